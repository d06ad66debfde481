// NCCL communicator for the data-parallel MLP step (new: the reference is a
// single process). One process per GPU; the unique id travels
// over the host-side bootstrap (torch.distributed's TCP store) and every rank
// calls ncclCommInitRank. NCCL is loaded with dlopen so that libb2 itself
// loads on hosts without it (the CPU test suite checks the exports).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>

#include "common.cuh"

namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
};

Nccl g_nccl;
ncclComm_t g_comm = nullptr;

int load_nccl() {
  if (g_nccl.h) return 0;
  const char* cands[3] = {getenv("B2_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
  for (const char* c : cands) {
    if (!c || !*c) continue;
    g_nccl.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.h) break;
  }
  if (!g_nccl.h) return b2::fail("libnccl.so.2 not found (set B2_NCCL_LIB)");
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(g_nccl.h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(g_nccl.h, "ncclCommInitRank");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(g_nccl.h, "ncclCommDestroy");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(g_nccl.h, "ncclAllReduce");
  g_nccl.ReduceScatter = (decltype(g_nccl.ReduceScatter))dlsym(g_nccl.h, "ncclReduceScatter");
  g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(g_nccl.h, "ncclAllGather");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(g_nccl.h, "ncclGetErrorString");
  g_nccl.CommGetAsyncError =
      (decltype(g_nccl.CommGetAsyncError))dlsym(g_nccl.h, "ncclCommGetAsyncError");
  g_nccl.CommAbort = (decltype(g_nccl.CommAbort))dlsym(g_nccl.h, "ncclCommAbort");
  if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.AllReduce)
    return b2::fail("libnccl is missing required symbols");
  return 0;
}

int nccl_fail(ncclResult_t r, const char* what) {
  std::string m = std::string(what) + ": NCCL error " + std::to_string((int)r);
  if (g_nccl.GetErrorString) m += std::string(" (") + g_nccl.GetErrorString(r) + ")";
  return b2::fail(m);
}

}  // namespace

extern "C" {

int b2_comm_unique_id(unsigned char* out128) {
  B2_TRY(load_nccl());
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out128, &id, 128);
  return 0;
}

int b2_comm_init(int rank, int nranks, const unsigned char* uid128) {
  B2_TRY(b2::ensure_init());
  B2_TRY(load_nccl());
  if (g_comm) return 0;
  ncclUniqueId id;
  memcpy(&id, uid128, 128);
  ncclResult_t r = g_nccl.CommInitRank(&g_comm, nranks, id, rank);
  if (r != ncclSuccess) {
    g_comm = nullptr;
    return nccl_fail(r, "ncclCommInitRank");
  }
  return 0;
}

int b2_comm_destroy(void) {
  if (g_comm && g_nccl.CommDestroy) g_nccl.CommDestroy(g_comm);
  g_comm = nullptr;
  return 0;
}

int b2_allreduce_f32(float* buf, int64_t n, int op, void* stream) {
  if (!g_comm) return b2::fail("b2_allreduce_f32: communicator not initialised");
  ncclRedOp_t rop = op == 1 ? ncclAvg : (op == 2 ? ncclMax : ncclSum);
  ncclResult_t r = g_nccl.AllReduce(buf, buf, (size_t)n, ncclFloat32, rop, g_comm, b2::resolve(stream));
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  return 0;
}

// Sharded optimizer step (ZeRO-1 style): the gradient is reduce-scattered so
// every rank holds the average of its contiguous 1/N shard (out = recv, count
// elements per rank), updates only that shard of the parameter, and the
// updated shards are all-gathered back into the full parameter in place
// (sendbuff = buf + rank * count, NCCL's in-place form). Same bytes on the
// wire as one all-reduce; 1/N of the optimizer's HBM traffic and slot memory.
int b2_reduce_scatter_f32(const float* send, float* recv, int64_t count, int op, void* stream) {
  if (!g_comm) return b2::fail("b2_reduce_scatter_f32: communicator not initialised");
  if (!g_nccl.ReduceScatter) return b2::fail("b2_reduce_scatter_f32: libnccl lacks ncclReduceScatter");
  ncclRedOp_t rop = op == 1 ? ncclAvg : (op == 2 ? ncclMax : ncclSum);
  ncclResult_t r = g_nccl.ReduceScatter(send, recv, (size_t)count, ncclFloat32, rop, g_comm, b2::resolve(stream));
  if (r != ncclSuccess) return nccl_fail(r, "ncclReduceScatter");
  return 0;
}

int b2_all_gather_f32(float* buf, int64_t count, int rank, void* stream) {
  if (!g_comm) return b2::fail("b2_all_gather_f32: communicator not initialised");
  if (!g_nccl.AllGather) return b2::fail("b2_all_gather_f32: libnccl lacks ncclAllGather");
  ncclResult_t r = g_nccl.AllGather(buf + (int64_t)rank * count, buf, (size_t)count, ncclFloat32, g_comm,
                                    b2::resolve(stream));
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
  return 0;
}

// Failure detection: the communicator's asynchronous error state
// (0 = ok; a peer that died or a network fault shows up here, not as a hang)
int b2_comm_async_error(int* err) {
  *err = 0;
  if (!g_comm || !g_nccl.CommGetAsyncError) return 0;
  ncclResult_t r = ncclSuccess;
  ncclResult_t q = g_nccl.CommGetAsyncError(g_comm, &r);
  if (q != ncclSuccess) return nccl_fail(q, "ncclCommGetAsyncError");
  *err = (int)r;
  return 0;
}

int b2_comm_abort(void) {
  if (g_comm && g_nccl.CommAbort) g_nccl.CommAbort(g_comm);
  g_comm = nullptr;
  return 0;
}

// Host wait for `stream` with a deadline, polling the communicator's async
// error: returns 0 when the stream drained, fails (and aborts the
// communicator so no rank blocks forever) on an NCCL error or a timeout.
int b2_stream_wait_timeout(void* stream, double timeout_ms) {
  cudaStream_t st = b2::resolve(stream);
  cudaEvent_t ev;
  B2_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  cudaError_t e = cudaEventRecord(ev, st);
  if (e != cudaSuccess) {
    cudaEventDestroy(ev);
    return b2::cuda_fail(e, "cudaEventRecord");
  }
  const auto t0 = std::chrono::steady_clock::now();
  int rc = 0;
  for (;;) {
    e = cudaEventQuery(ev);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) {
      rc = b2::cuda_fail(e, "b2_stream_wait_timeout");
      break;
    }
    int err = 0;
    if (b2_comm_async_error(&err) == 0 && err != 0 && err != (int)ncclInProgress) {
      b2_comm_abort();
      rc = b2::fail("NCCL asynchronous error " + std::to_string(err) + "; communicator aborted");
      break;
    }
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms > timeout_ms) {
      b2_comm_abort();
      rc = b2::fail("stream did not drain within " + std::to_string(timeout_ms) +
                    " ms; communicator aborted");
      break;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  cudaEventDestroy(ev);
  return rc;
}

}  // extern "C"
