// NCCL communicator for the data-parallel MLP step (new: the reference is a
// single process). One process per GPU; the unique id travels
// over the host-side bootstrap (torch.distributed's TCP store) and every rank
// calls ncclCommInitRank. NCCL is loaded with dlopen so that libb2 itself
// loads on hosts without it (the CPU test suite checks the exports).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"

namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
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
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(g_nccl.h, "ncclGetErrorString");
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

}  // extern "C"
