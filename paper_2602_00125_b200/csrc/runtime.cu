// Runtime plumbing + the caching device allocator.
//
// Replaces the reference's per-op `Buffer(array('f'))` storage
// (tensorlite/core.py:68-75, 315-330): device blocks come from size-class
// free lists and are returned on free in STREAM ORDER -- a block freed on its
// owning stream is reusable immediately by later work on that stream (the
// stream serialises the old and new users); a block freed from another
// stream is parked behind a CUDA event until that stream passes the free.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace b2 {

static thread_local std::string t_err;
std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { t_err = msg; }
int fail(const std::string& msg) {
  set_error(msg);
  return 1;
}
int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
  return 2;
}

static std::mutex g_init_mu;
static int g_device = -1;
static int g_sms = 0;
static cudaStream_t g_stream = nullptr;
static std::thread::id g_main_thread;

// One engine stream per host thread (the reference keeps one tape per thread,
// autograd.py:48-56; here each thread's ops also queue on their own CUDA
// stream, so two threads' work is independent and each thread's launches stay
// in program order). The thread that calls b2_init owns g_stream; any other
// thread gets a stream on its first call (and the device selected, since
// cudaSetDevice is per thread). A finished thread's stream goes back to a
// pool for the next new thread: blocks cached on it stay valid (same stream).
static std::mutex g_pool_mu;
static std::vector<cudaStream_t> g_stream_pool;

struct ThreadStream {
  cudaStream_t st = nullptr;
  bool owned = false;  // taken from the pool / created for this thread
  ~ThreadStream() {
    if (owned && st) {
      std::lock_guard<std::mutex> lk(g_pool_mu);
      g_stream_pool.push_back(st);
    }
  }
};
static thread_local ThreadStream t_stream;

static cudaStream_t thread_stream() {
  if (t_stream.st) return t_stream.st;
  if (!g_stream && b2_init(-1) != 0) return nullptr;
  if (std::this_thread::get_id() == g_main_thread) {
    t_stream.st = g_stream;
    return g_stream;
  }
  cudaSetDevice(g_device);
  cudaStream_t st = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (!g_stream_pool.empty()) {
      st = g_stream_pool.back();
      g_stream_pool.pop_back();
    }
  }
  if (!st && cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    return g_stream;
  }
  tickets(st);
  t_stream.st = st;
  t_stream.owned = true;
  return st;
}

int ensure_init() {
  if (!g_stream) B2_TRY(b2_init(-1));
  if (!t_stream.st) thread_stream();  // selects the device on a new thread
  return 0;
}

cudaStream_t resolve(void* stream) {
  if (stream) {
    if (!t_stream.st) thread_stream();  // this thread's device is selected
    return (cudaStream_t)stream;
  }
  return thread_stream();
}

// Per-stream arrival counters for single-launch two-stage reductions (the
// last CTA of a group folds the group's partials). Kernels on one stream run
// in order and every kernel leaves its counters at zero, so each stream owns
// one zeroed block, created on first use.
unsigned* tickets(cudaStream_t st) {
  static std::mutex mu;
  static std::map<cudaStream_t, unsigned*> blocks;
  std::lock_guard<std::mutex> lk(mu);
  auto it = blocks.find(st);
  if (it != blocks.end()) return it->second;
  unsigned* p = nullptr;
  if (cudaMalloc(&p, kTicketsAlloc * sizeof(unsigned)) != cudaSuccess) return nullptr;
  if (cudaMemset(p, 0, kTicketsAlloc * sizeof(unsigned)) != cudaSuccess) return nullptr;
  blocks[st] = p;
  return p;
}

int sm_count() {
  if (!g_sms) ensure_init();
  return g_sms ? g_sms : 148;
}

static std::atomic<int> g_gemm_reserve{0};

int gemm_sms() {
  const int n = sm_count();
  const int r = g_gemm_reserve.load(std::memory_order_relaxed);
  return n - r >= 2 ? n - r : 2;
}

// ------------------------------------------------------------ allocator

struct Block {
  void* ptr;
  size_t size;
  cudaStream_t stream;  // owning stream
  int graph = 0;        // CUDA graph that references this block (0: none)
};

// CUDA-graph capture support: while the engine stream is being captured,
// freed blocks stay private to the capture (reusable by later allocations of
// the same capture -- the captured stream order keeps that safe) and, once
// the graph exists, every block it touched is parked until b2_graph_destroy,
// so replays never race with other users of the memory.
struct GraphState {
  cudaGraphExec_t exec = nullptr;
  std::vector<Block*> parked;
};
static int g_capture = 0;  // id of the graph being captured (0: none)
static int g_next_graph = 1;
static std::multimap<size_t, Block*> g_cap_free;
static std::map<int, GraphState> g_graphs;

struct Pending {
  Block* blk;
  cudaEvent_t ev;
};

static std::mutex g_mu;
static std::unordered_map<void*, Block*> g_live;
// free lists keyed by (stream) -> size -> blocks
static std::map<cudaStream_t, std::multimap<size_t, Block*>> g_free;
static std::vector<Pending> g_pending;
static size_t g_in_use = 0, g_cached = 0, g_peak = 0;
static uint64_t g_nmalloc = 0;

static size_t round_size(size_t n) {
  if (n == 0) n = 1;
  if (n < (1u << 20)) return (n + 511) & ~size_t(511);        // 512 B classes
  return (n + (2u << 20) - 1) & ~size_t((2u << 20) - 1);       // 2 MiB classes
}

static void drain_pending_locked() {
  size_t w = 0;
  for (size_t i = 0; i < g_pending.size(); ++i) {
    Pending p = g_pending[i];
    if (cudaEventQuery(p.ev) == cudaSuccess) {
      cudaEventDestroy(p.ev);
      g_free[p.blk->stream].emplace(p.blk->size, p.blk);
    } else {
      g_pending[w++] = p;
    }
  }
  g_pending.resize(w);
  cudaGetLastError();  // clear cudaErrorNotReady
}

static int release_cached_locked() {
  drain_pending_locked();
  for (auto& kv : g_free) {
    for (auto& sb : kv.second) {
      cudaFree(sb.second->ptr);
      g_cached -= sb.second->size;
      delete sb.second;
    }
    kv.second.clear();
  }
  return 0;
}

}  // namespace b2

using namespace b2;

extern "C" {

const char* b2_last_error(void) { return t_err.c_str(); }

int b2_version(int* major, int* minor) {
  if (major) *major = 0;
  if (minor) *minor = 1;
  return 0;
}

int b2_init(int device) {
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (g_stream && (device < 0 || device == g_device)) return 0;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail("b2_init: no CUDA device visible (libb2 has no CPU fallback)");
  if (device < 0) {
    B2_CUDA(cudaGetDevice(&device));
  }
  B2_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  B2_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return fail("b2_init: libb2 is built for sm_100a (B200); found sm_" +
                std::to_string(prop.major) + std::to_string(prop.minor));
  g_sms = prop.multiProcessorCount;
  B2_CUDA(cudaStreamCreateWithFlags(&g_stream, cudaStreamNonBlocking));
  g_device = device;
  g_main_thread = std::this_thread::get_id();
  if (!tickets(g_stream)) return fail("b2_init: could not allocate reduction counters");
  return 0;
}

// Persistent GEMM grids leave `n` SMs free (0..sm_count-2): under data
// parallelism NCCL's collective kernels then run beside the backward GEMMs
// instead of waiting for a GEMM boundary (dist.Communicator sets it).
int b2_gemm_set_sm_reserve(int n) {
  B2_TRY(b2::ensure_init());
  if (n < 0 || n > b2::sm_count() - 2) return b2::fail("b2_gemm_set_sm_reserve: 0 <= n <= SMs - 2");
  b2::g_gemm_reserve.store(n, std::memory_order_relaxed);
  return 0;
}

int b2_gemm_get_sm_reserve(int* n) {
  *n = b2::g_gemm_reserve.load(std::memory_order_relaxed);
  return 0;
}

int b2_device_count(int* n) {
  cudaError_t e = cudaGetDeviceCount(n);
  if (e != cudaSuccess) {
    *n = 0;
    cudaGetLastError();
  }
  return 0;
}

int b2_device_info(int* sm, int* maj, int* min, size_t* total) {
  B2_TRY(ensure_init());
  cudaDeviceProp prop;
  B2_CUDA(cudaGetDeviceProperties(&prop, g_device));
  if (sm) *sm = prop.multiProcessorCount;
  if (maj) *maj = prop.major;
  if (min) *min = prop.minor;
  if (total) *total = prop.totalGlobalMem;
  return 0;
}

int b2_default_stream(void** s) {
  B2_TRY(ensure_init());
  *s = (void*)resolve(nullptr);  // the calling thread's engine stream
  return 0;
}
int b2_stream_create(void** s) {
  B2_TRY(ensure_init());
  cudaStream_t st;
  B2_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  *s = (void*)st;
  return 0;
}
// A non-blocking stream at the device's greatest priority: the block
// scheduler hands freed SMs to its kernels first (the data-parallel
// collectives and optimizer updates that overlap the backward GEMMs).
int b2_stream_create_priority(void** s) {
  B2_TRY(ensure_init());
  int least = 0, greatest = 0;
  B2_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  cudaStream_t st;
  B2_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, greatest));
  *s = (void*)st;
  return 0;
}
int b2_stream_destroy(void* s) {
  B2_CUDA(cudaStreamDestroy((cudaStream_t)s));
  return 0;
}
int b2_stream_sync(void* s) {
  B2_CUDA(cudaStreamSynchronize(resolve(s)));
  return 0;
}
int b2_device_sync(void) {
  B2_CUDA(cudaDeviceSynchronize());
  return 0;
}
int b2_event_create(void** ev) {
  B2_TRY(ensure_init());
  cudaEvent_t e;
  B2_CUDA(cudaEventCreate(&e));
  *ev = (void*)e;
  return 0;
}
int b2_event_destroy(void* ev) {
  B2_CUDA(cudaEventDestroy((cudaEvent_t)ev));
  return 0;
}
int b2_event_record(void* ev, void* s) {
  B2_CUDA(cudaEventRecord((cudaEvent_t)ev, resolve(s)));
  return 0;
}
int b2_event_elapsed_ms(void* a, void* b, float* ms) {
  B2_CUDA(cudaEventSynchronize((cudaEvent_t)b));
  B2_CUDA(cudaEventElapsedTime(ms, (cudaEvent_t)a, (cudaEvent_t)b));
  return 0;
}
int b2_stream_wait_event(void* s, void* ev) {
  B2_CUDA(cudaStreamWaitEvent(resolve(s), (cudaEvent_t)ev, 0));
  return 0;
}
int b2_launch_count(uint64_t* n) {
  *n = g_launches.load();
  return 0;
}

// ------------------------------------------------------------ allocator API

int b2_alloc(size_t bytes, void* stream, void** out) {
  B2_TRY(ensure_init());
  cudaStream_t st = resolve(stream);
  size_t sz = round_size(bytes);
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_pending.empty()) drain_pending_locked();
  if (g_capture) {  // reuse a block this capture already freed
    auto ci = g_cap_free.lower_bound(sz);
    if (ci != g_cap_free.end() && ci->first - sz <= (sz < (1u << 20) ? sz : sz / 8 + (2u << 20))) {
      Block* b = ci->second;
      g_cap_free.erase(ci);
      g_live[b->ptr] = b;
      g_in_use += b->size;
      if (g_in_use > g_peak) g_peak = g_in_use;
      *out = b->ptr;
      return 0;
    }
  }
  auto& fl = g_free[st];
  // best fit; small blocks may be up to 2x the request, large ones at most
  // 1/8 (>= 2 MiB) bigger, so steady-state reuse never balloons the footprint
  auto it = fl.lower_bound(sz);
  const size_t slack = sz < (1u << 20) ? sz : (sz / 8 > (2u << 20) ? sz / 8 : (2u << 20));
  if (it != fl.end() && it->first - sz <= slack) {
    Block* b = it->second;
    fl.erase(it);
    if (g_capture) b->graph = g_capture;
    g_live[b->ptr] = b;
    g_in_use += b->size;
    if (g_in_use > g_peak) g_peak = g_in_use;
    *out = b->ptr;
    return 0;
  }
  // a fitting block still waiting for another stream (the host ran ahead of
  // the device): wait for that stream instead of growing the pool -- bounded
  // memory and no cudaMalloc stall in steady state
  for (size_t i = 0; !g_capture && i < g_pending.size(); ++i) {
    Block* b = g_pending[i].blk;
    if (b->stream != st || b->size < sz || b->size - sz > slack) continue;
    cudaEventSynchronize(g_pending[i].ev);
    cudaEventDestroy(g_pending[i].ev);
    g_pending.erase(g_pending.begin() + (std::ptrdiff_t)i);
    g_live[b->ptr] = b;
    g_in_use += b->size;
    if (g_in_use > g_peak) g_peak = g_in_use;
    *out = b->ptr;
    return 0;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, sz);
  if (e != cudaSuccess) {
    cudaGetLastError();
    release_cached_locked();
    e = cudaMalloc(&p, sz);
    if (e != cudaSuccess) {
      char buf[160];
      snprintf(buf, sizeof buf, "b2_alloc: out of device memory allocating %zu bytes (in use %zu)",
               sz, g_in_use);
      cudaGetLastError();
      return fail(buf);
    }
  }
  ++g_nmalloc;
  Block* b = new Block{p, sz, st, g_capture};
  g_live[p] = b;
  g_in_use += sz;
  g_cached += sz;
  if (g_in_use > g_peak) g_peak = g_in_use;
  *out = p;
  return 0;
}

int b2_free(void* ptr, void* stream) {
  if (!ptr) return 0;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_live.find(ptr);
  if (it == g_live.end()) return fail("b2_free: pointer not owned by the allocator");
  Block* b = it->second;
  g_live.erase(it);
  g_in_use -= b->size;
  if (g_capture) {  // freed inside a capture: the graph may still touch it on replay
    b->graph = g_capture;
    g_cap_free.emplace(b->size, b);
    return 0;
  }
  if (b->graph) {  // owned by a live graph: park until the graph is destroyed
    auto gi = g_graphs.find(b->graph);
    if (gi != g_graphs.end()) {
      gi->second.parked.push_back(b);
      return 0;
    }
    b->graph = 0;
  }
  // last use: the given stream, else the calling thread's engine stream (a
  // block freed from another thread -- e.g. by the garbage collector -- waits
  // for that thread's queued work before its owner stream may reuse it)
  cudaStream_t fs = stream ? (cudaStream_t)stream : resolve(nullptr);
  if (fs == b->stream) {
    g_free[b->stream].emplace(b->size, b);
  } else {
    // last use was on another stream: reusable once that stream passes here
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ev, fs) != cudaSuccess) {
      cudaStreamSynchronize(fs);
      g_free[b->stream].emplace(b->size, b);
      cudaGetLastError();
    } else {
      g_pending.push_back({b, ev});
    }
  }
  return 0;
}

// ------------------------------------------------------------ CUDA graphs

int b2_graph_begin(void* stream) {
  B2_TRY(ensure_init());
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_capture) return fail("b2_graph_begin: a capture is already in progress");
    g_capture = g_next_graph++;
  }
  cudaError_t e = cudaStreamBeginCapture(resolve(stream), cudaStreamCaptureModeRelaxed);
  if (e != cudaSuccess) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_capture = 0;
    return cuda_fail(e, "cudaStreamBeginCapture");
  }
  return 0;
}

static void end_capture_locked(int id, cudaGraphExec_t exec) {
  GraphState& gs = g_graphs[id];
  gs.exec = exec;
  for (auto& kv : g_cap_free) gs.parked.push_back(kv.second);
  g_cap_free.clear();
  g_capture = 0;
}

int b2_graph_end(void* stream, int* graph_id) {
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(resolve(stream), &graph);
  std::lock_guard<std::mutex> lk(g_mu);
  int id = g_capture;
  if (e != cudaSuccess || !graph) {
    end_capture_locked(id, nullptr);  // keep the capture's blocks parked under a dead id
    return cuda_fail(e != cudaSuccess ? e : cudaErrorStreamCaptureInvalidated, "cudaStreamEndCapture");
  }
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  end_capture_locked(id, e == cudaSuccess ? exec : nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
  *graph_id = id;
  return 0;
}

int b2_graph_launch(int graph_id, void* stream) {
  cudaGraphExec_t exec = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_graphs.find(graph_id);
    if (it == g_graphs.end() || !it->second.exec) return fail("b2_graph_launch: unknown graph");
    exec = it->second.exec;
  }
  B2_CUDA(cudaGraphLaunch(exec, resolve(stream)));
  count_launch();
  return 0;
}

int b2_graph_destroy(int graph_id) {
  B2_CUDA(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_graphs.find(graph_id);
  if (it == g_graphs.end()) return 0;
  if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
  for (Block* b : it->second.parked) {
    b->graph = 0;
    g_free[b->stream].emplace(b->size, b);
  }
  for (auto& kv : g_live)
    if (kv.second->graph == graph_id) kv.second->graph = 0;
  g_graphs.erase(it);
  return 0;
}

int b2_alloc_stats(size_t* in_use, size_t* cached, size_t* peak, uint64_t* nm) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (in_use) *in_use = g_in_use;
  if (cached) *cached = g_cached;
  if (peak) *peak = g_peak;
  if (nm) *nm = g_nmalloc;
  return 0;
}

int b2_empty_cache(void) {
  B2_CUDA(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> lk(g_mu);
  return release_cached_locked();
}

int b2_host_alloc(size_t bytes, void** out) {
  B2_TRY(ensure_init());
  B2_CUDA(cudaMallocHost(out, bytes ? bytes : 1));
  return 0;
}
int b2_host_free(void* p) {
  B2_CUDA(cudaFreeHost(p));
  return 0;
}

int b2_memcpy_h2d(void* dst, const void* src, size_t bytes, void* s) {
  if (!bytes) return 0;
  B2_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, resolve(s)));
  return 0;
}
// synchronous w.r.t. the host: the data is valid when this returns
int b2_memcpy_d2h(void* dst, const void* src, size_t bytes, void* s) {
  if (!bytes) return 0;
  cudaStream_t st = resolve(s);
  B2_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
  B2_CUDA(cudaStreamSynchronize(st));
  return 0;
}
// stream-ordered D2H into pinned host memory; completion via an event
// (b2_event_sync) -- lets a training loop read step i's loss after step i+1
// is queued instead of draining the stream every step
int b2_memcpy_d2h_async(void* dst, const void* src, size_t bytes, void* s) {
  if (!bytes) return 0;
  B2_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, resolve(s)));
  return 0;
}
int b2_event_sync(void* ev) {
  B2_CUDA(cudaEventSynchronize((cudaEvent_t)ev));
  return 0;
}
int b2_memcpy_d2d(void* dst, const void* src, size_t bytes, void* s) {
  if (!bytes) return 0;
  B2_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, resolve(s)));
  return 0;
}

}  // extern "C"
