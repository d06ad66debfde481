// Multi-tensor fused SGD / Adam / RMSprop: one launch updates every parameter.
//
// Replaces Optimizer.step/_update and step_all (tensorlite/optim.py:39-136).
// Slot arithmetic is double and mirrors the reference expression order
// exactly (no FMA contraction: explicit __d*_rn), then theta is rounded to
// f32 once, like `param.write_flat` (optim.py:50, core.py:165-175).
//
// The tensor table travels as a __grid_constant__ kernel parameter (no H2D
// copy, no device table to keep alive); CTA b finds its tensor by a binary
// search over the per-tensor chunk prefix.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"

namespace {

constexpr int kMaxT = 48;
constexpr int kChunk = 8192;  // max elements per CTA (small steps use less: more CTAs)
constexpr int kThreads = 256;

struct Table {
  b2_opt_tensor t[kMaxT];
  int64_t prefix[kMaxT + 1];  // chunk prefix sums
  int64_t chunk;              // elements per CTA
  int count;
};

__device__ __forceinline__ int find_tensor(const Table& tb, int64_t chunk) {
  int lo = 0, hi = tb.count - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (tb.prefix[mid] <= chunk) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kThreads) k_sgd(const __grid_constant__ Table tb, double lr,
                                                  double mu, double wd) {
  int ti = find_tensor(tb, blockIdx.x);
  const b2_opt_tensor& T = tb.t[ti];
  int64_t base = (blockIdx.x - tb.prefix[ti]) * tb.chunk;
  int64_t end = min(T.n, base + tb.chunk);
  for (int64_t i = base + threadIdx.x; i < end; i += kThreads) {
    double th = (double)T.param[i];
    double g = (double)T.grad[i];
    if (wd != 0.0) g = __dadd_rn(g, __dmul_rn(wd, th));   // optim.py:47-49
    double v = __dadd_rn(__dmul_rn(mu, T.slot0[i]), g);   // optim.py:69
    T.slot0[i] = v;
    T.param[i] = __double2float_rn(__dsub_rn(th, __dmul_rn(lr, v)));  // :71
  }
}

__global__ void __launch_bounds__(kThreads) k_adam(const __grid_constant__ Table tb, double lr,
                                                   double b1, double b2, double omb1, double omb2,
                                                   double eps, double wd) {
  int ti = find_tensor(tb, blockIdx.x);
  const b2_opt_tensor& T = tb.t[ti];
  int64_t base = (blockIdx.x - tb.prefix[ti]) * tb.chunk;
  int64_t end = min(T.n, base + tb.chunk);
  double bc1 = T.bc1, bc2 = T.bc2;
  for (int64_t i = base + threadIdx.x; i < end; i += kThreads) {
    double th = (double)T.param[i];
    double g = (double)T.grad[i];
    if (wd != 0.0) g = __dadd_rn(g, __dmul_rn(wd, th));
    double m = __dadd_rn(__dmul_rn(b1, T.slot0[i]), __dmul_rn(omb1, g));               // :95
    double v = __dadd_rn(__dmul_rn(b2, T.slot1[i]), __dmul_rn(__dmul_rn(omb2, g), g)); // :96
    T.slot0[i] = m;
    T.slot1[i] = v;
    // theta - lr * (m / bc1) / (sqrt(v / bc2) + eps)                                    // :99
    double num = __dmul_rn(lr, __ddiv_rn(m, bc1));
    double den = __dadd_rn(__dsqrt_rn(__ddiv_rn(v, bc2)), eps);
    T.param[i] = __double2float_rn(__dsub_rn(th, __ddiv_rn(num, den)));
  }
}

__global__ void __launch_bounds__(kThreads) k_rmsprop(const __grid_constant__ Table tb, double lr,
                                                      double rho, double omrho, double eps,
                                                      double wd) {
  int ti = find_tensor(tb, blockIdx.x);
  const b2_opt_tensor& T = tb.t[ti];
  int64_t base = (blockIdx.x - tb.prefix[ti]) * tb.chunk;
  int64_t end = min(T.n, base + tb.chunk);
  for (int64_t i = base + threadIdx.x; i < end; i += kThreads) {
    double th = (double)T.param[i];
    double g = (double)T.grad[i];
    if (wd != 0.0) g = __dadd_rn(g, __dmul_rn(wd, th));
    // vi = rho * v + (1.0 - rho) * gi * gi (left to right)                     optim.py:118
    double v = __dadd_rn(__dmul_rn(rho, T.slot0[i]), __dmul_rn(__dmul_rn(omrho, g), g));
    T.slot0[i] = v;
    // theta - lr * gi / sqrt(vi + eps)                                           optim.py:120
    T.param[i] = __double2float_rn(
        __dsub_rn(th, __ddiv_rn(__dmul_rn(lr, g), __dsqrt_rn(__dadd_rn(v, eps)))));
  }
}

template <class Launch>
int run_multi(const b2_opt_tensor* ts, int count, Launch launch) {
  for (int off = 0; off < count; off += kMaxT) {
    Table tb;
    int k = 0;
    int64_t chunks = 0, total = 0;
    for (int i = off; i < count && i < off + kMaxT; ++i) total += ts[i].n > 0 ? ts[i].n : 0;
    // about 4 CTAs per SM for small steps (config 1: 203K params), 8K elements each for large
    int64_t chunk = total / (4 * (int64_t)b2::sm_count());
    chunk = std::max<int64_t>(1024, std::min<int64_t>(kChunk, (chunk + 255) / 256 * 256));
    tb.chunk = chunk;
    for (int i = off; i < count && k < kMaxT; ++i) {
      if (ts[i].n <= 0) continue;
      tb.t[k] = ts[i];
      tb.prefix[k] = chunks;
      chunks += (ts[i].n + chunk - 1) / chunk;
      ++k;
    }
    if (k == 0) continue;
    tb.prefix[k] = chunks;
    tb.count = k;
    B2_TRY(launch(tb, (unsigned)chunks));
  }
  return 0;
}

}  // namespace

extern "C" {

int b2_sgd_multi(const b2_opt_tensor* ts, int count, double lr, double mu, double wd,
                 void* stream) {
  cudaStream_t st = b2::resolve(stream);
  return run_multi(ts, count, [&](const Table& tb, unsigned grid) {
    k_sgd<<<grid, kThreads, 0, st>>>(tb, lr, mu, wd);
    return b2::launched("b2_sgd_multi");
  });
}

int b2_adam_multi(const b2_opt_tensor* ts, int count, double lr, double b1, double b2,
                  double eps, double wd, void* stream) {
  cudaStream_t st = b2::resolve(stream);
  double omb1 = 1.0 - b1, omb2 = 1.0 - b2;  // Python evaluates (1.0 - b1) in double
  return run_multi(ts, count, [&](const Table& tb, unsigned grid) {
    k_adam<<<grid, kThreads, 0, st>>>(tb, lr, b1, b2, omb1, omb2, eps, wd);
    return b2::launched("b2_adam_multi");
  });
}

int b2_rmsprop_multi(const b2_opt_tensor* ts, int count, double lr, double rho, double eps,
                     double wd, void* stream) {
  cudaStream_t st = b2::resolve(stream);
  double omrho = 1.0 - rho;
  return run_multi(ts, count, [&](const Table& tb, unsigned grid) {
    k_rmsprop<<<grid, kThreads, 0, st>>>(tb, lr, rho, omrho, eps, wd);
    return b2::launched("b2_rmsprop_multi");
  });
}

}  // extern "C"
