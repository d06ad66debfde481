// Row-wise losses: fused cross-entropy (fwd + pullback) and row softmax.
//
// cross_entropy mirrors tensorlite/nn.py:453-503 in double precision:
//   m = row max, se = sum exp(v - m), row loss = m + log(se) - z[y],
//   loss = f32((sum of row losses) / b);   pullback:
//   dz = f32((exp(v - m) / se - onehot) * (g / b)).
// The reference takes se from math.fsum in the pullback; here se is a
// compensated (Neumaier) sum in the forward, kept per row in `row_stats`, so
// the pullback does not redo the reductions.
//
// softmax mirrors the reference COMPOSITION (max detached, then
// sub/exp/sum/div as separate engine ops, each rounded to f32) and its
// GradStore-ordered pullback, so results are bit-identical to composing the
// ops on the reference engine.
#include <cuda_runtime.h>
#include <algorithm>
#include <math.h>

#include "common.cuh"
#include <cuda_bf16.h>

#include "fexp.cuh"

#ifndef B2_SOFTMAX_TMA
#define B2_SOFTMAX_TMA 1
#endif
constexpr bool kSoftmaxTma = B2_SOFTMAX_TMA;
// softmax rows: 3 resident 256-thread CTAs per SM (<= 85 registers). At the
// unconstrained 122 registers only 2 fit and the row loop's load -> max -> exp
// -> sum -> store chain leaves the SM idle (config-4 step 1.13 -> 0.94 ms).
#ifndef B2_SMX_MINB
#define B2_SMX_MINB 3
#endif

extern "C" int b2_alloc(size_t, void*, void**);
extern "C" int b2_free(void*, void*);

namespace {

__device__ __forceinline__ float warp_max_first(float m) {
  // row max VALUE (ties are irrelevant for the value); NaN handled by caller
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    float o = __shfl_xor_sync(0xffffffffu, m, off);
    m = o > m ? o : m;
  }
  return m;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// two-sum combine of Neumaier accumulators (s, c)
__device__ __forceinline__ void neu_add(double& s, double& c, double x) {
  double t = s + x;
  if (fabs(s) >= fabs(x))
    c += (s - t) + x;
  else
    c += (x - t) + s;
  s = t;
}

// Reference row max semantics for the value: strict '>' scan from v[0]
// (nn.py:478-481) -- a NaN at v[0] sticks, later NaNs are skipped.
__device__ __forceinline__ float row_max(const float* row, int64_t C, int lane) {
  float m = -INFINITY;
  bool any = false;
  for (int64_t j = lane; j < C; j += 32) {
    float v = row[j];
    if (!isnan(v)) {
      m = any ? (v > m ? v : m) : v;
      any = true;
    }
  }
  m = warp_max_first(any ? m : -INFINITY);
  float v0 = row[0];
  return isnan(v0) ? v0 : m;
}

// ---------------------------------------------------------------- cross-entropy
// one warp per row; grid-stride over rows
__global__ void __launch_bounds__(256) k_xent_rows(double* __restrict__ row_loss,
                                                   double* __restrict__ row_stats,
                                                   const float* __restrict__ z,
                                                   const int64_t* __restrict__ labels,
                                                   int64_t B, int64_t C) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < B; r += nw) {
    const float* row = z + r * C;
    double m = (double)row_max(row, C, lane);
    double s = 0, c = 0;
    for (int64_t j = lane; j < C; j += 32) neu_add(s, c, b2::exp_fast((double)row[j] - m));
    // per-lane compensated partials, then a fixed butterfly over 32 lanes
    double tot = warp_sum(s + c);
    if (lane == 0) {
      double se = tot;
      row_stats[2 * r] = m;
      row_stats[2 * r + 1] = se;
      const int64_t lab = labels[r];  // out of range (an unchecked Buffer): NaN loss, no stray read
      row_loss[r] = m + log(se) - (lab >= 0 && lab < C ? (double)row[lab] : (double)NAN);
    }
  }
}

// fixed-order sum of row losses by one CTA, loss = f32(total / denom)
__global__ void __launch_bounds__(1024) k_xent_final(float* __restrict__ loss,
                                                     const double* __restrict__ row_loss,
                                                     int64_t B, double denom) {
  __shared__ double sh[32];
  double acc = 0;
  for (int64_t r = threadIdx.x; r < B; r += blockDim.x) acc += row_loss[r];
  acc = warp_sum(acc);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = acc;
  __syncthreads();
  if (w == 0) {
    double t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) *loss = __double2float_rn(t / denom);
  }
}

__global__ void __launch_bounds__(256) k_xent_bwd(float* __restrict__ dz, const float* __restrict__ g,
                                                  const double* __restrict__ row_stats,
                                                  const float* __restrict__ z,
                                                  const int64_t* __restrict__ labels, int64_t B,
                                                  int64_t C, double denom) {
  double gv = (double)g[0] / denom;  // nn.py:489
  int64_t total = B * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / C;
    int64_t j = i - r * C;
    double m = row_stats[2 * r], se = row_stats[2 * r + 1];
    double p = b2::exp_fast((double)z[i] - m) / se - (j == labels[r] ? 1.0 : 0.0);
    dz[i] = __double2float_rn(p * gv);  // nn.py:500
  }
}

// ---------------------------------------------------------------- softmax (composed)
__global__ void __launch_bounds__(256) k_softmax_fwd(float* __restrict__ y, float* __restrict__ rs,
                                                     float* __restrict__ rm,
                                                     const float* __restrict__ z, int64_t B,
                                                     int64_t C) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < B; r += nw) {
    const float* row = z + r * C;
    float m = row_max(row, C, lane);
    double acc = 0;
    for (int64_t j = lane; j < C; j += 32) {
      float e = b2::exp_f32(__fsub_rn(row[j], m));  // exp(sub(z, m))
      acc += (double)e;
    }
    acc = warp_sum(acc);
    float s = __double2float_rn(acc);  // sum(e, -1, keepdims)
    float* yr = y + r * C;
    for (int64_t j = lane; j < C; j += 32) {
      float e = b2::exp_f32(__fsub_rn(row[j], m));
      yr[j] = __fdiv_rn(e, s);  // div(e, s)
    }
    if (lane == 0) {
      rs[r] = s;
      rm[r] = m;
    }
  }
}

__global__ void __launch_bounds__(256) k_softmax_bwd(float* __restrict__ gz,
                                                     const float* __restrict__ gy,
                                                     const float* __restrict__ z,
                                                     const float* __restrict__ rs,
                                                     const float* __restrict__ rm, int64_t B,
                                                     int64_t C) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < B; r += nw) {
    const float* row = z + r * C;
    const float* grow = gy + r * C;
    float s = rs[r], m = rm[r];
    float ss = __fmul_rn(s, s);
    double acc = 0;
    for (int64_t j = lane; j < C; j += 32) {
      float e = b2::exp_f32(__fsub_rn(row[j], m));
      float t = __fdiv_rn(__fmul_rn(grow[j], e), ss);  // div(mul(g, e), mul(s, s))
      acc += (double)(-t);                              // neg, then sum(axis=-1)
    }
    acc = warp_sum(acc);
    float gs = __double2float_rn(acc);
    float* out = gz + r * C;
    for (int64_t j = lane; j < C; j += 32) {
      float e = b2::exp_f32(__fsub_rn(row[j], m));
      float ge = __fdiv_rn(grow[j], s);            // div(g, s) -- stored first
      float tot = __fadd_rn(ge, gs);               // GradStore add(cur, g)
      out[j] = __fmul_rn(tot, e);                  // exp pullback mul(g, out)
    }
  }
}

// Register-resident variants for rows of up to 128*NV floats (C % 4 == 0,
// 16-B aligned rows): a warp loads its row once with NV 128-bit loads in
// flight per lane, computes each exp ONCE, and writes with 128-bit stores.
// Same arithmetic and rounding sequence as the looped kernels above.
__device__ __forceinline__ float f4get(const float4& q, int k) {
  return k == 0 ? q.x : k == 1 ? q.y : k == 2 ? q.z : q.w;
}
__device__ __forceinline__ void f4set(float4& q, int k, float v) {
  if (k == 0) q.x = v; else if (k == 1) q.y = v; else if (k == 2) q.z = v; else q.w = v;
}

// a / b rounded to nearest, for many a with one row-constant b: rb = RN(1/b)
// once per row, then Markstein's correction q' = RN(q + RN(a - b q) rb) with
// q = RN(a rb) -- exactly RN(a/b) whenever no intermediate under/overflows
// (Markstein 1990; Muller et al., Handbook of FP Arithmetic, Thm 4.10), which
// `ok` (b finite, >= 1) and the |a| window guarantee; anything else takes the
// IEEE division. Three FMA-pipe ops instead of __fdiv_rn's MUFU + fixups.
__device__ __forceinline__ float div_by(float a, float b, float rb, bool ok) {
  const float q = __fmul_rn(a, rb);
  const float r = __fmaf_rn(-q, b, a);
  const float q1 = __fmaf_rn(r, rb, q);
  const float aa = fabsf(a);
  return (ok && aa >= 0x1p-100f && aa <= 0x1p100f) ? q1 : __fdiv_rn(a, b);
}

// Row max VALUE over the registers (padding past C excluded): fmaxf skips
// NaNs like the strict '>' scan; the first-slot NaN rule is applied after the
// butterfly. The sign of a zero maximum may differ from the scan's first
// zero, which no consumer can observe: z - m and m + log(se) are the same
// for m = +0 and m = -0.
// The pieces of div_by for rows where the window check is hoisted: a row
// whose every dividend passes `in_window` (and whose divisor is `ok`) takes
// div_fast for all of its elements -- no IEEE division code on the path,
// which the per-element select of div_by made the compiler evaluate anyway.
__device__ __forceinline__ bool in_window(float a) {
  const float aa = fabsf(a);
  return aa == 0.0f || (aa >= 0x1p-100f && aa <= 0x1p100f);  // NaN: false
}
__device__ __forceinline__ float div_fast(float a, float b, float rb) {
  const float q = __fmul_rn(a, rb);
  const float r = __fmaf_rn(-q, b, a);
  return __fmaf_rn(r, rb, q);
}

template <int NV, bool FULL = false>
__device__ __forceinline__ float row_max_regs(const float4 (&v)[NV], int64_t C, int lane) {
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool in = FULL || (int64_t)(i * 32 + lane) * 4 + k < C;
      m = fmaxf(m, in ? f4get(v[i], k) : -INFINITY);
    }
  m = warp_max_first(m);
  const float v0 = __shfl_sync(0xffffffffu, v[0].x, 0);  // the first scanned slot
  return isnan(v0) ? v0 : m;
}

template <int NV>
__global__ void __launch_bounds__(256, B2_SMX_MINB) k_softmax_fwd_v(float* __restrict__ y, float* __restrict__ rs,
                                                       float* __restrict__ rm,
                                                       const float* __restrict__ z, int64_t B,
                                                       int64_t C) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < B; r += nw) {
    const float4* row = reinterpret_cast<const float4*>(z + r * C);
    float4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      v[i] = q * 4 < C ? __ldg(row + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float m = row_max_regs<NV>(v, C, lane);
    double acc = 0;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float e = b2::exp_f32(__fsub_rn(f4get(v[i], k), m));  // exp(sub(z, m))
        f4set(v[i], k, e);
        if ((int64_t)(i * 32 + lane) * 4 + k < C) acc += (double)e;
      }
    const float s = __double2float_rn(warp_sum(acc));  // sum(e, -1, keepdims)
    const bool ok = s >= 1.0f && s <= 0x1p100f;        // s >= 1 unless the row is NaN/-inf
    const float rs_ = __frcp_rn(s);
    float4* yr = reinterpret_cast<float4*>(y + r * C);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      if (q * 4 < C)
        yr[q] = make_float4(div_by(v[i].x, s, rs_, ok), div_by(v[i].y, s, rs_, ok),
                            div_by(v[i].z, s, rs_, ok), div_by(v[i].w, s, rs_, ok));  // div(e, s)
    }
    if (lane == 0) {
      rs[r] = s;
      rm[r] = m;
    }
  }
}

// TMA-staged rows (C % 4 == 0, 16-B aligned, 4*C bytes <= 16 KB): each warp
// owns two shared-memory row buffers; lane 0 issues the cp.async.bulk of the
// warp's NEXT row (mbarrier-tracked) before the warp works on the current
// one, so a row's load latency overlaps the previous row's max / exp / sum /
// divide chain -- the register-staged kernel above waits for every row's
// loads (config-4 forward 101 -> 81 us). Same arithmetic as k_softmax_fwd_v.
// The backward keeps the register-staged form: staging its two rows (z, g)
// per warp halves the warps per SM, and that measured slower.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void row_bulk(float* dst, const float* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of dst
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void row_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
               "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)), "r"(parity) : "memory");
}

template <int NV>
__global__ void __launch_bounds__(256, B2_SMX_MINB) k_softmax_fwd_tma(float* __restrict__ y, float* __restrict__ rs,
                                                                     float* __restrict__ rm,
                                                                     const float* __restrict__ z, int64_t B,
                                                                     int64_t C) {
  extern __shared__ __align__(128) float smx[];
  __shared__ __align__(8) uint64_t bars[8][2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* const buf0 = smx + (wid * 2) * (NV * 128);
  float* const buf1 = buf0 + NV * 128;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t bytes = (uint32_t)(C * 4);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bars[wid][0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bars[wid][1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (w < B) row_bulk(buf0, z + w * C, bytes, &bars[wid][0]);
  }
  __syncwarp();
  int it = 0;
  for (int64_t r = w; r < B; r += nw, ++it) {
    const int b = it & 1;
    if (lane == 0 && r + nw < B) row_bulk(b ? buf0 : buf1, z + (r + nw) * C, bytes, &bars[wid][b ^ 1]);
    row_wait(&bars[wid][b], (uint32_t)(it >> 1) & 1);
    const float4* row = reinterpret_cast<const float4*>(b ? buf1 : buf0);
    float4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      v[i] = q * 4 < C ? row[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncwarp();  // every lane has its values: the buffer may be refilled next iteration
    const float m = row_max_regs<NV>(v, C, lane);
    double acc = 0;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float e = b2::exp_f32(__fsub_rn(f4get(v[i], k), m));  // exp(sub(z, m))
        f4set(v[i], k, e);
        if ((int64_t)(i * 32 + lane) * 4 + k < C) acc += (double)e;
      }
    const float s = __double2float_rn(warp_sum(acc));  // sum(e, -1, keepdims)
    const bool ok = s >= 1.0f && s <= 0x1p100f;
    const float rs_ = __frcp_rn(s);
    float4* yr = reinterpret_cast<float4*>(y + r * C);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      if (q * 4 < C)
        yr[q] = make_float4(div_by(v[i].x, s, rs_, ok), div_by(v[i].y, s, rs_, ok),
                            div_by(v[i].z, s, rs_, ok), div_by(v[i].w, s, rs_, ok));  // div(e, s)
    }
    if (lane == 0) {
      rs[r] = s;
      rm[r] = m;
    }
  }
}

template <int NV>
__global__ void __launch_bounds__(256, B2_SMX_MINB) k_softmax_bwd_v(float* __restrict__ gz,
                                                       const float* __restrict__ gy,
                                                       const float* __restrict__ z,
                                                       const float* __restrict__ rs,
                                                       const float* __restrict__ rm, int64_t B,
                                                       int64_t C) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < B; r += nw) {
    const float4* zr = reinterpret_cast<const float4*>(z + r * C);
    const float4* gr = reinterpret_cast<const float4*>(gy + r * C);
    float4 ev[NV], gv[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      const bool in = q * 4 < C;
      ev[i] = in ? __ldg(zr + q) : make_float4(0.f, 0.f, 0.f, 0.f);
      gv[i] = in ? __ldg(gr + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float s = rs[r], m = rm[r];
    const float ss = __fmul_rn(s, s);
    const bool ok = s >= 1.0f && ss <= 0x1p100f;
    const float rs_ = __frcp_rn(s), rss = __frcp_rn(ss);
    double acc = 0;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float e = b2::exp_f32(__fsub_rn(f4get(ev[i], k), m));
        f4set(ev[i], k, e);
        const float t = div_by(__fmul_rn(f4get(gv[i], k), e), ss, rss, ok);  // div(mul(g, e), mul(s, s))
        if ((int64_t)(i * 32 + lane) * 4 + k < C) acc += (double)(-t);  // neg, then sum(axis=-1)
      }
    const float gs = __double2float_rn(warp_sum(acc));
    float4* out = reinterpret_cast<float4*>(gz + r * C);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      if (q * 4 < C) {
        float4 o;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float ge = div_by(f4get(gv[i], k), s, rs_, ok);  // div(g, s) -- stored first
          f4set(o, k, __fmul_rn(__fadd_rn(ge, gs), f4get(ev[i], k)));  // GradStore add, exp pullback
        }
        out[q] = o;
      }
    }
  }
}

// Row form of the cross-entropy pullback for C % 4 == 0, 16-B aligned rows:
// a warp per row, the row's (m, se) and label loaded once, 128-bit loads and
// stores, no per-element 64-bit index division. Same per-element arithmetic
// as k_xent_bwd (bit-identical).
template <int NV>
__global__ void __launch_bounds__(256, B2_SMX_MINB) k_xent_bwd_v(float* __restrict__ dz, const float* __restrict__ g,
                                                    const double* __restrict__ row_stats,
                                                    const float* __restrict__ z,
                                                    const int64_t* __restrict__ labels, int64_t B,
                                                    int64_t C, double denom) {
  const double gv = (double)g[0] / denom;  // nn.py:489
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < B; r += nw) {
    const double m = row_stats[2 * r], se = row_stats[2 * r + 1];
    const int64_t lab = labels[r];
    const float4* zr = reinterpret_cast<const float4*>(z + r * C);
    float4* out = reinterpret_cast<float4*>(dz + r * C);
    float4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      v[i] = q * 4 < C ? __ldg(zr + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      if (q * 4 < C) {
        float4 o;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t j = q * 4 + k;
          const double pr = b2::exp_fast((double)f4get(v[i], k) - m) / se - (j == lab ? 1.0 : 0.0);
          f4set(o, k, __double2float_rn(pr * gv));  // nn.py:500
        }
        out[q] = o;
      }
    }
  }
}

// Row form of the cross-entropy forward (C % 4 == 0, 16-B aligned rows): the
// row held in registers, one pass for the max and one for the compensated
// sum of exp(v - m) in double (each lane a Neumaier pair, fixed butterfly).
template <int NV>
__global__ void __launch_bounds__(256, B2_SMX_MINB) k_xent_rows_v(double* __restrict__ row_loss,
                                                     double* __restrict__ row_stats,
                                                     const float* __restrict__ z,
                                                     const int64_t* __restrict__ labels, int64_t B,
                                                     int64_t C) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < B; r += nw) {
    const float4* zr = reinterpret_cast<const float4*>(z + r * C);
    float4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      v[i] = q * 4 < C ? __ldg(zr + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const double m = (double)row_max_regs<NV>(v, C, lane);
    double sum = 0, comp = 0;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((int64_t)(i * 32 + lane) * 4 + k < C) neu_add(sum, comp, b2::exp_fast((double)f4get(v[i], k) - m));
    const double tot = warp_sum(sum + comp);
    if (lane == 0) {
      row_stats[2 * r] = m;
      row_stats[2 * r + 1] = tot;
      const int64_t lab = labels[r];
      row_loss[r] = m + log(tot) - (lab >= 0 && lab < C ? (double)z[r * C + lab] : (double)NAN);
    }
  }
}

// TMA-staged form of k_xent_rows_v (C % 4 == 0, 16-B aligned rows, C <= 1024):
// each warp bulk-copies its next row into its second shared-memory buffer
// while it reduces the current one, and reads the label's logit from the
// staged row instead of a dependent global load. Same arithmetic.
template <int NV>
__global__ void __launch_bounds__(256, B2_SMX_MINB) k_xent_rows_tma(double* __restrict__ row_loss,
                                                                   double* __restrict__ row_stats,
                                                                   const float* __restrict__ z,
                                                                   const int64_t* __restrict__ labels,
                                                                   int64_t B, int64_t C) {
  extern __shared__ __align__(128) float smx[];
  __shared__ __align__(8) uint64_t bars[8][2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* const buf0 = smx + (wid * 2) * (NV * 128);
  float* const buf1 = buf0 + NV * 128;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t bytes = (uint32_t)(C * 4);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bars[wid][0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bars[wid][1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (w < B) row_bulk(buf0, z + w * C, bytes, &bars[wid][0]);
  }
  __syncwarp();
  int it = 0;
  for (int64_t r = w; r < B; r += nw, ++it) {
    const int b = it & 1;
    if (lane == 0 && r + nw < B) row_bulk(b ? buf0 : buf1, z + (r + nw) * C, bytes, &bars[wid][b ^ 1]);
    const int64_t lab = labels[r];
    row_wait(&bars[wid][b], (uint32_t)(it >> 1) & 1);
    const float* rowp = b ? buf1 : buf0;
    const float4* row = reinterpret_cast<const float4*>(rowp);
    float4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      v[i] = q * 4 < C ? row[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float zl = (lab >= 0 && lab < C) ? rowp[lab] : __int_as_float(0x7fc00000);  // guarded read
    __syncwarp();  // every lane has its values: the buffer may be refilled next iteration
    const double m = (double)row_max_regs<NV>(v, C, lane);
    double sum = 0, comp = 0;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((int64_t)(i * 32 + lane) * 4 + k < C) neu_add(sum, comp, b2::exp_fast((double)f4get(v[i], k) - m));
    const double tot = warp_sum(sum + comp);
    if (lane == 0) {
      row_stats[2 * r] = m;
      row_stats[2 * r + 1] = tot;
      row_loss[r] = m + log(tot) - (double)zl;
    }
  }
}

// ---------------------------------------------------------------- softmax * t, mean (fused)
// BASELINE config 4's loss, loss = mean(softmax(z, -1) * t), as ONE row pass
// each way, bit-identical to composing the reference ops:
//   forward: m, e = f32(exp(f32(z - m))), s = f32(sum64 e), y = f32(e / s)
//     exactly as k_softmax_fwd_tma (y stored only if asked), p = f32(y * t),
//     row_dot[r] = sum64 p, then loss = f32(sum64 row_dot / count) (mean);
//   backward: gp = f32(g / f32(count)) (mean pullback), gy = f32(gp * t) (mul
//     pullback), then k_softmax_bwd_v's GradStore-ordered rounding sequence.
// The backward also emits what the next GEMMs and the bias gradient read:
// gz's 3xBF16 split (hi = bf16(gz), lo = bf16(gz - hi), as b2_bf16x3_split)
// and its column sums (per-warp fp64 column accumulators in shared memory,
// folded in a fixed order: warps, then CTAs), so neither a split pass nor a
// reduction re-reads gz -- and gz itself need not be stored in fp32.
#ifndef B2_WMEAN_MINB
#define B2_WMEAN_MINB 2
#endif
template <int NV, bool FULL>
__global__ void __launch_bounds__(256, B2_WMEAN_MINB) k_smx_wmean_fwd(float* __restrict__ y,
                                                                   float* __restrict__ rs,
                                                                   float* __restrict__ rm,
                                                                   double* __restrict__ row_dot,
                                                                   const float* __restrict__ z,
                                                                   const float* __restrict__ t,
                                                                   int64_t B, int64_t C) {
  extern __shared__ __align__(128) float smx[];
  __shared__ __align__(8) uint64_t bars[8][2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* const buf0 = smx + (wid * 2) * (NV * 128);
  float* const buf1 = buf0 + NV * 128;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t bytes = (uint32_t)(C * 4);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bars[wid][0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bars[wid][1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (w < B) row_bulk(buf0, z + w * C, bytes, &bars[wid][0]);
  }
  __syncwarp();
  int it = 0;
  for (int64_t r = w; r < B; r += nw, ++it) {
    const int b = it & 1;
    if (lane == 0 && r + nw < B) row_bulk(b ? buf0 : buf1, z + (r + nw) * C, bytes, &bars[wid][b ^ 1]);
    const float4* trow = reinterpret_cast<const float4*>(t + r * C);
    float4 tv[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {  // t's loads in flight while the z row lands
      const int64_t q = i * 32 + lane;
      tv[i] = (FULL || q * 4 < C) ? __ldg(trow + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    row_wait(&bars[wid][b], (uint32_t)(it >> 1) & 1);
    const float4* row = reinterpret_cast<const float4*>(b ? buf1 : buf0);
    float4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      v[i] = (FULL || q * 4 < C) ? row[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncwarp();
    const float m = row_max_regs<NV, FULL>(v, C, lane);
    double acc = 0;
    bool win = true;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float e = b2::exp_f32(__fsub_rn(f4get(v[i], k), m));  // exp(sub(z, m))
        f4set(v[i], k, e);
        win &= in_window(e);
        if (FULL || (int64_t)(i * 32 + lane) * 4 + k < C) acc += (double)e;
      }
    const float s = __double2float_rn(warp_sum(acc));  // sum(e, -1, keepdims)
    const bool ok = s >= 1.0f && s <= 0x1p100f;
    const float rs_ = __frcp_rn(s);
    const bool fast = __all_sync(0xffffffffu, win) && ok;  // warp-uniform
    double dot = 0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      if (FULL || q * 4 < C) {
        float4 yq;
        if (fast) {
#pragma unroll
          for (int k = 0; k < 4; ++k) f4set(yq, k, div_fast(f4get(v[i], k), s, rs_));  // div(e, s)
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) f4set(yq, k, __fdiv_rn(f4get(v[i], k), s));
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) dot += (double)__fmul_rn(f4get(yq, k), f4get(tv[i], k));  // mul(y, t), mean's sum
        if (y) reinterpret_cast<float4*>(y + r * C)[q] = yq;
      }
    }
    dot = warp_sum(dot);
    if (lane == 0) {
      rs[r] = s;
      rm[r] = m;
      row_dot[r] = dot;
    }
  }
}

__device__ __forceinline__ void split_store4(__nv_bfloat16* hi, __nv_bfloat16* lo, const float4& o) {
  __nv_bfloat16 h[4], l[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float x = f4get(o, k);
    h[k] = __float2bfloat16_rn(x);
    l[k] = __float2bfloat16_rn(__fsub_rn(x, __bfloat162float(h[k])));
  }
  *reinterpret_cast<uint2*>(hi) = *reinterpret_cast<const uint2*>(h);
  *reinterpret_cast<uint2*>(lo) = *reinterpret_cast<const uint2*>(l);
}

template <int NV, bool FULL>
__global__ void __launch_bounds__(256, B2_WMEAN_MINB) k_smx_wmean_bwd(float* __restrict__ gz,
                                                                   __nv_bfloat16* __restrict__ ghi,
                                                                   __nv_bfloat16* __restrict__ glo,
                                                                   double* __restrict__ colpart,
                                                                   const float* __restrict__ g,
                                                                   float count_f32,
                                                                   const float* __restrict__ z,
                                                                   const float* __restrict__ t,
                                                                   const float* __restrict__ rs,
                                                                   const float* __restrict__ rm,
                                                                   int64_t B, int64_t C) {
  extern __shared__ __align__(16) double colw[];  // [8 warps][4][NV*32] column accumulators
  constexpr int CP = NV * 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* const mycol = colw + wid * 4 * CP;
  if (colpart) {
    for (int i = threadIdx.x; i < 8 * 4 * CP; i += blockDim.x) colw[i] = 0.0;
    __syncthreads();
  }
  const float gp = __fdiv_rn(g[0], count_f32);  // mean pullback: div(g, f32(count))
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < B; r += nw) {
    const float4* zr = reinterpret_cast<const float4*>(z + r * C);
    const float4* tr = reinterpret_cast<const float4*>(t + r * C);
    float4 ev[NV], gv[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      const bool in = FULL || q * 4 < C;
      ev[i] = in ? __ldg(zr + q) : make_float4(0.f, 0.f, 0.f, 0.f);
      gv[i] = in ? __ldg(tr + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float s = rs[r], m = rm[r];
    const float ss = __fmul_rn(s, s);
    const bool ok = s >= 1.0f && ss <= 0x1p100f;
    const float rs_ = __frcp_rn(s), rss = __frcp_rn(ss);
    bool win = true;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float gy = __fmul_rn(gp, f4get(gv[i], k));  // mul pullback: mul(g, t)
        f4set(gv[i], k, gy);
        const float e = b2::exp_f32(__fsub_rn(f4get(ev[i], k), m));
        f4set(ev[i], k, e);
        win &= in_window(gy) && in_window(__fmul_rn(gy, e));
      }
    const bool fast = __all_sync(0xffffffffu, win) && ok;  // warp-uniform
    // the two divisions, with the window check hoisted to the row (warp-
    // uniform branch: the fast loops hold no IEEE-division code)
    double acc = 0;
    if (fast) {
#pragma unroll
      for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float tt = div_fast(__fmul_rn(f4get(gv[i], k), f4get(ev[i], k)), ss, rss);  // div(mul(g, e), mul(s, s))
          if (FULL || (int64_t)(i * 32 + lane) * 4 + k < C) acc += (double)(-tt);  // neg, then sum(axis=-1)
        }
    } else {
#pragma unroll
      for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float tt = __fdiv_rn(__fmul_rn(f4get(gv[i], k), f4get(ev[i], k)), ss);
          if (FULL || (int64_t)(i * 32 + lane) * 4 + k < C) acc += (double)(-tt);
        }
    }
    const float gs = __double2float_rn(warp_sum(acc));
    // ge = div(g, s) -- stored first; kept in gv
    if (fast) {
#pragma unroll
      for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) f4set(gv[i], k, div_fast(f4get(gv[i], k), s, rs_));
    } else {
#pragma unroll
      for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) f4set(gv[i], k, __fdiv_rn(f4get(gv[i], k), s));
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      if (FULL || q * 4 < C) {
        float4 o;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          f4set(o, k, __fmul_rn(__fadd_rn(f4get(gv[i], k), gs), f4get(ev[i], k)));  // GradStore add, exp pullback
        if (gz) reinterpret_cast<float4*>(gz + r * C)[q] = o;
        if (ghi) split_store4(ghi + r * C + q * 4, glo + r * C + q * 4, o);
        if (colpart) {
#pragma unroll
          for (int k = 0; k < 4; ++k) mycol[k * CP + q] += (double)f4get(o, k);
        }
      }
    }
  }
  if (colpart) {  // fold the 8 warps in order: this CTA's column partials
    __syncthreads();
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
      const int q = (int)(c >> 2), k = (int)(c & 3);
      double v = 0;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) v += colw[ww * 4 * CP + k * CP + q];
      colpart[blockIdx.x * C + c] = v;
    }
  }
}

// Cross-entropy pullback that hands its consumers what they read (the last
// Linear's dX / dW GEMMs and its bias gradient): dlogits' 3xBF16 split and
// its column sums (per-warp fp64 column accumulators in shared memory,
// warps then CTAs folded in order), instead of the fp32 tensor that a split
// pass and a column reduction would re-read. Same per-element arithmetic as
// k_xent_bwd_v (bit-identical values); C % 8 == 0, 16-B aligned rows.
template <int NV>
__global__ void __launch_bounds__(256, 2) k_xent_bwd_split(float* __restrict__ dz,
                                                          __nv_bfloat16* __restrict__ ghi,
                                                          __nv_bfloat16* __restrict__ glo,
                                                          double* __restrict__ colpart,
                                                          const float* __restrict__ g,
                                                          const double* __restrict__ row_stats,
                                                          const float* __restrict__ z,
                                                          const int64_t* __restrict__ labels, int64_t B,
                                                          int64_t C, double denom) {
  extern __shared__ __align__(16) double xcol[];  // [8 warps][4][NV*32]
  constexpr int CP = NV * 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* const mycol = xcol + wid * 4 * CP;
  if (colpart) {
    for (int i = threadIdx.x; i < 8 * 4 * CP; i += blockDim.x) xcol[i] = 0.0;
    __syncthreads();
  }
  const double gv = (double)g[0] / denom;  // nn.py:489
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < B; r += nw) {
    const double m = row_stats[2 * r], se = row_stats[2 * r + 1];
    const int64_t lab = labels[r];
    const float4* zr = reinterpret_cast<const float4*>(z + r * C);
    float4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      v[i] = q * 4 < C ? __ldg(zr + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t q = i * 32 + lane;
      if (q * 4 < C) {
        float4 o;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t j = q * 4 + k;
          const double pr = b2::exp_fast((double)f4get(v[i], k) - m) / se - (j == lab ? 1.0 : 0.0);
          f4set(o, k, __double2float_rn(pr * gv));  // nn.py:500
        }
        if (dz) reinterpret_cast<float4*>(dz + r * C)[q] = o;
        if (ghi) split_store4(ghi + r * C + q * 4, glo + r * C + q * 4, o);
        if (colpart) {
#pragma unroll
          for (int k = 0; k < 4; ++k) mycol[k * CP + q] += (double)f4get(o, k);
        }
      }
    }
  }
  if (colpart) {
    __syncthreads();
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
      const int q = (int)(c >> 2), k = (int)(c & 3);
      double t = 0;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) t += xcol[ww * 4 * CP + k * CP + q];
      colpart[blockIdx.x * C + c] = t;
    }
  }
}

// column sums of per-CTA fp64 partials, one f32 rounding: 32 columns x 8
// partial lanes per CTA (lane k folds partial rows k, k+8, ... in order), then
// a fixed shared-memory tree over the 8 lanes -- deterministic
__global__ void __launch_bounds__(256) k_colpart_fold(float* __restrict__ out, const double* __restrict__ part,
                                                      int nparts, int64_t C) {
  __shared__ double sh[256];
  const int c = threadIdx.x & 31, k = threadIdx.x >> 5;
  const int64_t n = blockIdx.x * 32LL + c;
  double s = 0.0;
  if (n < C)
    for (int r = k; r < nparts; r += 8) s += part[(int64_t)r * C + n];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int h = 4; h > 0; h >>= 1) {
    if (k < h) sh[threadIdx.x] += sh[threadIdx.x + 32 * h];
    __syncthreads();
  }
  if (k == 0 && n < C) out[n] = __double2float_rn(sh[c]);
}

int rows_grid(int64_t B) {
  int64_t warps = B;
  int64_t ctas = (warps + 7) / 8;
  int64_t cap = (int64_t)b2::sm_count() * 16;
  return (int)(ctas < cap ? (ctas > 0 ? ctas : 1) : cap);
}

}  // namespace

extern "C" {

int b2_xent_fwd(float* loss, double* row_stats, const float* logits, const int64_t* labels,
                int64_t rows, int64_t cols, double denom, void* stream) {
  if (rows <= 0 || cols <= 0) return b2::fail("b2_xent_fwd: empty logits");
  cudaStream_t st = b2::resolve(stream);
  void* ws = nullptr;
  B2_TRY(b2_alloc((size_t)rows * sizeof(double), st, &ws));
  const bool vec = cols % 4 == 0 && cols <= 2048 && ((uintptr_t)logits & 15) == 0;
  if (vec && cols <= 1024 && kSoftmaxTma) {
    const int nv = (int)((cols + 127) / 128);
    const int64_t ctas = std::min<int64_t>((rows + 7) / 8, 3LL * b2::sm_count());
#define B2_XT(NV)                                                                               \
  {                                                                                             \
    const int smem = 8 * 2 * NV * 128 * 4;                                                      \
    static bool attr = false;                                                                   \
    if (!attr) {                                                                                \
      B2_CUDA(cudaFuncSetAttribute(k_xent_rows_tma<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
      attr = true;                                                                              \
    }                                                                                           \
    k_xent_rows_tma<NV><<<(unsigned)ctas, 256, smem, st>>>((double*)ws, row_stats, logits, labels, rows, cols); \
  }
    if (nv <= 1) B2_XT(1)
    else if (nv <= 2) B2_XT(2)
    else if (nv <= 4) B2_XT(4)
    else B2_XT(8)
#undef B2_XT
  } else if (vec) {
    const int nv = (int)((cols + 127) / 128);
#define B2_XF(NV) \
  k_xent_rows_v<NV><<<rows_grid(rows), 256, 0, st>>>((double*)ws, row_stats, logits, labels, rows, cols)
    if (nv <= 1) B2_XF(1);
    else if (nv <= 2) B2_XF(2);
    else if (nv <= 4) B2_XF(4);
    else if (nv <= 8) B2_XF(8);
    else B2_XF(16);
#undef B2_XF
  } else {
    k_xent_rows<<<rows_grid(rows), 256, 0, st>>>((double*)ws, row_stats, logits, labels, rows, cols);
  }
  int rc = b2::launched("b2_xent_fwd(rows)");
  if (!rc) {
    k_xent_final<<<1, 1024, 0, st>>>(loss, (const double*)ws, rows, denom);
    rc = b2::launched("b2_xent_fwd(final)");
  }
  b2_free(ws, st);
  return rc;
}

int b2_xent_bwd(float* dlogits, const float* g, const double* row_stats, const float* logits,
                const int64_t* labels, int64_t rows, int64_t cols, double denom, void* stream) {
  if (rows <= 0 || cols <= 0) return 0;
  cudaStream_t st = b2::resolve(stream);
  const bool vec = cols % 4 == 0 && cols <= 2048 && ((uintptr_t)logits & 15) == 0 &&
                   ((uintptr_t)dlogits & 15) == 0;
  if (vec) {
    const int nv = (int)((cols + 127) / 128);
#define B2_XB(NV) \
  k_xent_bwd_v<NV><<<rows_grid(rows), 256, 0, st>>>(dlogits, g, row_stats, logits, labels, rows, cols, denom)
    if (nv <= 1) B2_XB(1);
    else if (nv <= 2) B2_XB(2);
    else if (nv <= 4) B2_XB(4);
    else if (nv <= 8) B2_XB(8);
    else B2_XB(16);
#undef B2_XB
    return b2::launched("b2_xent_bwd");
  }
  // one element per thread while that fills the chip (config 1's [256, 10]: 10 CTAs
  // of latency-bound fp64 exp + div chains instead of 2 CTAs x 5 elements deep)
  int grid = b2::grid_for(rows * cols, rows * cols <= 256LL * 8 * b2::sm_count() ? 256 : 256 * 8, 8);
  k_xent_bwd<<<grid, 256, 0, st>>>(dlogits, g, row_stats, logits, labels, rows, cols, denom);
  return b2::launched("b2_xent_bwd");
}

int b2_softmax_fwd(float* y, float* row_s, float* row_m, const float* z, int64_t rows,
                   int64_t cols, void* stream) {
  if (rows <= 0 || cols <= 0) return 0;
  cudaStream_t st = b2::resolve(stream);
  const bool vec = cols % 4 == 0 && cols <= 2048 && ((uintptr_t)z & 15) == 0 && ((uintptr_t)y & 15) == 0;
  if (vec && cols <= 1024 && ((uintptr_t)y & 15) == 0 && kSoftmaxTma) {
    // TMA-staged rows, persistent: 3 CTAs of 8 warps per SM, 2 row buffers per warp
    const int nv = (int)((cols + 127) / 128);
    const int64_t ctas = std::min<int64_t>((rows + 7) / 8, 3LL * b2::sm_count());
#define B2_SMT(NV)                                                                              \
  {                                                                                             \
    const int smem = 8 * 2 * NV * 128 * 4;                                                      \
    static bool attr = false;                                                                   \
    if (!attr) {                                                                                \
      B2_CUDA(cudaFuncSetAttribute(k_softmax_fwd_tma<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
      attr = true;                                                                              \
    }                                                                                           \
    k_softmax_fwd_tma<NV><<<(unsigned)ctas, 256, smem, st>>>(y, row_s, row_m, z, rows, cols);   \
  }
    if (nv <= 1) B2_SMT(1)
    else if (nv <= 2) B2_SMT(2)
    else if (nv <= 4) B2_SMT(4)
    else B2_SMT(8)
#undef B2_SMT
    return b2::launched("b2_softmax_fwd(tma)");
  }
  if (vec) {
    const int nv = (int)((cols + 127) / 128);
#define B2_SMF(NV) k_softmax_fwd_v<NV><<<rows_grid(rows), 256, 0, st>>>(y, row_s, row_m, z, rows, cols)
    if (nv <= 1) B2_SMF(1);
    else if (nv <= 2) B2_SMF(2);
    else if (nv <= 4) B2_SMF(4);
    else if (nv <= 8) B2_SMF(8);
    else B2_SMF(16);
#undef B2_SMF
  } else {
    k_softmax_fwd<<<rows_grid(rows), 256, 0, st>>>(y, row_s, row_m, z, rows, cols);
  }
  return b2::launched("b2_softmax_fwd");
}

int b2_softmax_bwd(float* gz, const float* gy, const float* z, const float* row_s,
                   const float* row_m, int64_t rows, int64_t cols, void* stream) {
  if (rows <= 0 || cols <= 0) return 0;
  cudaStream_t st = b2::resolve(stream);
  const bool vec = cols % 4 == 0 && cols <= 2048 && ((uintptr_t)z & 15) == 0 &&
                   ((uintptr_t)gy & 15) == 0 && ((uintptr_t)gz & 15) == 0;
  if (vec) {
    const int nv = (int)((cols + 127) / 128);
#define B2_SMB(NV) k_softmax_bwd_v<NV><<<rows_grid(rows), 256, 0, st>>>(gz, gy, z, row_s, row_m, rows, cols)
    if (nv <= 1) B2_SMB(1);
    else if (nv <= 2) B2_SMB(2);
    else if (nv <= 4) B2_SMB(4);
    else if (nv <= 8) B2_SMB(8);
    else B2_SMB(16);
#undef B2_SMB
  } else {
    k_softmax_bwd<<<rows_grid(rows), 256, 0, st>>>(gz, gy, z, row_s, row_m, rows, cols);
  }
  return b2::launched("b2_softmax_bwd");
}

int b2_softmax_wmean_fwd(float* loss, float* y, float* row_s, float* row_m, double* row_dot,
                         const float* z, const float* t, int64_t rows, int64_t cols, void* stream) {
  if (rows <= 0 || cols <= 0) return b2::fail("b2_softmax_wmean_fwd: empty input");
  if (cols % 4 || cols > 1024 || ((uintptr_t)z & 15) || ((uintptr_t)t & 15) || ((uintptr_t)y & 15))
    return b2::fail("b2_softmax_wmean_fwd: rows must be 16-B aligned with cols % 4 == 0, cols <= 1024");
  cudaStream_t st = b2::resolve(stream);
  const int nv = (int)((cols + 127) / 128);
  const int64_t ctas = std::min<int64_t>((rows + 7) / 8, (int64_t)B2_WMEAN_MINB * b2::sm_count());
#define B2_SWF(NV)                                                                              \
  {                                                                                             \
    const int smem = 8 * 2 * NV * 128 * 4;                                                      \
    static bool attr = false;                                                                   \
    if (!attr) {                                                                                \
      B2_CUDA(cudaFuncSetAttribute(k_smx_wmean_fwd<NV, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
      B2_CUDA(cudaFuncSetAttribute(k_smx_wmean_fwd<NV, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
      attr = true;                                                                              \
    }                                                                                           \
    if (cols == NV * 128)                                                                       \
      k_smx_wmean_fwd<NV, true><<<(unsigned)ctas, 256, smem, st>>>(y, row_s, row_m, row_dot, z, t, rows, cols); \
    else                                                                                        \
      k_smx_wmean_fwd<NV, false><<<(unsigned)ctas, 256, smem, st>>>(y, row_s, row_m, row_dot, z, t, rows, cols); \
  }
  if (nv <= 1) B2_SWF(1)
  else if (nv <= 2) B2_SWF(2)
  else if (nv <= 4) B2_SWF(4)
  else B2_SWF(8)
#undef B2_SWF
  B2_TRY(b2::launched("b2_softmax_wmean_fwd(rows)"));
  k_xent_final<<<1, 1024, 0, st>>>(loss, row_dot, rows, (double)rows * (double)cols);
  return b2::launched("b2_softmax_wmean_fwd(final)");
}

int b2_softmax_wmean_bwd(float* gz, void* gz_hi, void* gz_lo, float* colsum, const float* g,
                         float count_f32, const float* z, const float* t, const float* row_s,
                         const float* row_m, int64_t rows, int64_t cols, void* stream) {
  if (rows <= 0 || cols <= 0) return 0;
  if (cols % 4 || cols > 1024 || ((uintptr_t)z & 15) || ((uintptr_t)t & 15) || ((uintptr_t)gz & 15) ||
      ((uintptr_t)gz_hi & 7) || ((uintptr_t)gz_lo & 7) || (!gz_hi != !gz_lo))
    return b2::fail("b2_softmax_wmean_bwd: rows must be 16-B aligned with cols % 4 == 0, cols <= 1024");
  cudaStream_t st = b2::resolve(stream);
  const int nv = (int)((cols + 127) / 128);
  const int64_t ctas = std::min<int64_t>((rows + 7) / 8, (int64_t)B2_WMEAN_MINB * b2::sm_count());
  double* part = nullptr;
  if (colsum) B2_TRY(b2_alloc((size_t)ctas * cols * sizeof(double), st, (void**)&part));
#define B2_SWB(NV)                                                                              \
  {                                                                                             \
    const int smem = colsum ? 8 * 4 * NV * 32 * 8 : 0;                                          \
    static bool attr = false;                                                                   \
    if (!attr) {                                                                                \
      B2_CUDA(cudaFuncSetAttribute(k_smx_wmean_bwd<NV, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * NV * 32 * 8)); \
      B2_CUDA(cudaFuncSetAttribute(k_smx_wmean_bwd<NV, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * NV * 32 * 8)); \
      attr = true;                                                                              \
    }                                                                                           \
    if (cols == NV * 128)                                                                       \
      k_smx_wmean_bwd<NV, true><<<(unsigned)ctas, 256, smem, st>>>(gz, (__nv_bfloat16*)gz_hi,   \
          (__nv_bfloat16*)gz_lo, part, g, count_f32, z, t, row_s, row_m, rows, cols);            \
    else                                                                                        \
      k_smx_wmean_bwd<NV, false><<<(unsigned)ctas, 256, smem, st>>>(gz, (__nv_bfloat16*)gz_hi,  \
          (__nv_bfloat16*)gz_lo, part, g, count_f32, z, t, row_s, row_m, rows, cols);            \
  }
  if (nv <= 1) B2_SWB(1)
  else if (nv <= 2) B2_SWB(2)
  else if (nv <= 4) B2_SWB(4)
  else B2_SWB(8)
#undef B2_SWB
  int rc = b2::launched("b2_softmax_wmean_bwd");
  if (!rc && colsum) {
    k_colpart_fold<<<(unsigned)((cols + 31) / 32), 256, 0, st>>>(colsum, part, (int)ctas, cols);
    rc = b2::launched("b2_softmax_wmean_bwd(colsum)");
  }
  if (part) b2_free(part, st);
  return rc;
}

int b2_xent_bwd_split(float* dlogits, void* dl_hi, void* dl_lo, float* colsum, const float* g,
                      const double* row_stats, const float* logits, const int64_t* labels, int64_t rows,
                      int64_t cols, double denom, void* stream) {
  if (rows <= 0 || cols <= 0) return 0;
  if (cols % 8 || cols > 1024 || ((uintptr_t)logits & 15) || ((uintptr_t)dlogits & 15) ||
      ((uintptr_t)dl_hi & 15) || ((uintptr_t)dl_lo & 15) || (!dl_hi != !dl_lo))
    return b2::fail("b2_xent_bwd_split: needs cols % 8 == 0, cols <= 1024 and 16-B aligned rows");
  cudaStream_t st = b2::resolve(stream);
  const int nv = (int)((cols + 127) / 128);
  const int64_t ctas = std::min<int64_t>((rows + 7) / 8, 2LL * b2::sm_count());
  double* part = nullptr;
  if (colsum) B2_TRY(b2_alloc((size_t)ctas * cols * sizeof(double), st, (void**)&part));
#define B2_XBS(NV)                                                                              \
  {                                                                                             \
    const int smem = colsum ? 8 * 4 * NV * 32 * 8 : 0;                                          \
    static bool attr = false;                                                                   \
    if (!attr) {                                                                                \
      B2_CUDA(cudaFuncSetAttribute(k_xent_bwd_split<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * NV * 32 * 8)); \
      attr = true;                                                                              \
    }                                                                                           \
    k_xent_bwd_split<NV><<<(unsigned)ctas, 256, smem, st>>>(dlogits, (__nv_bfloat16*)dl_hi,     \
        (__nv_bfloat16*)dl_lo, part, g, row_stats, logits, labels, rows, cols, denom);           \
  }
  if (nv <= 1) B2_XBS(1)
  else if (nv <= 2) B2_XBS(2)
  else if (nv <= 4) B2_XBS(4)
  else B2_XBS(8)
#undef B2_XBS
  int rc = b2::launched("b2_xent_bwd_split");
  if (!rc && colsum) {
    k_colpart_fold<<<(unsigned)((cols + 31) / 32), 256, 0, st>>>(colsum, part, (int)ctas, cols);
    rc = b2::launched("b2_xent_bwd_split(colsum)");
  }
  if (part) b2_free(part, st);
  return rc;
}

}  // extern "C"
