// Broadcasting / strided elementwise engine.
//
// Replaces tensorlite/core.py:430-546 (_elementwise/_binary/_unary) and the
// pointwise activations of nn.py:95-111. Semantics: every result is the
// IEEE fp32 op, which equals the reference's f32(double op) for + - * /
// (double rounding is innocuous since 53 >= 2*24+2); exp/log are computed as
// f32(double libm) exactly like the reference. No FMA contraction anywhere in
// this file (explicit __f*_rn intrinsics, and the TU is built -fmad=false).
//
// Layout strategy (HBM-bound; index math hoisted per row, never per element):
//  * shapes/strides are collapsed on the host (adjacent dims merged when every
//    operand is contiguous across them, size-1 dims dropped);
//  * 1-D result  -> flat grid-stride kernel, 128-bit loads/stores;
//  * N-D result  -> "rows" kernel: rows = product of outer dims, the row base
//    offset of each operand is computed once per row, the innermost dim is
//    walked with float4 when its stride is 1 and rows are 16-B aligned, a
//    stride-0 operand is a register broadcast.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "fexp.cuh"

namespace {

constexpr int kThreads = 256;

struct Nd {
  int ndim;  // collapsed rank (>= 1)
  int64_t shape[B2_MAX_DIMS];
  int64_t st[3][B2_MAX_DIMS];  // [0]=out (contiguous), [1]=a, [2]=b
};

// merge dims and drop size-1 axes; nops operands (out first)
Nd collapse(int ndim, const int64_t* shape, int nops, const int64_t* const* strides) {
  Nd r;
  r.ndim = 0;
  for (int d = 0; d < ndim; ++d) {
    if (shape[d] == 1) continue;
    int k = r.ndim;
    if (k > 0) {
      bool merge = true;
      for (int o = 0; o < nops; ++o)
        if (r.st[o][k - 1] != strides[o][d] * shape[d]) merge = false;
      if (merge) {
        r.shape[k - 1] *= shape[d];
        for (int o = 0; o < nops; ++o) r.st[o][k - 1] = strides[o][d];
        continue;
      }
    }
    r.shape[k] = shape[d];
    for (int o = 0; o < nops; ++o) r.st[o][k] = strides[o][d];
    r.ndim++;
  }
  if (r.ndim == 0) {
    r.ndim = 1;
    r.shape[0] = 1;
    for (int o = 0; o < nops; ++o) r.st[o][0] = 1;
  }
  return r;
}

void contig_strides(int ndim, const int64_t* shape, int64_t* st) {
  int64_t acc = 1;
  for (int d = ndim - 1; d >= 0; --d) {
    st[d] = acc;
    acc *= shape[d];
  }
}

int64_t numel(int ndim, const int64_t* shape) {
  int64_t n = 1;
  for (int d = 0; d < ndim; ++d) n *= shape[d];
  return n;
}

// ------------------------------------------------------------------ ops

__device__ __forceinline__ float sign_of(float v) {
  return v > 0.0f ? 1.0f : (v < 0.0f ? -1.0f : 0.0f);  // core.py:533-538
}

// activations and their derivatives in double, like the reference's
// math.* on Python floats (nn.py:114-144); one f32 rounding at the store
__device__ __forceinline__ double sigmoid_d(double v) {
  if (v >= 0.0) return 1.0 / (1.0 + b2::exp_fast(-v));  // split on sign: exp never overflows
  const double e = b2::exp_fast(v);
  return e / (1.0 + e);
}
constexpr double kSqrt2 = 1.4142135623730951;          // math.sqrt(2.0)
constexpr double kInvSqrt2Pi = 0.3989422804014327;     // 1 / math.sqrt(2 pi)
__device__ __forceinline__ double gelu_d(double v) { return 0.5 * v * (1.0 + erf(v / kSqrt2)); }
__device__ __forceinline__ double gelu_deriv_d(double v) {
  const double cdf = 0.5 * (1.0 + erf(v / kSqrt2));
  const double pdf = kInvSqrt2Pi * b2::exp_fast(-0.5 * v * v);
  return cdf + v * pdf;
}

template <int OP>
struct Bin {
  __device__ __forceinline__ float operator()(float a, float b) const {
    if constexpr (OP == B2_ADD) return __fadd_rn(a, b);
    if constexpr (OP == B2_SUB) return __fsub_rn(a, b);
    if constexpr (OP == B2_MUL) return __fmul_rn(a, b);
    if constexpr (OP == B2_DIV) return __fdiv_rn(a, b);
    if constexpr (OP == B2_RELU_BWD) return __fmul_rn(a, b > 0.0f ? 1.0f : 0.0f);
    if constexpr (OP == B2_SIGN_MUL) return __fmul_rn(a, sign_of(b));
    if constexpr (OP == B2_SIGMOID_BWD) {
      const double y = b;
      return __fmul_rn(a, __double2float_rn(__dmul_rn(y, __dsub_rn(1.0, y))));
    }
    if constexpr (OP == B2_TANH_BWD) {
      const double y = b;
      return __fmul_rn(a, __double2float_rn(__dsub_rn(1.0, __dmul_rn(y, y))));
    }
    if constexpr (OP == B2_GELU_BWD) return __fmul_rn(a, __double2float_rn(gelu_deriv_d(b)));
    return 0.0f;
  }
};

template <int OP>
struct Un {
  double alpha, beta;
  __device__ __forceinline__ float operator()(float x) const {
    if constexpr (OP == B2_NEG) return -x;
    if constexpr (OP == B2_EXP) return b2::exp_f32(x);
    if constexpr (OP == B2_LOG) return __double2float_rn(log((double)x));
    if constexpr (OP == B2_SQRT) return __fsqrt_rn(x);
    if constexpr (OP == B2_ABS) return fabsf(x);
    if constexpr (OP == B2_RELU) return x > 0.0f ? x : 0.0f;  // nn.py:110
    if constexpr (OP == B2_RELU_MASK) return x > 0.0f ? 1.0f : 0.0f;
    if constexpr (OP == B2_COPY) return x;
    if constexpr (OP == B2_CLAMP) return x != x ? x : fminf(fmaxf(x, (float)alpha), (float)beta);  // NaN passes (np.clip)
    if constexpr (OP == B2_SCALE) return __fmul_rn(x, (float)alpha);
    if constexpr (OP == B2_DIV_SCALAR) return __fdiv_rn(x, (float)alpha);
    if constexpr (OP == B2_CLAMP_MASK) return (x >= (float)alpha && x <= (float)beta) ? 1.0f : 0.0f;
    if constexpr (OP == B2_SIGMOID) return __double2float_rn(sigmoid_d(x));
    if constexpr (OP == B2_TANH) return __double2float_rn(tanh((double)x));
    if constexpr (OP == B2_GELU) return __double2float_rn(gelu_d(x));
    return x;
  }
};

struct Fill {
  float v;
  __device__ __forceinline__ float operator()(float) const { return v; }
};

// binary with one operand replaced by an fp32 scalar
template <int OP, bool LEFT>
struct BinScalar {
  float s;
  __device__ __forceinline__ float operator()(float x) const {
    Bin<OP> f;
    return LEFT ? f(s, x) : f(x, s);
  }
};

// ------------------------------------------------------------------ kernels

// flat: out[i] = f(a[i*sa], b[i*sb]); sa, sb in {0, 1}
template <class F, bool VEC>
__global__ void __launch_bounds__(kThreads) k_bin_flat(float* __restrict__ out,
                                                       const float* __restrict__ a,
                                                       const float* __restrict__ b, int64_t n,
                                                       int sa, int sb, F f) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t nth = (int64_t)gridDim.x * blockDim.x;
  if (VEC) {
    int64_t n4 = n >> 2;
    float as = a[0], bs = b[0];
    for (int64_t i = tid; i < n4; i += nth) {
      float4 va = sa ? reinterpret_cast<const float4*>(a)[i] : make_float4(as, as, as, as);
      float4 vb = sb ? reinterpret_cast<const float4*>(b)[i] : make_float4(bs, bs, bs, bs);
      float4 r;
      r.x = f(va.x, vb.x);
      r.y = f(va.y, vb.y);
      r.z = f(va.z, vb.z);
      r.w = f(va.w, vb.w);
      reinterpret_cast<float4*>(out)[i] = r;
    }
    for (int64_t i = (n4 << 2) + tid; i < n; i += nth) out[i] = f(a[i * sa], b[i * sb]);
  } else {
    for (int64_t i = tid; i < n; i += nth) out[i] = f(a[i * sa], b[i * sb]);
  }
}

template <class F, bool VEC>
__global__ void __launch_bounds__(kThreads) k_un_flat(float* __restrict__ out,
                                                      const float* __restrict__ x, int64_t n,
                                                      int64_t sx, F f) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t nth = (int64_t)gridDim.x * blockDim.x;
  if (VEC) {
    // software-pipelined: the next 128-bit load is in flight while this one's
    // results are computed (exp's FP64 polynomial would otherwise serialise
    // with the memory latency)
    const int64_t n4 = n >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    int64_t i = tid;
    float4 v = i < n4 ? __ldg(x4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    for (; i < n4; i += nth) {
      const int64_t nx = i + nth;
      const float4 vn = nx < n4 ? __ldg(x4 + nx) : v;
      float4 r;
      r.x = f(v.x);
      r.y = f(v.y);
      r.z = f(v.z);
      r.w = f(v.w);
      reinterpret_cast<float4*>(out)[i] = r;
      v = vn;
    }
    for (int64_t i = (n4 << 2) + tid; i < n; i += nth) out[i] = f(x[i]);
  } else {
    for (int64_t i = tid; i < n; i += nth) out[i] = f(x[i * sx]);
  }
}

struct RowGeom {
  int nd;                         // number of OUTER dims (collapsed ndim - 1)
  int64_t oshape[B2_MAX_DIMS];    // outer dims
  int64_t ost[3][B2_MAX_DIMS];    // outer strides per operand
  int64_t inner;                  // innermost extent
  int64_t ist[3];                 // innermost stride per operand
  int64_t rows;
};

__device__ __forceinline__ void row_base(const RowGeom& g, int64_t r, int64_t* base, int nops) {
  for (int o = 0; o < nops; ++o) base[o] = 0;
  for (int d = g.nd - 1; d >= 0; --d) {
    int64_t ext = g.oshape[d];
    int64_t q = r / ext;
    int64_t i = r - q * ext;
    r = q;
    for (int o = 0; o < nops; ++o) base[o] += i * g.ost[o][d];
  }
}

// N-d binary: grid.x strides rows, grid.y splits the inner extent
template <class F, bool VEC>
__global__ void __launch_bounds__(kThreads) k_bin_rows(float* __restrict__ out,
                                                       const float* __restrict__ a,
                                                       const float* __restrict__ b, RowGeom g,
                                                       int64_t chunk, F f) {
  int64_t c0 = blockIdx.y * chunk;
  int64_t c1 = min(g.inner, c0 + chunk);
  for (int64_t r = blockIdx.x; r < g.rows; r += gridDim.x) {
    int64_t base[3];
    row_base(g, r, base, 3);
    float* o = out + base[0];
    const float* pa = a + base[1];
    const float* pb = b + base[2];
    if (VEC) {  // ist[0]==1, ist[1],ist[2] in {0,1}, rows 16B aligned, chunk%4==0
      float as = pa[0], bs = pb[0];
      for (int64_t c = c0 + 4 * threadIdx.x; c < c1; c += 4 * blockDim.x) {
        if (c + 3 < c1) {
          float4 va = g.ist[1] ? *reinterpret_cast<const float4*>(pa + c) : make_float4(as, as, as, as);
          float4 vb = g.ist[2] ? *reinterpret_cast<const float4*>(pb + c) : make_float4(bs, bs, bs, bs);
          float4 rr;
          rr.x = f(va.x, vb.x);
          rr.y = f(va.y, vb.y);
          rr.z = f(va.z, vb.z);
          rr.w = f(va.w, vb.w);
          *reinterpret_cast<float4*>(o + c) = rr;
        } else {
          for (int64_t k = c; k < c1; ++k) o[k] = f(pa[k * g.ist[1]], pb[k * g.ist[2]]);
        }
      }
    } else {
      for (int64_t c = c0 + threadIdx.x; c < c1; c += blockDim.x)
        o[c * g.ist[0]] = f(pa[c * g.ist[1]], pb[c * g.ist[2]]);
    }
  }
}

template <class F, bool VEC>
__global__ void __launch_bounds__(kThreads) k_un_rows(float* __restrict__ out,
                                                      const float* __restrict__ x, RowGeom g,
                                                      int64_t chunk, F f) {
  int64_t c0 = blockIdx.y * chunk;
  int64_t c1 = min(g.inner, c0 + chunk);
  for (int64_t r = blockIdx.x; r < g.rows; r += gridDim.x) {
    int64_t base[3];
    row_base(g, r, base, 2);
    float* o = out + base[0];
    const float* px = x + base[1];
    if (VEC) {
      float xs = px[0];
      for (int64_t c = c0 + 4 * threadIdx.x; c < c1; c += 4 * blockDim.x) {
        if (c + 3 < c1) {
          float4 v = g.ist[1] ? *reinterpret_cast<const float4*>(px + c) : make_float4(xs, xs, xs, xs);
          float4 rr;
          rr.x = f(v.x);
          rr.y = f(v.y);
          rr.z = f(v.z);
          rr.w = f(v.w);
          *reinterpret_cast<float4*>(o + c * g.ist[0]) = rr;
        } else {
          for (int64_t k = c; k < c1; ++k) o[k * g.ist[0]] = f(px[k * g.ist[1]]);
        }
      }
    } else {
      for (int64_t c = c0 + threadIdx.x; c < c1; c += blockDim.x)
        o[c * g.ist[0]] = f(px[c * g.ist[1]]);
    }
  }
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

RowGeom make_rows(const Nd& nd, int nops) {
  RowGeom g;
  g.nd = nd.ndim - 1;
  g.rows = 1;
  for (int d = 0; d < g.nd; ++d) {
    g.oshape[d] = nd.shape[d];
    g.rows *= nd.shape[d];
    for (int o = 0; o < nops; ++o) g.ost[o][d] = nd.st[o][d];
  }
  for (int o = nops; o < 3; ++o)
    for (int d = 0; d < g.nd; ++d) g.ost[o][d] = 0;
  g.inner = nd.shape[nd.ndim - 1];
  for (int o = 0; o < 3; ++o) g.ist[o] = o < nops ? nd.st[o][nd.ndim - 1] : 0;
  return g;
}

// rows 16B-aligned for every vector operand
bool rows_vec_ok(const RowGeom& g, const float* const* ptrs, int nops) {
  for (int o = 0; o < nops; ++o) {
    if (g.ist[o] != 1 && !(o > 0 && g.ist[o] == 0)) return false;
    if (g.ist[o] == 1) {
      if (!aligned16(ptrs[o])) return false;
      for (int d = 0; d < g.nd; ++d)
        if (g.ost[o][d] % 4) return false;
    }
  }
  return true;
}

void rows_grid(const RowGeom& g, dim3* grid, int64_t* chunk) {
  int target = b2::sm_count() * 8;
  int64_t gx = std::min<int64_t>(g.rows, target);
  int64_t gy = 1;
  if (g.rows < target) {
    gy = std::max<int64_t>(1, target / std::max<int64_t>(g.rows, 1));
    gy = std::min<int64_t>(gy, std::max<int64_t>(1, g.inner / (4 * kThreads)));
  }
  int64_t ch = (g.inner + gy - 1) / gy;
  ch = (ch + 3) & ~int64_t(3);
  gy = (g.inner + ch - 1) / ch;
  if (gy < 1) gy = 1;
  *grid = dim3((unsigned)std::max<int64_t>(gx, 1), (unsigned)gy);
  *chunk = ch;
}

template <class F>
int launch_binary(float* out, const Nd& nd, const float* a, const float* b, F f, cudaStream_t st) {
  int64_t n = 1;
  for (int d = 0; d < nd.ndim; ++d) n *= nd.shape[d];
  if (n == 0) return 0;
  if (nd.ndim == 1 && (nd.st[1][0] == 0 || nd.st[1][0] == 1) && (nd.st[2][0] == 0 || nd.st[2][0] == 1)) {
    bool vec = aligned16(out) && (nd.st[1][0] == 0 || aligned16(a)) && (nd.st[2][0] == 0 || aligned16(b));
    int grid = b2::grid_for(n, kThreads * 4 * 4, 8);
    if (vec)
      k_bin_flat<F, true><<<grid, kThreads, 0, st>>>(out, a, b, n, (int)nd.st[1][0], (int)nd.st[2][0], f);
    else
      k_bin_flat<F, false><<<grid, kThreads, 0, st>>>(out, a, b, n, (int)nd.st[1][0], (int)nd.st[2][0], f);
    return b2::launched("b2_binary(flat)");
  }
  RowGeom g = make_rows(nd, 3);
  dim3 grid;
  int64_t chunk;
  rows_grid(g, &grid, &chunk);
  const float* ptrs[3] = {out, a, b};
  if (rows_vec_ok(g, ptrs, 3))
    k_bin_rows<F, true><<<grid, kThreads, 0, st>>>(out, a, b, g, chunk, f);
  else
    k_bin_rows<F, false><<<grid, kThreads, 0, st>>>(out, a, b, g, chunk, f);
  return b2::launched("b2_binary(rows)");
}

template <class F>
int launch_unary(float* out, const Nd& nd, const float* x, F f, cudaStream_t st) {
  int64_t n = 1;
  for (int d = 0; d < nd.ndim; ++d) n *= nd.shape[d];
  if (n == 0) return 0;
  if (nd.ndim == 1 && nd.st[0][0] == 1) {
    bool vec = nd.st[1][0] == 1 && aligned16(out) && aligned16(x);
    int grid = b2::grid_for(n, kThreads * 4 * 4, 8);
    if (vec)
      k_un_flat<F, true><<<grid, kThreads, 0, st>>>(out, x, n, 1, f);
    else
      k_un_flat<F, false><<<grid, kThreads, 0, st>>>(out, x, n, nd.st[1][0], f);
    return b2::launched("b2_unary(flat)");
  }
  RowGeom g = make_rows(nd, 2);
  dim3 grid;
  int64_t chunk;
  rows_grid(g, &grid, &chunk);
  const float* ptrs[2] = {out, x};
  if (rows_vec_ok(g, ptrs, 2))
    k_un_rows<F, true><<<grid, kThreads, 0, st>>>(out, x, g, chunk, f);
  else
    k_un_rows<F, false><<<grid, kThreads, 0, st>>>(out, x, g, chunk, f);
  return b2::launched("b2_unary(rows)");
}

int check_nd(int ndim, const int64_t* shape) {
  if (ndim < 0 || ndim > B2_MAX_DIMS) return b2::fail("rank exceeds B2_MAX_DIMS (8)");
  for (int d = 0; d < ndim; ++d)
    if (shape[d] < 0) return b2::fail("negative extent");
  return 0;
}

// ------------------------------------------------------------------ fused config-2 chain

// y = relu(f32(f32(a*b) + c)); a:[R,C] contiguous, b,c: [C]
__global__ void __launch_bounds__(kThreads) k_muladd_relu_fwd(float* __restrict__ y,
                                                              const float* __restrict__ a,
                                                              const float* __restrict__ b,
                                                              const float* __restrict__ c,
                                                              int64_t rows, int64_t cols) {
  const int64_t c4 = cols >> 2;
  auto one = [&](const float4& va, int64_t j) {
    const float4 vb = reinterpret_cast<const float4*>(b)[j];
    const float4 vc = reinterpret_cast<const float4*>(c)[j];
    float4 o;
    float q;
    q = __fadd_rn(__fmul_rn(va.x, vb.x), vc.x); o.x = q > 0.f ? q : 0.f;
    q = __fadd_rn(__fmul_rn(va.y, vb.y), vc.y); o.y = q > 0.f ? q : 0.f;
    q = __fadd_rn(__fmul_rn(va.z, vb.z), vc.z); o.z = q > 0.f ? q : 0.f;
    q = __fadd_rn(__fmul_rn(va.w, vb.w), vc.w); o.w = q > 0.f ? q : 0.f;
    return o;
  };
  const int64_t B = blockDim.x;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const float4* pa = reinterpret_cast<const float4*>(a + r * cols);
    float4* py = reinterpret_cast<float4*>(y + r * cols);
    int64_t j = threadIdx.x;
    for (; j + 3 * B < c4; j += 4 * B) {  // 4 independent 128-bit loads in flight
      const float4 v0 = pa[j], v1 = pa[j + B], v2 = pa[j + 2 * B], v3 = pa[j + 3 * B];
      py[j] = one(v0, j);
      py[j + B] = one(v1, j + B);
      py[j + 2 * B] = one(v2, j + 2 * B);
      py[j + 3 * B] = one(v3, j + 3 * B);
    }
    for (; j < c4; j += B) py[j] = one(pa[j], j);
  }
}

#ifndef B2_MULADD_CL
#define B2_MULADD_CL 32
#endif
#ifndef B2_MULADD_CL_CLUSTER
#define B2_MULADD_CL_CLUSTER 8
#endif
constexpr int kMuladdCL = B2_MULADD_CL;  // column lanes per CTA (x4 columns each)

// backward of sum(relu(a*b + b)): ga = f32(mask*b); partial column sums of
// mask*a (fp64) and mask counts per row-split.
__global__ void __launch_bounds__(kThreads) k_muladd_relu_bwd(float* __restrict__ ga,
                                                              double* __restrict__ psum,
                                                              int* __restrict__ pcnt,
                                                              const float* __restrict__ a,
                                                              const float* __restrict__ b,
                                                              int64_t rows, int64_t cols,
                                                              int64_t rows_per_split) {
  // grid: x = strip of 4*CL columns (CL column lanes x float4), y = row split;
  // 256/CL row lanes per CTA (a warp touches 32/CL rows x 16*CL B), folded in smem
  constexpr int CL = kMuladdCL, RL = kThreads / CL;
  __shared__ double sh_s[kThreads * 4];
  __shared__ int sh_n[kThreads * 4];
  const int cl = threadIdx.x % CL, rl = threadIdx.x / CL;
  const int64_t col = (blockIdx.x * (int64_t)CL + cl) * 4;
  const int64_t r0 = blockIdx.y * rows_per_split;
  const int64_t r1 = min(rows, r0 + rows_per_split);
  const bool live = col < cols;
  const float4 vb = live ? *reinterpret_cast<const float4*>(b + col) : make_float4(0, 0, 0, 0);
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int n0 = 0, n1 = 0, n2 = 0, n3 = 0;
  auto one = [&](const float4& va, float4* dst) {
    const float m0 = __fadd_rn(__fmul_rn(va.x, vb.x), vb.x) > 0.f ? 1.f : 0.f;
    const float m1 = __fadd_rn(__fmul_rn(va.y, vb.y), vb.y) > 0.f ? 1.f : 0.f;
    const float m2 = __fadd_rn(__fmul_rn(va.z, vb.z), vb.z) > 0.f ? 1.f : 0.f;
    const float m3 = __fadd_rn(__fmul_rn(va.w, vb.w), vb.w) > 0.f ? 1.f : 0.f;
    *dst = make_float4(__fmul_rn(m0, vb.x), __fmul_rn(m1, vb.y), __fmul_rn(m2, vb.z),
                       __fmul_rn(m3, vb.w));
    s0 += (double)__fmul_rn(m0, va.x);
    s1 += (double)__fmul_rn(m1, va.y);
    s2 += (double)__fmul_rn(m2, va.z);
    s3 += (double)__fmul_rn(m3, va.w);
    n0 += m0 > 0.f;
    n1 += m1 > 0.f;
    n2 += m2 > 0.f;
    n3 += m3 > 0.f;
  };
  if (live) {
    int64_t r = r0 + rl;
    for (; r + 3 * RL < r1; r += 4 * RL) {  // 4 independent 128-bit loads in flight
      const float4 v0 = *reinterpret_cast<const float4*>(a + r * cols + col);
      const float4 v1 = *reinterpret_cast<const float4*>(a + (r + RL) * cols + col);
      const float4 v2 = *reinterpret_cast<const float4*>(a + (r + 2 * RL) * cols + col);
      const float4 v3 = *reinterpret_cast<const float4*>(a + (r + 3 * RL) * cols + col);
      one(v0, reinterpret_cast<float4*>(ga + r * cols + col));
      one(v1, reinterpret_cast<float4*>(ga + (r + RL) * cols + col));
      one(v2, reinterpret_cast<float4*>(ga + (r + 2 * RL) * cols + col));
      one(v3, reinterpret_cast<float4*>(ga + (r + 3 * RL) * cols + col));
    }
    for (; r < r1; r += RL)
      one(*reinterpret_cast<const float4*>(a + r * cols + col),
          reinterpret_cast<float4*>(ga + r * cols + col));
  }
  const int me = (rl * CL + cl) * 4;
  sh_s[me] = s0; sh_s[me + 1] = s1; sh_s[me + 2] = s2; sh_s[me + 3] = s3;
  sh_n[me] = n0; sh_n[me + 1] = n1; sh_n[me + 2] = n2; sh_n[me + 3] = n3;
  __syncthreads();
  for (int h = RL / 2; h > 0; h >>= 1) {  // fixed fold order -> deterministic
    if (rl < h) {
      const int other = ((rl + h) * CL + cl) * 4;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        sh_s[me + j] += sh_s[other + j];
        sh_n[me + j] += sh_n[other + j];
      }
    }
    __syncthreads();
  }
  if (rl == 0 && live) {
    const int64_t o = blockIdx.y * cols + col;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      psum[o + j] = sh_s[cl * 4 + j];
      pcnt[o + j] = sh_n[cl * 4 + j];
    }
  }
}

// 32 columns per CTA x 8 split-lanes per column: lane k folds splits k, k+8,
// ... (warps read 32 consecutive columns), then a fixed smem tree -> deterministic
__global__ void __launch_bounds__(256) k_muladd_relu_bwd_final(float* __restrict__ gb,
                                                               const double* __restrict__ psum,
                                                               const int* __restrict__ pcnt,
                                                               int64_t cols, int splits) {
  __shared__ double ss[256];
  __shared__ int64_t sn[256];
  const int c = threadIdx.x & 31, k = threadIdx.x >> 5;
  const int64_t col = blockIdx.x * 32ll + c;
  double s = 0;
  int64_t n = 0;
  if (col < cols)
    for (int q = k; q < splits; q += 8) {
      s += psum[q * cols + col];
      n += pcnt[q * cols + col];
    }
  ss[threadIdx.x] = s;
  sn[threadIdx.x] = n;
  __syncthreads();
  for (int h = 4; h > 0; h >>= 1) {
    if (k < h) {
      ss[threadIdx.x] += ss[threadIdx.x + 32 * h];
      sn[threadIdx.x] += sn[threadIdx.x + 32 * h];
    }
    __syncthreads();
  }
  // GradStore: count (add pullback) first, then f32(sum mask*a) (mul pullback)
  if (k == 0 && col < cols) gb[col] = __fadd_rn((float)sn[c], __double2float_rn(ss[c]));
}


// Cluster form of the fused backward (the reduce.cu k_cols scheme): a CTA
// owns a strip of 4*CL columns and one of CS row splits; its RL = 256/CL row
// lanes fold through shared memory in lane order, and the CS CTAs of the
// cluster (the row splits of one strip) fold through distributed shared
// memory in rank order -- b-bar is written by cluster rank 0, with no
// partials pass through HBM and no second launch. Deterministic.
template <int CL>
__global__ void __launch_bounds__(kThreads) k_muladd_relu_bwd_cl(float* __restrict__ ga,
                                                                 float* __restrict__ gb,
                                                                 const float* __restrict__ a,
                                                                 const float* __restrict__ b,
                                                                 int64_t rows, int64_t cols,
                                                                 int64_t rows_per_split) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int RL = kThreads / CL, W = 4 * CL;  // W columns per strip
  __shared__ double sh_s[RL][W];
  __shared__ int sh_n[RL][W];
  __shared__ double cs_s[W];
  __shared__ int cs_n[W];
  const int cl = threadIdx.x % CL, rl = threadIdx.x / CL;
  const int64_t col = (blockIdx.x * (int64_t)CL + cl) * 4;
  const int64_t r0 = blockIdx.y * rows_per_split;
  const int64_t r1 = min(rows, r0 + rows_per_split);
  const bool live = col < cols;
  const float4 vb = live ? *reinterpret_cast<const float4*>(b + col) : make_float4(0, 0, 0, 0);
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int n0 = 0, n1 = 0, n2 = 0, n3 = 0;
  auto one = [&](const float4& va, float4* dst) {
    const float m0 = __fadd_rn(__fmul_rn(va.x, vb.x), vb.x) > 0.f ? 1.f : 0.f;
    const float m1 = __fadd_rn(__fmul_rn(va.y, vb.y), vb.y) > 0.f ? 1.f : 0.f;
    const float m2 = __fadd_rn(__fmul_rn(va.z, vb.z), vb.z) > 0.f ? 1.f : 0.f;
    const float m3 = __fadd_rn(__fmul_rn(va.w, vb.w), vb.w) > 0.f ? 1.f : 0.f;
    *dst = make_float4(__fmul_rn(m0, vb.x), __fmul_rn(m1, vb.y), __fmul_rn(m2, vb.z),
                       __fmul_rn(m3, vb.w));
    s0 += (double)__fmul_rn(m0, va.x);
    s1 += (double)__fmul_rn(m1, va.y);
    s2 += (double)__fmul_rn(m2, va.z);
    s3 += (double)__fmul_rn(m3, va.w);
    n0 += m0 > 0.f;
    n1 += m1 > 0.f;
    n2 += m2 > 0.f;
    n3 += m3 > 0.f;
  };
  if (live) {
    int64_t r = r0 + rl;
    for (; r + 7 * RL < r1; r += 8 * RL) {  // 8 independent 128-bit loads in flight
      float4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldg(reinterpret_cast<const float4*>(a + (r + k * RL) * cols + col));
#pragma unroll
      for (int k = 0; k < 8; ++k) one(v[k], reinterpret_cast<float4*>(ga + (r + k * RL) * cols + col));
    }
    for (; r < r1; r += RL)
      one(__ldg(reinterpret_cast<const float4*>(a + r * cols + col)),
          reinterpret_cast<float4*>(ga + r * cols + col));
  }
  sh_s[rl][cl * 4 + 0] = s0; sh_s[rl][cl * 4 + 1] = s1; sh_s[rl][cl * 4 + 2] = s2; sh_s[rl][cl * 4 + 3] = s3;
  sh_n[rl][cl * 4 + 0] = n0; sh_n[rl][cl * 4 + 1] = n1; sh_n[rl][cl * 4 + 2] = n2; sh_n[rl][cl * 4 + 3] = n3;
  __syncthreads();
  if (threadIdx.x < W) {  // row lanes in order
    double t = sh_s[0][threadIdx.x];
    int n = sh_n[0][threadIdx.x];
    for (int k = 1; k < RL; ++k) {
      t += sh_s[k][threadIdx.x];
      n += sh_n[k][threadIdx.x];
    }
    cs_s[threadIdx.x] = t;
    cs_n[threadIdx.x] = n;
  }
  cluster.sync();
  if (blockIdx.y % cluster.dim_blocks().y == 0 && threadIdx.x < W) {  // rank 0: splits in rank order
    const unsigned cs = cluster.dim_blocks().y;
    double t = cs_s[threadIdx.x];
    int64_t n = cs_n[threadIdx.x];
    for (unsigned q = 1; q < cs; ++q) {
      t += cluster.map_shared_rank(cs_s, q)[threadIdx.x];
      n += cluster.map_shared_rank(cs_n, q)[threadIdx.x];
    }
    const int64_t c = blockIdx.x * (int64_t)W + threadIdx.x;
    // GradStore: count (add pullback) first, then f32(sum mask*a) (mul pullback)
    if (c < cols) gb[c] = __fadd_rn((float)n, __double2float_rn(t));
  }
  cluster.sync();  // keep each CTA's shared memory alive until rank 0 has read it
}

}  // namespace

extern "C" {

int b2_fill_f32(float* dst, float v, int64_t n, void* stream) {
  if (n <= 0) return 0;
  Nd nd;
  nd.ndim = 1;
  nd.shape[0] = n;
  nd.st[0][0] = 1;
  nd.st[1][0] = 1;
  return launch_unary(dst, nd, dst, Fill{v}, b2::resolve(stream));
}

int b2_binary(int op, float* out, int ndim, const int64_t* shape, const float* a,
              const int64_t* as, const float* b, const int64_t* bs, void* stream) {
  B2_TRY(check_nd(ndim, shape));
  int64_t os[B2_MAX_DIMS];
  contig_strides(ndim, shape, os);
  const int64_t* sts[3] = {os, as, bs};
  Nd nd = collapse(ndim, shape, 3, sts);
  cudaStream_t st = b2::resolve(stream);
  switch (op) {
    case B2_ADD: return launch_binary(out, nd, a, b, Bin<B2_ADD>{}, st);
    case B2_SUB: return launch_binary(out, nd, a, b, Bin<B2_SUB>{}, st);
    case B2_MUL: return launch_binary(out, nd, a, b, Bin<B2_MUL>{}, st);
    case B2_DIV: return launch_binary(out, nd, a, b, Bin<B2_DIV>{}, st);
    case B2_RELU_BWD: return launch_binary(out, nd, a, b, Bin<B2_RELU_BWD>{}, st);
    case B2_SIGN_MUL: return launch_binary(out, nd, a, b, Bin<B2_SIGN_MUL>{}, st);
    case B2_SIGMOID_BWD: return launch_binary(out, nd, a, b, Bin<B2_SIGMOID_BWD>{}, st);
    case B2_TANH_BWD: return launch_binary(out, nd, a, b, Bin<B2_TANH_BWD>{}, st);
    case B2_GELU_BWD: return launch_binary(out, nd, a, b, Bin<B2_GELU_BWD>{}, st);
  }
  return b2::fail("b2_binary: unknown op");
}

int b2_binary_scalar(int op, float* out, int ndim, const int64_t* shape, const float* x,
                     const int64_t* xs, float s, int scalar_left, void* stream) {
  B2_TRY(check_nd(ndim, shape));
  int64_t os[B2_MAX_DIMS];
  contig_strides(ndim, shape, os);
  const int64_t* sts[2] = {os, xs};
  Nd nd = collapse(ndim, shape, 2, sts);
  cudaStream_t st = b2::resolve(stream);
#define B2_BS(OPC)                                                                     \
  case OPC:                                                                            \
    return scalar_left ? launch_unary(out, nd, x, BinScalar<OPC, true>{s}, st)        \
                       : launch_unary(out, nd, x, BinScalar<OPC, false>{s}, st);
  switch (op) {
    B2_BS(B2_ADD)
    B2_BS(B2_SUB)
    B2_BS(B2_MUL)
    B2_BS(B2_DIV)
    B2_BS(B2_RELU_BWD)
  }
#undef B2_BS
  return b2::fail("b2_binary_scalar: unknown op");
}

int b2_unary(int op, float* out, int ndim, const int64_t* shape, const float* x,
             const int64_t* xs, double alpha, double beta, void* stream) {
  B2_TRY(check_nd(ndim, shape));
  int64_t os[B2_MAX_DIMS];
  contig_strides(ndim, shape, os);
  const int64_t* sts[2] = {os, xs};
  Nd nd = collapse(ndim, shape, 2, sts);
  cudaStream_t st = b2::resolve(stream);
  switch (op) {
    case B2_NEG: return launch_unary(out, nd, x, Un<B2_NEG>{alpha, beta}, st);
    case B2_EXP: return launch_unary(out, nd, x, Un<B2_EXP>{alpha, beta}, st);
    case B2_LOG: return launch_unary(out, nd, x, Un<B2_LOG>{alpha, beta}, st);
    case B2_SQRT: return launch_unary(out, nd, x, Un<B2_SQRT>{alpha, beta}, st);
    case B2_ABS: return launch_unary(out, nd, x, Un<B2_ABS>{alpha, beta}, st);
    case B2_RELU: return launch_unary(out, nd, x, Un<B2_RELU>{alpha, beta}, st);
    case B2_RELU_MASK: return launch_unary(out, nd, x, Un<B2_RELU_MASK>{alpha, beta}, st);
    case B2_COPY: return launch_unary(out, nd, x, Un<B2_COPY>{alpha, beta}, st);
    case B2_CLAMP: return launch_unary(out, nd, x, Un<B2_CLAMP>{alpha, beta}, st);
    case B2_SCALE: return launch_unary(out, nd, x, Un<B2_SCALE>{alpha, beta}, st);
    case B2_DIV_SCALAR: return launch_unary(out, nd, x, Un<B2_DIV_SCALAR>{alpha, beta}, st);
    case B2_CLAMP_MASK: return launch_unary(out, nd, x, Un<B2_CLAMP_MASK>{alpha, beta}, st);
    case B2_SIGMOID: return launch_unary(out, nd, x, Un<B2_SIGMOID>{alpha, beta}, st);
    case B2_TANH: return launch_unary(out, nd, x, Un<B2_TANH>{alpha, beta}, st);
    case B2_GELU: return launch_unary(out, nd, x, Un<B2_GELU>{alpha, beta}, st);
  }
  return b2::fail("b2_unary: unknown op");
}

int b2_copy_strided(float* out, int ndim, const int64_t* shape, const float* x,
                    const int64_t* xs, void* stream) {
  return b2_unary(B2_COPY, out, ndim, shape, x, xs, 0.0, 0.0, stream);
}

int b2_write_strided(float* dst, int ndim, const int64_t* shape, const int64_t* ds,
                     const float* src, void* stream) {
  B2_TRY(check_nd(ndim, shape));
  int64_t ss[B2_MAX_DIMS];
  contig_strides(ndim, shape, ss);
  const int64_t* sts[2] = {ds, ss};
  Nd nd = collapse(ndim, shape, 2, sts);
  int64_t n = numel(ndim, shape);
  if (n == 0) return 0;
  RowGeom g = make_rows(nd, 2);
  dim3 grid;
  int64_t chunk;
  rows_grid(g, &grid, &chunk);
  k_un_rows<Un<B2_COPY>, false><<<grid, kThreads, 0, b2::resolve(stream)>>>(dst, src, g, chunk,
                                                                              Un<B2_COPY>{0, 0});
  return b2::launched("b2_write_strided");
}

int b2_fused_muladd_relu_fwd(float* y, const float* a, const float* b, const float* c,
                             int64_t rows, int64_t cols, void* stream) {
  if (rows * cols == 0) return 0;
  if (cols % 4 || !aligned16(a) || !aligned16(b) || !aligned16(c) || !aligned16(y))
    return b2::fail("b2_fused_muladd_relu_fwd: needs cols%4==0 and 16-B aligned rows");
  int grid = (int)std::min<int64_t>(rows, b2::sm_count() * 8);
  k_muladd_relu_fwd<<<grid, kThreads, 0, b2::resolve(stream)>>>(y, a, b, c, rows, cols);
  return b2::launched("b2_fused_muladd_relu_fwd");
}

int b2_fused_muladd_relu_bwd(float* ga, float* gb, const float* a, const float* b,
                             int64_t rows, int64_t cols, void* stream) {
  if (cols == 0) return 0;
  if (cols % 4 || !aligned16(a) || !aligned16(b) || !aligned16(ga))
    return b2::fail("b2_fused_muladd_relu_bwd: needs cols%4==0 and 16-B aligned rows");
  cudaStream_t st = b2::resolve(stream);
  {
    // cluster path: strips x CS row splits folded through DSMEM (one launch)
    constexpr int CL = B2_MULADD_CL_CLUSTER, RL = kThreads / CL;
    const int64_t strips = (cols + 4 * CL - 1) / (4 * CL);
    const int64_t target = 3LL * b2::sm_count();
    int cs = 1;
    while (cs < 8 && strips * cs < target && rows >= (int64_t)(cs * 2) * RL * 8) cs *= 2;
    if (strips * cs >= 2LL * b2::sm_count() && strips <= INT32_MAX) {
      const int64_t rps = (rows + cs - 1) / cs;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)strips, (unsigned)cs, 1);
      cfg.blockDim = dim3(kThreads, 1, 1);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 1;
      attr[0].val.clusterDim.y = cs;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_muladd_relu_bwd_cl<CL>, ga, gb, a, b, rows, cols, rps);
      if (e != cudaSuccess) return b2::cuda_fail(e, "b2_fused_muladd_relu_bwd(cluster)");
      return b2::launched("b2_fused_muladd_relu_bwd(cluster)");
    }
  }
  int64_t colblocks = (cols + 4 * kMuladdCL - 1) / (4 * kMuladdCL);  // strips of 4*CL columns
  static int occ = 0;  // resident CTAs per SM: the splits fill exactly one wave
  if (!occ && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_muladd_relu_bwd, kThreads, 0) !=
                   cudaSuccess || occ < 1))
    occ = 1;
  int64_t splits = std::max<int64_t>(1, ((int64_t)b2::sm_count() * occ) / colblocks);
  splits = std::min<int64_t>(splits, std::max<int64_t>(rows / 64, 1));
  int64_t rps = (rows + splits - 1) / splits;
  if (rps == 0) rps = 1;
  splits = std::max<int64_t>(1, (rows + rps - 1) / rps);
  void* ws = nullptr;
  size_t bytes = (size_t)splits * cols * (sizeof(double) + sizeof(int));
  B2_TRY(b2_alloc(bytes, stream, &ws));
  double* psum = (double*)ws;
  int* pcnt = (int*)(psum + splits * cols);
  dim3 grid((unsigned)colblocks, (unsigned)splits);
  k_muladd_relu_bwd<<<grid, kThreads, 0, st>>>(ga, psum, pcnt, a, b, rows, cols, rps);
  int rc = b2::launched("b2_fused_muladd_relu_bwd");
  if (!rc) {
    k_muladd_relu_bwd_final<<<(unsigned)((cols + 31) / 32), 256, 0, st>>>(gb, psum, pcnt, cols,
                                                                         (int)splits);
    rc = b2::launched("b2_fused_muladd_relu_bwd_final");
  }
  b2_free(ws, stream);
  return rc;
}

}  // extern "C"
