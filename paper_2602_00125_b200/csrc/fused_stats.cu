// BASELINE config 2 as ONE pass over its input (multi-output fusion).
//
// The config's workload -- y = relu(a*b + b), e = exp(clamp(a, lo, hi)),
// sum/mean/max of y over dim 0 and dim 1, the full sum of y, and the
// gradients of sum(y) w.r.t. a and b -- composed from engine ops reads `a`
// nine times (~1 GB of traffic for a 64 MiB input). Its compulsory traffic is
// one read of a and the writes of y, e and a_bar (256 MiB at 4096^2). This
// kernel reads each element once and produces every output, with the
// arithmetic of the separate ops (bit-identical):
//   y     = relu(__fadd_rn(__fmul_rn(a, b), b))        core.py:453-483, nn.py:108-111
//   e     = f32(exp(double(clamp(a, lo, hi))))          b2_unary CLAMP (NaN passes) then EXP
//   a_bar = __fmul_rn(mask, b)                         mul pullback of the relu mask
//   b_bar = __fadd_rn(f32(count(mask)), f32(sum64 __fmul_rn(mask, a)))  GradStore order
//   sums / means in fp64 with one f32 rounding, max as the value (y >= +0, no NaN)
// Stage 1 (k_c2_pass): a CTA owns a 128-row x 256-column block; each warp
// walks rows w, w+8, ... with 8 columns per lane; a row's strip partial (fp64
// sum, max) is a warp butterfly, written to [strip][row]; column partials stay
// in registers across the warp's rows and fold over the 8 warps in order
// through shared memory to [row block][column]. Stage 2 (k_c2_fold) folds row
// partials over strips and column partials over row blocks in order; stage 3
// (k_c2_total) sums the fp64 row sums for the full sum. Deterministic: the
// partition depends only on the shape.
#include <cuda_runtime.h>

#include "common.cuh"
#include "fexp.cuh"

extern "C" int b2_alloc(size_t, void*, void**);
extern "C" int b2_free(void*, void*);

namespace {

constexpr int kSW = 256;  // columns per CTA strip (32 lanes x 8)
constexpr int kRB = 128;  // rows per CTA block

struct C2Part {
  double* rsum;  // [strips][R]
  float* rmax;   // [strips][R]
  double* csum;  // [rblocks][C]
  float* cmax;
  double* cma;   // sum of mask*a
  int* ccnt;     // count of mask
};

__global__ void __launch_bounds__(256) k_c2_pass(const float* __restrict__ a, const float* __restrict__ b,
                                                 float lo, float hi, float* __restrict__ y,
                                                 float* __restrict__ e, float* __restrict__ ga,
                                                 C2Part p, int64_t R, int64_t C) {
  __shared__ double sh_s[8][kSW];
  __shared__ double sh_a[8][kSW];
  __shared__ float sh_m[8][kSW];
  __shared__ int sh_n[8][kSW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int strip = blockIdx.x, rb = blockIdx.y;
  const int64_t c0 = (int64_t)strip * kSW + lane * 8;  // this lane's 8 columns
  const bool in0 = c0 < C, in1 = c0 + 4 < C;           // C % 4 == 0 (host)
  float bv[8];
  {
    const float4 b0 = in0 ? *reinterpret_cast<const float4*>(b + c0) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 b1 = in1 ? *reinterpret_cast<const float4*>(b + c0 + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
    bv[0] = b0.x; bv[1] = b0.y; bv[2] = b0.z; bv[3] = b0.w;
    bv[4] = b1.x; bv[5] = b1.y; bv[6] = b1.z; bv[7] = b1.w;
  }
  double cs[8], ca[8];
  float cm[8];
  int cn[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    cs[k] = 0.0;
    ca[k] = 0.0;
    cm[k] = -INFINITY;
    cn[k] = 0;
  }
  const int64_t r0 = (int64_t)rb * kRB, r1 = min(R, r0 + kRB);
  // the next row's loads are issued before this row is processed (two rows
  // of a in flight per warp)
  auto load = [&](int64_t r, float4& a0, float4& a1) {
    const float* ar = a + r * C + c0;
    a0 = (in0 && r < r1) ? __ldg(reinterpret_cast<const float4*>(ar)) : make_float4(0.f, 0.f, 0.f, 0.f);
    a1 = (in1 && r < r1) ? __ldg(reinterpret_cast<const float4*>(ar + 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  float4 n0, n1;
  load(r0 + w, n0, n1);
  for (int64_t r = r0 + w; r < r1; r += 8) {
    float av[8];
    av[0] = n0.x; av[1] = n0.y; av[2] = n0.z; av[3] = n0.w;
    av[4] = n1.x; av[5] = n1.y; av[6] = n1.z; av[7] = n1.w;
    load(r + 8, n0, n1);
    float yv[8], ev[8], gv[8];
    double rs = 0.0;
    float rm = -INFINITY;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool live = k < 4 ? in0 : in1;
      const float q = __fadd_rn(__fmul_rn(av[k], bv[k]), bv[k]);
      const float mf = q > 0.f ? 1.f : 0.f;
      yv[k] = q > 0.f ? q : 0.f;
      gv[k] = __fmul_rn(mf, bv[k]);
      ev[k] = b2::exp_f32(av[k] != av[k] ? av[k] : fminf(fmaxf(av[k], lo), hi));  // clamp keeps NaN
      if (live) {
        rs += (double)yv[k];
        rm = fmaxf(rm, yv[k]);
        cs[k] += (double)yv[k];
        cm[k] = fmaxf(cm[k], yv[k]);
        ca[k] += (double)__fmul_rn(mf, av[k]);
        cn[k] += q > 0.f;
      }
    }
    const int64_t o = r * C + c0;
    if (y) {
      if (in0) *reinterpret_cast<float4*>(y + o) = make_float4(yv[0], yv[1], yv[2], yv[3]);
      if (in1) *reinterpret_cast<float4*>(y + o + 4) = make_float4(yv[4], yv[5], yv[6], yv[7]);
    }
    if (e) {
      if (in0) *reinterpret_cast<float4*>(e + o) = make_float4(ev[0], ev[1], ev[2], ev[3]);
      if (in1) *reinterpret_cast<float4*>(e + o + 4) = make_float4(ev[4], ev[5], ev[6], ev[7]);
    }
    if (ga) {
      if (in0) *reinterpret_cast<float4*>(ga + o) = make_float4(gv[0], gv[1], gv[2], gv[3]);
      if (in1) *reinterpret_cast<float4*>(ga + o + 4) = make_float4(gv[4], gv[5], gv[6], gv[7]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      rs += __shfl_xor_sync(0xffffffffu, rs, off);
      rm = fmaxf(rm, __shfl_xor_sync(0xffffffffu, rm, off));
    }
    if (lane == 0) {
      p.rsum[(int64_t)strip * R + r] = rs;
      p.rmax[(int64_t)strip * R + r] = rm;
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    sh_s[w][lane * 8 + k] = cs[k];
    sh_a[w][lane * 8 + k] = ca[k];
    sh_m[w][lane * 8 + k] = cm[k];
    sh_n[w][lane * 8 + k] = cn[k];
  }
  __syncthreads();
  const int j = threadIdx.x;  // one column of the strip per thread, warps folded in order
  const int64_t c = (int64_t)strip * kSW + j;
  if (c < C) {
    double s = sh_s[0][j], sa = sh_a[0][j];
    float m = sh_m[0][j];
    int n = sh_n[0][j];
#pragma unroll
    for (int ww = 1; ww < 8; ++ww) {
      s += sh_s[ww][j];
      sa += sh_a[ww][j];
      m = fmaxf(m, sh_m[ww][j]);
      n += sh_n[ww][j];
    }
    const int64_t q = (int64_t)rb * C + c;
    p.csum[q] = s;
    p.cma[q] = sa;
    p.cmax[q] = m;
    p.ccnt[q] = n;
  }
}

struct C2Out {
  float *sum0, *mean0, *max0;  // [C] over dim 0
  float *sum1, *mean1, *max1;  // [R] over dim 1
  float* gb;                   // [C]
  double* rsum64;              // [R] scratch for the total
};

__global__ void __launch_bounds__(256) k_c2_fold(C2Part p, C2Out o, int strips, int rblocks, int64_t R,
                                                 int64_t C) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < R) {
    double s = 0.0;
    float m = -INFINITY;
    for (int q = 0; q < strips; ++q) {
      s += p.rsum[(int64_t)q * R + i];
      m = fmaxf(m, p.rmax[(int64_t)q * R + i]);
    }
    o.rsum64[i] = s;
    if (o.sum1) o.sum1[i] = __double2float_rn(s);
    if (o.mean1) o.mean1[i] = __double2float_rn(s / (double)C);
    if (o.max1) o.max1[i] = m;
  }
  if (i < C) {
    double s = 0.0, sa = 0.0;
    float m = -INFINITY;
    int64_t n = 0;
    for (int q = 0; q < rblocks; ++q) {
      const int64_t k = (int64_t)q * C + i;
      s += p.csum[k];
      sa += p.cma[k];
      m = fmaxf(m, p.cmax[k]);
      n += p.ccnt[k];
    }
    if (o.sum0) o.sum0[i] = __double2float_rn(s);
    if (o.mean0) o.mean0[i] = __double2float_rn(s / (double)R);
    if (o.max0) o.max0[i] = m;
    // GradStore: the add pullback's count first, then f32(sum mask*a) (mul pullback)
    if (o.gb) o.gb[i] = __fadd_rn((float)n, __double2float_rn(sa));
  }
}

__global__ void __launch_bounds__(1024) k_c2_total(float* __restrict__ total, const double* __restrict__ rsum,
                                                   int64_t R) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t r = threadIdx.x; r < R; r += blockDim.x) s += rsum[r];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = s;
  __syncthreads();
  if (w == 0) {
    double t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (lane == 0) *total = __double2float_rn(t);
  }
}

}  // namespace

extern "C" int b2_muladd_relu_stats(float* y, float* e, float* ga, float* gb, float* sum0, float* mean0,
                                    float* max0, float* sum1, float* mean1, float* max1, float* total,
                                    const float* a, const float* b, float clamp_lo, float clamp_hi,
                                    int64_t rows, int64_t cols, void* stream) {
  if (rows <= 0 || cols <= 0) return b2::fail("b2_muladd_relu_stats: empty input");
  if (cols % 4 || ((uintptr_t)a & 15) || ((uintptr_t)b & 15) || ((uintptr_t)y & 15) ||
      ((uintptr_t)e & 15) || ((uintptr_t)ga & 15))
    return b2::fail("b2_muladd_relu_stats: needs cols % 4 == 0 and 16-B aligned rows");
  cudaStream_t st = b2::resolve(stream);
  const int strips = (int)((cols + kSW - 1) / kSW);
  const int rblocks = (int)((rows + kRB - 1) / kRB);
  const size_t rn = (size_t)strips * rows, cn = (size_t)rblocks * cols;
  const size_t bytes = rn * (8 + 4) + cn * (8 + 4 + 8 + 4) + (size_t)rows * 8 + 1024;
  void* ws = nullptr;
  B2_TRY(b2_alloc(bytes, st, &ws));
  char* w = (char*)ws;
  C2Part p;
  p.rsum = (double*)w; w += rn * 8;
  p.csum = (double*)w; w += cn * 8;
  p.cma = (double*)w; w += cn * 8;
  double* rsum64 = (double*)w; w += (size_t)rows * 8;
  p.rmax = (float*)w; w += rn * 4;
  p.cmax = (float*)w; w += cn * 4;
  p.ccnt = (int*)w;
  k_c2_pass<<<dim3((unsigned)strips, (unsigned)rblocks), 256, 0, st>>>(a, b, clamp_lo, clamp_hi, y, e, ga, p,
                                                                       rows, cols);
  int rc = b2::launched("b2_muladd_relu_stats(pass)");
  if (!rc) {
    C2Out o{sum0, mean0, max0, sum1, mean1, max1, gb, rsum64};
    const int64_t n = rows > cols ? rows : cols;
    k_c2_fold<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, o, strips, rblocks, rows, cols);
    rc = b2::launched("b2_muladd_relu_stats(fold)");
  }
  if (!rc && total) {
    k_c2_total<<<1, 1024, 0, st>>>(total, rsum64, rows);
    rc = b2::launched("b2_muladd_relu_stats(total)");
  }
  b2_free(ws, st);
  return rc;
}
