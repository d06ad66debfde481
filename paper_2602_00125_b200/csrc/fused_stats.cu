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
// Stage 1 (k_c2_pass): a CTA owns a block of rows x 128 columns (3 CTAs of
// 8 warps per SM, one wave); each warp walks rows w, w+8, ... with 4 columns
// per lane, its rows streamed through a shared-memory ring by cp.async.bulk; a row's strip partial (fp64
// sum, max) is a warp butterfly, written to [strip][row]; column partials stay
// in registers across the warp's rows and fold over the 8 warps in order
// through shared memory to [row block][column]. Stage 2 (k_c2_fold) folds row
// partials over strips and column partials over row blocks in order; stage 3
// (k_c2_total) sums the fp64 row sums for the full sum. Deterministic: the
// partition depends only on the shape.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "fexp.cuh"

extern "C" int b2_alloc(size_t, void*, void**);
extern "C" int b2_free(void*, void*);

namespace {

#ifndef B2_C2_MINB
#define B2_C2_MINB 3
#endif
#ifndef B2_C2_CPL
#define B2_C2_CPL 4
#endif
constexpr int kCPL = B2_C2_CPL;        // columns per lane (4 or 8)
constexpr int kSW = 32 * kCPL;         // columns per CTA strip
#ifndef B2_C2_STAGES
#define B2_C2_STAGES 4
#endif
constexpr int kC2Stages = B2_C2_STAGES;  // 1-KB row segments in flight per warp
// rows per CTA block: chosen on the host so strips x row blocks fills one wave
// of 2 resident CTAs per SM (a partial second wave left ~30% of the SMs idle)

struct C2Part {
  double* rsum;  // [strips][R]
  float* rmax;   // [strips][R]
  double* csum;  // [rblocks][C]
  float* cmax;
  double* cma;   // sum of mask*a
  int* ccnt;     // count of mask
};

__global__ void __launch_bounds__(256, kCPL == 4 ? B2_C2_MINB : 2) k_c2_pass(const float* __restrict__ a, const float* __restrict__ b,
                                                 float lo, float hi, float* __restrict__ y,
                                                 float* __restrict__ e, float* __restrict__ ga,
                                                 C2Part p, int64_t R, int64_t C, int64_t kRB) {
  // dynamic shared memory: the row ring during the sweep, then (overlaid)
  // the 8 warps' column partials for the ordered fold
  extern __shared__ __align__(128) unsigned char c2_smem[];
  double(*sh_s)[kSW] = reinterpret_cast<double(*)[kSW]>(c2_smem);
  double(*sh_a)[kSW] = sh_s + 8;
  float(*sh_m)[kSW] = reinterpret_cast<float(*)[kSW]>(sh_a + 8);
  int(*sh_n)[kSW] = reinterpret_cast<int(*)[kSW]>(sh_m + 8);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int strip = blockIdx.x, rb = blockIdx.y;
  const int64_t c0 = (int64_t)strip * kSW + lane * kCPL;  // this lane's columns
  const bool in0 = c0 < C, in1 = kCPL == 8 && c0 + 4 < C;  // C % 4 == 0 (host)
  float bv[kCPL];
  {
    const float4 b0 = in0 ? *reinterpret_cast<const float4*>(b + c0) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 b1 = in1 ? *reinterpret_cast<const float4*>(b + c0 + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
    bv[0] = b0.x; bv[1] = b0.y; bv[2] = b0.z; bv[3] = b0.w;
    if (kCPL == 8) {
      bv[4 % kCPL] = b1.x; bv[5 % kCPL] = b1.y; bv[6 % kCPL] = b1.z; bv[7 % kCPL] = b1.w;
    }
  }
  double cs[kCPL], ca[kCPL];
  float cm[kCPL];
  int cn[kCPL];
#pragma unroll
  for (int k = 0; k < kCPL; ++k) {
    cs[k] = 0.0;
    ca[k] = 0.0;
    cm[k] = -INFINITY;
    cn[k] = 0;
  }
  const int64_t r0 = (int64_t)rb * kRB, r1 = min(R, r0 + kRB);
  // The warp's rows (r0 + w, r0 + w + 8, ...) stream through a kC2Stages-deep
  // shared-memory ring of 1-KB strip segments filled by cp.async.bulk (lane 0
  // issues, an mbarrier per stage carries the byte count): ~64 KB of a in
  // flight per SM without holding prefetched rows in registers.
  constexpr int kStages = kC2Stages;
  float(*ring)[kStages][kSW] = reinterpret_cast<float(*)[kStages][kSW]>(c2_smem);
  __shared__ __align__(8) uint64_t bars[8][kStages];
  const uint32_t seg_bytes = (uint32_t)(min((int64_t)kSW, C - (int64_t)strip * kSW) * 4);
  const float* abase = a + (int64_t)strip * kSW;
  auto issue = [&](int stg, int64_t r) {
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[w][stg]);
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&ring[w][stg][0]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(seg_bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(abase + r * C), "r"(seg_bytes), "r"(bar) : "memory");
  };
  if (lane == 0) {
    for (int k = 0; k < kStages; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[w][k])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 0; k < kStages; ++k)
      if (r0 + w + 8 * k < r1) issue(k, r0 + w + 8 * k);
  }
  __syncwarp();
  int it = 0;
  for (int64_t r = r0 + w; r < r1; r += 8, ++it) {
    const int stg = it % kStages;
    {
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[w][stg]);
      const uint32_t par = (uint32_t)(it / kStages) & 1;
      asm volatile("{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                   "@!P1 bra WAIT_%=;\n}\n" ::"r"(bar), "r"(par) : "memory");
    }
    float av[kCPL];
    {
      const float* seg = &ring[w][stg][lane * kCPL];
      const float4 a0 = in0 ? *reinterpret_cast<const float4*>(seg) : make_float4(0.f, 0.f, 0.f, 0.f);
      av[0] = a0.x; av[1] = a0.y; av[2] = a0.z; av[3] = a0.w;
      if (kCPL == 8) {
        const float4 a1 = in1 ? *reinterpret_cast<const float4*>(seg + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
        av[4 % kCPL] = a1.x; av[5 % kCPL] = a1.y; av[6 % kCPL] = a1.z; av[7 % kCPL] = a1.w;
      }
    }
    __syncwarp();  // every lane has read the stage: refill it with the row kStages ahead
    if (lane == 0 && r + 8 * kStages < r1) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(stg, r + 8 * kStages);
    }
    float yv[kCPL], ev[kCPL], gv[kCPL];
    double rs = 0.0;
    float rm = -INFINITY;
#pragma unroll
    for (int k = 0; k < kCPL; ++k) {
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
      if (in1) *reinterpret_cast<float4*>(y + o + 4) = make_float4(yv[4 % kCPL], yv[5 % kCPL], yv[6 % kCPL], yv[7 % kCPL]);
    }
    if (e) {
      if (in0) *reinterpret_cast<float4*>(e + o) = make_float4(ev[0], ev[1], ev[2], ev[3]);
      if (in1) *reinterpret_cast<float4*>(e + o + 4) = make_float4(ev[4 % kCPL], ev[5 % kCPL], ev[6 % kCPL], ev[7 % kCPL]);
    }
    if (ga) {
      if (in0) *reinterpret_cast<float4*>(ga + o) = make_float4(gv[0], gv[1], gv[2], gv[3]);
      if (in1) *reinterpret_cast<float4*>(ga + o + 4) = make_float4(gv[4 % kCPL], gv[5 % kCPL], gv[6 % kCPL], gv[7 % kCPL]);
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
  __syncthreads();  // every warp is done with the ring before the partials overlay it
#pragma unroll
  for (int k = 0; k < kCPL; ++k) {
    sh_s[w][lane * kCPL + k] = cs[k];
    sh_a[w][lane * kCPL + k] = ca[k];
    sh_m[w][lane * kCPL + k] = cm[k];
    sh_n[w][lane * kCPL + k] = cn[k];
  }
  __syncthreads();
  const int j = threadIdx.x;  // one column of the strip per thread, warps folded in order
  const int64_t c = (int64_t)strip * kSW + j;
  if (j < kSW && c < C) {
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

// Stage 2: 32 outputs x 8 lanes per CTA (lane k folds partial rows k, k+8,
// ... in order), then a fixed tree over the 8 lanes -- deterministic. CTAs
// [0, ceil(R/32)) fold the row partials, the rest the column partials.
__global__ void __launch_bounds__(256) k_c2_fold(C2Part p, C2Out o, int strips, int rblocks, int64_t R,
                                                 int64_t C) {
  __shared__ double s1[8][33], s2[8][33];
  __shared__ float sm[8][33];
  __shared__ int64_t sn[8][33];
  const int c = threadIdx.x & 31, k = threadIdx.x >> 5;
  const int64_t rowc = (R + 31) / 32;
  const bool rows_part = blockIdx.x < rowc;
  const int64_t i = (rows_part ? blockIdx.x : blockIdx.x - rowc) * 32 + c;
  double a1 = 0.0, a2 = 0.0;
  float m = -INFINITY;
  int64_t n = 0;
  if (rows_part && i < R) {
    for (int q = k; q < strips; q += 8) {
      a1 += p.rsum[(int64_t)q * R + i];
      m = fmaxf(m, p.rmax[(int64_t)q * R + i]);
    }
  } else if (!rows_part && i < C) {
    for (int q = k; q < rblocks; q += 8) {
      const int64_t x = (int64_t)q * C + i;
      a1 += p.csum[x];
      a2 += p.cma[x];
      m = fmaxf(m, p.cmax[x]);
      n += p.ccnt[x];
    }
  }
  s1[k][c] = a1;
  s2[k][c] = a2;
  sm[k][c] = m;
  sn[k][c] = n;
  __syncthreads();
  if (k != 0) return;
  for (int h = 1; h < 8; ++h) {
    a1 += s1[h][c];
    a2 += s2[h][c];
    m = fmaxf(m, sm[h][c]);
    n += sn[h][c];
  }
  if (rows_part) {
    if (i >= R) return;
    o.rsum64[i] = a1;
    if (o.sum1) o.sum1[i] = __double2float_rn(a1);
    if (o.mean1) o.mean1[i] = __double2float_rn(a1 / (double)C);
    if (o.max1) o.max1[i] = m;
  } else {
    if (i >= C) return;
    if (o.sum0) o.sum0[i] = __double2float_rn(a1);
    if (o.mean0) o.mean0[i] = __double2float_rn(a1 / (double)R);
    if (o.max0) o.max0[i] = m;
    // GradStore: the add pullback's count first, then f32(sum mask*a) (mul pullback)
    if (o.gb) o.gb[i] = __fadd_rn((float)n, __double2float_rn(a2));
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
  const int64_t slots = (kCPL == 4 ? (int64_t)B2_C2_MINB : 2LL) * b2::sm_count();
  const int64_t want_rb = std::max<int64_t>(1, slots / strips);
  int64_t kRB = std::max<int64_t>(8, (rows + want_rb - 1) / want_rb);
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
  constexpr int smem = std::max(8 * kSW * (8 + 8 + 4 + 4), 8 * kC2Stages * kSW * 4);  // fold area / row ring
  static bool attr = false;
  if (!attr) {
    B2_CUDA(cudaFuncSetAttribute(k_c2_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  if (((uintptr_t)a & 15) || (cols * 4) % 16) return b2::fail("b2_muladd_relu_stats: rows must be 16-B aligned");
  k_c2_pass<<<dim3((unsigned)strips, (unsigned)rblocks), 256, smem, st>>>(a, b, clamp_lo, clamp_hi, y, e, ga,
                                                                          p, rows, cols, kRB);
  int rc = b2::launched("b2_muladd_relu_stats(pass)");
  if (!rc) {
    C2Out o{sum0, mean0, max0, sum1, mean1, max1, gb, rsum64};
    const int64_t ctas = (rows + 31) / 32 + (cols + 31) / 32;
    k_c2_fold<<<(unsigned)ctas, 256, 0, st>>>(p, o, strips, rblocks, rows, cols);
    rc = b2::launched("b2_muladd_relu_stats(fold)");
  }
  if (!rc && total) {
    k_c2_total<<<1, 1024, 0, st>>>(total, rsum64, rows);
    rc = b2::launched("b2_muladd_relu_stats(total)");
  }
  b2_free(ws, st);
  return rc;
}
