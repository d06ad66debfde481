// Reference-arithmetic GEMM (B2_GEMM_REF): the reference's own dot product
// (tensorlite/core.py:802-807, matmul.block): every output is
// `sum(map(mul, xrow, wrow))` over Python floats, rounded once to f32 on store.
// CPython 3.12's builtin sum() of floats is Neumaier-compensated: it carries
// the exact rounding error of every addition in a second double and returns
// s + c. This kernel does the same, in the same left-to-right k order:
//   * fp32 x fp32 products are exact in fp64 (24 + 24 <= 53 bits);
//   * s, c per output: t = s + p; e = TwoSum error of that addition (exact,
//     branch-free; equal to Neumaier's branchy form); c += e; s = t;
//   * out = f32(s + c).
// So a finite output is bit-identical to the reference's, independent of K
// (the NumPy oracle's BLAS f64 GEMM is the one that may differ, by one f32
// ulp where its uncompensated sum straddles a rounding boundary).
//
// This is the parity mode (exact-arithmetic control for the BASELINE config-5
// gradients and updated weights), not a performance path: 8 FP64 ops per MAC,
// 64x64x16 CTA tiles, 256 threads, 4x4 compensated accumulators per thread,
// operands converted to double when staged to shared memory (double-buffered
// through registers).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace {

constexpr int RBM = 64, RBN = 64, RBK = 16;

// BF16IN: the operands are first rounded to bf16 (RN) -- the bf16 variant's
// operand rounding with exact products and compensated sums: the
// exact-arithmetic control for the bf16 variant (B2_GEMM_REF_BF16)
template <bool TA, bool TB, bool BF16IN>
__global__ void __launch_bounds__(256) k_gemm_f64acc(int64_t M, int64_t N, int64_t K,
                                                     const float* __restrict__ A, int64_t lda,
                                                     const float* __restrict__ B, int64_t ldb,
                                                     float* __restrict__ C, int64_t ldc,
                                                     const float* __restrict__ bias, int epi) {
  __shared__ __align__(16) double As[2][RBK][RBM];
  __shared__ __align__(16) double Bs[2][RBK][RBN];
  const int t = threadIdx.x, tx = t % 16, ty = t / 16;
  const int64_t m0 = blockIdx.y * (int64_t)RBM, n0 = blockIdx.x * (int64_t)RBN;
  double acc[4][4], cmp[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = cmp[i][j] = 0.0;
  float ra[4], rb[4];
  // each thread stages 4 elements of each 64x16 operand tile; the fastest
  // index follows the operand's contiguous axis so global reads coalesce
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int64_t m, k;
      if (!TA) { m = m0 + t / 4; k = k0 + (t % 4) * 4 + i; }
      else     { k = k0 + t / 16; m = m0 + (t % 16) * 4 + i; }
      ra[i] = (m < M && k < K) ? (TA ? A[k * lda + m] : A[m * lda + k]) : 0.0f;
      int64_t n, kk;
      if (TB) { n = n0 + t / 4; kk = k0 + (t % 4) * 4 + i; }
      else    { kk = k0 + t / 16; n = n0 + (t % 16) * 4 + i; }
      rb[i] = (n < N && kk < K) ? (TB ? B[n * ldb + kk] : B[kk * ldb + n]) : 0.0f;
    }
  };
  auto store = [&](int buf) {
    if (BF16IN) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ra[i] = __bfloat162float(__float2bfloat16_rn(ra[i]));
        rb[i] = __bfloat162float(__float2bfloat16_rn(rb[i]));
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (!TA) As[buf][(t % 4) * 4 + i][t / 4] = (double)ra[i];
      else     As[buf][t / 16][(t % 16) * 4 + i] = (double)ra[i];
      if (TB)  Bs[buf][(t % 4) * 4 + i][t / 4] = (double)rb[i];
      else     Bs[buf][t / 16][(t % 16) * 4 + i] = (double)rb[i];
    }
  };
  const int nk = (int)((K + RBK - 1) / RBK);
  load(0);
  store(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nk) load((int64_t)(kt + 1) * RBK);
#pragma unroll
    for (int k = 0; k < RBK; ++k) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        av[i] = As[cur][k][ty + 16 * i];  // rows ty, ty+16, ...: conflict-free broadcast
        bv[i] = Bs[cur][k][tx + 16 * i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double p = __dmul_rn(av[i], bv[j]);  // exact
          const double t = __dadd_rn(acc[i][j], p);
          const double z = __dsub_rn(t, acc[i][j]);
          const double e = __dadd_rn(__dsub_rn(acc[i][j], __dsub_rn(t, z)), __dsub_rn(p, z));
          cmp[i][j] = __dadd_rn(cmp[i][j], e);
          acc[i][j] = t;
        }
    }
    if (kt + 1 < nk) {
      store(cur ^ 1);
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx + 16 * j;
      if (n >= N) continue;
      // CPython adds the compensation only when it is nonzero and finite
      const double c = cmp[i][j];
      const double d = (c != 0.0 && isfinite(c)) ? __dadd_rn(acc[i][j], c) : acc[i][j];
      float v = __double2float_rn(d);  // the single f32 rounding (array('f') store)
      // separate f32 bias add and relu, as add(matmul(x, w), b) then relu
      if (epi == B2_EPI_BIAS || epi == B2_EPI_BIAS_RELU) v = __fadd_rn(v, bias[n]);
      if (epi == B2_EPI_BIAS_RELU || epi == B2_EPI_RELU) v = v > 0.0f ? v : 0.0f;
      C[m * ldc + n] = v;
    }
  }
}

}  // namespace

namespace b2 {

int gemm_ref(int ta, int tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
             const float* B, int64_t ldb, float* C, int64_t ldc, const float* bias, int epi,
             cudaStream_t st, bool bf16_operands) {
  if (M == 0 || N == 0) return 0;
  dim3 grid((unsigned)((N + RBN - 1) / RBN), (unsigned)((M + RBM - 1) / RBM));
  if (grid.y > 65535) return fail("b2_gemm(ref): M too large for the reference-arithmetic grid");
#define B2_REF(TA_, TB_)                                                                           \
  if (bf16_operands)                                                                               \
    k_gemm_f64acc<TA_, TB_, true><<<grid, 256, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, bias, epi); \
  else                                                                                             \
    k_gemm_f64acc<TA_, TB_, false><<<grid, 256, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, bias, epi)
  if (!ta && !tb) {
    B2_REF(false, false);
  } else if (!ta && tb) {
    B2_REF(false, true);
  } else if (ta && !tb) {
    B2_REF(true, false);
  } else {
    B2_REF(true, true);
  }
#undef B2_REF
  return launched("b2_gemm(ref)");
}

}  // namespace b2
