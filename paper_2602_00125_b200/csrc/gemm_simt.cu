// FP32 SIMT GEMM (FFMA, fp32 accumulate): the exact-fp32 fallback of the
// matmul engine for shapes the tcgen05 path does not take (tiny problems,
// operands whose leading dimension breaks TMA's 16-byte stride rule).
//
// Replaces matmul.block (tensorlite/core.py:802-807) and its pullbacks
// (core.py:815-817); the three operand layouts of those pullbacks are
// template parameters, so transposed views are read in place, never copied.
// 128x128x8 CTA tile, 256 threads, 8x8 outputs per thread (two 4x4 quads per
// axis to keep shared-memory reads conflict-free), register double buffering.
#include <cuda_runtime.h>

#include "common.cuh"

namespace {

constexpr int BM = 128, BN = 128, BK = 8;

template <bool TA, bool TB>
__device__ __forceinline__ void load_tiles(const float* __restrict__ A, int64_t lda,
                                           const float* __restrict__ B, int64_t ldb, int64_t M,
                                           int64_t N, int64_t K, int64_t m0, int64_t n0,
                                           int64_t k0, float ra[4], float rb[4]) {
  int tid = threadIdx.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m, k;
    if (!TA) { m = m0 + tid / 2; k = k0 + (tid % 2) * 4 + i; }
    else     { k = k0 + tid / 32; m = m0 + (tid % 32) * 4 + i; }
    ra[i] = (m < M && k < K) ? (TA ? A[k * lda + m] : A[m * lda + k]) : 0.0f;
    int64_t n, kb;
    if (TB) { n = n0 + tid / 2; kb = k0 + (tid % 2) * 4 + i; }
    else    { kb = k0 + tid / 32; n = n0 + (tid % 32) * 4 + i; }
    rb[i] = (n < N && kb < K) ? (TB ? B[n * ldb + kb] : B[kb * ldb + n]) : 0.0f;
  }
}

template <bool TA, bool TB>
__device__ __forceinline__ void store_tiles(float (*As)[BM], float (*Bs)[BN], const float ra[4],
                                            const float rb[4]) {
  int tid = threadIdx.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (!TA) As[(tid % 2) * 4 + i][tid / 2] = ra[i];
    else     As[tid / 32][(tid % 32) * 4 + i] = ra[i];
    if (TB)  Bs[(tid % 2) * 4 + i][tid / 2] = rb[i];
    else     Bs[tid / 32][(tid % 32) * 4 + i] = rb[i];
  }
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_gemm_simt(int64_t M, int64_t N, int64_t K,
                                                   const float* __restrict__ A, int64_t lda,
                                                   const float* __restrict__ B, int64_t ldb,
                                                   float* __restrict__ C, int64_t ldc,
                                                   const float* __restrict__ bias, int epi) {
  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];
  int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  int64_t m0 = blockIdx.y * (int64_t)BM, n0 = blockIdx.x * (int64_t)BN;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
  float ra[4], rb[4];
  load_tiles<TA, TB>(A, lda, B, ldb, M, N, K, m0, n0, 0, ra, rb);
  store_tiles<TA, TB>(As[0], Bs[0], ra, rb);
  __syncthreads();
  int nk = (int)((K + BK - 1) / BK);
  for (int kt = 0; kt < nk; ++kt) {
    int cur = kt & 1;
    if (kt + 1 < nk) load_tiles<TA, TB>(A, lda, B, ldb, M, N, K, m0, n0, (int64_t)(kt + 1) * BK, ra, rb);
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float4 a0 = *reinterpret_cast<const float4*>(&As[cur][k][ty * 4]);
      float4 a1 = *reinterpret_cast<const float4*>(&As[cur][k][64 + ty * 4]);
      float4 b0 = *reinterpret_cast<const float4*>(&Bs[cur][k][tx * 4]);
      float4 b1 = *reinterpret_cast<const float4*>(&Bs[cur][k][64 + tx * 4]);
      float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < nk) {
      store_tiles<TA, TB>(As[cur ^ 1], Bs[cur ^ 1], ra, rb);
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int64_t n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (n >= N) continue;
      float v = acc[i][j];
      if (epi == B2_EPI_BIAS || epi == B2_EPI_BIAS_RELU) v = __fadd_rn(v, bias[n]);
      if (epi == B2_EPI_BIAS_RELU || epi == B2_EPI_RELU) v = v > 0.0f ? v : 0.0f;
      C[m * ldc + n] = v;
    }
  }
}

__global__ void k_fill_bias(float* C, int64_t M, int64_t N, int64_t ldc, const float* bias, int epi) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M * N) return;
  int64_t m = i / N, n = i - m * N;
  float v = 0.0f;
  if (epi == B2_EPI_BIAS || epi == B2_EPI_BIAS_RELU) v = __fadd_rn(v, bias[n]);
  if (epi == B2_EPI_BIAS_RELU || epi == B2_EPI_RELU) v = v > 0.0f ? v : 0.0f;
  C[m * ldc + n] = v;
}

}  // namespace

namespace b2 {

int gemm_simt(int ta, int tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
              const float* B, int64_t ldb, float* C, int64_t ldc, const float* bias, int epi,
              cudaStream_t st) {
  if (M == 0 || N == 0) return 0;
  if (K == 0) {  // empty inner dimension: zeros (core.py matmul of (m,0)x(d,0))
    k_fill_bias<<<(unsigned)((M * N + 255) / 256), 256, 0, st>>>(C, M, N, ldc, bias, epi);
    return launched("b2_gemm(empty-K)");
  }
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM));
  if (grid.y > 65535) return fail("b2_gemm(simt): M too large for the SIMT grid");
#define B2_SIMT(TA_, TB_) \
  k_gemm_simt<TA_, TB_><<<grid, 256, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, bias, epi)
  if (!ta && !tb) B2_SIMT(false, false);
  else if (!ta && tb) B2_SIMT(false, true);
  else if (ta && !tb) B2_SIMT(true, false);
  else B2_SIMT(true, true);
#undef B2_SIMT
  return launched("b2_gemm(simt)");
}

}  // namespace b2
