// Matmul engine dispatch: C = opA(A) . opB(B) (+bias) (relu).
// Replaces tensorlite/core.py:784-820 (matmul and its pullbacks).
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace b2 {
int gemm_simt(int ta, int tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
              const float* B, int64_t ldb, float* C, int64_t ldc, const float* bias, int epi,
              cudaStream_t st);
int gemm_tc(int ta, int tb, int nprod, int64_t M, int64_t N, int64_t K, const float* Ahi,
            const float* Alo, int64_t lda, const float* Bhi, const float* Blo, int64_t ldb,
            float* C, int64_t ldc, const float* bias, int epi, cudaStream_t st);
int tf32_split(float* hi, float* lo, const float* x, int64_t rows, int64_t cols, int64_t ld,
               cudaStream_t st);
bool tc_supported(int ta, int tb, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb);
}  // namespace b2

namespace {

int forced_algo() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("B2_GEMM_ALGO");
    v = 0;
    if (e) {
      if (!strcmp(e, "simt")) v = B2_GEMM_SIMT;
      else if (!strcmp(e, "3xtf32")) v = B2_GEMM_3XTF32;
      else if (!strcmp(e, "1xtf32")) v = B2_GEMM_1XTF32;
    }
  }
  return v;
}

int select(int ta, int tb, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb) {
  int f = forced_algo();
  bool tc = b2::tc_supported(ta, tb, M, N, K, lda, ldb);
  if (f == B2_GEMM_SIMT || !tc) return B2_GEMM_SIMT;
  if (f) return f;
  // the tensor-core path pays a split pass + TMEM setup; small problems stay on FFMA
  double work = (double)M * (double)N * (double)K;
  return work >= (double)(1 << 26) ? B2_GEMM_3XTF32 : B2_GEMM_SIMT;
}

}  // namespace

extern "C" {

int b2_gemm_select(int ta, int tb, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb,
                   int* algo) {
  *algo = select(ta, tb, M, N, K, lda, ldb);
  return 0;
}

int b2_tf32_split(float* hi, float* lo, const float* x, int64_t rows, int64_t cols, int64_t ld,
                  void* stream) {
  return b2::tf32_split(hi, lo, x, rows, cols, ld, b2::resolve(stream));
}

int b2_gemm(int ta, int tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
            const float* B, int64_t ldb, float* C, int64_t ldc, const float* bias, int epi,
            int algo, void* stream) {
  if (M < 0 || N < 0 || K < 0) return b2::fail("b2_gemm: negative extent");
  if ((epi == B2_EPI_BIAS || epi == B2_EPI_BIAS_RELU) && !bias)
    return b2::fail("b2_gemm: bias epilogue without a bias pointer");
  cudaStream_t st = b2::resolve(stream);
  if (M == 0 || N == 0) return 0;
  if (K == 0) return b2::gemm_simt(ta, tb, M, N, 0, A, lda, B, ldb, C, ldc, bias, epi, st);
  if (algo == B2_GEMM_AUTO) algo = select(ta, tb, M, N, K, lda, ldb);
  if (algo != B2_GEMM_SIMT && !b2::tc_supported(ta, tb, M, N, K, lda, ldb))
    return b2::fail("b2_gemm: operands not TMA-compatible (leading dims must be multiples of 4)");
  switch (algo) {
    case B2_GEMM_SIMT:
      return b2::gemm_simt(ta, tb, M, N, K, A, lda, B, ldb, C, ldc, bias, epi, st);
    case B2_GEMM_1XTF32:
      if (((uintptr_t)A & 15) || ((uintptr_t)B & 15))
        return b2::fail("b2_gemm(1xtf32): operands must be 16-byte aligned for TMA");
      return b2::gemm_tc(ta, tb, 1, M, N, K, A, nullptr, lda, B, nullptr, ldb, C, ldc, bias, epi, st);
    case B2_GEMM_3XTF32: {
      // A: [M,K] (K-major) or stored [K,M]; B: [N,K] (trans_b) or stored [K,N]
      int64_t ar = ta ? K : M, ac = ta ? M : K;
      int64_t br = tb ? N : K, bc = tb ? K : N;
      size_t abytes = (size_t)ar * ac * 4, bbytes = (size_t)br * bc * 4;
      void* ws = nullptr;
      B2_TRY(b2_alloc(2 * (abytes + bbytes), st, &ws));
      float* ahi = (float*)ws;
      float* alo = (float*)((char*)ws + abytes);
      float* bhi = (float*)((char*)ws + 2 * abytes);
      float* blo = (float*)((char*)ws + 2 * abytes + bbytes);
      int rc = b2::tf32_split(ahi, alo, A, ar, ac, lda, st);
      if (!rc) rc = b2::tf32_split(bhi, blo, B, br, bc, ldb, st);
      if (!rc) rc = b2::gemm_tc(ta, tb, 3, M, N, K, ahi, alo, ac, bhi, blo, bc, C, ldc, bias, epi, st);
      b2_free(ws, st);
      return rc;
    }
  }
  return b2::fail("b2_gemm: unknown algo");
}

// 3xTF32 with caller-provided contiguous split operands (lets the host cache
// the split of a tensor that feeds several GEMMs, e.g. X in fwd and in dW).
int b2_gemm_presplit(int ta, int tb, int64_t M, int64_t N, int64_t K, const float* Ahi,
                     const float* Alo, const float* Bhi, const float* Blo, float* C, int64_t ldc,
                     const float* bias, int epi, void* stream) {
  if (M == 0 || N == 0) return 0;
  int64_t ac = ta ? M : K, bc = tb ? K : N;
  if (!b2::tc_supported(ta, tb, M, N, K, ac, bc))
    return b2::fail("b2_gemm_presplit: operands not TMA-compatible");
  return b2::gemm_tc(ta, tb, 3, M, N, K, Ahi, Alo, ac, Bhi, Blo, bc, C, ldc, bias, epi,
                     b2::resolve(stream));
}

}  // extern "C"
