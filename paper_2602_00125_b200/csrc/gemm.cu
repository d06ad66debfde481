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
int gemm_tc(int ta, int tb, int mode, int64_t M, int64_t N, int64_t K, const void* a0,
            const void* a1, const void* a2, int64_t lda, const void* b0, const void* b1,
            const void* b2_, int64_t ldb, float* C, int64_t ldc, const float* bias, int epi,
            cudaStream_t st, const float* mask = nullptr, void* s_hi = nullptr,
            void* s_lo = nullptr, float* colsum = nullptr, const uint64_t* mask_bits = nullptr,
            uint64_t* bits_out = nullptr);
int gemm_ref(int ta, int tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
             const float* B, int64_t ldb, float* C, int64_t ldc, const float* bias, int epi,
             cudaStream_t st, bool bf16_operands);
int tf32_split(float* hi, float* lo, const float* x, int64_t rows, int64_t cols, int64_t ld,
               cudaStream_t st);
int bf16_cast(void* out, const float* x, int64_t rows, int64_t cols, int64_t ld, cudaStream_t st);
int bf16x3_join(float* out, const void* hi, const void* lo, int64_t n, cudaStream_t st);
int bf16x3_split2(void* hia, void* loa, const float* xa, int64_t ra, int64_t ca, int64_t lda, void* hib,
                  void* lob, const float* xb, int64_t rb, int64_t cb, int64_t ldb, cudaStream_t st);
int bf16x2_split(void* hi, void* lo, const float* x, int64_t rows, int64_t cols, int64_t ld,
                 cudaStream_t st, int mode = 2);
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
      else if (!strcmp(e, "tf32x")) v = B2_GEMM_TF32X;
      else if (!strcmp(e, "3xbf16")) v = B2_GEMM_3XBF16;
      else if (!strcmp(e, "ref")) v = B2_GEMM_REF;
      else if (!strcmp(e, "ref_bf16")) v = B2_GEMM_REF_BF16;
    }
  }
  return v;
}

int select(int ta, int tb, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb) {
  int f = forced_algo();
  bool tc = b2::tc_supported(ta, tb, M, N, K, lda, ldb);
  if (f == B2_GEMM_REF || f == B2_GEMM_REF_BF16) return f;
  if (f == B2_GEMM_SIMT || !tc) return B2_GEMM_SIMT;
  if (f) return f;
  // the tensor-core path pays a split pass + TMEM setup; small problems stay on FFMA.
  // 3xBF16 (normwise ~4e-6) beats TF32X (~2e-6) by 1.4x at every measured size
  // and holds the 1e-4 fp32 contract with a 25x margin.
  double work = (double)M * (double)N * (double)K;
  return work >= (double)(1 << 26) ? B2_GEMM_3XBF16 : B2_GEMM_SIMT;
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
  if (algo == B2_GEMM_REF || algo == B2_GEMM_REF_BF16)
    return b2::gemm_ref(ta, tb, M, N, K, A, lda, B, ldb, C, ldc, bias, epi, st, algo == B2_GEMM_REF_BF16);
  if (algo != B2_GEMM_SIMT && !b2::tc_supported(ta, tb, M, N, K, lda, ldb))
    return b2::fail("b2_gemm: operands not TMA-compatible (leading dims must be multiples of 4)");
  switch (algo) {
    case B2_GEMM_SIMT:
      return b2::gemm_simt(ta, tb, M, N, K, A, lda, B, ldb, C, ldc, bias, epi, st);
    case B2_GEMM_1XTF32:
      if (((uintptr_t)A & 15) || ((uintptr_t)B & 15))
        return b2::fail("b2_gemm(1xtf32): operands must be 16-byte aligned for TMA");
      return b2::gemm_tc(ta, tb, 1, M, N, K, A, nullptr, nullptr, lda, B, nullptr, nullptr, ldb, C,
                         ldc, bias, epi, st);
    case B2_GEMM_3XBF16: {
      int64_t ar = ta ? K : M, ac = ta ? M : K;
      int64_t br = tb ? N : K, bc = tb ? K : N;
      size_t abytes = ((size_t)ar * ac * 2 + 255) & ~(size_t)255;
      size_t bbytes = ((size_t)br * bc * 2 + 255) & ~(size_t)255;
      void* ws = nullptr;
      B2_TRY(b2_alloc(2 * (abytes + bbytes), st, &ws));
      char* w = (char*)ws;
      int rc = b2::bf16x2_split(w, w + abytes, A, ar, ac, lda, st, 5);
      if (!rc) rc = b2::bf16x2_split(w + 2 * abytes, w + 2 * abytes + bbytes, B, br, bc, ldb, st, 5);
      if (!rc)
        rc = b2::gemm_tc(ta, tb, 5, M, N, K, w, w + abytes, nullptr, ac, w + 2 * abytes,
                         w + 2 * abytes + bbytes, nullptr, bc, C, ldc, bias, epi, st);
      b2_free(ws, st);
      return rc;
    }
    case B2_GEMM_TF32X: {
      if (((uintptr_t)A & 15) || ((uintptr_t)B & 15))
        return b2::fail("b2_gemm(tf32x): operands must be 16-byte aligned for TMA");
      int64_t ar = ta ? K : M, ac = ta ? M : K;
      int64_t br = tb ? N : K, bc = tb ? K : N;
      size_t abytes = (size_t)ar * ac * 2, bbytes = (size_t)br * bc * 2;
      abytes = (abytes + 255) & ~(size_t)255;
      bbytes = (bbytes + 255) & ~(size_t)255;
      void* ws = nullptr;
      B2_TRY(b2_alloc(2 * (abytes + bbytes), st, &ws));
      char* w = (char*)ws;
      int rc = b2::bf16x2_split(w, w + abytes, A, ar, ac, lda, st);
      if (!rc) rc = b2::bf16x2_split(w + 2 * abytes, w + 2 * abytes + bbytes, B, br, bc, ldb, st);
      if (!rc)
        rc = b2::gemm_tc(ta, tb, 2, M, N, K, A, w, w + abytes, lda, B, w + 2 * abytes,
                         w + 2 * abytes + bbytes, ldb, C, ldc, bias, epi, st);
      b2_free(ws, st);
      return rc;
    }
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
      if (!rc)
        rc = b2::gemm_tc(ta, tb, 3, M, N, K, ahi, alo, nullptr, ac, bhi, blo, nullptr, bc, C, ldc,
                         bias, epi, st);
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
  return b2::gemm_tc(ta, tb, 3, M, N, K, Ahi, Alo, nullptr, ac, Bhi, Blo, nullptr, bc, C, ldc, bias,
                     epi, b2::resolve(stream));
}

int b2_bf16x2_split(void* hi16, void* lo16, const float* x, int64_t rows, int64_t cols, int64_t ld,
                    void* stream) {
  return b2::bf16x2_split(hi16, lo16, x, rows, cols, ld, b2::resolve(stream));
}

// TF32 main product on the raw fp32 operands + the two cross terms as bf16
// MMAs on caller-provided contiguous splits (b2_bf16x2_split of A and B).
int b2_gemm_tf32x(int ta, int tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                  const void* A_hi16, const void* A_lo16, const float* B, int64_t ldb,
                  const void* B_hi16, const void* B_lo16, float* C, int64_t ldc, const float* bias,
                  int epi, void* stream) {
  if (M == 0 || N == 0) return 0;
  if (!b2::tc_supported(ta, tb, M, N, K, lda, ldb) || ((uintptr_t)A & 15) || ((uintptr_t)B & 15))
    return b2::fail("b2_gemm_tf32x: operands not TMA-compatible");
  return b2::gemm_tc(ta, tb, 2, M, N, K, A, A_hi16, A_lo16, lda, B, B_hi16, B_lo16, ldb, C, ldc,
                     bias, epi, b2::resolve(stream));
}

int b2_bf16_cast(void* out16, const float* x, int64_t rows, int64_t cols, int64_t ld,
                 void* stream) {
  return b2::bf16_cast(out16, x, rows, cols, ld, b2::resolve(stream));
}

// BF16 GEMM (the config-5 bf16 variant): one kind::f16 MMA per MAC on
// contiguous bf16 operand casts (A16: [M,K] or [K,M]; B16: [N,K] or [K,N]),
// fp32 accumulation with the same K-chunk promotion; same fused epilogue
// stages (bias, relu, ReLU-pullback mask, C's own bf16 cast for the next GEMM).
int b2_gemm_bf16(int ta, int tb, int64_t M, int64_t N, int64_t K, const void* A16,
                 const void* B16, float* C, int64_t ldc, const float* bias, int epi,
                 const float* mask, void* C16, float* colsum, void* stream) {
  if (M == 0 || N == 0) return 0;
  int64_t ac = ta ? M : K, bc = tb ? K : N;
  if (!b2::tc_supported(ta, tb, M, N, K, ac, bc) || ((uintptr_t)A16 & 15) || ((uintptr_t)B16 & 15))
    return b2::fail("b2_gemm_bf16: operands not TMA-compatible");
  if (mask && (((uintptr_t)mask & 15) || ldc % 4)) return b2::fail("b2_gemm_bf16: mask alignment");
  return b2::gemm_tc(ta, tb, 4, M, N, K, A16, nullptr, nullptr, ac, B16, nullptr, nullptr, bc, C,
                     ldc, bias, epi, b2::resolve(stream), mask, C16, nullptr, colsum);
}

int b2_bf16x3_split(void* hi16, void* lo16, const float* x, int64_t rows, int64_t cols, int64_t ld,
                    void* stream) {
  return b2::bf16x2_split(hi16, lo16, x, rows, cols, ld, b2::resolve(stream), 5);
}

int b2_bf16x3_split2(void* hi_a, void* lo_a, const float* a, int64_t rows_a, int64_t cols_a,
                     int64_t ld_a, void* hi_b, void* lo_b, const float* b, int64_t rows_b,
                     int64_t cols_b, int64_t ld_b, void* stream) {
  return b2::bf16x3_split2(hi_a, lo_a, a, rows_a, cols_a, ld_a, hi_b, lo_b, b, rows_b, cols_b, ld_b,
                           b2::resolve(stream));
}

int b2_bf16x3_join(float* out, const void* hi16, const void* lo16, int64_t n, void* stream) {
  return b2::bf16x3_join(out, hi16, lo16, n, b2::resolve(stream));
}

// 3xBF16: hi*hi + hi*lo + lo*hi as kind::f16 MMAs on caller-provided
// contiguous b2_bf16x3_split operands; fused epilogue as b2_gemm_tf32x_ex
// (the emitted C split is C's own 3xBF16 split).
int b2_gemm_3xbf16(int ta, int tb, int64_t M, int64_t N, int64_t K, const void* A_hi16,
                   const void* A_lo16, const void* B_hi16, const void* B_lo16, float* C,
                   int64_t ldc, const float* bias, int epi, const float* mask, void* C_hi16,
                   void* C_lo16, float* colsum, void* stream) {
  if (M == 0 || N == 0) return 0;
  int64_t ac = ta ? M : K, bc = tb ? K : N;
  if (!b2::tc_supported(ta, tb, M, N, K, ac, bc))
    return b2::fail("b2_gemm_3xbf16: operands not TMA-compatible");
  if (mask && (((uintptr_t)mask & 15) || ldc % 4)) return b2::fail("b2_gemm_3xbf16: mask alignment");
  return b2::gemm_tc(ta, tb, 5, M, N, K, A_hi16, A_lo16, nullptr, ac, B_hi16, B_lo16, nullptr, bc,
                     C, ldc, bias, epi, b2::resolve(stream), mask, C_hi16, C_lo16, colsum);
}

// b2_gemm_tf32x with the fused MLP epilogue stages: optional ReLU-pullback
// mask (C *= mask > 0, mask [M,N] with ld = ldc) and optional emission of C's
// own TF32X split (bf16 hi/lo, [M,N] contiguous) for the GEMMs that consume C.
int b2_gemm_tf32x_ex(int ta, int tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                     const void* A_hi16, const void* A_lo16, const float* B, int64_t ldb,
                     const void* B_hi16, const void* B_lo16, float* C, int64_t ldc,
                     const float* bias, int epi, const float* mask, void* C_hi16, void* C_lo16,
                     float* colsum, void* stream) {
  if (M == 0 || N == 0) return 0;
  if (!b2::tc_supported(ta, tb, M, N, K, lda, ldb) || ((uintptr_t)A & 15) || ((uintptr_t)B & 15))
    return b2::fail("b2_gemm_tf32x_ex: operands not TMA-compatible");
  if (mask && (((uintptr_t)mask & 15) || ldc % 4)) return b2::fail("b2_gemm_tf32x_ex: mask alignment");
  return b2::gemm_tc(ta, tb, 2, M, N, K, A, A_hi16, A_lo16, lda, B, B_hi16, B_lo16, ldb, C, ldc,
                     bias, epi, b2::resolve(stream), mask, C_hi16, C_lo16, colsum);
}

// The fused tensor-core GEMM behind one descriptor (include/b2.h
// b2_gemm_desc): every epilogue stage of the MLP chain in one launch.
static int desc_to_tc(const b2_gemm_desc* d, b2::TcDesc* t, int* mode_out) {
  const int ta = d->trans_a, tb = d->trans_b;
  const int64_t M = d->M, N = d->N, K = d->K;
  const int64_t ac = ta ? M : K, bc = tb ? K : N;
  int mode;
  int64_t lda = d->lda, ldb = d->ldb;
  switch (d->algo) {
    case B2_GEMM_3XBF16: mode = 5; lda = ac; ldb = bc; break;
    case B2_GEMM_TF32X: mode = 2; break;
    case B2_GEMM_BF16_VARIANT: mode = 4; lda = ac; ldb = bc; break;
    default: return b2::fail("b2_gemm_fused: algo must be 3XBF16, TF32X or BF16_VARIANT");
  }
  if (M < 0 || N < 0 || K < 0) return b2::fail("b2_gemm_fused: negative extent");
  if (!b2::tc_supported(ta, tb, M, N, K, lda, ldb))
    return b2::fail("b2_gemm_fused: operands not TMA-compatible");
  if (d->mask && (((uintptr_t)d->mask & 15) || d->ldc % 4))
    return b2::fail("b2_gemm_fused: mask alignment");
  if (d->relu_bits_out && !(d->epilogue == B2_EPI_RELU || d->epilogue == B2_EPI_BIAS_RELU))
    return b2::fail("b2_gemm_fused: relu_bits_out needs a ReLU epilogue");
  if ((d->epilogue == B2_EPI_BIAS || d->epilogue == B2_EPI_BIAS_RELU) && !d->bias)
    return b2::fail("b2_gemm_fused: bias epilogue without a bias pointer");
  *t = b2::TcDesc{ta, tb, M, N, K, d->a[0], d->a[1], mode == 2 ? d->a[2] : nullptr, lda,
                  d->b[0], d->b[1], mode == 2 ? d->b[2] : nullptr, ldb, d->C, d->ldc, d->bias,
                  d->epilogue, d->mask, d->c_hi, mode == 4 ? nullptr : d->c_lo, d->colsum,
                  d->mask_bits, d->relu_bits_out};
  *mode_out = mode;
  return 0;
}

int b2_gemm_fused(const b2_gemm_desc* d, void* stream) {
  if (!d) return b2::fail("b2_gemm_fused: null descriptor");
  if (d->M == 0 || d->N == 0) return 0;
  b2::TcDesc t;
  int mode;
  B2_TRY(desc_to_tc(d, &t, &mode));
  return b2::gemm_tc_group(mode, &t, 1, b2::resolve(stream));
}

// Up to 3 independent fused GEMMs of one algo in ONE persistent launch (the
// dX and dW GEMMs of a matmul/linear pullback: they read the same cotangent
// and write different outputs). Units are drawn dynamically, the most
// expensive first; every output is bit-identical to b2_gemm_fused of the
// same descriptor. No output may alias another problem's input.
int b2_gemm_fused_group(const b2_gemm_desc* d, int n, void* stream) {
  if (!d || n < 1 || n > 3) return b2::fail("b2_gemm_fused_group: 1 to 3 descriptors");
  b2::TcDesc t[3];
  int modes[3], m = 0;
  for (int i = 0; i < n; ++i) {
    if (d[i].M == 0 || d[i].N == 0) continue;  // empty output: nothing to launch
    B2_TRY(desc_to_tc(&d[i], &t[m], &modes[m]));
    if (m && modes[m] != modes[0]) return b2::fail("b2_gemm_fused_group: descriptors differ in algo");
    ++m;
  }
  if (!m) return 0;
  return b2::gemm_tc_group(modes[0], t, m, b2::resolve(stream));
}

}  // extern "C"
