/*
 * b2.h -- C ABI of the B200-native dense core (libb2.so).
 *
 * Plain pointers and sizes only; no torch or Python types. Every entry point
 * returns 0 on success and a nonzero status otherwise; b2_last_error()
 * returns the message of the most recent failure on the calling thread.
 * Device pointers are float32 (or int64 labels / double slots where named)
 * allocated with b2_alloc. Strides are in ELEMENTS; a stride of 0 marks a
 * broadcast axis (the reference's stride-0 expand view, core.py:381-392).
 * `stream` may be NULL for the engine's default compute stream.
 *
 * Each group below names the reference seam it replaces (paths relative to
 * /root/reference/pkg/src/tensorlite/). The reference is pure Python; these
 * are the pure-compute calls inside each op (SURVEY 8b "Kernel seams").
 */
#ifndef B2_H
#define B2_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B2_MAX_DIMS 8

/* ---------------------------------------------------------------- runtime */
const char* b2_last_error(void);
int b2_version(int* major, int* minor);
int b2_init(int device);                 /* select device, create streams */
int b2_device_count(int* n);
int b2_device_info(int* sm_count, int* cc_major, int* cc_minor, size_t* total_mem);
int b2_default_stream(void** stream);
int b2_stream_create(void** stream);
/* the same at the device's greatest stream priority (collectives beside the GEMMs) */
int b2_stream_create_priority(void** stream);
int b2_stream_destroy(void* stream);
int b2_stream_sync(void* stream);
int b2_device_sync(void);
int b2_event_create(void** ev);
int b2_event_destroy(void* ev);
int b2_event_record(void* ev, void* stream);
int b2_event_elapsed_ms(void* start, void* end, float* ms);
int b2_stream_wait_event(void* stream, void* ev);
/* kernels launched by this library since process start (launch counter) */
int b2_launch_count(uint64_t* n);
/* CUDA-graph capture of the engine stream (a training step replayed as one
 * launch). Blocks freed during capture stay private to the graph; every block
 * the graph touches is parked until b2_graph_destroy. No host syncs inside. */
int b2_graph_begin(void* stream);
int b2_graph_end(void* stream, int* graph_id);
int b2_graph_launch(int graph_id, void* stream);
int b2_graph_destroy(int graph_id);

/* ---------------------------------------------------------------- storage
 * Replaces Buffer(array('f')) per op output (core.py:68-75, 315-330): a
 * caching device allocator with size-class bins and stream-ordered frees.
 */
int b2_alloc(size_t bytes, void* stream, void** out);
int b2_free(void* ptr, void* stream);
int b2_alloc_stats(size_t* in_use, size_t* cached, size_t* peak, uint64_t* n_cuda_malloc);
int b2_empty_cache(void);
int b2_host_alloc(size_t bytes, void** out);   /* pinned host staging */
int b2_host_free(void* ptr);
int b2_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream);
int b2_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream);
int b2_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream);
/* stream-ordered D2H into pinned host memory (no stream drain); wait with
 * b2_event_sync on an event recorded after it */
int b2_memcpy_d2h_async(void* dst, const void* src, size_t bytes, void* stream);
int b2_event_sync(void* ev);
int b2_fill_f32(float* dst, float value, int64_t n, void* stream);

/* ---------------------------------------------------------------- elementwise
 * Replaces _elementwise/_binary/_unary (core.py:430-546) and the fused
 * pointwise activations (nn.py:95-111). out is contiguous with `shape`.
 */
enum b2_binary_op { B2_ADD = 0, B2_SUB = 1, B2_MUL = 2, B2_DIV = 3,
                    B2_RELU_BWD = 4 /* a * (b > 0 ? 1 : 0), nn.py:101-103 */,
                    B2_SIGN_MUL = 5 /* a * sign(b), core.py:533-546 */,
                    /* activation pullbacks (nn.py:95-144 _pointwise): a * f32(dfn(b)),
                       dfn in double on the saved value b */
                    B2_SIGMOID_BWD = 6 /* b = y: y * (1 - y) */,
                    B2_TANH_BWD = 7 /* b = y: 1 - y * y */,
                    B2_GELU_BWD = 8 /* b = x: Phi(x) + x * phi(x) */ };
enum b2_unary_op { B2_NEG = 0, B2_EXP = 1, B2_LOG = 2, B2_SQRT = 3, B2_ABS = 4,
                   B2_RELU = 5, B2_RELU_MASK = 6, B2_COPY = 7, B2_CLAMP = 8 /* min(max(x, alpha), beta); NaN passes */,
                   B2_SCALE = 9 /* x * alpha */, B2_DIV_SCALAR = 10 /* x / f32(alpha) */,
                   B2_CLAMP_MASK = 11 /* alpha <= x <= beta ? 1 : 0 */,
                   /* activations: f32(fn(double x)) (nn.py:114-144) */
                   B2_SIGMOID = 12 /* sign-split 1/(1+e^-x) | e^x/(1+e^x) */,
                   B2_TANH = 13, B2_GELU = 14 /* 0.5 x (1 + erf(x / sqrt 2)) */ };
int b2_binary(int op, float* out, int ndim, const int64_t* shape,
              const float* a, const int64_t* a_strides,
              const float* b, const int64_t* b_strides, void* stream);
/* binary op with one operand a Python scalar promoted to f32 (core.py:352-357) */
int b2_binary_scalar(int op, float* out, int ndim, const int64_t* shape,
                     const float* x, const int64_t* x_strides, float scalar,
                     int scalar_left, void* stream);
int b2_unary(int op, float* out, int ndim, const int64_t* shape,
             const float* x, const int64_t* x_strides,
             double alpha, double beta, void* stream);
/* strided (or stride-0 broadcast) gather into a contiguous tensor */
int b2_copy_strided(float* out, int ndim, const int64_t* shape,
                    const float* x, const int64_t* x_strides, void* stream);
/* strided scatter-write of a contiguous source into a (possibly strided) view */
int b2_write_strided(float* dst, int ndim, const int64_t* shape,
                     const int64_t* dst_strides, const float* src, void* stream);

/* Fused op+grad for y = relu(a*b + c) with a:[R,C], b,c broadcast rows [C]
 * (BASELINE config 2; core.py:453-483 + nn.py:108-111 in one pass).
 * fwd writes y (and optionally the pre-activation q). bwd of sum(y) w.r.t.
 * a and b in GradStore order: ga = mask*b, gb = f32(count) + f32(sum mask*a)
 * (autograd.py:140-145). */
int b2_fused_muladd_relu_fwd(float* y, const float* a, const float* b,
                             const float* c, int64_t rows, int64_t cols, void* stream);
int b2_fused_muladd_relu_bwd(float* ga, float* gb, const float* a,
                             const float* b, int64_t rows, int64_t cols, void* stream);

/* BASELINE config 2's whole workload in ONE pass over a [R, C] (b broadcast
 * rows [C]): y = relu(a*b + b), e = exp(clamp(a, lo, hi)), a_bar / b_bar of
 * sum(y) (as b2_fused_muladd_relu_bwd), sum/mean/max of y over dim 0 ([C])
 * and dim 1 ([R]) and the full sum -- the arithmetic of the separate ops
 * (core.py:453-483, 581-728; nn.py:108-111), bit-identical. Every output
 * pointer is nullable; C % 4 == 0, 16-B aligned rows. */
int b2_muladd_relu_stats(float* y, float* e, float* ga, float* gb, float* sum0, float* mean0,
                         float* max0, float* sum1, float* mean1, float* max1, float* total,
                         const float* a, const float* b, float clamp_lo, float clamp_hi,
                         int64_t rows, int64_t cols, void* stream);

/* ---------------------------------------------------------------- reductions
 * Replaces _sum_all / _axis_scan + sum/mean/max (core.py:581-728).
 * reduce_mask: bit d set => axis d is reduced. out is contiguous over the
 * kept axes (row-major). For B2_RED_MAX, argr (int64, may be NULL) receives
 * the index of the first maximum within the reduced subspace (row-major over
 * the reduced axes), the position the gradient is routed to.
 * Sums accumulate in fp64 with a fixed-order two-stage combine.
 */
enum b2_reduce_op { B2_RED_SUM = 0, B2_RED_MEAN = 1, B2_RED_MAX = 2 };
int b2_reduce(int op, float* out, int64_t* argr, int ndim, const int64_t* shape,
              const float* x, const int64_t* x_strides, uint32_t reduce_mask,
              void* stream);
/* max pullback (core.py:721-726): gx = zeros(shape); gx[pos(o, argr[o])] = g[o] */
int b2_max_scatter(float* gx, int ndim, const int64_t* shape, uint32_t reduce_mask,
                   const float* g, const int64_t* argr, void* stream);

/* ---------------------------------------------------------------- matmul
 * Replaces matmul.block (core.py:802-807) and its pullbacks (:815-817).
 * C[M,N] = opA(A) . opB(B) (+ bias[N]) (relu). Row-major with leading
 * dimensions lda/ldb/ldc in elements. trans_a: A stored [K,M]; trans_b: B
 * stored [N,K] (the reference's x.w^T is trans_b=1).
 * algo: 0 auto, 1 FP32 SIMT (FFMA), 2 3xTF32 on tcgen05 (fp32 accuracy),
 *       3 1xTF32 on tcgen05 (fast, ~1e-3 rel; never chosen by auto),
 *       4 TF32X: tf32 main product + the two cross terms as bf16 MMAs
 *         (2 tf32-equivalent MMAs per fp32 MAC, fp32-grade accuracy),
 *       5 3xBF16: hi = bf16_rn(x), lo = bf16_rn(x - hi); hi*hi + hi*lo + lo*hi
 *         as bf16 MMAs (1.5 tf32-equivalents per MAC, half TF32X's operand
 *         bytes, normwise error ~4e-6: inside the 1e-4 fp32 contract),
 *       7 REF: the reference's arithmetic -- exact fp32 products summed in fp64,
 *         one f32 rounding (core.py:802-807 matmul.block) -- on the FP64 pipe.
 *         Parity mode (the exact-arithmetic control), never chosen by auto.
 *       8 REF_BF16: the same on operands rounded to bf16 first -- the bf16
 *         variant's operand rounding with exact accumulation (its control).
 */
enum b2_gemm_algo { B2_GEMM_AUTO = 0, B2_GEMM_SIMT = 1, B2_GEMM_3XTF32 = 2,
                    B2_GEMM_1XTF32 = 3, B2_GEMM_TF32X = 4 /* tf32 hi*hi + bf16 hi*lo + lo*hi */,
                    B2_GEMM_3XBF16 = 5, B2_GEMM_REF = 7,
                    B2_GEMM_REF_BF16 = 8 };
enum b2_epilogue { B2_EPI_NONE = 0, B2_EPI_BIAS = 1, B2_EPI_BIAS_RELU = 2, B2_EPI_RELU = 3 };
int b2_gemm(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K,
            const float* A, int64_t lda, const float* B, int64_t ldb,
            float* C, int64_t ldc, const float* bias, int epilogue, int algo,
            void* stream);
/* which algorithm b2_gemm(algo=0) picks for a shape (for tests/bench) */
int b2_gemm_select(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K,
                   int64_t lda, int64_t ldb, int* algo);
/* split a [rows, cols] (leading dim ld) matrix into contiguous hi = tf32(x)
 * (round to nearest) and lo = x - hi, both exact fp32 (3xTF32 operands) */
int b2_tf32_split(float* hi, float* lo, const float* x, int64_t rows, int64_t cols,
                  int64_t ld, void* stream);
/* 3xTF32 GEMM on caller-provided contiguous splits (A: [M,K] or [K,M] if
 * trans_a; B: [N,K] if trans_b else [K,N]); lets the host reuse a split. */
int b2_gemm_presplit(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K,
                     const float* A_hi, const float* A_lo, const float* B_hi,
                     const float* B_lo, float* C, int64_t ldc, const float* bias,
                     int epilogue, void* stream);

/* split into contiguous bf16(trunc_tf32(x)) and bf16(x - trunc_tf32(x)); cols % 8 == 0 */
int b2_bf16x2_split(void* hi16, void* lo16, const float* x, int64_t rows, int64_t cols,
                    int64_t ld, void* stream);
/* TF32X GEMM: A/B raw fp32 (lda/ldb) + their contiguous b2_bf16x2_split halves */
int b2_gemm_tf32x(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K,
                  const float* A, int64_t lda, const void* A_hi16, const void* A_lo16,
                  const float* B, int64_t ldb, const void* B_hi16, const void* B_lo16,
                  float* C, int64_t ldc, const float* bias, int epilogue, void* stream);

/* TF32X GEMM with the fused MLP epilogue stages (nn.py:78-111 chained):
 * mask (nullable): C *= (mask > 0 ? 1 : 0) elementwise, mask [M,N] with ld = ldc
 *   -- the ReLU pullback of the layer below, applied to x_bar in the epilogue;
 * C_hi16/C_lo16 (nullable pair): also write C's TF32X split ([M,N] contiguous)
 *   so the GEMMs consuming C skip the b2_bf16x2_split pass;
 * colsum (nullable, [N] f32): column sums of the stored C over its M rows,
 *   f32(fp64 sum) -- the bias gradient of the layer below (core.py:405-423),
 *   computed in the epilogue instead of a separate pass over C. */
int b2_gemm_tf32x_ex(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K,
                     const float* A, int64_t lda, const void* A_hi16, const void* A_lo16,
                     const float* B, int64_t ldb, const void* B_hi16, const void* B_lo16,
                     float* C, int64_t ldc, const float* bias, int epilogue,
                     const float* mask, void* C_hi16, void* C_lo16, float* colsum, void* stream);

/* 3xBF16 split (hi = bf16_rn(x), lo = bf16_rn(x - hi), contiguous; cols % 8 == 0)
 * and the GEMM on such splits, with the same fused epilogue as
 * b2_gemm_tf32x_ex (C_hi16/C_lo16 receive C's own 3xBF16 split). */
int b2_bf16x3_split(void* hi16, void* lo16, const float* x, int64_t rows, int64_t cols,
                    int64_t ld, void* stream);
/* b2_bf16x3_split of two matrices in one launch (a GEMM's two fresh operands) */
int b2_bf16x3_split2(void* hi_a, void* lo_a, const float* a, int64_t rows_a, int64_t cols_a,
                     int64_t ld_a, void* hi_b, void* lo_b, const float* b, int64_t rows_b,
                     int64_t cols_b, int64_t ld_b, void* stream);
/* fp32 from a contiguous 3xBF16 split: out[i] = f32(hi[i]) + f32(lo[i]) (exact
 * in fp32; within 2^-16 relative of the split's source). n % 8 == 0, 16-B
 * aligned. Materialises a b2_gemm_fused output written with C == NULL (only
 * its operand split), on first host-visible use. */
int b2_bf16x3_join(float* out, const void* hi16, const void* lo16, int64_t n, void* stream);
int b2_gemm_3xbf16(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K,
                   const void* A_hi16, const void* A_lo16, const void* B_hi16,
                   const void* B_lo16, float* C, int64_t ldc, const float* bias, int epilogue,
                   const float* mask, void* C_hi16, void* C_lo16, float* colsum, void* stream);

/* The fused tensor-core GEMM of the MLP chain, one descriptor for every
 * epilogue stage (C = opA(A) . opB(B) as b2_gemm):
 *   algo B2_GEMM_3XBF16: a = {A_hi16, A_lo16}, b = {B_hi16, B_lo16} (contiguous splits);
 *   algo B2_GEMM_TF32X:  a = {A, A_hi16, A_lo16} (A with lda), b likewise;
 *   algo B2_GEMM_BF16_VARIANT: a = {A16}, b = {B16} (contiguous bf16 casts).
 * Epilogue, in order: + bias, ReLU, then the ReLU pullback of the layer below
 * (mask_bits: 1 bit per element as written by relu_bits_out, else mask: a
 * float tensor read as > 0), stores, C's own operand split (c_hi/c_lo; c_hi
 * alone = bf16 cast for BF16_VARIANT), relu_bits_out (C > 0 as bits, words
 * of 64 columns, ceil(N/64) words per row; needs a ReLU epilogue), colsum
 * (column sums of C, f32(fp64)). All pointers nullable except the operands;
 * C == NULL skips the fp32 store when only C's split/bits/column sums are
 * consumed (the host materialises C later with b2_bf16x3_join if it is read). */
enum { B2_GEMM_BF16_VARIANT = 6 };
typedef struct b2_gemm_desc {
  int algo, trans_a, trans_b;
  int64_t M, N, K;
  const void* a[3];
  int64_t lda;
  const void* b[3];
  int64_t ldb;
  float* C;
  int64_t ldc;
  const float* bias;
  int epilogue;
  const float* mask;
  const uint64_t* mask_bits;
  void* c_hi;
  void* c_lo;
  uint64_t* relu_bits_out;
  float* colsum;
} b2_gemm_desc;
int b2_gemm_fused(const b2_gemm_desc* desc, void* stream);
/* Up to 3 independent b2_gemm_fused problems of one algo in ONE persistent
 * launch -- the x_bar and w_bar GEMMs of a matmul pullback (core.py:815-817),
 * which read the same cotangent: units of all problems are drawn from one
 * queue, the most expensive first, so short-K and long-K GEMMs fill each
 * other's idle SMs. Outputs are bit-identical to separate b2_gemm_fused
 * calls; no output may alias another descriptor's input. Replaces the two
 * matmul calls of the pullback pair (core.py:815-817). */
int b2_gemm_fused_group(const b2_gemm_desc* descs, int n, void* stream);
/* SMs the persistent GEMM grids leave free (default 0): under data
 * parallelism the collectives' kernels run beside the backward GEMMs. */
int b2_gemm_set_sm_reserve(int n);
int b2_gemm_get_sm_reserve(int* n);

/* BF16 variant (explicitly requested precision only; bf16 tolerance 2e-2):
 * contiguous round-to-nearest bf16 cast of a [rows, cols] (ld) matrix, and a
 * GEMM on such casts (one kind::f16 MMA per MAC, fp32 accumulation) with the
 * same fused epilogue; C16 (nullable) receives C's own bf16 cast. */
int b2_bf16_cast(void* out16, const float* x, int64_t rows, int64_t cols, int64_t ld,
                 void* stream);
int b2_gemm_bf16(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const void* A16,
                 const void* B16, float* C, int64_t ldc, const float* bias, int epilogue,
                 const float* mask, void* C16, float* colsum, void* stream);

/* ---------------------------------------------------------------- conv2d
 * im2col / col2im of tensorlite's conv2d (nn.py:191-303); the GEMMs between
 * them run on b2_gemm*. x: (B, C, H, W) contiguous; patches: (B*OH*OW, C*KH*KW)
 * with rows = output positions (b, i, j), cols = taps (c, u, v), zero padding.
 * col2im gathers each input element's taps in increasing output-row order,
 * accumulating in double (the reference's scatter order), one f32 rounding. */
int b2_im2col(float* patches, const float* x, int64_t B, int64_t C, int64_t H, int64_t W,
              int64_t KH, int64_t KW, int64_t stride, int64_t pad, int64_t OH, int64_t OW,
              void* stream);
int b2_col2im(float* dx, const float* dpatches, int64_t B, int64_t C, int64_t H, int64_t W,
              int64_t KH, int64_t KW, int64_t stride, int64_t pad, int64_t OH, int64_t OW,
              void* stream);

/* ---------------------------------------------------------------- losses
 * cross_entropy (nn.py:453-503): fwd writes the mean loss (f32 scalar) and
 * per-row stats (max, sum exp) in double; bwd writes
 * dlogits = (exp(z-m)/se - onehot) * (g[0] / denom) (denom: the mean's divisor, b).
 * labels are int64, validated on the host (nn.py:465-472).
 */
int b2_xent_fwd(float* loss, double* row_stats, const float* logits,
                const int64_t* labels, int64_t rows, int64_t cols, double denom,
                void* stream);
int b2_xent_bwd(float* dlogits, const float* g, const double* row_stats,
                const float* logits, const int64_t* labels, int64_t rows,
                int64_t cols, double denom, void* stream);
/* b2_xent_bwd with the outputs the last Linear's pullbacks read: dlogits'
 * 3xBF16 split (dl_hi/dl_lo, as b2_bf16x3_split) and its column sums
 * (f32(sum64 over rows), the bias gradient); every output nullable (dlogits
 * too: the split alone when only GEMMs consume it). cols % 8 == 0, <= 1024. */
int b2_xent_bwd_split(float* dlogits, void* dl_hi, void* dl_lo, float* colsum, const float* g,
                      const double* row_stats, const float* logits, const int64_t* labels, int64_t rows,
                      int64_t cols, double denom, void* stream);
/* row softmax over the last axis, composed-semantics:
 * m = rowmax (detached), e = f32(exp(f32(z-m))), s = f32(sum64 e), y = f32(e/s).
 * bwd mirrors the GradStore order of the composition:
 * gz = f32(f32(f32(gy/s) + f32(sum64 f32(-f32(f32(gy*e)/f32(s*s))))) * e). */
int b2_softmax_fwd(float* y, float* row_s, float* row_m, const float* z,
                   int64_t rows, int64_t cols, void* stream);
int b2_softmax_bwd(float* gz, const float* gy, const float* z, const float* row_s,
                   const float* row_m, int64_t rows, int64_t cols, void* stream);

/* Fused row softmax * t, mean -- BASELINE config 4's loss mean(softmax(z) * t),
 * bit-identical to composing softmax (above) -> mul (core.py:469-476) -> mean
 * (core.py:663-689), with one row pass each way (cols % 4 == 0, cols <= 1024,
 * 16-B aligned rows).
 * fwd: y (nullable) = softmax(z); row_s/row_m as b2_softmax_fwd; row_dot[r] =
 *   sum64_j f32(y*t); loss = f32(sum64_r row_dot / (rows*cols)).
 * bwd: g = the loss cotangent (device scalar); gz = the composed pullback
 *   (mean: f32(g / count_f32); mul: f32(gp * t); softmax as b2_softmax_bwd).
 *   Outputs, each nullable: gz (fp32), gz_hi/gz_lo (gz's 3xBF16 split, as
 *   b2_bf16x3_split), colsum[cols] = f32(sum64 over rows of gz) (the bias
 *   gradient of a Linear feeding z, core.py:405-423). */
int b2_softmax_wmean_fwd(float* loss, float* y, float* row_s, float* row_m, double* row_dot,
                         const float* z, const float* t, int64_t rows, int64_t cols, void* stream);
int b2_softmax_wmean_bwd(float* gz, void* gz_hi, void* gz_lo, float* colsum, const float* g,
                         float count_f32, const float* z, const float* t, const float* row_s,
                         const float* row_m, int64_t rows, int64_t cols, void* stream);

/* ---------------------------------------------------------------- optimizers
 * Optimizer.step/_update + step_all (optim.py:39-136) as ONE multi-tensor
 * launch. Slots are double, like the reference. Per-tensor bias corrections
 * (Adam's t is per parameter, optim.py:84-91) come from the host.
 */
typedef struct b2_opt_tensor {
  float* param;
  const float* grad;
  double* slot0;      /* SGD v / Adam m */
  double* slot1;      /* Adam v (unused by SGD) */
  int64_t n;
  double bc1, bc2;    /* Adam: 1-b1^t, 1-b2^t */
} b2_opt_tensor;
int b2_sgd_multi(const b2_opt_tensor* tensors, int count, double lr, double momentum,
                 double weight_decay, void* stream);
int b2_adam_multi(const b2_opt_tensor* tensors, int count, double lr, double beta1,
                  double beta2, double eps, double weight_decay, void* stream);
/* RMSprop (optim.py:103-122): v = rho*v + (1-rho)*g*g; theta -= lr*g/sqrt(v+eps);
 * slot0 = v (fp64) */
int b2_rmsprop_multi(const b2_opt_tensor* tensors, int count, double lr, double rho, double eps,
                     double weight_decay, void* stream);

/* ---------------------------------------------------------------- collectives
 * Data-parallel gradient exchange (new; the reference is single-process).
 * NCCL over NVLink/NVSwitch; one communicator per process (one GPU each).
 */
int b2_comm_unique_id(unsigned char* out128);
int b2_comm_init(int rank, int nranks, const unsigned char* uid128);
int b2_comm_destroy(void);
/* in-place sum (op=0) / average (op=1) / max (op=2) over all ranks, fp32 */
int b2_allreduce_f32(float* buf, int64_t n, int op, void* stream);
/* sharded optimizer step: reduce-scatter (recv = this rank's count-element
 * shard of the reduced send[count * nranks]) and in-place all-gather (buf
 * [count * nranks], this rank's shard at buf + rank * count) */
int b2_reduce_scatter_f32(const float* send, float* recv, int64_t count, int op, void* stream);
int b2_all_gather_f32(float* buf, int64_t count, int rank, void* stream);
/* failure detection: the communicator's asynchronous NCCL error (0 = ok),
 * abort, and a host wait for a stream with a deadline that polls the async
 * error and aborts the communicator on error or timeout */
int b2_comm_async_error(int* err);
int b2_comm_abort(void);
int b2_stream_wait_timeout(void* stream, double timeout_ms);

#ifdef __cplusplus
}
#endif
#endif /* B2_H */
