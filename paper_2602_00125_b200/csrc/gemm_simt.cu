// FP32 SIMT GEMM (FFMA, fp32 accumulate): the exact-fp32 fallback of the
// matmul engine for shapes the tcgen05 path does not take (tiny problems,
// operands whose leading dimension breaks TMA's 16-byte stride rule).
//
// Replaces matmul.block (tensorlite/core.py:802-807) and its pullbacks
// (core.py:815-817); the three operand layouts of those pullbacks are
// template parameters, so transposed views are read in place, never copied.
// 128x128x16 CTA tile, 256 threads, 8x8 outputs per thread (two 4x4 quads per
// axis to keep shared-memory reads conflict-free), 128-bit global loads staged
// through registers across the k-tile (double-buffered shared memory).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"

extern "C" int b2_alloc(size_t, void*, void**);
extern "C" int b2_free(void*, void*);

namespace {

constexpr int BM = 128, BN = 128, BK = 16, GW = 16;
// Shared-memory tiles are [k][r] rows of 128 floats with the column XOR-swizzled by
// the k-quad, c = r ^ (8 * ((k >> 2) & 3)): the transposing stores of a
// k-contiguous operand (a warp holds 8 rows x 4 k-quads) then hit 32 distinct banks,
// and 16-byte groups stay whole for the 128-bit fragment reads.
constexpr int LDS = BM;
__device__ __forceinline__ int swz(int k) { return 8 * ((k >> 2) & 3); }

// One operand tile (128 rows/columns r x 16 k) from global memory into registers.
// KC: element (r, k) at X[r * ld + k] (k contiguous), else X[k * ld + r].
// VEC: base pointer 16-byte aligned and ld % 4 == 0, so a quad that lies inside
// the matrix is one 128-bit load; edge quads (and VEC = false) take guarded
// scalar loads with zero fill.
template <bool KC, bool VEC>
__device__ __forceinline__ void gload(const float* __restrict__ X, int64_t ld, int64_t R, int64_t K,
                                      int64_t r0, int64_t k0, float4 q[2]) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    int64_t r, k;
    if (KC) { r = r0 + (tid >> 2) + 64 * i; k = k0 + (tid & 3) * 4; }
    else    { k = k0 + (tid >> 5) + 8 * i;  r = r0 + (tid & 31) * 4; }
    const bool whole = KC ? (r < R && k + 3 < K) : (k < K && r + 3 < R);
    if (VEC && whole) {
      q[i] = __ldg(reinterpret_cast<const float4*>(KC ? X + r * ld + k : X + k * ld + r));
    } else {
      float v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t rr = KC ? r : r + j, kk = KC ? k + j : k;
        v[j] = (rr < R && kk < K) ? (KC ? X[rr * ld + kk] : X[kk * ld + rr]) : 0.0f;
      }
      q[i] = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
}

// registers -> the [k][r] shared-memory tile (transposing when k-contiguous)
template <bool KC>
__device__ __forceinline__ void sstore(float (*S)[LDS], const float4 q[2]) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    if (KC) {
      const int k = (tid & 3) * 4, c = ((tid >> 2) + 64 * i) ^ swz(k);
      S[k + 0][c] = q[i].x;
      S[k + 1][c] = q[i].y;
      S[k + 2][c] = q[i].z;
      S[k + 3][c] = q[i].w;
    } else {
      const int k = (tid >> 5) + 8 * i;
      *reinterpret_cast<float4*>(&S[k][((tid & 31) * 4) ^ swz(k)]) = q[i];
    }
  }
}

// Two fp32 FMAs in one instruction (Blackwell FFMA2, PTX fma.rn.f32x2): each half
// is an IEEE round-to-nearest fmaf, so results are bit-identical to scalar FFMAs,
// at half the issue slots -- an 8x8 FFMA micro-tile otherwise needs every issue
// slot of the SM sub-partition for the FMAs alone. ptxas folds the {a, a} pack
// into a broadcast operand (FFMA2 Rc, Ra.F32, Rb.F32x2, Rc.F32x2): no extra moves.
__device__ __forceinline__ void fma2(float2& c, float a, float2 b) {
  unsigned long long aa, bb, cc;
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(cc) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(cc) : "l"(aa), "l"(bb));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(c.x), "=f"(c.y) : "l"(cc));
}

// 128x128x16 CTA tile, 256 threads (2 CTAs per SM), 8x8 outputs per thread as
// four 4x4 quads 64 apart on each axis. A warp is 4 threads along m x 8 along n,
// so a k-step's fragment reads are 2 x 64 B of A and 2 x 128 B of B (one
// wavefront each) for 64 FFMAs per thread; the next k-tile's global loads are in
// flight in registers across the 16 k-steps, one __syncthreads per k-tile.
// Every output is a sequential fp32 fmaf chain over k = 0..K-1 (fixed order).
template <bool TA, bool TB, bool VEC>
__global__ void __launch_bounds__(256, 2) k_gemm_simt(int64_t M, int64_t N, int64_t K,
                                                      const float* __restrict__ A, int64_t lda,
                                                      const float* __restrict__ B, int64_t ldb,
                                                      float* __restrict__ C, int64_t ldc,
                                                      const float* __restrict__ bias, int epi) {
  __shared__ __align__(16) float As[2][BK][LDS];
  __shared__ __align__(16) float Bs[2][BK][LDS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // warp w: m-quads 4 * (w / 2) .. +3, n-quads 8 * (w % 2) .. +7
  // (2 x 16, 8 x 4 and the transposed 4 x 8 arrangements measured the same: every
  // 128-bit fragment read costs 3 shared-memory wavefronts whatever the lanes share)
  const int ty = (warp >> 1) * 4 + (lane >> 3), tx = (warp & 1) * 8 + (lane & 7);
  // grouped raster over a 1-D grid: tiles run down M inside groups of GW tile
  // columns, so the CTAs resident together (2 per SM) cover a ~16 x 18 block of
  // tiles -- each operand tile they fetch is shared by 16-18 of them in L2
  const int tiles_m = (int)((M + BM - 1) / BM), tiles_n = (int)((N + BN - 1) / BN);
  const int per_group = GW * tiles_m, g = blockIdx.x / per_group, t = blockIdx.x - g * per_group;
  const int gw = min(GW, tiles_n - g * GW);
  const int64_t m0 = (int64_t)(t / gw) * BM, n0 = (int64_t)(g * GW + t % gw) * BN;
  float2 acc[8][4];  // acc[i][j] = outputs (i, 2j) and (i, 2j + 1) of the micro-tile
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.0f, 0.0f);
  float4 qa[2], qb[2];
  gload<!TA, VEC>(A, lda, M, K, m0, 0, qa);
  gload<TB, VEC>(B, ldb, N, K, n0, 0, qb);
  sstore<!TA>(As[0], qa);
  sstore<TB>(Bs[0], qb);
  __syncthreads();
  const int nk = (int)((K + BK - 1) / BK);
  // interior CTAs (whole 128x128 tile inside the matrix) load whole k-tiles with
  // four unguarded 128-bit loads from pointers that advance by one k-tile
  const bool interior = VEC && m0 + BM <= M && n0 + BN <= N;
  const int nk_whole = (int)(K / BK);
  const float* pa = !TA ? A + (m0 + (tid >> 2)) * lda + (tid & 3) * 4
                        : A + (int64_t)(tid >> 5) * lda + m0 + (tid & 31) * 4;
  const float* pb = TB ? B + (n0 + (tid >> 2)) * ldb + (tid & 3) * 4
                       : B + (int64_t)(tid >> 5) * ldb + n0 + (tid & 31) * 4;
  const int64_t ha = (!TA ? 64 : 8) * lda, hb = (TB ? 64 : 8) * ldb;  // the thread's second quad
  const int64_t sa = !TA ? BK : BK * lda, sb = TB ? BK : BK * ldb;    // one k-tile ahead
  for (int kt = 0; kt < nk; ++kt) {
    const int cur = kt & 1;
    if (interior && kt + 1 < nk_whole) {
      pa += sa;
      pb += sb;
      qa[0] = __ldg(reinterpret_cast<const float4*>(pa));
      qa[1] = __ldg(reinterpret_cast<const float4*>(pa + ha));
      qb[0] = __ldg(reinterpret_cast<const float4*>(pb));
      qb[1] = __ldg(reinterpret_cast<const float4*>(pb + hb));
    } else if (kt + 1 < nk) {
      gload<!TA, VEC>(A, lda, M, K, m0, (int64_t)(kt + 1) * BK, qa);
      gload<TB, VEC>(B, ldb, N, K, n0, (int64_t)(kt + 1) * BK, qb);
    }
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[cur][k][(ty * 4) ^ swz(k)]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[cur][k][64 + ((ty * 4) ^ swz(k))]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[cur][k][(tx * 4) ^ swz(k)]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[cur][k][64 + ((tx * 4) ^ swz(k))]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                            make_float2(b1.z, b1.w)};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) fma2(acc[i][j], av[i], bv[j]);
    }
    if (kt + 1 < nk) {
      sstore<!TA>(As[cur ^ 1], qa);
      sstore<TB>(Bs[cur ^ 1], qb);
      __syncthreads();
    }
  }
  const bool vec_out = VEC && (ldc & 3) == 0 && ((uintptr_t)C & 15) == 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (m >= M) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t n = n0 + 64 * h + tx * 4;
      float v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[j] = (j & 1) ? acc[i][2 * h + j / 2].y : acc[i][2 * h + j / 2].x;
        if (n + j < N) {
          if (epi == B2_EPI_BIAS || epi == B2_EPI_BIAS_RELU) v[j] = __fadd_rn(v[j], bias[n + j]);
          if (epi == B2_EPI_BIAS_RELU || epi == B2_EPI_RELU) v[j] = v[j] > 0.0f ? v[j] : 0.0f;
        }
      }
      if (vec_out && n + 3 < N) {
        *reinterpret_cast<float4*>(&C[m * ldc + n]) = make_float4(v[0], v[1], v[2], v[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (n + j < N) C[m * ldc + n + j] = v[j];
      }
    }
  }
}

// ---------------------------------------------------------------- small / skinny GEMMs
// Latency path for problems whose 128x128 tiling leaves most SMs idle (BASELINE
// config 1: 256x256x784, 256x10x256, ...): 64x64x16 tiles, 4x4 outputs per
// thread, and the K loop split over S CTAs (grid.z). S > 1 writes fp32 partials
// [S][M][N] that k_splitk_reduce sums in fixed order s = 0..S-1 (deterministic)
// before the bias/ReLU epilogue.
constexpr int SBM = 64, SBN = 64, SBK = 16;

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_gemm_small(int64_t M, int64_t N, int64_t K, int64_t kslice,
                                                    const float* __restrict__ A, int64_t lda,
                                                    const float* __restrict__ B, int64_t ldb,
                                                    float* __restrict__ C, int64_t ldc,
                                                    const float* __restrict__ bias, int epi,
                                                    float* __restrict__ part) {
  __shared__ __align__(16) float As[2][SBK][SBM];
  __shared__ __align__(16) float Bs[2][SBK][SBN];
  const int t = threadIdx.x, tx = t % 16, ty = t / 16;
  const int64_t m0 = blockIdx.y * (int64_t)SBM, n0 = blockIdx.x * (int64_t)SBN;
  const int64_t kb = blockIdx.z * kslice, ke = min(K, kb + kslice);
  float acc[4][4] = {};
  float ra[4], rb[4];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int64_t m, k;
      if (!TA) { m = m0 + t / 4; k = k0 + (t % 4) * 4 + i; }
      else     { k = k0 + t / 16; m = m0 + (t % 16) * 4 + i; }
      ra[i] = (m < M && k < ke) ? (TA ? A[k * lda + m] : A[m * lda + k]) : 0.0f;
      int64_t n, kk;
      if (TB) { n = n0 + t / 4; kk = k0 + (t % 4) * 4 + i; }
      else    { kk = k0 + t / 16; n = n0 + (t % 16) * 4 + i; }
      rb[i] = (n < N && kk < ke) ? (TB ? B[n * ldb + kk] : B[kk * ldb + n]) : 0.0f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (!TA) As[buf][(t % 4) * 4 + i][t / 4] = ra[i];
      else     As[buf][t / 16][(t % 16) * 4 + i] = ra[i];
      if (TB)  Bs[buf][(t % 4) * 4 + i][t / 4] = rb[i];
      else     Bs[buf][t / 16][(t % 16) * 4 + i] = rb[i];
    }
  };
  const int nk = (int)((ke - kb + SBK - 1) / SBK);
  if (nk > 0) {
    load(kb);
    store(0);
  }
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nk) load(kb + (int64_t)(kt + 1) * SBK);
#pragma unroll
    for (int k = 0; k < SBK; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(&As[cur][k][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[cur][k][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < nk) {
      store(cur ^ 1);
      __syncthreads();
    }
  }
  const bool split = gridDim.z > 1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j];
      if (split) {
        part[(blockIdx.z * M + m) * N + n] = v;
        continue;
      }
      if (epi == B2_EPI_BIAS || epi == B2_EPI_BIAS_RELU) v = __fadd_rn(v, bias[n]);
      if (epi == B2_EPI_BIAS_RELU || epi == B2_EPI_RELU) v = v > 0.0f ? v : 0.0f;
      C[m * ldc + n] = v;
    }
  }
}

__global__ void k_splitk_reduce(float* __restrict__ C, int64_t ldc, const float* __restrict__ part,
                                int64_t M, int64_t N, int S, const float* __restrict__ bias, int epi) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M * N) return;
  const int64_t m = i / N, n = i - m * N;
  float v = 0.0f;
  for (int s = 0; s < S; ++s) v = __fadd_rn(v, part[s * M * N + i]);  // fixed order
  if (epi == B2_EPI_BIAS || epi == B2_EPI_BIAS_RELU) v = __fadd_rn(v, bias[n]);
  if (epi == B2_EPI_BIAS_RELU || epi == B2_EPI_RELU) v = v > 0.0f ? v : 0.0f;
  C[m * ldc + n] = v;
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
  const int64_t big_tiles = ((N + BN - 1) / BN) * ((M + BM - 1) / BM);
  if (big_tiles < sm_count() / 2) {
    // latency path: 64x64 tiles, K split so the grid covers ~2 CTAs per SM
    const int64_t tiles = ((N + SBN - 1) / SBN) * ((M + SBM - 1) / SBM);
    int64_t S = std::max<int64_t>(1, std::min<int64_t>((2 * sm_count()) / tiles, K / (4 * SBK)));
    S = std::min<int64_t>(S, 32);
    int64_t kslice = (K + S - 1) / S;
    kslice = (kslice + SBK - 1) / SBK * SBK;
    S = (K + kslice - 1) / kslice;
    dim3 g((unsigned)((N + SBN - 1) / SBN), (unsigned)((M + SBM - 1) / SBM), (unsigned)S);
    void* ws = nullptr;
    if (S > 1) B2_TRY(b2_alloc((size_t)S * M * N * sizeof(float), st, &ws));
    float* part = (float*)ws;
#define B2_SMALL(TA_, TB_) \
  k_gemm_small<TA_, TB_><<<g, 256, 0, st>>>(M, N, K, kslice, A, lda, B, ldb, C, ldc, bias, epi, part)
    if (!ta && !tb) B2_SMALL(false, false);
    else if (!ta && tb) B2_SMALL(false, true);
    else if (ta && !tb) B2_SMALL(true, false);
    else B2_SMALL(true, true);
#undef B2_SMALL
    int rc = launched("b2_gemm(simt-small)");
    if (!rc && S > 1) {
      k_splitk_reduce<<<(unsigned)((M * N + 255) / 256), 256, 0, st>>>(C, ldc, part, M, N, (int)S, bias, epi);
      rc = launched("b2_gemm(splitk-reduce)");
    }
    if (ws) b2_free(ws, st);
    return rc;
  }
  if (big_tiles > INT32_MAX) return fail("b2_gemm(simt): too many tiles for the SIMT grid");
  dim3 grid((unsigned)big_tiles);
  const bool vec = (lda & 3) == 0 && (ldb & 3) == 0 && (((uintptr_t)A | (uintptr_t)B) & 15) == 0;
#define B2_SIMT(TA_, TB_)                                                                      \
  do {                                                                                         \
    if (vec) k_gemm_simt<TA_, TB_, true><<<grid, 256, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, bias, epi);  \
    else k_gemm_simt<TA_, TB_, false><<<grid, 256, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, bias, epi); \
  } while (0)
  if (!ta && !tb) B2_SIMT(false, false);
  else if (!ta && tb) B2_SIMT(false, true);
  else if (ta && !tb) B2_SIMT(true, false);
  else B2_SIMT(true, true);
#undef B2_SIMT
  return launched("b2_gemm(simt)");
}

}  // namespace b2
