// FP32 SIMT GEMM (FFMA2, exact fp32 FMA chains): the FP32-pipe path of the matmul
// engine -- the north star's "FP32 SIMT" scheme, and the fallback for shapes the
// tcgen05 path does not take (tiny problems, operands whose leading dimension
// breaks TMA's 16-byte stride rule).
//
// Replaces matmul.block (tensorlite/core.py:802-807) and its pullbacks
// (core.py:815-817); the operand layouts of those pullbacks are template
// parameters, so transposed views are read in place, never copied.
// Many tiles: 128x128x16 CTA tiles, 256 threads x 8x8 outputs, 128-bit global
// loads staged through registers across the k-tile, double-buffered swizzled
// shared memory, grouped raster (k_gemm_simt). Few tiles: 64x64 tiles with K
// split over a thread-block cluster and folded through distributed shared
// memory (k_gemm_small).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"

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
// config 1: 256x256x784, 256x10x256, ...): 64x64 tiles, 4x4 outputs per thread
// (FFMA2), and the K loop split over the S <= 6 CTAs of a thread-block cluster
// (grid.z). A CTA stages its whole K slice (up to 112 k at a time) in shared
// memory with every global load issued before the first is consumed -- one
// memory latency per slice instead of one per k-tile -- and keeps its 64x64 fp32
// partial in shared memory; after a cluster barrier CTA r finishes its 1/S of the
// tile by reading the S partials through distributed shared memory, summed in
// slice order s = 0..S-1 (deterministic), then bias / ReLU and the store. No
// partials through L2, no second launch.
constexpr int SBM = 64, SBN = 64, SBK = 16, SKT = 7;  // SKT k-tiles (112 k) staged per pass

// one 64 x 16 operand sub-tile: a quad per thread (layouts as gload)
template <bool KC, bool VEC>
__device__ __forceinline__ float4 gload_small(const float* __restrict__ X, int64_t ld, int64_t R,
                                              int64_t kend, int64_t r0, int64_t k0) {
  const int tid = threadIdx.x;
  int64_t r, k;
  if (KC) { r = r0 + (tid >> 2); k = k0 + (tid & 3) * 4; }
  else    { k = k0 + (tid >> 4); r = r0 + (tid & 15) * 4; }
  const bool whole = KC ? (r < R && k + 3 < kend) : (k < kend && r + 3 < R);
  if (VEC && whole) return __ldg(reinterpret_cast<const float4*>(KC ? X + r * ld + k : X + k * ld + r));
  float v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t rr = KC ? r : r + j, kk = KC ? k + j : k;
    v[j] = (rr < R && kk < kend) ? (KC ? X[rr * ld + kk] : X[kk * ld + rr]) : 0.0f;
  }
  return make_float4(v[0], v[1], v[2], v[3]);
}

// into the [k][64] tile (swizzled like the big kernel's: conflict-free transposing stores)
template <bool KC>
__device__ __forceinline__ void sstore_small(float* S, int kt, const float4& q) {
  const int tid = threadIdx.x;
  if (KC) {
    const int k = (tid & 3) * 4, c = (tid >> 2) ^ swz(k);
    float* row = S + (kt * SBK + k) * SBM + c;
    row[0] = q.x;
    row[SBM] = q.y;
    row[2 * SBM] = q.z;
    row[3 * SBM] = q.w;
  } else {
    const int k = tid >> 4;
    *reinterpret_cast<float4*>(S + (kt * SBK + k) * SBM + (((tid & 15) * 4) ^ swz(k))) = q;
  }
}

__device__ __forceinline__ float4 ld_cluster_f4(const float* p, unsigned rank) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(ra)
               : "memory");
  return v;
}

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <bool TA, bool TB, bool VEC>
__global__ void __launch_bounds__(256) k_gemm_small(int64_t M, int64_t N, int64_t K, int64_t kslice,
                                                    const float* __restrict__ A, int64_t lda,
                                                    const float* __restrict__ B, int64_t ldb,
                                                    float* __restrict__ C, int64_t ldc,
                                                    const float* __restrict__ bias, int epi) {
  extern __shared__ __align__(16) float sm_small[];
  float* const As = sm_small;                     // [SKT * 16][64]
  float* const Bs = sm_small + SKT * SBK * SBM;   // [SKT * 16][64]
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int S = (int)gridDim.z, rank = (int)blockIdx.z;  // the cluster spans grid.z
  const int64_t m0 = blockIdx.y * (int64_t)SBM, n0 = blockIdx.x * (int64_t)SBN;
  const int64_t kb = rank * kslice, ke = min(K, kb + kslice);
  float2 acc[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = make_float2(0.0f, 0.0f);
  for (int64_t kc = kb; kc < ke; kc += SKT * SBK) {
    const int64_t left = (ke - kc + SBK - 1) / SBK;
    const int nkt = left < SKT ? (int)left : SKT;
    // (prefetching the next pass over this pass's FMAs measured slower: the 14 staged
    // quads then live across the FMA loop)
    float4 qa[SKT], qb[SKT];
#pragma unroll
    for (int i = 0; i < SKT; ++i)
      if (i < nkt) {
        qa[i] = gload_small<!TA, VEC>(A, lda, M, ke, m0, kc + i * SBK);
        qb[i] = gload_small<TB, VEC>(B, ldb, N, ke, n0, kc + i * SBK);
      }
    if (kc != kb) __syncthreads();  // the previous pass's tiles have been consumed
#pragma unroll
    for (int i = 0; i < SKT; ++i)
      if (i < nkt) {
        sstore_small<!TA>(As, i, qa[i]);
        sstore_small<TB>(Bs, i, qb[i]);
      }
    __syncthreads();
    for (int i = 0; i < nkt; ++i) {
      const float* ar = As + i * SBK * SBM;
      const float* br = Bs + i * SBK * SBM;
#pragma unroll
      for (int k = 0; k < SBK; ++k) {
        const float4 a = *reinterpret_cast<const float4*>(ar + k * SBM + ((ty * 4) ^ swz(k)));
        const float4 b = *reinterpret_cast<const float4*>(br + k * SBM + ((tx * 4) ^ swz(k)));
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float2 b01 = make_float2(b.x, b.y), b23 = make_float2(b.z, b.w);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          fma2(acc[r][0], av[r], b01);
          fma2(acc[r][1], av[r], b23);
        }
      }
    }
  }
  const bool vec_out = VEC && (ldc & 3) == 0 && ((uintptr_t)C & 15) == 0;
  auto finish = [&](int r, int c4, float4 v) {  // bias / ReLU epilogue + store of one quad
    const int64_t m = m0 + r, n = n0 + c4;
    if (m >= M) return;
    float o[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (n + j < N) {
        if (epi == B2_EPI_BIAS || epi == B2_EPI_BIAS_RELU) o[j] = __fadd_rn(o[j], bias[n + j]);
        if (epi == B2_EPI_BIAS_RELU || epi == B2_EPI_RELU) o[j] = o[j] > 0.0f ? o[j] : 0.0f;
      }
    if (vec_out && n + 3 < N) {
      *reinterpret_cast<float4*>(&C[m * ldc + n]) = make_float4(o[0], o[1], o[2], o[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (n + j < N) C[m * ldc + n + j] = o[j];
    }
  };
  if (S == 1) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
      finish(ty * 4 + r, tx * 4, make_float4(acc[r][0].x, acc[r][0].y, acc[r][1].x, acc[r][1].y));
    return;
  }
  // this CTA's partial tile, [64][64] row-major over the (consumed) A tiles
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 4; ++r)
    *reinterpret_cast<float4*>(As + (ty * 4 + r) * SBN + tx * 4) =
        make_float4(acc[r][0].x, acc[r][0].y, acc[r][1].x, acc[r][1].y);
  cluster_barrier();  // every slice's partial is staged and visible cluster-wide
  // CTA r finishes quads [r * Q, (r + 1) * Q) of the tile's 1024: the S remote
  // reads of a quad are issued together, then added in slice order
  const int Q = (SBM * (SBN / 4) + S - 1) / S;
  const int q_end = min((rank + 1) * Q, SBM * (SBN / 4));
  for (int qi = rank * Q + t; qi < q_end; qi += 256) {
    const int r = qi >> 4, c4 = (qi & 15) * 4;
    float4 p[8];
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2)
      if (s2 < S) p[s2] = ld_cluster_f4(As + r * SBN + c4, (unsigned)s2);
    float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2)
      if (s2 < S) {  // fixed slice order
        v.x = __fadd_rn(v.x, p[s2].x);
        v.y = __fadd_rn(v.y, p[s2].y);
        v.z = __fadd_rn(v.z, p[s2].z);
        v.w = __fadd_rn(v.w, p[s2].w);
      }
    finish(r, c4, v);
  }
  cluster_barrier();  // no CTA leaves while a peer still reads its partial
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
    // latency path: 64x64 tiles, K split over a cluster of S <= 6 CTAs so the grid
    // covers ~2 CTAs per SM (at least 64 k per slice)
    const int64_t tiles = ((N + SBN - 1) / SBN) * ((M + SBM - 1) / SBM);
    int64_t S = std::max<int64_t>(1, std::min<int64_t>((2 * sm_count()) / tiles, K / (4 * SBK)));
    // clusters of up to 6: 7 and 8 CTAs measured slower (256x256x784: 8.6 us at S = 6
    // with two staging passes per CTA, 9.9-10.3 us at S = 7 / 8 with one)
    S = std::min<int64_t>(S, 6);
    int64_t kslice = (K + S - 1) / S;
    kslice = (kslice + 3) / 4 * 4;  // slices start on 16-byte boundaries of k-contiguous rows
    S = (K + kslice - 1) / kslice;
    dim3 g((unsigned)((N + SBN - 1) / SBN), (unsigned)((M + SBM - 1) / SBM), (unsigned)S);
    if (g.y > 65535) return fail("b2_gemm(simt-small): M too large");
    const bool vec = (lda & 3) == 0 && (ldb & 3) == 0 && (((uintptr_t)A | (uintptr_t)B) & 15) == 0;
    constexpr int kSmem = 2 * SKT * SBK * SBM * (int)sizeof(float);  // 56 KB
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = (unsigned)S;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaSuccess;
#define B2_SMALL(TA_, TB_, V_)                                                                       \
  do {                                                                                               \
    static bool attr_set = false;                                                                    \
    if (!attr_set) {                                                                                 \
      B2_CUDA(cudaFuncSetAttribute(k_gemm_small<TA_, TB_, V_>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem)); \
      attr_set = true;                                                                               \
    }                                                                                                \
    e = cudaLaunchKernelEx(&cfg, k_gemm_small<TA_, TB_, V_>, M, N, K, kslice, A, lda, B, ldb, C, ldc, bias, epi); \
  } while (0)
#define B2_SMALL_V(TA_, TB_) \
  do { if (vec) B2_SMALL(TA_, TB_, true); else B2_SMALL(TA_, TB_, false); } while (0)
    if (!ta && !tb) B2_SMALL_V(false, false);
    else if (!ta && tb) B2_SMALL_V(false, true);
    else if (ta && !tb) B2_SMALL_V(true, false);
    else B2_SMALL_V(true, true);
    if (e != cudaSuccess && S > 1) {
      // the clusters could not be placed (MIG / MPS partitions): one CTA per tile
      // walks the whole K in staging passes, no cluster
      cudaGetLastError();
      S = 1;
      kslice = K;
      cfg.gridDim = dim3(g.x, g.y, 1);
      attr[0].val.clusterDim.z = 1;
      if (!ta && !tb) B2_SMALL_V(false, false);
      else if (!ta && tb) B2_SMALL_V(false, true);
      else if (ta && !tb) B2_SMALL_V(true, false);
      else B2_SMALL_V(true, true);
    }
#undef B2_SMALL_V
#undef B2_SMALL
    if (e != cudaSuccess) return cuda_fail(e, "b2_gemm(simt-small)");
    return launched("b2_gemm(simt-small)");
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
