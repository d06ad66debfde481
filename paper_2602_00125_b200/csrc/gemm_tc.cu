// tcgen05 / TMEM / TMA GEMM for sm_100a with fp32 accuracy.
//
// Replaces matmul.block (tensorlite/core.py:802-807) + pullbacks (:815-817)
// for every shape big enough to fill the chip. The reference computes each
// output as one double dot rounded to f32; the fp32 tolerance (1e-4, SURVEY
// 8a.3) rules out plain TF32 (~2.5e-4 normwise), so operands are split
// x = hi + lo and the tensor cores accumulate hi*hi + hi*lo + lo*hi:
//   3xBF16 (MODE 5, default): hi = bf16_rn(x), lo = bf16_rn(x - hi), three
//          kind::f16 MMAs per fp32 MAC (1.5 tf32-equivalents), ~5e-6 normwise;
//   TF32X  (MODE 2): the tf32 MMA reads the raw fp32 operand (the hardware
//          truncates to tf32, so hi = trunc(x)) and the two cross terms run as
//          kind::f16 MMAs on bf16(hi), bf16(lo): 2 tf32-equivalents, ~2e-6;
//   3xTF32 (MODE 3): three kind::tf32 MMAs on fp32 hi/lo arrays, ~1e-6;
//   1xTF32 (MODE 1, TF32 accuracy) and BF16 (MODE 4, the explicit bf16
//          variant) are single-MMA modes.
//
// Structure (persistent; one CTA per SM, CTA pairs for big problems):
//   warp 0      TMA producer: per k-block loads the mode's operand tiles
//               (cp.async.bulk.tensor, 128/64-byte swizzles, L2 cache hints)
//               into a ring of up to 8 stages
//   warp 1      MMA issuer (leader CTA): one thread issues the tcgen05.mma's
//               (M=128 per CTA or 256 per pair, N=256, K=8/16), tcgen05.commit
//               frees smem slots and hands K-chunks to the epilogue
//   warp 2      TMEM allocator (512 columns = two 128x256 fp32 accumulators,
//               ping-ponged per K-chunk: K = 1024 for the bf16 modes, 256 for tf32)
//   warps 4..19 epilogue: drain each K-chunk (tcgen05.ld) into RN fp32
//               running sums in registers while the MMAs fill the other
//               accumulator; after the last chunk +bias -> relu -> ReLU-pullback
//               mask -> stores (+ the result's own operand split for the next GEMM)
// The partial last wave (and few-tile long-K problems) split K over CTAs:
// fp32 partial slices, fixed-order second stage k_tail_epilogue. Operand majorness comes from the
// reference's three layouts: NT (forward, x.w^T), NN (x_bar = g.w), TN (w_bar
// = g^T.x): K-major tiles are one TMA box per operand; MN-major tiles are
// 128-byte-wide boxes laid side by side (UMMA LBO = box bytes).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"

extern "C" int b2_alloc(size_t, void*, void**);
extern "C" int b2_free(void*, void*);
extern "C" int b2_reduce(int, float*, int64_t*, int, const int64_t*, const float*, const int64_t*,
                         uint32_t, void*);

namespace {

// B2_GEMM_TRACE builds (scripts/gemm_trace.py, a separate library) stamp the
// global timer at the phases of every CTA's first unit -- where a few-tile
// GEMM's fixed cost goes. Not in the product library.
#ifdef B2_GEMM_TRACE
__device__ unsigned long long g_trace[1024][8];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define B2_TRACE(slot) g_trace[blockIdx.x & 1023][slot] = gtime()
#else
#define B2_TRACE(slot) ((void)0)
#endif

constexpr int BM = 128, BN = 256, BK = 32;  // BK fp32 = 128 bytes = one swizzle row
constexpr int kThreads = 640;  // 4 control warps + 16 epilogue warps
constexpr int KC_BASE = 8;     // k-blocks per accumulation chunk for the tf32 modes (K = 256)
constexpr int kTmemCols = 512;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---- cluster (CTA pair) helpers for cta_group::2
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of `local`'s twin in CTA `rank` of this cluster
__device__ __forceinline__ uint32_t mapa(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// 2-SM TMA: data lands in this CTA's smem, the transaction bytes are counted on
// the mbarrier at `bar_cluster` (the leader CTA's barrier)
__device__ __forceinline__ void tma_load_2d_cg2(void* dst, const CUtensorMap* tm, uint32_t bar_cluster,
                                                int c0, int c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)tm), "r"(bar_cluster), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0,
                                            int c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}

// L2 cache policies for the operand streams: the raster keeps a group of B
// panels hot across every wave of the group sweep (evict_last), A panels are
// shared only by the tiles of one wave (evict_normal)
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// commit this CTA pair's MMAs to the barrier at the same offset in both CTAs
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

template <int CG>
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accum, bool f16) {
  if (CG == 1) {
    if (f16)
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
          "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
          : "memory");
    else
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
          "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
          : "memory");
  } else {
    if (f16)
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
          "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
          : "memory");
    else
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
          "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
          : "memory");
  }
}

// UMMA shared-memory descriptor (sm_100): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version=1 [46,48), base_offset=0, layout type [61,64):
// SWIZZLE_128B=2 for K-major tiles; SWIZZLE_128B_BASE32B=1 for MN-major tf32
// tiles (the only MN-major layout kind::tf32 accepts: 32-B chunks swizzled
// within 128-B rows, 4-row atoms).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// 32 lanes x 32 bit x 16 columns of TMEM -> 16 registers per thread
#define TMEM_LD16(taddr, v)                                                                        \
  asm volatile(                                                                                    \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "                                                   \
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"                           \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),       \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),   \
        "=r"(v[14]), "=r"(v[15])                                                                   \
      : "r"(taddr))

// instruction descriptor: D=F32 [4,6), A/B format [7,10)/[10,13) (TF32=2, BF16=1),
// a_major [15], b_major [16], N>>3 [17,23), M>>4 [24,29). M = 128 per CTA (256 per pair).
__host__ __device__ constexpr uint32_t make_idesc(bool f16, bool a_mn, bool b_mn, int m) {
  return (1u << 4) | ((f16 ? 1u : 2u) << 7) | ((f16 ? 1u : 2u) << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

struct TcParams {
  float* C;
  const float* bias;
  int64_t ldc;
  int M, N, K;
  int epi;
  int tiles_n, num_tiles;  // tiles of BM*CG x BN
  int tiles_m;
  // optional fused epilogue stages (MLP backward / forward chaining):
  const float* mask;        // C = C * (mask > 0 ? 1 : 0), mask [M, N] with ld = ldc (ReLU pullback)
  __nv_bfloat16* s_hi;      // emit the TF32X split of C: bf16(trunc_tf32(C)) ...
  __nv_bfloat16* s_lo;      // ... and bf16(C - trunc_tf32(C)), both [M, N] contiguous
  int group_n;              // raster group width in tile-columns
  // work units: units [0, full_tiles) are whole tiles (all of K); the rest
  // split the remaining tail tiles into `splits` K slices of kbps k-blocks
  // (slices slowest), whose fp32 partials go to ws (tile-local, BM*CG x BN
  // each) for k_tail_epilogue. full_tiles = whole waves of the persistent
  // grid, so the last, partial wave runs on all SMs in thinner K slices.
  int full_tiles;
  int splits;
  int kbps;
  float* ws;
  int nkb;                  // k-blocks of K
  double* colsum;           // optional [ceil(M/128)][N] fp64 column partial sums of the stored C
  const uint64_t* mask_bits;  // ReLU-pullback mask as bits ([M][bits_ld] words, bit j = column 64w+j)
  uint64_t* bits_out;         // emit C > 0 as bits (ReLU forward): the next backward's mask
  int bits_ld;                // words per row of both bit arrays = ceil(N / 64)
  int a_mn, b_mn;             // operand layouts: A stored [K,M] (MN-major) / B stored [K,N]
};

// Epilogue stores of outputs that are read next as another launch's operand
// (too large to stay in L2): with G.l2hint & 4 they go out as cache-streaming
// stores (L2 evict-first), so they do not push the raster's A / B panels out.
__device__ __forceinline__ void st_out16(void* p, uint4 v, bool cs) {
  if (cs)
    asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  else
    *reinterpret_cast<uint4*>(p) = v;
}


// One launch runs up to kMaxProb independent problems of one mode (the dX and
// dW GEMMs of a pullback): their work units are numbered back to back
// (problem g owns units [ustart[g], ustart[g+1])). Every CTA (pair) takes
// units from a ring in shared memory that its producer thread fills: with
// sched == nullptr unit i of cluster c is c + i * clusters (the static
// persistent raster of a single problem); otherwise the producer draws units
// from an atomic counter (sched[0]; sched[1] counts finished clusters, the
// last one re-zeroes both), so problems whose units differ in cost (long-K dW
// slices first, then dX tiles) balance dynamically. Which CTA computes a unit
// never changes its result (K-slice partials have fixed slots, folded in
// slice order): deterministic either way.
constexpr int kMaxProb = 3;
// Unit ids published ahead of the consumers. The ring needs no "slot free"
// barrier: every consumer is within 2 + STAGES + 1 units of the producer
// (the producer publishes unit k+1 only after issuing unit k-1's loads, which
// needs all but STAGES k-blocks consumed by the MMAs; the MMAs of unit m
// need the epilogue warps of both CTAs to have drained up to unit m-2; the
// peer's loads gate the leader's MMAs), so with STAGES <= 8 a ring of 16
// never overwrites an id a consumer has yet to read -- and a consumer's
// release would cost a memory barrier behind its own global stores.
constexpr int kUnitRing = 16;
struct TcGroup {
  TcParams p[kMaxProb];
  int nprob;
  int ustart[kMaxProb + 1];
  int num_units;
  unsigned* sched;
  int kc;         // k-blocks per fp32 promotion chunk
  int l2hint;     // B operand loads with L2 evict_last (B2_GEMM_L2HINT=0 disables)
  int stage_out;  // every CTA runs at most one unit: fp32 tile stores go through shared memory
  int csplit;     // > 1: cluster split-K -- the S CTAs of a cluster compute the S K slices of one
                  // tile and fold them through distributed shared memory (no partials, no second
                  // kernel); every CTA runs exactly one unit
};
struct TcMaps {
  CUtensorMap m[kMaxProb][6];  // per problem: MODE 1 {A, B}; 3/5 {A, B, Alo, Blo}; 2 {A, B, Ah, Bh, Al, Bl}; 4 {A, B}
};

// unit u -> (output tile, k-block range, partial slot); slot -1 = a whole
// tile finished in the fused epilogue, else the unit's index into ws
__device__ __forceinline__ void tile_coords(const TcParams& p, int t, int& tm, int& tn);
__device__ __forceinline__ void tile_info(const TcParams& p, int u, int& tm, int& tn, int& kb0,
                                          int& kb1, int& slot) {
  const int nkb = p.nkb;
  if (u < p.full_tiles) {
    tile_coords(p, u, tm, tn);
    kb0 = 0;
    kb1 = nkb;
    slot = -1;
    return;
  }
  const int tail = p.tiles_m * p.tiles_n - p.full_tiles;
  slot = u - p.full_tiles;
  const int ks = slot / tail;
  tile_coords(p, p.full_tiles + (slot - ks * tail), tm, tn);
  kb0 = ks * p.kbps;
  kb1 = min(nkb, kb0 + p.kbps);
}

// Grouped raster: tiles walk M inside groups of kGroupN tile-columns, so the
// ~74-148 tiles resident at once cover a ~9 x 8 block of the output and the
// B panels of a group stay in L2 across waves (the plain row-major order
// re-read all of B from DRAM every wave: 12.8 GB/launch for 3.4 GB of data).
constexpr int kGroupN = 8;  // default group width (B2_GEMM_GROUPN overrides, p.group_n)
__device__ __forceinline__ void tile_coords(const TcParams& p, int t, int& tm, int& tn) {
  const int gn = p.group_n;
  const int group = gn * p.tiles_m;
  const int g = t / group, r = t - g * group;
  const int w = min(gn, p.tiles_n - g * gn);
  tm = r / w;
  tn = g * gn + (r - tm * w);
}

// MODE 1: 1xTF32            tiles A32 | B32
// MODE 3: 3xTF32            tiles Ahi | Alo | Bhi | Blo (fp32 arrays, hi = tf32(x))
// MODE 2: TF32 + 2xBF16     tiles A32 | B32 | Ah16 | Al16 | Bh16 | Bl16: the main
//         product runs on the raw fp32 operands (the tensor core truncates them
//         to tf32: hi = trunc(x), probed on B200) and the two cross terms
//         hi*lo + lo*hi run as kind::f16 MMAs on bf16(hi), bf16(lo) at twice the
//         tf32 rate -- 2 tf32-equivalents per fp32 MAC instead of 3.
// MODE 4: BF16 (explicit bf16 variant) tiles Ah16 | Bh16, one kind::f16 MMA per MAC.
// MODE 5: 3xBF16            tiles Ah16 | Al16 | Bh16 | Bl16 with hi = bf16_rn(x),
//         lo = bf16_rn(x - hi) (16 significant bits): hi*hi + hi*lo + lo*hi, all
//         kind::f16 -- 3 bf16 MMAs per fp32 MAC (1.5 tf32-equivalents) on half
//         MODE 2's operand bytes; normwise error ~4e-6 against the 1e-4 contract.
// CG 1: one CTA computes a 128x256 tile. CG 2: a CTA pair (cluster of 2)
//         computes 256x256 with tcgen05 cta_group::2: each CTA holds its 128
//         rows of A and HALF (128 rows) of B, the leader issues M=256 MMAs that
//         read both CTAs' smem -- per-SM operand ingress drops by a third.
template <int MODE, int CG>
struct Cfg {
  static constexpr int BNL = BN / CG;      // B rows loaded per CTA
  // k-block depth: 32 for every mode that stages fp32 tiles (128-B rows), 64
  // for the pure-bf16 modes (128-B rows of bf16, SW128): twice the MMAs per
  // barrier round trip
  static constexpr bool W64 = MODE == 4 || MODE == 5 || MODE == 6;
  static constexpr int BKM = W64 ? 64 : BK;
  // MODE 6 (bf16 variant, 512-row pair tiles): each CTA holds two 128-row
  // blocks of A and the pair issues two M=256 MMAs per k-step into TMEM
  // columns [0, 256) and [256, 512) -- a quarter fewer operand bytes per MAC
  // (the bf16 mode is bound by the ~43 B/clk of shared-memory ingress per SM);
  // the single 512-column accumulator is not double-buffered
  static constexpr int RM = MODE == 6 ? 2 : 1;
  static constexpr int A32 = BM * BK * 4;  // 16 KB
  static constexpr int B32 = BNL * BK * 4;
  static constexpr int A16 = BM * BKM * 2;
  static constexpr int B16 = BNL * BKM * 2;
  static constexpr int STAGE_BYTES =
      MODE == 1 ? A32 + B32
      : MODE == 3 ? 2 * (A32 + B32)
      : MODE == 4 ? A16 + B16
      : MODE == 6 ? 2 * A16 + B16
      : MODE == 5 ? 2 * (A16 + B16)
                  : A32 + B32 + 2 * (A16 + B16);
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 8 ? 8 : (200 * 1024) / STAGE_BYTES;
  // + the column-sum exchange (4 column groups x 4 warps x 64 doubles)
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 512 /*barriers, unit ring*/ + 8192;
  // byte offsets inside a stage
  static constexpr int OFF_A = 0;
  static constexpr int OFF_ALO = A32;                                 // MODE 3
  static constexpr int OFF_B = MODE == 3 ? 2 * A32 : A32;
  static constexpr int OFF_BLO = 2 * A32 + B32;                       // MODE 3
  static constexpr int F32 = (MODE == 4 || MODE == 5 || MODE == 6) ? 0 : A32 + B32;  // fp32 part (MODE 2)
  static constexpr int OFF_AH16 = F32;                                // MODE 2 / 4 / 5 / 6 (block 0)
  static constexpr int OFF_AL16 = F32 + A16;                          // MODE 2 / 5; MODE 6: block 1
  static constexpr int OFF_BH16 = MODE == 4 ? A16 : F32 + 2 * A16;
  static constexpr int OFF_BL16 = F32 + 2 * A16 + B16;
};

// Loads a tile into this CTA's smem, counting bytes on `bar` (a local
// barrier for CG 1, the leader's barrier as a shared::cluster address for CG 2).
template <int CG>
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* tm, uint64_t* bar, uint32_t bar_cl,
                                      int c0, int c1, uint64_t pol) {
  if (CG == 1)
    tma_load_2d(dst, tm, bar, c0, c1, pol);
  else
    tma_load_2d_cg2(dst, tm, bar_cl, c0, c1, pol);
}

// fp32 tile (tf32 consumption): K-major = one box {32 K, rows}; MN-major = 32x32 boxes
template <int ROWS, int CG>
__device__ __forceinline__ void load32(bool mn, uint8_t* dst, const CUtensorMap* tm, uint64_t* bar,
                                       uint32_t bar_cl, int mn0, int k0, uint64_t pol) {
  if (mn) {
#pragma unroll
    for (int j = 0; j < ROWS / 32; ++j) tma2d<CG>(dst + j * 4096, tm, bar, bar_cl, mn0 + 32 * j, k0, pol);
  } else {
    tma2d<CG>(dst, tm, bar, bar_cl, k0, mn0, pol);
  }
}

// bf16 tile: K-major = one box {KB K, rows}; MN-major = boxes {64 MN (128 B), KB K}
// (KB = 32 with 64-B rows in MODE 2, 64 with 128-B rows in the pure-bf16 modes)
template <int ROWS, int CG, int KB = 32>
__device__ __forceinline__ void load16(bool mn, uint8_t* dst, const CUtensorMap* tm, uint64_t* bar,
                                       uint32_t bar_cl, int mn0, int k0, uint64_t pol) {
  if (mn) {
#pragma unroll
    for (int j = 0; j < ROWS / 64; ++j)
      tma2d<CG>(dst + j * (KB * 128), tm, bar, bar_cl, mn0 + 64 * j, k0, pol);
  } else {
    tma2d<CG>(dst, tm, bar, bar_cl, k0, mn0, pol);
  }
}

// UMMA descriptors for one k-step
__device__ __forceinline__ uint64_t desc32(uint32_t base, bool mn, int ks) {
  // tf32, K=8 per MMA. K-major: 128-B swizzle, +32 B per k-step, SBO 8 rows x 128 B.
  // MN-major: 128-B/32-B-atom swizzle, +8 rows x 128 B per k-step, LBO = next
  // 32-element box (4 KB), SBO = next 4-row atom (512 B).
  return mn ? umma_desc(base + ks * 1024, 4096, 512, 1) : umma_desc(base + ks * 32, 16, 1024, 2);
}
template <int KB = 32>
__device__ __forceinline__ uint64_t desc16(uint32_t base, bool mn, int ks) {
  // bf16, K=16 per MMA. KB = 32: K-major 64-B swizzle (rows of 32 bf16), +32 B
  // per k-step, SBO 8 rows x 64 B. KB = 64: K-major 128-B swizzle (rows of 64
  // bf16), +32 B per k-step, SBO 8 rows x 128 B. MN-major: 128-B swizzle, +16
  // rows x 128 B per k-step, LBO = next 64-element box (KB x 128 B), SBO 8 x 128 B.
  if (mn) return umma_desc(base + ks * 2048, KB * 128, 1024, 2);
  return KB == 64 ? umma_desc(base + ks * 32, 16, 1024, 2) : umma_desc(base + ks * 32, 16, 512, 4);
}

// operand split written by the epilogue for the next GEMM: TF32X (MODE 2)
// = bf16(trunc_tf32(x)), bf16(x - trunc_tf32(x)); 3xBF16 (MODE 5) = hi =
// bf16_rn(x), lo = bf16_rn(x - hi). Same arithmetic as the split kernels.
template <int MODE>
__device__ __forceinline__ void split_pair(float x, __nv_bfloat16& h, __nv_bfloat16& l) {
  if (MODE == 5) {
    h = __float2bfloat16_rn(x);
    l = __float2bfloat16_rn(__fsub_rn(x, __bfloat162float(h)));
  } else {
    const float t = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    h = __float2bfloat16_rn(t);
    l = __float2bfloat16_rn(__fsub_rn(x, t));
  }
}

// Two elements at once (packed F2FP conversions): the same bits as two
// split_pair calls, packed as bf16x2 words (element a in the low half).
template <int MODE>
__device__ __forceinline__ void split_pair2(float a, float b, uint32_t& h, uint32_t& l) {
  float ta = a, tb = b;
  if (MODE != 5) {
    ta = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
    tb = __uint_as_float(__float_as_uint(b) & 0xFFFFE000u);
  }
  const __nv_bfloat162 hh = __floats2bfloat162_rn(ta, tb);
  const float ha = MODE == 5 ? __low2float(hh) : ta;
  const float hb = MODE == 5 ? __high2float(hh) : tb;
  const __nv_bfloat162 ll = __floats2bfloat162_rn(__fsub_rn(a, ha), __fsub_rn(b, hb));
  h = *reinterpret_cast<const uint32_t*>(&hh);
  l = *reinterpret_cast<const uint32_t*>(&ll);
}

// Coalesced fp32 tile store for CTAs that run a single unit (few-tile GEMMs,
// where the epilogue is exposed): each epilogue thread owns one row and 64
// columns, so direct stores are 32 rows x 16 B per warp instruction (one L2
// transaction per row). Instead the 16 epilogue warps stage the 128 x 256 tile
// in the (now idle) pipeline buffers -- rows padded to 260 floats, so a warp's
// 16-B writes hit the minimum 4 wavefronts -- then store whole rows, 1 KB per
// warp instruction pair. Named barrier 5 spans the 512 epilogue threads.
constexpr int kStageLd = BN + 4;
__device__ __forceinline__ void stage_tile_store(uint8_t* smem, const float (&acc)[64], int row, int cg,
                                                 int warp, int lane, float* dst, int64_t ld, int rows,
                                                 int cols) {
  float* t = reinterpret_cast<float*>(smem);
  float* mine = t + row * kStageLd + cg * 64;
#pragma unroll
  for (int j = 0; j < 64; j += 4)
    *reinterpret_cast<float4*>(mine + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
  asm volatile("bar.sync 5, 512;" ::: "memory");
  const int ew = warp - 4;  // 0..15
  const bool vec = (ld % 4) == 0 && (((uintptr_t)dst) & 15) == 0;
  for (int r = ew; r < rows; r += 16) {
    const float* src = t + r * kStageLd;
    float* out = dst + (int64_t)r * ld;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = (h * 32 + lane) * 4;
      if (vec && c + 4 <= cols) {
        *reinterpret_cast<float4*>(out + c) = *reinterpret_cast<const float4*>(src + c);
      } else {
        for (int q = 0; q < 4; ++q)
          if (c + q < cols) out[c + q] = src[c + q];
      }
    }
  }
  asm volatile("bar.sync 5, 512;" ::: "memory");  // the buffer may be reused by the next store
}

// ---- unit ring (see TcGroup): shared::cluster store + cluster-scope waits
__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// The MMAs of one k-block (stage at shared address s0) for one operand
// layout; acc_flag = 0 starts a new accumulation chunk.
template <int MODE, int CG, bool A_MN, bool B_MN>
__device__ __forceinline__ void mma_kblock(uint32_t d_tmem, uint32_t s0, uint32_t acc_flag,
                                           int blocks = 3 /* MODE 6: bit b = row block b */) {
  using CF = Cfg<MODE, CG>;
  constexpr uint32_t id32 = make_idesc(false, A_MN, B_MN, BM * CG);
  constexpr uint32_t id16 = make_idesc(true, A_MN, B_MN, BM * CG);
  if (MODE == 4 || MODE == 6) {
#pragma unroll
    for (int b = 0; b < CF::RM; ++b)
      if (CF::RM == 1 || ((blocks >> b) & 1))
#pragma unroll
        for (int ks = 0; ks < CF::BKM / 16; ++ks)
          tc_mma<CG>(d_tmem + b * BN, desc16<CF::BKM>(s0 + CF::OFF_AH16 + b * CF::A16, A_MN, ks),
                     desc16<CF::BKM>(s0 + CF::OFF_BH16, B_MN, ks), id16, (acc_flag | ks) ? 1u : 0u, true);
  }
  if (MODE == 5) {
#pragma unroll
    for (int ks = 0; ks < CF::BKM / 16; ++ks) {
      const uint64_t ah = desc16<CF::BKM>(s0 + CF::OFF_AH16, A_MN, ks);
      const uint64_t bh = desc16<CF::BKM>(s0 + CF::OFF_BH16, B_MN, ks);
      tc_mma<CG>(d_tmem, ah, bh, id16, (acc_flag | ks) ? 1u : 0u, true);
      tc_mma<CG>(d_tmem, ah, desc16<CF::BKM>(s0 + CF::OFF_BL16, B_MN, ks), id16, 1u, true);
      tc_mma<CG>(d_tmem, desc16<CF::BKM>(s0 + CF::OFF_AL16, A_MN, ks), bh, id16, 1u, true);
    }
  }
#pragma unroll
  for (int ks = 0; ks < ((MODE == 4 || MODE == 5 || MODE == 6) ? 0 : BK / 8); ++ks) {
    const uint64_t a = desc32(s0 + CF::OFF_A, A_MN, ks);
    const uint64_t b = desc32(s0 + CF::OFF_B, B_MN, ks);
    tc_mma<CG>(d_tmem, a, b, id32, (acc_flag | ks) ? 1u : 0u, false);
    if (MODE == 3) {
      tc_mma<CG>(d_tmem, a, desc32(s0 + CF::OFF_BLO, B_MN, ks), id32, 1u, false);
      tc_mma<CG>(d_tmem, desc32(s0 + CF::OFF_ALO, A_MN, ks), b, id32, 1u, false);
    }
  }
  if (MODE == 2) {
#pragma unroll
    for (int ks = 0; ks < BK / 16; ++ks) {
      tc_mma<CG>(d_tmem, desc16(s0 + CF::OFF_AH16, A_MN, ks), desc16(s0 + CF::OFF_BL16, B_MN, ks), id16,
                 1u, true);
      tc_mma<CG>(d_tmem, desc16(s0 + CF::OFF_AL16, A_MN, ks), desc16(s0 + CF::OFF_BH16, B_MN, ks), id16,
                 1u, true);
    }
  }
}

__device__ __forceinline__ float ld_dsmem_f32(uint32_t cluster_addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(cluster_addr) : "memory");
  return v;
}
__device__ __forceinline__ double ld_dsmem_f64(uint32_t cluster_addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(cluster_addr) : "memory");
  return v;
}

// Cluster split-K (TcGroup::csplit = S): every CTA of the cluster staged its
// K slice's fp32 partial tile (rows padded to kStageLd) at the start of its
// shared memory; CTA `krank` finishes rows [krank*128/S, +128/S) of the tile:
// the S partials added in slice order (as k_tail_epilogue adds them), then
// k_tail_epilogue's epilogue stages, with its 8-row groups and fixed-order
// fp64 column sums -- the fold of the 16 group sums per column is done by
// krank 0 (csplit_colsum) -- so outputs are bit-identical to the partials +
// second-stage path. Epilogue warps only (512 threads; ew = warp - 4).
template <int EMIT, int S>
__device__ __forceinline__ void csplit_reduce(const TcParams& p, uint8_t* smem, int tm, int tn,
                                              int krank, int ew, int lane) {
  constexpr int RPG = 8;  // rows per group (k_tail_epilogue: BM / 16)
  const int R = BM / S, ngroups = R / RPG;
  const int r0 = krank * R;
  const int64_t m0 = (int64_t)tm * BM, n0 = (int64_t)tn * BN;
  uint32_t base[S];
#pragma unroll
  for (int s2 = 0; s2 < S; ++s2) base[s2] = mapa(smem_u32(smem), (uint32_t)s2);
  double* gsum = reinterpret_cast<double*>(smem + BM * kStageLd * 4);  // [16 groups][BN]
  uint32_t* bits32 = reinterpret_cast<uint32_t*>(p.bits_out);
  const uint32_t* mbits32 = reinterpret_cast<const uint32_t*>(p.mask_bits);
  // a lane owns 4 consecutive columns (16-B distributed shared memory loads:
  // the cluster network is request-bound, 4-B loads ran at ~14 GB/s per SM);
  // a warp covers a 128-column strip of one 8-row group
  constexpr int STRIPS = BN / 128;
  for (int it = ew; it < ngroups * STRIPS; it += 16) {
    const int grp = it / STRIPS, strip = it % STRIPS;
    const int c = strip * 128 + lane * 4;
    const int64_t n = n0 + c;
    bool cok[4];
    float bias[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      cok[k] = n + k < p.N;
      bias[k] = (cok[k] && (p.epi == B2_EPI_BIAS || p.epi == B2_EPI_BIAS_RELU)) ? p.bias[n + k] : 0.0f;
    }
    const bool vec = cok[3] && (p.ldc % 4) == 0 && ((((uintptr_t)p.C) + 4 * (n + m0 * p.ldc)) & 15) == 0;
    double cs[4] = {0.0, 0.0, 0.0, 0.0};
    const int rbase = r0 + grp * RPG;
#pragma unroll 2
    for (int q = 0; q < RPG; ++q) {
      const int64_t m = m0 + rbase + q;
      if (m >= p.M) break;
      float4 v[S];  // the row's S partials in flight, added in slice order
#pragma unroll
      for (int s2 = 0; s2 < S; ++s2) {
        const uint32_t a = base[s2] + (uint32_t)((rbase + q) * kStageLd + c) * 4u;
        asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v[s2].x), "=f"(v[s2].y), "=f"(v[s2].z), "=f"(v[s2].w)
                     : "r"(a)
                     : "memory");
      }
      float x[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int s2 = 0; s2 < S; ++s2) {
        x[0] = __fadd_rn(x[0], v[s2].x);
        x[1] = __fadd_rn(x[1], v[s2].y);
        x[2] = __fadd_rn(x[2], v[s2].z);
        x[3] = __fadd_rn(x[3], v[s2].w);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (p.epi == B2_EPI_BIAS || p.epi == B2_EPI_BIAS_RELU) x[k] = __fadd_rn(x[k], bias[k]);
        if (p.epi == B2_EPI_BIAS_RELU || p.epi == B2_EPI_RELU) x[k] = x[k] > 0.0f ? x[k] : 0.0f;
      }
      if (bits32) {  // 8 lanes x 4 columns = one 32-bit word of y > 0
        uint32_t nib = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) nib |= (cok[k] && x[k] > 0.0f ? 1u : 0u) << k;
        uint32_t word = nib << (4 * (lane & 7));
        word |= __shfl_xor_sync(0xffffffffu, word, 1);
        word |= __shfl_xor_sync(0xffffffffu, word, 2);
        word |= __shfl_xor_sync(0xffffffffu, word, 4);
        const int64_t wn = (n0 + strip * 128 + (lane & ~7) * 4) >> 5;
        if ((lane & 7) == 0 && wn < 2 * (int64_t)p.bits_ld) bits32[m * 2 * p.bits_ld + wn] = word;
      }
      if (mbits32) {
        const uint32_t w = mbits32[m * 2 * p.bits_ld + (n >> 5)];
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = __fmul_rn(x[k], (w >> ((n + k) & 31)) & 1 ? 1.0f : 0.0f);
      } else if (p.mask) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (cok[k]) x[k] = __fmul_rn(x[k], p.mask[m * p.ldc + n + k] > 0.0f ? 1.0f : 0.0f);
      }
      if (p.C) {
        if (vec) {
          *reinterpret_cast<float4*>(p.C + m * p.ldc + n) = make_float4(x[0], x[1], x[2], x[3]);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (cok[k]) p.C[m * p.ldc + n + k] = x[k];
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (!cok[k]) continue;
        if (EMIT == 4 && p.s_hi) p.s_hi[m * p.N + n + k] = __float2bfloat16_rn(x[k]);
        if ((EMIT == 2 || EMIT == 5) && p.s_hi)
          split_pair<EMIT>(x[k], p.s_hi[m * p.N + n + k], p.s_lo[m * p.N + n + k]);
        cs[k] += (double)x[k];
      }
    }
    if (p.colsum) {
#pragma unroll
      for (int k = 0; k < 4; ++k) gsum[(krank * ngroups + grp) * BN + c + k] = cs[k];
    }
  }
}

// krank 0 of a cluster split-K tile: the tile's 128-row block column sums,
// the 16 group sums folded in group order across the cluster's CTAs.
__device__ __forceinline__ void csplit_colsum(const TcParams& p, uint8_t* smem, int tm, int tn, int S,
                                              int tid) {
  const int ngroups = BM / S / 8;
  const int64_t m0 = (int64_t)tm * BM, n0 = (int64_t)tn * BN;
  if (m0 >= p.M) return;
  const uint32_t goff = (uint32_t)(BM * kStageLd * 4);
  for (int c = tid; c < BN; c += 512) {
    const int64_t n = n0 + c;
    if (n >= p.N) continue;
    double v[16];  // all 16 group sums in flight, folded in group order
#pragma unroll
    for (int g = 0; g < 16; ++g)
      v[g] = ld_dsmem_f64(mapa(smem_u32(smem) + goff, (uint32_t)(g / ngroups)) + (uint32_t)((g * BN + c) * 8));
    double t = v[0];
#pragma unroll
    for (int g = 1; g < 16; ++g) t += v[g];
    p.colsum[(m0 / BM) * p.N + n] = t;
  }
}

// problem of unit u (MULTI = false: a single-problem launch, problem 0 with
// every parameter at a static offset)
template <bool MULTI>
__device__ __forceinline__ int prob_of(const TcGroup& G, int u) {
  if (!MULTI) return 0;
  int g = 0;
  while (g + 1 < G.nprob && u >= G.ustart[g + 1]) ++g;
  return g;
}

// cluster split-K: the unit of CTA b -- cluster b / S takes the cluster-th
// tile of the launch (problems back to back), its CTA of rank r the r-th K
// slice (units of a split problem are numbered slice-major)
__device__ __forceinline__ int csplit_unit(const TcGroup& G, int b) {
  const int S = G.csplit;
  int c = b / S;
  const int r = b - c * S;
  for (int g = 0; g < G.nprob; ++g) {
    const int tiles = G.p[g].tiles_m * G.p[g].tiles_n;
    if (c < tiles) return G.ustart[g] + r * tiles + c;
    c -= tiles;
  }
  return G.num_units;
}

template <int MODE, int CG, bool MULTI>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_tc(const __grid_constant__ TcMaps tmaps, const __grid_constant__ TcGroup G) {
  using CF = Cfg<MODE, CG>;
  constexpr int STAGES = CF::STAGES;
  // bf16 operands carry 2^-9 relative error: promote every K = 1024 instead
  const int KC = G.kc;  // k-blocks per accumulation chunk (host: kc_for_mode)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + STAGES * CF::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * STAGES + 4);
  uint64_t* ufull = bars + 2 * STAGES + 5;
  int* uring = (int*)(ufull + kUnitRing);
  double* colsum_smem = (double*)(smem + STAGES * CF::STAGE_BYTES + 512);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) B2_TRACE(0);  // entry
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  const bool leader = rank == 0;
  const int cl_id = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int cl_num = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int num_units = G.num_units;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 16 * CG);  // every epilogue warp of the pair drains before reuse
    }
    for (int s = 0; s < kUnitRing; ++s) mbar_init(&ufull[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int g = 0; g < (MULTI ? G.nprob : 1); ++g) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmaps.m[g][0]) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmaps.m[g][1]) : "memory");
    }
  }
  if (warp == 2) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();  // peer barriers initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: everything above (barrier init, TMEM
  // allocation, descriptor prefetch) may overlap the previous kernel's tail;
  // no global memory is touched before the prerequisite grids are complete.
  // Then let the next kernel start its own prologue as SMs free up.
  if (threadIdx.x == 0) B2_TRACE(1);  // prologue done (barriers, TMEM)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0) B2_TRACE(2);  // prerequisite grids complete

  // consumer side of the unit ring: unit i of this cluster (see kUnitRing)
  auto take = [&](int i) -> int {
    const int slot = i & (kUnitRing - 1);
    const uint32_t ph = (uint32_t)(i / kUnitRing) & 1u;
    if (CG == 2 && !leader)
      mbar_wait_cl(&ufull[slot], ph);
    else
      mbar_wait(&ufull[slot], ph);
    return *(volatile int*)&uring[slot];
  };

  int cs_unit = -1;  // cluster split-K: this CTA's unit (epilogue warps)
  if (warp == 0) {
    // ------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t pa = (G.l2hint & 3) == 2 ? l2_policy_first() : l2_policy_normal();
      const uint64_t pb = (G.l2hint & 3) ? l2_policy_last() : pa;
      auto produce = [&](int u) {
        const int gi = prob_of<MULTI>(G, u);
        const TcParams& p = G.p[gi];
        const CUtensorMap* mp = &tmaps.m[gi][0];
        const bool amn = p.a_mn != 0, bmn = p.b_mn != 0;
        int tm, tn, kb0, kb1, ks;
        tile_info(p, u - G.ustart[gi], tm, tn, kb0, kb1, ks);
        const int m0 = tm * (BM * CG * CF::RM) + (int)rank * BM;
        const int n0 = tn * BN + (int)rank * CF::BNL;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * CF::STAGE_BYTES;
          uint64_t* fb = &full[stage];
          const uint32_t fb_cl = CG == 2 ? mapa(smem_u32(fb), 0) : 0;
          if (leader) mbar_expect_tx(fb, CF::STAGE_BYTES * CG);
          const int k0 = kb * CF::BKM;
          if (MODE == 4 || MODE == 5 || MODE == 6) {  // bf16 operands only
            load16<BM, CG, CF::BKM>(amn, st + CF::OFF_AH16, mp + 0, fb, fb_cl, m0, k0, pa);
            if (MODE == 6)  // the second 256-row block of the pair tile
              load16<BM, CG, CF::BKM>(amn, st + CF::OFF_AL16, mp + 0, fb, fb_cl, m0 + BM * CG, k0, pa);
            load16<CF::BNL, CG, CF::BKM>(bmn, st + CF::OFF_BH16, mp + 1, fb, fb_cl, n0, k0, pb);
            if (MODE == 5) {
              load16<BM, CG, CF::BKM>(amn, st + CF::OFF_AL16, mp + 2, fb, fb_cl, m0, k0, pa);
              load16<CF::BNL, CG, CF::BKM>(bmn, st + CF::OFF_BL16, mp + 3, fb, fb_cl, n0, k0, pb);
            }
          } else {
            load32<BM, CG>(amn, st + CF::OFF_A, mp + 0, fb, fb_cl, m0, k0, pa);
            load32<CF::BNL, CG>(bmn, st + CF::OFF_B, mp + 1, fb, fb_cl, n0, k0, pb);
          }
          if (MODE == 3) {
            load32<BM, CG>(amn, st + CF::OFF_ALO, mp + 2, fb, fb_cl, m0, k0, pa);
            load32<CF::BNL, CG>(bmn, st + CF::OFF_BLO, mp + 3, fb, fb_cl, n0, k0, pb);
          } else if (MODE == 2) {
            load16<BM, CG>(amn, st + CF::OFF_AH16, mp + 2, fb, fb_cl, m0, k0, pa);
            load16<BM, CG>(amn, st + CF::OFF_AL16, mp + 4, fb, fb_cl, m0, k0, pa);
            load16<CF::BNL, CG>(bmn, st + CF::OFF_BH16, mp + 3, fb, fb_cl, n0, k0, pb);
            load16<CF::BNL, CG>(bmn, st + CF::OFF_BL16, mp + 5, fb, fb_cl, n0, k0, pb);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      };
      if (leader) {
        // draw units (static raster or the atomic counter) and publish them
        // one ahead of the loads, to this CTA's ring and the peer's
        auto next_unit = [&](int i) -> int {
          if (G.csplit > 1) return i == 0 ? csplit_unit(G, (int)blockIdx.x) : num_units;
          return G.sched ? (int)atomicAdd(G.sched, 1u) : cl_id + i * cl_num;
        };
        auto publish = [&](int i, int u) {
          const int slot = i & (kUnitRing - 1);
          uring[slot] = u;
          if (CG == 2) {
            st_cluster_u32(mapa(smem_u32(&uring[slot]), 1), u);
            mbar_arrive_remote(mapa(smem_u32(&ufull[slot]), 1));
          }
          mbar_arrive(&ufull[slot]);
        };
        int i = 0;
        int u = next_unit(0);
        publish(0, u);
        while (u < num_units) {
          const int un = next_unit(i + 1);
          publish(i + 1, un);
          produce(u);
          u = un;
          ++i;
        }
        if (G.sched) {  // the last cluster to finish drawing re-zeroes the counters
          __threadfence();
          if (atomicAdd(G.sched + 1, 1u) == (unsigned)cl_num - 1) {
            atomicExch(G.sched, 0u);
            atomicExch(G.sched + 1, 0u);
          }
        }
      } else {
        for (int i = 0;; ++i) {
          const int u = take(i);
          if (u >= num_units) break;
          produce(u);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader CTA only)
    // The accumulator restarts every KC k-blocks (kc_for_mode): the tensor core's
    // fp32 accumulation loses ~1 ulp per MMA step (2e-5 normwise at K=8192 with
    // exact inputs), so the epilogue promotes each chunk into RN fp32 sums.
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int chunk = 0;
      uint32_t d_tmem = tmem_base;
      for (int i = 0;; ++i) {
        const int u = take(i);
        if (u >= num_units) break;
        const int gi = prob_of<MULTI>(G, u);
        const TcParams& p = G.p[gi];
        const bool amn = p.a_mn != 0, bmn = p.b_mn != 0;
        int tm, tn, kb0, kb1, ks_;
        tile_info(p, u - G.ustart[gi], tm, tn, kb0, kb1, ks_);
        auto issue = [&](uint32_t s0, uint32_t acc_flag, int blocks) {
          if (amn) {
            if (bmn) mma_kblock<MODE, CG, true, true>(d_tmem, s0, acc_flag, blocks);
            else mma_kblock<MODE, CG, true, false>(d_tmem, s0, acc_flag, blocks);
          } else {
            if (bmn) mma_kblock<MODE, CG, false, true>(d_tmem, s0, acc_flag, blocks);
            else mma_kblock<MODE, CG, false, false>(d_tmem, s0, acc_flag, blocks);
          }
        };
        if (CF::RM > 1) {
          // MODE 6: the epilogue frees row block 0 of the accumulator (tempty[0])
          // before it has even drained block 1 (tempty[1]); the next unit's
          // block-0 MMAs run ahead over every k-block already staged, and its
          // block-1 MMAs (and the stage releases) follow once block 1 is free
          const int L = min(STAGES, kb1 - kb0);
          mbar_wait(&tempty[0], (chunk & 1) ^ 1);
          tc_fence_after();
          d_tmem = tmem_base;
          int st0 = stage;
          uint32_t ph0 = phase;
          for (int j = 0; j < L; ++j) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (lane == 0) issue(smem_u32(smem + stage * CF::STAGE_BYTES), j ? 1u : 0u, 1);
            __syncwarp();
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          mbar_wait(&tempty[1], (chunk & 1) ^ 1);
          tc_fence_after();
          stage = st0;
          phase = ph0;
          for (int kb = kb0; kb < kb1; ++kb) {
            const int j = kb - kb0;
            if (j >= L) {
              mbar_wait(&full[stage], phase);
              tc_fence_after();
            }
            if (lane == 0) {
              const uint32_t s0 = smem_u32(smem + stage * CF::STAGE_BYTES);
              issue(s0, j ? 1u : 0u, j < L ? 2 : 3);
              if (CG == 1) {
                tc_commit(&empty[stage]);
                if (kb == kb1 - 1) tc_commit(&tfull[0]);
              } else {
                tc_commit_pair(&empty[stage]);
                if (kb == kb1 - 1) tc_commit_pair(&tfull[0]);
              }
            }
            __syncwarp();
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          ++chunk;
          continue;
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          const int kc = (kb - kb0) % KC;
          if (kc == 0) {  // claim the next chunk accumulator (ping-pong; MODE 6: the whole TMEM)
            if (CF::RM == 1) {
              const int cb = chunk & 1;
              mbar_wait(&tempty[cb], ((chunk >> 1) & 1) ^ 1);
              d_tmem = tmem_base + cb * BN;
            } else {
              mbar_wait(&tempty[0], (chunk & 1) ^ 1);
              d_tmem = tmem_base;
            }
            tc_fence_after();
          }
          mbar_wait(&full[stage], phase);
          tc_fence_after();
#ifdef B2_GEMM_TRACE
          if (lane == 0 && kb == kb0 && i == 0) B2_TRACE(3);  // first operands landed
#endif
          if (lane == 0) {
            const uint32_t s0 = smem_u32(smem + stage * CF::STAGE_BYTES);
            // one branch per k-block into layout-specialised issue code (the
            // descriptors fold to constants: no address math between MMAs)
            issue(s0, kc ? 1u : 0u, 3);
            // smem slot free (in both CTAs) once these MMAs retire; chunk ready
            const bool last = kc == KC - 1 || kb == kb1 - 1;
            const int fb2 = CF::RM == 1 ? (chunk & 1) : 0;
            if (CG == 1) {
              tc_commit(&empty[stage]);
              if (last) tc_commit(&tfull[fb2]);
            } else {
              tc_commit_pair(&empty[stage]);
              if (last) tc_commit_pair(&tfull[fb2]);
            }
          }
          __syncwarp();
          if (kc == KC - 1 || kb == kb1 - 1) ++chunk;
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue (warps 4..19, both CTAs)
    // warp w drains TMEM lanes 32*(w%4).. (its lane quarter) for the 64-column
    // group (w-4)/4, keeps the tile's running sums for those 64 outputs of its
    // row in registers, and stores them (+bias, relu) after the last chunk.
    const int q = warp & 3;
    const int cg = (warp - 4) >> 2;
    const int row = q * 32 + lane;
    int chunk = 0;
    for (int i = 0;; ++i) {
      const int u = take(i);
      if (u >= num_units) break;
      const int gi = prob_of<MULTI>(G, u);
      const TcParams& p = G.p[gi];
      const bool vec_ok = (p.ldc % 4) == 0 && (((uintptr_t)p.C) & 15) == 0;
      int tm, tn, kb0, kb1, ks;
      tile_info(p, u - G.ustart[gi], tm, tn, kb0, kb1, ks);
      const int nch = (kb1 - kb0 + KC - 1) / KC;
      const int n0 = tn * BN;
#pragma unroll 1
      for (int blk = 0; blk < CF::RM; ++blk) {  // 128-row blocks of this CTA (MODE 6: two)
      const int m0 = tm * (BM * CG * CF::RM) + blk * (BM * CG) + (int)rank * BM;
      float acc[64];
#pragma unroll
      for (int j = 0; j < 64; ++j) acc[j] = 0.0f;
      if (CF::RM > 1) {  // MODE 6: one chunk per unit, block blk in TMEM columns [blk*256, +256)
        if (blk == 0) {
          mbar_wait(&tfull[0], chunk & 1);
          tc_fence_after();
        }
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(blk * BN + cg * 64);
#pragma unroll
        for (int j = 0; j < 64; j += 16) {
          uint32_t v[16];
          TMEM_LD16(tbase + j, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int t = 0; t < 16; ++t) acc[j + t] = __fadd_rn(acc[j + t], __uint_as_float(v[t]));
        }
        // this row block of the accumulator is free (the next unit's MMAs for
        // block 0 may start while block 0's outputs are still being stored)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(mapa(smem_u32(&tempty[blk]), 0));
        if (blk == CF::RM - 1) ++chunk;
      }
      for (int c = 0; c < (CF::RM > 1 ? 0 : nch); ++c, ++chunk) {
        const int cb = chunk & 1;
        mbar_wait(&tfull[cb], (chunk >> 1) & 1);
        tc_fence_after();
#ifdef B2_GEMM_TRACE
        if (warp == 4 && lane == 0 && c == nch - 1 && i == 0) B2_TRACE(4);  // last chunk's MMAs done
#endif
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(cb * BN + cg * 64);
#pragma unroll
        for (int j = 0; j < 64; j += 16) {
          uint32_t v[16];
          TMEM_LD16(tbase + j, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int t = 0; t < 16; ++t) acc[j + t] = __fadd_rn(acc[j + t], __uint_as_float(v[t]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 1)
            mbar_arrive(&tempty[cb]);
          else
            mbar_arrive_remote(mapa(smem_u32(&tempty[cb]), 0));  // the leader's barrier
        }
      }
      if (ks >= 0 && G.csplit > 1) {  // cluster split-K: the partial stays in shared memory
        float* mine = reinterpret_cast<float*>(smem) + row * kStageLd + cg * 64;
#pragma unroll
        for (int j = 0; j < 64; j += 4)
          *reinterpret_cast<float4*>(mine + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        cs_unit = u;
        continue;
      }
      if (ks >= 0) {  // a K slice of a tail tile: raw partial sums, tile-local
        float* w0 = p.ws + ((int64_t)ks * (BM * CG) + (int)rank * BM) * BN;
        if (G.stage_out) {
          stage_tile_store(smem, acc, row, cg, warp, lane, w0, BN, BM, BN);
          continue;
        }
        float* w = w0 + (int64_t)row * BN + cg * 64;
#pragma unroll
        for (int j = 0; j < 64; j += 4)
          *reinterpret_cast<float4*>(w + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        continue;
      }
      const int64_t m = m0 + row;
      if (m < p.M) {
        float* crow = p.C + m * p.ldc;
        const int nb = n0 + cg * 64;
        if (p.epi == B2_EPI_BIAS || p.epi == B2_EPI_BIAS_RELU) {
          if (nb + 64 <= p.N && (((uintptr_t)(p.bias + nb)) & 15) == 0) {
#pragma unroll
            for (int j = 0; j < 64; j += 4) {  // one broadcast 16-B load per 4 columns
              const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + nb + j));
              acc[j] = __fadd_rn(acc[j], b.x);
              acc[j + 1] = __fadd_rn(acc[j + 1], b.y);
              acc[j + 2] = __fadd_rn(acc[j + 2], b.z);
              acc[j + 3] = __fadd_rn(acc[j + 3], b.w);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 64; ++j) acc[j] = __fadd_rn(acc[j], nb + j < p.N ? __ldg(p.bias + nb + j) : 0.0f);
          }
        }
        if (p.epi == B2_EPI_BIAS_RELU || p.epi == B2_EPI_RELU) {
#pragma unroll
          for (int j = 0; j < 64; ++j) acc[j] = acc[j] > 0.0f ? acc[j] : 0.0f;
        }
        const bool full64 = vec_ok && nb + 64 <= p.N;
        const bool stcs = (G.l2hint & 4) != 0;
        if (p.bits_out) {  // ReLU forward: record y > 0 as 64 bits per (row, column group)
          uint32_t lo = 0, hi = 0;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            lo |= (acc[j] > 0.0f ? 1u : 0u) << j;
            hi |= (acc[32 + j] > 0.0f ? 1u : 0u) << j;
          }
          if (nb < p.N) p.bits_out[m * p.bits_ld + (nb >> 6)] = ((uint64_t)hi << 32) | lo;
        }
        if (p.mask_bits) {  // ReLU pullback from the forward's bits: g * (y > 0 ? 1 : 0)
          const uint64_t b = __ldg(reinterpret_cast<const unsigned long long*>(p.mask_bits) +
                                   m * p.bits_ld + (nb >> 6));
#pragma unroll
          for (int j = 0; j < 64; ++j) acc[j] = __fmul_rn(acc[j], (b >> j) & 1 ? 1.0f : 0.0f);
        } else if (p.mask) {  // ReLU pullback of the layer below: g * (y > 0 ? 1 : 0) (nn.py:101-103)
          const float* mrow = p.mask + m * p.ldc;
          if (full64) {
#pragma unroll
            for (int j = 0; j < 64; j += 4) {
              const float4 y = __ldg(reinterpret_cast<const float4*>(mrow + nb + j));
              acc[j] = __fmul_rn(acc[j], y.x > 0.0f ? 1.0f : 0.0f);
              acc[j + 1] = __fmul_rn(acc[j + 1], y.y > 0.0f ? 1.0f : 0.0f);
              acc[j + 2] = __fmul_rn(acc[j + 2], y.z > 0.0f ? 1.0f : 0.0f);
              acc[j + 3] = __fmul_rn(acc[j + 3], y.w > 0.0f ? 1.0f : 0.0f);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 64; ++j)
              if (nb + j < p.N) acc[j] = __fmul_rn(acc[j], mrow[nb + j] > 0.0f ? 1.0f : 0.0f);
          }
        }
        if (!p.C) {
          // fp32 C not wanted: only its operand split / bits / column sums
        } else if (G.stage_out) {
          // stored below, coalesced through shared memory (all rows of the tile)
        } else if (full64) {
#pragma unroll
          for (int j = 0; j < 64; j += 4)
            st_out16(crow + nb + j,
                     make_uint4(__float_as_uint(acc[j]), __float_as_uint(acc[j + 1]), __float_as_uint(acc[j + 2]),
                                __float_as_uint(acc[j + 3])),
                     stcs);
        } else {
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (nb + j < p.N) crow[nb + j] = acc[j];
        }
        if ((MODE == 4 || MODE == 6) && p.s_hi) {  // BF16 mode: the next GEMM's bf16 operand (RN cast)
          __nv_bfloat16* hrow = p.s_hi + m * (int64_t)p.N;
          if (full64 && (p.N % 8) == 0) {
#pragma unroll
            for (int j = 0; j < 64; j += 8) {
              __align__(16) __nv_bfloat16 h[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) h[i] = __float2bfloat16_rn(acc[j + i]);
              st_out16(hrow + nb + j, *reinterpret_cast<const uint4*>(h), stcs);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 64; ++j)
              if (nb + j < p.N) hrow[nb + j] = __float2bfloat16_rn(acc[j]);
          }
        } else if (p.s_hi) {  // the next GEMM's operand split (TF32X / 3xBF16), no separate pass
          __nv_bfloat16* hrow = p.s_hi + m * (int64_t)p.N;
          __nv_bfloat16* lrow = p.s_lo + m * (int64_t)p.N;
          if (full64 && (p.N % 8) == 0) {
#pragma unroll
            for (int j = 0; j < 64; j += 8) {
              uint4 hv, lv;
              split_pair2<MODE>(acc[j], acc[j + 1], hv.x, lv.x);
              split_pair2<MODE>(acc[j + 2], acc[j + 3], hv.y, lv.y);
              split_pair2<MODE>(acc[j + 4], acc[j + 5], hv.z, lv.z);
              split_pair2<MODE>(acc[j + 6], acc[j + 7], hv.w, lv.w);
              st_out16(hrow + nb + j, hv, stcs);
              st_out16(lrow + nb + j, lv, stcs);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 64; ++j)
              if (nb + j < p.N) split_pair<MODE>(acc[j], hrow[nb + j], lrow[nb + j]);
          }
        }
      }
      if (G.stage_out && p.C) {  // every epilogue warp takes part (rows past M are not stored)
        const int rows_left = p.M - m0;
        const int cols_left = p.N - n0;
        stage_tile_store(smem, acc, row, cg, warp, lane, p.C + (int64_t)m0 * p.ldc + n0, p.ldc,
                         rows_left < BM ? rows_left : BM, cols_left < BN ? cols_left : BN);
      }
      if (p.colsum) {
        // Column sums of the stored tile over this CTA's 128 rows (the bias
        // gradient of the layer below, fused): per 8-column group a
        // transpose-reduce butterfly in fp64 (lane l ends with column l & 7
        // over its 8 lanes) + two xor stages; the 4 row-quarter warps then
        // add in fixed order through shared memory -- deterministic.
        const bool valid = m < p.M;
        double* cb = colsum_smem + cg * 256;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          double v[8];
          {  // first stage on the fp32 values (one shuffle each); the pair sum in fp64
            const bool up = (lane & 4) != 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float a = valid ? acc[g * 8 + j] : 0.0f, b = valid ? acc[g * 8 + j + 4] : 0.0f;
              const float send = up ? a : b;
              const float keep = up ? b : a;
              v[j] = (double)keep + (double)__shfl_xor_sync(0xffffffffu, send, 4);
            }
          }
#pragma unroll
          for (int s = 2; s >= 1; s >>= 1) {
            const bool up = (lane & s) != 0;
#pragma unroll
            for (int j = 0; j < s; ++j) {
              const double send = up ? v[j] : v[j + s];
              const double keep = up ? v[j + s] : v[j];
              v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
            }
          }
          double t = v[0];
          t += __shfl_xor_sync(0xffffffffu, t, 8);
          t += __shfl_xor_sync(0xffffffffu, t, 16);
          if (lane < 8) cb[q * 64 + g * 8 + lane] = t;
        }
        asm volatile("bar.sync %0, 128;" ::"r"(1 + cg) : "memory");
        if (q == 0 && m0 < p.M) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = h * 32 + lane;
            const int n = n0 + cg * 64 + col;
            if (n < p.N)
              p.colsum[(int64_t)(m0 / BM) * p.N + n] = ((cb[col] + cb[64 + col]) + cb[128 + col]) + cb[192 + col];
          }
        }
        asm volatile("bar.sync %0, 128;" ::"r"(1 + cg) : "memory");
      }
      }  // blk
    }
  }
  if (threadIdx.x == 4 * 32) B2_TRACE(5);  // this epilogue warp's stores issued
  __syncthreads();
  if (threadIdx.x == 0) B2_TRACE(6);  // every warp done
  if (CG == 1 && G.csplit > 1) {
    // every CTA of the cluster has staged its K slice: fold, finish, store
    const int S = G.csplit;
    const int krank = (int)cluster_rank();
    cluster_sync();
    if (threadIdx.x == 4 * 32) B2_TRACE(5);  // (trace builds: cluster split-K -- all partials staged)
    int gi = 0, tm = 0, tn = 0;
    if (warp >= 4 && cs_unit >= 0) {
      gi = prob_of<MULTI>(G, cs_unit);
      int kb0, kb1, ks;
      tile_info(G.p[gi], cs_unit - G.ustart[gi], tm, tn, kb0, kb1, ks);
      const TcParams& p = G.p[gi];
      constexpr int EM = (MODE == 4 || MODE == 6) ? 4 : (MODE == 5 ? 5 : 2);
#define B2_CSR(SS)                                                                        \
  if (S == SS) {                                                                          \
    if (!p.s_hi) csplit_reduce<0, SS>(p, smem, tm, tn, krank, warp - 4, lane);           \
    else csplit_reduce<EM, SS>(p, smem, tm, tn, krank, warp - 4, lane);                  \
  }
      B2_CSR(2) B2_CSR(4) B2_CSR(8)
#undef B2_CSR
    }
    if (threadIdx.x == 4 * 32) B2_TRACE(6);  // (trace builds: this CTA's rows folded and stored)
    cluster_sync();  // the group column sums are visible
    if (warp >= 4 && cs_unit >= 0 && krank == 0 && G.p[gi].colsum)
      csplit_colsum(G.p[gi], smem, tm, tn, S, threadIdx.x - 128);
    cluster_sync();  // no CTA leaves while a peer reads its shared memory
  }
  if (CG == 2) cluster_sync();  // the peer may still be reading our smem / arriving on us
  if (warp == 2) {
    tc_fence_after();
#ifdef B2_GEMM_TRACE
    if (lane == 0) B2_TRACE(7);  // teardown
#endif
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(kTmemCols));
  }
}

// ---------------------------------------------------------------- split kernels
// 3xTF32: hi = tf32 round-to-nearest(x), lo = x - hi (exact).
__global__ void k_tf32_split(float* __restrict__ hi, float* __restrict__ lo,
                             const float* __restrict__ x, int64_t rows, int64_t cols, int64_t ld) {
  int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / cols, c = i - r * cols;
    float v = x[r * ld + c];
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
    float hf = __uint_as_float(h);
    if (hi) hi[r * cols + c] = hf;
    lo[r * cols + c] = __fsub_rn(v, hf);
  }
}

__global__ void k_tf32_split_vec(float* __restrict__ hi, float* __restrict__ lo,
                                 const float* __restrict__ x, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = reinterpret_cast<const float4*>(x)[i];
    float in[4] = {v.x, v.y, v.z, v.w}, h[4], l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t b;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(in[j]));
      h[j] = __uint_as_float(b);
      l[j] = __fsub_rn(in[j], h[j]);
    }
    if (hi) reinterpret_cast<float4*>(hi)[i] = make_float4(h[0], h[1], h[2], h[3]);
    reinterpret_cast<float4*>(lo)[i] = make_float4(l[0], l[1], l[2], l[3]);
  }
}

// Operand split (split_pair<MODE>): TF32X (MODE 2) or 3xBF16 (MODE 5).
// 8 elements per thread-iteration (32 B in, 2 x 16 B out).
template <int MODE>
__global__ void k_bf16x2_split(__nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo,
                               const float* __restrict__ x, int64_t rows, int64_t cols, int64_t ld) {
  asm volatile("griddepcontrol.launch_dependents;");  // the consuming GEMM may start its prologue
  const int64_t c8 = cols >> 3;  // cols % 8 == 0 (checked on the host)
  const int64_t n8 = rows * c8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / c8, c = (i - r * c8) * 8;
    const float* src = x + r * ld + c;
    float v[8];
    if (((uintptr_t)src & 15) == 0) {
      float4 a = reinterpret_cast<const float4*>(src)[0], b = reinterpret_cast<const float4*>(src)[1];
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = src[j];
    }
    __align__(16) __nv_bfloat16 h[8], l[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) split_pair<MODE>(v[j], h[j], l[j]);
    *reinterpret_cast<uint4*>(hi + r * cols + c) = *reinterpret_cast<const uint4*>(h);
    *reinterpret_cast<uint4*>(lo + r * cols + c) = *reinterpret_cast<const uint4*>(l);
  }
}

// Two matrices' 3xBF16 splits in one launch (a GEMM's two fresh operands):
// threads [0, n8a) take the first matrix's 8-element groups, the rest the
// second's -- the same per-element arithmetic as k_bf16x2_split<5>.
struct SplitJob {
  __nv_bfloat16* hi;
  __nv_bfloat16* lo;
  const float* x;
  int64_t rows, cols, ld;
};
__global__ void k_bf16x3_split2(const SplitJob ja, const SplitJob jb) {
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t n8a = ja.rows * (ja.cols >> 3), n8 = n8a + jb.rows * (jb.cols >> 3);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool first = i < n8a;
    const SplitJob& j = first ? ja : jb;
    const int64_t k = first ? i : i - n8a;
    const int64_t c8 = j.cols >> 3;
    const int64_t r = k / c8, c = (k - r * c8) * 8;
    const float* src = j.x + r * j.ld + c;
    float v[8];
    if (((uintptr_t)src & 15) == 0) {
      float4 a = reinterpret_cast<const float4*>(src)[0], b = reinterpret_cast<const float4*>(src)[1];
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = src[q];
    }
    __align__(16) __nv_bfloat16 h[8], l[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) split_pair<5>(v[q], h[q], l[q]);
    *reinterpret_cast<uint4*>(j.hi + r * j.cols + c) = *reinterpret_cast<const uint4*>(h);
    *reinterpret_cast<uint4*>(j.lo + r * j.cols + c) = *reinterpret_cast<const uint4*>(l);
  }
}

// BF16 mode operand: contiguous bf16 round-to-nearest copy of a [rows, cols] (ld) matrix
__global__ void k_bf16_cast(__nv_bfloat16* __restrict__ out, const float* __restrict__ x,
                            int64_t rows, int64_t cols, int64_t ld) {
  const int64_t c8 = cols >> 3;  // cols % 8 == 0 (checked on the host)
  const int64_t n8 = rows * c8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / c8, c = (i - r * c8) * 8;
    const float* src = x + r * ld + c;
    __align__(16) __nv_bfloat16 h[8];
    if (((uintptr_t)src & 15) == 0) {
      const float4 a = reinterpret_cast<const float4*>(src)[0], b = reinterpret_cast<const float4*>(src)[1];
      h[0] = __float2bfloat16_rn(a.x); h[1] = __float2bfloat16_rn(a.y);
      h[2] = __float2bfloat16_rn(a.z); h[3] = __float2bfloat16_rn(a.w);
      h[4] = __float2bfloat16_rn(b.x); h[5] = __float2bfloat16_rn(b.y);
      h[6] = __float2bfloat16_rn(b.z); h[7] = __float2bfloat16_rn(b.w);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) h[j] = __float2bfloat16_rn(src[j]);
    }
    *reinterpret_cast<uint4*>(out + r * cols + c) = *reinterpret_cast<const uint4*>(h);
  }
}

// Tail second stage: for each split tail tile, C = epilogue(sum_s ws[s]) in
// fixed slice order (deterministic) with the GEMM epilogue's stages: bias,
// ReLU, relu bits (ballot per 32 columns), the ReLU-pullback mask (bits or
// fp32), the stores, C's operand split (EMIT = GEMM mode: 2 TF32X, 5 3xBF16,
// 4 bf16 cast, 0 none) and the fp64 column partial sums of its 128-row block.
// grid (tail tiles, CG row blocks of 128, BN/32 column strips), 32 x 16
// threads: x = 32 consecutive columns (one relu-bits word per warp row),
// y = an 8-row group walked in order; the groups' fp64 column sums are added
// in fixed order. 8 CTAs per tile x row block keep the SMs busy (one CTA of
// 512 threads per 128 columns left most of them idle: latency-bound).
template <int EMIT>
__global__ void __launch_bounds__(512) k_tail_epilogue(const TcParams p) {
  constexpr int RG = 16, RPG = BM / RG;  // row groups x rows per group
  __shared__ double csum[RG][32];
  const int i = blockIdx.x, cg = (int)gridDim.y;
  const int tail = p.tiles_m * p.tiles_n - p.full_tiles;
  int tm, tn;
  tile_coords(p, p.full_tiles + i, tm, tn);
  const int r0 = blockIdx.y * BM + threadIdx.y * RPG;
  const int c = blockIdx.z * 32 + threadIdx.x;
  const int64_t n = (int64_t)tn * BN + c;
  const int64_t mb = (int64_t)tm * (BM * cg) + blockIdx.y * BM;
  const bool col_ok = n < p.N;
  const float bias = (col_ok && (p.epi == B2_EPI_BIAS || p.epi == B2_EPI_BIAS_RELU)) ? p.bias[n] : 0.0f;
  const int64_t slice = (int64_t)tail * (BM * cg) * BN;
  const float* w = p.ws + ((int64_t)i * (BM * cg) + r0) * BN + c;
  uint32_t* bits32 = reinterpret_cast<uint32_t*>(p.bits_out);
  const uint32_t* mbits32 = reinterpret_cast<const uint32_t*>(p.mask_bits);
  const bool word_ok = (n >> 5) < 2 * (int64_t)p.bits_ld;  // the words cover N rounded up to 64
  double cs = 0.0;
  const int64_t mrow0 = (int64_t)tm * (BM * cg) + r0;
  const int64_t left = p.M - mrow0;
  const int nrows = left <= 0 ? 0 : (left < RPG ? (int)left : RPG);
  // 8 rows x 4 slices of partials in flight per round (a serial walk over
  // rows and slices would pay one L2 round trip per partial); every row still
  // adds its slices in slice order
  for (int rb = 0; rb < nrows; rb += 8) {
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
    for (int sl = 0; sl < p.splits; sl += 4) {
      float v[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < 8; ++q)
          v[u][q] = (sl + u < p.splits && rb + q < nrows)
                        ? __ldcg(w + (int64_t)(sl + u) * slice + (int64_t)(rb + q) * BN)
                        : 0.0f;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (sl + u < p.splits) acc[q] = __fadd_rn(acc[q], v[u][q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
    if (rb + q >= nrows) break;
    const int r = rb + q;
    const int64_t m = mrow0 + r;
    float x = acc[q];
    if (p.epi == B2_EPI_BIAS || p.epi == B2_EPI_BIAS_RELU) x = __fadd_rn(x, bias);
    if (p.epi == B2_EPI_BIAS_RELU || p.epi == B2_EPI_RELU) x = x > 0.0f ? x : 0.0f;
    if (bits32) {
      const uint32_t word = __ballot_sync(0xffffffffu, col_ok && x > 0.0f);
      if ((threadIdx.x & 31) == 0 && word_ok) bits32[m * 2 * p.bits_ld + (n >> 5)] = word;
    }
    if (!col_ok) continue;
    if (mbits32)
      x = __fmul_rn(x, (mbits32[m * 2 * p.bits_ld + (n >> 5)] >> (n & 31)) & 1 ? 1.0f : 0.0f);
    else if (p.mask)
      x = __fmul_rn(x, p.mask[m * p.ldc + n] > 0.0f ? 1.0f : 0.0f);
    if (p.C) p.C[m * p.ldc + n] = x;
    if (EMIT == 4 && p.s_hi) p.s_hi[m * p.N + n] = __float2bfloat16_rn(x);
    if ((EMIT == 2 || EMIT == 5) && p.s_hi) split_pair<EMIT>(x, p.s_hi[m * p.N + n], p.s_lo[m * p.N + n]);
    cs += (double)x;
    }
  }
  if (!p.colsum) return;
  csum[threadIdx.y][threadIdx.x] = cs;
  __syncthreads();
  if (threadIdx.y == 0 && col_ok && mb < p.M)
  {
    double t = csum[0][threadIdx.x];
#pragma unroll
    for (int g = 1; g < RG; ++g) t += csum[g][threadIdx.x];
    p.colsum[(mb / BM) * p.N + n] = t;
  }
}

// colsum[n] = f32(sum over the row blocks of the fp64 partials): 32 columns x
// 8 row lanes per CTA (lane k folds row blocks k, k+8, ...), then a fixed
// shared-memory tree over the 8 lanes -- deterministic
__global__ void __launch_bounds__(256) k_colsum_final(float* __restrict__ out,
                                                      const double* __restrict__ part, int rows, int N) {
  __shared__ double sh[256];
  const int c = threadIdx.x & 31, k = threadIdx.x >> 5;
  const int n = blockIdx.x * 32 + c;
  double s = 0.0;
  if (n < N)
    for (int r = k; r < rows; r += 8) s += part[(int64_t)r * N + n];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int h = 4; h > 0; h >>= 1) {
    if (k < h) sh[threadIdx.x] += sh[threadIdx.x + 32 * h];
    __syncthreads();
  }
  if (k == 0 && n < N) out[n] = __double2float_rn(sh[c]);
}

// ---------------------------------------------------------------- host side

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

int get_encode() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    cudaGetLastError();
  });
  return g_encode ? 0 : b2::fail("cuTensorMapEncodeTiled unavailable from the driver");
}

// 2-D tensor map over a row-major [rows, cols] matrix with leading dim ld (elements).
//   fp32 operand (tf32): box {32, box_rows}; K-major 128-B swizzle, MN-major
//     128-B swizzle with 32-B atoms (UMMA SWIZZLE_128B_BASE32B).
//   bf16 operand: K-major box {32 (64 B), box_rows} with 64-B swizzle; MN-major
//     box {64 (128 B), 32} with 128-B swizzle.
//   wide (pure-bf16 modes): K-major box {64 (128 B), box_rows} with 128-B
//     swizzle; MN-major box {64, 64}.
int make_map(CUtensorMap* tm, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
             bool mn_major, bool bf16, bool wide = false) {
  const int esz = bf16 ? 2 : 4;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * esz};
  const int kb = bf16 && wide ? 64 : 32;  // k extent of a box
  // box = {inner (contiguous) extent, outer extent}; for MN-major tiles the
  // inner extent is 64 MN elements and box_rows carries the k extent
  cuuint32_t box[2] = {(cuuint32_t)(bf16 && mn_major ? 64 : kb), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapSwizzle sw = bf16 ? ((mn_major || wide) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B)
                               : (mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B);
  CUresult r = g_encode(tm, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                        (void*)base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return b2::fail("cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) + ")");
  return 0;
}

struct Operands {
  const void* a[3];   // MODE 1: {A}; MODE 3/5: {Ahi, Alo}; MODE 2: {A, Ah16, Al16}; MODE 4: {A16}
  const void* b[3];
  int64_t lda, ldb;   // leading dims of a[0], b[0]; the other arrays are contiguous
};

// fp32 promotion interval: the tensor core's accumulation truncates (~1 ulp
// per MMA, biased), so the accumulator restarts every KC k-blocks and the
// epilogue sums chunks in RN fp32. K = 256 for the tf32 modes; K = 1024 for
// 3xBF16 (measured: normwise 5e-6 at K = 8192 vs 4e-6 at K = 256, +8% speed
// from 4x fewer TMEM drains) and for the bf16 variant (2^-9 operand error).
// B2_GEMM_KC overrides (scripts/gemm_kc_probe.py).
static int kc_for_mode(int mode) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("B2_GEMM_KC");
    env = e ? atoi(e) : 0;
  }
  if (env > 0) return env;
  // BF16 (bf16 variant): bf16 operand rounding dwarfs the accumulator's
  // truncation, so chunks of K = 4096 -- one TMEM drain per tile for the
  // config-5 shapes, the epilogue's slack a whole tile (bf16 step -7%)
  if (mode == 4) return 8 * KC_BASE;
  if (mode == 6) return 1 << 30;  // one chunk per unit: the single 512-column accumulator
  return mode == 5 ? 2 * KC_BASE : KC_BASE;  // K = 1024 (BK 64) / 256 (BK 32)
}

static int pdl_enabled() {
  static int v = -1;  // B2_GEMM_PDL=0: plain stream serialisation (A/B measurements)
  if (v < 0) {
    const char* e = getenv("B2_GEMM_PDL");
    v = !(e && e[0] == '0');
  }
  return v;
}

static int stage_out_enabled() {
  static int v = -1;  // B2_GEMM_STAGE_OUT=0: direct per-row stores everywhere (A/B measurements)
  if (v < 0) {
    const char* e = getenv("B2_GEMM_STAGE_OUT");
    v = !(e && e[0] == '0');
  }
  return v;
}

// One problem of a launch as the host prepares it (gemm_tc_group).
struct Prob {
  TcParams p;
  Operands o;
  int64_t tiles;      // output tiles at the launch's CTA grouping
  int S;              // K slices of the split tiles (1: whole tiles only)
  int64_t T;          // tiles split into S slices
  void* part;         // K-slice partials
  void* cs_part;      // fp64 column partials
  float* colsum_out;
  int cs_rows;
};

constexpr int kCsplitNoFit = -77;  // launch_tc: the split-K clusters cannot all be resident

static int group_n_env() {
  static int gn = -1;
  if (gn < 0) {
    const char* e = getenv("B2_GEMM_GROUPN");
    gn = e ? atoi(e) : 0;
    if (gn <= 0) gn = kGroupN;
  }
  return gn;
}

// Tensor maps of every problem (box shapes from the mode's Cfg), the
// TcGroup, one launch. A is [M,K] (K-major) or stored [K,M] (MN-major); B is
// [N,K] or stored [K,N].
template <int MODE, int CG>
int launch_tc(Prob* pr, int n, TcGroup& G, cudaStream_t st) {
  using CF = Cfg<MODE, CG>;
  static TcMaps maps;  // host staging (copied into the launch's parameters)
  constexpr bool kB16 = MODE == 4 || MODE == 5 || MODE == 6;
  for (int g = 0; g < n; ++g) {
    const TcParams& p = pr[g].p;
    const Operands& o = pr[g].o;
    CUtensorMap* m = maps.m[g];
    const bool A_MN = p.a_mn != 0, B_MN = p.b_mn != 0;
    const int64_t ar = A_MN ? p.K : p.M, ac = A_MN ? p.M : p.K;
    const int64_t br = B_MN ? p.K : p.N, bc = B_MN ? p.N : p.K;
    const int abox = A_MN ? CF::BKM : BM, bbox = B_MN ? CF::BKM : CF::BNL;
    B2_TRY(make_map(&m[0], o.a[0], ar, ac, o.lda, abox, A_MN, kB16, CF::W64));
    B2_TRY(make_map(&m[1], o.b[0], br, bc, o.ldb, bbox, B_MN, kB16, CF::W64));
    m[2] = m[0]; m[3] = m[1]; m[4] = m[0]; m[5] = m[1];
    if (MODE == 5) {
      B2_TRY(make_map(&m[2], o.a[1], ar, ac, ac, abox, A_MN, true, CF::W64));
      B2_TRY(make_map(&m[3], o.b[1], br, bc, bc, bbox, B_MN, true, CF::W64));
    } else if (MODE == 3) {
      B2_TRY(make_map(&m[2], o.a[1], ar, ac, ac, abox, A_MN, false));
      B2_TRY(make_map(&m[3], o.b[1], br, bc, bc, bbox, B_MN, false));
    } else if (MODE == 2) {
      B2_TRY(make_map(&m[2], o.a[1], ar, ac, ac, abox, A_MN, true));
      B2_TRY(make_map(&m[4], o.a[2], ar, ac, ac, abox, A_MN, true));
      B2_TRY(make_map(&m[3], o.b[1], br, bc, bc, bbox, B_MN, true));
      B2_TRY(make_map(&m[5], o.b[2], br, bc, bc, bbox, B_MN, true));
    }
    G.p[g] = p;
  }
  G.kc = kc_for_mode(MODE);
  auto kern = n > 1 ? k_gemm_tc<MODE, CG, true> : k_gemm_tc<MODE, CG, false>;
  static bool attr_set = false;
  if (!attr_set) {
    for (auto k : {k_gemm_tc<MODE, CG, true>, k_gemm_tc<MODE, CG, false>}) {
      B2_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));
      if (CG == 2) B2_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
    }
    attr_set = true;
  }
  const int sms = b2::gemm_sms();
  const int grid = (G.num_units * CG < sms) ? G.num_units * CG : (sms / CG) * CG;
  static_assert(CF::STAGES * CF::STAGE_BYTES >= BM * kStageLd * 4, "staged tile store needs the stage buffers");
  G.stage_out = G.num_units <= grid / CG && stage_out_enabled();
  // several problems with more units than CTA (pairs): units are drawn from
  // the stream's zeroed scheduler counters (dynamic balance); else the raster
  G.sched = nullptr;
  if (G.csplit > 1) {
    if (CG != 1 || grid != G.num_units || grid % G.csplit) return b2::fail("gemm_tc: bad cluster split-K launch");
    G.stage_out = 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = CF::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  static_assert(CG == 2 || CF::STAGES * CF::STAGE_BYTES >= BM * kStageLd * 4 + 16 * BN * 8,
                "cluster split-K stages the partial tile and the group column sums in the stage buffers");
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (CG == 1 && G.csplit > 1) ? G.csplit : CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  if (G.csplit > 1) {
    // every cluster must be resident at once (S CTAs of ~200 KB in one GPC):
    // otherwise the K slices go through L2 partials instead (host fallback)
    int fit = 0;
    cudaLaunchConfig_t q = cfg;
    q.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&fit, (void*)kern, &q) != cudaSuccess) {
      cudaGetLastError();
      fit = 0;
    }
    if (fit * G.csplit < G.num_units) return kCsplitNoFit;
  }
  // Units are drawn dynamically whenever there are more than CTA (pairs):
  // also for one problem, where the next clusters to finish take the next
  // tiles of the raster, so the 8 consumers of an A panel stay in step and
  // find it in L2 -- config-5 forward GEMM: DRAM reads 3.92 -> 3.35 GB and
  // 4.22 -> 4.11 ms per launch (ncu) against the static raster, which lets
  // the clusters drift apart over ~56 waves. B2_GEMM_DYNAMIC=0: static (A/B).
  static int dyn = -1;
  if (dyn < 0) {
    const char* e = getenv("B2_GEMM_DYNAMIC");
    dyn = !(e && e[0] == '0');
  }
  if ((n > 1 || dyn) && G.num_units > grid / CG && G.csplit == 1) {
    unsigned* tk = b2::tickets(st);
    if (!tk) return b2::fail("gemm_tc: no scheduler counters for this stream");
    G.sched = tk + b2::kGemmTicket;
  }
  B2_CUDA(cudaLaunchKernelEx(&cfg, kern, maps, G));
  return b2::launched(n > 1 ? "b2_gemm(tcgen05, grouped)" : "b2_gemm(tcgen05)");
}

}  // namespace

#ifdef B2_GEMM_TRACE
extern "C" int b2_gemm_trace_read(unsigned long long* out /* [1024][8] */) {
  return cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace)) == cudaSuccess ? 0 : 1;
}
#endif

namespace b2 {

// split a [rows, cols] (ld) matrix into contiguous hi/lo fp32 arrays (3xTF32)
int tf32_split(float* hi, float* lo, const float* x, int64_t rows, int64_t cols, int64_t ld,
               cudaStream_t st) {
  int64_t n = rows * cols;
  if (n == 0) return 0;
  if (ld == cols && ((uintptr_t)x & 15) == 0 && ((uintptr_t)lo & 15) == 0 &&
      (!hi || ((uintptr_t)hi & 15) == 0) && n % 4 == 0) {
    k_tf32_split_vec<<<grid_for(n / 4, 256 * 4, 8), 256, 0, st>>>(hi, lo, x, n / 4);
  } else {
    k_tf32_split<<<grid_for(n, 256 * 4, 8), 256, 0, st>>>(hi, lo, x, rows, cols, ld);
  }
  return launched("b2_tf32_split");
}

// split a [rows, cols] (ld) matrix into contiguous bf16 hi/lo arrays:
// mode 2 (TF32X) bf16(trunc_tf32(x)), bf16(x - trunc); mode 5 (3xBF16)
// bf16_rn(x), bf16_rn(x - hi)
int bf16x2_split(void* hi, void* lo, const float* x, int64_t rows, int64_t cols, int64_t ld,
                 cudaStream_t st, int mode) {
  int64_t n = rows * cols;
  if (n == 0) return 0;
  if (cols % 8 || ((uintptr_t)hi & 15) || ((uintptr_t)lo & 15))
    return fail("b2_bf16x2_split: cols must be a multiple of 8 and outputs 16-B aligned");
  if (mode == 5)
    k_bf16x2_split<5><<<grid_for(n / 8, 256 * 4, 8), 256, 0, st>>>(
        (__nv_bfloat16*)hi, (__nv_bfloat16*)lo, x, rows, cols, ld);
  else
    k_bf16x2_split<2><<<grid_for(n / 8, 256 * 4, 8), 256, 0, st>>>(
        (__nv_bfloat16*)hi, (__nv_bfloat16*)lo, x, rows, cols, ld);
  return launched(mode == 5 ? "b2_bf16x3_split" : "b2_bf16x2_split");
}

// fp32 view of a 3xBF16 split: out = f32(hi) + f32(lo), exact in fp32 (hi has
// 8 significant bits, lo sits below them), within 2^-16 relative of the
// value the split was made from. Materialises a GEMM output whose epilogue
// wrote only its operand split (b2_bf16x3_join).
__global__ void __launch_bounds__(256) k_bf16x3_join(float* __restrict__ out, const __nv_bfloat16* __restrict__ hi,
                                                     const __nv_bfloat16* __restrict__ lo, int64_t n8) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += st) {
    const uint4 h = __ldg(reinterpret_cast<const uint4*>(hi) + i);
    const uint4 l = __ldg(reinterpret_cast<const uint4*>(lo) + i);
    const __nv_bfloat162* hp = reinterpret_cast<const __nv_bfloat162*>(&h);
    const __nv_bfloat162* lp = reinterpret_cast<const __nv_bfloat162*>(&l);
    float r[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 a = __bfloat1622float2(hp[k]), b = __bfloat1622float2(lp[k]);
      r[2 * k] = __fadd_rn(a.x, b.x);
      r[2 * k + 1] = __fadd_rn(a.y, b.y);
    }
    float4* o = reinterpret_cast<float4*>(out) + 2 * i;
    o[0] = make_float4(r[0], r[1], r[2], r[3]);
    o[1] = make_float4(r[4], r[5], r[6], r[7]);
  }
}

int bf16x3_split2(void* hia, void* loa, const float* xa, int64_t ra, int64_t ca, int64_t lda, void* hib,
                  void* lob, const float* xb, int64_t rb, int64_t cb, int64_t ldb, cudaStream_t st) {
  if (ca % 8 || cb % 8 || ((uintptr_t)hia & 15) || ((uintptr_t)loa & 15) || ((uintptr_t)hib & 15) ||
      ((uintptr_t)lob & 15))
    return fail("b2_bf16x3_split2: cols must be multiples of 8 and outputs 16-B aligned");
  const int64_t n8 = ra * (ca / 8) + rb * (cb / 8);
  if (n8 == 0) return 0;
  const SplitJob ja{(__nv_bfloat16*)hia, (__nv_bfloat16*)loa, xa, ra, ca, lda};
  const SplitJob jb{(__nv_bfloat16*)hib, (__nv_bfloat16*)lob, xb, rb, cb, ldb};
  k_bf16x3_split2<<<grid_for(n8, 256 * 4, 8), 256, 0, st>>>(ja, jb);
  return launched("b2_bf16x3_split2");
}

int bf16x3_join(float* out, const void* hi, const void* lo, int64_t n, cudaStream_t st) {
  if (n == 0) return 0;
  if (n % 8 || ((uintptr_t)out & 15) || ((uintptr_t)hi & 15) || ((uintptr_t)lo & 15))
    return fail("b2_bf16x3_join: n % 8 == 0 and 16-B aligned buffers needed");
  k_bf16x3_join<<<grid_for(n / 8, 256 * 2, 8), 256, 0, st>>>(out, (const __nv_bfloat16*)hi,
                                                               (const __nv_bfloat16*)lo, n / 8);
  return launched("b2_bf16x3_join");
}

int bf16_cast(void* out, const float* x, int64_t rows, int64_t cols, int64_t ld, cudaStream_t st) {
  int64_t n = rows * cols;
  if (n == 0) return 0;
  if (cols % 8 || ((uintptr_t)out & 15)) return fail("b2_bf16_cast: cols % 8 and 16-B output needed");
  k_bf16_cast<<<grid_for(n / 8, 256 * 4, 8), 256, 0, st>>>((__nv_bfloat16*)out, x, rows, cols, ld);
  return launched("b2_bf16_cast");
}

bool tc_supported(int ta, int tb, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb) {
  if (M > INT32_MAX / 2 || N > INT32_MAX / 2 || K > INT32_MAX / 2) return false;
  if (lda % 4 || ldb % 4) return false;  // TMA: row strides multiple of 16 bytes
  // the contiguous split copies use their column count as leading dimension
  // (bf16 rows need 16-byte strides: multiples of 8 elements)
  if ((ta ? M : K) % 8 || (tb ? K : N) % 8) return false;
  if (M < 1 || N < 1 || K < 1) return false;
  return true;
}

static int splitk_enabled() {
  static int v = -1;  // B2_GEMM_SPLITK=0 disables split-K (A/B measurements)
  if (v < 0) {
    const char* e = getenv("B2_GEMM_SPLITK");
    v = !(e && e[0] == '0');
  }
  return v;
}

static int m2_enabled() {
  static int v = -1;  // B2_GEMM_M2=0: the bf16 variant keeps 256-row pair tiles (A/B)
  if (v < 0) {
    const char* e = getenv("B2_GEMM_M2");
    v = !(e && e[0] == '0');
  }
  return v;
}

static int csplit_enabled() {
  static int v = -1;  // B2_GEMM_CSPLIT=0: K slices through L2 partials + k_tail_epilogue (A/B)
  if (v < 0) {
    const char* e = getenv("B2_GEMM_CSPLIT");
    v = !(e && e[0] == '0');
  }
  return v;
}

static int cg_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("B2_GEMM_CG");
    v = e ? atoi(e) : 0;  // 0 auto, 1 or 2 forced
  }
  return v;
}

int gemm_tc_group(int mode, const TcDesc* d, int n, cudaStream_t st) {
  B2_TRY(get_encode());
  if (n < 1 || n > kMaxProb) return fail("gemm_tc: 1 to 3 problems per launch");
  Prob pr[kMaxProb];
  for (int g = 0; g < n; ++g) {
    const TcDesc& x = d[g];
    TcParams& p = pr[g].p;
    memset(&p, 0, sizeof(p));
    p.C = x.C;
    p.bias = x.bias;
    p.ldc = x.ldc;
    p.M = (int)x.M;
    p.N = (int)x.N;
    p.K = (int)x.K;
    p.epi = x.epi;
    p.mask = x.mask;
    p.mask_bits = x.mask_bits;
    p.bits_out = x.bits_out;
    p.bits_ld = (int)((x.N + 63) / 64);
    if (((uintptr_t)x.mask_bits & 7) || ((uintptr_t)x.bits_out & 7))
      return fail("gemm_tc: bit masks need 8-B aligned word arrays");
    p.s_hi = (__nv_bfloat16*)x.s_hi;
    p.s_lo = (__nv_bfloat16*)x.s_lo;
    if ((x.s_hi == nullptr) != (x.s_lo == nullptr) && mode != 4)
      return fail("gemm_tc: split outputs come in pairs");
    if (((uintptr_t)x.s_hi & 15) || ((uintptr_t)x.s_lo & 15) || ((uintptr_t)x.C & 3))
      return fail("gemm_tc: C must be 4-B and the emitted split arrays 16-B aligned");
    if (mode == 4) p.s_lo = nullptr;  // BF16 mode emits a single bf16 cast
    p.a_mn = x.ta != 0;
    p.b_mn = x.tb == 0;
    p.group_n = group_n_env();
    pr[g].o = Operands{{x.a0, x.a1, x.a2}, {x.b0, x.b1, x.b2}, x.lda, x.ldb};
    pr[g].part = pr[g].cs_part = nullptr;
    pr[g].colsum_out = x.colsum;
    pr[g].S = 1;
    pr[g].T = 0;
  }
  const int sms = gemm_sms();
  const int bk = (mode == 4 || mode == 5) ? 64 : BK;  // Cfg::BKM
  // CTA pairs once there are enough 256-row tiles to fill the chip
  auto cg_alone = [&](const TcDesc& x) -> int {
    const int f = cg_mode();
    if (f == 1 || f == 2) return f;
    const int64_t pair_tiles = ((x.M + 2 * BM - 1) / (2 * BM)) * ((x.N + BN - 1) / BN);
    if (pair_tiles >= sms / 2) return 2;
    // few tiles over a long K (the dW GEMMs of config 4: 1024^2 over K = 32768)
    // run as K slices for many k-blocks per unit: there a pair's per-SM operand
    // ingress (64 KB per k-block instead of 96 KB) is the limit, not the tile
    // count (measured: 174 -> 158 us; short-K few-tile GEMMs stay single-CTA)
    return (x.K >= 8192 && x.M >= 2 * BM) ? 2 : 1;
  };
  int cg = 1;
  for (int g = 0; g < n; ++g) cg = std::max(cg, cg_alone(d[g]));
  // a group of few tiles in all (config 3's dA + dB at n = 1024) fills the
  // chip once with K slices of every tile: one unit per CTA (pair)
  int64_t group_tiles = 0;
  for (int g = 0; g < n; ++g)
    group_tiles += ((d[g].M + (int64_t)BM * cg - 1) / ((int64_t)BM * cg)) * ((d[g].N + BN - 1) / BN);
  const bool few_group = n > 1 && group_tiles * cg <= sms / 2;
  // bf16 variant with CTA pairs and at least two waves of 512-row pair tiles:
  // MODE 6 (Cfg::RM), whole tiles only (no K slices; one chunk per unit)
  bool m2 = false;
  if (mode == 4 && cg == 2 && m2_enabled()) {
    int64_t t2 = 0;
    for (int g = 0; g < n; ++g) t2 += ((d[g].M + 4 * BM - 1) / (4 * BM)) * ((d[g].N + BN - 1) / BN);
    m2 = t2 >= 2 * (int64_t)(sms / 2);
  }
  const int rows_per_tile = BM * cg * (m2 ? 2 : 1);
  // Work units (TcParams): whole tiles, and tiles split into S K slices
  // whose fp32 partials a fixed-order second stage folds. Taken where it pays
  // for the partials' round trip and the second stage (measured,
  // scripts/tail_probe.py): few-tile long-K GEMMs split every tile (dW
  // [1024 x 1024] over K = 32768, square n = 1024); a short run of waves
  // whose last wave is at most half full splits its tail tiles (dW
  // [4096 x 4096] over K = 65536: 3 waves + 34 of 74 tiles). Slices >= 256
  // of K, S <= 16. The K partition of a problem is the one it gets when
  // launched alone -- it fixes the rounding of every output, so a grouped
  // launch is bit-identical to separate ones -- except in a group of few
  // tiles (below); either way it depends only on the shapes and the SM count
  // (deterministic).
  for (int g = 0; g < n; ++g) {
    TcParams& p = pr[g].p;
    p.nkb = (int)((d[g].K + bk - 1) / bk);
    p.tiles_n = (int)((d[g].N + BN - 1) / BN);
    p.tiles_m = (int)((d[g].M + (int64_t)rows_per_tile - 1) / rows_per_tile);
    pr[g].tiles = (int64_t)p.tiles_m * p.tiles_n;
    const int ca = cg_alone(d[g]);
    const int64_t Pa = sms / ca;
    const int64_t tiles_a = ((d[g].M + (int64_t)BM * ca - 1) / ((int64_t)BM * ca)) * p.tiles_n;
    const int nkb = p.nkb;
    int64_t full = pr[g].tiles, T = 0;
    int S = 1;
    if (m2) {
      // whole 512-row tiles (the unit queue balances them dynamically)
    } else if (few_group && nkb >= 16 && splitk_enabled()) {
      // the group's own partition (outputs differ from separate launches in
      // rounding only; still a function of the shapes and the SM count)
      S = (int)std::max<int64_t>(
          1, std::min<int64_t>({(sms / cg) / group_tiles, (int64_t)nkb * bk / 256, 16}));
      if (S > 1) {
        full = 0;
        T = pr[g].tiles;
      }
    } else if (nkb >= 16 && splitk_enabled()) {
      int64_t fa = tiles_a, Ta = 0;
      if (tiles_a * ca <= sms / 2) {
        fa = 0;
        Ta = tiles_a;
      } else if (tiles_a >= Pa && tiles_a < 8 * Pa && 2 * (tiles_a % Pa) <= Pa) {
        fa = (tiles_a / Pa) * Pa;
        Ta = tiles_a - fa;
      }
      if (Ta > 0)
        S = (int)std::max<int64_t>(1, std::min<int64_t>({Pa / Ta, (int64_t)nkb * bk / 256, 16}));
      if (S > 1) {
        if (fa == 0) {  // every tile split: any tile shape gives the same K partition
          full = 0;
          T = pr[g].tiles;
        } else if (ca == cg) {  // the same tiles as alone
          full = fa;
          T = Ta;
        } else {
          S = 1;
        }
      }
    }
    p.full_tiles = (int)full;
    p.kbps = nkb;
    p.splits = 1;
    p.ws = nullptr;
    if (S > 1) {
      p.kbps = (nkb + S - 1) / S;
      S = (nkb + p.kbps - 1) / p.kbps;
      p.splits = S;
    } else {
      p.full_tiles = (int)pr[g].tiles;
      T = 0;
    }
    pr[g].S = S;
    pr[g].T = T;
  }
  // most expensive units first (longest-processing-time order for the
  // dynamic draw); a stable order otherwise
  if (n > 1)
    std::stable_sort(pr, pr + n, [](const Prob& a, const Prob& b) {
      return (a.S > 1 ? a.p.kbps : a.p.nkb) > (b.S > 1 ? b.p.kbps : b.p.nkb);
    });
  TcGroup G;
  memset(&G, 0, sizeof(G));
  G.nprob = n;
  int units = 0;
  for (int g = 0; g < n; ++g) {
    TcParams& p = pr[g].p;
    p.num_tiles = (int)(p.full_tiles + (pr[g].tiles - p.full_tiles) * p.splits);  // units
    G.ustart[g] = units;
    units += p.num_tiles;
  }
  G.ustart[n] = units;
  G.num_units = units;
  // Cluster split-K: a launch whose every tile is split into the same S slices
  // with one unit per CTA (the few-tile regime at cg 1: config 3 at n = 1024)
  // folds the slices through distributed shared memory inside each cluster of
  // S CTAs -- no fp32 partials through L2, no second-stage kernel.
  G.csplit = 1;
  if (cg == 1 && csplit_enabled() && units <= sms) {
    const int S0 = pr[0].S;
    bool ok = S0 == 2 || S0 == 4 || S0 == 8;
    for (int g = 0; g < n && ok; ++g) ok = pr[g].S == S0 && pr[g].p.full_tiles == 0;
    if (ok) G.csplit = S0;
  }
  {
    static int h = -1;
    if (h < 0) {
      const char* e = getenv("B2_GEMM_L2HINT");  // 0: no hints; 2: also A evict_first (A/B); +4: streaming output stores
      h = !e ? 1 : atoi(e);
    }
    G.l2hint = h;
  }
  int rc = 0;
  for (int g = 0; g < n && !rc; ++g) {
    TcParams& p = pr[g].p;
    if (pr[g].S > 1 && G.csplit == 1) {
      rc = b2_alloc((size_t)pr[g].S * pr[g].T * (BM * cg) * BN * sizeof(float), st, &pr[g].part);
      p.ws = (float*)pr[g].part;
    }
    // fused column sums (bias gradient of the layer below): fp64 partials per
    // 128-row block from the GEMM epilogue (whole tiles) and the tail stage
    pr[g].cs_rows = (p.M + BM - 1) / BM;
    if (!rc && pr[g].colsum_out) {
      rc = b2_alloc((size_t)pr[g].cs_rows * p.N * sizeof(double), st, &pr[g].cs_part);
      p.colsum = (double*)pr[g].cs_part;
    }
  }
  auto alloc_parts = [&]() -> int {  // K-slice partials (the L2 path)
    for (int g = 0; g < n; ++g) {
      TcParams& p = pr[g].p;
      if (pr[g].S > 1 && G.csplit == 1 && !pr[g].part) {
        B2_TRY(b2_alloc((size_t)pr[g].S * pr[g].T * (BM * cg) * BN * sizeof(float), st, &pr[g].part));
        p.ws = (float*)pr[g].part;
      }
    }
    return 0;
  };
  if (!rc) {
    auto run = [&]() -> int {
#define B2_TC(MD)                                                        \
  if (mode == MD) return cg == 2 ? launch_tc<MD, 2>(pr, n, G, st) : launch_tc<MD, 1>(pr, n, G, st);
      if (m2) return launch_tc<6, 2>(pr, n, G, st);
      B2_TC(1) B2_TC(2) B2_TC(3) B2_TC(4) B2_TC(5)
#undef B2_TC
      return fail("gemm_tc: unknown mode");
    };
    rc = run();
    if (rc == kCsplitNoFit) {  // not every cluster fits at once: partials through L2
      G.csplit = 1;
      rc = alloc_parts();
      if (!rc) rc = run();
    }
  }
  for (int g = 0; g < n; ++g) {
    const TcParams& p = pr[g].p;
    if (!rc && pr[g].S > 1 && G.csplit == 1) {
      dim3 grid2((unsigned)pr[g].T, cg, BN / 32);
#define B2_SKE(E) k_tail_epilogue<E><<<grid2, dim3(32, 16), 0, st>>>(p)
      if (!p.s_hi) B2_SKE(0);
      else if (mode == 4) B2_SKE(4);
      else if (mode == 5) B2_SKE(5);
      else B2_SKE(2);
#undef B2_SKE
      rc = launched("b2_gemm(tcgen05 tail K-slice epilogue)");
    }
    if (pr[g].part) b2_free(pr[g].part, st);
    if (!rc && pr[g].cs_part) {
      k_colsum_final<<<(unsigned)((p.N + 31) / 32), 256, 0, st>>>(
          pr[g].colsum_out, (const double*)pr[g].cs_part, pr[g].cs_rows, p.N);
      rc = launched("b2_gemm(tcgen05 column sums)");
    }
    if (pr[g].cs_part) b2_free(pr[g].cs_part, st);
  }
  return rc;
}

// mode 1: a0/b0 raw; mode 3: a0/b0 = hi arrays, a1/b1 = lo arrays (contiguous);
// mode 2: a0/b0 raw fp32 (lda/ldb), a1/b1 = bf16 hi, a2/b2 = bf16 lo (contiguous);
// mode 4: a0/b0 = bf16 casts; mode 5: a0/b0 = bf16 hi, a1/b1 = bf16 lo (contiguous)
int gemm_tc(int ta, int tb, int mode, int64_t M, int64_t N, int64_t K, const void* a0,
            const void* a1, const void* a2, int64_t lda, const void* b0, const void* b1,
            const void* b2_, int64_t ldb, float* C, int64_t ldc, const float* bias, int epi,
            cudaStream_t st, const float* mask, void* s_hi, void* s_lo, float* colsum_out,
            const uint64_t* mask_bits, uint64_t* bits_out) {
  TcDesc d{ta, tb, M, N, K, a0, a1, a2, lda, b0, b1, b2_, ldb, C, ldc, bias, epi,
           mask, s_hi, s_lo, colsum_out, mask_bits, bits_out};
  return gemm_tc_group(mode, &d, 1, st);
}

}  // namespace b2
