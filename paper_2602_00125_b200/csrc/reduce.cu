// Reduction engine: sum / mean / max over any axis set.
//
// Replaces tensorlite/core.py:581-728 (_sum_all, _axis_scan, sum, mean, max).
// * sums accumulate in fp64 and round to f32 once (the reference accumulates
//   Python doubles); mean = f32(dsum / count) in double (core.py:671, 682);
// * max keeps (value, first index): strict '>' scan semantics, ties go to the
//   lower row-major index, a NaN in the first scanned slot sticks and later
//   NaNs are skipped (core.py:709-713). Inside a thread a plain `v > best`
//   scan skips NaNs for free; the first-slot NaN is checked once per output;
//   the cross-thread combine is associative so the parallel order cannot
//   change the winner;
// * deterministic: work is partitioned by a fixed function of the shape and
//   the SM count, partials combine in a fixed order (the reference's
//   worker-count-independent chunk contract, parallel.py:1-8, 48-63).
//
// HBM-bound: every thread keeps 4 independent 128-bit loads in flight
// (unrolled, independent accumulators).
//
// Canonical forms (after dropping size-1 axes):
//   contiguous x with the reduced axes one contiguous block  -> [O1, R, I]
//   (I == 1 is a row reduction); anything else is first gathered into a
//   [kept..., reduced...] contiguous temp and reduced as rows.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "common.cuh"

extern "C" int b2_alloc(size_t, void*, void**);
extern "C" int b2_free(void*, void*);

namespace {

constexpr int64_t kNone = INT64_MAX;
// internal op: max without the first-index routing (no gradient to route)
constexpr int kMaxValue = 3;

struct MaxAcc {
  float v;
  int64_t i;
};

__device__ __forceinline__ bool sticky(const MaxAcc& a) { return a.i == 0 && isnan(a.v); }

__device__ __forceinline__ MaxAcc max_combine(const MaxAcc& a, const MaxAcc& b) {
  if (sticky(a)) return a;
  if (sticky(b)) return b;
  if (a.i == kNone) return b;
  if (b.i == kNone) return a;
  if (a.v > b.v) return a;
  if (b.v > a.v) return b;
  return a.i < b.i ? a : b;
}

// in-order scan step: NaN never compares greater, so it is skipped
// indices inside a scan are 32-bit (reduced extents < 2^31, checked on the host)
constexpr int kNone32 = INT32_MAX;
__device__ __forceinline__ void max_scan(float& best, int& bi, float v, int64_t i) {
  const bool gt = v > best;  // predicated selects, no branch
  best = gt ? v : best;
  bi = gt ? (int)i : bi;
}
__device__ __forceinline__ MaxAcc mk(float b, int i) {
  return MaxAcc{b, i == kNone32 ? kNone : (int64_t)i};
}

__device__ __forceinline__ MaxAcc shfl_max(MaxAcc a, int off) {
  MaxAcc b;
  b.v = __shfl_xor_sync(0xffffffffu, a.v, off);
  b.i = __shfl_xor_sync(0xffffffffu, a.i, off);
  return b;
}

template <int GROUP>
__device__ __forceinline__ double group_sum(double v, double* sh) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if (GROUP == 32) return v;
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < GROUP / 32 ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
  }
  __syncthreads();
  return t;  // valid in thread 0
}

template <int GROUP>
__device__ __forceinline__ MaxAcc group_max(MaxAcc a, MaxAcc* sh) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) a = max_combine(a, shfl_max(a, off));
  if (GROUP == 32) return a;
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = a;
  __syncthreads();
  MaxAcc t{0.f, kNone};
  if (threadIdx.x < 32) {
    if (threadIdx.x < GROUP / 32) t = sh[threadIdx.x];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t = max_combine(t, shfl_max(t, off));
  }
  __syncthreads();
  return t;
}

// Single-launch second stage: thread 0 of every CTA of a group publishes the
// CTA's partials, then arrives on the group's counter with release/acquire
// semantics; the CTA that arrives last (it sees every other partial) folds
// them and re-arms the counter for the next launch on this stream.
__device__ __forceinline__ bool arrive_last(unsigned* ctr, int n, unsigned* flag) {
  __syncthreads();  // this CTA's partial stores precede the arrival
  if (threadIdx.x == 0) {
    unsigned prev;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(ctr) : "memory");
    const bool is_last = prev == (unsigned)n - 1;
    if (is_last) *ctr = 0;
    *flag = is_last;
  }
  __syncthreads();
  return *flag != 0;
}

// ---------------------------------------------------------------- row reduce
// x: [O, R] contiguous rows. grid = (ceil(O / rows_per_cta), S); each group of
// GROUP threads owns one row and the split range [s*Rs, min(R,(s+1)*Rs)).
// S == 1 -> final outputs; S > 1 -> partials [S][O].
template <int OP, int GROUP, bool VEC>
__global__ void __launch_bounds__(256) k_rows(const float* __restrict__ x, int64_t O, int64_t R,
                                              int64_t Rs, float* __restrict__ out,
                                              int64_t* __restrict__ argr, double* __restrict__ psum,
                                              MaxAcc* __restrict__ pmax, double count,
                                              unsigned* __restrict__ ticket) {
  __shared__ double shd[8];
  __shared__ MaxAcc shm[8];
  __shared__ unsigned last;
  constexpr int RPC = 256 / GROUP;
  const int g = threadIdx.x / GROUP, t = threadIdx.x % GROUP;
  const int64_t o = blockIdx.x * (int64_t)RPC + g;
  const int S = gridDim.y, s = blockIdx.y;
  const int64_t r0 = s * Rs, r1 = min(R, r0 + Rs);
  const bool live = o < O;
  const float* row = x + (live ? o : 0) * R;
  if (OP != B2_RED_MAX) {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    if (live) {
      if (VEC) {
        int64_t r = r0 + 4 * t;
        for (; r + 28 * GROUP + 3 < r1; r += 32 * GROUP) {  // 8 x 128-bit loads in flight
          float4 v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = __ldg(reinterpret_cast<const float4*>(row + r + 4 * k * GROUP));
#pragma unroll
          for (int k = 0; k < 8; k += 4) {
            a0 += (double)v[k].x + (double)v[k].y + (double)v[k].z + (double)v[k].w;
            a1 += (double)v[k + 1].x + (double)v[k + 1].y + (double)v[k + 1].z + (double)v[k + 1].w;
            a2 += (double)v[k + 2].x + (double)v[k + 2].y + (double)v[k + 2].z + (double)v[k + 2].w;
            a3 += (double)v[k + 3].x + (double)v[k + 3].y + (double)v[k + 3].z + (double)v[k + 3].w;
          }
        }
        for (; r + 12 * GROUP + 3 < r1; r += 16 * GROUP) {  // 4 x 128-bit loads in flight
          const float4 v0 = *reinterpret_cast<const float4*>(row + r);
          const float4 v1 = *reinterpret_cast<const float4*>(row + r + 4 * GROUP);
          const float4 v2 = *reinterpret_cast<const float4*>(row + r + 8 * GROUP);
          const float4 v3 = *reinterpret_cast<const float4*>(row + r + 12 * GROUP);
          a0 += (double)v0.x + (double)v0.y + (double)v0.z + (double)v0.w;
          a1 += (double)v1.x + (double)v1.y + (double)v1.z + (double)v1.w;
          a2 += (double)v2.x + (double)v2.y + (double)v2.z + (double)v2.w;
          a3 += (double)v3.x + (double)v3.y + (double)v3.z + (double)v3.w;
        }
        for (; r < r1; r += 4 * GROUP) {
          if (r + 3 < r1) {
            const float4 v = *reinterpret_cast<const float4*>(row + r);
            a0 += (double)v.x + (double)v.y + (double)v.z + (double)v.w;
          } else {
            for (int64_t k = r; k < r1; ++k) a0 += (double)row[k];
          }
        }
      } else {
        int64_t r = r0 + t;
        for (; r + 3 * GROUP < r1; r += 4 * GROUP) {
          a0 += (double)row[r];
          a1 += (double)row[r + GROUP];
          a2 += (double)row[r + 2 * GROUP];
          a3 += (double)row[r + 3 * GROUP];
        }
        for (; r < r1; r += GROUP) a0 += (double)row[r];
      }
    }
    const double tot = group_sum<GROUP>((a0 + a1) + (a2 + a3), shd);
    if (S == 1) {
      if (live && t == 0) out[o] = OP == B2_RED_MEAN ? __double2float_rn(tot / count) : __double2float_rn(tot);
      return;
    }
    // thread 0 publishes the CTA's partials itself, so its release covers them
    __shared__ double stage[RPC];
    if (t == 0) stage[g] = tot;
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 0; k < RPC; ++k)
        if (blockIdx.x * (int64_t)RPC + k < O) psum[(int64_t)s * O + blockIdx.x * (int64_t)RPC + k] = stage[k];
    if (!arrive_last(ticket + blockIdx.x, S, &last)) return;
    // the last CTA of this row block folds the S partials of its rows in a
    // fixed order: group lane t takes splits t, t+GROUP, ..., then the fixed tree
    double f = 0;
    if (live)
      for (int q = t; q < S; q += GROUP) f += __ldcg(psum + (int64_t)q * O + o);
    f = group_sum<GROUP>(f, shd);
    if (live && t == 0) out[o] = OP == B2_RED_MEAN ? __double2float_rn(f / count) : __double2float_rn(f);
  } else {
    // each of the 4 lanes of the unroll scans its own index sequence in order
    float b0 = -INFINITY, b1 = -INFINITY, b2 = -INFINITY, b3 = -INFINITY;
    int i0 = kNone32, i1 = kNone32, i2 = kNone32, i3 = kNone32;
    if (live) {
      if (VEC) {
        int64_t r = r0 + 4 * t;
        for (; r + 12 * GROUP + 3 < r1; r += 16 * GROUP) {  // 4 x 128-bit loads in flight
          const float4 v0 = *reinterpret_cast<const float4*>(row + r);
          const float4 v1 = *reinterpret_cast<const float4*>(row + r + 4 * GROUP);
          const float4 v2 = *reinterpret_cast<const float4*>(row + r + 8 * GROUP);
          const float4 v3 = *reinterpret_cast<const float4*>(row + r + 12 * GROUP);
          const int64_t q1 = r + 4 * GROUP, q2 = r + 8 * GROUP, q3 = r + 12 * GROUP;
          max_scan(b0, i0, v0.x, r);  max_scan(b1, i1, v0.y, r + 1);
          max_scan(b2, i2, v0.z, r + 2);  max_scan(b3, i3, v0.w, r + 3);
          max_scan(b0, i0, v1.x, q1);  max_scan(b1, i1, v1.y, q1 + 1);
          max_scan(b2, i2, v1.z, q1 + 2);  max_scan(b3, i3, v1.w, q1 + 3);
          max_scan(b0, i0, v2.x, q2);  max_scan(b1, i1, v2.y, q2 + 1);
          max_scan(b2, i2, v2.z, q2 + 2);  max_scan(b3, i3, v2.w, q2 + 3);
          max_scan(b0, i0, v3.x, q3);  max_scan(b1, i1, v3.y, q3 + 1);
          max_scan(b2, i2, v3.z, q3 + 2);  max_scan(b3, i3, v3.w, q3 + 3);
        }
        for (; r < r1; r += 4 * GROUP) {
          if (r + 3 < r1) {
            const float4 v = *reinterpret_cast<const float4*>(row + r);
            max_scan(b0, i0, v.x, r);
            max_scan(b1, i1, v.y, r + 1);
            max_scan(b2, i2, v.z, r + 2);
            max_scan(b3, i3, v.w, r + 3);
          } else {
            for (int64_t k = r; k < r1; ++k) max_scan(b0, i0, row[k], k);
          }
        }
      } else {
        for (int64_t r = r0 + t; r < r1; r += GROUP) max_scan(b0, i0, row[r], r);
      }
    }
    MaxAcc acc = max_combine(max_combine(mk(b0, i0), mk(b1, i1)), max_combine(mk(b2, i2), mk(b3, i3)));
    if (live && s == 0 && t == 0) {
      const float v0 = row[0];
      if (isnan(v0)) acc = MaxAcc{v0, 0};          // first-slot NaN sticks
      else if (acc.i == kNone || !(acc.v > v0)) {  // all -inf/NaN: x0 at index 0
        if (acc.i == kNone || acc.v == v0) acc = max_combine(acc, MaxAcc{v0, 0});
      }
    }
    const MaxAcc best = group_max<GROUP>(acc, shm);
    if (S == 1) {
      if (live && t == 0) {
        out[o] = best.v;
        if (argr) argr[o] = best.i;
      }
      return;
    }
    __shared__ MaxAcc stagem[RPC];
    if (t == 0) stagem[g] = best;
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 0; k < RPC; ++k)
        if (blockIdx.x * (int64_t)RPC + k < O) pmax[(int64_t)s * O + blockIdx.x * (int64_t)RPC + k] = stagem[k];
    if (!arrive_last(ticket + blockIdx.x, S, &last)) return;
    MaxAcc f{0.f, kNone};
    if (live)
      for (int q = t; q < S; q += GROUP) {
        const MaxAcc* pq = pmax + (int64_t)q * O + o;
        f = max_combine(f, MaxAcc{__ldcg(&pq->v), __ldcg(&pq->i)});
      }
    f = group_max<GROUP>(f, shm);
    if (live && t == 0) {
      out[o] = f.v;
      if (argr) argr[o] = f.i;
    }
  }
}

// ---------------------------------------------------------------- mid reduce
// x: [O1, R, I] contiguous; output o = o1*I + i. Each thread owns 4
// consecutive columns (float4; I % 4 == 0) or one column; rows unrolled x4.
// grid = (cb * O1, S), cb = ceil(I / (256 * V)).
// Column strips with in-CTA row lanes: a CTA owns CL*V consecutive columns
// (CL column lanes x V columns each) and RL = 256/CL row lanes; row lane k
// scans rows k, k+RL, ... of the CTA's row split (a warp reads 2 rows x 256 B,
// coalesced), then a fixed shared-memory tree folds the RL lanes. Splits S
// stay small (~8), so the second stage is cheap. grid = (strips * O1, S).
template <int OP, int V, int CL>
__global__ void __launch_bounds__(256) k_strip(const float* __restrict__ x, int64_t O1, int64_t R,
                                               int64_t I, int64_t Rs, float* __restrict__ out,
                                               int64_t* __restrict__ argr,
                                               double* __restrict__ psum,
                                               MaxAcc* __restrict__ pmax, double count,
                                               int64_t strips) {
  constexpr int RL = 256 / CL;  // CL column lanes x RL row lanes
  __shared__ double shd[256 * V];
  __shared__ MaxAcc shm[OP == B2_RED_MAX ? 256 * V : 1];
  const int cl = threadIdx.x % CL, rl = threadIdx.x / CL;
  const int64_t o1 = blockIdx.x / strips;
  const int64_t i = ((blockIdx.x - o1 * strips) * CL + cl) * V;
  const int S = gridDim.y, s = blockIdx.y;
  const int64_t r0 = s * Rs, r1 = min(R, r0 + Rs);
  const bool live = i < I;
  const float* base = x + o1 * R * I + (live ? i : 0);
  if constexpr (OP == B2_RED_SUM || OP == B2_RED_MEAN) {
    double a[V];
#pragma unroll
    for (int j = 0; j < V; ++j) a[j] = 0.0;
    if (live) {
      int64_t r = r0 + rl;
      if (V == 4) {  // 8 independent 128-bit loads in flight, then fold
        for (; r + 7 * RL < r1; r += 8 * RL) {
          float4 v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = __ldg(reinterpret_cast<const float4*>(base + (r + k * RL) * I));
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            a[0] += (double)v[k].x;
            a[V > 1 ? 1 : 0] += (double)v[k].y;
            a[V > 2 ? 2 : 0] += (double)v[k].z;
            a[V > 3 ? 3 : 0] += (double)v[k].w;
          }
        }
      }
      for (; r + 3 * RL < r1; r += 4 * RL) {  // 4 independent loads in flight
        if (V == 4) {
          const float4 v0 = *reinterpret_cast<const float4*>(base + r * I);
          const float4 v1 = *reinterpret_cast<const float4*>(base + (r + RL) * I);
          const float4 v2 = *reinterpret_cast<const float4*>(base + (r + 2 * RL) * I);
          const float4 v3 = *reinterpret_cast<const float4*>(base + (r + 3 * RL) * I);
          a[0] += (double)v0.x + (double)v1.x + (double)v2.x + (double)v3.x;
          a[V > 1 ? 1 : 0] += (double)v0.y + (double)v1.y + (double)v2.y + (double)v3.y;
          a[V > 2 ? 2 : 0] += (double)v0.z + (double)v1.z + (double)v2.z + (double)v3.z;
          a[V > 3 ? 3 : 0] += (double)v0.w + (double)v1.w + (double)v2.w + (double)v3.w;
        } else {
          a[0] += (double)base[r * I] + (double)base[(r + RL) * I] + (double)base[(r + 2 * RL) * I] +
                  (double)base[(r + 3 * RL) * I];
        }
      }
      for (; r < r1; r += RL) {
        if (V == 4) {
          const float4 v = *reinterpret_cast<const float4*>(base + r * I);
          a[0] += (double)v.x;
          a[V > 1 ? 1 : 0] += (double)v.y;
          a[V > 2 ? 2 : 0] += (double)v.z;
          a[V > 3 ? 3 : 0] += (double)v.w;
        } else {
          a[0] += (double)base[r * I];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < V; ++j) shd[(rl * CL + cl) * V + j] = a[j];
    __syncthreads();
    for (int h = RL / 2; h > 0; h >>= 1) {
      if (rl < h)
#pragma unroll
        for (int j = 0; j < V; ++j) shd[(rl * CL + cl) * V + j] += shd[((rl + h) * CL + cl) * V + j];
      __syncthreads();
    }
    if (rl == 0 && live) {
      const int64_t o = o1 * I + i;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const double t = shd[cl * V + j];
        if (S > 1)
          psum[(int64_t)s * O1 * I + o + j] = t;
        else
          out[o + j] = OP == B2_RED_MEAN ? __double2float_rn(t / count) : __double2float_rn(t);
      }
    }
  } else {
    float b[V];
    int bi[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      b[j] = -INFINITY;
      bi[j] = kNone32;
    }
    if (live) {
      auto scan4 = [&](const float4& v, int64_t r) {
        max_scan(b[0], bi[0], v.x, r);
        max_scan(b[V > 1 ? 1 : 0], bi[V > 1 ? 1 : 0], v.y, r);
        max_scan(b[V > 2 ? 2 : 0], bi[V > 2 ? 2 : 0], v.z, r);
        max_scan(b[V > 3 ? 3 : 0], bi[V > 3 ? 3 : 0], v.w, r);
      };
      int64_t r = r0 + rl;
      if (V == 4) {
        // 8 x 128-bit loads in flight; per column the block maximum is an
        // FMNMX tree (NaNs drop out unless all are NaN) and only a block that
        // beats the running best (rare after the first few) locates its first
        // maximal row -- the in-order strict '>' scan's answer for the block.
        constexpr int U = 8;
        auto comp = [](const float4& q, int j) { return j == 0 ? q.x : j == 1 ? q.y : j == 2 ? q.z : q.w; };
        for (; r + (U - 1) * RL < r1; r += U * RL) {
          float4 v[U];
#pragma unroll
          for (int k = 0; k < U; ++k) v[k] = __ldg(reinterpret_cast<const float4*>(base + (r + k * RL) * I));
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float m = comp(v[0], j);
#pragma unroll
            for (int k = 1; k < U; ++k) m = fmaxf(m, comp(v[k], j));
            if (m > b[j]) {
              int kk = U - 1;
#pragma unroll
              for (int k = U - 2; k >= 0; --k) kk = comp(v[k], j) == m ? k : kk;
              // the element itself, not m: keeps the sign of a zero maximum
#pragma unroll
              for (int k = 0; k < U; ++k) b[j] = k == kk ? comp(v[k], j) : b[j];
              bi[j] = (int)(r + kk * RL);
            }
          }
        }
        for (; r < r1; r += RL) scan4(*reinterpret_cast<const float4*>(base + r * I), r);
      } else {
        for (; r + 3 * RL < r1; r += 4 * RL) {
          const float v0 = base[r * I], v1 = base[(r + RL) * I], v2 = base[(r + 2 * RL) * I],
                      v3 = base[(r + 3 * RL) * I];
          max_scan(b[0], bi[0], v0, r);
          max_scan(b[0], bi[0], v1, r + RL);
          max_scan(b[0], bi[0], v2, r + 2 * RL);
          max_scan(b[0], bi[0], v3, r + 3 * RL);
        }
        for (; r < r1; r += RL) max_scan(b[0], bi[0], base[r * I], r);
      }
    }
#pragma unroll
    for (int j = 0; j < V; ++j) shm[(rl * CL + cl) * V + j] = mk(b[j], bi[j]);
    __syncthreads();
    for (int h = RL / 2; h > 0; h >>= 1) {
      if (rl < h)
#pragma unroll
        for (int j = 0; j < V; ++j)
          shm[(rl * CL + cl) * V + j] =
              max_combine(shm[(rl * CL + cl) * V + j], shm[((rl + h) * CL + cl) * V + j]);
      __syncthreads();
    }
    if (rl == 0 && live) {
      const int64_t o = o1 * I + i;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        MaxAcc acc = shm[cl * V + j];
        if (s == 0) {  // the first scanned slot of this column: NaN sticks, -inf ties at 0
          const float v0 = base[j];
          if (isnan(v0)) acc = MaxAcc{v0, 0};
          else acc = max_combine(acc, MaxAcc{v0, 0});
        }
        if (S > 1) {
          pmax[(int64_t)s * O1 * I + o + j] = acc;
        } else {
          out[o + j] = acc.v;
          if (argr) argr[o + j] = acc.i;
        }
      }
    }
  }
}

// ---------------------------------------------------------------- column reduce, cluster fold
// x: [O1, R, I] contiguous, I % 4 == 0, 16-B aligned; reduce R. A CTA owns a
// 32-column strip (8 column lanes x float4) and one of CS row splits; its 32
// row lanes scan rows rl, rl+32, ... with 8 x 128-bit loads in flight (a warp
// reads 4 rows x 128 B). The row lanes fold in a fixed order (warp butterfly,
// then warps in index order), and the CS CTAs of a cluster -- the row splits
// of one strip -- fold through distributed shared memory in rank order: no
// global partials and no second launch. Measured (scripts/hbm_probe.cu): the
// read pattern alone reaches ~82% of HBM at 512 CTAs; a separate partials
// pass + second kernel costs ~2 us of a ~12 us op.
template <int OP>
__global__ void __launch_bounds__(256) k_cols(const float* __restrict__ x, int64_t R, int64_t I,
                                              int64_t Rs, float* __restrict__ out,
                                              int64_t* __restrict__ argr, double count,
                                              int64_t strips) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ double shd[8][32];
  __shared__ MaxAcc shm[OP == B2_RED_MAX ? 8 : 1][32];
  __shared__ double cpd[32];
  __shared__ MaxAcc cpm[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cl = lane & 7, rl = w * 4 + (lane >> 3);  // 8 column lanes x 32 row lanes
  constexpr int RL = 32;
  const int64_t o1 = blockIdx.x / strips;
  const int64_t i = ((blockIdx.x - o1 * strips) * 8 + cl) * 4;
  const int s = blockIdx.y, S = gridDim.y;
  const int64_t r0 = s * Rs, r1 = min(R, r0 + Rs);
  const bool live = i < I;
  const float* base = x + o1 * R * I + (live ? i : 0);
  if constexpr (OP == B2_RED_SUM || OP == B2_RED_MEAN) {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    if (live) {
      int64_t r = r0 + rl;
      for (; r + 7 * RL < r1; r += 8 * RL) {
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldg(reinterpret_cast<const float4*>(base + (r + k * RL) * I));
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          a0 += (double)v[k].x;
          a1 += (double)v[k].y;
          a2 += (double)v[k].z;
          a3 += (double)v[k].w;
        }
      }
      for (; r < r1; r += RL) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(base + r * I));
        a0 += (double)v.x;
        a1 += (double)v.y;
        a2 += (double)v.z;
        a3 += (double)v.w;
      }
    }
    // fold the warp's 4 row lanes (lane bits 3, 4), then the 8 warps in order
#pragma unroll
    for (int off = 8; off <= 16; off <<= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, off);
      a1 += __shfl_xor_sync(0xffffffffu, a1, off);
      a2 += __shfl_xor_sync(0xffffffffu, a2, off);
      a3 += __shfl_xor_sync(0xffffffffu, a3, off);
    }
    if (lane < 8) {
      shd[w][cl * 4 + 0] = a0;
      shd[w][cl * 4 + 1] = a1;
      shd[w][cl * 4 + 2] = a2;
      shd[w][cl * 4 + 3] = a3;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      double t = shd[0][threadIdx.x];
#pragma unroll
      for (int k = 1; k < 8; ++k) t += shd[k][threadIdx.x];
      cpd[threadIdx.x] = t;
    }
    cluster.sync();
    if (s == 0 && threadIdx.x < 32) {  // cluster rank 0 folds the row splits in rank order
      const int64_t c = ((blockIdx.x - o1 * strips) * 8) * 4 + threadIdx.x;
      double t = cpd[threadIdx.x];
      for (int q = 1; q < S; ++q) t += cluster.map_shared_rank(cpd, q)[threadIdx.x];
      if (c < I) {
        const int64_t o = o1 * I + c;
        out[o] = OP == B2_RED_MEAN ? __double2float_rn(t / count) : __double2float_rn(t);
      }
    }
    cluster.sync();  // keep every CTA's shared memory alive until rank 0 has read it
  } else if constexpr (OP == kMaxValue) {
    // value-only max (no gradient will be routed, so no index is tracked):
    // fmaxf skips NaN like the strict '>' scan; the first-slot NaN rule is
    // applied at the end, and a zero maximum takes the sign of the column's
    // first zero (the in-order scan keeps the first of +-0 ties)
    __shared__ float shv[8][32];
    __shared__ float cpv[32];
    float b[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    const int64_t cfirst = ((blockIdx.x - o1 * strips) * 8) * 4 + threadIdx.x;
    const float v0 = (s == 0 && threadIdx.x < 32 && cfirst < I) ? x[o1 * R * I + cfirst] : 0.0f;
    if (live) {
      int64_t r = r0 + rl;
      constexpr int U = 8;
      for (; r + (U - 1) * RL < r1; r += U * RL) {
        float4 v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) v[k] = __ldg(reinterpret_cast<const float4*>(base + (r + k * RL) * I));
#pragma unroll
        for (int k = 0; k < U; ++k) {
          b[0] = fmaxf(b[0], v[k].x);
          b[1] = fmaxf(b[1], v[k].y);
          b[2] = fmaxf(b[2], v[k].z);
          b[3] = fmaxf(b[3], v[k].w);
        }
      }
      for (; r < r1; r += RL) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(base + r * I));
        b[0] = fmaxf(b[0], v.x);
        b[1] = fmaxf(b[1], v.y);
        b[2] = fmaxf(b[2], v.z);
        b[3] = fmaxf(b[3], v.w);
      }
    }
#pragma unroll
    for (int off = 8; off <= 16; off <<= 1)
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = fmaxf(b[j], __shfl_xor_sync(0xffffffffu, b[j], off));
    if (lane < 8)
#pragma unroll
      for (int j = 0; j < 4; ++j) shv[w][cl * 4 + j] = b[j];
    __syncthreads();
    if (threadIdx.x < 32) {
      float t = shv[0][threadIdx.x];
#pragma unroll
      for (int k = 1; k < 8; ++k) t = fmaxf(t, shv[k][threadIdx.x]);
      cpv[threadIdx.x] = t;
    }
    cluster.sync();
    if (s == 0 && threadIdx.x < 32) {
      const int64_t c = cfirst;
      float t = cpv[threadIdx.x];
      for (int q = 1; q < S; ++q) t = fmaxf(t, cluster.map_shared_rank(cpv, q)[threadIdx.x]);
      if (c < I) {
        if (isnan(v0)) {
          t = v0;
        } else {
          t = fmaxf(t, v0);
          if (t == 0.0f) {  // every non-NaN value <= 0: the first zero in scan order wins
            const float* col = x + o1 * R * I + c;
            for (int64_t r = 0; r < R; ++r) {
              const float v = col[r * I];
              if (v == 0.0f) {
                t = v;
                break;
              }
            }
          }
        }
        out[o1 * I + c] = t;
      }
    }
    cluster.sync();
  } else {
    float b[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    int bi[4] = {kNone32, kNone32, kNone32, kNone32};
    // the first scanned slot of each column (NaN sticks, -inf ties at 0), loaded
    // up front so the fold at the end does not wait on a global load
    const int64_t cfirst = ((blockIdx.x - o1 * strips) * 8) * 4 + threadIdx.x;
    const float v0 = (s == 0 && threadIdx.x < 32 && cfirst < I) ? x[o1 * R * I + cfirst] : 0.0f;
    auto comp = [](const float4& q, int j) { return j == 0 ? q.x : j == 1 ? q.y : j == 2 ? q.z : q.w; };
    if (live) {
      int64_t r = r0 + rl;
      constexpr int U = 8;
      for (; r + (U - 1) * RL < r1; r += U * RL) {
        float4 v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) v[k] = __ldg(reinterpret_cast<const float4*>(base + (r + k * RL) * I));
        // per column: FMNMX tree over the U rows; only a block that beats the
        // running best locates its first maximal row (the in-order scan's answer)
        // branch-free: the block's first maximal row is located for every
        // column and kept only where the block beats the running best (a
        // divergent locate doubled the warp's instructions). The value kept is
        // the FMNMX result; a zero maximum's sign is restored from the winning
        // element at the end (fmaxf may return +0 for -0).
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float m = comp(v[0], j);
#pragma unroll
          for (int k = 1; k < U; ++k) m = fmaxf(m, comp(v[k], j));
          int kk = U - 1;
#pragma unroll
          for (int k = U - 2; k >= 0; --k) kk = comp(v[k], j) == m ? k : kk;
          const bool gt = m > b[j];
          b[j] = gt ? m : b[j];
          bi[j] = gt ? (int)(r + kk * RL) : bi[j];
        }
      }
      for (; r < r1; r += RL) {
        const float4 w = __ldg(reinterpret_cast<const float4*>(base + r * I));
#pragma unroll
        for (int j = 0; j < 4; ++j) max_scan(b[j], bi[j], comp(w, j), r);
      }
    }
    MaxAcc acc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j] = mk(b[j], bi[j]);
#pragma unroll
    for (int off = 8; off <= 16; off <<= 1)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = max_combine(acc[j], shfl_max(acc[j], off));
    if (lane < 8)
#pragma unroll
      for (int j = 0; j < 4; ++j) shm[w][cl * 4 + j] = acc[j];
    __syncthreads();
    if (threadIdx.x < 32) {
      MaxAcc t = shm[0][threadIdx.x];
#pragma unroll
      for (int k = 1; k < 8; ++k) t = max_combine(t, shm[k][threadIdx.x]);
      cpm[threadIdx.x] = t;
    }
    cluster.sync();
    if (s == 0 && threadIdx.x < 32) {
      const int64_t c = ((blockIdx.x - o1 * strips) * 8) * 4 + threadIdx.x;
      MaxAcc t = cpm[threadIdx.x];
      for (int q = 1; q < S; ++q) t = max_combine(t, cluster.map_shared_rank(cpm, q)[threadIdx.x]);
      if (c < I) {
        if (isnan(v0)) t = MaxAcc{v0, 0};
        else t = max_combine(t, MaxAcc{v0, 0});
        if (t.v == 0.0f && t.i != kNone) t.v = x[o1 * R * I + t.i * I + c];  // the winner's own zero sign
        const int64_t o = o1 * I + c;
        out[o] = t.v;
        if (argr) argr[o] = t.i;
      }
    }
    cluster.sync();
  }
}


// ---------------------------------------------------------------- row splits streamed by TMA
// Few long rows (the full sum, row sums of a handful of rows): each CTA owns a
// run of 16-KB chunks of one row and streams them through a 4-deep
// shared-memory ring with cp.async.bulk (one elected thread issues, an
// mbarrier per stage carries the byte count), so the bytes in flight per SM
// (2 CTAs x 64 KB) do not depend on registers; the threads scan shared memory
// in row order. The row's tail past the last whole chunk goes to the last
// split with plain loads; partials fold in the last-arriving CTA (arrive_last).
// Measured (scripts/hbm_probe.cu): 77% of HBM for a 64 MiB full sum vs 69% for
// register-staged loads at the best split count.
constexpr int kBulkStages = 4, kBulkChunk = 4096;  // floats per chunk (16 KB)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk_chunk(float* dst, const float* src, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)),
               "r"(kBulkChunk * 4) : "memory");
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(kBulkChunk * 4), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(su32(bar)), "r"(parity) : "memory");
}

template <int OP>
__global__ void __launch_bounds__(256) k_bulk_rows(const float* __restrict__ x, int64_t O, int64_t R,
                                                   int64_t cps, float* __restrict__ out,
                                                   int64_t* __restrict__ argr, double* __restrict__ psum,
                                                   MaxAcc* __restrict__ pmax, double count,
                                                   unsigned* __restrict__ ticket) {
  extern __shared__ __align__(128) float sbuf[];
  __shared__ __align__(8) uint64_t bars[kBulkStages];
  __shared__ double shd[8];
  __shared__ MaxAcc shm[8];
  __shared__ unsigned last;
  const int64_t o = blockIdx.x;
  const int s = blockIdx.y, S = gridDim.y;
  const float* row = x + o * R;
  const int64_t nfull = R / kBulkChunk;
  const int64_t c0 = min(nfull, s * cps), c1 = min(nfull, c0 + cps), nc = c1 - c0;
  const int t = threadIdx.x;
  if (t == 0) {
    for (int b = 0; b < kBulkStages; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int b = 0; b < kBulkStages && b < nc; ++b)
      bulk_chunk(sbuf + b * kBulkChunk, row + (c0 + b) * kBulkChunk, &bars[b]);
  }
  __syncthreads();
  double a0 = 0, a1 = 0;
  float b0 = -INFINITY, b1 = -INFINITY, b2 = -INFINITY, b3 = -INFINITY;
  int i0 = kNone32, i1 = kNone32, i2 = kNone32, i3 = kNone32;
  for (int64_t c = 0; c < nc; ++c) {
    const int st = (int)(c % kBulkStages);
    bar_wait(&bars[st], (uint32_t)(c / kBulkStages) & 1);
    const float4* q = reinterpret_cast<const float4*>(sbuf + st * kBulkChunk) + t;
    const float4 v0 = q[0], v1 = q[256], v2 = q[512], v3 = q[768];
    if (OP != B2_RED_MAX) {
      a0 += ((double)v0.x + (double)v0.y) + ((double)v0.z + (double)v0.w);
      a1 += ((double)v1.x + (double)v1.y) + ((double)v1.z + (double)v1.w);
      a0 += ((double)v2.x + (double)v2.y) + ((double)v2.z + (double)v2.w);
      a1 += ((double)v3.x + (double)v3.y) + ((double)v3.z + (double)v3.w);
    } else {
      const int64_t e = (c0 + c) * kBulkChunk + 4 * t;  // row-order scan per component lane
      max_scan(b0, i0, v0.x, e);        max_scan(b1, i1, v0.y, e + 1);
      max_scan(b2, i2, v0.z, e + 2);    max_scan(b3, i3, v0.w, e + 3);
      max_scan(b0, i0, v1.x, e + 1024); max_scan(b1, i1, v1.y, e + 1025);
      max_scan(b2, i2, v1.z, e + 1026); max_scan(b3, i3, v1.w, e + 1027);
      max_scan(b0, i0, v2.x, e + 2048); max_scan(b1, i1, v2.y, e + 2049);
      max_scan(b2, i2, v2.z, e + 2050); max_scan(b3, i3, v2.w, e + 2051);
      max_scan(b0, i0, v3.x, e + 3072); max_scan(b1, i1, v3.y, e + 3073);
      max_scan(b2, i2, v3.z, e + 3074); max_scan(b3, i3, v3.w, e + 3075);
    }
    __syncthreads();  // every thread is done with this stage before it is refilled
    if (t == 0 && c + kBulkStages < nc)
      bulk_chunk(sbuf + st * kBulkChunk, row + (c0 + c + kBulkStages) * kBulkChunk, &bars[st]);
  }
  if (s == S - 1)  // the row's tail past the last whole chunk
    for (int64_t k = nfull * kBulkChunk + t; k < R; k += 256) {
      if (OP != B2_RED_MAX) a0 += (double)row[k];
      else max_scan(b0, i0, row[k], k);
    }
  if (OP != B2_RED_MAX) {
    const double tot = group_sum<256>(a0 + a1, shd);
    if (t == 0) psum[(int64_t)s * O + o] = tot;
    if (!arrive_last(ticket + o, S, &last)) return;
    double f = 0;
    for (int q = t; q < S; q += 256) f += __ldcg(psum + (int64_t)q * O + o);
    f = group_sum<256>(f, shd);
    if (t == 0) out[o] = OP == B2_RED_MEAN ? __double2float_rn(f / count) : __double2float_rn(f);
  } else {
    MaxAcc acc = max_combine(max_combine(mk(b0, i0), mk(b1, i1)), max_combine(mk(b2, i2), mk(b3, i3)));
    if (s == 0 && t == 0) {  // the first scanned slot: NaN sticks, -inf ties at index 0
      const float v0 = row[0];
      if (isnan(v0)) acc = MaxAcc{v0, 0};
      else acc = max_combine(acc, MaxAcc{v0, 0});
    }
    const MaxAcc best = group_max<256>(acc, shm);
    if (t == 0) pmax[(int64_t)s * O + o] = best;
    if (!arrive_last(ticket + o, S, &last)) return;
    MaxAcc f{0.f, kNone};
    for (int q = t; q < S; q += 256) {
      const MaxAcc* pq = pmax + (int64_t)q * O + o;
      f = max_combine(f, MaxAcc{__ldcg(&pq->v), __ldcg(&pq->i)});
    }
    f = group_max<256>(f, shm);
    if (t == 0) {
      out[o] = f.v;
      if (argr) argr[o] = f.i;
    }
  }
}

// Second stage over partials [S][O]. A CTA owns `cpt` consecutive outputs
// (a power of two <= 32) with 256/cpt threads per output: thread (c, k) folds
// partials s = k, k + lpc, ... (warps read consecutive outputs: coalesced) and
// a fixed shared-memory tree combines the k's -- deterministic for a given S.
template <int OP>
__global__ void __launch_bounds__(256) k_final(int64_t O, int S, const double* __restrict__ psum,
                                               const MaxAcc* __restrict__ pmax,
                                               float* __restrict__ out, int64_t* __restrict__ argr,
                                               double count, int cpt) {
  __shared__ double shd[256];
  __shared__ MaxAcc shm[256];
  const int lpc = 256 / cpt;
  const int c = threadIdx.x % cpt, k = threadIdx.x / cpt;
  const int64_t o = blockIdx.x * (int64_t)cpt + c;
  const bool live = o < O;
  if (OP != B2_RED_MAX) {
    double acc = 0;
    if (live)
      for (int s = k; s < S; s += lpc) acc += psum[(int64_t)s * O + o];
    shd[threadIdx.x] = acc;
    __syncthreads();
    for (int h = lpc / 2; h > 0; h >>= 1) {
      if (k < h) shd[threadIdx.x] += shd[threadIdx.x + h * cpt];
      __syncthreads();
    }
    if (live && k == 0) {
      const double tot = shd[c];
      out[o] = OP == B2_RED_MEAN ? __double2float_rn(tot / count) : __double2float_rn(tot);
    }
  } else {
    MaxAcc a{0.f, kNone};
    if (live)
      for (int s = k; s < S; s += lpc) a = max_combine(a, pmax[(int64_t)s * O + o]);
    shm[threadIdx.x] = a;
    __syncthreads();
    for (int h = lpc / 2; h > 0; h >>= 1) {
      if (k < h) shm[threadIdx.x] = max_combine(shm[threadIdx.x], shm[threadIdx.x + h * cpt]);
      __syncthreads();
    }
    if (live && k == 0) {
      out[o] = shm[c].v;
      if (argr) argr[o] = shm[c].i;
    }
  }
}

template <int OP>
void launch_final(int64_t O, int64_t S, const double* psum, const MaxAcc* pmax, float* out,
                  int64_t* argr, double count, cudaStream_t st) {
  int cpt = 32;
  while (cpt > 1 && cpt / 2 >= O) cpt /= 2;
  k_final<OP><<<(unsigned)((O + cpt - 1) / cpt), 256, 0, st>>>(O, (int)S, psum, pmax, out, argr,
                                                                count, cpt);
}

__global__ void k_fill_out(float* out, int64_t* argr, int64_t n, float v) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    out[i] = v;
    if (argr) argr[i] = 0;
  }
}

struct ScatterGeom {
  int nk, nr;
  int64_t kshape[B2_MAX_DIMS], kstride[B2_MAX_DIMS];  // kept dims, contiguous input strides
  int64_t rshape[B2_MAX_DIMS], rstride[B2_MAX_DIMS];  // reduced dims
};

__global__ void k_max_scatter(float* __restrict__ gx, const float* __restrict__ g,
                              const int64_t* __restrict__ argr, int64_t O, ScatterGeom sg) {
  int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= O) return;
  int64_t pos = 0, q = o;
  for (int d = sg.nk - 1; d >= 0; --d) {
    int64_t e = sg.kshape[d];
    pos += (q % e) * sg.kstride[d];
    q /= e;
  }
  q = argr[o];
  for (int d = sg.nr - 1; d >= 0; --d) {
    int64_t e = sg.rshape[d];
    pos += (q % e) * sg.rstride[d];
    q /= e;
  }
  gx[pos] = __fadd_rn(0.0f, g[o]);  // acc[pos] += g with acc = 0.0 (core.py:723-726): -0 -> +0
}

// resident CTAs per SM of a 256-thread reduction kernel (cached per kernel)
template <int OP>
int resident(const void* kern) {
  static const void* kerns[8] = {};
  static int occ[8] = {};
  for (int i = 0; i < 8; ++i)
    if (kerns[i] == kern) return occ[i];
  int n = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, 256, 0) != cudaSuccess || n < 1) n = 1;
  for (int i = 0; i < 8; ++i)
    if (!kerns[i]) {
      kerns[i] = kern;
      occ[i] = n;
      break;
    }
  return n;
}

template <int OP>
int run_rows(const float* x, int64_t O, int64_t R, float* out, int64_t* argr, double count,
             cudaStream_t st) {
  const bool vec = ((uintptr_t)x & 15) == 0 && R % 4 == 0;
  const int sms = b2::sm_count();
  if (vec && O < 2 * sms && R >= 8 * kBulkChunk && O <= b2::kTickets) {
    // few long rows: TMA-streamed splits, ~2 CTAs per SM in total
    const int64_t nfull = R / kBulkChunk;
    int64_t S = std::max<int64_t>(1, (2LL * sms) / O);
    S = std::min<int64_t>(S, nfull);
    const int64_t cps = (nfull + S - 1) / S;
    S = (nfull + cps - 1) / cps;
    unsigned* tk = b2::tickets(st);
    if (!tk) return b2::fail("b2_reduce: no reduction counters for this stream");
    void* ws = nullptr;
    B2_TRY(b2_alloc((size_t)S * O * (OP == B2_RED_MAX ? sizeof(MaxAcc) : sizeof(double)), st, &ws));
    const int smem = kBulkStages * kBulkChunk * 4;
    static bool attr = false;
    if (!attr) {
      B2_CUDA(cudaFuncSetAttribute(k_bulk_rows<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr = true;
    }
    k_bulk_rows<OP><<<dim3((unsigned)O, (unsigned)S), 256, smem, st>>>(x, O, R, cps, out, argr, (double*)ws,
                                                                       (MaxAcc*)ws, count, tk);
    int rc = b2::launched("b2_reduce(bulk rows)");
    b2_free(ws, st);
    return rc;
  }
  // a warp per row up to 16K elements (8 rows per CTA: no block barrier, and
  // enough bytes in flight per CTA); a whole CTA per row beyond that
  const int group = R > 16384 ? 256 : 32;
  const int rpc = 256 / group;
  const int64_t ctas = (O + rpc - 1) / rpc;
  int64_t S = 1;
  if (ctas < 2 * sms && R >= 16384) {  // few long rows: split R to fill one resident wave
    const int64_t cap = (int64_t)sms * resident<OP>(group == 256 ? (const void*)k_rows<OP, 256, true>
                                                                 : (const void*)k_rows<OP, 32, true>);
    S = std::min<int64_t>(std::max<int64_t>(cap / ctas, 1), (R + 8191) / 8192);
    S = std::max<int64_t>(S, 1);
  }
  int64_t Rs = (R + S - 1) / S;
  Rs = (Rs + 3) & ~int64_t(3);
  S = (R + Rs - 1) / Rs;
  if (S < 1) S = 1;
  void* ws = nullptr;
  double* psum = nullptr;
  MaxAcc* pmax = nullptr;
  if (S > 1) {
    size_t bytes = (size_t)S * O * (OP == B2_RED_MAX ? sizeof(MaxAcc) : sizeof(double));
    B2_TRY(b2_alloc(bytes, st, &ws));
    psum = (double*)ws;
    pmax = (MaxAcc*)ws;
  }
  unsigned* tk = nullptr;
  if (S > 1) {
    tk = b2::tickets(st);
    if (!tk) return b2::fail("b2_reduce: no reduction counters for this stream");
    if (ctas > b2::kTickets) return b2::fail("b2_reduce: too many row blocks for a split reduction");
  }
  dim3 grid((unsigned)ctas, (unsigned)S);
#define B2_ROWS(G, V) k_rows<OP, G, V><<<grid, 256, 0, st>>>(x, O, R, Rs, out, argr, psum, pmax, count, tk)
  if (group == 256) {
    if (vec) B2_ROWS(256, true); else B2_ROWS(256, false);
  } else {
    if (vec) B2_ROWS(32, true); else B2_ROWS(32, false);
  }
#undef B2_ROWS
  int rc = b2::launched("b2_reduce(rows)");
  if (ws) b2_free(ws, st);
  return rc;
}

template <int OP>
int run_mid(const float* x, int64_t O1, int64_t R, int64_t I, float* out, int64_t* argr,
            double count, cudaStream_t st) {
  const int sms = b2::sm_count();
  const int V = (I % 4 == 0 && ((uintptr_t)x & 15) == 0) ? 4 : 1;
  if (V == 4) {
    // cluster path: 32-column strips x CS row splits folded through DSMEM.
    // Target ~4 resident 256-thread CTAs per SM (the probe's best); CS is a
    // power of two <= 16 and leaves every row lane >= 8 rows.
    const int64_t cstrips = (I + 31) / 32, base_ctas = cstrips * O1;
    const int64_t target = 3LL * sms;  // 4 x 148 strips-splits -> cs 4 for a 4096-wide input (probe best)
    int cs = 1;
    while (cs < 16 && base_ctas * cs < target && R >= (int64_t)(cs * 2) * 32 * 8) cs *= 2;
    if (cs == 16) {  // a non-portable cluster size (narrow, tall inputs: e.g. 1024 bias columns)
      static bool np_ok =
          cudaFuncSetAttribute(k_cols<OP>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
          (OP != B2_RED_MAX ||
           cudaFuncSetAttribute(k_cols<kMaxValue>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess);
      if (!np_ok) {
        cudaGetLastError();
        cs = 8;
      }
    }
    while (base_ctas * cs >= 2LL * sms && base_ctas <= INT32_MAX) {
      const int64_t Rs = (R + cs - 1) / cs;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)base_ctas, (unsigned)cs, 1);
      cfg.blockDim = dim3(256, 1, 1);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 1;
      attr[0].val.clusterDim.y = cs;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaError_t e = (OP == B2_RED_MAX && !argr)
                          ? cudaLaunchKernelEx(&cfg, k_cols<kMaxValue>, x, R, I, Rs, out, argr, count, cstrips)
                          : cudaLaunchKernelEx(&cfg, k_cols<OP>, x, R, I, Rs, out, argr, count, cstrips);
      if (e != cudaSuccess && cs > 8) {
        // 16-CTA clusters could not be placed (MIG/MPS partitions, busy GPCs):
        // retry with the portable cluster size
        cudaGetLastError();
        cs = 8;
        continue;
      }
      if (e != cudaSuccess) return b2::cuda_fail(e, "b2_reduce(cols)");
      return b2::launched("b2_reduce(cols)");
    }
  }
  // Column lanes and split policy (measured on 4096x4096, scripts/red_bench.py):
  // sums use 8 column lanes x 4 columns (128 B per row segment) and split rows
  // to fill one wave; max uses 4 x 4 (64 B segments, 4x more strips) and does
  // not split once the strips alone cover the SMs -- its 16-B (value, index)
  // partials and second stage cost more than the narrower segments.
  const int CL = V == 4 ? (OP == B2_RED_MAX ? 4 : 8) : 32, RL = 256 / CL;
  const bool single = OP == B2_RED_MAX;
  const void* kern = V == 4 ? (CL == 4 ? (const void*)k_strip<OP, 4, 4> : (const void*)k_strip<OP, 4, 8>)
                            : (const void*)k_strip<OP, 1, 32>;
  const int64_t strips = (I + CL * V - 1) / (CL * V);
  const int64_t ctas = strips * O1;
  int64_t S = 1;
  // splits: as many as ONE resident wave holds (a partial second wave would
  // double the tail), but at least 8 row-lane passes per CTA
  const int64_t cap = (int64_t)sms * resident<OP>(kern);
  if (ctas < cap && !(single && ctas >= sms)) {
    S = std::min<int64_t>(cap / ctas, R / (RL * 8));
    S = std::max<int64_t>(S, 1);
  }
  int64_t Rs = (R + S - 1) / S;
  S = (R + Rs - 1) / Rs;
  if (S < 1) S = 1;
  const int64_t O = O1 * I;
  void* ws = nullptr;
  double* psum = nullptr;
  MaxAcc* pmax = nullptr;
  if (S > 1) {
    size_t bytes = (size_t)S * O * (OP == B2_RED_MAX ? sizeof(MaxAcc) : sizeof(double));
    B2_TRY(b2_alloc(bytes, st, &ws));
    psum = (double*)ws;
    pmax = (MaxAcc*)ws;
  }
  dim3 grid((unsigned)(strips * O1), (unsigned)S);
  if (V == 4 && CL == 4)
    k_strip<OP, 4, 4><<<grid, 256, 0, st>>>(x, O1, R, I, Rs, out, argr, psum, pmax, count, strips);
  else if (V == 4)
    k_strip<OP, 4, 8><<<grid, 256, 0, st>>>(x, O1, R, I, Rs, out, argr, psum, pmax, count, strips);
  else
    k_strip<OP, 1, 32><<<grid, 256, 0, st>>>(x, O1, R, I, Rs, out, argr, psum, pmax, count, strips);
  int rc = b2::launched("b2_reduce(mid)");
  if (!rc && S > 1) {
    launch_final<OP>(O, S, psum, pmax, out, argr, count, st);
    rc = b2::launched("b2_reduce(final)");
  }
  if (ws) b2_free(ws, st);
  return rc;
}

template <int OP>
int dispatch(int canon, const float* x, int64_t O1, int64_t R, int64_t I, float* out, int64_t* argr,
             double count, cudaStream_t st) {
  if (canon == 0) return run_rows<OP>(x, O1, R, out, argr, count, st);
  return run_mid<OP>(x, O1, R, I, out, argr, count, st);
}

}  // namespace

extern "C" int b2_copy_strided(float*, int, const int64_t*, const float*, const int64_t*, void*);

extern "C" int b2_reduce(int op, float* out, int64_t* argr, int ndim, const int64_t* shape,
                         const float* x, const int64_t* xs, uint32_t mask, void* stream) {
  if (ndim < 0 || ndim > B2_MAX_DIMS) return b2::fail("b2_reduce: rank exceeds 8");
  if (op < 0 || op > 2) return b2::fail("b2_reduce: unknown op");
  cudaStream_t st = b2::resolve(stream);
  int64_t nkept = 1, nred = 1;
  for (int d = 0; d < ndim; ++d) {
    if (mask >> d & 1)
      nred *= shape[d];
    else
      nkept *= shape[d];
  }
  if (nkept == 0) return 0;
  if (op == B2_RED_MAX && nred >= INT32_MAX)
    return b2::fail("b2_reduce: max over more than 2^31-1 elements per output");
  if (nred == 0) {
    if (op == B2_RED_MAX) return b2::fail("max over a zero-extent axis is undefined");
    float v = op == B2_RED_MEAN ? NAN : 0.0f;
    k_fill_out<<<(unsigned)((nkept + 255) / 256), 256, 0, st>>>(out, argr, nkept, v);
    return b2::launched("b2_reduce(empty)");
  }
  double count = (double)nred;
  // drop size-1 axes; check contiguity and whether the reduced axes are one block
  int64_t cshape[B2_MAX_DIMS], cst[B2_MAX_DIMS];
  bool cred[B2_MAX_DIMS];
  int n = 0;
  for (int d = 0; d < ndim; ++d) {
    if (shape[d] == 1) continue;
    cshape[n] = shape[d];
    cst[n] = xs[d];
    cred[n] = mask >> d & 1;
    ++n;
  }
  bool contig = true;
  int64_t acc = 1;
  for (int d = n - 1; d >= 0; --d) {
    if (cst[d] != acc) contig = false;
    acc *= cshape[d];
  }
  int lo = -1, hi = -1;
  bool block = true;
  for (int d = 0; d < n; ++d) {
    if (cred[d]) {
      if (lo < 0) lo = d;
      else if (hi != d) block = false;
      hi = d + 1;
    }
  }
  if (lo < 0) {  // nothing (non-trivial) reduced: a copy
    int rc = b2_copy_strided(out, ndim, shape, x, xs, stream);
    if (!rc && argr) {
      B2_CUDA(cudaMemsetAsync(argr, 0, nkept * sizeof(int64_t), st));
    }
    return rc;
  }
  const float* src = x;
  void* tmp = nullptr;
  int64_t O1, R, I;
  int canon;
  if (contig && block) {
    O1 = 1;
    R = 1;
    I = 1;
    for (int d = 0; d < lo; ++d) O1 *= cshape[d];
    for (int d = lo; d < hi; ++d) R *= cshape[d];
    for (int d = hi; d < n; ++d) I *= cshape[d];
    canon = I == 1 ? 0 : 1;
  } else {
    // gather into [kept..., reduced...] order (reduced dims in increasing axis order)
    int64_t pshape[B2_MAX_DIMS], pst[B2_MAX_DIMS];
    int k = 0;
    for (int d = 0; d < n; ++d)
      if (!cred[d]) { pshape[k] = cshape[d]; pst[k] = cst[d]; ++k; }
    for (int d = 0; d < n; ++d)
      if (cred[d]) { pshape[k] = cshape[d]; pst[k] = cst[d]; ++k; }
    B2_TRY(b2_alloc((size_t)(nkept * nred) * sizeof(float), st, &tmp));
    int rc = b2_copy_strided((float*)tmp, n, pshape, x, pst, st);
    if (rc) {
      b2_free(tmp, st);
      return rc;
    }
    src = (const float*)tmp;
    O1 = nkept;
    R = nred;
    I = 1;
    canon = 0;
  }
  int rc;
  switch (op) {
    case B2_RED_SUM: rc = dispatch<B2_RED_SUM>(canon, src, O1, R, I, out, argr, count, st); break;
    case B2_RED_MEAN: rc = dispatch<B2_RED_MEAN>(canon, src, O1, R, I, out, argr, count, st); break;
    default: rc = dispatch<B2_RED_MAX>(canon, src, O1, R, I, out, argr, count, st); break;
  }
  if (tmp) b2_free(tmp, st);
  return rc;
}

extern "C" int b2_max_scatter(float* gx, int ndim, const int64_t* shape, uint32_t mask,
                              const float* g, const int64_t* argr, void* stream) {
  if (ndim < 0 || ndim > B2_MAX_DIMS) return b2::fail("b2_max_scatter: rank exceeds 8");
  cudaStream_t st = b2::resolve(stream);
  int64_t total = 1, O = 1;
  for (int d = 0; d < ndim; ++d) {
    total *= shape[d];
    if (!(mask >> d & 1)) O *= shape[d];
  }
  if (total == 0) return 0;
  B2_CUDA(cudaMemsetAsync(gx, 0, total * sizeof(float), st));
  if (O == 0) return 0;
  ScatterGeom sg;
  sg.nk = sg.nr = 0;
  int64_t stride[B2_MAX_DIMS], acc = 1;
  for (int d = ndim - 1; d >= 0; --d) {
    stride[d] = acc;
    acc *= shape[d];
  }
  for (int d = 0; d < ndim; ++d) {
    if (mask >> d & 1) {
      sg.rshape[sg.nr] = shape[d];
      sg.rstride[sg.nr++] = stride[d];
    } else {
      sg.kshape[sg.nk] = shape[d];
      sg.kstride[sg.nk++] = stride[d];
    }
  }
  k_max_scatter<<<(unsigned)((O + 255) / 256), 256, 0, st>>>(gx, g, argr, O, sg);
  return b2::launched("b2_max_scatter");
}
