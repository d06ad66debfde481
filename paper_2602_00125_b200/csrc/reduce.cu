// Reduction engine: sum / mean / max over any axis set.
//
// Replaces tensorlite/core.py:581-728 (_sum_all, _axis_scan, sum, mean, max).
// * sums accumulate in fp64 and round to f32 once (the reference accumulates
//   Python doubles); mean = f32(dsum / count) in double (core.py:671, 682);
// * max keeps (value, first index): strict '>' scan semantics, ties go to the
//   lower row-major index, a NaN in the first scanned slot sticks and later
//   NaNs are skipped (core.py:709-713) -- the combine below is associative so
//   the parallel order cannot change the winner;
// * deterministic: work is partitioned by a fixed function of the shape and
//   the SM count, partials combine in a fixed order (the reference's
//   worker-count-independent chunk contract, parallel.py:1-8, 48-63).
//
// Canonical forms (after dropping size-1 axes):
//   contiguous x with the reduced axes one contiguous block  -> [O1, R, I]
//   (I == 1 is a row reduction); anything else is first gathered into a
//   [kept..., reduced...] contiguous temp and reduced as rows.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "common.cuh"

extern "C" int b2_alloc(size_t, void*, void**);
extern "C" int b2_free(void*, void*);

namespace {

constexpr int64_t kNone = INT64_MAX;

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

__device__ __forceinline__ void max_push(MaxAcc& a, float v, int64_t i) {
  if (isnan(v)) {
    if (i == 0) a = MaxAcc{v, 0};
    return;
  }
  if (sticky(a)) return;
  if (a.i == kNone || v > a.v || (v == a.v && i < a.i)) a = MaxAcc{v, i};
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

// ---------------------------------------------------------------- row reduce
// x: [O, R] contiguous rows. grid = (ceil(O / rows_per_cta), S); each group of
// GROUP threads owns one row and the split range [s*Rs, min(R,(s+1)*Rs)).
// S == 1 -> final outputs; S > 1 -> partials [S][O].
template <int OP, int GROUP, bool VEC>
__global__ void __launch_bounds__(256) k_rows(const float* __restrict__ x, int64_t O, int64_t R,
                                              int64_t Rs, float* __restrict__ out,
                                              int64_t* __restrict__ argr, double* __restrict__ psum,
                                              MaxAcc* __restrict__ pmax, double count) {
  __shared__ double shd[8];
  __shared__ MaxAcc shm[8];
  constexpr int RPC = 256 / GROUP;
  int g = threadIdx.x / GROUP, t = threadIdx.x % GROUP;
  int64_t o = blockIdx.x * (int64_t)RPC + g;
  int S = gridDim.y, s = blockIdx.y;
  int64_t r0 = s * Rs, r1 = min(R, r0 + Rs);
  bool live = o < O;
  const float* row = x + (live ? o : 0) * R;
  if (OP != B2_RED_MAX) {
    double acc = 0;
    if (live) {
      if (VEC) {
        for (int64_t r = r0 + 4 * t; r < r1; r += 4 * GROUP) {
          if (r + 3 < r1) {
            float4 v = *reinterpret_cast<const float4*>(row + r);
            acc += (double)v.x;
            acc += (double)v.y;
            acc += (double)v.z;
            acc += (double)v.w;
          } else {
            for (int64_t k = r; k < r1; ++k) acc += (double)row[k];
          }
        }
      } else {
        for (int64_t r = r0 + t; r < r1; r += GROUP) acc += (double)row[r];
      }
    }
    double tot = group_sum<GROUP>(acc, shd);
    if (live && t == 0) {
      if (S > 1) {
        psum[(int64_t)s * O + o] = tot;
      } else {
        out[o] = OP == B2_RED_MEAN ? __double2float_rn(tot / count) : __double2float_rn(tot);
      }
    }
  } else {
    MaxAcc acc{0.f, kNone};
    if (live) {
      if (VEC) {
        for (int64_t r = r0 + 4 * t; r < r1; r += 4 * GROUP) {
          if (r + 3 < r1) {
            float4 v = *reinterpret_cast<const float4*>(row + r);
            max_push(acc, v.x, r);
            max_push(acc, v.y, r + 1);
            max_push(acc, v.z, r + 2);
            max_push(acc, v.w, r + 3);
          } else {
            for (int64_t k = r; k < r1; ++k) max_push(acc, row[k], k);
          }
        }
      } else {
        for (int64_t r = r0 + t; r < r1; r += GROUP) max_push(acc, row[r], r);
      }
    }
    MaxAcc best = group_max<GROUP>(acc, shm);
    if (live && t == 0) {
      if (S > 1) {
        pmax[(int64_t)s * O + o] = best;
      } else {
        out[o] = best.v;
        if (argr) argr[o] = best.i;
      }
    }
  }
}

// ---------------------------------------------------------------- mid reduce
// x: [O1, R, I] contiguous; output o = o1*I + i. grid = (cb * O1, S), cb = ceil(I/256)
template <int OP>
__global__ void __launch_bounds__(256) k_mid(const float* __restrict__ x, int64_t O1, int64_t R,
                                             int64_t I, int64_t Rs, float* __restrict__ out,
                                             int64_t* __restrict__ argr, double* __restrict__ psum,
                                             MaxAcc* __restrict__ pmax, double count, int64_t cb) {
  int64_t o1 = blockIdx.x / cb;
  int64_t i = (blockIdx.x - o1 * cb) * (int64_t)blockDim.x + threadIdx.x;
  int S = gridDim.y, s = blockIdx.y;
  if (i >= I) return;
  int64_t r0 = s * Rs, r1 = min(R, r0 + Rs);
  const float* base = x + o1 * R * I + i;
  int64_t o = o1 * I + i;
  int64_t O = O1 * I;
  if (OP != B2_RED_MAX) {
    double acc = 0;
    int64_t r = r0;
    for (; r + 3 < r1; r += 4) {  // 4 independent loads in flight
      float a0 = base[r * I], a1 = base[(r + 1) * I], a2 = base[(r + 2) * I], a3 = base[(r + 3) * I];
      acc += (double)a0;
      acc += (double)a1;
      acc += (double)a2;
      acc += (double)a3;
    }
    for (; r < r1; ++r) acc += (double)base[r * I];
    if (S > 1)
      psum[(int64_t)s * O + o] = acc;
    else
      out[o] = OP == B2_RED_MEAN ? __double2float_rn(acc / count) : __double2float_rn(acc);
  } else {
    MaxAcc acc{0.f, kNone};
    for (int64_t r = r0; r < r1; ++r) max_push(acc, base[r * I], r);
    if (S > 1) {
      pmax[(int64_t)s * O + o] = acc;
    } else {
      out[o] = acc.v;
      if (argr) argr[o] = acc.i;
    }
  }
}

template <int OP>
__global__ void k_final(int64_t O, int S, const double* __restrict__ psum,
                        const MaxAcc* __restrict__ pmax, float* __restrict__ out,
                        int64_t* __restrict__ argr, double count) {
  int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= O) return;
  if (OP != B2_RED_MAX) {
    double acc = 0;
    for (int s = 0; s < S; ++s) acc += psum[(int64_t)s * O + o];
    out[o] = OP == B2_RED_MEAN ? __double2float_rn(acc / count) : __double2float_rn(acc);
  } else {
    MaxAcc a{0.f, kNone};
    for (int s = 0; s < S; ++s) a = max_combine(a, pmax[(int64_t)s * O + o]);
    out[o] = a.v;
    if (argr) argr[o] = a.i;
  }
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

template <int OP>
int run_rows(const float* x, int64_t O, int64_t R, float* out, int64_t* argr, double count,
             cudaStream_t st) {
  bool vec = ((uintptr_t)x & 15) == 0 && R % 4 == 0;
  int sms = b2::sm_count();
  int group = R >= 2048 ? 256 : 32;
  int rpc = 256 / group;
  int64_t ctas = (O + rpc - 1) / rpc;
  int64_t S = 1;
  if (ctas < 2 * sms && R >= 8192) {  // few long rows: split R across CTAs
    S = std::min<int64_t>((4 * sms + ctas - 1) / ctas, (R + 4095) / 4096);
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
  dim3 grid((unsigned)ctas, (unsigned)S);
#define B2_ROWS(G, V) k_rows<OP, G, V><<<grid, 256, 0, st>>>(x, O, R, Rs, out, argr, psum, pmax, count)
  if (group == 256) {
    if (vec) B2_ROWS(256, true); else B2_ROWS(256, false);
  } else {
    if (vec) B2_ROWS(32, true); else B2_ROWS(32, false);
  }
#undef B2_ROWS
  int rc = b2::launched("b2_reduce(rows)");
  if (!rc && S > 1) {
    k_final<OP><<<(unsigned)((O + 255) / 256), 256, 0, st>>>(O, (int)S, psum, pmax, out, argr, count);
    rc = b2::launched("b2_reduce(final)");
  }
  if (ws) b2_free(ws, st);
  return rc;
}

template <int OP>
int run_mid(const float* x, int64_t O1, int64_t R, int64_t I, float* out, int64_t* argr,
            double count, cudaStream_t st) {
  int sms = b2::sm_count();
  int64_t cb = (I + 255) / 256;
  int64_t ctas = cb * O1;
  int64_t S = 1;
  if (ctas < 4 * sms && R >= 64) {
    S = std::min<int64_t>((4 * sms + ctas - 1) / ctas, R / 16);
    S = std::max<int64_t>(S, 1);
  }
  int64_t Rs = (R + S - 1) / S;
  S = (R + Rs - 1) / Rs;
  if (S < 1) S = 1;
  int64_t O = O1 * I;
  void* ws = nullptr;
  double* psum = nullptr;
  MaxAcc* pmax = nullptr;
  if (S > 1) {
    size_t bytes = (size_t)S * O * (OP == B2_RED_MAX ? sizeof(MaxAcc) : sizeof(double));
    B2_TRY(b2_alloc(bytes, st, &ws));
    psum = (double*)ws;
    pmax = (MaxAcc*)ws;
  }
  dim3 grid((unsigned)(cb * O1), (unsigned)S);
  k_mid<OP><<<grid, 256, 0, st>>>(x, O1, R, I, Rs, out, argr, psum, pmax, count, cb);
  int rc = b2::launched("b2_reduce(mid)");
  if (!rc && S > 1) {
    k_final<OP><<<(unsigned)((O + 255) / 256), 256, 0, st>>>(O, (int)S, psum, pmax, out, argr, count);
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
