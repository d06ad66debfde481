// HBM probe for the 64 MiB config-2 reductions: what a 4096x4096 fp32 read
// can reach when timed the way bench.py times the ops (24 calls captured in a
// CUDA graph, rotating over 6 input copies so every call streams from HBM).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/hbm_probe scripts/hbm_probe.cu
//
// Variants (full sum, fp64 accumulation):
//   two   : partial per CTA, then a 1-CTA second kernel
//   tick  : one kernel; the last CTA to finish (release/acquire ticket) folds
//           the partials in CTA order -- deterministic
//   readf : fp32 accumulate, no second stage (upper bound of the read loop)
//   copy  : read + write 64 MiB each (the elementwise shape)
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int T = 256;

template <int U>
__device__ __forceinline__ double chunk_sum(const float4* __restrict__ x, int64_t n4, int64_t b0, int64_t b1) {
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  int64_t i = b0 + threadIdx.x;
  for (; i + (U - 1) * T < b1; i += U * T) {
    float4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = __ldg(x + i + k * T);
#pragma unroll
    for (int k = 0; k < U; k += 4) {
      a0 += ((double)v[k].x + (double)v[k].y) + ((double)v[k].z + (double)v[k].w);
      if (k + 1 < U) a1 += ((double)v[k + 1].x + (double)v[k + 1].y) + ((double)v[k + 1].z + (double)v[k + 1].w);
      if (k + 2 < U) a2 += ((double)v[k + 2].x + (double)v[k + 2].y) + ((double)v[k + 2].z + (double)v[k + 2].w);
      if (k + 3 < U) a3 += ((double)v[k + 3].x + (double)v[k + 3].y) + ((double)v[k + 3].z + (double)v[k + 3].w);
    }
  }
  for (; i < b1; i += T) {
    float4 v = __ldg(x + i);
    a0 += ((double)v.x + (double)v.y) + ((double)v.z + (double)v.w);
  }
  return (a0 + a1) + (a2 + a3);
}

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[T / 32];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < T / 32 ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(~0u, t, o);
  }
  return t;
}

template <int U>
__global__ void __launch_bounds__(T) k_part(const float4* x, int64_t n4, double* part) {
  const int64_t per = (n4 + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = min(n4, b0 + per);
  double s = block_sum(chunk_sum<U>(x, n4, b0, b1));
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_fin(const double* part, int G, float* out) {
  double s = 0;
  for (int i = threadIdx.x; i < G; i += T) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) *out = (float)s;
}

template <int U>
__global__ void __launch_bounds__(T) k_tick(const float4* x, int64_t n4, double* part, unsigned* ticket, float* out) {
  const int64_t per = (n4 + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = min(n4, b0 + per);
  double s = block_sum(chunk_sum<U>(x, n4, b0, b1));
  __shared__ unsigned last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    unsigned t;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(ticket) : "memory");
    last = t == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    double a = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += T) {
      a += __ldcg(part + i);
    }
    a = block_sum(a);
    if (threadIdx.x == 0) {
      *out = (float)a;
      *ticket = 0;  // re-arm for the next launch (stream-ordered)
    }
  }
}

template <int U>
__global__ void __launch_bounds__(T) k_readf(const float4* x, int64_t n4, float* out) {
  const int64_t per = (n4 + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = min(n4, b0 + per);
  float a = 0;
  int64_t i = b0 + threadIdx.x;
  for (; i + (U - 1) * T < b1; i += U * T) {
    float4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = __ldg(x + i + k * T);
#pragma unroll
    for (int k = 0; k < U; ++k) a += v[k].x + v[k].y + v[k].z + v[k].w;
  }
  for (; i < b1; i += T) { float4 v = __ldg(x + i); a += v.x + v.y + v.z + v.w; }
  if (a == 12345.f) *out = a;
}

__global__ void __launch_bounds__(T) k_copy(const float4* x, float4* y, int64_t n4) {
  int64_t i = blockIdx.x * (int64_t)T + threadIdx.x, st = (int64_t)gridDim.x * T;
  for (; i + 3 * st < n4; i += 4 * st) {
    float4 a = __ldg(x + i), b = __ldg(x + i + st), c = __ldg(x + i + 2 * st), d = __ldg(x + i + 3 * st);
    y[i] = a; y[i + st] = b; y[i + 2 * st] = c; y[i + 3 * st] = d;
  }
  for (; i < n4; i += st) y[i] = __ldg(x + i);
}


// ---- TMA bulk streaming: each CTA copies its contiguous range through a
// STAGES-deep ring of CH-byte shared-memory chunks (cp.async.bulk + mbarrier);
// the threads only read shared memory, so the bytes in flight do not depend
// on registers.
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(b)) : "memory");
}

template <int STAGES, int CH>
__global__ void __launch_bounds__(T) k_bulk(const float4* x, int64_t n4, double* part, unsigned* ticket, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * CH);
  constexpr int V = CH / 16;  // float4 per chunk
  const int64_t nch = n4 / V;  // whole chunks (n4 % V == 0 here)
  const int64_t per = (nch + gridDim.x - 1) / gridDim.x;
  const int64_t c0 = blockIdx.x * per, c1 = min(nch, c0 + per);
  const int64_t nc = c1 > c0 ? c1 - c0 : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) bar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < STAGES && s < nc; ++s) bulk_load(smem + s * CH, x + (c0 + s) * V, CH, &bars[s]);
  }
  __syncthreads();
  double a0 = 0, a1 = 0;
  for (int64_t c = 0; c < nc; ++c) {
    const int s = c % STAGES;
    bar_wait(&bars[s], (c / STAGES) & 1);
    const float4* q = reinterpret_cast<const float4*>(smem + s * CH);
#pragma unroll
    for (int k = 0; k < V / T; k += 2) {
      float4 v = q[threadIdx.x + k * T];
      float4 w = q[threadIdx.x + (k + 1) * T];
      a0 += ((double)v.x + (double)v.y) + ((double)v.z + (double)v.w);
      a1 += ((double)w.x + (double)w.y) + ((double)w.z + (double)w.w);
    }
    __syncthreads();
    if (threadIdx.x == 0 && c + STAGES < nc) bulk_load(smem + s * CH, x + (c0 + c + STAGES) * V, CH, &bars[s]);
  }
  double s = block_sum(a0 + a1);
  __shared__ unsigned last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    unsigned t;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(ticket) : "memory");
    last = t == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    double a = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += T) {
      a += __ldcg(part + i);
    }
    a = block_sum(a);
    if (threadIdx.x == 0) { *out = (float)a; *ticket = 0; }
  }
}

// ---- column sums of [R, C]: plain loads, CTA = (row split, 1024-column block),
// thread owns 4 columns; partials [S][C] then a ticket per column block
template <int U>
__global__ void __launch_bounds__(T) k_col(const float* x, int64_t R, int64_t C, int64_t Rs, double* part,
                                           unsigned* tickets, float* out) {
  const int cb = blockIdx.x, s = blockIdx.y, S = gridDim.y;
  const int64_t col = cb * 1024 + threadIdx.x * 4;
  const int64_t r0 = s * Rs, r1 = min(R, r0 + Rs);
  double a[4] = {0, 0, 0, 0};
  int64_t r = r0;
  for (; r + U <= r1; r += U) {
    float4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = __ldg(reinterpret_cast<const float4*>(x + (r + k) * C + col));
#pragma unroll
    for (int k = 0; k < U; ++k) { a[0] += v[k].x; a[1] += v[k].y; a[2] += v[k].z; a[3] += v[k].w; }
  }
  for (; r < r1; ++r) {
    float4 v = __ldg(reinterpret_cast<const float4*>(x + r * C + col));
    a[0] += v.x; a[1] += v.y; a[2] += v.z; a[3] += v.w;
  }
  double* p = part + (int64_t)s * C + col;
  p[0] = a[0]; p[1] = a[1]; p[2] = a[2]; p[3] = a[3];
  __shared__ unsigned last;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(tickets + cb) : "memory");
    last = t == (unsigned)S - 1;
  }
  __syncthreads();
  if (last) {
    double b[4] = {0, 0, 0, 0};
#pragma unroll 8
    for (int q = 0; q < S; ++q) {
      const double* pp = part + (int64_t)q * C + col;
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] += __ldcg(pp + j);
    }
    for (int j = 0; j < 4; ++j) out[col + j] = (float)b[j];
    if (threadIdx.x == 0) tickets[cb] = 0;
  }
}

// ---- column sums with TMA bulk row segments: CTA = (1024-column block, row
// split); a stage holds RPS rows x 4 KB; thread t owns columns 4t..4t+3
template <int STAGES, int RPS>
__global__ void __launch_bounds__(T) k_bcol(const float* x, int64_t R, int64_t C, int64_t Rs, double* part,
                                            unsigned* tickets, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int SB = RPS * 4096;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * SB);
  const int cb = blockIdx.x, s = blockIdx.y, S = gridDim.y;
  const int64_t c0 = cb * 1024;
  const int64_t r0 = s * Rs, r1 = min(R, r0 + Rs);
  const int64_t nst = (r1 - r0 + RPS - 1) / RPS;
  auto issue = [&](int64_t st) {
    const int b = st % STAGES;
    const int64_t ra = r0 + st * RPS;
    const int nr = (int)min((int64_t)RPS, r1 - ra);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[b])), "r"(nr * 4096) : "memory");
    for (int k = 0; k < nr; ++k)
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];"
                   ::"r"(su32(smem + b * SB + k * 4096)), "l"(x + (ra + k) * C + c0), "r"(su32(&bars[b])) : "memory");
  };
  if (threadIdx.x == 0) {
    for (int b = 0; b < STAGES; ++b) bar_init(&bars[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int b = 0; b < STAGES && b < nst; ++b) issue(b);
  }
  __syncthreads();
  double a[4] = {0, 0, 0, 0};
  for (int64_t st = 0; st < nst; ++st) {
    const int b = st % STAGES;
    bar_wait(&bars[b], (st / STAGES) & 1);
    const int nr = (int)min((int64_t)RPS, r1 - (r0 + st * RPS));
    const float4* q = reinterpret_cast<const float4*>(smem + b * SB) + threadIdx.x;
    if (nr == RPS) {
#pragma unroll
      for (int k = 0; k < RPS; ++k) { float4 v = q[k * 256]; a[0] += v.x; a[1] += v.y; a[2] += v.z; a[3] += v.w; }
    } else {
      for (int k = 0; k < nr; ++k) { float4 v = q[k * 256]; a[0] += v.x; a[1] += v.y; a[2] += v.z; a[3] += v.w; }
    }
    __syncthreads();
    if (threadIdx.x == 0 && st + STAGES < nst) issue(st + STAGES);
  }
  const int64_t col = c0 + threadIdx.x * 4;
  double* p = part + (int64_t)s * C + col;
  p[0] = a[0]; p[1] = a[1]; p[2] = a[2]; p[3] = a[3];
  __shared__ unsigned last;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(tickets + cb) : "memory");
    last = t == (unsigned)S - 1;
  }
  __syncthreads();
  if (last) {
    double b2[4] = {0, 0, 0, 0};
#pragma unroll 8
    for (int q = 0; q < S; ++q) {
      const double* pp = part + (int64_t)q * C + col;
#pragma unroll
      for (int j = 0; j < 4; ++j) b2[j] += __ldcg(pp + j);
    }
    for (int j = 0; j < 4; ++j) out[col + j] = (float)b2[j];
    if (threadIdx.x == 0) tickets[cb] = 0;
  }
}

// ---- dim-0 streaming efficiency vs segment width: CTA = (W-column block,
// H-row split); 256 threads = (256/(W/4)) row lanes x (W/4) column lanes when
// W <= 1024 floats; thread owns 4 columns; U rows in flight; partial written,
// no fold (measures the read pattern only)
template <int W, int U>
__global__ void __launch_bounds__(T) k_colw(const float* x, int64_t R, int64_t C, int64_t Rs, double* part) {
  constexpr int CL = W / 4 < 256 ? W / 4 : 256, RL = 256 / CL;
  const int cl = threadIdx.x % CL, rl = threadIdx.x / CL;
  const int cb = blockIdx.x, s = blockIdx.y;
  const int64_t col = (int64_t)cb * W + cl * 4;
  const int64_t r0 = s * Rs, r1 = min(R, r0 + Rs);
  double a[4] = {0, 0, 0, 0};
  int64_t r = r0 + rl;
  for (; r + (U - 1) * RL < r1; r += U * RL) {
    float4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = __ldg(reinterpret_cast<const float4*>(x + (r + k * RL) * C + col));
#pragma unroll
    for (int k = 0; k < U; ++k) { a[0] += v[k].x; a[1] += v[k].y; a[2] += v[k].z; a[3] += v[k].w; }
  }
  for (; r < r1; r += RL) {
    float4 v = __ldg(reinterpret_cast<const float4*>(x + r * C + col));
    a[0] += v.x; a[1] += v.y; a[2] += v.z; a[3] += v.w;
  }
  if (a[0] + a[1] + a[2] + a[3] == 1234.5) part[0] = a[0];
}

int main() {
  const int64_t n = 4096LL * 4096, n4 = n / 4;
  const int NC = 6, IT = 24;
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<float4*> bufs(NC);
  for (auto& b : bufs) { CK(cudaMalloc(&b, n * 4)); CK(cudaMemset(b, 0, n * 4)); }
  float4* ybuf; CK(cudaMalloc(&ybuf, n * 4 * NC));
  double* part; CK(cudaMalloc(&part, 1 << 20));
  unsigned* ticket; CK(cudaMalloc(&ticket, 4)); CK(cudaMemset(ticket, 0, 4));
  float* out; CK(cudaMalloc(&out, 64));
  cudaStream_t st; CK(cudaStreamCreate(&st));
  auto time = [&](const char* name, double bytes, auto body) {
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
    for (int it = 0; it < IT; ++it) body(it % NC, st);
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, st)); CK(cudaStreamSynchronize(st));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0, st)); CK(cudaGraphLaunch(ge, st)); CK(cudaEventRecord(e1, st));
      CK(cudaStreamSynchronize(st));
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    double us = best * 1000 / IT;
    printf("%-34s %8.2f us/call %8.0f GB/s\n", name, us, bytes / us / 1e3);
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
  };
  const double rb = n * 4.0;
  for (int mult : {1, 2, 4}) {
    int G = sms * mult;
    char nm[64];
    snprintf(nm, 64, "two   U=8 G=%d", G);
    time(nm, rb, [&](int c, cudaStream_t s) { k_part<8><<<G, T, 0, s>>>(bufs[c], n4, part); k_fin<<<1, T, 0, s>>>(part, G, out); });
    snprintf(nm, 64, "part only U=8 G=%d", G);
    time(nm, rb, [&](int c, cudaStream_t s) { k_part<8><<<G, T, 0, s>>>(bufs[c], n4, part); });
    snprintf(nm, 64, "tick  U=8 G=%d", G);
    time(nm, rb, [&](int c, cudaStream_t s) { k_tick<8><<<G, T, 0, s>>>(bufs[c], n4, part, ticket, out); });
    snprintf(nm, 64, "tick  U=4 G=%d", G);
    time(nm, rb, [&](int c, cudaStream_t s) { k_tick<4><<<G, T, 0, s>>>(bufs[c], n4, part, ticket, out); });
    snprintf(nm, 64, "tick  U=16 G=%d", G);
    time(nm, rb, [&](int c, cudaStream_t s) { k_tick<16><<<G, T, 0, s>>>(bufs[c], n4, part, ticket, out); });
    snprintf(nm, 64, "readf U=8 G=%d", G);
    time(nm, rb, [&](int c, cudaStream_t s) { k_readf<8><<<G, T, 0, s>>>(bufs[c], n4, out); });
    snprintf(nm, 64, "copy  G=%d", G);
    time(nm, 2 * rb, [&](int c, cudaStream_t s) { k_copy<<<G, T, 0, s>>>(bufs[c], ybuf + c * n4, n4); });
  }
  for (int mult : {8, 16}) {
    int G = sms * mult;
    char nm[64];
    snprintf(nm, 64, "tick  U=8 G=%d", G);
    time(nm, rb, [&](int c, cudaStream_t s) { k_tick<8><<<G, T, 0, s>>>(bufs[c], n4, part, ticket, out); });
    snprintf(nm, 64, "copy  G=%d", G);
    time(nm, 2 * rb, [&](int c, cudaStream_t s) { k_copy<<<G, T, 0, s>>>(bufs[c], ybuf + c * n4, n4); });
  }


  {
    double* cpart2; CK(cudaMalloc(&cpart2, 1 << 20));
    auto runw = [&](auto kern, int W, int ctas_target, const char* tag) {
      int cbs = 4096 / W;
      int S = ctas_target / cbs; if (S < 1) S = 1;
      int64_t Rs = (4096 + S - 1) / S;
      dim3 grid(cbs, S);
      char nm[64];
      snprintf(nm, 64, "colw %s W=%d CTAs=%d H=%lld", tag, W * 4, cbs * S, (long long)Rs);
      time(nm, rb, [&](int c, cudaStream_t s) { kern<<<grid, T, 0, s>>>((const float*)bufs[c], 4096, 4096, Rs, cpart2); });
    };
    for (int ct : {296, 592, 1184}) {
      runw(k_colw<32, 8>, 32, ct, "U8");
      runw(k_colw<128, 8>, 128, ct, "U8");
      runw(k_colw<512, 8>, 512, ct, "U8");
      runw(k_colw<1024, 8>, 1024, ct, "U8");
    }
  }
  {
    auto run_bulk = [&](auto kern, int stages, int ch, int per_sm, const char* tag) {
      int smem = stages * ch + 64;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      int G = sms * per_sm;
      char nm[64];
      snprintf(nm, 64, "bulk %s G=%d", tag, G);
      time(nm, rb, [&](int c, cudaStream_t s) { kern<<<G, T, smem, s>>>(bufs[c], n4, part, ticket, out); });
    };
    run_bulk(k_bulk<4, 16384>, 4, 16384, 2, "4x16K");
    run_bulk(k_bulk<4, 16384>, 4, 16384, 3, "4x16K");
    run_bulk(k_bulk<6, 8192>, 6, 8192, 4, "6x8K");
    run_bulk(k_bulk<8, 8192>, 8, 8192, 2, "8x8K");
    run_bulk(k_bulk<8, 8192>, 8, 8192, 3, "8x8K");
    run_bulk(k_bulk<3, 32768>, 3, 32768, 2, "3x32K");
  }
  {
    unsigned* tk; CK(cudaMalloc(&tk, 4096)); CK(cudaMemset(tk, 0, 4096));
    double* cpart; CK(cudaMalloc(&cpart, 256 << 20));

    for (int S : {37, 74, 111, 148}) {
      int64_t Rs = (4096 + S - 1) / S;
      char nm[64];
      dim3 grid(4, S);
      {
        auto kern = k_bcol<4, 4>; int smem = 4 * 4 * 4096 + 64;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        snprintf(nm, 64, "bcol 4x4rows S=%d", S);
        time(nm, rb, [&](int c, cudaStream_t s) { kern<<<grid, T, smem, s>>>((const float*)bufs[c], 4096, 4096, Rs, cpart, tk, out); });
      }
      {
        auto kern = k_bcol<6, 2>; int smem = 6 * 2 * 4096 + 64;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        snprintf(nm, 64, "bcol 6x2rows S=%d", S);
        time(nm, rb, [&](int c, cudaStream_t s) { kern<<<grid, T, smem, s>>>((const float*)bufs[c], 4096, 4096, Rs, cpart, tk, out); });
      }
    }
    for (int S : {74}) for (int U : {8}) {
      int64_t Rs = (4096 + S - 1) / S;
      char nm[64];
      snprintf(nm, 64, "col U=%d S=%d", U, S);
      dim3 grid(4, S);
      time(nm, rb, [&](int c, cudaStream_t s) {
        if (U == 4) k_col<4><<<grid, T, 0, s>>>((const float*)bufs[c], 4096, 4096, Rs, cpart, tk, out);
        else k_col<8><<<grid, T, 0, s>>>((const float*)bufs[c], 4096, 4096, Rs, cpart, tk, out);
      });
    }
  }
  for (int mult : {8}) {
    int G = sms * mult;
    char nm[64];
    snprintf(nm, 64, "part only U=8 G=%d", G);
    time(nm, rb, [&](int c, cudaStream_t s) { k_part<8><<<G, T, 0, s>>>(bufs[c], n4, part); });
    snprintf(nm, 64, "readf U=8 G=%d", G);
    time(nm, rb, [&](int c, cudaStream_t s) { k_readf<8><<<G, T, 0, s>>>(bufs[c], n4, out); });
  }
  // a big copy for reference (the MEASURED_PEAKS method: 2 GiB each way)
  {
    float4 *a, *b; int64_t m4 = (1LL << 31) / 16;
    CK(cudaMalloc(&a, m4 * 16)); CK(cudaMalloc(&b, m4 * 16));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k_copy<<<sms * 4, T, 0, st>>>(a, b, m4);
    CK(cudaEventRecord(e0, st)); k_copy<<<sms * 4, T, 0, st>>>(a, b, m4); CK(cudaEventRecord(e1, st));
    CK(cudaStreamSynchronize(st));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-34s %8.2f us/call %8.0f GB/s\n", "copy 2 GiB", ms * 1000, 2.0 * m4 * 16 / ms / 1e6);
  }
  return 0;
}
