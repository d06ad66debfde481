// Exhaustive check of b2::exp_f32 (fexp.cuh) over all 2^32 float inputs.
// Every input where it differs from f32(libdevice exp(double x)) is written
// out as (x, device, libdevice) bit triples; scripts/exp_exhaustive_check.py
// then settles each one against f32(math.exp(x)) -- glibc, the reference's
// exp (tensorlite core.py:509) -- on the host. The previous table variant
// (degree 6, explicit range selects) runs alongside as `v0` for comparison.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2602_00125_b200/csrc \
//        -o scripts/exp_exhaustive scripts/exp_exhaustive.cu
//   ./scripts/exp_exhaustive gpurun_out/exp_new.bin gpurun_out/exp_v0.bin
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include "fexp.cuh"

__device__ __forceinline__ float exp_f32_v0(float x) {
  const float xc = fminf(fmaxf(x, -104.5f), 88.8f);
  const double xd = (double)xc;
  const double t_ = fma(xd, 0x1.71547652b82fep+6, 0x1.8p52);
  const double n = t_ - 0x1.8p52;
  const int ni = __double2loint(t_);
  double r = fma(-n, 0x1.62e42fef00000p-7, xd);
  r = fma(-n, 0x1.473de6af278edp-40, r);
  const int j = ni & 63, m = (ni - j) >> 6;
  double p = fma(r, 1.0 / 720.0, 1.0 / 120.0);
  p = fma(r, p, 1.0 / 24.0);
  p = fma(r, p, 1.0 / 6.0);
  p = fma(r, p, 0.5);
  p = fma(r, p, 1.0);
  p = p * r;
  const double t = __ldg(&b2::kExp2Tab[j]);
  const double y = fma(t, p, t);
  float v = __double2float_rn(__longlong_as_double(__double_as_longlong(y) + ((long long)m << 52)));
  v = x < 88.8f ? v : INFINITY;
  v = x > -104.5f ? v : 0.0f;
  return x == x ? v : x;
}

template <int V>
__global__ void k_check(uint64_t base, unsigned* count, uint32_t* out, unsigned cap) {
  const uint64_t i = base + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i > 0xffffffffull) return;
  const uint32_t bits = (uint32_t)i;
  const float x = __uint_as_float(bits);
  const float got = V == 0 ? b2::exp_f32(x) : exp_f32_v0(x);
  const float want = __double2float_rn(exp((double)x));
  const bool same = (__float_as_uint(got) == __float_as_uint(want)) || (isnan(got) && isnan(want));
  if (!same) {
    unsigned k = atomicAdd(count, 1u);
    if (k < cap) {
      out[3 * k] = bits;
      out[3 * k + 1] = __float_as_uint(got);
      out[3 * k + 2] = __float_as_uint(want);
    }
  }
}

template <int V>
int run(const char* path) {
  const unsigned cap = 1 << 22;
  unsigned* count; uint32_t* out;
  cudaMalloc(&count, 4); cudaMemset(count, 0, 4);
  cudaMalloc(&out, cap * 12ull);
  const uint64_t total = 1ull << 32, per = 1ull << 30;
  for (uint64_t b = 0; b < total; b += per)
    k_check<V><<<(unsigned)(per / 256), 256>>>(b, count, out, cap);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  unsigned n; cudaMemcpy(&n, count, 4, cudaMemcpyDeviceToHost);
  unsigned m = n < cap ? n : cap;
  uint32_t* h = new uint32_t[3ull * (m ? m : 1)];
  cudaMemcpy(h, out, m * 12ull, cudaMemcpyDeviceToHost);
  FILE* f = fopen(path, "wb");
  fwrite(h, 12, m, f); fclose(f);
  printf("%s: %u inputs differ from f32(libdevice exp) (saved %u)\n", V == 0 ? "exp_f32" : "v0", n, m);
  cudaFree(count); cudaFree(out); delete[] h;
  return 0;
}

int main(int argc, char** argv) {
  if (run<0>(argc > 1 ? argv[1] : "exp_new.bin")) return 1;
  if (run<1>(argc > 2 ? argv[2] : "exp_v0.bin")) return 1;
  return 0;
}
