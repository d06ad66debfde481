// Conv2D data movement for the im2col formulation of tensorlite's conv2d
// (nn.py:191-303): the patch matrix feeds the tcgen05 / FFMA
// GEMM engine, and the input cotangent is gathered back from the patch
// cotangent.
//
// im2col: patches[r, col] with r = (b, i, j) output position (row-major) and
//   col = (c, u, v) kernel tap; zero where the tap falls in the padding.
// col2im: dx[b, c, ih, iw] = sum over the taps that read (ih, iw) of dp[r, col],
//   accumulated in double in increasing r -- the order of the reference's
//   scatter loop (nn.py:275-292, Python floats) -- and rounded to f32 once.
//   A gather per input element: deterministic, no atomics.
#include <cuda_runtime.h>

#include "common.cuh"

namespace {

struct ConvGeom {
  int64_t B, C, H, W, KH, KW, S, P, OH, OW;
};

__global__ void __launch_bounds__(256) k_im2col(float* __restrict__ patches,
                                                const float* __restrict__ x, ConvGeom g) {
  const int64_t cols = g.C * g.KH * g.KW;
  const int64_t total = g.B * g.OH * g.OW * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, col = e - r * cols;
    const int64_t plane = g.OH * g.OW;
    const int64_t b = r / plane, pos = r - b * plane;
    const int64_t i = pos / g.OW, j = pos - i * g.OW;
    const int64_t c = col / (g.KH * g.KW), uv = col - c * g.KH * g.KW;
    const int64_t u = uv / g.KW, v = uv - u * g.KW;
    const int64_t ih = i * g.S - g.P + u, iw = j * g.S - g.P + v;
    float val = 0.0f;
    if (ih >= 0 && ih < g.H && iw >= 0 && iw < g.W) val = x[((b * g.C + c) * g.H + ih) * g.W + iw];
    patches[e] = val;
  }
}

__global__ void __launch_bounds__(256) k_col2im(float* __restrict__ dx, const float* __restrict__ dp,
                                                ConvGeom g) {
  const int64_t cols = g.C * g.KH * g.KW;
  const int64_t total = g.B * g.C * g.H * g.W;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t iw = e % g.W;
    int64_t q = e / g.W;
    const int64_t ih = q % g.H;
    q /= g.H;
    const int64_t c = q % g.C, b = q / g.C;
    double acc = 0.0;
    // taps (u, v) descending -> output rows r = (i, j) ascending
    for (int64_t u = g.KH - 1; u >= 0; --u) {
      const int64_t ti = ih + g.P - u;
      if (ti < 0 || ti % g.S) continue;
      const int64_t i = ti / g.S;
      if (i >= g.OH) continue;
      for (int64_t v = g.KW - 1; v >= 0; --v) {
        const int64_t tj = iw + g.P - v;
        if (tj < 0 || tj % g.S) continue;
        const int64_t j = tj / g.S;
        if (j >= g.OW) continue;
        const int64_t r = (b * g.OH + i) * g.OW + j;
        acc += (double)dp[r * cols + (c * g.KH + u) * g.KW + v];
      }
    }
    dx[e] = __double2float_rn(acc);
  }
}

int check(const ConvGeom& g) {
  if (g.B < 0 || g.C < 1 || g.H < 1 || g.W < 1 || g.KH < 1 || g.KW < 1 || g.S < 1 || g.P < 0)
    return b2::fail("conv2d: invalid geometry");
  if (g.OH != (g.H + 2 * g.P - g.KH) / g.S + 1 || g.OW != (g.W + 2 * g.P - g.KW) / g.S + 1 ||
      g.OH < 1 || g.OW < 1)
    return b2::fail("conv2d: output extent does not match the geometry");
  return 0;
}

}  // namespace

extern "C" {

int b2_im2col(float* patches, const float* x, int64_t B, int64_t C, int64_t H, int64_t W,
              int64_t KH, int64_t KW, int64_t stride, int64_t pad, int64_t OH, int64_t OW,
              void* stream) {
  ConvGeom g{B, C, H, W, KH, KW, stride, pad, OH, OW};
  B2_TRY(check(g));
  const int64_t total = B * OH * OW * C * KH * KW;
  if (total == 0) return 0;
  k_im2col<<<b2::grid_for(total, 256 * 4, 8), 256, 0, b2::resolve(stream)>>>(patches, x, g);
  return b2::launched("b2_im2col");
}

int b2_col2im(float* dx, const float* dp, int64_t B, int64_t C, int64_t H, int64_t W, int64_t KH,
              int64_t KW, int64_t stride, int64_t pad, int64_t OH, int64_t OW, void* stream) {
  ConvGeom g{B, C, H, W, KH, KW, stride, pad, OH, OW};
  B2_TRY(check(g));
  const int64_t total = B * C * H * W;
  if (total == 0) return 0;
  k_col2im<<<b2::grid_for(total, 256 * 4, 8), 256, 0, b2::resolve(stream)>>>(dx, dp, g);
  return b2::launched("b2_col2im");
}

}  // extern "C"
