// Table-driven double-precision exp for the f32(exp(double x)) stores the
// reference makes (core.py:41-45, nn.py:474-501). x = (64 m + j) ln2/64 + r,
// |r| <= ln2/128; exp(x) = 2^m * 2^(j/64) * (1 + p(r)), p of degree 6
// (truncation ~1e-19). Error ~2 ulp in double, so the final f32 rounding
// matches a correctly rounded exp except within ~2^-50 of a midpoint. About
// 12 FP64 ops instead of libdevice exp's ~25: keeps the elementwise exp and
// the softmax/cross-entropy rows HBM-bound.
#pragma once
#include <math.h>

namespace b2 {

static __device__ const double kExp2Tab[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0,
};

__device__ __forceinline__ double exp_fast(double x) {
  if (!(x > -746.0)) return isnan(x) ? x : 0.0;  // NaN propagates; underflow -> +0
  if (x > 709.0) return INFINITY;
  const double kInv = 0x1.71547652b82fep+6;      // 64 / ln 2
  const double kHi = 0x1.62e42fef00000p-7;       // ln2/64, 33 bits: n*kHi exact
  const double kLo = 0x1.473de6af278edp-40;
  // round-to-integer by the 1.5*2^52 shift (n lands in the low mantissa bits):
  // no FRND/F2I conversions, which issue at a fraction of the FMA rate
  const double t_ = fma(x, kInv, 0x1.8p52);
  const double n = t_ - 0x1.8p52;
  const int ni = __double2loint(t_);
  double r = fma(-n, kHi, x);
  r = fma(-n, kLo, r);
  const int j = ni & 63, m = (ni - j) >> 6;
  double p = fma(r, 1.0 / 720.0, 1.0 / 120.0);
  p = fma(r, p, 1.0 / 24.0);
  p = fma(r, p, 1.0 / 6.0);
  p = fma(r, p, 0.5);
  p = fma(r, p, 1.0);
  p = p * r;                                      // exp(r) - 1
  const double t = __ldg(&kExp2Tab[j]);
  const double y = fma(t, p, t);                  // 2^(j/64) * exp(r), in [1, 2)
  if (m >= -1022) {                               // normal range: scale by an exact 2^m
    const double s = __longlong_as_double((long long)(m + 1023) << 52);
    return y * s;
  }
  return ldexp(y, m);                              // subnormal results (x < -708)
}

// f32(exp(double(x))) for a float x: the same table algorithm trimmed to
// what the f32 result needs (this loop is instruction-issue bound in the
// elementwise exp and the softmax rows):
// * degree-5 polynomial: truncation (ln2/128)^6/720 ~ 2^-54.7 relative;
// * the input is clamped to [-104.5, 88.8] and the clamped ends round by
//   themselves (exp(88.8) > FLT_MAX -> +inf, exp(-104.5) < 2^-150 -> +0), so
//   only NaN needs a select (fminf/fmaxf map it to an end);
// * 2^m is added to the high word of y in [0.99, 2): m in [-151, 128] keeps
//   the double normal, one f64->f32 rounding at the end.
// Verified against f32(glibc exp(double x)) -- the reference's math.exp --
// over every float input (scripts/exp_exhaustive.cu + exp_exhaustive_check.py).
__device__ __forceinline__ float exp_f32(float x) {
  const float xc = fminf(fmaxf(x, -104.5f), 88.8f);
  const double xd = (double)xc;
  const double t_ = fma(xd, 0x1.71547652b82fep+6, 0x1.8p52);  // 64/ln2; rint via the shift
  const double n = t_ - 0x1.8p52;
  const int ni = __double2loint(t_);
  double r = fma(-n, 0x1.62e42fef00000p-7, xd);
  r = fma(-n, 0x1.473de6af278edp-40, r);
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(r, p, 1.0 / 6.0);
  p = fma(r, p, 0.5);
  p = fma(r, p, 1.0);
  p = p * r;
  const double t = __ldg(&kExp2Tab[ni & 63]);
  const double y = fma(t, p, t);
  const double z = __hiloint2double(__double2hiint(y) + ((ni << 14) & (int)0xFFF00000u), __double2loint(y));
  const float v = __double2float_rn(z);
  return x == x ? v : x;
}

}  // namespace b2
