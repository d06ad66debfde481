/* The device's f32 exp (paper_2602_00125_b200/csrc/fexp.cuh, exp_f32),
 * restated in C with the same IEEE double operations (fma, the same table and
 * constants, the same exponent arithmetic), compared over all 2^32 float
 * inputs with f32(glibc exp(double x)) -- what the reference computes
 * (tensorlite core.py:509 through CPython's math.exp). Together with
 * scripts/exp_exhaustive.cu (device == f32(libdevice exp) on every input)
 * this pins the device exp bit-for-bit on the whole float domain.
 *   (tests/test_exp_exhaustive.py writes exp_table.inc from fexp.cuh, compiles with gcc -O2 -fopenmp and runs it) */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

static double T[64];

static float dev_exp(float x) {
  float xc = fminf(fmaxf(x, -104.5f), 88.8f);
  if (isnan(x)) xc = -104.5f; /* fmaxf(NaN, a) = a on the device too */
  double xd = (double)xc;
  double t_ = fma(xd, 0x1.71547652b82fep+6, 0x1.8p52);
  double n = t_ - 0x1.8p52;
  uint64_t tb; memcpy(&tb, &t_, 8);
  int32_t ni = (int32_t)(uint32_t)tb;
  double r = fma(-n, 0x1.62e42fef00000p-7, xd);
  r = fma(-n, 0x1.473de6af278edp-40, r);
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(r, p, 1.0 / 6.0);
  p = fma(r, p, 0.5);
  p = fma(r, p, 1.0);
  p = p * r;
  double t = T[ni & 63];
  double y = fma(t, p, t);
  uint64_t yb; memcpy(&yb, &y, 8);
  uint32_t hi = (uint32_t)(yb >> 32) + (((uint32_t)ni << 14) & 0xFFF00000u);
  yb = ((uint64_t)hi << 32) | (yb & 0xffffffffu);
  double z; memcpy(&z, &yb, 8);
  float v = (float)z;
  return x == x ? v : x;
}

int main(void) {
  /* the device table, as hex literals (fexp.cuh kExp2Tab) */
  static const double tab[64] = {
#include "exp_table.inc"
  };
  memcpy(T, tab, sizeof T);
  long long bad = 0, first = -1;
#pragma omp parallel for reduction(+ : bad) schedule(static, 1 << 20)
  for (long long i = 0; i < (1LL << 32); ++i) {
    uint32_t b = (uint32_t)i;
    float x; memcpy(&x, &b, 4);
    float want = (float)exp((double)x);
    float got = dev_exp(x);
    uint32_t wb, gb; memcpy(&wb, &want, 4); memcpy(&gb, &got, 4);
    if (wb != gb && !(isnan(want) && isnan(got))) {
      ++bad;
#pragma omp critical
      if (first < 0) first = i;
    }
  }
  printf("{\"inputs\": 4294967296, \"mismatches_vs_glibc\": %lld, \"first_bits\": %lld}\n", bad, first);
  return bad != 0;
}
