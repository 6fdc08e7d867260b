/* Host build of glibm.cuh checked bit for bit against the host libm (glibc 2.39, FMA variants) on
 * random arguments from the ranges standardize_2x2 produces and beyond, plus special values.
 * Build: gcc -O2 -ffp-contract=off tests/glibm_check.c -lm (tests/test_glibm_cpu.py). Usage: glibm_check N [seed] */
#include <stdbool.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include "../paper_1704_04549_b200/csrc/glibm.cuh"

static uint64_t s;
static uint64_t rnd(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double uni(double a, double b) { return a + (b - a) * ((rnd() >> 11) * 0x1p-53); }
static double logu(int emin, int emax) {  /* random sign and mantissa, exponent uniform in [emin, emax] */
  int e = emin + (int)(rnd() % (uint64_t)(emax - emin + 1));
  return ldexp(1.0 + (rnd() >> 12) * 0x1p-52, e) * ((rnd() & 1) ? -1 : 1);
}
static int same(double a, double b) { return memcmp(&a, &b, 8) == 0 || (a != a && b != b); }
static long bad[4], shown;
static void chk(int fn, double x, double y) {
  double g, m;
  switch (fn) {
    case 0: g = sin(x); m = glibm_sin(x); break;
    case 1: g = cos(x); m = glibm_cos(x); break;
    case 2: g = atan(x); m = glibm_atan(x); break;
    default: g = atan2(x, y); m = glibm_atan2(x, y); break;
  }
  if (!same(g, m)) {
    bad[fn]++;
    if (shown++ < 10) printf("fn %d (%a, %a): libm %a restated %a\n", fn, x, y, g, m);
  }
}
int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 1000000;
  s = argc > 2 ? strtoull(argv[2], 0, 10) : 0x9E3779B97F4A7C15ull;
  const double sp[] = {0.0, -0.0, 1.0, -1.0, 0.0625, 16.0, 0x1.49ff2p52, 0x1p-1074, 0x1p-1022, 1e300,
                       INFINITY, -INFINITY, NAN, M_PI, M_PI_2, M_PI_4, 0.855469, 2.426265, 0.126, 1e-8};
  int nsp = sizeof sp / sizeof sp[0];
  for (int i = 0; i < nsp; ++i) {
    chk(0, sp[i], 0); chk(1, sp[i], 0); chk(2, sp[i], 0);
    for (int j = 0; j < nsp; ++j) chk(3, sp[i], sp[j]);
  }
  for (long i = 0; i < n; ++i) {
    double x;
    switch (i % 4) {
      case 0: x = uni(-M_PI, M_PI); break;     /* standardize_2x2's theta range */
      case 1: x = logu(-40, 6); break;
      case 2: x = uni(-1e5, 1e5); break;
      default: x = uni(-2.5, 2.5); break;
    }
    chk(0, x, 0); chk(1, x, 0);
    double t = (i & 1) ? logu(-40, 60) : uni(-20, 20);
    chk(2, t, 0);
    double y = (i % 3) ? logu(-40, 40) : uni(-2, 2), z = (i % 5) ? logu(-40, 40) : uni(-2, 2);
    if (i % 7 == 0) z = y * uni(0.9, 1.1);
    if (i % 11 == 0) y = logu(-1070, 1023), z = logu(-1070, 1023);
    chk(3, y, z);
  }
  printf("n=%ld mismatches: sin %ld cos %ld atan %ld atan2 %ld\n", n, bad[0], bad[1], bad[2], bad[3]);
  return (bad[0] || bad[1] || bad[2] || bad[3]) ? 1 : 0;
}
