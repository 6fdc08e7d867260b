/* LD_PRELOAD shim (study tool): logs every atan2/atan/sin/cos argument the oracle's formation
 * passes to libm (standardize_2x2, reference tensor/schur.hpp:91-108) into $TRIG_LOG (binary
 * records {fn, x, y}) and forwards to the real libm. */
#define _GNU_SOURCE
#include <dlfcn.h>
#include <stdio.h>
#include <stdlib.h>
static FILE* f;
static void rec(double fn, double x, double y) {
  if (!f) { const char* p = getenv("TRIG_LOG"); if (!p) return; f = fopen(p, "ab"); }
  double r[3] = {fn, x, y};
  fwrite(r, 8, 3, f);
}
double atan2(double y, double x) { static double (*g)(double, double); if (!g) g = dlsym(RTLD_NEXT, "atan2"); rec(3, y, x); return g(y, x); }
double atan(double x) { static double (*g)(double); if (!g) g = dlsym(RTLD_NEXT, "atan"); rec(2, x, 0); return g(x); }
double sin(double x) { static double (*g)(double); if (!g) g = dlsym(RTLD_NEXT, "sin"); rec(0, x, 0); return g(x); }
double cos(double x) { static double (*g)(double); if (!g) g = dlsym(RTLD_NEXT, "cos"); rec(1, x, 0); return g(x); }
