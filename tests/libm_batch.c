/* Host libm (glibc) over arrays, for tests/test_gpu_glibm.py: fn 0 sin, 1 cos, 2 atan, 3 atan2(x, y). */
#include <math.h>
void libm_batch(int fn, long n, const double* x, const double* y, double* out) {
  for (long i = 0; i < n; ++i)
    out[i] = fn == 0 ? sin(x[i]) : fn == 1 ? cos(x[i]) : fn == 2 ? atan(x[i]) : atan2(x[i], y[i]);
}
