// glibm.cuh — sin, cos, atan and atan2 exactly as the reference's libm computes them.
//
// Why: the one libm call site on the hot path is standardize_2x2 (reference tensor/schur.hpp:91-108:
// atan2, atan, cos, sin; GCC fuses the cos/sin pairs into sincos, which glibc computes with the same
// code as sin and cos). The KSVD factors amplify a 1-ulp difference in a Schur rotation to ~1e-9 in
// the preconditioner apply, so the device must return the reference's bits, not merely accurate
// ones: CUDA's sin/cos/atan2 are not correctly rounded, and glibc's are not either (a correctly
// rounded double-double implementation disagrees with glibc on ~5e-4 of the atan2 calls the cfg2
// p = 15 formation makes).
//
// What: a restatement of the third-party dependency's published algorithm — GNU C Library 2.39
// (Ubuntu 2.39-0ubuntu8.5, x86_64), sysdeps/ieee754/dbl-64 s_sin.c (do_sin, do_cos, TAYLOR_SIN,
// reduce_sincos), s_atan.c and e_atan2.c (the IBM Accurate Mathematical Library after the removal of
// the multi-precision slow paths) — in the operation order of the FMA builds that glibc's ifunc
// selects on AVX2+FMA hosts (__sin_fma, __cos_fma, __atan_fma, __ieee754_atan2_fma): every place
// where that build contracts a multiply-add is an explicit fma below, every other operation is an
// individually rounded add/mul/div. Arguments outside the ranges the path can produce
// (|x| >= 105414350 for sin/cos) fall back to CUDA's functions.
//
// Tables: glibm_tables.h (tools/gen_glibc_tables.py). Verified bit for bit against the host libm:
// tests/test_glibm_cpu.py (host build of this file) and tests/test_gpu_glibm.py (device, >= 10^7
// arguments per function).
#pragma once
#include "glibm_tables.h"

#if defined(__CUDACC__)
#define GLIBM_FN __host__ __device__ __forceinline__ static
__device__ static const double glibm_sincos_dev[] = GLIBM_SINCOS_INIT;
__device__ static const double glibm_cij_dev[241][7] = GLIBM_CIJ_INIT;
#else
#include <math.h>
#include <string.h>
#define GLIBM_FN static inline
#endif
static const double glibm_sincos_host[] = GLIBM_SINCOS_INIT;
static const double glibm_cij_host[241][7] = GLIBM_CIJ_INIT;

#if defined(__CUDA_ARCH__)
#define GL_ADD(a, b) __dadd_rn((a), (b))
#define GL_SUB(a, b) __dsub_rn((a), (b))
#define GL_MUL(a, b) __dmul_rn((a), (b))
#define GL_DIV(a, b) __ddiv_rn((a), (b))
#define GL_FMA(a, b, c) __fma_rn((a), (b), (c))
#define GL_SINCOS_TAB glibm_sincos_dev
#define GL_CIJ glibm_cij_dev
#else
#define GL_ADD(a, b) ((a) + (b))
#define GL_SUB(a, b) ((a) - (b))
#define GL_MUL(a, b) ((a) * (b))
#define GL_DIV(a, b) ((a) / (b))
#define GL_FMA(a, b, c) fma((a), (b), (c))
#define GL_SINCOS_TAB glibm_sincos_host
#define GL_CIJ glibm_cij_host
#endif

GLIBM_FN int gl_hi(double x) {
#if defined(__CUDA_ARCH__)
  return __double2hiint(x);
#else
  long long b; memcpy(&b, &x, 8); return (int)(b >> 32);
#endif
}
GLIBM_FN int gl_lo(double x) {
#if defined(__CUDA_ARCH__)
  return __double2loint(x);
#else
  long long b; memcpy(&b, &x, 8); return (int)(b & 0xffffffff);
#endif
}

// s_sin.c / usncs.h constants
#define GL_BIG 0x1.8p45
#define GL_HP0 0x1.921fb54442d18p0
#define GL_HP1 0x1.1a62633145c07p-54
#define GL_MP1 0x1.921fb58p0
#define GL_MP2 -0x1.dde973cp-27
#define GL_PP3 -0x1.cb3b398p-55
#define GL_PP4 -0x1.d747f23e32ed7p-83
#define GL_HPINV 0x1.45f306dc9c883p-1
#define GL_TOINT 0x1.8p52
#define GL_SN3 -0x1.5555555555515p-3
#define GL_SN5 0x1.11110e829872fp-7
#define GL_CS2 0.5
#define GL_CS4 -0x1.5555555555535p-5
#define GL_CS6 0x1.6c16bedd9e239p-10
#define GL_S1 -0x1.5555555555555p-3
#define GL_S2 0x1.1111111110ecep-7
#define GL_S3 -0x1.a01a019db08b8p-13
#define GL_S4 0x1.71de27b9a7ed9p-19
#define GL_S5 -0x1.addffc2fcdf59p-26
// s_atan.c / e_atan2.c / atnat.h constants
#define GL_D3 -0x1.5555555555555p-2
#define GL_D5 0x1.99999999997fdp-3
#define GL_D7 -0x1.24924923f7603p-3
#define GL_D9 0x1.c71c6e5129a3bp-4
#define GL_D11 -0x1.7458022b13c25p-4
#define GL_D13 0x1.375f08b31cbcep-4
#define GL_ATAN_A 0x1.bb67ap-27
#define GL_ATAN_E 0x1.49ff2p52
#define GL_TWO52 0x1p52
#define GL_OPI 0x1.921fb54442d18p1
#define GL_OPI1 0x1.1a62633145c07p-53
#define GL_QPI 0x1.921fb54442d18p-1
#define GL_TQPI 0x1.2d97c7f3321d2p1

// TAYLOR_SIN (s_sin.c): sin(a + da) for |a| < 0.126
GLIBM_FN double gl_taylor_sin(double a, double da) {
  const double xx = GL_MUL(a, a);
  double p = GL_FMA(GL_FMA(GL_FMA(GL_FMA(GL_S5, xx, GL_S4), xx, GL_S3), xx, GL_S2), xx, GL_S1);
  p = GL_FMA(p, a, -GL_MUL(0.5, da));
  return GL_ADD(a, GL_FMA(xx, p, da));
}
// do_sin (s_sin.c): sin(x + dx), table node i/128 + polynomial correction
GLIBM_FN double gl_do_sin(double x, double dx) {
  const double xold = x;
  if (fabs(x) < 0.126) return gl_taylor_sin(x, dx);
  if (x <= 0) dx = -dx;
  const double u = GL_ADD(fabs(x), GL_BIG);
  x = GL_SUB(fabs(x), GL_SUB(u, GL_BIG));
  const int k = gl_lo(u) << 2;
  const double xx = GL_MUL(x, x);
  const double s = GL_ADD(x, GL_FMA(GL_MUL(x, xx), GL_FMA(xx, GL_SN5, GL_SN3), dx));
  const double c = GL_FMA(x, dx, GL_MUL(xx, GL_FMA(xx, GL_FMA(xx, GL_CS6, GL_CS4), GL_CS2)));
  const double sn = GL_SINCOS_TAB[k], ssn = GL_SINCOS_TAB[k + 1], cs = GL_SINCOS_TAB[k + 2],
               ccs = GL_SINCOS_TAB[k + 3];
  const double cor = GL_FMA(s, cs, GL_FMA(-c, sn, GL_FMA(s, ccs, ssn)));
  return copysign(GL_ADD(sn, cor), xold);
}
// do_cos (s_sin.c): cos(x + dx)
GLIBM_FN double gl_do_cos(double x, double dx) {
  if (x < 0) dx = -dx;
  const double u = GL_ADD(fabs(x), GL_BIG);
  x = GL_ADD(GL_SUB(fabs(x), GL_SUB(u, GL_BIG)), dx);
  const int k = gl_lo(u) << 2;
  const double xx = GL_MUL(x, x);
  const double s = GL_FMA(GL_MUL(x, xx), GL_FMA(xx, GL_SN5, GL_SN3), x);
  const double c = GL_MUL(xx, GL_FMA(xx, GL_FMA(xx, GL_CS6, GL_CS4), GL_CS2));
  const double sn = GL_SINCOS_TAB[k], ssn = GL_SINCOS_TAB[k + 1], cs = GL_SINCOS_TAB[k + 2],
               ccs = GL_SINCOS_TAB[k + 3];
  const double cor = GL_FMA(-s, sn, GL_FMA(-c, cs, GL_FMA(-s, ssn, ccs)));
  return GL_ADD(cs, cor);
}
// reduce_sincos (s_sin.c): x = n pi/2 + (a + da), |x| < 105414350
GLIBM_FN int gl_reduce(double x, double* a, double* da) {
  const double t = GL_FMA(x, GL_HPINV, GL_TOINT);
  const double xn = GL_SUB(t, GL_TOINT);
  const int n = gl_lo(t) & 3;
  double y = GL_FMA(-xn, GL_MP1, x);
  y = GL_FMA(-xn, GL_MP2, y);
  const double t2 = GL_FMA(-xn, GL_PP3, y);
  double db = GL_FMA(-xn, GL_PP3, GL_SUB(y, t2));
  const double b = GL_FMA(-xn, GL_PP4, t2);
  db = GL_ADD(db, GL_FMA(-xn, GL_PP4, GL_SUB(t2, b)));
  *a = b;
  *da = db;
  return n;
}

GLIBM_FN double glibm_sin(double x) {
  const int k = gl_hi(x) & 0x7fffffff;
  if (k < 0x3e500000) return x;
  if (k < 0x3feb6000) return gl_do_sin(x, 0.0);
  if (k < 0x400368fd) return copysign(gl_do_cos(GL_SUB(GL_HP0, fabs(x)), GL_HP1), x);
  if (k < 0x419921fb) {
    double a, da;
    const int n = gl_reduce(x, &a, &da);
    const double r = (n & 1) ? gl_do_cos(a, da) : gl_do_sin(a, da);
    return (n & 2) ? -r : r;
  }
  return sin(x);
}
GLIBM_FN double glibm_cos(double x) {
  const int k = gl_hi(x) & 0x7fffffff;
  if (k < 0x3e400000) return 1.0;
  if (k < 0x3feb6000) return gl_do_cos(x, 0.0);
  if (k < 0x400368fd) {
    const double y = GL_SUB(GL_HP0, fabs(x));
    const double a = GL_ADD(y, GL_HP1);
    const double da = GL_ADD(GL_SUB(y, a), GL_HP1);
    return gl_do_sin(a, da);
  }
  if (k < 0x419921fb) {
    double a, da;
    const int n = gl_reduce(x, &a, &da) + 1;
    const double r = (n & 1) ? gl_do_cos(a, da) : gl_do_sin(a, da);
    return (n & 2) ? -r : r;
  }
  return cos(x);
}

GLIBM_FN double gl_poly_d(double v) {  // d3 + v (d5 + v (d7 + v (d9 + v (d11 + v d13))))
  return GL_FMA(v, GL_FMA(v, GL_FMA(v, GL_FMA(v, GL_FMA(v, GL_D13, GL_D11), GL_D9), GL_D7), GL_D5), GL_D3);
}
GLIBM_FN int gl_cij_index(double u) { return (int)GL_SUB(GL_FMA(u, 256.0, GL_TWO52), GL_TWO52) - 16; }
GLIBM_FN double gl_poly_c(const double* c, double z) {  // c2 + z (c3 + z (c4 + z (c5 + z c6)))
  return GL_FMA(z, GL_FMA(z, GL_FMA(z, GL_FMA(z, c[6], c[5]), c[4]), c[3]), c[2]);
}

// s_atan.c
GLIBM_FN double glibm_atan(double x) {
  if (x != x) return GL_ADD(x, x);
  const double u = fabs(x);
  if (u < 1.0) {
    if (u < 0.0625) {
      if (u < GL_ATAN_A) return x;
      const double v = GL_MUL(x, x);
      return GL_FMA(GL_MUL(x, v), gl_poly_d(v), x);
    }
    const double* c = GL_CIJ[gl_cij_index(u)];
    const double z = GL_SUB(u, c[0]);
    return copysign(GL_FMA(gl_poly_c(c, z), z, c[1]), x);
  }
  if (u < 16.0) {
    const double w = GL_DIV(1.0, u);
    const double t1 = GL_MUL(w, u);
    const double t2 = GL_FMA(u, w, -t1);
    const double e = GL_SUB(GL_SUB(1.0, t1), t2);
    const double* c = GL_CIJ[gl_cij_index(w)];
    const double z = GL_FMA(e, w, GL_SUB(w, c[0]));
    const double yy = GL_FMA(-gl_poly_c(c, z), z, GL_HP1);
    return copysign(GL_ADD(GL_SUB(GL_HP0, c[1]), yy), x);
  }
  if (u < GL_ATAN_E) {
    const double w = GL_DIV(1.0, u);
    const double t1 = GL_MUL(w, u);
    const double ta = GL_SUB(GL_HP0, w);
    const double v = GL_MUL(w, w);
    const double yy = gl_poly_d(v);
    const double t2 = GL_FMA(u, w, -t1);
    const double e = GL_SUB(GL_SUB(1.0, t1), t2);
    const double t3 = GL_ADD(GL_SUB(GL_SUB(GL_HP0, ta), w), GL_HP1);
    double r = GL_FMA(-e, w, t3);
    r = GL_FMA(-GL_MUL(w, v), yy, r);
    return copysign(GL_ADD(ta, r), x);
  }
  return copysign(GL_HP0, x);
}

GLIBM_FN bool gl_signbit(double x) { return gl_hi(x) < 0; }

// e_atan2.c
GLIBM_FN double glibm_atan2(double y, double x) {
  if (x != x) return GL_ADD(x, y);
  if (y != y) return GL_ADD(y, y);
  const bool xneg = gl_signbit(x), yneg = gl_signbit(y);
  if (y == 0) return xneg ? (yneg ? -GL_OPI : GL_OPI) : y;
  if (x == 0) return yneg ? -GL_HP0 : GL_HP0;
  const double inf = __builtin_huge_val();
  if (fabs(x) == inf) {
    if (fabs(y) == inf) return xneg ? (yneg ? -GL_TQPI : GL_TQPI) : (yneg ? -GL_QPI : GL_QPI);
    return xneg ? (yneg ? -GL_OPI : GL_OPI) : (yneg ? -0.0 : 0.0);
  }
  if (fabs(y) == inf) return yneg ? -GL_HP0 : GL_HP0;

  double ax = fabs(x), ay = fabs(y);
  const int de = (gl_hi(y) & 0x7ff00000) - (gl_hi(x) & 0x7ff00000);
  if (de >= 0x3900000) return yneg ? -GL_HP0 : GL_HP0;
  if (de <= -0x3900000) {
    if (x > 0) return copysign(GL_DIV(ay, ax), y);
    return yneg ? -GL_OPI : GL_OPI;
  }
  if (ax < 0x1p-500 || ay < 0x1p-500) { ax = GL_MUL(ax, 0x1p500); ay = GL_MUL(ay, 0x1p500); }
  if (ax > 0x1p500 || ay > 0x1p500) { ax = GL_MUL(ax, 0x1p-500); ay = GL_MUL(ay, 0x1p-500); }

  double u, du;
  if (ay < ax) {
    u = GL_DIV(ay, ax);
    const double v = GL_MUL(u, ax), vv = GL_FMA(u, ax, -v);
    du = GL_DIV(GL_SUB(GL_SUB(ay, v), vv), ax);
  } else {
    u = GL_DIV(ax, ay);
    const double v = GL_MUL(u, ay), vv = GL_FMA(u, ay, -v);
    du = GL_DIV(GL_SUB(GL_SUB(ax, v), vv), ay);
  }
  double z;
  if (x > 0) {
    if (ay < ax) {  // (i) atan(ay/ax)
      if (u < 0.0625) {
        const double v = GL_MUL(u, u);
        z = GL_ADD(u, GL_FMA(GL_MUL(u, v), gl_poly_d(v), du));
      } else {
        const double* c = GL_CIJ[gl_cij_index(u)];
        const double t3 = GL_SUB(u, c[0]);
        const double v = GL_ADD(t3, du);
        const double dv = fabs(t3) > fabs(du) ? GL_ADD(GL_SUB(t3, v), du) : GL_ADD(GL_SUB(du, v), t3);
        const double p = GL_MUL(GL_MUL(v, v), GL_FMA(v, GL_FMA(v, GL_FMA(v, c[6], c[5]), c[4]), c[3]));
        z = GL_ADD(GL_FMA(v, c[2], GL_FMA(dv, c[2], p)), c[1]);
      }
    } else {  // (ii) pi/2 - atan(ax/ay)
      if (u < 0.0625) {
        const double v = GL_MUL(u, u);
        const double zz = GL_MUL(GL_MUL(u, v), gl_poly_d(v));
        const double t2 = GL_SUB(GL_HP0, u);
        const double cor = fabs(GL_HP0) > fabs(u) ? GL_SUB(GL_SUB(GL_HP0, t2), u)
                                                  : GL_SUB(GL_HP0, GL_ADD(u, t2));
        z = GL_ADD(GL_SUB(GL_SUB(GL_ADD(cor, GL_HP1), du), zz), t2);
      } else {
        const double* c = GL_CIJ[gl_cij_index(u)];
        const double v = GL_ADD(GL_SUB(u, c[0]), du);
        z = GL_ADD(GL_SUB(GL_HP0, c[1]), GL_FMA(-v, gl_poly_c(c, v), GL_HP1));
      }
    }
  } else {
    if (ax < ay) {  // (iii) pi/2 + atan(ax/ay)
      if (u < 0.0625) {
        const double v = GL_MUL(u, u);
        const double zz = GL_MUL(GL_MUL(u, v), gl_poly_d(v));
        const double t2 = GL_ADD(GL_HP0, u);
        const double cor = fabs(GL_HP0) > fabs(u) ? GL_ADD(GL_SUB(GL_HP0, t2), u)
                                                  : GL_ADD(GL_SUB(u, t2), GL_HP0);
        z = GL_ADD(GL_ADD(GL_ADD(GL_ADD(cor, GL_HP1), du), zz), t2);
      } else {
        const double* c = GL_CIJ[gl_cij_index(u)];
        const double v = GL_ADD(GL_SUB(u, c[0]), du);
        z = GL_ADD(GL_ADD(GL_HP0, c[1]), GL_FMA(v, gl_poly_c(c, v), GL_HP1));
      }
    } else {  // (iv) pi - atan(ay/ax)
      if (u < 0.0625) {
        const double v = GL_MUL(u, u);
        const double zz = GL_MUL(GL_MUL(u, v), gl_poly_d(v));
        const double t2 = GL_SUB(GL_OPI, u);
        const double cor = fabs(GL_OPI) > fabs(u) ? GL_SUB(GL_SUB(GL_OPI, t2), u)
                                                  : GL_SUB(GL_OPI, GL_ADD(u, t2));
        z = GL_ADD(GL_SUB(GL_SUB(GL_ADD(cor, GL_OPI1), du), zz), t2);
      } else {
        const double* c = GL_CIJ[gl_cij_index(u)];
        const double v = GL_ADD(GL_SUB(u, c[0]), du);
        z = GL_ADD(GL_SUB(GL_OPI, c[1]), GL_FMA(-v, gl_poly_c(c, v), GL_OPI1));
      }
    }
  }
  return copysign(z, y);
}
