// Order-preserving, contraction-free fp64 arithmetic for the "faithful" kernels.
//
// The KSVD factors of the BASELINE configurations are ill-conditioned (kappa_inf up to ~1e11,
// SURVEY.md sec.7): the reference's own FMA and no-FMA builds disagree by up to 7e-7 on the PC
// apply. Kernels that must agree with the reference bit for bit therefore (1) use __dmul_rn /
// __dadd_rn / __dsub_rn (never contracted into FMA, whatever -fmad says), and (2) keep the
// reference's per-entry summation order (ascending index, starting from +0.0). IEEE add, mul,
// div and sqrt are correctly rounded on sm_100 and on x86-64, so this reproduces the reference
// compiled with its own CMake Release flags (no -march => no FMA).
#pragma once

namespace tpdg_gpu {

__device__ __forceinline__ double fmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double fsub(double a, double b) { return __dsub_rn(a, b); }
// s + a*b, rounded twice (reference `s += a * b` without contraction)
__device__ __forceinline__ double fmac(double s, double a, double b) { return __dadd_rn(s, __dmul_rn(a, b)); }
// s - a*b, rounded twice
__device__ __forceinline__ double fmsc(double s, double a, double b) { return __dsub_rn(s, __dmul_rn(a, b)); }
__device__ __forceinline__ double fdiv(double a, double b) { return __ddiv_rn(a, b); }
// a / d correctly rounded, given y = __drcp_rn(d) (computed once per divisor): one Newton step
// brings q within 1 ulp, then Markstein's correction q + (a - d q) y rounds to RN(a / d). The
// residuals are exact (FMA); r0 == 0 means q0 is already the exact quotient (also keeps -0).
// Equal to fdiv for finite, normal operands; the bit-exact parity tests pin it.
__device__ __forceinline__ double fdiv_rcp(double a, double d, double y) {
  const double q0 = __dmul_rn(a, y);
  const double r0 = __fma_rn(-d, q0, a);
  const double q1 = __fma_rn(r0, y, q0);
  const double r1 = __fma_rn(-d, q1, a);
  const double q2 = __fma_rn(r1, y, q1);
  return r0 == 0.0 ? q0 : q2;
}

} // namespace tpdg_gpu
