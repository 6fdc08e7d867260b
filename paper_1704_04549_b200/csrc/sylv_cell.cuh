// Factored tiny systems of the quasi-triangular Sylvester solve (shared by kron.cu and kron_ew.cu).
#pragma once

#include "faithful.cuh"

namespace tpdg_gpu {

// The tiny system of a Sylvester cell, (T1_ii (x) I + I (x) T2_kk) y = r (sylvester.hpp:84-107),
// does not depend on the data: sylv_cells_kernel runs solve_tiny's elimination once per PC and
// stores what it applies to the right-hand side, so that the apply only replays those row
// operations. Cell slot: [code, L (strict lower, row-major), U (strict upper, row-major),
// diag(U), 1/diag(U)]; code = perm[u] in bits 2u..2u+1 | singular << 8. The row swaps of the
// interleaved elimination are composed LAPACK-style (swapped together with the stored
// multipliers), so every right-hand side entry sees the same operations in the same order.
template <int IS, int KS>
__device__ __forceinline__ void factor_cell(const double* t1, int n1, const double* t2, int n2, int i0, int k0, double tol,
                            double* c) {
  constexpr int NS = IS * KS;
  double a[NS][NS], L[NS][NS];
  int perm[NS];
  bool sing = false;
#pragma unroll
  for (int ai = 0; ai < IS; ++ai)
#pragma unroll
    for (int kb = 0; kb < KS; ++kb)
#pragma unroll
      for (int a2 = 0; a2 < IS; ++a2)
#pragma unroll
        for (int kb2 = 0; kb2 < KS; ++kb2) {
          double coef = 0.0;
          if (kb == kb2) coef = fadd(coef, t1[(i0 + ai) * n1 + i0 + a2]);
          if (ai == a2) coef = fadd(coef, t2[(k0 + kb) * n2 + k0 + kb2]);
          a[ai * KS + kb][a2 * KS + kb2] = coef;
        }
#pragma unroll
  for (int u = 0; u < NS; ++u) {
    perm[u] = u;
#pragma unroll
    for (int v = 0; v < NS; ++v) L[u][v] = 0.0;
  }
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    int piv = k;
    double pv = a[k][k];
#pragma unroll
    for (int i = k + 1; i < NS; ++i)
      if (fabs(a[i][k]) > fabs(pv)) {
        pv = a[i][k];
        piv = i;
      }
    if (fabs(pv) < tol) {
      sing = true;
      break;
    }
#pragma unroll
    for (int i = k + 1; i < NS; ++i)
      if (piv == i) {
#pragma unroll
        for (int j = 0; j < NS; ++j) {
          double t = a[i][j];
          a[i][j] = a[k][j];
          a[k][j] = t;
          t = L[i][j];
          L[i][j] = L[k][j];
          L[k][j] = t;
        }
        const int t = perm[i];
        perm[i] = perm[k];
        perm[k] = t;
      }
    const double inv = fdiv(1.0, a[k][k]);
#pragma unroll
    for (int i = k + 1; i < NS; ++i) {
      const double m = fmul(a[i][k], inv);
      L[i][k] = m;
      if (m == 0.0) continue;
#pragma unroll
      for (int j = k; j < NS; ++j) a[i][j] = fmsc(a[i][j], m, a[k][j]);
    }
  }
  long long code = sing ? 256 : 0;
#pragma unroll
  for (int u = 0; u < NS; ++u) code |= (long long)perm[u] << (2 * u);
  int o = 0;
  c[o++] = __longlong_as_double(code);
#pragma unroll
  for (int i = 1; i < NS; ++i)
#pragma unroll
    for (int j = 0; j < i; ++j) c[o++] = L[i][j];
#pragma unroll
  for (int i = 0; i < NS; ++i)
#pragma unroll
    for (int j = i + 1; j < NS; ++j) c[o++] = a[i][j];
#pragma unroll
  for (int i = 0; i < NS; ++i) c[o + i] = a[i][i];
#pragma unroll
  for (int i = 0; i < NS; ++i) c[o + NS + i] = __drcp_rn(a[i][i]);
}

} // namespace tpdg_gpu
