// Per-element application of the approximate Kronecker inverse P^{-1}, P = A1 (x) B1 + A2 (x) B2
// (2D) or A1 (x) (B1 (x) C1 + B2 (x) C2) (3D), one CTA per block.
//
// Restates KsvdPC2D::apply / KsvdPC3D::apply (reference precond/ksvd.hpp:172-233) and
// apply_factors_2d / apply_factors_3d (:112-153): LU axis solves (ops/kernels.hpp:36-51,
// tensor/small_matrix.hpp:177-187), rotation to Schur coordinates (matmul, :103-113), the
// quasi-triangular Sylvester solve T1 Y + Y T2^T = M (tensor/sylvester.hpp:72-127), rotation back.
//
// "Faithful" arithmetic (faithful.cuh): no FMA, the reference's per-entry summation order, so
// given the same factors the result equals the reference's bit for bit. The parallelism is over
// independent entries (fibers, matrix entries, Sylvester cells on one anti-diagonal of the
// block wavefront), never inside one sum.
//
// Fallback blocks (kind == 0) are solved by kron_fallback_kernel with the exact block LU
// (LuFactor::solve_inplace, tensor/small_matrix.hpp:189-192), stored column-major so that the
// column sweeps read coalesced columns; its forward sweep keeps the reference order, the backward
// sweep runs column-descending (per-row order reversed; the block itself is well conditioned).
#include <cstdint>
#include <cstdlib>

#include "faithful.cuh"
#include "sylv_cell.cuh"
#include "mma.cuh"
#include "tma.cuh"
#include "tpdg_internal.hpp"

namespace tpdg_gpu {

namespace {

constexpr int kApplyThreads = 128;

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Quasi-triangular diagonal block structure (tensor/sylvester.hpp:16-30); returns block count.
__device__ int quasi_blocks_dev(const double* t, int n, int* start, int* size) {
  int i = 0, nb = 0;
  while (i < n) {
    if (i + 1 < n && t[(i + 1) * n + i] != 0.0) {
      start[nb] = i;
      size[nb++] = 2;
      i += 2;
    } else {
      start[nb] = i;
      size[nb++] = 1;
      ++i;
    }
  }
  return nb;
}

// solve_tiny<4> (tensor/sylvester.hpp:34-59); returns false on a singular pivot.
__device__ bool solve_tiny_dev(double a[4][4], double b[4], int n, double tol) {
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int i = k + 1; i < n; ++i)
      if (fabs(a[i][k]) > fabs(a[piv][k])) piv = i;
    if (fabs(a[piv][k]) < tol) return false;
    if (piv != k) {
      for (int j = 0; j < 4; ++j) {
        const double t = a[piv][j];
        a[piv][j] = a[k][j];
        a[k][j] = t;
      }
      const double t = b[piv];
      b[piv] = b[k];
      b[k] = t;
    }
    const double inv = fdiv(1.0, a[k][k]);
    for (int i = k + 1; i < n; ++i) {
      const double m = fmul(a[i][k], inv);
      if (m == 0.0) continue;
      for (int j = k; j < n; ++j) a[i][j] = fmsc(a[i][j], m, a[k][j]);
      b[i] = fmsc(b[i], m, b[k]);
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    for (int j = i + 1; j < n; ++j) b[i] = fmsc(b[i], a[i][j], b[j]);
    b[i] = fdiv(b[i], a[i][i]);
  }
  return true;
}

// In-place LU solve of one strided fiber (LuFactor::solve: x = b[perm], forward, backward).
__device__ void lu_solve_fiber(const double* lu, const int* perm, int n, double* x, int stride, double* tmp,
                               int tstride) {
  for (int k = 0; k < n; ++k) tmp[k * tstride] = x[perm[k] * stride];
  for (int r = 0; r < n; ++r) {
    double s = tmp[r * tstride];
    for (int j = 0; j < r; ++j) s = fmsc(s, lu[r * n + j], tmp[j * tstride]);
    tmp[r * tstride] = s;
  }
  for (int r = n - 1; r >= 0; --r) {
    double s = tmp[r * tstride];
    for (int j = r + 1; j < n; ++j) s = fmsc(s, lu[r * n + j], tmp[j * tstride]);
    tmp[r * tstride] = fdiv(s, lu[r * n + r]);
  }
  for (int k = 0; k < n; ++k) x[k * stride] = tmp[k * tstride];
}

// Shared state of the Sylvester wavefront for one (T1, T2) pair.
struct SylvPlan {
  int nb1, nb2;
  int *s1, *z1, *s2, *z2;
  double tol;
};

// Plan (block structure, pivot tolerance 1e-14 (||T1||_inf + ||T2||_inf)); thread-cooperative.
__device__ void sylv_plan(const double* t1, int n1, const double* t2, int n2, SylvPlan& P, double* rowsum) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < n1 + n2; i += nt) {
    const double* row = i < n1 ? t1 + i * n1 : t2 + (i - n1) * n2;
    const int n = i < n1 ? n1 : n2;
    double s = 0.0;
    for (int j = 0; j < n; ++j) s = fadd(s, fabs(row[j]));
    rowsum[i] = s;
  }
  __syncthreads();
  if (tid == 0) {
    double m1 = 0.0, m2 = 0.0;
    for (int i = 0; i < n1; ++i) m1 = fmax(m1, rowsum[i]);
    for (int i = 0; i < n2; ++i) m2 = fmax(m2, rowsum[n1 + i]);
    P.tol = fmul(1e-14, fmax(fadd(m1, m2), 1e-300));
    P.nb1 = quasi_blocks_dev(t1, n1, P.s1, P.z1);
    P.nb2 = quasi_blocks_dev(t2, n2, P.s2, P.z2);
  }
  __syncthreads();
}

// Solve T1 Y + Y T2^T = M for `nslices` independent slices (M, Y: [slice][n1][ld]) by the
// block anti-diagonal wavefront; each cell restates the reference's per-cell arithmetic.
__device__ void sylv_wavefront(const double* t1, int n1, const double* t2, int n2, const SylvPlan& P,
                               const double* M, double* Y, int ld, int slice_stride, int nslices, int* status) {
  const int nb1 = P.nb1, nb2 = P.nb2;
  for (int step = 0; step <= nb1 + nb2 - 2; ++step) {
    const int d1lo = step - (nb2 - 1) > 0 ? step - (nb2 - 1) : 0;
    const int d1hi = step < nb1 - 1 ? step : nb1 - 1;
    const int ncell = d1hi - d1lo + 1;
    for (int t = threadIdx.x; t < ncell * nslices; t += blockDim.x) {
      const int sl = t / ncell, d1 = d1lo + t % ncell, d2 = step - d1;
      const int bi = nb1 - 1 - d1, bj = nb2 - 1 - d2;
      const int i0 = P.s1[bi], isz = P.z1[bi], k0 = P.s2[bj], ksz = P.z2[bj];
      const double* Ms = M + sl * slice_stride;
      double* Ys = Y + sl * slice_stride;
      double mm[4][4], rhs[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        rhs[u] = 0.0;
#pragma unroll
        for (int v = 0; v < 4; ++v) mm[u][v] = 0.0;
      }
      for (int a = 0; a < isz; ++a)
        for (int kb = 0; kb < ksz; ++kb) {
          // R rows: B minus coupling to solved rows below (sylvester.hpp:84-90) ...
          double s = Ms[(i0 + a) * ld + k0 + kb];
          for (int j = i0 + isz; j < n1; ++j) s = fmsc(s, t1[(i0 + a) * n1 + j], Ys[j * ld + k0 + kb]);
          // ... then the solved columns to the right (sylvester.hpp:93-99)
          for (int l = k0 + ksz; l < n2; ++l) s = fmsc(s, t2[(k0 + kb) * n2 + l], Ys[(i0 + a) * ld + l]);
          const int row = a * ksz + kb;
          rhs[row] = s;
          for (int a2 = 0; a2 < isz; ++a2)
            for (int kb2 = 0; kb2 < ksz; ++kb2) {
              double coef = 0.0;
              if (kb == kb2) coef = fadd(coef, t1[(i0 + a) * n1 + i0 + a2]);
              if (a == a2) coef = fadd(coef, t2[(k0 + kb) * n2 + k0 + kb2]);
              mm[row][a2 * ksz + kb2] = coef;
            }
        }
      if (!solve_tiny_dev(mm, rhs, isz * ksz, P.tol)) atomicExch(status, int(TPDG_SINGULAR));
      for (int a = 0; a < isz; ++a)
        for (int kb = 0; kb < ksz; ++kb) Ys[(i0 + a) * ld + k0 + kb] = rhs[a * ksz + kb];
    }
    __syncthreads();
  }
}

// C[i][j] = sum_k A(i,k) B(k,j) for `nslices` slices, generic strides, k ascending (matmul).
// a_t: A(i,k) = a[k*lda + i] (transposed access); b_t likewise for B.
__device__ void mm_slices(int r, int kk, int c, const double* a, int lda, bool a_t, int a_slice, const double* b,
                          int ldb, bool b_t, int b_slice, double* out, int ldo, int o_slice, int nslices) {
  const int per = r * c;
  for (int t = threadIdx.x; t < per * nslices; t += blockDim.x) {
    const int sl = t / per, i = (t % per) / c, j = t % c;
    const double* as = a + sl * a_slice;
    const double* bs = b + sl * b_slice;
    double s = 0.0;
    for (int k = 0; k < kk; ++k) {
      const double av = a_t ? as[k * lda + i] : as[i * lda + k];
      const double bv = b_t ? bs[j * ldb + k] : bs[k * ldb + j];
      s = fmac(s, av, bv);
    }
    out[sl * o_slice + i * ldo + j] = s;
  }
}

// ------------------------------------------------------------------------------------ 2D
__global__ void __launch_bounds__(kApplyThreads) kron2d_apply_kernel(DevPC pc, const double* __restrict__ in,
                                                                      double* __restrict__ out) {
  const int blk = blockIdx.x;
  if (pc.kind[blk] == 0 || (pc.skip && *pc.skip)) return;
  extern __shared__ double sm[];
  const int n1 = pc.n1, n2 = pc.q, ld = n2 | 1;
  double* sX = sm;
  double* sT = sX + n1 * ld;
  double* sR = sT + n1 * ld;
  double* rowsum = sR + pc.rec_len;
  int* sPiv = reinterpret_cast<int*>(rowsum + n1 + n2);
  int* sb = sPiv + pc.piv_len;
  __shared__ SylvPlan P;
  const int tid = threadIdx.x, nt = blockDim.x;
  const double* rec = pc.rec + size_t(blk) * pc.rec_len;
  for (int i = tid; i < pc.rec_len; i += nt) sR[i] = rec[i];
  for (int i = tid; i < pc.piv_len; i += nt) sPiv[i] = pc.piv[size_t(blk) * pc.piv_len + i];
  const double* x = in + size_t(blk) * pc.blk_len;
  for (int i = tid; i < n1 * n2; i += nt) sX[(i / n2) * ld + i % n2] = x[i];
  if (tid == 0) {
    P.s1 = sb;
    P.z1 = sb + n1;
    P.s2 = sb + 2 * n1;
    P.z2 = sb + 2 * n1 + n2;
  }
  __syncthreads();
  const double* luA2 = sR;
  const double* luB1 = luA2 + n1 * n1;
  const double* Q1 = luB1 + n2 * n2;
  const double* T1 = Q1 + n1 * n1;
  const double* Q2 = T1 + n1 * n1;
  const double* T2 = Q2 + n2 * n2;
  // (A2^{-1} (x) I): fibers along the outer axis (one per inner column i)
  for (int i = tid; i < n2; i += nt) lu_solve_fiber(luA2, sPiv, n1, sX + i, ld, sT + i, ld);
  __syncthreads();
  // (I (x) B1^{-1}): rows
  for (int o = tid; o < n1; o += nt) lu_solve_fiber(luB1, sPiv + n1, n2, sX + o * ld, 1, sT + o * ld, 1);
  __syncthreads();
  // M = (Q1^T X) Q2
  mm_slices(n1, n1, n2, Q1, n1, true, 0, sX, ld, false, 0, sT, ld, 0, 1);
  sylv_plan(T1, n1, T2, n2, P, rowsum);  // contains __syncthreads
  mm_slices(n1, n2, n2, sT, ld, false, 0, Q2, n2, false, 0, sX, ld, 0, 1);
  __syncthreads();
  // Y: T1 Y + Y T2^T = M
  sylv_wavefront(T1, n1, T2, n2, P, sX, sT, ld, 0, 1, pc.status);
  // back = (Q1 Y) Q2^T
  mm_slices(n1, n1, n2, Q1, n1, false, 0, sT, ld, false, 0, sX, ld, 0, 1);
  __syncthreads();
  double* o = out + size_t(blk) * pc.blk_len;
  mm_slices(n1, n2, n2, sX, ld, false, 0, Q2, n2, true, 0, o, n2, 0, 1);
}

size_t kron2d_smem(const DevPC& pc) {
  const int n1 = pc.n1, n2 = pc.q, ld = n2 | 1;
  return sizeof(double) * size_t(2 * n1 * ld + pc.rec_len + n1 + n2) +
         sizeof(int) * size_t(pc.piv_len + 2 * n1 + 2 * n2) + 16;
}

// ------------------------------------------------------------------------------------ 2D, sized
// Latency-oriented variant for compile-time (N1, N2): the element's work is a chain of
// dependent fp64 operations (LU substitutions with divisions, the Sylvester wavefront), so the
// kernel minimizes the chain: fibers live in registers with fully unrolled substitutions, the
// Sylvester cells are specialized on their block shape (1x1 / 1x2 / 2x1 / 2x2) with the tiny
// pivoted solve unrolled in registers, and the wavefront runs in one warp (__syncwarp per step).
// 64 threads per element keep many elements resident per SM. Same arithmetic as above.
constexpr int kSizedThreads = 64;


template <int N>
__device__ __forceinline__ void lu_fiber_reg(const double* __restrict__ lu, const double* __restrict__ rcp,
                                             const int* __restrict__ perm, double* col, int stride) {
  double x[N];
#pragma unroll
  for (int k = 0; k < N; ++k) x[k] = col[perm[k] * stride];
#pragma unroll
  for (int r = 1; r < N; ++r) {
    double s = x[r];
#pragma unroll
    for (int j = 0; j < r; ++j) s = fmsc(s, lu[r * N + j], x[j]);
    x[r] = s;
  }
#pragma unroll
  for (int r = N - 1; r >= 0; --r) {
    double s = x[r];
#pragma unroll
    for (int j = r + 1; j < N; ++j) s = fmsc(s, lu[r * N + j], x[j]);
    x[r] = fdiv_rcp(s, lu[r * N + r], rcp[r]);
  }
#pragma unroll
  for (int k = 0; k < N; ++k) col[k * stride] = x[k];
}

// Same solve for long fibers (N > 32) whose LU stays in global memory (lu_g): the NF fibers
// (columns c < NF of X, one per lane) are permuted into a shared scratch column (tmp) and solved
// there, and the LU rows stream through a D-deep shared ring (cp.async, issued D - 1 rows ahead)
// so that every row is read from L2 once and broadcast from shared memory to the chains.
template <int N, int NF>
__device__ __forceinline__ void lu_cols_ring(const double* __restrict__ lu_g, const double* __restrict__ rcp,
                                             const int* __restrict__ perm, double* X, int ld, double* tmp,
                                             double* ring, int lane) {
  constexpr int D = 4;
  static_assert(NF <= 32 && N % 2 == 0, "one fiber per lane, 16-byte row copies");
  auto issue = [&](int r) {
    for (int i = 2 * lane; i < N; i += 64) cp_async16(ring + (r % D) * N + i, lu_g + size_t(r) * N + i);
  };
  const bool act = lane < NF;
  const int c = lane;
  if (act)
#pragma unroll 1
    for (int k = 0; k < N; ++k) tmp[k * ld + c] = X[perm[k] * ld + c];
  // forward (unit lower, j ascending), rows 1 .. N-1
#pragma unroll
  for (int u = 1; u < D; ++u) {
    if (u < N) issue(u);
    cp_async_commit();
  }
#pragma unroll 1
  for (int r = 1; r < N; ++r) {
    if (r + D - 1 < N) issue(r + D - 1);
    cp_async_commit();
    cp_async_wait_group<D - 1>();
    __syncwarp();
    if (act) {
      const double* L = ring + (r % D) * N;
      double s = tmp[r * ld + c];
#pragma unroll 8
      for (int j = 0; j < r; ++j) s = fmsc(s, L[j], tmp[j * ld + c]);
      tmp[r * ld + c] = s;
    }
    __syncwarp();
  }
  // backward (j ascending after the diagonal), rows N-1 .. 0
#pragma unroll
  for (int u = 0; u < D - 1; ++u) {
    if (N - 1 - u >= 0) issue(N - 1 - u);
    cp_async_commit();
  }
#pragma unroll 1
  for (int r = N - 1; r >= 0; --r) {
    if (r - (D - 1) >= 0) issue(r - (D - 1));
    cp_async_commit();
    cp_async_wait_group<D - 1>();
    __syncwarp();
    if (act) {
      const double* U = ring + (r % D) * N;
      double s = tmp[r * ld + c];
#pragma unroll 8
      for (int j = r + 1; j < N; ++j) s = fmsc(s, U[j], tmp[j * ld + c]);
      tmp[r * ld + c] = fdiv_rcp(s, U[r], rcp[r]);
    }
    __syncwarp();
  }
  if (act)
#pragma unroll 1
    for (int k = 0; k < N; ++k) X[k * ld + c] = tmp[k * ld + c];
  __syncwarp();
}

// Warp-level tiled product O = op(A) op(B) (R x K x C), lane tile TI x TJ; each output still
// accumulates k ascending from +0.0 with separate mul / add roundings (faithful).
template <int R, int K, int C, bool AT, bool BT, int TI, int TJ>
__device__ __forceinline__ void warp_mm(const double* A, int lda, const double* B, int ldb, double* O, int ldo,
                                        int lane) {
  constexpr int NTI = (R + TI - 1) / TI, NTJ = (C + TJ - 1) / TJ;
  for (int t = lane; t < NTI * NTJ; t += 32) {
    const int i0 = (t / NTJ) * TI, j0 = (t % NTJ) * TJ;
    double acc[TI][TJ];
#pragma unroll
    for (int ii = 0; ii < TI; ++ii)
#pragma unroll
      for (int jj = 0; jj < TJ; ++jj) acc[ii][jj] = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double a[TI], b[TJ];
#pragma unroll
      for (int ii = 0; ii < TI; ++ii) {
        const int i = i0 + ii < R ? i0 + ii : R - 1;
        a[ii] = AT ? A[k * lda + i] : A[i * lda + k];
      }
#pragma unroll
      for (int jj = 0; jj < TJ; ++jj) {
        const int j = j0 + jj < C ? j0 + jj : C - 1;
        b[jj] = BT ? B[j * ldb + k] : B[k * ldb + j];
      }
#pragma unroll
      for (int ii = 0; ii < TI; ++ii)
#pragma unroll
        for (int jj = 0; jj < TJ; ++jj) acc[ii][jj] = fmac(acc[ii][jj], a[ii], b[jj]);
    }
#pragma unroll
    for (int ii = 0; ii < TI; ++ii)
#pragma unroll
      for (int jj = 0; jj < TJ; ++jj)
        if (i0 + ii < R && j0 + jj < C) O[(i0 + ii) * ldo + j0 + jj] = acc[ii][jj];
  }
}

// Right-hand side of one Sylvester entry: B minus the solved rows below (j ascending), then the
// solved columns to the right (l ascending), exactly sylvester.hpp:84-99.
__device__ __forceinline__ double sylv_rhs(const double* __restrict__ t1, int n1, const double* __restrict__ t2,
                                           int n2, const double* M, const double* Y, int ld, int i, int k,
                                           int jfirst, int lfirst) {
  double s = M[i * ld + k];
  // one loop over both segments: the lanes of a wavefront step then share one trip count
  const int nj = n1 - jfirst, nt = nj + n2 - lfirst;
  const double* a1 = t1 + i * n1 + jfirst;
  const double* b1 = Y + jfirst * ld + k;
  const double* a2 = t2 + k * n2 + lfirst - nj;
  const double* b2 = Y + i * ld + lfirst - nj;
#pragma unroll 4
  for (int t = 0; t < nt; ++t) {
    const bool first = t < nj;
    const double* pa = first ? a1 + t : a2 + t;
    const double* pb = first ? b1 + t * ld : b2 + t;
    s = fmsc(s, *pa, *pb);
  }
  return s;
}

// Sylvester cell factors: factor_cell (sylv_cell.cuh).

// Replays a factored cell on the permuted right-hand side b (b[u] = r[perm[u]]); returns entry e.
template <int NS>
__device__ __forceinline__ double cell_solve(const double (&cf)[22], double (&b)[4], int e) {
  constexpr int NL = NS * (NS - 1) / 2;
  int o = 1;
#pragma unroll
  for (int i = 1; i < NS; ++i)
#pragma unroll
    for (int j = 0; j < i; ++j) {
      const double m = cf[o++];
      b[i] = m != 0.0 ? fmsc(b[i], m, b[j]) : b[i];
    }
#pragma unroll
  for (int i = NS - 1; i >= 0; --i) {
    int u = 1 + NL;
#pragma unroll
    for (int r = 0; r < i; ++r) u += NS - 1 - r;
#pragma unroll
    for (int j = i + 1; j < NS; ++j) b[i] = fmsc(b[i], cf[u + j - i - 1], b[j]);
    b[i] = fdiv_rcp(b[i], cf[1 + 2 * NL + i], cf[1 + 2 * NL + NS + i]);
  }
  double y = b[0];
#pragma unroll
  for (int t = 1; t < NS; ++t)
    if (e == t) y = b[t];
  return y;
}

// One warp per Kronecker block: lane 0 builds the plan (tol from the row sums, quasi-blocks),
// the lanes factor the cells.
__global__ void sylv_cells_kernel(DevPC pc, double* __restrict__ cells) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= pc.nblk || pc.kind[warp] == 0) return;
  const int t1n = pc.dim == 2 ? pc.n1 : pc.q, t2n = pc.q;
  const double* r = pc.rec + size_t(warp) * pc.rec_len;
  const double* t1 = pc.dim == 2 ? r + 2 * pc.n1 * pc.n1 + pc.q * pc.q : r + pc.n1 * pc.n1 + 3 * pc.q * pc.q;
  const double* t2 = t1 + t1n * t1n + pc.q * pc.q;  // T1, Q2, T2 (rec layout of make_factors)
  double* c = cells + size_t(warp) * pc.cells_len;
  int* h = reinterpret_cast<int*>(c);
  if (lane == 0) {
    double m1 = 0.0, m2 = 0.0;
    for (int i = 0; i < t1n; ++i) {
      double s = 0.0;
      for (int j = 0; j < t1n; ++j) s = fadd(s, fabs(t1[i * t1n + j]));
      m1 = fmax(m1, s);
    }
    for (int i = 0; i < t2n; ++i) {
      double s = 0.0;
      for (int j = 0; j < t2n; ++j) s = fadd(s, fabs(t2[i * t2n + j]));
      m2 = fmax(m2, s);
    }
    const int nb1 = quasi_blocks_dev(t1, t1n, h + 4, h + 4 + t1n);
    const int nb2 = quasi_blocks_dev(t2, t2n, h + 4 + 2 * t1n, h + 4 + 2 * t1n + t2n);
    h[0] = nb1;
    h[1] = nb2;
    h[2] = (nb1 == t1n && nb2 == t2n) ? 1 : 0;
    h[3] = 0;
    reinterpret_cast<double*>(h)[sylv_hdr_doubles(t1n, t2n) - 1] = fmul(1e-14, fmax(fadd(m1, m2), 1e-300));
  }
  __syncwarp();
  const int nb1 = h[0], nb2 = h[1];
  const int *s1 = h + 4, *z1 = s1 + t1n, *s2 = z1 + t1n, *z2 = s2 + t2n;
  const double tol = c[sylv_hdr_doubles(t1n, t2n) - 1];
  double* cc = c + sylv_hdr_doubles(t1n, t2n);
  for (int cell = lane; cell < nb1 * nb2; cell += 32) {
    const int bi = cell / nb2, bk = cell % nb2;
    const int i0 = s1[bi], isz = z1[bi], k0 = s2[bk], ksz = z2[bk];
    double* slot = cc + 6 * (i0 * t2n + isz * k0);
    const int code = (isz - 1) * 2 + (ksz - 1);
    if (code == 0) factor_cell<1, 1>(t1, t1n, t2, t2n, i0, k0, tol, slot);
    else if (code == 1) factor_cell<1, 2>(t1, t1n, t2, t2n, i0, k0, tol, slot);
    else if (code == 2) factor_cell<2, 1>(t1, t1n, t2, t2n, i0, k0, tol, slot);
    else factor_cell<2, 2>(t1, t1n, t2, t2n, i0, k0, tol, slot);
    const long long cw = __double_as_longlong(slot[0]);
    if (cw & 256) atomicOr(h + 3, 1);
  }
}


// Block anti-diagonal wavefront of the quasi-triangular Sylvester solve over NSL slices that
// share one plan (2D: 1, 3D: the outer slices). Work items are (step, pass) pairs, each pass a
// set of NT/4 (cell, slice) groups of 4 lanes (lane e of a group = entry e of the cell); a
// barrier separates the steps. (Loading the next item's factors one item ahead was measured
// slower: the extra registers cost more occupancy than the hidden latency gained.)
template <int TN1, int TN2, int NSL, int NT, bool CTA>
__device__ __forceinline__ void sylv_wavefront(const double* T1, const double* T2, double* X, int ld, int ss,
                                               const double* __restrict__ cc, const int* sb, int tid, int* status) {
  // cc = the replay slots of the factored cells (sylv_cells_kernel).
  const int nb1 = sb[0], nb2 = sb[1];
  const int *s1 = sb + 4, *z1 = s1 + TN1, *s2 = z1 + TN1, *z2 = s2 + TN2;
  const int last = nb1 + nb2 - 2, lane = tid & 31, e = lane & 3, g = lane & ~3;
  constexpr int NCF = 22;
  struct Item {
    int bi, bj, sl;
    bool ok;
  };
  auto locate = [&](int st, int bs) {
    Item it;
    const int d1lo = st - (nb2 - 1) > 0 ? st - (nb2 - 1) : 0;
    const int d1hi = st < nb1 - 1 ? st : nb1 - 1;
    const int ncell = d1hi - d1lo + 1;
    const int grp = (bs + tid) >> 2;
    it.ok = grp < ncell * NSL;
    const int cell = !it.ok ? 0 : NSL == 1 ? grp : grp % ncell;
    it.sl = !it.ok || NSL == 1 ? 0 : grp / ncell;
    const int d1 = d1lo + cell;
    it.bi = nb1 - 1 - d1;
    it.bj = nb2 - 1 - (st - d1);
    return it;
  };
  auto load = [&](const Item& it, double (&c)[NCF]) {
#pragma unroll
    for (int u = 0; u < NCF; ++u) c[u] = 0.0;
    if (!it.ok) return;
    const int i0 = s1[it.bi], isz = z1[it.bi], k0 = s2[it.bj], ksz = z2[it.bj];
    {
      const double2* p = reinterpret_cast<const double2*>(cc + 6 * (i0 * TN2 + isz * k0));
#pragma unroll
      for (int u = 0; u < NCF / 2; ++u) {
        const double2 v = __ldg(p + u);
        c[2 * u] = v.x;
        c[2 * u + 1] = v.y;
      }
    }
  };
  int step = 0, base = 0;
  Item cur = locate(0, 0);
  double cf[NCF];
  load(cur, cf);
  while (step <= last) {
    // next work item: the next pass of this step, else the first pass of the next step
    int nstep = step, nbase = base + NT;
    {
      const int d1lo = step - (nb2 - 1) > 0 ? step - (nb2 - 1) : 0;
      const int d1hi = step < nb1 - 1 ? step : nb1 - 1;
      if (nbase >= (d1hi - d1lo + 1) * NSL * 4) {
        ++nstep;
        nbase = 0;
      }
    }
    const Item nxt = locate(nstep, nbase);
    double cn[NCF];
    double* Ms = X + cur.sl * ss;
    int i0 = 0, k0 = 0, isz = 1, ksz = 1;
    double s = 0.0;
    if (cur.ok) {
      i0 = s1[cur.bi];
      isz = z1[cur.bi];
      k0 = s2[cur.bj];
      ksz = z2[cur.bj];
      if (e < isz * ksz)
        s = sylv_rhs(T1, TN1, T2, TN2, Ms, Ms, ld, i0 + (ksz == 2 ? e >> 1 : e), k0 + (ksz == 2 ? e & 1 : 0),
                          i0 + isz, k0 + ksz);
    }
    const int ns = isz * ksz;
    double y = 0.0;
    {
      const long long code = __double_as_longlong(cf[0]);
      double b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = __shfl_sync(0xffffffffu, s, g + int((code >> (2 * u)) & 3));
      if (cur.ok && e < ns) {
        if (code & 256) atomicExch(status, int(TPDG_SINGULAR));
        y = ns == 1 ? cell_solve<1>(cf, b, e) : ns == 2 ? cell_solve<2>(cf, b, e) : cell_solve<4>(cf, b, e);
      }
    }
    if (cur.ok && e < ns) Ms[(i0 + (ksz == 2 ? e >> 1 : e)) * ld + k0 + (ksz == 2 ? e & 1 : 0)] = y;
    if (nstep != step) {
      if (CTA) __syncthreads();
      else __syncwarp();
    }
    if (nstep <= last) load(nxt, cn);
#pragma unroll
    for (int u = 0; u < NCF; ++u) cf[u] = cn[u];
    cur = nxt;
    step = nstep;
    base = nbase;
  }
}

// Faithful quasi-triangular Sylvester solve (sylvester.hpp:72-127) of one block by one warp, in
// place on X (ld), for a T1 that stays in global memory (kron2d_sized_kernel<.., GREC>): the block
// anti-diagonal wavefront with one lane per Sylvester entry, and the rows of T1 the current step
// reads held in a window of R rows in shared memory (win, slot = row % R). The steps move down T1
// (the active block rows at step st are the ones below nb1 - 1 - st, at most nb2 blocks), so the
// rows entering at step st + 1 are prefetched with cp.async while step st runs; a step whose rows
// do not fit in the window reads T1 from global memory. Cells of a step are processed in groups
// of gs lanes (gs = the largest cell of the block: 1, 2 or 4), so 32 / gs cells per pass. Each lane
// forms its entry's right-hand side in the reference order (B, then the solved rows below j
// ascending, then the solved columns to the right l ascending, separate mul / sub roundings); the
// gs lanes of a cell exchange their right-hand sides with shuffles and each replays the cell's
// factored tiny system (sylv_cells_kernel). 1 x 1 cells divide by t1_ii + t2_kk (solve_tiny<1>).
template <int N1, int N2, int R>
__device__ __forceinline__ void sylv_window(const double* __restrict__ T1g, const double* __restrict__ T2, double* X,
                                            int ld, const int* sb, const double* __restrict__ cc, double* win,
                                            int lane, int* status) {
  static_assert(N1 % 2 == 0, "16-byte row copies");
  const int nb1 = sb[0], nb2 = sb[1];
  const int *s1 = sb + 4, *z1 = s1 + N1, *s2 = z1 + N1, *z2 = s2 + N2;
  if (sb[3] && lane == 0) atomicExch(status, int(TPDG_SINGULAR));
  const int lg = (nb1 < N1 ? 1 : 0) + (nb2 < N2 ? 1 : 0);  // log2 of the group size
  const int gs = 1 << lg, per = 32 >> lg;
  const int g = lane >> lg, e = lane & (gs - 1), gbase = g << lg;
  const int last = nb1 + nb2 - 2;
  // rows of T1 read at step st: the block rows d1 in [d1lo, d1hi] (bi = nb1 - 1 - d1)
  auto rows = [&](int st, int& lo, int& hi) {
    const int d1lo = st - (nb2 - 1) > 0 ? st - (nb2 - 1) : 0;
    const int d1hi = st < nb1 - 1 ? st : nb1 - 1;
    lo = s1[nb1 - 1 - d1hi];
    hi = s1[nb1 - 1 - d1lo] + z1[nb1 - 1 - d1lo] - 1;
  };
  auto load_rows = [&](int a, int b) {  // rows a..b into their slots (cp.async, this lane's share)
    for (int r = a; r <= b; ++r)
      for (int i = 2 * lane; i < N1; i += 64) cp_async16(win + (r % R) * N1 + i, T1g + size_t(r) * N1 + i);
  };
  int res_lo = 0, res_hi = -1;  // resident rows (empty)
  auto ensure = [&](int st) {  // make the rows of step st resident, synchronously; false if they do not fit
    int lo, hi;
    rows(st, lo, hi);
    if (hi - lo + 1 > R) {
      res_lo = 0;
      res_hi = -1;
      return;
    }
    if (res_hi < res_lo || hi < res_lo || lo > res_hi) load_rows(lo, hi);
    else if (lo < res_lo) load_rows(lo, res_lo - 1);
    cp_async_commit();
    cp_async_wait_group<0>();
    __syncwarp();
    res_lo = lo;
    res_hi = hi;
  };
  ensure(0);
  for (int st = 0; st <= last; ++st) {
    int lo, hi;
    rows(st, lo, hi);
    const bool inwin = res_hi >= res_lo && lo >= res_lo && hi <= res_hi;
    if (st < last && inwin) {  // prefetch the rows entering at st + 1 if their slots are free now
      int lo1, hi1;
      rows(st + 1, lo1, hi1);
      if (hi - lo1 + 1 <= R && lo1 < res_lo) {
        load_rows(lo1, res_lo - 1);
        res_lo = lo1;
      }
      cp_async_commit();
    }
    const int d1lo = st - (nb2 - 1) > 0 ? st - (nb2 - 1) : 0;
    const int d1hi = st < nb1 - 1 ? st : nb1 - 1;
    const int ncell = d1hi - d1lo + 1;
    for (int c0 = 0; c0 < ncell; c0 += per) {
      const int cell = c0 + g;
      const bool ok = cell < ncell;
      int i0 = 0, isz = 1, k0 = 0, ksz = 1;
      if (ok) {
        const int d1 = d1lo + cell, bi = nb1 - 1 - d1, bk = nb2 - 1 - (st - d1);
        i0 = s1[bi];
        isz = z1[bi];
        k0 = s2[bk];
        ksz = z2[bk];
      }
      const int ns = isz * ksz;
      const bool act = ok && e < ns;
      const int i = i0 + (ksz == 2 ? e >> 1 : e), k = k0 + (ksz == 2 ? e & 1 : 0);
      const double* t1r = inwin ? win + (i % R) * N1 : T1g + size_t(i) * N1;  // row i of T1
      // the cell's factored system (ns > 1), loaded ahead of the chains
      double cf[22];
      cf[0] = 0.0;
      if (ns > 1) {
        const double* slot = cc + 6 * (i0 * N2 + isz * k0);
        const int ncf = ns == 2 ? 7 : 21;
#pragma unroll
        for (int u = 0; u < 21; ++u) cf[u] = (ok && u < ncf) ? __ldg(slot + u) : 0.0;
      }
      double s = 0.0, diag = 0.0;
      if (act) {
        s = X[i * ld + k];
        diag = ns == 1 ? fadd(t1r[i0], T2[k0 * N2 + k0]) : 0.0;
        const int jf = i0 + isz, lf = k0 + ksz;
        const double* py = X + jf * ld + k;
#pragma unroll 4
        for (int t = 0; t < N1 - jf; ++t) s = fmsc(s, t1r[jf + t], py[t * ld]);
        const double* pt = T2 + k * N2 + lf;
        py = X + i * ld + lf;
#pragma unroll 4
        for (int t = 0; t < N2 - lf; ++t) s = fmsc(s, pt[t], py[t]);
      }
      double y = 0.0;
      if (lg == 0) {
        if (act) y = fdiv(s, diag);
      } else {
        const long long code = __double_as_longlong(cf[0]);
        double b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int src = ns > 1 ? int((code >> (2 * u)) & 3) : u;
          b[u] = __shfl_sync(0xffffffffu, s, gbase + (src & (gs - 1)));
        }
        if (act) {
          if (ns == 1) y = fdiv(s, diag);
          else if (ns == 2) y = cell_solve<2>(cf, b, e);
          else y = cell_solve<4>(cf, b, e);
        }
      }
      if (act) X[i * ld + k] = y;
    }
    if (st < last) {
      if (inwin) cp_async_wait_group<0>();
      __syncwarp();
      ensure(st + 1);
    } else {
      __syncwarp();
    }
  }
}

// One warp per element: every phase is warp-synchronous (no CTA barriers), so several elements
// proceed independently on an SM and their dependency chains overlap.
template <int N1, int N2>
struct Kron2dWarpLayout {
  static constexpr int ld = N2 | 1;  // odd: row fibers and column accesses are conflict-free
  static constexpr int xsz = (N1 * ld + 1) & ~1;
  static constexpr int rec = 3 * N1 * N1 + 3 * N2 * N2;
  static constexpr int hdr = (((4 + 2 * N1 + 2 * N2) / 2 + 2) & ~1);
  static constexpr int ints = N1 + N2;
  static constexpr int per = xsz + rec + ((N1 + N2 + 1) & ~1) + hdr + (ints + 1) / 2;
  static constexpr int per_even = (per + 1) & ~1;
  // GREC: the record stays in global memory (read through L1) and only X, the product scratch,
  // the reciprocals and the plan live in shared memory (large N1: cfg3's n_c q = 64 record is 104 KB)
  static constexpr int per_g = 2 * xsz + 4 * N1 + 3 * N2 * N2 + ((N1 + N2 + 1) & ~1) + hdr + (ints + 1) / 2;
  static constexpr int per_g_even = (per_g + 1) & ~1;
};

template <int N1, int N2, bool GREC = false>
__global__ void __launch_bounds__(kSizedThreads) kron2d_sized_kernel(DevPC pc, const double* __restrict__ in,
                                                                      double* __restrict__ out) {
  using L = Kron2dWarpLayout<N1, N2>;
  static_assert(GREC || N1 <= 32, "register fibers");
  static_assert(!GREC || N2 <= 32, "lu_cols_ring: one column fiber per lane");
  constexpr int ld = L::ld, rec = L::rec, hdr = L::hdr;
  extern __shared__ double sm_all[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int blk = blockIdx.x * (kSizedThreads / 32) + warp;
  if (blk >= pc.nblk || pc.kind[blk] == 0 || (pc.skip && *pc.skip)) return;
  double* sX = sm_all + size_t(warp) * (GREC ? L::per_g_even : L::per_even);
  const double* gR = pc.rec + size_t(blk) * rec;
  double* sR = sX + L::xsz;
  double* sT = sR;  // product scratch: aliases LU(A2), LU(B1) once both fiber solves are done
  double* sSmall = sR + L::xsz;  // GREC: LU(B1), Q2, T2 (3 N2^2) staged in shared memory
  double* sRing = sSmall + 3 * N2 * N2;  // GREC: 4-row ring of LU(A2)
  double* sRcp = sR + (GREC ? L::xsz + 3 * N2 * N2 + 4 * N1 : rec);
  double* sH = sRcp + ((N1 + N2 + 1) & ~1);  // Sylvester plan header (ints)
  int* sPiv = reinterpret_cast<int*>(sH + hdr);
  const double* cells = pc.cells + size_t(blk) * pc.cells_len;
  {  // asynchronous global -> shared copies (LDGSTS), one round trip for the whole record
    const double* r = gR;
    if (GREC) {
      for (int i = lane; i < N2 * N2; i += 32) cp_async8(sSmall + i, r + N1 * N1 + i);
      for (int i = lane; i < 2 * N2 * N2; i += 32) cp_async8(sSmall + N2 * N2 + i, r + 3 * N1 * N1 + N2 * N2 + i);
    } else if ((reinterpret_cast<uintptr_t>(r) & 15) == 0) {
      for (int i = 2 * lane; i + 1 < rec; i += 64) cp_async16(sR + i, r + i);
      if ((rec & 1) && lane == 0) sR[rec - 1] = r[rec - 1];
    } else {
      for (int i = lane; i < rec; i += 32) cp_async8(sR + i, r + i);
    }
    for (int i = 2 * lane; i < hdr; i += 64) cp_async16(sH + i, cells + i);
    for (int i = lane; i < N1 + N2; i += 32) sPiv[i] = pc.piv[size_t(blk) * (N1 + N2) + i];
    const double* x = in + size_t(blk) * (N1 * N2);
    for (int i = lane; i < N1 * N2; i += 32) cp_async8(sX + (i / N2) * ld + i % N2, x + i);
    cp_async_wait_all();
  }
  __syncwarp();
  const double* luA2 = GREC ? gR : sR;
  const double* luB1 = GREC ? sSmall : luA2 + N1 * N1;
  const double* Q1 = luA2 + N1 * N1 + N2 * N2;
  const double* T1 = Q1 + N1 * N1;
  const double* Q2 = GREC ? sSmall + N2 * N2 : T1 + N1 * N1;
  const double* T2 = Q2 + N2 * N2;
  for (int i = lane; i < N1 + N2; i += 32)
    sRcp[i] = __drcp_rn(i < N1 ? luA2[i * N1 + i] : luB1[(i - N1) * N2 + i - N1]);
  __syncwarp();
  // (A2^{-1} (x) I): one column fiber per lane
  if constexpr (GREC) {
    lu_cols_ring<N1, N2>(luA2, sRcp, sPiv, sX, ld, sT, sRing, lane);
  } else {
    for (int c = lane; c < N2; c += 32) lu_fiber_reg<N1>(luA2, sRcp, sPiv, sX + c, ld);
  }
  __syncwarp();
  // (I (x) B1^{-1}): one row fiber per lane
  for (int r = lane; r < N1; r += 32) lu_fiber_reg<N2>(luB1, sRcp + N1, sPiv + N1, sX + r * ld, 1);
  __syncwarp();
  warp_mm<N1, N1, N2, true, false, 2, 4>(Q1, N1, sX, ld, sT, ld, lane);  // Q1^T X
  __syncwarp();
  warp_mm<N1, N2, N2, false, false, 2, 4>(sT, ld, Q2, N2, sX, ld, lane);  // (.) Q2 -> M
  __syncwarp();
  {  // Y overwrites M in place (sX): T1 Y + Y T2^T = M, block anti-diagonal wavefront
    const int* sb = reinterpret_cast<const int*>(sH);
    const double* cc = cells + hdr;
    if constexpr (GREC) {  // T1 rows through a shared window in the (free) product scratch
      sylv_window<N1, N2, ld>(T1, T2, sX, ld, sb, cc, sT, lane, pc.status);
    } else if (sb[2]) {  // 1 x 1 blocks: one lane per cell; solve_tiny<1> is y = r / (t1_ii + t2_kk)
      const int nb1 = sb[0], nb2 = sb[1];
      for (int step = 0; step <= nb1 + nb2 - 2; ++step) {
        const int d1lo = step - (nb2 - 1) > 0 ? step - (nb2 - 1) : 0;
        const int d1hi = step < nb1 - 1 ? step : nb1 - 1;
        for (int d1 = d1lo + lane; d1 <= d1hi; d1 += 32) {
          const int i = nb1 - 1 - d1, k = nb2 - 1 - (step - d1);
          const double* c = cc + 6 * (i * N2 + k);
          const double code = __ldg(c), coef = __ldg(c + 1), rcp = __ldg(c + 2);
          const double s = sylv_rhs(T1, N1, T2, N2, sX, sX, ld, i, k, i + 1, k + 1);
          if (__double_as_longlong(code) & 256) atomicExch(pc.status, int(TPDG_SINGULAR));
          sX[i * ld + k] = fdiv_rcp(s, coef, rcp);
        }
        __syncwarp();
      }
    } else {  // 4 lanes per cell (one per entry), the cell's factored tiny system replayed in the group
      sylv_wavefront<N1, N2, 1, 32, false>(T1, T2, sX, ld, 0, cc, sb, lane, pc.status);
      __syncwarp();
    }
  }
  warp_mm<N1, N1, N2, false, false, 2, 4>(Q1, N1, sX, ld, sT, ld, lane);  // Q1 Y
  __syncwarp();
  warp_mm<N1, N2, N2, false, true, 2, 4>(sT, ld, Q2, N2, out + size_t(blk) * (N1 * N2), N2, lane);  // (.) Q2^T
}

template <int N1, int N2, bool GREC = false>
size_t kron2d_sized_smem() {
  using L = Kron2dWarpLayout<N1, N2>;
  return sizeof(double) * size_t(GREC ? L::per_g_even : L::per_even) * (kSizedThreads / 32);
}

template <int N1, int N2, bool GREC = false>
bool try_kron2d_sized(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  if (pc.n1 != N1 || pc.q != N2) return false;
  const size_t smem = kron2d_sized_smem<N1, N2, GREC>();
  ensure_smem(kron2d_sized_kernel<N1, N2, GREC>, smem, true);
  const int per_cta = kSizedThreads / 32;
  kron2d_sized_kernel<N1, N2, GREC><<<(pc.nblk + per_cta - 1) / per_cta, kSizedThreads, smem, st>>>(pc, in, out);
  return true;
}

bool launch_kron2d_sized(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  return try_kron2d_sized<5, 5>(pc, in, out, st) || try_kron2d_sized<9, 9>(pc, in, out, st) ||
         try_kron2d_sized<16, 16>(pc, in, out, st) || try_kron2d_sized<21, 21>(pc, in, out, st) ||
         try_kron2d_sized<31, 31>(pc, in, out, st) ||
         try_kron2d_sized<64, 16, true>(pc, in, out, st);  // cfg3 stand-in: n_c = 4, q = 16
}

// ------------------------------------------------------------------------------------ 3D, sized
// apply_factors_3d (precond/ksvd.hpp:132-153) with compile-time (N1 outer, Q): one 128-thread CTA
// per block. Three LU axis solves with register-resident fibers, then the N1 outer slices share
// one Sylvester plan: the wavefront runs all slices at once (4 lanes per cell and slice, tiny
// solve replicated in the group), and the rotations are tiled CTA products over all slices.
constexpr int k3Threads = 128;

template <int R, int K, int C, bool AT, bool BT, int TI, int TJ>
__device__ __forceinline__ void cta_mm_slices(const double* A, int lda, int a_slice, const double* B, int ldb,
                                              int b_slice, double* O, int ldo, int o_slice, int nslices) {
  constexpr int NTI = (R + TI - 1) / TI, NTJ = (C + TJ - 1) / TJ, PER = NTI * NTJ;
  for (int t = threadIdx.x; t < PER * nslices; t += k3Threads) {
    const int sl = t / PER, tt = t % PER, i0 = (tt / NTJ) * TI, j0 = (tt % NTJ) * TJ;
    const double* As = A + sl * a_slice;
    const double* Bs = B + sl * b_slice;
    double acc[TI][TJ];
#pragma unroll
    for (int ii = 0; ii < TI; ++ii)
#pragma unroll
      for (int jj = 0; jj < TJ; ++jj) acc[ii][jj] = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double a[TI], b[TJ];
#pragma unroll
      for (int ii = 0; ii < TI; ++ii) {
        const int i = i0 + ii < R ? i0 + ii : R - 1;
        a[ii] = AT ? As[k * lda + i] : As[i * lda + k];
      }
#pragma unroll
      for (int jj = 0; jj < TJ; ++jj) {
        const int j = j0 + jj < C ? j0 + jj : C - 1;
        b[jj] = BT ? Bs[j * ldb + k] : Bs[k * ldb + j];
      }
#pragma unroll
      for (int ii = 0; ii < TI; ++ii)
#pragma unroll
        for (int jj = 0; jj < TJ; ++jj) acc[ii][jj] = fmac(acc[ii][jj], a[ii], b[jj]);
    }
    double* Os = O + sl * o_slice;
#pragma unroll
    for (int ii = 0; ii < TI; ++ii)
#pragma unroll
      for (int jj = 0; jj < TJ; ++jj)
        if (i0 + ii < R && j0 + jj < C) Os[(i0 + ii) * ldo + j0 + jj] = acc[ii][jj];
  }
}

template <int N1, int Q>
struct Kron3dLayout {
  static constexpr int ld = Q | 1, ss = Q * ld;  // row stride, slice stride (odd: conflict-free fibers)
  static constexpr int rec = N1 * N1 + 6 * Q * Q;
  static constexpr int hdr = (((4 + 4 * Q) / 2 + 2) & ~1);
  static constexpr int rcp = (N1 + 2 * Q + 1) & ~1;
  static constexpr int total = 2 * N1 * ss + rec + rcp + hdr + (N1 + 2 * Q + 1) / 2 + 2;
};

template <int N1, int Q>
__global__ void __launch_bounds__(k3Threads) kron3d_sized_kernel(DevPC pc, const double* __restrict__ in,
                                                                  double* __restrict__ out) {
  const int blk = blockIdx.x;
  if (pc.kind[blk] == 0 || (pc.skip && *pc.skip)) return;
  using L = Kron3dLayout<N1, Q>;
  constexpr int ld = L::ld, ss = L::ss, rec = L::rec, hdr = L::hdr;
  extern __shared__ double sm[];
  double* sX = sm;
  double* sT = sX + N1 * ss;
  double* sR = sT + N1 * ss;
  double* sRcp = sR + rec;
  double* sH = sRcp + L::rcp;
  int* sPiv = reinterpret_cast<int*>(sH + hdr);
  const int tid = threadIdx.x;
  const double* cells = pc.cells + size_t(blk) * pc.cells_len;
  {
    const double* r = pc.rec + size_t(blk) * rec;
    if ((reinterpret_cast<uintptr_t>(r) & 15) == 0 && (reinterpret_cast<uintptr_t>(sR) & 15) == 0) {
      for (int i = 2 * tid; i + 1 < rec; i += 2 * k3Threads) cp_async16(sR + i, r + i);
      if ((rec & 1) && tid == 0) sR[rec - 1] = r[rec - 1];
    } else {
      for (int i = tid; i < rec; i += k3Threads) cp_async8(sR + i, r + i);
    }
    for (int i = tid; i < hdr; i += k3Threads) cp_async8(sH + i, cells + i);
    for (int i = tid; i < N1 + 2 * Q; i += k3Threads) sPiv[i] = pc.piv[size_t(blk) * (N1 + 2 * Q) + i];
    const double* x = in + size_t(blk) * (N1 * Q * Q);
    for (int i = tid; i < N1 * Q * Q; i += k3Threads) {
      const int j = i % Q, rr = (i / Q) % Q, sl = i / (Q * Q);
      cp_async8(sX + sl * ss + rr * ld + j, x + i);
    }
    cp_async_wait_all();
  }
  __syncthreads();
  const double* luA1 = sR;
  const double* luB2 = luA1 + N1 * N1;
  const double* luC1 = luB2 + Q * Q;
  const double* Q1 = luC1 + Q * Q;
  const double* T1 = Q1 + Q * Q;
  const double* Q2 = T1 + Q * Q;
  const double* T2 = Q2 + Q * Q;
  for (int i = tid; i < N1 + 2 * Q; i += k3Threads)
    sRcp[i] = __drcp_rn(i < N1 ? luA1[i * N1 + i] : i < N1 + Q ? luB2[(i - N1) * (Q + 1)] : luC1[(i - N1 - Q) * (Q + 1)]);
  __syncthreads();
  // axis 2 (outer, A1): fibers over (r, j)
  for (int f = tid; f < Q * Q; f += k3Threads) lu_fiber_reg<N1>(luA1, sRcp, sPiv, sX + (f / Q) * ld + f % Q, ss);
  __syncthreads();
  // axis 1 (middle, B2): fibers over (s, j)
  for (int f = tid; f < N1 * Q; f += k3Threads)
    lu_fiber_reg<Q>(luB2, sRcp + N1, sPiv + N1, sX + (f / Q) * ss + f % Q, ld);
  __syncthreads();
  // axis 0 (inner, C1): rows
  for (int f = tid; f < N1 * Q; f += k3Threads)
    lu_fiber_reg<Q>(luC1, sRcp + N1 + Q, sPiv + N1 + Q, sX + (f / Q) * ss + (f % Q) * ld, 1);
  __syncthreads();
  cta_mm_slices<Q, Q, Q, true, false, 2, 4>(Q1, Q, 0, sX, ld, ss, sT, ld, ss, N1);  // Q1^T X_s
  __syncthreads();
  cta_mm_slices<Q, Q, Q, false, false, 2, 4>(sT, ld, ss, Q2, Q, 0, sX, ld, ss, N1);  // (.) Q2 -> M_s
  __syncthreads();
  {  // Y_s overwrites M_s: wavefront over all slices at once
    const int* sb = reinterpret_cast<const int*>(sH);
    const double* cc = cells + hdr;
    if (sb[2]) {
      const int nb1 = sb[0], nb2 = sb[1];
      for (int step = 0; step <= nb1 + nb2 - 2; ++step) {
        const int d1lo = step - (nb2 - 1) > 0 ? step - (nb2 - 1) : 0;
        const int d1hi = step < nb1 - 1 ? step : nb1 - 1;
        const int ncell = d1hi - d1lo + 1;
        for (int t = tid; t < ncell * N1; t += k3Threads) {
          const int sl = t / ncell, d1 = d1lo + t % ncell;
          double* Ms = sX + sl * ss;
          const int i = nb1 - 1 - d1, k = nb2 - 1 - (step - d1);
          const double* c = cc + 6 * (i * Q + k);
          const double code = __ldg(c), coef = __ldg(c + 1), rcp = __ldg(c + 2);
          const double s = sylv_rhs(T1, Q, T2, Q, Ms, Ms, ld, i, k, i + 1, k + 1);
          if (__double_as_longlong(code) & 256) atomicExch(pc.status, int(TPDG_SINGULAR));
          Ms[i * ld + k] = fdiv_rcp(s, coef, rcp);
        }
        __syncthreads();
      }
    } else {
      sylv_wavefront<Q, Q, N1, k3Threads, true>(T1, T2, sX, ld, ss, cc, sb, tid, pc.status);
      __syncthreads();
    }
  }
  cta_mm_slices<Q, Q, Q, false, false, 2, 4>(Q1, Q, 0, sX, ld, ss, sT, ld, ss, N1);  // Q1 Y_s
  __syncthreads();
  cta_mm_slices<Q, Q, Q, false, true, 2, 4>(sT, ld, ss, Q2, Q, 0, out + size_t(blk) * (N1 * Q * Q), Q, Q * Q,
                                            N1);  // (.) Q2^T
}

// ------------------------------------------------------------------------------------ 3D, DMMA
// apply_factors_3d (precond/ksvd.hpp:132-153) as dense products on the FP64 tensor cores. The
// formation-time prep (kron3d_inv_prep_kernel) turns each block's record into
//   A1^-1, L^T = B2^-T Q1, R = C1^-T Q2, Q1, Q2, T2 and G_b = (I (x) T1 + T2_bb (x) I)^-1 for every
//   quasi-diagonal block b of T2 (1x1 or 2x2),
// so that the three LU axis solves fold into the rotations: M_s = L (A1^-1 x)_s R. The Sylvester
// solve T1 Y_s + Y_s T2^T = M_s runs over T2's blocks right to left, as DMMA products of the
// right-hand sides of eight slices with G_b^T per block (each lane forms the right-hand sides of its own
// (slice, row) entries from its solved entries and T2; no barrier). The whole apply is DMMA products
// plus those right-hand sides. (Round 2's first version applied G_b row by row on the CUDA cores, one
// thread per (slice, row): 8.9k shared-memory wavefronts per element, 85 % of the SM's shared-memory
// bandwidth, most of them G_b rows re-read by every warp.) Not bit-faithful
// (explicit inverses; ~1e-13 from the reference at cfg4, tools/study/kron3d_inv_emul.py; gate 1e-12).

// Column c of A^-1 from the packed LU (unit lower L, U, perm) of a record.
__device__ void lu_inverse_col(const double* lu, const int* perm, int n, int c, double* x) {
  for (int k = 0; k < n; ++k) x[k] = perm[k] == c ? 1.0 : 0.0;
  for (int r = 1; r < n; ++r) {
    double s = x[r];
    for (int j = 0; j < r; ++j) s = fma(-lu[r * n + j], x[j], s);
    x[r] = s;
  }
  for (int r = n - 1; r >= 0; --r) {
    double s = x[r];
    for (int j = r + 1; j < n; ++j) s = fma(-lu[r * n + j], x[j], s);
    x[r] = s / lu[r * n + r];
  }
}

// One warp per block: irec = A1^-1 | L^T | R | Q1 | Q2 | T2 | G blocks (block b of size m = sz q stored
// transposed, Gt[k'][n] = G_b[n][k'], m rows of g_t_ld(q, sz) = 2 (mod 8) doubles: the DMMA B-fragment loads
// of the apply's Sylvester sweep -- eight consecutive n by four k' two rows apart -- are conflict-free).
// Lanes take inverse columns, product entries and, in the Gauss-Jordan inverse of (I (x) T1 + T2_bb (x) I),
// rows (elimination) or columns (swap / scaling); every entry sees the same operations in the same
// order as a serial elimination. Shared memory per warp: K, G (m x m, m <= 2 q) and B2^-1, C1^-1.
constexpr int kPrepWarps = 4;
__host__ __device__ inline size_t kron3d_prep_smem_per_warp(int q) { return sizeof(double) * size_t(2 * 4 * q * q + 2 * q * q); }

__global__ void __launch_bounds__(32 * kPrepWarps) kron3d_inv_prep_kernel(DevPC pc, double* __restrict__ irec) {
  extern __shared__ double prep_sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int blk = blockIdx.x * kPrepWarps + wid;
  if (blk >= pc.nblk || pc.kind[blk] == 0) return;
  const int n1 = pc.n1, q = pc.q;
  const double* r = pc.rec + size_t(blk) * pc.rec_len;  // LU(A1) | LU(B2) | LU(C1) | Q1 | T1 | Q2 | T2
  const int* piv = pc.piv + size_t(blk) * pc.piv_len;
  const double *luA1 = r, *luB2 = luA1 + n1 * n1, *luC1 = luB2 + q * q, *Q1 = luC1 + q * q, *T1 = Q1 + q * q,
               *Q2 = T1 + q * q, *T2 = Q2 + q * q;
  double* o = irec + size_t(blk) * irec3_doubles(n1, q);
  double *oA = o, *oLt = oA + n1 * n1, *oR = oLt + q * q, *oQ1 = oR + q * q, *oQ2 = oQ1 + q * q, *oT2 = oQ2 + q * q,
         *oG = oT2 + q * q;
  double* K = prep_sm + size_t(wid) * (kron3d_prep_smem_per_warp(q) / sizeof(double));
  double* G = K + 4 * q * q;
  double* binv = G + 4 * q * q;
  double* cinv = binv + q * q;
  double col[64];
  for (int c = lane; c < n1; c += 32) {
    lu_inverse_col(luA1, piv, n1, c, col);
    for (int k = 0; k < n1; ++k) oA[k * n1 + c] = col[k];
  }
  for (int c = lane; c < q; c += 32) {
    lu_inverse_col(luB2, piv + n1, q, c, col);
    for (int k = 0; k < q; ++k) binv[k * q + c] = col[k];
    lu_inverse_col(luC1, piv + n1 + q, q, c, col);
    for (int k = 0; k < q; ++k) cinv[k * q + c] = col[k];
  }
  __syncwarp();
  for (int e = lane; e < q * q; e += 32) {
    const int i = e / q, j = e % q;
    double lt = 0.0, rr = 0.0;
    for (int k = 0; k < q; ++k) {
      lt = fma(binv[k * q + i], Q1[k * q + j], lt);  // (B2^-T Q1)[i][j]
      rr = fma(cinv[k * q + i], Q2[k * q + j], rr);  // (C1^-T Q2)[i][j]
    }
    oLt[e] = lt;
    oR[e] = rr;
    oQ1[e] = Q1[e];
    oQ2[e] = Q2[e];
    oT2[e] = T2[e];
  }
  int off = 0;
  for (int k0 = 0; k0 < q;) {
    const int sz = (k0 + 1 < q && T2[(k0 + 1) * q + k0] != 0.0) ? 2 : 1;
    const int m = sz * q;  // vec(Y_b) column-major: index c q + i
    for (int e = lane; e < m * m; e += 32) {
      const int a = e / m, b = e % m, ca = a / q, ia = a % q, cb = b / q, ib = b % q;
      K[e] = (ca == cb ? T1[ia * q + ib] : 0.0) + (ia == ib ? T2[(k0 + ca) * q + k0 + cb] : 0.0);
      G[e] = a == b ? 1.0 : 0.0;
    }
    __syncwarp();
    for (int c = 0; c < m; ++c) {  // Gauss-Jordan with partial pivoting (first maximum), as a serial sweep
      int pr = c;
      for (int rr = c + 1; rr < m; ++rr)
        if (fabs(K[rr * m + c]) > fabs(K[pr * m + c])) pr = rr;
      if (pr != c)
        for (int j = lane; j < m; j += 32) {
          double t = K[c * m + j]; K[c * m + j] = K[pr * m + j]; K[pr * m + j] = t;
          t = G[c * m + j]; G[c * m + j] = G[pr * m + j]; G[pr * m + j] = t;
        }
      __syncwarp();
      const double d = 1.0 / K[c * m + c];
      __syncwarp();
      for (int j = lane; j < m; j += 32) {
        K[c * m + j] *= d;
        G[c * m + j] *= d;
      }
      __syncwarp();
      for (int rr = lane; rr < m; rr += 32) {  // lane = row: each row's entries in j order
        if (rr == c) continue;
        const double f = K[rr * m + c];
        if (f == 0.0) continue;
        for (int j = 0; j < m; ++j) {
          K[rr * m + j] = fma(-f, K[c * m + j], K[rr * m + j]);
          G[rr * m + j] = fma(-f, G[c * m + j], G[rr * m + j]);
        }
      }
      __syncwarp();
    }
    const int ld = g_t_ld(q, sz);  // transposed: Gt[k'][n] = G[n][k'], m rows of ld (= 2 mod 8) doubles
    for (int e = lane; e < m * ld; e += 32) {
      const int kk = e / ld, n = e % ld;
      oG[off + e] = n < m ? G[n * m + kk] : 0.0;
    }
    __syncwarp();
    off += m * ld;
    k0 += sz;
  }
}

template <int N1, int Q>
struct Kron3dInvLayout {
  static constexpr int SPW = 32 / Q, NW = (N1 + SPW - 1) / SPW, NTH = 32 * NW;  // slices per warp, warps
  static constexpr int N1P = p8(N1), K1 = p4(N1), QQ = Q * Q, QQP = p8(QQ);
  static constexpr int QP = p8(Q), KQ = p4(Q), NC = N1 * Q, NCP = p8(NC);
  static constexpr int LDS0 = lda4(QQP), LDA = lda4(K1), LDR = lda4(NCP), LDP = lda4(KQ), LQ = lda4(QP);
  static constexpr int NWS = (N1 + 7) / 8;  // Sylvester warps: slices 8 w .. 8 w + 7 are the rows of their tiles
  static_assert(NWS <= NW, "Sylvester warps");
  static constexpr int LD1 = g_t_ld(Q, 1), LD2 = g_t_ld(Q, 2);
  static constexpr int GB = 2 * Q * LD2;   // largest G block (a 2x2 T2 block), doubles
  static constexpr int NG = 3;             // G ring slots (two blocks in flight ahead of the one in use)
  static constexpr int mx(int a, int b) { return a > b ? a : b; }
  // one region, reused: x staged as [s][(r, j)] (GEMM 0) -> P rows (GEMM 1/2) -> G ring (Sylvester) -> Z rows
  static constexpr int S0 = mx(mx(K1 * LDS0, NCP * LDP), NG * GB);
  static constexpr int o_s0 = 0;
  static constexpr int o_x = o_s0 + S0;                // Xr[r][(s, j)]: KQ x LDR
  static constexpr int o_a = o_x + KQ * LDR;           // A1^-1: N1P x LDA
  static constexpr int o_lt = o_a + N1P * LDA;         // L^T, R, Q1, Q2: QP x LQ each
  static constexpr int o_r = o_lt + QP * LQ;
  static constexpr int o_q1 = o_r + QP * LQ;
  static constexpr int o_q2 = o_q1 + QP * LQ;
  static constexpr int o_t2 = o_q2 + QP * LQ;          // T2
  static constexpr int o_lut = (o_t2 + QQ + 1) & ~1;  // int LUTs: Xr offset of (r, j) = n; P offset of (s, r')
  static constexpr int total = o_lut + (QQP + NCP + 1) / 2 + 1;
};

template <int N1, int Q>
__global__ void __launch_bounds__(Kron3dInvLayout<N1, Q>::NTH) kron3d_inv_kernel(DevPC pc,
                                                                                  const double* __restrict__ in,
                                                                                  double* __restrict__ out) {
  const int blk = blockIdx.x;
  if (pc.kind[blk] == 0 || (pc.skip && *pc.skip)) return;
  using L = Kron3dInvLayout<N1, Q>;
  constexpr int NW = L::NW, NTH = L::NTH, QQ = L::QQ, QP = L::QP, KQ = L::KQ, NC = L::NC,
                LDS0 = L::LDS0, LDA = L::LDA, LDR = L::LDR, LDP = L::LDP, LQ = L::LQ, K1 = L::K1;
  extern __shared__ double sm[];
  double* S0 = sm + L::o_s0;
  double* Xr = sm + L::o_x;
  double* Pr = sm + L::o_s0;  // aliases S0 (x staging is dead after GEMM 0, the G ring before GEMM 3)
  double* sA = sm + L::o_a;
  double* sLt = sm + L::o_lt;
  double* sR = sm + L::o_r;
  double* sQ1 = sm + L::o_q1;
  double* sQ2 = sm + L::o_q2;
  double* sT2 = sm + L::o_t2;
  int* lutX = reinterpret_cast<int*>(sm + L::o_lut);  // n = r Q + j -> r LDR + j
  int* lutP = lutX + L::QQP;                          // n = s Q + j -> s Q LDP + j
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // per column k: kind [0, 16) (0 single, 1 second column of a 2x2 block, 2 its first), G offset [16, 32);
  // per Sylvester step (right to left): G offset [34, 50), bytes [50, 66); [32] total G length, [33] steps
  __shared__ int bplan[66];
  __shared__ __align__(8) uint64_t gfull[3], gempty[3];
  const double* ir = pc.irec + size_t(blk) * int(irec3_doubles(N1, Q));
  const double* gG = ir + N1 * N1 + 5 * QQ;
  {
    for (int i = tid; i < N1 * N1; i += NTH) cp_async8(sA + (i / N1) * LDA + i % N1, ir + i);
    for (int i = tid; i < QQ; i += NTH) {
      const int rr = i / Q, cc = i % Q;
      cp_async8(sLt + rr * LQ + cc, ir + N1 * N1 + i);
      cp_async8(sR + rr * LQ + cc, ir + N1 * N1 + QQ + i);
      cp_async8(sQ1 + rr * LQ + cc, ir + N1 * N1 + 2 * QQ + i);
      cp_async8(sQ2 + rr * LQ + cc, ir + N1 * N1 + 3 * QQ + i);
      cp_async8(sT2 + i, ir + N1 * N1 + 4 * QQ + i);
    }
    const double* x = in + size_t(blk) * (N1 * QQ);
    for (int sl = 0; sl < N1; ++sl)
      for (int n = tid; n < QQ; n += NTH) cp_async8(S0 + sl * LDS0 + n, x + sl * QQ + n);
    // K-padding of every product operand must be zero (M / N padding only feeds discarded outputs)
    for (int c = tid; c < LDS0; c += NTH)
      for (int r = N1; r < K1; ++r) S0[r * LDS0 + c] = 0.0;
    for (int r = tid; r < L::N1P; r += NTH)
      for (int c = N1; c < K1; ++c) sA[r * LDA + c] = 0.0;
    for (int c = tid; c < LDR; c += NTH)
      for (int r = Q; r < KQ; ++r) Xr[r * LDR + c] = 0.0;
    for (int c = tid; c < LQ; c += NTH)
      for (int r = Q; r < KQ; ++r) sLt[r * LQ + c] = sR[r * LQ + c] = 0.0;
    for (int r = tid; r < QP; r += NTH)
      for (int c = Q; c < KQ; ++c) sQ1[r * LQ + c] = sQ2[r * LQ + c] = 0.0;
    for (int n = tid; n < L::QQP; n += NTH) lutX[n] = (n / Q) * LDR + n % Q;
    for (int n = tid; n < L::NCP; n += NTH) lutP[n] = (n / Q) * Q * LDP + n % Q;
    cp_async_wait_all();
  }
  __syncthreads();
  if (tid == 0) {
    int goff = 0;
    for (int k0 = 0; k0 < Q;) {
      const int sz = (k0 + 1 < Q && sT2[(k0 + 1) * Q + k0] != 0.0) ? 2 : 1;
      bplan[k0] = sz == 1 ? 0 : 2;
      if (sz == 2) bplan[k0 + 1] = 1;
      bplan[16 + k0 + sz - 1] = goff;
      goff += sz * Q * (sz == 1 ? L::LD1 : L::LD2);
      k0 += sz;
    }
    bplan[32] = goff;
    int ns = 0;
    for (int k = Q - 1; k >= 0; --k) {
      if (bplan[k] == 2) continue;
      const int sz = bplan[k] == 0 ? 1 : 2;
      bplan[34 + ns] = bplan[16 + k];
      bplan[50 + ns++] = 8 * sz * Q * (sz == 1 ? L::LD1 : L::LD2);
    }
    bplan[33] = ns;
    // the element's G blocks go HBM -> L2 now, during the rotations: the ring's copies (two blocks ahead of the
    // sweep) then see L2 latency instead of HBM latency, which paced the sweep
    bulk_prefetch_l2(gG, unsigned(goff) * 8u);
    for (int i = 0; i < L::NG; ++i) {
      mbar_init(&gfull[i], 1);
      mbar_init(&gempty[i], L::NWS);
    }
    mbar_fence_init();
  }
  const int fr = lane >> 2, fc = 2 * (lane & 3);
  {  // X = A1^-1 x along the outer axis: (N1 x N1)(N1 x Q^2) -> Xr[r][s Q + j]
    constexpr int NT0 = L::QQP / 8, NTW0 = (NT0 + NW - 1) / NW;
    double acc[L::N1P / 8][NTW0][2];
    zero_tiles(acc);
    const int nt0 = warp * NTW0;
    if (nt0 < NT0) {
      mma_tiles<L::N1P / 8, NTW0, L::K1 / 4, false>(acc, sA, LDA, S0 + 8 * nt0, LDS0, lane);
#pragma unroll
      for (int nt = 0; nt < NTW0; ++nt)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int n = 8 * (nt0 + nt) + fc + u;
          if (n < QQ) {
            const int o = lutX[n];
#pragma unroll
            for (int mt = 0; mt < L::N1P / 8; ++mt)
              if (8 * mt + fr < N1) Xr[o + (8 * mt + fr) * Q] = acc[mt][nt][u];
          }
        }
    }
  }
  __syncthreads();
  for (int r = tid; r < L::NCP; r += NTH)  // S0 now holds P: its K padding (column Q) must be zero
    for (int c = Q; c < KQ; ++c) Pr[r * LDP + c] = 0.0;
  constexpr int NT = L::NCP / 8, NTW = (NT + NW - 1) / NW;
  {  // P = L Xr (L read through L^T) -> P rows (s Q + r', j)
    double acc[QP / 8][NTW][2];
    zero_tiles(acc);
    const int nt0 = warp * NTW;
    if (nt0 < NT) {
      mma_tiles<QP / 8, NTW, KQ / 4, false, true>(acc, sLt, LQ, Xr + 8 * nt0, LDR, lane);
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int n = 8 * (nt0 + nt) + fc + u;
          if (n < NC) {
            const int o = lutP[n];
#pragma unroll
            for (int mt = 0; mt < QP / 8; ++mt)
              if (8 * mt + fr < Q) Pr[o + (8 * mt + fr) * LDP] = acc[mt][nt][u];
          }
        }
    }
  }
  __syncthreads();
  {  // M = P_rows R -> Xr[r'][s Q + j']
    double acc[NTW][QP / 8][2];
    zero_tiles(acc);
    const int mt0 = warp * NTW;
    if (mt0 < NT) {
      mma_tiles<NTW, QP / 8, KQ / 4, false>(acc, Pr + 8 * mt0 * LDP, LDP, sR, LQ, lane);
#pragma unroll
      for (int mt = 0; mt < NTW; ++mt) {
        const int m = 8 * (mt0 + mt) + fr;
        if (m < NC) {
          const int o = (m % Q) * LDR + (m / Q) * Q;
#pragma unroll
          for (int nt = 0; nt < QP / 8; ++nt)
#pragma unroll
            for (int u = 0; u < 2; ++u)
              if (8 * nt + fc + u < Q) Xr[o + 8 * nt + fc + u] = acc[mt][nt][u];
        }
      }
    }
  }
  __syncthreads();
  // G ring (TMA): slot u % NG holds the block of Sylvester step u; the first two are issued now (P is dead)
  auto g_issue = [&](int u) {
    const int slot = u % L::NG;
    mbar_expect_tx(&gfull[slot], unsigned(bplan[50 + u]));
    bulk_g2s(S0 + slot * L::GB, gG + bplan[34 + u], unsigned(bplan[50 + u]), &gfull[slot]);
  };
  if (tid == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic accesses to P before the TMA writes
    for (int u = 0; u < 2 && u < bplan[33]; ++u) g_issue(u);
  }
  if (warp < L::NWS) {
    // Sylvester T1 Y_s + Y_s T2^T = M_s over T2's quasi-diagonal blocks, right to left, on the tensor cores:
    // for block b (columns c of Y_s, m = |b| q unknowns per slice) [y_c]^T = [rhs_c]^T G_b^T with
    // rhs_c = m_c - sum_{l > b} T2[c][l] y_l, all slices of the warp at once. Warp w takes slices
    // s = 8 w + lane / 4 (the rows of its DMMA tiles); lane quad q = lane % 4 owns the rows
    // i = 8 (t >> 1) + 2 q + (t & 1), t < 2 NTQ, of every column of its slice: exactly the accumulator
    // entries (tile t >> 1, entry t & 1) a product returns to it and the A-fragment entries it supplies
    // at k-step t (the K order of the product is permuted accordingly, Gt rows read in the same order).
    // A lane reads and writes only its own (s, i) entries of Xr, so the sweep needs no barrier.
    constexpr int NTQ = (Q + 7) / 8, NSL = 2 * NTQ, LD1 = L::LD1, LD2 = L::LD2;
    const int r8 = lane >> 2, q4 = lane & 3, sl = 8 * warp + r8;
    const bool sok = sl < N1;
    double* xs = Xr + (sok ? sl : 0) * Q;  // Y_s[i][l] at xs[i LDR + l]
    int step = 0;
#pragma unroll
    for (int k = Q - 1; k >= 0; --k) {
      const int kind = bplan[k];
      if (kind == 2) continue;
      const int slot = step % L::NG;
      const double* g = S0 + slot * L::GB;
      if (tid == 0 && step + 2 < bplan[33]) {  // refill the slot freed by step - 1
        if (step >= 1) mbar_wait(&gempty[(step + 2) % L::NG], unsigned((step - 1) / L::NG) & 1u);
        g_issue(step + 2);
      }
      if (kind == 0) {  // 1x1 block, column k
        double a[NSL];
#pragma unroll
        for (int t = 0; t < NSL; ++t) {
          const int i = 8 * (t >> 1) + 2 * q4 + (t & 1);
          double s0 = 0.0, s1 = 0.0;
          if (sok && i < Q) {
            const double* xr = xs + i * LDR;
            s0 = xr[k];
#pragma unroll
            for (int l = k + 1; l < Q; ++l) {
              if ((l - k) & 1) s0 = fma(-xr[l], sT2[k * Q + l], s0);
              else s1 = fma(-xr[l], sT2[k * Q + l], s1);
            }
          }
          a[t] = s0 + s1;
        }
        mbar_wait(&gfull[slot], unsigned(step / L::NG) & 1u);
        double acc[NTQ][2];
#pragma unroll
        for (int nt = 0; nt < NTQ; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
        for (int kc = 0; kc < NSL; ++kc) {
          const int kk = 8 * (kc >> 1) + 2 * q4 + (kc & 1);
#pragma unroll
          for (int nt = 0; nt < NTQ; ++nt) {
            const int n = 8 * nt + r8;
            dmma(acc[nt], a[kc], (kk < Q && n < Q) ? g[kk * LD1 + n] : 0.0);
          }
        }
        if (sok)
#pragma unroll
          for (int nt = 0; nt < NTQ; ++nt)
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int i = 8 * nt + 2 * q4 + u;
              if (i < Q) xs[i * LDR + k] = acc[nt][u];
            }
      } else if (k > 0) {  // 2x2 block, columns k - 1, k: the 2 Q unknowns (c, i) of a slice as one index n' = c Q + i
        // lane quad q owns n' = 8 (t >> 1) + 2 q + (t & 1), t < NS2: the accumulator entries a product returns to it
        // and the A entries it supplies at k-step t (K order permuted accordingly, Gt rows read in that order)
        constexpr int NT2 = (2 * Q + 7) / 8, NS2 = 2 * NT2;
        double a[NS2];
#pragma unroll
        for (int t = 0; t < NS2; ++t) {
          const int np = 8 * (t >> 1) + 2 * q4 + (t & 1);
          const int c = np >= Q ? 1 : 0, i = np - c * Q;
          double v = 0.0;
          if (sok && np < 2 * Q) {
            const double* xr = xs + i * LDR;
            const double* t2 = sT2 + (k - 1 + c) * Q;
            v = xr[k - 1 + c];
#pragma unroll
            for (int l = k + 1; l < Q; ++l) v = fma(-xr[l], t2[l], v);
          }
          a[t] = v;
        }
        mbar_wait(&gfull[slot], unsigned(step / L::NG) & 1u);
        double acc[NT2][2];
#pragma unroll
        for (int nt = 0; nt < NT2; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
        for (int kc = 0; kc < NS2; ++kc) {
          const int kk = 8 * (kc >> 1) + 2 * q4 + (kc & 1);
#pragma unroll
          for (int nt = 0; nt < NT2; ++nt) {
            const int n = 8 * nt + r8;
            dmma(acc[nt], a[kc], (kk < 2 * Q && n < 2 * Q) ? g[kk * LD2 + n] : 0.0);
          }
        }
        if (sok)
#pragma unroll
          for (int nt = 0; nt < NT2; ++nt)
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int np = 8 * nt + 2 * q4 + u;
              const int c = np >= Q ? 1 : 0, i = np - c * Q;
              if (np < 2 * Q) xs[i * LDR + k - 1 + c] = acc[nt][u];
            }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&gempty[slot]);
      ++step;
    }
  }
  __syncthreads();
  for (int r = tid; r < L::NCP; r += NTH)  // the G ring overwrote P's K padding
    for (int c = Q; c < KQ; ++c) Pr[r * LDP + c] = 0.0;
  {  // Z = Q1 Y -> Z rows (s Q + r, j')
    double acc[QP / 8][NTW][2];
    zero_tiles(acc);
    const int nt0 = warp * NTW;
    if (nt0 < NT) {
      mma_tiles<QP / 8, NTW, KQ / 4, false>(acc, sQ1, LQ, Xr + 8 * nt0, LDR, lane);
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int n = 8 * (nt0 + nt) + fc + u;
          if (n < NC) {
            const int o = lutP[n];
#pragma unroll
            for (int mt = 0; mt < QP / 8; ++mt)
              if (8 * mt + fr < Q) Pr[o + (8 * mt + fr) * LDP] = acc[mt][nt][u];
          }
        }
    }
  }
  __syncthreads();
  {  // out = Z_rows Q2^T -> out[s][r][j]
    double acc[NTW][QP / 8][2];
    zero_tiles(acc);
    const int mt0 = warp * NTW;
    if (mt0 < NT) {
      mma_tiles<NTW, QP / 8, KQ / 4, true>(acc, Pr + 8 * mt0 * LDP, LDP, sQ2, LQ, lane);
      double* o = out + size_t(blk) * (N1 * QQ);
#pragma unroll
      for (int mt = 0; mt < NTW; ++mt) {
        const int m = 8 * (mt0 + mt) + fr;
        if (m < NC)
#pragma unroll
          for (int nt = 0; nt < QP / 8; ++nt)
#pragma unroll
            for (int u = 0; u < 2; ++u)
              if (8 * nt + fc + u < Q) o[m * Q + 8 * nt + fc + u] = acc[mt][nt][u];
      }
    }
  }
}

template <int N1, int Q>
bool try_kron3d_inv(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  if (pc.dim != 3 || pc.n1 != N1 || pc.q != Q || !pc.irec) return false;
  using L = Kron3dInvLayout<N1, Q>;
  const size_t smem = sizeof(double) * size_t(L::total);
  ensure_smem(kron3d_inv_kernel<N1, Q>, smem);
  kron3d_inv_kernel<N1, Q><<<pc.nblk, L::NTH, smem, st>>>(pc, in, out);
  return true;
}

bool launch_kron3d_inv(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  return try_kron3d_inv<4, 4>(pc, in, out, st) || try_kron3d_inv<5, 5>(pc, in, out, st) ||
         try_kron3d_inv<8, 8>(pc, in, out, st) || try_kron3d_inv<11, 11>(pc, in, out, st) ||
         try_kron3d_inv<15, 3>(pc, in, out, st) || try_kron3d_inv<40, 8>(pc, in, out, st);
}

template <int N1, int Q>
bool try_kron3d_sized(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  if (pc.dim != 3 || pc.n1 != N1 || pc.q != Q) return false;
  const size_t smem = sizeof(double) * size_t(Kron3dLayout<N1, Q>::total);
  ensure_smem(kron3d_sized_kernel<N1, Q>, smem, true);
  kron3d_sized_kernel<N1, Q><<<pc.nblk, k3Threads, smem, st>>>(pc, in, out);
  return true;
}

bool launch_kron3d_sized(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  return try_kron3d_sized<4, 4>(pc, in, out, st) || try_kron3d_sized<5, 5>(pc, in, out, st) ||
         try_kron3d_sized<8, 8>(pc, in, out, st) || try_kron3d_sized<11, 11>(pc, in, out, st);
}

// ------------------------------------------------------------------------------------ 3D
__global__ void __launch_bounds__(kApplyThreads) kron3d_apply_kernel(DevPC pc, const double* __restrict__ in,
                                                                      double* __restrict__ out) {
  const int blk = blockIdx.x;
  if (pc.kind[blk] == 0 || (pc.skip && *pc.skip)) return;
  extern __shared__ double sm[];
  const int n1 = pc.n1, q = pc.q, ld = q | 1, ss = q * ld;  // slice stride
  double* sX = sm;
  double* sT = sX + n1 * ss;
  double* sR = sT + n1 * ss;
  double* rowsum = sR + pc.rec_len;
  int* sPiv = reinterpret_cast<int*>(rowsum + 2 * q);
  int* sb = sPiv + pc.piv_len;
  __shared__ SylvPlan P;
  const int tid = threadIdx.x, nt = blockDim.x;
  const double* rec = pc.rec + size_t(blk) * pc.rec_len;
  for (int i = tid; i < pc.rec_len; i += nt) sR[i] = rec[i];
  for (int i = tid; i < pc.piv_len; i += nt) sPiv[i] = pc.piv[size_t(blk) * pc.piv_len + i];
  const double* x = in + size_t(blk) * pc.blk_len;
  for (int i = tid; i < n1 * q * q; i += nt) {
    const int j = i % q, r = (i / q) % q, s = i / (q * q);
    sX[s * ss + r * ld + j] = x[i];
  }
  if (tid == 0) {
    P.s1 = sb;
    P.z1 = sb + q;
    P.s2 = sb + 2 * q;
    P.z2 = sb + 3 * q;
  }
  __syncthreads();
  const double* luA1 = sR;
  const double* luB2 = luA1 + n1 * n1;
  const double* luC1 = luB2 + q * q;
  const double* Q1 = luC1 + q * q;
  const double* T1 = Q1 + q * q;
  const double* Q2 = T1 + q * q;
  const double* T2 = Q2 + q * q;
  // axis 2 (outer, A1): fibers over (r, j)
  for (int f = tid; f < q * q; f += nt) {
    const int r = f / q, j = f % q;
    lu_solve_fiber(luA1, sPiv, n1, sX + r * ld + j, ss, sT + r * ld + j, ss);
  }
  __syncthreads();
  // axis 1 (middle, B2): fibers over (s, j)
  for (int f = tid; f < n1 * q; f += nt) {
    const int s = f / q, j = f % q;
    lu_solve_fiber(luB2, sPiv + n1, q, sX + s * ss + j, ld, sT + s * ss + j, ld);
  }
  __syncthreads();
  // axis 0 (inner, C1): rows
  for (int f = tid; f < n1 * q; f += nt) {
    const int s = f / q, r = f % q;
    lu_solve_fiber(luC1, sPiv + n1 + q, q, sX + s * ss + r * ld, 1, sT + s * ss + r * ld, 1);
  }
  __syncthreads();
  mm_slices(q, q, q, Q1, q, true, 0, sX, ld, false, ss, sT, ld, ss, n1);
  sylv_plan(T1, q, T2, q, P, rowsum);
  mm_slices(q, q, q, sT, ld, false, ss, Q2, q, false, 0, sX, ld, ss, n1);
  __syncthreads();
  sylv_wavefront(T1, q, T2, q, P, sX, sT, ld, ss, n1, pc.status);
  mm_slices(q, q, q, Q1, q, false, 0, sT, ld, false, ss, sX, ld, ss, n1);
  __syncthreads();
  double* o = out + size_t(blk) * pc.blk_len;
  mm_slices(q, q, q, sX, ld, false, ss, Q2, q, true, 0, o, q, q * q, n1);
}

size_t kron3d_smem(const DevPC& pc) {
  const int n1 = pc.n1, q = pc.q, ld = q | 1;
  return sizeof(double) * size_t(2 * n1 * q * ld + pc.rec_len + 2 * q) +
         sizeof(int) * size_t(pc.piv_len + 4 * q) + 16;
}

// ------------------------------------------------------------------------------------ fallback
// x = LU^{-1} b for one dense block; LU column-major (lu[j*n + i] = LU(i, j)).
__global__ void __launch_bounds__(256) kron_fallback_kernel(DevPC pc, const double* __restrict__ in,
                                                             double* __restrict__ out) {
  const int blk = blockIdx.x;
  if (pc.kind[blk] != 0 || (pc.skip && *pc.skip)) return;
  extern __shared__ double sx[];
  const int n = pc.blk_len;
  const int slot = pc.fb_slot[blk];
  const double* lu = pc.fb_lu + size_t(slot) * n * n;
  const int* perm = pc.fb_piv + size_t(slot) * n;
  const double* b = in + size_t(blk) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sx[i] = b[perm[i]];
  __syncthreads();
  for (int j = 0; j < n; ++j) {  // forward: row i gets j = 0, 1, ... in order (reference order)
    const double xj = sx[j];
    const double* col = lu + size_t(j) * n;
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) sx[i] = fmsc(sx[i], col[i], xj);
    __syncthreads();
  }
  for (int j = n - 1; j >= 0; --j) {  // backward, column-descending
    const double* col = lu + size_t(j) * n;
    const double xj = fdiv(sx[j], col[j]);
    __syncthreads();
    if (threadIdx.x == 0) sx[j] = xj;
    for (int i = threadIdx.x; i < j; i += blockDim.x) sx[i] = fmsc(sx[i], col[i], xj);
    __syncthreads();
  }
  double* o = out + size_t(blk) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) o[i] = sx[i];
}


} // namespace

void launch_kron3d_inv_prep(const DevPC& pc, double* irec, cudaStream_t st) {
  if (pc.nblk == 0) return;
  const size_t smem = kron3d_prep_smem_per_warp(pc.q) * kPrepWarps;
  ensure_smem(kron3d_inv_prep_kernel, smem);
  kron3d_inv_prep_kernel<<<(pc.nblk + kPrepWarps - 1) / kPrepWarps, 32 * kPrepWarps, smem, st>>>(pc, irec);
  TPDG_CUDA_CHECK(cudaGetLastError());
}

void launch_sylv_cells(const DevPC& pc, double* cells, cudaStream_t st) {
  if (pc.nblk == 0) return;
  sylv_cells_kernel<<<(pc.nblk + 3) / 4, 128, 0, st>>>(pc, cells);
  TPDG_CUDA_CHECK(cudaGetLastError());
}

void launch_pc_apply(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  if (pc.nblk == 0) return;
  const size_t smem = pc.dim == 2 ? kron2d_smem(pc) : kron3d_smem(pc);
  if (smem > 227 * 1024)
    throw Failure{TPDG_CONFIG, "pc_apply: factor record of " + std::to_string(smem) + " B exceeds shared memory"};
  if (pc.dim == 2) {
    // the bit-faithful multi-block kernel (kron_ew.cu), else one block per warp (sized), else generic
    if (!launch_kron2d_ew(pc, in, out, st) && !launch_kron2d_sized(pc, in, out, st)) {
      ensure_smem(kron2d_apply_kernel, smem);
      kron2d_apply_kernel<<<pc.nblk, kApplyThreads, smem, st>>>(pc, in, out);
    }
  } else if (!(!pc.faithful && launch_kron3d_inv(pc, in, out, st)) && !launch_kron3d_sized(pc, in, out, st)) {
    ensure_smem(kron3d_apply_kernel, smem);
    kron3d_apply_kernel<<<pc.nblk, kApplyThreads, smem, st>>>(pc, in, out);
  }
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
  if (pc.fb_lu) {
    const size_t fsm = sizeof(double) * size_t(pc.blk_len);
    if (!launch_fallback_apply(pc, in, out, st)) {  // blocks beyond 2048 rows: one column sweep per step
      ensure_smem(kron_fallback_kernel, fsm);
      kron_fallback_kernel<<<pc.nblk, 256, fsm, st>>>(pc, in, out);
    }
    TPDG_CUDA_CHECK(cudaGetLastError());
    ++g_launches;
  }
}

} // namespace tpdg_gpu
