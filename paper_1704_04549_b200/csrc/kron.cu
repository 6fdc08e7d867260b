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
#include "faithful.cuh"
#include "tpdg_internal.hpp"

namespace tpdg_gpu {

namespace {

constexpr int kApplyThreads = 128;

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
  if (pc.kind[blk] == 0) return;
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

// ------------------------------------------------------------------------------------ 3D
__global__ void __launch_bounds__(kApplyThreads) kron3d_apply_kernel(DevPC pc, const double* __restrict__ in,
                                                                      double* __restrict__ out) {
  const int blk = blockIdx.x;
  if (pc.kind[blk] == 0) return;
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
  if (pc.kind[blk] != 0) return;
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

template <typename K>
void set_smem(K kernel, size_t bytes, size_t& configured) {
  if (bytes > configured) {
    TPDG_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    configured = bytes;
  }
}

} // namespace

void launch_pc_apply(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  if (pc.nblk == 0) return;
  static size_t c2 = 0, c3 = 0, cf = 0;
  const size_t smem = pc.dim == 2 ? kron2d_smem(pc) : kron3d_smem(pc);
  if (smem > 227 * 1024)
    throw Failure{TPDG_CONFIG, "pc_apply: factor record of " + std::to_string(smem) + " B exceeds shared memory"};
  if (pc.dim == 2) {
    set_smem(kron2d_apply_kernel, smem, c2);
    kron2d_apply_kernel<<<pc.nblk, kApplyThreads, smem, st>>>(pc, in, out);
  } else {
    set_smem(kron3d_apply_kernel, smem, c3);
    kron3d_apply_kernel<<<pc.nblk, kApplyThreads, smem, st>>>(pc, in, out);
  }
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
  if (pc.fb_lu) {
    const size_t fsm = sizeof(double) * size_t(pc.blk_len);
    set_smem(kron_fallback_kernel, fsm, cf);
    kron_fallback_kernel<<<pc.nblk, 256, fsm, st>>>(pc, in, out);
    TPDG_CUDA_CHECK(cudaGetLastError());
    ++g_launches;
  }
}

} // namespace tpdg_gpu
