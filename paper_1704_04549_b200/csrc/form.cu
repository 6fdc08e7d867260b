// KSVD formation on the device, one CTA per block (persistent grid, per-CTA global workspace).
//
// Restates form_ksvd_2d / form_ksvd_3d (reference precond/ksvd.hpp:252-372):
//   lanczos_form_kernel : Golub-Kahan Lanczos with full 2-pass MGS reorthogonalization
//                         (tensor/lanczos.hpp:85-190) on the matrix-free shuffled products
//                         (shuffled.cuh), one-sided Jacobi SVD of the bidiagonal
//                         (tensor/svd_small.hpp:20-84), reshape to Kronecker factors, degenerate
//                         collapse (ksvd.hpp:279-283); 3D: stage 1 (r=1) + stage 2 on the
//                         explicitly shuffled D1 (ksvd.hpp:335-352).
//   make_factors_kernel : LuFactor (tensor/small_matrix.hpp:143-172), C = A^{-1} B
//                         (ksvd.hpp:48-57), real_schur (tensor/schur.hpp:38-232),
//                         check_sylvester_pair (ksvd.hpp:61-73), term swap on failure
//                         (ksvd.hpp:284-291 / 353-358).
//   assemble + dense LU : exact block fallback (ksvd.hpp:292-300, ops/linearized.hpp:245-285).
//
// Compiled with -fmad=false. Every reduction is summed in the reference's order by a single
// thread; the parallelism is across independent accumulators (matrix entries, fibers,
// Householder columns/rows, rotation columns), which leaves each result bit-identical to the
// reference's sequential code. The only non-bit-identical operations are CUDA's libm sin / cos /
// atan / atan2 inside standardize_2x2 (<= 2 ulp vs glibc).
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <type_traits>

#include "faithful.cuh"
#include "glibm.cuh"
#include "shuffled.cuh"
#include "tpdg_internal.hpp"

namespace tpdg_gpu {

namespace {

constexpr int kFormThreads = 256;

constexpr int kMaxGroups = kFormThreads / 32;
#ifndef FORM_GLOBAL_CTAS
#define FORM_GLOBAL_CTAS 4  // measured at cfg2 p=15: 2 -> 8.2 ms, 3 -> 7.1, 4 -> 5.3, 6 -> 6.5, 8 -> 6.9
#endif
constexpr int kFormGlobalCtas = FORM_GLOBAL_CTAS;  // resident CTAs per SM of the global-working-set make_factors
template <class G>
__device__ __forceinline__ int groups_per_cta() {
  return 1;
}
template <>
__device__ __forceinline__ int groups_per_cta<WarpGroup>() {
  return int(blockDim.x >> 5);
}

__device__ __forceinline__ void bsync() { __syncthreads(); }

// ---------------------------------------------------------------- sequential reductions
// dot / norm in the reference's order. A CTA group sums on one thread and broadcasts through shared memory. A warp
// group spreads the loads and the products over its lanes (coalesced; each product is rounded on its own, as in the
// serial loop: no FMA in this file) and every lane then adds the 32 products of a chunk in index order, fetched by
// shuffle: the same additions in the same order, so the same bits, but the chain is one DADD per element instead of
// a load-to-use latency per element (the serial sums were 34 % of the cfg4 Lanczos kernel, ncu).
__device__ __forceinline__ double warp_ordered_sum(double s, double p, int cnt) {
  if (cnt == 32) {
#pragma unroll
    for (int l = 0; l < 32; ++l) s += __shfl_sync(0xffffffffu, p, l);
  } else {
    for (int l = 0; l < cnt; ++l) s += __shfl_sync(0xffffffffu, p, l);
  }
  return s;
}
template <class Grp>
__device__ double seq_dot(const Grp& g, const double* a, const double* b, long n, double* sh) {
  if constexpr (std::is_same<Grp, WarpGroup>::value) {
    const int lane = g.rank();
    double s = 0.0;
    for (long base = 0; base < n; base += 32) {
      const long i = base + lane;
      const double p = i < n ? a[i] * b[i] : 0.0;
      s = warp_ordered_sum(s, p, int(n - base < 32 ? n - base : 32));
    }
    g.sync();
    return s;
  } else {
    if (g.rank() == 0) {
      double s = 0.0;
      for (long i = 0; i < n; ++i) s += a[i] * b[i];
      *sh = s;
    }
    g.sync();
    const double r = *sh;
    g.sync();
    return r;
  }
}
template <class Grp>
__device__ double seq_norm(const Grp& g, const double* a, long n, double* sh) {
  if constexpr (std::is_same<Grp, WarpGroup>::value) {
    const int lane = g.rank();
    double s = 0.0;
    for (long base = 0; base < n; base += 32) {
      const long i = base + lane;
      const double p = i < n ? a[i] * a[i] : 0.0;
      s = warp_ordered_sum(s, p, int(n - base < 32 ? n - base : 32));
    }
    g.sync();
    return sqrt(s);
  } else {
    if (g.rank() == 0) {
      double s = 0.0;
      for (long i = 0; i < n; ++i) s += a[i] * a[i];
      *sh = sqrt(s);
    }
    g.sync();
    const double r = *sh;
    g.sync();
    return r;
  }
}

// ---------------------------------------------------------------- shuffled operator wrapper
struct LzOp {
  int kind;           // 0 = element shuffled, 1 = dense matrix (3D stage 2)
  ShufCtx k;
  const double* dense;  // rows x cols, row-major
  int m1, n1, m2, n2;
  __host__ __device__ long rows() const { return long(m1) * n1; }
  __host__ __device__ long cols() const { return long(m2) * n2; }
};

template <class Grp>
__device__ void op_apply(const Grp& g, const LzOp& op, const double* x, double* y, double* ws) {
  if (op.kind == 0) {
    if (op.k.s.dim == 2) shuf_apply_2d_dev(g, op.k, x, y, ws); else shuf_apply_3d_dev(g, op.k, x, y, ws);
    return;
  }
  const long R = op.rows(), Cn = op.cols();
  for (long i = g.rank(); i < R; i += g.size()) {  // matvec (small_matrix.hpp:116-124)
    double s = 0.0;
    for (long j = 0; j < Cn; ++j) s += op.dense[i * Cn + j] * x[j];
    y[i] = s;
  }
  g.sync();
}
template <class Grp>
__device__ void op_apply_t(const Grp& g, const LzOp& op, const double* x, double* y, double* ws) {
  if (op.kind == 0) {
    if (op.k.s.dim == 2) shuf_apply_t_2d_dev(g, op.k, x, y, ws); else shuf_apply_t_3d_dev(g, op.k, x, y, ws);
    return;
  }
  const long R = op.rows(), Cn = op.cols();
  for (long j = g.rank(); j < Cn; j += g.size()) {  // matvec_transpose (small_matrix.hpp:127-135)
    double s = 0.0;
    for (long i = 0; i < R; ++i) s += op.dense[i * Cn + j] * x[i];
    y[j] = s;
  }
  g.sync();
}

// ---------------------------------------------------------------- Jacobi SVD (single thread)
// svd_small on the tall orientation; u: m x k, v: n x k, k = min(m, n).
__device__ void svd_small_dev(int m, int n, const double* a, double* u, double* sigma, double* v, double* w,
                              double* vv, double* sig, int* order) {
  const bool tr = m < n;
  const int M = tr ? n : m, N = tr ? m : n;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) w[i * N + j] = tr ? a[j * n + i] : a[i * n + j];
  for (int i = 0; i < N * N; ++i) vv[i] = 0.0;
  for (int i = 0; i < N; ++i) vv[i * N + i] = 1.0;
  double scale = 0.0;
  for (int i = 0; i < M * N; ++i) scale = fmax(scale, fabs(w[i]));
  scale = fmax(scale, 1e-300);
  const double tol = 1e-14;
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < N - 1; ++p)
      for (int qq = p + 1; qq < N; ++qq) {
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (int i = 0; i < M; ++i) {
          app += w[i * N + p] * w[i * N + p];
          aqq += w[i * N + qq] * w[i * N + qq];
          apq += w[i * N + p] * w[i * N + qq];
        }
        if (fabs(apq) <= tol * scale * scale) continue;
        rotated = true;
        const double zeta = (aqq - app) / (2.0 * apq);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = c * t;
        for (int i = 0; i < M; ++i) {
          const double wp = w[i * N + p], wq = w[i * N + qq];
          w[i * N + p] = c * wp - s * wq;
          w[i * N + qq] = s * wp + c * wq;
        }
        for (int i = 0; i < N; ++i) {
          const double vp = vv[i * N + p], vq = vv[i * N + qq];
          vv[i * N + p] = c * vp - s * vq;
          vv[i * N + qq] = s * vp + c * vq;
        }
      }
    if (!rotated) break;
  }
  for (int j = 0; j < N; ++j) {
    double s = 0.0;
    for (int i = 0; i < M; ++i) s += w[i * N + j] * w[i * N + j];
    sig[j] = sqrt(s);
    order[j] = j;
  }
  for (int i = 1; i < N; ++i) {  // descending; == libstdc++ std::sort for distinct values
    const int key = order[i];
    int j = i - 1;
    while (j >= 0 && sig[key] > sig[order[j]]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = key;
  }
  // tall result: U_t (M x N) = w / sig, V_t (N x N) = vv; transposed input swaps the roles.
  double* Ut = tr ? v : u;
  double* Vt = tr ? u : v;
  for (int kk = 0; kk < N; ++kk) {
    const int j = order[kk];
    sigma[kk] = sig[j];
    const double inv = sig[j] > 0.0 ? 1.0 / sig[j] : 0.0;
    for (int i = 0; i < M; ++i) Ut[i * N + kk] = w[i * N + j] * inv;
    for (int i = 0; i < N; ++i) Vt[i * N + kk] = vv[i * N + j];
  }
}

// ---------------------------------------------------------------- Lanczos KSVD (one CTA)
struct LzWork {
  double* V;      // (J+1) x cols
  double* U;      // (J+1) x rows
  double* alpha;  // J+1
  double* beta;   // J+1
  double* B;      // (J+1)^2
  double* bu;     // (J+1)^2
  double* bv;     // (J+1)^2
  double* bs;     // J+1
  double* sw;     // 2 (J+1)^2 + 2 (J+1) svd scratch
  int* order;     // J+1
  double* opws;   // shuffled scratch
};

// fa: r x (m1 x n1), fb: r x (m2 x n2), sig: r. Returns iterations (reference `iterations`).
template <class Grp>
__device__ int lanczos_dev(const Grp& g, const LzOp& op, int r, int max_iter, double breakdown, const double* start, double* fa,
                           double* fb, double* sig, LzWork& W, double* sh) {
  const long nrows = op.rows(), ncols = op.cols();
  const int tid = g.rank(), nt = g.size();
  for (long i = tid; i < r * nrows; i += nt) fa[i] = 0.0;
  for (long i = tid; i < r * ncols; i += nt) fb[i] = 0.0;
  if (tid < r) sig[tid] = 0.0;
  for (long i = tid; i < ncols; i += nt) W.V[i] = start[i];
  g.sync();
  op_apply(g, op, W.V, W.U, W.opws);
  double alpha = seq_norm(g, W.U, nrows, sh);
  const double tol = breakdown * fmax(alpha, 1e-300);
  if (alpha < 1e-300) return 0;
  for (long i = tid; i < nrows; i += nt) W.U[i] = W.U[i] / alpha;
  if (tid == 0) W.alpha[0] = alpha;
  int nv = 1, nu = 1, na = 1, nb = 0, iters = 1;
  g.sync();
  while (na < max_iter) {
    double* p = W.V + size_t(nv) * ncols;
    op_apply_t(g, op, W.U + size_t(nu - 1) * nrows, p, W.opws);
    const double al = W.alpha[na - 1];
    const double* vl = W.V + size_t(nv - 1) * ncols;
    for (long i = tid; i < ncols; i += nt) p[i] = p[i] - al * vl[i];
    g.sync();
    for (int pass = 0; pass < 2; ++pass)
      for (int j = 0; j < nv; ++j) {
        const double* qj = W.V + size_t(j) * ncols;
        const double dot = seq_dot(g, qj, p, ncols, sh);
        for (long i = tid; i < ncols; i += nt) p[i] = p[i] - dot * qj[i];
        g.sync();
      }
    const double beta = seq_norm(g, p, ncols, sh);
    ++iters;
    if (beta < tol) break;
    for (long i = tid; i < ncols; i += nt) p[i] = p[i] / beta;
    if (tid == 0) W.beta[nb] = beta;
    ++nv;
    ++nb;
    g.sync();
    double* rv = W.U + size_t(nu) * nrows;
    op_apply(g, op, W.V + size_t(nv - 1) * ncols, rv, W.opws);
    const double* ul = W.U + size_t(nu - 1) * nrows;
    for (long i = tid; i < nrows; i += nt) rv[i] = rv[i] - beta * ul[i];
    g.sync();
    for (int pass = 0; pass < 2; ++pass)
      for (int j = 0; j < nu; ++j) {
        const double* qj = W.U + size_t(j) * nrows;
        const double dot = seq_dot(g, qj, rv, nrows, sh);
        for (long i = tid; i < nrows; i += nt) rv[i] = rv[i] - dot * qj[i];
        g.sync();
      }
    alpha = seq_norm(g, rv, nrows, sh);
    if (alpha < tol) break;
    for (long i = tid; i < nrows; i += nt) rv[i] = rv[i] / alpha;
    if (tid == 0) W.alpha[na] = alpha;
    ++nu;
    ++na;
    g.sync();
  }
  const int ku = nu, kv = nv, kmin = ku < kv ? ku : kv;
  if (tid == 0) {
    for (int i = 0; i < ku * kv; ++i) W.B[i] = 0.0;
    for (int i = 0; i < ku; ++i) {
      W.B[i * kv + i] = W.alpha[i];
      if (i + 1 < kv && i < nb) W.B[i * kv + i + 1] = W.beta[i];
    }
    const int J1 = max_iter + 1;
    svd_small_dev(ku, kv, W.B, W.bu, W.bs, W.bv, W.sw, W.sw + J1 * J1, W.sw + 2 * J1 * J1, W.order);
    for (int j = 0; j < r; ++j) sig[j] = (j < kmin && W.bs[j] > 0.0) ? W.bs[j] : 0.0;
  }
  g.sync();
  for (int j = 0; j < r; ++j) {
    if (!(j < kmin && W.bs[j] > 0.0)) continue;
    const double scale = sqrt(W.bs[j]);
    for (long i = tid; i < nrows; i += nt) {
      double s = 0.0;
      for (int l = 0; l < ku; ++l) s += W.U[size_t(l) * nrows + i] * W.bu[l * kmin + j];
      fa[j * nrows + (i % op.m1) * op.n1 + i / op.m1] = scale * s;
    }
    for (long i = tid; i < ncols; i += nt) {
      double s = 0.0;
      for (int l = 0; l < kv; ++l) s += W.V[size_t(l) * ncols + i] * W.bv[l * kmin + j];
      fb[j * ncols + (i % op.m2) * op.n2 + i / op.m2] = scale * s;
    }
  }
  g.sync();
  return iters;
}

template <class Grp>
__device__ void set_identity_dev(const Grp& g, int n, double* m) {
  for (int i = g.rank(); i < n * n; i += g.size()) m[i] = (i / n == i % n) ? 1.0 : 0.0;
}

// Lanczos work layout per CTA.
__host__ __device__ inline size_t lz_work_doubles(int J, long rows, long cols, size_t opws) {
  const size_t J1 = J + 1;
  return J1 * cols + J1 * rows + 4 * J1 + 3 * J1 * J1 + 2 * J1 * J1 + 2 * J1 + J1 + opws + 64;
}

__device__ LzWork carve_lz(double* base, int J, long rows, long cols) {
  const size_t J1 = J + 1;
  LzWork W;
  W.V = base;
  W.U = W.V + J1 * cols;
  W.alpha = W.U + J1 * rows;
  W.beta = W.alpha + J1;
  W.bs = W.beta + J1;
  W.B = W.bs + 2 * J1;
  W.bu = W.B + J1 * J1;
  W.bv = W.bu + J1 * J1;
  W.sw = W.bv + J1 * J1;
  W.order = reinterpret_cast<int*>(W.sw + 2 * J1 * J1 + 2 * J1);
  W.opws = W.sw + 2 * J1 * J1 + 2 * J1 + J1;
  return W;
}

// Per block: raw factors (2D: a1 b1 a2 b2 ; 3D: a1 b1 c1 b2 c2) after the degenerate collapse;
// kind[blk] = 0 when the 3D stage-1 singular value vanishes (-> fallback), else 1 (pending).
template <class Grp>
__global__ void __launch_bounds__(kFormThreads, 2) lanczos_form_kernel(DevSys s, tpdg_gpu_ksvd_config cfg,
                                                                     const double* start_vec,
                                                                     const double* start_vec2, double* raw,
                                                                     int* kind, double* work, size_t work_per_cta,
                                                                     int nblk) {
  const int NG = groups_per_cta<Grp>();
  const Grp g;
  const int gid = NG == 1 ? 0 : int(threadIdx.x >> 5);
  __shared__ double sh_all[kMaxGroups][4];
  double* sh = sh_all[gid];
  const int q = s.q, ncb = s.small ? 1 : s.n_c, m1 = ncb * q, m2 = s.dim == 2 ? q : q * q;
  const int terms = cfg.terms;
  const int J = cfg.lanczos_max_it > 0 ? cfg.lanczos_max_it : 2 * terms + 20;
  const int J1 = cfg.lanczos_max_it > 0 ? cfg.lanczos_max_it : 2 * 1 + 20;
  const int rl = raw_len_of(s.dim, m1, q);
  double* wbase = work + (size_t(blockIdx.x) * NG + gid) * work_per_cta;
  for (int blk = blockIdx.x * NG + gid; blk < nblk; blk += gridDim.x * NG) {
    const int bpe = s.small ? s.n_c : 1;
    const int e = blk / bpe, comp = blk % bpe;
    LzOp op;
    op.kind = 0;
    op.k.s = s;
    op.k.e = e;
    op.k.comp = comp;
    op.k.ncb = ncb;
    op.dense = nullptr;
    op.m1 = op.n1 = m1;
    op.m2 = op.n2 = m2;
    double* rb = raw + size_t(blk) * rl;
    const size_t opws = shuffled_ws_doubles(s.dim, q, s.mu, ncb);
    if (s.dim == 2) {
      const int Jm = J;
      LzWork W = carve_lz(wbase, Jm, op.rows(), op.cols());
      double* fa = W.opws + opws;              // terms x m1^2
      double* fb = fa + size_t(terms) * m1 * m1;  // terms x q^2
      double* sig = fb + size_t(terms) * q * q;
      lanczos_dev(g, op, terms, Jm, cfg.breakdown_tol, start_vec, fa, fb, sig, W, sh);
      double* a1 = rb;
      double* b1 = a1 + m1 * m1;
      double* a2 = b1 + q * q;
      double* b2 = a2 + m1 * m1;
      for (int i = g.rank(); i < m1 * m1; i += g.size()) {
        a1[i] = fa[i];
        a2[i] = terms > 1 ? fa[m1 * m1 + i] : 0.0;
      }
      for (int i = g.rank(); i < q * q; i += g.size()) {
        b1[i] = fb[i];
        b2[i] = terms > 1 ? fb[q * q + i] : 0.0;
      }
      g.sync();
      if (terms < 2 || sig[1] <= cfg.degenerate_tol * sig[0]) {
        set_identity_dev(g, m1, a2);
        for (int i = g.rank(); i < q * q; i += g.size()) b2[i] = 0.0;
      }
      if (g.rank() == 0) kind[blk] = 1;
      g.sync();
    } else {
      // stage 1: A ~ A1 (x) D1 (r = 1)
      LzWork W = carve_lz(wbase, J1, op.rows(), op.cols());
      double* fa = W.opws + opws;         // m1^2
      double* d1 = fa + size_t(m1) * m1;  // q^4
      double* sig1 = d1 + size_t(m2) * m2;
      double* shd = sig1 + 2;             // q^4 shuffled D1
      double* fb2 = shd + size_t(m2) * m2;  // terms x q^2
      double* fc2 = fb2 + size_t(terms) * q * q;
      double* sig2 = fc2 + size_t(terms) * q * q;
      lanczos_dev(g, op, 1, J1, cfg.breakdown_tol, start_vec, fa, d1, sig1, W, sh);
      if (!(sig1[0] > 0.0)) {
        if (g.rank() == 0) kind[blk] = 0;
        g.sync();
        continue;
      }
      // shuffle_dense(D1, q, q, q, q) (tensor/shuffle.hpp:16-25)
      for (int t = g.rank(); t < m2 * m2; t += g.size()) {
        const int c = t % q, r = (t / q) % q, j = (t / (q * q)) % q, i = t / (q * q * q);
        shd[(j * q + i) * (q * q) + c * q + r] = d1[(i * q + r) * (q * q) + j * q + c];
      }
      g.sync();
      LzOp op2;
      op2.kind = 1;
      op2.k = op.k;
      op2.dense = shd;
      op2.m1 = op2.n1 = op2.m2 = op2.n2 = q;
      LzWork W2 = carve_lz(wbase, J, op2.rows(), op2.cols());
      lanczos_dev(g, op2, terms, J, cfg.breakdown_tol, start_vec2, fb2, fc2, sig2, W2, sh);
      double* a1 = rb;
      double* b1 = a1 + m1 * m1;
      double* c1 = b1 + q * q;
      double* b2 = c1 + q * q;
      double* c2 = b2 + q * q;
      for (int i = g.rank(); i < m1 * m1; i += g.size()) a1[i] = fa[i];
      for (int i = g.rank(); i < q * q; i += g.size()) {
        b1[i] = fb2[i];
        c1[i] = fc2[i];
        b2[i] = terms > 1 ? fb2[q * q + i] : 0.0;
        c2[i] = terms > 1 ? fc2[q * q + i] : 0.0;
      }
      g.sync();
      if (terms < 2 || sig2[1] <= cfg.degenerate_tol * sig2[0]) {
        set_identity_dev(g, q, b2);
        for (int i = g.rank(); i < q * q; i += g.size()) c2[i] = 0.0;
      }
      if (g.rank() == 0) kind[blk] = 1;
      g.sync();
    }
  }
}

// ---------------------------------------------------------------- dense LU (CTA-cooperative)
// LuFactor ctor on an n x n row-major matrix (copied to lu). Returns false if singular.
template <class Grp>
__device__ bool lu_factor_dev(const Grp& g, int n, const double* a, double* lu, int* perm, double* sh, int* ish) {
  const int tid = g.rank(), nt = g.size();
  for (int i = tid; i < n * n; i += nt) lu[i] = a[i];
  for (int i = tid; i < n; i += nt) perm[i] = i;
  // inf_norm: row sums in order, then max
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int j = 0; j < n; ++j) s += fabs(a[i * n + j]);
      m = fmax(m, s);
    }
    sh[0] = 1e-14 * fmax(m, 1e-300);
  }
  g.sync();
  const double tol = sh[0];
  for (int k = 0; k < n; ++k) {
    if (tid == 0) {
      int piv = k;
      double best = fabs(lu[k * n + k]);
      for (int i = k + 1; i < n; ++i) {
        const double v = fabs(lu[i * n + k]);
        if (v > best) {
          best = v;
          piv = i;
        }
      }
      ish[0] = best < tol ? -1 : piv;
      if (best >= tol && piv != k) {
        const int t = perm[k];
        perm[k] = perm[piv];
        perm[piv] = t;
      }
    }
    g.sync();
    const int piv = ish[0];
    if (piv < 0) return false;
    if (piv != k)
      for (int j = tid; j < n; j += nt) {
        const double t = lu[k * n + j];
        lu[k * n + j] = lu[piv * n + j];
        lu[piv * n + j] = t;
      }
    g.sync();
    const double inv = 1.0 / lu[k * n + k];
    for (int i = k + 1 + tid; i < n; i += nt) lu[i * n + k] = lu[i * n + k] * inv;
    g.sync();
    const int rem = n - k - 1;
    for (int t = tid; t < rem * rem; t += nt) {
      const int i = k + 1 + t / rem, j = k + 1 + t % rem;
      lu[i * n + j] -= lu[i * n + k] * lu[k * n + j];
    }
    g.sync();
  }
  return true;
}

// lu_solve_matrix (ksvd.hpp:48-57): x(:, j) = LU^{-1} rhs(:, j), columns in parallel.
template <class Grp>
__device__ void lu_solve_cols_dev(const Grp& g, int n, const double* lu, const int* perm, int cols, const double* rhs, double* x) {
  for (int j = g.rank(); j < cols; j += g.size()) {
    for (int i = 0; i < n; ++i) x[i * cols + j] = rhs[perm[i] * cols + j];
    for (int i = 0; i < n; ++i) {
      double s = x[i * cols + j];
      for (int k = 0; k < i; ++k) s -= lu[i * n + k] * x[k * cols + j];
      x[i * cols + j] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = x[i * cols + j];
      for (int k = i + 1; k < n; ++k) s -= lu[i * n + k] * x[k * cols + j];
      x[i * cols + j] = s / lu[i * n + i];
    }
  }
  g.sync();
}

// ---------------------------------------------------------------- real Schur (CTA-cooperative)
template <class Grp>
__device__ void rot_left_dev(const Grp& g, double* m, int n, int i, int j, double c, double s) {
  for (int k = g.rank(); k < n; k += g.size()) {
    const double x = m[i * n + k], y = m[j * n + k];
    m[i * n + k] = c * x + s * y;
    m[j * n + k] = -s * x + c * y;
  }
}
template <class Grp>
__device__ void rot_right_dev(const Grp& g, double* m, int n, int i, int j, double c, double s) {
  for (int k = g.rank(); k < n; k += g.size()) {
    const double x = m[k * n + i], y = m[k * n + j];
    m[k * n + i] = c * x + s * y;
    m[k * n + j] = -s * x + c * y;
  }
}

// standardize_2x2 (schur.hpp:86-113)
template <class Grp>
__device__ void standardize_2x2_dev(const Grp& g, double* h, double* q, int n, int l, double* sh) {
  if (g.rank() == 0) {
    const double a = h[l * n + l], b = h[l * n + l + 1], c = h[(l + 1) * n + l], d = h[(l + 1) * n + l + 1];
    sh[2] = 0.0;
    if (c == 0.0) {
      sh[3] = -1.0;
    } else {
      // libm calls in glibc's own arithmetic (glibm.cuh): bit-identical rotations to the reference
      const double th1 = 0.5 * glibm_atan2(d - a, b + c);
      double cc = glibm_cos(th1), ss = glibm_sin(th1);
      const double bt = cc * cc * b - ss * ss * c + cc * ss * (d - a);
      const double ct = cc * cc * c - ss * ss * b + cc * ss * (d - a);
      const bool real_pair = bt * ct >= 0.0;
      double th = th1;
      if (real_pair) {
        double th2;
        if (bt == 0.0)
          th2 = (ct == 0.0) ? 0.0 : 2.0 * glibm_atan(1.0);
        else
          th2 = glibm_atan(sqrt(ct / bt));
        th += th2;
      }
      sh[0] = glibm_cos(th);
      sh[1] = glibm_sin(th);
      sh[2] = real_pair ? 1.0 : 0.0;
      sh[3] = 1.0;
    }
  }
  g.sync();
  if (sh[3] < 0.0) {
    g.sync();
    return;
  }
  const double cc = sh[0], ss = sh[1];
  const bool real_pair = sh[2] != 0.0;
  rot_left_dev(g, h, n, l, l + 1, cc, ss);
  g.sync();
  rot_right_dev(g, h, n, l, l + 1, cc, ss);
  rot_right_dev(g, q, n, l, l + 1, cc, ss);
  g.sync();
  if (g.rank() == 0 && real_pair) h[(l + 1) * n + l] = 0.0;
  g.sync();
}

// real_schur (schur.hpp:119-232). h holds C on entry, T on exit; returns false on budget exhaustion.
template <class Grp>
__device__ bool real_schur_dev(const Grp& g, int n, double* h, double* q, double* v, double* sh, int* ish) {
  const int tid = g.rank(), nt = g.size();
  for (int i = tid; i < n * n; i += nt) q[i] = (i / n == i % n) ? 1.0 : 0.0;
  g.sync();
  if (n == 1) return true;
  // Householder Hessenberg (schur.hpp:38-79)
  for (int k = 0; k + 2 < n; ++k) {
    if (tid == 0) {
      double norm = 0.0;
      for (int i = k + 1; i < n; ++i) norm += h[i * n + k] * h[i * n + k];
      norm = sqrt(norm);
      ish[0] = 0;
      if (norm != 0.0) {
        const double alpha = h[(k + 1) * n + k] >= 0.0 ? -norm : norm;
        double vn2 = 0.0;
        for (int i = k + 1; i < n; ++i) {
          v[i] = h[i * n + k];
          if (i == k + 1) v[i] -= alpha;
          vn2 += v[i] * v[i];
        }
        if (vn2 != 0.0) {
          ish[0] = 1;
          sh[0] = 2.0 / vn2;
          sh[1] = alpha;
        }
      }
    }
    g.sync();
    if (ish[0] == 0) continue;
    const double beta = sh[0], alpha = sh[1];
    for (int j = k + tid; j < n; j += nt) {  // H <- P H
      double dot = 0.0;
      for (int i = k + 1; i < n; ++i) dot += v[i] * h[i * n + j];
      dot *= beta;
      for (int i = k + 1; i < n; ++i) h[i * n + j] -= dot * v[i];
    }
    g.sync();
    for (int i = tid; i < n; i += nt) {  // H <- H P ; Q <- Q P
      double dot = 0.0;
      for (int j = k + 1; j < n; ++j) dot += h[i * n + j] * v[j];
      dot *= beta;
      for (int j = k + 1; j < n; ++j) h[i * n + j] -= dot * v[j];
      double dq = 0.0;
      for (int j = k + 1; j < n; ++j) dq += q[i * n + j] * v[j];
      dq *= beta;
      for (int j = k + 1; j < n; ++j) q[i * n + j] -= dq * v[j];
    }
    g.sync();
    if (tid == 0) {
      for (int i = k + 2; i < n; ++i) h[i * n + k] = 0.0;
      h[(k + 1) * n + k] = alpha;
    }
    g.sync();
  }
  double hnorm;
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int j = 0; j < n; ++j) s += fabs(h[i * n + j]);
      m = fmax(m, s);
    }
    sh[0] = fmax(m, 1e-300);
  }
  g.sync();
  hnorm = sh[0];
  g.sync();
  const double eps = 2.3e-16;
  int m = n - 1, iter = 0, total = 0;
  const int budget = 60 * n;
  while (m >= 0) {
    if (++total > budget) return false;
    // deflation scan (thread 0), shift vector
    if (tid == 0) {
      int l = m;
      while (l > 0) {
        const double s = fabs(h[(l - 1) * n + l - 1]) + fabs(h[l * n + l]);
        if (fabs(h[l * n + l - 1]) <= eps * fmax(s, hnorm)) {
          h[l * n + l - 1] = 0.0;
          break;
        }
        --l;
      }
      ish[0] = l;
    }
    g.sync();
    const int l = ish[0];
    g.sync();
    if (l == m) {
      m -= 1;
      iter = 0;
      continue;
    }
    if (l == m - 1) {
      standardize_2x2_dev(g, h, q, n, l, sh);
      m -= 2;
      iter = 0;
      continue;
    }
    ++iter;
    double x, y, z;
#define H(i, j) h[(i) * n + (j)]
    if (iter % 11 == 0) {
      const double s = fabs(H(m, m - 1)) + fabs(H(m - 1, m - 2));
      const double shf = H(m, m) + 0.75 * s;
      const double tdet = shf * shf - 0.4375 * s * s;
      x = H(l, l) * H(l, l) + H(l, l + 1) * H(l + 1, l) - 2.0 * shf * H(l, l) + tdet;
      y = H(l + 1, l) * (H(l, l) + H(l + 1, l + 1) - 2.0 * shf);
      z = (l + 2 <= m) ? H(l + 1, l) * H(l + 2, l + 1) : 0.0;
    } else {
      const double tr = H(m - 1, m - 1) + H(m, m);
      const double det = H(m - 1, m - 1) * H(m, m) - H(m - 1, m) * H(m, m - 1);
      x = H(l, l) * H(l, l) + H(l, l + 1) * H(l + 1, l) - tr * H(l, l) + det;
      y = H(l + 1, l) * (H(l, l) + H(l + 1, l + 1) - tr);
      z = (l + 2 <= m) ? H(l + 1, l) * H(l + 2, l + 1) : 0.0;
    }
    for (int k = l; k <= m - 1; ++k) {
      const int len = (k + 2 <= m) ? 3 : 2;
      if (tid == 0) {
        v[0] = x;
        v[1] = y;
        v[2] = (len == 3) ? z : 0.0;
        double nrm = 0.0;
        for (int i = 0; i < len; ++i) nrm += v[i] * v[i];
        nrm = sqrt(nrm);
        ish[1] = 0;
        if (nrm != 0.0) {
          const double alpha = v[0] >= 0.0 ? -nrm : nrm;
          v[0] -= alpha;
          double vn2 = 0.0;
          for (int i = 0; i < len; ++i) vn2 += v[i] * v[i];
          if (vn2 != 0.0) {
            ish[1] = 1;
            sh[0] = 2.0 / vn2;
          }
        }
      }
      g.sync();
      if (ish[1]) {
        const double beta = sh[0];
        const int row_hi = (k + len < n) ? k + len : n;
        const int col_lo = (k > l) ? k - 1 : l;
        for (int j = col_lo + tid; j < n; j += nt) {
          double dot = 0.0;
          for (int i = 0; i < len; ++i) dot += v[i] * H(k + i, j);
          dot *= beta;
          for (int i = 0; i < len; ++i) H(k + i, j) -= dot * v[i];
        }
        g.sync();
        const int row_top = ((m < k + len) ? m : k + len) + 1;
        for (int i = tid; i < n; i += nt) {
          if (i < row_top) {
            double dot = 0.0;
            for (int j = k; j < row_hi; ++j) dot += H(i, j) * v[j - k];
            dot *= beta;
            for (int j = k; j < row_hi; ++j) H(i, j) -= dot * v[j - k];
          }
          double dq = 0.0;
          for (int j = k; j < row_hi; ++j) dq += q[i * n + j] * v[j - k];
          dq *= beta;
          for (int j = k; j < row_hi; ++j) q[i * n + j] -= dq * v[j - k];
        }
        g.sync();
      }
      x = H(k + 1, k);
      if (k + 2 <= m) y = H(k + 2, k);
      if (k + 3 <= m) z = H(k + 3, k);
      g.sync();
    }
    for (int t = tid; t < n * n; t += nt) {
      const int i = t / n, j = t % n;
      if (i >= l + 2 && i <= m && j >= l && j <= i - 2) H(i, j) = 0.0;
    }
    g.sync();
#undef H
  }
  for (int l = 0; l + 1 < n; ++l) {
    const double sub = h[(l + 1) * n + l];
    g.sync();
    if (sub != 0.0) standardize_2x2_dev(g, h, q, n, l, sh);
  }
  return true;
}

// quasi_triangular_eigenvalues (schur.hpp:235-266), single thread.
__device__ int quasi_eigs_dev(int n, const double* t, double* re, double* im) {
  int i = 0, k = 0;
  while (i < n) {
    if (i + 1 < n && t[(i + 1) * n + i] != 0.0) {
      const double a = t[i * n + i], b = t[i * n + i + 1], c = t[(i + 1) * n + i], d = t[(i + 1) * n + i + 1];
      const double tr = 0.5 * (a + d);
      const double disc = tr * tr - (a * d - b * c);
      if (disc >= 0.0) {
        const double sq = sqrt(disc);
        re[k] = tr + sq;
        im[k++] = 0.0;
        re[k] = tr - sq;
        im[k++] = 0.0;
      } else {
        const double sq = sqrt(-disc);
        re[k] = tr;
        im[k++] = sq;
        re[k] = tr;
        im[k++] = -sq;
      }
      i += 2;
    } else {
      re[k] = t[i * n + i];
      im[k++] = 0.0;
      ++i;
    }
  }
  return k;
}

__device__ double inf_norm_seq(int n, const double* a) {
  double m = 0.0;
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += fabs(a[i * n + j]);
    m = fmax(m, s);
  }
  return m;
}

// check_sylvester_pair (ksvd.hpp:61-73): true when usable.
template <class Grp>
__device__ bool check_pair_dev(const Grp& g, int n1, const double* t1, int n2, const double* t2, double* eig, double* sh,
                               int* ish) {
  double* re1 = eig;
  double* im1 = re1 + n1;
  double* re2 = im1 + n1;
  double* im2 = re2 + n2;
  if (g.rank() == 0) {
    quasi_eigs_dev(n1, t1, re1, im1);
    quasi_eigs_dev(n2, t2, re2, im2);
    sh[0] = inf_norm_seq(n1, t1) + inf_norm_seq(n2, t2);
    ish[0] = 0;
  }
  g.sync();
  const double thr = 1e-12 * fmax(sh[0], 1e-300);
  for (int t = g.rank(); t < n1 * n2; t += g.size()) {
    const int i = t / n2, j = t % n2;
    const double re = re1[i] + re2[j], im = im1[i] + im2[j];
    if (sqrt(re * re + im * im) < thr) ish[0] = 1;
  }
  g.sync();
  const bool ok = ish[0] == 0;
  g.sync();
  return ok;
}

// make_factors_2d / 3d into a record (layout in tpdg_internal.hpp). Returns true when usable.
template <class Grp>
__device__ bool make_factors_dev(const Grp& g, int dim, int q, int n1, const double* raw, double* rec, int* piv, double* w,
                                 double* sh, int* ish) {
  if (dim == 2) {
    const double* a1 = raw;
    const double* b1 = a1 + n1 * n1;
    const double* a2 = b1 + q * q;
    const double* b2 = a2 + n1 * n1;
    double* luA2 = rec;
    double* luB1 = luA2 + n1 * n1;
    double* Q1 = luB1 + q * q;
    double* T1 = Q1 + n1 * n1;
    double* Q2 = T1 + n1 * n1;
    double* T2 = Q2 + q * q;
    if (!lu_factor_dev(g, n1, a2, luA2, piv, sh, ish)) return false;
    if (!lu_factor_dev(g, q, b1, luB1, piv + n1, sh, ish)) return false;
    lu_solve_cols_dev(g, n1, luA2, piv, n1, a1, T1);      // C1 = A2^{-1} A1 (Schur in place in T1)
    lu_solve_cols_dev(g, q, luB1, piv + n1, q, b2, T2);   // C2 = B1^{-1} B2
    if (!real_schur_dev(g, n1, T1, Q1, w, sh, ish)) return false;
    if (!real_schur_dev(g, q, T2, Q2, w, sh, ish)) return false;
    return check_pair_dev(g, n1, T1, q, T2, w, sh, ish);
  }
  const double* a1 = raw;
  const double* b1 = a1 + n1 * n1;
  const double* c1 = b1 + q * q;
  const double* b2 = c1 + q * q;
  const double* c2 = b2 + q * q;
  double* luA1 = rec;
  double* luB2 = luA1 + n1 * n1;
  double* luC1 = luB2 + q * q;
  double* Q1 = luC1 + q * q;
  double* T1 = Q1 + q * q;
  double* Q2 = T1 + q * q;
  double* T2 = Q2 + q * q;
  if (!lu_factor_dev(g, n1, a1, luA1, piv, sh, ish)) return false;
  if (!lu_factor_dev(g, q, b2, luB2, piv + n1, sh, ish)) return false;
  if (!lu_factor_dev(g, q, c1, luC1, piv + n1 + q, sh, ish)) return false;
  lu_solve_cols_dev(g, q, luB2, piv + n1, q, b1, T1);       // G1 = B2^{-1} B1
  lu_solve_cols_dev(g, q, luC1, piv + n1 + q, q, c2, T2);   // G2 = C1^{-1} C2
  if (!real_schur_dev(g, q, T1, Q1, w, sh, ish)) return false;
  if (!real_schur_dev(g, q, T2, Q2, w, sh, ish)) return false;
  return check_pair_dev(g, q, T1, q, T2, w, sh, ish);
}

// Per block with kind == 1: factors; on failure swap the (second-stage) terms and retry;
// on second failure kind = 0 (fallback). NOTE: the reference lets a Schur ConvergenceError
// escape (process abort); here it is routed to the swap / fallback path.
// The whole per-block working set (raw factors, the record being built, pivots, scratch) lives in
// shared memory when it fits (SMEM = true): the serial sections of LU / Hessenberg / Francis QR then
// pay shared-memory rather than L2 latency per access. Results are copied out at the end.
template <bool SMEM, class Grp>
__global__ void __launch_bounds__(kFormThreads, SMEM ? 1 : kFormGlobalCtas) make_factors_kernel(int dim, int q, int n1, int nblk,
                                                                     double* raw, double* rec, int* piv, int* kind,
                                                                     double* work) {
  const int NG = groups_per_cta<Grp>();
  const Grp g;
  const int gid = NG == 1 ? 0 : int(threadIdx.x >> 5);
  __shared__ double sh_all[kMaxGroups][8];
  __shared__ int ish_all[kMaxGroups][4];
  double* sh = sh_all[gid];
  int* ish = ish_all[gid];
  extern __shared__ double fsm_all[];
  const int rl = raw_len_of(dim, n1, q), rcl = rec_len_of(dim, n1, q), pl = piv_len_of(dim, n1, q);
  const int wl = 4 * (n1 > q ? n1 : q) + 16;
  const size_t per_group = size_t(wl + rl + rcl) + size_t(pl + 1) / 2 + 2;
  double* fsm = fsm_all + (SMEM ? size_t(gid) * per_group : 0);
  double* w = SMEM ? fsm : work + (size_t(blockIdx.x) * NG + gid) * wl;
  double* rb_s = fsm + wl;
  double* rc_s = rb_s + rl;
  int* pv_s = reinterpret_cast<int*>(rc_s + rcl);
  for (int blk = blockIdx.x * NG + gid; blk < nblk; blk += gridDim.x * NG) {
    if (kind[blk] == 0) continue;
    double* rb_g = raw + size_t(blk) * rl;
    double* rb = SMEM ? rb_s : rb_g;
    double* rc = SMEM ? rc_s : rec + size_t(blk) * rcl;
    int* pv = SMEM ? pv_s : piv + size_t(blk) * pl;
    if (SMEM) {
      for (int i = g.rank(); i < rl; i += g.size()) rb_s[i] = rb_g[i];
      g.sync();
    }
    bool ok = make_factors_dev(g, dim, q, n1, rb, rc, pv, w, sh, ish);
    if (!ok) {
      // swap: 2D (a1,b1,a2,b2) -> (a2,b2,a1,b1); 3D (b1,c1) <-> (b2,c2)
      if (dim == 2) {
        const int la = n1 * n1, lb = q * q;
        for (int i = g.rank(); i < la; i += g.size()) {
          const double t = rb[i];
          rb[i] = rb[la + lb + i];
          rb[la + lb + i] = t;
        }
        for (int i = g.rank(); i < lb; i += g.size()) {
          const double t = rb[la + i];
          rb[la + i] = rb[2 * la + lb + i];
          rb[2 * la + lb + i] = t;
        }
      } else {
        const int base = n1 * n1, lb = q * q;
        for (int i = g.rank(); i < 2 * lb; i += g.size()) {
          const double t = rb[base + i];
          rb[base + i] = rb[base + 2 * lb + i];
          rb[base + 2 * lb + i] = t;
        }
      }
      g.sync();
      ok = make_factors_dev(g, dim, q, n1, rb, rc, pv, w, sh, ish);
      if (SMEM)
        for (int i = g.rank(); i < rl; i += g.size()) rb_g[i] = rb_s[i];  // export the swapped terms
    }
    if (SMEM && ok) {
      double* rcg = rec + size_t(blk) * rcl;
      int* pvg = piv + size_t(blk) * pl;
      for (int i = g.rank(); i < rcl; i += g.size()) rcg[i] = rc_s[i];
      for (int i = g.rank(); i < pl; i += g.size()) pvg[i] = pv_s[i];
    }
    if (g.rank() == 0) kind[blk] = ok ? 1 : 0;
    g.sync();
  }
}

// ---------------------------------------------------------------- fallback blocks
// Dense block by probing element_diag_apply with unit vectors (ops/linearized.hpp:245-285).
// One CTA per (column j, fallback block); column-major result = the probe's output vector.
__global__ void __launch_bounds__(kFormThreads) probe_kernel(DevSys s, const int* blocks, int nfb, double* fb_lu,
                                                              double* work, size_t work_per_cta) {
  const int ncols = s.small ? s.npe : s.n_c * s.npe;
  for (int task = blockIdx.x; task < ncols * nfb; task += gridDim.x) {
  const int j = task % ncols, f = task / ncols;
  const int blk = blocks[f];
  const int bpe = s.small ? s.n_c : 1;
  const int e = blk / bpe, comp = blk % bpe;
  const int npe = s.npe, nfull = s.n_c * npe, n = s.small ? npe : nfull;
  const int q = s.q, mu = s.mu, nc = s.n_c, d = s.dim, nqv = s.nqv, nqf = s.nqf;
  double* vin = work + size_t(blockIdx.x) * work_per_cta;
  double* vals = vin + nfull;
  double* field = vals + nc * nqv;
  double* t1 = field + nqv;  // scratch for the sum-factorized stages (mu^d * q^... bounded below)
  const int off = s.small ? comp * npe : 0;
  for (int i = threadIdx.x; i < nfull; i += blockDim.x) vin[i] = (i == off + j) ? 1.0 : 0.0;
  double* out = fb_lu + size_t(f) * n * n + size_t(j) * n;
  double* vout = t1 + 2 * size_t(nqv) * q + nfull;  // full-length accumulator
  for (int i = threadIdx.x; i < nfull; i += blockDim.x) vout[i] = 0.0;
  bsync();
  const int ext0 = q;
  (void)ext0;
  // vals = G x..x G vin_c (eval_at_quad)
  for (int c = 0; c < nc; ++c) {
    const double* co = vin + c * npe;
    double* vv = vals + c * nqv;
    if (d == 2) {
      for (int t = threadIdx.x; t < mu * q; t += blockDim.x) {
        const int al = t % mu, jj = t / mu;
        double acc = 0.0;
        for (int i = 0; i < q; ++i) acc += s.g[al * q + i] * co[jj * q + i];
        t1[t] = acc;  // [j][al]
      }
      bsync();
      for (int t = threadIdx.x; t < mu * mu; t += blockDim.x) {
        const int al = t % mu, be = t / mu;
        double acc = 0.0;
        for (int jj = 0; jj < q; ++jj) acc += s.g[be * q + jj] * t1[jj * mu + al];
        vv[t] = acc;
      }
      bsync();
    } else {
      double* t2 = t1 + size_t(q) * q * mu;
      for (int t = threadIdx.x; t < mu * q * q; t += blockDim.x) {
        const int al = t % mu, jk = t / mu;
        double acc = 0.0;
        for (int i = 0; i < q; ++i) acc += s.g[al * q + i] * co[jk * q + i];
        t1[t] = acc;  // [k][j][al]
      }
      bsync();
      for (int t = threadIdx.x; t < mu * mu * q; t += blockDim.x) {
        const int al = t % mu, be = (t / mu) % mu, k = t / (mu * mu);
        double acc = 0.0;
        for (int jj = 0; jj < q; ++jj) acc += s.g[be * q + jj] * t1[(k * q + jj) * mu + al];
        t2[t] = acc;  // [k][be][al]
      }
      bsync();
      for (int t = threadIdx.x; t < nqv; t += blockDim.x) {
        const int ab = t % (mu * mu), ga = t / (mu * mu);
        double acc = 0.0;
        for (int k = 0; k < q; ++k) acc += s.g[ga * q + k] * t2[k * mu * mu + ab];
        vv[t] = acc;
      }
      bsync();
    }
  }
  // integrate_back of one field into vout_r with D^T W in slot dslot
  auto integrate = [&](int dslot, const double* fld, double* o) {
    if (d == 2) {
      for (int t = threadIdx.x; t < q * mu; t += blockDim.x) {
        const int i = t % q, be = t / q;
        const double* X = dslot == 0 ? s.dw : s.gw;
        double acc = 0.0;
        for (int al = 0; al < mu; ++al) acc += X[i * mu + al] * fld[be * mu + al];
        t1[t] = acc;  // [be][i]
      }
      bsync();
      for (int t = threadIdx.x; t < q * q; t += blockDim.x) {
        const int i = t % q, jj = t / q;
        const double* Y = dslot == 1 ? s.dw : s.gw;
        double acc = 0.0;
        for (int be = 0; be < mu; ++be) acc += Y[jj * mu + be] * t1[be * q + i];
        o[t] += acc;
      }
      bsync();
    } else {
      double* t2 = t1 + size_t(q) * mu * mu;
      for (int t = threadIdx.x; t < q * mu * mu; t += blockDim.x) {
        const int i = t % q, gb = t / q;
        const double* X = dslot == 0 ? s.dw : s.gw;
        double acc = 0.0;
        for (int al = 0; al < mu; ++al) acc += X[i * mu + al] * fld[gb * mu + al];
        t1[t] = acc;  // [ga][be][i]
      }
      bsync();
      for (int t = threadIdx.x; t < q * q * mu; t += blockDim.x) {
        const int i = t % q, jj = (t / q) % q, ga = t / (q * q);
        const double* Y = dslot == 1 ? s.dw : s.gw;
        double acc = 0.0;
        for (int be = 0; be < mu; ++be) acc += Y[jj * mu + be] * t1[(ga * mu + be) * q + i];
        t2[t] = acc;  // [ga][j][i]
      }
      bsync();
      for (int t = threadIdx.x; t < q * q * q; t += blockDim.x) {
        const int ij = t % (q * q), k = t / (q * q);
        const double* Z = dslot == 2 ? s.dw : s.gw;
        double acc = 0.0;
        for (int ga = 0; ga < mu; ++ga) acc += Z[k * mu + ga] * t2[ga * q * q + ij];
        o[t] += acc;
      }
      bsync();
    }
  };
  const double* jd = s.jdet + size_t(e) * nqv;
  if (s.a != 0.0)
    for (int c = 0; c < nc; ++c) {
      for (int t = threadIdx.x; t < nqv; t += blockDim.x) field[t] = s.a * jd[t] * vals[c * nqv + t];
      bsync();
      integrate(-1, field, vout + c * npe);
    }
  if (s.b != 0.0) {
    for (int dir = 0; dir < d; ++dir) {
      const double* dft = s.dft + ((size_t(e) * d + dir) * nqv) * nc * nc;
      for (int r = 0; r < nc; ++r) {
        for (int t = threadIdx.x; t < nqv; t += blockDim.x) {
          double acc = 0.0;
          if (!s.small)
            for (int c = 0; c < nc; ++c) acc += dft[size_t(t) * nc * nc + r * nc + c] * vals[c * nqv + t];
          else
            acc = dft[size_t(t) * nc * nc + r * nc + r] * vals[r * nqv + t];
          field[t] = s.b * acc;
        }
        bsync();
        integrate(dir, field, vout + r * npe);
      }
    }
    // own-trace face terms (face_trace / face_lift, ops/discretization.hpp:89-166)
    for (int fc = 0; fc < 2 * d; ++fc) {
      const int axis = fc / 2, layer = (fc % 2) == 0 ? 0 : q - 1;
      double* tm = field;  // nc * nqf (nqf <= nqv)
      for (int t = threadIdx.x; t < nc * nqf; t += blockDim.x) {
        const int c = t / nqf, qf = t % nqf;
        const double* co = vin + c * npe;
        double acc = 0.0;
        if (d == 2) {
          for (int jj = 0; jj < q; ++jj) acc += s.g[qf * q + jj] * (axis == 0 ? co[jj * q + layer] : co[layer * q + jj]);
        } else {
          const int a = qf % mu, bb = qf / mu;
          for (int j1 = 0; j1 < q; ++j1) {
            double inner = 0.0;
            for (int j0 = 0; j0 < q; ++j0) {
              int idx[3];
              idx[axis] = layer;
              idx[axis == 0 ? 1 : 0] = j0;
              idx[axis == 2 ? 1 : 2] = j1;
              inner += s.g[a * q + j0] * co[(idx[2] * q + idx[1]) * q + idx[0]];
            }
            acc += s.g[bb * q + j1] * inner;
          }
        }
        tm[t] = acc;
      }
      bsync();
      const double* dfm = s.dfm + ((size_t(e) * 2 * d + fc) * nqf) * nc * nc;
      const double* fw = s.face_w + (size_t(e) * 2 * d + fc) * nqf;
      double* gq = t1;
      for (int t = threadIdx.x; t < nc * nqf; t += blockDim.x) {
        const int r = t / nqf, qf = t % nqf;
        double acc = 0.0;
        if (!s.small)
          for (int c = 0; c < nc; ++c) acc += dfm[size_t(qf) * nc * nc + r * nc + c] * tm[c * nqf + qf];
        else
          acc = dfm[size_t(qf) * nc * nc + r * nc + r] * tm[r * nqf + qf];
        gq[t] = -s.b * fw[qf] * acc;
      }
      bsync();
      const int nlay = d == 2 ? q : q * q;
      for (int t = threadIdx.x; t < nc * nlay; t += blockDim.x) {
        const int r = t / nlay, l = t % nlay;
        const double* g = gq + r * nqf;
        double acc = 0.0;
        int node;
        if (d == 2) {
          for (int a = 0; a < mu; ++a) acc += s.g[a * q + l] * g[a];
          node = axis == 0 ? l * q + layer : layer * q + l;
        } else {
          const int j0 = l % q, j1 = l / q;
          for (int bb = 0; bb < mu; ++bb) {
            double inner = 0.0;
            for (int a = 0; a < mu; ++a) inner += s.g[a * q + j0] * g[bb * mu + a];
            acc += s.g[bb * q + j1] * inner;
          }
          int idx[3];
          idx[axis] = layer;
          idx[axis == 0 ? 1 : 0] = j0;
          idx[axis == 2 ? 1 : 2] = j1;
          node = (idx[2] * q + idx[1]) * q + idx[0];
        }
        vout[r * npe + node] += acc;
      }
      bsync();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = vout[off + i];
  bsync();
  }
}

// Dense LU with partial pivoting of column-major n x n blocks (LuFactor semantics: reference
// pivot tolerance 1e-14 ||A||_inf, strict '>' first-maximum pivot choice, per-entry k order).
__global__ void __launch_bounds__(1024) dense_lu_kernel(int n, double* lu_all, int* piv_all, int* status) {
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ double tol_sh;
  __shared__ int piv_sh;
  double* lu = lu_all + size_t(blockIdx.x) * n * n;
  int* perm = piv_all + size_t(blockIdx.x) * n;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
#define A(i, j) lu[size_t(j) * n + (i)]
  for (int i = tid; i < n; i += nt) perm[i] = i;
  // ||A||_inf: row sums in order
  double m = 0.0;
  for (int i = tid; i < n; i += nt) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += fabs(A(i, j));
    m = fmax(m, s);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red_v[wid] = m;
  __syncthreads();
  if (tid == 0) {
    double mm = 0.0;
    for (int w = 0; w < nw; ++w) mm = fmax(mm, red_v[w]);
    tol_sh = 1e-14 * fmax(mm, 1e-300);
  }
  __syncthreads();
  const double tol = tol_sh;
  for (int k = 0; k < n; ++k) {
    // first maximum of |A(i,k)|, i >= k
    double best = -1.0;
    int bi = n;
    for (int i = k + tid; i < n; i += nt) {
      const double v = fabs(A(i, k));
      if (v > best) {
        best = v;
        bi = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      red_v[wid] = best;
      red_i[wid] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double bv = red_v[0];
      int bix = red_i[0];
      for (int w = 1; w < nw; ++w)
        if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < bix)) {
          bv = red_v[w];
          bix = red_i[w];
        }
      if (bv < tol) {
        atomicExch(status, int(TPDG_SINGULAR));
        bix = k;
      }
      piv_sh = bix;
      if (bix != k) {
        const int t = perm[k];
        perm[k] = perm[bix];
        perm[bix] = t;
      }
    }
    __syncthreads();
    const int piv = piv_sh;
    if (piv != k)
      for (int j = tid; j < n; j += nt) {
        const double t = A(k, j);
        A(k, j) = A(piv, j);
        A(piv, j) = t;
      }
    __syncthreads();
    const double inv = 1.0 / A(k, k);
    for (int i = k + 1 + tid; i < n; i += nt) A(i, k) = A(i, k) * inv;
    __syncthreads();
    const int rem = n - k - 1;
    for (int j = k + 1 + wid; j < n; j += nw) {  // column j: warp-strided, coalesced along i
      const double ukj = A(k, j);
      for (int i = k + 1 + lane; i < n; i += 32) A(i, j) -= A(i, k) * ukj;
    }
    (void)rem;
    __syncthreads();
  }
#undef A
}

// Test hook: one element's shuffled product.
__global__ void __launch_bounds__(kFormThreads) shuffled_kernel(DevSys s, int e, int comp, int transpose,
                                                                 const double* in, double* out, double* ws) {
  const CtaGroup g;
  ShufCtx k;
  k.s = s;
  k.e = e;
  k.comp = comp;
  k.ncb = s.small ? 1 : s.n_c;
  if (s.dim == 2) {
    if (transpose) shuf_apply_t_2d_dev(g, k, in, out, ws); else shuf_apply_2d_dev(g, k, in, out, ws);
  } else {
    if (transpose) shuf_apply_t_3d_dev(g, k, in, out, ws); else shuf_apply_3d_dev(g, k, in, out, ws);
  }
}

} // namespace

size_t shuffled_scratch_doubles(const DevSys& s) {
  return shuffled_ws_doubles(s.dim, s.q, s.mu, s.small ? 1 : s.n_c);
}

void launch_shuffled(const DevSys& s, int e, int comp, int transpose, const double* in, double* out, double* scratch,
                     cudaStream_t st) {
  shuffled_kernel<<<1, kFormThreads, 0, st>>>(s, e, comp, transpose, in, out, scratch);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

size_t lanczos_work_doubles(const DevSys& s, int max_it) {
  const int q = s.q, ncb = s.small ? 1 : s.n_c, m1 = ncb * q, m2 = s.dim == 2 ? q : q * q;
  const long rows = long(m1) * m1, cols = long(m2) * m2;
  const size_t opws = shuffled_scratch_doubles(s);
  const int J = max_it;
  size_t w = lz_work_doubles(J, rows, cols, opws);
  // factor outputs after opws: 2D: 2 m1^2 + 2 q^2 + 2 ; 3D: m1^2 + 2 m2^2 + 4 q^2 + 4
  w += 2 * size_t(m1) * m1 + 2 * size_t(m2) * m2 + 8 * size_t(q) * q + 16;
  return w;
}

void launch_lanczos_form(const DevSys& s, const tpdg_gpu_ksvd_config& cfg, const double* start_vec,
                         const double* start_vec2, double* raw, double* sigma, int* kind, double* work,
                         size_t work_per_block, int grid, cudaStream_t st) {
  (void)sigma;
  const int nblk = s.n_local * (s.small ? s.n_c : 1);
  lanczos_form_kernel<WarpGroup><<<grid, kFormThreads, 0, st>>>(s, cfg, start_vec, start_vec2, raw, kind, work,
                                                      work_per_block, nblk);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

void launch_make_factors(int dim, int q, int n1, int nblk, const double* raw, double* rec, int* piv, int* kind,
                         double* work, cudaStream_t st) {
  // One warp per block with a global (L1-resident) working set (work holds make_factors_work_groups() x
  // (4 max(n1, q) + 16) doubles), four 8-warp CTAs per SM: the Francis QR sweeps are dependent chains, so
  // resident warps matter more than access latency (a shared-memory working set with one CTA per SM
  // measured 10.5 vs 5.3 ms at cfg2 p = 15).
  const int grid = std::min((nblk + kMaxGroups - 1) / kMaxGroups, 148 * kFormGlobalCtas);
  make_factors_kernel<false, WarpGroup><<<grid, kFormThreads, 0, st>>>(dim, q, n1, nblk, const_cast<double*>(raw),
                                                                      rec, piv, kind, work);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

int make_factors_work_groups() { return 148 * kFormGlobalCtas * kMaxGroups; }

size_t probe_work_doubles(const DevSys& s) {
  const size_t nfull = size_t(s.n_c) * s.npe;
  return nfull + size_t(s.n_c) * s.nqv + s.nqv + 2 * size_t(s.nqv) * s.q + nfull + size_t(s.q) * s.mu * s.mu * 2 + 64;
}

int probe_grid(int n, int nfb) {
  const long total = long(n) * nfb;
  return int(total < 148 * 4 ? total : 148 * 4);
}

void launch_assemble_fallback(const DevSys& s, const int* blocks, int nfb, double* fb_lu, double* work,
                              cudaStream_t st) {
  const int n = s.small ? s.npe : s.n_c * s.npe;
  probe_kernel<<<probe_grid(n, nfb), kFormThreads, 0, st>>>(s, blocks, nfb, fb_lu, work, probe_work_doubles(s));
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

// Blocked variant of dense_lu_kernel with the same operations in the same order per entry
// (LuFactor, tensor/small_matrix.hpp:143-172: partial pivoting with full-row swaps, multipliers
// a_ik * (1 / a_kk), rank-1 updates a_ij -= l_ik u_kj in k order, separate mul / sub roundings).
// Columns are processed in panels of KB: the panel is factored right-looking (its rows swapped at
// each step), the panel's swaps are then applied to the other columns, and the trailing columns
// receive the panel's KB rank-1 updates in k order in one pass (U-block rows first, by shuffles
// inside the column's warp; then the rows below with the panel's multipliers staged in shared
// memory). Each trailing entry sees exactly the unblocked sequence; the trailing matrix streams
// once per panel instead of once per pivot (p = 30: 961^2 blocks).
template <int KB>
__global__ void __launch_bounds__(1024) dense_lu_blocked_kernel(int n, double* lu_all, int* piv_all, int* status) {
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ double tol_sh;
  __shared__ int piv_sh, piv_blk[KB];
  extern __shared__ double Ls[];  // panel multipliers, [kk][i - k0] (n - k0 <= n rows)
  double* lu = lu_all + size_t(blockIdx.x) * n * n;
  int* perm = piv_all + size_t(blockIdx.x) * n;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
#define A(i, j) lu[size_t(j) * n + (i)]
  for (int i = tid; i < n; i += nt) perm[i] = i;
  double m = 0.0;
  for (int i = tid; i < n; i += nt) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += fabs(A(i, j));
    m = fmax(m, s);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red_v[wid] = m;
  __syncthreads();
  if (tid == 0) {
    double mm = 0.0;
    for (int w = 0; w < nw; ++w) mm = fmax(mm, red_v[w]);
    tol_sh = 1e-14 * fmax(mm, 1e-300);
  }
  __syncthreads();
  const double tol = tol_sh;
  for (int k0 = 0; k0 < n; k0 += KB) {
    const int kb = n - k0 < KB ? n - k0 : KB, kend = k0 + kb;
    // ---- (1) panel factorization (columns [k0, kend))
    for (int k = k0; k < kend; ++k) {
      double best = -1.0;
      int bi = n;
      for (int i = k + tid; i < n; i += nt) {
        const double v = fabs(A(i, k));
        if (v > best) {
          best = v;
          bi = i;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
          best = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        red_v[wid] = best;
        red_i[wid] = bi;
      }
      __syncthreads();
      if (tid == 0) {
        double bv = red_v[0];
        int bix = red_i[0];
        for (int w = 1; w < nw; ++w)
          if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < bix)) {
            bv = red_v[w];
            bix = red_i[w];
          }
        if (bv < tol) {
          atomicExch(status, int(TPDG_SINGULAR));
          bix = k;
        }
        piv_sh = bix;
        piv_blk[k - k0] = bix;
        if (bix != k) {
          const int t = perm[k];
          perm[k] = perm[bix];
          perm[bix] = t;
        }
      }
      __syncthreads();
      const int piv = piv_sh;
      if (piv != k)
        for (int j = k0 + tid; j < kend; j += nt) {
          const double t = A(k, j);
          A(k, j) = A(piv, j);
          A(piv, j) = t;
        }
      __syncthreads();
      const double inv = 1.0 / A(k, k);
      for (int i = k + 1 + tid; i < n; i += nt) A(i, k) = A(i, k) * inv;
      __syncthreads();
      for (int j = k + 1 + wid; j < kend; j += nw) {
        const double ukj = A(k, j);
        for (int i = k + 1 + lane; i < n; i += 32) A(i, j) -= A(i, k) * ukj;
      }
      __syncthreads();
    }
    // ---- (2) the panel's row swaps on the other columns (per column, in pivot order)
    for (int j = tid; j < n; j += nt) {
      if (j >= k0 && j < kend) continue;
      for (int kk = 0; kk < kb; ++kk) {
        const int k = k0 + kk, piv = piv_blk[kk];
        if (piv != k) {
          const double t = A(k, j);
          A(k, j) = A(piv, j);
          A(piv, j) = t;
        }
      }
    }
    // panel multipliers of the rows below the panel into shared memory
    for (int kk = 0; kk < kb; ++kk)
      for (int i = kend + tid; i < n; i += nt) Ls[size_t(kk) * (n - kend) + (i - kend)] = A(i, k0 + kk);
    __syncthreads();
    // ---- (3) trailing columns: the panel's kb rank-1 updates in k order, one warp per column
    for (int j = kend + wid; j < n; j += nw) {
      // (3a) U-block rows k0 .. kend-1 (lane kk holds row k0 + kk)
      double u = lane < kb ? A(k0 + lane, j) : 0.0;
      for (int kk = 0; kk < kb; ++kk) {
        const double ukk = __shfl_sync(0xffffffffu, u, kk);
        const double l = (lane > kk && lane < kb) ? A(k0 + lane, k0 + kk) : 0.0;
        if (lane > kk && lane < kb) u -= l * ukk;
      }
      if (lane < kb) A(k0 + lane, j) = u;
      double ub[KB];  // the column's U-block values, broadcast while the warp is converged
#pragma unroll
      for (int kk = 0; kk < KB; ++kk) ub[kk] = __shfl_sync(0xffffffffu, u, kk);
      // (3b) rows below the panel
      for (int i = kend + lane; i < n; i += 32) {
        double a = A(i, j);
#pragma unroll
        for (int kk = 0; kk < KB; ++kk)
          if (kk < kb) a -= Ls[size_t(kk) * (n - kend) + (i - kend)] * ub[kk];
        A(i, j) = a;
      }
    }
    __syncthreads();
  }
#undef A
}

void launch_dense_lu(int n, int nfb, double* fb_lu, int* fb_piv, int* fb_status, cudaStream_t st) {
  // test hook TPDG_GPU_DENSE_LU=unblocked: the unblocked kernel (one trailing pass per pivot), which the
  // blocked one must equal bit for bit (tests/test_gpu_block_jacobi.py); it also serves n > 1600
  static const bool unblocked = [] {
    const char* f = std::getenv("TPDG_GPU_DENSE_LU");
    return f && f[0] == 'u';
  }();
  constexpr int KB = 16;
  const size_t ls = sizeof(double) * size_t(KB) * size_t(n);
  if (!unblocked && ls <= 200 * 1024) {
    ensure_smem(dense_lu_blocked_kernel<KB>, ls);
    dense_lu_blocked_kernel<KB><<<nfb, 1024, ls, st>>>(n, fb_lu, fb_piv, fb_status);
  } else {
    dense_lu_kernel<<<nfb, 1024, 0, st>>>(n, fb_lu, fb_piv, fb_status);
  }
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

} // namespace tpdg_gpu
