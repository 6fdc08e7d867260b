// build_cache on the device for scalar upwind advection (reference
// ops/linearized.hpp:38-100 with the advection law's flux Jacobian / numerical-flux Jacobians,
// laws/advection.hpp:25-80). The cache is state independent for linear advection, so it is a map
// over quadrature points of the geometry:
//   dft[e][k][q] = sum_m adj[e][q][k][m] v_m(x_q)           (volume points, m ascending)
//   dfm[e][f][q] = max(v(x_q) . n_q, 0)                     (face points, upwind side)
//   dfp[e][f][q] = min(v(x_q) . n_q, 0) on interior faces, 0 on boundary faces.
// field 0 / 2: constant velocity (2D / 3D); 1: (sin 2 pi y, cos 2 pi x). Same operation order as
// the host restatement (host_setup.cpp, bit-exact vs the reference) and no FMA (-fmad=false): the
// fields reproduce it bit for bit (the swirl field's sin/cos in glibc's arithmetic, glibm.cuh).
#include <cstdint>

#include "glibm.cuh"
#include "tpdg_internal.hpp"

namespace tpdg_gpu {

namespace {

__device__ __forceinline__ void velocity(int field, const double* vel, const double* x, double* v) {
  if (field == 1) {
    v[0] = glibm_sin(2.0 * 3.14159265358979323846 * x[1]);
    v[1] = glibm_cos(2.0 * 3.14159265358979323846 * x[0]);
    v[2] = 0.0;
  } else {
    v[0] = vel[0];
    v[1] = vel[1];
    v[2] = vel[2];
  }
}

struct CacheArgs {
  int dim, n_elements, nvol, nface, field;
  double vel[3];
  const double *adj, *vol_x, *face_n, *face_x;
  const int64_t* conn;
  double *dft, *dfm, *dfp;
};

__global__ void cache_volume_kernel(CacheArgs a) {
  const int64_t total = int64_t(a.n_elements) * a.nvol;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = t / a.nvol, qv = t % a.nvol;
    double v[3];
    velocity(a.field, a.vel, a.vol_x + t * a.dim, v);
    const double* adj = a.adj + t * a.dim * a.dim;
    for (int k = 0; k < a.dim; ++k) {
      double s = 0.0;
      for (int m = 0; m < a.dim; ++m) s += adj[k * a.dim + m] * v[m];
      a.dft[(e * a.dim + k) * a.nvol + qv] = s;
    }
  }
}

__global__ void cache_face_kernel(CacheArgs a) {
  const int64_t total = int64_t(a.n_elements) * 2 * a.dim * a.nface;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t ef = t / a.nface;  // e * 2d + f
    const bool interior = a.conn[ef * 3] >= 0;
    double v[3];
    velocity(a.field, a.vel, a.face_x + t * a.dim, v);
    double vn = 0.0;
    for (int m = 0; m < a.dim; ++m) vn += v[m] * a.face_n[t * a.dim + m];
    a.dfm[t] = vn < 0.0 ? 0.0 : vn;                 // std::max(vn, 0.0)
    a.dfp[t] = interior ? (0.0 < vn ? 0.0 : vn) : 0.0;  // std::min(vn, 0.0)
  }
}

// ------------------------------------------------------------------ LLF Euler law (laws/euler.hpp)
// Restated in the reference's operation order (this file builds with -fmad=false): pressure
// (euler.hpp:29-34), flux_jacobian_dir (:37-75), wave_speed (:78-105), num_flux_jac_minus/plus
// (:164-206), boundary_state = copy (:208-210). check_state (:14-27) raises StateError via *status.
constexpr double kGamma = 1.4;

__device__ double eu_pressure(int d, const double* u) {
  const int nc = d + 2;
  double ke = 0.0;
  for (int m = 0; m < d; ++m) ke += u[1 + m] * u[1 + m];
  return (kGamma - 1.0) * (u[nc - 1] - 0.5 * ke / u[0]);
}
__device__ void eu_check(int d, const double* u, int* status) {
  const double p = eu_pressure(d, u);
  if (!(u[0] > 0.0) || !(p > 0.0)) atomicExch(status, int(TPDG_STATE));
}
__device__ void eu_flux_jacobian_dir(int d, int dir, const double* u, double* df) {
  const int nc = d + 2;
  const double inv_rho = 1.0 / u[0];
  double vel[3] = {0, 0, 0};
  double ke2 = 0.0;
  for (int m = 0; m < d; ++m) {
    vel[m] = u[1 + m] * inv_rho;
    ke2 += 0.5 * vel[m] * vel[m];
  }
  const double p = eu_pressure(d, u);
  const double h = (u[nc - 1] + p) * inv_rho;
  const double vd = vel[dir];
  double dp[5];
  dp[0] = (kGamma - 1.0) * ke2;
  for (int m = 0; m < d; ++m) dp[1 + m] = -(kGamma - 1.0) * vel[m];
  dp[nc - 1] = kGamma - 1.0;
  for (int c = 0; c < nc; ++c) df[c] = 0.0;
  df[1 + dir] = 1.0;
  for (int i = 0; i < d; ++i) {
    double* row = df + (1 + i) * nc;
    row[0] = -vel[i] * vd;
    for (int c = 1; c < nc; ++c) row[c] = 0.0;
    row[1 + i] += vd;
    row[1 + dir] += vel[i];
    if (i == dir)
      for (int c = 0; c < nc; ++c) row[c] += dp[c];
  }
  double* row = df + (nc - 1) * nc;
  row[0] = vd * (dp[0] - h);
  for (int m = 0; m < d; ++m) row[1 + m] = vd * dp[1 + m];
  row[1 + dir] += h;
  row[nc - 1] = vd * (1.0 + dp[nc - 1]);
}
__device__ double eu_wave_speed(int d, const double* u, const double* n, double* ds) {
  const int nc = d + 2;
  const double inv_rho = 1.0 / u[0];
  double mn = 0.0, ke = 0.0;
  for (int m = 0; m < d; ++m) {
    mn += u[1 + m] * n[m];
    ke += u[1 + m] * u[1 + m];
  }
  const double vn = mn * inv_rho;
  const double p = eu_pressure(d, u);
  const double c = sqrt(kGamma * p * inv_rho);
  if (ds) {
    const double sgn = vn >= 0.0 ? 1.0 : -1.0;
    const double gm1 = kGamma - 1.0;
    double dpr[5];
    dpr[0] = gm1 * (-u[nc - 1] * inv_rho * inv_rho + ke * inv_rho * inv_rho * inv_rho);
    for (int m = 0; m < d; ++m) dpr[1 + m] = -gm1 * u[1 + m] * inv_rho * inv_rho;
    dpr[nc - 1] = gm1 * inv_rho;
    ds[0] = sgn * (-vn * inv_rho) + kGamma / (2.0 * c) * dpr[0];
    for (int m = 0; m < d; ++m) ds[1 + m] = sgn * n[m] * inv_rho + kGamma / (2.0 * c) * dpr[1 + m];
    ds[nc - 1] = kGamma / (2.0 * c) * dpr[nc - 1];
  }
  return fabs(vn) + c;
}
// side 0: num_flux_jac_minus (d/du^-), 1: num_flux_jac_plus (d/du^+)
__device__ void eu_num_flux_jac(int d, int side, const double* um, const double* up, const double* n, double* out) {
  const int nc = d + 2;
  double ds[5];
  const double sm = eu_wave_speed(d, um, n, side == 0 ? ds : nullptr);
  const double sp = eu_wave_speed(d, up, n, side == 1 ? ds : nullptr);
  const double lam = sm > sp ? sm : sp;  // std::max(sm, sp)
  const double* us = side == 0 ? um : up;
  double df[3 * 25];
  for (int dir = 0; dir < d; ++dir) eu_flux_jacobian_dir(d, dir, us, df + dir * nc * nc);
  for (int r = 0; r < nc; ++r)
    for (int c = 0; c < nc; ++c) {
      double v = 0.0;
      for (int dir = 0; dir < d; ++dir) v += n[dir] * df[(dir * nc + r) * nc + c];
      v *= 0.5;
      if (r == c) v = side == 0 ? v + 0.5 * lam : v - 0.5 * lam;
      if (side == 0 ? sm >= sp : sm < sp) v += 0.5 * (um[r] - up[r]) * ds[c];
      out[r * nc + c] = v;
    }
}

// dst[o][i'][inner] = sum_j M(i', j) src[o][j][inner] (kernels::axis_apply, kernels.hpp:11-32: j ascending
// from +0, zero entries skipped), parallel over the outputs.
__device__ void eu_axis_apply(const double* m, int nout, int nin, int inner, int outer, const double* src, double* dst) {
  const int total = outer * nout * inner;
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int q = t % inner, i = (t / inner) % nout, o = t / (inner * nout);
    double s = 0.0;
    for (int j = 0; j < nin; ++j) {
      const double mij = m[i * nin + j];
      if (mij == 0.0) continue;
      s += mij * src[(o * nin + j) * inner + q];
    }
    dst[t] = s;
  }
}

// face_trace (ops/discretization.hpp:89-129) of a component's coefficients at face f, first tangential
// axis fastest; one thread per output point (qf < nqf), tmp: q^2 doubles (3D).
__device__ double eu_face_trace_point(int d, int q, int mu, const double* g, int f, const double* coeff, int qf) {
  const int axis = f / 2, layer = (f % 2) == 0 ? 0 : q - 1;
  if (d == 2) {
    double s = 0.0;
    for (int j = 0; j < q; ++j) s += g[qf * q + j] * (axis == 0 ? coeff[j * q + layer] : coeff[layer * q + j]);
    return s;
  }
  const int t0 = axis == 0 ? 1 : 0, t1 = axis == 2 ? 1 : 2;
  const int a = qf % mu, b = qf / mu;
  double vb = 0.0;
  for (int j1 = 0; j1 < q; ++j1) {
    double sa = 0.0;  // ws.a[j1 * mu + a]
    for (int j0 = 0; j0 < q; ++j0) {
      int idx[3];
      idx[axis] = layer;
      idx[t0] = j0;
      idx[t1] = j1;
      sa += g[a * q + j0] * coeff[(idx[2] * q + idx[1]) * q + idx[0]];
    }
    vb += g[b * q + j1] * sa;
  }
  return vb;
}

// build_cache (ops/linearized.hpp:38-100) of one element per CTA.
__global__ void cache_euler_kernel(int d, int q, int mu, const double* __restrict__ g, const double* __restrict__ state,
                                   const double* __restrict__ adj, const double* __restrict__ face_n,
                                   const int64_t* __restrict__ conn, double* __restrict__ dft,
                                   double* __restrict__ dfm, double* __restrict__ dfp, int* status) {
  extern __shared__ double cs[];
  const int e = blockIdx.x, nc = d + 2;
  const int npe = d == 2 ? q * q : q * q * q, nqv = d == 2 ? mu * mu : mu * mu * mu, nqf = nqv / mu;
  double* vals = cs;                       // [c][nqv]
  double* w1 = vals + nc * nqv;            // axis-apply scratch: mu q^(d-1) (per component)
  double* w2 = w1 + mu * q * q;            // mu^2 q (3D)
  double* tr = w2 + mu * mu * q;           // [side][c][nqf]
  const double* ue = state + size_t(e) * nc * npe;
  for (int c = 0; c < nc; ++c) {  // eval_at_quad (kernels.hpp:60-78)
    const double* coeff = ue + size_t(c) * npe;
    if (d == 2) {
      eu_axis_apply(g, mu, q, 1, q, coeff, w1);
      __syncthreads();
      eu_axis_apply(g, mu, q, mu, 1, w1, vals + c * nqv);
    } else {
      eu_axis_apply(g, mu, q, 1, q * q, coeff, w1);
      __syncthreads();
      eu_axis_apply(g, mu, q, mu, q, w1, w2);
      __syncthreads();
      eu_axis_apply(g, mu, q, mu * mu, 1, w2, vals + c * nqv);
    }
    __syncthreads();
  }
  for (int qv = threadIdx.x; qv < nqv; qv += blockDim.x) {
    double uq[5], df[3 * 25];
    for (int c = 0; c < nc; ++c) uq[c] = vals[c * nqv + qv];
    eu_check(d, uq, status);
    for (int m = 0; m < d; ++m) eu_flux_jacobian_dir(d, m, uq, df + m * nc * nc);
    const double* a = adj + (size_t(e) * nqv + qv) * d * d;
    for (int k = 0; k < d; ++k)
      for (int r = 0; r < nc; ++r)
        for (int c = 0; c < nc; ++c) {
          double s = 0.0;
          for (int m = 0; m < d; ++m) s += a[k * d + m] * df[(m * nc + r) * nc + c];
          dft[((size_t(e) * d + k) * nqv + qv) * nc * nc + r * nc + c] = s;
        }
  }
  for (int f = 0; f < 2 * d; ++f) {
    const int64_t* fc = conn + (size_t(e) * 2 * d + f) * 3;
    const bool interior = fc[0] >= 0;
    __syncthreads();
    for (int t = threadIdx.x; t < nc * nqf; t += blockDim.x) {
      const int c = t / nqf, qf = t % nqf;
      tr[t] = eu_face_trace_point(d, q, mu, g, f, ue + size_t(c) * npe, qf);
      if (interior) {  // neighbor_trace (discretization.hpp:170-181): oriented into this face's enumeration
        const int code = int(fc[2]);
        int qa, qb;
        if (d == 2) {
          qa = code == 0 ? qf : mu - 1 - qf;
          qb = 0;
        } else {
          const int a0 = qf % mu, b0 = qf / mu;
          int u = (code & 4) ? b0 : a0, v = (code & 4) ? a0 : b0;
          if (code & 1) u = mu - 1 - u;
          if (code & 2) v = mu - 1 - v;
          qa = u;
          qb = v;
        }
        const double* un = state + (size_t(fc[0]) * nc + c) * npe;
        tr[nc * nqf + t] = eu_face_trace_point(d, q, mu, g, int(fc[1]), un, (d == 3 ? qb * mu : 0) + qa);
      }
    }
    __syncthreads();
    for (int qf = threadIdx.x; qf < nqf; qf += blockDim.x) {
      double um[5], up[5];
      for (int c = 0; c < nc; ++c) {
        um[c] = tr[c * nqf + qf];
        up[c] = interior ? tr[nc * nqf + c * nqf + qf] : um[c];  // boundary_state: copy
      }
      const double* n = face_n + ((size_t(e) * 2 * d + f) * nqf + qf) * d;
      const size_t o = ((size_t(e) * 2 * d + f) * nqf + qf) * nc * nc;
      eu_check(d, um, status);
      eu_num_flux_jac(d, 0, um, up, n, dfm + o);
      if (interior) {
        eu_check(d, up, status);
        eu_num_flux_jac(d, 1, um, up, n, dfp + o);
      } else {
        for (int k = 0; k < nc * nc; ++k) dfp[o + k] = 0.0;
      }
    }
  }
}

// ------------------------------------------------------------------ residual r(u, t) of the Euler law
// ops/discretization.hpp:188-254: volume fluxes contracted with the adjugate and integrated against the
// test-function gradients (integrate_back, kernels.hpp:82-104), minus the lifted LLF numerical flux
// (face_lift, discretization.hpp:133-166). Per output entry the reference's accumulation sequence:
// out = 0; += the d volume terms (k ascending); += the 2d face lifts (f ascending).
__device__ void eu_flux(int d, const double* u, double* f) {  // laws/euler.hpp:125-136, F[dir][c]
  const int nc = d + 2;
  const double inv_rho = 1.0 / u[0];
  const double p = eu_pressure(d, u);
  for (int dir = 0; dir < d; ++dir) {
    const double vd = u[1 + dir] * inv_rho;
    double* fd = f + dir * nc;
    fd[0] = u[1 + dir];
    for (int i = 0; i < d; ++i) fd[1 + i] = u[1 + i] * vd;
    fd[1 + dir] += p;
    fd[nc - 1] = (u[nc - 1] + p) * vd;
  }
}
__device__ void eu_num_flux(int d, const double* um, const double* up, const double* n, double* fhat) {
  const int nc = d + 2;  // laws/euler.hpp:138-162
  const double sm = eu_wave_speed(d, um, n, nullptr), sp = eu_wave_speed(d, up, n, nullptr);
  const double lam = sm > sp ? sm : sp;
  double fm[5], fp[5];
  const double invm = 1.0 / um[0], invp = 1.0 / up[0];
  const double pm = eu_pressure(d, um), pp = eu_pressure(d, up);
  for (int c = 0; c < nc; ++c) fhat[c] = 0.0;
  for (int dir = 0; dir < d; ++dir) {
    const double vdm = um[1 + dir] * invm, vdp = up[1 + dir] * invp;
    fm[0] = um[1 + dir];
    fp[0] = up[1 + dir];
    for (int i = 0; i < d; ++i) {
      fm[1 + i] = um[1 + i] * vdm;
      fp[1 + i] = up[1 + i] * vdp;
    }
    fm[1 + dir] += pm;
    fp[1 + dir] += pp;
    fm[nc - 1] = (um[nc - 1] + pm) * vdm;
    fp[nc - 1] = (up[nc - 1] + pp) * vdp;
    for (int c = 0; c < nc; ++c) fhat[c] += 0.5 * n[dir] * (fm[c] + fp[c]);
  }
  for (int c = 0; c < nc; ++c) fhat[c] += 0.5 * lam * (um[c] - up[c]);
}

// One element per CTA. Shared: vals [c][nqv] (reused for ft), scratch, out [c][npe], face buffers.
__global__ void residual_euler_kernel(int d, int q, int mu, const double* __restrict__ g,
                                      const double* __restrict__ gw, const double* __restrict__ dw,
                                      const double* __restrict__ state, const double* __restrict__ adj,
                                      const double* __restrict__ face_n, const double* __restrict__ face_w,
                                      const int64_t* __restrict__ conn, double* __restrict__ out, int* status) {
  extern __shared__ double rs[];
  const int e = blockIdx.x, nc = d + 2;
  const int npe = d == 2 ? q * q : q * q * q, nqv = d == 2 ? mu * mu : mu * mu * mu, nqf = nqv / mu;
  double* vals = rs;                 // [c][nqv]
  double* ft = vals + nc * nqv;      // [k][c][nqv]
  double* w1 = ft + d * nc * nqv;    // mu q^2 (>= q mu^2 for the back integration)
  double* w2 = w1 + mu * mu * q;     // mu^2 q
  double* acc = w2 + mu * mu * q;    // [c][npe]
  double* lift = acc + nc * npe;     // [c][nqf]
  double* tr = lift + nc * nqf;      // [side][c][nqf]
  const double* ue = state + size_t(e) * nc * npe;
  for (int c = 0; c < nc; ++c) {  // eval_at_quad
    const double* coeff = ue + size_t(c) * npe;
    if (d == 2) {
      eu_axis_apply(g, mu, q, 1, q, coeff, w1);
      __syncthreads();
      eu_axis_apply(g, mu, q, mu, 1, w1, vals + c * nqv);
    } else {
      eu_axis_apply(g, mu, q, 1, q * q, coeff, w1);
      __syncthreads();
      eu_axis_apply(g, mu, q, mu, q, w1, w2);
      __syncthreads();
      eu_axis_apply(g, mu, q, mu * mu, 1, w2, vals + c * nqv);
    }
    __syncthreads();
  }
  for (int qv = threadIdx.x; qv < nqv; qv += blockDim.x) {
    double uq[5], fq[15];
    for (int c = 0; c < nc; ++c) uq[c] = vals[c * nqv + qv];
    eu_check(d, uq, status);
    eu_flux(d, uq, fq);
    const double* a = adj + (size_t(e) * nqv + qv) * d * d;
    for (int k = 0; k < d; ++k)
      for (int c = 0; c < nc; ++c) {
        double s = 0.0;
        for (int m = 0; m < d; ++m) s += a[k * d + m] * fq[m * nc + c];
        ft[(k * nc + c) * nqv + qv] = s;
      }
  }
  for (int i = threadIdx.x; i < nc * npe; i += blockDim.x) acc[i] = 0.0;
  __syncthreads();
  for (int k = 0; k < d; ++k)  // integrate_back(gw, dw, d, dslot = k): M_0 along x, M_1 along y (, M_2 along z)
    for (int c = 0; c < nc; ++c) {
      const double* field = ft + (k * nc + c) * nqv;
      const double* m0 = k == 0 ? dw : gw;
      const double* m1 = k == 1 ? dw : gw;
      if (d == 2) {
        eu_axis_apply(m0, q, mu, 1, mu, field, w1);
        __syncthreads();
        for (int t = threadIdx.x; t < npe; t += blockDim.x) {  // second pass fused with out += ws.d
          const int i = t % q, j = t / q;
          double s = 0.0;
          for (int b = 0; b < mu; ++b) {
            const double mij = m1[j * mu + b];
            if (mij == 0.0) continue;
            s += mij * w1[b * q + i];
          }
          acc[c * npe + t] += s;
        }
      } else {
        const double* m2 = k == 2 ? dw : gw;
        eu_axis_apply(m0, q, mu, 1, mu * mu, field, w1);
        __syncthreads();
        eu_axis_apply(m1, q, mu, q, mu, w1, w2);
        __syncthreads();
        for (int t = threadIdx.x; t < npe; t += blockDim.x) {
          const int ij = t % (q * q), l = t / (q * q);
          double s = 0.0;
          for (int b = 0; b < mu; ++b) {
            const double mij = m2[l * mu + b];
            if (mij == 0.0) continue;
            s += mij * w2[b * q * q + ij];
          }
          acc[c * npe + t] += s;
        }
      }
      __syncthreads();
    }
  for (int f = 0; f < 2 * d; ++f) {
    const int64_t* fc = conn + (size_t(e) * 2 * d + f) * 3;
    const bool interior = fc[0] >= 0;
    for (int t = threadIdx.x; t < nc * nqf; t += blockDim.x) {
      const int c = t / nqf, qf = t % nqf;
      tr[t] = eu_face_trace_point(d, q, mu, g, f, ue + size_t(c) * npe, qf);
      if (interior) {
        const int code = int(fc[2]);
        int qa, qb;
        if (d == 2) {
          qa = code == 0 ? qf : mu - 1 - qf;
          qb = 0;
        } else {
          const int a0 = qf % mu, b0 = qf / mu;
          int u = (code & 4) ? b0 : a0, v = (code & 4) ? a0 : b0;
          if (code & 1) u = mu - 1 - u;
          if (code & 2) v = mu - 1 - v;
          qa = u;
          qb = v;
        }
        const double* un = state + (size_t(fc[0]) * nc + c) * npe;
        tr[nc * nqf + t] = eu_face_trace_point(d, q, mu, g, int(fc[1]), un, (d == 3 ? qb * mu : 0) + qa);
      }
    }
    __syncthreads();
    for (int qf = threadIdx.x; qf < nqf; qf += blockDim.x) {
      double um[5], up[5], fh[5];
      for (int c = 0; c < nc; ++c) {
        um[c] = tr[c * nqf + qf];
        up[c] = interior ? tr[nc * nqf + c * nqf + qf] : um[c];
      }
      eu_check(d, um, status);
      eu_check(d, up, status);
      const size_t fq = (size_t(e) * 2 * d + f) * nqf + qf;
      eu_num_flux(d, um, up, face_n + fq * d, fh);
      for (int c = 0; c < nc; ++c) lift[c * nqf + qf] = -face_w[fq] * fh[c];
    }
    __syncthreads();
    // face_lift (discretization.hpp:133-166) into the face node layer
    const int axis = f / 2, layer = (f % 2) == 0 ? 0 : q - 1;
    if (d == 2) {
      for (int t = threadIdx.x; t < nc * q; t += blockDim.x) {
        const int c = t / q, j = t % q;
        double s = 0.0;
        for (int a = 0; a < mu; ++a) s += g[a * q + j] * lift[c * nqf + a];
        acc[c * npe + (axis == 0 ? j * q + layer : layer * q + j)] += s;
      }
    } else {
      const int t0 = axis == 0 ? 1 : 0, t1 = axis == 2 ? 1 : 2;
      for (int t = threadIdx.x; t < nc * q * q; t += blockDim.x) {
        const int c = t / (q * q), j0 = t % q, j1 = (t / q) % q;
        double s = 0.0;
        for (int b = 0; b < mu; ++b) {
          double sa = 0.0;  // ws.a[j0 * mu + b]
          for (int a = 0; a < mu; ++a) sa += g[a * q + j0] * lift[c * nqf + b * mu + a];
          s += g[b * q + j1] * sa;
        }
        int idx[3];
        idx[axis] = layer;
        idx[t0] = j0;
        idx[t1] = j1;
        acc[c * npe + (idx[2] * q + idx[1]) * q + idx[0]] += s;
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < nc * npe; i += blockDim.x) out[size_t(e) * nc * npe + i] = acc[i];
}

// Test hook: fn 0 sin, 1 cos, 2 atan, 3 atan2(x, y) of glibm.cuh over n arguments.
__global__ void libm_eval_kernel(int fn, int64_t n, const double* x, const double* y, double* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double a = x[i];
    out[i] = fn == 0 ? glibm_sin(a) : fn == 1 ? glibm_cos(a) : fn == 2 ? glibm_atan(a) : glibm_atan2(a, y[i]);
  }
}

} // namespace

void launch_libm_eval(int fn, int64_t n, const double* x, const double* y, double* out, cudaStream_t st) {
  libm_eval_kernel<<<148 * 8, 256, 0, st>>>(fn, n, x, y, out);
  TPDG_CUDA_CHECK(cudaGetLastError());
  g_launches += 1;
}

void launch_build_cache_euler(int dim, int q, int mu, int n_elements, const double* g, const double* state,
                              const double* adj, const double* face_n, const int64_t* conn, double* dft, double* dfm,
                              double* dfp, int* status, cudaStream_t st) {
  const int nc = dim + 2, nqv = dim == 2 ? mu * mu : mu * mu * mu, nqf = nqv / mu;
  const size_t smem = sizeof(double) * (size_t(nc) * nqv + size_t(mu) * q * q + size_t(mu) * mu * q + 2 * nc * nqf);
  ensure_smem(cache_euler_kernel, smem);
  if (n_elements) cache_euler_kernel<<<n_elements, 256, smem, st>>>(dim, q, mu, g, state, adj, face_n, conn, dft, dfm,
                                                                    dfp, status);
  TPDG_CUDA_CHECK(cudaGetLastError());
  g_launches += 1;
}

void launch_residual_euler(int dim, int q, int mu, int n_elements, const double* g, const double* gw, const double* dw,
                           const double* state, const double* adj, const double* face_n, const double* face_w,
                           const int64_t* conn, double* out, int* status, cudaStream_t st) {
  const int nc = dim + 2, nqv = dim == 2 ? mu * mu : mu * mu * mu, nqf = nqv / mu;
  const int npe = dim == 2 ? q * q : q * q * q;
  const size_t smem = sizeof(double) * (size_t(nc) * nqv * (1 + dim) + 2 * size_t(mu) * mu * q + size_t(nc) * npe +
                                        3 * size_t(nc) * nqf);
  ensure_smem(residual_euler_kernel, smem);
  if (n_elements)
    residual_euler_kernel<<<n_elements, 256, smem, st>>>(dim, q, mu, g, gw, dw, state, adj, face_n, face_w, conn, out,
                                                         status);
  TPDG_CUDA_CHECK(cudaGetLastError());
  g_launches += 1;
}

void launch_build_cache_advection(int dim, int n_elements, int nvol, int nface, const double* adj,
                                  const double* vol_x, const double* face_n, const double* face_x,
                                  const int64_t* conn, int field, const double* vel, double* dft, double* dfm,
                                  double* dfp, cudaStream_t st) {
  CacheArgs a{dim, n_elements, nvol, nface, field, {vel[0], vel[1], dim == 3 ? vel[2] : 0.0}, adj, vol_x, face_n,
              face_x, conn, dft, dfm, dfp};
  cache_volume_kernel<<<148 * 8, 256, 0, st>>>(a);
  TPDG_CUDA_CHECK(cudaGetLastError());
  cache_face_kernel<<<148 * 8, 256, 0, st>>>(a);
  TPDG_CUDA_CHECK(cudaGetLastError());
  g_launches += 2;
}

} // namespace tpdg_gpu
