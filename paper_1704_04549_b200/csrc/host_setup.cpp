// Host-side input production for the BASELINE configurations (outside the kernel scope;
// SURVEY.md sec.2 marks reference element / mesh / laws as host setup whose matrices are
// uploaded once). Restates, in the reference's operation order (built with
// -ffp-contract=off, so the arrays match the reference's bit for bit):
//   legendre / gauss_rule / gauss_lobatto_rule / lagrange_*  dg/quadrature.hpp:10-114
//   build_reference                                           dg/reference_element.hpp:43-84
//   generate_mesh (cartesian) + MeshGeometry::precompute      dg/mesh.hpp:111-355
//   build_cache for scalar advection (upwind)                 ops/linearized.hpp:38-100,
//                                                              laws/advection.hpp:25-80
#include <array>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "tpdg_gpu.h"
#include "tpdg_internal.hpp"

namespace tpdg_gpu {
namespace {

std::pair<double, double> legendre(int n, double x) {
  double p0 = 1.0, p1 = x;
  if (n == 0) return {1.0, 0.0};
  for (int k = 1; k < n; ++k) {
    const double p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
    p0 = p1;
    p1 = p2;
  }
  const double dp = (std::abs(x) < 1.0) ? n * (x * p1 - p0) / (x * x - 1.0)
                                        : 0.5 * n * (n + 1) * (x >= 1.0 ? 1.0 : (n % 2 ? 1.0 : -1.0));
  return {p1, dp};
}

void gauss(int n, std::vector<double>& pts, std::vector<double>& wts) {
  pts.assign(n, 0.0);
  wts.assign(n, 0.0);
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      const auto pr = legendre(n, x);
      const double dx = pr.first / pr.second;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    const double dp = legendre(n, x).second;
    const double w = 2.0 / ((1.0 - x * x) * dp * dp);
    pts[i] = 0.5 * (1.0 - x);
    pts[n - 1 - i] = 0.5 * (1.0 + x);
    wts[i] = 0.5 * w;
    wts[n - 1 - i] = 0.5 * w;
  }
}

std::vector<double> lobatto_points(int n) {
  const int m = n - 1;
  std::vector<double> pts(n, 0.0);
  pts[0] = 0.0;
  pts[n - 1] = 1.0;
  for (int i = 1; i < n - 1; ++i) {
    double x = std::cos(M_PI * i / m);
    for (int it = 0; it < 100; ++it) {
      const auto pr = legendre(m, x);
      const double ddp = (2.0 * x * pr.second - m * (m + 1) * pr.first) / (1.0 - x * x);
      const double dx = pr.second / ddp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    pts[n - 1 - i] = 0.5 * (1.0 + x);
  }
  return pts;
}

double lag_value(const std::vector<double>& nodes, int j, double x) {
  double v = 1.0;
  for (int k = 0; k < int(nodes.size()); ++k) {
    if (k == j) continue;
    v *= (x - nodes[k]) / (nodes[j] - nodes[k]);
  }
  return v;
}

double lag_derivative(const std::vector<double>& nodes, int j, double x) {
  const int n = int(nodes.size());
  double denom = 1.0;
  for (int k = 0; k < n; ++k)
    if (k != j) denom *= nodes[j] - nodes[k];
  double sum = 0.0;
  for (int l = 0; l < n; ++l) {
    if (l == j) continue;
    double prod = 1.0;
    for (int k = 0; k < n; ++k)
      if (k != j && k != l) prod *= x - nodes[k];
    sum += prod;
  }
  return sum / denom;
}

struct Geometry {
  int dim = 2, n_elements = 0, mu = 0, nvol = 0, nface = 0;
  std::vector<std::array<double, 3>> nodes;
  std::vector<std::array<int, 8>> elem_nodes;
  std::vector<double> map1d{0.0, 1.0};

  void map_point(int e, const double* xi, double* x) const {
    double shape[3][2];
    for (int a = 0; a < dim; ++a)
      for (int i = 0; i < 2; ++i) shape[a][i] = lag_value(map1d, i, xi[a]);
    for (int m = 0; m < dim; ++m) x[m] = 0.0;
    const int npts = dim == 2 ? 4 : 8;
    for (int idx = 0; idx < npts; ++idx) {
      int rem = idx;
      double s = 1.0;
      for (int a = 0; a < dim; ++a) {
        s *= shape[a][rem % 2];
        rem /= 2;
      }
      for (int m = 0; m < dim; ++m) x[m] += s * nodes[elem_nodes[e][idx]][m];
    }
  }

  void map_jacobian(int e, const double* xi, double* jac) const {
    double shape[3][2], dshape[3][2];
    for (int a = 0; a < dim; ++a)
      for (int i = 0; i < 2; ++i) {
        shape[a][i] = lag_value(map1d, i, xi[a]);
        dshape[a][i] = lag_derivative(map1d, i, xi[a]);
      }
    for (int i = 0; i < dim * dim; ++i) jac[i] = 0.0;
    const int npts = dim == 2 ? 4 : 8;
    for (int idx = 0; idx < npts; ++idx)
      for (int k = 0; k < dim; ++k) {
        int rem = idx;
        double s = 1.0;
        for (int a = 0; a < dim; ++a) {
          s *= (a == k) ? dshape[a][rem % 2] : shape[a][rem % 2];
          rem /= 2;
        }
        for (int m = 0; m < dim; ++m) jac[m * dim + k] += s * nodes[elem_nodes[e][idx]][m];
      }
  }

  double adjugate(const double* jac, double* out) const {
    if (dim == 2) {
      const double a = jac[0], b = jac[1], c = jac[2], d = jac[3];
      out[0] = d;
      out[1] = -b;
      out[2] = -c;
      out[3] = a;
      return a * d - b * c;
    }
    auto J = [&](int m, int k) { return jac[m * 3 + k]; };
    out[0] = J(1, 1) * J(2, 2) - J(1, 2) * J(2, 1);
    out[1] = -(J(0, 1) * J(2, 2) - J(0, 2) * J(2, 1));
    out[2] = J(0, 1) * J(1, 2) - J(0, 2) * J(1, 1);
    out[3] = -(J(1, 0) * J(2, 2) - J(1, 2) * J(2, 0));
    out[4] = J(0, 0) * J(2, 2) - J(0, 2) * J(2, 0);
    out[5] = -(J(0, 0) * J(1, 2) - J(0, 2) * J(1, 0));
    out[6] = J(1, 0) * J(2, 1) - J(1, 1) * J(2, 0);
    out[7] = -(J(0, 0) * J(2, 1) - J(0, 1) * J(2, 0));
    out[8] = J(0, 0) * J(1, 1) - J(0, 1) * J(1, 0);
    return J(0, 0) * out[0] + J(0, 1) * out[3] + J(0, 2) * out[6];
  }
};

void face_tangents(int dim, int axis, int* t) {
  if (dim == 2) {
    t[0] = axis == 0 ? 1 : 0;
    t[1] = -1;
  } else {
    t[0] = axis == 0 ? 1 : 0;
    t[1] = axis == 2 ? 1 : 2;
  }
}

} // namespace

namespace {
// Linearization states of the Euler stand-ins (BASELINE.json configs[2] / configs[4], inviscid): the
// reference interpolates a pointwise state onto the nodes (ops/discretization.hpp:356-375). cfg3:
// rho = 1 + 0.2 exp(-r^2/2) about the centre of [0,10]^2, velocity (1, 1) plus the tangential swirl
// 0.5 r exp((1 - r^2)/2), pressure from the isentropic relation p = rho^gamma. cfg5: Taylor-Green on
// [0, 2 pi]^3 at Mach 0.1 (rho = 1, p0 = 1 / (gamma M^2)). gamma = 1.4. The same expressions are in
// oracle/ref_driver.cpp (the reference's own interpolate), so the states agree bit for bit.
void euler_state(int kind, const double* x, double* u) {
  const double gamma = 1.4;
  if (kind == 3) {
    const double dx = x[0] - 5.0, dy = x[1] - 5.0;
    const double r2 = dx * dx + dy * dy;
    const double rho = 1.0 + 0.2 * std::exp(-0.5 * r2);
    const double sw = 0.5 * std::exp(0.5 * (1.0 - r2));  // swirl speed / r
    const double vx = 1.0 - sw * dy, vy = 1.0 + sw * dx;
    const double pr = std::pow(rho, gamma);
    u[0] = rho;
    u[1] = rho * vx;
    u[2] = rho * vy;
    u[3] = pr / (gamma - 1.0) + 0.5 * rho * (vx * vx + vy * vy);
  } else {
    const double mach = 0.1, p0 = 1.0 / (gamma * mach * mach);
    const double vx = std::sin(x[0]) * std::cos(x[1]) * std::cos(x[2]);
    const double vy = -std::cos(x[0]) * std::sin(x[1]) * std::cos(x[2]);
    const double pr = p0 + (std::cos(2.0 * x[0]) + std::cos(2.0 * x[1])) * (std::cos(2.0 * x[2]) + 2.0) / 16.0;
    u[0] = 1.0;
    u[1] = vx;
    u[2] = vy;
    u[3] = 0.0;
    u[4] = pr / (gamma - 1.0) + 0.5 * (vx * vx + vy * vy);
  }
}
} // namespace

int setup_advection(int kind, const double* vel, int nx, int ny, int nz, int p, int periodic, Setup& S) {
  const bool euler = kind == 3 || kind == 5;
  const int dim = kind == 2 || kind == 5 ? 3 : 2;
  const double lo = 0.0, hi = kind == 3 ? 10.0 : kind == 5 ? 2.0 * M_PI : 1.0;
  const int n = p + 1, mu = p + 2;
  S.dim = dim;
  S.n_c = 1;
  S.p = p;
  S.mu = mu;
  // ---- reference element
  const std::vector<double> nodes = lobatto_points(n);
  std::vector<double> qp, qw;
  gauss(mu, qp, qw);
  S.g.assign(std::size_t(mu) * n, 0.0);
  S.d.assign(std::size_t(mu) * n, 0.0);
  S.gw.assign(std::size_t(n) * mu, 0.0);
  S.dw.assign(std::size_t(n) * mu, 0.0);
  for (int a = 0; a < mu; ++a)
    for (int j = 0; j < n; ++j) {
      S.g[a * n + j] = lag_value(nodes, j, qp[a]);
      S.d[a * n + j] = lag_derivative(nodes, j, qp[a]);
      S.gw[j * mu + a] = S.g[a * n + j] * qw[a];
      S.dw[j * mu + a] = S.d[a * n + j] * qw[a];
    }
  S.w = qw;
  S.qpoints = qp;
  // ---- structured cartesian mesh on the unit square/cube (dg/mesh.hpp:265-355)
  Geometry G;
  G.dim = dim;
  const int cnt[3] = {nx, ny, dim == 3 ? nz : 1};
  const int nv[3] = {nx + 1, ny + 1, dim == 3 ? nz + 1 : 1};
  double h[3] = {1.0, 1.0, 1.0};
  for (int a = 0; a < dim; ++a) h[a] = (hi - lo) / cnt[a];
  G.nodes.resize(std::size_t(nv[0]) * nv[1] * nv[2]);
  for (int k = 0; k < nv[2]; ++k)
    for (int j = 0; j < nv[1]; ++j)
      for (int i = 0; i < nv[0]; ++i)
        G.nodes[(std::size_t(k) * nv[1] + j) * nv[0] + i] = {lo + i * h[0], lo + j * h[1],
                                                             dim == 3 ? lo + k * h[2] : 0.0};
  const int E = cnt[0] * cnt[1] * cnt[2];
  S.n_elements = E;
  G.n_elements = E;
  G.elem_nodes.resize(E);
  S.conn.assign(std::size_t(E) * 2 * dim * 3, 0);
  auto vid = [&](int i, int j, int k) { return (k * nv[1] + j) * nv[0] + i; };
  for (int k = 0; k < cnt[2]; ++k)
    for (int j = 0; j < cnt[1]; ++j)
      for (int i = 0; i < cnt[0]; ++i) {
        const int e = (k * cnt[1] + j) * cnt[0] + i;
        int c = 0;
        for (int ck = 0; ck <= (dim == 3 ? 1 : 0); ++ck)
          for (int cj = 0; cj <= 1; ++cj)
            for (int ci = 0; ci <= 1; ++ci) G.elem_nodes[e][c++] = vid(i + ci, j + cj, k + ck);
        const int pos[3] = {i, j, k};
        for (int f = 0; f < 2 * dim; ++f) {
          const int axis = f / 2, side = f % 2;
          int np[3] = {pos[0], pos[1], pos[2]};
          const int npos = pos[axis] + (side == 1 ? 1 : -1);
          int64_t* fc = &S.conn[(std::size_t(e) * 2 * dim + f) * 3];
          if (npos >= 0 && npos < cnt[axis]) {
            np[axis] = npos;
          } else if (periodic) {
            np[axis] = (npos + cnt[axis]) % cnt[axis];
          } else {
            fc[0] = -1;
            fc[1] = -1;
            fc[2] = 0;
            continue;
          }
          fc[0] = (np[2] * cnt[1] + np[1]) * cnt[0] + np[0];
          fc[1] = 2 * axis + (1 - side);
          fc[2] = 0;
        }
      }
  // ---- geometry caches at quadrature points (dg/mesh.hpp:158-231)
  const int nvol = dim == 2 ? mu * mu : mu * mu * mu;
  const int nface = nvol / mu;
  S.jdet.assign(std::size_t(E) * nvol, 0.0);
  S.face_w.assign(std::size_t(E) * 2 * dim * nface, 0.0);
  std::vector<double> adj(std::size_t(E) * nvol * dim * dim), vol_x(std::size_t(E) * nvol * dim);
  std::vector<double> face_n(std::size_t(E) * 2 * dim * nface * dim), face_x(face_n.size());
  double jac[9], adj_pt[9], xi[3] = {0, 0, 0}, x[3];
  for (int e = 0; e < E; ++e) {
    for (int qv = 0; qv < nvol; ++qv) {
      int rem = qv;
      for (int a = 0; a < dim; ++a) {
        xi[a] = qp[rem % mu];
        rem /= mu;
      }
      G.map_jacobian(e, xi, jac);
      const double det = G.adjugate(jac, adj_pt);
      S.jdet[std::size_t(e) * nvol + qv] = det;
      for (int i = 0; i < dim * dim; ++i) adj[(std::size_t(e) * nvol + qv) * dim * dim + i] = adj_pt[i];
      G.map_point(e, xi, x);
      for (int m = 0; m < dim; ++m) vol_x[(std::size_t(e) * nvol + qv) * dim + m] = x[m];
    }
    for (int f = 0; f < 2 * dim; ++f) {
      const int axis = f / 2, side = f % 2;
      int tang[2];
      face_tangents(dim, axis, tang);
      for (int qf = 0; qf < nface; ++qf) {
        const int alpha = qf % mu, beta = dim == 3 ? qf / mu : 0;
        xi[axis] = double(side);
        xi[tang[0]] = qp[alpha];
        if (dim == 3) xi[tang[1]] = qp[beta];
        G.map_jacobian(e, xi, jac);
        G.adjugate(jac, adj_pt);
        const double sign = side == 1 ? 1.0 : -1.0;
        double len = 0.0, nvec[3];
        for (int m = 0; m < dim; ++m) {
          nvec[m] = sign * adj_pt[axis * dim + m];
          len += nvec[m] * nvec[m];
        }
        len = std::sqrt(len);
        double wt = qw[alpha];
        if (dim == 3) wt *= qw[beta];
        const std::size_t base = (std::size_t(e) * 2 * dim + f) * nface + qf;
        S.face_w[base] = wt * len;
        G.map_point(e, xi, x);
        for (int m = 0; m < dim; ++m) {
          face_n[base * dim + m] = nvec[m] / len;
          face_x[base * dim + m] = x[m];
        }
      }
    }
  }
  S.vol_x = vol_x;
  S.adj = adj;
  S.face_n = face_n;
  S.face_x = face_x;
  if (euler) {  // nodal linearization state (ops/discretization.hpp:356-375); the cache is built on the device
    const int nc = dim + 2, npe = dim == 2 ? n * n : n * n * n;
    S.n_c = nc;
    S.state.assign(std::size_t(E) * nc * npe, 0.0);
    double u[5];
    for (int e = 0; e < E; ++e)
      for (int qn = 0; qn < npe; ++qn) {
        int rem = qn;
        for (int a = 0; a < dim; ++a) {
          xi[a] = nodes[rem % n];
          rem /= n;
        }
        G.map_point(e, xi, x);
        euler_state(kind, x, u);
        for (int c = 0; c < nc; ++c) S.state[(std::size_t(e) * nc + c) * npe + qn] = u[c];
      }
    S.dft.assign(std::size_t(E) * dim * nvol * nc * nc, 0.0);
    S.dfm.assign(std::size_t(E) * 2 * dim * nface * nc * nc, 0.0);
    S.dfp.assign(S.dfm.size(), 0.0);
    // FNV-1a of the state bytes (ops/state.hpp:52-61)
    std::uint64_t hsh = 1469598103934665603ULL;
    const unsigned char* bytes = reinterpret_cast<const unsigned char*>(S.state.data());
    for (std::size_t i = 0; i < S.state.size() * sizeof(double); ++i) {
      hsh ^= bytes[i];
      hsh *= 1099511628211ULL;
    }
    S.state_hash = hsh;
    return TPDG_OK;
  }
  // ---- linearization cache of scalar upwind advection (ops/linearized.hpp:38-100)
  auto velocity = [&](const double* xx, double* v) {
    if (kind == 1) {
      v[0] = std::sin(2.0 * M_PI * xx[1]);
      v[1] = std::cos(2.0 * M_PI * xx[0]);
      v[2] = 0.0;
    } else {
      v[0] = vel[0];
      v[1] = vel[1];
      v[2] = dim == 3 ? vel[2] : 0.0;
    }
  };
  S.dft.assign(std::size_t(E) * dim * nvol, 0.0);
  S.dfm.assign(std::size_t(E) * 2 * dim * nface, 0.0);
  S.dfp.assign(std::size_t(E) * 2 * dim * nface, 0.0);
  for (int e = 0; e < E; ++e) {
    for (int qv = 0; qv < nvol; ++qv) {
      double v[3];
      velocity(&vol_x[(std::size_t(e) * nvol + qv) * dim], v);
      const double* a = &adj[(std::size_t(e) * nvol + qv) * dim * dim];
      for (int k = 0; k < dim; ++k) {
        double s = 0.0;
        for (int m = 0; m < dim; ++m) s += a[k * dim + m] * v[m];
        S.dft[(std::size_t(e) * dim + k) * nvol + qv] = s;
      }
    }
    for (int f = 0; f < 2 * dim; ++f) {
      const bool interior = S.conn[(std::size_t(e) * 2 * dim + f) * 3] >= 0;
      for (int qf = 0; qf < nface; ++qf) {
        const std::size_t base = (std::size_t(e) * 2 * dim + f) * nface + qf;
        double v[3];
        velocity(&face_x[base * dim], v);
        double vn = 0.0;
        for (int m = 0; m < dim; ++m) vn += v[m] * face_n[base * dim + m];
        S.dfm[base] = std::max(vn, 0.0);
        if (interior) S.dfp[base] = std::min(vn, 0.0);
      }
    }
  }
  // FNV-1a of the (zero) linearization state (ops/state.hpp:52-61): advection's Jacobian is
  // state independent, the reference binds the zero state.
  std::uint64_t hsh = 1469598103934665603ULL;
  const std::size_t nbytes = std::size_t(E) * std::size_t(dim == 2 ? n * n : n * n * n) * sizeof(double);
  for (std::size_t i = 0; i < nbytes; ++i) {
    hsh ^= 0u;
    hsh *= 1099511628211ULL;
  }
  S.state_hash = hsh;
  return TPDG_OK;
}

void uniform_vector(std::uint64_t seed, std::int64_t n, double scale, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-scale, scale);
  for (std::int64_t i = 0; i < n; ++i) out[i] = dist(rng);
}

void seeded_unit_vector(std::int64_t n, std::uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> dist(0.0, 1.0);
  double nrm = 0.0;
  while (nrm == 0.0) {
    for (std::int64_t i = 0; i < n; ++i) out[i] = dist(rng);
    double s = 0.0;
    for (std::int64_t i = 0; i < n; ++i) s += out[i] * out[i];
    nrm = std::sqrt(s);
  }
  for (std::int64_t i = 0; i < n; ++i) out[i] /= nrm;
}

} // namespace tpdg_gpu
