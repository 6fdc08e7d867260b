// Reference driver: compiles the UNMODIFIED reference headers in place
// (-I/root/reference/proj/include; nothing is copied into this repo) and
//   * `golden <case> <dir>` dumps inputs and outputs of the hot path as .npy
//     files (tests/golden/make_golden.py packs them into committed fixtures);
//   * `bench <case> <threads> <max_its> <reps>` times the reference CPU path
//     (form_ksvd, KsvdPC::apply, jacobian_apply, gmres) and prints one JSON line.
// Test infrastructure only (oracle/): never linked into the product.
//
// The hot path driven here is exactly the one newton_linear_solve runs
// (reference proj/include/tpdg/solve/time_step.hpp:57-122): build_cache ->
// form_ksvd_2d/3d -> gmres(jacobian_apply, KsvdPC::apply), with a seeded
// uniform RHS as in tests/unit/test_precond.cpp:64-74,390-392.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "tpdg/laws/advection.hpp"
#include "tpdg/laws/euler.hpp"
#include "tpdg/precond/ksvd.hpp"
#include "tpdg/solve/gmres.hpp"
#include "tpdg/solve/time_step.hpp"

using namespace tpdg;

namespace {

// ---------------------------------------------------------------- npy output
void write_npy(const std::string& path, const void* data, std::size_t count, const char* descr,
               std::size_t elem) {
  std::ostringstream hdr;
  hdr << "{'descr': '" << descr << "', 'fortran_order': False, 'shape': (" << count << ",), }";
  std::string h = hdr.str();
  const std::size_t pre = 10;
  std::size_t total = pre + h.size() + 1;
  std::size_t pad = (64 - total % 64) % 64;
  h.append(pad, ' ');
  h.push_back('\n');
  std::ofstream f(path, std::ios::binary);
  const char magic[] = "\x93NUMPY";
  f.write(magic, 6);
  const unsigned char ver[2] = {1, 0};
  f.write(reinterpret_cast<const char*>(ver), 2);
  const std::uint16_t hl = std::uint16_t(h.size());
  f.write(reinterpret_cast<const char*>(&hl), 2);
  f.write(h.data(), std::streamsize(h.size()));
  f.write(reinterpret_cast<const char*>(data), std::streamsize(count * elem));
}
void dump(const std::string& dir, const std::string& name, const std::vector<double>& v) {
  write_npy(dir + "/" + name + ".npy", v.data(), v.size(), "<f8", 8);
}
void dump_i(const std::string& dir, const std::string& name, const std::vector<std::int64_t>& v) {
  write_npy(dir + "/" + name + ".npy", v.data(), v.size(), "<i8", 8);
}
void dump_m(const std::string& dir, const std::string& name, const SmallMatrix& m) {
  std::vector<double> v(m.data(), m.data() + m.size());
  dump(dir, name, v);
}

// ---------------------------------------------------------------- cases
struct CaseSpec {
  int dim = 2;
  std::string law;            // adv_const | adv_swirl | adv_b | euler | euler_cfg3 | euler_cfg5
  double hi = 1.0;            // domain [0, hi]^d
  int gmres_budget = 0;       // > 0: fixed GMRES iteration budget (history gate)
  double vel[3] = {1.0, 0.5, 0.0};
  int counts[3] = {1, 1, 1};
  int p = 1;
  double dt = 0.01;
  double amplitude = 0.0;
  bool periodic = true;
  std::uint64_t mesh_seed = 0;
  BlockMode mode = BlockMode::full;
  double rhs_scale = 1.0;
  bool light = false;         // big case: dump decisions and counts only
};

CaseSpec lookup(const std::string& name) {
  CaseSpec c;
  auto adv2 = [&](double vx, double vy, int n, int p, double dt) {
    c.dim = 2; c.law = "adv_const"; c.vel[0] = vx; c.vel[1] = vy;
    c.counts[0] = c.counts[1] = n; c.p = p; c.dt = dt;
  };
  auto swirl = [&](int n, int p) {
    c.dim = 2; c.law = "adv_swirl"; c.counts[0] = c.counts[1] = n; c.p = p; c.dt = 0.005;
  };
  auto adv3 = [&](int n, int p) {
    c.dim = 3; c.law = "adv_const"; c.vel[0] = 1.0; c.vel[1] = 0.7; c.vel[2] = 0.4;
    c.counts[0] = c.counts[1] = c.counts[2] = n; c.p = p; c.dt = 0.01;
  };
  // BASELINE.json configs[0]: 2D advection (1, 0.5), 8x8, p=8, dt=0.01.
  if (name == "cfg1") { adv2(1.0, 0.5, 8, 8, 0.01); return c; }
  // configs[1] at reduced mesh sizes (same field, dt, p values).
  if (name == "cfg2s_p4") { swirl(8, 4); return c; }
  if (name == "cfg2s_p8") { swirl(4, 8); return c; }
  if (name == "cfg2s_p15") { swirl(2, 15); return c; }
  // configs[1] at full size: decisions + counts only.
  for (int p : {4, 8, 15, 20, 30})
    if (name == "cfg2_p" + std::to_string(p)) { swirl(64, p); c.light = true; return c; }
  // Perturbed, non-periodic mesh with boundary faces (field b of the reference).
  if (name == "pert2d") {
    c.dim = 2; c.law = "adv_b"; c.counts[0] = c.counts[1] = 3; c.p = 3; c.dt = 0.5;
    c.amplitude = 0.1; c.periodic = false; c.mesh_seed = 7; return c;
  }
  // BASELINE.json configs[3] at reduced sizes, and full size (light).
  if (name == "adv3d_p3") { adv3(2, 3); return c; }
  if (name == "adv3d_p4") { adv3(3, 4); return c; }
  if (name == "cfg4") { adv3(16, 10); c.light = true; return c; }
  // Systems (reference LLF Euler law) for the n_c > 1 kernel paths.
  if (name == "euler2d" || name == "euler2d_small") {
    c.dim = 2; c.law = "euler"; c.counts[0] = c.counts[1] = 2; c.p = 2; c.dt = 0.05;
    c.amplitude = 0.08; c.mesh_seed = 23; c.rhs_scale = 1e-3;
    if (name == "euler2d_small") c.mode = BlockMode::small;
    return c;
  }
  if (name == "euler3d") {
    c.dim = 3; c.law = "euler"; c.counts[0] = 2; c.counts[1] = 2; c.counts[2] = 1; c.p = 2;
    c.dt = 2.5e-3; c.rhs_scale = 1e-3; return c;
  }
  // Euler stand-ins of BASELINE configs[2] / configs[4] (LLF flux: the reference has no Roe flux and no
  // BR2 viscous terms), states of host_setup.cpp's euler_state; reduced sizes with full dumps, and the
  // configured sizes with a fixed GMRES budget (neither converges to 1e-10).
  if (name == "cfg3s" || name == "cfg3") {
    c.dim = 2; c.law = "euler_cfg3"; c.hi = 10.0; c.dt = 0.05; c.rhs_scale = 1e-3;
    if (name == "cfg3s") { c.counts[0] = c.counts[1] = 4; c.p = 4; }
    else { c.counts[0] = c.counts[1] = 32; c.p = 15; c.light = true; c.gmres_budget = 40; }
    return c;
  }
  if (name == "cfg5s" || name == "cfg5") {
    c.dim = 3; c.law = "euler_cfg5"; c.hi = 2.0 * M_PI; c.dt = 0.01; c.rhs_scale = 1e-3;
    if (name == "cfg5s") { c.counts[0] = c.counts[1] = c.counts[2] = 2; c.p = 3; }
    else { c.counts[0] = c.counts[1] = c.counts[2] = 8; c.p = 7; c.light = true; c.gmres_budget = 40; }
    return c;
  }
  std::fprintf(stderr, "unknown case %s\n", name.c_str());
  std::exit(2);
}

// Scalar advection with a user velocity field, written against the reference
// Law plugin exactly like advection_law (reference laws/advection.hpp:25-54).
template <class Vel>
Law make_adv_law(int dim, Vel vel) {
  Law law;
  law.dim = dim;
  law.n_c = 1;
  law.flux = [vel, dim](const double* u, const double* x, double* f) {
    double v[3]; vel(x, v);
    for (int m = 0; m < dim; ++m) f[m] = v[m] * u[0];
  };
  law.flux_jacobian = [vel, dim](const double*, const double* x, double* df) {
    double v[3]; vel(x, v);
    for (int m = 0; m < dim; ++m) df[m] = v[m];
  };
  law.num_flux = [vel, dim](const double* um, const double* up, const double* n, const double* x, double* fh) {
    double v[3]; vel(x, v);
    double vn = 0.0;
    for (int m = 0; m < dim; ++m) vn += v[m] * n[m];
    fh[0] = vn * (vn >= 0.0 ? um[0] : up[0]);
  };
  law.num_flux_jac_minus = [vel, dim](const double*, const double*, const double* n, const double* x, double* d) {
    double v[3]; vel(x, v);
    double vn = 0.0;
    for (int m = 0; m < dim; ++m) vn += v[m] * n[m];
    d[0] = std::max(vn, 0.0);
  };
  law.num_flux_jac_plus = [vel, dim](const double*, const double*, const double* n, const double* x, double* d) {
    double v[3]; vel(x, v);
    double vn = 0.0;
    for (int m = 0; m < dim; ++m) vn += v[m] * n[m];
    d[0] = std::min(vn, 0.0);
  };
  law.boundary_state = [](const double*, double, const double*, double* u_out) { u_out[0] = 0.0; };
  return law;
}

struct Built {
  Discretization sys;
  StateVector state;
};

Built build(const CaseSpec& c) {
  auto ref = build_reference(c.p);
  MeshSpec spec;
  spec.dim = c.dim;
  spec.kind = c.amplitude == 0.0 ? MeshKind::cartesian : MeshKind::perturbed;
  spec.counts = {c.counts[0], c.counts[1], c.counts[2]};
  spec.amplitude = c.amplitude;
  spec.seed = c.mesh_seed;
  spec.periodic = c.periodic;
  for (int a = 0; a < c.dim; ++a) spec.hi[a] = c.hi;
  auto mesh = generate_mesh(spec, ref);
  Law law;
  if (c.law == "adv_const") {
    const double v0 = c.vel[0], v1 = c.vel[1], v2 = c.vel[2];
    law = make_adv_law(c.dim, [v0, v1, v2](const double*, double* v) { v[0] = v0; v[1] = v1; v[2] = v2; });
  } else if (c.law == "adv_swirl") {
    law = make_adv_law(2, [](const double* x, double* v) {
      v[0] = std::sin(2.0 * M_PI * x[1]);
      v[1] = std::cos(2.0 * M_PI * x[0]);
      v[2] = 0.0;
    });
  } else if (c.law == "adv_b") {
    law = advection_law(AdvectionField::b);
  } else {
    law = euler_law(c.dim);  // also euler_cfg3 / euler_cfg5
  }
  Built b{make_discretization(std::move(ref), std::move(mesh), std::move(law)), StateVector()};
  if (c.law == "euler" && c.dim == 2) {
    // smooth_euler_state2d, reference tests/unit/test_precond.cpp:43-54.
    b.state = interpolate(b.sys, [](const double* x, double* u) {
      const double rho = 1.0 + 0.15 * std::sin(2.0 * M_PI * x[0]) * std::cos(2.0 * M_PI * x[1]);
      const double vx = 0.4 + 0.1 * std::cos(2.0 * M_PI * x[1]);
      const double vy = -0.3;
      const double p = 1.0 + 0.1 * std::cos(2.0 * M_PI * x[0]);
      u[0] = rho; u[1] = rho * vx; u[2] = rho * vy;
      u[3] = p / 0.4 + 0.5 * rho * (vx * vx + vy * vy);
    });
  } else if (c.law == "euler_cfg3") {
    b.state = interpolate(b.sys, [](const double* x, double* u) {
      const double gamma = 1.4;
      const double dx = x[0] - 5.0, dy = x[1] - 5.0;
      const double r2 = dx * dx + dy * dy;
      const double rho = 1.0 + 0.2 * std::exp(-0.5 * r2);
      const double sw = 0.5 * std::exp(0.5 * (1.0 - r2));
      const double vx = 1.0 - sw * dy, vy = 1.0 + sw * dx;
      const double pr = std::pow(rho, gamma);
      u[0] = rho;
      u[1] = rho * vx;
      u[2] = rho * vy;
      u[3] = pr / (gamma - 1.0) + 0.5 * rho * (vx * vx + vy * vy);
    });
  } else if (c.law == "euler_cfg5") {
    b.state = interpolate(b.sys, [](const double* x, double* u) {
      const double gamma = 1.4, mach = 0.1, p0 = 1.0 / (gamma * mach * mach);
      const double vx = std::sin(x[0]) * std::cos(x[1]) * std::cos(x[2]);
      const double vy = -std::cos(x[0]) * std::sin(x[1]) * std::cos(x[2]);
      const double pr = p0 + (std::cos(2.0 * x[0]) + std::cos(2.0 * x[1])) * (std::cos(2.0 * x[2]) + 2.0) / 16.0;
      u[0] = 1.0;
      u[1] = vx;
      u[2] = vy;
      u[3] = 0.0;
      u[4] = pr / (gamma - 1.0) + 0.5 * (vx * vx + vy * vy);
    });
  } else if (c.law == "euler") {
    // reference tests/unit/test_precond.cpp:266-273.
    b.state = interpolate(b.sys, [](const double* x, double* s) {
      const double rho = 1.0 + 0.2 * std::sin(M_PI * (x[0] + x[1] + x[2]));
      s[0] = rho; s[1] = rho; s[2] = -0.5 * rho; s[3] = rho; s[4] = 1.0 / 0.4 + 0.5 * rho * 2.25;
    });
  } else {
    b.state = b.sys.make_state();
  }
  return b;
}

std::vector<double> uniform_vector(std::uint64_t seed, std::size_t n, double scale) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-scale, scale);
  std::vector<double> v(n);
  for (auto& x : v) x = dist(rng);
  return v;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

struct PcHolder {
  KsvdPC2D k2;
  KsvdPC3D k3;
  int dim = 2;
  void apply(std::span<const double> in, std::span<double> out) const {
    if (dim == 2) k2.apply(in, out); else k3.apply(in, out);
  }
  const std::vector<FallbackEvent>& fallbacks() const { return dim == 2 ? k2.fallbacks : k3.fallbacks; }
};

PcHolder form(const LinearizedOperator& lin, int dim, BlockMode mode) {
  PcHolder h;
  h.dim = dim;
  if (dim == 2) h.k2 = form_ksvd_2d(lin, mode); else h.k3 = form_ksvd_3d(lin, mode);
  return h;
}

LinearAction make_op(const Discretization& sys, const LinearizedOperator& lin) {
  return [&sys, &lin](std::span<const double> in, std::span<double> out) {
    StateVector v = sys.make_state();
    std::copy(in.begin(), in.end(), v.data.begin());
    const StateVector w = jacobian_apply(lin, v);
    std::copy(w.data.begin(), w.data.end(), out.begin());
  };
}

GmresConfig gmres_cfg(int max_its) {
  GmresConfig g;
  g.tol = 1e-10;        // BASELINE.json configs: GMRES(30) to rel. tol 1e-10
  g.restart = 30;
  g.max_iterations = max_its;
  g.side = PrecondSide::right;
  return g;
}

// ---------------------------------------------------------------- golden
int run_golden(const std::string& name, const std::string& dir) {
  const CaseSpec c = lookup(name);
  std::filesystem::create_directories(dir);
  Built bt = build(c);
  const Discretization& sys = bt.sys;
  const auto cache = build_cache(sys, bt.state);
  const auto lin = [&] {
    auto l = make_linearized_operator(sys, cache, c.dt);
    l.block_mode = c.mode;
    return l;
  }();
  const int d = sys.dim, q = sys.n1d, E = sys.mesh.n_elements;
  const std::size_t N = std::size_t(E) * sys.n_c * sys.npe;

  std::vector<double> meta = {double(d), double(sys.n_c), double(sys.ref.p), double(sys.mu), double(E),
                              c.dt, c.mode == BlockMode::full ? 0.0 : 1.0, double(c.counts[0]),
                              double(c.counts[1]), double(c.counts[2]), c.rhs_scale, c.periodic ? 1.0 : 0.0};
  dump(dir, "meta", meta);

  if (!c.light) {
    dump_m(dir, "ref_g", sys.ref.g);
    dump_m(dir, "ref_d", sys.ref.d);
    dump_m(dir, "ref_gw", sys.ref.gw);
    dump_m(dir, "ref_dw", sys.ref.dw);
    dump(dir, "ref_w", sys.ref.qweights);
    dump(dir, "ref_qpoints", sys.ref.qpoints);
    dump(dir, "ref_nodes", sys.ref.nodes);
    dump(dir, "jdet", sys.mesh.jdet);
    dump(dir, "face_w", sys.mesh.face_w);
    dump(dir, "face_n", sys.mesh.face_n);
    dump(dir, "adj", sys.mesh.adj);
    dump(dir, "vol_x", sys.mesh.vol_x);
    dump(dir, "face_x", sys.mesh.face_x);
    std::vector<std::int64_t> conn;
    for (int e = 0; e < E; ++e)
      for (int f = 0; f < 2 * d; ++f) {
        conn.push_back(sys.mesh.faces[e][f].neighbor);
        conn.push_back(sys.mesh.faces[e][f].neighbor_face);
        conn.push_back(sys.mesh.faces[e][f].orientation);
      }
    dump_i(dir, "conn", conn);
    dump(dir, "state", bt.state.data);
    dump(dir, "dft", cache.dft);
    dump(dir, "dfm", cache.dfm);
    dump(dir, "dfp", cache.dfp);

    // Jv on a seeded vector.
    StateVector v = sys.make_state();
    v.data = uniform_vector(1001, N, 1.0);
    dump(dir, "jv_in", v.data);
    dump(dir, "jv_out", jacobian_apply(lin, v).data);

    // Shuffled products of element 0 (and the last element).
    for (int e : {0, E - 1}) {
      for (int comp = 0; comp < (c.mode == BlockMode::full ? 1 : sys.n_c); ++comp) {
        const auto op = make_element_shuffled_operator(lin, e, c.mode, comp);
        const std::string tag = "e" + std::to_string(e) + "c" + std::to_string(comp);
        const auto v0 = uniform_vector(2000 + e, std::size_t(op.cols()), 1.0);
        const auto u1 = uniform_vector(3000 + e, std::size_t(op.rows()), 1.0);
        std::vector<double> u0(op.rows()), v1(op.cols());
        op.apply(v0, u0);
        op.apply_transpose(u1, v1);
        dump(dir, "shuf_" + tag + "_v", v0);
        dump(dir, "shuf_" + tag + "_av", u0);
        dump(dir, "shuf_" + tag + "_u", u1);
        dump(dir, "shuf_" + tag + "_atu", v1);
        // Lanczos on this operator as form_ksvd runs it.
        KsvdConfig kc;
        const auto lres = lanczos_ksvd(op, ksvd_detail::block_lanczos_config(kc, d == 2 ? kc.terms : 1));
        dump(dir, "lanczos_" + tag + "_sigma", lres.singular_values);
        dump(dir, "lanczos_" + tag + "_iters", {double(lres.iterations), lres.converged ? 1.0 : 0.0});
        for (std::size_t t = 0; t < lres.factors.terms.size(); ++t) {
          dump_m(dir, "lanczos_" + tag + "_t" + std::to_string(t) + "_a", lres.factors.terms[t][0]);
          dump_m(dir, "lanczos_" + tag + "_t" + std::to_string(t) + "_b", lres.factors.terms[t][1]);
        }
        // Dense diagonal block (for the block-error gate).
        if (c.mode == BlockMode::full) dump_m(dir, "block_e" + std::to_string(e), assemble_diag_block(lin, e));
      }
    }
    // Start vectors (reference tensor/lanczos.hpp:61-72), seed 0x5eed.
    {
      const long n2d = d == 2 ? long(q) * q : long(q) * q * q * q;
      dump(dir, "start_vec", detail::seeded_unit_vector(n2d, 0x5eedULL));
      if (d == 3) dump(dir, "start_vec2", detail::seeded_unit_vector(long(q) * q, 0x5eedULL));
    }
  }

  if (!c.light && c.law.rfind("euler_cfg", 0) == 0) {
    // residual r(u, t) (ops/discretization.hpp:188-254) at the linearization state, M v on the seeded vector
    // (mass_apply), and one backward Euler step by Newton-GMRES with the KSVD preconditioner
    // (solve/time_step.hpp:126-146, newton.hpp:32-68): GMRES(30) to 1e-10, Newton defaults.
    dump(dir, "resid", residual(sys, bt.state, 0.0).data);
    {
      StateVector v = sys.make_state();
      v.data = uniform_vector(1001, N, 1.0);
      dump(dir, "mass_out", mass_apply(sys, v).data);
    }
    ImplicitConfig icfg;
    icfg.gmres = gmres_cfg(2000);
    icfg.precond = c.mode == BlockMode::full ? PrecondKind::ksvd_full : PrecondKind::ksvd_small;
    StepStats st;
    st.keep_residual_history = true;
    const StateVector u1 = step_backward_euler(sys, bt.state, 0.0, c.dt, icfg, &st);
    dump(dir, "newton_state", u1.data);
    std::vector<double> gits(st.gmres_per_solve.begin(), st.gmres_per_solve.end());
    dump(dir, "newton_gmres", gits);
    dump(dir, "newton_steps", {double(st.newton_steps)});
    std::printf("%s: newton steps %d, gmres per solve:", name.c_str(), st.newton_steps);
    for (int g : st.gmres_per_solve) std::printf(" %d", g);
    std::printf("\n");
  }

  const PcHolder pc = form(lin, d, c.mode);
  // Formed factors, element-major (full) or element*n_c+c (small).
  {
    std::vector<double> fac, sq1, st1, sq2, st2;
    std::vector<std::int64_t> has;
    auto append = [](std::vector<double>& dst, const SmallMatrix& m) { dst.insert(dst.end(), m.data(), m.data() + m.size()); };
    const std::size_t nblk = d == 2 ? pc.k2.factors.size() : pc.k3.factors.size();
    for (std::size_t i = 0; i < nblk; ++i) {
      if (d == 2) {
        const auto& f = pc.k2.factors[i];
        has.push_back(f.has_value() ? 1 : 0);
        if (f && !c.light) {
          append(fac, f->a1); append(fac, f->b1); append(fac, f->a2); append(fac, f->b2);
          append(sq1, f->s1.q); append(st1, f->s1.t); append(sq2, f->s2.q); append(st2, f->s2.t);
        }
      } else {
        const auto& f = pc.k3.factors[i];
        has.push_back(f.has_value() ? 1 : 0);
        if (f && !c.light) {
          append(fac, f->a1); append(fac, f->b1); append(fac, f->c1); append(fac, f->b2); append(fac, f->c2);
          append(sq1, f->s1.q); append(st1, f->s1.t); append(sq2, f->s2.q); append(st2, f->s2.t);
        }
      }
    }
    dump_i(dir, "has_factors", has);
    if (!c.light) {
      dump(dir, "factors", fac);
      dump(dir, "schur_q1", sq1); dump(dir, "schur_t1", st1);
      dump(dir, "schur_q2", sq2); dump(dir, "schur_t2", st2);
    }
    std::vector<std::int64_t> fb;
    for (const auto& ev : pc.fallbacks()) { fb.push_back(ev.element); fb.push_back(ev.component); }
    dump_i(dir, "fallbacks", fb);
  }

  const auto b = uniform_vector(12345, N, c.rhs_scale);
  if (!c.light) {
    std::vector<double> z(N);
    pc.apply(b, z);
    dump(dir, "rhs", b);
    dump(dir, "pc_out", z);
  }
  const auto op = make_op(sys, lin);
  const LinearAction pca = [&pc](std::span<const double> in, std::span<double> out) { pc.apply(in, out); };
  GmresResult gr;
  bool converged = true;
  try {
    gr = gmres(op, pca, b, gmres_cfg(c.gmres_budget > 0 ? c.gmres_budget : c.light ? 400 : 2000));
  } catch (const GmresFailure& f) {
    gr = f.result;
    converged = false;
  }
  dump(dir, "gmres_meta", {double(gr.iterations), converged ? 1.0 : 0.0});
  dump(dir, "gmres_hist", gr.residual_history);
  if (!c.light) dump(dir, "gmres_x", gr.x);
  std::printf("%s: N=%zu fallbacks=%zu gmres_its=%d converged=%d\n", name.c_str(), N, pc.fallbacks().size(),
              gr.iterations, int(converged));
  return 0;
}

// ---------------------------------------------------------------- bench
// Times the reference CPU path on one case. `max_its` caps GMRES so that one
// step is a bounded sample of the workload (GDOF-iterations/s is per iteration).
int run_bench(const std::string& name, int threads, int max_its, int reps) {
  thread_count() = threads;
  const CaseSpec c = lookup(name);
  Built bt = build(c);
  const Discretization& sys = bt.sys;
  const auto cache = build_cache(sys, bt.state);
  auto lin = make_linearized_operator(sys, cache, c.dt);
  lin.block_mode = c.mode;
  const std::size_t N = std::size_t(sys.mesh.n_elements) * sys.n_c * sys.npe;
  const auto b = uniform_vector(12345, N, c.rhs_scale);

  auto t0 = std::chrono::steady_clock::now();
  PcHolder pc = form(lin, sys.dim, c.mode);
  const double t_form = seconds_since(t0);

  std::vector<double> z(N);
  t0 = std::chrono::steady_clock::now();
  pc.apply(b, z);
  const double t_apply = seconds_since(t0);

  StateVector v = sys.make_state();
  v.data = b;
  t0 = std::chrono::steady_clock::now();
  const StateVector jv = jacobian_apply(lin, v);
  const double t_jv = seconds_since(t0);

  const auto op = make_op(sys, lin);
  const LinearAction pca = [&pc](std::span<const double> in, std::span<double> out) { pc.apply(in, out); };
  std::vector<double> t_gmres;
  int its = 0;
  bool converged = false;
  for (int r = 0; r < reps; ++r) {
    t0 = std::chrono::steady_clock::now();
    try {
      const auto gr = gmres(op, pca, b, gmres_cfg(max_its));
      its = gr.iterations;
      converged = gr.converged;
    } catch (const GmresFailure& f) {
      its = f.result.iterations;
      converged = false;
    }
    t_gmres.push_back(seconds_since(t0));
  }
  std::printf("{\"case\": \"%s\", \"N\": %zu, \"threads\": %d, \"form_s\": %.6e, \"pc_apply_s\": %.6e, "
              "\"jv_s\": %.6e, \"gmres_its\": %d, \"gmres_converged\": %d, \"fallbacks\": %zu, \"gmres_s\": [",
              name.c_str(), N, threads, t_form, t_apply, t_jv, its, int(converged), pc.fallbacks().size());
  for (std::size_t i = 0; i < t_gmres.size(); ++i) std::printf("%s%.6e", i ? ", " : "", t_gmres[i]);
  std::printf("]}\n");
  return 0;
}

} // namespace

int main(int argc, char** argv) {
  if (argc >= 4 && std::string(argv[1]) == "golden") {
    thread_count() = int(std::thread::hardware_concurrency());
    return run_golden(argv[2], argv[3]);
  }
  if (argc >= 6 && std::string(argv[1]) == "bench")
    return run_bench(argv[2], std::atoi(argv[3]), std::atoi(argv[4]), std::atoi(argv[5]));
  std::fprintf(stderr, "usage: %s golden <case> <dir> | bench <case> <threads> <max_its> <reps>\n", argv[0]);
  return 2;
}
