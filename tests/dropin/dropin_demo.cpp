// Drop-in demonstration (built in the build container against the UNMODIFIED reference headers,
// run on the GPU box): the reference's own Discretization / LinearizationCache / LinearizedOperator
// feed the B200 path through include/tpdg_gpu.hpp, and the reference's CPU gmres runs beside it.
// Prints one JSON line: GMRES counts of both, Jv and PC-apply differences.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>

#define TPDG_GPU_WITH_REFERENCE 1
#include "tpdg/laws/advection.hpp"
#include "tpdg/precond/block_jacobi.hpp"
#include "tpdg/precond/ksvd.hpp"
#include "tpdg/solve/gmres.hpp"
#include "tpdg_gpu.hpp"

using namespace tpdg;

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 8;
  const int p = argc > 2 ? std::atoi(argv[2]) : 8;
  // BASELINE configs[1] field on an n x n periodic mesh, through the reference's Law plugin.
  auto ref = build_reference(p);
  MeshSpec spec;
  spec.dim = 2;
  spec.counts = {n, n, 1};
  spec.periodic = true;
  auto mesh = generate_mesh(spec, ref);
  Law law = advection_law(AdvectionField::a);
  auto vel = [](const double* x, double* v) {
    v[0] = std::sin(2.0 * M_PI * x[1]);
    v[1] = std::cos(2.0 * M_PI * x[0]);
  };
  law.flux_jacobian = [vel](const double*, const double* x, double* df) { vel(x, df); };
  law.num_flux_jac_minus = [vel](const double*, const double*, const double* nn, const double* x, double* d) {
    double v[2];
    vel(x, v);
    d[0] = std::max(v[0] * nn[0] + v[1] * nn[1], 0.0);
  };
  law.num_flux_jac_plus = [vel](const double*, const double*, const double* nn, const double* x, double* d) {
    double v[2];
    vel(x, v);
    d[0] = std::min(v[0] * nn[0] + v[1] * nn[1], 0.0);
  };
  const Discretization sys = make_discretization(std::move(ref), std::move(mesh), law);
  const StateVector u = sys.make_state();
  const auto cache = build_cache(sys, u);
  const auto lin = make_linearized_operator(sys, cache, 0.005);

  std::mt19937_64 rng(12345);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  std::vector<double> b(u.data.size());
  for (auto& x : b) x = dist(rng);

  // reference CPU path
  const auto kpc = form_ksvd_2d(lin);
  auto op = [&](std::span<const double> in, std::span<double> out) {
    StateVector v = sys.make_state();
    std::copy(in.begin(), in.end(), v.data.begin());
    const StateVector w = jacobian_apply(lin, v);
    std::copy(w.data.begin(), w.data.end(), out.begin());
  };
  GmresConfig gc;
  gc.tol = 1e-10;
  gc.restart = 30;
  const auto ref_res = gmres(op, [&](auto in, auto out) { kpc.apply(in, out); }, b, gc);

  // drop-in B200 path fed by the same reference objects
  tpdg::gpu::Context ctx(0);
  tpdg::gpu::LinearizedOperator gop(ctx, lin);
  const auto gpc = tpdg::gpu::form_ksvd(gop);
  const auto gres = tpdg::gpu::gmres(gop, gpc, b, {1e-10, 30, 2000, 0});

  std::vector<double> jr(b.size()), jg(b.size()), zr(b.size()), zg(b.size());
  op(b, jr);
  gop.apply(b, jg);
  kpc.apply(b, zr);
  gpc.apply(b, zg);
  auto rel = [](const std::vector<double>& a, const std::vector<double>& c) {
    double nn = 0, dd = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
      nn += (a[i] - c[i]) * (a[i] - c[i]);
      dd += c[i] * c[i];
    }
    return std::sqrt(nn / dd);
  };

  // Mode::jacobian_only (ops/linearized.hpp:167-178): the drop-in honours lin.mode
  auto lin_j = make_linearized_operator(sys, cache, 0.005, LinearizedOperator::Mode::jacobian_only);
  tpdg::gpu::LinearizedOperator gop_j(ctx, lin_j);
  StateVector vb = sys.make_state();
  vb.data = b;
  const StateVector jref_j = jacobian_apply(lin_j, vb);
  std::vector<double> jg_j(b.size());
  gop_j.apply(b, jg_j);

  // budget exhausted: both implementations throw GmresFailure carrying the best iterate (gmres.hpp:165-178)
  GmresConfig gf = gc;
  gf.max_iterations = 3;
  int ref_fail_its = -1, gpu_fail_its = -1;
  double fail_hist_rel = -1.0, fail_x_rel = -1.0;
  std::vector<double> ref_fail_x, ref_fail_hist;
  try {
    gmres(op, [&](auto in, auto out) { kpc.apply(in, out); }, b, gf);
  } catch (const GmresFailure& f) {
    ref_fail_its = f.result.iterations;
    ref_fail_x = f.result.x;
    ref_fail_hist = f.result.residual_history;
  }
  try {
    tpdg::gpu::gmres(gop, gpc, b, {1e-10, 30, 3, 0});
  } catch (const GmresFailure& f) {  // tpdg::GmresFailure: the reference's own class
    gpu_fail_its = f.result.iterations;
    fail_x_rel = rel(f.result.x, ref_fail_x);
    double mx = 0.0;
    for (std::size_t i = 0; i < f.result.residual_history.size() && i < ref_fail_hist.size(); ++i)
      mx = std::max(mx, std::abs(f.result.residual_history[i] - ref_fail_hist[i]) / ref_fail_hist[i]);
    fail_hist_rel = f.result.residual_history.size() == ref_fail_hist.size() ? mx : 1.0;
  }

  // form_block_jacobi (precond/block_jacobi.hpp:38-72) through the same wrapper
  const auto bj = form_block_jacobi(lin);
  const auto gbj = tpdg::gpu::form_block_jacobi(gop);
  std::vector<double> br(b.size()), bg(b.size());
  bj.apply(b, br);
  gbj.apply(b, bg);
  const bool fields = gpc.mode == 0 && gpc.n_elements == kpc.n_elements && gpc.n_c == kpc.n_c && gpc.npe == kpc.npe &&
                      gpc.n1d == kpc.n1d;

  std::printf("{\"n\": %d, \"p\": %d, \"ref_its\": %d, \"gpu_its\": %d, \"ref_fallbacks\": %zu, "
              "\"gpu_fallbacks\": %zu, \"jv_rel\": %.3e, \"pc_rel\": %.3e, \"jv_jacobian_only_rel\": %.3e, "
              "\"ref_fail_its\": %d, \"gpu_fail_its\": %d, \"fail_x_rel\": %.3e, \"fail_hist_rel\": %.3e, "
              "\"block_jacobi_rel\": %.3e, \"pc_fields_match\": %d}\n",
              n, p, ref_res.iterations, gres.iterations, kpc.fallbacks.size(), gpc.fallbacks().size(), rel(jg, jr),
              rel(zg, zr), rel(jg_j, jref_j.data), ref_fail_its, gpu_fail_its, fail_x_rel, fail_hist_rel,
              rel(bg, br), int(fields));
  return ref_res.iterations == gres.iterations ? 0 : 1;
}
