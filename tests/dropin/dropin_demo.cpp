// Drop-in demonstration (built in the build container against the UNMODIFIED reference headers,
// run on the GPU box): the reference's own Discretization / LinearizationCache / LinearizedOperator
// feed the B200 path through include/tpdg_gpu.hpp, and the reference's CPU gmres runs beside it.
// Prints one JSON line: GMRES counts of both, Jv and PC-apply differences.
#include <cmath>
#include <cstdio>
#include <random>

#define TPDG_GPU_WITH_REFERENCE 1
#include "tpdg/laws/advection.hpp"
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
  std::printf("{\"n\": %d, \"p\": %d, \"ref_its\": %d, \"gpu_its\": %d, \"ref_fallbacks\": %zu, "
              "\"gpu_fallbacks\": %zu, \"jv_rel\": %.3e, \"pc_rel\": %.3e}\n",
              n, p, ref_res.iterations, gres.iterations, kpc.fallbacks.size(), gpc.fallbacks().size(), rel(jg, jr),
              rel(zg, zr));
  return ref_res.iterations == gres.iterations ? 0 : 1;
}
