// tpdg_gpu.hpp -- header-only C++ drop-in over the C ABI (tpdg_gpu.h).
//
// Mirrors the reference's operator / preconditioner interface so that a newton_linear_solve-style
// caller (reference solve/time_step.hpp:57-122) switches implementation without changing shape:
//
//   reference                                   drop-in
//   make_linearized_operator(sys, cache, dt)    tpdg::gpu::LinearizedOperator(ctx, lin)
//   jacobian_apply(lin, v)                      op.apply(in, out)            (host spans)
//   form_ksvd_2d / form_ksvd_3d(lin, mode, cfg) tpdg::gpu::form_ksvd(op, cfg)
//   KsvdPC2D::apply(in, out)                    pc.apply(in, out)            (host spans)
//   KsvdPC2D::fallbacks                         pc.fallbacks()
//   gmres(op, pc, b, GmresConfig)               tpdg::gpu::gmres(op, pc, b, cfg)
//   form_block_jacobi(lin, mode, budget)        tpdg::gpu::form_block_jacobi(op, budget)
//   GmresFailure{what, GmresResult}             tpdg::GmresFailure (reference types) / gpu::GmresFailure
//
// Define TPDG_GPU_WITH_REFERENCE (with the reference's proj/include on the include path) to get the
// constructors taking the reference's own types and errors re-thrown as the reference's exception
// classes; otherwise errors surface as tpdg::gpu::Error carrying the status code.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <algorithm>
#include <string>
#include <utility>
#include <vector>

#include "tpdg_gpu.h"

#if __has_include("tpdg/precond/ksvd.hpp") && defined(TPDG_GPU_WITH_REFERENCE)
#include "tpdg/precond/ksvd.hpp"
#include "tpdg/solve/gmres.hpp"
#define TPDG_GPU_REFERENCE_TYPES 1
#endif

namespace tpdg::gpu {

struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& what) : std::runtime_error(what), status(s) {}
};

inline void check(int rc) {
  if (rc == TPDG_OK) return;
  const std::string msg = tpdg_gpu_last_error();
#ifdef TPDG_GPU_REFERENCE_TYPES
  switch (rc) {  // the reference's hierarchy (common/error.hpp:9-42)
    case TPDG_SHAPE: throw tpdg::ShapeError(msg);
    case TPDG_SINGULAR: throw tpdg::SingularError(msg);
    case TPDG_STATE: throw tpdg::StateError(msg);
    case TPDG_CONVERGENCE: throw tpdg::ConvergenceError(msg);
    case TPDG_CONFIG: throw tpdg::ConfigError(msg);
    default: break;
  }
#endif
  throw Error(rc, msg);
}

class Context {
 public:
  explicit Context(int device = 0, int rank = 0, int nranks = 1, const void* nccl_id = nullptr) {
    check(tpdg_gpu_ctx_create(device, rank, nranks, nccl_id, &h_));
  }
  ~Context() { tpdg_gpu_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  tpdg_gpu_ctx handle() const { return h_; }

 private:
  tpdg_gpu_ctx h_ = nullptr;
};

// Flat views of a Discretization + LinearizationCache (reference layouts, no copies).
struct SystemArrays {
  tpdg_gpu_system sys{};
  std::vector<int64_t> conn;  // the reference stores FaceConn structs; the ABI wants [E][2d][3]
};

#ifdef TPDG_GPU_REFERENCE_TYPES
inline SystemArrays system_of(const tpdg::LinearizedOperator& lin) {
  lin.check_cache();
  const tpdg::Discretization& d = *lin.sys;
  SystemArrays a;
  a.conn.reserve(std::size_t(d.mesh.n_elements) * 2 * d.dim * 3);
  for (int e = 0; e < d.mesh.n_elements; ++e)
    for (int f = 0; f < 2 * d.dim; ++f) {
      const auto& fc = d.mesh.faces[e][f];
      a.conn.push_back(fc.neighbor);
      a.conn.push_back(fc.neighbor_face);
      a.conn.push_back(fc.orientation);
    }
  tpdg_gpu_system& s = a.sys;
  s.dim = d.dim;
  s.n_c = d.n_c;
  s.p = d.ref.p;
  s.mu = d.mu;
  s.n_elements = d.mesh.n_elements;
  s.g = d.ref.g.data();
  s.d = d.ref.d.data();
  s.gw = d.ref.gw.data();
  s.dw = d.ref.dw.data();
  s.w = d.ref.qweights.data();
  s.jdet = d.mesh.jdet.data();
  s.face_w = d.mesh.face_w.data();
  s.conn = a.conn.data();
  s.dft = lin.cache->dft.data();
  s.dfm = lin.cache->dfm.data();
  s.dfp = lin.cache->dfp.data();
  s.state_hash = lin.cache->hash;
  return a;
}
#endif

class LinearizedOperator {
 public:
  // dt: backward-Euler step (operator M - dt J, the reference's mass_minus_dt_jacobian mode).
  // jacobian_only = 1: J alone (LinearizedOperator::Mode::jacobian_only, ops/linearized.hpp:167-178).
  LinearizedOperator(const Context& ctx, const tpdg_gpu_system& sys, double dt, int block_mode = 0,
                     int e_begin = 0, int e_end = -1, int jacobian_only = 0)
      : n_c_(sys.n_c), npe_(sys.dim == 2 ? (sys.p + 1) * (sys.p + 1) : (sys.p + 1) * (sys.p + 1) * (sys.p + 1)),
        block_mode_(block_mode), jacobian_only_(jacobian_only), n1d_(sys.p + 1) {
    check(tpdg_gpu_op_create(ctx.handle(), &sys, dt, jacobian_only, block_mode, e_begin,
                             e_end < 0 ? sys.n_elements : e_end, &h_));
    check(tpdg_gpu_op_local_size(h_, &n_));
    n_elements_ = int(n_ / (std::int64_t(n_c_) * npe_));
  }
#ifdef TPDG_GPU_REFERENCE_TYPES
  // Honours lin.mode and lin.block_mode; lin.check_cache() runs inside system_of (stale hash -> ConfigError).
  LinearizedOperator(const Context& ctx, const tpdg::LinearizedOperator& lin)
      : LinearizedOperator(ctx, system_of(lin).sys, lin.dt, lin.block_mode == tpdg::BlockMode::small ? 1 : 0, 0, -1,
                           lin.mode == tpdg::LinearizedOperator::Mode::jacobian_only ? 1 : 0) {}
#endif
  ~LinearizedOperator() { tpdg_gpu_op_destroy(h_); }
  LinearizedOperator(const LinearizedOperator&) = delete;
  LinearizedOperator& operator=(const LinearizedOperator&) = delete;

  void apply(std::span<const double> in, std::span<double> out) const {
    if (std::int64_t(in.size()) != n_ || std::int64_t(out.size()) != n_) check_shape();
    check(tpdg_gpu_jv_host(h_, in.data(), out.data()));
  }
  std::int64_t size() const { return n_; }
  tpdg_gpu_op handle() const { return h_; }
  int n_elements() const { return n_elements_; }
  int n_c() const { return n_c_; }
  int npe() const { return npe_; }
  int n1d() const { return n1d_; }
  int block_mode() const { return block_mode_; }
  bool jacobian_only() const { return jacobian_only_ != 0; }

 private:
  [[noreturn]] static void check_shape() { throw Error(TPDG_SHAPE, "jacobian_apply: state shape mismatch"); }
  tpdg_gpu_op h_ = nullptr;
  std::int64_t n_ = 0;
  int n_c_ = 1, npe_ = 1, block_mode_ = 0, jacobian_only_ = 0, n1d_ = 1, n_elements_ = 0;
};

struct FallbackEvent {
  int element = 0;
  int component = -1;
};

// KsvdPC2D / KsvdPC3D (precond/ksvd.hpp:161-170, 199-208) and BlockJacobiPC (block_jacobi.hpp:13-19):
// the public shape fields of the reference classes, the factors stay on the device.
class KsvdPC {
 public:
  KsvdPC(tpdg_gpu_pc h, const LinearizedOperator& op)
      : mode(op.block_mode()), n_elements(op.n_elements()), n_c(op.n_c()), npe(op.npe()), n1d(op.n1d()), h_(h),
        n_(op.size()) {}
  ~KsvdPC() { tpdg_gpu_pc_destroy(h_); }
  KsvdPC(const KsvdPC&) = delete;
  KsvdPC& operator=(const KsvdPC&) = delete;
  KsvdPC(KsvdPC&& o) noexcept
      : mode(o.mode), n_elements(o.n_elements), n_c(o.n_c), npe(o.npe), n1d(o.n1d), h_(std::exchange(o.h_, nullptr)),
        n_(o.n_) {}

  int mode = 0;  // BlockMode: 0 = full, 1 = small
  int n_elements = 0;
  int n_c = 0;
  int npe = 0;
  int n1d = 0;

  void apply(std::span<const double> in, std::span<double> out) const {
    check(tpdg_gpu_pc_apply_host(h_, in.data(), out.data()));
  }
  std::vector<FallbackEvent> fallbacks() const {
    int n = 0;
    check(tpdg_gpu_pc_num_fallbacks(h_, &n));
    std::vector<int64_t> pairs(2 * std::size_t(n));
    if (n) check(tpdg_gpu_pc_fallbacks(h_, pairs.data()));
    std::vector<FallbackEvent> ev(n);
    for (int i = 0; i < n; ++i) ev[i] = {int(pairs[2 * i]), int(pairs[2 * i + 1])};
    return ev;
  }
  tpdg_gpu_pc handle() const { return h_; }

 private:
  tpdg_gpu_pc h_ = nullptr;
  std::int64_t n_ = 0;
};

inline KsvdPC form_ksvd(const LinearizedOperator& op, tpdg_gpu_ksvd_config cfg = {2, 0, 1e-12, 0x5eedULL, 1e-12}) {
  tpdg_gpu_pc h = nullptr;
  check(tpdg_gpu_form_ksvd(op.handle(), &cfg, &h));
  return KsvdPC(h, op);
}

// form_block_jacobi (precond/block_jacobi.hpp:38-72): the block mode is the operator's; max_total_entries <= 0
// selects the reference's default budget (3e8). ConfigError over budget, SingularError on a singular block.
inline KsvdPC form_block_jacobi(const LinearizedOperator& op, long max_total_entries = 300'000'000) {
  tpdg_gpu_pc h = nullptr;
  check(tpdg_gpu_form_block_jacobi(op.handle(), max_total_entries, &h));
  return KsvdPC(h, op);
}

#ifdef TPDG_GPU_REFERENCE_TYPES
using GmresResult = tpdg::GmresResult;
using GmresFailure = tpdg::GmresFailure;
#else
struct GmresResult {
  std::vector<double> x;
  int iterations = 0;
  std::vector<double> residual_history;
  bool converged = false;
};
// solve/gmres.hpp:39-44: thrown when the iteration budget runs out; carries the best iterate.
struct GmresFailure : Error {
  GmresFailure(const std::string& what, GmresResult r) : Error(TPDG_CONVERGENCE, what), result(std::move(r)) {}
  GmresResult result;
};
#endif

inline GmresResult gmres(const LinearizedOperator& op, const KsvdPC& pc, std::span<const double> b,
                         tpdg_gpu_gmres_config cfg = {1e-5, 60, 2000, 0}) {
  GmresResult r;
  r.x.assign(b.size(), 0.0);
  r.residual_history.assign(std::size_t(cfg.max_iterations) + 1, 0.0);
  int conv = 0;
  const int rc = tpdg_gpu_gmres_host(op.handle(), pc.handle(), b.data(), r.x.data(), &cfg, &r.iterations,
                                     r.residual_history.data(), int(r.residual_history.size()), &conv);
  r.residual_history.resize(std::min(r.residual_history.size(), std::size_t(r.iterations)));
  r.converged = conv != 0;
  // budget exhausted: GmresFailure carrying the best iterate, like gmres.hpp:165-178
  if (rc == TPDG_CONVERGENCE) throw GmresFailure(tpdg_gpu_last_error(), std::move(r));
  if (rc != TPDG_OK) check(rc);
  return r;
}

} // namespace tpdg::gpu
