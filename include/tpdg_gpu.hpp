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
//
// Define TPDG_GPU_WITH_REFERENCE (with the reference's proj/include on the include path) to get the
// constructors taking the reference's own types and errors re-thrown as the reference's exception
// classes; otherwise errors surface as tpdg::gpu::Error carrying the status code.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
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
  LinearizedOperator(const Context& ctx, const tpdg_gpu_system& sys, double dt, int block_mode = 0,
                     int e_begin = 0, int e_end = -1) {
    check(tpdg_gpu_op_create(ctx.handle(), &sys, dt, 0, block_mode, e_begin, e_end < 0 ? sys.n_elements : e_end,
                             &h_));
    check(tpdg_gpu_op_local_size(h_, &n_));
  }
#ifdef TPDG_GPU_REFERENCE_TYPES
  LinearizedOperator(const Context& ctx, const tpdg::LinearizedOperator& lin)
      : LinearizedOperator(ctx, system_of(lin).sys, lin.dt, lin.block_mode == tpdg::BlockMode::small ? 1 : 0) {}
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

 private:
  [[noreturn]] static void check_shape() { throw Error(TPDG_SHAPE, "jacobian_apply: state shape mismatch"); }
  tpdg_gpu_op h_ = nullptr;
  std::int64_t n_ = 0;
};

struct FallbackEvent {
  int element = 0;
  int component = -1;
};

class KsvdPC {
 public:
  explicit KsvdPC(tpdg_gpu_pc h, std::int64_t n) : h_(h), n_(n) {}
  ~KsvdPC() { tpdg_gpu_pc_destroy(h_); }
  KsvdPC(const KsvdPC&) = delete;
  KsvdPC& operator=(const KsvdPC&) = delete;
  KsvdPC(KsvdPC&& o) noexcept : h_(std::exchange(o.h_, nullptr)), n_(o.n_) {}

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
  return KsvdPC(h, op.size());
}

struct GmresResult {
  std::vector<double> x;
  int iterations = 0;
  std::vector<double> residual_history;
  bool converged = false;
};

inline GmresResult gmres(const LinearizedOperator& op, const KsvdPC& pc, std::span<const double> b,
                         tpdg_gpu_gmres_config cfg = {1e-5, 60, 2000, 0}) {
  GmresResult r;
  r.x.assign(b.size(), 0.0);
  r.residual_history.assign(std::size_t(cfg.max_iterations) + 1, 0.0);
  int conv = 0;
  const int rc = tpdg_gpu_gmres_host(op.handle(), pc.handle(), b.data(), r.x.data(), &cfg, &r.iterations,
                                     r.residual_history.data(), int(r.residual_history.size()), &conv);
  r.residual_history.resize(std::size_t(r.iterations));
  r.converged = conv != 0;
  if (rc != TPDG_OK) check(rc);  // TPDG_CONVERGENCE <-> GmresFailure (best iterate in r.x)
  return r;
}

} // namespace tpdg::gpu
