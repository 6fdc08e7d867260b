/* tpdg_gpu.h -- C ABI of the B200 (sm_100a) KSVD-preconditioned matrix-free GMRES hot path.
 *
 * Drop-in boundary for the reference library `tpdg` (header-only C++20). Every entry point
 * replaces one reference interface on the path newton_linear_solve runs
 * (reference proj/include/tpdg/solve/time_step.hpp:57-122); citations are relative to
 * /root/reference/proj/include/tpdg/:
 *
 *   tpdg_gpu_op_create        make_linearized_operator        ops/linearized.hpp:187-196
 *                             (+ the LinearizationCache it binds, ops/linearized.hpp:15-33)
 *   tpdg_gpu_jv               jacobian_apply                  ops/linearized.hpp:201-240
 *   tpdg_gpu_shuffled         shuffled_apply(_transpose)      ops/shuffled.hpp:509-531
 *   tpdg_gpu_form_ksvd        form_ksvd_2d / form_ksvd_3d     precond/ksvd.hpp:252-306, 312-372
 *   tpdg_gpu_form_block_jacobi form_block_jacobi              precond/block_jacobi.hpp:38-72
 *   tpdg_gpu_pc_apply         KsvdPC2D::apply / KsvdPC3D::apply precond/ksvd.hpp:172-195, 210-233
 *   tpdg_gpu_pc_fallbacks     KsvdPC*::fallbacks (FallbackEvent) precond/ksvd.hpp:22-28
 *   tpdg_gpu_gmres            gmres(op, pc, b, GmresConfig)   solve/gmres.hpp:52-179
 *   status codes              tpdg::Error hierarchy           common/error.hpp:9-42
 *
 * Conventions
 *  - Plain C types only. Arrays are in the reference's own index orders (no re-layout at the
 *    boundary; kernels re-tile internally):
 *      state vectors  [e][c][tensor index, x fastest]                  (ops/state.hpp:12-13)
 *      g, d           mu x (p+1) row-major; gw, dw (p+1) x mu          (dg/reference_element.hpp:24-27)
 *      w              mu quadrature weights on [0,1]
 *      jdet           [e][mu^dim]; face_w [e][2*dim][mu^(dim-1)]       (dg/mesh.hpp:87-92)
 *      conn           [e][2*dim][3] = neighbor, neighbor_face, orientation (dg/mesh.hpp:37-42);
 *                     neighbor < 0 marks a boundary face
 *      dft            [e][dir][mu^dim][n_c][n_c]; dfm, dfp [e][face][mu^(dim-1)][n_c][n_c]
 *  - Functions never throw; they return a tpdg_status. tpdg_gpu_last_error() gives the message of
 *    the last failure on the calling thread. Per-element singularity is NOT an error: it is
 *    reported through the fallback list exactly like FallbackEvent.
 *  - `_host` entry points take host pointers and copy in/out inside the call; the others take
 *    device pointers and are ordered on the context's CUDA stream (synchronous on return unless
 *    stated otherwise).
 *  - Objects are owned by the caller and released with tpdg_gpu_*_destroy.
 */
#ifndef TPDG_GPU_H
#define TPDG_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TPDG_OK = 0,
  TPDG_SHAPE = 1,        /* tpdg::ShapeError */
  TPDG_SINGULAR = 2,     /* tpdg::SingularError */
  TPDG_STATE = 3,        /* tpdg::StateError */
  TPDG_CONVERGENCE = 4,  /* tpdg::ConvergenceError / GmresFailure (best iterate still returned) */
  TPDG_CONFIG = 5,       /* tpdg::ConfigError (incl. stale-cache hash mismatch) */
  TPDG_CUDA = 6          /* CUDA / NCCL runtime failure (no reference equivalent) */
} tpdg_status;

typedef struct tpdg_gpu_ctx_s *tpdg_gpu_ctx;
typedef struct tpdg_gpu_op_s *tpdg_gpu_op;
typedef struct tpdg_gpu_pc_s *tpdg_gpu_pc;

/* Discretization + linearization as flat host arrays (GLOBAL mesh; see layouts above).
 * Mirrors Discretization (ops/discretization.hpp:17-35) + LinearizationCache. */
typedef struct {
  int dim, n_c, p, mu, n_elements;
  const double *g, *d, *gw, *dw, *w;
  const double *jdet, *face_w;
  const int64_t *conn;
  const double *dft, *dfm, *dfp;
  uint64_t state_hash; /* LinearizationCache::hash (ops/linearized.hpp:16) */
} tpdg_gpu_system;

/* KsvdConfig + LanczosConfig (precond/ksvd.hpp:16-20, tensor/lanczos.hpp:15-30). */
typedef struct {
  int terms;               /* r, default 2 */
  int lanczos_max_it;      /* J, 0 = 2r + 20 */
  double breakdown_tol;    /* default 1e-12 */
  uint64_t seed;           /* default 0x5eed */
  double degenerate_tol;   /* default 1e-12 */
} tpdg_gpu_ksvd_config;

/* GmresConfig (solve/gmres.hpp:14-29). side: 0 = right (default), 1 = left. */
typedef struct {
  double tol;
  int restart;
  int max_iterations;
  int side;
} tpdg_gpu_gmres_config;

const char *tpdg_gpu_last_error(void);
const char *tpdg_gpu_version(void);

/* ---- context: one per GPU / rank. nccl_id: 128-byte ncclUniqueId for nranks > 1, else NULL. */
int tpdg_gpu_ctx_create(int device, int rank, int nranks, const void *nccl_id, tpdg_gpu_ctx *out);
int tpdg_gpu_ctx_destroy(tpdg_gpu_ctx ctx);
int tpdg_gpu_ctx_stream(tpdg_gpu_ctx ctx, void **cuda_stream);
int tpdg_gpu_ctx_sync(tpdg_gpu_ctx ctx);
int tpdg_gpu_nccl_unique_id(void *out128);
/* Count of this library's kernel launches on the context so far (bench evidence). */
int tpdg_gpu_ctx_launches(tpdg_gpu_ctx ctx, int64_t *count);
/* CUDA-event timing per kernel class on the context stream (enable resets the record):
 * class 0 = Kronecker PC apply, 1 = Jv, 2 = MGS + norm passes, 3 = other. */
int tpdg_gpu_ctx_profile(tpdg_gpu_ctx ctx, int enable);
int tpdg_gpu_ctx_profile_read(tpdg_gpu_ctx ctx, double *ms /* [4] */, int64_t *counts /* [4] */);

/* ---- operator (M - dt J) (jacobian_only = 0) or J (jacobian_only = 1) of the elements
 * [e_begin, e_end) owned by this rank. block_mode: 0 = full, 1 = small. */
int tpdg_gpu_op_create(tpdg_gpu_ctx ctx, const tpdg_gpu_system *sys, double dt, int jacobian_only, int block_mode,
                       int e_begin, int e_end, tpdg_gpu_op *out);
int tpdg_gpu_op_destroy(tpdg_gpu_op op);
int tpdg_gpu_op_local_size(tpdg_gpu_op op, int64_t *n_local);
/* check_cache (ops/linearized.hpp:180-184): TPDG_CONFIG when hash != the op's bound hash */
int tpdg_gpu_op_check_hash(tpdg_gpu_op op, uint64_t expected_hash);
int tpdg_gpu_jv(tpdg_gpu_op op, const double *d_in, double *d_out);
int tpdg_gpu_jv_host(tpdg_gpu_op op, const double *h_in, double *h_out);
/* Matrix-free shuffled product of one (local) element block; test hook. */
int tpdg_gpu_shuffled_host(tpdg_gpu_op op, int e, int comp, int transpose, const double *h_in, double *h_out);

/* ---- KSVD preconditioner, formed on the device (no host fallback). */
int tpdg_gpu_form_ksvd(tpdg_gpu_op op, const tpdg_gpu_ksvd_config *cfg, tpdg_gpu_pc *out);
/* Exact block-Jacobi preconditioner (BlockJacobiPC / form_block_jacobi, precond/block_jacobi.hpp:13-72):
 * every diagonal block (element, or element x component in small mode) assembled on the device by
 * probing the element operator and LU-factored with partial pivoting; applied with the same
 * tpdg_gpu_pc_apply. ConfigError when block^2 x blocks exceeds max_total_entries (<= 0: the
 * reference's default 3e8), SingularError on a singular block. The paper's comparison baseline. */
int tpdg_gpu_form_block_jacobi(tpdg_gpu_op op, int64_t max_total_entries, tpdg_gpu_pc *out);
/* Test hook: build the apply state from externally formed raw factors (2D: a1 b1 a2 b2,
 * 3D: a1 b1 c1 b2 c2 per block, concatenated for blocks with has[blk] != 0; LU and Schur are
 * recomputed on the device exactly as make_factors_2d/3d do). Blocks with has == 0 get the
 * exact block-LU fallback. */
int tpdg_gpu_pc_import_factors(tpdg_gpu_op op, const double *h_factors, const int64_t *h_has, tpdg_gpu_pc *out);
/* As import_factors, but the apply state of every factored block is taken as given instead of
 * recomputed: h_rec = per block (has != 0, concatenated) the LU factors then the Schur pairs
 * (2D: LU(A2) LU(B1) Q1 T1 Q2 T2; 3D: LU(A1) LU(B2) LU(C1) Q1 T1 Q2 T2, the LuFactor and
 * SchurPair members of Factors2D / Factors3D, precond/ksvd.hpp:34-46), h_piv = their pivots.
 * Isolates the apply (ksvd.hpp:112-153) from the formation's libm-dependent Schur rotations. */
int tpdg_gpu_pc_import_record(tpdg_gpu_op op, const double *h_factors, const int64_t *h_has, const double *h_rec,
                              const int *h_piv, tpdg_gpu_pc *out);
int tpdg_gpu_pc_destroy(tpdg_gpu_pc pc);
int tpdg_gpu_pc_num_fallbacks(tpdg_gpu_pc pc, int *n);
int tpdg_gpu_pc_fallbacks(tpdg_gpu_pc pc, int64_t *pairs /* (element, component) x n */);
int tpdg_gpu_pc_factor_len(tpdg_gpu_pc pc, int *len);
int tpdg_gpu_pc_export_factors(tpdg_gpu_pc pc, int blk, double *h_out, int *has);
int tpdg_gpu_pc_apply(tpdg_gpu_pc pc, const double *d_in, double *d_out);
int tpdg_gpu_pc_apply_host(tpdg_gpu_pc pc, const double *h_in, double *h_out);

/* ---- restarted GMRES, device resident. hist (may be NULL) receives |g_{k+1}| per iteration
 * (GmresResult::residual_history). Returns TPDG_CONVERGENCE (with x = best iterate) when the
 * budget runs out, like GmresFailure. */
int tpdg_gpu_gmres(tpdg_gpu_op op, tpdg_gpu_pc pc, const double *d_b, double *d_x, const tpdg_gpu_gmres_config *cfg,
                   int *iterations, double *hist, int hist_cap, int *converged);
int tpdg_gpu_gmres_host(tpdg_gpu_op op, tpdg_gpu_pc pc, const double *h_b, double *h_x,
                        const tpdg_gpu_gmres_config *cfg, int *iterations, double *hist, int hist_cap,
                        int *converged);

/* ---- multi-rank element partition and face-neighbour halo plan (host only; what op_create uses
 * for nranks > 1). Rank r owns [E r / N, E (r+1) / N). conn: [n_local][2d][3] with neighbours
 * mapped to local ids (< n_local) or halo slots (n_local + s); halo_gid: global id per slot;
 * peer i: elements this rank sends (local ids, ascending) and the halo slot range it receives. */
typedef struct tpdg_halo_plan_s *tpdg_halo_plan;
int tpdg_halo_plan_create(const tpdg_gpu_system *sys, int rank, int nranks, tpdg_halo_plan *out);
int tpdg_halo_plan_query(tpdg_halo_plan h, int *e_begin, int *e_end, int *n_halo, int *n_peers);
int tpdg_halo_plan_conn(tpdg_halo_plan h, int *conn_out);
int tpdg_halo_plan_halo_gid(tpdg_halo_plan h, int *gid_out);
/* Per peer: n_send face layers sent (send_pairs: local element, face) and n_recv received (recv_pairs: halo
 * slot, face of the halo element), both ordered by (global element, face); one layer = n_c q^(d-1) doubles
 * (the neighbour trace of ops/discretization.hpp:89-97 / 170-181). Pair arrays may be NULL (counts only). */
int tpdg_halo_plan_peer(tpdg_halo_plan h, int i, int *rank, int *n_send, int *send_pairs, int *n_recv,
                        int *recv_pairs);
int tpdg_halo_plan_destroy(tpdg_halo_plan h);
/* In-process transport: nranks contexts in one process (one host thread each, same or different GPUs) run
 * the multi-rank data plane (face-layer halo exchange, GMRES allreduces) with device copies and a fixed-order
 * sum instead of NCCL. Used to validate the distributed path on one GPU (tests/test_gpu_loopback.py). */
typedef struct tpdg_gpu_loopback_s *tpdg_gpu_loopback;
int tpdg_gpu_loopback_create(int nranks, tpdg_gpu_loopback *out);
int tpdg_gpu_loopback_destroy(tpdg_gpu_loopback h);
int tpdg_gpu_ctx_create_loopback(int device, int rank, tpdg_gpu_loopback hub, tpdg_gpu_ctx *out);

/* ---- host-side input production for the BASELINE configurations (out of the kernel scope;
 * restates build_reference / generate_mesh(cartesian) / build_cache for scalar advection).
 * case_kind: 0 = 2D constant velocity (vel[0], vel[1]); 1 = 2D swirl (sin 2 pi y, cos 2 pi x);
 *            2 = 3D constant velocity (vel[0..2]).
 * Returned arrays are owned by the setup object. */
typedef struct tpdg_setup_s *tpdg_setup;
int tpdg_setup_advection(int case_kind, const double *vel, int nx, int ny, int nz, int p, int periodic,
                         tpdg_setup *out);
int tpdg_setup_system(tpdg_setup s, tpdg_gpu_system *sys);
/* geometry at the quadrature points: adjugates [E][nvol][d][d], points [E][nvol][d], face unit normals and
 * points [E][2d][nface][d] (mesh.hpp:72-106 adj_at / vol_x_at / face_n_at / face_x_at) */
int tpdg_setup_geometry(tpdg_setup s, const double **adj, const double **vol_x, const double **face_n,
                        const double **face_x, int *nvol, int *nface);
/* build_cache (ops/linearized.hpp:38-100) of scalar upwind advection on the device, from device copies of the
 * geometry: dft [E][d][nvol], dfm / dfp [E][2d][nface] (n_c = 1). field: 0 / 2 constant velocity vel (2D / 3D),
 * 1 = (sin 2 pi y, cos 2 pi x). SURVEY.md sec.8f row 1 for the advection laws. */
int tpdg_gpu_build_cache_advection(tpdg_gpu_ctx ctx, int dim, int n_elements, int nvol, int nface, const double *d_adj,
                                   const double *d_vol_x, const double *d_face_n, const double *d_face_x,
                                   const int64_t *d_conn, int field, const double *vel, double *d_dft, double *d_dfm,
                                   double *d_dfp);
/* Test hook: the device libm of the formation (csrc/glibm.cuh, glibc 2.39's sin/cos/atan/atan2 as called by
 * standardize_2x2, tensor/schur.hpp:91-108) on n device arguments. fn: 0 sin, 1 cos, 2 atan, 3 atan2(x, y). */
int tpdg_gpu_libm_eval(tpdg_gpu_ctx ctx, int fn, int64_t n, const double *d_x, const double *d_y, double *d_out);
/* Test hook: one modified Gram-Schmidt step of the Arnoldi process as the GMRES driver launches it
 * (solve/gmres.hpp:112-121): d_V holds rows v_0 .. v_k (orthonormal basis) and row k+1 = w, each of n doubles at
 * stride ldv (a multiple of 2, >= n); on return h[0 .. k] = the projections, h[k+1] = ||w||, and row k+1 is the
 * normalized w. h: host array of k + 2 doubles. */
int tpdg_gpu_mgs_step(tpdg_gpu_ctx ctx, double *d_V, int64_t ldv, int k, int64_t n, double *h);
/* build_cache (ops/linearized.hpp:38-100) of the LLF Euler law (laws/euler.hpp:106-211) on the device from the
 * nodal linearization state [e][c][node] and the quadrature-point geometry (adj [e][q][d][d], face_n
 * [e][f][qf][d]); G is the reference element's (mu x p+1) interpolation matrix. TPDG_STATE on a
 * non-physical state (check_state, euler.hpp:14-27). Single rank (neighbour states are local). */
int tpdg_gpu_build_cache_euler(tpdg_gpu_ctx ctx, int dim, int p, int mu, int n_elements, const double *d_g,
                               const double *d_state, const double *d_adj, const double *d_face_n,
                               const int64_t *d_conn, double *d_dft, double *d_dfm, double *d_dfp);
/* residual r(u, t) (ops/discretization.hpp:188-254) of the LLF Euler law on the device (device pointers,
 * global mesh, single rank). TPDG_STATE on a non-physical state. */
int tpdg_gpu_residual_euler(tpdg_gpu_ctx ctx, int dim, int p, int mu, int n_elements, const double *d_g,
                            const double *d_gw, const double *d_dw, const double *d_state, const double *d_adj,
                            const double *d_face_n, const double *d_face_w, const int64_t *d_conn, double *d_out);
/* One backward Euler step of the Euler law by Newton-GMRES with the KSVD preconditioner, everything on the
 * device (step_backward_euler, solve/time_step.hpp:136-146; newton, solve/newton.hpp:32-68;
 * newton_linear_solve, time_step.hpp:57-122): per Newton step the linearization cache is rebuilt at the
 * iterate, the preconditioner formed, GMRES run on -G(w), G(w) = M (w - u) - dt r(w). h_u: u in, u' out
 * (host, [e][c][node]); newton_tol / max_iterations / floor as NewtonConfig; statistics per solve are
 * written up to cap entries (residual_norms: cap + 1). TPDG_CONVERGENCE on the reference's failure modes. */
int tpdg_gpu_step_backward_euler(tpdg_gpu_ctx ctx, const tpdg_gpu_system *sys, const double *h_adj,
                                 const double *h_face_n, double *h_u, double dt, double newton_tol,
                                 int newton_max_iterations, double newton_floor, const tpdg_gpu_gmres_config *gcfg,
                                 const tpdg_gpu_ksvd_config *kcfg, int block_mode, int *newton_steps,
                                 int *gmres_per_solve, double *residual_norms, int cap);
/* Euler stand-ins of BASELINE configs[2] (case 3: 2D, [0,10]^2) and configs[4] (case 5: 3D, [0,2pi]^3):
 * geometry plus the interpolated nodal state (host_setup.cpp); the cache is left zero for the device. */
int tpdg_setup_euler(int case_kind, int nx, int ny, int nz, int p, tpdg_setup *out);
int tpdg_setup_state(tpdg_setup s, const double **state, int64_t *n);
int tpdg_setup_destroy(tpdg_setup s);
/* libstdc++ std::mt19937_64 + uniform_real_distribution(-scale, scale) (tests/support/test_rng.hpp) */
int tpdg_uniform_vector(uint64_t seed, int64_t n, double scale, double *out);
/* tpdg::detail::seeded_unit_vector (tensor/lanczos.hpp:61-72) */
int tpdg_seeded_unit_vector(int64_t n, uint64_t seed, double *out);

#ifdef __cplusplus
}
#endif
#endif /* TPDG_GPU_H */
