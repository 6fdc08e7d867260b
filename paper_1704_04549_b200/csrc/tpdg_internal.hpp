// Internal declarations shared by the C-ABI layer (capi.cu), the kernels and the host setup.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "tpdg_gpu.h"

namespace tpdg_gpu {

// ---------------------------------------------------------------- errors
struct Failure {
  int status;
  std::string what;
};
void set_error(const std::string& what);

#define TPDG_CUDA_CHECK(expr)                                                                         \
  do {                                                                                                \
    cudaError_t err__ = (expr);                                                                       \
    if (err__ != cudaSuccess)                                                                         \
      throw ::tpdg_gpu::Failure{TPDG_CUDA, std::string(#expr) + ": " + cudaGetErrorString(err__)};    \
  } while (0)

// ---------------------------------------------------------------- host setup
struct Setup {
  int dim = 2, n_c = 1, p = 1, mu = 3, n_elements = 0;
  std::vector<double> g, d, gw, dw, w, qpoints, jdet, face_w, dft, dfm, dfp, vol_x;
  std::vector<double> adj, face_n, face_x;  // geometry at the quadrature points (build_cache inputs)
  std::vector<double> state;                // nodal linearization state (Euler stand-ins) [e][c][node]
  std::vector<int64_t> conn;
  uint64_t state_hash = 0;
};
int setup_advection(int kind, const double* vel, int nx, int ny, int nz, int p, int periodic, Setup& s);
void uniform_vector(uint64_t seed, int64_t n, double scale, double* out);
// build_cache of scalar upwind advection on the device (cache.cu); device pointers
void launch_libm_eval(int fn, int64_t n, const double* x, const double* y, double* out, cudaStream_t st);
// build_cache of the LLF Euler law (laws/euler.hpp) on the device from the nodal state
void launch_build_cache_euler(int dim, int q, int mu, int n_elements, const double* g, const double* state,
                              const double* adj, const double* face_n, const int64_t* conn, double* dft, double* dfm,
                              double* dfp, int* status, cudaStream_t st);
// residual r(u) of the LLF Euler law (ops/discretization.hpp:188-254) on the device
void launch_residual_euler(int dim, int q, int mu, int n_elements, const double* g, const double* gw, const double* dw,
                           const double* state, const double* adj, const double* face_n, const double* face_w,
                           const int64_t* conn, double* out, int* status, cudaStream_t st);
void launch_build_cache_advection(int dim, int n_elements, int nvol, int nface, const double* adj,
                                  const double* vol_x, const double* face_n, const double* face_x,
                                  const int64_t* conn, int field, const double* vel, double* dft, double* dfm,
                                  double* dfp, cudaStream_t st);
void seeded_unit_vector(int64_t n, uint64_t seed, double* out);

// ---------------------------------------------------------------- multi-rank plan (halo.cpp)
struct HaloPlan {
  int e_begin = 0, e_end = 0, n_halo = 0;
  std::vector<int> conn;          // [n_local][2d][3]: neighbour -> local id (< n_local) or halo slot
  std::vector<int> halo_gid;      // global element id of each halo slot
  // Face traces: what crosses ranks is, per cut face, the neighbour's face node layer (GL nodes: the
  // trace is that layer, ops/discretization.hpp:89-97), n_c q^(d-1) doubles, not the element block.
  struct Peer {
    int rank = 0;
    std::vector<int> send_elem, send_face;  // local element and face of each layer sent (ascending (gid, face))
    std::vector<int> recv_slot, recv_face;  // halo slot and face of each layer received (same order)
  };
  std::vector<Peer> peers;
};
HaloPlan build_halo_plan(const tpdg_gpu_system* sys, int rank, int nranks, int e_begin, int e_end);
// Element-block offset of node t of face f's node layer (t < q^(d-1); lower tangential axis fastest).
__host__ __device__ inline int face_layer_index(int d, int q, int f, int t) {
  const int axis = f / 2, layer = (f % 2) == 0 ? 0 : q - 1;
  if (d == 2) return axis == 0 ? layer + q * t : t + q * layer;
  const int u = t % q, v = t / q;
  return axis == 0 ? layer + q * (u + q * v) : axis == 1 ? u + q * (layer + q * v) : u + q * (v + q * layer);
}

// ---------------------------------------------------------------- device views (POD, by value)
// Discretization + linearization of the local elements, reference layouts.
struct DevSys {
  int dim, n_c, q, mu, npe, nqv, nqf, n_local, n_halo;
  int e_lo, e_hi;     // the launch processes local elements [e_lo, e_hi) (interior / boundary split)
  int small;          // BlockMode::small
  double a, b;        // mass / jacobian coefficients (ops/linearized.hpp:177-178)
  const double *g, *d, *gw, *dw, *w;
  const double *jdet, *face_w, *dft, *dfm, *dfp;  // local element 0 first
  const int* conn;    // [n_local][2d][3]; neighbor index < n_local: local, >= n_local: halo slot
  const int* skip;    // optional device flag: kernels return immediately when *skip != 0
  const double *cdfm, *cdfp;  // face Jacobians pre-scaled by -b fw (device; read by jv3d_fast)
  const double* pw;           // 3D n_c = 1: [e][mu^3][a jdet, b dft_x, b dft_y, b dft_z] (device)
  // n_c > 1: the Jacobians regrouped by output component (row r of every point contiguous over the
  // points), dftr [e][r][dir][point][n_c], dfmr / dfpr [e][f][r][face point][n_c] (device; generic Jv)
  const double *dftr, *dfmr, *dfpr;
  const double *hg, *hgw, *hdw;  // HOST copies of g, gw, dw (packed into kernel parameters at launch)
};

// Formed KSVD preconditioner, device side. One factor record per block (element, or element x
// component in small mode); record layout (doubles), n1 = ncb*q:
//   2D: LU(A2) n1^2 | LU(B1) q^2 | Q1 n1^2 | T1 n1^2 | Q2 q^2 | T2 q^2
//   3D: LU(A1) n1^2 | LU(B2) q^2 | LU(C1) q^2 | Q1 q^2 | T1 q^2 | Q2 q^2 | T2 q^2
// plus int pivots  2D: n1 + q ; 3D: n1 + 2q.
struct DevPC {
  int dim, q, n1, nblk, blk_len;
  int rec_len, piv_len;
  const double* rec;     // [nblk][rec_len]
  const int* piv;        // [nblk][piv_len]
  const int* kind;       // [nblk]: 1 = Kronecker factors, 0 = dense fallback
  const int* fb_slot;    // [nblk]: slot into fb_lu for fallback blocks, -1 otherwise
  const double* fb_lu;   // [n_fb][blk_len^2]
  const int* fb_piv;     // [n_fb][blk_len]
  const int* fb_list;    // [n_fb]: block of each fallback slot
  int n_fb;
  int faithful;          // 1: bit-faithful kernels only (TPDG_GPU_FAITHFUL=1), 0: tensor-core apply
  const double* cells;   // [nblk][cells_len]: Sylvester plan + factored tiny systems (sylv_cells_len)
  int cells_len;
  const double* irec;    // [nblk][irec3_len]: 3D tensor-core apply operands (kron3d_inv_prep_kernel)
  int* status;           // device error flag (SingularError inside the Sylvester solve)
  const int* skip;       // optional device flag: kernels return immediately when *skip != 0
};

__host__ __device__ inline int rec_len_of(int dim, int n1, int q) {
  return dim == 2 ? 3 * n1 * n1 + 3 * q * q : n1 * n1 + 6 * q * q;
}
__host__ __device__ inline int piv_len_of(int dim, int n1, int q) { return dim == 2 ? n1 + q : n1 + 2 * q; }
// Sylvester cell record of one block (T1: t1 x t1, T2: t2 x t2): an int header [nb1, nb2, all11,
// 0, s1[t1], z1[t1], s2[t2], z2[t2]], tol in its last double (even count), then 6 doubles per
// Sylvester entry; the cell of quasi-blocks (bi, bk) starts at 6 (s1[bi] t2 + z1[bi] s2[bk]).
__host__ __device__ inline int sylv_hdr_doubles(int t1, int t2) { return ((4 + 2 * t1 + 2 * t2) / 2 + 2) & ~1; }
__host__ __device__ inline int sylv_cells_len(int dim, int n1, int q) {
  const int t1 = dim == 2 ? n1 : q;
  return sylv_hdr_doubles(t1, q) + 6 * t1 * q;
}
__host__ __device__ inline int raw_len_of(int dim, int n1, int q) { return dim == 2 ? 2 * n1 * n1 + 2 * q * q : n1 * n1 + 4 * q * q; }

// ---------------------------------------------------------------- kernel launchers
void launch_jv(const DevSys& s, const double* vin, const double* halo, double* vout, cudaStream_t st);
// 3D n_c = 1 operator with constant-bank weights (jv3d.cu); false if no instance fits
bool launch_jv3d_fast(const DevSys& s, const double* vin, const double* halo, double* vout, cudaStream_t st);
bool launch_jv2d_mma(const DevSys& s, const double* vin, const double* halo, double* vout, cudaStream_t st);
size_t jv_smem_bytes(const DevSys& s);
void launch_pc_apply(const DevPC& pc, const double* in, double* out, cudaStream_t st);
// 3D tensor-core apply operands of every factored block (formation time)
void launch_kron3d_inv_prep(const DevPC& pc, double* irec, cudaStream_t st);
// Row stride of the 3D Sylvester block inverses G (sz = 1, 2): segments of even(q) doubles, rows 2 (mod 4) apart
// leading dimension of a transposed G block of sz x sz T2 cells: the smallest >= sz q that is 4 (mod 8)
// Row stride of a transposed G block: >= sz q and = 2 (mod 8). The Sylvester sweep's DMMA B fragments read, per
// half-warp (LDS.64 is served one half-warp at a time), four rows k' two apart by four consecutive n: with
// 2 ld = 4 (mod 16) doubles those 16 lanes hit 16 distinct bank pairs (ld = 4 (mod 8) gave a two-way conflict:
// 4 wavefronts per load instead of 2, 19 % of the apply kernel's shared-memory wavefronts, ncu).
__host__ __device__ constexpr int g_t_ld(int q, int sz) { return (sz * q + 5) / 8 * 8 + 2; }
// A1^-1 | L^T | R | Q1 | Q2 | T2 | G blocks (<= q^2 g_t_ld(q, 2): every block 2 x 2)
__host__ __device__ inline size_t irec3_doubles(int n1, int q) { return size_t(n1) * n1 + 5 * q * q + size_t(q) * q * g_t_ld(q, 2); }
// bit-faithful 2D apply, several blocks per warp (kron_ew.cu); false if no sized variant fits
bool launch_kron2d_ew(const DevPC& pc, const double* in, double* out, cudaStream_t st);
// dense-LU fallback blocks, one CTA per fallback block (kron_fallback.cu); false if n is too large
bool launch_fallback_apply(const DevPC& pc, const double* in, double* out, cudaStream_t st);
// Factor the data-independent tiny Sylvester systems of every Kronecker block into pc.cells.
void launch_sylv_cells(const DevPC& pc, double* cells, cudaStream_t st);
void launch_shuffled(const DevSys& s, int e, int comp, int transpose, const double* in, double* out,
                     double* scratch, cudaStream_t st);
size_t shuffled_scratch_doubles(const DevSys& s);

// Form: raw factors -> records (LU, C = A^{-1} B, Schur, Sylvester check, swap).
// kind_out[blk] = 1 ok, 0 singular (needs fallback).
struct FormBuffers {
  double* raw;      // [nblk][raw_len]
  double* rec;      // [nblk][rec_len]
  int* piv;         // [nblk][piv_len]
  int* kind;        // [nblk]
  double* work;     // scratch
};
void launch_lanczos_form(const DevSys& s, const tpdg_gpu_ksvd_config& cfg, const double* start_vec,
                         const double* start_vec2, double* raw, double* sigma, int* lz_iters, double* work,
                         size_t work_per_block, int grid, cudaStream_t st);
size_t lanczos_work_doubles(const DevSys& s, int max_it);
void launch_make_factors(int dim, int q, int n1, int nblk, const double* raw, double* rec, int* piv, int* kind,
                         double* work, cudaStream_t st);
int make_factors_work_groups();
size_t probe_work_doubles(const DevSys& s);
int probe_grid(int n, int nfb);
void launch_assemble_fallback(const DevSys& s, const int* blocks, int nfb, double* fb_lu, double* work,
                              cudaStream_t st);
void launch_dense_lu(int n, int nfb, double* fb_lu, int* fb_piv, int* fb_status, cudaStream_t st);

// GMRES vector kernels
void launch_dot(const double* x, const double* y, int64_t n, double* partial, double* result, unsigned* counter,
                cudaStream_t st);
void launch_norm(const double* x, int64_t n, double* partial, double* result, unsigned* counter, cudaStream_t st);
void launch_mgs_step(double* w, const double* vprev, const double* hprev, const double* vj, int64_t n,
                     double* partial, double* result, unsigned* counter, cudaStream_t st, const int* skip,
                     bool sqrt_norm = true);
void launch_axpy_neg(double* w, const double* h, const double* v, int64_t n, cudaStream_t st);
void launch_scale_div(const double* in, const double* den, double* out, int64_t n, cudaStream_t st,
                      const int* skip = nullptr);
// Device-side Givens step of GMRES iteration k (solve/gmres.hpp:122-141); see blas.cu.
struct GmresDev {
  double *hc, *H, *cs, *sn, *g, *y;
  int* done;
  double target;
  int m;
};
struct GmresStatus {  // host-mapped, one per iteration of a cycle
  double res;
  int conv;
  int valid;
};
void launch_givens(const GmresDev& G, int k, GmresStatus* status, cudaStream_t st);
// All MGS passes + normalization of iteration k in one cooperative launch (single rank).
// With G / status, the iteration's Givens step runs at the end of the same launch (m <= 62).
void launch_mgs_iteration(double* V, int64_t ldv, int k, int64_t n, double* hc, double* partial, unsigned* bar,
                          const int* skip, cudaStream_t st, const GmresDev* G = nullptr,
                          GmresStatus* status = nullptr);
bool mgs_fuses_givens(int m);
int mgs_partial_doubles(int m);
void launch_backsolve(const GmresDev& G, int k, cudaStream_t st);
void launch_sub(const double* b, const double* ax, double* r, int64_t n, cudaStream_t st);
void launch_combine(const double* v, int64_t ldv, const double* y, int k, double* out, int64_t n, cudaStream_t st);
void launch_add(double* x, const double* dx, int64_t n, cudaStream_t st);
int reduce_grid(int64_t n);

extern thread_local int64_t g_launches;


// cudaFuncSetAttribute(MaxDynamicSharedMemorySize = bytes [, carveout 100 %]) once per (device, kernel)
// and size (launch_cfg.cpp; thread-safe, per device).
void ensure_smem(const void* fn, size_t bytes, bool carveout = false);
template <typename K>
inline void ensure_smem(K* kernel, size_t bytes, bool carveout = false) {
  ensure_smem(reinterpret_cast<const void*>(kernel), bytes, carveout);
}


} // namespace tpdg_gpu
