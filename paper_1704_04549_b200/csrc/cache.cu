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
