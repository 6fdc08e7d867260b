// GMRES vector kernels (HBM-bound streaming passes) for the device-resident restarted GMRES
// (reference solve/gmres.hpp:52-179).
//
// Reductions are deterministic: each CTA reduces a fixed grid-stride slice (per-thread
// sequential, then warp-shuffle + shared tree), writes one partial, and the last CTA to finish
// (atomic ticket) sums the partials in CTA order. The reference sums left to right over all N
// entries; the tree order differs by O(sqrt(N) eps) relative, which is why the parity gate for
// GMRES is the iteration count.
//
// MGS is fused: pass j computes w <- w - h_{j-1} v_{j-1} and the partial dot <v_j, w> in one read
// of (w, v_{j-1}, v_j) and one write of w, so the k+1 MGS steps of iteration k cost k+2 passes.
#include "tpdg_internal.hpp"

namespace tpdg_gpu {

thread_local int64_t g_launches = 0;

namespace {

constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < int(blockDim.x >> 5); ++w) s += sh[w];
  __syncthreads();
  return s;  // valid in thread 0
}

// Last-CTA finalization: result[0] = sum of partials in CTA order (optionally sqrt).
__device__ __forceinline__ void finalize(double local, double* partial, double* result, unsigned* counter,
                                         bool take_sqrt) {
  __shared__ double sh[32];
  __shared__ bool last;
  const double s = block_sum(local, sh);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = s;
    __threadfence();
    const unsigned t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double tot = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) tot += ((volatile double*)partial)[b];
    result[0] = take_sqrt ? sqrt(tot) : tot;
    *counter = 0u;  // re-arm for the next launch (stream ordered)
  }
}

__global__ void __launch_bounds__(kRedThreads) dot_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                           int64_t n, double* partial, double* result,
                                                           unsigned* counter, int take_sqrt) {
  double s = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    s += x[i] * y[i];
  finalize(s, partial, result, counter, take_sqrt != 0);
}

// w <- w - hprev[0] * vprev (if vprev), then partial <vj, w>.
__global__ void __launch_bounds__(kRedThreads) mgs_kernel(double* __restrict__ w, const double* __restrict__ vprev,
                                                           const double* __restrict__ hprev,
                                                           const double* __restrict__ vj, int64_t n, double* partial,
                                                           double* result, unsigned* counter, int take_sqrt) {
  const double h = vprev ? hprev[0] : 0.0;
  double s = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double wi = w[i];
    if (vprev) {
      wi = wi - h * vprev[i];
      w[i] = wi;
    }
    s += (vj ? vj[i] : wi) * wi;
  }
  finalize(s, partial, result, counter, take_sqrt != 0);
}

__global__ void axpy_neg_kernel(double* __restrict__ w, const double* __restrict__ h, const double* __restrict__ v,
                                int64_t n) {
  const double hv = h[0];
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    w[i] = w[i] - hv * v[i];
}

// out = in / den[0] when den[0] > 0 (reference: `if (hkk > 0) v /= hkk`), else out = in.
__global__ void scale_div_kernel(const double* __restrict__ in, const double* __restrict__ den,
                                 double* __restrict__ out, int64_t n) {
  const double d = den[0];
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = d > 0.0 ? in[i] / d : in[i];
}

__global__ void sub_kernel(const double* __restrict__ b, const double* __restrict__ ax, double* __restrict__ r,
                           int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    r[i] = b[i] - ax[i];
}

// out[i] = sum_j y_j v_j[i], j ascending (reference: tmp[i] += y[j] * v[j][i]).
__global__ void combine_kernel(const double* __restrict__ v, int64_t ldv, const double* __restrict__ y, int k,
                               double* __restrict__ out, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < k; ++j) s += y[j] * v[j * ldv + i];
    out[i] = s;
  }
}

__global__ void add_kernel(double* __restrict__ x, const double* __restrict__ dx, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    x[i] = x[i] + dx[i];
}

int stream_grid(int64_t n) {
  const int64_t want = (n + 255) / 256;
  const int64_t cap = 148 * 8;
  return int(want < cap ? (want > 0 ? want : 1) : cap);
}

} // namespace

int reduce_grid(int64_t n) {
  const int64_t want = (n + kRedThreads * 4 - 1) / (kRedThreads * 4);
  const int64_t cap = 148 * 4;
  return int(want < cap ? (want > 0 ? want : 1) : cap);
}

void launch_dot(const double* x, const double* y, int64_t n, double* partial, double* result, unsigned* counter,
                cudaStream_t st) {
  dot_kernel<<<reduce_grid(n), kRedThreads, 0, st>>>(x, y, n, partial, result, counter, 0);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

void launch_norm(const double* x, int64_t n, double* partial, double* result, unsigned* counter, cudaStream_t st) {
  dot_kernel<<<reduce_grid(n), kRedThreads, 0, st>>>(x, x, n, partial, result, counter, 1);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

void launch_mgs_step(double* w, const double* vprev, const double* hprev, const double* vj, int64_t n,
                     double* partial, double* result, unsigned* counter, cudaStream_t st) {
  mgs_kernel<<<reduce_grid(n), kRedThreads, 0, st>>>(w, vprev, hprev, vj, n, partial, result, counter,
                                                      vj == nullptr ? 1 : 0);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

void launch_axpy_neg(double* w, const double* h, const double* v, int64_t n, cudaStream_t st) {
  axpy_neg_kernel<<<stream_grid(n), 256, 0, st>>>(w, h, v, n);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

void launch_scale_div(const double* in, const double* den, double* out, int64_t n, cudaStream_t st) {
  scale_div_kernel<<<stream_grid(n), 256, 0, st>>>(in, den, out, n);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

void launch_sub(const double* b, const double* ax, double* r, int64_t n, cudaStream_t st) {
  sub_kernel<<<stream_grid(n), 256, 0, st>>>(b, ax, r, n);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

void launch_combine(const double* v, int64_t ldv, const double* y, int k, double* out, int64_t n, cudaStream_t st) {
  combine_kernel<<<stream_grid(n), 256, 0, st>>>(v, ldv, y, k, out, n);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

void launch_add(double* x, const double* dx, int64_t n, cudaStream_t st) {
  add_kernel<<<stream_grid(n), 256, 0, st>>>(x, dx, n);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

} // namespace tpdg_gpu
