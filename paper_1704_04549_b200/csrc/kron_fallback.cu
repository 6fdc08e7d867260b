// Dense block-LU fallback of the KSVD preconditioner: x = A_e^{-1} b for the blocks whose Kronecker
// factors were rejected (form_ksvd_2d / _3d fallback, reference precond/ksvd.hpp:292-300 and
// :359-366; LuFactor::solve_inplace, tensor/small_matrix.hpp:177-192).
//
// One 256-thread CTA per fallback block, thread t owning rows t + 256 r (r < R). The LU factor is
// stored column-major (lu[j n + i] = LU(i, j)), so every step of both sweeps reads one coalesced
// column; the columns are streamed through a register ring D steps ahead of their use, which
// keeps the HBM stream (n^2 doubles per block and apply: the fallback blocks dominate the bytes at
// p = 20 / 30) independent of the per-step latency.
//   forward  (unit lower, reference order): step j publishes x_j (its row has received every
//            term j' < j), then each row i > j subtracts L(i, j) x_j -- row i sees j ascending,
//            with separate mul / sub roundings, exactly as the reference;
//   backward (column-descending): step j forms x_j = s_j / U(j, j) (correctly rounded division
//            via the precomputed reciprocal) and rows i < j subtract U(i, j) x_j. The per-row order
//            is reversed with respect to the reference (well-conditioned dense block:
//            tests/test_gpu_full_pc_parity.py measures ~1e-15).
#include <cstdint>

#include "faithful.cuh"
#include "tpdg_internal.hpp"

namespace tpdg_gpu {

namespace {

constexpr int kFbThreads = 256;

template <int R>
__device__ __forceinline__ void fetch_col(const double* __restrict__ lu, int n, int j, int t, bool lower,
                                          double (&dst)[R]) {
  // rows of column j that the sweep uses: i > j (forward, unit lower) or i <= j (backward, upper)
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = t + kFbThreads * r;
    const bool use = j >= 0 && j < n && i < n && (lower ? i > j : i <= j);
    dst[r] = use ? __ldcs(lu + size_t(j) * n + i) : 0.0;
  }
}

template <int R, int D>
__global__ void __launch_bounds__(kFbThreads) fb_apply_kernel(DevPC pc, const double* __restrict__ in,
                                                               double* __restrict__ out) {
  if (pc.skip && *pc.skip) return;
  extern __shared__ double sx[];
  const int slot = blockIdx.x, blk = pc.fb_list[slot];
  const int n = pc.blk_len, t = threadIdx.x;
  const double* lu = pc.fb_lu + size_t(slot) * n * n;
  const int* perm = pc.fb_piv + size_t(slot) * n;
  const double* b = in + size_t(blk) * n;
  double s[R], rd[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = t + kFbThreads * r;
    s[r] = i < n ? b[perm[i]] : 0.0;
    rd[r] = i < n ? __drcp_rn(lu[size_t(i) * n + i]) : 1.0;
  }
  const int nr = (n + D - 1) / D * D;
  double ring[D][R];
  // forward sweep, j ascending
#pragma unroll
  for (int d = 0; d < D; ++d) fetch_col<R>(lu, n, d, t, true, ring[d]);
  for (int j0 = 0; j0 < nr; j0 += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int j = j0 + d;
      const int own = j & (kFbThreads - 1), orow = j / kFbThreads;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (t == own && r == orow && j < n) sx[j] = s[r];
      __syncthreads();
      const double xj = j < n ? sx[j] : 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (t + kFbThreads * r > j && j < n) s[r] = fmsc(s[r], ring[d][r], xj);
      fetch_col<R>(lu, n, j + D, t, true, ring[d]);
    }
  }
  // backward sweep, j descending (rows padded up to nr: j = nr - 1 - jj)
#pragma unroll
  for (int d = 0; d < D; ++d) fetch_col<R>(lu, n, nr - 1 - d, t, false, ring[d]);
  __syncthreads();
  for (int jj0 = 0; jj0 < nr; jj0 += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int j = nr - 1 - (jj0 + d);
      const int own = j & (kFbThreads - 1), orow = j / kFbThreads;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (t == own && r == orow && j < n) {
          s[r] = fdiv_rcp(s[r], ring[d][r], rd[r]);
          sx[j] = s[r];
        }
      __syncthreads();
      const double xj = j < n ? sx[j] : 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (t + kFbThreads * r < j && j < n) s[r] = fmsc(s[r], ring[d][r], xj);
      fetch_col<R>(lu, n, j - D, t, false, ring[d]);
    }
  }
  __syncthreads();
  double* o = out + size_t(blk) * n;
  for (int i = t; i < n; i += kFbThreads) o[i] = sx[i];
}

template <int R>
bool try_fb(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  if (pc.blk_len > R * kFbThreads) return false;
  constexpr int D = R <= 2 ? 16 : 8;
  const size_t smem = sizeof(double) * size_t(pc.blk_len);
  static size_t configured = 0;
  if (smem > configured) {
    TPDG_CUDA_CHECK(cudaFuncSetAttribute(fb_apply_kernel<R, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    configured = smem;
  }
  fb_apply_kernel<R, D><<<pc.n_fb, kFbThreads, smem, st>>>(pc, in, out);
  return true;
}

} // namespace

bool launch_fallback_apply(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  if (pc.n_fb == 0) return true;
  return try_fb<1>(pc, in, out, st) || try_fb<2>(pc, in, out, st) || try_fb<4>(pc, in, out, st) ||
         try_fb<8>(pc, in, out, st);
}

} // namespace tpdg_gpu
