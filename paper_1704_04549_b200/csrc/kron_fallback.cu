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
#include <cstdlib>

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

// Panel-blocked variant (default): the same per-row operation order as fb_apply_kernel, with two
// block barriers per 32-column panel instead of one per column. Forward, panel [c0, c0 + 32):
// (1) the panel's 32 rows go to warp 0, which solves the unit-lower 32 x 32 triangle with shuffles
// (row r subtracts L(r, c) x_c for c ascending) and publishes x; (2) every thread subtracts the
// panel's 32 columns from its rows below the panel (c ascending, coalesced column loads, eight
// columns in flight). Backward mirrors it with panels from the bottom, columns descending,
// divisions by the diagonal in the triangle. Per-element latency drops ~16x, so the kernel is
// bound by the n^2 stream of the factor.
constexpr int kPanel = 32;

template <int R>
__global__ void __launch_bounds__(kFbThreads, R <= 4 ? 3 : 1) fb_panel_kernel(DevPC pc, const double* __restrict__ in,
                                                               double* __restrict__ out) {
  if (pc.skip && *pc.skip) return;
  extern __shared__ double sx[];  // x (n) | panel rows (kPanel)
  double* sp = sx + pc.blk_len;
  const int slot = blockIdx.x, blk = pc.fb_list[slot];
  const int n = pc.blk_len, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const double* lu = pc.fb_lu + size_t(slot) * n * n;
  const int* perm = pc.fb_piv + size_t(slot) * n;
  const double* b = in + size_t(blk) * n;
  double s[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = t + kFbThreads * r;
    s[r] = i < n ? b[perm[i]] : 0.0;
  }
  const int np = (n + kPanel - 1) / kPanel;
  // ---- forward (unit lower), panels ascending
  for (int pp = 0; pp < np; ++pp) {
    const int c0 = pp * kPanel, cw = n - c0 < kPanel ? n - c0 : kPanel;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = t + kFbThreads * r;
      if (i >= c0 && i < c0 + cw) sp[i - c0] = s[r];
    }
    __syncthreads();
    if (warp == 0) {
      const double* col = lu + size_t(c0) * n + c0 + lane;  // L(c0 + lane, c0 + c) at col[c n]
      double tl[kPanel];
#pragma unroll
      for (int c = 0; c < kPanel; ++c) tl[c] = (lane > c && lane < cw) ? col[size_t(c) * n] : 0.0;
      double v = lane < cw ? sp[lane] : 0.0;
#pragma unroll
      for (int c = 0; c < kPanel; ++c) {
        const double xc = __shfl_sync(0xffffffffu, v, c);
        if (lane > c && lane < cw) v = fmsc(v, tl[c], xc);
      }
      if (lane < cw) sx[c0 + lane] = v;
    }
    __syncthreads();
    // rows below the panel: s_i -= L(i, c0 + c) x_{c0 + c}, c ascending
    for (int cb = 0; cb < cw; cb += 8) {
      double lv[8][R];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = t + kFbThreads * r, c = cb + u;
          lv[u][r] = (c < cw && i >= c0 + cw && i < n) ? __ldcs(lu + size_t(c0 + c) * n + i) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = cb + u;
        if (c < cw) {
          const double xc = sx[c0 + c];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int i = t + kFbThreads * r;
            if (i >= c0 + cw && i < n) s[r] = fmsc(s[r], lv[u][r], xc);
          }
        }
      }
    }
  }
  // the forward solution is in sx; rows keep it in s as the backward right-hand side
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = t + kFbThreads * r;
    if (i < n) s[r] = sx[i];
  }
  __syncthreads();
  // ---- backward (upper, with the diagonal), panels descending, columns descending
  for (int pp = np - 1; pp >= 0; --pp) {
    const int c0 = pp * kPanel, cw = n - c0 < kPanel ? n - c0 : kPanel;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = t + kFbThreads * r;
      if (i >= c0 && i < c0 + cw) sp[i - c0] = s[r];
    }
    __syncthreads();
    if (warp == 0) {
      const double* col = lu + size_t(c0) * n + c0 + lane;  // U(c0 + lane, c0 + c) at col[c n]
      double tu[kPanel];
#pragma unroll
      for (int c = 0; c < kPanel; ++c) tu[c] = (lane < c && c < cw) ? col[size_t(c) * n] : 0.0;
      const double d = lane < cw ? lu[size_t(c0 + lane) * n + c0 + lane] : 1.0;
      const double rdv = __drcp_rn(d);
      double v = lane < cw ? sp[lane] : 0.0;
#pragma unroll
      for (int c = kPanel - 1; c >= 0; --c) {
        if (c < cw) {
          if (lane == c) v = fdiv_rcp(v, d, rdv);
          const double xc = __shfl_sync(0xffffffffu, v, c);
          if (lane < c) v = fmsc(v, tu[c], xc);
        }
      }
      if (lane < cw) sx[c0 + lane] = v;
    }
    __syncthreads();
    // rows above the panel: s_i -= U(i, c0 + c) x_{c0 + c}, c descending
    for (int cb = cw - 1; cb >= 0; cb -= 8) {
      double lv[8][R];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = t + kFbThreads * r, c = cb - u;
          lv[u][r] = (c >= 0 && i < c0) ? __ldcs(lu + size_t(c0 + c) * n + i) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = cb - u;
        if (c >= 0) {
          const double xc = sx[c0 + c];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int i = t + kFbThreads * r;
            if (i < c0) s[r] = fmsc(s[r], lv[u][r], xc);
          }
        }
      }
    }
  }
  __syncthreads();
  double* o = out + size_t(blk) * n;
  for (int i = t; i < n; i += kFbThreads) o[i] = sx[i];
}

template <int R>
bool try_fb_panel(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  if (pc.blk_len > R * kFbThreads) return false;
  const size_t smem = sizeof(double) * size_t(pc.blk_len + kPanel);
  ensure_smem(fb_panel_kernel<R>, smem);
  fb_panel_kernel<R><<<pc.n_fb, kFbThreads, smem, st>>>(pc, in, out);
  return true;
}

template <int R>
bool try_fb(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  if (pc.blk_len > R * kFbThreads) return false;
  constexpr int D = R <= 2 ? 16 : 8;
  const size_t smem = sizeof(double) * size_t(pc.blk_len);
  ensure_smem(fb_apply_kernel<R, D>, smem);
  fb_apply_kernel<R, D><<<pc.n_fb, kFbThreads, smem, st>>>(pc, in, out);
  return true;
}

} // namespace

bool launch_fallback_apply(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  if (pc.n_fb == 0) return true;
  // panels pay off for large blocks (cfg2 p = 30, n = 961: 1.44 -> 0.91 ms); at n = 441 (p = 20) the
  // per-column kernel's deeper prefetch ring is faster (209 vs 232 us)
  if (pc.blk_len > 2 * kFbThreads)
    return try_fb_panel<4>(pc, in, out, st) || try_fb_panel<8>(pc, in, out, st);
  return try_fb<1>(pc, in, out, st) || try_fb<2>(pc, in, out, st) || try_fb<4>(pc, in, out, st) ||
         try_fb<8>(pc, in, out, st);
}

} // namespace tpdg_gpu
