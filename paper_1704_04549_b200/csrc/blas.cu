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
#include <map>
#include <mutex>
#include <type_traits>
#include <algorithm>
#include <cstdint>

#include <cooperative_groups.h>

#include <cstdlib>

#include "tma.cuh"
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

// Last-CTA finalization: result[0] = fixed-order tree sum of the per-CTA partials (optionally sqrt).
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
  if (!last) return;
  __threadfence();
  double v = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) v += ((volatile double*)partial)[b];
  const double tot = block_sum(v, sh);
  if (threadIdx.x == 0) {
    result[0] = take_sqrt ? sqrt(tot) : tot;
    *counter = 0u;  // re-arm for the next launch (stream ordered)
  }
}

__device__ __forceinline__ bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Grid-stride over double2 pairs when every operand is 16 B aligned (an odd n is finished by the
// scalar tail in the first CTA); otherwise a scalar grid-stride loop.
__global__ void __launch_bounds__(kRedThreads) dot_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                           int64_t n, double* partial, double* result,
                                                           unsigned* counter, int take_sqrt) {
  double s0 = 0.0, s1 = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x, t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (aligned16(x) && aligned16(y)) {
    const int64_t n2 = n / 2;
    const double2* x2 = reinterpret_cast<const double2*>(x);
    const double2* y2 = reinterpret_cast<const double2*>(y);
    for (int64_t i = t0; i < n2; i += stride) {
      const double2 a = x2[i], b = y2[i];
      s0 += a.x * b.x;
      s1 += a.y * b.y;
    }
    if ((n & 1) && t0 == 0) s0 += x[n - 1] * y[n - 1];
  } else {
    for (int64_t i = t0; i < n; i += stride) s0 += x[i] * y[i];
  }
  finalize(s0 + s1, partial, result, counter, take_sqrt != 0);
}

// w <- w - hprev[0] * vprev (if vprev), then partial <vj, w> (or <w, w> when vj is null).
__global__ void __launch_bounds__(kRedThreads) mgs_kernel(double* __restrict__ w, const double* __restrict__ vprev,
                                                           const double* __restrict__ hprev,
                                                           const double* __restrict__ vj, int64_t n, double* partial,
                                                           double* result, unsigned* counter, int take_sqrt,
                                                           const int* skip) {
  if (skip && *skip) return;
  const double h = vprev ? hprev[0] : 0.0;
  double s0 = 0.0, s1 = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x, t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (aligned16(w) && (!vprev || aligned16(vprev)) && (!vj || aligned16(vj))) {
    const int64_t n2 = n / 2;
    double2* w2 = reinterpret_cast<double2*>(w);
    const double2* p2 = reinterpret_cast<const double2*>(vprev);
    const double2* j2 = reinterpret_cast<const double2*>(vj);
    for (int64_t i = t0; i < n2; i += stride) {
      double2 wi = w2[i];
      if (vprev) {
        const double2 pv = p2[i];
        wi.x = wi.x - h * pv.x;
        wi.y = wi.y - h * pv.y;
        w2[i] = wi;
      }
      const double2 a = vj ? j2[i] : wi;
      s0 += a.x * wi.x;
      s1 += a.y * wi.y;
    }
    if ((n & 1) && t0 == 0) {
      double wi = w[n - 1];
      if (vprev) {
        wi = wi - h * vprev[n - 1];
        w[n - 1] = wi;
      }
      s0 += (vj ? vj[n - 1] : wi) * wi;
    }
  } else {
    for (int64_t i = t0; i < n; i += stride) {
      double wi = w[i];
      if (vprev) {
        wi = wi - h * vprev[i];
        w[i] = wi;
      }
      s0 += (vj ? vj[i] : wi) * wi;
    }
  }
  finalize(s0 + s1, partial, result, counter, take_sqrt != 0);
}

__global__ void axpy_neg_kernel(double* __restrict__ w, const double* __restrict__ h, const double* __restrict__ v,
                                int64_t n) {
  const double hv = h[0];
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    w[i] = w[i] - hv * v[i];
}

// out = in / den[0] when den[0] > 0 (reference: `if (hkk > 0) v /= hkk`), else out = in.
__global__ void scale_div_kernel(const double* __restrict__ in, const double* __restrict__ den,
                                 double* __restrict__ out, int64_t n, const int* skip) {
  if (skip && *skip) return;
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
  __shared__ double ys[64];
  for (int j = threadIdx.x; j < k && j < 64; j += blockDim.x) ys[j] = y[j];
  __syncthreads();
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    // same j-ascending chain; unrolled so that the basis loads are in flight together
#pragma unroll 8
    for (int j = 0; j < k; ++j) s += (j < 64 ? ys[j] : y[j]) * v[j * ldv + i];
    out[i] = s;
  }
}

__global__ void add_kernel(double* __restrict__ x, const double* __restrict__ dx, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    x[i] = x[i] + dx[i];
}

// Givens step of iteration k (solve/gmres.hpp:122-141), one thread. hc holds the raw Hessenberg
// column h(0..k+1, k) from MGS; the rotated column goes to H(:, k). Writes |g_{k+1}| and the
// convergence decision to the host-mapped status slot and raises `done` on convergence.
__device__ __forceinline__ void givens_warp(const GmresDev& G, int k, GmresStatus* status, double* gsm) {
  // one warp stages the column and the previous rotations in shared memory (independent loads,
  // one round trip), then lane 0 runs the dependent rotation chain on-chip; gsm: col[m + 2] | cs[m + 1] | sn[m + 1]
  const int m = G.m;
  double* col = gsm;
  double* cs = col + m + 2;
  double* sn = cs + m + 1;
  // every operand is loaded in one round trip (done flag, g_k, the column, the old rotations)
  const int done = *G.done;
  const double gk = G.g[k];
  for (int j = threadIdx.x; j <= k + 1; j += 32) col[j] = G.hc[j];
  for (int j = threadIdx.x; j < k; j += 32) {
    cs[j] = G.cs[j];
    sn[j] = G.sn[j];
  }
  if (done) return;
  __syncwarp();
  if (threadIdx.x == 0) {
    for (int j = 0; j < k; ++j) {
      const double t1 = col[j], t2 = col[j + 1];
      col[j] = cs[j] * t1 + sn[j] * t2;
      col[j + 1] = -sn[j] * t1 + cs[j] * t2;
    }
    const double t1 = col[k], t2 = col[k + 1];
    const double denom = hypot(t1, t2);
    const double c = denom == 0.0 ? 1.0 : t1 / denom, sv = denom == 0.0 ? 0.0 : t2 / denom;
    const double res = fabs(sv * gk);
    const int conv = res <= G.target ? 1 : 0;
    status[k].res = res;
    status[k].conv = conv;
    __threadfence_system();  // payload before the valid flag (the host polls `valid`)
    status[k].valid = 1;
    if (conv) *G.done = 1;
    G.cs[k] = c;
    G.sn[k] = sv;
    G.g[k] = c * gk;
    G.g[k + 1] = -sv * gk;
    col[k] = denom;
    col[k + 1] = 0.0;
  }
  __syncwarp();
  for (int j = threadIdx.x; j <= k + 1; j += 32) G.H[j * m + k] = col[j];
}

__global__ void givens_kernel(GmresDev G, int k, GmresStatus* status) {
  extern __shared__ double gsm[];
  givens_warp(G, k, status, gsm);
}

// The Givens step fused at the end of the cooperative MGS launch (single rank): block 0's first
// warp runs it once the iteration's column h(0..k+1, k) is complete (written by block 0 itself).
constexpr int kFusedGivensMaxM = 62;
__device__ __forceinline__ void fused_givens(const GmresDev& G, int k, GmresStatus* status) {
  __shared__ double gsm[3 * kFusedGivensMaxM + 4];
  if (status == nullptr || blockIdx.x != 0) return;
  __syncthreads();
  if (threadIdx.x < 32) givens_warp(G, k, status, gsm);
}

// y = H(0:k, 0:k)^{-1} g (back substitution, solve/gmres.hpp:145-150), one thread.
// Restarts whose H(0:k, 0:k) does not fit in shared memory (k > kBacksolveSmemMax) run the same
// sequence straight from global memory (G.y as the solution buffer).
constexpr int kBacksolveSmemMax = 160;  // 8 (k^2 + 2k + 1) B <= 227 KB
__global__ void backsolve_global_kernel(GmresDev G, int k) {
  if (threadIdx.x != 0) return;
  const int m = G.m;
  for (int i = k - 1; i >= 0; --i) {
    double s = G.g[i];
    for (int j = i + 1; j < k; ++j) s -= G.H[i * m + j] * G.y[j];
    G.y[i] = s / G.H[i * m + i];
  }
}

__global__ void backsolve_kernel(GmresDev G, int k) {
  // the warp stages H(0:k, 0:k) and g in shared memory (one round trip), then lane 0 runs the
  // sequential back substitution on-chip (same order as before)
  extern __shared__ double bs_sm[];  // H rows (k x k) | g (k) | y (k)
  const int m = G.m;
  double* Hs = bs_sm;
  double* gs = Hs + k * k;
  double* ys = gs + k;
  if (k <= 32) {  // all loads of a lane issued before any store (one memory round trip)
    double hv[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) hv[r] = (r < k && int(threadIdx.x) < k) ? G.H[r * m + threadIdx.x] : 0.0;
    const double gv = int(threadIdx.x) < k ? G.g[threadIdx.x] : 0.0;
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (r < k && int(threadIdx.x) < k) Hs[r * k + threadIdx.x] = hv[r];
    if (int(threadIdx.x) < k) gs[threadIdx.x] = gv;
  } else {
    for (int t = threadIdx.x; t < k * k; t += blockDim.x) Hs[t] = G.H[(t / k) * m + t % k];
    for (int t = threadIdx.x; t < k; t += blockDim.x) gs[t] = G.g[t];
  }
  __syncwarp();
  if (threadIdx.x == 0) {
    for (int i = k - 1; i >= 0; --i) {
      double s = gs[i];
      for (int j = i + 1; j < k; ++j) s -= Hs[i * k + j] * ys[j];
      ys[i] = s / Hs[i * k + i];
    }
  }
  __syncwarp();
  for (int t = threadIdx.x; t < k; t += blockDim.x) G.y[t] = ys[t];
}

// All MGS passes of Arnoldi iteration k in one cooperative persistent launch (single rank):
//   pass j <= k : w <- w - h_{j-1} v_{j-1} (j > 0), partial <v_j, w>
//   pass k+1    : w <- w - h_k v_k, partial <w, w>; then w /= ||w|| when > 0.
// Each CTA owns a fixed contiguous slice of w (updated only by it), so passes need no data
// exchange; between passes a grid-wide barrier publishes the per-CTA partials, and every CTA sums
// them in the same fixed order (deterministic, identical on all CTAs).
constexpr int kCoopThreads = 1024;

// L2 eviction-priority hints (createpolicy + .L2::cache_hint): in mgs_global_kernel the working vector w
// and the current basis vector are kept L2-resident across passes (evict_last), so a pass streams
// only v_j from HBM instead of w (read + write), v_{j-1} and v_j.
// thread-private cp.async ring of the streaming MGS kernel (dst: shared-space byte address)
__device__ __forceinline__ void cp_async16(uint32_t dst, const double* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16z(uint32_t dst, const double* gmem, unsigned src_bytes) {  // rest zero-filled
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ double2 lds128(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld2_hint(const double* a, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st2_hint(double* a, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(a), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}

// Grid reduction of one MGS pass: CTA partial (warp trees, then the 32 warp sums in order), the
// grid barrier, and every thread summing the per-CTA partials in the same fixed order.
// The barrier is a monotonic arrival counter bar[0]: pass p of a launch is complete when it reaches
// base + (p + 1) nb, base = bar[1], which the launch reads at its start and CTA 0 advances at its
// end (mgs_epoch_*). One atomic and one acquire poll per pass; no re-arming store, no generation
// flag (2.1 vs 3.0 us per empty grid sum, tools/gridsum_bench.cu). Returns the total.
// The running target lives in shared memory (thread 0 only uses it), so the kernels carry no extra
// register for it.
__device__ __forceinline__ void mgs_epoch_begin(const unsigned* bar, unsigned* target) {
  if (threadIdx.x == 0) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(*target) : "l"(bar + 1) : "memory");
}
__device__ __forceinline__ void mgs_epoch_end(unsigned* bar, const unsigned* target) {
  // every CTA read bar[1] before its first arrival, and CTA 0 gets here only after all arrivals
  if (blockIdx.x == 0 && threadIdx.x == 0) bar[1] = *target;
}
__device__ __forceinline__ double mgs_grid_sum(double v, double* part, unsigned* bar, unsigned* target, double* shA,
                                               double* shB) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned nb = gridDim.x;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) shA[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double bs = 0.0;
    for (int w2 = 0; w2 < int(blockDim.x >> 5); ++w2) bs += shA[w2];
    part[blockIdx.x] = bs;
    const unsigned tg = *target + nb;
    *target = tg;
    unsigned t;  // the release arrival publishes this CTA's partial; waiters acquire the count
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(bar) : "memory");
    if (t + 1u != tg) {
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
      } while (int(cur - tg) < 0);
    }
  }
  __syncthreads();
  double pv = threadIdx.x < nb ? reinterpret_cast<volatile double*>(part)[threadIdx.x] : 0.0;
  for (unsigned b = threadIdx.x + blockDim.x; b < nb; b += blockDim.x) pv += reinterpret_cast<volatile double*>(part)[b];
  // only the warps holding partials reduce; warp 0 then sums the warp sums in order and
  // broadcasts (the ordered 32-term sum in every thread cost more issue slots than a barrier)
  const int nw = int((nb + 31) / 32);
  if (wid < nw) {
    for (int o = 16; o > 0; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
    if (lane == 0) shB[wid] = pv;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w2 = 0; w2 < nw; ++w2) tot += shB[w2];
    shB[32] = tot;
  }
  __syncthreads();
  return shB[32];
}

// General fallback (slices too large to keep w on chip): w in global memory / L2.
__global__ void __launch_bounds__(kCoopThreads) mgs_global_kernel(double* __restrict__ V, int64_t ldv, int k,
                                                                 int64_t n, int64_t chunk, double* __restrict__ hc,
                                                                 double* __restrict__ partial, unsigned* bar,
                                                                 const int* skip, GmresDev G, GmresStatus* gstatus) {
  if (skip && *skip) return;
  __shared__ unsigned tgt;
  mgs_epoch_begin(bar, &tgt);
  __shared__ double shA[32], shB[33];
  const unsigned nb = gridDim.x;
  const int64_t lo = int64_t(blockIdx.x) * chunk;
  const int64_t hi = lo + chunk < n ? lo + chunk : n;
  const int64_t len = hi > lo ? hi - lo : 0;
  double* wg = V + int64_t(k + 1) * ldv + lo;
  double* w = wg;
  double h = 0.0;
  const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
  for (int j = 0; j <= k + 1; ++j) {
    const double* vp = j > 0 ? V + int64_t(j - 1) * ldv + lo : nullptr;
    const double* vj = j <= k ? V + int64_t(j) * ldv + lo : nullptr;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll 4
    for (int64_t i = 2 * threadIdx.x; i < len; i += 2 * blockDim.x) {
      if (i + 1 < len) {
        double2 wi = ld2_hint(w + i, keep);
        if (vp) {
          const double2 pv = ld2_hint(vp + i, drop);
          wi.x = wi.x - h * pv.x;
          wi.y = wi.y - h * pv.y;
          st2_hint(w + i, wi, keep);
        }
        double2 a = wi;
        if (vj) a = ld2_hint(vj + i, keep);
        s0 += a.x * wi.x;
        s1 += a.y * wi.y;
      } else {
        double wi = w[i];
        if (vp) {
          wi = wi - h * vp[i];
          w[i] = wi;
        }
        double a = wi;
        if (vj) a = vj[i];
        s0 += a * wi;
      }
    }
    // prefetch the next basis vector's slice into L2 while the grid waits at the barrier
    if (j + 1 <= k)
      for (int64_t i = 16 * int64_t(threadIdx.x); i < len; i += 16 * int64_t(blockDim.x))
        asm volatile("prefetch.global.L2 [%0];" ::"l"(V + int64_t(j + 1) * ldv + lo + i));
    const double tot = mgs_grid_sum(s0 + s1, partial + size_t(j) * nb, bar, &tgt, shA, shB);
    h = j <= k ? tot : sqrt(tot);
    if (blockIdx.x == 0 && threadIdx.x == 0) hc[j] = h;
  }
  // reference: if (hkk > 0) v[k+1] /= hkk
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) wg[i] = h > 0.0 ? w[i] / h : w[i];
  mgs_epoch_end(bar, &tgt);
  fused_givens(G, k, gstatus);
}

// ---- streaming MGS: every slice that fits on chip (all BASELINE configs) ----------------------
// Element assignment: thread t of 512 owns the pairs t + 512 u, u < PPT, of every 2048-double row of
// its CTA's slice; accumulation order: rows ascending, even/odd elements in s0/s1, then warp
// butterflies, the warp sums and the CTA partials in index order (tools/mgs_bench.cu checks the first
// dot against a host emulation of this order bit for bit). How a basis row reaches its thread:
//  * v_j comes from HBM once, through a thread-private cp.async ring: every thread copies the 16-byte
//    pieces it will consume itself (a warp's pieces are 512 contiguous bytes), D rows ahead, and waits
//    on its own cp.async groups only -- no mbarrier, no producer, no block-level handshake per row
//    (tools/tma_ring_bench.cu: a cp.async.bulk ring with full/empty mbarriers costs 700-900 cycles per
//    row whatever the row size or depth, 11.7 us per cfg4 pass; tools/cpasync_ring_bench.cu: this ring
//    streams the same pass in 6.0 us, HBM speed);
//  * v_{j-1}, needed for the update w -= h_{j-1} v_{j-1} one pass later, does not come back through L2:
//    after using its pairs of v_j for the dot, the thread parks them in tensor memory (rows r < TMR:
//    8 columns per row, the four warps of a TMEM lane quarter take 128 columns each; tcgen05.st, read
//    back with tcgen05.ld one pass later). 256 KB of TMEM hold 16 rows per SM; rows >= TMR (two at
//    cfg4) are parked in shared memory instead. Every basis vector is read exactly once per pass.
// w lives on chip for the whole launch: rows r < RW in registers, the rest in shared memory.
template <int NT, int RW, int D, int PPT, int TMR>
__global__ void __launch_bounds__(NT, 1) mgs_stream_kernel(double* __restrict__ V, int64_t ldv, int k, int64_t n,
                                                           int64_t chunk, double* __restrict__ hc,
                                                           double* __restrict__ partial, unsigned* bar, const int* skip,
                                                           GmresDev G, GmresStatus* gstatus) {
  if (skip && *skip) return;
  static_assert(PPT == 2 && RW <= TMR && TMR * 8 * (NT / 128) <= 512 && (D & (D - 1)) == 0, "TMEM rows / ring depth");
  __shared__ unsigned tgt;
  mgs_epoch_begin(bar, &tgt);
  constexpr int ROW = 2 * NT * PPT;      // doubles per row
  constexpr unsigned ROWB = 8u * ROW;    // bytes per row
  constexpr unsigned P1 = 16u * NT;      // byte offset of a thread's second pair in a row
  extern __shared__ __align__(128) double bsm[];
  __shared__ double shA[32], shB[33];
  __shared__ uint32_t tm_slot;
  const unsigned nb = gridDim.x;
  const int64_t lo = int64_t(blockIdx.x) * chunk;
  const int64_t hi = lo + chunk < n ? lo + chunk : n;
  const int len = int(hi > lo ? hi - lo : 0);
  const int nrows = (len + ROW - 1) / ROW, nfull = len / ROW;  // rows, rows with every pair inside len
  // shared memory: ring of D rows (v_j of task q in slot q % D) | parked rows r >= TMR of v_{j-1} | w rows r >= RW
  double* wsm = bsm + (D + (nrows > TMR ? nrows - TMR : 0)) * ROW;
  double* wg = V + int64_t(k + 1) * ldv + lo;
  const int t = threadIdx.x;
  if (t < 32) tmem_alloc512(&tm_slot);
  tmem_fence_before_sync();
  // every shared-memory access below is to the thread's own pairs, through 32-bit shared-space addresses
  const uint32_t ring_s = smem_u32(bsm) + 16u * unsigned(t);
  const uint32_t park_s = ring_s + D * ROWB - TMR * ROWB;  // row r >= TMR parked at park_s + ROWB r
  const uint32_t w_s = smem_u32(wsm) + 16u * unsigned(t) - RW * ROWB;  // w row r >= RW at w_s + ROWB r
  // The copies of v-task q = (pass j <= k, row r), j-major, by their consumer, D - 1 tasks ahead; one cp.async group
  // per task. Pieces past len are zero-filled (src-size 8 / 0) and w is zero there too, so the row arithmetic needs
  // no bounds: the padding adds +0.0 to the sums and stays zero under the update.
  auto piece_bytes = [&](int r, int u) {  // bytes of pair t + NT u of row r inside len
    const int left = len - (r * ROW + 2 * (t + NT * u));
    return unsigned(left >= 2 ? 16 : left > 0 ? 8 : 0);
  };
  const int nvtask = (k + 1) * nrows;
  const int64_t wrapinc = ldv - int64_t(nrows - 1) * ROW;
  const double* isrc = V + lo + 2 * t;  // this thread's first pair of the next task's row
  int iq = 0, ir = 0;
  unsigned islot = 0;
  auto issue_any = [&]() {  // any task: partial last row, pass wrap, past the last v-task (zero-fill, no read)
    const bool live = iq < nvtask, fullrow = ir < nfull, wrap = ir + 1 == nrows;
    const unsigned pb0 = piece_bytes(nfull, 0), pb1 = piece_bytes(nfull, 1);
    const unsigned z0 = live ? (fullrow ? 16u : pb0) : 0u, z1 = live ? (fullrow ? 16u : pb1) : 0u;
    cp_async16z(ring_s + islot, isrc, z0);
    cp_async16z(ring_s + islot + P1, isrc + 2 * NT, z1);
    cp_async_commit();
    islot = (islot + ROWB) & (D * ROWB - 1);
    ++iq;
    isrc += live ? (wrap ? wrapinc : int64_t(ROW)) : int64_t(0);
    ir = wrap ? 0 : ir + 1;
  };
  auto issue_mid = [&]() {  // a full row of a pass j <= k that is not the pass's last row
    cp_async16(ring_s + islot, isrc);
    cp_async16(ring_s + islot + P1, isrc + 2 * NT);
    cp_async_commit();
    islot = (islot + ROWB) & (D * ROWB - 1);
    ++iq;
    isrc += ROW;
    ++ir;
  };
  for (int q = 0; q < D - 1; ++q) issue_any();
  // w rows >= RW go straight to shared memory (the thread's own pairs, zero-filled past len) as one cp.async group
  // behind the ring's first rows: all of them in flight at once, complete by the third row of pass 0 (group order)
  for (int r = RW; r < nrows; ++r) {
#pragma unroll
    for (int u = 0; u < PPT; ++u)
      cp_async16z(w_s + ROWB * unsigned(r) + P1 * unsigned(u), wg + r * ROW + 2 * (t + NT * u), piece_bytes(r, u));
  }
  cp_async_commit();
  double2 wr[RW][PPT];
#pragma unroll
  for (int r = 0; r < RW; ++r)
#pragma unroll
    for (int u = 0; u < PPT; ++u) {
      const int i = 2 * (t + NT * u) + ROW * r;
      wr[r][u] = i + 1 < len ? *reinterpret_cast<const double2*>(wg + i) : make_double2(i < len ? wg[i] : 0.0, 0.0);
    }
  __syncthreads();
  tmem_fence_after_sync();
  const uint32_t tm = tm_slot + ((32u * unsigned((t >> 5) & 3)) << 16) + unsigned(t >> 7) * (512u / (NT / 128));
  double h = 0.0, s0 = 0.0, s1 = 0.0;
  unsigned cslot = 0;
  // KIND 0: first pass (dot with v_0); 1: update with v_{j-1}, dot with v_j; 2: last update and <w, w>
  auto row = [&](auto kind, auto mid, double2 (&wi)[PPT], int r) {
    constexpr int KIND = decltype(kind)::value;
    constexpr bool MID = decltype(mid)::value;  // the task issued here is a full, non-last row of this pass
    const bool tmrow = r < TMR;  // uniform over the CTA; folds for the register rows
    double2 pv[PPT];
    if (KIND > 0 && tmrow) {
      tmem_ld4(tm + 8u * unsigned(r), pv[0]);
      tmem_ld4(tm + 8u * unsigned(r) + 4u, pv[1]);
    }
    if (KIND < 2) {  // v-task + D - 1, into the slot this thread finished reading one row ago
      if (MID) issue_mid();
      else issue_any();
      cp_async_wait<D - 1>();
    }
    if (KIND > 0) {
      if (tmrow) {
        tmem_wait_ld(pv[0], pv[1]);
      } else {
        pv[0] = lds128(park_s + ROWB * unsigned(r));
        pv[1] = lds128(park_s + ROWB * unsigned(r) + P1);
      }
#pragma unroll
      for (int u = 0; u < PPT; ++u) {
        wi[u].x = fma(-h, pv[u].x, wi[u].x);
        wi[u].y = fma(-h, pv[u].y, wi[u].y);
      }
    }
    if (KIND < 2) {
      double2 vj[PPT];
      vj[0] = lds128(ring_s + cslot);
      vj[1] = lds128(ring_s + cslot + P1);
      cslot = (cslot + ROWB) & (D * ROWB - 1);
      if (tmrow) {
        tmem_st4(tm + 8u * unsigned(r), vj[0]);
        tmem_st4(tm + 8u * unsigned(r) + 4u, vj[1]);
      } else {
        sts128(park_s + ROWB * unsigned(r), vj[0]);
        sts128(park_s + ROWB * unsigned(r) + P1, vj[1]);
      }
#pragma unroll
      for (int u = 0; u < PPT; ++u) {
        s0 = fma(vj[u].x, wi[u].x, s0);
        s1 = fma(vj[u].y, wi[u].y, s1);
      }
    } else {
#pragma unroll
      for (int u = 0; u < PPT; ++u) {
        s0 = fma(wi[u].x, wi[u].x, s0);
        s1 = fma(wi[u].y, wi[u].y, s1);
      }
    }
  };
  // Row r issues the task of row r + D - 1: a full row inside the same pass as long as r + D - 1 < nrows - 1.
  const bool regs_mid = nrows - 1 > RW - 1 + D - 1;
  auto pass = [&](auto kind, int j) {
    constexpr int KIND = decltype(kind)::value;
    constexpr std::true_type yes{};
    constexpr std::false_type no{};
    s0 = s1 = 0.0;
    if (regs_mid) {
#pragma unroll
      for (int r = 0; r < RW; ++r) row(kind, yes, wr[r], r);
    } else {
#pragma unroll
      for (int r = 0; r < RW; ++r)
        if (r < nrows) row(kind, no, wr[r], r);
    }
    for (int r = RW; r < nrows; ++r) {
      double2 wi[PPT];
      wi[0] = lds128(w_s + ROWB * unsigned(r));
      wi[1] = lds128(w_s + ROWB * unsigned(r) + P1);
      if (r + D - 1 < nrows - 1) row(kind, yes, wi, r);
      else row(kind, no, wi, r);
      if (KIND > 0) {
        sts128(w_s + ROWB * unsigned(r), wi[0]);
        sts128(w_s + ROWB * unsigned(r) + P1, wi[1]);
      }
    }
    if (KIND < 2) tmem_wait_st();
    const double tot = mgs_grid_sum(s0 + s1, partial + size_t(j) * nb, bar, &tgt, shA, shB);
    h = KIND < 2 ? tot : sqrt(tot);
    if (blockIdx.x == 0 && t == 0) hc[j] = h;
  };
  pass(std::integral_constant<int, 0>{}, 0);
  for (int j = 1; j <= k; ++j) pass(std::integral_constant<int, 1>{}, j);
  pass(std::integral_constant<int, 2>{}, k + 1);
  cp_async_wait<0>();
  tmem_fence_before_sync();
  __syncthreads();
  if (t < 32) tmem_dealloc512(tm_slot);
#pragma unroll
  for (int r = 0; r < RW; ++r)
#pragma unroll
    for (int u = 0; u < PPT; ++u) {
      const int i = 2 * (t + NT * u) + ROW * r;
      if (i + 1 < len)
        *reinterpret_cast<double2*>(wg + i) = h > 0.0 ? make_double2(wr[r][u].x / h, wr[r][u].y / h) : wr[r][u];
      else if (i < len)
        wg[i] = h > 0.0 ? wr[r][u].x / h : wr[r][u].x;
    }
  for (int i = ROW * RW + 2 * t; i < len; i += 2 * NT) {  // the pairs this thread owns
    wg[i] = h > 0.0 ? wsm[i - ROW * RW] / h : wsm[i - ROW * RW];
    if (i + 1 < len) wg[i + 1] = h > 0.0 ? wsm[i + 1 - ROW * RW] / h : wsm[i + 1 - ROW * RW];
  }
  mgs_epoch_end(bar, &tgt);
  fused_givens(G, k, gstatus);
}

struct CoopPlan {
  int grid;
  int64_t chunk;
  size_t smem;
  int mode;  // 1..3: mgs_stream_kernel shapes (mgs_coop_plan); 0: mgs_global_kernel
  int threads = kCoopThreads;
};

// One CTA per SM (cheap barrier); the most on-chip residency that fits. Shapes of the streaming kernel: 512 threads
// x 2 pairs per 2048-double row, 16 rows of v_{j-1} in tensor memory, and by slice length (rows per CTA):
//   <= 4 rows  (cfg2 p <= 15): 4 register rows of w, ring depth 8 (the ring reaches two passes ahead);
//   <= 10 rows (cfg2 p = 20):  10 register rows, ring depth 8;
//   <= 18 rows (cfg2 p = 30, cfg4): 10 register rows + w rows in shared memory, ring depth 4.
// tools/mgs_bench.cu, us per launch at K = 25: n = 1048576: 63.0 (registers only, round-2 kernel) -> 54.8;
// 1806336: 104.1 (TMA ring) -> 73.4; 3936256: 190.1 -> 125; 5451776: 264.6 -> 160.
constexpr int kBulkThreads = 512, kBulkPPT = 2, kBulkTMR = 16;
constexpr int kBulkRow = 2 * kBulkThreads * kBulkPPT;

template <int RW, int D>
bool stream_plan(int sms, int64_t chunk, int mode, CoopPlan* out) {
  const int64_t rows = (chunk + kBulkRow - 1) / kBulkRow;
  const size_t sm = sizeof(double) * kBulkRow *
                    (D + size_t(rows > kBulkTMR ? rows - kBulkTMR : 0) + size_t(rows > RW ? rows - RW : 0));
  if (sm > 227 * 1024) return false;
  const void* fn = reinterpret_cast<const void*>(mgs_stream_kernel<kBulkThreads, RW, D, kBulkPPT, kBulkTMR>);
  ensure_smem(fn, sm);
  int fit = 0;
  TPDG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, fn, kBulkThreads, sm));
  if (fit < 1) return false;
  *out = {sms, chunk, sm, mode, kBulkThreads};
  return true;
}

CoopPlan mgs_coop_plan(int64_t n) {
  int dev = 0, sms = 0;
  TPDG_CUDA_CHECK(cudaGetDevice(&dev));
  TPDG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int64_t chunk = (n + sms - 1) / sms;
  chunk = (chunk + 1) & ~int64_t(1);
  CoopPlan plan{sms, chunk, 0, 0};  // fallback: w in global memory
  if (chunk <= 4 * kBulkRow && stream_plan<4, 8>(sms, chunk, 1, &plan)) return plan;
  if (chunk <= 10 * kBulkRow && stream_plan<10, 8>(sms, chunk, 2, &plan)) return plan;
  if (stream_plan<10, 4>(sms, chunk, 3, &plan)) return plan;
  return plan;
}

int stream_grid(int64_t n) {
  const int64_t want = (n + 255) / 256;
  const int64_t cap = 148 * 8;
  return int(want < cap ? (want > 0 ? want : 1) : cap);
}

} // namespace

int reduce_grid(int64_t n) {
  const int64_t want = (n / 2 + kRedThreads - 1) / kRedThreads;
  const int64_t cap = 148 * 8;
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
                     double* partial, double* result, unsigned* counter, cudaStream_t st, const int* skip,
                     bool sqrt_norm) {
  mgs_kernel<<<reduce_grid(n), kRedThreads, 0, st>>>(w, vprev, hprev, vj, n, partial, result, counter,
                                                      vj == nullptr && sqrt_norm ? 1 : 0, skip);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

void launch_axpy_neg(double* w, const double* h, const double* v, int64_t n, cudaStream_t st) {
  axpy_neg_kernel<<<stream_grid(n), 256, 0, st>>>(w, h, v, n);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

void launch_scale_div(const double* in, const double* den, double* out, int64_t n, cudaStream_t st,
                      const int* skip) {
  scale_div_kernel<<<stream_grid(n), 256, 0, st>>>(in, den, out, n, skip);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

void launch_mgs_iteration(double* V, int64_t ldv, int k, int64_t n, double* hc, double* partial, unsigned* bar,
                          const int* skip, cudaStream_t st, const GmresDev* G, GmresStatus* status) {
  // plans per (device, slice length): rank threads of the loopback transport may hold different n
  static std::mutex mu;
  static std::map<std::pair<int, int64_t>, CoopPlan> plans;
  int dev = 0;
  TPDG_CUDA_CHECK(cudaGetDevice(&dev));
  CoopPlan plan;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = plans.find({dev, n});
    if (it == plans.end()) it = plans.emplace(std::make_pair(dev, n), mgs_coop_plan(n)).first;
    plan = it->second;
  }
  int64_t chunk = plan.chunk;
  GmresDev g = G && G->m <= kFusedGivensMaxM ? *G : GmresDev{};
  GmresStatus* gs = G && G->m <= kFusedGivensMaxM ? status : nullptr;
  void* args[] = {&V, &ldv, &k, &n, &chunk, &hc, &partial, &bar, &skip, &g, &gs};
  void* fn = plan.mode == 1   ? reinterpret_cast<void*>(mgs_stream_kernel<kBulkThreads, 4, 8, kBulkPPT, kBulkTMR>)
             : plan.mode == 2 ? reinterpret_cast<void*>(mgs_stream_kernel<kBulkThreads, 10, 8, kBulkPPT, kBulkTMR>)
             : plan.mode == 3 ? reinterpret_cast<void*>(mgs_stream_kernel<kBulkThreads, 10, 4, kBulkPPT, kBulkTMR>)
                              : reinterpret_cast<void*>(mgs_global_kernel);
  TPDG_CUDA_CHECK(cudaLaunchCooperativeKernel(fn, dim3(plan.grid), dim3(plan.threads), args, plan.smem, st));
  ++g_launches;
}

int mgs_partial_doubles(int m) { return (m + 2) * 256; }

bool mgs_fuses_givens(int m) { return m <= kFusedGivensMaxM; }

void launch_givens(const GmresDev& G, int k, GmresStatus* status, cudaStream_t st) {
  givens_kernel<<<1, 32, sizeof(double) * size_t(3 * G.m + 4), st>>>(G, k, status);
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

void launch_backsolve(const GmresDev& G, int k, cudaStream_t st) {
  if (k > kBacksolveSmemMax) {
    backsolve_global_kernel<<<1, 32, 0, st>>>(G, k);
    TPDG_CUDA_CHECK(cudaGetLastError());
    ++g_launches;
    return;
  }
  const size_t smem = sizeof(double) * size_t(k * k + 2 * k + 1);
  if (smem > 48 * 1024)  // per call: cudaFuncSetAttribute is per device and cheap
    TPDG_CUDA_CHECK(cudaFuncSetAttribute(backsolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  backsolve_kernel<<<1, 32, smem, st>>>(G, k);
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
