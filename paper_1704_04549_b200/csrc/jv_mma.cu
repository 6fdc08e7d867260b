// Scalar 2D operator (a M + b J) v on the FP64 tensor cores (DMMA.8x8x4, mma.sync m8n8k4 f64),
// one warp per element, persistent grid. Same operator as jv2d_sized_kernel (jv.cu; reference
// ops/linearized.hpp:107-162,201-240), with every sum-factorized stage a warp-level DMMA product:
//
//   (1) t    = v G^T                    Q x Q   . Q x MU      (+ 6 spare columns, see below)
//   (2) vals = G t                      MU x Q  . Q x NT1
//   (3) A    = [M | F0] [GW^T ; DW^T]   MU x 2MU . 2MU x Q
//   (4) B    = F1 GW^T                  MU x MU . MU x Q
//   (5) out  = [GW | DW] [A ; B]        Q x 2MU . 2MU x Q      + face lifts, straight to HBM
//
// The face traces ride along in (1)-(2): the spare columns of t hold the element's two x-face
// layers v[:, 0], v[:, Q-1] and the four neighbour face layers, so that (2) also returns
// G v[:, layer] (own x-face traces) and G (neighbour layer) (neighbour traces); the own y-face
// traces are rows 0 and Q-1 of t. F1 overwrites vals in place.
//
// Fragment layouts (PTX mma.m8n8k4 .f64, row.col): A 8x4: lane l holds A[l/4][l%4]; B 4x8:
// B[l%4][l/4]; C 8x8: C[l/4][2(l%4) + {0,1}]. Leading dimensions are chosen so that every
// fragment load is two conflict-free shared-memory wavefronts: ld = 4 (mod 8) for A and for
// column-major B, ld = 8 (mod 16) for row-major B.
//
// Parity: FMA and DMMA change the summation order; the operator's gate is rel-L2 <= 1e-12
// (SURVEY.md sec.8c), measured ~1e-16.
#include <algorithm>

#include "mma.cuh"
#include "tpdg_internal.hpp"

namespace tpdg_gpu {

namespace {

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}

__device__ __forceinline__ const double* nbr_vals(const DevSys& s, const double* vin, const double* halo, int nbr,
                                                  int qq) {
  return nbr < s.n_local ? vin + size_t(nbr) * qq : halo + size_t(nbr - s.n_local) * qq;
}

constexpr int kJvWarps = 16;  // most warps per CTA (q = 16); JvMmaLayout::wcap per instantiation

template <int Q, int MU>
struct JvMmaLayout {
  static constexpr int QP = p8(Q), MP = p8(MU), KQ = p4(Q), KM = p4(MU), K2 = p4(2 * MU);
  static constexpr int NT1 = p8(MU + 6);  // t / vals columns: MU + 6 spare (2 own x layers, 4 neighbour layers)
  static constexpr int LV = lda4(KQ), LG = lda4(KQ), LT = ldb8(NT1), LVAL = lda4(NT1), LMF = lda4(K2),
                       LAB = ldb8(QP), LW5 = lda4(K2), LWG = lda4(KM);
  static constexpr int GROWS = NT1 > MP ? NT1 : MP;
  // CTA-shared weights
  static constexpr int w_G = 0;                       // G (GROWS x LG), zero padded
  static constexpr int w_W5 = w_G + GROWS * LG;       // [GW | DW] (QP x LW5), zero padded
  static constexpr int w_WG = w_W5 + QP * LW5;        // GW (QP x LWG), columns >= MU zero
  static constexpr int weights = (w_WG + QP * LWG + 1) & ~1;
  // per-warp workspace: region 0 = v, t (early) / [A ; B] (late); vals/F1; [M | F0]; faces
  static constexpr int e_v = 0;
  static constexpr int e_t = e_v + QP * LV;
  static constexpr int r0_early = e_t + KQ * LT;
  static constexpr int r0_late = K2 * LAB;
  static constexpr int r0 = ((r0_early > r0_late ? r0_early : r0_late) + 1) & ~1;
  static constexpr int e_val = r0;
  // [M | F0] is written by the point-wise pass, after v and t are dead, and read by product (3) before
  // [A ; B] is stored: it shares region 0 when it fits
  static constexpr bool mf_in_r0 = MP * LMF <= r0;
  static constexpr int e_mf = mf_in_r0 ? 0 : e_val + MP * LVAL;
  static constexpr int e_g = mf_in_r0 ? e_val + MP * LVAL : e_mf + MP * LMF;  // g[4][MU]
  static constexpr int e_lift = e_g + 4 * MU;          // lift vectors [4][Q]
  static constexpr int e_pw = (e_lift + 4 * Q + 1) & ~1; // jd | dft0 | dft1 of the element (cp.async, prefetched)
  // q <= 16: the element's jd / dft are not staged (they are read once, from L2, bulk-prefetched one element ahead):
  // the workspace shrinks by a third and 16 warps fit (cfg2 p = 15: 36.2 -> 34.0 us); larger q keeps the staging
  // (p = 30 measured 190 us staged vs 197 direct)
  static constexpr bool stage_pw = Q > 16;
  static constexpr int per_warp = stage_pw ? ((e_pw + 3 * MU * MU + 1) & ~1) : e_pw;
  static constexpr int budget = (227 * 1024) / 8 - weights - 16;
  // 12 warps pay at q >= 16 (p = 15 / 20 / 30: 42 -> 41, 83 -> 81, 249 -> 207 us); p = 8 is faster with 8
  static constexpr int wcap = Q > 16 ? 12 : Q == 16 ? kJvWarps : 8;
  static constexpr int warps = budget / per_warp > wcap ? wcap : budget / per_warp;
};

template <int Q, int MU>
__global__ void __launch_bounds__(32 * JvMmaLayout<Q, MU>::wcap) jv2d_mma_kernel(DevSys s, const double* __restrict__ vin,
                                                        const double* __restrict__ halo, double* __restrict__ vout) {
  if (s.skip && *s.skip) return;
  using L = JvMmaLayout<Q, MU>;
  constexpr int QP = L::QP, MP = L::MP, KQ = L::KQ, KM = L::KM, K2 = L::K2, NT1 = L::NT1;
  constexpr int LV = L::LV, LG = L::LG, LT = L::LT, LVAL = L::LVAL, LMF = L::LMF, LAB = L::LAB, LW5 = L::LW5,
                LWG = L::LWG, NW = L::warps, QQ = Q * Q, MM = MU * MU;
  extern __shared__ double sm[];
  double* W = sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < L::weights; i += blockDim.x) W[i] = 0.0;
  __syncthreads();
  for (int i = threadIdx.x; i < MU * Q; i += blockDim.x) {
    const int a = i / Q, j = i % Q;
    W[L::w_G + a * LG + j] = s.g[i];                   // G[a][j]
    W[L::w_W5 + j * LW5 + a] = s.gw[j * MU + a];       // GW[j][a]
    W[L::w_W5 + j * LW5 + MU + a] = s.dw[j * MU + a];  // DW[j][a]
    W[L::w_WG + j * LWG + a] = s.gw[j * MU + a];
  }
  double* E = sm + L::weights + warp * L::per_warp;
  for (int i = lane; i < L::per_warp; i += 32) E[i] = 0.0;  // zero pads (rows / columns never written)
  __syncthreads();
  if (warp >= NW) return;
  const double* G = W + L::w_G;
  const double* W5 = W + L::w_W5;
  const double* WG = W + L::w_WG;
  double* sv = E + L::e_v;
  double* st = E + L::e_t;
  double* sab = E;
  double* sval = E + L::e_val;
  double* smf = E + L::e_mf;
  double* sg = E + L::e_g;
  double* slift = E + L::e_lift;
  const int r = lane >> 2, c2 = 2 * (lane & 3);

  double* spw = E + L::e_pw;
  constexpr int NL = (4 * Q + 31) / 32, NV = (QQ + 31) / 32, NF = (4 * MU + 31) / 32;
  // per-element global data, fetched one element ahead: v and the neighbour face layers into
  // registers, jd / dft into shared memory with cp.async (consumed by the point-wise pass)
  auto fetch_regs = [&](int e, double (&vr)[NV], double (&nr)[NL]) {
    if (e >= s.e_hi) return;
    const double* ve = vin + size_t(e) * QQ;
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const int i = lane + 32 * u;
      vr[u] = i < QQ ? ve[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < NL; ++u) {
      const int idx = lane + 32 * u;
      double x = 0.0;
      if (idx < 4 * Q) {
        const int f = idx / Q, j = idx % Q;
        const int* fc = s.conn + (size_t(e) * 4 + f) * 3;
        if (fc[0] >= 0) {
          const int nf = fc[1], layer = (nf % 2) == 0 ? 0 : Q - 1;
          const double* cf = nbr_vals(s, vin, halo, fc[0], QQ);
          x = nf / 2 == 0 ? cf[j * Q + layer] : cf[layer * Q + j];
        }
      }
      nr[u] = x;
    }
  };
  auto fetch_pw = [&](int e) {
    if (e >= s.e_hi) return;
    const double* jd = s.jdet + size_t(e) * MM;
    const double* d0 = s.dft + size_t(e) * 2 * MM;
    if constexpr (L::stage_pw) {
      for (int i = lane; i < MM; i += 32) cp_async8(spw + i, jd + i);
      for (int i = lane; i < 2 * MM; i += 32) cp_async8(spw + MM + i, d0 + i);
    } else if (lane == 0) {  // HBM -> L2; ranges widened to 16-byte boundaries
      const uintptr_t a = reinterpret_cast<uintptr_t>(jd) & ~uintptr_t(15), b = reinterpret_cast<uintptr_t>(d0) & ~uintptr_t(15);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(unsigned((MM * 8 + 31) & ~15)) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b), "r"(unsigned((2 * MM * 8 + 31) & ~15)) : "memory");
    }
  };
  const int stride = gridDim.x * NW;
  double vr[NV], nr[NL];
  int e = s.e_lo + blockIdx.x * NW + warp;
  fetch_regs(e, vr, nr);
  fetch_pw(e);
  for (; e < s.e_hi; e += stride) {
    // face data of this element (registers; consumed after step 2)
    double fdm[NF], fdp[NF], ffw[NF];
    int fnb[NF], ffl[NF];
#pragma unroll
    for (int u = 0; u < NF; ++u) {
      const int idx = lane + 32 * u;
      fdm[u] = fdp[u] = ffw[u] = 0.0;
      fnb[u] = -1;
      ffl[u] = 0;
      if (idx < 4 * MU) {
        const int f = idx / MU;
        const size_t fq = size_t(e) * 4 * MU + idx;
        const int* fc = s.conn + (size_t(e) * 4 + f) * 3;
        fdm[u] = s.dfm[fq];
        fdp[u] = s.dfp[fq];
        ffw[u] = s.face_w[fq];
        fnb[u] = fc[0];
        ffl[u] = fc[2];
      }
    }
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const int i = lane + 32 * u;
      if (i < QQ) sv[(i / Q) * LV + i % Q] = vr[u];
    }
    double nl[NL];
#pragma unroll
    for (int u = 0; u < NL; ++u) nl[u] = nr[u];
    fetch_regs(e + stride, vr, nr);  // next element, in flight during this one
    __syncwarp();
    {  // (1) t = v G^T
      double acc[QP / 8][NT1 / 8][2];
      zero_tiles(acc);
      mma_tiles<QP / 8, NT1 / 8, KQ / 4, true>(acc, sv, LV, G, LG, lane);
      store_tiles(acc, st, LT, KQ, lane);
    }
    __syncwarp();
    for (int j = lane; j < Q; j += 32) {  // spare columns: own x-face layers
      st[j * LT + MU] = sv[j * LV];
      st[j * LT + MU + 1] = sv[j * LV + Q - 1];
    }
#pragma unroll
    for (int u = 0; u < NL; ++u) {
      const int idx = lane + 32 * u;
      if (idx < 4 * Q) st[(idx % Q) * LT + MU + 2 + idx / Q] = nl[u];
    }
    __syncwarp();
    {  // (2) vals = G t
      double acc[MP / 8][NT1 / 8][2];
      zero_tiles(acc);
      mma_tiles<MP / 8, NT1 / 8, KQ / 4, false>(acc, G, LG, st, LT, lane);
      store_tiles(acc, sval, LVAL, MP, lane);
    }
    __syncwarp();
    // face data g[f][a] = -b fw (dfm tm + dfp tp)
#pragma unroll
    for (int u = 0; u < NF; ++u) {
      const int idx = lane + 32 * u;
      if (idx < 4 * MU) {
        const int a = idx % MU, f = idx / MU;
        const double tm = f < 2 ? sval[a * LVAL + MU + f] : st[(f == 2 ? 0 : Q - 1) * LT + a];
        double tp = 0.0;
        if (fnb[u] >= 0) tp = sval[(ffl[u] == 0 ? a : MU - 1 - a) * LVAL + MU + 2 + f];
        sg[idx] = -s.b * ffw[u] * fma(fdm[u], tm, fdp[u] * tp);
      }
    }
    // point-wise fields: [M | F0] -> smf, F1 -> vals in place
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    for (int qv = lane; qv < MM; qv += 32) {
      const int be = qv / MU, al = qv % MU;
      const double x = sval[be * LVAL + al];
      double cj, c0, c1;
      if constexpr (L::stage_pw) {
        cj = spw[qv], c0 = spw[MM + qv], c1 = spw[2 * MM + qv];
      } else {
        const double* pd = s.dft + size_t(e) * 2 * MM;
        cj = __ldg(s.jdet + size_t(e) * MM + qv), c0 = __ldg(pd + qv), c1 = __ldg(pd + MM + qv);
      }
      smf[be * LMF + al] = s.a * cj * x;
      smf[be * LMF + MU + al] = s.b * (c0 * x);
      sval[be * LVAL + al] = s.b * (c1 * x);
    }
    __syncwarp();
    fetch_pw(e + stride);  // the buffer is free: next element's jd / dft
    // lift vectors: x faces Lf[j] = sum_a G[a][j] g[f][a]; y faces the same over i
    for (int idx = lane; idx < 4 * Q; idx += 32) {
      const int f = idx / Q, j = idx % Q;
      double acc = 0.0;
      for (int a = 0; a < MU; ++a) acc = fma(G[a * LG + j], sg[f * MU + a], acc);
      slift[idx] = acc;
    }
    {  // (3) A = [M | F0] [GW^T ; DW^T] -> rows 0..MU-1 of [A ; B]; (4) B = F1 GW^T -> rows MU..2MU-1
      double acc[MP / 8][QP / 8][2];
      zero_tiles(acc);
      mma_tiles<MP / 8, QP / 8, K2 / 4, true>(acc, smf, LMF, W5, LW5, lane);
      double acc4[MP / 8][QP / 8][2];
      zero_tiles(acc4);
      mma_tiles<MP / 8, QP / 8, KM / 4, true>(acc4, sval, LVAL, WG, LWG, lane);
      store_tiles(acc, sab, LAB, MU, lane);
      store_tiles(acc4, sab + MU * LAB, LAB, MU, lane);
    }
    __syncwarp();
    {  // (5) out = [GW | DW] [A ; B] + lifts
      double acc[QP / 8][QP / 8][2];
      zero_tiles(acc);
      mma_tiles<QP / 8, QP / 8, K2 / 4, false>(acc, W5, LW5, sab, LAB, lane);
      double* oe = vout + size_t(e) * QQ;
#pragma unroll
      for (int mt = 0; mt < QP / 8; ++mt)
#pragma unroll
        for (int nt = 0; nt < QP / 8; ++nt) {
          const int j = 8 * mt + r;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int i = 8 * nt + c2 + u;
            if (j < Q && i < Q) {
              double x = acc[mt][nt][u];
              if (i == 0) x += slift[0 * Q + j];
              if (i == Q - 1) x += slift[1 * Q + j];
              if (j == 0) x += slift[2 * Q + i];
              if (j == Q - 1) x += slift[3 * Q + i];
              oe[j * Q + i] = x;
            }
          }
        }
    }
    __syncwarp();
  }
}

template <int Q, int MU>
bool try_jv2d_mma(const DevSys& s, const double* vin, const double* halo, double* vout, cudaStream_t st) {
  if (s.dim != 2 || s.n_c != 1 || s.q != Q || s.mu != MU) return false;
  using L = JvMmaLayout<Q, MU>;
  static_assert(L::warps >= 1, "element workspace exceeds shared memory");
  const size_t smem = sizeof(double) * size_t(L::weights + L::warps * L::per_warp);
  ensure_smem(jv2d_mma_kernel<Q, MU>, smem, true);
  static int grid = 0;
  if (!grid) {
    int per_sm = 0;
    TPDG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jv2d_mma_kernel<Q, MU>, 32 * L::warps,
                                                                  smem));
    int dev = 0, sms = 0;
    TPDG_CUDA_CHECK(cudaGetDevice(&dev));
    TPDG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = std::max(1, per_sm) * sms;
  }
  const int need = (s.e_hi - s.e_lo + L::warps - 1) / L::warps;
  jv2d_mma_kernel<Q, MU><<<std::min(grid, need), 32 * L::warps, smem, st>>>(s, vin, halo, vout);
  return true;
}

} // namespace

bool launch_jv2d_mma(const DevSys& s, const double* vin, const double* halo, double* vout, cudaStream_t st) {
  return try_jv2d_mma<5, 6>(s, vin, halo, vout, st) || try_jv2d_mma<9, 10>(s, vin, halo, vout, st) ||
         try_jv2d_mma<16, 17>(s, vin, halo, vout, st) || try_jv2d_mma<21, 22>(s, vin, halo, vout, st) ||
         try_jv2d_mma<31, 32>(s, vin, halo, vout, st);
}

} // namespace tpdg_gpu
