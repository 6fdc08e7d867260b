// Matrix-free DG operator (a M + b J) v, sum-factorized, one CTA per element.
//
// Restates jacobian_apply (reference ops/linearized.hpp:201-240) = element_diag_apply
// (:107-162: eval_at_quad, mass + contravariant-flux fields, integrate_back, own-trace face
// terms) + the neighbour coupling through dfp (:216-236), with face_trace / face_lift /
// neighbor_trace from ops/discretization.hpp:89-181.
//
// Parity contract: rel-L2 <= 1e-12 against the reference. The volume and face
// contributions are fused (one lift per face for own + neighbour trace, one combined
// integrate-back for the mass and flux fields), so the summation order differs from the
// reference's; the reference's own FMA/no-FMA builds differ by ~2.5e-16 here.
//
// HBM layout (reference orders, read once per launch): v [e][c][tensor, x fastest],
// jdet [e][mu^d], dft [e][dir][mu^d][nc][nc], dfm/dfp [e][f][mu^(d-1)][nc][nc], face_w.
#include <algorithm>

#include "tpdg_internal.hpp"

namespace tpdg_gpu {

namespace {

__device__ __forceinline__ const double* nbr_block(const DevSys& s, const double* vin, const double* halo, int nbr) {
  const size_t blk = size_t(s.n_c) * s.npe;
  return nbr < s.n_local ? vin + size_t(nbr) * blk : halo + size_t(nbr - s.n_local) * blk;
}

// ------------------------------------------------------------------------------------ 2D
// NC, Q, MU: compile-time sizes of an instantiated system (0: runtime, from s)
template <int NT, int NC = 0, int Q = 0, int MU = 0>
__global__ void __launch_bounds__(NT) jv2d_kernel(DevSys s, const double* __restrict__ vin,
                                                    const double* __restrict__ halo, double* __restrict__ vout) {
  extern __shared__ double sm[];
  if (s.skip && *s.skip) return;
  const int e = s.e_lo + blockIdx.x;
  const int q = Q ? Q : s.q, mu = MU ? MU : s.mu, nc = NC ? NC : s.n_c, qq = q * q, mm = mu * mu;
  const int tid = threadIdx.x, nt = blockDim.x;
  double* sG = sm;                 // mu*q
  double* sGW = sG + mu * q;       // q*mu
  double* sDW = sGW + q * mu;      // q*mu
  double* sv = sDW + q * mu;       // nc*q*q
  double* st = sv + nc * qq;       // nc*q*mu    t[c][j][al]
  double* sval = st + nc * q * mu; // nc*mu*mu   vals[c][be][al]
  double* sf = sval + nc * mm;     // 3*nc*mu*mu fields M, F0, F1 [r][be][al]
  double* sA = sf + 3 * nc * mm;   // nc*mu*q    A[r][be][i]
  double* sB = sA + nc * mu * q;   // nc*mu*q
  double* str = sB + nc * mu * q;  // 2*4*nc*mu  own / neighbour traces [side][f][c][a]
  double* sg = str + 8 * nc * mu;  // 4*nc*mu    lifted face data [f][r][a]

  for (int i = tid; i < mu * q; i += nt) {
    sG[i] = s.g[i];
    sGW[i] = s.gw[i];
    sDW[i] = s.dw[i];
  }
  const double* ve = vin + size_t(e) * nc * qq;
  for (int i = tid; i < nc * qq; i += nt) sv[i] = ve[i];
  __syncthreads();

  // eval_at_quad: x then y contraction with G.
  for (int idx = tid; idx < nc * q * mu; idx += nt) {
    const int al = idx % mu, j = (idx / mu) % q, c = idx / (mu * q);
    const double* row = sv + c * qq + j * q;
    double acc = 0.0;
    for (int i = 0; i < q; ++i) acc = fma(sG[al * q + i], row[i], acc);
    st[idx] = acc;
  }
  // own + neighbour face traces (need only sv / global v)
  for (int idx = tid; idx < 8 * nc * mu; idx += nt) {
    const int a = idx % mu, c = (idx / mu) % nc, f = (idx / (mu * nc)) % 4, side = idx / (4 * mu * nc);
    const int* fc = s.conn + (size_t(e) * 4 + f) * 3;
    double acc = 0.0;
    if (side == 0) {
      const int layer = (f % 2) == 0 ? 0 : q - 1;
      const double* cf = sv + c * qq;
      if (f / 2 == 0)
        for (int j = 0; j < q; ++j) acc = fma(sG[a * q + j], cf[j * q + layer], acc);
      else
        for (int j = 0; j < q; ++j) acc = fma(sG[a * q + j], cf[layer * q + j], acc);
    } else if (fc[0] >= 0) {
      const int nf = fc[1];
      const int aa = fc[2] == 0 ? a : mu - 1 - a;  // orient_face_coords, dg/mesh.hpp:57-67
      const int layer = (nf % 2) == 0 ? 0 : q - 1;
      const double* cf = nbr_block(s, vin, halo, fc[0]) + size_t(c) * qq;
      if (nf / 2 == 0)
        for (int j = 0; j < q; ++j) acc = fma(sG[aa * q + j], cf[j * q + layer], acc);
      else
        for (int j = 0; j < q; ++j) acc = fma(sG[aa * q + j], cf[layer * q + j], acc);
    }
    str[idx] = acc;
  }
  __syncthreads();
  for (int idx = tid; idx < nc * mm; idx += nt) {
    const int al = idx % mu, be = (idx / mu) % mu, c = idx / mm;
    const double* tc = st + c * q * mu;
    double acc = 0.0;
    for (int j = 0; j < q; ++j) acc = fma(sG[be * q + j], tc[j * mu + al], acc);
    sval[idx] = acc;
  }
  // face data g[f][r][a] = -b fw (dfm tm + dfp tp)
  for (int idx = tid; idx < 4 * nc * mu; idx += nt) {
    const int a = idx % mu, r = (idx / mu) % nc, f = idx / (mu * nc);
    const size_t fq = (size_t(e) * 4 + f) * mu + a;
    const size_t fr = (((size_t(e) * 4 + f) * nc + r) * mu + a) * nc;  // regrouped: [e][f][r][a][c]
    const double* dfm = s.dfmr ? s.dfmr + fr : s.dfm + fq * nc * nc + r * nc;
    const double* dfp = s.dfpr ? s.dfpr + fr : s.dfp + fq * nc * nc + r * nc;
    const double* tm = str + (f * nc) * mu + a;
    const double* tp = str + ((4 + f) * nc) * mu + a;
    double acc = 0.0;
    if (!s.small) {
      for (int c = 0; c < nc; ++c) acc = fma(dfm[c], tm[c * mu], fma(dfp[c], tp[c * mu], acc));
    } else {
      acc = fma(dfm[r], tm[r * mu], dfp[r] * tp[r * mu]);
    }
    sg[idx] = -s.b * s.face_w[fq] * acc;
  }
  __syncthreads();
  // point-wise fields: M = a jd vals_r ; F_dir = b sum_c dft[dir][q][r][c] vals_c
  for (int idx = tid; idx < nc * mm; idx += nt) {
    const int qv = idx % mm, r = idx / mm;
    const double* d0 = s.dftr ? s.dftr + ((size_t(e) * nc + r) * 2 * mm + qv) * nc
                              : s.dft + ((size_t(e) * 2 + 0) * mm + qv) * nc * nc + r * nc;
    const double* d1 = s.dftr ? d0 + size_t(mm) * nc : s.dft + ((size_t(e) * 2 + 1) * mm + qv) * nc * nc + r * nc;
    double f0 = 0.0, f1 = 0.0;
    if (!s.small) {
      for (int c = 0; c < nc; ++c) {
        const double vc = sval[c * mm + qv];
        f0 = fma(d0[c], vc, f0);
        f1 = fma(d1[c], vc, f1);
      }
    } else {
      f0 = d0[r] * sval[r * mm + qv];
      f1 = d1[r] * sval[r * mm + qv];
    }
    sf[idx] = s.a * s.jdet[size_t(e) * mm + qv] * sval[idx];
    sf[nc * mm + idx] = s.b * f0;
    sf[2 * nc * mm + idx] = s.b * f1;
  }
  __syncthreads();
  // integrate_back, x direction: A = GW M + DW F0 ; B = GW F1
  for (int idx = tid; idx < nc * mu * q; idx += nt) {
    const int i = idx % q, be = (idx / q) % mu, r = idx / (q * mu);
    const double* M = sf + r * mm + be * mu;
    const double* F0 = sf + nc * mm + r * mm + be * mu;
    const double* F1 = sf + 2 * nc * mm + r * mm + be * mu;
    double acc_a = 0.0, acc_b = 0.0;
    for (int al = 0; al < mu; ++al) {
      acc_a = fma(sGW[i * mu + al], M[al], fma(sDW[i * mu + al], F0[al], acc_a));
      acc_b = fma(sGW[i * mu + al], F1[al], acc_b);
    }
    sA[idx] = acc_a;
    sB[idx] = acc_b;
  }
  __syncthreads();
  // y direction + face lifts, written straight to HBM
  double* oe = vout + size_t(e) * nc * qq;
  for (int idx = tid; idx < nc * qq; idx += nt) {
    const int i = idx % q, j = (idx / q) % q, r = idx / qq;
    const double* A = sA + r * mu * q + i;
    const double* B = sB + r * mu * q + i;
    double acc = 0.0;
    for (int be = 0; be < mu; ++be) acc = fma(sGW[j * mu + be], A[be * q], fma(sDW[j * mu + be], B[be * q], acc));
    // face_lift: x faces hit column i = layer at row j, y faces row j = layer at column i
    if (i == 0 || i == q - 1) {
      const double* gf = sg + ((i == 0 ? 0 : 1) * nc + r) * mu;
      for (int a = 0; a < mu; ++a) acc = fma(sG[a * q + j], gf[a], acc);
    }
    if (j == 0 || j == q - 1) {
      const double* gf = sg + ((j == 0 ? 2 : 3) * nc + r) * mu;
      for (int a = 0; a < mu; ++a) acc = fma(sG[a * q + i], gf[a], acc);
    }
    oe[idx] = acc;
  }
}

size_t jv2d_smem(const DevSys& s) {
  const int q = s.q, mu = s.mu, nc = s.n_c;
  return sizeof(double) * size_t(3 * mu * q + nc * q * q + nc * q * mu + 4 * nc * mu * mu + 2 * nc * mu * q +
                                 12 * nc * mu);
}

// ------------------------------------------------------------------------------------ 2D, sized
// Scalar (n_c = 1) 2D operator with compile-time (Q, MU), one warp per element, CTA-shared
// weights, persistent grid. The five sum-factorized stages are written as register-tiled small
// products with stacked K so that the mass and flux integrations share one pass:
//   t    = v G^T                      (q x q) (q x mu)
//   vals = G t                        (mu x q) (q x mu)
//   AB   = [a jd vals | b dft0 vals ; b dft1 vals | 0] [GW^T ; DW^T]     (2 mu x 2 mu)(2 mu x q)
//   out  = [GW | DW] AB  + face lifts (q x 2 mu)(2 mu x q)
// FMA contraction is allowed here (the operator's parity gate is 1e-12).

template <int R, int K, int C, bool BT, int TI, int TJ>
__device__ __forceinline__ void warp_mm_fma(const double* A, int lda, const double* B, int ldb, double* O, int ldo,
                                            int lane) {
  constexpr int NTI = (R + TI - 1) / TI, NTJ = (C + TJ - 1) / TJ;
  for (int t = lane; t < NTI * NTJ; t += 32) {
    const int i0 = (t / NTJ) * TI, j0 = (t % NTJ) * TJ;
    double acc[TI][TJ];
#pragma unroll
    for (int ii = 0; ii < TI; ++ii)
#pragma unroll
      for (int jj = 0; jj < TJ; ++jj) acc[ii][jj] = 0.0;
#pragma unroll 2
    for (int k = 0; k < K; ++k) {
      double a[TI], b[TJ];
#pragma unroll
      for (int ii = 0; ii < TI; ++ii) a[ii] = A[(i0 + ii < R ? i0 + ii : R - 1) * lda + k];
#pragma unroll
      for (int jj = 0; jj < TJ; ++jj) {
        const int j = j0 + jj < C ? j0 + jj : C - 1;
        b[jj] = BT ? B[j * ldb + k] : B[k * ldb + j];
      }
#pragma unroll
      for (int ii = 0; ii < TI; ++ii)
#pragma unroll
        for (int jj = 0; jj < TJ; ++jj) acc[ii][jj] = fma(a[ii], b[jj], acc[ii][jj]);
    }
#pragma unroll
    for (int ii = 0; ii < TI; ++ii)
#pragma unroll
      for (int jj = 0; jj < TJ; ++jj)
        if (i0 + ii < R && j0 + jj < C) O[(i0 + ii) * ldo + j0 + jj] = acc[ii][jj];
  }
}

template <int Q, int MU>
struct Jv2dLayout {
  static constexpr int M2 = 2 * MU;
  // CTA-shared weights
  static constexpr int w_G = 0;                      // G      MU x Q
  static constexpr int w_W4 = w_G + MU * Q;          // [GW^T ; DW^T]  2MU x Q
  static constexpr int w_W5 = w_W4 + M2 * Q;         // [GW | DW]      Q x 2MU
  static constexpr int weights = w_W5 + Q * M2;
  // per-warp element workspace (dead buffers aliased)
  static constexpr int e_v = 0;                      // v (Q x Q), later out
  static constexpr int e_t = e_v + Q * Q;            // t (Q x MU), later AB (2MU x Q)
  static constexpr int e_val = e_t + M2 * Q;         // vals (MU x MU)
  static constexpr int e_mf = e_val + MU * MU;       // [M | F0] (MU x 2MU), F1 (MU x MU)
  static constexpr int e_tr = e_mf + 3 * MU * MU;    // traces 8 x MU, face data 4 x MU
  static constexpr int per_elem = ((e_tr + 12 * MU) + 1) & ~1;
  static constexpr int budget = (227 * 1024) / 8 - weights - 64;
  static constexpr int warps = budget / per_elem >= 4 ? 4 : (budget / per_elem >= 1 ? budget / per_elem : 1);
};

template <int Q, int MU>
__global__ void __launch_bounds__(128) jv2d_sized_kernel(DevSys s, const double* __restrict__ vin,
                                                          const double* __restrict__ halo, double* __restrict__ vout) {
  if (s.skip && *s.skip) return;
  using L = Jv2dLayout<Q, MU>;
  constexpr int M2 = L::M2, QQ = Q * Q, MM = MU * MU, NW = L::warps;
  extern __shared__ double sm[];
  double* W = sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* E = sm + L::weights + warp * L::per_elem;
  for (int i = threadIdx.x; i < MU * Q; i += blockDim.x) {
    const int a = i / Q, j = i % Q;
    W[L::w_G + i] = s.g[i];
    W[L::w_W4 + a * Q + j] = s.gw[j * MU + a];          // GW^T
    W[L::w_W4 + (MU + a) * Q + j] = s.dw[j * MU + a];   // DW^T
    W[L::w_W5 + j * M2 + a] = s.gw[j * MU + a];         // GW
    W[L::w_W5 + j * M2 + MU + a] = s.dw[j * MU + a];    // DW
  }
  __syncthreads();
  if (warp >= NW) return;
  const double* G = W + L::w_G;
  for (int e = s.e_lo + blockIdx.x * NW + warp; e < s.e_hi; e += gridDim.x * NW) {
    double* v = E + L::e_v;
    double* t = E + L::e_t;
    double* ab = E + L::e_t;
    double* val = E + L::e_val;
    double* mf = E + L::e_mf;
    double* f1 = mf + MU * M2;
    double* tr = E + L::e_tr;
    const double* ve = vin + size_t(e) * QQ;
    for (int i = lane; i < QQ; i += 32) v[i] = ve[i];
    __syncwarp();
    // face traces: own (from v) and neighbour (global), tr[side][f][a]
    for (int idx = lane; idx < 8 * MU; idx += 32) {
      const int a = idx % MU, f = (idx / MU) % 4, side = idx / (4 * MU);
      double acc = 0.0;
      if (side == 0) {
        const int layer = (f % 2) == 0 ? 0 : Q - 1;
        if (f / 2 == 0)
          for (int j = 0; j < Q; ++j) acc = fma(G[a * Q + j], v[j * Q + layer], acc);
        else
          for (int j = 0; j < Q; ++j) acc = fma(G[a * Q + j], v[layer * Q + j], acc);
      } else {
        const int* fc = s.conn + (size_t(e) * 4 + f) * 3;
        if (fc[0] >= 0) {
          const int nf = fc[1];
          const int aa = fc[2] == 0 ? a : MU - 1 - a;
          const int layer = (nf % 2) == 0 ? 0 : Q - 1;
          const double* cf = nbr_block(s, vin, halo, fc[0]);
          if (nf / 2 == 0)
            for (int j = 0; j < Q; ++j) acc = fma(G[aa * Q + j], cf[j * Q + layer], acc);
          else
            for (int j = 0; j < Q; ++j) acc = fma(G[aa * Q + j], cf[layer * Q + j], acc);
        }
      }
      tr[idx] = acc;
    }
    warp_mm_fma<Q, Q, MU, true, 2, 4>(v, Q, G, Q, t, MU, lane);  // t = v G^T
    __syncwarp();
    for (int idx = lane; idx < 4 * MU; idx += 32) {  // face data g[f][a]
      const int a = idx % MU, f = idx / MU;
      const size_t fq = (size_t(e) * 4 + f) * MU + a;
      const double acc = fma(s.dfm[fq], tr[f * MU + a], s.dfp[fq] * tr[(4 + f) * MU + a]);
      tr[8 * MU + idx] = -s.b * s.face_w[fq] * acc;
    }
    warp_mm_fma<MU, Q, MU, false, 2, 4>(G, Q, t, MU, val, MU, lane);  // vals = G t
    __syncwarp();
    const double* jd = s.jdet + size_t(e) * MM;
    const double* d0 = s.dft + size_t(e) * 2 * MM;
    const double* d1 = d0 + MM;
    for (int qv = lane; qv < MM; qv += 32) {
      const int be = qv / MU, al = qv % MU;
      const double x = val[qv];
      mf[be * M2 + al] = s.a * jd[qv] * x;
      mf[be * M2 + MU + al] = s.b * (d0[qv] * x);
      f1[qv] = s.b * (d1[qv] * x);
    }
    __syncwarp();
    warp_mm_fma<MU, M2, Q, false, 2, 4>(mf, M2, W + L::w_W4, Q, ab, Q, lane);       // A = [M|F0][GW^T;DW^T]
    warp_mm_fma<MU, MU, Q, false, 2, 4>(f1, MU, W + L::w_W4, Q, ab + MU * Q, Q, lane);  // B = F1 GW^T
    __syncwarp();
    warp_mm_fma<Q, M2, Q, false, 2, 4>(W + L::w_W5, M2, ab, Q, v, Q, lane);  // out = [GW|DW][A;B] (into v)
    __syncwarp();
    double* oe = vout + size_t(e) * QQ;
    const double* gf = tr + 8 * MU;
    for (int idx = lane; idx < QQ; idx += 32) {
      const int i = idx % Q, j = idx / Q;
      double acc = v[idx];
      if (i == 0 || i == Q - 1) {
        const double* g = gf + (i == 0 ? 0 : 1) * MU;
        for (int a = 0; a < MU; ++a) acc = fma(G[a * Q + j], g[a], acc);
      }
      if (j == 0 || j == Q - 1) {
        const double* g = gf + (j == 0 ? 2 : 3) * MU;
        for (int a = 0; a < MU; ++a) acc = fma(G[a * Q + i], g[a], acc);
      }
      oe[idx] = acc;
    }
    __syncwarp();
  }
}

template <int Q, int MU>
bool try_jv2d_sized(const DevSys& s, const double* vin, const double* halo, double* vout, cudaStream_t st) {
  if (s.dim != 2 || s.n_c != 1 || s.q != Q || s.mu != MU) return false;
  using L = Jv2dLayout<Q, MU>;
  const size_t smem = sizeof(double) * size_t(L::weights + L::warps * L::per_elem);
  ensure_smem(jv2d_sized_kernel<Q, MU>, smem, true);
  static int grid = 0;
  if (!grid) {
    int per_sm = 0;
    TPDG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jv2d_sized_kernel<Q, MU>, 128, smem));
    int dev = 0, sms = 0;
    TPDG_CUDA_CHECK(cudaGetDevice(&dev));
    TPDG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = std::max(1, per_sm) * sms;
  }
  const int need = (s.e_hi - s.e_lo + L::warps - 1) / L::warps;
  jv2d_sized_kernel<Q, MU><<<std::min(grid, need), 128, smem, st>>>(s, vin, halo, vout);
  return true;
}

bool launch_jv2d_sized(const DevSys& s, const double* vin, const double* halo, double* vout, cudaStream_t st) {
  return try_jv2d_sized<5, 6>(s, vin, halo, vout, st) || try_jv2d_sized<9, 10>(s, vin, halo, vout, st) ||
         try_jv2d_sized<16, 17>(s, vin, halo, vout, st) || try_jv2d_sized<21, 22>(s, vin, halo, vout, st) ||
         try_jv2d_sized<31, 32>(s, vin, halo, vout, st);
}

// ------------------------------------------------------------------------------------ 3D
// Face f: axis = f/2, tangents (dg/mesh.hpp:47-52): axis0 -> (y,z), axis1 -> (x,z), axis2 -> (x,y).
__device__ __forceinline__ int flat_face_node(int q, int f, int j0, int j1) {
  const int axis = f / 2, layer = (f % 2) == 0 ? 0 : q - 1;
  int idx[3];
  idx[axis] = layer;
  idx[axis == 0 ? 1 : 0] = j0;
  idx[axis == 2 ? 1 : 2] = j1;
  return (idx[2] * q + idx[1]) * q + idx[0];
}

template <int NT, int NC = 0, int Q = 0, int MU = 0>
__global__ void __launch_bounds__(NT) jv3d_kernel(DevSys s, const double* __restrict__ vin,
                                                    const double* __restrict__ halo, double* __restrict__ vout) {
  extern __shared__ double sm[];
  if (s.skip && *s.skip) return;
  const int e = s.e_lo + blockIdx.x;
  const int q = Q ? Q : s.q, mu = MU ? MU : s.mu, nc = NC ? NC : s.n_c;
  const int q3 = q * q * q, m3 = mu * mu * mu, m2 = mu * mu, q2 = q * q;
  const int tid = threadIdx.x, nt = blockDim.x;
  double* sG = sm;
  double* sGW = sG + mu * q;
  double* sDW = sGW + q * mu;
  double* sv = sDW + q * mu;          // nc*q^3
  double* sval = sv + nc * q3;        // nc*mu^3
  double* sbuf = sval + nc * m3;      // big scratch: max(t1+t2 eval, fields + X + Y)
  // eval temporaries
  double* t1 = sbuf;                  // nc * q*q*mu  [c][k][j][al]
  double* t2 = t1 + nc * q2 * mu;     // nc * q*mu*mu [c][k][be][al]
  // per-r temporaries
  double* fM = sbuf;                  // 4 fields mu^3: M, F0, F1, F2
  double* Xa = fM + 4 * m3;           // mu*mu*q [ga][be][i]
  double* Xb = Xa + m2 * q;
  double* Xc = Xb + m2 * q;
  double* Ya = Xc + m2 * q;           // mu*q*q [ga][j][i]
  double* Yc = Ya + mu * q2;
  double* str = Yc + mu * q2;         // 2*6*nc*m2 traces
  double* wa = str + 12 * nc * m2;    // trace temp: 12*nc*q*mu
  double* sg = wa + 12 * nc * q * mu; // 6*nc*m2 face data
  double* sacc = sg + 6 * nc * m2;    // nc*q^3 output accumulator

  for (int i = tid; i < mu * q; i += nt) {
    sG[i] = s.g[i];
    sGW[i] = s.gw[i];
    sDW[i] = s.dw[i];
  }
  const double* ve = vin + size_t(e) * nc * q3;
  for (int i = tid; i < nc * q3; i += nt) sv[i] = ve[i];
  __syncthreads();
  // ---- eval_at_quad
  for (int idx = tid; idx < nc * q2 * mu; idx += nt) {
    const int al = idx % mu, jk = (idx / mu) % q2, c = idx / (mu * q2);
    const double* row = sv + c * q3 + jk * q;
    double acc = 0.0;
    for (int i = 0; i < q; ++i) acc = fma(sG[al * q + i], row[i], acc);
    t1[idx] = acc;
  }
  __syncthreads();
  for (int idx = tid; idx < nc * q * m2; idx += nt) {
    const int al = idx % mu, be = (idx / mu) % mu, k = (idx / m2) % q, c = idx / (m2 * q);
    const double* col = t1 + (c * q + k) * q * mu + al;
    double acc = 0.0;
    for (int j = 0; j < q; ++j) acc = fma(sG[be * q + j], col[j * mu], acc);
    t2[idx] = acc;
  }
  __syncthreads();
  for (int idx = tid; idx < nc * m3; idx += nt) {
    const int ab = idx % m2, ga = (idx / m2) % mu, c = idx / m3;
    const double* col = t2 + c * q * m2 + ab;
    double acc = 0.0;
    for (int k = 0; k < q; ++k) acc = fma(sG[ga * q + k], col[k * m2], acc);
    sval[idx] = acc;
  }
  __syncthreads();
  // ---- face traces (own: side 0, neighbour: side 1), two-stage G along the tangents
  for (int idx = tid; idx < 12 * nc * q * mu; idx += nt) {
    const int a = idx % mu, j1 = (idx / mu) % q, c = (idx / (mu * q)) % nc, f = (idx / (mu * q * nc)) % 6;
    const int side = idx / (6 * mu * q * nc);
    const int* fc = s.conn + (size_t(e) * 6 + f) * 3;
    double acc = 0.0;
    if (side == 0) {
      const double* cf = sv + c * q3;
      for (int j0 = 0; j0 < q; ++j0) acc = fma(sG[a * q + j0], cf[flat_face_node(q, f, j0, j1)], acc);
    } else if (fc[0] >= 0) {
      const double* cf = nbr_block(s, vin, halo, fc[0]) + size_t(c) * q3;
      for (int j0 = 0; j0 < q; ++j0) acc = fma(sG[a * q + j0], cf[flat_face_node(q, fc[1], j0, j1)], acc);
    }
    wa[idx] = acc;  // [side][f][c][j1][a]
  }
  __syncthreads();
  for (int idx = tid; idx < 12 * nc * m2; idx += nt) {
    const int a = idx % mu, bb = (idx / mu) % mu, rest = idx / m2;  // rest = (side*6 + f)*nc + c
    const double* w = wa + size_t(rest) * q * mu + a;
    double acc = 0.0;
    for (int j1 = 0; j1 < q; ++j1) acc = fma(sG[bb * q + j1], w[j1 * mu], acc);
    str[idx] = acc;  // [side][f][c][b][a] in the face's own (a, b) enumeration
  }
  __syncthreads();
  for (int idx = tid; idx < 6 * nc * m2; idx += nt) {
    const int qf = idx % m2, r = (idx / m2) % nc, f = idx / (m2 * nc);
    const int* fc = s.conn + (size_t(e) * 6 + f) * 3;
    const size_t fq = (size_t(e) * 6 + f) * m2 + qf;
    const size_t fr = (((size_t(e) * 6 + f) * nc + r) * m2 + qf) * nc;  // regrouped: [e][f][r][point][c]
    const double* dfm = s.dfmr ? s.dfmr + fr : s.dfm + fq * nc * nc + r * nc;
    const double* dfp = s.dfpr ? s.dfpr + fr : s.dfp + fq * nc * nc + r * nc;
    // neighbour trace permuted into this face's enumeration (orient_face_coords, dg/mesh.hpp:57-67)
    const int qa = qf % mu, qb = qf / mu;
    const int code = fc[2];
    int u = (code & 4) ? qb : qa, v = (code & 4) ? qa : qb;
    if (code & 1) u = mu - 1 - u;
    if (code & 2) v = mu - 1 - v;
    const int qn = v * mu + u;
    const double* tm = str + (f * nc) * m2;
    const double* tp = str + ((6 + f) * nc) * m2;
    double acc = 0.0;
    if (!s.small) {
      for (int c = 0; c < nc; ++c) acc = fma(dfm[c], tm[c * m2 + qf], fma(dfp[c], tp[c * m2 + qn], acc));
    } else {
      acc = fma(dfm[r], tm[r * m2 + qf], dfp[r] * tp[r * m2 + qn]);
    }
    sg[idx] = -s.b * s.face_w[fq] * acc;
  }
  __syncthreads();
  // first stage of face_lift: la[f][r][j0][b] = sum_a G(a, j0) g[f][r][b][a]   (reuses wa)
  double* la = wa;
  for (int idx = tid; idx < 6 * nc * q * mu; idx += nt) {
    const int bb = idx % mu, j0 = (idx / mu) % q, fr = idx / (mu * q);
    const double* gf = sg + fr * m2 + bb * mu;
    double acc = 0.0;
    for (int a = 0; a < mu; ++a) acc = fma(sG[a * q + j0], gf[a], acc);
    la[idx] = acc;
  }
  __syncthreads();
  // ---- per output component r: fields, three integrate_back contractions
  for (int r = 0; r < nc; ++r) {
    for (int idx = tid; idx < m3; idx += nt) {
      // row r of the point's three flux Jacobians (coalesced over the points from the regrouped copy)
      const double* d0 = s.dftr ? s.dftr + ((size_t(e) * nc + r) * 3 * m3 + idx) * nc
                                : s.dft + ((size_t(e) * 3 + 0) * m3 + idx) * nc * nc + r * nc;
      const double* d1 = s.dftr ? d0 + size_t(m3) * nc : s.dft + ((size_t(e) * 3 + 1) * m3 + idx) * nc * nc + r * nc;
      const double* d2 = s.dftr ? d1 + size_t(m3) * nc : s.dft + ((size_t(e) * 3 + 2) * m3 + idx) * nc * nc + r * nc;
      double f0 = 0.0, f1 = 0.0, f2 = 0.0;
      if (!s.small) {
        for (int c = 0; c < nc; ++c) {
          const double vc = sval[c * m3 + idx];
          f0 = fma(d0[c], vc, f0);
          f1 = fma(d1[c], vc, f1);
          f2 = fma(d2[c], vc, f2);
        }
      } else {
        const double vc = sval[r * m3 + idx];
        f0 = d0[r] * vc;
        f1 = d1[r] * vc;
        f2 = d2[r] * vc;
      }
      fM[idx] = s.a * s.jdet[size_t(e) * m3 + idx] * sval[r * m3 + idx];
      fM[m3 + idx] = s.b * f0;
      fM[2 * m3 + idx] = s.b * f1;
      fM[3 * m3 + idx] = s.b * f2;
    }
    __syncthreads();
    // x: Xa = GW M + DW F0 ; Xb = GW F1 ; Xc = GW F2
    for (int idx = tid; idx < m2 * q; idx += nt) {
      const int i = idx % q, gb = idx / q;  // gb = ga*mu + be
      const double* M = fM + gb * mu;
      double xa = 0.0, xb = 0.0, xc = 0.0;
      for (int al = 0; al < mu; ++al) {
        const double gw = sGW[i * mu + al];
        xa = fma(gw, M[al], fma(sDW[i * mu + al], M[m3 + al], xa));
        xb = fma(gw, M[2 * m3 + al], xb);
        xc = fma(gw, M[3 * m3 + al], xc);
      }
      Xa[idx] = xa;
      Xb[idx] = xb;
      Xc[idx] = xc;
    }
    __syncthreads();
    // y: Ya = GW Xa + DW Xb ; Yc = GW Xc
    for (int idx = tid; idx < mu * q2; idx += nt) {
      const int i = idx % q, j = (idx / q) % q, ga = idx / q2;
      double ya = 0.0, yc = 0.0;
      for (int be = 0; be < mu; ++be) {
        const int src = (ga * mu + be) * q + i;
        ya = fma(sGW[j * mu + be], Xa[src], fma(sDW[j * mu + be], Xb[src], ya));
        yc = fma(sGW[j * mu + be], Xc[src], yc);
      }
      Ya[idx] = ya;
      Yc[idx] = yc;
    }
    __syncthreads();
    // z: out = GW Ya + DW Yc
    for (int idx = tid; idx < q3; idx += nt) {
      const int ij = idx % q2, k = idx / q2;
      double acc = 0.0;
      for (int ga = 0; ga < mu; ++ga) acc = fma(sGW[k * mu + ga], Ya[ga * q2 + ij], fma(sDW[k * mu + ga], Yc[ga * q2 + ij], acc));
      sacc[r * q3 + idx] = acc;
    }
    __syncthreads();
  }
  // ---- face lifts (face_lift, ops/discretization.hpp:148-165): layer nodes only, gathered per node
  double* oe = vout + size_t(e) * nc * q3;
  for (int idx = tid; idx < nc * q3; idx += nt) {
    const int i = idx % q, j = (idx / q) % q, k = (idx / q2) % q, r = idx / q3;
    double acc = sacc[idx];
    const int pos[3] = {i, j, k};
    for (int axis = 0; axis < 3; ++axis) {
      const int p = pos[axis];
      if (p != 0 && p != q - 1) continue;
      const int f = 2 * axis + (p == 0 ? 0 : 1);
      const int j0 = pos[axis == 0 ? 1 : 0], j1 = pos[axis == 2 ? 1 : 2];
      const double* lf = la + ((f * nc + r) * q + j0) * mu;
      double sacc2 = 0.0;
      for (int bb = 0; bb < mu; ++bb) sacc2 = fma(sG[bb * q + j1], lf[bb], sacc2);
      acc += sacc2;
    }
    oe[idx] = acc;
  }
}

// ------------------------------------------------------------------------------------ 3D, sized
// Scalar 3D operator with compile-time (Q, MU), one CTA per element (persistent). Every stage is a
// set of independent 1D "pencil" contractions: a thread owns one pencil, keeps its accumulators in
// registers and reads the (broadcast) 1D weights from shared memory. The point-wise fields are
// formed inside the x-direction integration (never stored), and dead buffers are aliased, so an
// element needs ~11 K doubles of shared memory (cfg4) instead of ~24 K.
template <int Q, int MU>
struct Jv3dLayout {
  static constexpr int Q2 = Q * Q, Q3 = Q * Q * Q, M2 = MU * MU, M3 = MU * MU * MU;
  static constexpr int SLAB = (MU + 1) / 2;  // quadrature z-slabs per integration round
  static constexpr int w_G = 0, w_GW = MU * Q, w_DW = 2 * MU * Q, weights = 3 * MU * Q;
  // A: t1 + t2 (eval) | X for one slab group (3 SLAB MU Q)
  static constexpr int a_size = (Q2 * MU + Q * M2) > 3 * SLAB * MU * Q ? (Q2 * MU + Q * M2) : 3 * SLAB * MU * Q;
  // C: v (Q3) | traces str (12 M2) | Ya, Yc (2 MU Q2)
  static constexpr int c_a = Q3 > 12 * M2 ? Q3 : 12 * M2;
  static constexpr int c_size = c_a > 2 * MU * Q2 ? c_a : 2 * MU * Q2;
  static constexpr int val_size = M3 > 12 * Q * MU ? M3 : 12 * Q * MU;  // vals | trace stage 1
  static constexpr int r_a = weights, r_val = r_a + a_size, r_c = r_val + val_size, r_d = r_c + c_size;
  static constexpr int total = r_d + 6 * Q * MU + 6 * M2;  // D: lift stage wa (6 Q MU), face data sg (6 M2)
};

template <int Q, int MU>
__global__ void __launch_bounds__(256) jv3d_sized_kernel(DevSys s, const double* __restrict__ vin,
                                                          const double* __restrict__ halo, double* __restrict__ vout) {
  if (s.skip && *s.skip) return;
  using L = Jv3dLayout<Q, MU>;
  constexpr int Q2 = L::Q2, Q3 = L::Q3, M2 = L::M2, M3 = L::M3, SLAB = L::SLAB;
  constexpr int QH = (Q + 1) / 2;  // output halves per pencil in the integration stages
  extern __shared__ double sm[];
  double* G = sm + L::w_G;    // [a][j]
  double* GW = sm + L::w_GW;  // [j][a]
  double* DW = sm + L::w_DW;  // [j][a]
  double* t1 = sm + L::r_a;
  double* t2 = t1 + Q2 * MU;
  double* X = sm + L::r_a;
  double* val = sm + L::r_val;
  double* v = sm + L::r_c;
  double* str = sm + L::r_c;
  double* Ya = sm + L::r_c;
  double* Yc = Ya + MU * Q2;
  double* wa = sm + L::r_d;       // lift stage [f][j0][b]
  double* sg = wa + 6 * Q * MU;   // face data [f][b][a]
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < MU * Q; i += nt) {
    G[i] = s.g[i];
    GW[i] = s.gw[i];
    DW[i] = s.dw[i];
  }
  for (int e = s.e_lo + blockIdx.x; e < s.e_hi; e += gridDim.x) {
    __syncthreads();
    const double* ve = vin + size_t(e) * Q3;
    for (int i = tid; i < Q3; i += nt) v[i] = ve[i];
    __syncthreads();
    // ---- eval_at_quad, x pencils (k,j) -> t1[k][j][al]; trace stage 1 into val (free until z-eval)
    double* tw = val;  // [side][f][j1][a], 12 Q MU <= M3
    for (int p = tid; p < Q2 + 12 * Q; p += nt) {
      double acc[MU];
#pragma unroll
      for (int a = 0; a < MU; ++a) acc[a] = 0.0;
      if (p < Q2) {
        const double* row = v + p * Q;
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          const double x = row[i];
#pragma unroll
          for (int a = 0; a < MU; ++a) acc[a] = fma(G[a * Q + i], x, acc[a]);
        }
#pragma unroll
        for (int a = 0; a < MU; ++a) t1[p * MU + a] = acc[a];
      } else {
        const int idx = p - Q2, j1 = idx % Q, f = (idx / Q) % 6, side = idx / (6 * Q);
        const double* cf = v;
        int ff = f;
        bool ok = true;
        if (side == 1) {
          const int* fc = s.conn + (size_t(e) * 6 + f) * 3;
          ok = fc[0] >= 0;
          if (ok) {
            cf = nbr_block(s, vin, halo, fc[0]);
            ff = fc[1];
          }
        }
        if (ok)
          for (int j0 = 0; j0 < Q; ++j0) {
            const double x = cf[flat_face_node(Q, ff, j0, j1)];
#pragma unroll
            for (int a = 0; a < MU; ++a) acc[a] = fma(G[a * Q + j0], x, acc[a]);
          }
#pragma unroll
        for (int a = 0; a < MU; ++a) tw[(idx / Q) * Q * MU + j1 * MU + a] = acc[a];
      }
    }
    __syncthreads();
    // y pencils (k, al) -> t2[k][be][al]; trace stage 2 -> str[side][f][b][a] (over v, now dead)
    for (int p = tid; p < Q * MU + 12 * MU; p += nt) {
      double acc[MU];
#pragma unroll
      for (int b = 0; b < MU; ++b) acc[b] = 0.0;
      if (p < Q * MU) {
        const int k = p / MU, al = p % MU;
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          const double x = t1[(k * Q + j) * MU + al];
#pragma unroll
          for (int b = 0; b < MU; ++b) acc[b] = fma(G[b * Q + j], x, acc[b]);
        }
#pragma unroll
        for (int b = 0; b < MU; ++b) t2[(k * MU + b) * MU + al] = acc[b];
      } else {
        const int idx = p - Q * MU, a = idx % MU, sf = idx / MU;
        for (int j1 = 0; j1 < Q; ++j1) {
          const double x = tw[sf * Q * MU + j1 * MU + a];
#pragma unroll
          for (int b = 0; b < MU; ++b) acc[b] = fma(G[b * Q + j1], x, acc[b]);
        }
#pragma unroll
        for (int b = 0; b < MU; ++b) str[sf * M2 + b * MU + a] = acc[b];
      }
    }
    __syncthreads();
    // z pencils (be, al) -> vals[ga][be][al]; face data g[f][qf] (neighbour trace oriented)
    for (int p = tid; p < M2 + 6 * M2; p += nt) {
      if (p < M2) {
        double acc[MU];
#pragma unroll
        for (int g = 0; g < MU; ++g) acc[g] = 0.0;
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          const double x = t2[k * M2 + p];
#pragma unroll
          for (int g = 0; g < MU; ++g) acc[g] = fma(G[g * Q + k], x, acc[g]);
        }
#pragma unroll
        for (int g = 0; g < MU; ++g) val[g * M2 + p] = acc[g];
      } else {
        const int idx = p - M2, qf = idx % M2, f = idx / M2;
        const int* fc = s.conn + (size_t(e) * 6 + f) * 3;
        const size_t fq = (size_t(e) * 6 + f) * M2 + qf;
        const int qa = qf % MU, qb = qf / MU, code = fc[2];
        int u = (code & 4) ? qb : qa, w = (code & 4) ? qa : qb;
        if (code & 1) u = MU - 1 - u;
        if (code & 2) w = MU - 1 - w;
        const double tm = str[f * M2 + qf], tp = str[(6 + f) * M2 + w * MU + u];
        sg[idx] = -s.b * s.face_w[fq] * fma(s.dfm[fq], tm, s.dfp[fq] * tp);
      }
    }
    __syncthreads();
    // lift stage 1: wa[f][j0][b] = sum_a G(a, j0) g[f][b][a]
    for (int idx = tid; idx < 6 * MU; idx += nt) {
      const int b = idx % MU, f = idx / MU;
      double acc[Q];
#pragma unroll
      for (int j = 0; j < Q; ++j) acc[j] = 0.0;
      for (int a = 0; a < MU; ++a) {
        const double x = sg[f * M2 + b * MU + a];
#pragma unroll
        for (int j = 0; j < Q; ++j) acc[j] = fma(G[a * Q + j], x, acc[j]);
      }
#pragma unroll
      for (int j = 0; j < Q; ++j) wa[(f * Q + j) * MU + b] = acc[j];
    }
    // ---- integration in rounds of SLAB quadrature z-slabs: fields + x (into X), then y (into Ya, Yc)
    const double* jd = s.jdet + size_t(e) * M3;
    const double* d0 = s.dft + size_t(e) * 3 * M3;
    const double* d1 = d0 + M3;
    const double* d2 = d1 + M3;
    for (int g0 = 0; g0 < MU; g0 += SLAB) {
      const int ng = MU - g0 < SLAB ? MU - g0 : SLAB;
      for (int p = tid; p < ng * MU * 2; p += nt) {  // pencil (ga, be), half h of the outputs i
        const int hh = p % 2, pb = p / 2, ga = g0 + pb / MU, be = pb % MU;
        const int i0 = hh * QH, ni = hh == 0 ? QH : Q - QH;
        double xa[QH], xb[QH], xc[QH];
#pragma unroll
        for (int i = 0; i < QH; ++i) xa[i] = xb[i] = xc[i] = 0.0;
        for (int al = 0; al < MU; ++al) {
          const int qv = (ga * MU + be) * MU + al;
          const double x = val[qv];
          const double fm = s.a * jd[qv] * x, f0 = s.b * (d0[qv] * x), f1 = s.b * (d1[qv] * x),
                       f2 = s.b * (d2[qv] * x);
#pragma unroll
          for (int i = 0; i < QH; ++i) {
            if (i < ni) {
              const double gw = GW[(i0 + i) * MU + al];
              xa[i] = fma(gw, fm, fma(DW[(i0 + i) * MU + al], f0, xa[i]));
              xb[i] = fma(gw, f1, xb[i]);
              xc[i] = fma(gw, f2, xc[i]);
            }
          }
        }
        const int row = (pb)*Q + i0;  // X[(ga-g0)][be][i]
#pragma unroll
        for (int i = 0; i < QH; ++i)
          if (i < ni) {
            X[row + i] = xa[i];
            X[SLAB * MU * Q + row + i] = xb[i];
            X[2 * SLAB * MU * Q + row + i] = xc[i];
          }
      }
      __syncthreads();
      for (int p = tid; p < ng * Q * 2; p += nt) {  // pencil (ga, i), half of the outputs j
        const int hh = p % 2, pb = p / 2, gl = pb / Q, i = pb % Q, ga = g0 + gl;
        const int j0 = hh * QH, nj = hh == 0 ? QH : Q - QH;
        double ya[QH], yc[QH];
#pragma unroll
        for (int j = 0; j < QH; ++j) ya[j] = yc[j] = 0.0;
        for (int be = 0; be < MU; ++be) {
          const int src = (gl * MU + be) * Q + i;
          const double xa = X[src], xb = X[SLAB * MU * Q + src], xc = X[2 * SLAB * MU * Q + src];
#pragma unroll
          for (int j = 0; j < QH; ++j)
            if (j < nj) {
              ya[j] = fma(GW[(j0 + j) * MU + be], xa, fma(DW[(j0 + j) * MU + be], xb, ya[j]));
              yc[j] = fma(GW[(j0 + j) * MU + be], xc, yc[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < QH; ++j)
          if (j < nj) {
            Ya[(ga * Q + j0 + j) * Q + i] = ya[j];
            Yc[(ga * Q + j0 + j) * Q + i] = yc[j];
          }
      }
      __syncthreads();
    }
    // z integration, pencils (j, i) + face lifts, straight to HBM
    double* oe = vout + size_t(e) * Q3;
    for (int p = tid; p < Q2; p += nt) {
      double acc[Q];
#pragma unroll
      for (int k = 0; k < Q; ++k) acc[k] = 0.0;
      for (int ga = 0; ga < MU; ++ga) {
        const double ya = Ya[ga * Q2 + p], yc = Yc[ga * Q2 + p];
#pragma unroll
        for (int k = 0; k < Q; ++k) acc[k] = fma(GW[k * MU + ga], ya, fma(DW[k * MU + ga], yc, acc[k]));
      }
      const int i = p % Q, j = p / Q;
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        double r = acc[k];
        const int pos[3] = {i, j, k};
#pragma unroll
        for (int axis = 0; axis < 3; ++axis) {
          const int pp = pos[axis];
          if (pp != 0 && pp != Q - 1) continue;
          const int f = 2 * axis + (pp == 0 ? 0 : 1);
          const int j0 = pos[axis == 0 ? 1 : 0], j1 = pos[axis == 2 ? 1 : 2];
          const double* lf = wa + (f * Q + j0) * MU;
          double s2 = 0.0;
          for (int bb = 0; bb < MU; ++bb) s2 = fma(G[bb * Q + j1], lf[bb], s2);
          r += s2;
        }
        oe[k * Q2 + p] = r;
      }
    }
  }
}

template <int Q, int MU>
bool try_jv3d_sized(const DevSys& s, const double* vin, const double* halo, double* vout, cudaStream_t st) {
  if (s.dim != 3 || s.n_c != 1 || s.q != Q || s.mu != MU) return false;
  const size_t smem = sizeof(double) * size_t(Jv3dLayout<Q, MU>::total);
  ensure_smem(jv3d_sized_kernel<Q, MU>, smem, true);
  static int grid = 0;
  if (!grid) {
    int per_sm = 0, dev = 0, sms = 0;
    TPDG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jv3d_sized_kernel<Q, MU>, 256, smem));
    TPDG_CUDA_CHECK(cudaGetDevice(&dev));
    TPDG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = std::max(1, per_sm) * sms;
  }
  jv3d_sized_kernel<Q, MU><<<std::min(grid, s.e_hi - s.e_lo), 256, smem, st>>>(s, vin, halo, vout);
  return true;
}

bool launch_jv3d_sized(const DevSys& s, const double* vin, const double* halo, double* vout, cudaStream_t st) {
  return try_jv3d_sized<4, 5>(s, vin, halo, vout, st) || try_jv3d_sized<5, 6>(s, vin, halo, vout, st) ||
         try_jv3d_sized<8, 9>(s, vin, halo, vout, st) || try_jv3d_sized<11, 12>(s, vin, halo, vout, st);
}

size_t jv3d_smem(const DevSys& s) {
  const size_t q = s.q, mu = s.mu, nc = s.n_c;
  const size_t q3 = q * q * q, m3 = mu * mu * mu, m2 = mu * mu, q2 = q * q;
  const size_t eval = nc * q2 * mu + nc * q * m2;
  const size_t per_r = 4 * m3 + 3 * m2 * q + 2 * mu * q2 + 12 * nc * m2 + 12 * nc * q * mu + 6 * nc * m2 + nc * q3;
  return sizeof(double) * (3 * mu * q + nc * q3 + nc * m3 + (eval > per_r ? eval : per_r));
}

} // namespace

size_t jv_smem_bytes(const DevSys& s) { return s.dim == 2 ? jv2d_smem(s) : jv3d_smem(s); }

namespace {
template <typename K>
void launch_generic(K kernel, int nt, size_t smem, const DevSys& s, const double* vin, const double* halo,
                    double* vout, cudaStream_t st) {
  ensure_smem(kernel, smem);
  kernel<<<s.e_hi - s.e_lo, nt, smem, st>>>(s, vin, halo, vout);
}
}  // namespace

void launch_jv(const DevSys& s, const double* vin, const double* halo, double* vout, cudaStream_t st) {
  if (s.e_hi <= s.e_lo) return;
  const size_t smem = jv_smem_bytes(s);
  if (s.dim == 2 && (launch_jv2d_mma(s, vin, halo, vout, st) || launch_jv2d_sized(s, vin, halo, vout, st))) {
    TPDG_CUDA_CHECK(cudaGetLastError());
    ++g_launches;
    return;
  }
  if (s.dim == 3 && (launch_jv3d_fast(s, vin, halo, vout, st) || launch_jv3d_sized(s, vin, halo, vout, st))) {
    TPDG_CUDA_CHECK(cudaGetLastError());
    ++g_launches;
    return;
  }
  // generic (runtime-size) kernels, one CTA per element; systems (n_c > 1) use wider CTAs: their
  // shared-memory footprint allows one or two CTAs per SM, so the stages need more threads
  // (instances with compile-time sizes for the BASELINE systems: cfg3 2D n_c = 4, q = 16; cfg5 3D n_c = 5, q = 8)
  const bool full = !s.small;
  if (s.dim == 2) {
    if (full && s.n_c == 4 && s.q == 16 && s.mu == 17)
      launch_generic(jv2d_kernel<512, 4, 16, 17>, 512, smem, s, vin, halo, vout, st);
    else if (s.n_c > 1) launch_generic(jv2d_kernel<512>, 512, smem, s, vin, halo, vout, st);
    else launch_generic(jv2d_kernel<256>, 256, smem, s, vin, halo, vout, st);
  } else {
    if (full && s.n_c == 5 && s.q == 8 && s.mu == 9)
      launch_generic(jv3d_kernel<1024, 5, 8, 9>, 1024, smem, s, vin, halo, vout, st);
    else if (s.n_c > 1) launch_generic(jv3d_kernel<1024>, 1024, smem, s, vin, halo, vout, st);
    else launch_generic(jv3d_kernel<256>, 256, smem, s, vin, halo, vout, st);
  }
  TPDG_CUDA_CHECK(cudaGetLastError());
  ++g_launches;
}

} // namespace tpdg_gpu
