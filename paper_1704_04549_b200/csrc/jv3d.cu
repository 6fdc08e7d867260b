// 3D scalar matrix-free operator (a M + b J) v, sum-factorized, constant-bank weights.
//
// Restates jacobian_apply for dim = 3, n_c = 1 (reference ops/linearized.hpp:201-240):
// element_diag_apply (:107-162: eval_at_quad kernels.hpp:60-78, the mass and contravariant-flux
// fields, integrate_back kernels.hpp:82-104, the own-trace face terms) plus the neighbour
// coupling through dfp (:216-236), with face_trace / face_lift / neighbor_trace from
// ops/discretization.hpp:89-181.
//
// B200 design (cfg4: q = 11, mu = 12, 4096 elements, 370 MB and 2.8 GFLOP per launch at the
// SURVEY.md sec.8d accounting, FP64-bound on the CUDA cores):
//  * The three 1D matrices (G, G^T W, D^T W) live in constant memory; every contraction is fully
//    unrolled over compile-time (Q, MU), so each DFMA takes its weight as a uniform register
//    loaded by LDCU right before it (no per-thread weight registers, no shared-memory weight
//    traffic). The only shared-memory traffic is the pencil input, one LDS per MU (or Q) DFMAs.
//  * One 160-thread CTA per element (persistent grid, 3 CTAs per SM); each stage is a set of
//    independent 1D pencil contractions, one pencil per thread, accumulators in registers.
//  * Integration is factored so that the (d + 2) reference transforms share their stages:
//      z: A1 = Gz fm + Dz f2, A2 = Gz f0, A3 = Gz f1      (pencil = quadrature column (beta, alpha))
//      y: S1 = Gy A1 + Dy A3, S2 = Gy A2                 (pencil (k, alpha))
//      x: out = Gx S1 + Dx S2                            (pencil (k, j)) + face lifts
//    The z stage is fused with the last eval stage and the point-wise fields: the quadrature
//    values of a column never leave registers. A and S overwrite their inputs per thread (a thread
//    reads its whole column before writing its own outputs into the same slots).
//  * Face data arrive pre-scaled (cdfm = -b fw dfm, cdfp = -b fw dfp) and the point-wise coefficients
//    interleaved per quadrature point (pw = [a jdet, b dft_x, b dft_y, b dft_z], two 16-byte loads),
//    both folded once at op_create.
//  * Latency: the next element's operator data are prefetched into L2 with bulk prefetches
//    (cp.async.bulk.prefetch.L2, the TMA unit) one element ahead, and its v and neighbour face
//    layers are copied into shared memory with cp.async during the current element's last two
//    stages (shared-memory regions are reused by liveness: X1 t1|tw -> A, X2 t2|str -> next v).
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "tpdg_internal.hpp"

namespace tpdg_gpu {

namespace {

// The 1D matrices of each (Q, MU) instance in constant memory: slot s holds G (mu x q, G(a, j) at
// a Q + j, reference_element.hpp:24-27), G^T W (q x mu, at i MU + a) and D^T W (q x mu).
constexpr int kJv3dSlots = 5, kJv3dSlotLen = 3 * 12 * 11;
__constant__ double c_jv3d[kJv3dSlots][kJv3dSlotLen];

// One weight from constant memory. The asm volatile keeps the load next to its use: ptxas then
// emits LDCU (uniform datapath) + a DFMA with a uniform-register operand, instead of hoisting all
// the weights out of the loops into ~150 regular registers (what it does for plain array reads).
__device__ __forceinline__ double cld(const double* p) {
  double r;
  asm volatile("{\n\t.reg .u64 t;\n\tcvta.to.const.u64 t, %1;\n\tld.const.f64 %0, [t];\n\t}" : "=d"(r) : "l"(p));
  return r;
}

template <int SLOT, int Q, int MU>
struct Jv3dW {
  __device__ __forceinline__ static double G(int i) { return cld(&c_jv3d[SLOT][i]); }
  __device__ __forceinline__ static double GW(int i) { return cld(&c_jv3d[SLOT][MU * Q + i]); }
  __device__ __forceinline__ static double DW(int i) { return cld(&c_jv3d[SLOT][2 * MU * Q + i]); }
};

template <int Q, int MU>
struct Jv3dLayout {
  static constexpr int Q2 = Q * Q, Q3 = Q * Q * Q, M2 = MU * MU, M3 = MU * MU * MU;
  static constexpr int cmax(int a, int b) { return a > b ? a : b; }
  // Regions reused by liveness (doubles):
  //   X1: t1 | tw (E1-E2), then A1 | A2 | A3 (E3-E4; S1, S2 over A1, A2 until E5)
  //   X2: t2 | str (E2-E3), then the next element's v | neighbour face layers (cp.async, E4 -> E1)
  //   X3: lifted face data wa (E3-E5)
  // Rows of MU entries that consecutive lanes read or write one row apart (t1 / tw stores, str, wa and
  // S loads) are MP = MU | 1 doubles apart: an odd stride spreads the 16 lanes of a 64-bit wavefront
  // over all banks (stride 12 was a 4-way conflict).
  static constexpr int MP = MU | 1;
  static constexpr int t1 = 0, tw = Q2 * MP, A1 = 0, A2 = Q * M2, A3 = 2 * Q * M2;
  static constexpr int x1 = cmax(3 * Q * M2, Q2 * MP + 12 * Q * MP);
  static constexpr int t2 = x1, str = t2 + Q * M2, v = x1, nbl = v + Q3;
  static constexpr int x2 = cmax(Q * M2 + 12 * MU * MP, Q3 + 6 * Q2);
  static constexpr int wa = x1 + x2;
  static constexpr int total = wa + 6 * Q * MP;
  // X2 tail (free while the next element's v | neighbour layers travel, E4 -> E1): a shared copy of G
  // and the lifted face contributions lift[f][j1][j0] (E5a), read by the x-integration pencils (E5b)
  static constexpr int sg = v + Q3 + 6 * Q2, lift = sg + MU * Q;
  static_assert(lift + 6 * Q2 <= x1 + x2, "X2 tail too small for the lifted face layers");
};

__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  // TMA-unit bulk prefetch into L2 (16-byte granularity)
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const unsigned b = (bytes + 15 + unsigned(reinterpret_cast<uintptr_t>(p) & 15)) & ~15u;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(b) : "memory");
}

template <int Q>
__device__ __forceinline__ int face_node(int f, int j0, int j1) {
  // node of a face layer (face_trace, discretization.hpp:89-129): axis f/2 fixed at 0 or Q-1, the
  // tangential axes in face_param_axes order (mesh.hpp:45-50)
  const int axis = f >> 1, layer = (f & 1) ? Q - 1 : 0;
  const int i = axis == 0 ? layer : j0;
  const int j = axis == 1 ? layer : (axis == 0 ? j0 : j1);
  const int k = axis == 2 ? layer : j1;
  return (k * Q + j) * Q + i;
}

template <int Q, int MU>
__device__ __forceinline__ void prefetch_element(const DevSys& s, const double* __restrict__ vin, int e) {
  constexpr int Q3 = Q * Q * Q, M2 = MU * MU, M3 = MU * MU * MU;
  const int t = threadIdx.x;
  if (t == 0) prefetch_l2(s.pw + size_t(e) * 4 * M3, 2 * M3 * 8);
  if (t == 32) prefetch_l2(s.pw + size_t(e) * 4 * M3 + 2 * M3, 2 * M3 * 8);
  if (t == 64) prefetch_l2(s.cdfm + size_t(e) * 6 * M2, 6 * M2 * 8);
  if (t == 96) prefetch_l2(s.cdfp + size_t(e) * 6 * M2, 6 * M2 * 8);
  if (t == 128) prefetch_l2(vin + size_t(e) * Q3, Q3 * 8);
}

__device__ __forceinline__ void cp8(double* smem, const double* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// v of element e and its six neighbour face layers (in the neighbour's own (j0, j1) enumeration) into
// shared memory, asynchronously (LDGSTS); boundary faces are zero-filled.
template <int Q, int NT>
__device__ __forceinline__ void load_element_async(const DevSys& s, const double* __restrict__ vin,
                                                   const double* __restrict__ halo, int e, double* sv, double* snb) {
  constexpr int Q2 = Q * Q, Q3 = Q * Q * Q;
  const double* ve = vin + size_t(e) * Q3;
  for (int i = threadIdx.x; i < Q3; i += NT) cp8(sv + i, ve + i);
  for (int i = threadIdx.x; i < 6 * Q2; i += NT) {
    const int f = i / Q2, r = i % Q2, j0 = r / Q, j1 = r % Q;
    const int* fc = s.conn + (size_t(e) * 6 + f) * 3;
    if (fc[0] >= 0) {
      const double* nb = fc[0] < s.n_local ? vin + size_t(fc[0]) * Q3 : halo + size_t(fc[0] - s.n_local) * Q3;
      cp8(snb + f * Q2 + j0 * Q + j1, nb + face_node<Q>(fc[1], j0, j1));
    } else {
      snb[f * Q2 + j0 * Q + j1] = 0.0;
    }
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

template <int SLOT, int Q, int MU, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) jv3d_fast_kernel(DevSys s, const double* __restrict__ vin,
                                                           const double* __restrict__ halo,
                                                           double* __restrict__ vout) {
  if (s.skip && *s.skip) return;
  using L = Jv3dLayout<Q, MU>;
  using W = Jv3dW<SLOT, Q, MU>;
  constexpr int Q2 = L::Q2, Q3 = L::Q3, M2 = L::M2, M3 = L::M3;
  extern __shared__ double sm[];
  const int tid = threadIdx.x;
  if (s.e_lo + int(blockIdx.x) < s.e_hi) {
    prefetch_element<Q, MU>(s, vin, s.e_lo + blockIdx.x);
    load_element_async<Q, NT>(s, vin, halo, s.e_lo + blockIdx.x, sm + L::v, sm + L::nbl);
  }
  for (int e = s.e_lo + blockIdx.x; e < s.e_hi; e += gridDim.x) {
    const int e_next = e + int(gridDim.x);
    if (e_next < s.e_hi) prefetch_element<Q, MU>(s, vin, e_next);
    // ---- E0: this element's v and neighbour layers (cp.async issued during the previous element's E4)
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    // ---- E1: eval x pencils (k, j) -> t1[k][j][al]; trace stage 1: tw[sf][j1][a] = sum_j0 G(a, j0) layer(j0, j1)
    for (int p = tid; p < Q2 + 12 * Q; p += NT) {
      double x[Q];
      double* dst;
      if (p < Q2) {
#pragma unroll
        for (int i = 0; i < Q; ++i) x[i] = sm[L::v + p * Q + i];
        dst = sm + L::t1 + p * L::MP;
      } else {
        const int idx = p - Q2, j1 = idx % Q, sf = idx / Q, f = sf % 6;
        if (sf < 6) {
#pragma unroll
          for (int j0 = 0; j0 < Q; ++j0) x[j0] = sm[L::v + face_node<Q>(f, j0, j1)];
        } else {
#pragma unroll
          for (int j0 = 0; j0 < Q; ++j0) x[j0] = sm[L::nbl + f * Q2 + j0 * Q + j1];
        }
        dst = sm + L::tw + (sf * Q + j1) * L::MP;
      }
#pragma unroll
      for (int al = 0; al < MU; ++al) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < Q; ++i) acc = fma(W::G(al * Q + i), x[i], acc);
        dst[al] = acc;
      }
    }
    __syncthreads();
    // ---- E2: eval y pencils (k, al) -> t2[k][be][al]; trace stage 2: str[sf][b][a]
    for (int p = tid; p < Q * MU + 12 * MU; p += NT) {
      double x[Q];
      if (p < Q * MU) {
        const int k = p / MU, al = p % MU;
#pragma unroll
        for (int j = 0; j < Q; ++j) x[j] = sm[L::t1 + (k * Q + j) * L::MP + al];
#pragma unroll
        for (int be = 0; be < MU; ++be) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < Q; ++j) acc = fma(W::G(be * Q + j), x[j], acc);
          sm[L::t2 + (k * MU + be) * MU + al] = acc;
        }
      } else {
        const int idx = p - Q * MU, a = idx % MU, sf = idx / MU;
#pragma unroll
        for (int j1 = 0; j1 < Q; ++j1) x[j1] = sm[L::tw + (sf * Q + j1) * L::MP + a];
#pragma unroll
        for (int b = 0; b < MU; ++b) {
          double acc = 0.0;
#pragma unroll
          for (int j1 = 0; j1 < Q; ++j1) acc = fma(W::G(b * Q + j1), x[j1], acc);
          sm[L::str + (sf * MU + b) * L::MP + a] = acc;
        }
      }
    }
    __syncthreads();
    // ---- E3: face lifts (pencils (f, b), first) and the quadrature columns (be, al):
    //      eval z + point-wise fields + z integration, all in registers
    for (int p = tid; p < 6 * MU + M2; p += NT) {
      if (p < 6 * MU) {
        // face data g = -b fw (dfm t^- + dfp t^+) (discretization.hpp:133-181, linearized.hpp:143-161,
        // 216-236) at the points (a, b) of face f, then wa[f][j][b] = sum_a G(a, j) g(a, b)
        const int f = p / MU, b = p % MU;
        const int code = s.conn[(size_t(e) * 6 + f) * 3 + 2];
        const double* cm = s.cdfm + (size_t(e) * 6 + f) * M2 + b * MU;
        const double* cp = s.cdfp + (size_t(e) * 6 + f) * M2 + b * MU;
        double g[MU];
#pragma unroll
        for (int a = 0; a < MU; ++a) {
          int u = (code & 4) ? b : a, w = (code & 4) ? a : b;  // orient_face_coords (mesh.hpp:57-67)
          if (code & 1) u = MU - 1 - u;
          if (code & 2) w = MU - 1 - w;
          const double tm = sm[L::str + (f * MU + b) * L::MP + a], tp = sm[L::str + ((6 + f) * MU + w) * L::MP + u];
          g[a] = fma(__ldg(cm + a), tm, __ldg(cp + a) * tp);
        }
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          double acc = 0.0;
#pragma unroll
          for (int a = 0; a < MU; ++a) acc = fma(W::G(a * Q + j), g[a], acc);
          sm[L::wa + (f * Q + j) * L::MP + b] = acc;
        }
      } else {
        const int c = p - 6 * MU;  // column (be, al) = c
        double x[Q];
#pragma unroll
        for (int k = 0; k < Q; ++k) x[k] = sm[L::t2 + k * M2 + c];
        // point-wise coefficients (a jdet, b dft_x, b dft_y, b dft_z) interleaved per quadrature point
        const double2* pw = reinterpret_cast<const double2*>(s.pw + (size_t(e) * M3 + c) * 4);
        double A1[Q], A2[Q], A3[Q];
#pragma unroll
        for (int k = 0; k < Q; ++k) A1[k] = A2[k] = A3[k] = 0.0;
#pragma unroll
        for (int ga = 0; ga < MU; ++ga) {
          double val = 0.0;
#pragma unroll
          for (int k = 0; k < Q; ++k) val = fma(W::G(ga * Q + k), x[k], val);
          const double2 c01 = __ldg(pw + 2 * ga * M2), c23 = __ldg(pw + 2 * ga * M2 + 1);
          const double fm = c01.x * val;  // mass field a jdet u
          const double f0 = c01.y * val;  // b (adjugate-contracted flux Jacobian)_x u
          const double f1 = c23.x * val;
          const double f2 = c23.y * val;
#pragma unroll
          for (int k = 0; k < Q; ++k) {
            const double gw = W::GW(k * MU + ga);
            A1[k] = fma(gw, fm, fma(W::DW(k * MU + ga), f2, A1[k]));
            A2[k] = fma(gw, f0, A2[k]);
            A3[k] = fma(gw, f1, A3[k]);
          }
        }
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          sm[L::A1 + k * M2 + c] = A1[k];
          sm[L::A2 + k * M2 + c] = A2[k];
          sm[L::A3 + k * M2 + c] = A3[k];
        }
      }
    }
    __syncthreads();
    // the next element's v and neighbour layers travel during E4 / E5 (X2 is free from here on)
    if (e_next < s.e_hi) load_element_async<Q, NT>(s, vin, halo, e_next, sm + L::v, sm + L::nbl);
    // ---- E4: y integration, pencils (k, al): S1 = Gy A1 + Dy A3 (-> A1 slots), S2 = Gy A2 (-> A2 slots);
    //      the threads without a pencil stage G in shared memory for E5a
    for (int p = Q * MU + (tid - Q * MU); tid >= Q * MU && p < Q * MU + MU * Q; p += NT - Q * MU)
      sm[L::sg + p - Q * MU] = W::G(p - Q * MU);
    for (int p = tid; p < Q * MU; p += NT) {
      const int k = p / MU, al = p % MU;
      const int base = k * M2 + al;
      double x1[MU], x2[MU], x3[MU];
#pragma unroll
      for (int be = 0; be < MU; ++be) {
        x1[be] = sm[L::A1 + base + be * MU];
        x2[be] = sm[L::A2 + base + be * MU];
        x3[be] = sm[L::A3 + base + be * MU];
      }
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        double s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int be = 0; be < MU; ++be) {
          const double gw = W::GW(j * MU + be);
          s1 = fma(gw, x1[be], fma(W::DW(j * MU + be), x3[be], s1));
          s2 = fma(gw, x2[be], s2);
        }
        sm[L::A1 + base + j * MU] = s1;
        sm[L::A2 + base + j * MU] = s2;
      }
    }
    __syncthreads();
    // ---- E5a: second stage of the face lifts (face_lift, discretization.hpp:133-166), spread over all
    //      threads: lift[f][j1][j0] = sum_bb G(bb, j1) wa[f][j0][bb]
    for (int it = tid; it < 6 * Q2; it += NT) {
      const int f = it / Q2, j1 = (it % Q2) / Q, j0 = it % Q;
      const double* w = sm + L::wa + (f * Q + j0) * L::MP;
      double l = 0.0;
#pragma unroll
      for (int bb = 0; bb < MU; ++bb) l = fma(sm[L::sg + bb * Q + j1], w[bb], l);
      sm[L::lift + it] = l;
    }
    __syncthreads();
    // ---- E5b: x integration, pencils (k, j): out = Gx S1 + Dx S2, plus the lifted layers, straight to HBM
    for (int p = tid; p < Q2; p += NT) {
      const int k = p / Q, j = p % Q;
      const int base = k * M2 + j * MU;
      double x1[MU], x2[MU];
      if constexpr (MU % 2 == 0) {  // rows are 16-byte aligned: 16-byte loads halve the cost of the stride-MU bank conflict
#pragma unroll
        for (int al = 0; al < MU; al += 2) {
          const double2 a = *reinterpret_cast<const double2*>(sm + L::A1 + base + al);
          const double2 b = *reinterpret_cast<const double2*>(sm + L::A2 + base + al);
          x1[al] = a.x, x1[al + 1] = a.y, x2[al] = b.x, x2[al + 1] = b.y;
        }
      } else {
#pragma unroll
        for (int al = 0; al < MU; ++al) {
          x1[al] = sm[L::A1 + base + al];
          x2[al] = sm[L::A2 + base + al];
        }
      }
      // lifted layers of the faces whose layer contains the whole pencil (y, z faces), tangential (i, k) / (i, j)
      const double* ly = (j == 0) ? sm + L::lift + 2 * Q2 + k * Q : (j == Q - 1 ? sm + L::lift + 3 * Q2 + k * Q : nullptr);
      const double* lz = (k == 0) ? sm + L::lift + 4 * Q2 + j * Q : (k == Q - 1 ? sm + L::lift + 5 * Q2 + j * Q : nullptr);
      double* oe = vout + size_t(e) * Q3 + p * Q;
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int al = 0; al < MU; ++al) acc = fma(W::GW(i * MU + al), x1[al], fma(W::DW(i * MU + al), x2[al], acc));
        if (ly) acc += ly[i];  // face 2/3: (j0, j1) = (i, k)
        if (lz) acc += lz[i];  // face 4/5: (j0, j1) = (i, j)
        if (i == 0 || i == Q - 1) acc += sm[L::lift + (i == 0 ? 0 : 1) * Q2 + k * Q + j];  // face 0/1: (j0, j1) = (j, k)
        oe[i] = acc;
      }
    }
    __syncthreads();
  }
}

template <int SLOT, int Q, int MU, int MINB = 3>
bool try_jv3d_fast(const DevSys& s, const double* vin, const double* halo, double* vout, cudaStream_t st) {
  static_assert(SLOT < kJv3dSlots && 3 * MU * Q <= kJv3dSlotLen, "constant slot too small");
  if (s.dim != 3 || s.n_c != 1 || s.q != Q || s.mu != MU || !s.cdfm || !s.pw || !s.hg) return false;
  constexpr int NT = 160;
  constexpr int kMaxDev = 16;
  const size_t smem = sizeof(double) * size_t(Jv3dLayout<Q, MU>::total);
  static int grid[kMaxDev] = {0};
  static double loaded[kMaxDev][3 * MU * Q];
  static bool has[kMaxDev] = {false};
  static std::mutex mu;
  int dev = 0;
  TPDG_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDev) return false;
  double w[3 * MU * Q];
  std::copy(s.hg, s.hg + MU * Q, w);
  std::copy(s.hgw, s.hgw + MU * Q, w + MU * Q);
  std::copy(s.hdw, s.hdw + MU * Q, w + 2 * MU * Q);
  ensure_smem(jv3d_fast_kernel<SLOT, Q, MU, NT, MINB>, smem);
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!grid[dev]) {
      int per_sm = 0, sms = 0;
      TPDG_CUDA_CHECK(
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jv3d_fast_kernel<SLOT, Q, MU, NT, MINB>, NT, smem));
      TPDG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      grid[dev] = std::max(1, per_sm) * sms;
    }
    // the reference element's matrices of this (Q, MU) into the instance's constant slot, stream-ordered
    // before the launch; re-uploaded only when an operator with different matrices uses the slot
    if (!has[dev] || !std::equal(w, w + 3 * MU * Q, loaded[dev])) {
      TPDG_CUDA_CHECK(cudaMemcpyToSymbolAsync(c_jv3d, w, sizeof(w), sizeof(double) * SLOT * kJv3dSlotLen,
                                              cudaMemcpyHostToDevice, st));
      TPDG_CUDA_CHECK(cudaStreamSynchronize(st));  // w is a stack buffer
      std::copy(w, w + 3 * MU * Q, loaded[dev]);
      has[dev] = true;
    }
  }
  jv3d_fast_kernel<SLOT, Q, MU, NT, MINB><<<std::min(grid[dev], s.e_hi - s.e_lo), NT, smem, st>>>(s, vin, halo, vout);
  return true;
}

}  // namespace

bool launch_jv3d_fast(const DevSys& s, const double* vin, const double* halo, double* vout, cudaStream_t st) {
  return try_jv3d_fast<0, 11, 12>(s, vin, halo, vout, st) || try_jv3d_fast<1, 5, 6>(s, vin, halo, vout, st) ||
         try_jv3d_fast<2, 8, 9>(s, vin, halo, vout, st) || try_jv3d_fast<3, 4, 5>(s, vin, halo, vout, st) ||
         try_jv3d_fast<4, 3, 4>(s, vin, halo, vout, st);
}

}  // namespace tpdg_gpu
