// Bit-faithful 2D Kronecker apply, several blocks per warp (n_c = 1: n1 = n2 = N = q).
//
// apply_factors_2d (reference precond/ksvd.hpp:112-129) for the scalar 2D configurations
// (BASELINE cfg1, cfg2 at p = 4 ... 30): LU axis solves (ops/kernels.hpp:36-51 with
// LuFactor::solve, tensor/small_matrix.hpp:177-187), rotation to Schur coordinates
// M = Q1^T X Q2 (matmul, :103-113), the quasi-triangular Sylvester solve T1 Y + Y T2^T = M
// (tensor/sylvester.hpp:72-127) and the rotation back X = Q1 Y Q2^T. Every value is formed with
// the reference's operations in the reference's order (faithful.cuh: separate mul / add
// roundings, ascending summation, correctly rounded divisions), so with the reference's LU and
// Schur factors the result equals the reference's bit for bit
// (tests/test_gpu_full_pc_parity.py); parallelism is only across independent values.
//
// Layout: EW = 32 / N blocks per warp (N lanes each), so all phases keep the lanes busy:
//   * LU phase: lane = one column fiber, then one row fiber of its block (register fibers);
//   * rotations: lane = a TI x TJ tile of its block's N x N product;
//   * Sylvester: lane = one cell (quasi-block pair) of the current block anti-diagonal; the lane
//     forms the right-hand sides of the cell's <= 4 entries together (shared T / Y loads, four
//     independent chains) and replays the cell's factored tiny system (sylv_cells_kernel).
// Shared memory per block: R1 = LU(A2) | LU(B1) -> P (product scratch) -> T1 | T2 -> P,
// X (ld = N + 3: conflict-free fibers and anti-diagonal accesses), pivots,
// reciprocal pivots and the Sylvester plan. T1 / T2 and the cell factors are prefetched to L2 at
// the start and copied in after the first rotation.
#include <cstdint>

#include "faithful.cuh"
#include "tpdg_internal.hpp"

namespace tpdg_gpu {

namespace {

__device__ __forceinline__ void cpa8(double* smem, const double* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cpa16(double* smem, const double* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cpa4(int* smem, const int* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// LEN contiguous doubles global -> shared by the N lanes of one block: 16-byte copies when both
// ends are aligned (even N: every offset used here is even), else 8-byte copies.
template <int LEN, int N, int P>
__device__ __forceinline__ void copy_mat(double* dst, const double* src, int li) {
  if ((N & 1) == 0 && ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    for (int i = 2 * li; i < LEN; i += 2 * P) cpa16(dst + i, src + i);
  } else {
    for (int i = li; i < LEN; i += P) cpa8(dst + i, src + i);
  }
}

constexpr int kEwBigN = 24;     // N above which the kernel may use up to 254 registers (8 warps per SM)
constexpr int kEwLdPad = 3;     // X row padding
constexpr int kEw16Lanes = 16;  // lanes per block at N = 16 (2 blocks per warp); 8 (4 per warp) measured 114 vs 91 us

template <int N, int P = N>  // P lanes per block
struct Ew {
  static constexpr int EW = 32 / P;  // blocks per warp
  // X leading dimension. The Sylvester wavefront's lanes sit on an anti-diagonal of X, one quasi-block apart:
  // consecutive lanes' right-hand-side loads are (LD - 1) doubles apart for 1 x 1 blocks and 2 (LD - 1) for 2 x 2
  // blocks, so LD - 1 must be odd for those (up to 8 / 16) lanes to hit distinct bank pairs. N + 3 is even for the
  // odd N; N = 16 takes N + 2 (N + 3 = 19 was a two-way conflict on 54 % of the kernel's shared-memory wavefronts,
  // ncu; the row fibers' two-way conflict at an even LD costs far less).
  static constexpr int LD = N + (N % 2 == 0 ? 2 : kEwLdPad);
  static constexpr int XSZ = (N * LD + 1) & ~1;
  static constexpr int R1 = (2 * N * N > XSZ ? 2 * N * N : XSZ);
  static constexpr int HDR = ((4 + 4 * N) / 2 + 2) & ~1;  // sylv_hdr_doubles(N, N)
  static constexpr int O_X = R1, O_RCP = O_X + XSZ, O_H = O_RCP + 2 * N, O_PIV = O_H + HDR;
  static constexpr int PER0 = O_PIV + N;                   // 2N int pivots
  static constexpr int PER = PER0 + ((8 - PER0 % 16) + 16) % 16;  // = 8 (mod 16): slots start half a bank row apart
  // rotation tile (TI x TJ per lane, P lanes per block)
  static constexpr int TI = P == 8 && N == 16 ? 4 : N == 16 ? 4 : N == 9 ? 3 : N == 21 ? 3 : 1;
  static constexpr int TJ = P == 8 && N == 16 ? 8 : N == 16 ? 4 : N == 9 ? 3 : N == 21 ? 7 : N;
  static constexpr int NTJ = N / TJ;
  static_assert((N / TI) * (N / TJ) == P, "one tile per lane");
  static_assert(EW * P <= 32, "lanes");
};

// x := A^{-1} x for one fiber (LuFactor::solve): gather through the pivots, forward then backward
// substitution in the reference's order, division by the pivot via its reciprocal (exact RN).
template <int N>
__device__ __forceinline__ void lu_fiber(const double* __restrict__ lu, const double* __restrict__ rcp,
                                         const int* __restrict__ perm, double* col, int stride) {
  double x[N];
#pragma unroll
  for (int k = 0; k < N; ++k) x[k] = col[perm[k] * stride];
#pragma unroll
  for (int r = 1; r < N; ++r) {
    double s = x[r];
#pragma unroll
    for (int j = 0; j < r; ++j) s = fmsc(s, lu[r * N + j], x[j]);
    x[r] = s;
  }
#pragma unroll
  for (int r = N - 1; r >= 0; --r) {
    double s = x[r];
#pragma unroll
    for (int j = r + 1; j < N; ++j) s = fmsc(s, lu[r * N + j], x[j]);
    x[r] = fdiv_rcp(s, lu[r * N + r], rcp[r]);
  }
#pragma unroll
  for (int k = 0; k < N; ++k) col[k * stride] = x[k];
}

// fibers li, li + P, ... of a block (P lanes per block), one call each
template <int N, int P, typename F>
__device__ __forceinline__ void for_fibers(int li, F&& f) {
  f(li);
  if constexpr (P < N) {
    asm volatile("" ::: "memory");  // one fiber at a time (interleaving two unrolled fibers spills)
    if (li + P < N) f(li + P);
  }
  if constexpr (2 * P < N) {
    for (int c = li + 2 * P; c < N; c += P) f(c);
  }
}

// One lane's TI x TJ tile of O = op(A) op(B) (N x N x N), k ascending (matmul order). AG / BG:
// that operand is a Schur factor read from global memory through L1 (read-only path; the two
// rotations reuse it), 16-byte loads when N is even; the other operand is in shared memory.
template <int N, int P, bool AT, bool BT, bool AG, bool BG>
__device__ __forceinline__ void mm_tile(const double* A, int lda, const double* B, int ldb, double* O, int ldo,
                                        int li) {
  using C = Ew<N, P>;
  constexpr int TI = C::TI, TJ = C::TJ, KP = (N % 2 == 0 && TI * TJ <= 16) ? 2 : 1;
  const int i0 = (li / C::NTJ) * TI, j0 = (li % C::NTJ) * TJ;
  double acc[TI][TJ];
#pragma unroll
  for (int k = 0; k < N; k += KP) {
    double a[KP][TI], b[KP][TJ];
    if constexpr (AG && KP == 2 && AT && TI % 2 == 0) {  // A[k][i0 + ii], contiguous in ii
#pragma unroll
      for (int kk = 0; kk < 2; ++kk)
#pragma unroll
        for (int ii = 0; ii < TI; ii += 2) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(A + (k + kk) * lda + i0 + ii));
          a[kk][ii] = v.x;
          a[kk][ii + 1] = v.y;
        }
    } else if constexpr (AG && KP == 2 && !AT) {  // A[i0 + ii][k .. k + 1]
#pragma unroll
      for (int ii = 0; ii < TI; ++ii) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(A + (i0 + ii) * lda + k));
        a[0][ii] = v.x;
        a[1][ii] = v.y;
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < KP; ++kk)
#pragma unroll
        for (int ii = 0; ii < TI; ++ii) {
          const double* pa = AT ? A + (k + kk) * lda + i0 + ii : A + (i0 + ii) * lda + k + kk;
          a[kk][ii] = AG ? __ldg(pa) : *pa;
        }
    }
    if constexpr (BG && KP == 2 && !BT && TJ % 2 == 0) {  // B[k][j0 + jj], contiguous in jj
#pragma unroll
      for (int kk = 0; kk < 2; ++kk)
#pragma unroll
        for (int jj = 0; jj < TJ; jj += 2) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(B + (k + kk) * ldb + j0 + jj));
          b[kk][jj] = v.x;
          b[kk][jj + 1] = v.y;
        }
    } else if constexpr (BG && KP == 2 && BT) {  // B[j0 + jj][k .. k + 1]
#pragma unroll
      for (int jj = 0; jj < TJ; ++jj) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(B + (j0 + jj) * ldb + k));
        b[0][jj] = v.x;
        b[1][jj] = v.y;
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < KP; ++kk)
#pragma unroll
        for (int jj = 0; jj < TJ; ++jj) {
          const double* pb = BT ? B + (j0 + jj) * ldb + k + kk : B + (k + kk) * ldb + j0 + jj;
          b[kk][jj] = BG ? __ldg(pb) : *pb;
        }
    }
#pragma unroll
    for (int kk = 0; kk < KP; ++kk)
#pragma unroll
      for (int ii = 0; ii < TI; ++ii)
#pragma unroll
        for (int jj = 0; jj < TJ; ++jj)
          acc[ii][jj] = k + kk == 0 ? fmul(a[kk][ii], b[kk][jj]) : fmac(acc[ii][jj], a[kk][ii], b[kk][jj]);
  }
#pragma unroll
  for (int ii = 0; ii < TI; ++ii)
#pragma unroll
    for (int jj = 0; jj < TJ; ++jj) O[(i0 + ii) * ldo + j0 + jj] = acc[ii][jj];
}

// Replays a factored tiny system (slot [code, L, U, diag, 1/diag], sylv_cells_kernel) on the
// permuted right-hand side b; on return b[u] is unknown u (solve_tiny, sylvester.hpp:34-61).
template <int NS>
__device__ __forceinline__ void replay(const double* cf, double (&b)[4]) {
  constexpr int NL = NS * (NS - 1) / 2;
  int o = 1;
#pragma unroll
  for (int i = 1; i < NS; ++i)
#pragma unroll
    for (int j = 0; j < i; ++j) {
      const double m = cf[o++];
      b[i] = m != 0.0 ? fmsc(b[i], m, b[j]) : b[i];
    }
#pragma unroll
  for (int i = NS - 1; i >= 0; --i) {
    int u = 1 + NL;
#pragma unroll
    for (int r = 0; r < i; ++r) u += NS - 1 - r;
#pragma unroll
    for (int j = i + 1; j < NS; ++j) b[i] = fmsc(b[i], cf[u + j - i - 1], b[j]);
    b[i] = fdiv_rcp(b[i], cf[1 + 2 * NL + i], cf[1 + 2 * NL + NS + i]);
  }
}

template <int N, int P>
__global__ void __launch_bounds__(32, P < N ? 7 : N > kEwBigN ? 8 : 16) kron2d_ew_kernel(DevPC pc, const double* __restrict__ in,
                                                        double* __restrict__ out) {
  using C = Ew<N, P>;
  constexpr int EW = C::EW, LD = C::LD;
  extern __shared__ double sm_all[];
  const int lane = threadIdx.x, g = lane / P, li = lane % P;
  const int blk = blockIdx.x * EW + g;
  const bool act = g < EW && blk < pc.nblk && pc.kind[blk] != 0 && !(pc.skip && *pc.skip);
  double* S = sm_all + (g < EW ? g : 0) * C::PER;
  double* R1 = S;
  const double* Q1 = pc.rec + size_t(act ? blk : 0) * (6 * N * N) + 2 * N * N;  // Schur factors: global, via L1
  const double* Q2 = Q1 + 2 * N * N;
  double* X = S + C::O_X;
  double* rcp = S + C::O_RCP;
  int* hdr = reinterpret_cast<int*>(S + C::O_H);
  int* piv = reinterpret_cast<int*>(S + C::O_PIV);
  const double* rec = pc.rec + size_t(act ? blk : 0) * (6 * N * N);
  const double* cells = pc.cells + size_t(act ? blk : 0) * pc.cells_len;
  if (act) {
    // L2 prefetch of what the later phases read: Q1 | T1 | Q2 | T2 (the cell factors are read only
    // for the 2 x 2 quasi-blocks' cells, on demand)
    for (int o = 16 * li; o < 4 * N * N; o += 16 * P) prefetch_l2(rec + 2 * N * N + o);
    copy_mat<2 * N * N, N, P>(R1, rec, li);               // LU(A2) | LU(B1)
    for (int i = 2 * li; i < C::HDR; i += 2 * P) cpa16(reinterpret_cast<double*>(hdr) + i, cells + i);
    for (int i = li; i < 2 * N; i += P) cpa4(piv + i, pc.piv + size_t(blk) * (2 * N) + i);
    const double* x = in + size_t(blk) * (N * N);
    for (int i = li; i < N * N; i += P) cpa8(X + (i / N) * LD + i % N, x + i);
  }
  cpa_wait();
  __syncwarp();
  if (act)
    for (int i = li; i < N; i += P) {
      rcp[i] = __drcp_rn(R1[i * N + i]);
      rcp[N + i] = __drcp_rn(R1[N * N + i * N + i]);
    }
  __syncwarp();
  // (A2^{-1} (x) I): column fibers, then (I (x) B1^{-1}): row fibers
  if (act)
    for_fibers<N, P>(li, [&](int c) { lu_fiber<N>(R1, rcp, piv, X + c, LD); });
  __syncwarp();
  if (act)
    for_fibers<N, P>(li, [&](int r) { lu_fiber<N>(R1 + N * N, rcp + N, piv + N, X + r * LD, 1); });
  __syncwarp();
  // M = (Q1^T X) Q2
  if (act) mm_tile<N, P, true, false, true, false>(Q1, N, X, LD, R1, LD, li);
  __syncwarp();
  if (act) mm_tile<N, P, false, false, false, true>(R1, LD, Q2, N, X, LD, li);
  __syncwarp();
  // T1 | T2 into R1
  if (act) {
    copy_mat<N * N, N, P>(R1, rec + 3 * N * N, li);
    copy_mat<N * N, N, P>(R1 + N * N, rec + 5 * N * N, li);
  }
  cpa_wait();
  __syncwarp();
  {  // Sylvester: T1 Y + Y T2^T = M, Y over M in X
    const double* T1 = R1;
    const double* T2 = R1 + N * N;
    const int nb1 = act ? hdr[0] : 0, nb2 = act ? hdr[1] : 0;
    if (act && li == 0 && hdr[3]) atomicExch(pc.status, int(TPDG_SINGULAR));
    const int *s1 = hdr + 4, *z1 = s1 + N, *s2 = z1 + N, *z2 = s2 + N;
    const double* cc = cells + C::HDR;
    double* scr = sm_all + C::EW * C::PER + 4 * lane;  // per-lane scratch: the cell's right-hand sides
    const int last = __reduce_max_sync(0xffffffffu, act ? nb1 + nb2 - 2 : -1);
    // cell of this lane at step st (valid = inside the anti-diagonal) and its factor slot
    auto cell_at = [&](int st, int& i0, int& isz, int& k0, int& ksz, int off = 0) {
      const int d1lo = st - (nb2 - 1) > 0 ? st - (nb2 - 1) : 0;
      const int d1hi = st < nb1 - 1 ? st : nb1 - 1;
      const int d1 = d1lo + li + off;
      const bool ok = act && st <= nb1 + nb2 - 2 && d1 <= d1hi;
      const int bi = ok ? nb1 - 1 - d1 : 0, bk = ok ? nb2 - 1 - (st - d1) : 0;
      i0 = s1[bi];
      isz = z1[bi];
      k0 = s2[bk];
      ksz = z2[bk];
      return ok;
    };
    auto load_cf = [&](bool ok, int i0, int isz, int k0, int ksz, double (&c)[22]) {
      const int ns = isz * ksz, npair = !ok ? 0 : ns == 1 ? 2 : ns == 2 ? 4 : 11;
      const double2* sp = reinterpret_cast<const double2*>(cc + 6 * (i0 * N + isz * k0));
#pragma unroll
      for (int u = 0; u < 11; ++u) {
        const double2 v = u < npair ? __ldg(sp + u) : make_double2(0.0, 0.0);
        c[2 * u] = v.x;
        c[2 * u + 1] = v.y;
      }
    };
    // one wavefront step with this lane's cell (ok, i0, isz, k0, ksz); the next step's cell is
    // located first and its factor slot prefetched into L1, so that the factors, loaded after
    // the chains (registers stay free for the chains' load pipelining), arrive from L1
    // chains + tiny-system replay of one cell (ok, i0, isz, k0, ksz)
    auto do_cell = [&](bool ok, int i0, int isz, int k0, int ksz) {
      if (ok) {
        const int ns = isz * ksz;
        const int i1 = i0 + isz - 1, k1 = k0 + ksz - 1;
        double s00 = X[i0 * LD + k0], s01 = X[i0 * LD + k1], s10 = X[i1 * LD + k0], s11 = X[i1 * LD + k1];
        {  // solved rows below (j ascending), then solved columns to the right (l ascending)
          const double* ta = T1 + i0 * N + i0 + isz;
          const double* tb = ta + (isz - 1) * N;
          const double* ya = X + (i0 + isz) * LD + k0;
          const int dk = ksz - 1;
#pragma unroll 4
          for (int t = 0; t < N - i0 - isz; ++t) {
            const double a0 = ta[t], a1 = tb[t], y0 = ya[t * LD], y1 = ya[t * LD + dk];
            s00 = fmsc(s00, a0, y0);
            s01 = fmsc(s01, a0, y1);
            s10 = fmsc(s10, a1, y0);
            s11 = fmsc(s11, a1, y1);
          }
          const double* ua = T2 + k0 * N + k0 + ksz;
          const double* ub = ua + (ksz - 1) * N;
          const double* wa = X + i0 * LD + k0 + ksz;
          const double* wb = wa + (isz - 1) * LD;
#pragma unroll 4
          for (int t = 0; t < N - k0 - ksz; ++t) {
            const double u0 = ua[t], u1 = ub[t], w0 = wa[t], w1 = wb[t];
            s00 = fmsc(s00, u0, w0);
            s01 = fmsc(s01, u1, w0);
            s10 = fmsc(s10, u0, w1);
            s11 = fmsc(s11, u1, w1);
          }
        }
        if (ns == 1) {  // solve_tiny<1>: the cell's coefficient (0 + t1_ii) + t2_kk, recomputed
          const double coef = fadd(fadd(0.0, T1[i0 * N + i0]), T2[k0 * N + k0]);
          X[i0 * LD + k0] = fdiv_rcp(s00, coef, __drcp_rn(coef));
        } else {
          double cf[22];
          load_cf(true, i0, isz, k0, ksz, cf);
          // unknowns in (a, kb) order, a * ksz + kb; rows permuted by the elimination's pivots
          const long long code = __double_as_longlong(cf[0]);
          scr[0] = s00;
          scr[1] = ksz == 2 ? s01 : s10;
          scr[2] = s10;
          scr[3] = s11;
          double b[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) b[u] = scr[int((code >> (2 * u)) & 3)];
          if (ns == 2) {
            replay<2>(cf, b);
            X[i0 * LD + k0] = b[0];
            X[i1 * LD + k1] = b[1];  // (0, 1) or (1, 0)
          } else {
            replay<4>(cf, b);
            X[i0 * LD + k0] = b[0];
            X[i0 * LD + k1] = b[1];
            X[i1 * LD + k0] = b[2];
            X[i1 * LD + k1] = b[3];
          }
        }
      }
    };
    auto step = [&](int st, bool ok, int i0, int isz, int k0, int ksz, bool& nok, int& ni0, int& nisz, int& nk0,
                    int& nksz) {
      nok = cell_at(st + 1, ni0, nisz, nk0, nksz);
      if (nok && nisz * nksz > 1) {
        const double* sp = cc + 6 * (ni0 * N + nisz * nk0);
        asm volatile("prefetch.global.L1 [%0];" ::"l"(sp));
        if (nisz * nksz == 4) asm volatile("prefetch.global.L1 [%0];" ::"l"(sp + 16));
      }
      do_cell(ok, i0, isz, k0, ksz);
      if constexpr (P < N) {  // more cells on this anti-diagonal than lanes per block: further passes
        const int d1lo = st - (nb2 - 1) > 0 ? st - (nb2 - 1) : 0;
        const int d1hi = st < nb1 - 1 ? st : nb1 - 1;
        const int nc = __reduce_max_sync(0xffffffffu, act && st <= nb1 + nb2 - 2 ? d1hi - d1lo + 1 : 0);
        for (int off = P; off < nc; off += P) {
          int xi0, xisz, xk0, xksz;
          const bool xok = cell_at(st, xi0, xisz, xk0, xksz, off);
          do_cell(xok, xi0, xisz, xk0, xksz);
        }
      }
      __syncwarp();
    };
    bool aok, bok;
    int ai0, aisz, ak0, aksz, bi0, bisz, bk0, bksz;
    aok = cell_at(0, ai0, aisz, ak0, aksz);
    for (int st = 0; st <= last; st += 2) {  // ping-pong between the two cell descriptors
      step(st, aok, ai0, aisz, ak0, aksz, bok, bi0, bisz, bk0, bksz);
      if (st + 1 <= last) step(st + 1, bok, bi0, bisz, bk0, bksz, aok, ai0, aisz, ak0, aksz);
    }
  }
  // X = (Q1 Y) Q2^T
  if (act) mm_tile<N, P, false, false, true, false>(Q1, N, X, LD, R1, LD, li);
  __syncwarp();
  if (act) mm_tile<N, P, false, true, false, true>(R1, LD, Q2, N, X, LD, li);
  __syncwarp();
  if (act) {
    double* o = out + size_t(blk) * (N * N);
    for (int i = li; i < N * N; i += P) o[i] = X[(i / N) * LD + i % N];
  }
}

template <int N, int P = N>
bool try_ew(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  if (pc.dim != 2 || pc.n1 != N || pc.q != N) return false;
  using C = Ew<N, P>;
  const size_t smem = sizeof(double) * (size_t(C::PER) * C::EW + 4 * 32);
  ensure_smem(kron2d_ew_kernel<N, P>, smem, true);
  kron2d_ew_kernel<N, P><<<(pc.nblk + C::EW - 1) / C::EW, 32, smem, st>>>(pc, in, out);
  return true;
}

} // namespace

bool launch_kron2d_ew(const DevPC& pc, const double* in, double* out, cudaStream_t st) {
  return try_ew<5>(pc, in, out, st) || try_ew<9>(pc, in, out, st) || try_ew<16, kEw16Lanes>(pc, in, out, st) ||
         try_ew<21>(pc, in, out, st) || try_ew<31>(pc, in, out, st);
}

} // namespace tpdg_gpu
