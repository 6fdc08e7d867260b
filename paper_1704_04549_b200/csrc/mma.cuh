// Warp-level FP64 tensor-core products (DMMA.8x8x4 = mma.sync.aligned.m8n8k4.row.col.f64).
//
// Fragment layouts (PTX ISA, mma.m8n8k4 .f64): A 8x4: lane l holds A[l/4][l%4]; B 4x8: B[l%4][l/4];
// C/D 8x8: C[l/4][2(l%4) + {0,1}]. With a shared-memory leading dimension ld = 4 (mod 8) (lda4)
// every fragment load -- A[m][k] at m*ld + k, or the transposed access k*ld + m -- hits each bank
// pair exactly twice: two wavefronts for 256 bytes, the minimum.
#pragma once

namespace tpdg_gpu {

constexpr int p8(int x) { return (x + 7) & ~7; }
constexpr int p4(int x) { return (x + 3) & ~3; }
constexpr int lda4(int x) { return (x + 3) / 8 * 8 + 4; }   // smallest y >= x with y = 4 (mod 8)
constexpr int ldb8(int x) { return (x + 7) / 16 * 16 + 8; }  // smallest y >= x with y = 8 (mod 16)

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// acc[MT][NT] += op(A)[8MT x 4KC] op(B)[4KC x 8NT].
//   ATR: A[m][k] = As[k * lda + m] (else As[m * lda + k]);
//   BCOL: B[k][n] = Bs[n * ldb + k] (else Bs[k * ldb + n]).
template <int MT, int NT, int KC, bool BCOL, bool ATR = false>
__device__ __forceinline__ void mma_tiles(double (&acc)[MT][NT][2], const double* A, int lda, const double* B, int ldb,
                                          int lane) {
  const int r = lane >> 2, kq = lane & 3;
#pragma unroll
  for (int kc = 0; kc < KC; ++kc) {
    double a[MT], b[NT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
      a[mt] = ATR ? A[(4 * kc + kq) * lda + 8 * mt + r] : A[(8 * mt + r) * lda + 4 * kc + kq];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
      b[nt] = BCOL ? B[(8 * nt + r) * ldb + 4 * kc + kq] : B[(4 * kc + kq) * ldb + 8 * nt + r];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt], a[mt], b[nt]);
  }
}

template <int MT, int NT>
__device__ __forceinline__ void zero_tiles(double (&acc)[MT][NT][2]) {
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
}

// Store rows [0, rows) of the tiles to O (ldo even: 16-byte stores).
template <int MT, int NT>
__device__ __forceinline__ void store_tiles(const double (&acc)[MT][NT][2], double* O, int ldo, int rows, int lane) {
  const int r = lane >> 2, c = 2 * (lane & 3);
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
      if (8 * mt + r < rows)
        *reinterpret_cast<double2*>(O + (8 * mt + r) * ldo + 8 * nt + c) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
}

} // namespace tpdg_gpu
