// Study tool: FP64 FMA throughput with the weight operand (a) in a register, (b) loaded from the constant
// bank right before every DFMA (LDCU + uniform-operand DFMA, as jv3d.cu does), (c) one LDCU per two DFMAs,
// (d) one per four, at several warps per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/ldcu_bench_bin tools/ldcu_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__constant__ double cw[512];

__device__ __forceinline__ double cld(const double* p) {
  double r;
  asm volatile("{\n\t.reg .u64 t;\n\tcvta.to.const.u64 t, %1;\n\tld.const.f64 %0, [t];\n\t}" : "=d"(r) : "l"(p));
  return r;
}

__device__ __forceinline__ double2 cld2(const double* p) {
  double2 r;
  asm volatile("{\n\t.reg .u64 t;\n\tcvta.to.const.u64 t, %2;\n\tld.const.v2.f64 {%0, %1}, [t];\n\t}" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

template <int MODE>
__global__ void k(double* out, int iters) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  double x0 = 1.0 + threadIdx.x * 1e-9, x1 = x0 + 0.5, x2 = x0 + 0.25, x3 = x0 + 0.125;
  double wr[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) wr[i] = cw[i] + out[0];
  if (MODE == 5 || MODE == 6) {
    extern __shared__ double sw[];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) sw[i] = cw[i];
    __syncthreads();
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (MODE == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(wr[i], x0, a[i]);
      } else if (MODE == 1) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(cld(&cw[u * 8 + i]), x0, a[i]);
      } else if (MODE == 2) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double w = cld(&cw[u * 4 + i]);
          a[2 * i] = fma(w, x0, a[2 * i]);
          a[2 * i + 1] = fma(w, x1, a[2 * i + 1]);
        }
      } else if (MODE == 4) {  // one 16-byte constant load per two DFMAs with different weights
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double2 w = cld2(&cw[u * 8 + 2 * i]);
          a[2 * i] = fma(w.x, x0, a[2 * i]);
          a[2 * i + 1] = fma(w.y, x0, a[2 * i + 1]);
        }
      } else if (MODE == 5) {  // weights from shared memory, broadcast 16-byte loads
        extern __shared__ double sw[];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double2 w = *reinterpret_cast<const double2*>(&sw[u * 8 + 2 * i]);
          a[2 * i] = fma(w.x, x0, a[2 * i]);
          a[2 * i + 1] = fma(w.y, x0, a[2 * i + 1]);
        }
      } else if (MODE == 6) {  // alternate: constant bank (8 B) and shared memory (8 B)
        extern __shared__ double sw[];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double w0 = cld(&cw[u * 8 + 2 * i]);
          const double w1 = sw[u * 8 + 2 * i + 1];
          a[2 * i] = fma(w0, x0, a[2 * i]);
          a[2 * i + 1] = fma(w1, x0, a[2 * i + 1]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const double w = cld(&cw[u * 2 + i]);
          a[4 * i] = fma(w, x0, a[4 * i]);
          a[4 * i + 1] = fma(w, x1, a[4 * i + 1]);
          a[4 * i + 2] = fma(w, x2, a[4 * i + 2]);
          a[4 * i + 3] = fma(w, x3, a[4 * i + 3]);
        }
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345) out[1] = s;
}

template <int MODE>
void run(double* out, int warps_per_sm) {
  const int iters = 2000;
  int nt = 32 * (warps_per_sm >= 8 ? 8 : warps_per_sm), nb = 148 * (warps_per_sm >= 8 ? warps_per_sm / 8 : 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<MODE><<<nb, nt, 4096>>>(out, 10);
  cudaEventRecord(a);
  k<MODE><<<nb, nt, 4096>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double fl = 2.0 * 128.0 * iters * double(nb) * nt;
  printf("mode %d warps/SM %2d: %.2f TFLOP/s\n", MODE, warps_per_sm, fl / ms * 1e-9);
}

int main() {
  double* out;
  cudaMalloc(&out, 64);
  cudaMemset(out, 0, 64);
  double h[512];
  for (int i = 0; i < 512; ++i) h[i] = 1.0 / (i + 3);
  cudaMemcpyToSymbol(cw, h, sizeof(h));
  for (int w : {4, 8, 16, 24, 32}) {
    run<0>(out, w);
    run<1>(out, w);
    run<2>(out, w);
    run<3>(out, w);
    run<4>(out, w);
    run<5>(out, w);
    run<6>(out, w);
  }
  return 0;
}
