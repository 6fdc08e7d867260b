// Study tool: DMMA.8x8x4 dependent-chain latency and multi-warp throughput on B200.  tools/dmma_lat_bin
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, long long* cyc, int iters) {
  double c[CH][2];
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i], a, b);
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8 << 20); cudaMallocManaged(&cyc, 8);
  const int iters = 2000;
  for (int warps : {1, 2, 4, 8, 16, 32}) {
    printf("warps/SM %2d:", warps);
    k<1><<<148, 32 * warps>>>(out, cyc, iters); cudaDeviceSynchronize(); printf("  1 chain: %.1f cyc/dmma", double(cyc[0]) / iters);
    k<2><<<148, 32 * warps>>>(out, cyc, iters); cudaDeviceSynchronize(); printf("  2 chains: %.1f cyc/dmma/warp", double(cyc[0]) / iters / 2);
    k<4><<<148, 32 * warps>>>(out, cyc, iters); cudaDeviceSynchronize(); printf("  4 chains: %.1f", double(cyc[0]) / iters / 4);
    k<8><<<148, 32 * warps>>>(out, cyc, iters); cudaDeviceSynchronize(); printf("  8 chains: %.1f\n", double(cyc[0]) / iters / 8);
  }
  return 0;
}
