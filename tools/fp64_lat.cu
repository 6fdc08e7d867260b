// FP64 dependent-chain latencies on the device (one warp): DADD, DMUL, DFMA, __ddiv_rn, __drcp_rn,
// LDS->DADD, SHFL. nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_lat.cu -o /tmp/fp64_lat
#include <cstdio>
#include <cuda_runtime.h>
constexpr int R = 1024;
__global__ void k(double* out, long long* cyc, double a, double b) {
  __shared__ double sm[64];
  sm[threadIdx.x] = a + threadIdx.x; sm[threadIdx.x + 32] = b;
  __syncwarp();
  double x = a; long long t0, t1;
  t0 = clock64(); for (int i = 0; i < R; ++i) x = __dadd_rn(x, b); t1 = clock64(); cyc[0] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < R; ++i) x = __dmul_rn(x, b); t1 = clock64(); cyc[1] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < R; ++i) x = __fma_rn(x, b, a); t1 = clock64(); cyc[2] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < R; ++i) x = __ddiv_rn(x, b); t1 = clock64(); cyc[3] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < R; ++i) x = __drcp_rn(x); t1 = clock64(); cyc[4] = t1 - t0;
  int idx = threadIdx.x;
  t0 = clock64(); for (int i = 0; i < R; ++i) { x = __dadd_rn(x, sm[idx]); idx = (idx + int(x != 0.0)) & 31; } t1 = clock64(); cyc[5] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < R; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31); t1 = clock64(); cyc[6] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < R; ++i) x = __dsub_rn(x, __dmul_rn(sm[i & 31], b)); t1 = clock64(); cyc[7] = t1 - t0;
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMallocManaged(&c, 64 * 8);
  k<<<1, 32>>>(o, c, 1.0000001, 0.9999999); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.0000001, 0.9999999); cudaDeviceSynchronize();
  const char* n[] = {"dadd", "dmul", "dfma", "ddiv_rn", "drcp_rn", "lds+dadd(+int)", "shfl", "lds-dmul-dsub chain"};
  for (int i = 0; i < 8; ++i) printf("%-22s %.1f cycles\n", n[i], double(c[i]) / R);
}
