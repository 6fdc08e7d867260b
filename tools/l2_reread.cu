// Study tool: effective L2 capacity for a streamed re-read on B200. Reads buffer A (size S), then
// reads A again; prints the time of the second read vs the first (HBM) for a range of sizes.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/l2_reread_bin tools/l2_reread.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const double2* __restrict__ a, size_t n, double* out, int mode) {
  double s = 0;
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    double2 v;
    if (mode == 1) {
      uint64_t p;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
      asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a + i), "l"(p));
    } else {
      v = __ldcg(a + i);
    }
    s += v.x + v.y;
  }
  if (s == 123.456) out[0] = s;
}

int main() {
  double2* a;
  double* out;
  const size_t maxb = size_t(200) << 20;
  cudaMalloc(&a, maxb);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, maxb);
  double2* flush;
  cudaMalloc(&flush, size_t(512) << 20);
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  for (int mode = 0; mode < 2; ++mode)
    for (int mb : {8, 16, 24, 32, 40, 44, 48, 56, 64, 80, 96, 112}) {
      const size_t n = (size_t(mb) << 20) / 16;
      cudaMemset(flush, mb, size_t(512) << 20);
      cudaEventRecord(e0);
      rd<<<148 * 8, 512>>>(a, n, out, mode);
      cudaEventRecord(e1);
      rd<<<148 * 8, 512>>>(a, n, out, mode);
      cudaEventRecord(e2);
      cudaEventSynchronize(e2);
      float t1, t2;
      cudaEventElapsedTime(&t1, e0, e1);
      cudaEventElapsedTime(&t2, e1, e2);
      printf("mode %d %3d MB: first %.1f us (%.0f GB/s), second %.1f us (%.0f GB/s)\n", mode, mb, t1 * 1e3,
             mb * 1.048576e6 / (t1 * 1e-3) / 1e9, t2 * 1e3, mb * 1.048576e6 / (t2 * 1e-3) / 1e9);
    }
  return 0;
}
