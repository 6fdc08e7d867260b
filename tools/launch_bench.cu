// Launch-overhead probe (study tool): back-to-back launches of an empty 148 x 1024 kernel,
// regular vs cooperative, with and without 170 KB of dynamic shared memory.
#include <cstdio>
__global__ void __launch_bounds__(1024) empty_kernel(int* p) {
  extern __shared__ double s[];
  if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = int(s[0]);
}
int main() {
  cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int* p = nullptr;
  for (int coop = 0; coop < 2; ++coop)
    for (int big = 0; big < 2; ++big) {
      const size_t smem = big ? 170 * 1024 : 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a, st);
        for (int i = 0; i < 200; ++i) {
          if (coop) {
            void* args[] = {&p};
            cudaLaunchCooperativeKernel((void*)empty_kernel, dim3(148), dim3(1024), args, smem, st);
          } else {
            empty_kernel<<<148, 1024, smem, st>>>(p);
          }
        }
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("coop=%d smem=%zu: %.2f us per launch\n", coop, smem, ms * 1e3 / 200);
      }
    }
  return 0;
}
