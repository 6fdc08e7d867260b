// Measures the FP64 peaks the roofline needs (SURVEY.md sec.8d asks for them; MEASURED_PEAKS.json
// has only HBM and bf16): DFMA (CUDA cores) and DMMA.8x8x4 (mma.sync f64 tensor cores).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void dfma_kernel(double* out, double s) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 0.5);
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 1234.5) out[0] = r;
}

__global__ void dmma_kernel(double* out, double s) {
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = threadIdx.x * 1e-3 + i;
  const double x = s, y = s * 0.5;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(x), "d"(y));
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += d[i][0] + d[i][1];
  if (r == 1234.5) out[0] = r;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    float ms = 0;
    cudaEventRecord(a);
    dfma_kernel<<<blocks, threads>>>(out, 0.999);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    const double dfma = 2.0 * 8 * kIters * double(blocks) * threads / (ms * 1e-3) / 1e12;
    cudaEventRecord(a);
    dmma_kernel<<<blocks, threads>>>(out, 0.999);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    const double dmma = 2.0 * 256 * 8 * kIters * double(blocks) * (threads / 32) / (ms * 1e-3) / 1e12;
    if (rep) printf("{\"fp64_dfma_tflops\": %.2f, \"fp64_dmma_tflops\": %.2f, \"sms\": %d}\n", dfma, dmma, sms);
  }
  return 0;
}
