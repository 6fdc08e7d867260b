// Study tool: completion times of a burst of cp.async.bulk copies issued by one thread (one CTA), each to its own
// mbarrier: are consecutive bulk copies pipelined by the copy engine?  tools/tma_lat_bench_bin
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "tma.cuh"
using namespace tpdg_gpu;

__global__ void k(const double* V, int bytes, int nops, int gap, long long* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < nops; ++i) mbar_init(&bar[i], 1);
    mbar_fence_init();
    const long long t0 = clock64();
    for (int i = 0; i < nops; ++i) {
      mbar_expect_tx(&bar[i], unsigned(bytes));
      bulk_g2s(sm + size_t(i) * bytes, reinterpret_cast<const unsigned char*>(V) + size_t(i) * bytes + size_t(blockIdx.x) * (1 << 20), unsigned(bytes), &bar[i]);
      out[16 + i] = clock64() - t0;
      if (gap) { const long long t1 = clock64(); while (clock64() - t1 < gap) {} }
    }
    for (int i = 0; i < nops; ++i) {
      mbar_wait(&bar[i], 0);
      out[i] = clock64() - t0;
    }
  }
}

int main() {
  double* V; long long* out;
  cudaMalloc(&V, size_t(512) << 20);
  cudaMemset(V, 0, size_t(512) << 20);
  cudaMallocManaged(&out, 64 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int grid : {1, 148})
  for (int gap : {0, 300})
  for (int bytes : {1024, 4096, 16384, 32768}) {
    const int nops = bytes * 6 <= 200 * 1024 ? 6 : 200 * 1024 / bytes;
    for (int rep = 0; rep < 2; ++rep) {  // rep 0: from HBM (cold), rep 1: L2
      k<<<grid, 32, 200 * 1024>>>(V, bytes, nops, gap, out);
      cudaDeviceSynchronize();
      printf("grid %3d gap %3d bytes %5d %s: issue", grid, gap, bytes, rep ? "L2 " : "HBM");
      for (int i = 0; i < nops; ++i) printf(" %lld", out[16 + i]);
      printf(" | done");
      for (int i = 0; i < nops; ++i) printf(" %lld", out[i]);
      printf("\n");
    }
    cudaMemset(V, 1, size_t(512) << 20);  // flush L2 for the next size
  }
  return 0;
}
