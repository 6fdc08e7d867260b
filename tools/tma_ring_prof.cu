// Study tool: clock64 breakdown of one ring iteration (issue / wait full / read / arrive), per warp.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "tma.cuh"
using namespace tpdg_gpu;

template <int NS, int ROWB>
__global__ void __launch_bounds__(512, 1) k(const double* __restrict__ V, int64_t ldv, int64_t chunk, int passes, double* out,
                                            long long* prof, int variant) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t lo = int64_t(blockIdx.x) * chunk;
  constexpr int rowd = ROWB / 8;
  const int nrows = int(chunk / rowd);
  if (t == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 16); }
    mbar_fence_init();
  }
  __syncthreads();
  const int ntask = passes * nrows;
  auto issue = [&](int task) {
    const int j = task / nrows, r = task - j * nrows, s = task % NS;
    mbar_expect_tx(&full[s], unsigned(ROWB));
    bulk_g2s(sm + size_t(s) * ROWB, V + int64_t(j & 1) * ldv + lo + int64_t(r) * rowd, unsigned(ROWB), &full[s]);
  };
  if (t == 0) for (int q = 0; q < NS - 1 && q < ntask; ++q) issue(q);
  double acc = 0.0;
  long long tI = 0, tW = 0, tR = 0, tA = 0;
  for (int task = 0; task < ntask; ++task) {
    const int s = task % NS;
    long long c0 = clock64();
    if (t == 0 && task + NS - 1 < ntask) {
      const int nt = task + NS - 1;
      if (nt >= NS) mbar_wait(&empty[nt % NS], unsigned(nt / NS - 1) & 1u);
      issue(nt);
    }
    long long c1 = clock64();
    if (variant == 1) { if (lane == 0) mbar_wait(&full[s], unsigned(task / NS) & 1u); __syncwarp(); }
    else mbar_wait(&full[s], unsigned(task / NS) & 1u);
    long long c2 = clock64();
    const double2* p = reinterpret_cast<const double2*>(sm + size_t(s) * ROWB);
#pragma unroll
    for (int i = 0; i < rowd / 2 / 512; ++i) { const double2 v = p[t + 512 * i]; acc += v.x + v.y; }
    long long c3 = clock64();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    long long c4 = clock64();
    tI += c1 - c0; tW += c2 - c1; tR += c3 - c2; tA += c4 - c3;
  }
  if (acc == 123.456) out[0] = acc;
  if (blockIdx.x == 0 && lane == 0) { prof[4 * warp] = tI / ntask; prof[4 * warp + 1] = tW / ntask; prof[4 * warp + 2] = tR / ntask; prof[4 * warp + 3] = tA / ntask; }
}

template <int NS, int ROWB>
void run(const double* V, int64_t ldv, double* out, long long* prof, int variant) {
  const int64_t n = 5451776; const int sms = 148;
  const int rowd = ROWB / 8; const int64_t chunk = n / sms / rowd * rowd;
  cudaFuncSetAttribute(k<NS, ROWB>, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * ROWB);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k<NS, ROWB><<<sms, 512, NS * ROWB>>>(V, ldv, chunk, 16, out, prof, variant);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  }
  printf("NS %d ROWB %5d variant %d: %.2f us per pass, %.0f cycles per row; cycles per task (issue wait read arrive):", NS, ROWB,
         variant, ms * 1e3 / 16, ms * 1e-3 / 16 / (chunk / rowd) * 1.965e9);
  for (int w : {0, 1, 15}) printf("  w%d %lld %lld %lld %lld", w, prof[4 * w], prof[4 * w + 1], prof[4 * w + 2], prof[4 * w + 3]);
  printf("\n");
}

int main() {
  const int64_t ldv = 5451776 + 4096;
  double *V, *out; long long* prof;
  cudaMalloc(&V, sizeof(double) * ldv * 2); cudaMemset(V, 0, sizeof(double) * ldv * 2);
  cudaMalloc(&out, 8); cudaMallocManaged(&prof, 64 * 8);
  for (int variant = 0; variant < 2; ++variant) {
    run<3, 4096>(V, ldv, out, prof, variant);
    run<3, 16384>(V, ldv, out, prof, variant);
    run<6, 16384>(V, ldv, out, prof, variant);
    run<3, 32768>(V, ldv, out, prof, variant);
  }
  return 0;
}
