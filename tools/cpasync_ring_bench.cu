// Study tool: thread-private cp.async ring (no barriers): each of 512 threads copies the 16-byte pieces it will
// consume itself (pairs t + 512 u of every 2048-double row), D rows in flight, cp.async.wait_group per row.
//   tools/cpasync_ring_bench_bin
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cpa16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(uint32_t(__cvta_generic_to_shared(dst))), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int D, int PPT>
__global__ void __launch_bounds__(512, 1) k(const double* __restrict__ V, int64_t ldv, int nvec, int64_t chunk, int passes,
                                            double* out, int reread) {
  extern __shared__ __align__(128) double sm[];
  constexpr int ROW = 2 * 512 * PPT;
  const int t = threadIdx.x;
  const int64_t lo = int64_t(blockIdx.x) * chunk;
  const int nrows = int(chunk / ROW);
  const int ntask = passes * nrows;
  auto issue = [&](int task) {
    if (task < ntask) {
      const int j = task / nrows, r = task - j * nrows, s = task % D;
      const double* src = V + int64_t(reread ? (j & 1) : (j % nvec)) * ldv + lo + int64_t(r) * ROW;
#pragma unroll
      for (int u = 0; u < PPT; ++u) cpa16(sm + s * ROW + 2 * (t + 512 * u), src + 2 * (t + 512 * u));
    }
    cpa_commit();
  };
  for (int q = 0; q < D - 1; ++q) issue(q);
  double acc = 0.0;
  for (int task = 0; task < ntask; ++task) {
    issue(task + D - 1);  // into the slot consumed at task - 1 (by this same thread)
    cpa_wait<D - 1>();
    const int s = task % D;
#pragma unroll
    for (int u = 0; u < PPT; ++u) {
      const double2 v = *reinterpret_cast<const double2*>(sm + s * ROW + 2 * (t + 512 * u));
      acc += v.x + v.y;
    }
  }
  if (acc == 123.456) out[0] = acc;
}

template <int D, int PPT>
void run(const double* V, int64_t ldv, int nvec, double* out) {
  const int64_t n = 5451776; const int sms = 148;
  constexpr int ROW = 2 * 512 * PPT;
  const int64_t chunk = n / sms / ROW * ROW;
  const size_t smem = sizeof(double) * ROW * D;
  cudaFuncSetAttribute(k<D, PPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int reread = 0; reread < 2; ++reread) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      k<D, PPT><<<sms, 512, smem>>>(V, ldv, nvec, chunk, 16, out, reread);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    const double bytes = double(chunk) * 8 * sms * 16;
    printf("%s depth %2d row %5d B: %6.2f us per pass, %5.2f TB/s  %s\n", reread ? "L2 " : "HBM", D, ROW * 8, best * 1e3 / 16,
           bytes / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  const int nvec = 16; const int64_t ldv = 5451776 + 4096;
  double *V, *out;
  cudaMalloc(&V, sizeof(double) * ldv * nvec); cudaMemset(V, 0, sizeof(double) * ldv * nvec);
  cudaMalloc(&out, 8);
  run<2, 2>(V, ldv, nvec, out); run<3, 2>(V, ldv, nvec, out); run<4, 2>(V, ldv, nvec, out); run<6, 2>(V, ldv, nvec, out);
  run<8, 2>(V, ldv, nvec, out); run<12, 2>(V, ldv, nvec, out);
  run<4, 1>(V, ldv, nvec, out); run<8, 1>(V, ldv, nvec, out); run<16, 1>(V, ldv, nvec, out);
  run<3, 4>(V, ldv, nvec, out); run<6, 4>(V, ldv, nvec, out);
  return 0;
}
