// Study tool: what a per-SM cp.async.bulk (TMA 1D) ring can stream on B200, in the MGS kernel's shape:
// one 512-thread CTA per SM, each streaming its own contiguous slice of a vector, pass after pass
// (a different vector per pass, so every pass comes from HBM), rows of ROWB bytes through an NS-stage ring,
// the copy of a row split into NI pieces issued by NI different threads (lane 0 of NI warps).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_1704_04549_b200/csrc \
//        -o tools/tma_ring_bench_bin tools/tma_ring_bench.cu
//   tools/tma_ring_bench_bin            (sweeps row size x stages x issuers; prints us per pass, B/clk/SM, TB/s)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tma.cuh"
using namespace tpdg_gpu;

__device__ __forceinline__ void wait_test(uint64_t* b, unsigned parity) {  // non-blocking test_wait spin
  unsigned ok;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void wait_hint(uint64_t* b, unsigned parity, unsigned ns_hint) {  // try_wait with a time hint
  unsigned ok;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(parity), "r"(ns_hint) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void wait_sleep(uint64_t* b, unsigned parity) {  // test_wait with nanosleep backoff
  unsigned ok;
  for (;;) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
    if (ok) break;
    __nanosleep(40);
  }
}
#define WAITX(b, par) do { if (wmode == 1) wait_test(b, par); else if (wmode == 2) wait_hint(b, par, 20u); else if (wmode == 4) wait_sleep(b, par); else mbar_wait(b, par); } while (0)

__global__ void __launch_bounds__(544, 1) ring_kernel(const double* __restrict__ V, int64_t ldv, int nvec, int64_t chunk,
                                                      int rowb, int ns, int ni, int passes, double* out, int reread, int mode, int wmode) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t lo = int64_t(blockIdx.x) * chunk;
  const int rowd = rowb / 8;
  const int nrows = int(chunk / rowd);
  if (t == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], (mode == 1 || mode == 3) ? 1 : ni);
      mbar_init(&empty[s], 16);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int ntask = passes * nrows;
  const int piece = rowb / ni;
  auto issue = [&](int task) {  // by lane 0 of warps < ni
    const int j = task / nrows, r = task - j * nrows, s = task % ns;
    const int vec = reread ? (j & 1) : (j % nvec);
    mbar_expect_tx(&full[s], unsigned(piece));
    bulk_g2s(sm + size_t(s) * rowb + size_t(warp) * piece,
             reinterpret_cast<const unsigned char*>(V + int64_t(vec) * ldv + lo + int64_t(r) * rowd) + size_t(warp) * piece,
             unsigned(piece), &full[s]);
  };
  if (mode == 1) {  // dedicated producer warp: free-running, bounded by the empty barriers only
    if (warp == 16) {
      if (lane == 0)
        for (int q = 0; q < ntask; ++q) {
          if (q >= ns) WAITX(&empty[q % ns], unsigned(q / ns - 1) & 1u);
          const int j = q / nrows, r = q - j * nrows, s = q % ns;
          const int vec = reread ? (j & 1) : (j % nvec);
          mbar_expect_tx(&full[s], unsigned(rowb));
          bulk_g2s(sm + size_t(s) * rowb, V + int64_t(vec) * ldv + lo + int64_t(r) * rowd, unsigned(rowb), &full[s]);
        }
      return;
    }
  } else if (warp == 16) {
    return;
  }
  const bool issuer = mode != 1 && mode != 3 && lane == 0 && warp < ni;
  if (issuer)
    for (int q = 0; q < ns - 1 && q < ntask; ++q) issue(q);
  auto issue_rr = [&](int q) {  // mode 3: the whole row of task q by lane 0 of warp q % 16
    const int j = q / nrows, r = q - j * nrows, s = q % ns;
    const int vec = reread ? (j & 1) : (j % nvec);
    mbar_expect_tx(&full[s], unsigned(rowb));
    bulk_g2s(sm + size_t(s) * rowb, V + int64_t(vec) * ldv + lo + int64_t(r) * rowd, unsigned(rowb), &full[s]);
  };
  if (mode == 3 && lane == 0)
    for (int q = 0; q < ns - 1 && q < ntask; ++q)
      if (q % 16 == warp) issue_rr(q);
  double acc = 0.0;
  for (int task = 0; task < ntask; ++task) {
    const int s = task % ns;
    if (issuer && task + ns - 1 < ntask) {
      const int nt = task + ns - 1;
      if (nt >= ns) WAITX(&empty[nt % ns], unsigned(nt / ns - 1) & 1u);
      issue(nt);
    }
    if (mode == 3 && lane == 0 && task + ns - 1 < ntask && (task + ns - 1) % 16 == warp) {
      const int nt = task + ns - 1;
      if (nt >= ns) WAITX(&empty[nt % ns], unsigned(nt / ns - 1) & 1u);
      issue_rr(nt);
    }
    if (wmode == 3) {  // one warp polls, the CTA's consumers meet at a hardware barrier
      if (warp == 0) mbar_wait(&full[s], unsigned(task / ns) & 1u);
      asm volatile("bar.sync 1, 512;" ::: "memory");
    } else if (mode == 2) {
      if (lane == 0) WAITX(&full[s], unsigned(task / ns) & 1u);
      __syncwarp();
    } else {
      WAITX(&full[s], unsigned(task / ns) & 1u);
    }
    const double2* p = reinterpret_cast<const double2*>(sm + size_t(s) * rowb);
    for (int i = t; i < rowd / 2; i += 512) {
      const double2 v = p[i];
      acc += v.x + v.y;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (acc == 123.456) out[0] = acc;
}

int main() {
  const int64_t n = 5451776;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int nvec = 16;
  const int64_t ldv = (n + 4095) & ~int64_t(4095);
  double *V, *out;
  cudaMalloc(&V, sizeof(double) * ldv * nvec);
  cudaMalloc(&out, 8);
  cudaMemset(V, 0, sizeof(double) * ldv * nvec);
  cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int passes = 16;
  printf("SMs %d, clock %d kHz; slice %lld doubles per SM, %d passes over %d vectors (HBM) or 2 vectors (L2 reread)\n", sms,
         clk, (long long)(n / sms), passes, nvec);
  for (int grid : {sms})
  for (int wmode : {0, 3, 4})
  for (int mode : {0, 1})
  for (int reread = 1; reread < 2; ++reread)
    for (int rowb : {4096, 16384})
      for (int ns : {2, 3, 6})
        for (int ni : {1}) {
          if (size_t(rowb) * ns > 200 * 1024) continue;
          const int rowd = rowb / 8;
          int64_t chunk = n / sms / rowd * rowd;  // whole rows only
          float best = 1e30f;
          for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            ring_kernel<<<grid, 544, size_t(rowb) * ns>>>(V, ldv, nvec, chunk, rowb, ns, ni, passes, out, reread, mode, wmode);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
          }
          cudaError_t e = cudaGetLastError();
          const double bytes = double(chunk) * 8 * grid * passes;
          printf("wait %d grid %3d mode %d %s row %5d B stages %2d issuers %2d: %6.2f us per pass, %5.2f TB/s, %5.1f B/clk/SM %s\n",
                 wmode, grid, mode, reread ? "L2 " : "HBM", rowb, ns, ni, best * 1e3 / passes, bytes / (best * 1e-3) / 1e12,
                 bytes / grid / (best * 1e-3) / (clk * 1e3), e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
  return 0;
}
