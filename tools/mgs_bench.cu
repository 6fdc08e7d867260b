// MGS kernel microbenchmark (study tool): times launch_mgs_iteration for k = 0..K-1 on random
// data of size n, as inside one GMRES(30) cycle.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_1704_04549_b200/csrc -Iinclude \
//        -o /tmp/mgs_bench tools/mgs_bench.cu paper_1704_04549_b200/csrc/blas.cu
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cmath>
#include <vector>

#include "tpdg_internal.hpp"

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 1048576;
  const int K = argc > 2 ? atoi(argv[2]) : 25;
  const int64_t ldv = (n + 31) & ~int64_t(31);
  double *V, *hc, *part;
  unsigned* ctr;
  cudaMalloc(&V, sizeof(double) * ldv * 32);
  cudaMalloc(&hc, sizeof(double) * 64);
  cudaMalloc(&part, sizeof(double) * 256 * 64);
  cudaMalloc(&ctr, sizeof(unsigned) * 512);
  cudaMemset(ctr, 0, sizeof(unsigned) * 512);
  std::vector<double> h(ldv * 32);
  srand(1);
  for (auto& x : h) x = rand() / double(RAND_MAX) - 0.5;
  cudaStream_t st;
  cudaStreamCreate(&st);
  if (getenv("L2P")) {  // persisting L2 set-aside (evict_last lines) = the device maximum
    int mx = 0;
    cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, 0);
    const size_t want = size_t(atof(getenv("L2P")) * mx);
    cudaError_t e = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
    printf("max persisting L2 %d B, set %zu -> %s, now %zu\n", mx, want, cudaGetErrorString(e), got);
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(V, h.data(), sizeof(double) * ldv * 32, cudaMemcpyHostToDevice);
    cudaEventRecord(a, st);
    for (int k = 0; k < K; ++k) tpdg_gpu::launch_mgs_iteration(V, ldv, k, n, hc, part, ctr + 4, nullptr, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (rep == 2) printf("n=%lld K=%d: %.1f us per MGS launch (avg k+1 = %.1f), %.2f us per pass\n", (long long)n, K,
                         ms * 1e3 / K, (K + 1) / 2.0, ms * 1e3 / (K * ((K + 1) / 2.0 + 1)));
  }
  {  // host emulation of hc[0] of the last launch (<v_0, V[K]> in the kernels' fixed order)
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int64_t chunk = (n + sms - 1) / sms;
    chunk = (chunk + 1) & ~int64_t(1);
    const double* v = h.data();
    const double* w = h.data() + int64_t(K) * ldv;
    std::vector<double> part(sms);
    for (int b = 0; b < sms; ++b) {
      const int64_t lo = b * chunk, hi = std::min<int64_t>(lo + chunk, n);
      const int len = int(hi > lo ? hi - lo : 0);
      // ownership of the bulk kernel (blas.cu kBulkThreads = 512, kBulkPPT = 2): thread t sums the pairs
      // t + 512 u (u = 0, 1) of every 2048-double row, rows ascending; 16 warp sums in order
      constexpr int NT = 512, PPT = 2, ROW = 2 * NT * PPT;
      double lanev[NT];
      for (int t = 0; t < NT; ++t) {
        double s0 = 0.0, s1 = 0.0;
        for (int r0 = 0; r0 < len; r0 += ROW)
          for (int u = 0; u < PPT; ++u) {
            const int i = r0 + 2 * (t + NT * u);
            if (i + 1 < len) {
              s0 = fma(v[lo + i], w[lo + i], s0);
              s1 = fma(v[lo + i + 1], w[lo + i + 1], s1);
            } else if (i < len) {
              s0 = fma(v[lo + i], w[lo + i], s0);
            }
          }
        lanev[t] = s0 + s1;
      }
      double bs = 0.0;
      for (int wi = 0; wi < NT / 32; ++wi) {
        double x[32];
        for (int l = 0; l < 32; ++l) x[l] = lanev[32 * wi + l];
        for (int o = 16; o > 0; o >>= 1) {
          double y[32];
          for (int l = 0; l < 32; ++l) y[l] = x[l] + x[l ^ o];
          for (int l = 0; l < 32; ++l) x[l] = y[l];
        }
        bs += x[0];
      }
      part[b] = bs;
    }
    const int nw = (sms + 31) / 32;
    double tot = 0.0;
    for (int wi = 0; wi < nw; ++wi) {
      double x[32];
      for (int l = 0; l < 32; ++l) x[l] = 32 * wi + l < sms ? part[32 * wi + l] : 0.0;
      for (int o = 16; o > 0; o >>= 1) {
        double y[32];
        for (int l = 0; l < 32; ++l) y[l] = x[l] + x[l ^ o];
        for (int l = 0; l < 32; ++l) x[l] = y[l];
      }
      tot += x[0];
    }
    printf("host emulation h0 %.17g\n", tot);
  }
  std::vector<double> hh(64);
  cudaMemcpy(hh.data(), hc, sizeof(double) * 64, cudaMemcpyDeviceToHost);
  unsigned long long x = 0;
  for (int j = 0; j <= K; ++j) x ^= reinterpret_cast<unsigned long long&>(hh[j]) * (j + 1);
  printf("hc checksum %016llx (h0 %.17g)\n", x, hh[0]);
  {  // the whole basis after the last launch (w normalized into V[K])
    std::vector<double> vv(ldv * 32);
    cudaMemcpy(vv.data(), V, sizeof(double) * ldv * 32, cudaMemcpyDeviceToHost);
    unsigned long long y = 0;
    for (size_t i = 0; i < vv.size(); ++i) y = y * 1000003ull + reinterpret_cast<unsigned long long&>(vv[i]);
    printf("V checksum %016llx\n", y);
  }
  return 0;
}
