// Grid-reduction latency microbenchmark (study tool): P back-to-back deterministic grid sums in one
// cooperative launch of 148 x 1024 threads, as one MGS pass would do with no data.
//   A: generation barrier (atomic arrival + generation flag) then every CTA reads all partials
//   B: monotonic arrival counter (target known from the pass index) then every CTA reads all partials
//   C: per-CTA slots {value, epoch} (16 B, st.release), spread 512 B apart, polled by lanes 0..nb-1
//   D<S>: B with the arrival counter sharded over S counters 256 B apart (CTA b arrives on counter b % S; same-address
//         L2 atomics serialize at ~27 cycles each, 148 of them ~2 us); lanes 0..S-1 of warp 0 each poll one shard
//   E: per-CTA slots of two 8-byte words {32 bits of the partial | 32-bit epoch} (each word single-copy atomic: the data
//      carries its own flag, no fence, no atomic, relaxed stores and polls), parity double buffer, polled by lanes 0..nb-1
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/gsb tools/gridsum_bench.cu
#include <cstdio>
#include <cstdint>

constexpr int NT = 1024;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double cta_partial(double v, double* shA) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) shA[wid] = v;
  __syncthreads();
  double bs = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < NT / 32; ++w) bs += shA[w];
  return bs;  // thread 0
}
__device__ __forceinline__ double finish(double pv, double* shB) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = int((gridDim.x + 31) / 32);
  if (wid < nw) {
    pv = warp_sum(pv);
    if (lane == 0) shB[wid] = pv;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < nw; ++w) tot += shB[w];
    shB[32] = tot;
  }
  __syncthreads();
  return shB[32];
}

template <int V, int S = 1>
__global__ void __launch_bounds__(NT) gsum(int P, double* part, unsigned* bar, double* out, unsigned base) {
  __shared__ double shA[32], shB[33];
  const unsigned nb = gridDim.x;
  double acc = 0.0, x = 1.0 + blockIdx.x * 1e-3 + threadIdx.x * 1e-6;
  for (int p = 0; p < P; ++p) {
    const double bs = cta_partial(x, shA);
    double pv = 0.0;
    if (V == 0) {
      if (threadIdx.x == 0) {
        part[size_t(p % 64) * nb + blockIdx.x] = bs;
        unsigned g, t;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(bar) : "memory");
        if (t == nb - 1) {
          asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
        } else {
          unsigned cur;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
          } while (cur == g);
        }
      }
      __syncthreads();
      pv = threadIdx.x < nb ? reinterpret_cast<volatile double*>(part)[size_t(p % 64) * nb + threadIdx.x] : 0.0;
    } else if (V == 1) {
      if (threadIdx.x == 0) {
        part[size_t(p % 64) * nb + blockIdx.x] = bs;
        const unsigned target = base + (p + 1) * nb;
        unsigned t;
        asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(bar) : "memory");
        if (t + 1 != target) {
          unsigned cur;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
          } while (int(cur - target) < 0);
        }
      }
      __syncthreads();
      pv = threadIdx.x < nb ? reinterpret_cast<volatile double*>(part)[size_t(p % 64) * nb + threadIdx.x] : 0.0;
    } else if (V == 3) {
      if (threadIdx.x == 0) {
        part[size_t(p % 64) * nb + blockIdx.x] = bs;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 64 * (blockIdx.x % S)) : "memory");
      }
      if (threadIdx.x < S) {  // shard c gets the CTAs b = c (mod S)
        const unsigned nc = (nb - threadIdx.x + S - 1) / S, target = (base + p + 1) * nc;
        unsigned cur;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 64 * threadIdx.x) : "memory");
        } while (int(cur - target) < 0);
      }
      __syncthreads();
      pv = threadIdx.x < nb ? reinterpret_cast<volatile double*>(part)[size_t(p % 64) * nb + threadIdx.x] : 0.0;
    } else if (V == 4) {
      const unsigned epoch = base + p + 1;
      unsigned long long* slots = reinterpret_cast<unsigned long long*>(part) + 2 * size_t(nb) * (p & 1);
      if (threadIdx.x == 0) {
        const unsigned long long bits = (unsigned long long)__double_as_longlong(bs);
        const unsigned long long w0 = (bits & 0xffffffffull) | ((unsigned long long)epoch << 32);
        const unsigned long long w1 = (bits >> 32) | ((unsigned long long)epoch << 32);
        asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(slots + 2 * blockIdx.x), "l"(w0), "l"(w1) : "memory");
      }
      if (threadIdx.x < nb) {
        unsigned long long w0, w1;
        do {
          asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(slots + 2 * threadIdx.x) : "memory");
        } while (unsigned(w0 >> 32) != epoch || unsigned(w1 >> 32) != epoch);
        pv = __longlong_as_double((long long)((w0 & 0xffffffffull) | (w1 << 32)));
      }
    } else {
      // slot b at part + 64 b doubles (512 B apart): {value, epoch}
      const unsigned epoch = base + p + 1;
      if (threadIdx.x == 0) {
        double* sl = part + 64 * (size_t(blockIdx.x) + nb * (p & 1));  // parity double buffer
        asm volatile("st.release.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(sl), "l"(__double_as_longlong(bs)),
                     "l"((unsigned long long)epoch)
                     : "memory");
      }
      if (threadIdx.x < nb) {
        const double* sl = part + 64 * (size_t(threadIdx.x) + nb * (p & 1));
        unsigned long long v, e;
        do {
          asm volatile("ld.acquire.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v), "=l"(e) : "l"(sl) : "memory");
        } while (int(unsigned(e) - epoch) < 0);
        pv = __longlong_as_double(v);
      }
    }
    const double tot = finish(pv, shB);
    acc += tot;
    x = x * 0.5 + 1e-9 * tot;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *part, *out;
  unsigned* bar;
  cudaMalloc(&part, sizeof(double) * 64 * 256 * 2);
  cudaMalloc(&out, 8);
  cudaMalloc(&bar, 256 * 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int P = 2000;
  for (int grid : {sms, sms / 2, sms / 4}) {  // variant B with fewer CTAs: does the reduction get cheaper?
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(bar, 0, 256 * 64);
      unsigned base = 0;
      int Pv = P;
      void* args[] = {&Pv, &part, &bar, &out, &base};
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)gsum<1>, dim3(grid), dim3(NT), args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("variant B, %d CTAs: %.3f us per grid sum\n", grid, ms * 1e3 / P);
    }
  }
  for (int v = 0; v < 9; ++v) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(bar, 0, 256 * 64);
      cudaMemset(part, 0, sizeof(double) * 64 * 256 * 2);
      unsigned base = 0;
      int Pv = P;
      void* args[] = {&Pv, &part, &bar, &out, &base};
      void* fn = v == 0 ? (void*)gsum<0> : v == 1 ? (void*)gsum<1> : v == 2 ? (void*)gsum<2> : v == 3 ? (void*)gsum<3, 4>
                 : v == 4 ? (void*)gsum<3, 8> : v == 5 ? (void*)gsum<3, 16> : v == 6 ? (void*)gsum<3, 32> : v == 7 ? (void*)gsum<3, 1> : (void*)gsum<4>;
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel(fn, dim3(sms), dim3(NT), args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      double o = 0;
      cudaMemcpy(&o, out, 8, cudaMemcpyDeviceToHost);
      const char* names[] = {"A", "B", "C", "D<4>", "D<8>", "D<16>", "D<32>", "D<1>", "E"};
      if (rep == 2) printf("variant %s: %.3f us per grid sum (%s) acc %.17g\n", names[v], ms * 1e3 / P,
                           cudaGetErrorString(cudaGetLastError()), o);
    }
  }
  return 0;
}
