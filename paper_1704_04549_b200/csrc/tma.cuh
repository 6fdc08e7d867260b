// tma.cuh — mbarrier + cp.async.bulk (TMA 1D global -> shared) helpers shared by the MGS ring (blas.cu)
// and the 3D preconditioner's G-block ring (kron.cu); tensor-memory (TMEM) scratch helpers for the MGS kernel.
#pragma once
#include <cstdint>

namespace tpdg_gpu {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!ok);
}
// bytes: multiple of 16; dst / src 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
      : "memory");
}

// HBM -> L2 only (no shared-memory destination, nothing to wait for); bytes: multiple of 16, src 16-byte aligned
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// ---- tensor memory as a per-thread scratchpad (tcgen05.ld / st, shape 32x32b: lane l of warp w reads
// and writes TMEM lane 32 (w % 4) + l, consecutive 32-bit columns). One warp allocates all 512 columns.
__device__ __forceinline__ void tmem_alloc512(uint32_t* slot) {  // one converged warp; *slot (shared) = base address
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc512(uint32_t base) {  // one converged warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
}
__device__ __forceinline__ void tmem_fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// one double2 per access (4 columns)
__device__ __forceinline__ void tmem_ld4(uint32_t addr, double2& v) {
  asm volatile(
      "{\n\t.reg .b32 a, b, c, d;\n\ttcgen05.ld.sync.aligned.32x32b.x4.b32 {a, b, c, d}, [%2];\n\t"
      "mov.b64 %0, {a, b};\n\tmov.b64 %1, {c, d};\n}"
      : "=d"(v.x), "=d"(v.y)
      : "r"(addr)
      : "memory");
}
// the wait carries the loaded values so that no use is scheduled before it
__device__ __forceinline__ void tmem_wait_ld(double2& a, double2& b) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+d"(a.x), "+d"(a.y), "+d"(b.x), "+d"(b.y) : : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t addr, double2 v) {
  asm volatile(
      "{\n\t.reg .b32 a, b, c, d;\n\tmov.b64 {a, b}, %1;\n\tmov.b64 {c, d}, %2;\n\t"
      "tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {a, b, c, d};\n}" ::"r"(addr),
      "d"(v.x), "d"(v.y)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

} // namespace tpdg_gpu
