// Kernel launch attributes, per device and thread-safe (cudaFuncSetAttribute acts on the current
// device only; several contexts on several devices, or several rank threads of the loopback
// transport, may launch the same kernel).
#include <map>
#include <mutex>
#include <utility>

#include "tpdg_internal.hpp"

namespace tpdg_gpu {

void ensure_smem(const void* fn, size_t bytes, bool carveout) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;  // (device, kernel) -> configured bytes + 1
  int dev = 0;
  TPDG_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = done[{dev, fn}];
  if (cur > bytes) return;
  TPDG_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
  if (carveout) TPDG_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  cur = bytes + 1;
}

}  // namespace tpdg_gpu
