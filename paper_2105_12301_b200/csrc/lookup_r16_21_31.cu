// K3 instantiation unit: the 16-warp resident kernel for 21 <= k <= 31
// (fallbacks of the class split: long series, CMB_LOOKUP_ROT=0/1, k > 24).
#include "lookup_impl.cuh"

namespace cmb {

cudaError_t launch_lookup_r16_21_31(const LookupArgs& a, int grid, int smem, cudaStream_t st) {
  auto kern = lookup_xmap_kernel<true, 0, kLookupWarps, 21, 31>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kLookupWarps * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace cmb
