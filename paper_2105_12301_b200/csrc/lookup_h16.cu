// K3 instantiation unit: the opt-in 16-bit target lookups (CMB_LOOKUP_FP16=1 fp16, =2 q16).
#include "lookup_impl.cuh"

namespace cmb {

cudaError_t launch_lookup_h16(const LookupArgs& a, int grid, int smem, cudaStream_t st) {
  auto kern = a.h16 == 2 ? lookup_xmap_kernel<true, 2> : lookup_xmap_kernel<true, 1>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kLookupWarps * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace cmb
