// K3 instantiation unit: the 12-warp two-target class kernel (4 <= k <= 16).
#include "lookup_impl.cuh"

namespace cmb {

cudaError_t launch_lookup_w12(const LookupArgs& a, int grid, int smem, cudaStream_t st) {
  auto kern = lookup_xmap_kernel<true, 0, 12>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, 12 * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace cmb
