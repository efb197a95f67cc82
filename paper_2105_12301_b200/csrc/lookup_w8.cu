// K3 instantiation unit: the 8-warp two-target class kernel (17 <= k <= 24).
#include "lookup_impl.cuh"

namespace cmb {

cudaError_t launch_lookup_w8(const LookupArgs& a, int grid, int smem, cudaStream_t st) {
  auto kern = lookup_xmap_kernel<true, 0, 8>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, 8 * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace cmb
