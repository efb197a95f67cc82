// K3 instantiation unit: the non-resident lookup (targets gathered from L2; T past shared memory).
#include "lookup_impl.cuh"

namespace cmb {

cudaError_t launch_lookup_nonresident(const LookupArgs& a, int grid, int smem, cudaStream_t st) {
  auto kern = lookup_xmap_kernel<false, 0, kNonResWarps>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kNonResWarps * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace cmb
