// K3: cross-map lookup with fused Pearson skill -- host launchers, the
// 16-warp resident kernel, the fp64 fixup and the predictions kernel.  The
// device code is in lookup_impl.cuh.
#include "lookup_impl.cuh"

#include <algorithm>

namespace cmb {

int lookup_stage_bytes(int T, int max_rec_bytes, int warps) {
  const int budget = 232448 - (T + 1) * 128 - warps * 2 * 8 - 1024;  // 1 KB static reserve
  int sb = budget / (warps * 2);
  sb = sb - sb % 16;
  if (sb > 4096) sb = 4096;
  // resident targets need room for at least two records per slot; otherwise
  // the kernel gathers targets from L2 with 4 KB staging slots
  if (sb < 2 * max_rec_bytes) return kNonResidentStage;
  return sb;
}

bool lookup_rot2_fits(int stage_bytes, int k) {
  return k >= 2 && k <= kRot2MaxK && rot_records(stage_bytes, 2, k) >= 8;
}

// the kernel instantiations live in separate translation units so that nvcc
// builds them in parallel (lookup_nr.cu, lookup_h16.cu, lookup_w12.cu, lookup_w8.cu)
cudaError_t launch_lookup_r16_2_3(const LookupArgs& a, int grid, int smem, cudaStream_t st) {
  auto kern = lookup_xmap_kernel<true, 0, kLookupWarps, 2, 3>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kLookupWarps * 32, smem, st>>>(a);
  return cudaGetLastError();
}

// 16-warp resident launch: every group of `a` lies in one k range
// (lookup_r16_range), served by its own instantiation unit
cudaError_t launch_lookup_resident16(const LookupArgs& a, int grid, int smem, cudaStream_t st) {
  int kmax = 0;
  for (int g = 0; g < a.ngroups; ++g) kmax = std::max(kmax, a.g_E[g] + 1);
  switch (lookup_r16_range(kmax)) {
    case 0: return launch_lookup_r16_2_3(a, grid, smem, st);
    case 1: return launch_lookup_r16_4_12(a, grid, smem, st);
    case 2: return launch_lookup_r16_13_20(a, grid, smem, st);
    default: return launch_lookup_r16_21_31(a, grid, smem, st);
  }
}

cudaError_t launch_lookup_xmap(const LookupArgs& a, int grid, cudaStream_t st) {
  const bool resident = a.stage_bytes != kNonResidentStage;
  const int warps = !resident ? kNonResWarps : ((!a.h16 && a.warps) ? a.warps : kLookupWarps);
  const int smem = (resident ? (a.T + 1) * 128 : 0) + warps * 2 * a.stage_bytes + warps * 2 * 8;
  count_launch();
  if (!resident) return launch_lookup_nonresident(a, grid, smem, st);
  if (a.h16) return launch_lookup_h16(a, grid, smem, st);
  if (warps == 12) return launch_lookup_w12(a, grid, smem, st);
  if (warps == 8) return launch_lookup_w8(a, grid, smem, st);
  return launch_lookup_resident16(a, grid, smem, st);
}

cudaError_t launch_predict_pairs(const LookupArgs& a, const int4* pairs, int64_t npairs, int64_t c0,
                                 const double* shift, float* pred, int64_t ldp, cudaStream_t st) {
  if (npairs == 0) return cudaSuccess;
  count_launch();
  const int64_t blocks = std::min<int64_t>((npairs + 7) / 8, 148 * 16);
  predict_pairs_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, pairs, npairs, c0, shift, pred, ldp);
  return cudaGetLastError();
}

cudaError_t launch_lookup_fixup(const LookupArgs& a, cudaStream_t st) {
  count_launch();
  lookup_fixup_kernel<<<148 * 8, kFixWarps * 32, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace cmb
