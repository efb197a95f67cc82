// Library-size convergence sweep (kEDM `ccm`).
//
// No reference implementation exists; the semantics are the
// oracle's restatement (oracle/crossmap_oracle.py: ccm_convergence): for each
// library size and random library sample (sorted embedded-point indices drawn
// on the host with the reference's PCG64 convention), every embedded point of
// the library is matched to its k = E + 1 nearest neighbours AMONG THE SAMPLED
// POINTS (self excluded, key (distance, index), knn.py semantics), simplex
// weights follow knn.py:180-202, and every target of the pair list is
// predicted at all points (Tp = 0) and scored with Pearson.
//
// The restricted tables are built exactly in float64 (reference operation
// order, no fused multiply-add) -- the candidate sets are small -- by one warp
// per query row with a register list; the lookup reuses the float64 kernels of
// the public lookup_batch path.
#include "cmb_common.cuh"
#include "kernels.cuh"

#include <float.h>

namespace cmb {

namespace {

__device__ __forceinline__ double inf64() { return __longlong_as_double(0x7ff0000000000000ll); }

// grid: (ceil(n / 8), samples); block 256 = 8 warps, one row each
__global__ void restricted_table_kernel(const double* __restrict__ x, int n, int E, int tau, int k,
                                        const int32_t* __restrict__ pts, int npts,
                                        int64_t* __restrict__ idx_out, double* __restrict__ w_out) {
  const int lane = lane_id();
  const int row = blockIdx.x * 8 + warp_id();
  const int smp = blockIdx.y;
  if (row >= n) return;
  const int32_t* S = pts + (size_t)smp * npts;
  double dd = inf64();
  int jj = 0x7fffffff;
  double thr = inf64();
  for (int c0 = 0; c0 < npts; c0 += 32) {
    const int c = c0 + lane;
    double D = inf64();
    int j = 0x7fffffff;
    if (c < npts) {
      j = S[c];
      if (j != row) {
        double acc = 0.0;
        for (int e = 0; e < E; ++e) {
          const double df = __dsub_rn(__ldg(x + row + e * tau), __ldg(x + j + e * tau));
          acc = __dadd_rn(acc, __dmul_rn(df, df));
        }
        D = acc;
      }
    }
    unsigned m = __ballot_sync(CMB_FULL, D < thr);
    while (m) {
      const int src = __ffs(m) - 1;
      const double dc = __shfl_sync(CMB_FULL, D, src);
      const int jc = __shfl_sync(CMB_FULL, j, src);
      const double pd = __shfl_up_sync(CMB_FULL, dd, 1);
      const int pj = __shfl_up_sync(CMB_FULL, jj, 1);
      if (dd > dc) {
        const bool prev = lane > 0 && pd > dc;
        dd = prev ? pd : dc;
        jj = prev ? pj : jc;
      }
      thr = __shfl_sync(CMB_FULL, dd, k - 1);
      m &= (src == 31) ? 0u : (~0u << (src + 1));
      m &= __ballot_sync(CMB_FULL, D < thr);
    }
  }
  // simplex weights on the exact distances (knn.py:194-202)
  const double dist = (lane < k) ? sqrt(dd) : 0.0;
  double scale = __shfl_sync(CMB_FULL, dist, 0);
  if (scale == 0.0) {
    const unsigned pm = __ballot_sync(CMB_FULL, lane < k && dist > 0.0);
    scale = pm ? __shfl_sync(CMB_FULL, dist, __ffs(pm) - 1) : 1.0;
  }
  double raw = 0.0;
  if (lane < k) raw = fmax(exp(-dist / scale), DBL_MIN);
  const double wgt = raw / warp_sum_d(raw);
  if (lane < k) {
    const size_t at = ((size_t)smp * n + row) * k + lane;
    idx_out[at] = jj;
    w_out[at] = wgt;
  }
}

}  // namespace

cudaError_t launch_restricted_tables(const double* x, int n, int E, int tau, int k, const int32_t* pts,
                                     int npts, int samples, int64_t* idx, double* w, cudaStream_t st) {
  if (n <= 0 || samples <= 0) return cudaSuccess;
  dim3 grid((n + 7) / 8, samples);
  count_launch();
  restricted_table_kernel<<<grid, 256, 0, st>>>(x, n, E, tau, k, pts, npts, idx, w);
  return cudaGetLastError();
}

}  // namespace cmb
