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
// order, no fused multiply-add) by one warp per query row with a register
// list.  Every (library, size, sample) is a "pseudo-library": its table is
// written in the cross-map record format (cmb_common.cuh rec_*), and the
// shared-memory-resident lookup of the cross map (lookup.cu) scores all targets
// of the E group against a chunk of pseudo-libraries per launch.
#include "cmb_common.cuh"
#include "kernels.cuh"

#include <float.h>

namespace cmb {

namespace {

__device__ __forceinline__ double inf64() { return __longlong_as_double(0x7ff0000000000000ll); }

// Same selection, one warp per (pseudo-library, row), writing xmap records
// (fp32 weights from the exact fp64 ones, u16 rows idx + (E-1) tau).
// grid: (n_pseudo, ceil(n / 8)); pseudo-library pl = chunk0 + blockIdx.x is
// (library index li, size s, sample q) = ((pl / samples) / n_sizes, ...).
__global__ void restricted_records_kernel(const double* __restrict__ X, int64_t len,
                                          const int32_t* __restrict__ libs, int n, int E, int tau,
                                          int k, const int32_t* __restrict__ pts,
                                          const int64_t* __restrict__ size_off,
                                          const int32_t* __restrict__ sizes, int n_sizes, int samples,
                                          int64_t chunk0, uint8_t* __restrict__ tab) {
  const int lane = lane_id();
  const int row = blockIdx.y * 8 + warp_id();
  const int64_t pl = chunk0 + blockIdx.x;
  if (row >= n) return;
  const int q = (int)(pl % samples);
  const int64_t ls = pl / samples;
  const int s = (int)(ls % n_sizes);
  const int li = (int)(ls / n_sizes);
  const double* x = X + (int64_t)libs[li] * len;
  const int npts = sizes[s];
  const int32_t* S = pts + size_off[s] + (int64_t)q * npts;
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
  const double dist = (lane < k) ? sqrt(dd) : 0.0;
  double scale = __shfl_sync(CMB_FULL, dist, 0);
  if (scale == 0.0) {
    const unsigned pm = __ballot_sync(CMB_FULL, lane < k && dist > 0.0);
    scale = pm ? __shfl_sync(CMB_FULL, dist, __ffs(pm) - 1) : 1.0;
  }
  double raw = 0.0;
  if (lane < k) raw = fmax(exp(-dist / scale), DBL_MIN);
  const double wgt = raw / warp_sum_d(raw);
  uint8_t* rec = tab + (size_t)blockIdx.x * rec_lib_stride(k, n) + (size_t)row * rec_bytes(k);
  if (lane < rec_nw(k)) reinterpret_cast<float*>(rec)[lane] = (lane < k) ? (float)wgt : 0.f;
  if (lane < rec_nr(k))
    reinterpret_cast<uint16_t*>(rec + rec_row_off(k))[lane] = (lane < k) ? (uint16_t)(jj + (E - 1) * tau) : (uint16_t)0;
}

// tau = 1 variant: a warp owns 4 consecutive rows.  Each candidate's window
// x[j .. j + E - 1] is loaded into registers once and serves the 4 rows, whose
// query samples x[row .. row + E + 2] are one sliding register window, so the
// L1 traffic per candidate drops 4x; the distance arithmetic and the selection
// are those of restricted_records_kernel (exact fp64, reference order).
template <int E>
__global__ void __launch_bounds__(256) restricted_records4_kernel(
    const double* __restrict__ X, int64_t len, const int32_t* __restrict__ libs, int n,
    const int32_t* __restrict__ pts, const int64_t* __restrict__ size_off, const int32_t* __restrict__ sizes,
    int n_sizes, int samples, int64_t chunk0, uint8_t* __restrict__ tab) {
  constexpr int R = 4, k = E + 1;
  const int lane = lane_id();
  const int row0 = (blockIdx.y * 8 + warp_id()) * R;
  const int64_t pl = chunk0 + blockIdx.x;
  if (row0 >= n) return;
  const int q = (int)(pl % samples);
  const int64_t ls = pl / samples;
  const int s = (int)(ls % n_sizes);
  const int li = (int)(ls / n_sizes);
  const double* x = X + (int64_t)libs[li] * len;
  const int npts = sizes[s];
  const int32_t* S = pts + size_off[s] + (int64_t)q * npts;
  double qw[R + E - 1];
#pragma unroll
  for (int m = 0; m < R + E - 1; ++m) qw[m] = (row0 + m < len) ? __ldg(x + row0 + m) : 0.0;
  double dd[R], thr[R];
  int jj[R];
#pragma unroll
  for (int r = 0; r < R; ++r) { dd[r] = inf64(); thr[r] = inf64(); jj[r] = 0x7fffffff; }
  for (int c0 = 0; c0 < npts; c0 += 32) {
    const int c = c0 + lane;
    const bool valid = c < npts;
    const int j = valid ? S[c] : 0x7fffffff;
    double w[E];
#pragma unroll
    for (int e = 0; e < E; ++e) w[e] = valid ? __ldg(x + j + e) : 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double D = inf64();
      if (valid && j != row0 + r) {
        double acc = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const double df = __dsub_rn(qw[r + e], w[e]);
          acc = __dadd_rn(acc, __dmul_rn(df, df));
        }
        D = acc;
      }
      unsigned m = __ballot_sync(CMB_FULL, D < thr[r]);
      while (m) {
        const int src = __ffs(m) - 1;
        const double dc = __shfl_sync(CMB_FULL, D, src);
        const int jc = __shfl_sync(CMB_FULL, j, src);
        const double pd = __shfl_up_sync(CMB_FULL, dd[r], 1);
        const int pj = __shfl_up_sync(CMB_FULL, jj[r], 1);
        if (dd[r] > dc) {
          const bool prev = lane > 0 && pd > dc;
          dd[r] = prev ? pd : dc;
          jj[r] = prev ? pj : jc;
        }
        thr[r] = __shfl_sync(CMB_FULL, dd[r], k - 1);
        m &= (src == 31) ? 0u : (~0u << (src + 1));
        m &= __ballot_sync(CMB_FULL, D < thr[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int row = row0 + r;
    if (row >= n) break;
    const double dist = (lane < k) ? sqrt(dd[r]) : 0.0;
    double scale = __shfl_sync(CMB_FULL, dist, 0);
    if (scale == 0.0) {
      const unsigned pm = __ballot_sync(CMB_FULL, lane < k && dist > 0.0);
      scale = pm ? __shfl_sync(CMB_FULL, dist, __ffs(pm) - 1) : 1.0;
    }
    double raw = 0.0;
    if (lane < k) raw = fmax(exp(-dist / scale), DBL_MIN);
    const double wgt = raw / warp_sum_d(raw);
    uint8_t* rec = tab + (size_t)blockIdx.x * rec_lib_stride(k, n) + (size_t)row * rec_bytes(k);
    if (lane < rec_nw(k)) reinterpret_cast<float*>(rec)[lane] = (lane < k) ? (float)wgt : 0.f;
    if (lane < rec_nr(k))
      reinterpret_cast<uint16_t*>(rec + rec_row_off(k))[lane] = (lane < k) ? (uint16_t)(jj[r] + (E - 1)) : (uint16_t)0;
  }
}

}  // namespace

cudaError_t launch_restricted_records(const double* X, int64_t len, const int32_t* libs, int n, int E,
                                      int tau, const int32_t* pts, const int64_t* size_off,
                                      const int32_t* sizes, int n_sizes, int samples, int64_t chunk0,
                                      int64_t n_pseudo, uint8_t* tab, cudaStream_t st) {
  if (n <= 0 || n_pseudo <= 0) return cudaSuccess;
  if (tau == 1 && E <= 20) {
    dim3 grid4((unsigned)n_pseudo, (n + 31) / 32);
    count_launch();
    switch (E) {
#define CMB_E(ee) case ee: restricted_records4_kernel<ee><<<grid4, 256, 0, st>>>(X, len, libs, n, pts, size_off, sizes, n_sizes, samples, chunk0, tab); break;
      CMB_E(1) CMB_E(2) CMB_E(3) CMB_E(4) CMB_E(5) CMB_E(6) CMB_E(7) CMB_E(8) CMB_E(9) CMB_E(10)
      CMB_E(11) CMB_E(12) CMB_E(13) CMB_E(14) CMB_E(15) CMB_E(16) CMB_E(17) CMB_E(18) CMB_E(19) CMB_E(20)
#undef CMB_E
      default: break;
    }
    return cudaGetLastError();
  }
  dim3 grid((unsigned)n_pseudo, (n + 7) / 8);
  count_launch();
  restricted_records_kernel<<<grid, 256, 0, st>>>(X, len, libs, n, E, tau, E + 1, pts, size_off, sizes,
                                                  n_sizes, samples, chunk0, tab);
  return cudaGetLastError();
}

}  // namespace cmb
