// K1/K2: fused delay-embedding distance sweep + exact top-(E+1) selection +
// simplex weights, for every embedding dimension E <= E_HI in one pass.
//
// Replaces, per library series, the reference's materialised n x n distance
// matrix and its per-row argpartition:
//   pairwise_distances   knn.py:97-128   (fused: coordinates read from the raw
//                                          series in shared memory)
//   _self_skill_curve    prediction.py:197-240 (incremental E: one running sum
//                                          per candidate, extended one
//                                          coordinate per E)
//   partial_sort_topk    knn.py:144-177   (warp register lists, ties -> lower j)
//   normalize_to_weights knn.py:180-202   (fp64 weights from exact distances)
//
// Exactness.  The sweep runs in FP32 on the CUDA cores (contraction depth
// E <= 30 gives nothing to a tensor core).  Each per-(row, E) list keeps
// k + 1 candidates ordered by (fp32 distance, index).  The epilogue recomputes
// those candidates' distances in fp64 with the reference's exact operation
// order, re-sorts by (fp64 distance, index), and CERTIFIES the result: every
// candidate outside the list has fp32 distance >= the list threshold t, hence
// fp64 distance >= t - err(t) with err() a rigorous bound on the fp32
// accumulation + input rounding error.  If the k-th fp64 distance is not
// strictly below that bound, the row is re-selected by an exact fp64 scan
// (counted in diagnostics).  Indices are therefore identical to the
// reference's in every case, and weights are the reference's formula on the
// identical fp64 distances.
//
// Layout: one CTA = (library, block of rows); one warp = one query row i;
// lanes = 32 consecutive candidates j (conflict-free shared-memory reads);
// list entry l of dimension E lives in lane l.
#include "cmb_common.cuh"
#include "kernels.cuh"

#include <float.h>

namespace cmb {

namespace {

#define kInfF __int_as_float(0x7f800000)
__device__ __forceinline__ double inf_d() { return __longlong_as_double(0x7ff0000000000000ll); }

// Rigorous bound on |fp32 sweep distance - reference fp64 distance| for a
// candidate whose fp32 distance is t ("kNN certification").
__device__ __forceinline__ double sweep_err_bound(double t, int E, double M) {
  const double u = 5.9604644775390625e-08;  // 2^-24
  const double gam = E * u / (1.0 - E * u);
  const double e1 = (4.0 * M * sqrt((double)E * t) + 4.0 * E * M * M) * (1.0 + 3.0 * u) + 3.0 * u * t;
  return 1.001 * (gam * (t + e1) + e1) + 1e-15 * t;
}

// Exact fp64 selection for one (row, E): scan every candidate, keep the k
// smallest by (distance, index).  lanes < k end with the sorted list.
__device__ void exact_row_select(const double* __restrict__ x64, int i, int E, int tau, int nE,
                                 int k, double& dd, int& jj) {
  const int lane = lane_id();
  dd = inf_d();
  jj = 0x7fffffff;
  double thr = inf_d();
  for (int jc = 0; jc < nE; jc += 32) {
    const int j = jc + lane;
    double D = inf_d();
    if (j < nE && j != i) D = exact_sqdist(x64, i, j, E, tau);
    unsigned m = __ballot_sync(CMB_FULL, D < thr);
    while (m) {
      const int src = __ffs(m) - 1;
      const double dc = __shfl_sync(CMB_FULL, D, src);
      const double pd = __shfl_up_sync(CMB_FULL, dd, 1);
      const int pj = __shfl_up_sync(CMB_FULL, jj, 1);
      if (dd > dc) {
        const bool prev = lane > 0 && pd > dc;
        dd = prev ? pd : dc;
        jj = prev ? pj : jc + src;
      }
      thr = __shfl_sync(CMB_FULL, dd, k - 1);
      m &= (src == 31) ? 0u : (~0u << (src + 1));
      m &= __ballot_sync(CMB_FULL, D < thr);
    }
  }
}

// Odd-even transposition sort of lanes [0, Kp) by (dd, jj); early exit when
// already ordered (the common case: the fp32 order is almost always exact).
__device__ __forceinline__ void sort_lanes(double& dd, int& jj, int Kp) {
  const int lane = lane_id();
  for (int round = 0; round < Kp; ++round) {
    unsigned any = 0;
#pragma unroll
    for (int par = 0; par < 2; ++par) {
      const int partner = ((lane & 1) == par) ? lane + 1 : lane - 1;
      const double od = __shfl_sync(CMB_FULL, dd, partner & 31);
      const int oj = __shfl_sync(CMB_FULL, jj, partner & 31);
      const bool valid = lane < Kp && partner >= 0 && partner < Kp;
      const bool mine_less = dd < od || (dd == od && jj < oj);
      const bool swap = valid && ((lane < partner) ? !mine_less : mine_less);
      if (swap) { dd = od; jj = oj; }
      any |= __ballot_sync(CMB_FULL, swap);
    }
    if (!any) break;
  }
}

template <int E_HI>
__global__ void __launch_bounds__(256)
knn_sweep_kernel(KnnArgs a) {
  extern __shared__ float xs[];
  __shared__ double red[8][E_HI > 0 ? E_HI : 1][5];
  __shared__ double s_mean;
  __shared__ int s_last;

  const int lib = blockIdx.x / a.nrb;
  const int rb = blockIdx.x - lib * a.nrb;
  const int64_t srow = a.lib_rows ? a.lib_rows[lib] : lib;
  const float* __restrict__ gx = a.x32 + srow * a.ld;
  const double* __restrict__ gx64 = a.x64 + srow * a.ld;
  const int L = a.L, tau = a.tau;
  const int lane = lane_id(), w = warp_id(), nw = blockDim.x >> 5;

  // stage the library series (plus zero padding for out-of-range candidates)
  const int span = L + E_HI * tau + 64;
  for (int t = threadIdx.x; t < span; t += blockDim.x) xs[t] = (t < L) ? gx[t] : 0.f;

  // EDIM: series mean (Pearson shift) and position of the last sample change
  if (a.mode == KNN_EDIM) {
    const int Tfull = L + a.Tp;
    double s = 0.0;
    int last = 0;
    for (int t = threadIdx.x; t < Tfull; t += blockDim.x) {
      const double v = gx64[t];
      s += v;
      if (t > 0 && v != gx64[t - 1]) last = max(last, t);
    }
    s = warp_sum_d(s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(CMB_FULL, last, o));
    __shared__ double ws[8];
    __shared__ int wl[8];
    if (lane == 0) { ws[w] = s; wl[w] = last; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      int lst = 0;
      for (int q = 0; q < nw; ++q) { tot += ws[q]; lst = max(lst, wl[q]); }
      s_mean = tot / Tfull;
      s_last = lst;
    }
  }
  __syncthreads();

  const double M = a.err_m ? (double)a.err_m[lib] : 0.0;
  const int e_hi = a.e_hi;
  const int r0 = rb * a.rows_per_block;
  const int r1 = min(L, r0 + a.rows_per_block);

  // per-lane EDIM accumulators for E = lane + 1
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0, acc4 = 0;
  const double shift = (a.mode == KNN_EDIM) ? s_mean : 0.0;

  for (int i = r0 + w; i < r1; i += nw) {
    // dimensions that have row i and are wanted
    uint32_t act = 0;
#pragma unroll
    for (int e = 0; e < E_HI; ++e)
      if (e < e_hi && ((a.need >> e) & 1u) && i < L - e * tau) act |= 1u << e;
    if (!act) continue;
    const int eh = 32 - __clz(act);  // highest active E

    float xi[E_HI], ld[E_HI], thr[E_HI];
    int lj[E_HI];
#pragma unroll
    for (int e = 0; e < E_HI; ++e) {
      xi[e] = xs[i + e * tau];
      ld[e] = kInfF;
      thr[e] = kInfF;
      lj[e] = 0x7fffffff;
    }

    // ---------------- fp32 sweep over all candidates
    for (int jc = 0; jc < L; jc += 32) {
      const int j = jc + lane;
      float d = 0.f;
#pragma unroll
      for (int e = 0; e < E_HI; ++e) {
        if (e < eh) {
          const float df = xs[j + e * tau] - xi[e];
          d = __fmaf_rn(df, df, d);
          if ((act >> e) & 1u) {
            const int nE = L - e * tau;
            const int k = (a.mode == KNN_RAW) ? a.k_raw : e + 2;
            const int Kp = min(k + 1, nE - 1);
            unsigned m = __ballot_sync(CMB_FULL, (d < thr[e]) && (j < nE) && (j != i));
            while (m) {
              const int src = __ffs(m) - 1;
              const float dc = __shfl_sync(CMB_FULL, d, src);
              const float pd = __shfl_up_sync(CMB_FULL, ld[e], 1);
              const int pj = __shfl_up_sync(CMB_FULL, lj[e], 1);
              if (ld[e] > dc) {
                const bool prev = lane > 0 && pd > dc;
                ld[e] = prev ? pd : dc;
                lj[e] = prev ? pj : jc + src;
              }
              thr[e] = __shfl_sync(CMB_FULL, ld[e], Kp - 1);
              m &= (src == 31) ? 0u : (~0u << (src + 1));
              m &= __ballot_sync(CMB_FULL, d < thr[e]);
            }
          }
        }
      }
    }

    // ---------------- per-E epilogue: exact re-rank, certify, weights, emit
#pragma unroll
    for (int e = 0; e < E_HI; ++e) {
      if (!((act >> e) & 1u)) continue;
      const int E = e + 1;
      const int nE = L - e * tau;
      const int k = (a.mode == KNN_RAW) ? a.k_raw : e + 2;
      const int Kp = min(k + 1, nE - 1);
      int jj = lj[e];
      double dd = inf_d();
      if (lane < Kp && jj != 0x7fffffff) dd = exact_sqdist(gx64, i, jj, E, tau);
      if (lane >= Kp) jj = 0x7fffffff;
      sort_lanes(dd, jj, Kp);
      bool ok = (Kp == nE - 1);  // every candidate was listed
      if (!ok) {
        const float t32 = thr[e];
        const double dk = __shfl_sync(CMB_FULL, dd, k - 1);
        if (isfinite(t32) && t32 > 1e-30f) {
          const double t = (double)t32;
          ok = dk < t - sweep_err_bound(t, E, M);
        }
      }
      if (!ok) {
        exact_row_select(gx64, i, E, tau, nE, k, dd, jj);
        if (lane == 0 && a.diag) atomicAdd(a.diag + 0, 1ull);
      }
      if (lane == 0 && a.diag) atomicAdd(a.diag + 1, 1ull);

      // simplex weights (knn.py:194-202) on the exact distances
      const double dist = (lane < k) ? sqrt(dd) : 0.0;
      double scale = __shfl_sync(CMB_FULL, dist, 0);
      if (scale == 0.0) {
        const unsigned pm = __ballot_sync(CMB_FULL, lane < k && dist > 0.0);
        scale = pm ? __shfl_sync(CMB_FULL, dist, __ffs(pm) - 1) : 1.0;
      }
      double raw = 0.0;
      if (lane < k) raw = fmax(exp(-dist / scale), DBL_MIN);
      const double wgt = raw / warp_sum_d(raw);

      if (a.mode == KNN_TABLE) {
        const int kp4 = rec_kp4(k), kp8 = rec_kp8(k);
        uint8_t* rec = a.tab[E] + ((size_t)lib * nE + i) * (size_t)rec_bytes(k);
        if (lane < kp4) reinterpret_cast<float*>(rec)[lane] = (lane < k) ? (float)wgt : 0.f;
        if (lane < kp8)
          reinterpret_cast<uint16_t*>(rec + 4 * kp4)[lane] =
              (lane < k) ? (uint16_t)(jj + e * tau) : (uint16_t)0;
      } else if (a.mode == KNN_EDIM) {
        // prediction of x[i + (E-1)tau + Tp] from the neighbours' futures
        const int off = e * tau + a.Tp;
        const double term = (lane < k) ? wgt * gx64[jj + off] : 0.0;
        const double p = warp_sum_d(term) - shift;
        const double o = gx64[i + off] - shift;
        if (lane == e) {
          acc0 += o;
          acc1 += p;
          acc2 += o * o;
          acc3 += p * p;
          acc4 += o * p;
        }
      } else {  // KNN_RAW: one E only
        if (lane < k) {
          const size_t at = (size_t)i * k + lane;
          a.raw_idx[at] = jj;
          a.raw_w[at] = wgt;
          if (a.raw_d) a.raw_d[at] = dd;
        }
      }
    }
  }

  if (a.mode == KNN_EDIM) {
    // fixed-order CTA reduction of the per-warp partial moments
    if (lane < E_HI) {
      red[w][lane < E_HI ? lane : 0][0] = acc0;
      red[w][lane < E_HI ? lane : 0][1] = acc1;
      red[w][lane < E_HI ? lane : 0][2] = acc2;
      red[w][lane < E_HI ? lane : 0][3] = acc3;
      red[w][lane < E_HI ? lane : 0][4] = acc4;
    }
    __syncthreads();
    if (threadIdx.x < e_hi * 5) {
      const int e = threadIdx.x / 5, c = threadIdx.x % 5;
      double s = 0.0;
      for (int q = 0; q < nw; ++q) s += red[q][e][c];
      a.part[(((size_t)lib * a.nrb + rb) * e_hi + e) * 5 + c] = s;
    }
    if (rb == 0 && threadIdx.x == 0) {
      a.last_change[lib] = s_last;
      a.mean[lib] = s_mean;
    }
  }
}

// instantiated widths; a request rounds up to the next one
constexpr int kWidths[] = {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 24, 28, 30};

template <int W>
cudaError_t launch_w(const KnnArgs& a, int grid, size_t smem, cudaStream_t st) {
  auto kern = knn_sweep_kernel<W>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  count_launch();
  kern<<<grid, 256, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

int sweep_width(int e_hi) {
  for (int w : kWidths)
    if (w >= e_hi) return w;
  return -1;
}

cudaError_t launch_knn_sweep(const KnnArgs& a, cudaStream_t st) {
  const int W = sweep_width(a.e_hi);
  if (W < 0) return cudaErrorInvalidValue;
  const size_t smem = sizeof(float) * (size_t)(a.L + W * a.tau + 64);
  const int grid = a.nlib * a.nrb;
  if (grid == 0) return cudaSuccess;
  switch (W) {
#define CMB_W(n) case n: return launch_w<n>(a, grid, smem, st);
    CMB_W(1) CMB_W(2) CMB_W(3) CMB_W(4) CMB_W(5) CMB_W(6) CMB_W(7) CMB_W(8) CMB_W(9) CMB_W(10)
    CMB_W(11) CMB_W(12) CMB_W(13) CMB_W(14) CMB_W(15) CMB_W(16) CMB_W(17) CMB_W(18) CMB_W(19)
    CMB_W(20) CMB_W(24) CMB_W(28) CMB_W(30)
#undef CMB_W
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------- EDIM finalize
// Merge per-row-block partial moments in fixed order, Pearson per E, then the
// argmax (prediction.py:257-261: strict '>' so ties go to the smaller E; values
// within kTieEps of the best are treated as ties).
__global__ void edim_finalize_kernel(const double* __restrict__ part, const int* __restrict__ last_change,
                                     int nlib, int nrb, int e_hi, int L, int tau, int Tp,
                                     double* __restrict__ rho, int32_t* __restrict__ estar,
                                     const int32_t* __restrict__ valid) {
  const int lib = blockIdx.x * blockDim.x + threadIdx.x;
  if (lib >= nlib) return;
  const double kTieEps = 1e-13;
  int best = 0;
  double bestv = 0.0;
  bool all_def = true;
  for (int e = 0; e < e_hi; ++e) {
    double s[5] = {0, 0, 0, 0, 0};
    for (int r = 0; r < nrb; ++r)
      for (int c = 0; c < 5; ++c) s[c] += part[(((size_t)lib * nrb + r) * e_hi + e) * 5 + c];
    const double n = (double)(L - e * tau);
    const double m2o = s[2] - s[0] * s[0] / n;
    const double m2p = s[3] - s[1] * s[1] / n;
    const double com = s[4] - s[0] * s[1] / n;
    // observed segment x[e*tau + Tp, T) is constant iff no sample changes after it starts
    const bool obs_const = last_change[lib] <= e * tau + Tp;
    double r;
    if (obs_const || !(m2o > 0.0) || !(m2p > 0.0) || n < 2) {
      r = __longlong_as_double(0x7ff8000000000000ll);
      all_def = false;
    } else {
      r = fmin(1.0, fmax(-1.0, com / sqrt(m2o * m2p)));
      if (best == 0 || r > bestv + kTieEps) { best = e + 1; bestv = r; }
    }
    rho[(size_t)lib * e_hi + e] = r;
  }
  if (estar) estar[lib] = (all_def && (!valid || valid[lib])) ? best : 0;
}

cudaError_t launch_edim_finalize(const double* part, const int* last_change, int nlib, int nrb,
                                 int e_hi, int L, int tau, int Tp, double* rho, int32_t* estar,
                                 const int32_t* valid, cudaStream_t st) {
  if (nlib == 0) return cudaSuccess;
  count_launch();
  edim_finalize_kernel<<<(nlib + 127) / 128, 128, 0, st>>>(part, last_change, nlib, nrb, e_hi, L,
                                                             tau, Tp, rho, estar, valid);
  return cudaGetLastError();
}

}  // namespace cmb
