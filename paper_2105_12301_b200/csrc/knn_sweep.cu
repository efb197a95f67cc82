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
//   partial_sort_topk    knn.py:144-177   (warp-cooperative lists, ties -> lower j)
//   normalize_to_weights knn.py:180-202
//
// Layout: one CTA = (library, block of rows), 8 warps; one warp = a run of
// consecutive query rows; lanes = candidates j (4 per lane per step, 128 per
// warp: conflict-free shared-memory reads, 4 independent FMA chains).  Every
// needed dimension E keeps a list of k + 1 (distance, index) entries per warp
// in shared memory and a warp-uniform threshold in a register; a ballot
// against the threshold admits candidates, inserted cooperatively (ties keep
// the lower j because candidates arrive in ascending j).  The threshold of row
// i is seeded from row i-1's neighbours shifted by one sample (a valid upper
// bound on the (k+1)-th distance), which removes most list inserts on
// deterministic series.
//
// Exactness.  The sweep runs in FP32 on the CUDA cores (contraction depth
// E <= 30 gives nothing to a tensor core).  err(t) below is a rigorous bound
// on |fp32 sweep distance - reference fp64 distance| ("kNN
// certification").  TABLE mode (cross-map tables, fp32 weights) accepts the
// fp32 top-k set when the k-th and (k+1)-th distances are separated by more
// than the error bounds.  Otherwise -- and always in EDIM/RAW modes, whose
// outputs are fp64 -- the listed candidates' distances are recomputed in fp64
// in the reference's exact operation order, re-sorted by (d64, j), and
// certified against the list threshold; rows that still cannot be certified
// are re-selected by an exact fp64 scan (counted in diagnostics).  Neighbour
// indices therefore equal the reference's in every case.
#include "cmb_common.cuh"
#include "kernels.cuh"

#include <float.h>

namespace cmb {

namespace {

#define kInfF __int_as_float(0x7f800000)
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kCand = 4;                 // candidates per lane per sweep step
constexpr int kStep = 32 * kCand;        // candidates per warp per sweep step
constexpr int kNoJ = 0x7fffffff;

struct __align__(8) Entry {
  float d;
  int j;
};

__device__ __forceinline__ double inf_d() { return __longlong_as_double(0x7ff0000000000000ll); }

// list for dimension index e (E = e + 1) holds up to e + 3 entries (k + 1, k = E + 1)
__host__ __device__ constexpr int list_off(int e) { return e * (e + 5) / 2; }
template <int E_HI>
__host__ __device__ constexpr int list_total() {
  return list_off(E_HI) < 32 ? 32 : list_off(E_HI);
}

// Rigorous bound on |fp32 sweep distance - reference fp64 distance| for a
// candidate whose fp32 distance is t.  u = 2^-24; M = max |x32 - x64|.
__device__ __forceinline__ double sweep_err_bound(double t, int E, double M) {
  const double u = 5.9604644775390625e-08;
  const double gam = E * u / (1.0 - E * u);
  const double e1 = (4.0 * M * sqrt((double)E * t) + 4.0 * E * M * M) * (1.0 + 3.0 * u) + 3.0 * u * t;
  return 1.001 * (gam * (t + e1) + e1) + 1e-15 * t;
}

template <int E_HI>
__device__ __forceinline__ double exact_sqdist_u(const double* x, int i, int j, int E, int tau) {
  double acc = 0.0;
#pragma unroll
  for (int e = 0; e < E_HI; ++e) {
    if (e < E) {
      const double df = __dsub_rn(x[i + e * tau], x[j + e * tau]);
      acc = __dadd_rn(acc, __dmul_rn(df, df));
    }
  }
  return acc;
}

// Exact fp64 selection for one (row, E): scan every candidate, keep the k
// smallest by (distance, index).  Lanes < k end with the sorted list.
template <int E_HI>
__device__ void exact_row_select(const double* x64, int i, int E, int tau, int nE, int k,
                                 double& dd, int& jj) {
  const int lane = lane_id();
  dd = inf_d();
  jj = kNoJ;
  double thr = inf_d();
  for (int jc = 0; jc < nE; jc += 32) {
    const int j = jc + lane;
    double D = inf_d();
    if (j < nE && j != i) D = exact_sqdist_u<E_HI>(x64, i, j, E, tau);
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

// Insert (dc, jn) into the warp's sorted list L[0, Kp); returns the new threshold.
__device__ __forceinline__ float list_insert(Entry* L, int Kp, float dc, int jn) {
  const int lane = lane_id();
  Entry cur;
  cur.d = kInfF;
  cur.j = kNoJ;
  if (lane < Kp) cur = L[lane];
  const float pd = __shfl_up_sync(CMB_FULL, cur.d, 1);
  const int pj = __shfl_up_sync(CMB_FULL, cur.j, 1);
  if (lane < Kp && cur.d > dc) {
    const bool prev = lane > 0 && pd > dc;
    cur.d = prev ? pd : dc;
    cur.j = prev ? pj : jn;
    L[lane] = cur;
  }
  return __shfl_sync(CMB_FULL, cur.d, Kp - 1);
}

struct RowCtx {
  int i, L, tau, mode, k_raw;
  uint32_t act;
};

__device__ __forceinline__ int k_of(const RowCtx& r, int e) { return r.mode == KNN_RAW ? r.k_raw : e + 2; }
__device__ __forceinline__ int kp_of(const RowCtx& r, int e) {
  return min(k_of(r, e) + 1, r.L - e * r.tau - 1);
}
__device__ __forceinline__ Entry* list_of(Entry* wl, const RowCtx& r, int e) {
  return wl + (r.mode == KNN_RAW ? 0 : list_off(e));
}

template <int E_HI, bool CHECK>
__device__ __forceinline__ void sweep_step(const float* __restrict__ xs, int jc, const RowCtx& r,
                                           int eh, const float (&xi)[E_HI], float (&thr)[E_HI],
                                           Entry* wl) {
  const int lane = lane_id();
  float d[kCand];
#pragma unroll
  for (int q = 0; q < kCand; ++q) d[q] = 0.f;
#pragma unroll
  for (int e = 0; e < E_HI; ++e) {
    if (e < eh) {
#pragma unroll
      for (int q = 0; q < kCand; ++q) {
        const float df = __fsub_rn(xs[jc + 32 * q + lane + e * r.tau], xi[e]);
        d[q] = __fmaf_rn(df, df, d[q]);
      }
      if ((r.act >> e) & 1u) {
        const float t = thr[e];
        const int nE = r.L - e * r.tau;
        bool hit = false;
#pragma unroll
        for (int q = 0; q < kCand; ++q) {
          const int j = jc + 32 * q + lane;
          hit |= CHECK ? (d[q] < t && j < nE && j != r.i) : (d[q] < t);
        }
        if (__any_sync(CMB_FULL, hit)) {
          const int Kp = kp_of(r, e);
          Entry* Le = list_of(wl, r, e);
#pragma unroll
          for (int q = 0; q < kCand; ++q) {
            const int j = jc + 32 * q + lane;
            const bool ok = CHECK ? (j < nE && j != r.i) : true;
            unsigned m = __ballot_sync(CMB_FULL, ok && d[q] < thr[e]);
            while (m) {
              const int src = __ffs(m) - 1;
              const float dc = __shfl_sync(CMB_FULL, d[q], src);
              thr[e] = list_insert(Le, Kp, dc, jc + 32 * q + src);
              m &= (src == 31) ? 0u : (~0u << (src + 1));
              m &= __ballot_sync(CMB_FULL, d[q] < thr[e]);
            }
          }
        }
      }
    }
  }
}

template <int E_HI>
__global__ void __launch_bounds__(kThreads, 2)
knn_sweep_kernel(KnnArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int LT = list_total<E_HI>();
  __shared__ double red[kWarps][E_HI][5];
  __shared__ double s_mean;
  __shared__ int s_last;

  const int lib = blockIdx.x / a.nrb;
  const int rb = blockIdx.x - lib * a.nrb;
  const int64_t srow = a.lib_rows ? a.lib_rows[lib] : lib;
  const float* __restrict__ gx = a.x32 + srow * a.ld;
  const double* __restrict__ gx64 = a.x64 + srow * a.ld;
  const int L = a.L, tau = a.tau;
  const int Tfull = L + a.Tp;
  const int lane = lane_id(), w = warp_id();

  Entry* lists = reinterpret_cast<Entry*>(smem);
  double* x64s = reinterpret_cast<double*>(lists + kWarps * LT);
  const int x64n = a.x64_smem ? ((Tfull + 1) & ~1) : 0;
  float* xs = reinterpret_cast<float*>(x64s + x64n);

  // stage the library series (plus zero padding for out-of-range candidates)
  const int span = L + E_HI * tau + kStep + 32;
  for (int t = threadIdx.x; t < span; t += kThreads) xs[t] = (t < L) ? gx[t] : 0.f;
  if (a.x64_smem)
    for (int t = threadIdx.x; t < Tfull; t += kThreads) x64s[t] = gx64[t];
  const double* __restrict__ xp = a.x64_smem ? x64s : gx64;

  // EDIM: series mean (Pearson shift) and position of the last sample change
  if (a.mode == KNN_EDIM) {
    double s = 0.0;
    int last = 0;
    for (int t = threadIdx.x; t < Tfull; t += kThreads) {
      const double v = gx64[t];
      s += v;
      if (t > 0 && v != gx64[t - 1]) last = max(last, t);
    }
    s = warp_sum_d(s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(CMB_FULL, last, o));
    __shared__ double ws[kWarps];
    __shared__ int wl[kWarps];
    if (lane == 0) { ws[w] = s; wl[w] = last; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      int lst = 0;
      for (int q = 0; q < kWarps; ++q) { tot += ws[q]; lst = max(lst, wl[q]); }
      s_mean = tot / Tfull;
      s_last = lst;
    }
  }
  __syncthreads();

  const double M = a.err_m ? (double)a.err_m[lib] : 0.0;
  const int e_hi = a.e_hi;
  const int rpw = (a.rows_per_block + kWarps - 1) / kWarps;
  const int r0 = rb * a.rows_per_block + w * rpw;
  const int r1 = min(min(L, rb * a.rows_per_block + a.rows_per_block), r0 + rpw);
  Entry* wl = lists + w * LT;

  // per-lane EDIM accumulators for E = lane + 1
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0, acc4 = 0;
  const double shift = (a.mode == KNN_EDIM) ? s_mean : 0.0;

  RowCtx r;
  r.L = L;
  r.tau = tau;
  r.mode = a.mode;
  r.k_raw = a.k_raw;
  uint32_t prev_act = 0;

  for (int i = r0; i < r1; ++i) {
    r.i = i;
    uint32_t act = 0;
#pragma unroll
    for (int e = 0; e < E_HI; ++e)
      if (e < e_hi && ((a.need >> e) & 1u) && i < L - e * tau) act |= 1u << e;
    r.act = act;
    if (!act) { prev_act = 0; continue; }
    const int eh = 32 - __clz(act);

    float xi[E_HI], thr[E_HI];
#pragma unroll
    for (int e = 0; e < E_HI; ++e) {
      xi[e] = xs[i + e * tau];
      thr[e] = kInfF;
    }

    // ---- threshold seeding from row i-1's neighbours shifted by one sample,
    //      then list reset
#pragma unroll
    for (int e = 0; e < E_HI; ++e) {
      if (!((act >> e) & 1u)) continue;
      const int Kp = kp_of(r, e);
      const int nE = L - e * tau;
      Entry* Le = list_of(wl, r, e);
      if ((prev_act >> e) & 1u) {
        bool ok = true;
        float ds = -kInfF;
        if (lane < Kp) {
          const int jp = Le[lane].j;
          const int js = jp + 1;
          ok = jp != kNoJ && js < nE && js != i;
          if (ok) {
            float dv = 0.f;
#pragma unroll
            for (int q = 0; q < E_HI; ++q)
              if (q <= e) {
                const float df = __fsub_rn(xs[js + q * tau], xi[q]);
                dv = __fmaf_rn(df, df, dv);
              }
            ds = dv;
          }
        }
        if (__all_sync(CMB_FULL, ok)) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) ds = fmaxf(ds, __shfl_xor_sync(CMB_FULL, ds, o));
          if (ds < kInfF) thr[e] = __int_as_float(__float_as_int(ds) + 1);  // next float above
        }
      }
      __syncwarp();
      if (lane < Kp) {
        Entry z;
        z.d = kInfF;
        z.j = kNoJ;
        Le[lane] = z;
      }
    }
    __syncwarp();

    // ---- fp32 sweep over all candidates
    const int nmin = L - (eh - 1) * tau;
    for (int jc = 0; jc < L; jc += kStep) {
      const bool special = (jc + kStep > nmin) || (i >= jc && i < jc + kStep);
      if (special)
        sweep_step<E_HI, true>(xs, jc, r, eh, xi, thr, wl);
      else
        sweep_step<E_HI, false>(xs, jc, r, eh, xi, thr, wl);
    }
    __syncwarp();

    // ---- per-E epilogue: certify, weights, emit
#pragma unroll
    for (int e = 0; e < E_HI; ++e) {
      if (!((act >> e) & 1u)) continue;
      const int E = e + 1;
      const int nE = L - e * tau;
      const int k = k_of(r, e);
      const int Kp = kp_of(r, e);
      Entry* Le = list_of(wl, r, e);
      Entry en;
      en.d = kInfF;
      en.j = kNoJ;
      if (lane < Kp) en = Le[lane];
      const bool full = (Kp == nE - 1);  // every candidate was listed

      if (a.mode == KNN_TABLE) {
        // fp32 set certification: k-th and (k+1)-th separated beyond the error bounds
        const float dk1 = __shfl_sync(CMB_FULL, en.d, k - 1);
        const float dk = __shfl_sync(CMB_FULL, en.d, min(k, Kp - 1));
        bool ok = full || (M == 0.0 && dk == 0.f);  // exact zeros: only identical vectors
        if (!ok && isfinite(dk) && dk > 1e-30f) {
          const double A = dk1, B = dk;
          ok = A + sweep_err_bound(A, E, M) < B - sweep_err_bound(B, E, M);
        }
        if (ok) {
          const float dist = (lane < k) ? sqrtf(en.d) : 0.f;
          float scale = __shfl_sync(CMB_FULL, dist, 0);
          if (scale == 0.f) {
            const unsigned pm = __ballot_sync(CMB_FULL, lane < k && dist > 0.f);
            scale = pm ? __shfl_sync(CMB_FULL, dist, __ffs(pm) - 1) : 1.f;
          }
          float raw = 0.f;
          if (lane < k) raw = fmaxf(expf(-dist / scale), FLT_MIN);
          float tot = raw;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(CMB_FULL, tot, o);
          const int kp4 = rec_kp4(k), kp8 = rec_kp8(k);
          uint8_t* rec = a.tab[E] + ((size_t)lib * nE + i) * (size_t)rec_bytes(k);
          if (lane < kp4) reinterpret_cast<float*>(rec)[lane] = (lane < k) ? raw / tot : 0.f;
          if (lane < kp8)
            reinterpret_cast<uint16_t*>(rec + 4 * kp4)[lane] =
                (lane < k) ? (uint16_t)(en.j + e * tau) : (uint16_t)0;
          if (lane == 0 && a.diag) atomicAdd(a.diag + 1, 1ull);
          continue;
        }
      }

      // fp64 path: exact distances of the listed candidates, re-sort, certify
      int jj = (lane < Kp) ? en.j : kNoJ;
      double dd = inf_d();
      if (lane < Kp && jj != kNoJ) dd = exact_sqdist_u<E_HI>(xp, i, jj, E, tau);
      sort_lanes(dd, jj, Kp);
      const float t32 = __shfl_sync(CMB_FULL, en.d, Kp - 1);  // list threshold
      bool ok = full || (M == 0.0 && t32 == 0.f);
      if (!ok) {
        const double dk = __shfl_sync(CMB_FULL, dd, k - 1);
        if (isfinite(t32) && t32 > 1e-30f) {
          const double t = (double)t32;
          ok = dk < t - sweep_err_bound(t, E, M);
        }
      }
      if (!ok) {
        exact_row_select<E_HI>(xp, i, E, tau, nE, k, dd, jj);
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
        const double term = (lane < k) ? wgt * xp[jj + off] : 0.0;
        const double p = warp_sum_d(term) - shift;
        const double o = xp[i + off] - shift;
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
      // keep the exact order in the list for the next row's seeding
      if (lane < Kp) {
        Entry z;
        z.d = (float)dd;
        z.j = jj;
        Le[lane] = z;
      }
    }
    prev_act = act;
    __syncwarp();
  }

  if (a.mode == KNN_EDIM) {
    // fixed-order CTA reduction of the per-warp partial moments
    if (lane < E_HI) {
      red[w][lane][0] = acc0;
      red[w][lane][1] = acc1;
      red[w][lane][2] = acc2;
      red[w][lane][3] = acc3;
      red[w][lane][4] = acc4;
    }
    __syncthreads();
    if (threadIdx.x < e_hi * 5) {
      const int e = threadIdx.x / 5, c = threadIdx.x % 5;
      double s = 0.0;
      for (int q = 0; q < kWarps; ++q) s += red[q][e][c];
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
size_t smem_bytes(const KnnArgs& a) {
  const int Tfull = a.L + a.Tp;
  size_t b = sizeof(Entry) * kWarps * list_total<W>();
  if (a.x64_smem) b += sizeof(double) * ((Tfull + 1) & ~1);
  b += sizeof(float) * (size_t)(a.L + W * a.tau + kStep + 32);
  return b;
}

template <int W>
cudaError_t launch_w(const KnnArgs& a, int grid, cudaStream_t st) {
  auto kern = knn_sweep_kernel<W>;
  const size_t smem = smem_bytes<W>(a);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  count_launch();
  kern<<<grid, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

int sweep_width(int e_hi) {
  for (int w : kWidths)
    if (w >= e_hi) return w;
  return -1;
}

cudaError_t launch_knn_sweep(const KnnArgs& a_in, cudaStream_t st) {
  KnnArgs a = a_in;
  const int W = sweep_width(a.e_hi);
  if (W < 0) return cudaErrorInvalidValue;
  const int grid = a.nlib * a.nrb;
  if (grid == 0) return cudaSuccess;
  a.x64_smem = (a.L + a.Tp) <= 6144 ? 1 : 0;
  switch (W) {
#define CMB_W(n) case n: return launch_w<n>(a, grid, st);
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
