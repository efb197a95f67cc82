// Kernel template of K1/K2 (included by knn_sweep.cu and the width-instantiation
// units knn_w*.cu, which compile in parallel).
#pragma once
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
namespace knn_detail {

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

// A nonzero fp32 sample below 2^-50 can make the squared difference of two
// distinct samples underflow to zero (or lose the relative error model of
// sweep_err_bound), so such a library never takes the fp32 certification:
// library_err returns NaN for it and every row goes through the fp64 path
// (exact re-sort, or exact_row_select).  ADVICE r01.
__device__ __forceinline__ bool tiny_sample(float v) { return v != 0.f && fabsf(v) < 8.881784197001252e-16f; }

// Certification perturbation M of a library: max |x32 - x64| of its series
// (err_m, indexed by series row; 0 for float32 inputs), NaN when tiny.
template <class A>
__device__ __forceinline__ double library_err(const A& a, int64_t srow, bool tiny) {
  if (tiny) return __longlong_as_double(0x7ff8000000000000ll);
  return a.err_m ? (double)a.err_m[srow] : 0.0;
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

// ---------------------------------------------------------------- selection state
// Per warp and dimension index e: a sorted list L_e (up to Kp entries) and an
// unsorted hit buffer B_e (up to kCap entries), counts in shared memory.  The
// sweep tests candidates against a warp-uniform threshold in bulk and appends
// hits; full buffers are merged into the list by a warp bitonic sort + merge
// (compact_lists), which also tightens the threshold.
constexpr int kCap = 32;
constexpr unsigned long long kMaxKey = ~0ull;

// order-preserving key of (distance, index): distances are >= 0
__device__ __forceinline__ unsigned long long pack_key(float d, int j) {
  return ((unsigned long long)__float_as_uint(d) << 32) | (unsigned int)j;
}
__device__ __forceinline__ Entry unpack_key(unsigned long long k) {
  Entry e;
  e.d = __uint_as_float((unsigned int)(k >> 32));
  e.j = (int)(unsigned int)k;
  return e;
}

// ascending bitonic sort of one key per lane
__device__ __forceinline__ unsigned long long warp_sort32(unsigned long long v) {
  const int lane = lane_id();
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const unsigned long long o = __shfl_xor_sync(CMB_FULL, v, stride);
      const bool keep_min = ((lane & stride) == 0) == ((lane & size) == 0);
      v = keep_min ? (o < v ? o : v) : (o > v ? o : v);
    }
  }
  return v;
}

// number of lanes whose key in the ascending lane-sorted S is below x (per lane x)
__device__ __forceinline__ int count_below(unsigned long long S, unsigned long long x) {
  int pos = 0;
#pragma unroll
  for (int step = 16; step > 0; step >>= 1) {
    const unsigned long long sv = __shfl_sync(CMB_FULL, S, pos + step - 1);
    if (sv < x) pos += step;
  }
  const unsigned long long last = __shfl_sync(CMB_FULL, S, 31);
  return pos + ((pos == 31 && last < x) ? 1 : 0);
}

// Merge buffer B[0, bc) into the sorted list L[0, lc); keep the Kp smallest.
// Returns the new list count.  With an empty list this is a plain sort.
static __device__ __noinline__ int compact_lists(Entry* L, Entry* B, int lc, int bc, int Kp) {
  const int lane = lane_id();
  unsigned long long kb = kMaxKey, kl = kMaxKey;
  if (lane < bc) kb = pack_key(B[lane].d, B[lane].j);
  kb = warp_sort32(kb);
  if (lc == 0) {
    __syncwarp();
    if (lane < bc && lane < Kp) L[lane] = unpack_key(kb);
    __syncwarp();
    return min(Kp, bc);
  }
  if (lane < lc) kl = pack_key(L[lane].d, L[lane].j);
  const int rb = lane + count_below(kl, kb);
  const int rl = lane + count_below(kb, kl);
  __syncwarp();
  if (lane < bc && rb < Kp) L[rb] = unpack_key(kb);
  if (lane < lc && rl < Kp) L[rl] = unpack_key(kl);
  __syncwarp();
  return min(Kp, lc + bc);
}

// Tile-kernel hit buffers (knn_tile.cuh): kCap entries per dimension; a RAW
// sweep (one list) uses the first.
__device__ __forceinline__ int tile_buf_off(int mode, int e) { return mode == KNN_RAW ? 0 : e * kCap; }

struct RowCtx {
  int i, L, tau, mode, k_raw;
  uint32_t act;
  unsigned long long* diag;  // [3] hits appended, [4] compactions, [5] hit events
};

__device__ __forceinline__ int k_of(int mode, int k_raw, int e) { return mode == KNN_RAW ? k_raw : e + 2; }
__device__ __forceinline__ int kp_of(int mode, int k_raw, int L, int tau, int e) {
  return min(k_of(mode, k_raw, e) + 1, L - e * tau - 1);
}
__device__ __forceinline__ Entry* list_of(Entry* wl, int mode, int e) {
  return wl + (mode == KNN_RAW ? 0 : list_off(e));
}

// Merge the hit buffer into the list and tighten the shared threshold (out of
// line: rare, and keeps the sweep loop small in the instruction cache).
static __device__ __noinline__ void compact_into(Entry* Le, Entry* Be, int* cnt, float* thr_slot,
                                                 int Kp) {
  const int lc = compact_lists(Le, Be, cnt[0], cnt[1], Kp);
  float t = *thr_slot;
  if (lc == Kp) t = fminf(t, Le[Kp - 1].d);
  __syncwarp();
  if (lane_id() == 0) {
    cnt[0] = lc;
    cnt[1] = 0;
    *thr_slot = t;
  }
  __syncwarp();
}

// One sweep step: kCand x 32 consecutive candidates, every swept dimension.
// Runtime loop over e (xi and thresholds are warp-uniform shared values), so
// the hot loop stays a few hundred bytes of code.  TAIL: candidates may run
// past n_E of the active dimensions and need per-dimension masking.  Hits are
// appended to the dimension's buffer; a buffer holding Kp candidates while
// the list is still empty, or half full, is compacted so the threshold becomes
// exact early.
template <bool TAIL>
__device__ __forceinline__ void sweep_step(const float* __restrict__ xs, int jc, const RowCtx& r,
                                           int eh, const float* __restrict__ xi_w,
                                           float* thr_w, Entry* wl, Entry* wb, int* wc) {
  const int lane = lane_id();
  const unsigned below = (1u << lane) - 1u;
  float d[kCand];
#pragma unroll
  for (int q = 0; q < kCand; ++q) {
    const int j = jc + 32 * q + lane;
    d[q] = (j == r.i || j >= r.L) ? kInfF : 0.f;  // self and past-the-end excluded
  }
  const float* xj = xs + jc + lane;
#pragma unroll 1
  for (int e = 0; e < eh; ++e, xj += r.tau) {
    const float xe = xi_w[e];
#pragma unroll
    for (int q = 0; q < kCand; ++q) {
      const float df = __fsub_rn(xj[32 * q], xe);
      d[q] = __fmaf_rn(df, df, d[q]);
    }
    if ((r.act >> e) & 1u) {
      float dm[kCand];
#pragma unroll
      for (int q = 0; q < kCand; ++q) {
        dm[q] = d[q];
        if (TAIL && jc + 32 * q + lane >= r.L - e * r.tau) dm[q] = kInfF;
      }
      float t = thr_w[e];
      const float mn = fminf(fminf(dm[0], dm[1]), fminf(dm[2], dm[3]));
      if (__any_sync(CMB_FULL, mn < t)) {
        int* c = wc + 2 * e;
        Entry* Be = wb + e * kCap;
        Entry* Le = list_of(wl, r.mode, e);
        const int Kp = kp_of(r.mode, r.k_raw, r.L, r.tau, e);
        int bc = c[1];
#pragma unroll
        for (int q = 0; q < kCand; ++q) {
          unsigned m = __ballot_sync(CMB_FULL, dm[q] < t);
          if (m) {
            if (bc + __popc(m) > kCap) {
              __syncwarp();
              if (lane == 0) c[1] = bc;
              __syncwarp();
              compact_into(Le, Be, c, thr_w + e, Kp);
              bc = 0;
              t = thr_w[e];
              m = __ballot_sync(CMB_FULL, dm[q] < t);
            }
            if ((m >> lane) & 1u) {
              Entry h;
              h.d = dm[q];
              h.j = jc + 32 * q + lane;
              Be[bc + __popc(m & below)] = h;
            }
            bc += __popc(m);
          }
        }
        __syncwarp();
        if (lane == 0) c[1] = bc;
        __syncwarp();
        if (bc >= Kp && (c[0] == 0 || 2 * bc >= kCap)) compact_into(Le, Be, c, thr_w + e, Kp);
      }
    }
  }
}

// Threshold seeding for row i, dimension index e, from row i-1's final list
// shifted by one sample, then state reset.  The seed distances use exactly the
// sweep's fp32 operation sequence, so thr = next float above their maximum is
// a valid upper bound on the list threshold (every seed is collected).
static __device__ __noinline__ void seed_and_reset(Entry* Le, int* cnt, float* thr_slot,
                                                   const float* __restrict__ xs, int i, int e,
                                                   int tau, int nE, int Kp, bool seed) {
  const int lane = lane_id();
  float thr = kInfF;
  if (seed) {
    bool ok = true;
    float ds = -kInfF;
    if (lane < Kp) {
      const int jp = Le[lane].j;
      const int js = jp + 1;
      ok = jp != kNoJ && js < nE && js != i;
      if (ok) {
        float dv = 0.f;
        for (int q = 0; q <= e; ++q) {
          const float df = __fsub_rn(xs[js + q * tau], xs[i + q * tau]);
          dv = __fmaf_rn(df, df, dv);
        }
        ds = dv;
      }
    }
    if (__all_sync(CMB_FULL, ok)) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ds = fmaxf(ds, __shfl_xor_sync(CMB_FULL, ds, o));
      if (ds < kInfF) thr = __int_as_float(__float_as_int(ds) + 1);  // next float above
    }
  }
  __syncwarp();
  if (lane == 0) {
    cnt[0] = 0;
    cnt[1] = 0;
    *thr_slot = thr;
  }
  __syncwarp();
}

// Final merge of the hit buffer into the list (end of row).
static __device__ __noinline__ void finish_list(Entry* Le, Entry* Be, int* cnt, int Kp) {
  const int lc = cnt[0], bc = cnt[1];
  const int n = (bc > 0) ? compact_lists(Le, Be, lc, bc, Kp) : lc;
  __syncwarp();
  if (lane_id() == 0) {
    cnt[0] = n;
    cnt[1] = 0;
  }
  __syncwarp();
  // entries beyond n (fewer candidates than Kp cannot happen: Kp <= nE - 1)
}

struct PredObs {
  double p, o;
};

// Lane-parallel end of row: lane e merges dimension e's hit buffer into its
// list (sequential insertion by (distance, index)) and, in TABLE mode, when the
// fp32 top-k set certifies, computes the fp32 weights and writes the record.
// One lane per dimension keeps all 32 lanes busy instead of k of them.
// Returns the mask of dimensions that still need the warp fp64 path.
template <int E_HI>
static __device__ __noinline__ unsigned lane_finish(const KnnArgs* __restrict__ ap, Entry* wl,
                                                    Entry* wb, int* wc, int lib, int i,
                                                    uint32_t act, double M, bool emit,
                                                    bool tile_layout = false) {
  const KnnArgs& a = *ap;
  const int lane = lane_id();
  const int e = lane;
  bool pending = false;
  if (e < E_HI && ((act >> e) & 1u)) {
    Entry* Le = list_of(wl, a.mode, e);
    const Entry* Be = wb + (tile_layout ? tile_buf_off(a.mode, e) : e * kCap);
    int* c = wc + 2 * e;
    const int Kp = kp_of(a.mode, a.k_raw, a.L, a.tau, e);
    int lc = c[0];
    const int bc = c[1];
    {
      // insertion by (distance, index): binary search for the slot, then an
      // unrolled block move (independent loads/stores pipeline, unlike a
      // compare-and-shift chain whose every step waits on the previous load)
      for (int b = 0; b < bc; ++b) {
        const Entry x = Be[b];
        const unsigned long long key = pack_key(x.d, x.j);
        int n = lc;
        if (lc == Kp) {
          if (key >= pack_key(Le[Kp - 1].d, Le[Kp - 1].j)) continue;
          n = Kp - 1;  // the last entry drops out
        } else {
          ++lc;
        }
        int lo = 0, hi = n;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (pack_key(Le[mid].d, Le[mid].j) < key) lo = mid + 1; else hi = mid;
        }
#pragma unroll 4
        for (int m = n; m > lo; --m) Le[m] = Le[m - 1];
        Le[lo] = x;
      }
    }
    c[0] = lc;
    c[1] = 0;
    if (emit) {
      pending = true;
      if (a.mode == KNN_TABLE) {
        const int E = e + 1;
        const int nE = a.L - e * a.tau;
        const int k = k_of(a.mode, a.k_raw, e);
        const float dk1 = Le[k - 1].d;
        const float dk = Le[min(k, Kp - 1)].d;
        bool ok = !isnan(M) && ((Kp == nE - 1) || (M == 0.0 && dk == 0.f));
        if (!ok && isfinite(dk) && dk > 1e-30f) {
          const double A = dk1, B = dk;
          ok = A + sweep_err_bound(A, E, M) < B - sweep_err_bound(B, E, M);
        }
        if (ok && M != 0.0) {
          // float64 inputs (M > 0): the weights exp(-d_q / d_scale) are as
          // sensitive as the smallest listed distance, so every fp32 distance
          // must be known to 1e-5 relative -- an fp32 zero could be a tiny
          // positive fp64 distance that the reference uses as its scale.  (With
          // M = 0 the bound is < 2e-6 relative and zeros are exact.)
          for (int q = 0; q < k && ok; ++q) {
            const float dq = Le[q].d;
            ok = dq > 0.f && sweep_err_bound(dq, E, M) <= 1e-5 * (double)dq;
          }
        }
        if (ok) {
          // scale: the smallest distance, or the first positive one (knn.py:194-199)
          float scale = sqrtf(Le[0].d);
          if (scale == 0.f) {
            scale = 1.f;
            for (int q = 1; q < k; ++q) {
              const float dq = sqrtf(Le[q].d);
              if (dq > 0.f) { scale = dq; break; }
            }
          }
          // raw weights once (parked in the list entries, whose distances are not
          // needed after this row), then normalised
          const float inv = __fdividef(1.f, scale);
          float tot = 0.f;
          for (int q = 0; q < k; ++q) {
            const float raw = fmaxf(expf(-sqrtf(Le[q].d) * inv), FLT_MIN);
            Le[q].d = raw;
            tot += raw;
          }
          const float itot = __fdividef(1.f, tot);
          uint8_t* rec = a.tab[E] + (size_t)lib * rec_lib_stride(k, nE) + (size_t)i * rec_bytes(k);
          float* wr = reinterpret_cast<float*>(rec);
          uint16_t* rr = reinterpret_cast<uint16_t*>(rec + rec_row_off(k));
          for (int q = 0; q < rec_nw(k); ++q) wr[q] = (q < k) ? Le[q].d * itot : 0.f;
          for (int q = 0; q < rec_nr(k); ++q) rr[q] = (q < k) ? (uint16_t)(Le[q].j + e * a.tau) : (uint16_t)0;
          pending = false;
        }
      }
    }
  }
  const unsigned need = __ballot_sync(CMB_FULL, pending);
  if (a.diag) {
    const unsigned done = __ballot_sync(CMB_FULL, emit && e < E_HI && ((act >> e) & 1u) && !pending);
    if (lane == 0 && done) atomicAdd(a.diag + 1, (unsigned long long)__popc(done));
  }
  return need;
}

// Per-(row, E) epilogue: certification, weights, emission.  Returns the EDIM
// prediction and observation (shifted), zeros otherwise.
template <int E_HI>
__device__ __noinline__ PredObs epilogue_e(const KnnArgs* __restrict__ ap, Entry* Le, int lib, int i,
                                           int e, const double* __restrict__ xp, double M,
                                           double shift) {
  const KnnArgs& a = *ap;
  const int lane = lane_id();
  const int L = a.L, tau = a.tau;
  const int E = e + 1;
  const int nE = L - e * tau;
  const int k = k_of(a.mode, a.k_raw, e);
  const int Kp = kp_of(a.mode, a.k_raw, L, tau, e);
  PredObs po;
  po.p = 0.0;
  po.o = 0.0;
  Entry en;
  en.d = kInfF;
  en.j = kNoJ;
  if (lane < Kp) en = Le[lane];
  const bool full = (Kp == nE - 1);  // every candidate was listed

  // (the fp32 set certification already failed in lane_finish for every row
  // that reaches this path)
  // fp64 path: exact distances of the listed candidates, re-sort, certify
  int jj = (lane < Kp) ? en.j : kNoJ;
  double dd = inf_d();
  if (lane < Kp && jj != kNoJ) dd = exact_sqdist_u<E_HI>(xp, i, jj, E, tau);
  sort_lanes(dd, jj, Kp);
  // list threshold: its largest fp32 distance (the list is sorted, or a heap)
  float t32 = (lane < Kp) ? en.d : -kInfF;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t32 = fmaxf(t32, __shfl_xor_sync(CMB_FULL, t32, o));
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
    uint8_t* rec = a.tab[E] + (size_t)lib * rec_lib_stride(k, nE) + (size_t)i * rec_bytes(k);
    if (lane < rec_nw(k)) reinterpret_cast<float*>(rec)[lane] = (lane < k) ? (float)wgt : 0.f;
    if (lane < rec_nr(k))
      reinterpret_cast<uint16_t*>(rec + rec_row_off(k))[lane] = (lane < k) ? (uint16_t)(jj + e * tau) : (uint16_t)0;
  } else if (a.mode == KNN_EDIM) {
    // prediction of x[i + (E-1)tau + Tp] from the neighbours' futures
    const int off = e * tau + a.Tp;
    const double term = (lane < k) ? wgt * xp[jj + off] : 0.0;
    po.p = warp_sum_d(term) - shift;
    po.o = xp[i + off] - shift;
  } else {  // KNN_RAW: one E only
    if (lane < k) {
      const size_t at = (size_t)i * k + lane;
      a.raw_idx[at] = jj;
      a.raw_w[at] = wgt;
      if (a.raw_d) a.raw_d[at] = dd;
    }
  }
  // keep the exact order in the list for the next row's seeding
  __syncwarp();
  if (lane < Kp) {
    Entry z;
    z.d = (float)dd;
    z.j = jj;
    Le[lane] = z;
  }
  __syncwarp();
  return po;
}

template <int E_HI>
__global__ void __launch_bounds__(kThreads, 3)
knn_sweep_kernel(const __grid_constant__ KnnArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int LT = list_total<E_HI>();
  __shared__ double red[kWarps][E_HI][5];
  __shared__ float thr_s[kWarps][E_HI];
  __shared__ float xi_s[kWarps][E_HI];
  __shared__ int cnt_s[kWarps][E_HI][2];
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
  Entry* bufs = lists + kWarps * LT;
  double* x64s = reinterpret_cast<double*>(bufs + kWarps * E_HI * kCap);
  const int x64n = a.x64_smem ? ((Tfull + 1) & ~1) : 0;
  float* xs = reinterpret_cast<float*>(x64s + x64n);

  // stage the library series (plus zero padding for out-of-range candidates)
  const int span = L + E_HI * tau + kStep + 32;
  bool tiny = false;
  for (int t = threadIdx.x; t < span; t += kThreads) {
    const float v = (t < L) ? gx[t] : 0.f;
    xs[t] = v;
    tiny |= tiny_sample(v);
  }
  tiny = __syncthreads_or(tiny);
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

  const double M = library_err(a, srow, tiny);
  const int e_hi = a.e_hi;
  const int rpw = (a.rows_per_block + kWarps - 1) / kWarps;
  const int r0 = rb * a.rows_per_block + w * rpw;
  const int r1 = min(min(L, rb * a.rows_per_block + a.rows_per_block), r0 + rpw);
  Entry* wl = lists + w * LT;
  Entry* wb = bufs + w * E_HI * kCap;
  int* wc = &cnt_s[w][0][0];

  // per-lane EDIM accumulators for E = lane + 1
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0, acc4 = 0;
  const double shift = (a.mode == KNN_EDIM) ? s_mean : 0.0;

  RowCtx r;
  r.L = L;
  r.tau = tau;
  r.mode = a.mode;
  r.k_raw = a.k_raw;
  r.diag = a.diag;
  uint32_t prev_act = 0;

  // rows r0 - 1 (warm-up, not emitted: seeds the thresholds of row r0) .. r1 - 1
  for (int i = max(0, r0 - 1); i < r1; ++i) {
    const bool emit = i >= r0;
    r.i = i;
    uint32_t act = 0;
    for (int e = 0; e < e_hi; ++e)
      if (((a.need >> e) & 1u) && i < L - e * tau) act |= 1u << e;
    r.act = act;
    if (!act) { prev_act = 0; continue; }
    const int eh = 32 - __clz(act);

    // ---- thresholds seeded from row i-1, lists reset (runtime loop, no unrolling)
#pragma unroll 1
    for (int e = 0; e < eh; ++e) {
      if (!((act >> e) & 1u)) continue;
      seed_and_reset(list_of(wl, r.mode, e), wc + 2 * e, &thr_s[w][e], xs, i, e, tau, L - e * tau,
                     kp_of(r.mode, r.k_raw, L, tau, e), ((prev_act >> e) & 1u) != 0);
    }

    // query coordinates x[i + e tau] as warp-uniform shared values
    if (lane < eh) xi_s[w][lane] = xs[i + lane * tau];
    __syncwarp();

    // ---- fp32 sweep over all candidates, one register-resident chunk at a time
    const int nmin = L - (eh - 1) * tau;
    for (int c0 = 0; c0 < L; c0 += kStep) {
      if (c0 + kStep > nmin)
        sweep_step<true>(xs, c0, r, eh, xi_s[w], thr_s[w], wl, wb, wc);
      else
        sweep_step<false>(xs, c0, r, eh, xi_s[w], thr_s[w], wl, wb, wc);
    }
    __syncwarp();

    // ---- end of row: lane-parallel merge (+ fp32 TABLE records), then the warp
    //      fp64 path for the dimensions that need it
    __syncwarp();
    unsigned need = lane_finish<E_HI>(&a, wl, wb, wc, lib, i, act, M, emit);
    __syncwarp();
#pragma unroll 1
    while (need) {
      const int e = __ffs(need) - 1;
      need &= need - 1;
      const PredObs po = epilogue_e<E_HI>(&a, list_of(wl, r.mode, e), lib, i, e, xp, M, shift);
      if (a.mode == KNN_EDIM && lane == e) {
        acc0 += po.o;
        acc1 += po.p;
        acc2 += po.o * po.o;
        acc3 += po.p * po.p;
        acc4 += po.o * po.p;
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

template <int W>
size_t smem_bytes(const KnnArgs& a) {
  const int Tfull = a.L + a.Tp;
  size_t b = sizeof(Entry) * kWarps * (list_total<W>() + W * kCap);
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

}  // namespace knn_detail
}  // namespace cmb
