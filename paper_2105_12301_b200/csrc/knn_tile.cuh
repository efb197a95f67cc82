// K1/K2 v6: two-pass register-window tile sweep (tau = 1).
//
// Same contract as knn_sweep_kernel (knn_sweep.cuh) -- every dimension
// E <= E_HI of one library in one pass over the candidates, exact top-(E+1)
// selection, TABLE / EDIM / RAW epilogues -- with a different selection
// strategy, chosen from ncu captures (profiles/r01_*): in v4 the warp-uniform
// threshold seeded from row i-1 was loose for noise-like series, 78% of the
// (step, E) iterations took the ballot/insert path and the sweep ran at
// ~2,500 warp instructions per (row, E); a first fully unrolled tile variant
// cut the work but its 200 KB body stalled on instruction fetch (no_inst 85%),
// so the hot loop here is a ~250-instruction block.
//
// Layout.  A warp owns one query row i at a time.  A tile is 768 candidates;
// lane l owns two runs of 12 consecutive candidates half a tile apart,
// p = tile0 + 12 l + c and p + 384 + c (c < 12).  The candidate window slides
// by one sample per dimension (x[j + e], e = 0..E-1), so a block of four
// dimensions needs only the 15 sample pairs (x[p+m], x[p+384+m]) -- loaded
// once per block into registers from a pair-packed shared copy of the series
// (one pad pair per 4, so the 32 lanes' 8-byte loads are bank-conflict free
// and the offsets are compile-time constants) -- and each dimension is then
// 12 FADD2 + 12 FFMA2 (sm_100 packed fp32) on registers.  Samples past the end
// of the library are +inf, so a candidate's distance becomes +inf exactly at
// the first dimension E with j >= n_E (no tail masking).
//
// Selection, per row:
//   pass 1  distances of all tiles, per lane and dimension the running minimum
//           over its candidates; the threshold t_E = the Kp-th smallest of the
//           32 lane minima (Kp = k + 1 list entries) is an upper bound on the
//           Kp-th smallest distance (Kp distinct lanes each hold a candidate
//           <= t_E).  Rows are independent (no state carries from row i-1).
//   pass 2  distances again; per (tile, E) a lane-min test against t_E, and
//           when some lane has a candidate <= t_E the hitting lanes park their
//           distances in a scratch row and an out-of-line collector appends
//           the hits to the dimension's buffer.
//   end     each buffer is sorted by (distance, index) (warp bitonic) into the
//           list; certification, weights and records are the v4 epilogue.
// Distances use exactly the v4 fp32 operation sequence (sub, then fma
// accumulation in e order; the packed ops round identically), so the
// certification bounds of knn_sweep.cuh apply unchanged.
#pragma once

#include "knn_sweep.cuh"

namespace cmb {
namespace knn_detail {

constexpr int kRun = 12;              // consecutive candidates per run (two runs per lane)
constexpr int kTC = 2 * kRun;         // candidates per lane per tile
constexpr int kHalf = 32 * kRun;      // offset of the second run
constexpr int kTile = 2 * kHalf;      // candidates per warp tile
constexpr int kEB = 4;                // dimensions per unrolled block
constexpr int kNW = kRun + kEB - 1;   // window pairs per block
constexpr int kScrWarp = 800;        // per-warp scratch: carried + tile pool, or E_HI x 33 lane minima

// pair-packed series: pair p = (x[p], x[p + kHalf]) at index zi(p), one pad pair per 4
__device__ __forceinline__ int zi(int p) { return p + (p >> 2); }
__host__ __device__ constexpr int z_len(int n) { return n + (n >> 2) + 1; }
__device__ __forceinline__ float xval(const float2* Z, int p) { return Z[zi(p)].x; }


// ascending bitonic sort of one key per lane over groups of W lanes
template <int W>
__device__ __forceinline__ unsigned long long warp_sortw(unsigned long long v) {
  const int lane = lane_id();
#pragma unroll
  for (int size = 2; size <= W; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const unsigned long long o = __shfl_xor_sync(CMB_FULL, v, stride);
      const bool keep_min = ((lane & stride) == 0) == ((lane & size) == 0);
      v = keep_min ? (o < v ? o : v) : (o > v ? o : v);
    }
  }
  return v;
}

// Merge buffer B[0, bc) (bc <= 32) into the sorted list L[0, lc); keep the Kp
// smallest.  Sort width adapts to the buffer size.
static __device__ __noinline__ int merge_buffer(Entry* L, const Entry* B, int lc, int bc, int Kp) {
  const int lane = lane_id();
  unsigned long long kb = kMaxKey, kl = kMaxKey;
  if (lane < bc) kb = pack_key(B[lane].d, B[lane].j);
  if (bc <= 8) kb = warp_sortw<8>(kb);
  else if (bc <= 16) kb = warp_sortw<16>(kb);
  else kb = warp_sortw<32>(kb);
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

// Thresholds after pass 1, lane-parallel: lane e sorts the 32 lane minima of
// dimension e (mins[e * kMinStride + q]) with a register bitonic network and
// takes the Kp-th smallest.  It is an upper bound on the Kp-th smallest
// distance (Kp distinct lanes each hold a candidate at or below it).  ntp[e] =
// -(next float above t) in both halves: D <= t  <=>  D + ntp < 0 (exact: a
// difference of distinct floats never rounds to zero without flush-to-zero).
constexpr int kMinStride = 33;  // conflict-free transposed reads
static __device__ __noinline__ void lane_min_thresholds(const float* mins, float* thr, float2* ntp,
                                                        uint32_t act, int mode, int k_raw, int L) {
  const int e = lane_id();
  if (e < 32 && ((act >> e) & 1u)) {
    float v[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = mins[e * kMinStride + q];
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const int r = q ^ stride;
          if (r > q) {
            const float lo = fminf(v[q], v[r]), hi = fmaxf(v[q], v[r]);
            const bool up = (q & size) == 0;
            v[q] = up ? lo : hi;
            v[r] = up ? hi : lo;
          }
        }
      }
    }
    const int kp = kp_of(mode, k_raw, L, 1, e);
    // t = v[kp - 1] by a select tree over the bits of kp - 1 (five dependent
    // levels instead of a 31-step chain; ncu: the chain was 2.6% of the stalls)
    const int q1 = kp - 1;
#pragma unroll
    for (int lv = 0; lv < 5; ++lv) {
      const bool hi = (q1 >> lv) & 1;
#pragma unroll
      for (int q = 0; q < (32 >> (lv + 1)); ++q) v[q] = hi ? v[2 * q + 1] : v[2 * q];
    }
    const float t = v[0];
    const float tn = (t < kInfF) ? -__int_as_float(__float_as_int(t) + 1) : -kInfF;
    thr[e] = t;
    ntp[e] = make_float2(tn, tn);
  }
  __syncwarp();
}

// Pool round: each lane takes one pool candidate j (or none; the pool is in
// increasing j), recomputes its distances for every dimension in the sweep's
// exact fp32 operation order, and the warp appends the hits (D_e(j) <= t_e) to
// the dimension buffers by ballot.  Buffer counts live in lane e's register
// (bc); a buffer that would overflow is first merged into its list, which
// tightens the threshold to strictly below the list's last distance.  Buffer
// order is otherwise irrelevant (lane_finish inserts by (distance, index)).
static __device__ __noinline__ int pool_round(const int* pool, int n, const float2* __restrict__ Z,
                                              const float2* nq, float* thr, int* wc, Entry* wl, Entry* wb,
                                              uint32_t act, int eh, int mode, int k_raw, int L, int bc,
                                              unsigned long long* g_stats) {
  const int lane = lane_id();
  const unsigned below = (1u << lane) - 1u;
  const bool valid = lane < n;
  const int j = valid ? pool[lane] : 0;
  float d = valid ? 0.f : kInfF;
  const float2* zj = Z + zi(j);
#pragma unroll 1
  for (int e = 0; e < eh; ++e) {
    const float xv = valid ? Z[zi(j + e)].x : 0.f;
    const float df = __fadd_rn(xv, nq[e].x);
    d = __fmaf_rn(df, df, d);
    unsigned m = __ballot_sync(CMB_FULL, d <= thr[e]);  // inactive dimensions: thr = -1
    if (!m) continue;
    int b0 = __shfl_sync(CMB_FULL, bc, e);
    Entry* Be = wb + tile_buf_off(mode, e);
#ifdef CMB_KNN_STATS
    if (lane == 0 && g_stats) atomicAdd(g_stats + 0, (unsigned long long)__popc(m));
#endif
    if (b0 + __popc(m) > kCap) {
#ifdef CMB_KNN_STATS
      if (lane == 0 && g_stats) atomicAdd(g_stats + 1, 1ull);
#endif
      const int Kp = kp_of(mode, k_raw, L, 1, e);
      Entry* Le = list_of(wl, mode, e);
      const int lc = merge_buffer(Le, Be, wc[2 * e], b0, Kp);
      // pool candidates arrive in increasing j, so once the list is full a later
      // candidate enters only with a strictly smaller distance than its last entry
      float t2 = thr[e];
      if (lc == Kp) {
        const float last = Le[Kp - 1].d;
        const float below = last > 0.f ? __int_as_float(__float_as_int(last) - 1) : -1.f;
        t2 = fminf(t2, below);
      }
      __syncwarp();
      if (lane == 0) {
        wc[2 * e] = lc;
        thr[e] = t2;
      }
      b0 = 0;
      m = __ballot_sync(CMB_FULL, d <= t2);
    }
    if ((m >> lane) & 1u) {
      Entry h;
      h.d = d;
      h.j = j;
      Be[b0 + __popc(m & below)] = h;
    }
    if (lane == e) bc = b0 + __popc(m);
  }
  (void)zj;
  __syncwarp();
  return bc;
}

// Window of one dimension block and the initial distances of the lane's 24
// candidates (pair c = candidates p + c and p + kHalf + c).
__device__ __forceinline__ void block_window(const float2* __restrict__ Z, int zb, int eb,
                                             float2 (&W)[kNW]) {
  const float2* zp = Z + zb + (kEB + 1) * eb;  // zi(p + kEB eb + m) = zb + 5 eb + m + m / 4
#pragma unroll
  for (int m = 0; m < kNW; ++m) W[m] = zp[m + (m >> 2)];
}

__device__ __forceinline__ float tile_min(const float2 (&D)[kRun]) {
  float m[kRun / 3];
#pragma unroll
  for (int q = 0; q < kRun / 3; ++q)
    m[q] = fminf(fminf(fminf(D[3 * q].x, D[3 * q].y), fminf(D[3 * q + 1].x, D[3 * q + 1].y)),
                 fminf(D[3 * q + 2].x, D[3 * q + 2].y));
  return fminf(fminf(m[0], m[1]), fminf(m[2], m[3]));
}

template <int E_HI>
__global__ void __launch_bounds__(kThreads, 2)
knn_tile_kernel(const __grid_constant__ KnnArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int LT = list_total<E_HI>();
  constexpr int EHR = (E_HI + kEB - 1) / kEB * kEB;  // dimensions rounded up to whole blocks
  __shared__ float thr_s[kWarps][E_HI];
  __shared__ float2 nq_s[kWarps][EHR];
  __shared__ float2 ntp_s[kWarps][EHR];
  __shared__ int cnt_s[kWarps][E_HI][2];
  __shared__ double s_mean;
  __shared__ int s_last;

  const int lib = blockIdx.x / a.nrb;
  const int rb = blockIdx.x - lib * a.nrb;
  const int64_t srow = a.lib_rows ? a.lib_rows[lib] : lib;
  const float* __restrict__ gx = a.x32 + srow * a.ld;
  const double* __restrict__ gx64 = a.x64 + srow * a.ld;
  const int L = a.L;
  const int Tfull = L + a.Tp;
  const int lane = lane_id(), w = warp_id();

  Entry* lists = reinterpret_cast<Entry*>(smem);
  Entry* bufs = lists + kWarps * LT;
  float* scratch = reinterpret_cast<float*>(bufs + kWarps * E_HI * kCap);
  // EDIM reduction after the row loop reuses the (then idle) hit buffers
  double (*red)[E_HI][5] = reinterpret_cast<double (*)[E_HI][5]>(bufs);
  double* x64s = reinterpret_cast<double*>(scratch + kWarps * kScrWarp);
  const int x64n = a.x64_smem ? ((Tfull + 1) & ~1) : 0;
  float2* Z = reinterpret_cast<float2*>(x64s + x64n);

  // stage the library series as (x[p], x[p + kHalf]) pairs, +inf past the end
  const int zspan = L + kHalf + 32 + EHR;
  bool tiny = false;
  for (int q = threadIdx.x; q < zspan; q += kThreads) {
    float2 v;
    v.x = (q < L) ? gx[q] : kInfF;
    v.y = (q + kHalf < L) ? gx[q + kHalf] : kInfF;
    Z[zi(q)] = v;
    tiny |= tiny_sample(v.x);
  }
  tiny = __syncthreads_or(tiny);
  if (a.x64_smem)
    for (int t = threadIdx.x; t < Tfull; t += kThreads) x64s[t] = gx64[t];
  const double* __restrict__ xp = a.x64_smem ? x64s : gx64;

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
  // rows interleaved over the warps (no state carries between rows), so the
  // last, partial block of a library keeps all eight warps busy
  const int r0 = rb * a.rows_per_block + w;
  const int r1 = min(L, rb * a.rows_per_block + a.rows_per_block);
  Entry* wl = lists + w * LT;
  Entry* wb = bufs + w * E_HI * kCap;
  float* wscr = scratch + w * kScrWarp;
  float* mins = wscr;  // pass 1 / thresholds: [e][lane] (the scratch is free until pass 2)
  int* wc = &cnt_s[w][0][0];

  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0, acc4 = 0;
  const double shift = (a.mode == KNN_EDIM) ? s_mean : 0.0;

  for (int i = r0; i < r1; i += kWarps) {
    uint32_t act = 0;
    for (int e = 0; e < e_hi; ++e)
      if (((a.need >> e) & 1u) && i < L - e) act |= 1u << e;
    if (!act) continue;
    const int eh = 32 - __clz(act);
    const int nb = (eh + kEB - 1) / kEB;

    // ---- list/buffer reset, query coordinates, pass-1 minima
    if (lane < E_HI) {
      wc[2 * lane] = 0;
      wc[2 * lane + 1] = 0;
      thr_s[w][lane] = ((act >> lane) & 1u) ? kInfF : -1.f;  // inactive: no candidate qualifies
    }
    if (lane < EHR) {
      const float q = (lane < eh) ? xval(Z, i + lane) : 0.f;
      nq_s[w][lane] = make_float2(-q, -q);
      ntp_s[w][lane] = make_float2(kInfF, kInfF);  // inactive dimensions never hit
    }
    for (int e = 0; e < kEB * nb; ++e) mins[e * kMinStride + lane] = kInfF;
    __syncwarp();

    // ---- pass 1: per-lane minima
    for (int tile0 = 0; tile0 < L; tile0 += kTile) {
      const int p = tile0 + kRun * lane;
      const int zb = zi(p);
      float2 D[kRun];
#pragma unroll
      for (int c = 0; c < kRun; ++c) {
        D[c].x = (p + c == i) ? kInfF : 0.f;
        D[c].y = (p + kHalf + c == i) ? kInfF : 0.f;
      }
#pragma unroll 1
      for (int eb = 0; eb < nb; ++eb) {
        float2 W[kNW];
        block_window(Z, zb, eb, W);
        // whole blocks without per-dimension guards: dimensions past eh or
        // outside act compute harmlessly (their minima are never read)
#pragma unroll
        for (int r = 0; r < kEB; ++r) {
          const int e = kEB * eb + r;
          const float2 nq = nq_s[w][e];
#pragma unroll
          for (int c = 0; c < kRun; ++c) {
            const float2 df = __fadd2_rn(W[c + r], nq);
            D[c] = __ffma2_rn(df, df, D[c]);
          }
          mins[e * kMinStride + lane] = fminf(mins[e * kMinStride + lane], tile_min(D));
        }
      }
    }
    __syncwarp();
    // thresholds: Kp-th smallest lane minimum, tightened by the seed
    lane_min_thresholds(mins, thr_s[w], ntp_s[w], act, a.mode, a.k_raw, L);

    // ---- pass 2: per candidate min_E (D_E - t'_E) < 0 marks a hit for some E;
    //      the tile's marked candidates form a pool, processed in 32-lane rounds
    int* pool = reinterpret_cast<int*>(wscr);
    int bcount = 0;  // lane e: entries in dimension e's buffer
    int carry = 0;   // pool entries (< 32) carried into the next tile's rounds
    for (int tile0 = 0; tile0 < L; tile0 += kTile) {
      const int p = tile0 + kRun * lane;
      const int zb = zi(p);
      float2 D[kRun], Mn[kRun];
#pragma unroll
      for (int c = 0; c < kRun; ++c) {
        D[c].x = (p + c == i) ? kInfF : 0.f;
        D[c].y = (p + kHalf + c == i) ? kInfF : 0.f;
        Mn[c] = make_float2(kInfF, kInfF);
      }
#pragma unroll 1
      for (int eb = 0; eb < nb; ++eb) {
        float2 W[kNW];
        block_window(Z, zb, eb, W);
        // whole blocks, two dimensions per min step (FMNMX3); inactive
        // dimensions carry ntp = +inf and never mark
#pragma unroll
        for (int r = 0; r < kEB; r += 2) {
          const int e = kEB * eb + r;
          const float2 nq0 = nq_s[w][e], nq1 = nq_s[w][e + 1];
          const float2 nt0 = ntp_s[w][e], nt1 = ntp_s[w][e + 1];
#pragma unroll
          for (int c = 0; c < kRun; ++c) {
            const float2 df0 = __fadd2_rn(W[c + r], nq0);
            D[c] = __ffma2_rn(df0, df0, D[c]);
            const float2 u0 = __fadd2_rn(D[c], nt0);
            const float2 df1 = __fadd2_rn(W[c + r + 1], nq1);
            D[c] = __ffma2_rn(df1, df1, D[c]);
            const float2 u1 = __fadd2_rn(D[c], nt1);
            Mn[c].x = fminf(Mn[c].x, fminf(u0.x, u1.x));
            Mn[c].y = fminf(Mn[c].y, fminf(u0.y, u1.y));
          }
        }
      }
      // pool of the tile in increasing j: every lane's first-run hits, then second-run hits
      unsigned ha = 0, hb = 0;
#pragma unroll
      for (int c = 0; c < kRun; ++c) {
        ha |= (Mn[c].x < 0.f ? 1u : 0u) << c;
        hb |= (Mn[c].y < 0.f ? 1u : 0u) << c;
      }
      const int na = __popc(ha), nb2 = __popc(hb);
      int ia = na, ib = nb2;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int ua = __shfl_up_sync(CMB_FULL, ia, o);
        const int ub = __shfl_up_sync(CMB_FULL, ib, o);
        if (lane >= o) { ia += ua; ib += ub; }
      }
      const int tot_a = __shfl_sync(CMB_FULL, ia, 31);
      const int total = tot_a + __shfl_sync(CMB_FULL, ib, 31);
      int* da = pool + carry + ia - na;
      while (ha) {
        const int c = __ffs(ha) - 1;
        ha &= ha - 1;
        *da++ = p + c;
      }
      int* db = pool + carry + tot_a + ib - nb2;
      while (hb) {
        const int c = __ffs(hb) - 1;
        hb &= hb - 1;
        *db++ = p + kHalf + c;
      }
      __syncwarp();
#ifdef CMB_KNN_STATS
      if (a.diag && lane == 0) {
        atomicAdd(a.diag + 3, (unsigned long long)total);
        atomicAdd(a.diag + 4, (unsigned long long)((total + 31) / 32));
      }
#endif
      // full rounds now; a remainder waits for the next tile (the pool stays j-ordered)
      const int avail = carry + total;
      const bool last_tile = tile0 + kTile >= L;
      int q0 = 0;
#pragma unroll 1
      for (; q0 + 32 <= avail || (last_tile && q0 < avail); q0 += 32)
        bcount = pool_round(pool + q0, min(32, avail - q0), Z, nq_s[w], thr_s[w], wc, wl, wb, act, eh,
                            a.mode, a.k_raw, L, bcount, a.diag ? a.diag + 5 : nullptr);
      carry = last_tile ? 0 : avail - q0;
      if (carry) {
        const int v = (lane < carry) ? pool[q0 + lane] : 0;
        __syncwarp();
        if (lane < carry) pool[lane] = v;
      }
      __syncwarp();
    }
    if (lane < E_HI) wc[2 * lane + 1] = bcount;
    __syncwarp();

    // ---- certification, weights, records / predictions (v4 epilogue)
    unsigned need = lane_finish<E_HI>(&a, wl, wb, wc, lib, i, act, M, true, true);
    __syncwarp();
#pragma unroll 1
    while (need) {
      const int e = __ffs(need) - 1;
      need &= need - 1;
      const PredObs po = epilogue_e<E_HI>(&a, list_of(wl, a.mode, e), lib, i, e, xp, M, shift);
      if (a.mode == KNN_EDIM && lane == e) {
        acc0 += po.o;
        acc1 += po.p;
        acc2 += po.o * po.o;
        acc3 += po.p * po.p;
        acc4 += po.o * po.p;
      }
    }
    __syncwarp();
  }

  if (a.mode == KNN_EDIM) {
    __syncthreads();  // every warp is done with its hit buffers
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

// dynamic shared memory of the tile kernel for width W and library length L
inline size_t tile_smem_bytes_rt(int W, int L) {
  const int lt = list_off(W) < 32 ? 32 : list_off(W);
  return sizeof(Entry) * kWarps * (size_t)(lt + W * kCap) + sizeof(float) * (kWarps * kScrWarp) +
         sizeof(float2) * (size_t)z_len(L + kHalf + 32 + (W + kEB - 1) / kEB * kEB);
}

template <int W>
size_t tile_smem_bytes(const KnnArgs& a) {
  const int Tfull = a.L + a.Tp;
  size_t b = sizeof(Entry) * kWarps * (list_total<W>() + W * kCap);
  b += sizeof(float) * (kWarps * kScrWarp);
  if (a.x64_smem) b += sizeof(double) * ((Tfull + 1) & ~1);
  b += sizeof(float2) * (size_t)z_len(a.L + kHalf + 32 + (W + kEB - 1) / kEB * kEB);
  return b;
}

template <int W>
cudaError_t launch_tile_w(const KnnArgs& a, int grid, cudaStream_t st) {
  auto kern = knn_tile_kernel<W>;
  const size_t smem = tile_smem_bytes<W>(a);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  count_launch();
  kern<<<grid, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace knn_detail
}  // namespace cmb
