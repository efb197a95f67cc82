// K3: cross-map lookup with fused Pearson skill -- the hot kernel of xmap.
//
// Replaces lookup_batch (prediction.py:122-161) and PearsonAggregate
// (prediction.py:25-79) as called from ccm_pairwise (ccm.py:131-149): for
// every (library, target) pair, predictions
//     p_t = sum_k w[t,k] * y[row[t,k]],  row = idx + (E-1)*tau
// for all n_E embedded points, and rho(y[(E-1)tau + t], p_t).  Only rho
// leaves the SM.
//
// B200 mapping.  A CTA keeps one block of 32 targets (all with the same E*)
// resident in shared memory, time-major: tgt[t][lane] -- T = 1,450 samples x
// 128 B = 185.6 KB of the 227 KB -- so every gathered row is one
// conflict-free 128-byte shared-memory wavefront (lane = target).  Its 16
// warps each stream their own libraries' neighbour tables (records of k
// fp32 weights + k u16 rows) from L2/HBM into a 2-slot shared-memory ring
// with cp.async.bulk (TMA bulk copies) completing on an mbarrier, so table
// bytes are fetched once per (library, target block) and read back as
// broadcast 16-byte shared loads.  Skill is accumulated per lane in fp32 over
// a staging slot and folded into fp64; rho is evaluated in fp64 against the
// precomputed observed-segment moments.
//
// Work items are (E group, library sub-range, target block), handed out by
// an atomic counter so concurrently running CTAs share the same libraries'
// tables in L2.
#include "cmb_common.cuh"
#include "kernels.cuh"

#include <cuda_fp16.h>

namespace cmb {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// shared-memory load at a 32-bit shared address (targets are written only
// before the __syncthreads that opens a work item, so no memory clobber)
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ float2 h2f2(uint32_t u) {
  __half2 h;
  memcpy(&h, &u, 4);
  return __half22float2(h);
}

// 16-bit target words (two targets per lane): raw values whose differences are
// exact, and debias() to the value itself.  MODE 1: fp16.  MODE 2 (q16): each
// biased u16 is placed under the exponent of 2^23 by one PRMT, i.e. the float
// 2^23 + 32768 + v, so differences of raw values are exact integers.
template <int MODE>
__device__ __forceinline__ float2 t16_raw(uint32_t u) {
  if constexpr (MODE == 1) return h2f2(u);
  else
    return make_float2(__uint_as_float(__byte_perm(u, 0x4B000000u, 0x7610)),
                       __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7632)));
}
template <int MODE>
__device__ __forceinline__ float2 t16_debias(float2 f) {
  if constexpr (MODE == 1) return f;
  else return __fadd2_rn(f, make_float2(-8421376.f, -8421376.f));
}

__device__ __forceinline__ void lds_v2(uint32_t addr, float& x, float& y) {
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(addr));
}
__device__ __forceinline__ void lds_v2(uint32_t addr, uint32_t& x, uint32_t& y) {
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(addr));
}

struct WarpStream {
  const uint8_t* base;  // table of the warp's first library
  size_t stride;        // bytes per library table (16-byte multiple)
  int n;                // records per library
  int R;                // record bytes
  int RS;               // records per stage
  int nst;              // stages per library
  int total;            // stages in the stream
};

__device__ __forceinline__ void issue_stage(const WarpStream& ws, int q, uint8_t* slot, uint64_t* bar) {
  const int l = q / ws.nst, s = q - l * ws.nst;
  const int r0 = s * ws.RS;
  const int nrec = min(ws.RS, ws.n - r0);
  // bulk copies move 16-byte multiples; a library's table is padded to 16 bytes
  const uint32_t bytes = (uint32_t)((nrec * ws.R + 15) & ~15);
  const uint8_t* src = ws.base + (size_t)l * ws.stride + (size_t)r0 * ws.R;
  mbar_expect_tx(bar, bytes);
  bulk_g2s(slot, src, bytes, bar);
}

// Prediction of one embedded point from its record in a shared-memory stage
// (used once per library for the accumulation shift below).  y(row) reads the
// lane's target sample; the arithmetic matches the main loop.
template <int K, typename Y>
__device__ __forceinline__ float record_predict(uint32_t rec, Y y) {
  constexpr int RO = rec_row_off(K);
  const auto row = [&](int kk) {
    return __byte_perm(lds_u32(rec + RO + 4 * (kk >> 1)), 0, (kk & 1) ? 0x4432 : 0x4410);
  };
  if constexpr (rec_implicit(K)) {
    const float ylast = y(row(K - 1));
    float p = ylast;
#pragma unroll
    for (int kk = 0; kk < K - 1; ++kk) p = __fmaf_rn(lds_f32(rec + 4 * kk), __fsub_rn(y(row(kk)), ylast), p);
    return p;
  } else {
    float p = 0.f;
#pragma unroll
    for (int kk = 0; kk < K; ++kk) p = __fmaf_rn(lds_f32(rec + 4 * kk), y(row(kk)), p);
    return p;
  }
}

// RESIDENT: targets staged in shared memory with row stride 32; otherwise
// gathered from the time-major global array (row stride ldy) through L1/L2.
template <int K, bool RESIDENT>
__device__ __forceinline__ void warp_libraries(const LookupArgs& a, const float* __restrict__ tgt,
                                               uint8_t* ring, uint64_t* bars, uint32_t& qglob,
                                               int E, int lib0, int nl, int slot_base) {
  constexpr int R = rec_bytes(K);
  constexpr int RO = rec_row_off(K);
  const int64_t stride = RESIDENT ? 32 : a.ldy;
  const int lane = lane_id();
  const int n = a.T - (E - 1) * a.tau;
  const int off = (E - 1) * a.tau;
  WarpStream ws;
  ws.stride = rec_lib_stride(K, n);
  ws.base = a.tab[E] + (size_t)lib0 * ws.stride;
  ws.n = n;
  ws.R = R;
  ws.RS = a.stage_bytes / R;
  ws.nst = (n + ws.RS - 1) / ws.RS;
  ws.total = nl * ws.nst;

  // observed-segment moments of this lane's target
  const int slot = slot_base + lane;
  const int tgt_id = a.slot_tgt[slot];
  const double So = a.obs_s[slot], Soo = a.obs_ss[slot];
  const bool ocst = a.obs_const[slot] != 0;
  const float* __restrict__ tcol = tgt + lane;
  const uint32_t tbase = RESIDENT ? smem_u32(tcol) : 0u;

  // prologue: two stages in flight
  if (lane == 0) {
    for (int q = 0; q < 2 && q < ws.total; ++q) {
      const uint32_t g = qglob + q;
      issue_stage(ws, q, ring + (g & 1) * a.stage_bytes, bars + (g & 1));
    }
  }
  __syncwarp();

  // Moments are accumulated about a per-(library, target) shift, the prediction
  // of the library's first point: m2p and the comoment are shift-invariant, and
  // a near-constant prediction (e.g. from a constant library) would otherwise
  // cancel catastrophically in sum p^2 - (sum p)^2 / n.
  double Sp = 0.0, Spp = 0.0, Sop = 0.0;
  float shift = 0.f;
  for (int q = 0; q < ws.total; ++q) {
    const uint32_t g = qglob + q;
    uint8_t* slotp = ring + (g & 1) * a.stage_bytes;
    const int l = q / ws.nst, s = q - l * ws.nst;
    mbar_wait(bars + (g & 1), (g >> 1) & 1);
    const uint32_t slot_s = smem_u32(slotp);
    if (s == 0) {
      if (RESIDENT)
        shift = record_predict<K>(slot_s, [&](uint32_t row) { return lds_f32(tbase + (row << 7)); });
      else
        shift = record_predict<K>(slot_s, [&](uint32_t row) { return tcol[(int64_t)row * stride]; });
    }
    const int r0 = s * ws.RS;
    const int nrec = min(ws.RS, n - r0);
    float sp = 0.f, spp = 0.f, sop = 0.f;
    // non-resident gathers come from L2: unroll over points so enough independent
    // loads are in flight (small k would otherwise leave the warp latency-bound)
    constexpr int UNR = RESIDENT ? 2 : (K <= 3 ? 8 : (K <= 8 ? 4 : 2));
#pragma unroll UNR
    for (int r = 0; r < nrec; ++r) {
      const uint32_t rec = slot_s + r * R;
      // broadcast reads as 8-byte loads (one shared wavefront each; a
      // broadcast 16-byte load costs two, so keep the compiler from merging)
      float wv[2 * ((K + 1) / 2)];
      uint32_t rv[2 * ((K + 3) / 4)];
      float o, p = -shift;
      if constexpr (K == 2) {
        // [w0][r0 r1]: the last weight is 1 - w0, p = y1 + w0 (y0 - y1)
        uint32_t u0;
        lds_v2(rec, u0, rv[0]);
        wv[0] = __uint_as_float(u0);
      } else {
#pragma unroll
        // weights used: k (explicit) or k - 1 (implicit last weight)
        for (int c = 0; c < ((rec_implicit(K) ? K - 1 : K) + 1) / 2; ++c)
          lds_v2(rec + 8 * c, wv[2 * c], wv[2 * c + 1]);
#pragma unroll
        for (int c = 0; c < (K + 3) / 4; ++c) lds_v2(rec + RO + 8 * c, rv[2 * c], rv[2 * c + 1]);
      }
      if constexpr (rec_implicit(K)) {
        // k - 1 stored weights, the last implied: p = y_last + sum w_q (y_q - y_last)
        float yv[K];
        if (RESIDENT) {
          // 32-bit shared addresses: byte offset of sample row s is s << 7
          o = lds_f32(tbase + ((uint32_t)(off + r0 + r) << 7));
#pragma unroll
          for (int kk = 0; kk < K; ++kk) {
            const uint32_t row = __byte_perm(rv[kk >> 1], 0, (kk & 1) ? 0x4432 : 0x4410);
            yv[kk] = lds_f32(tbase + (row << 7));
          }
        } else {
          o = tcol[(int64_t)(off + r0 + r) * stride];
#pragma unroll
          for (int kk = 0; kk < K; ++kk) {
            const uint32_t row = __byte_perm(rv[kk >> 1], 0, (kk & 1) ? 0x4432 : 0x4410);
            yv[kk] = tcol[(int64_t)row * stride];
          }
        }
        p = __fsub_rn(yv[K - 1], shift);
#pragma unroll
        for (int kk = 0; kk < K - 1; ++kk) p = __fmaf_rn(wv[kk], __fsub_rn(yv[kk], yv[K - 1]), p);
      } else if (RESIDENT) {
        o = lds_f32(tbase + ((uint32_t)(off + r0 + r) << 7));
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
          const uint32_t row = __byte_perm(rv[kk >> 1], 0, (kk & 1) ? 0x4432 : 0x4410);
          p = __fmaf_rn(wv[kk], lds_f32(tbase + (row << 7)), p);
        }
      } else {
        o = tcol[(int64_t)(off + r0 + r) * stride];
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
          const uint32_t row = __byte_perm(rv[kk >> 1], 0, (kk & 1) ? 0x4432 : 0x4410);
          p = __fmaf_rn(wv[kk], tcol[(int64_t)row * stride], p);
        }
      }
      sp += p;
      spp = __fmaf_rn(p, p, spp);
      sop = __fmaf_rn(o, p, sop);
    }
    Sp += sp;
    Spp += spp;
    Sop += sop;
    __syncwarp();
    if (lane == 0 && q + 2 < ws.total) issue_stage(ws, q + 2, slotp, bars + (g & 1));
    if (s == ws.nst - 1) {
      // library complete: skill of (library, this lane's target)
      const double nn = (double)n;
      const double m2o = Soo - So * So / nn;
      const double m2p = Spp - Sp * Sp / nn;
      const double com = Sop - So * Sp / nn;
      float r = __int_as_float(0x7fc00000);
      if (!ocst && m2o > 0.0 && m2p > 0.0) r = (float)fmin(1.0, fmax(-1.0, com / sqrt(m2o * m2p)));
      if (tgt_id >= 0) a.rhoT[(size_t)tgt_id * a.ldr + a.lib_col[lib0 + l]] = r;
      Sp = Spp = Sop = 0.0;
    }
  }
  qglob += ws.total;
}

// Prediction of one point from its record in a shared-memory stage: the
// arithmetic of warp_libraries (shift folded into the first operation); y(row)
// gathers the lane's target sample (shared memory when resident, else L1/L2).
template <int K, typename Y>
__device__ __forceinline__ float rec_predict(uint32_t rec, Y y, float shift) {
  constexpr int RO = rec_row_off(K);
  float wv[2 * ((K + 1) / 2)];
  uint32_t rv[2 * ((K + 3) / 4)];
  if constexpr (K == 2) {
    uint32_t u0;
    lds_v2(rec, u0, rv[0]);
    wv[0] = __uint_as_float(u0);
  } else {
#pragma unroll
    for (int c = 0; c < ((rec_implicit(K) ? K - 1 : K) + 1) / 2; ++c) lds_v2(rec + 8 * c, wv[2 * c], wv[2 * c + 1]);
#pragma unroll
    for (int c = 0; c < (K + 3) / 4; ++c) lds_v2(rec + RO + 8 * c, rv[2 * c], rv[2 * c + 1]);
  }
  if constexpr (rec_implicit(K)) {
    float yv[K];
#pragma unroll
    for (int kk = 0; kk < K; ++kk) yv[kk] = y(__byte_perm(rv[kk >> 1], 0, (kk & 1) ? 0x4432 : 0x4410));
    float p = __fsub_rn(yv[K - 1], shift);
#pragma unroll
    for (int kk = 0; kk < K - 1; ++kk) p = __fmaf_rn(wv[kk], __fsub_rn(yv[kk], yv[K - 1]), p);
    return p;
  } else {
    float p = -shift;
#pragma unroll
    for (int kk = 0; kk < K; ++kk) p = __fmaf_rn(wv[kk], y(__byte_perm(rv[kk >> 1], 0, (kk & 1) ? 0x4432 : 0x4410)), p);
    return p;
  }
}

__device__ __forceinline__ float pair_rho(double So, double Soo, bool ocst, double Sp, double Spp, double Sop,
                                          int n) {
  const double nn = (double)n;
  const double m2o = Soo - So * So / nn;
  const double m2p = Spp - Sp * Sp / nn;
  const double com = Sop - So * Sp / nn;
  float r = __int_as_float(0x7fc00000);
  if (!ocst && m2o > 0.0 && m2p > 0.0) r = (float)fmin(1.0, fmax(-1.0, com / sqrt(m2o * m2p)));
  return r;
}

// Libraries in lockstep (resident targets), NL = 2 or 4 at a time: each stage
// slot holds the same record range of libraries l .. l + NL - 1 in NL parts,
// and every point's observed value -- one shared-memory wavefront -- serves
// all NL predictions; the libraries' moment sums are packed FADD2/FFMA2 pairs.
// For k = 2 (E* = 1, half the targets of the mixed data) pairs take 7 instead
// of 8 wavefronts and 27.5 instead of 34 instructions per point pair.  Each
// library's arithmetic is warp_libraries' (rho differs from the single path
// only through the fp32 per-stage grouping of the moment sums).
template <int K, bool RESIDENT, int NL>
__device__ __forceinline__ void warp_library_group(const LookupArgs& a, const float* __restrict__ tgt,
                                                   uint8_t* ring, uint64_t* bars, uint32_t& qglob,
                                                   int E, int lib0, int ngroup, int slot_base) {
  static_assert(NL == 2 || NL == 4, "libraries per group");
  constexpr int R = rec_bytes(K);
  const int lane = lane_id();
  const int n = a.T - (E - 1) * a.tau;
  const int off = (E - 1) * a.tau;
  const size_t lstride = rec_lib_stride(K, n);
  const uint8_t* base = a.tab[E] + (size_t)lib0 * lstride;
  const int part = (a.stage_bytes / NL) & ~15;
  const int RS = part / R;
  const int nst = (n + RS - 1) / RS;
  const int total = ngroup * nst;

  const int slot = slot_base + lane;
  const int tgt_id = a.slot_tgt[slot];
  const double So = a.obs_s[slot], Soo = a.obs_ss[slot];
  const bool ocst = a.obs_const[slot] != 0;
  const float* __restrict__ tcol = tgt + lane;
  const int64_t stride = RESIDENT ? 32 : a.ldy;
  const uint32_t tbase = RESIDENT ? smem_u32(tcol) : 0u;
  const auto y = [&](uint32_t row) {
    if constexpr (RESIDENT) return lds_f32(tbase + (row << 7));
    else return tcol[(int64_t)row * stride];
  };

  auto issue = [&](int q, uint8_t* dst, uint64_t* bar) {
    const int lg = q / nst, s = q - lg * nst;
    const int r0 = s * RS;
    const int nrec = min(RS, n - r0);
    const uint32_t bytes = (uint32_t)((nrec * R + 15) & ~15);
    const uint8_t* src = base + (size_t)(NL * lg) * lstride + (size_t)r0 * R;
    mbar_expect_tx(bar, NL * bytes);
#pragma unroll
    for (int h = 0; h < NL; ++h) bulk_g2s(dst + h * part, src + h * lstride, bytes, bar);
  };
  if (lane == 0) {
    for (int q = 0; q < 2 && q < total; ++q) {
      const uint32_t g = qglob + q;
      issue(q, ring + (g & 1) * a.stage_bytes, bars + (g & 1));
    }
  }
  __syncwarp();

  double Sp[NL], Spp[NL], Sop[NL];
  float sh[NL];
#pragma unroll
  for (int h = 0; h < NL; ++h) Sp[h] = Spp[h] = Sop[h] = 0.0, sh[h] = 0.f;
  for (int q = 0; q < total; ++q) {
    const uint32_t g = qglob + q;
    uint8_t* slotp = ring + (g & 1) * a.stage_bytes;
    const int lg = q / nst, s = q - lg * nst;
    mbar_wait(bars + (g & 1), (g >> 1) & 1);
    const uint32_t s0 = smem_u32(slotp);
    if (s == 0) {  // per-library shifts (see warp_libraries)
#pragma unroll
      for (int h = 0; h < NL; ++h) sh[h] = rec_predict<K>(s0 + h * part, y, 0.f);
    }
    const int r0 = s * RS;
    const int nrec = min(RS, n - r0);
    float2 sp[NL / 2], spp[NL / 2], sop[NL / 2];
#pragma unroll
    for (int h = 0; h < NL / 2; ++h) sp[h] = spp[h] = sop[h] = make_float2(0.f, 0.f);
    // non-resident gathers come from L2: unroll over points for loads in flight
    constexpr int UNR = RESIDENT ? 2 : (K <= 3 ? 4 : 2);
#pragma unroll UNR
    for (int r = 0; r < nrec; ++r) {
      const float o = y((uint32_t)(off + r0 + r));
#pragma unroll
      for (int h = 0; h < NL / 2; ++h) {
        const float2 p = make_float2(rec_predict<K>(s0 + (2 * h) * part + r * R, y, sh[2 * h]),
                                     rec_predict<K>(s0 + (2 * h + 1) * part + r * R, y, sh[2 * h + 1]));
        sp[h] = __fadd2_rn(sp[h], p);
        spp[h] = __ffma2_rn(p, p, spp[h]);
        sop[h] = __ffma2_rn(make_float2(o, o), p, sop[h]);
      }
    }
#pragma unroll
    for (int h = 0; h < NL / 2; ++h) {
      Sp[2 * h] += sp[h].x;
      Spp[2 * h] += spp[h].x;
      Sop[2 * h] += sop[h].x;
      Sp[2 * h + 1] += sp[h].y;
      Spp[2 * h + 1] += spp[h].y;
      Sop[2 * h + 1] += sop[h].y;
    }
    __syncwarp();
    if (lane == 0 && q + 2 < total) issue(q + 2, slotp, bars + (g & 1));
    if (s == nst - 1) {
      if (tgt_id >= 0) {
        float* dst = a.rhoT + (size_t)tgt_id * a.ldr;
#pragma unroll
        for (int h = 0; h < NL; ++h) dst[a.lib_col[lib0 + NL * lg + h]] = pair_rho(So, Soo, ocst, Sp[h], Spp[h], Sop[h], n);
      }
#pragma unroll
      for (int h = 0; h < NL; ++h) Sp[h] = Spp[h] = Sop[h] = 0.0;
    }
  }
  qglob += total;
}

// fp16-target variant (opt-in, CMB_LOOKUP_FP16=1): the resident block holds 64
// targets as fp16 scaled to [-1, 1] -- the same 128 bytes per sample row -- and
// lane l owns targets 2l and 2l + 1, so every shared-memory wavefront (gathers,
// record broadcasts, observed values) serves 64 pairs instead of 32.  Values are
// widened to fp32 and accumulated with packed FFMA2; rho as in the fp32 path.
template <int K, int MODE>
__device__ __forceinline__ void warp_libraries_h16(const LookupArgs& a, const uint8_t* tgt,
                                                   uint8_t* ring, uint64_t* bars, uint32_t& qglob,
                                                   int E, int lib0, int nl, int slot_base) {
  constexpr int R = rec_bytes(K);
  constexpr int RO = rec_row_off(K);
  const int lane = lane_id();
  const int n = a.T - (E - 1) * a.tau;
  const int off = (E - 1) * a.tau;
  WarpStream ws;
  ws.stride = rec_lib_stride(K, n);
  ws.base = a.tab[E] + (size_t)lib0 * ws.stride;
  ws.n = n;
  ws.R = R;
  ws.RS = a.stage_bytes / R;
  ws.nst = (n + ws.RS - 1) / ws.RS;
  ws.total = nl * ws.nst;

  int tid[2];
  double So[2], Soo[2];
  bool ocst[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int slot = slot_base + 2 * lane + h;
    tid[h] = a.slot_tgt[slot];
    So[h] = a.obs_s[slot];
    Soo[h] = a.obs_ss[slot];
    ocst[h] = a.obs_const[slot] != 0;
  }
  const uint32_t tbase = smem_u32(tgt) + 4 * lane;

  if (lane == 0) {
    for (int q = 0; q < 2 && q < ws.total; ++q) {
      const uint32_t g = qglob + q;
      issue_stage(ws, q, ring + (g & 1) * a.stage_bytes, bars + (g & 1));
    }
  }
  __syncwarp();

  // prediction of one point from its record (debiased values); the moments
  // are accumulated about the library's first prediction as in warp_libraries
  const auto predict = [&](uint32_t rec) {
    float wv[2 * ((K + 1) / 2)];
    uint32_t rv[2 * ((K + 3) / 4)];
    if constexpr (K == 2) {
      uint32_t u0;
      lds_v2(rec, u0, rv[0]);
      wv[0] = __uint_as_float(u0);
    } else {
#pragma unroll
      for (int c = 0; c < ((rec_implicit(K) ? K - 1 : K) + 1) / 2; ++c)
        lds_v2(rec + 8 * c, wv[2 * c], wv[2 * c + 1]);
#pragma unroll
      for (int c = 0; c < (K + 3) / 4; ++c) lds_v2(rec + RO + 8 * c, rv[2 * c], rv[2 * c + 1]);
    }
    float2 p;
    if constexpr (rec_implicit(K)) {
      float2 yv[K];
#pragma unroll
      for (int kk = 0; kk < K; ++kk) {
        const uint32_t row = __byte_perm(rv[kk >> 1], 0, (kk & 1) ? 0x4432 : 0x4410);
        yv[kk] = t16_raw<MODE>(lds_u32(tbase + (row << 7)));
      }
      p = t16_debias<MODE>(yv[K - 1]);
#pragma unroll
      for (int kk = 0; kk < K - 1; ++kk) {
        const float2 d = make_float2(__fsub_rn(yv[kk].x, yv[K - 1].x), __fsub_rn(yv[kk].y, yv[K - 1].y));
        p = __ffma2_rn(make_float2(wv[kk], wv[kk]), d, p);
      }
    } else {
      p = make_float2(0.f, 0.f);
#pragma unroll
      for (int kk = 0; kk < K; ++kk) {
        const uint32_t row = __byte_perm(rv[kk >> 1], 0, (kk & 1) ? 0x4432 : 0x4410);
        p = __ffma2_rn(make_float2(wv[kk], wv[kk]), t16_debias<MODE>(t16_raw<MODE>(lds_u32(tbase + (row << 7)))), p);
      }
    }
    return p;
  };

  double Sp0 = 0, Sp1 = 0, Spp0 = 0, Spp1 = 0, Sop0 = 0, Sop1 = 0;
  float2 nshift = make_float2(0.f, 0.f);
  for (int q = 0; q < ws.total; ++q) {
    const uint32_t g = qglob + q;
    uint8_t* slotp = ring + (g & 1) * a.stage_bytes;
    mbar_wait(bars + (g & 1), (g >> 1) & 1);
    const uint32_t slot_s = smem_u32(slotp);
    const int l = q / ws.nst, s = q - l * ws.nst;
    if (s == 0) {
      const float2 f = predict(slot_s);
      nshift = make_float2(-f.x, -f.y);
    }
    const int r0 = s * ws.RS;
    const int nrec = min(ws.RS, n - r0);
    float2 sp = make_float2(0.f, 0.f), spp = sp, sop = sp;
#pragma unroll 2
    for (int r = 0; r < nrec; ++r) {
      const float2 o = t16_debias<MODE>(t16_raw<MODE>(lds_u32(tbase + ((uint32_t)(off + r0 + r) << 7))));
      // the shift is subtracted from the complete prediction, so a prediction
      // equal to the library's first one contributes exactly zero
      const float2 p = __fadd2_rn(predict(slot_s + r * R), nshift);
      sp = __fadd2_rn(sp, p);
      spp = __ffma2_rn(p, p, spp);
      sop = __ffma2_rn(o, p, sop);
    }
    Sp0 += sp.x; Sp1 += sp.y;
    Spp0 += spp.x; Spp1 += spp.y;
    Sop0 += sop.x; Sop1 += sop.y;
    __syncwarp();
    if (lane == 0 && q + 2 < ws.total) issue_stage(ws, q + 2, slotp, bars + (g & 1));
    if (s == ws.nst - 1) {
      const double nn = (double)n;
      const double Sp[2] = {Sp0, Sp1}, Spp[2] = {Spp0, Spp1}, Sop[2] = {Sop0, Sop1};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double m2o = Soo[h] - So[h] * So[h] / nn;
        const double m2p = Spp[h] - Sp[h] * Sp[h] / nn;
        const double com = Sop[h] - So[h] * Sp[h] / nn;
        float rr = __int_as_float(0x7fc00000);
        if (!ocst[h] && m2o > 0.0 && m2p > 0.0) rr = (float)fmin(1.0, fmax(-1.0, com / sqrt(m2o * m2p)));
        if (tid[h] >= 0) a.rhoT[(size_t)tid[h] * a.ldr + a.lib_col[lib0 + l]] = rr;
      }
      Sp0 = Sp1 = Spp0 = Spp1 = Sop0 = Sop1 = 0.0;
    }
  }
  qglob += ws.total;
}

constexpr int kPairMaxK = 31;  // library pairs for every k (A/B: k <= 8 5.83 s, all 5.81 s)
// non-resident targets (T past shared memory): pairs measured neutral at
// N = 1,024, T = 10,000 (81.2 vs 80.8 ms, L2-latency-bound gathers), so off
constexpr int kPairMaxKL2 = 1;
constexpr int kQuadMaxK = 4;  // four libraries in lockstep for k <= 4

template <bool RESIDENT, int H16>
__global__ void __launch_bounds__(kLookupWarps * 32, 1) lookup_xmap_kernel(LookupArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  float* tgt = reinterpret_cast<float*>(smem);
  const size_t tgt_bytes = RESIDENT ? (size_t)a.T * 128 : 0;
  uint8_t* rings = smem + tgt_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(rings + (size_t)kLookupWarps * 2 * a.stage_bytes);
  __shared__ int64_t s_item;

  const int lane = lane_id(), w = warp_id();
  if (threadIdx.x < kLookupWarps * 2) mbar_init(bars + threadIdx.x, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  uint8_t* ring = rings + (size_t)w * 2 * a.stage_bytes;
  uint64_t* wbars = bars + 2 * w;
  uint32_t qglob = 0;

  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(a.counter, 1);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= a.n_items) break;
    int g = 0;
    while (g + 1 < a.ngroups && a.g_item0[g + 1] <= item) ++g;
    const int64_t rem = item - a.g_item0[g];
    const int nblk = a.g_nblk[g];
    const int lsub = (int)(rem / nblk);
    const int blk = a.g_blk0[g] + (int)(rem - (int64_t)lsub * nblk);
    const int E = a.g_E[g];

    // stage the target block (32 fp32 or 64 fp16 targets: 128 bytes per row), time-major
    if (RESIDENT) {
      const float4* src = H16 ? reinterpret_cast<const float4*>(reinterpret_cast<const uint8_t*>(a.Y) + (size_t)blk * 128)
                              : reinterpret_cast<const float4*>(a.Y + (size_t)blk * 32);
      float4* dst = reinterpret_cast<float4*>(tgt);
      const int64_t ld4 = H16 ? a.ldy / 8 : a.ldy / 4;
      for (int v = threadIdx.x; v < a.T * 8; v += blockDim.x) {
        const int t = v >> 3, c = v & 7;
        dst[v] = src[(size_t)t * ld4 + c];
      }
    }
    __syncthreads();

    const int per_warp = a.LS / kLookupWarps;
    const int lib0 = lsub * a.LS + w * per_warp;
    const int nl = max(0, min(per_warp, a.nlib - lib0));
    if (nl > 0) {
      const int k = E + 1;
      switch (k) {
#define CMB_K(kk)                                                                                   \
  case kk:                                                                                          \
    if constexpr (H16)                                                                              \
      warp_libraries_h16<kk, H16>(a, reinterpret_cast<const uint8_t*>(tgt), ring, wbars, qglob, E, lib0, nl, blk * 64); \
    else if constexpr (kk <= (RESIDENT ? kPairMaxK : kPairMaxKL2)) {                                \
      const float* tb = RESIDENT ? tgt : a.Y + (size_t)blk * 32;                                      \
      int l = 0;                                                                                      \
      if constexpr (kk <= kQuadMaxK) {                                                                \
        const int nq = nl >> 2;                                                                       \
        if (nq) warp_library_group<kk, RESIDENT, 4>(a, tb, ring, wbars, qglob, E, lib0, nq, blk * 32); \
        l = 4 * nq;                                                                                   \
      }                                                                                               \
      const int np = (nl - l) >> 1;                                                                   \
      if (np) warp_library_group<kk, RESIDENT, 2>(a, tb, ring, wbars, qglob, E, lib0 + l, np, blk * 32); \
      l += 2 * np;                                                                                    \
      if (l < nl) warp_libraries<kk, RESIDENT>(a, tb, ring, wbars, qglob, E, lib0 + l, 1, blk * 32);  \
    } else                                                                                            \
      warp_libraries<kk, RESIDENT>(a, RESIDENT ? tgt : a.Y + (size_t)blk * 32, ring, wbars, qglob, E, lib0, nl, blk * 32); \
    break;
        CMB_K(2) CMB_K(3) CMB_K(4) CMB_K(5) CMB_K(6) CMB_K(7) CMB_K(8) CMB_K(9) CMB_K(10)
        CMB_K(11) CMB_K(12) CMB_K(13) CMB_K(14) CMB_K(15) CMB_K(16) CMB_K(17) CMB_K(18) CMB_K(19)
        CMB_K(20) CMB_K(21) CMB_K(22) CMB_K(23) CMB_K(24) CMB_K(25) CMB_K(26) CMB_K(27) CMB_K(28)
        CMB_K(29) CMB_K(30) CMB_K(31)
#undef CMB_K
        default: break;
      }
    }
    __syncthreads();
  }
  (void)lane;
}

}  // namespace

int lookup_stage_bytes(int T, int max_rec_bytes) {
  const int budget = 232448 - T * 128 - kLookupWarps * 2 * 8 - 1024;  // 1 KB static reserve
  int sb = budget / (kLookupWarps * 2);
  sb = sb - sb % 16;
  if (sb > 4096) sb = 4096;
  // resident targets need room for at least two records per slot; otherwise
  // the kernel gathers targets from L2 with 4 KB staging slots
  if (sb < 2 * max_rec_bytes) return kNonResidentStage;
  return sb;
}

cudaError_t launch_lookup_xmap(const LookupArgs& a, int grid, cudaStream_t st) {
  const bool resident = a.stage_bytes != kNonResidentStage;
  const int smem = (resident ? a.T * 128 : 0) + kLookupWarps * 2 * a.stage_bytes + kLookupWarps * 2 * 8;
  auto kern = !resident      ? lookup_xmap_kernel<false, 0>
              : a.h16 == 2 ? lookup_xmap_kernel<true, 2>
              : a.h16      ? lookup_xmap_kernel<true, 1>
                           : lookup_xmap_kernel<true, 0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  count_launch();
  kern<<<grid, kLookupWarps * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace cmb
