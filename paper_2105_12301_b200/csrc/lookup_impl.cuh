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
// resident in shared memory, time-major: tgt[t][32] -- T = 1,450 samples x
// 128 B = 185.6 KB of the 227 KB -- plus a zero row.  Its warps stream their
// own libraries' neighbour tables (records of k fp32 weights + k u16 rows)
// from L2/HBM into per-warp 2-slot shared-memory rings with cp.async.bulk
// (TMA bulk copies) completing on mbarriers, so table bytes are fetched once
// per (library, target block).  Work items are (E group, library sub-range,
// target block), handed out by an atomic counter so concurrently running
// CTAs share the same libraries' tables in L2.
//
// The default (resident fp32) path is the rotated-lane layout
// (rot_library_group / rot2_library_pairs below): a lane owns an embedded
// point, loads its record once, and rotates over the block's target columns,
// so every gather is one conflict-free wavefront and no record is broadcast;
// the moments stay in registers for a whole library and are transposed once.
// It runs as one launch per neighbour-count class (kernels.cuh
// lookup_class_warps: 12 warps for k <= 16, 8 for 17..24, both on the
// two-target path; 16 otherwise).  The lane = target layout with broadcast
// records (warp_libraries / warp_library_group) remains for the non-resident
// case (targets gathered from L2), the 16-bit target modes and fallbacks.
// Skill is evaluated in fp64 against the precomputed observed-segment
// moments; ill-conditioned pairs of the rotated path are finished in fp64 by
// lookup_fixup_kernel.
#pragma once

#include "cmb_common.cuh"
#include "kernels.cuh"

#include <cuda_fp16.h>

#include <algorithm>

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

// ---------------------------------------------------------------- rotated-lane lookup
// The paths above give every lane one target and broadcast each point's record
// (k weights + k rows) to all 32 lanes: on the mixed data those broadcasts are
// ~40% of the shared-memory wavefronts, the kernel's binding resource.  Here a
// lane owns a POINT instead: the warp works on batches of 8 consecutive
// points; lane l (group g = l / 8, point p = l % 8) loads the record of point
// p once into registers and, at rotation step j = 0..7, predicts target
// column 8g + ((p + j) & 7) of the resident block.  At every step the 32 lanes
// gather 32 distinct columns -- 32 distinct banks whatever the rows -- so each
// gather is one wavefront for 32 (point, target) pairs and the record costs
// ~k/16 wavefronts per 32 pairs instead of ~k/2 + k/4.  Lane l's accumulator j
// always belongs to target column 8g + ((p + j) & 7), so the moments stay in
// registers for the whole library and are transposed once at its end (a
// barrel rotation by p and an 8-lane butterfly reduce-scatter in fp64).
//
// The moments are raw fp32 sums (no per-target shift: it would cost 8
// registers per library); a pair whose prediction variance is small against
// its second moment (m2p <= fix_ratio * Spp, e.g. a near-constant library), where
// those sums could cancel, is queued and recomputed exactly in fp64 by
// lookup_fixup_kernel.  Elsewhere |d m2p| / m2p <= 16 (|d Spp| + 2 |d Sp| max|p|)
// / Spp (fix_ratio = 1/16, CMB_FIX_RATIO), i.e. a few fp32 ulps of a ~n/8-term
// sum.  Measured at N = 8,192 against an all-fp64 run (ratio 2): max |d rho|
// 3.3e-6 at ratios 1/4 and 1/16 (0.7% and 0.04% of the (library, block) items
// queued), 1.4e-5 at 1/64, 3.1e-5 at 1/256 with no queue at all.
template <int NL> struct RotV;
template <> struct RotV<1> { using T = float; };
template <> struct RotV<2> { using T = float2; };
__device__ __forceinline__ float v_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float2 v_add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float v_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float2 v_fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float v_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float2 v_mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ void v_set(float& v, int, float x) { v = x; }
__device__ __forceinline__ void v_set(float2& v, int h, float x) { (h ? v.y : v.x) = x; }
__device__ __forceinline__ float v_get(float v, int) { return v; }
__device__ __forceinline__ float v_get(float2 v, int h) { return h ? v.y : v.x; }
template <class V> __device__ __forceinline__ V v_splat(float x);
template <> __device__ __forceinline__ float v_splat<float>(float x) { return x; }
template <> __device__ __forceinline__ float2 v_splat<float2>(float x) { return make_float2(x, x); }

__device__ __forceinline__ void lds_v4(uint32_t addr, uint32_t& x, uint32_t& y, uint32_t& z, uint32_t& w) {
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(addr));
}

// Sum over the 8 lanes of this lane's group of the accumulators that belong
// to target column (lane & 24) + (lane & 7): lane p's m[j] belongs to column
// (p + j) & 7, so rotate by p (v[c] = m[(c - p) & 7]) and reduce-scatter.
__device__ __forceinline__ double rot_reduce(const float (&m)[8], int p) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = m[i];
#pragma unroll
  for (int b = 1; b < 8; b <<= 1) {
    const bool on = (p & b) != 0;
    float u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) u[i] = on ? v[(i - b) & 7] : v[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = u[i];
  }
  const bool b4 = (p & 4) != 0, b2 = (p & 2) != 0, b1 = (p & 1) != 0;
  double d[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    d[i] = (double)(b4 ? v[i + 4] : v[i]) + (double)__shfl_xor_sync(CMB_FULL, b4 ? v[i] : v[i + 4], 4);
  double e[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) e[i] = (b2 ? d[i + 2] : d[i]) + __shfl_xor_sync(CMB_FULL, b2 ? d[i] : d[i + 2], 2);
  return (b1 ? e[1] : e[0]) + __shfl_xor_sync(CMB_FULL, b1 ? e[0] : e[1], 1);
}

// records per stage part for the rotated path (a multiple of the 8-point batch)
__host__ __device__ constexpr int rot_records(int stage_bytes, int nl, int k) {
  return (((stage_bytes / nl) & ~15) / rec_bytes(k)) & ~7;
}

template <int K, int NL>
__device__ __forceinline__ void rot_library_group(const LookupArgs& a, uint32_t tsm, uint8_t* ring,
                                                  uint64_t* bars, uint32_t& qglob, int E, int lib0,
                                                  int ngroup, int slot_base) {
  using V = typename RotV<NL>::T;
  constexpr int R = rec_bytes(K);
  constexpr int RO = rec_row_off(K);
  const int lane = lane_id();
  const int pl = lane & 7;
  const int n = a.T - (E - 1) * a.tau;
  const int off = (E - 1) * a.tau;
  const size_t lstride = rec_lib_stride(K, n);
  const uint8_t* base = a.tab[E] + (size_t)lib0 * lstride;
  const int part = (a.stage_bytes / NL) & ~15;
  const int RS = rot_records(a.stage_bytes, NL, K);
  const int nst = (n + RS - 1) / RS;
  const int total = ngroup * nst;
  const uint32_t zrow = tsm + (uint32_t)a.T * 128u;  // a zero sample row: masked points gather 0
  uint32_t col[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) col[j] = (uint32_t)((lane & 24) | ((pl + j) & 7)) << 2;

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

  V sp[8], spp[8], sop[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) sp[j] = spp[j] = sop[j] = v_splat<V>(0.f);
  for (int q = 0; q < total; ++q) {
    const uint32_t g = qglob + q;
    uint8_t* slotp = ring + (g & 1) * a.stage_bytes;
    const int lg = q / nst, s = q - lg * nst;
    mbar_wait(bars + (g & 1), (g >> 1) & 1);
    const uint32_t s0 = smem_u32(slotp);
    const int r0 = s * RS;
    const int nrec = min(RS, n - r0);
    for (int b = 0; b < nrec; b += 8) {
      const int r = b + pl;
      uint32_t ra[NL][K];
      V w[K];
#pragma unroll
      for (int h = 0; h < NL; ++h) {
        uint32_t wd[R / 4];
        const uint32_t rec = s0 + h * part + r * R;
        if constexpr (R == 8) {
          lds_v2(rec, wd[0], wd[1]);
        } else {
#pragma unroll
          for (int c = 0; c < R / 16; ++c) lds_v4(rec + 16 * c, wd[4 * c], wd[4 * c + 1], wd[4 * c + 2], wd[4 * c + 3]);
        }
        float ws = 0.f;
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
          float wk;
          if (rec_implicit(K) && kk == K - 1) {
            wk = __fsub_rn(1.f, ws);  // k <= 3 records store k - 1 weights
          } else {
            wk = __uint_as_float(wd[kk]);
            ws = __fadd_rn(ws, wk);
          }
          const uint32_t row = (wd[RO / 4 + (kk >> 1)] >> ((kk & 1) * 16)) & 0xffffu;
          ra[h][kk] = tsm + (row << 7);
          v_set(w[kk], h, wk);
        }
      }
      uint32_t oa = tsm + ((uint32_t)(off + r0 + r) << 7);
      if (b + 8 > nrec) {
        // the library's last, partial batch: lanes past its end gather the zero
        // row with zero weights, so they add nothing to the moments
        const bool valid = r < nrec;
#pragma unroll
        for (int h = 0; h < NL; ++h)
#pragma unroll
          for (int kk = 0; kk < K; ++kk) {
            ra[h][kk] = valid ? ra[h][kk] : zrow;
            v_set(w[kk], h, valid ? v_get(w[kk], h) : 0.f);
          }
        oa = valid ? oa : zrow;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float o = lds_f32(oa + col[j]);
        V p;
        if constexpr (NL == 1 && K >= 4) {
          // one library: even and odd neighbours as the two halves of packed
          // FFMA2s (half the FMA instructions; two shorter dependency chains)
          float2 p2 = __fmul2_rn(make_float2(v_get(w[0], 0), v_get(w[1], 0)),
                                 make_float2(lds_f32(ra[0][0] + col[j]), lds_f32(ra[0][1] + col[j])));
#pragma unroll
          for (int kk = 2; kk + 1 < K; kk += 2)
            p2 = __ffma2_rn(make_float2(v_get(w[kk], 0), v_get(w[kk + 1], 0)),
                            make_float2(lds_f32(ra[0][kk] + col[j]), lds_f32(ra[0][kk + 1] + col[j])), p2);
          float pp = __fadd_rn(p2.x, p2.y);
          if constexpr (K & 1) pp = __fmaf_rn(v_get(w[K - 1], 0), lds_f32(ra[0][K - 1] + col[j]), pp);
          v_set(p, 0, pp);
        } else {
          V y;
#pragma unroll
          for (int h = 0; h < NL; ++h) v_set(y, h, lds_f32(ra[h][0] + col[j]));
          p = v_mul(w[0], y);
#pragma unroll
          for (int kk = 1; kk < K; ++kk) {
#pragma unroll
            for (int h = 0; h < NL; ++h) v_set(y, h, lds_f32(ra[h][kk] + col[j]));
            p = v_fma(w[kk], y, p);
          }
        }
        sp[j] = v_add(sp[j], p);
        spp[j] = v_fma(p, p, spp[j]);
        sop[j] = v_fma(v_splat<V>(o), p, sop[j]);
      }
    }
    __syncwarp();
    if (lane == 0 && q + 2 < total) issue(q + 2, slotp, bars + (g & 1));
    if (s == nst - 1) {
      // library group complete: lane l ends with target column l of the block
      const int slot = slot_base + lane;
      const int tgt_id = a.slot_tgt[slot];
      const double So = a.obs_s[slot], Soo = a.obs_ss[slot];
      const bool ocst = a.obs_const[slot] != 0;
      const double nn = (double)n;
#pragma unroll
      for (int h = 0; h < NL; ++h) {
        bool fix = false;
        float m[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = v_get(sp[j], h);
        const double Sp = rot_reduce(m, pl);
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = v_get(spp[j], h);
        const double Spp = rot_reduce(m, pl);
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = v_get(sop[j], h);
        const double Sop = rot_reduce(m, pl);
        const int l = lib0 + NL * lg + h;
        if (tgt_id >= 0) {
          float* dst = a.rhoT + (size_t)tgt_id * a.ldr + a.lib_col[l];
          const double m2o = Soo - So * So / nn;
          const double m2p = Spp - Sp * Sp / nn;
          const double com = Sop - So * Sp / nn;
          if (ocst || !(m2o > 0.0)) *dst = __int_as_float(0x7fc00000);
          else if (m2p > a.fix_ratio * Spp) *dst = (float)fmin(1.0, fmax(-1.0, com / sqrt(m2o * m2p)));
          else fix = true;
        }
        // ill-conditioned pairs: queue (library, target block) once per warp
        const unsigned bal = __ballot_sync(CMB_FULL, fix);
        if (bal && lane == __ffs(bal) - 1) {
          const int f = atomicAdd(a.fix_count, 1);
          if (f < a.fix_cap) a.fix[f] = make_int2(l, slot_base);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) sp[j] = spp[j] = sop[j] = v_splat<V>(0.f);
    }
  }
  qglob += total;
}

// Two-target variant for larger k (rot2): each half-warp runs its own
// library of a pair; lane l (half h = l / 16, group g = (l / 8) & 1, point
// p = l % 8) gathers a COLUMN PAIR per neighbour with one 8-byte load -- pair
// 8g + ((p + j) & 7) at step j, so a half-warp's 16 lanes read 16 distinct
// pairs (all 32 banks) whatever the rows.  Per 32 (point, target) pairs that is
// the same k gather wavefronts, half the record traffic (a record serves 16
// targets instead of 8) and about half the instructions of rot_library_group
// (one load + address per two targets), which leaves the shared-memory pipe as
// the only limiter for large k.  Accumulators: 8 steps x 3 moments x float2.
__device__ __forceinline__ float2 lds_f2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}

template <int K>
__device__ __forceinline__ void rot2_library_pairs(const LookupArgs& a, uint32_t tsm, uint8_t* ring,
                                                   uint64_t* bars, uint32_t& qglob, int E, int lib0,
                                                   int nl, int slot_base) {
  constexpr int R = rec_bytes(K);
  constexpr int RO = rec_row_off(K);
  const int lane = lane_id();
  const int h = lane >> 4;
  const int pl = lane & 7;
  const uint32_t gcol = (uint32_t)(lane & 8) << 3;  // byte offset of the group's 8 column pairs
  const int n = a.T - (E - 1) * a.tau;
  const int off = (E - 1) * a.tau;
  const size_t lstride = rec_lib_stride(K, n);
  const uint8_t* base = a.tab[E] + (size_t)lib0 * lstride;
  const int part = (a.stage_bytes / 2) & ~15;
  const int RS = rot_records(a.stage_bytes, 2, K);
  const int nst = (n + RS - 1) / RS;
  const int npair = (nl + 1) >> 1;
  const int total = npair * nst;
  const uint32_t zrow = tsm + (uint32_t)a.T * 128u;

  auto issue = [&](int q, uint8_t* dst, uint64_t* bar) {
    const int lg = q / nst, s = q - lg * nst;
    const int r0 = s * RS;
    const int nrec = min(RS, n - r0);
    const uint32_t bytes = (uint32_t)((nrec * R + 15) & ~15);
    const int nh = (2 * lg + 1 < nl) ? 2 : 1;
    const uint8_t* src = base + (size_t)(2 * lg) * lstride + (size_t)r0 * R;
    mbar_expect_tx(bar, nh * bytes);
    for (int hh = 0; hh < nh; ++hh) bulk_g2s(dst + hh * part, src + hh * lstride, bytes, bar);
  };
  if (lane == 0) {
    for (int q = 0; q < 2 && q < total; ++q) {
      const uint32_t g = qglob + q;
      issue(q, ring + (g & 1) * a.stage_bytes, bars + (g & 1));
    }
  }
  __syncwarp();

  float2 sp[8], spp[8], sop[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) sp[j] = spp[j] = sop[j] = make_float2(0.f, 0.f);
  for (int q = 0; q < total; ++q) {
    const uint32_t g = qglob + q;
    uint8_t* slotp = ring + (g & 1) * a.stage_bytes;
    const int lg = q / nst, s = q - lg * nst;
    const bool second = 2 * lg + 1 < nl;  // the pair has a second library
    mbar_wait(bars + (g & 1), (g >> 1) & 1);
    const uint32_t s0 = smem_u32(slotp) + ((h && second) ? part : 0);
    const int r0 = s * RS;
    const int nrec = min(RS, n - r0);
    for (int b = 0; b < nrec; b += 8) {
      const int r = b + pl;
      uint32_t ra[K];
      float w[K];
      {
        uint32_t wd[R / 4];
        const uint32_t rec = s0 + r * R;
        if constexpr (R == 8) {
          lds_v2(rec, wd[0], wd[1]);
        } else {
#pragma unroll
          for (int c = 0; c < R / 16; ++c) lds_v4(rec + 16 * c, wd[4 * c], wd[4 * c + 1], wd[4 * c + 2], wd[4 * c + 3]);
        }
        float ws = 0.f;
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
          if (rec_implicit(K) && kk == K - 1) {
            w[kk] = __fsub_rn(1.f, ws);  // k <= 3 records store k - 1 weights
          } else {
            w[kk] = __uint_as_float(wd[kk]);
            ws = __fadd_rn(ws, w[kk]);
          }
          const uint32_t row = (wd[RO / 4 + (kk >> 1)] >> ((kk & 1) * 16)) & 0xffffu;
          ra[kk] = tsm + (row << 7);
        }
      }
      uint32_t oa = tsm + ((uint32_t)(off + r0 + r) << 7);
      if (b + 8 > nrec) {
        const bool valid = r < nrec;
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
          ra[kk] = valid ? ra[kk] : zrow;
          w[kk] = valid ? w[kk] : 0.f;
        }
        oa = valid ? oa : zrow;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t c = gcol | ((uint32_t)((pl + j) & 7) << 3);
        const float2 o = lds_f2(oa + c);
        float2 y = lds_f2(ra[0] + c);
        float2 p = make_float2(__fmul_rn(w[0], y.x), __fmul_rn(w[0], y.y));
#pragma unroll
        for (int kk = 1; kk < K; ++kk) {
          y = lds_f2(ra[kk] + c);
          p.x = __fmaf_rn(w[kk], y.x, p.x);
          p.y = __fmaf_rn(w[kk], y.y, p.y);
        }
        sp[j] = __fadd2_rn(sp[j], p);
        spp[j] = __ffma2_rn(p, p, spp[j]);
        sop[j] = __ffma2_rn(o, p, sop[j]);
      }
    }
    __syncwarp();
    if (lane == 0 && q + 2 < total) issue(q + 2, slotp, bars + (g & 1));
    if (s == nst - 1) {
      // pair complete: lane (h, g, p) holds column pair 8g + p of library 2 lg + h
      const int l = lib0 + 2 * lg + h;
      const bool live = h == 0 || second;
      const double nn = (double)n;
      bool fix = false;
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
        float m[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = c2 ? sp[j].y : sp[j].x;
        const double Sp = rot_reduce(m, pl);
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = c2 ? spp[j].y : spp[j].x;
        const double Spp = rot_reduce(m, pl);
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = c2 ? sop[j].y : sop[j].x;
        const double Sop = rot_reduce(m, pl);
        const int slot = slot_base + 2 * ((lane & 8) | pl) + c2;
        const int tgt_id = a.slot_tgt[slot];
        if (live && tgt_id >= 0) {
          const double So = a.obs_s[slot], Soo = a.obs_ss[slot];
          float* dst = a.rhoT + (size_t)tgt_id * a.ldr + a.lib_col[l];
          const double m2o = Soo - So * So / nn;
          const double m2p = Spp - Sp * Sp / nn;
          const double com = Sop - So * Sp / nn;
          if (a.obs_const[slot] != 0 || !(m2o > 0.0)) *dst = __int_as_float(0x7fc00000);
          else if (m2p > a.fix_ratio * Spp) *dst = (float)fmin(1.0, fmax(-1.0, com / sqrt(m2o * m2p)));
          else fix = true;
        }
      }
      // ill-conditioned pairs: queue (library, target block) once per half-warp
      const unsigned bal = __ballot_sync(CMB_FULL, fix) & (0xffffu << (16 * h));
      if (bal && lane == __ffs(bal) - 1) {
        const int f = atomicAdd(a.fix_count, 1);
        if (f < a.fix_cap) a.fix[f] = make_int2(l, slot_base);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) sp[j] = spp[j] = sop[j] = make_float2(0.f, 0.f);
    }
  }
  qglob += total;
}

// Exact completion of the queued (library, target block) entries: one CTA
// per entry, lane = target as in warp_libraries, warp w taking the points
// t = w (mod 8); fp64 predictions from the same fp32 records and targets (the
// record read as warp-uniform loads, the samples as coalesced 128-byte rows of
// the time-major array through L1/L2), moments about the lane's first
// prediction (the shift of warp_libraries) so near-constant predictions do
// not cancel, and a fixed-order fp64 reduction over the 8 warps.
constexpr int kFixWarps = 8;
__global__ void __launch_bounds__(kFixWarps * 32) lookup_fixup_kernel(LookupArgs a) {
  __shared__ double red[3][kFixWarps][32];
  const int nfix = min(*a.fix_count, a.fix_cap);
  const int lane = lane_id(), w = warp_id();
  for (int e = blockIdx.x; e < nfix; e += gridDim.x) {
    const int2 f = a.fix[e];
    const int l = f.x, slot = f.y + lane;
    const int blk = f.y / 32;
    int g = 0;
    while (g + 1 < a.ngroups && a.g_blk0[g + 1] <= blk) ++g;
    const int E = a.g_E[g], K = E + 1;
    const int n = a.T - (E - 1) * a.tau, off = (E - 1) * a.tau;
    const int R = rec_bytes(K), RO = rec_row_off(K);
    const uint8_t* rec0 = a.tab[E] + (size_t)l * rec_lib_stride(K, n);
    const float* __restrict__ ycol = a.Y + slot;
    const auto pred = [&](int t) {
      const uint8_t* rp = rec0 + (size_t)t * R;
      const float* wp = reinterpret_cast<const float*>(rp);
      const uint16_t* rw = reinterpret_cast<const uint16_t*>(rp + RO);
      double p = 0.0, ws = 0.0;
      for (int kk = 0; kk < K; ++kk) {
        const double wk = (rec_implicit(K) && kk == K - 1) ? 1.0 - ws : (double)__ldg(wp + kk);
        ws += wk;
        p += wk * (double)__ldg(ycol + (size_t)__ldg(rw + kk) * a.ldy);
      }
      return p;
    };
    const double s = pred(0);
    double Sp = 0.0, Spp = 0.0, Sop = 0.0;
#pragma unroll 2
    for (int t = w; t < n; t += kFixWarps) {
      const double p = pred(t) - s;
      const double o = (double)__ldg(ycol + (size_t)(off + t) * a.ldy);
      Sp += p;
      Spp += p * p;
      Sop += o * p;
    }
    red[0][w][lane] = Sp;
    red[1][w][lane] = Spp;
    red[2][w][lane] = Sop;
    __syncthreads();
    if (w == 0) {
      Sp = Spp = Sop = 0.0;
      for (int q = 0; q < kFixWarps; ++q) {
        Sp += red[0][q][lane];
        Spp += red[1][q][lane];
        Sop += red[2][q][lane];
      }
      const int tgt_id = a.slot_tgt[slot];
      if (tgt_id >= 0) {
        const double nn = (double)n;
        const double So = a.obs_s[slot], Soo = a.obs_ss[slot];
        const double m2o = Soo - So * So / nn;
        const double m2p = Spp - Sp * Sp / nn;
        const double com = Sop - So * Sp / nn;
        float r = __int_as_float(0x7fc00000);
        if (a.obs_const[slot] == 0 && m2o > 0.0 && m2p > 0.0) r = (float)fmin(1.0, fmax(-1.0, com / sqrt(m2o * m2p)));
        a.rhoT[(size_t)tgt_id * a.ldr + a.lib_col[l]] = r;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- materialised predictions
// lookup_batch(want_predictions=True) of the cross map (prediction.py:145-153,
// ccm.py:148-149) for a caller-given set of (library, target) pairs, from the
// SAME tables and centred targets the rho lookup used (so the predictions are
// the ones behind rho).  One warp per pair, lanes over embedded points:
// p_t = sum_q w_q y[row_q] in fp32 (explicit last weight 1 - sum of the others
// for k <= 3 records, as in rot_library_group), plus the target's mean back.
// pred[pair][t] for t < n_E, NaN after.
__global__ void predict_pairs_kernel(LookupArgs a, const int4* __restrict__ pairs, int64_t npairs, int64_t c0,
                                     const double* __restrict__ shift, float* __restrict__ pred, int64_t ldp) {
  const int lane = lane_id();
  const int64_t nw = (int64_t)gridDim.x * blockDim.x / 32;
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; q < npairs; q += nw) {
    const int4 pr = pairs[q];  // (library index in the library list, target slot, E, output row)
    const int E = pr.z, K = E + 1;
    const int n = a.T - (E - 1) * a.tau;
    const int R = rec_bytes(K), RO = rec_row_off(K);
    const uint8_t* rec0 = a.tab[E] + (size_t)(pr.x - c0) * rec_lib_stride(K, n);
    const float* __restrict__ ycol = a.Y + pr.y;
    const double mu = shift[pr.y];
    float* out = pred + (size_t)pr.w * ldp;
    for (int t = lane; t < a.T; t += 32) {
      if (t >= n) {
        out[t] = __int_as_float(0x7fc00000);
        continue;
      }
      const uint8_t* rp = rec0 + (size_t)t * R;
      const float* w = reinterpret_cast<const float*>(rp);
      const uint16_t* rw = reinterpret_cast<const uint16_t*>(rp + RO);
      float ws = 0.f, p = 0.f;
      for (int kk = 0; kk < K; ++kk) {
        float wk;
        if (rec_implicit(K) && kk == K - 1) {
          wk = __fsub_rn(1.f, ws);
        } else {
          wk = __ldg(w + kk);
          ws = __fadd_rn(ws, wk);
        }
        p = __fmaf_rn(wk, __ldg(ycol + (size_t)__ldg(rw + kk) * a.ldy), p);
      }
      out[t] = (float)((double)p + mu);
    }
  }
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
constexpr int kRotPairMaxK = 8;  // rotated path: two libraries in lockstep (packed FFMA2) for k <= 8
// two-target rotated path (rot2_library_pairs) for 4 <= k <= 24 (where the stage
// slots hold 8 records of two libraries: k <= 12 at T = 1,450); A/B at full
// size on one box (lookup seconds): rot2 from k = 9 4.764, from k = 4 4.719;
// library pairs up to k = 12 instead of rot2 4.969; OR-formed gather addresses
// (LOP3 instead of IMAD) 4.851
constexpr int kRot2MinK = 4;
constexpr int kRot2MaxK = 24;

// Rotated-lane lookup of one warp's libraries [lib0, lib0 + nl); returns the
// number handled (0 when the staging slot is too small for an 8-point batch).
template <int K>
__device__ __forceinline__ int rot_dispatch(const LookupArgs& a, uint32_t tsm, uint8_t* ring, uint64_t* bars,
                                            uint32_t& qglob, int E, int lib0, int nl, int slot_base) {
  int l = 0;
  if constexpr (K >= kRot2MinK && K <= kRot2MaxK) {
    if (a.rot == 2 && rot_records(a.stage_bytes, 2, K) >= 8) {
      rot2_library_pairs<K>(a, tsm, ring, bars, qglob, E, lib0, nl, slot_base);
      return nl;
    }
  }
  if constexpr (K <= kRotPairMaxK) {
    const int np = nl >> 1;
    if (np && rot_records(a.stage_bytes, 2, K) >= 8) {
      rot_library_group<K, 2>(a, tsm, ring, bars, qglob, E, lib0, np, slot_base);
      l = 2 * np;
    }
  }
  if (l < nl && rot_records(a.stage_bytes, 1, K) >= 8) {
    rot_library_group<K, 1>(a, tsm, ring, bars, qglob, E, lib0 + l, nl - l, slot_base);
    l = nl;
  }
  return l;
}

// WARPS = 16: every path (the small-k rotated class, fallbacks, non-resident and
// 16-bit modes).  WARPS = 12 / 8: only the two-target rotated path for the
// mid / large k classes (lookup_class_warps), whose larger stage slots hold 8
// records of two libraries.
// KLO..KHI: the neighbour counts this instantiation compiles (the host sends a
// launch only groups inside the range): the 16-warp resident kernel is split
// into k ranges so that nvcc builds the pieces in parallel.
template <bool RESIDENT, int H16, int WARPS = kLookupWarps, int KLO = 2, int KHI = 31>
__global__ void __launch_bounds__(WARPS * 32, 1) lookup_xmap_kernel(LookupArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  float* tgt = reinterpret_cast<float*>(smem);
  // resident targets: T sample rows + one zero row (rotated path: masked points)
  const size_t tgt_bytes = RESIDENT ? (size_t)(a.T + 1) * 128 : 0;
  uint8_t* rings = smem + tgt_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(rings + (size_t)WARPS * 2 * a.stage_bytes);
  __shared__ int64_t s_item;

  const int lane = lane_id(), w = warp_id();
  if (threadIdx.x < WARPS * 2) mbar_init(bars + threadIdx.x, 1);
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
    // resident: library-major items (concurrent CTAs share the libraries'
    // tables in L2, each keeps its own target block in shared memory);
    // non-resident: target-block-major (concurrent CTAs gather from the same
    // target block in L2 and stream their own libraries' tables)
    int lsub, blk;
    if (RESIDENT || !a.tmajor) {
      lsub = (int)(rem / nblk);
      blk = a.g_blk0[g] + (int)(rem - (int64_t)lsub * nblk);
    } else {
      const int b = (int)(rem / a.n_lsub);
      lsub = (int)(rem - (int64_t)b * a.n_lsub);
      blk = a.g_blk0[g] + b;
    }
    const int E = a.g_E[g];

    // stage the target block (32 fp32 or 64 fp16 targets: 128 bytes per row), time-major
    if (RESIDENT) {
      const float4* src = H16 ? reinterpret_cast<const float4*>(reinterpret_cast<const uint8_t*>(a.Y) + (size_t)blk * 128)
                              : reinterpret_cast<const float4*>(a.Y + (size_t)blk * 32);
      float4* dst = reinterpret_cast<float4*>(tgt);
      const int64_t ld4 = H16 ? a.ldy / 8 : a.ldy / 4;
      for (int v = threadIdx.x; v < (a.T + 1) * 8; v += blockDim.x) {
        const int t = v >> 3, c = v & 7;
        dst[v] = t < a.T ? src[(size_t)t * ld4 + c] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    __syncthreads();

    // the item's libraries [lsub LS, (lsub + 1) LS) split over the warps (the
    // non-resident kernel's warp count need not divide LS)
    int per_warp, nl, lib0;
    if constexpr (RESIDENT) {
      per_warp = a.LS / WARPS;
      lib0 = lsub * a.LS + w * per_warp;
      nl = max(0, min(per_warp, a.nlib - lib0));
    } else {
      per_warp = (a.LS + WARPS - 1) / WARPS;
      lib0 = lsub * a.LS + w * per_warp;
      nl = max(0, min(per_warp, min(a.nlib, (lsub + 1) * a.LS) - lib0));
    }
    if constexpr (RESIDENT && WARPS != kLookupWarps) {
      // class kernels: the host only sends them k with a feasible two-target stage
      if (nl > 0) {
        switch (E + 1) {
#define CMB_K2(kk) \
  case kk:         \
    rot2_library_pairs<kk>(a, smem_u32(tgt), ring, wbars, qglob, E, lib0, nl, blk * 32); \
    break;
          CMB_K2(2) CMB_K2(3) CMB_K2(4) CMB_K2(5) CMB_K2(6) CMB_K2(7) CMB_K2(8) CMB_K2(9) CMB_K2(10) CMB_K2(11) CMB_K2(12)
          CMB_K2(13) CMB_K2(14) CMB_K2(15) CMB_K2(16) CMB_K2(17) CMB_K2(18) CMB_K2(19) CMB_K2(20)
          CMB_K2(21) CMB_K2(22) CMB_K2(23) CMB_K2(24)
#undef CMB_K2
          default: __trap();
        }
      }
    } else if (nl > 0) {
      const int k = E + 1;
      switch (k) {
#define CMB_K(kk)                                                                                   \
  case kk:                                                                                          \
    if constexpr (kk < KLO || kk > KHI) { __trap(); } else {                                        \
    if constexpr (RESIDENT && !H16)                                                                 \
      if (a.rot && rot_dispatch<kk>(a, smem_u32(tgt), ring, wbars, qglob, E, lib0, nl, blk * 32) == nl) \
        break;                                                                                      \
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
    }                                                                                                 \
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

}  // namespace cmb
