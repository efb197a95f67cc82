// Supporting kernels: data staging for the cross map, the materialised
// reference-shaped primitives of the public API (pairwise_distances,
// partial_sort_topk, normalize_to_weights, PearsonAggregate.from_arrays,
// lookup_batch with predictions) and small layout kernels.
#include "cmb_common.cuh"
#include "kernels.cuh"

#include <cuda_fp16.h>
#include <float.h>

namespace cmb {

namespace {

__device__ __forceinline__ double nan_d() { return __longlong_as_double(0x7ff8000000000000ll); }

// ---------------------------------------------------------------- series statistics
__global__ void series_mean_kernel(const float* __restrict__ x, int64_t N, int64_t T, int64_t ld,
                                   double* __restrict__ mean) {
  const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= N) return;
  const float* p = x + s * ld;
  double acc = 0.0;
  for (int64_t t = lane_id(); t < T; t += 32) acc += (double)p[t];
  acc = warp_sum_d(acc);
  if (lane_id() == 0) mean[s] = acc / (double)T;
}

__global__ void promote_kernel(const float* __restrict__ x, int64_t N, int64_t T, int64_t ld,
                               double* __restrict__ y) {
  const int64_t total = N * ld;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total;
       v += (int64_t)gridDim.x * blockDim.x)
    y[v] = (double)x[v];
}

__global__ void demote_kernel(const double* __restrict__ x, int64_t N, int64_t T,
                              float* __restrict__ y, float* __restrict__ err) {
  const int64_t s = blockIdx.x;
  float m = 0.f;
  for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
    const double v = x[s * T + t];
    const float f = (float)v;
    y[s * T + t] = f;
    m = fmaxf(m, (float)fabs((double)f - v) * 1.0000001f);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(CMB_FULL, m, o));
  __shared__ float wm[32];
  if (lane_id() == 0) wm[warp_id()] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float r = 0.f;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) r = fmaxf(r, wm[q]);
    err[s] = r;
  }
}

// float64 series -> float32 samples about the series mean (the cross map's
// float64 entry): x32 = fl32(x64 - mean64), so large offsets do not eat the
// fp32 mantissa; err = max |x32 - (x64 - mean64)| (+ the fp64 rounding of the
// subtraction), the perturbation M the kNN certification bounds.  Distances
// are translation invariant; the exact fp64 paths use the uncentred x64.
__global__ void demote_center_kernel(const double* __restrict__ x, int64_t T, float* __restrict__ y,
                                     float* __restrict__ err, double* __restrict__ mu_out) {
  const int64_t s = blockIdx.x;
  __shared__ double wsum[32];
  __shared__ float wm[32];
  __shared__ double s_mean;
  double acc = 0.0;
  for (int64_t t = threadIdx.x; t < T; t += blockDim.x) acc += x[s * T + t];
  acc = warp_sum_d(acc);
  if (lane_id() == 0) wsum[warp_id()] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) tot += wsum[q];
    s_mean = tot / (double)T;
    if (mu_out) mu_out[s] = s_mean;
  }
  __syncthreads();
  const double mu = s_mean;
  float m = 0.f;
  double amax = 0.0;
  for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
    const double v = x[s * T + t];
    const double c = v - mu;
    const float f = (float)c;
    y[s * T + t] = f;
    m = fmaxf(m, (float)fabs((double)f - c) * 1.0000001f);
    amax = fmax(amax, fabs(v));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m = fmaxf(m, __shfl_xor_sync(CMB_FULL, m, o));
    amax = fmax(amax, __shfl_xor_sync(CMB_FULL, amax, o));
  }
  if (lane_id() == 0) { wm[warp_id()] = m; wsum[warp_id()] = amax; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float r = 0.f;
    double a = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { r = fmaxf(r, wm[q]); a = fmax(a, wsum[q]); }
    // |fl(v - mu) - (v - mu)| <= 2^-53 (|v| + |mu|)
    err[s] = r + (float)(2.3e-16 * (a + fabs(mu)));
  }
}

// Y[t][slot] = x[tgt(slot)][t] - mean(tgt)   (32 x 32 shared-memory transpose)
__global__ void build_targets_kernel(const float* __restrict__ x, int64_t ld,
                                     const double* __restrict__ mean,
                                     const int32_t* __restrict__ slot_tgt, int64_t slots, int T,
                                     float* __restrict__ Y, int64_t ldy) {
  __shared__ float tile[32][33];
  const int64_t s0 = (int64_t)blockIdx.y * 32;
  const int t0 = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t s = s0 + r;
    const int t = t0 + threadIdx.x;
    float v = 0.f;
    if (s < slots && t < T) {
      const int tg = slot_tgt[s];
      if (tg >= 0) v = __fsub_rn(x[(int64_t)tg * ld + t], (float)mean[tg]);
    }
    tile[r][threadIdx.x] = v;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int t = t0 + r;
    const int64_t s = s0 + threadIdx.x;
    if (t < T && s < ldy) Y[(int64_t)t * ldy + s] = tile[threadIdx.x][r];
  }
}

__global__ void obs_moments_kernel(const float* __restrict__ Y, int64_t ldy, int T, int tau,
                                   const int32_t* __restrict__ slot_E, int64_t slots,
                                   double* __restrict__ s1, double* __restrict__ s2,
                                   uint8_t* __restrict__ cst) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= slots) return;
  const int E = slot_E[s];
  if (E <= 0) { s1[s] = 0; s2[s] = 0; cst[s] = 1; return; }
  const int off = (E - 1) * tau;
  const int n = T - off;
  double a = 0.0, b = 0.0;
  const float first = Y[(int64_t)off * ldy + s];
  bool c = true;
  for (int t = 0; t < n; ++t) {
    const float v = Y[(int64_t)(off + t) * ldy + s];
    a += (double)v;
    b += (double)v * (double)v;
    c = c && (v == first);
  }
  s1[s] = a;
  s2[s] = b;
  cst[s] = c ? 1 : 0;
}

// fp16 target staging (opt-in lookup mode, CMB_LOOKUP_FP16=1): per slot the
// centred series is scaled into [-1, 1] (rho is invariant to the scale), rounded
// to fp16, and the observed-segment moments are taken from the rounded values
// so Pearson is evaluated on one consistent set of numbers.
__global__ void targets_to_half_kernel(const float* __restrict__ Y, int64_t ldy, int T, int tau,
                                       const int32_t* __restrict__ slot_E, int64_t slots,
                                       __half* __restrict__ Yh, double* __restrict__ s1,
                                       double* __restrict__ s2, uint8_t* __restrict__ cst, int mode) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= slots) return;
  float m = 0.f, mn = INFINITY, mx = -INFINITY;
  for (int t = 0; t < T; ++t) {
    const float y = Y[(int64_t)t * ldy + s];
    m = fmaxf(m, fabsf(y));
    mn = fminf(mn, y);
    mx = fmaxf(mx, y);
  }
  // mode 2 (q16): signed 16-bit fixed point v = rint((y - mid) * 32767 / half
  // range) over the full [-32767, 32767] (rho is invariant to the affine map),
  // stored biased by 32768 so the lookup rebuilds 2^23 + 32768 + v with one PRMT
  const float mid = mode == 2 ? 0.5f * (mn + mx) : 0.f;
  if (mode == 2) m = 0.5f * (mx - mn);
  const float inv = (m > 0.f) ? (mode == 2 ? 32767.f : 1.f) / m : 1.f;
  uint16_t* Yq = reinterpret_cast<uint16_t*>(Yh);
  const auto rd = [&](int64_t t) {
    return mode == 2 ? (float)((int)Yq[t * ldy + s] - 32768) : __half2float(Yh[t * ldy + s]);
  };
  for (int t = 0; t < T; ++t) {
    const float y = (Y[(int64_t)t * ldy + s] - mid) * inv;
    if (mode == 2)
      Yq[(int64_t)t * ldy + s] = (uint16_t)((int)fminf(32767.f, fmaxf(-32767.f, rintf(y))) + 32768);
    else
      Yh[(int64_t)t * ldy + s] = __float2half_rn(y);
  }
  const int E = slot_E[s];
  if (E <= 0) { s1[s] = 0; s2[s] = 0; cst[s] = 1; return; }
  const int off = (E - 1) * tau;
  const int n = T - off;
  double a = 0.0, b = 0.0;
  const float first = rd(off);
  bool c = true;
  for (int t = 0; t < n; ++t) {
    const float v = rd(off + t);
    a += (double)v;
    b += (double)v * (double)v;
    c = c && (v == first);
  }
  s1[s] = a;
  s2[s] = b;
  cst[s] = c ? 1 : 0;
}

__global__ void fill_nan_kernel(float* p, int64_t rows, int64_t cols, int64_t ld) {
  const int64_t total = rows * cols;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = v / cols, c = v - r * cols;
    p[r * ld + c] = __int_as_float(0x7fc00000);
  }
}

// ---------------------------------------------------------------- materialised primitives
__global__ void pairwise_kernel(const double* __restrict__ x, int n, int E, int tau,
                                double* __restrict__ D) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= n) return;
  D[(int64_t)i * n + j] = exact_sqdist(x, i, j, E, tau);
}

// One CTA per row: bitonic sort of (value, column) keys with the diagonal
// poisoned to +inf, first k kept.  Keys are unique (column breaks ties), so
// the order is the reference's (value, column) lexicographic order.
__global__ void topk_rows_kernel(const double* __restrict__ D, int n, int npad, int k,
                                 double* __restrict__ d_out, int64_t* __restrict__ i_out) {
  extern __shared__ unsigned char sm[];
  double* key = reinterpret_cast<double*>(sm);
  int* col = reinterpret_cast<int*>(key + npad);
  const int row = blockIdx.x;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  for (int j = threadIdx.x; j < npad; j += blockDim.x) {
    key[j] = (j < n && j != row) ? D[(int64_t)row * n + j] : inf;
    col[j] = (j < n) ? j : 0x7fffffff;
  }
  __syncthreads();
  for (int size = 2; size <= npad; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < npad / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const double kl = key[lo], kh = key[hi];
        const int cl = col[lo], ch = col[hi];
        const bool gt = kl > kh || (kl == kh && cl > ch);
        if (gt == up) { key[lo] = kh; key[hi] = kl; col[lo] = ch; col[hi] = cl; }
      }
      __syncthreads();
    }
  }
  for (int q = threadIdx.x; q < k; q += blockDim.x) {
    d_out[(int64_t)row * k + q] = key[q];
    i_out[(int64_t)row * k + q] = col[q];
  }
}

// flags: bit0 negative entry, bit1 non-ascending row
__global__ void weights_kernel(const double* __restrict__ sq, int64_t n, int k,
                               double* __restrict__ w, int* __restrict__ flags) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double* s = sq + r * k;
  double* o = w + r * k;
  int f = 0;
  for (int q = 0; q < k; ++q) {
    if (s[q] < 0.0) f |= 1;
    if (q > 0 && s[q] < s[q - 1]) f |= 2;
  }
  if (f) { atomicOr(flags, f); return; }
  double scale = sqrt(s[0]);
  if (scale == 0.0) {
    scale = 1.0;
    for (int q = 0; q < k; ++q) {
      const double d = sqrt(s[q]);
      if (d > 0.0) { scale = d; break; }
    }
  }
  double tot = 0.0;
  for (int q = 0; q < k; ++q) {
    const double raw = fmax(exp(-sqrt(s[q]) / scale), DBL_MIN);
    o[q] = raw;
    tot += raw;
  }
  for (int q = 0; q < k; ++q) o[q] = o[q] / tot;
}

// deterministic block sum (blockDim = 1024)
__device__ double block_sum(double v, double* scratch) {
  v = warp_sum_d(v);
  if (lane_id() == 0) scratch[warp_id()] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = (threadIdx.x < (blockDim.x >> 5)) ? scratch[threadIdx.x] : 0.0;
    r = warp_sum_d(r);
    if (threadIdx.x == 0) scratch[32] = r;
  }
  __syncthreads();
  r = scratch[32];
  __syncthreads();
  return r;
}

// Pearson aggregate of a[0,n), b[0,n) in 4096-point blocks merged with the
// pooled rule (prediction.py:45-73).  One CTA; writes 6 doubles.
__device__ void pearson_blocks(const double* __restrict__ a, const double* __restrict__ b,
                               int64_t n, double* out, double* scratch) {
  double cnt = 0, ma = 0, mb = 0, m2a = 0, m2b = 0, cm = 0;
  for (int64_t s0 = 0; s0 < n; s0 += 4096) {
    const int64_t e0 = min(n, s0 + (int64_t)4096);
    const double nb = (double)(e0 - s0);
    double sa = 0, sb = 0;
    for (int64_t t = s0 + threadIdx.x; t < e0; t += blockDim.x) { sa += a[t]; sb += b[t]; }
    const double xa = block_sum(sa, scratch) / nb;
    const double xb = block_sum(sb, scratch) / nb;
    double paa = 0, pbb = 0, pab = 0;
    for (int64_t t = s0 + threadIdx.x; t < e0; t += blockDim.x) {
      const double da = a[t] - xa, db = b[t] - xb;
      paa += da * da;
      pbb += db * db;
      pab += da * db;
    }
    const double baa = block_sum(paa, scratch);
    const double bbb = block_sum(pbb, scratch);
    const double bab = block_sum(pab, scratch);
    if (cnt == 0) {
      cnt = nb; ma = xa; mb = xb; m2a = baa; m2b = bbb; cm = bab;
    } else {
      const double nt = cnt + nb;
      const double ga = xa - ma, gb = xb - mb, pooled = cnt * nb / nt;
      ma += ga * nb / nt;
      mb += gb * nb / nt;
      m2a += baa + ga * ga * pooled;
      m2b += bbb + gb * gb * pooled;
      cm += bab + ga * gb * pooled;
      cnt = nt;
    }
  }
  if (threadIdx.x == 0) {
    out[0] = cnt; out[1] = ma; out[2] = mb; out[3] = m2a; out[4] = m2b; out[5] = cm;
  }
}

__global__ void __launch_bounds__(1024) pearson_kernel(const double* a, const double* b, int64_t n,
                                                        double* agg) {
  __shared__ double scratch[33];
  pearson_blocks(a, b, n, agg, scratch);
}

__global__ void lookup64_pred_kernel(const int64_t* __restrict__ idx, const double* __restrict__ w,
                                     int64_t n, int k, int offset, const double* __restrict__ Y,
                                     int64_t len, int64_t M, double* __restrict__ pred) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t m = blockIdx.y;
  if (t >= n || m >= M) return;
  const double* y = Y + m * len;
  double p = 0.0;
  for (int q = 0; q < k; ++q) p = __dadd_rn(p, __dmul_rn(w[t * k + q], y[idx[t * k + q] + offset]));
  pred[m * n + t] = p;
}

__global__ void __launch_bounds__(1024) lookup64_rho_kernel(const double* __restrict__ Y, int64_t len,
                                                             int64_t n, int offset,
                                                             const double* __restrict__ pred,
                                                             double* __restrict__ rho) {
  __shared__ double scratch[33];
  __shared__ double agg[6];
  const int64_t m = blockIdx.x;
  pearson_blocks(Y + m * len + offset, pred + m * n, n, agg, scratch);
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = nan_d();
    if (agg[0] >= 2 && agg[3] > 0.0 && agg[4] > 0.0) r = fmin(1.0, fmax(-1.0, agg[5] / sqrt(agg[3] * agg[4])));
    rho[m] = r;
  }
}

__global__ void transpose_kernel(const float* __restrict__ src, int64_t rows, int64_t cols,
                                 int64_t lds, float* __restrict__ dst, int64_t ldd) {
  __shared__ float tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t rr = r0 + r, cc = c0 + threadIdx.x;
    if (rr < rows && cc < cols) tile[r][threadIdx.x] = src[rr * lds + cc];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t cc = c0 + r, rr = r0 + threadIdx.x;
    if (rr < rows && cc < cols) dst[cc * ldd + rr] = tile[threadIdx.x][r];
  }
}

int grid_for(int64_t total, int block) {
  int64_t g = (total + block - 1) / block;
  if (g > 148 * 64) g = 148 * 64;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

cudaError_t launch_series_stats(const float* x32, int64_t N, int64_t T, int64_t ld, double* mean,
                                cudaStream_t st) {
  if (N == 0) return cudaSuccess;
  count_launch();
  series_mean_kernel<<<(unsigned)((N + 7) / 8), 256, 0, st>>>(x32, N, T, ld, mean);
  return cudaGetLastError();
}

cudaError_t launch_promote(const float* x32, int64_t N, int64_t T, int64_t ld, double* x64,
                           cudaStream_t st) {
  count_launch();
  promote_kernel<<<grid_for(N * ld, 256), 256, 0, st>>>(x32, N, T, ld, x64);
  return cudaGetLastError();
}

cudaError_t launch_demote(const double* x64, int64_t N, int64_t T, float* x32, float* err_m,
                          cudaStream_t st) {
  if (N == 0) return cudaSuccess;
  count_launch();
  demote_kernel<<<(unsigned)N, 256, 0, st>>>(x64, N, T, x32, err_m);
  return cudaGetLastError();
}

cudaError_t launch_demote_center(const double* x64, int64_t N, int64_t T, float* x32, float* err_m,
                                 double* mu, cudaStream_t st) {
  if (N == 0) return cudaSuccess;
  count_launch();
  demote_center_kernel<<<(unsigned)N, 256, 0, st>>>(x64, T, x32, err_m, mu);
  return cudaGetLastError();
}

__global__ void slot_shift_kernel(const double* __restrict__ mean, const double* __restrict__ mu,
                                  const int32_t* __restrict__ slot_tgt, int64_t slots, double* __restrict__ shift) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= slots) return;
  const int t = slot_tgt[s];
  shift[s] = t < 0 ? 0.0 : (double)(float)mean[t] + (mu ? mu[t] : 0.0);
}

cudaError_t launch_slot_shift(const double* mean, const double* mu, const int32_t* slot_tgt, int64_t slots,
                              double* shift, cudaStream_t st) {
  if (slots == 0) return cudaSuccess;
  count_launch();
  slot_shift_kernel<<<(unsigned)((slots + 255) / 256), 256, 0, st>>>(mean, mu, slot_tgt, slots, shift);
  return cudaGetLastError();
}

cudaError_t launch_build_targets(const float* x32, int64_t ld, const double* mean,
                                 const int32_t* slot_tgt, int64_t slots, int T, float* Y,
                                 int64_t ldy, cudaStream_t st) {
  dim3 grid((T + 31) / 32, (unsigned)((ldy + 31) / 32));
  count_launch();
  build_targets_kernel<<<grid, dim3(32, 8), 0, st>>>(x32, ld, mean, slot_tgt, slots, T, Y, ldy);
  return cudaGetLastError();
}

cudaError_t launch_obs_moments(const float* Y, int64_t ldy, int T, int tau, const int32_t* slot_E,
                               int64_t slots, double* s, double* ss, uint8_t* cst, cudaStream_t st) {
  if (slots == 0) return cudaSuccess;
  count_launch();
  obs_moments_kernel<<<(unsigned)((slots + 127) / 128), 128, 0, st>>>(Y, ldy, T, tau, slot_E, slots,
                                                                     s, ss, cst);
  return cudaGetLastError();
}

cudaError_t launch_targets_to_half(const float* Y, int64_t ldy, int T, int tau, const int32_t* slot_E,
                                   int64_t slots, void* Yh, double* s, double* ss, uint8_t* cst,
                                   int mode, cudaStream_t st) {
  if (slots == 0) return cudaSuccess;
  count_launch();
  targets_to_half_kernel<<<(unsigned)((slots + 127) / 128), 128, 0, st>>>(
      Y, ldy, T, tau, slot_E, slots, reinterpret_cast<__half*>(Yh), s, ss, cst, mode);
  return cudaGetLastError();
}

__global__ void copy_count_kernel(const int* __restrict__ src, volatile int* dst) { *dst = *src; }

cudaError_t launch_copy_count(const int* src, int* dst, cudaStream_t st) {
  count_launch();
  copy_count_kernel<<<1, 1, 0, st>>>(src, dst);
  return cudaGetLastError();
}

cudaError_t launch_fill_nan(float* p, int64_t rows, int64_t cols, int64_t ld, cudaStream_t st) {
  if (rows * cols == 0) return cudaSuccess;
  count_launch();
  fill_nan_kernel<<<grid_for(rows * cols, 256), 256, 0, st>>>(p, rows, cols, ld);
  return cudaGetLastError();
}

cudaError_t launch_pairwise(const double* x, int n, int E, int tau, double* D, cudaStream_t st) {
  dim3 grid((n + 127) / 128, n);
  count_launch();
  pairwise_kernel<<<grid, 128, 0, st>>>(x, n, E, tau, D);
  return cudaGetLastError();
}

cudaError_t launch_topk_rows(const double* D, int n, int k, double* d_out, int64_t* i_out,
                             cudaStream_t st) {
  int npad = 1;
  while (npad < n) npad <<= 1;
  if (npad < 2) npad = 2;
  const size_t smem = (size_t)npad * (sizeof(double) + sizeof(int));
  if (smem > 232448) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(topk_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  count_launch();
  topk_rows_kernel<<<n, 512, smem, st>>>(D, n, npad, k, d_out, i_out);
  return cudaGetLastError();
}

cudaError_t launch_weights(const double* sq, int64_t n, int k, double* w, int* flags,
                           cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  count_launch();
  weights_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(sq, n, k, w, flags);
  return cudaGetLastError();
}

cudaError_t launch_pearson(const double* a, const double* b, int64_t n, double* agg,
                           cudaStream_t st) {
  count_launch();
  pearson_kernel<<<1, 1024, 0, st>>>(a, b, n, agg);
  return cudaGetLastError();
}

cudaError_t launch_lookup64(const int64_t* idx, const double* w, int64_t n, int k, int offset,
                            const double* Y, int64_t len, int64_t M, double* pred, double* rho,
                            cudaStream_t st) {
  if (M == 0 || n == 0) return cudaSuccess;
  dim3 g1((unsigned)((n + 255) / 256), (unsigned)M);
  count_launch();
  lookup64_pred_kernel<<<g1, 256, 0, st>>>(idx, w, n, k, offset, Y, len, M, pred);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  count_launch();
  lookup64_rho_kernel<<<(unsigned)M, 1024, 0, st>>>(Y, len, n, offset, pred, rho);
  return cudaGetLastError();
}

cudaError_t launch_transpose_f32(const float* src, int64_t rows, int64_t cols, int64_t lds,
                                 float* dst, int64_t ldd, cudaStream_t st) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  count_launch();
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src, rows, cols, lds, dst, ldd);
  return cudaGetLastError();
}

}  // namespace cmb
