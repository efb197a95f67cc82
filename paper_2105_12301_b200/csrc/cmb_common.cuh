// Shared device/host helpers for libcmb200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "../../include/cmb200.h"

#define CMB_WARP 32
#define CMB_FULL 0xffffffffu

// Largest embedding dimension handled by the fused register-list kNN sweep
// (list length E + 2 <= 32 lanes).
#define CMB_SWEEP_MAX_E 30

namespace cmb {

// ---------------------------------------------------------------- host errors
void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define CMB_CUDA(call)                                                          \
  do {                                                                          \
    cudaError_t _e = (call);                                                    \
    if (_e != cudaSuccess) return ::cmb::cuda_fail(_e, #call, __FILE__, __LINE__); \
  } while (0)

#define CMB_PARAM(cond, ...)                                                    \
  do {                                                                          \
    if (!(cond)) { ::cmb::set_error(__VA_ARGS__); return CMB_ERR_PARAM; }      \
  } while (0)

// ---------------------------------------------------------------- lookup table records
// One record per embedded point t of a library at dimension E (k = E + 1):
//   float    w[rec_nw(k)]  simplex weights
//   uint16_t row[rec_nr(k)] target sample positions idx + (E-1)*tau, zero padded
// k >= 4: kp4 = round_up(k, 4) weights (zero padded) and kp8 = round_up(k, 8)
// rows (zero padded to fill the record) -- an odd multiple of 16 bytes.  k <= 3 (E = 1, 2: half of all targets in the
// mixed data) stores k - 1 weights, the last being 1 - (sum of the others), so
// an E = 1 record is 8 bytes: one broadcast shared-memory load in the lookup
// instead of two.  A library's records start on a 16-byte boundary
// (rec_lib_stride) so tables move with cp.async.bulk.
__host__ __device__ constexpr int rec_kp4(int k) { return (k + 3) & ~3; }
__host__ __device__ constexpr int rec_kp8(int k) { return (k + 7) & ~7; }
__host__ __device__ constexpr bool rec_implicit(int k) { return k <= 3; }
__host__ __device__ constexpr int rec_nw(int k) { return rec_implicit(k) ? k - 1 : rec_kp4(k); }
__host__ __device__ constexpr int rec_row_off(int k) { return 4 * rec_nw(k); }
// k >= 4 records are an ODD number of 16-byte chunks (one zero chunk appended
// when the packed size is even): the rotated lookup reads 8 consecutive records
// per quarter-warp with 16-byte loads, and an odd chunk stride puts them in 8
// distinct bank quads (an even stride such as 128 B would be an 8-way conflict).
__host__ __device__ constexpr int rec_bytes_packed(int k) { return 4 * rec_kp4(k) + 2 * rec_kp8(k); }
__host__ __device__ constexpr int rec_bytes(int k) {
  return rec_implicit(k) ? ((4 * (k - 1) + 2 * k + 7) & ~7)
                         : rec_bytes_packed(k) + (((rec_bytes_packed(k) >> 4) & 1) ? 0 : 16);
}
// row slots (zero padded) filling the record after the weights
__host__ __device__ constexpr int rec_nr(int k) { return (rec_bytes(k) - rec_row_off(k)) / 2; }
__host__ __device__ constexpr size_t rec_lib_stride(int k, int64_t n) {
  return ((size_t)n * (size_t)rec_bytes(k) + 15) & ~(size_t)15;
}
static_assert(rec_bytes(2) == 8 && rec_bytes(3) == 16 && rec_bytes(4) == 48 && rec_bytes(8) == 48 &&
                  rec_bytes(20) == 144 && rec_bytes(21) == 144, "record layout");
static_assert(rec_nr(2) == 2 && rec_nr(3) == 4 && rec_nr(4) == 16 && rec_nr(21) == 24, "record rows");

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

// Squared fp64 distance between embedded points i and j in exactly the
// reference's operation order: (a - b), square, running sum over e = 0..E-1,
// no fused multiply-add (knn.py:118-125 / prediction.py:211-230).
__device__ __forceinline__ double exact_sqdist(const double* __restrict__ x, int i, int j,
                                               int E, int tau) {
  double acc = 0.0;
  for (int e = 0; e < E; ++e) {
    double d = __dsub_rn(__ldg(x + i + e * tau), __ldg(x + j + e * tau));
    acc = __dadd_rn(acc, __dmul_rn(d, d));
  }
  return acc;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(CMB_FULL, v, o);
  return v;
}

}  // namespace cmb
