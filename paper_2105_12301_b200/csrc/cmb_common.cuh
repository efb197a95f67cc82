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
//   float    w[kp4]   simplex weights, zero padded        (16-byte aligned)
//   uint16_t row[kp8] target sample positions idx + (E-1)*tau, zero padded
// kp4 = round_up(k, 4), kp8 = round_up(k, 8).  Record bytes are a multiple
// of 16 so records and tables can be moved with cp.async.bulk.
__host__ __device__ constexpr int rec_kp4(int k) { return (k + 3) & ~3; }
__host__ __device__ constexpr int rec_kp8(int k) { return (k + 7) & ~7; }
__host__ __device__ constexpr int rec_bytes(int k) { return 4 * rec_kp4(k) + 2 * rec_kp8(k); }

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
