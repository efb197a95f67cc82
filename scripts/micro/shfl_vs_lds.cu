// Microbenchmark: throughput of broadcast LDS.64, per-lane LDS.32 and SHFL.IDX on one SM type.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o shfl_vs_lds shfl_vs_lds.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lds_bcast(float* out, int iters) {
  __shared__ float2 s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_float2(i, i);
  __syncthreads();
  float acc = 0.f; int a = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) { float2 v = s[(a + u * 7 + it) & 1023]; acc += v.x * v.y; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_lds_lane(float* out, int iters) {
  __shared__ float s[32 * 64];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = i;
  __syncthreads();
  float acc = 0.f; int l = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += s[(((u * 5 + it) & 63) << 5) + l];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_shfl(float* out, int iters) {
  float v = threadIdx.x, acc = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += __shfl_sync(0xffffffff, v, (u + it) & 31);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_mix(float* out, int iters) {  // 8 per-lane LDS + 8 SHFL per step
  __shared__ float s[32 * 64];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = i;
  __syncthreads();
  float acc = 0.f, v = threadIdx.x; int l = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc += s[(((u * 5 + it) & 63) << 5) + l];
      acc += __shfl_sync(0xffffffff, v, (u + it) & 31);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sizeof(float) * sms * 4 * 1024);
  const int iters = 4096, threads = 1024, blocks = sms * 2;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"lds64_bcast", "lds32_lane", "shfl", "mix8lds+8shfl"};
  void (*ks[])(float*, int) = {k_lds_bcast, k_lds_lane, k_shfl, k_mix};
  for (int q = 0; q < 4; ++q) {
    ks[q]<<<blocks, threads>>>(out, 16);
    cudaEventRecord(a);
    ks[q]<<<blocks, threads>>>(out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double warp_ops = (double)blocks * (threads / 32) * iters * 16;  // memory/shuffle warp-instructions
    printf("%-16s %8.3f ms  %.3f warp-ops/clk/SM (at %d MHz)\n", names[q], ms,
           warp_ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
