// Gather strategies for 80-byte dimension rows into shared memory (32-row blocks per warp).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cpa16(void* d, const void* s) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(d)), "l"(s) : "memory");
}
// (a) cp.async 16B pieces, lane -> (row, piece)
__global__ void k_cpasync(const double* __restrict__ V, const int* __restrict__ keys, long n, double* out) {
  __shared__ __align__(16) double buf[8][32 * 10];
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long nb = n / 32, gw = blockIdx.x * 8 + w, W = gridDim.x * 8;
  double acc = 0;
  for (long b = gw; b < nb; b += W) {
    const int* kk = keys + b * 32;
    for (int j = lane; j < 160; j += 32) {
      int rr = j / 5, pc = j % 5;
      cpa16(&buf[w][rr * 10 + 2 * pc], V + (long)kk[rr] * 12 + 2 * pc);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    acc += buf[w][lane * 10];
    __syncwarp();
  }
  if (acc == 1.2345) out[0] = acc;
}
// (b) LDG.128 lane = row, 5 loads, STS
__global__ void k_ldg(const double* __restrict__ V, const int* __restrict__ keys, long n, double* out) {
  __shared__ __align__(16) double buf[8][32 * 10];
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long nb = n / 32, gw = blockIdx.x * 8 + w, W = gridDim.x * 8;
  double acc = 0;
  for (long b = gw; b < nb; b += W) {
    int key = keys[b * 32 + lane];
    const double2* r = reinterpret_cast<const double2*>(V + (long)key * 12);
    double2 v0 = r[0], v1 = r[1], v2 = r[2], v3 = r[3], v4 = r[4];
    double2* d = reinterpret_cast<double2*>(&buf[w][lane * 10]);
    d[0] = v0; d[1] = v1; d[2] = v2; d[3] = v3; d[4] = v4;
    __syncwarp();
    acc += buf[w][((lane + 1) & 31) * 10];
    __syncwarp();
  }
  if (acc == 1.2345) out[0] = acc;
}
// (c) LDG.64 in DMMA layout directly (lane (m,k): col m and 8+m of row k), 8 groups per block
__global__ void k_ldg_dmma(const double* __restrict__ V, const int* __restrict__ keys, long n, double* out) {
  int lane = threadIdx.x & 31, k = lane & 3, m = lane >> 2;
  long nb = n / 32, gw = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), W = gridDim.x * (blockDim.x / 32);
  double acc = 0;
  for (long b = gw; b < nb; b += W) {
    int kl = keys[b * 32 + lane];
#pragma unroll
    for (int j = 0; j < 8; j++) {
      int key = __shfl_sync(0xffffffffu, kl, 4 * j + k);
      const double* r = V + (long)key * 12;
      acc += r[m] + (m < 2 ? r[8 + m] : 0.0);
    }
  }
  if (acc == 1.2345) out[0] = acc;
}
__global__ void k_init(int* keys, long n, int nrows) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    unsigned long long x = (unsigned long long)(i / 2) * 0x9E3779B97F4A7C15ull;  // runs of 2
    x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    keys[i] = (int)(x % (unsigned long long)nrows);
  }
}
template <typename F> float tm(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); f(); cudaDeviceSynchronize();
  float best = 1e9;
  for (int r = 0; r < 5; r++) { cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best; }
  return best;
}
int main() {
  long n = 10l << 20; int nr = 100000;
  int* keys; double* V; double* out;
  cudaMalloc(&keys, n * 4); cudaMalloc(&V, (long)nr * 12 * 8 + 1024); cudaMalloc(&out, 64);
  cudaMemset(V, 0, (long)nr * 12 * 8);
  k_init<<<1184, 256>>>(keys, n, nr);
  printf("cp.async 16B     : %.3f ms\n", tm([&] { k_cpasync<<<148 * 2, 256>>>(V, keys, n, out); }));
  printf("LDG.128 lane=row : %.3f ms\n", tm([&] { k_ldg<<<148 * 2, 256>>>(V, keys, n, out); }));
  printf("LDG.64 dmma 8w   : %.3f ms\n", tm([&] { k_ldg_dmma<<<148 * 2, 256>>>(V, keys, n, out); }));
  printf("LDG.64 dmma 16w  : %.3f ms\n", tm([&] { k_ldg_dmma<<<148 * 4, 256>>>(V, keys, n, out); }));
  return 0;
}
