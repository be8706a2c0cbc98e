// Step-0 microbenchmarks for the B200 (sm_100a) hot path of lmfao_gpu.
// Measures the rates SURVEY.md §7 step 0 asks for, which decide the design of
// the root-scan kernel (c) and its Gram tiles (d):
//   * FP64 DFMA throughput and FP64 DMMA (mma.sync m8n8k4 .f64) throughput,
//     alone and interleaved (do they share a pipe?);
//   * shared-memory and global FP64/u32 atomic rates;
//   * L2-resident random row-gather bandwidth (view lookups);
//   * HBM streaming read bandwidth.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks peaks.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void k_dfma(double* out, int iters, double a) {
  double r[16];
#pragma unroll
  for (int i = 0; i < 16; i++) r[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) r[i] = fma(r[i], a, 1e-7);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += r[i];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, int iters, double a) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
  double av = a + threadIdx.x * 1e-9, bv = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) dmma(c[i][0], c[i][1], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// interleave: per iteration 4 DMMA (4*256 FMA/warp) + 32 DFMA per lane (32*32 FMA/warp)
__global__ void k_mixed(double* out, int iters, double a) {
  double c[4][2];
  double r[16];
#pragma unroll
  for (int i = 0; i < 4; i++) { c[i][0] = 0; c[i][1] = 0; }
#pragma unroll
  for (int i = 0; i < 16; i++) r[i] = threadIdx.x * 1e-9 + i;
  double av = a + threadIdx.x * 1e-9, bv = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++) dmma(c[i][0], c[i][1], av, bv);
#pragma unroll
    for (int i = 0; i < 16; i++) r[i] = fma(r[i], a, 1e-7);
#pragma unroll
    for (int i = 0; i < 16; i++) r[i] = fma(r[i], a, 1e-7);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 16; i++) s += r[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_smem_atomic_f64(double* out, int iters, int spread) {
  __shared__ double h[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
  __syncthreads();
  unsigned idx = (threadIdx.x * 7919u) % (unsigned)spread;
  for (int it = 0; it < iters; it++) {
    atomicAdd(&h[idx], 1.0);
    idx = (idx * 1103515245u + 12345u) % (unsigned)spread;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[0];
}

__global__ void k_smem_atomic_u32(unsigned* out, int iters, int spread) {
  __shared__ unsigned h[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
  __syncthreads();
  unsigned idx = (threadIdx.x * 7919u) % (unsigned)spread;
  for (int it = 0; it < iters; it++) {
    atomicAdd(&h[idx], (unsigned)(it & 3) + 1u);
    idx = (idx * 1103515245u + 12345u) % (unsigned)spread;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[0];
}

__global__ void k_gmem_red_f64(double* tab, int iters, unsigned spread) {
  unsigned idx = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u % spread;
  for (int it = 0; it < iters; it++) {
    atomicAdd(&tab[idx], 1.0);
    idx = (idx * 1103515245u + 12345u) % spread;
  }
}

__global__ void k_gmem_red_u32(unsigned* tab, int iters, unsigned spread) {
  unsigned idx = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u % spread;
  for (int it = 0; it < iters; it++) {
    atomicAdd(&tab[idx], 1u);
    idx = (idx * 1103515245u + 12345u) % spread;
  }
}

// gather rows of W doubles from a table of nrows (L2 resident), random keys
template <int W>
__global__ void k_gather(const double* __restrict__ tab, const int* __restrict__ keys, long n, double* out) {
  double acc = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const double* row = tab + (long)keys[i] * W;
#pragma unroll
    for (int j = 0; j < W; j += 2) {
      double2 v = *reinterpret_cast<const double2*>(row + j);
      acc += v.x + v.y;
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void k_stream(const double2* __restrict__ a, long n2, double* out) {
  double acc = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
    double2 v = __ldcs(a + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void k_init_keys(int* keys, long n, int nrows) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    unsigned long long x = (unsigned long long)i * 0x9E3779B97F4A7C15ull;
    x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    keys[i] = (int)(x % (unsigned long long)nrows);
  }
}

template <typename F>
float time_ms(F f, int reps = 5) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_block_optin\": %zu, \"clock_khz\": %d,\n",
         p.name, sms, p.l2CacheSize, p.sharedMemPerBlockOptin, p.clockRate);
  double* dout; CK(cudaMalloc(&dout, 1 << 20));
  const int iters = 4096;
  // DFMA: blocks = sms*8, 256 thr, 16 fma per iter
  {
    int blocks = sms * 8, thr = 256;
    float ms = time_ms([&] { k_dfma<<<blocks, thr>>>(dout, iters, 0.999999); });
    double fmas = (double)blocks * thr * iters * 16;
    printf(" \"dfma_tfma_per_s\": %.3f,\n", fmas / ms / 1e9);
  }
  {
    int blocks = sms * 8, thr = 256;
    float ms = time_ms([&] { k_dmma<<<blocks, thr>>>(dout, iters, 0.999999); });
    double fmas = (double)blocks * (thr / 32) * iters * 8 * 256;
    printf(" \"dmma_tfma_per_s\": %.3f,\n", fmas / ms / 1e9);
  }
  {
    int blocks = sms * 8, thr = 256;
    float ms = time_ms([&] { k_mixed<<<blocks, thr>>>(dout, iters, 0.999999); });
    double f_dmma = (double)blocks * (thr / 32) * iters * 4 * 256;
    double f_dfma = (double)blocks * thr * iters * 32;
    printf(" \"mixed_ms\": %.4f, \"mixed_dmma_tfma\": %.3f, \"mixed_dfma_tfma\": %.3f, \"mixed_total_tfma\": %.3f,\n",
           ms, f_dmma / ms / 1e9, f_dfma / ms / 1e9, (f_dmma + f_dfma) / ms / 1e9);
  }
  const int aiters = 2048;
  for (int spread : {1, 32, 1024, 4096}) {
    int blocks = sms * 4, thr = 512;
    float ms = time_ms([&] { k_smem_atomic_f64<<<blocks, thr>>>(dout, aiters, spread); });
    double ops = (double)blocks * thr * aiters;
    printf(" \"smem_atom_f64_spread%d_gops\": %.2f,\n", spread, ops / ms / 1e6);
    ms = time_ms([&] { k_smem_atomic_u32<<<blocks, thr>>>((unsigned*)dout, aiters, spread); });
    printf(" \"smem_atom_u32_spread%d_gops\": %.2f,\n", spread, ops / ms / 1e6);
  }
  {
    size_t tabn = 16u << 20;  // 16M entries
    double* tab; CK(cudaMalloc(&tab, tabn * 8)); CK(cudaMemset(tab, 0, tabn * 8));
    for (unsigned spread : {1u << 10, 100000u, 1u << 20, 16u << 20}) {
      int blocks = sms * 8, thr = 256, it = 256;
      float ms = time_ms([&] { k_gmem_red_f64<<<blocks, thr>>>(tab, it, spread); });
      double ops = (double)blocks * thr * it;
      printf(" \"gmem_red_f64_spread%u_gops\": %.2f,\n", spread, ops / ms / 1e6);
      ms = time_ms([&] { k_gmem_red_u32<<<blocks, thr>>>((unsigned*)tab, it, spread); });
      printf(" \"gmem_red_u32_spread%u_gops\": %.2f,\n", spread, ops / ms / 1e6);
    }
    cudaFree(tab);
  }
  {
    long n = 10l << 20;
    int* keys; CK(cudaMalloc(&keys, n * 4));
    double* tab; CK(cudaMalloc(&tab, 100000l * 16 * 8)); CK(cudaMemset(tab, 0, 100000l * 16 * 8));
    k_init_keys<<<sms * 4, 256>>>(keys, n, 100000);
    float ms = time_ms([&] { k_gather<12><<<sms * 8, 256>>>(tab, keys, n, dout); });
    printf(" \"gather12_rows_per_s_G\": %.2f, \"gather12_GBps\": %.1f,\n", n / ms / 1e6, n * (96.0 + 4) / ms / 1e6);
    ms = time_ms([&] { k_gather<16><<<sms * 8, 256>>>(tab, keys, n, dout); });
    printf(" \"gather16_rows_per_s_G\": %.2f, \"gather16_GBps\": %.1f,\n", n / ms / 1e6, n * (128.0 + 4) / ms / 1e6);
    cudaFree(keys); cudaFree(tab);
  }
  {
    long bytes = 2l << 30;
    double2* a; CK(cudaMalloc(&a, bytes)); CK(cudaMemset(a, 0, bytes));
    for (int occ : {4, 8, 16}) {
      float ms = time_ms([&] { k_stream<<<sms * occ, 256>>>(a, bytes / 16, dout); });
      printf(" \"stream_read_occ%d_GBps\": %.1f,\n", occ, bytes / ms / 1e6);
    }
    cudaFree(a);
  }
  printf(" \"ok\": true}\n");
  return 0;
}
