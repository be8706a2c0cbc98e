// microbench/atomics.cu — round-2 companion of peaks.cu: FP64 pipe sharing re-checked, plus
// random-address global atomics over a 2 GiB table (the C5 cube design question).
//
// Not part of the product path: a standalone program printing one JSON object with
//   dfma      FP64 FMA throughput (independent chains, all SMs)
//   dmma      FP64 mma.sync m8n8k4 throughput (256 FMA per instruction)
//   mixed     DMMA and DFMA interleaved in the same warps (do they share a pipe?)
//   dmma_lat  dependent DMMA latency (cycles), one warp
//   red_f64   global red.add.f64 to random addresses of a 2 GiB table, and to 64 hot lines
//   ratom_cas global atomicCAS to random addresses (a hash-insert probe)
//   sred_f64  shared red.add.f64 (per-lane private addresses)
//   hbm_read  streaming read (int4 loads, grid-stride)
//   l2_gather 96-byte rows gathered at random from a 9.6 MB table (L2 resident)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o microbench/atomics microbench/atomics.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

constexpr int CH = 8;  // independent chains per thread

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double c[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) c[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) s += c[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma(double* out, int iters, double a, double b) {
  double d[CH][2];
#pragma unroll
  for (int i = 0; i < CH; i++) d[i][0] = d[i][1] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) dmma(d[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) s += d[i][0] + d[i][1];
  if (s == 12345.678) out[0] = s;
}

// per iteration: CH/2 DMMA (128 FMA each per lane-equivalent: 256 per warp) + CH DFMA per lane
__global__ void k_mixed(double* out, int iters, double a, double b) {
  double d[CH / 2][2], c[CH];
#pragma unroll
  for (int i = 0; i < CH / 2; i++) d[i][0] = d[i][1] = i;
#pragma unroll
  for (int i = 0; i < CH; i++) c[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH / 2; i++) {
      dmma(d[i], a, b);
      c[2 * i] = fma(c[2 * i], a, b);
      c[2 * i + 1] = fma(c[2 * i + 1], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH / 2; i++) s += d[i][0] + d[i][1];
#pragma unroll
  for (int i = 0; i < CH; i++) s += c[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma_lat(double* out, long long* cyc, int iters, double a, double b) {
  double d[2] = {1.0, 2.0};
  const long long t0 = clock64();
  for (int it = 0; it < iters; it++) dmma(d, a + d[0] * 1e-30, b);
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (d[0] == 12345.678) out[0] = d[1];
}

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

__global__ void k_red_rand(double* t, uint64_t mask, int per_thread) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (int i = 0; i < per_thread; i++) {
    const uint64_t h = mix(tid * 1315423911ull + i) & mask;
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(t + h), "d"(1.0) : "memory");
  }
}

__global__ void k_cas_rand(unsigned long long* t, uint64_t mask, int per_thread, unsigned long long* hits) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  unsigned long long n = 0;
  for (int i = 0; i < per_thread; i++) {
    const uint64_t h = mix(tid * 2654435761ull + i) & mask;
    n += atomicCAS(t + h, 0ull, tid + 1) == 0ull;
  }
  if (n == 0xffffffffffull) hits[0] = n;
}

__global__ void k_sred(double* out, int iters) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm) + 8u * ((threadIdx.x * 7) & 2047);
  for (int it = 0; it < iters; it++)
    asm volatile("red.shared.add.f64 [%0], %1;" ::"r"(base), "d"(1.0) : "memory");
  __syncthreads();
  if (threadIdx.x == 0 && sm[5] == 12345.678) out[0] = sm[5];
}

__global__ void k_read(const int4* __restrict__ p, size_t n, int* out) {
  int acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int4 v = __ldg(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

// one row = 12 doubles (96 B); each lane gathers a whole row (6 x 16 B)
__global__ void k_gather(const double2* __restrict__ tab, uint64_t nrow, int per_thread, double* out) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  double s = 0;
  for (int i = 0; i < per_thread; i++) {
    const uint64_t r = mix(tid * 40503ull + i) % nrow;
#pragma unroll
    for (int j = 0; j < 6; j++) {
      const double2 v = __ldg(tab + r * 6 + j);
      s += v.x + v.y;
    }
  }
  if (s == 12345.678) out[0] = s;
}

template <class F>
static float time_ms(F f, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int nsm = p.multiProcessorCount;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double* out;
  long long* cyc;
  CK(cudaMalloc(&out, 64));
  CK(cudaMalloc(&cyc, 64));
  const int iters = 4096, thr = 256, blocks = nsm * 8;
  const double a = 1.0000001, b = 1e-9;

  const float t_dfma = time_ms([&] { k_dfma<<<blocks, thr>>>(out, iters, a, b); });
  const double dfma = (double)blocks * thr * iters * CH / (t_dfma * 1e-3);
  const float t_dmma = time_ms([&] { k_dmma<<<blocks, thr>>>(out, iters, a, b); });
  const double dmma_fma = (double)blocks * (thr / 32) * iters * CH * 256.0 / (t_dmma * 1e-3);
  const float t_mix = time_ms([&] { k_mixed<<<blocks, thr>>>(out, iters, a, b); });
  const double mix_fma = ((double)blocks * (thr / 32) * iters * (CH / 2) * 256.0 +
                          (double)blocks * thr * iters * CH) / (t_mix * 1e-3);
  k_dmma_lat<<<1, 32>>>(out, cyc, iters, a, b);
  CK(cudaDeviceSynchronize());
  long long cy = 0;
  CK(cudaMemcpy(&cy, cyc, 8, cudaMemcpyDeviceToHost));
  const double lat = (double)cy / iters;

  // global REDs: 2 GiB table (256 Mi doubles), random; and 64 hot 128-B lines (1024 doubles)
  const uint64_t nt = 1ull << 28;
  double* tab;
  CK(cudaMalloc(&tab, nt * 8));
  CK(cudaMemset(tab, 0, nt * 8));
  const int per = 64, rb = nsm * 16;
  const float t_red = time_ms([&] { k_red_rand<<<rb, thr>>>(tab, nt - 1, per); });
  const double red_rand = (double)rb * thr * per / (t_red * 1e-3);
  const float t_redh = time_ms([&] { k_red_rand<<<rb, thr>>>(tab, 1023, per); });
  const double red_hot = (double)rb * thr * per / (t_redh * 1e-3);
  CK(cudaMemset(tab, 0, nt * 8));
  const float t_cas = time_ms([&] { k_cas_rand<<<rb, thr>>>(reinterpret_cast<unsigned long long*>(tab), nt - 1, per,
                                                         reinterpret_cast<unsigned long long*>(out)); }, 1);
  const double cas_rand = (double)rb * thr * per / (t_cas * 1e-3);

  const float t_sred = time_ms([&] { k_sred<<<nsm * 4, thr, 32 * 64 * 8>>>(out, iters); });
  const double sred = (double)nsm * 4 * thr * iters / (t_sred * 1e-3);

  // HBM streaming read of the 2 GiB table
  const float t_rd = time_ms([&] { k_read<<<nsm * 8, 512>>>(reinterpret_cast<const int4*>(tab), nt * 8 / 16,
                                                           reinterpret_cast<int*>(out)); });
  const double hbm = (double)nt * 8 / (t_rd * 1e-3) / 1e9;

  // L2-resident gather: 100k rows x 96 B (9.6 MB)
  const uint64_t nrow = 100000;
  const int gper = 64;
  const float t_g = time_ms([&] { k_gather<<<nsm * 16, thr>>>(reinterpret_cast<const double2*>(tab), nrow, gper, out); });
  const double gather = (double)nsm * 16 * thr * gper / (t_g * 1e-3);

  CK(cudaGetLastError());
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %.0f,\n", p.name, nsm, clk_khz / 1e3);
  printf(" \"dfma_tfma_s\": %.2f, \"dmma_tfma_s\": %.2f, \"mixed_dmma_dfma_tfma_s\": %.2f,\n", dfma / 1e12, dmma_fma / 1e12,
         mix_fma / 1e12);
  printf(" \"dmma_dependent_latency_cycles\": %.1f,\n", lat);
  printf(" \"red_f64_random_2GiB_g_s\": %.2f, \"red_f64_hot_64lines_g_s\": %.2f, \"cas_u64_random_2GiB_g_s\": %.2f,\n",
         red_rand / 1e9, red_hot / 1e9, cas_rand / 1e9);
  printf(" \"sred_f64_g_s\": %.1f, \"hbm_stream_read_gb_s\": %.0f, \"l2_gather_96B_rows_g_s\": %.1f,\n", sred / 1e9, hbm,
         gather / 1e9);
  printf(" \"how\": \"microbench/atomics.cu: best of 5 (CAS: 1) CUDA-event-timed launches after a warm-up; %d blocks x %d threads for FP64\"}\n",
         blocks, thr);
  return 0;
}
