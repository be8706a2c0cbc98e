// Latency microbenchmarks (single warp, dependent chains): DMMA m8n8k4 f64, DFMA, LDS.64.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void k(long long* out, double a, int n, int chains) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = i * 0.5;
  __syncwarp();
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    dmma(c[0][0], c[0][1], a, a);
    if (chains > 1) dmma(c[1][0], c[1][1], a, a);
    if (chains > 2) dmma(c[2][0], c[2][1], a, a);
    if (chains > 3) dmma(c[3][0], c[3][1], a, a);
  }
  long long t1 = clock64();
  double r = a;
  for (int i = 0; i < n; i++) r = fma(r, a, 1e-9);
  long long t2 = clock64();
  unsigned idx = threadIdx.x;
  for (int i = 0; i < n; i++) { double v = sm[idx & 1023]; idx = (unsigned)v + threadIdx.x; }
  long long t3 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; }
  if (c[0][0] + c[1][1] + c[2][0] + c[3][1] + r + idx == 1234.5) out[3] = 1;
}
int main() {
  long long* d; cudaMalloc(&d, 64); long long h[4];
  for (int ch : {1, 2, 4}) {
    k<<<1, 32>>>(d, 1.0000001, 1000, ch); cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("chains=%d: DMMA %.1f cyc/iter (per dependent DMMA), DFMA dep %.1f cyc, LDS dep %.1f cyc\n",
           ch, h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0);
  }
  return 0;
}
