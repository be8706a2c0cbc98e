// microbench/columns.cu — does reading NC separate fp64 columns chunk by chunk (the view build's
// access pattern: a warp sums 512 rows of each column, chunks dealt round-robin to the warps)
// stream as fast as one array?  Prints GB/s for: one array grid-stride; NC columns with the
// chunked pattern; NC columns grid-stride (all columns at the same row window).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o microbench/columns microbench/columns.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NC = 10;
struct Cols { const double* c[NC]; };

__global__ void k_one(const double2* __restrict__ a, long n2, double* out) {
  double s = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
    const double2 v = a[i];
    s += v.x + v.y;
  }
  if (s == 1.2345) out[0] = s;
}
template <int CH>
__global__ void __launch_bounds__(256, 4) k_chunked(Cols cs, long nrows, double* out) {
  const int lane = threadIdx.x & 31;
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = ((long)gridDim.x * blockDim.x) >> 5;
  const long nch = nrows / (32 * CH);
  double tot = 0;
  for (long ch = gw; ch < nch; ch += nw) {
#pragma unroll
    for (int s = 0; s < NC; s++) {
      const double2* c = reinterpret_cast<const double2*>(cs.c[s] + ch * 32 * CH);
      double x = 0, y = 0;
#pragma unroll
      for (int j = 0; j < CH / 2; j++) {
        const double2 w = c[lane + 32 * j];
        x += w.x;
        y += w.y;
      }
      tot += x + y;
    }
  }
  if (tot == 1.2345) out[0] = tot;
}
__global__ void k_cols_stride(Cols cs, long nrows, double* out) {
  double s = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < nrows / 2; i += (long)gridDim.x * blockDim.x)
#pragma unroll
    for (int c = 0; c < NC; c++) {
      const double2 v = reinterpret_cast<const double2*>(cs.c[c])[i];
      s += v.x + v.y;
    }
  if (s == 1.2345) out[0] = s;
}
template <class F>
float best(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float m = 1e30f;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    m = ms < m ? ms : m;
  }
  return m;
}
int main() {
  const long nrows = 50000000 / 512 * 512;
  double* out;
  cudaMalloc(&out, 64);
  Cols cs;
  for (int c = 0; c < NC; c++) {
    double* p;
    cudaMalloc(&p, nrows * 8);
    cudaMemset(p, 0, nrows * 8);
    cs.c[c] = p;
  }
  double* big;
  cudaMalloc(&big, nrows * 8 * NC);
  cudaMemset(big, 0, nrows * 8 * NC);
  const double bytes = (double)nrows * 8 * NC;
  const float t1 = best([&] { k_one<<<148 * 8, 512>>>(reinterpret_cast<const double2*>(big), nrows * NC / 2, out); });
  const float t2 = best([&] { k_chunked<16><<<148 * 4, 256>>>(cs, nrows, out); });
  const float t3 = best([&] { k_chunked<64><<<148 * 4, 256>>>(cs, nrows, out); });
  const float t4 = best([&] { k_cols_stride<<<148 * 8, 256>>>(cs, nrows, out); });
  printf("{\"bytes\": %.0f, \"one_array_gbs\": %.0f, \"chunked512_gbs\": %.0f, \"chunked2048_gbs\": %.0f, \"cols_gridstride_gbs\": %.0f}\n",
         bytes, bytes / t1 / 1e6, bytes / t2 / 1e6, bytes / t3 / 1e6, bytes / t4 / 1e6);
  return 0;
}
