// FP64 throughput per SM: W warps, each lane runs 8 independent DADD/DMUL chains.
#include <cstdio>
__global__ void k(double* out, long long* cyc, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double m = 1.0000001, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = a[i] * m + c;  // DMUL + DADD (no fma)
  }
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMallocManaged(&o, 1024 * 8); cudaMallocManaged(&c, 64);
  const int it = 2048;
  for (int w : {1, 2, 4, 8, 16}) {
    k<<<1, 32 * w>>>(o, c, it); cudaDeviceSynchronize();
    k<<<1, 32 * w>>>(o, c, it); cudaDeviceSynchronize();
    const double ops = 2.0 * 8 * it * 32 * w;  // thread FP64 ops
    printf("%2d warps: %.1f cycles/iter, %.2f FP64 thread-ops/clk/SM\n", w, double(c[0]) / it, ops / c[0]);
  }
  return 0;
}
