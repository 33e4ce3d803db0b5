// Microbenchmark: dependent-chain latency of FP64 ops on sm_100a (one thread).
#include <cstdio>
#include <cmath>
__global__ void k(double* out, long long* cyc, double seed, int iters) {
  double x = seed, y = seed * 0.5;
  long long t0, t1;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x + y;
  t1 = clock64(); cyc[0] = t1 - t0; out[0] = x;
  // DMUL chain
  x = seed; t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x * 1.0000001;
  t1 = clock64(); cyc[1] = t1 - t0; out[1] = x;
  // DIV chain
  x = seed; t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64(); cyc[2] = t1 - t0; out[2] = x;
  // SQRT chain
  x = seed + 2.0; t0 = clock64();
  for (int i = 0; i < iters; ++i) x = sqrt(x + 1.0);
  t1 = clock64(); cyc[3] = t1 - t0; out[3] = x;
  // Jacobi params chain (eigen.hpp:66-80) with the next-pivot update
  double apq = seed, dp = 3.0, dq = 1.0, s = 0, tau = 0, yv = 0.25;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    apq = apq - s * (yv + apq * tau);
    const double g = 100.0 * fabs(apq);
    double hh = dq - dp, tt;
    if (fabs(hh) + g == fabs(hh)) tt = apq / hh;
    else {
      const double theta = 0.5 * hh / apq;
      tt = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta));
      if (theta < 0.0) tt = -tt;
    }
    const double c = 1.0 / sqrt(1.0 + tt * tt);
    s = tt * c;
    tau = s / (1.0 + c);
    const double h = tt * apq;
    dp -= h;
    apq = apq + 0.3;  // keep it alive
  }
  t1 = clock64(); cyc[4] = t1 - t0; out[4] = apq + dp + s + tau;
}
int main() {
  double* o; long long* c; cudaMallocManaged(&o, 64); cudaMallocManaged(&c, 64);
  const int it = 4096;
  k<<<1,1>>>(o, c, 0.7, it); cudaDeviceSynchronize();
  k<<<1,1>>>(o, c, 0.7, it); cudaDeviceSynchronize();
  const char* nm[5] = {"dadd", "dmul", "div", "sqrt", "jacobi-params"};
  for (int i = 0; i < 5; ++i) printf("%-14s %.1f cycles/iter\n", nm[i], double(c[i]) / it);
  return 0;
}
