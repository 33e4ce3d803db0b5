// Latency of the Jacobi rotation-parameter chain: branchy (eigen.hpp) vs branch-free, 1 vs 32 lanes.
#include <cstdio>
#include <cmath>
__device__ __forceinline__ void pf(double apq, double dp, double dq, double tresh, bool late, double& s, double& tau, double& h, bool& rot) {
  const double g = 100.0 * fabs(apq);
  const bool zero = late && (fabs(dp) + g == fabs(dp)) && (fabs(dq) + g == fabs(dq));
  rot = !zero && (fabs(apq) > tresh);
  const double hh = dq - dp;
  const double t1 = apq / hh;
  const double theta = 0.5 * hh / apq;
  double t2 = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta));
  t2 = theta < 0.0 ? -t2 : t2;
  const double tt = (fabs(hh) + g == fabs(hh)) ? t1 : t2;
  const double c = 1.0 / sqrt(1.0 + tt * tt);
  const double sv = tt * c; const double tv = sv / (1.0 + c); const double hv = tt * apq;
  s = rot ? sv : 0.0; tau = rot ? tv : 0.0; h = rot ? hv : 0.0;
}
__global__ void k(double* out, long long* cyc, double seed, int iters) {
  double apq = seed + threadIdx.x * 1e-9, dp = 3.0, dq = 1.0, s = 0, tau = 0, h = 0, y = 0.25; bool rot;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    apq = apq - s * (y + apq * tau);
    pf(apq, dp, dq, 1e-300, false, s, tau, h, rot);
    dp -= h; apq = apq + 0.3;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = apq + s + dp;
}
int main() {
  double* o; long long* c; cudaMallocManaged(&o, 64 * 8); cudaMallocManaged(&c, 64);
  for (int th : {1, 32}) {
    k<<<1, th>>>(o, c, 0.7, 4096); cudaDeviceSynchronize();
    k<<<1, th>>>(o, c, 0.7, 4096); cudaDeviceSynchronize();
    printf("branch-free params chain, %d lanes: %.1f cycles/iter\n", th, double(c[0]) / 4096);
  }
  return 0;
}
