// rsqrt_check.cu -- maximum relative error of rsqrt.approx.ftz.f64 on [2^-60, 128) (one B200):
// decides how many refinement steps bm_sqrt (philox.cuh) needs.
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k(const double* x, double* y, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[i])); y[i] = r; }
}

int main() {
  const int n = 1 << 22;
  double *hx = new double[n], *hy = new double[n], *dx, *dy;
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const double u = (double)(s >> 11) * 0x1p-53;            // [0, 1)
    hx[i] = std::ldexp(1.0 + u, (int)(s % 67) - 60);          // [2^-60, 2^7)
  }
  cudaMalloc(&dx, n * 8); cudaMalloc(&dy, n * 8);
  cudaMemcpy(dx, hx, n * 8, cudaMemcpyHostToDevice);
  k<<<(n + 255) / 256, 256>>>(dx, dy, n);
  cudaMemcpy(hy, dy, n * 8, cudaMemcpyDeviceToHost);
  double worst = 0;
  for (int i = 0; i < n; ++i) {
    const long double ref = 1.0L / sqrtl((long double)hx[i]);
    const double e = (double)fabsl(((long double)hy[i] - ref) / ref);
    if (e > worst) worst = e;
  }
  printf("rsqrt.approx.ftz.f64 max rel error %.3g = 2^%.1f over %d samples\n", worst, std::log2(worst), n);
  return 0;
}
