// microbench_sel.cu -- which pipe takes SEL vs FSEL on sm_100a, measured as the throughput
// of the ±1 sign-application loop of sk_rad_kernel<double> (one select + one DFMA per element).
// Variants: 0 = SEL (selp.b32), 1 = FSEL (selp.f32), 2 = alternate SEL/FSEL, 3 = DFMA only.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__device__ __forceinline__ int pick(uint32_t w, int b) {
  int h;
  if (V == 0 || (V == 2 && (b & 1) == 0)) {
    asm("{.reg .pred p; .reg .b32 t; and.b32 t, %1, %2; setp.ne.u32 p, t, 0; selp.b32 %0, -1074790400, 1072693248, p;}"
        : "=r"(h) : "r"(w), "r"(1u << b));
  } else {
    float f;
    asm("{.reg .pred p; .reg .b32 t; and.b32 t, %1, %2; setp.ne.u32 p, t, 0; selp.f32 %0, 0fBFF00000, 0f3FF00000, p;}"
        : "=f"(f) : "r"(w), "r"(1u << b));
    h = __float_as_int(f);
  }
  return h;
}

template <int V>
__global__ void k(const uint32_t* __restrict__ W, double a, double* out, int n) {
  double acc[32];
#pragma unroll
  for (int b = 0; b < 32; ++b) acc[b] = 0;
  uint32_t w = W[threadIdx.x];
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int b = 0; b < 32; ++b) {
      if constexpr (V == 3) acc[b] = fma(a, a, acc[b]);
      else acc[b] = fma(__hiloint2double(pick<V>(w, b), 0), a, acc[b]);
    }
    w = w * 1664525u + 1013904223u;
  }
  double s = 0;
#pragma unroll
  for (int b = 0; b < 32; ++b) s += acc[b];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  uint32_t* W; double* out;
  cudaMalloc(&W, 4096); cudaMalloc(&out, 148 * 8 * 256 * 8);
  cudaMemset(W, 0x5a, 4096);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = 148 * 4, threads = 512, n = 2000;
  const double elems = (double)blocks * threads * 32 * n;
  auto run = [&](auto kern, const char* name) {
    kern<<<blocks, threads>>>(W, 1.0000001, out, n);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(W, 1.0000001, out, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%s: %.3f elem/clk/SM (%.3g elem/s)\n", name, elems * 5 / (ms * 1e-3) / 148 / 1.965e9, elems * 5 / (ms * 1e-3));
  };
  run(k<0>, "SEL+DFMA");
  run(k<1>, "FSEL+DFMA");
  run(k<2>, "SEL/FSEL alternating+DFMA");
  run(k<3>, "DFMA only");
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
