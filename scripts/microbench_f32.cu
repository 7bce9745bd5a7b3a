// microbench_f32.cu -- FP32 issue / pipe rates on sm_100a for the ±1 x fp32 kernel (config c4):
//   mode 0: FADD            (1 lane-op per instruction)
//   mode 1: FADD2 (add.rn.f32x2: 2 lane-ops per instruction)
//   mode 2: FFMA2 (fma.rn.f32x2)
//   mode 3: predicated FADD from sign bits (the current c4 inner loop: R2P + @P FADD)
//   mode 4: FADD2 on sign-masked pairs: LOP3 (a & mask) x 2 + FADD2 per 2 entries
//   mode 5: FADD2 + independent LOP3 (can the ALU pipe issue while the FMA pipe runs FADD2?)
// Prints lane-ops (entries) per second per GPU and per clock per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o microbench_f32 microbench_f32.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void upk(unsigned long long r, float& x, float& y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(r));
}

template <int MODE>
__global__ void k(float* out, int iters, float a, uint32_t seed) {
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = (float)(threadIdx.x + i);
  unsigned long long acc2[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc2[i] = pk(acc[2 * i], acc[2 * i + 1]);
  uint32_t w = seed ^ threadIdx.x, z = 0;
  const unsigned long long a2 = pk(a, a * 0.5f);
  for (int it = 0; it < iters; ++it) {
    w = w * 1664525u + 1013904223u;     // new sign word (1 IMAD)
    if constexpr (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] += a;
    } else if constexpr (MODE == 1) {
#pragma unroll
      for (int i = 0; i < 16; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc2[i]) : "l"(a2));
    } else if constexpr (MODE == 2) {
#pragma unroll
      for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc2[i]) : "l"(a2));
    } else if constexpr (MODE == 3) {
#pragma unroll
      for (int b = 0; b < 32; ++b)
        if ((w >> b) & 1u) acc[b] += a;
    } else if constexpr (MODE == 4) {
      const uint32_t ab = __float_as_uint(a);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t m0 = (uint32_t)((int32_t)(w << (31 - 2 * i)) >> 31);
        const uint32_t m1 = (uint32_t)((int32_t)(w << (30 - 2 * i)) >> 31);
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc2[i]) : "l"(pk(__uint_as_float(ab & m0), __uint_as_float(ab & m1))));
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc2[i]) : "l"(a2));
        z = (z ^ (w >> i)) & 0x5555u;   // one LOP3-class ALU op per FADD2
      }
    }
  }
  float s = (float)z;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += acc[i];
#pragma unroll
  for (int i = 0; i < 16; ++i) { float x, y; upk(acc2[i], x, y); s += x + y; }
  if (s == -1234.5f) out[threadIdx.x] = s;
}

template <int MODE>
double run(int blocks, int threads, int iters, float* out, double clk_ghz, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<MODE><<<blocks, threads>>>(out, 10, 1.0f, 1u);
  cudaEventRecord(e0);
  k<MODE><<<blocks, threads>>>(out, iters, 1.0f, 1u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double entries = (double)blocks * threads * iters * 32.0;
  const double rate = entries / (ms * 1e-3);
  printf("mode %d: %.3f ms, %.3e entries/s, %.1f entries/clk/SM\n", MODE, ms, rate, rate / (sms * clk_ghz * 1e9));
  return rate;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double ghz = clk_khz / 1e6;
  printf("%s, %d SMs, %.3f GHz\n", p.name, p.multiProcessorCount, ghz);
  float* out;
  cudaMalloc(&out, 4096 * sizeof(float));
  const int blocks = p.multiProcessorCount * 4, threads = 512, iters = 20000;
  run<0>(blocks, threads, iters, out, ghz, p.multiProcessorCount);
  run<1>(blocks, threads, iters, out, ghz, p.multiProcessorCount);
  run<2>(blocks, threads, iters, out, ghz, p.multiProcessorCount);
  run<3>(blocks, threads, iters, out, ghz, p.multiProcessorCount);
  run<4>(blocks, threads, iters, out, ghz, p.multiProcessorCount);
  run<5>(blocks, threads, iters, out, ghz, p.multiProcessorCount);
  return 0;
}
