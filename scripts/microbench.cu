// microbench.cu -- measures the B200 pipe rates the roofline of DESIGN.md uses:
//   (1) FP64 DADD and DFMA throughput (lane-ops / s / GPU),
//   (2) FP32 FADD throughput,
//   (3) Philox4x32-10 blocks / s (INT pipe), XOR-folded so nothing is stored per call.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2310_15419_b200/csrc/philox.cuh"

template <typename T, int OP>
__global__ void pipe_kernel(T* out, int iters, T a) {
  T acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = T(threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if constexpr (OP == 0) acc[i] = acc[i] + a;       // add
      else acc[i] = acc[i] * a + a;                      // fma
    }
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == T(-1234.5)) out[threadIdx.x] = s;
}

__global__ void philox_kernel(uint32_t* out, int iters, sk::PhiloxKeys K) {
  uint32_t f = 0;
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    uint4 x = sk::s_block((uint32_t)it, (uint64_t)j, K);
    f ^= x.x ^ x.y ^ x.z ^ x.w;
  }
  if (f == 0x12345678u) out[0] = f;
}

// Philox with the products as mul.hi + mul.lo (IMAD.HI + IMAD) instead of mul.wide (IMAD.WIDE)
__device__ __forceinline__ uint4 philox_hilo(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                            const sk::PhiloxKeys& K) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t h0 = __umulhi(sk::kPhiloxM0, c0), l0 = sk::kPhiloxM0 * c0;
    const uint32_t h1 = __umulhi(sk::kPhiloxM1, c2), l1 = sk::kPhiloxM1 * c2;
    const uint32_t n0 = h1 ^ c1 ^ K.k0[r];
    const uint32_t n2 = h0 ^ c3 ^ K.k1[r];
    c1 = l1; c3 = l0; c0 = n0; c2 = n2;
  }
  return make_uint4(c0, c1, c2, c3);
}

template <int MODE>
__global__ void philox_kernel2(uint32_t* out, int iters, sk::PhiloxKeys K) {
  uint32_t f = 0;
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; it += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint4 x = MODE == 0 ? sk::s_block((uint32_t)(it + u), (uint64_t)j, K)
                                : philox_hilo((uint32_t)(it + u), 0u, j, 0u, K);
      f ^= x.x ^ x.y ^ x.z ^ x.w;
    }
  }
  if (f == 0x12345678u) out[0] = f;
}

// IMAD.WIDE.U32 vs (IMAD.HI.U32 + IMAD.LO) for the 32x32->64 products of a Philox round.
template <int MODE>
__global__ void mul_kernel(uint32_t* out, int iters, uint32_t m) {
  uint32_t a[8], f = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7919u + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (MODE == 0) {
        const uint64_t p = (uint64_t)m * a[i];
        a[i] = (uint32_t)(p >> 32) ^ (uint32_t)p;
      } else {
        uint32_t hi, lo;
        asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(m), "r"(a[i]));
        asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(m), "r"(a[i]));
        a[i] = hi ^ lo;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) f ^= a[i];
  if (f == 0x12345678u) out[0] = f;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d", p.name, p.multiProcessorCount, clk);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  void* buf; cudaMalloc(&buf, 1 << 20);
  const int blocks = p.multiProcessorCount * 8, threads = 256;
  auto timeit = [&](auto launch, double ops, const char* name) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf(", \"%s\": %.4g", name, ops * 5 / (ms * 1e-3));
  };
  const int iters = 20000;
  const double lanes = (double)blocks * threads * 16 * iters;
  timeit([&] { pipe_kernel<double, 0><<<blocks, threads>>>((double*)buf, iters, 1.0000001); }, lanes, "dadd_per_s");
  timeit([&] { pipe_kernel<double, 1><<<blocks, threads>>>((double*)buf, iters, 0.9999999); }, lanes, "dfma_per_s");
  timeit([&] { pipe_kernel<float, 0><<<blocks, threads>>>((float*)buf, iters, 1.0001f); }, lanes, "fadd_per_s");
  const int piters = 4000;
  timeit([&] { philox_kernel<<<blocks, threads>>>((uint32_t*)buf, piters, sk::make_keys(7)); },
         (double)blocks * threads * piters, "philox_blocks_per_s");
  timeit([&] { philox_kernel2<0><<<blocks, threads>>>((uint32_t*)buf, piters, sk::make_keys(7)); },
         (double)blocks * threads * piters, "philox_wide_x4_blocks_per_s");
  timeit([&] { philox_kernel2<1><<<blocks, threads>>>((uint32_t*)buf, piters, sk::make_keys(7)); },
         (double)blocks * threads * piters, "philox_hilo_x4_blocks_per_s");
  timeit([&] { mul_kernel<0><<<blocks, threads>>>((uint32_t*)buf, 20000, 0xD2511F53u); },
         (double)blocks * threads * 8 * 20000, "mulwide_per_s");
  timeit([&] { mul_kernel<1><<<blocks, threads>>>((uint32_t*)buf, 20000, 0xD2511F53u); },
         (double)blocks * threads * 8 * 20000, "mulhi_lo_per_s");
  printf("}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
