// microbench_producer.cu -- throughput of the fp4 tensor-core path's S producer loop alone
// (Philox4x32-10 -> 32x32 warp bit transpose -> e2m1 nibble expansion -> 4 x STS.128), with no
// barriers, for 4..16 warps per SM.  Reports (row, nonzero) entries per clock per SM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2310_15419_b200/csrc/philox.cuh"

__device__ __forceinline__ uint32_t stage_op(uint32_t x, uint32_t y, uint32_t sh, uint32_t keep) {
  uint32_t t, r;
  asm("shf.l.wrap.b32 %0, %1, %1, %2;" : "=r"(t) : "r"(y), "r"(sh));
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(x), "r"(t), "r"(keep));
  return r;
}
__device__ __forceinline__ uint32_t nib(uint32_t t) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(t), "r"(0x88888888u), "r"(0x22222222u));
  return r;
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k(int iters, sk::PhiloxKeys K, uint32_t* out) {
  __shared__ __align__(16) uint32_t buf[NW][4 * 32 * 4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const uint4 xb = sk::s_block((uint32_t)warp, (uint64_t)(it * 32 + lane), K);
    uint32_t x[4] = {xb.x, xb.y, xb.z, xb.w};
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
      const uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu : j == 2 ? 0x33333333u : 0x55555555u;
      const bool hi = (lane & j) != 0;
      const uint32_t keep = hi ? ~m : m, sh = hi ? (32 - j) : j;
      uint32_t y[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) y[q] = __shfl_xor_sync(0xFFFFFFFFu, x[q], j);
#pragma unroll
      for (int q = 0; q < 4; ++q) x[q] = stage_op(x[q], y[q], sh, keep);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t w0 = nib(x[q] << 3), w1 = nib(x[q] << 2), w2 = nib(x[q] << 1), w3 = nib(x[q]);
      const uint32_t a = (uint32_t)__cvta_generic_to_shared(&buf[warp][(q * 32 + lane) * 4]);
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(a), "r"(w0), "r"(w1), "r"(w2), "r"(w3) : "memory");
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NW * 512; i += blockDim.x) acc ^= (&buf[0][0])[i];
  if (acc == 0x12345678u) out[0] = acc;
}

template <int NW>
void run() {
  uint32_t* out;
  cudaMalloc(&out, 4);
  const int iters = 4000;
  k<NW><<<148, NW * 32>>>(iters, sk::make_keys(3), out);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<NW><<<148, NW * 32>>>(iters, sk::make_keys(3), out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double entries = 148.0 * NW * 32 * 128 * iters;   // each lane: one block = 128 entries / iter
  printf("%2d warps/SM: %.1f entries/clk/SM (%.3f ms)\n", NW, entries / (ms * 1e-3) / 148 / 1.965e9, ms);
  cudaFree(out);
}

int main() {
  run<4>(); run<8>(); run<12>(); run<16>(); run<20>();
  return 0;
}
