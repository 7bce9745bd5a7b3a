// microbench_producer.cu -- throughput of the fp4 tensor-core path's S producer loop alone
// (Philox4x32-10 -> 32x32 warp bit transpose -> e2m1 nibble expansion -> STS.128), with no
// barriers.  Reports (row, nonzero) entries per clock per SM for
//   MODE 2: Philox + rotated 5-stage transpose + nibbles + STS.128 (the f4 producer);
//   3: Philox + 3-stage partial exchange + nibbles + 16 STS.32 (SK_F4_PART); 4: Philox + nibbles +
//   STS.128 without the transpose; 6: mode 2 with a CTA-wide bar.sync after every U blocks
//   (all producer warps in lock step, as a stage barrier would force)
// with U Philox blocks per lane in flight and NW warps per SM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2310_15419_b200/csrc/philox.cuh"

__device__ __forceinline__ uint32_t nib(uint32_t t) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(t), "r"(0x88888888u), "r"(0x22222222u));
  return r;
}

template <int MODE, int U, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k(int iters, sk::PhiloxKeys K, uint32_t* out) {
  __shared__ __align__(16) uint32_t buf[NW][4 * 32 * 4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t acc = 0;
  const uint32_t m[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
  for (int it = 0; it < iters; it += U) {
    uint32_t x[4 * U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint4 xb = sk::s_block((uint32_t)warp, (uint64_t)((it + u) * 32 + lane), K);
      x[4 * u] = xb.x; x[4 * u + 1] = xb.y; x[4 * u + 2] = xb.z; x[4 * u + 3] = xb.w;
    }
    if (MODE == 3) {
      const uint32_t m0[3] = {0x0F0F0F0Fu, 0x00FF00FFu, 0x0000FFFFu};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const bool lower = (lane & (1 << a)) == 0;
        const uint32_t keep = lower ? m0[a] : ~m0[a];
        const uint32_t r = lower ? (4u << a) : 32u - (4u << a);
        uint32_t y[4 * U];
#pragma unroll
        for (int q = 0; q < 4 * U; ++q) y[q] = __shfl_xor_sync(0xFFFFFFFFu, x[q], 1 << a);
#pragma unroll
        for (int q = 0; q < 4 * U; ++q) {
          const uint32_t yr = __funnelshift_l(y[q], y[q], r);
          asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(x[q]) : "r"(x[q]), "r"(yr), "r"(keep));
        }
      }
      const uint32_t base = (uint32_t)__cvta_generic_to_shared(&buf[warp][0]) + (uint32_t)((lane & 7) * 16 + (lane >> 3) * 4);
#pragma unroll
      for (int q = 0; q < 4 * U; ++q)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          asm volatile("st.shared.b32 [%0], %1;" :: "r"(base + (uint32_t)((((q & 3) * 4 + c) & 15) * 128)), "r"(nib(x[q] << (3 - c))) : "memory");
    } else if (MODE == 1 || MODE == 2 || MODE == 6) {
#pragma unroll
      for (int q = 0; q < 4 * U; ++q) x[q] = __funnelshift_l(x[q], x[q], lane);
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        const uint32_t rm = __funnelshift_l(m[s], m[s], lane);
        const uint32_t keep = (lane & (16 >> s)) ? ~rm : rm;
        uint32_t y[4 * U];
#pragma unroll
        for (int q = 0; q < 4 * U; ++q) y[q] = __shfl_xor_sync(0xFFFFFFFFu, x[q], 16 >> s);
#pragma unroll
        for (int q = 0; q < 4 * U; ++q) asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(x[q]) : "r"(x[q]), "r"(y[q]), "r"(keep));
      }
#pragma unroll
      for (int q = 0; q < 4 * U; ++q) x[q] = __funnelshift_r(x[q], x[q], lane);
    }
    if (MODE == 2 || MODE == 4 || MODE == 6) {
#pragma unroll
      for (int q = 0; q < 4 * U; ++q) {
        const uint32_t w0 = nib(x[q] << 3), w1 = nib(x[q] << 2), w2 = nib(x[q] << 1), w3 = nib(x[q]);
        const uint32_t a = (uint32_t)__cvta_generic_to_shared(&buf[warp][((q & 3) * 32 + lane) * 4]);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(a), "r"(w0), "r"(w1), "r"(w2), "r"(w3) : "memory");
      }
    } else if (MODE != 3) {
#pragma unroll
      for (int q = 0; q < 4 * U; ++q) acc ^= x[q];
    }
    if (MODE == 6) asm volatile("bar.sync 1, %0;" :: "r"(NW * 32) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NW * 512; i += blockDim.x) acc ^= (&buf[0][0])[i];
  if (acc == 0x12345678u + (uint32_t)iters) out[0] = acc;
}

template <int MODE, int U, int NW>
void run() {
  uint32_t* out;
  cudaMalloc(&out, 4);
  const int iters = 4096;
  k<MODE, U, NW><<<148, NW * 32>>>(iters, sk::make_keys(3), out);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE, U, NW><<<148, NW * 32>>>(iters, sk::make_keys(3), out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  if (cudaGetLastError() != cudaSuccess) { printf("mode %d U %d NW %d: launch error\n", MODE, U, NW); return; }
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double entries = 148.0 * NW * 32 * 128 * iters;   // each lane: one block = 128 entries / iter
  printf("mode %d U %d %2d warps/SM: %6.1f entries/clk/SM (%.3f ms)\n", MODE, U, NW, entries / (ms * 1e-3) / 148 / 1.9e9, ms);
  cudaFree(out);
}

template <int MODE, int U>
void runs() { run<MODE, U, 4>(); run<MODE, U, 8>(); run<MODE, U, 12>(); run<MODE, U, 16>(); }

int main() {
  runs<4, 4>(); runs<2, 4>(); runs<3, 4>(); runs<6, 4>(); runs<6, 2>();
  return 0;
}
