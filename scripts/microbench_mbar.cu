// microbench_mbar.cu -- mbarrier hand-off latency on sm_100a: two warps ping-pong through two
// mbarriers (A arrives on b0, B waits b0 then arrives on b1, A waits b1), N round trips.
// MODE 0: try_wait loops, 1: test_wait spin, 2: try_wait with suspend-time hint 0x10.
// Extra "busy" warps run an ALU loop alongside (0 or 12 of them).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  if constexpr (MODE == 0) {
    asm volatile("{\n\t.reg .pred P;\n\tW%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W%=;\n\t}"
                 :: "r"(su(b)), "r"(par) : "memory");
  } else if constexpr (MODE == 1) {
    asm volatile("{\n\t.reg .pred P;\n\tW%=: mbarrier.test_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W%=;\n\t}"
                 :: "r"(su(b)), "r"(par) : "memory");
  } else {
    asm volatile("{\n\t.reg .pred P;\n\tW%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t@!P bra W%=;\n\t}"
                 :: "r"(su(b)), "r"(par), "r"(0x10) : "memory");
  }
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su(b)) : "memory");
}

template <int MODE>
__global__ void k(int iters, int busy, unsigned long long* out, unsigned* sink) {
  __shared__ uint64_t b[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&b[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&b[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      __syncwarp();
      if (lane == 0) arrive(&b[0]);
      wait<MODE>(&b[1], i & 1);
    }
    long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  } else if (warp == 1) {
    for (int i = 0; i < iters; ++i) {
      wait<MODE>(&b[0], i & 1);
      __syncwarp();
      if (lane == 0) arrive(&b[1]);
    }
  } else if (warp - 2 < busy) {
    unsigned x = threadIdx.x;
    for (int i = 0; i < iters * 64; ++i) x = x * 1664525u + 1013904223u ^ (x >> 7);
    sink[blockIdx.x * blockDim.x + threadIdx.x] = x;
  }
}

template <int MODE>
void run(int busy) {
  unsigned long long* d;
  unsigned* sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 148 * 512 * 4);
  const int iters = 20000;
  k<MODE><<<148, 32 * (2 + busy), 0>>>(iters, busy, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("mode %d busy warps %2d: %.1f clk per round trip (2 hand-offs) %s\n", MODE, busy, (double)c / iters,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int busy : {0, 12}) {
    run<0>(busy);
    run<1>(busy);
    run<2>(busy);
  }
  return 0;
}
