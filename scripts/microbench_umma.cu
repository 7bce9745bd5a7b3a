// microbench_umma.cu -- tcgen05.mma kind::i8 throughput on sm_100a for the shapes the ±1
// tensor-core sketch can use: A = 128 x 32 u8 tile (MN-major SWIZZLE_128B, or K-major
// SWIZZLE_128B), B = 32 x N s8 (MN-major no swizzle / K-major), N in {8, 16, 32, 64, 128, 256}.
// One CTA per SM; one thread issues `iters` x 16 MMAs (16 accumulators, like the sketch's 16
// row tiles) and commits once per 16; reports tensor cycles per MMA from clock64.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7u) << 61;
  return d;
}

template <int N, int AMAJOR, int STRESS>
__global__ void __launch_bounds__(544, 1) k(int iters, unsigned long long* cyc, volatile int* stop) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 16 * 4096 + 8192 + 65536; i += blockDim.x) sm[i] = (unsigned char)(i * 7);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 16) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(AMAJOR == 1) << 15) | (1u << 16) |
                         ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  const int ncols = N < 32 ? 32 : N;   // accumulator stride (columns)
  const int nacc = 512 / ncols < 16 ? 512 / ncols : 16;
  if (STRESS && warp < 16) {
    // 16 warps store 16 B per lane per iteration into a private 64 KB region (conflict-free)
    const uint32_t base = smem_u32(sm + 16 * 4096 + 8192 + 1024) ;
    uint32_t v = threadIdx.x;
    long long cnt = 0;
    while (*stop == 0 && cnt < 2000000) {
#pragma unroll 8
      for (int r = 0; r < 64; ++r) {
        asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" :: "r"(base + (uint32_t)((r * 512 + threadIdx.x * 16) & 0xFFFF)), "r"(v) : "memory");
      }
      cnt += 64;
    }
  }
  if (threadIdx.x == 16 * 32) {
    const uint32_t a0 = smem_u32(sm);
    const uint32_t b0 = smem_u32(sm + 16 * 4096);
    const uint64_t bdesc = make_desc(b0, 128u * (N / 16), 128u, 0u);   // K-group stride, N core-matrix stride
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int bi = it & 3;
      if (it >= 4) {   // at most 4 groups of 16 MMAs in flight; each barrier one phase ahead at most
        asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}"
                     :: "r"(smem_u32(&bar[bi])), "r"((uint32_t)(((it >> 2) - 1) & 1)) : "memory");
      }
      for (int t = 0; t < 16; ++t) {
        if constexpr (AMAJOR == 2) {
          const uint32_t d = tbase + (uint32_t)(t * 16);
          const uint32_t at = tbase + 256u + (uint32_t)(t * 8);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
                       :: "r"(d), "r"(at), "l"(bdesc), "r"(idesc), "r"(it > 0 ? 1u : 0u));
        } else {
        const uint64_t adesc = AMAJOR ? make_desc(a0 + t * 4096, 4096u, 1024u, 2u)
                                      : make_desc(a0 + t * 4096, 16u, 1024u, 2u);
        const uint32_t d = tbase + (uint32_t)((t % nacc) * ncols);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                     :: "r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(it > 0 ? 1u : 0u));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   :: "r"(smem_u32(&bar[bi])) : "memory");
    }
    for (int it = iters - 4; it < iters; ++it) {
      if (it < 0) continue;
      asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}"
                   :: "r"(smem_u32(&bar[it & 3])), "r"((uint32_t)((it >> 2) & 1)) : "memory");
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = (unsigned long long)(t1 - t0);
    *stop = 1;
  }
  __syncthreads();
  if (warp == 16) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tbase));
}

template <int N, int AM, int ST>
void run(const char* name) {
  unsigned long long* d;
  int* stop;
  cudaMalloc(&d, 8);
  cudaMalloc(&stop, 4);
  const int smem = 16 * 4096 + 8192 + 1024 + 65536;
  cudaFuncSetAttribute(k<N, AM, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 400;
  cudaMemset(stop, 0, 4);
  k<N, AM, ST><<<148, 544, smem>>>(iters, d, stop);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaMemset(stop, 0, 4);
  cudaEventRecord(a);
  k<N, AM, ST><<<148, 544, smem>>>(iters, d, stop);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned long long c = 0; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / (iters * 16.0);
  printf("%-28s N=%3d: %.1f cycles/MMA, %.1f A-bytes/clk, %.3f ms total %s\n", name, N, per, 4096.0 / per, ms,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<16, 2, 0>("A TMEM K-major (TS)");
  run<16, 2, 1>("A TMEM K-major (TS) + STS");
  run<16, 1, 0>("A MN-major SW128");
  run<16, 1, 1>("A MN-major SW128 + STS stress");
  run<64, 1, 0>("A MN-major SW128");
  run<64, 1, 1>("A MN-major SW128 + STS stress");
  run<256, 1, 1>("A MN-major SW128 + STS stress");
  return 0;
}
