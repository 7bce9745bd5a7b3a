// mxf4_mn_probe.cu -- does tcgen05.mma kind::mxf4 accept an MN-major (transposed) A operand on sm_100a?
// A = 128 x 64 random ±1 e2m1 (nibble 0x2 / 0xA), B = 8 x 64 random ±1 (K-major, no swizzle),
// D = A B^T (f32, TMEM).  A is laid out K-major (reference) or MN-major under four readings of the
// descriptor's LBO / SBO; each result is compared with the host product.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__global__ void __launch_bounds__(128, 1) k(const uint8_t* a_img, const uint8_t* b_img, uint32_t lbo, uint32_t sbo,
                                            int a_mn, float* out) {
  __shared__ __align__(1024) uint8_t sa[4096];
  __shared__ __align__(1024) uint8_t sb[256];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 4096; i += 128) sa[i] = a_img[i];
  for (int i = threadIdx.x; i < 256; i += 128) sb[i] = b_img[i];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const uint32_t tb = tbase;
  {
    const uint32_t taddr = tb + ((uint32_t)(32 * warp) << 16) + 448u;
    const uint32_t v = 0x7F7F7F7Fu;
    for (int c = 0; c < 64; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" :: "r"(taddr + c), "r"(v) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((8u >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
    const uint64_t adesc = a_mn ? make_desc(smem_u32(sa), lbo, sbo) : make_desc(smem_u32(sa), 128u, 256u);
    const uint64_t bdesc = make_desc(smem_u32(sb), 128u, 256u);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}"
                 :: "r"(tb), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(0u), "r"(tb + 448u), "r"(tb + 480u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred P1;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" :: "r"(smem_u32(&bar)) : "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(tb + ((uint32_t)(32 * warp) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int n = 0; n < 8; ++n) out[threadIdx.x * 8 + n] = __uint_as_float(v[n]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tb));
}

static void put_nib(std::vector<uint8_t>& img, size_t elem_byte_off, int nib, uint8_t v) {
  uint8_t& b = img[elem_byte_off];
  b = nib ? (uint8_t)((b & 0x0F) | (v << 4)) : (uint8_t)((b & 0xF0) | v);
}

int main() {
  srand(7);
  int S[128][64], B[8][64];
  for (int m = 0; m < 128; ++m) for (int q = 0; q < 64; ++q) S[m][q] = (rand() & 1) ? 1 : -1;
  for (int n = 0; n < 8; ++n) for (int q = 0; q < 64; ++q) B[n][q] = (rand() & 1) ? 1 : -1;
  auto nib = [](int s) -> uint8_t { return s > 0 ? 0x2 : 0xA; };
  // K-major no swizzle: core matrix 8 rows x 16 B (32 K elements), LBO = 128 (K), SBO = 256 (8-row groups);
  // element (r, q): group r/8 at 256 (r/8), K chunk q/32 at 128 (q/32), row r%8 at 16 (r%8), byte (q%32)/2, nibble q%2
  auto kmaj = [&](int rows, int (*M)[64]) {
    std::vector<uint8_t> img(rows * 32, 0);
    for (int r = 0; r < rows; ++r) for (int q = 0; q < 64; ++q)
      put_nib(img, (r / 8) * 256 + (q / 32) * 128 + (r % 8) * 16 + (q % 32) / 2, q % 2, nib(M[r][q]));
    return img;
  };
  std::vector<uint8_t> aK = kmaj(128, S), bK = kmaj(8, B);
  double ref[128][8];
  for (int m = 0; m < 128; ++m) for (int n = 0; n < 8; ++n) { int s = 0; for (int q = 0; q < 64; ++q) s += S[m][q] * B[n][q]; ref[m][n] = s; }
  uint8_t *da, *db; float* dout;
  cudaMalloc(&da, 4096); cudaMalloc(&db, 256); cudaMalloc(&dout, 128 * 8 * 4);
  cudaMemcpy(db, bK.data(), 256, cudaMemcpyHostToDevice);
  auto run = [&](const char* name, const std::vector<uint8_t>& a, uint32_t lbo, uint32_t sbo, int mn) {
    cudaMemcpy(da, a.data(), 4096, cudaMemcpyHostToDevice);
    cudaMemset(dout, 0, 128 * 8 * 4);
    k<<<1, 128>>>(da, db, lbo, sbo, mn, dout);
    cudaError_t e = cudaDeviceSynchronize();
    float h[128 * 8];
    cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 128; ++m) for (int n = 0; n < 8; ++n) bad += h[m * 8 + n] != (float)ref[m][n];
    printf("%-40s %s mismatches %d / 1024  (D[0][0..3] = %.0f %.0f %.0f %.0f, ref %.0f %.0f %.0f %.0f)\n", name,
           e == cudaSuccess ? "ok " : cudaGetErrorString(e), bad, h[0], h[1], h[2], h[3], ref[0][0], ref[0][1], ref[0][2], ref[0][3]);
    return e == cudaSuccess;
  };
  if (!run("A K-major (reference)", aK, 0, 0, 0)) return 1;
  // MN-major: core matrix = 8 K rows x 16 B (32 M elements); element (m, q): core (m/32, q/8), inside:
  // K row q%8 at 16 (q%8), byte (m%32)/2, nibble m%2.  Two placements of the cores x two descriptor readings.
  for (int place = 0; place < 2; ++place) {
    std::vector<uint8_t> aM(4096, 0);
    for (int m = 0; m < 128; ++m) for (int q = 0; q < 64; ++q) {
      const size_t core = place == 0 ? (size_t)(q / 8) * 512 + (m / 32) * 128 : (size_t)(m / 32) * 1024 + (q / 8) * 128;
      put_nib(aM, core + (q % 8) * 16 + (m % 32) / 2, m % 2, nib(S[m][q]));
    }
    const uint32_t mn_stride = place == 0 ? 128 : 1024, k_stride = place == 0 ? 512 : 128;
    char nm[80];
    snprintf(nm, sizeof nm, "A MN-major place %d LBO=MN SBO=K", place);
    if (!run(nm, aM, mn_stride, k_stride, 1)) return 1;
    snprintf(nm, sizeof nm, "A MN-major place %d LBO=K SBO=MN", place);
    if (!run(nm, aM, k_stride, mn_stride, 1)) return 1;
  }
  return 0;
}
