// tm_check.cu -- probe cuTensorMapEncodeTiled for the 1-D maps sketch_f4n.cu uses
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
int main() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  printf("entry point: %s q=%d p=%p\n", cudaGetErrorString(e), (int)q, p);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  void* buf; cudaMalloc(&buf, 1 << 20);
  CUtensorMap m;
  cuuint64_t dim[1] = {50000}; cuuint64_t str[1] = {4}; cuuint32_t box[1] = {256}; cuuint32_t es[1] = {1};
  for (int l2 = 0; l2 < 4; ++l2) {
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_INT32, 1, buf, dim, nullptr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = enc(&m, CU_TENSOR_MAP_DATA_TYPE_INT32, 1, buf, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("l2 %d: null strides -> %d, strides -> %d\n", l2, (int)r, (int)r2);
  }
  return 0;
}
