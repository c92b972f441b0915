// TMA box-shape probe: ./tma_probe BOXW BOXH GW GH X Y  (8-byte elements)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

__global__ void k(const CUtensorMap* tm, int x, int y, unsigned bytes, unsigned long long* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long mbar;
  unsigned mb = static_cast<unsigned>(__cvta_generic_to_shared(&mbar));
  unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(dst), "l"(reinterpret_cast<unsigned long long>(tm)), "r"(x), "r"(y), "r"(mb) : "memory");
  }
  __syncthreads();
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" ::"r"(mb) : "memory");
  if (threadIdx.x == 0) out[0] = reinterpret_cast<unsigned long long*>(sm)[0];
}

int main(int argc, char** argv) {
  int bw = atoi(argv[1]), bh = atoi(argv[2]), gw = atoi(argv[3]), gh = atoi(argv[4]);
  int x = atoi(argv[5]), y = atoi(argv[6]);
  void* fnp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto fn = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(fnp);
  void* g; cudaMalloc(&g, size_t(gw) * gh * 8);
  CUtensorMap m;
  cuuint64_t gd[2] = {cuuint64_t(gw), cuuint64_t(gh)}, gs[1] = {cuuint64_t(gw) * 8};
  cuuint32_t box[2] = {cuuint32_t(bw), cuuint32_t(bh)}, es[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, g, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap* dm; cudaMalloc(&dm, sizeof(m)); cudaMemcpy(dm, &m, sizeof(m), cudaMemcpyHostToDevice);
  unsigned long long* out; cudaMalloc(&out, 8);
  unsigned bytes = unsigned(bw) * bh * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  k<<<1, 128, bytes>>>(dm, x, y, bytes, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("box %dx%d (%d B rows) global %dx%d at (%d,%d): encode=%d run=%s\n", bw, bh, bw * 8, gw, gh, x, y, int(r), cudaGetErrorString(e));
  return 0;
}
