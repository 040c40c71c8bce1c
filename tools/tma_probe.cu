// TMA probe: variants (argv[1]) of a cp.async.bulk.tensor load into smem.
//  0: 4-D FLOAT64 box 34x10x20x1, descriptor as __grid_constant__ param
//  1: 2-D FLOAT64 box 32x8, param
//  2: 2-D FLOAT32 box 32x8, param
//  3: 4-D FLOAT64, descriptor in global memory
//  4: 2-D FLOAT64, .shared::cta destination form
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int kDim, bool kCta>
__global__ void k(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, unsigned bytes, float* out, int gx = 0, int gy = 0) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) unsigned long long bar;
  const CUtensorMap* map = gtm ? gtm : &tm;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes) : "memory");
    if (kDim == 3)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(su(sm)), "l"(map), "r"(su(&bar)), "r"(1), "r"(1), "r"(0) : "memory");
    else if (kDim == 5)
      asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                   ::"r"(su(sm)), "l"(map), "r"(su(&bar)), "r"(1), "r"(1), "r"(0), "r"(0), "r"(0) : "memory");
    else if (kDim == 4 && kCta)
      asm volatile("cp.async.bulk.tensor.4d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                   ::"r"(su(sm)), "l"(map), "r"(su(&bar)), "r"(-2), "r"(-1), "r"(0), "r"(1) : "memory");
    else if (kDim == 4)
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                   ::"r"(su(sm)), "l"(map), "r"(su(&bar)), "r"(-2), "r"(-1), "r"(0), "r"(1) : "memory");
    else if (!kCta)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(su(sm)), "l"(map), "r"(su(&bar)), "r"(gx), "r"(gy) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(su(sm)), "l"(map), "r"(su(&bar)), "r"(0), "r"(0) : "memory");
  }
  asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W_%=; }" ::"r"(su(&bar)) : "memory");
  for (unsigned e = threadIdx.x; e < bytes / 4; e += blockDim.x) out[e] = sm[e];
}
int main(int argc, char** argv) {
  const int v = argc > 1 ? atoi(argv[1]) : 0;
  const int nx = 200, ny = 40, pitch = 208, S = 2;
  const size_t plane = (size_t)ny * pitch, n = plane * 20 * S;
  std::vector<double> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = (double)i;
  double* d; float* o;
  cudaMalloc(&d, n * 8); cudaMalloc(&o, 1 << 20);
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaError_t ge = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  printf("entry %d q=%d fn=%p\n", (int)ge, (int)q, fn);
  CUtensorMap tm;
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r; unsigned bytes;
  const int B0 = argc > 2 ? atoi(argv[2]) : 34, B1 = argc > 3 ? atoi(argv[3]) : 10,
            B2 = argc > 4 ? atoi(argv[4]) : 20;
  if (v == 5 || v == 7) {
    cuuint64_t dims[5] = {nx, ny, 20, S, 1}, str[4] = {pitch * 8, plane * 8, plane * 20 * 8, plane * 40 * 8};
    cuuint32_t box[5] = {(cuuint32_t)B0, (cuuint32_t)B1, (cuuint32_t)B2, 1, 1};
    r = ((Enc)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, v == 5 ? 3 : 5, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    bytes = B0 * B1 * B2 * 8;
  } else if (v == 0 || v == 3 || v == 6) {
    cuuint64_t dims[4] = {nx, ny, 20, S}, str[3] = {pitch * 8, plane * 8, plane * 20 * 8};
    cuuint32_t box[4] = {(cuuint32_t)B0, (cuuint32_t)B1, (cuuint32_t)B2, 1};
    r = ((Enc)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    bytes = B0 * B1 * B2 * 8;
  } else if (v == 2) {
    cuuint64_t dims[2] = {2 * nx, ny}, str[1] = {pitch * 8};
    cuuint32_t box[2] = {64, 8};
    r = ((Enc)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    bytes = 64 * 8 * 4;
  } else {
    cuuint64_t dims[2] = {nx, ny}, str[1] = {pitch * 8};
    cuuint32_t box[2] = {(cuuint32_t)B0, (cuuint32_t)B1};
    r = ((Enc)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    bytes = B0 * B1 * 8;
  }
  printf("variant %d encode %d\n", v, (int)r);
  CUtensorMap* gtm = nullptr;
  if (v == 3) { cudaMalloc(&gtm, sizeof(CUtensorMap)); cudaMemcpy(gtm, &tm, sizeof tm, cudaMemcpyHostToDevice); }
  const int smem = 65536;
  if (v == 5) { cudaFuncSetAttribute(k<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<3, false><<<1, 128, smem>>>(tm, gtm, bytes, o); }
  else if (v == 7) { cudaFuncSetAttribute(k<5, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<5, false><<<1, 128, smem>>>(tm, gtm, bytes, o); }
  else if (v == 6) { cudaFuncSetAttribute(k<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<4, true><<<1, 128, smem>>>(tm, gtm, bytes, o); }
  else if (v == 0 || v == 3) { cudaFuncSetAttribute(k<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<4, false><<<1, 128, smem>>>(tm, gtm, bytes, o); }
  else if (v == 4) { cudaFuncSetAttribute(k<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<2, true><<<1, 128, smem>>>(tm, gtm, bytes, o); }
  else { cudaFuncSetAttribute(k<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<2, false><<<1, 128, smem>>>(tm, gtm, bytes, o, argc > 5 ? atoi(argv[5]) : 0, argc > 6 ? atoi(argv[6]) : 0); }
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> ho(bytes / 4);
  cudaMemcpy(ho.data(), o, bytes, cudaMemcpyDeviceToHost);
  double first = 0; memcpy(&first, ho.data(), 8);
  printf("variant %d box %d %d %d: %s first=%g\n", v, B0, B1, B2, cudaGetErrorString(e), first);
  return 0;
}
