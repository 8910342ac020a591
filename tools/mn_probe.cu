// Descriptor probe (diagnostics, not product): D[128 cols x 16] = V^T x P with
// V^T an MN-major SW128 operand loaded by 2-D TMA boxes {64 cols, 128 rows}
// and P a K-major SW128 operand written by CUDA cores (1 KB per 64 tokens,
// rows 0..3 valid, rows 8..15 aliased to the next block).  Checks against CPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2407_21118_b200/csrc \
//        -o tools/mn_probe tools/mn_probe.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "palu_sm100.cuh"

using namespace palu::tc;

__global__ void probe(const __grid_constant__ CUtensorMap map_v, const float* P, float* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = sm;               // 2 x 16 KB
  uint8_t* Bp = sm + 32768;      // 2 x 1 KB + slack
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 32768 + 4096);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // P (K-major SW128): token t, head h -> block t/64, row h, 16-B chunk ((t%64)/8) ^ h
  for (int i = tid; i < 4 * 128; i += blockDim.x) {
    const int h = i / 128, t = i % 128, w = t % 64;
    const uint32_t off = (t / 64) * 1024 + h * 128 + ((((w >> 3) ^ h) & 7) << 4) + (w & 7) * 2;
    *reinterpret_cast<__nv_bfloat16*>(Bp + off) = __float2bfloat16(P[h * 128 + t]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *slot;
  if (tid == 0) {
    mbar_expect_tx(&bar[0], 32768);
    tma_load_2d(&map_v, &bar[0], A, 0, 0);
    tma_load_2d(&map_v, &bar[0], A + 16384, 64, 0);
    mbar_wait(&bar[0], 0);
    fence_after();
    for (int kk = 0; kk < 8; ++kk)
      umma_bf16_id(tmem, sdesc_mn(smem_u32(A) + kk * 2048, 16384, 1024),
                   sdesc(smem_u32(Bp) + (kk / 4) * 1024 + (kk % 4) * 32), IDESC_V, kk > 0);
    umma_commit(&bar[1]);
  }
  mbar_wait(&bar[1], 0);
  fence_after();
  float v[16];
  tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
  tmem_wait_ld();
  for (int n = 0; n < 16; ++n) out[tid * 16 + n] = v[n];
  fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 256, cols = 256;
  std::vector<__nv_bfloat16> hv(rows * cols);
  std::vector<float> vf(rows * cols), P(4 * 128);
  srand(1);
  for (int i = 0; i < rows * cols; ++i) {
    vf[i] = (float)((rand() % 17) - 8) / 8.f;
    hv[i] = __float2bfloat16(vf[i]);
  }
  for (auto& x : P) x = (float)((rand() % 9) - 4) / 4.f;
  __nv_bfloat16* dv;
  float *dp, *dout;
  cudaMalloc(&dv, hv.size() * 2);
  cudaMalloc(&dp, P.size() * 4);
  cudaMalloc(&dout, 128 * 16 * 4);
  cudaMemcpy(dv, hv.data(), hv.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, P.data(), P.size() * 4, cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  const cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  CUresult r = ((EncodeFn)fp)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dv, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<<<1, 128, 48 * 1024>>>(map, dp, dout);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> out(128 * 16);
  cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 4; ++n) {
      double ref = 0;
      for (int t = 0; t < 128; ++t) ref += (double)vf[t * cols + m] * P[n * 128 + t];
      maxerr = fmax(maxerr, fabs(ref - out[m * 16 + n]));
      if (m < 2) printf("m %d n %d ref %.4f got %.4f\n", m, n, ref, out[m * 16 + n]);
    }
  printf("max abs err %.3e %s\n", maxerr, maxerr < 1e-3 ? "PASS" : "FAIL");
  return 0;
}
