// Short-stream HBM probe (diagnostics, not product): 148 CTAs each stream a
// contiguous per-CTA share through a 2-D TMA ring (one producer thread, 8
// consumer warps that only release slots), timed over back-to-back launches
// on rotating buffers (no L2 reuse).  Answers: how long does a 67 MB weight
// stream (the decode GEMV) take at best, and how much of it is ramp?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_probe tools/stream_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes));
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)));
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(su32(b)),
               "r"(ph));
}

// W viewed as rows of 256 B; a box = box_rows x 256 B contiguous
__global__ void __launch_bounds__(288, 1) stream(const __grid_constant__ CUtensorMap map, long long row0,
                                                 int rows_per_cta, int stages, int box_rows, int boxes_per_stage) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int chunk = box_rows * 256 * boxes_per_stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * chunk);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int n = rows_per_cta / (box_rows * boxes_per_stage);
  const long long base = row0 + (long long)blockIdx.x * rows_per_cta;
  if (warp == 8) {
    if (lane == 0)
      for (int i = 0; i < n; ++i) {
        const int s = i % stages;
        mb_wait(&empty[s], ((i / stages) & 1) ^ 1);
        mb_expect(&full[s], chunk);
        for (int b = 0; b < boxes_per_stage; ++b) {
          const int row = (int)(base + (long long)(i * boxes_per_stage + b) * box_rows);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                  su32(sm + (size_t)s * chunk + b * box_rows * 256)),
              "l"(&map), "r"(su32(&full[s])), "r"(0), "r"(row)
              : "memory");
        }
      }
    return;
  }
  for (int i = 0; i < n; ++i) {
    const int s = i % stages;
    mb_wait(&full[s], (i / stages) & 1);
    __syncwarp();
    if (lane == 0) mb_arrive(&empty[s]);
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t total = (size_t)4 << 30;
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const long long rows_total = (long long)(total / 256);
  for (size_t per_cta : {(size_t)458752, (size_t)1835008}) {   // 67.9 MB and 272 MB in total
    for (int box_rows : {32, 128}) {
      CUtensorMap map;
      const cuuint64_t dims[2] = {256, (cuuint64_t)rows_total};
      const cuuint64_t strides[1] = {256};
      const cuuint32_t box[2] = {256, (cuuint32_t)box_rows}, es[2] = {1, 1};
      ((EncodeFn)fp)(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int stage_kb : {16, 32, 64})
        for (int stages : {3, 5, 8, 12}) {
          const int chunk = stage_kb * 1024;
          if (chunk < box_rows * 256) continue;
          if ((size_t)chunk * stages > 210 * 1024) continue;
          const int bps = chunk / (box_rows * 256);
          const int rows_per_cta = (int)(per_cta / 256);
          const size_t smem = (size_t)chunk * stages + 16 * stages + 64;
          const long long per_launch_rows = (long long)rows_per_cta * 148;
          const int reps = 20;
          for (int w = 0; w < 2; ++w)
            stream<<<148, 288, smem>>>(map, 0, rows_per_cta, stages, box_rows, bps);
          cudaEventRecord(a);
          for (int r = 0; r < reps; ++r)
            stream<<<148, 288, smem>>>(map, (r % 8) * per_launch_rows, rows_per_cta, stages, box_rows, bps);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          const double us = ms * 1e3 / reps, bytes = (double)per_cta * 148;
          printf("per-CTA %7zu B, box %3d rows, stage %2d KB x %2d: %7.2f us/launch, %7.1f GB/s\n", per_cta,
                 box_rows, stage_kb, stages, us, bytes / (us * 1e3));
        }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
