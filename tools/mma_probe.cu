// tcgen05 throughput probe (diagnostics, not product): back-to-back
// kind::f16 MMAs on resident smem operands, one CTA (or CTA pair) per SM,
// all SMs busy; reports ns per MMA and TFLOP/s for several shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_21118_b200/csrc \
//        -I include -o tools/mma_probe tools/mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#include "palu_sm100.cuh"

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

using namespace palu::tc;

template <int M, int N, int CG>
__global__ void __launch_bounds__(320, 1) mma_probe(int iters, float* sink, int extra,
                                                    const __grid_constant__ CUtensorMap map) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 128 * 1024);  // [0] end [1] unused [2] commit [4..7] TMA ring
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 8);
  const int warp = threadIdx.x >> 5;
  uint32_t rank = 0;
  if (CG == 2) rank = cluster_rank();
  if (threadIdx.x == 0) {
    *reinterpret_cast<int*>(slot + 4) = 0;
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    mbar_init(&bar[0], 1);
    for (int r = 0; r < 4; ++r) mbar_init(&bar[4 + r], 1);
    mbar_init(&bar[3], 1);
    mbar_arrive(&bar[3]);  // phase 0 complete: waits on it return at once
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  if (extra & 16) {  // random bf16 operands in [-1, 1) (all-zero smem toggles no datapath bits)
    uint16_t* h = reinterpret_cast<uint16_t*>(sm);
    for (int i = threadIdx.x; i < 96 * 512; i += blockDim.x) {
      uint32_t x = (uint32_t)i * 2654435761u ^ (blockIdx.x * 40503u);
      x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
      const float f = (float)(x & 0xFFFF) / 32768.f - 1.f;
      h[i] = (uint16_t)(__float_as_uint(f) >> 16);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();
  fence_after();
  const uint32_t tmem = *slot;
  constexpr uint32_t ID = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                          ((uint32_t)(M >> 4) << 24);
  if (threadIdx.x == 0 && (CG == 1 || rank == 0)) {
    const unsigned long long c0 = clock64(), g0 = gtimer_ns();
    const uint32_t a0 = smem_u32(sm), b = smem_u32(sm + 32 * 1024);
    for (int i = 0; i < iters; ++i) {
      if (extra & 4) {  // a commit per 4 MMAs (the score kernel's per-k-block stage release)
        if (CG == 1) umma_commit(&bar[2]); else umma2_commit_both(&bar[2]);
      }
      if ((extra & 8) && (i & 3) == 0) {  // different A stage per k-block (16 KB apart)
      }
      const uint32_t a = (extra & 8) ? a0 + (uint32_t)((i & 1) * 16384) : a0;
      if (extra & 128) {  // the score kernel's per-k-block wait: satisfied mbarrier + tcgen05 fence
        mbar_wait(&bar[3], 0);
        fence_after();
      }
      if ((extra & 256) && (i & 3) == 0) {  // per unit: + a global store of a timestamp (trace)
        sink[4 + (i & 7)] = (float)gtimer_ns();
      }
      // extra 32: the score kernel's D pattern (slot alternates every 16 MMAs,
      // first MMA of a unit overwrites); extra 64: accumulate flag only
      const uint32_t dt = (extra & 32) ? tmem + (uint32_t)(((i >> 2) & 1) * 256) : tmem;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t acc = ((extra & 96) && (i & 3) == 0 && kk == 0) ? 0u : 1u;
        if (CG == 1)
          umma_bf16_id(dt, sdesc(a + kk * 32), sdesc(b + kk * 32), ID, acc);
        else
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dt),
              "l"(sdesc(a + kk * 32)), "l"(sdesc(b + kk * 32)), "r"(ID), "r"(acc)
              : "memory");
      }
    }
    if (CG == 1)
      umma_commit(&bar[0]);
    else
      umma2_commit_both(&bar[0]);
    mbar_wait(&bar[0], 0);
    if (blockIdx.x == 0) {
      sink[2] = (float)(clock64() - c0);
      sink[3] = (float)(gtimer_ns() - g0);
    }
  }
  volatile int* stop = reinterpret_cast<volatile int*>(slot + 4);
  if (threadIdx.x == 0) { if (!(CG == 1 || rank == 0)) mbar_wait(&bar[0], 0); *stop = 1; }
  if (warp == 1 && (extra & 1) && lane_id() == 0) {
    // continuous TMA tile loads, 4 x 16 KB in flight, into a ring at 64..128 KB
    // (no consumer): the score kernel's H-stage write pressure on shared memory
    for (int i = 0; *stop == 0 && i < 100000000; ++i) {
      const int r = i & 3;
      if (i >= 4) mbar_wait(&bar[4 + r], ((i >> 2) - 1) & 1);
      mbar_expect_tx(&bar[4 + r], 16384);
      tma_load_2d(&map, &bar[4 + r], sm + 64 * 1024 + r * 16384, 0,
                  (int)(((blockIdx.x * 28331u + (unsigned)i) * 128u) % (1u << 22)));
    }
  }
  if (warp >= 2 && (extra & 512)) {
    // 8 warps stream a 16 KB L1-resident table with 16-B __ldg loads (the
    // score epilogue's cos/sin base rows) while the MMAs run
    const float4* tab = reinterpret_cast<const float4*>(sink + 64);
    float acc = 0.f;
    for (int i = 0; *stop == 0 && i < 10000000; ++i) {
      float4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldg(tab + ((threadIdx.x + 256 * k + i * 8) & 1023));
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += v[k].x * v[k].y + v[k].z * v[k].w;
    }
    if (acc == 12345.f) sink[1] = acc;
  }
  if (warp >= 2 && (extra & 2)) {
    // 8 warps read the other TMEM slot like the score epilogue (2 x 16 columns, wait, FMAs)
    float v[16], w[16], acc = 0.f;
    for (int i = 0; *stop == 0 && i < 10000000; ++i) {
      const uint32_t col = 256 + (i & 3) * 32 + ((warp - 2) >> 2) * 128;
      tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + col, v);
      tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + col + 16, w);
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 16; ++k) acc = fmaf(v[k], w[k], acc);
    }
    if (acc == 12345.f) sink[1] = acc;
  }
  fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();
  if (warp == 0) {
    fence_after();
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
  if (iters < 0) sink[0] = 1.f;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static CUtensorMap g_map;
static int g_extra = 0;

template <int M, int N, int CG>
void run(const char* name) {
  auto k = mma_probe<M, N, CG>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = 140 * 1024;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = CG;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  float* sink;
  cudaMalloc(&sink, 64 * 1024);
  cudaMemset(sink, 0, 64 * 1024);
  const int iters = getenv("ITERS") ? atoi(getenv("ITERS")) : 4000;
  cudaLaunchKernelEx(&cfg, k, iters, sink, g_extra, g_map);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, k, iters, sink, g_extra, g_map);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double mmas = (double)iters * 4;  // per issuing CTA
  const int issuers = 148 / CG;
  const double flops = 2.0 * M * N * 16 * mmas * issuers;
  float hs[4];
  cudaMemcpy(hs, sink, 16, cudaMemcpyDeviceToHost);
  printf("extra %d %-24s %7.2f ns/MMA  %7.1f TFLOP/s  CTA0: %.3f GHz %.0f clk/MMA (%s)\n", g_extra, name,
         ms * 1e6 / mmas, flops / (ms * 1e-3) / 1e12, hs[2] / hs[3], hs[2] / mmas,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  void* buf;
  cudaMalloc(&buf, (size_t)1024 << 20);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  const cuuint64_t dims[2] = {64, 1u << 22};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  ((EncodeFn)fp)(&g_map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  for (int e : {0, 512, 16, 528}) {
    g_extra = e;
    run<256, 256, 2>("cta2 M256 N256 K16");
    run<128, 256, 1>("cta1 M128 N256 K16");
  }
  return 0;
}
