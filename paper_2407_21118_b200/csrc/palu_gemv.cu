// Weight-streaming GEMV for the decode step's projections (sm_100a):
//   y[b][n] (+)= sum_k W[n][k] x[b][k]      W bf16 row-major, x / y fp32
// attention.py:428-431 (q = x W_q), :343-347 (x A_k, x A_v; one GEMV over the
// stacked [W_q | A_k | A_v]^T rows) and :361 (ctx @ wo_fused).
//
// HBM-bound: every weight byte is read once per step.  One persistent CTA per
// SM owns a contiguous, balanced range of rows -- one contiguous byte range
// of W -- and streams it through a 5 x 32 KB shared-memory ring with 1-D bulk
// copies (cp.async.bulk, one producer thread, up to 160 KB in flight per SM).
// The weights do not depend on the preceding kernel, so the producer starts
// at launch (programmatic dependent launch) and the ring fills while the
// predecessor drains; the 8 consumer warps wait for it only before loading
// x.  Lane l of warp w owns the same K positions of every row
// (w K/8 + 8 l + 256 i), so its slice of x lives in registers for the whole
// kernel and each 16-byte weight load feeds 8 FMAs per batch row with no
// shared-memory x traffic; the cross-warp sum is a fixed-order reduction
// (deterministic, no atomics).
#include "palu_sm100.cuh"
#include "palu_tmap.cuh"

namespace palu {
namespace tc {

// ring geometry (overridable at build time for A/B builds)
#ifndef PALU_GS_WARPS
#define PALU_GS_WARPS 8
#endif
#ifndef PALU_GS_CHUNK
#define PALU_GS_CHUNK 32768
#endif
#ifndef PALU_GS_SLOTS
#define PALU_GS_SLOTS 5
#endif
constexpr int GS_WARPS = PALU_GS_WARPS;
constexpr int GS_THREADS = (GS_WARPS + 1) * 32;
constexpr int GS_CHUNK = PALU_GS_CHUNK;
constexpr int GS_SLOTS = PALU_GS_SLOTS;

// KR8: 16-byte weight loads per lane per row (= K / 2048); NB: batch rows
template <int KR8, int NB>
__global__ void __launch_bounds__(GS_THREADS, 1)
gemv_stream_kernel(const __grid_constant__ CUtensorMap map_w, const bf16* __restrict__ W, int N, int K,
                   const float* __restrict__ x, int ldx,
                   float* __restrict__ y, int ldy, int accumulate, int rpc, int diag) {
  pdl_launch();
  extern __shared__ __align__(128) uint8_t gs_smem[];
  uint8_t* ring = gs_smem;                                            // GS_SLOTS x GS_CHUNK
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + GS_SLOTS * GS_CHUNK);
  uint64_t* empty = full + GS_SLOTS;
  float* red = reinterpret_cast<float*>(empty + GS_SLOTS);            // [2][8 warps][rpc][NB]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = (int)(((long long)N * blockIdx.x) / gridDim.x);
  const int r1 = (int)(((long long)N * (blockIdx.x + 1)) / gridDim.x);
  const int nchunks = (r1 - r0 + rpc - 1) / rpc;
  const size_t row_bytes = (size_t)K * 2;
  if (threadIdx.x == 0) {
    prefetch_map(&map_w);
    for (int s = 0; s < GS_SLOTS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], GS_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == GS_WARPS) {
    // ---------------- producer: contiguous row chunks of W ----------------
    if (lane == 0) {
      const uint64_t pol_first = policy_evict_first();
      Ring rg;
      for (int c = 0; c < nchunks; ++c, rg.next(GS_SLOTS)) {
        const int row = r0 + c * rpc;
        const int nr = min(rpc, r1 - row);
        mbar_wait(&empty[rg.slot], rg.phase ^ 1);
        mbar_expect_tx(&full[rg.slot], (uint32_t)(nr * row_bytes));
        // one 2-D tensor box per weight row (W viewed as 256-byte rows); the
        // weights are read once per step: evict-first (an L2 hit on rows the
        // score kernel prefetched demotes them)
        for (int r = 0; r < nr; ++r)
          tma_load_2d_hint(&map_w, &full[rg.slot], ring + rg.slot * GS_CHUNK + r * row_bytes, 0,
                           (int)((size_t)(row + r) * (row_bytes / 256)), pol_first);
      }
    }
    return;  // the producer takes no part in the reductions below
  }
  // ---------------- consumers ----------------
  pdl_wait();  // x is the predecessor's output
  const int kw = K / GS_WARPS;
  float xr[NB][KR8][8];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int i = 0; i < KR8; ++i) {
      const float4* xp = reinterpret_cast<const float4*>(x + (size_t)b * ldx + warp * kw + 8 * lane + 256 * i);
      const float4 a = __ldg(xp), c = __ldg(xp + 1);
      xr[b][i][0] = a.x; xr[b][i][1] = a.y; xr[b][i][2] = a.z; xr[b][i][3] = a.w;
      xr[b][i][4] = c.x; xr[b][i][5] = c.y; xr[b][i][6] = c.z; xr[b][i][7] = c.w;
    }
  const uint32_t lane_off = (uint32_t)(warp * kw + 8 * lane) * 2;
  constexpr int MAXR = GS_CHUNK / (2048 * 2 * KR8) > 0 ? GS_CHUNK / (2048 * 2 * KR8) : 1;  // = rpc
  Ring rg;
  for (int c = 0; c < nchunks; ++c, rg.next(GS_SLOTS)) {
    const int row = r0 + c * rpc;
    const int nr = min(rpc, r1 - row);
    mbar_wait(&full[rg.slot], rg.phase);
    const uint32_t base = smem_u32(ring + rg.slot * GS_CHUNK) + lane_off;
    float* rb = red + (size_t)(c & 1) * GS_WARPS * rpc * NB;
    // all rows of the chunk at once: independent FMA and shuffle-reduction
    // chains per row (a row at a time left each warp waiting on one 5-step
    // shuffle chain after another)
    float acc[MAXR][NB];
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
#pragma unroll
      for (int b = 0; b < NB; ++b) acc[r][b] = 0.f;
      if (r < nr && !(diag & 1)) {  // diag 1 (diagnostic builds): stream without the math
        uint4 wv[KR8];
#pragma unroll
        for (int i = 0; i < KR8; ++i) wv[i] = lds128(base + (uint32_t)(r * row_bytes) + 512u * i);
#pragma unroll
        for (int i = 0; i < KR8; ++i) {
          float wf[8];
          Vec16<bf16>::unpack(wv[i], wf);
#pragma unroll
          for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[r][b] = fmaf(wf[e], xr[b][i][e], acc[r][b]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < MAXR; ++r)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[r][b] += __shfl_xor_sync(0xffffffffu, acc[r][b], o);
      }
    if (lane == 0)
#pragma unroll
      for (int r = 0; r < MAXR; ++r)
        if (r < nr)
#pragma unroll
          for (int b = 0; b < NB; ++b) rb[(warp * rpc + r) * NB + b] = acc[r][b];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[rg.slot]);  // all lanes' smem reads of the slot are done
    named_bar_sync(1, GS_WARPS * 32);
    for (int o = threadIdx.x; o < nr * NB; o += GS_WARPS * 32) {
      const int r = o / NB, b = o - r * NB;
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < GS_WARPS; ++w) v += rb[(w * rpc + r) * NB + b];
      float* dst = y + (size_t)b * ldy + row + r;
      *dst = accumulate ? *dst + v : v;
    }
  }
}

static int gemv_diag() {
#ifdef PALU_DIAG
  return getenv("PALU_GEMV_DIAG") ? atoi(getenv("PALU_GEMV_DIAG")) : 0;
#else
  return 0;
#endif
}

template <int KR8, int NB>
static int launch_stream(const bf16* W, int N, int K, const float* x, int ldx, float* y, int ldy,
                         int acc, cudaStream_t st) {
  const int rpc = GS_CHUNK / (K * 2);
  const size_t smem = (size_t)GS_SLOTS * GS_CHUNK + 2 * GS_SLOTS * 8 + 2 * GS_WARPS * rpc * NB * 4 + 16;
  static bool attr = false;
  if (!attr) {
    PALU_CK(cudaFuncSetAttribute(gemv_stream_kernel<KR8, NB>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = N < sms ? N : sms;
  CUtensorMap map_w;
  const CUresult mr = make_map_stream(&map_w, W, (uint64_t)N * K * 2, (uint32_t)(K * 2));
  if (mr != CUDA_SUCCESS) {
    set_error("gemv: cuTensorMapEncodeTiled failed (%d)", (int)mr);
    return PALU_ECUDA;
  }
  PALU_CK(launch_k(gemv_stream_kernel<KR8, NB>, dim3(grid), dim3(GS_THREADS), smem, st, map_w, W, N, K, x,
                   ldx, y, ldy, acc, rpc, gemv_diag()));
  PALU_LAUNCHED();
  return PALU_OK;
}

template <int KR8>
static int stream_nb(const bf16* W, int N, int K, const float* x, int B, int ldx, float* y, int ldy,
                     int acc, cudaStream_t st) {
  // x slice in registers: KR8 * 8 floats per batch row (<= 64 in total)
  constexpr int MAXB = KR8 <= 2 ? 4 : (KR8 <= 4 ? 2 : 1);
  for (int b0 = 0; b0 < B; b0 += MAXB) {
    const int nb = B - b0 < MAXB ? B - b0 : MAXB;
    const float* xb = x + (size_t)b0 * ldx;
    float* yb = y + (size_t)b0 * ldy;
    int rc;
    if (nb == 1) rc = launch_stream<KR8, 1>(W, N, K, xb, ldx, yb, ldy, acc, st);
    else if (nb == 2) rc = launch_stream<KR8, (MAXB >= 2 ? 2 : 1)>(W, N, K, xb, ldx, yb, ldy, acc, st);
    else if (nb == 3) {
      rc = launch_stream<KR8, (MAXB >= 2 ? 2 : 1)>(W, N, K, xb, ldx, yb, ldy, acc, st);
      if (!rc) rc = launch_stream<KR8, 1>(W, N, K, xb + 2 * (size_t)ldx, ldx, yb + 2 * (size_t)ldy, ldy, acc, st);
    } else rc = launch_stream<KR8, (MAXB >= 4 ? 4 : 1)>(W, N, K, xb, ldx, yb, ldy, acc, st);
    if (rc) return rc;
  }
  return PALU_OK;
}

}  // namespace tc

// Returns PALU_EUNSUPPORTED when the shape is not streamable (the caller then
// uses the warp-per-row kernel): K a multiple of 2048 up to 16384, batch <= 256
// (more than MAXB rows stream the weights once per MAXB-row chunk).
int gemv_stream(const bf16* W, int N, int K, const float* x, int B, int ldx, float* y, int ldy,
                int acc, cudaStream_t st) {
  using namespace tc;
  if (K % 2048 != 0 || K > 16384 || B > 256 || ldx % 4 != 0) return PALU_EUNSUPPORTED;
  switch (K / 2048) {
    case 1: return stream_nb<1>(W, N, K, x, B, ldx, y, ldy, acc, st);
    case 2: return stream_nb<2>(W, N, K, x, B, ldx, y, ldy, acc, st);
    case 3: return stream_nb<3>(W, N, K, x, B, ldx, y, ldy, acc, st);
    case 4: return stream_nb<4>(W, N, K, x, B, ldx, y, ldy, acc, st);
    case 6: return stream_nb<6>(W, N, K, x, B, ldx, y, ldy, acc, st);
    case 8: return stream_nb<8>(W, N, K, x, B, ldx, y, ldy, acc, st);
    default: return PALU_EUNSUPPORTED;
  }
}

}  // namespace palu
