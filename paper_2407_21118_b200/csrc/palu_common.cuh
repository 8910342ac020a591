// Shared helpers for the Palu B200 kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdarg.h>
#include <stdio.h>

#include "palu_b200.h"

namespace palu {

void set_error(const char* fmt, ...);

#define PALU_CK(x)                                                                   \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      ::palu::set_error("%s:%d %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return PALU_ECUDA;                                                             \
    }                                                                                \
  } while (0)

#define PALU_REQUIRE(cond, ...)               \
  do {                                        \
    if (!(cond)) {                            \
      ::palu::set_error(__VA_ARGS__);         \
      return PALU_EVALIDATION;                \
    }                                         \
  } while (0)

#define PALU_LAUNCHED() PALU_CK(cudaGetLastError())

// ---- programmatic dependent launch (PDL) -----------------------------------
// Every kernel of the decode step is launched with programmatic stream
// serialisation, triggers its dependents at entry and waits for its
// predecessor (griddepcontrol.wait) before touching any global data: the next
// kernel's launch and CTA ramp then overlap this kernel's tail.  Every kernel
// waits, so completion stays transitive along the stream.  PALU_PDL=0 turns
// the attribute off (griddepcontrol.* are no-ops then).
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Split form (GEMV, query absorb, score and value kernels): launch
// dependents first, wait for the predecessor only where its output is read.
// A kernel K starts once its predecessor P executed launch_dependents: if P
// waits first (pdl_enter), everything before P has completed; if P is split,
// only what precedes P's own wait is guaranteed.  In the step order
//   gemv (split) -> append K+V + absorb (split: one grid; append blocks wait
//   first, absorb blocks before reading q) -> score (split) -> value (split)
//   -> merge (enter) -> gemv (split)
// score and value may start while the append of row t still runs.  Rule:
// every thread that reads a latent row,
// scale or zero point of the NEWEST token (row t) executes pdl_wait() first
// (griddepcontrol.wait returns after the whole predecessor chain completed).
// Rows < t were written by earlier steps and may be read before the wait:
// the value producer streams them early and waits before the last tile; the
// score producer waits before its first UW load; the converter and epilogue
// warps wait at entry.  gemv and absorb read only constants early.
__device__ __forceinline__ void pdl_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();
int pdl_split();  // PALU_PDL_SPLIT=0: split-form kernels wait at entry (A/B diagnostics)

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

typedef __nv_bfloat16 bf16;

// Weight-streaming bf16 GEMV (palu_gemv.cu); PALU_EUNSUPPORTED if the shape
// is not streamable (the caller falls back to the warp-per-row kernel).
int gemv_stream(const bf16* W, int N, int K, const float* x, int B, int ldx, float* y, int ldy,
                int acc, cudaStream_t st);

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(bf16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

// 16-byte vector of storage elements -> fp32
template <typename T> struct Vec16;
template <> struct Vec16<float> {
  static constexpr int N = 4;
  static __device__ __forceinline__ void unpack(const uint4& v, float* f) {
    f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
  }
};
template <> struct Vec16<bf16> {
  static constexpr int N = 8;
  static __device__ __forceinline__ void unpack(const uint4& v, float* f) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
};

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <typename F>
__device__ __forceinline__ float warp_reduce(float v, F op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Extract code `k` from a little-endian packed row (quant.py:156-169 order).
__device__ __forceinline__ uint32_t packed_code(const uint8_t* row, int row_bytes, int k, int bits) {
  const int bit = k * bits;
  const int byte = bit >> 3;
  uint32_t v = row[byte];
  if (byte + 1 < row_bytes) v |= uint32_t(row[byte + 1]) << 8;
  return (v >> (bit & 7)) & ((1u << bits) - 1u);
}

// packed fp32x2 FMA (sm_100 FFMA2): d = a * b + c elementwise
__device__ __forceinline__ float2 ffma2_f(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

// Round half away from zero (quant.py:31-32), no contraction.
__device__ __forceinline__ double round_half_away(double x) {
  return x >= 0.0 ? floor(__dadd_rn(x, 0.5)) : ceil(__dsub_rn(x, 0.5));
}

// sincos of a large fp64 angle: Cody-Waite reduction by 2*pi first, so the
// library call stays on its fast path (t * theta reaches 1e5 rad at 128K).
__device__ __forceinline__ void sincos_big(double x, double* sn, double* cs) {
  const double k = rint(x * 0.15915494309189535);    // 1 / (2 pi)
  double r = fma(-k, 6.283185307179586, x);           // 2 pi (hi)
  r = fma(-k, 2.4492935982947064e-16, r);             // 2 pi (lo)
  sincos(r, sn, cs);
}

}  // namespace palu
