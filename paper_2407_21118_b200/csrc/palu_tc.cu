// tcgen05 (sm_100a) RoPE score kernel -- placeholder until the tensor-core
// path lands; the RoPE tables are final.
#include <math.h>

#include "palu_common.cuh"

namespace palu {

// tile bases: cos/sin(t0 * th_j) for t0 = 128 * tile, fp64 angle reduction;
// offsets: cos/sin(delta * th_j) for delta in [0, 128).
__global__ void rope_table_kernel(const double* __restrict__ theta, int half, int n_tiles,
                                  float2* __restrict__ tab) {
  const int total = (n_tiles + 128) * half;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int row = i / half, j = i - row * half;
    const double pos = row < n_tiles ? 128.0 * row : (double)(row - n_tiles);
    double sn, cs;
    sincos(pos * theta[j], &sn, &cs);
    tab[i] = make_float2((float)cs, (float)sn);
  }
}

}  // namespace palu

using namespace palu;

extern "C" {

size_t palu_rope_table_floats(int half, int T_cap) {
  const int n_tiles = (T_cap + 127) / 128 + 1;
  return (size_t)2 * (n_tiles + 128) * half;
}

int palu_rope_table(const double* theta, int half, int T_cap, float* rope_tab, void* stream) {
  PALU_REQUIRE(half > 0 && T_cap > 0, "palu_rope_table: bad sizes");
  const int n_tiles = (T_cap + 127) / 128 + 1;
  rope_table_kernel<<<256, 256, 0, (cudaStream_t)stream>>>(theta, half, n_tiles,
                                                           reinterpret_cast<float2*>(rope_tab));
  PALU_LAUNCHED();
  return PALU_OK;
}

int palu_rope_score_tc(int bits, const void* hk, const float* scales, const float* zps, int B,
                       int n_heads, int s_k, int G, int R_pad, int T_cap, const void* uw,
                       const float* rope_tab, const int* t_dev, float* logits, int ld_logits,
                       void* stream) {
  set_error("palu_rope_score_tc: tensor-core path not built yet");
  return PALU_EUNSUPPORTED;
}

}  // extern "C"
