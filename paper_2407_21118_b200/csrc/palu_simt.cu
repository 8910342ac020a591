// Palu latent-KV RoPE decode: CUDA-core kernels + the C ABI (sm_100a).
//
// Each kernel restates one stage of palu_decode_step_rope
// (/root/reference/pkg/src/palu/attention.py:392-448); see include/palu_b200.h
// for the contracts and DESIGN.md for the HBM layout and rooflines.
#include <math.h>
#include <string.h>

#include "palu_common.cuh"
#include <stdlib.h>

namespace palu {

static thread_local char g_err[1024] = "";

bool pdl_enabled() {
  static const int on = [] {
    const char* e = getenv("PALU_PDL");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return on != 0;
}

int pdl_split() {
  static const int on = [] {
    const char* e = getenv("PALU_PDL_SPLIT");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return on;
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// GEMV:  y[b][n] (+)= sum_k W[n][k] x[b][k].  Weight-streaming (HBM-bound):
// one warp per 2 output rows, 16-byte non-allocating loads, 4 in flight per
// lane, x staged in shared memory in K chunks, up to MAXB batch rows per pass.
// ---------------------------------------------------------------------------
constexpr int GEMV_WARPS = 8;
constexpr int GEMV_UNROLL_DEF = 8;  // 16-byte weight loads in flight per lane

template <typename T, int MAXB, int GEMV_UNROLL>
__global__ void __launch_bounds__(GEMV_WARPS * 32)
gemv_kernel(const T* __restrict__ W, int N, int K, const float* __restrict__ x, int B, int ldx,
            float* __restrict__ y, int ldy, int accumulate, int split) {
  // the weights are constant: the first batch of weight loads is issued
  // before waiting for the predecessor that writes x (PDL split form)
  pdl_launch();
  if (!split) pdl_wait();
  using V = Vec16<T>;
  constexpr int VEC = V::N;
  constexpr int STEP = 32 * VEC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * GEMV_WARPS + warp;
  if (row >= N) return;
  const T* wr = W + (size_t)row * K;
  float acc[MAXB];
#pragma unroll
  for (int b = 0; b < MAXB; ++b) acc[b] = 0.f;
  uint4 nxt[GEMV_UNROLL];
  auto load = [&](int k) {
#pragma unroll
    for (int u = 0; u < GEMV_UNROLL; ++u)
      if (k + u * STEP < K) nxt[u] = ldg_stream(wr + k + u * STEP);
  };
  load(lane * VEC);
  pdl_wait();
  for (int k = lane * VEC; k < K; k += GEMV_UNROLL * STEP) {
    uint4 v[GEMV_UNROLL];
#pragma unroll
    for (int u = 0; u < GEMV_UNROLL; ++u) v[u] = nxt[u];
    if (k + GEMV_UNROLL * STEP < K) load(k + GEMV_UNROLL * STEP);  // next batch in flight
#pragma unroll
    for (int u = 0; u < GEMV_UNROLL; ++u) {
      const int kk = k + u * STEP;
      if (kk < K) {
        float wf[VEC];
        V::unpack(v[u], wf);
#pragma unroll
        for (int b = 0; b < MAXB; ++b) {
          if (b < B) {
            const float4* xp = reinterpret_cast<const float4*>(x + (size_t)b * ldx + kk);
#pragma unroll
            for (int e4 = 0; e4 < VEC / 4; ++e4) {
              const float4 t4 = __ldg(xp + e4);
              acc[b] = fmaf(wf[4 * e4], t4.x, acc[b]);
              acc[b] = fmaf(wf[4 * e4 + 1], t4.y, acc[b]);
              acc[b] = fmaf(wf[4 * e4 + 2], t4.z, acc[b]);
              acc[b] = fmaf(wf[4 * e4 + 3], t4.w, acc[b]);
            }
          }
        }
      }
    }
  }
#pragma unroll
  for (int b = 0; b < MAXB; ++b) {
    const float v = warp_reduce(acc[b], [](float a, float c) { return a + c; });
    if (lane == 0 && b < B) {
      float* dst = y + (size_t)b * ldy + row;
      *dst = accumulate ? *dst + v : v;
    }
  }
}

template <typename T, int MAXB>
static int launch_gemv(const T* W, int N, int K, const float* x, int B, int ldx, float* y, int ldy,
                       int acc, cudaStream_t st) {
  dim3 grid((N + GEMV_WARPS - 1) / GEMV_WARPS);
  static const int unroll = getenv("PALU_GEMV_UNROLL") ? atoi(getenv("PALU_GEMV_UNROLL")) : GEMV_UNROLL_DEF;
  if (unroll >= 16)
    PALU_CK(launch_k(gemv_kernel<T, MAXB, 16>, grid, dim3(GEMV_WARPS * 32), 0, st, W, N, K, x, B,
                     ldx, y, ldy, acc, pdl_split()));
  else
    PALU_CK(launch_k(gemv_kernel<T, MAXB, 8>, grid, dim3(GEMV_WARPS * 32), 0, st, W, N, K, x, B,
                     ldx, y, ldy, acc, pdl_split()));
  PALU_LAUNCHED();
  return PALU_OK;
}

template <typename T>
static int gemv_dispatch(const T* W, int N, int K, const float* x, int B, int ldx, float* y,
                         int ldy, int acc, cudaStream_t st) {
  for (int b0 = 0; b0 < B; b0 += 8) {
    const int nb = B - b0 < 8 ? B - b0 : 8;
    const float* xb = x + (size_t)b0 * ldx;
    float* yb = y + (size_t)b0 * ldy;
    int rc;
    if (nb == 1) rc = launch_gemv<T, 1>(W, N, K, xb, nb, ldx, yb, ldy, acc, st);
    else if (nb == 2) rc = launch_gemv<T, 2>(W, N, K, xb, nb, ldx, yb, ldy, acc, st);
    else if (nb <= 4) rc = launch_gemv<T, 4>(W, N, K, xb, nb, ldx, yb, ldy, acc, st);
    else rc = launch_gemv<T, 8>(W, N, K, xb, nb, ldx, yb, ldy, acc, st);
    if (rc) return rc;
  }
  return PALU_OK;
}

// ---------------------------------------------------------------------------
// Latent append (attention.py:343-347 + _GroupStore.append :248-255).
// One CTA per (group, batch row).  Quantised sides run quant.py:87-99 in fp64.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void append_raw_body(const float* __restrict__ lat, int ld_lat, int G,
                                                const int* __restrict__ ranks,
                                                const int* __restrict__ lat_off, T* __restrict__ rows,
                                                int R_pad, int T_cap, int t, int g, int b) {
  if (t >= T_cap) return;
  const int r = ranks[g];
  const float* src = lat + (size_t)b * ld_lat + lat_off[g];
  T* dst = rows + (((size_t)b * G + g) * T_cap + t) * R_pad;
  for (int c = threadIdx.x; c < R_pad; c += blockDim.x) dst[c] = from_f<T>(c < r ? src[c] : 0.f);
}

template <typename T>
__global__ void append_raw_kernel(const float* __restrict__ lat, int ld_lat, int G,
                                  const int* __restrict__ ranks, const int* __restrict__ lat_off,
                                  T* __restrict__ rows, int R_pad, int T_cap,
                                  const int* __restrict__ t_dev) {
  pdl_enter();
  append_raw_body<T>(lat, ld_lat, G, ranks, lat_off, rows, R_pad, T_cap, *t_dev, blockIdx.x, blockIdx.y);
}

// Quantise one row held in shared memory (fp64).  Mirrors quant.py:93-98.
__device__ void quantize_row_dev(const double* xrow, int cols, int bits, uint8_t* codes_out,
                                 double* s_out, int64_t* z_out, double* red /*[64]*/) {
  const int tid = threadIdx.x, nt = blockDim.x;
  double lo = INFINITY, hi = -INFINITY;
  for (int c = tid; c < cols; c += nt) {
    lo = fmin(lo, xrow[c]);
    hi = fmax(hi, xrow[c]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const int warp = tid >> 5, lane = tid & 31, nw = (nt + 31) >> 5;
  if (lane == 0) { red[warp] = lo; red[32 + warp] = hi; }
  __syncthreads();
  if (tid == 0) {
    double l = red[0], h = red[32];
    for (int w = 1; w < nw; ++w) { l = fmin(l, red[w]); h = fmax(h, red[32 + w]); }
    red[0] = l; red[32] = h;
  }
  __syncthreads();
  lo = red[0];
  hi = red[32];
  const double qmax = double((1 << bits) - 1);
  // scales = max(hi - lo, 1e-8) / qmax ;  zps = rha(-lo / scales)
  const double s = __ddiv_rn(fmax(__dsub_rn(hi, lo), 1e-8), qmax);
  const double z = round_half_away(__ddiv_rn(-lo, s));
  for (int c = tid; c < cols; c += nt) {
    double q = __dadd_rn(round_half_away(__ddiv_rn(xrow[c], s)), z);
    q = fmin(fmax(q, 0.0), qmax);
    codes_out[c] = (uint8_t)q;
  }
  if (tid == 0) { *s_out = s; *z_out = (int64_t)z; }
  __syncthreads();
}

__device__ void pack_row_dev(const uint8_t* codes, int cols, int bits, uint8_t* out) {
  const int nbytes = cols * bits / 8;
  for (int j = threadIdx.x; j < nbytes; j += blockDim.x) {
    uint32_t byte = 0;
    if (bits == 8) {
      byte = codes[j];
    } else if (bits == 4) {
      byte = codes[2 * j] | (codes[2 * j + 1] << 4);
    } else if (bits == 2) {
      byte = codes[4 * j] | (codes[4 * j + 1] << 2) | (codes[4 * j + 2] << 4) | (codes[4 * j + 3] << 6);
    } else {
      for (int p = 0; p < 8; ++p) {
        const int bit = 8 * j + p;
        byte |= ((codes[bit / bits] >> (bit % bits)) & 1u) << p;
      }
    }
    out[j] = (uint8_t)byte;
  }
}

__device__ __forceinline__ void append_quant_body(const float* __restrict__ lat, int ld_lat, int G,
                                                  int bits, const int* __restrict__ ranks,
                                                  const int* __restrict__ lat_off,
                                                  uint8_t* __restrict__ rows, float* __restrict__ scales,
                                                  float* __restrict__ zps, double* __restrict__ scales64,
                                                  int64_t* __restrict__ zps64, int R_pad, int T_cap,
                                                  int t, int g, int b, double* qsm) {
  // qsm: [R_pad] values, 64 reduction slots, then codes
  double* xrow = qsm;
  double* red = qsm + R_pad;
  uint8_t* codes = reinterpret_cast<uint8_t*>(red + 64);
  __shared__ double s_sh;
  __shared__ int64_t z_sh;
  if (t >= T_cap) return;
  const int r = ranks[g];
  const float* src = lat + (size_t)b * ld_lat + lat_off[g];
  for (int c = threadIdx.x; c < r; c += blockDim.x) xrow[c] = (double)src[c];
  __syncthreads();
  quantize_row_dev(xrow, r, bits, codes, &s_sh, &z_sh, red);
  for (int c = r + threadIdx.x; c < R_pad; c += blockDim.x) codes[c] = 0;
  __syncthreads();
  const size_t tok = ((size_t)b * G + g) * T_cap + t;
  pack_row_dev(codes, R_pad, bits, rows + tok * (size_t)(R_pad * bits / 8));
  if (threadIdx.x == 0) {
    scales[tok] = (float)s_sh;
    zps[tok] = (float)z_sh;
    if (scales64) scales64[tok] = s_sh;
    if (zps64) zps64[tok] = z_sh;
  }
}

__global__ void append_quant_kernel(const float* __restrict__ lat, int ld_lat, int G, int bits,
                                    const int* __restrict__ ranks, const int* __restrict__ lat_off,
                                    uint8_t* __restrict__ rows, float* __restrict__ scales,
                                    float* __restrict__ zps, double* __restrict__ scales64,
                                    int64_t* __restrict__ zps64, int R_pad, int T_cap,
                                    const int* __restrict__ t_dev) {
  pdl_enter();
  extern __shared__ double qsm[];
  append_quant_body(lat, ld_lat, G, bits, ranks, lat_off, rows, scales, zps, scales64, zps64, R_pad,
                    T_cap, *t_dev, blockIdx.x, blockIdx.y, qsm);
}

// Both sides of one layer's append in one launch: blocks [0, G_k) of each
// batch row append the key latents, [G_k, G_k + G_v) the value latents.
struct AppendSide {
  int bits, G, R_pad;
  const float* lat;  // this side's latents inside the GEMV output
  const int* ranks;
  const int* lat_off;
  void* rows;
  float *scales, *zps;
  double* scales64;
  int64_t* zps64;
};

template <typename T>
__global__ void append_kv_kernel(AppendSide k, AppendSide v, int ld_lat, int T_cap,
                                 const int* __restrict__ t_dev) {
  pdl_enter();
  extern __shared__ double qsm[];
  const bool is_k = (int)blockIdx.x < k.G;
  const AppendSide& a = is_k ? k : v;
  const int g = is_k ? (int)blockIdx.x : (int)blockIdx.x - k.G, b = blockIdx.y;
  const int t = *t_dev;
  if (a.bits == 16)
    append_raw_body<T>(a.lat, ld_lat, a.G, a.ranks, a.lat_off, reinterpret_cast<T*>(a.rows), a.R_pad,
                       T_cap, t, g, b);
  else
    append_quant_body(a.lat, ld_lat, a.G, a.bits, a.ranks, a.lat_off,
                      reinterpret_cast<uint8_t*>(a.rows), a.scales, a.zps, a.scales64, a.zps64,
                      a.R_pad, T_cap, t, g, b, qsm);
}

__global__ void quantize_rows_kernel(const double* __restrict__ x, int cols, int bits,
                                     uint8_t* __restrict__ codes, double* __restrict__ scales,
                                     int64_t* __restrict__ zps) {
  extern __shared__ double qsm[];
  double* xrow = qsm;
  double* red = qsm + cols;
  __shared__ double s_sh;
  __shared__ int64_t z_sh;
  const int row = blockIdx.x;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) xrow[c] = x[(size_t)row * cols + c];
  __syncthreads();
  quantize_row_dev(xrow, cols, bits, codes + (size_t)row * cols, &s_sh, &z_sh, red);
  if (threadIdx.x == 0) { scales[row] = s_sh; zps[row] = z_sh; }
}

__global__ void pack_rows_kernel(const uint8_t* __restrict__ codes, int cols, int bits,
                                 uint8_t* __restrict__ packed) {
  const int row = blockIdx.x;
  pack_row_dev(codes + (size_t)row * cols, cols, bits, packed + (size_t)row * (cols * bits / 8));
}

// ---------------------------------------------------------------------------
// Query absorption (attention.py:428-431 queries, folded into the key factor).
// grid (n_heads, B); fp64 RoPE of q at t, then u/w columns per rank row k.
// ---------------------------------------------------------------------------
// One CTA: head i, rank rows [32 ky, +32), batch row b.  PDL split form: the
// fp64 angles (t, theta) and the B_k slice (constant) are prepared before the
// pdl_wait() for the GEMV that produced q.
template <typename T>
__device__ __forceinline__ void query_absorb_body(const float* __restrict__ q, int ld_q, int n_heads, int dh,
                                                  int s_k, const T* __restrict__ bk, int bk_rows, int R_pad,
                                                  const double* __restrict__ theta, float scale,
                                                  const int* __restrict__ t_dev, void* __restrict__ uw,
                                                  int layout, int i, int ky, int b) {
  // qr[dh], then bs[32][dh + 1] (row pad: the bf16 layouts read one column
  // across 32 rank rows per warp, which an unpadded dh stride maps to one
  // bank), then cos/sin[dh/2] in fp64
  extern __shared__ float qa_sm[];
  float* qr = qa_sm;
  float* bs = qa_sm + dh;
  const int bstr = dh + 1;
  const int k0 = ky * 32;
  const int half = dh / 2;
  double* csn = reinterpret_cast<double*>(qa_sm + dh + 32 * (dh + 1));  // [half] cos, [half] sin
  const int g = i / s_k, p = i - g * s_k;
  const int nk = min(32, R_pad - k0);
  const double pos = (double)(*t_dev);
  const float* qh = q + (size_t)b * ld_q + (size_t)i * dh;
  for (int j = threadIdx.x; j < half; j += blockDim.x) {
    double sn, cs;
    sincos_big(pos * theta[j], &sn, &cs);  // attention.py:108-112 (fp64 angles)
    csn[j] = cs;
    csn[half + j] = sn;
  }
  if (layout == 4) {
    // replicated-B groups (GQA as its MHA-equivalent layer): the score kernel
    // reconstructs K = H B once per KV head, so only the rotated query is
    // needed: uw = float [B][n_heads][dh] = scale x RoPE_pos(q) (fp64 angles)
    pdl_wait();  // q comes from the preceding GEMV
    __syncthreads();
    float* out = reinterpret_cast<float*>(uw) + ((size_t)b * n_heads + i) * dh;
    for (int j = threadIdx.x; j < half; j += blockDim.x) {
      const double cs = csn[j], sn = csn[half + j];
      const double lo = qh[j], hi = qh[j + half];
      out[j] = scale * (float)(lo * cs - hi * sn);
      out[j + half] = scale * (float)(lo * sn + hi * cs);
    }
    return;
  }
  const int width = s_k * dh;
  const T* bg = bk + ((size_t)g * bk_rows + k0) * width + (size_t)p * dh;
  constexpr int V = 16 / (int)sizeof(T);
  if (dh % V == 0 && (width % V) == 0) {
    // 16-byte loads, all issued before the shared stores
    const int per_row = dh / V;
    for (int base = threadIdx.x; base < nk * per_row; base += 4 * blockDim.x) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = base + u * blockDim.x;
        if (idx < nk * per_row) {
          const int kk = idx / per_row, c = (idx - kk * per_row) * V;
          v[u] = *reinterpret_cast<const uint4*>(bg + (size_t)kk * width + c);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = base + u * blockDim.x;
        if (idx < nk * per_row) {
          const int kk = idx / per_row, c = (idx - kk * per_row) * V;
          float f[V];
          Vec16<T>::unpack(v[u], f);
#pragma unroll
          for (int e = 0; e < V; ++e) bs[kk * bstr + c + e] = f[e];
        }
      }
    }
  } else {
    for (int idx = threadIdx.x; idx < nk * dh; idx += blockDim.x) {
      const int kk = idx / dh, c = idx - kk * dh;
      bs[kk * bstr + c] = to_f(bg[(size_t)kk * width + c]);
    }
  }
  pdl_wait();  // q comes from the preceding GEMV
  for (int j = threadIdx.x; j < half; j += blockDim.x) {
    const double cs = csn[j], sn = csn[half + j];
    const double lo = qh[j], hi = qh[j + half];
    qr[j] = (float)(lo * cs - hi * sn);
    qr[j + half] = (float)(lo * sn + hi * cs);
  }
  __syncthreads();
  if (layout == 0) {
    float* out = reinterpret_cast<float*>(uw) + (((size_t)b * n_heads + i) * R_pad + k0) * dh;
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int kk = threadIdx.x >> 5; kk < nk; kk += nw)
      for (int j = lane; j < half; j += 32) {
        const float b1 = bs[kk * bstr + j], b2 = bs[kk * bstr + j + half];
        out[(size_t)kk * dh + j] = scale * (qr[j] * b1 + qr[j + half] * b2);
        out[(size_t)kk * dh + j + half] = scale * (qr[j + half] * b1 - qr[j] * b2);
      }
  } else {
    // bf16 [B][G][s_k*dh][R_pad]: row n = p*dh + c, c < half -> u_c, else w_{c-half}.
    // layouts 2/3: rank k stored at the K position the tcgen05 converter gives
    // code k of an int4 / int2 key row (groups of 8 / 16: k < G/2 -> 2k,
    // else 2k - G + 1), so that the dot product is unchanged
    bf16* out = reinterpret_cast<bf16*>(uw) +
                (((size_t)b * (n_heads / s_k) + g) * width + (size_t)p * dh) * R_pad;
    const int grp = layout == 2 ? 8 : (layout == 3 ? 16 : 0);
    // lane = rank row kk (nk <= 32), warp strides over the frequencies j
    const int kk = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int j = threadIdx.x >> 5; j < half && kk < nk; j += nw) {
      const float b1 = bs[kk * bstr + j], b2 = bs[kk * bstr + j + half];
      int pos = k0 + kk;
      if (grp) {
        const int i = pos % grp;
        pos = pos - i + (i < grp / 2 ? 2 * i : 2 * i - grp + 1);
      }
      out[(size_t)j * R_pad + pos] = __float2bfloat16_rn(scale * (qr[j] * b1 + qr[j + half] * b2));
      out[(size_t)(j + half) * R_pad + pos] =
          __float2bfloat16_rn(scale * (qr[j + half] * b1 - qr[j] * b2));
    }
  }
}

// grid (n_heads, ceil(R_pad / 32), B)
template <typename T>
__global__ void query_absorb_kernel(const float* __restrict__ q, int ld_q, int n_heads, int dh,
                                    int s_k, const T* __restrict__ bk, int bk_rows, int R_pad,
                                    const double* __restrict__ theta, float scale,
                                    const int* __restrict__ t_dev, void* __restrict__ uw,
                                    int layout, int split) {
  pdl_launch();
  if (!split) pdl_wait();
  query_absorb_body<T>(q, ld_q, n_heads, dh, s_k, bk, bk_rows, R_pad, theta, scale, t_dev, uw, layout,
                       blockIdx.x, blockIdx.y, blockIdx.z);
}

// The latent append (both sides) and the query absorption of one layer in one
// launch: both read only the GEMV output (and t), and the score kernel needs
// both, so one grid takes the append off the serial launch chain.  Blocks
// [0, n_abs) absorb (head, rank block, batch row); the rest append.
struct AbsorbArgs {
  const float* q;
  int ld_q, n_heads, dh, s_k;
  const void* bk;
  int bk_rows, R_pad;
  const double* theta;
  float scale;
  void* uw;
  int layout, gy;
};
template <typename T>
__global__ void append_absorb_kernel(AppendSide k, AppendSide v, int ld_lat, int T_cap,
                                     const int* __restrict__ t_dev, AbsorbArgs a, int n_abs) {
  pdl_launch();
  const int bid = blockIdx.x;
  if (bid < n_abs) {
    const int i = bid % a.n_heads, rest = bid / a.n_heads;
    query_absorb_body<T>(a.q, a.ld_q, a.n_heads, a.dh, a.s_k, reinterpret_cast<const T*>(a.bk), a.bk_rows,
                         a.R_pad, a.theta, a.scale, t_dev, a.uw, a.layout, i, rest % a.gy, rest / a.gy);
    return;
  }
  pdl_wait();  // the GEMV's latents and the step position
  extern __shared__ double qsm[];
  const int r = bid - n_abs, gs = k.G + v.G;
  const int gi = r % gs, b = r / gs;
  const bool is_k = gi < k.G;
  const AppendSide& s = is_k ? k : v;
  const int g = is_k ? gi : gi - k.G;
  const int t = *t_dev;
  if (s.bits == 16)
    append_raw_body<T>(s.lat, ld_lat, s.G, s.ranks, s.lat_off, reinterpret_cast<T*>(s.rows), s.R_pad, T_cap, t,
                       g, b);
  else
    append_quant_body(s.lat, ld_lat, s.G, s.bits, s.ranks, s.lat_off, reinterpret_cast<uint8_t*>(s.rows),
                      s.scales, s.zps, s.scales64, s.zps64, s.R_pad, T_cap, t, g, b, qsm);
}

// ---------------------------------------------------------------------------
// RoPE score, CUDA-core path.  logits[b][i][t'] = sum_j cos(t' th_j) (h.u_j)
// + sin(t' th_j) (h.w_j) -- algebraically q_rot . RoPE_t'(h B) (see
// palu_query_absorb).  Tiled for d_h = 128: a CTA owns (b, group) and walks
// 64-token tiles; per head a 64 x 128 x R GEMM in registers, then the cos/sin
// epilogue.  cos/sin come from fp64 angles per tile (attention.py:108-110).
// ---------------------------------------------------------------------------
constexpr int SC_TT = 64;  // tokens per tile
constexpr int SC_KC = 32;  // rank rows per chunk

template <typename T, int BITS>
__device__ __forceinline__ float load_latent(const void* rows, const float* scales,
                                             const float* zps, size_t tok, int R_pad, int k) {
  if constexpr (BITS == 16) {
    return to_f(reinterpret_cast<const T*>(rows)[tok * R_pad + k]);
  } else {
    const int rb = R_pad * BITS / 8;
    const uint8_t* row = reinterpret_cast<const uint8_t*>(rows) + tok * rb;
    const float code = (float)packed_code(row, rb, k, BITS);
    return (code - zps[tok]) * scales[tok];
  }
}

template <typename T, int BITS>
__global__ void __launch_bounds__(256)
rope_score_tiled_kernel(const void* __restrict__ hk, const float* __restrict__ scales,
                        const float* __restrict__ zps, int n_heads, int s_k, int G, int R_pad,
                        int T_cap, const float* __restrict__ uw, const double* __restrict__ theta,
                        const int* __restrict__ t_dev, float* __restrict__ logits, int ld_logits) {
  pdl_enter();
  constexpr int DH = 128, HALF = 64, HS = SC_TT + 4;
  extern __shared__ __align__(16) float sc_sm[];
  float (*Hs)[HS] = reinterpret_cast<float (*)[HS]>(sc_sm);                  // [SC_KC][HS]
  float (*Us)[DH] = reinterpret_cast<float (*)[DH]>(sc_sm + SC_KC * HS);     // [SC_KC][DH]
  float2 (*CSs)[HALF] = reinterpret_cast<float2 (*)[HALF]>(sc_sm + SC_KC * HS + SC_KC * DH);
  const int g = blockIdx.y, b = blockIdx.z;
  const int T_rows = *t_dev + 1;
  const int n_tiles = (T_rows + SC_TT - 1) / SC_TT;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const size_t tok_base = ((size_t)b * G + g) * T_cap;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int t0 = tile * SC_TT;
    __syncthreads();
    for (int idx = tid; idx < SC_TT * HALF; idx += blockDim.x) {
      const int tt = idx / HALF, j = idx - tt * HALF;
      double sn, cs;
      sincos_big((double)(t0 + tt) * theta[j], &sn, &cs);
      CSs[tt][j] = make_float2((float)cs, (float)sn);
    }
    for (int p = 0; p < s_k; ++p) {
      const int head = g * s_k + p;
      const float* uwh = uw + ((size_t)b * n_heads + head) * R_pad * DH;
      float acc[4][8];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[a][c] = 0.f;
      for (int k0 = 0; k0 < R_pad; k0 += SC_KC) {
        __syncthreads();
        for (int idx = tid; idx < SC_KC * SC_TT; idx += blockDim.x) {
          const int tt = idx / SC_KC, kk = idx - tt * SC_KC;
          const int t = t0 + tt;
          Hs[kk][tt] = (t < T_rows) ? load_latent<T, BITS>(hk, scales, zps, tok_base + t, R_pad, k0 + kk)
                                    : 0.f;
        }
        for (int idx = tid; idx < SC_KC * DH / 4; idx += blockDim.x) {
          const int kk = idx / (DH / 4), c4 = idx - kk * (DH / 4);
          reinterpret_cast<float4*>(&Us[kk][0])[c4] =
              reinterpret_cast<const float4*>(uwh + (size_t)(k0 + kk) * DH)[c4];
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < SC_KC; ++kk) {
          const float4 a = reinterpret_cast<const float4*>(&Hs[kk][0])[ty];
          const float4 u = reinterpret_cast<const float4*>(&Us[kk][0])[tx];
          const float4 w = reinterpret_cast<const float4*>(&Us[kk][HALF])[tx];
          const float av[4] = {a.x, a.y, a.z, a.w};
          const float bv[8] = {u.x, u.y, u.z, u.w, w.x, w.y, w.z, w.w};
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
        }
      }
      // epilogue: sum_j cos_j * h.u_j + sin_j * h.w_j over this thread's 4 pairs
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int tt = ty * 4 + r;
        float v = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float2 cs = CSs[tt][tx * 4 + c];
          v = fmaf(cs.x, acc[r][c], v);
          v = fmaf(cs.y, acc[r][c + 4], v);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        const int t = t0 + tt;
        if (tx == 0 && t < T_rows) logits[((size_t)b * n_heads + head) * ld_logits + t] = v;
      }
    }
  }
}

// Generic (any even d_h) score: one thread per (token, head).  Used for the
// small reference-test shapes; the tiled/tcgen05 kernels cover d_h = 128.
template <typename T, int BITS>
__global__ void rope_score_generic_kernel(const void* __restrict__ hk, const float* __restrict__ scales,
                                          const float* __restrict__ zps, int n_heads, int dh,
                                          int s_k, int G, int R_pad, int T_cap,
                                          const float* __restrict__ uw,
                                          const double* __restrict__ theta,
                                          const int* __restrict__ t_dev, float* __restrict__ logits,
                                          int ld_logits) {
  pdl_enter();
  const int b = blockIdx.z, head = blockIdx.y;
  const int g = head / s_k;
  const int T_rows = *t_dev + 1;
  const int half = dh / 2;
  const float* uwh = uw + ((size_t)b * n_heads + head) * R_pad * dh;
  const size_t tok_base = ((size_t)b * G + g) * T_cap;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T_rows; t += gridDim.x * blockDim.x) {
    float v = 0.f;
    for (int j = 0; j < half; ++j) {
      float a = 0.f, w = 0.f;
      for (int k = 0; k < R_pad; ++k) {
        const float h = load_latent<T, BITS>(hk, scales, zps, tok_base + t, R_pad, k);
        a = fmaf(h, uwh[(size_t)k * dh + j], a);
        w = fmaf(h, uwh[(size_t)k * dh + j + half], w);
      }
      double sn, cs;
      sincos_big((double)t * theta[j], &sn, &cs);
      v += (float)cs * a + (float)sn * w;
    }
    logits[((size_t)b * n_heads + head) * ld_logits + t] = v;
  }
}

// ---------------------------------------------------------------------------
// Softmax + value (attention.py:445-446, 350-362).  Split-T partials, then a
// fixed-order merge (deterministic).
// ---------------------------------------------------------------------------
constexpr int SV_HP = 4;           // heads per pass
constexpr int SV_MAX_CHUNK = 8192;  // tokens per chunk cap (smem)

struct SvPartial {
  float* m;       // [B][n][NC]
  float* l;       // [B][n][NC]
  float* ctx;     // [B][n][NC][R_pad]
  unsigned* cnt;  // [B][G] arrival tickets (self-resetting)
};

__host__ __device__ inline SvPartial sv_carve(void* ws, int B, int n, int R_pad, int NC) {
  // tickets first: their offset must not depend on R_pad (layers may differ)
  SvPartial p;
  p.cnt = reinterpret_cast<unsigned*>(ws);
  float* f = reinterpret_cast<float*>(ws) + (((size_t)B * n + 31) & ~size_t(31));
  p.m = f;
  p.l = f + (size_t)B * n * NC;
  p.ctx = f + 2 * (size_t)B * n * NC;
  return p;
}

// Fixed-order merge of a group's NC chunk partials (flash-decoding combine)
// by one CTA of 8 warps: ctx = sum_c e^(m_c - M) ctx_c / sum_c e^(m_c - M) l_c.
// Warp w takes chunks c = w (mod 8) for every head of the group, lanes take
// columns; the 8 warp sums are added in a fixed order (deterministic).
__device__ void sv_merge_group(const SvPartial& part, size_t head_base, int hp, int NC, int R_pad,
                               int r, float* const* dst, float* sm, int tid) {
  constexpr int NW = 8;
  const int warp = tid >> 5, lane = tid & 31;
  float* wsm = sm;                     // [hp][NC] chunk weights
  float* inv_l = sm + SV_HP * NC;      // [hp]
  float* red = inv_l + SV_HP;          // [NW][hp][R_pad]
  if (warp < hp) {
    const size_t base = (head_base + warp) * NC;
    float M = -INFINITY;
    for (int c = lane; c < NC; c += 32) M = fmaxf(M, part.m[base + c]);
    M = warp_reduce(M, [](float a, float d) { return fmaxf(a, d); });
    float L = 0.f;
    for (int c = lane; c < NC; c += 32) {
      const float l = part.l[base + c];
      const float w = (l > 0.f) ? expf(part.m[base + c] - M) : 0.f;
      wsm[warp * NC + c] = w;
      L += w * l;
    }
    L = warp_reduce(L, [](float a, float d) { return a + d; });
    if (lane == 0) inv_l[warp] = 1.f / L;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
  for (int h = 0; h < hp; ++h) {
    const float* src = part.ctx + (head_base + h) * NC * (size_t)R_pad;
    for (int col0 = 0; col0 < r; col0 += 32 * 4) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int c = warp; c < NC; c += NW) {
        const float w = wsm[h * NC + c];
        const float* row = src + (size_t)c * R_pad + col0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int col = lane + 32 * k;
          if (col0 + col < r) acc[k] = fmaf(w, row[col], acc[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int col = col0 + lane + 32 * k;
        if (col < r) red[((size_t)warp * SV_HP + h) * R_pad + col] = acc[k];
      }
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
  for (int idx = tid; idx < hp * r; idx += NW * 32) {
    const int h = idx / r, col = idx - h * r;
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) v += red[((size_t)w * SV_HP + h) * R_pad + col];
    dst[h][col] = v * inv_l[h];
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
}

// ---------------------------------------------------------------------------
// Rope-off score (attention.py:380-388, both fusions active): the key-side
// reconstruction is absorbed into wq_fused offline, so per head i of key group
// g the logits are a latent-cache GEMV
//   logit[t] = (H_k[g][t] . q_lat_i) / sqrt(d_h),   q_lat_i = x @ wq_fused[:, q_off[i]:]
// CUDA-core version for every dtype / bit width: one warp per (token, group),
// lanes over the rank, the group's s heads reduced together.
template <typename T, int BITS>
__global__ void __launch_bounds__(256)
latent_score_kernel(const void* __restrict__ hk, const float* __restrict__ scales,
                    const float* __restrict__ zps, int n_heads, int s_k, int G, int R_pad,
                    int T_cap, const float* __restrict__ y, int ld_y, const int* __restrict__ q_off,
                    const int* __restrict__ ranks, float scale, const int* __restrict__ t_dev,
                    float* __restrict__ logits, int ld_logits) {
  pdl_enter();
  const int g = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T_rows = *t_dev + 1;
  const int r = ranks[g];
  const size_t tok_base = ((size_t)b * G + g) * T_cap;
  for (int t = blockIdx.x * 8 + warp; t < T_rows; t += gridDim.x * 8) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int k = lane; k < r; k += 32) {
      const float h = load_latent<T, BITS>(hk, scales, zps, tok_base + t, R_pad, k);
#pragma unroll
      for (int p = 0; p < 8; ++p)
        if (p < s_k) acc[p] = fmaf(h, y[(size_t)b * ld_y + q_off[g * s_k + p] + k], acc[p]);
    }
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      if (p < s_k) {
        const float v = warp_reduce(acc[p], [](float a, float c) { return a + c; });
        if (lane == 0) logits[((size_t)b * n_heads + g * s_k + p) * ld_logits + t] = v * scale;
      }
    }
  }
}

template <typename T, int BITS>
struct SvSeg {
  static constexpr bool RAW = BITS == 16;
  // raw: 16 B; packed: one 32-bit word, or 12 B (= 32 codes) for 3-bit rows
  static constexpr int BYTES = RAW ? 16 : (BITS == 3 ? 12 : 4);
  static constexpr int COLV = RAW ? 16 / (int)sizeof(T) : (BITS == 3 ? 32 : 32 / BITS);
  static __device__ __forceinline__ void unpack(const uint4& v, float* f) {
    if constexpr (RAW) {
      Vec16<T>::unpack(v, f);
    } else if constexpr (BITS == 3) {
      const uint32_t w[3] = {v.x, v.y, v.z};
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int bit = 3 * e, wi = bit >> 5, off = bit & 31;
        uint32_t c = w[wi] >> off;
        if (off > 29) c |= w[wi + 1] << (32 - off);
        f[e] = (float)(c & 7u);
      }
    } else {
      const uint32_t w = v.x;
#pragma unroll
      for (int e = 0; e < COLV; ++e) f[e] = (float)((w >> (e * BITS)) & ((1u << BITS) - 1u));
    }
  }
  static __device__ __forceinline__ uint4 load(const uint8_t* p) {
    if constexpr (RAW) {
      return ldg_stream(p);
    } else {
      const uint32_t* q = reinterpret_cast<const uint32_t*>(p);
      uint4 r;
      r.x = __ldg(q);
      r.y = BITS == 3 ? __ldg(q + 1) : 0u;
      r.z = BITS == 3 ? __ldg(q + 2) : 0u;
      r.w = 0u;
      return r;
    }
  }
};

__device__ __forceinline__ uint32_t sv_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void sv_mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = sv_smem_u32(bar);
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  }
}

constexpr int SV_CONSUMERS = 8;              // consumer warps
constexpr int SV_BLOCK = (SV_CONSUMERS + 1) * 32;
constexpr int SV_STAGE_BYTES = 16384;
constexpr int SV_NSTAGE = 4;

// Split-T softmax + value pass.  The chunk's H_v rows are contiguous in HBM,
// so one elected producer lane streams them with 1-D TMA bulk copies
// (cp.async.bulk, 16 KB stages, 4 in flight) while 8 consumer warps first
// compute the per-head softmax statistics and then reduce the staged rows
// out of shared memory.  Lr lanes cover a row (NSEG segments each); rows are
// spread over warps.  Quantised rows use ctx = sum_t (p_t s_t) code_t -
// sum_t p_t s_t z_t with the z term folded into the statistics pass.
template <typename T, int BITS, int NSEG>
__global__ void __launch_bounds__(SV_BLOCK)
softmax_value_partial_kernel(const void* __restrict__ hv, const float* __restrict__ scales,
                             const float* __restrict__ zps, int n_heads, int s_v, int G, int R_pad,
                             int T_cap, const float* __restrict__ logits, int ld_logits,
                             int n_planes, long long plane, const int* __restrict__ t_dev, int NC,
                             int Lr, SvPartial part, const int* __restrict__ ranks_v,
                             const int* __restrict__ o_off, float* __restrict__ ctx_out,
                             int ld_ctx) {
  pdl_enter();
  using Seg = SvSeg<T, BITS>;
  constexpr int COLV = Seg::COLV;
  extern __shared__ __align__(128) uint8_t sv_raw[];
  uint8_t* ring = sv_raw;                                            // SV_NSTAGE x 16 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + SV_NSTAGE * SV_STAGE_BYTES);
  uint64_t* empty = full + SV_NSTAGE;
  float* ps = reinterpret_cast<float*>(empty + SV_NSTAGE);           // [SV_HP][clen]
  __shared__ float zsum[SV_HP];
  const int c = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
  const int T_rows = *t_dev + 1;
  int clen = (T_rows + NC - 1) / NC;
  clen = (clen + 7) & ~7;
  const int c0 = min(T_rows, c * clen);
  const int c1 = min(T_rows, c0 + clen);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t tok_base = ((size_t)b * G + g) * T_cap;
  const int row_bytes = Seg::RAW ? R_pad * (int)sizeof(T) : R_pad * BITS / 8;
  const int segs = row_bytes / Seg::BYTES;
  const int RW = 32 / Lr;  // rows per warp step
  const int rs = lane / Lr, sb = lane - rs * Lr;
  const int stage_rows = SV_STAGE_BYTES / row_bytes;
  const int n_loads = (c1 - c0 + stage_rows - 1) / stage_rows;
  const uint8_t* src0 = reinterpret_cast<const uint8_t*>(hv) + (tok_base + c0) * (size_t)row_bytes;

  if (tid == 0) {
    for (int st = 0; st < SV_NSTAGE; ++st) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sv_smem_u32(&full[st])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sv_smem_u32(&empty[st])),
                   "r"(SV_CONSUMERS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  int load_ctr = 0;  // producer and consumers walk the same stage sequence
  for (int p0 = 0; p0 < s_v; p0 += SV_HP) {
    const int hp = min(SV_HP, s_v - p0);
    if (warp == SV_CONSUMERS) {
      // ---------------- producer: stream the chunk rows ----------------
      // the ring doubles as the consumers' reduction buffer: wait until the
      // previous head pass has finished with it
      if (p0 > 0) asm volatile("bar.sync 2, %0;" ::"r"(SV_BLOCK) : "memory");
      if (lane == 0) {
        for (int l = 0; l < n_loads; ++l) {
          const int ctr = load_ctr + l;
          const int st = ctr % SV_NSTAGE;
          sv_mbar_wait(&empty[st], ((ctr / SV_NSTAGE) & 1) ^ 1);
          const int r0 = l * stage_rows;
          const int nr = min(stage_rows, (c1 - c0) - r0);
          const uint32_t bytes = (uint32_t)(nr * row_bytes);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                           sv_smem_u32(&full[st])),
                       "r"(bytes)
                       : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  sv_smem_u32(ring + st * SV_STAGE_BYTES)),
              "l"(src0 + (size_t)r0 * row_bytes), "r"(bytes), "r"(sv_smem_u32(&full[st]))
              : "memory");
        }
      }
      load_ctr += n_loads;
      continue;
    }
    // (1) softmax statistics of the chunk for the hp heads, all 8 consumer
    // warps over tokens (independent loads, block reductions)
    __shared__ float red_m[SV_CONSUMERS][SV_HP], red_l[SV_CONSUMERS][SV_HP],
        red_z[SV_CONSUMERS][SV_HP];
    __shared__ float m_sh[SV_HP];
    {
      const float* lg[SV_HP];
#pragma unroll
      for (int h = 0; h < SV_HP; ++h)
        lg[h] = logits + ((size_t)b * n_heads + g * s_v + p0 + min(h, hp - 1)) * ld_logits;
      float m[SV_HP];
#pragma unroll
      for (int h = 0; h < SV_HP; ++h) m[h] = -INFINITY;
      for (int t = c0 + tid; t < c1; t += SV_CONSUMERS * 32) {
        float v[SV_HP];
#pragma unroll
        for (int h = 0; h < SV_HP; ++h) {
          v[h] = lg[h][t];
          for (int pl = 1; pl < n_planes; ++pl) v[h] += lg[h][pl * plane + t];
        }
#pragma unroll
        for (int h = 0; h < SV_HP; ++h) {
          ps[h * clen + (t - c0)] = v[h];
          m[h] = fmaxf(m[h], v[h]);
        }
      }
#pragma unroll
      for (int h = 0; h < SV_HP; ++h) {
        m[h] = warp_reduce(m[h], [](float x, float y) { return fmaxf(x, y); });
        if (lane == 0) red_m[warp][h] = m[h];
      }
      asm volatile("bar.sync 1, %0;" ::"r"(SV_CONSUMERS * 32) : "memory");
      if (tid < SV_HP) {
        float mm = red_m[0][tid];
        for (int w = 1; w < SV_CONSUMERS; ++w) mm = fmaxf(mm, red_m[w][tid]);
        m_sh[tid] = mm;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(SV_CONSUMERS * 32) : "memory");
#pragma unroll
      for (int h = 0; h < SV_HP; ++h) m[h] = m_sh[h];
      float l[SV_HP], zs[SV_HP];
#pragma unroll
      for (int h = 0; h < SV_HP; ++h) l[h] = zs[h] = 0.f;
      for (int t = c0 + tid; t < c1; t += SV_CONSUMERS * 32) {
        float sc = 1.f, zp = 0.f;
        if constexpr (!Seg::RAW) {
          sc = scales[tok_base + t];
          zp = zps[tok_base + t];
        }
#pragma unroll
        for (int h = 0; h < SV_HP; ++h) {
          float e = expf(ps[h * clen + (t - c0)] - m[h]);
          l[h] += e;
          if constexpr (!Seg::RAW) {
            zs[h] = fmaf(e * sc, zp, zs[h]);
            e *= sc;
          }
          ps[h * clen + (t - c0)] = e;
        }
      }
#pragma unroll
      for (int h = 0; h < SV_HP; ++h) {
        l[h] = warp_reduce(l[h], [](float x, float y) { return x + y; });
        zs[h] = warp_reduce(zs[h], [](float x, float y) { return x + y; });
        if (lane == 0) {
          red_l[warp][h] = l[h];
          red_z[warp][h] = zs[h];
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(SV_CONSUMERS * 32) : "memory");
      if (tid < hp) {
        float ll = 0.f, zz = 0.f;
        for (int w = 0; w < SV_CONSUMERS; ++w) {
          ll += red_l[w][tid];
          zz += red_z[w][tid];
        }
        const size_t pi = ((size_t)b * n_heads + g * s_v + p0 + tid) * NC + c;
        part.m[pi] = (c0 < c1) ? m_sh[tid] : -INFINITY;
        part.l[pi] = (c0 < c1) ? ll : 0.f;
        zsum[tid] = zz;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(SV_CONSUMERS * 32) : "memory");
    // (2) reduce the staged rows (packed FFMA2; probabilities of all SV_HP
    // head slots are read unconditionally -- slots >= hp hold stale values
    // whose accumulators are never stored)
    static_assert(COLV % 2 == 0, "COLV must be even");
    float2 acc[SV_HP][NSEG][COLV / 2];
#pragma unroll
    for (int h = 0; h < SV_HP; ++h)
#pragma unroll
      for (int q = 0; q < NSEG; ++q)
#pragma unroll
        for (int e = 0; e < COLV / 2; ++e) acc[h][q][e] = make_float2(0.f, 0.f);
    const int my_first = warp * RW + rs;
    const int row_step = SV_CONSUMERS * RW;
    for (int l = 0; l < n_loads; ++l) {
      const int ctr = load_ctr + l;
      const int st = ctr % SV_NSTAGE;
      sv_mbar_wait(&full[st], (ctr / SV_NSTAGE) & 1);
      const int r0 = l * stage_rows;
      const int nr = min(stage_rows, (c1 - c0) - r0);
      const uint8_t* sbase = ring + st * SV_STAGE_BYTES;
      const float* pst = ps + r0;
      for (int r = my_first; r < nr; r += row_step) {
        const uint8_t* row = sbase + (size_t)r * row_bytes;
        float pv[SV_HP];
#pragma unroll
        for (int h = 0; h < SV_HP; ++h) pv[h] = pst[h * clen + r];
#pragma unroll
        for (int q = 0; q < NSEG; ++q) {
          const int sg = sb + q * Lr;
          if (NSEG == 1 || sg < segs) {
            uint4 v;
            if constexpr (Seg::BYTES == 16) {
              v = *reinterpret_cast<const uint4*>(row + sg * 16);
            } else {
              const uint32_t* w = reinterpret_cast<const uint32_t*>(row + sg * Seg::BYTES);
              v.x = w[0];
              v.y = Seg::BYTES > 4 ? w[1] : 0u;
              v.z = Seg::BYTES > 8 ? w[2] : 0u;
              v.w = 0u;
            }
            float f[COLV];
            Seg::unpack(v, f);
#pragma unroll
            for (int h = 0; h < SV_HP; ++h) {
              const float2 p2 = make_float2(pv[h], pv[h]);
#pragma unroll
              for (int e = 0; e < COLV / 2; ++e)
                acc[h][q][e] = ffma2_f(p2, make_float2(f[2 * e], f[2 * e + 1]), acc[h][q][e]);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sv_smem_u32(&empty[st]))
                     : "memory");
    }
    load_ctr += n_loads;
    // (3) reduce: across row slots inside the warp, then across warps
#pragma unroll
    for (int h = 0; h < SV_HP; ++h)
#pragma unroll
      for (int q = 0; q < NSEG; ++q)
#pragma unroll
        for (int e = 0; e < COLV / 2; ++e)
          for (int o = Lr; o < 32; o <<= 1) {
            acc[h][q][e].x += __shfl_xor_sync(0xffffffffu, acc[h][q][e].x, o);
            acc[h][q][e].y += __shfl_xor_sync(0xffffffffu, acc[h][q][e].y, o);
          }
    asm volatile("bar.sync 1, %0;" ::"r"(SV_CONSUMERS * 32) : "memory");
    float* red = reinterpret_cast<float*>(ring);  // all stages consumed: reuse
    if (rs == 0) {
#pragma unroll
      for (int h = 0; h < SV_HP; ++h)
#pragma unroll
        for (int q = 0; q < NSEG; ++q) {
          const int sg = sb + q * Lr;
          if (sg < segs)
#pragma unroll
            for (int e = 0; e < COLV / 2; ++e) {
              red[((size_t)warp * SV_HP + h) * R_pad + sg * COLV + 2 * e] = acc[h][q][e].x;
              red[((size_t)warp * SV_HP + h) * R_pad + sg * COLV + 2 * e + 1] = acc[h][q][e].y;
            }
        }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(SV_CONSUMERS * 32) : "memory");
    for (int idx = tid; idx < hp * R_pad; idx += SV_CONSUMERS * 32) {
      const int h = idx / R_pad, col = idx - h * R_pad;
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < SV_CONSUMERS; ++w) v += red[((size_t)w * SV_HP + h) * R_pad + col];
      if constexpr (!Seg::RAW) v -= zsum[h];
      const int head = g * s_v + p0 + h;
      part.ctx[(((size_t)b * n_heads + head) * NC + c) * R_pad + col] = v;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(SV_CONSUMERS * 32) : "memory");
    if (p0 + SV_HP < s_v) asm volatile("bar.arrive 2, %0;" ::"r"(SV_BLOCK) : "memory");
  }
  if (warp == SV_CONSUMERS) return;
  // The last CTA of this (sequence, group) to finish merges the chunks.
  __shared__ unsigned ticket_sh;
  __threadfence();
  asm volatile("bar.sync 1, %0;" ::"r"(SV_CONSUMERS * 32) : "memory");
  if (tid == 0) ticket_sh = atomicAdd(&part.cnt[(size_t)b * G + g], 1u);
  asm volatile("bar.sync 1, %0;" ::"r"(SV_CONSUMERS * 32) : "memory");
  if (ticket_sh != (unsigned)(NC - 1)) return;
  __threadfence();
  const int r = ranks_v[g];
  for (int p0 = 0; p0 < s_v; p0 += SV_HP) {
    const int hp = min(SV_HP, s_v - p0);
    float* dst[SV_HP];
#pragma unroll
    for (int h = 0; h < SV_HP; ++h)
      dst[h] = ctx_out + (size_t)b * ld_ctx + o_off[g * s_v + p0 + min(h, hp - 1)];
    sv_merge_group(part, (size_t)b * n_heads + g * s_v + p0, hp, NC, R_pad, r, dst,
                   reinterpret_cast<float*>(ring), tid);
  }
  if (tid == 0) part.cnt[(size_t)b * G + g] = 0u;  // ready for the next launch
}

__global__ void advance_kernel(int* t_dev) { pdl_enter(); *t_dev += 1; }

// Comparator support (flashinfer trtllm-gen decode inside the uncompressed
// step graph): RoPE + append row t into an HND paged bf16 cache
// [page][2][n][P][d_h] (page = b * pages_per_seq + t / P), rotated q as bf16
// [B][n][d_h] for the attention kernel.
// qkv: fp32 [B][n dh + 2 n_kv dh] (q | k | v; GQA: n_kv < n KV heads); block
// (i, b) rotates query head i and, for i < n_kv, appends KV head i.
__global__ void dense_append_paged_kernel(const float* __restrict__ qkv, int n_heads, int n_kv, int dh,
                                          bf16* __restrict__ kv, int P, int pages_per_seq,
                                          const double* __restrict__ theta,
                                          const int* __restrict__ t_dev, bf16* __restrict__ qout) {
  pdl_enter();
  const int i = blockIdx.x, b = blockIdx.y;
  const int d = n_heads * dh, dkv = n_kv * dh, half = dh / 2;
  const int t = *t_dev;
  const float* row = qkv + (size_t)b * (d + 2 * dkv);
  const float* q = row + (size_t)i * dh;
  const float* k = row + d + (size_t)i * dh;
  const float* v = row + d + dkv + (size_t)i * dh;
  const bool kv_head = i < n_kv;
  const size_t page = (size_t)b * pages_per_seq + t / P;
  bf16* krow = kv + (((page * 2 + 0) * n_kv + i) * P + t % P) * dh;
  bf16* vrow = kv + (((page * 2 + 1) * n_kv + i) * P + t % P) * dh;
  bf16* qo = qout + ((size_t)b * n_heads + i) * dh;
  for (int j = threadIdx.x; j < half; j += blockDim.x) {
    double sn, cs;
    sincos_big((double)t * theta[j], &sn, &cs);
    const double qlo = q[j], qhi = q[j + half];
    qo[j] = __float2bfloat16_rn((float)(qlo * cs - qhi * sn));
    qo[j + half] = __float2bfloat16_rn((float)(qlo * sn + qhi * cs));
    if (kv_head) {
      const double klo = k[j], khi = k[j + half];
      krow[j] = __float2bfloat16_rn((float)(klo * cs - khi * sn));
      krow[j + half] = __float2bfloat16_rn((float)(klo * sn + khi * cs));
    }
  }
  if (kv_head)
    for (int j = threadIdx.x; j < dh; j += blockDim.x) vrow[j] = __float2bfloat16_rn(v[j]);
}

__global__ void cast_bf16_f32_kernel(const bf16* __restrict__ src, float* __restrict__ dst, int n) {
  pdl_enter();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = __bfloat162float(src[i]);
}

// ---------------------------------------------------------------------------
// Uncompressed baseline K0 (reference_decode, attention.py:133-168)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void dense_append_kernel(const float* __restrict__ qkv, int n_heads, int dh,
                                    T* __restrict__ kc, T* __restrict__ vc, int T_cap,
                                    const double* __restrict__ theta, const int* __restrict__ t_dev,
                                    float* __restrict__ qrot) {
  const int i = blockIdx.x, b = blockIdx.y;
  const int d = n_heads * dh, half = dh / 2;
  const int t = *t_dev;
  const float* q = qkv + (size_t)b * 3 * d + (size_t)i * dh;
  const float* k = q + d;
  const float* v = q + 2 * d;
  const size_t row = (((size_t)b * n_heads + i) * T_cap + t) * dh;
  for (int j = threadIdx.x; j < half; j += blockDim.x) {
    double sn, cs;
    sincos_big((double)t * theta[j], &sn, &cs);
    const double klo = k[j], khi = k[j + half], qlo = q[j], qhi = q[j + half];
    kc[row + j] = from_f<T>((float)(klo * cs - khi * sn));
    kc[row + j + half] = from_f<T>((float)(klo * sn + khi * cs));
    float* qo = qrot + ((size_t)b * n_heads + i) * dh;
    qo[j] = (float)(qlo * cs - qhi * sn);
    qo[j + half] = (float)(qlo * sn + qhi * cs);
  }
  for (int j = threadIdx.x; j < dh; j += blockDim.x) vc[row + j] = from_f<T>(v[j]);
}

// one warp per token: logit = k . q / sqrt(dh); chunk partials like K3
template <typename T>
__global__ void __launch_bounds__(256)
dense_partial_kernel(int n_heads, int dh, const T* __restrict__ kc, const T* __restrict__ vc,
                     int T_cap, const int* __restrict__ t_dev, const float* __restrict__ qrot,
                     int NC, SvPartial part) {
  extern __shared__ float dsm[];  // q[dh], lg[clen], acc[8][dh], red
  const int c = blockIdx.x, i = blockIdx.y, b = blockIdx.z;
  const int T_rows = *t_dev + 1;
  int clen = (T_rows + NC - 1) / NC;
  clen = (clen + 7) & ~7;
  const int c0 = c * clen, c1 = min(T_rows, c0 + clen);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* qs = dsm;
  float* lg = dsm + dh;
  float* accs = lg + clen;  // [8][dh]
  float* red = accs + 8 * dh;
  const float scale = rsqrtf((float)dh);
  for (int j = tid; j < dh; j += blockDim.x) qs[j] = qrot[((size_t)b * n_heads + i) * dh + j];
  __syncthreads();
  const size_t base = ((size_t)b * n_heads + i) * T_cap;
  float m = -INFINITY;
  for (int t = c0 + warp; t < c1; t += 8) {
    const T* kr = kc + (base + t) * dh;
    float s = 0.f;
    for (int j = lane; j < dh; j += 32) s = fmaf(to_f(kr[j]), qs[j], s);
    s = warp_reduce(s, [](float a, float e) { return a + e; });
    s *= scale;
    if (lane == 0) lg[t - c0] = s;
    m = fmaxf(m, s);
  }
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = red[0];
  for (int w = 1; w < 8; ++w) m = fmaxf(m, red[w]);
  float l = 0.f;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int t = c0 + warp; t < c1; t += 8) {
    const float p = expf(lg[t - c0] - m);
    l += p;
    const T* vr = vc + (base + t) * dh;
    for (int j = lane, q = 0; j < dh && q < 4; j += 32, ++q) acc[q] = fmaf(p, to_f(vr[j]), acc[q]);
  }
  for (int j = lane, q = 0; j < dh && q < 4; j += 32, ++q) accs[warp * dh + j] = acc[q];
  __syncthreads();
  if (lane == 0) red[8 + warp] = l;
  __syncthreads();
  const size_t pi = ((size_t)b * n_heads + i) * NC + c;
  if (tid == 0) {
    float ll = 0.f;
    for (int w = 0; w < 8; ++w) ll += red[8 + w];
    part.m[pi] = (c0 < c1) ? m : -INFINITY;
    part.l[pi] = (c0 < c1) ? ll : 0.f;
  }
  for (int j = tid; j < dh; j += blockDim.x) {
    float v = 0.f;
    for (int w = 0; w < 8; ++w) v += accs[w * dh + j];
    part.ctx[pi * dh + j] = v;
  }
}

__global__ void dense_combine_kernel(int n_heads, int dh, int NC, SvPartial part,
                                     float* __restrict__ attn) {
  const int i = blockIdx.x, b = blockIdx.y;
  const size_t base = ((size_t)b * n_heads + i) * NC;
  float M = -INFINITY;
  for (int c = 0; c < NC; ++c) M = fmaxf(M, part.m[base + c]);
  float L = 0.f;
  for (int c = 0; c < NC; ++c)
    if (part.l[base + c] > 0.f) L += expf(part.m[base + c] - M) * part.l[base + c];
  for (int j = threadIdx.x; j < dh; j += blockDim.x) {
    float v = 0.f;
    for (int c = 0; c < NC; ++c)
      if (part.l[base + c] > 0.f) v = fmaf(expf(part.m[base + c] - M), part.ctx[(base + c) * dh + j], v);
    attn[(size_t)b * n_heads * dh + (size_t)i * dh + j] = v / L;
  }
}

}  // namespace palu

namespace palu {
static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename T, int BITS>
static void launch_score(const void* hk, const float* scales, const float* zps, int B,
                         int n_heads, int head_dim, int s_k, int G, int R_pad, int T_cap,
                         const float* uw, const double* theta, const int* t_dev, float* logits,
                         int ld_logits, cudaStream_t st) {
  if (head_dim == 128 && R_pad % SC_KC == 0) {
    const int tiles = (T_cap + SC_TT - 1) / SC_TT;
    int px = (2 * sm_count() + G * B - 1) / (G * B);
    px = px < 1 ? 1 : (px > tiles ? tiles : px);
    dim3 grid(px, G, B);
    const size_t smem = sizeof(float) * (SC_KC * (SC_TT + 4) + SC_KC * 128 + 2 * SC_TT * 64);
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(rope_score_tiled_kernel<T, BITS>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr_set = true;
    }
    (void)(launch_k(rope_score_tiled_kernel<T, BITS>, dim3(grid), dim3(256), smem, st, hk, scales, zps, n_heads, s_k, G, R_pad,
                                                           T_cap, uw, theta, t_dev, logits,
                                                           ld_logits));
  } else {
    const int blocks = (T_cap + 127) / 128;
    dim3 grid(blocks < 64 ? blocks : 64, n_heads, B);
    (void)(launch_k(rope_score_generic_kernel<T, BITS>, dim3(grid), dim3(128), 0, st, hk, scales, zps, n_heads, head_dim,
                                                             s_k, G, R_pad, T_cap, uw, theta,
                                                             t_dev, logits, ld_logits));
  }
}

template <typename T, int BITS, int NSEG>
static int launch_sv_n(const void* hv, const float* scales, const float* zps, int B, int n_heads,
                       int s_v, int G, int R_pad, const int* ranks_v, const int* o_off, int T_cap,
                       const float* logits, int ld_logits, int n_planes, long long plane,
                       const int* t_dev, int NC, int Lr, SvPartial part, float* ctx, int ld_ctx,
                       cudaStream_t st) {
  int clen = (T_cap + NC - 1) / NC;
  clen = (clen + 7) & ~7;
  PALU_REQUIRE(clen <= SV_MAX_CHUNK, "palu_softmax_value: raise n_chunks (chunk %d > %d)", clen,
               SV_MAX_CHUNK);
  const size_t ring = (size_t)SV_NSTAGE * SV_STAGE_BYTES;
  const size_t red = (size_t)SV_CONSUMERS * SV_HP * R_pad * sizeof(float);
  PALU_REQUIRE(red <= ring, "palu_softmax_value: R_pad %d too large", R_pad);
  const size_t smem = ring + 2 * SV_NSTAGE * sizeof(uint64_t) + (size_t)SV_HP * clen * sizeof(float);
  static bool attr = false;
  if (!attr) {
    PALU_CK(cudaFuncSetAttribute(softmax_value_partial_kernel<T, BITS, NSEG>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  dim3 grid(NC, G, B);
  PALU_REQUIRE(sizeof(float) * ((size_t)SV_HP * NC + SV_HP + (size_t)8 * SV_HP * R_pad) <= ring,
               "palu_softmax_value: too many chunks for the merge buffer");
  PALU_CK(launch_k(softmax_value_partial_kernel<T, BITS, NSEG>, dim3(grid), dim3(SV_BLOCK), smem, st, 
      hv, scales, zps, n_heads, s_v, G, R_pad, T_cap, logits, ld_logits, n_planes, plane, t_dev, NC,
      Lr, part, ranks_v, o_off, ctx, ld_ctx));
  PALU_LAUNCHED();
  return PALU_OK;
}

template <typename T, int BITS>
static int launch_sv(const void* hv, const float* scales, const float* zps, int B, int n_heads,
                     int s_v, int G, int R_pad, const int* ranks_v, const int* o_off, int T_cap,
                     const float* logits, int ld_logits, int n_planes, long long plane,
                     const int* t_dev, int NC, SvPartial part, float* ctx, int ld_ctx,
                     cudaStream_t st) {
  using Seg = SvSeg<T, BITS>;
  const int row_bytes = Seg::RAW ? R_pad * (int)sizeof(T) : R_pad * BITS / 8;
  PALU_REQUIRE(row_bytes % Seg::BYTES == 0 && row_bytes % 16 == 0 && row_bytes <= SV_STAGE_BYTES,
               "palu_softmax_value: R_pad=%d unsupported", R_pad);
  const int segs = row_bytes / Seg::BYTES;
  const int nseg = (segs + 31) / 32;
  int lr = 1;
  while (lr < (segs + nseg - 1) / nseg) lr <<= 1;
  PALU_REQUIRE(nseg <= 4 && lr <= 32, "palu_softmax_value: R_pad=%d unsupported (segments %d)",
               R_pad, segs);
#define SVN(N_) return launch_sv_n<T, BITS, N_>(hv, scales, zps, B, n_heads, s_v, G, R_pad, ranks_v, \
                                                 o_off, T_cap, logits, ld_logits, n_planes, plane, \
                                                 t_dev, NC, lr, part, ctx, ld_ctx, st)
  if (nseg == 1) SVN(1);
  if (nseg == 2) SVN(2);
  if (nseg <= 4) SVN(4);
#undef SVN
  PALU_REQUIRE(false, "palu_softmax_value: unsupported segment count");
}

}  // namespace palu

// ===========================================================================
// C ABI
// ===========================================================================
using namespace palu;

extern "C" {

const char* palu_version(void) { return "palu_b200 0.1.0 (sm_100a)"; }
const char* palu_last_error(void) { return g_err; }

int palu_device_check(int device) {
  cudaDeviceProp prop;
  PALU_CK(cudaGetDeviceProperties(&prop, device));
  PALU_REQUIRE(prop.major == 10 && prop.minor == 0,
               "palu_b200 is built for sm_100a only; device %d is sm_%d%d (%s)", device,
               prop.major, prop.minor, prop.name);
  return PALU_OK;
}

int palu_gemv(int dtype, const void* W, int N, int K, const float* x, int B, int ldx, float* y,
              int ldy, int accumulate, void* stream) {
  PALU_REQUIRE(N > 0 && K > 0 && B > 0, "palu_gemv: bad sizes N=%d K=%d B=%d", N, K, B);
  const int vec = dtype == PALU_DTYPE_BF16 ? 8 : 4;
  PALU_REQUIRE(K % vec == 0, "palu_gemv: K=%d must be a multiple of %d", K, vec);
  PALU_REQUIRE(((uintptr_t)W & 15) == 0 && ((uintptr_t)x & 15) == 0 && ldx % 4 == 0,
               "palu_gemv: W/x must be 16-byte aligned");
  if (dtype == PALU_DTYPE_BF16) {
    static const bool warp_rows = getenv("PALU_GEMV") && strcmp(getenv("PALU_GEMV"), "warp") == 0;
    if (!warp_rows) {
      const int rc = gemv_stream((const bf16*)W, N, K, x, B, ldx, y, ldy, accumulate, S(stream));
      if (rc != PALU_EUNSUPPORTED) return rc;
    }
    return gemv_dispatch<bf16>((const bf16*)W, N, K, x, B, ldx, y, ldy, accumulate, S(stream));
  }
  PALU_REQUIRE(dtype == PALU_DTYPE_F32, "palu_gemv: unknown dtype %d", dtype);
  return gemv_dispatch<float>((const float*)W, N, K, x, B, ldx, y, ldy, accumulate, S(stream));
}

int palu_latent_append(int dtype, int bits, const float* lat, int B, int ld_lat, int G,
                       const int* ranks, const int* lat_off, void* rows, float* scales, float* zps,
                       double* scales64, int64_t* zps64, int R_pad, int T_cap, const int* t_dev,
                       void* stream) {
  PALU_REQUIRE(B > 0 && G > 0 && R_pad > 0 && T_cap > 0, "palu_latent_append: bad sizes");
  dim3 grid(G, B);
  if (bits == 16) {
    if (dtype == PALU_DTYPE_BF16)
      PALU_CK(launch_k(append_raw_kernel<bf16>, dim3(grid), dim3(128), 0, S(stream), lat, ld_lat, G, ranks, lat_off,
                                                            (bf16*)rows, R_pad, T_cap, t_dev));
    else
      PALU_CK(launch_k(append_raw_kernel<float>, dim3(grid), dim3(128), 0, S(stream), lat, ld_lat, G, ranks, lat_off,
                                                             (float*)rows, R_pad, T_cap, t_dev));
    PALU_LAUNCHED();
    return PALU_OK;
  }
  PALU_REQUIRE(bits == 2 || bits == 3 || bits == 4 || bits == 8,
               "bits must be one of (2, 3, 4, 8), got %d", bits);
  PALU_REQUIRE(R_pad % 32 == 0, "quantised rows need R_pad %% 32 == 0 (got %d)", R_pad);
  const size_t smem = (size_t)(R_pad + 64) * sizeof(double) + R_pad;
  PALU_CK(launch_k(append_quant_kernel, dim3(grid), dim3(128), smem, S(stream), lat, ld_lat, G, bits, ranks, lat_off,
                                                      (uint8_t*)rows, scales, zps, scales64, zps64,
                                                      R_pad, T_cap, t_dev));
  PALU_LAUNCHED();
  return PALU_OK;
}

int palu_latent_append_kv(int dtype, int bits_k, int bits_v, const float* lat_k, const float* lat_v,
                          int B, int ld_lat, int G_k, int G_v, const int* ranks_k,
                          const int* lat_off_k, const int* ranks_v, const int* lat_off_v,
                          void* rows_k, float* scales_k, float* zps_k, double* scales64_k,
                          int64_t* zps64_k, void* rows_v, float* scales_v, float* zps_v,
                          double* scales64_v, int64_t* zps64_v, int R_pad_k, int R_pad_v,
                          int T_cap, const int* t_dev, void* stream) {
  PALU_REQUIRE(B > 0 && G_k > 0 && G_v > 0 && R_pad_k > 0 && R_pad_v > 0 && T_cap > 0,
               "palu_latent_append_kv: bad sizes");
  size_t smem = 0;
  for (int side = 0; side < 2; ++side) {
    const int bits = side ? bits_v : bits_k, R_pad = side ? R_pad_v : R_pad_k;
    if (bits == 16) continue;
    PALU_REQUIRE(bits == 2 || bits == 3 || bits == 4 || bits == 8,
                 "bits must be one of (2, 3, 4, 8), got %d", bits);
    PALU_REQUIRE(R_pad % 32 == 0, "quantised rows need R_pad %% 32 == 0 (got %d)", R_pad);
    const size_t need = (size_t)(R_pad + 64) * sizeof(double) + R_pad;
    if (need > smem) smem = need;
  }
  const AppendSide k{bits_k, G_k, R_pad_k, lat_k, ranks_k, lat_off_k, rows_k,
                     scales_k, zps_k, scales64_k, zps64_k};
  const AppendSide v{bits_v, G_v, R_pad_v, lat_v, ranks_v, lat_off_v, rows_v,
                     scales_v, zps_v, scales64_v, zps64_v};
  const dim3 grid(G_k + G_v, B);
  if (dtype == PALU_DTYPE_BF16)
    PALU_CK(launch_k(append_kv_kernel<bf16>, grid, dim3(128), smem, S(stream), k, v, ld_lat, T_cap, t_dev));
  else
    PALU_CK(launch_k(append_kv_kernel<float>, grid, dim3(128), smem, S(stream), k, v, ld_lat, T_cap, t_dev));
  PALU_LAUNCHED();
  return PALU_OK;
}

// ---------------------------------------------------------------------------
// Container export (quant.py:156-169 pack_codes over a cache's stored rows):
// the first `rank` codes of each padded row, concatenated over T rows, as one
// LSB-first bitstream (code i at bits [i b, (i + 1) b)).  Thread = output byte.
// ---------------------------------------------------------------------------
__global__ void pack_stream_kernel(const uint8_t* __restrict__ rows, int row_bytes, int rank, int T,
                                   int bits, uint8_t* __restrict__ out, long long out_bytes) {
  pdl_enter();
  const long long n_codes = (long long)T * rank;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < out_bytes;
       j += (long long)gridDim.x * blockDim.x) {
    uint32_t byte = 0;
    for (int p = 0; p < 8; ++p) {
      const long long pos = 8 * j + p;
      const long long i = pos / bits;
      if (i >= n_codes) break;
      const int bit = (int)(pos - i * bits);
      const long long t = i / rank;
      const long long rb = (i - t * rank) * bits + bit;  // bit inside the stored row
      const uint32_t v = rows[t * row_bytes + (rb >> 3)];
      byte |= ((v >> (rb & 7)) & 1u) << p;
    }
    out[j] = (uint8_t)byte;
  }
}

int palu_pack_code_stream(int bits, const void* rows, int row_bytes, int rank, int T, void* out,
                          long long out_bytes, void* stream) {
  PALU_REQUIRE(bits == 2 || bits == 3 || bits == 4 || bits == 8,
               "palu_pack_code_stream: bits must be one of (2, 3, 4, 8), got %d", bits);
  PALU_REQUIRE(rank >= 0 && T >= 0 && (long long)rank * bits <= 8LL * row_bytes,
               "palu_pack_code_stream: rank %d does not fit rows of %d bytes", rank, row_bytes);
  const long long need = ((long long)T * rank * bits + 7) / 8;
  PALU_REQUIRE(out_bytes == need, "palu_pack_code_stream: out_bytes %lld, expected %lld", out_bytes,
               need);
  if (need == 0) return PALU_OK;
  const int threads = 256;
  const long long blocks = (need + threads - 1) / threads;
  PALU_CK(launch_k(pack_stream_kernel, dim3((unsigned)(blocks < 4096 ? blocks : 4096)),
                   dim3(threads), 0, S(stream), (const uint8_t*)rows, row_bytes, rank, T, bits,
                   (uint8_t*)out, out_bytes));
  PALU_LAUNCHED();
  return PALU_OK;
}

int palu_quantize_rows(const double* x, int rows, int cols, int bits, uint8_t* codes,
                       double* scales, int64_t* zps, void* stream) {
  PALU_REQUIRE(bits == 2 || bits == 3 || bits == 4 || bits == 8,
               "bits must be one of (2, 3, 4, 8), got %d", bits);
  PALU_REQUIRE(rows >= 0 && cols > 0, "palu_quantize_rows: bad sizes");
  if (rows == 0) return PALU_OK;
  const size_t smem = (size_t)(cols + 64) * sizeof(double);
  PALU_CK(cudaFuncSetAttribute(quantize_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  quantize_rows_kernel<<<rows, 128, smem, S(stream)>>>(x, cols, bits, codes, scales, zps);
  PALU_LAUNCHED();
  return PALU_OK;
}

int palu_pack_rows(const uint8_t* codes, int rows, int cols, int bits, uint8_t* packed,
                   void* stream) {
  PALU_REQUIRE(bits == 2 || bits == 3 || bits == 4 || bits == 8,
               "bits must be one of (2, 3, 4, 8), got %d", bits);
  PALU_REQUIRE((cols * bits) % 8 == 0, "palu_pack_rows: cols*bits must be byte aligned");
  if (rows == 0) return PALU_OK;
  pack_rows_kernel<<<rows, 128, 0, S(stream)>>>(codes, cols, bits, packed);
  PALU_LAUNCHED();
  return PALU_OK;
}

int palu_query_absorb(int dtype, const float* q, int B, int ld_q, int n_heads, int head_dim,
                      int s_k, const void* bk, int bk_rows, int R_pad, const double* theta,
                      float scale, const int* t_dev, void* uw, int layout, void* stream) {
  PALU_REQUIRE(bk_rows >= R_pad, "palu_query_absorb: bk has %d rows < R_pad %d", bk_rows, R_pad);
  PALU_REQUIRE(head_dim % 2 == 0, "rotary embedding requires an even head_dim");
  PALU_REQUIRE(s_k >= 1 && n_heads % s_k == 0, "group size %d does not divide %d heads", s_k,
               n_heads);
  PALU_REQUIRE(layout >= 0 && layout <= 3, "palu_query_absorb: layout must be 0..3");
  dim3 grid(n_heads, (R_pad + 31) / 32, B);
  const size_t smem = ((size_t)head_dim + 32 * ((size_t)head_dim + 1)) * sizeof(float) +
                      (size_t)head_dim * sizeof(double);
  if (dtype == PALU_DTYPE_BF16)
    PALU_CK(launch_k(query_absorb_kernel<bf16>, dim3(grid), dim3(256), smem, S(stream), q, ld_q,
                     n_heads, head_dim, s_k, (const bf16*)bk, bk_rows, R_pad, theta, scale, t_dev,
                     uw, layout, pdl_split()));
  else
    PALU_CK(launch_k(query_absorb_kernel<float>, dim3(grid), dim3(256), smem, S(stream), q, ld_q,
                     n_heads, head_dim, s_k, (const float*)bk, bk_rows, R_pad, theta, scale, t_dev,
                     uw, layout, pdl_split()));
  PALU_LAUNCHED();
  return PALU_OK;
}

int palu_append_absorb(int dtype, int bits_k, int bits_v, const float* lat_k, const float* lat_v, int B,
                       int ld_lat, int G_k, int G_v, const int* ranks_k, const int* lat_off_k,
                       const int* ranks_v, const int* lat_off_v, void* rows_k, float* scales_k,
                       float* zps_k, double* scales64_k, int64_t* zps64_k, void* rows_v, float* scales_v,
                       float* zps_v, double* scales64_v, int64_t* zps64_v, int R_pad_k, int R_pad_v,
                       int T_cap, const float* q, int ld_q, int n_heads, int head_dim, int s_k,
                       const void* bk, int bk_rows, const double* theta, float scale, void* uw, int layout,
                       const int* t_dev, void* stream) {
  PALU_REQUIRE(B > 0 && G_k > 0 && G_v > 0 && R_pad_k > 0 && R_pad_v > 0 && T_cap > 0,
               "palu_append_absorb: bad sizes");
  PALU_REQUIRE(bk_rows >= R_pad_k, "palu_append_absorb: bk has %d rows < R_pad %d", bk_rows, R_pad_k);
  PALU_REQUIRE(head_dim % 2 == 0, "rotary embedding requires an even head_dim");
  PALU_REQUIRE(s_k >= 1 && n_heads % s_k == 0, "group size %d does not divide %d heads", s_k, n_heads);
  PALU_REQUIRE(layout >= 0 && layout <= 4, "palu_append_absorb: layout must be 0..4");
  size_t smem = ((size_t)head_dim + 32 * ((size_t)head_dim + 1)) * sizeof(float) +
                (size_t)head_dim * sizeof(double);
  for (int side = 0; side < 2; ++side) {
    const int bits = side ? bits_v : bits_k, R_pad = side ? R_pad_v : R_pad_k;
    if (bits == 16) continue;
    PALU_REQUIRE(bits == 2 || bits == 3 || bits == 4 || bits == 8,
                 "bits must be one of (2, 3, 4, 8), got %d", bits);
    PALU_REQUIRE(R_pad % 32 == 0, "quantised rows need R_pad %% 32 == 0 (got %d)", R_pad);
    const size_t need = (size_t)(R_pad + 64) * sizeof(double) + R_pad;
    if (need > smem) smem = need;
  }
  const AppendSide k{bits_k, G_k, R_pad_k, lat_k, ranks_k, lat_off_k, rows_k,
                     scales_k, zps_k, scales64_k, zps64_k};
  const AppendSide v{bits_v, G_v, R_pad_v, lat_v, ranks_v, lat_off_v, rows_v,
                     scales_v, zps_v, scales64_v, zps64_v};
  const int gy = layout == 4 ? 1 : (R_pad_k + 31) / 32;  // layout 4: rotated query rows only
  const AbsorbArgs a{q, ld_q, n_heads, head_dim, s_k, bk, bk_rows, R_pad_k, theta, scale, uw, layout, gy};
  const int n_abs = n_heads * gy * B, n_app = (G_k + G_v) * B;
  if (dtype == PALU_DTYPE_BF16)
    PALU_CK(launch_k(append_absorb_kernel<bf16>, dim3(n_abs + n_app), dim3(256), smem, S(stream), k, v, ld_lat,
                     T_cap, t_dev, a, n_abs));
  else
    PALU_CK(launch_k(append_absorb_kernel<float>, dim3(n_abs + n_app), dim3(256), smem, S(stream), k, v, ld_lat,
                     T_cap, t_dev, a, n_abs));
  PALU_LAUNCHED();
  return PALU_OK;
}

int palu_latent_score(int dtype, int bits, const void* hk, const float* scales, const float* zps,
                      int B, int n_heads, int s_k, int G, int R_pad, int T_cap, const float* y,
                      int ld_y, const int* q_off, const int* ranks, float scale, const int* t_dev,
                      float* logits, int ld_logits, void* stream) {
  PALU_REQUIRE(G * s_k == n_heads, "palu_latent_score: G*s_k != n_heads");
  PALU_REQUIRE(s_k <= 8, "palu_latent_score: at most 8 heads per key group (got %d)", s_k);
  PALU_REQUIRE(ld_logits >= T_cap, "palu_latent_score: ld_logits < T_cap");
  dim3 grid((T_cap + 7) / 8 < 512 ? (T_cap + 7) / 8 : 512, G, B);
  cudaStream_t st = S(stream);
#define LS(T_, BITS_)                                                                          \
  PALU_CK(launch_k(latent_score_kernel<T_, BITS_>, grid, dim3(256), 0, st, hk, scales, zps, n_heads, \
                   s_k, G, R_pad, T_cap, y, ld_y, q_off, ranks, scale, t_dev, logits, ld_logits))
  if (bits == 16) {
    if (dtype == PALU_DTYPE_BF16) LS(bf16, 16);
    else LS(float, 16);
  } else if (bits == 2) LS(float, 2);
  else if (bits == 3) LS(float, 3);
  else if (bits == 4) LS(float, 4);
  else if (bits == 8) LS(float, 8);
  else PALU_REQUIRE(false, "bits must be one of (2, 3, 4, 8, 16), got %d", bits);
#undef LS
  return PALU_OK;
}

int palu_rope_score(int dtype, int bits, const void* hk, const float* scales, const float* zps,
                    int B, int n_heads, int head_dim, int s_k, int G, int R_pad, int T_cap,
                    const void* uw, const double* theta, const int* t_dev, float* logits,
                    int ld_logits, void* stream) {
  PALU_REQUIRE(G * s_k == n_heads, "palu_rope_score: G*s_k != n_heads");
  PALU_REQUIRE(ld_logits >= T_cap, "palu_rope_score: ld_logits < T_cap");
  cudaStream_t st = S(stream);
  const float* u = (const float*)uw;
#define SCORE(T_, B_) launch_score<T_, B_>(hk, scales, zps, B, n_heads, head_dim, s_k, G, R_pad, \
                                           T_cap, u, theta, t_dev, logits, ld_logits, st)
  if (bits == 16) {
    if (dtype == PALU_DTYPE_BF16) SCORE(bf16, 16);
    else SCORE(float, 16);
  } else if (bits == 8) SCORE(float, 8);
  else if (bits == 4) SCORE(float, 4);
  else if (bits == 3) SCORE(float, 3);
  else if (bits == 2) SCORE(float, 2);
  else PALU_REQUIRE(false, "bits must be one of (2, 3, 4, 8, 16), got %d", bits);
#undef SCORE
  PALU_LAUNCHED();
  return PALU_OK;
}

size_t palu_softmax_value_workspace(int B, int n_heads, int R_pad, int n_chunks) {
  // partial (m, l, ctx) per chunk + one ticket per (sequence, group) (zero-initialised)
  return sizeof(float) * (size_t)B * n_heads * n_chunks * (2 + (size_t)R_pad) +
         sizeof(unsigned) * (((size_t)B * n_heads + 31) & ~size_t(31));
}

int palu_softmax_value(int dtype, int bits, const void* hv, const float* scales, const float* zps,
                       int B, int n_heads, int s_v, int G, int R_pad, const int* ranks_v,
                       const int* o_off, int T_cap, const float* logits, int ld_logits,
                       int n_planes, size_t plane_stride, const int* t_dev, int n_chunks,
                       void* workspace, float* ctx, int ld_ctx, void* stream) {
  const long long plane = (long long)plane_stride;
  PALU_REQUIRE(n_planes >= 1, "palu_softmax_value: n_planes must be >= 1");
  PALU_REQUIRE(G * s_v == n_heads, "palu_softmax_value: G*s_v != n_heads");
  PALU_REQUIRE(n_chunks >= 1, "palu_softmax_value: n_chunks must be >= 1");
  SvPartial part = sv_carve(workspace, B, n_heads, R_pad, n_chunks);
  cudaStream_t st = S(stream);
#define SV(T_, B_) return launch_sv<T_, B_>(hv, scales, zps, B, n_heads, s_v, G, R_pad, ranks_v, \
                                            o_off, T_cap, logits, ld_logits, n_planes, plane,    \
                                            t_dev, n_chunks, part, ctx, ld_ctx, st)
  if (bits == 16) {
    if (dtype == PALU_DTYPE_BF16) SV(bf16, 16);
    SV(float, 16);
  }
  if (bits == 8) SV(float, 8);
  if (bits == 4) SV(float, 4);
  if (bits == 3) SV(float, 3);
  if (bits == 2) SV(float, 2);
#undef SV
  PALU_REQUIRE(false, "bits must be one of (2, 3, 4, 8, 16), got %d", bits);
}

int palu_advance(int* t_dev, void* stream) {
  PALU_CK(launch_k(advance_kernel, dim3(1), dim3(1), 0, S(stream), t_dev));
  PALU_LAUNCHED();
  return PALU_OK;
}

int palu_dense_append_paged(const float* qkv, int B, int n_heads, int n_kv, int head_dim, void* kv_pages,
                            int page_size, int pages_per_seq, const double* theta, const int* t_dev,
                            void* q_out, void* stream) {
  PALU_REQUIRE(head_dim % 2 == 0 && n_kv >= 1 && n_kv <= n_heads && n_heads % n_kv == 0,
               "palu_dense_append_paged: head_dim %d, %d query / %d KV heads", head_dim, n_heads, n_kv);
  PALU_CK(launch_k(dense_append_paged_kernel, dim3(n_heads, B), dim3(64), 0, S(stream), qkv, n_heads,
                   n_kv, head_dim, (bf16*)kv_pages, page_size, pages_per_seq, theta, t_dev, (bf16*)q_out));
  PALU_LAUNCHED();
  return PALU_OK;
}

int palu_cast_bf16_f32(const void* src, float* dst, int n, void* stream) {
  PALU_CK(launch_k(cast_bf16_f32_kernel, dim3((n + 255) / 256 < 148 ? (n + 255) / 256 : 148), dim3(256),
                   0, S(stream), (const bf16*)src, dst, n));
  PALU_LAUNCHED();
  return PALU_OK;
}

size_t palu_dense_workspace(int B, int n_heads, int head_dim, int n_chunks) {
  return sizeof(float) * ((size_t)B * n_heads * n_chunks * (2 + (size_t)head_dim) +
                          (size_t)B * n_heads * head_dim + (((size_t)B * n_heads + 31) & ~size_t(31)));
}

int palu_dense_decode(int dtype, const float* qkv, int B, int n_heads, int head_dim, void* kc,
                      void* vc, int T_cap, const double* theta, const int* t_dev, int n_chunks,
                      void* workspace, float* attn, void* stream) {
  PALU_REQUIRE(head_dim % 2 == 0 && head_dim <= 128, "palu_dense_decode: head_dim %d", head_dim);
  cudaStream_t st = S(stream);
  SvPartial part = sv_carve(workspace, B, n_heads, head_dim, n_chunks);
  float* qrot = part.ctx + (size_t)B * n_heads * n_chunks * head_dim;
  int clen = (T_cap + n_chunks - 1) / n_chunks;
  clen = (clen + 7) & ~7;
  const size_t smem = sizeof(float) * (head_dim + clen + 8 * head_dim + 16);
  PALU_REQUIRE(smem <= 200 * 1024, "palu_dense_decode: raise n_chunks");
  dim3 g1(n_heads, B), g2(n_chunks, n_heads, B);
  if (dtype == PALU_DTYPE_BF16) {
    dense_append_kernel<bf16><<<g1, 64, 0, st>>>(qkv, n_heads, head_dim, (bf16*)kc, (bf16*)vc,
                                                 T_cap, theta, t_dev, qrot);
    PALU_CK(cudaFuncSetAttribute(dense_partial_kernel<bf16>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dense_partial_kernel<bf16><<<g2, 256, smem, st>>>(n_heads, head_dim, (const bf16*)kc,
                                                      (const bf16*)vc, T_cap, t_dev, qrot,
                                                      n_chunks, part);
  } else {
    dense_append_kernel<float><<<g1, 64, 0, st>>>(qkv, n_heads, head_dim, (float*)kc, (float*)vc,
                                                  T_cap, theta, t_dev, qrot);
    PALU_CK(cudaFuncSetAttribute(dense_partial_kernel<float>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dense_partial_kernel<float><<<g2, 256, smem, st>>>(n_heads, head_dim, (const float*)kc,
                                                       (const float*)vc, T_cap, t_dev, qrot,
                                                       n_chunks, part);
  }
  PALU_LAUNCHED();
  dense_combine_kernel<<<g1, 128, 0, st>>>(n_heads, head_dim, n_chunks, part, attn);
  PALU_LAUNCHED();
  return PALU_OK;
}

}  // extern "C"
