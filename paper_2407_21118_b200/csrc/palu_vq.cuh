// Packed-V softmax + value kernel on the int8 tensor pipe (sm_100a
// tcgen05.mma.kind::i8).  Included by palu_tc.cu (namespace palu::tc).
//
// Restates attention.py:445 (_softmax) and :350-362 (_value_output up to
// wo_fused) for quantised value latents, dequantised as quant.py:106-107
// x = (c - z) s, without ever materialising x:
//
//   sum_t p_t x_t[c] = sum_t (p_t s_t) (c_t[c] - z_t)
//
// Per 512-token sub-block and head, u_t = p_t s_t / max_t(p_t s_t) is split
// into two signed 8-bit digits, w_t = 254 hi_t + lo_t = round(127 * 254 u_t)
// (|u_t - w_t / 32258| <= 1.6e-5 of the sub-block maximum).  The tensor pipe
// then accumulates EXACT integer sums
//   D[c][hi_h] = sum_t hi_t c_t,   D[c][lo_h] = sum_t lo_t c_t     (s32, TMEM)
// with A = the raw codes as u8 (MN-major SW128: the cache's own [token][col]
// order, nibbles / crumbs expanded to bytes by 4 converter warps; 8-bit codes
// are copied), B = the digits (K-major SW128, N = 16 rows: 4 heads x {hi, lo},
// 8 zero rows), K = 32 tokens per MMA.  The zero-point term
// sum_t w_t z_t is an exact int64 sum on the CUDA cores, so
//   ctx_sub[c] = (254 D_hi + D_lo - sum_t w_t z_t) * max(p s) / 32258
// carries only the digit rounding of the weights.  An online softmax across
// sub-blocks and the deterministic value_merge_kernel complete the path.
//
// The only bytes streamed are the packed codes (TMA, 128-token tiles of the
// whole row), the per-token fp32 scale and zero point, and the logits: the
// HBM-bound stream the north star names, with no bf16 staging of values.
//
// Warps: 0-3 softmax + digits (group A), 4-7 TMEM readback + online softmax
// (group B), 8 TMA producer, 9 MMA issuer + TMEM owner, 10-13 converters.

constexpr int VQ_THREADS = 448;
constexpr int VQ_SUB = 512;                 // tokens per digit sub-block
constexpr int VQ_NB = VQ_SUB / TILE_M;      // 128-token blocks per sub-block
constexpr int VQ_PBUF = VQ_NB * 2048;       // digits: per block 16 rows x 128 B
constexpr int VQ_STAGE = TILE_M * 128;      // one (block, 128-column tile) u8 operand
constexpr int VQ_TMEM = 128;                // 2 buffers x up to 4 tiles x 16 columns
constexpr float VQ_W = 127.f * 254.f;       // digit weight scale
// D s32, A u8 (MN-major), B s8 (K-major), M 128, N 16
constexpr uint32_t IDESC_Q = (2u << 4) | (0u << 7) | (1u << 10) | (1u << 15) |
                             ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(TILE_M >> 4) << 24);

struct VQParams {
  int B, n_heads, s, G, Rv_pad, T_cap, ld_logits;
  int row_bytes, box_bytes;  // packed row; TMA box width (row_bytes or 128)
  int raw_slots, stages, ns_cap;
  const int* t_dev;
  const float* logits;
  const float* scales;
  const float* zps;
  float *pm, *pl, *pctx;
};

__device__ __forceinline__ void umma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(IDESC_Q), "r"(accum)
      : "memory");
}

// This CTA's units: its contiguous items [i, i1) of (sequence x group,
// 256-token super-tile), split at group boundaries (value_merge_kernel's
// vc = per slot convention).
struct VQIter {
  int i, i1, n_super;
  __device__ VQIter(int a, int b, int ns) : i(a), i1(b), n_super(ns) {}
  __device__ __forceinline__ bool next(int& bg, int& st0, int& st1) {
    if (i >= i1) return false;
    bg = i / n_super;
    st0 = i - bg * n_super;
    const int se = min(i1, (bg + 1) * n_super);
    st1 = se - bg * n_super;
    i = se;
    return true;
  }
};

// Operand position (TMEM lane) -> value column, inverse of the converter's
// expansion order inside a 128-column tile.
template <int BITS>
__device__ __forceinline__ int vq_column(int m) {
  if constexpr (BITS == 4) {
    const int r = m & 31;
    return (m & ~31) + (r < 16 ? 2 * r : 2 * (r - 16) + 1);
  } else if constexpr (BITS == 2) {
    const int r = m & 63;
    return (m & ~63) + 4 * (r & 15) + (r >> 4);
  } else {
    return m;
  }
}

template <int BITS>
__global__ void __launch_bounds__(VQ_THREADS, 1)
value_q_kernel(const __grid_constant__ CUtensorMap map_c, const VQParams p) {
  // codes of older tokens stream while the score kernel drains; the producer
  // waits before the newest token's tile, group A before the logits
  pdl_launch();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int NJ = p.Rv_pad / 128;
  const int RB = TILE_M * p.row_bytes;
  uint8_t* ring = smem;                                          // stages x 16 KB
  uint8_t* pbuf = ring + p.stages * VQ_STAGE;                    // 2 x 8 KB digits
  uint8_t* raw = pbuf + 2 * VQ_PBUF;                             // raw_slots x RB codes
  float* stat = reinterpret_cast<float*>(raw + (size_t)p.raw_slots * RB);  // [2][3][V_HP]
  long long* statz = reinterpret_cast<long long*>(stat + 2 * 3 * V_HP);    // [2][V_HP]
  uint64_t* full = reinterpret_cast<uint64_t*>(statz + 2 * V_HP);
  uint64_t* empty = full + p.stages;
  uint64_t* rfull = empty + p.stages;
  uint64_t* rempty = rfull + p.raw_slots;
  uint64_t* pfull = rempty + p.raw_slots;  // [2] digits + statistics written
  uint64_t* dfull = pfull + 2;             // [2] sub-block accumulators complete
  uint64_t* dempty = dfull + 2;            // [2] sub-block accumulators read back
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dempty + 2);
  __shared__ float red_f[2][4][V_HP];
  __shared__ long long red_z[4][V_HP];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int T_rows = *p.t_dev + 1;  // final: advanced by the previous step's last launch
  const int n_super = (T_rows + SUPER - 1) / SUPER;
  const int total = p.B * p.G * n_super;
  const int per = (total + (int)gridDim.x - 1) / (int)gridDim.x;
  const int i0 = min(total, (int)blockIdx.x * per), i1 = min(total, i0 + per);

  if (tid == 0) {
    for (int st = 0; st < p.stages; ++st) {
      mbar_init(&full[st], 4);  // one arrive per converter warp
      mbar_init(&empty[st], 1);
    }
    for (int r = 0; r < p.raw_slots; ++r) {
      mbar_init(&rfull[r], 1);
      mbar_init(&rempty[r], 4);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&pfull[a], 1);
      mbar_init(&dfull[a], 1);
      mbar_init(&dempty[a], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // digit rows 8..15 of every block stay zero (N = 16 > 4 heads x 2 digits)
  for (int i = tid; i < 2 * VQ_NB * 64; i += VQ_THREADS) {
    const int blk = i >> 6, w = i & 63;
    reinterpret_cast<uint4*>(pbuf + blk * 2048 + 1024)[w] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(VQ_TMEM));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  int bg, s0u, s1u;

  if (warp == 8) {
    // ---------------- TMA producer: packed code tiles {row, 128 tokens} ----------------
    if (lane == 0) {
      prefetch_map(&map_c);
      VQIter it(i0, i1, n_super);
      Ring rg;
      bool waited = false;
      while (it.next(bg, s0u, s1u)) {
        const int c0 = s0u * SUPER, c1 = min(T_rows, s1u * SUPER);
        for (int t0 = c0; t0 < c1; t0 += TILE_M) {
          // the newest token (row T_rows - 1) comes from this step's append
          if (!waited && t0 + TILE_M >= T_rows) {
            pdl_wait();
            waited = true;
          }
          mbar_wait(&rempty[rg.slot], rg.phase ^ 1);
          mbar_expect_tx(&rfull[rg.slot], RB);
          uint8_t* dst = raw + (size_t)rg.slot * RB;
          for (int x = 0; x < p.row_bytes; x += p.box_bytes)
            tma_load_2d(&map_c, &rfull[rg.slot], dst + x * TILE_M, x, bg * p.T_cap + t0);
          rg.next(p.raw_slots);
        }
      }
    }
  } else if (warp >= 10) {
    // ---------------- converters: packed row -> u8 MN-major SW128 operand ----------------
    // work item (row, q): 16-byte raw chunk q of the row's slice for column
    // tile j; RC consecutive lanes share a row (conflict-free raw reads)
    constexpr int RC = BITS;  // raw 16-byte chunks per row per 128 columns
    const int ct = tid - 320;
    VQIter it(i0, i1, n_super);
    Ring rr, rs;
    while (it.next(bg, s0u, s1u)) {
      const int c0 = s0u * SUPER, c1 = min(T_rows, s1u * SUPER);
      for (int t0 = c0; t0 < c1; t0 += TILE_M) {
        mbar_wait(&rfull[rr.slot], rr.phase);
        const uint8_t* slot = raw + (size_t)rr.slot * RB;
        for (int j = 0; j < NJ; ++j) {
          mbar_wait(&empty[rs.slot], rs.phase ^ 1);
          uint8_t* st = ring + rs.slot * VQ_STAGE;
#pragma unroll
          for (int k = 0; k < RC; ++k) {
            const int w = ct + 128 * k;
            const int row = w / RC, q = w % RC;
            const int kb = j * 16 * BITS + 16 * q;  // byte inside the packed row
            const uint4 v = lds128(smem_u32(slot + (kb / p.box_bytes) * (TILE_M * p.box_bytes) +
                                            row * p.box_bytes + kb % p.box_bytes));
            const uint32_t rowa = smem_u32(st + row * 128);
            const int sw = row & 7;
            if constexpr (BITS == 8) {
              asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(rowa + ((q ^ sw) << 4)),
                           "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                           : "memory");
            } else if constexpr (BITS == 4) {
              constexpr uint32_t M = 0x0F0F0F0Fu;
              asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(rowa + (((2 * q) ^ sw) << 4)),
                           "r"(v.x & M), "r"(v.y & M), "r"(v.z & M), "r"(v.w & M)
                           : "memory");
              asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                               rowa + (((2 * q + 1) ^ sw) << 4)),
                           "r"((v.x >> 4) & M), "r"((v.y >> 4) & M), "r"((v.z >> 4) & M),
                           "r"((v.w >> 4) & M)
                           : "memory");
            } else {  // BITS == 2
              constexpr uint32_t M = 0x03030303u;
#pragma unroll
              for (int e = 0; e < 4; ++e)
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                                 rowa + (((4 * q + e) ^ sw) << 4)),
                             "r"((v.x >> (2 * e)) & M), "r"((v.y >> (2 * e)) & M),
                             "r"((v.z >> (2 * e)) & M), "r"((v.w >> (2 * e)) & M)
                             : "memory");
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[rs.slot]);
          rs.next(p.stages);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&rempty[rr.slot]);
        rr.next(p.raw_slots);
      }
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      VQIter it(i0, i1, n_super);
      Ring rs;
      int sb = 0;
      while (it.next(bg, s0u, s1u)) {
        const int c0 = s0u * SUPER, c1 = min(T_rows, s1u * SUPER);
        const int nblk = (c1 - c0 + TILE_M - 1) / TILE_M;
        for (int b0 = 0; b0 < nblk; b0 += VQ_NB, ++sb) {
          const int buf = sb & 1;
          mbar_wait(&pfull[buf], (sb >> 1) & 1);
          if (sb >= 2) mbar_wait(&dempty[buf], ((sb >> 1) - 1) & 1);
          fence_after();
          const uint32_t pb = smem_u32(pbuf + buf * VQ_PBUF);
          const int b1 = min(nblk, b0 + VQ_NB);
          for (int blk = b0; blk < b1; ++blk)
            for (int j = 0; j < NJ; ++j) {
              mbar_wait(&full[rs.slot], rs.phase);
              fence_after();
              const uint32_t a0 = smem_u32(ring + rs.slot * VQ_STAGE);
              const uint32_t d = tmem + (uint32_t)((buf * NJ + j) * 16);
              const uint64_t da = sdesc_mn(a0, VQ_STAGE, 1024);
              const uint64_t db = sdesc(pb + (blk - b0) * 2048);
#pragma unroll
              for (int kk = 0; kk < TILE_M / 32; ++kk)  // K = 32 tokens: 4 KB of A, 32 B of B
                umma_i8(d, da + (uint64_t)(kk * 256), db + (uint64_t)(kk * 2), (blk != b0) || (kk != 0));
              umma_commit(&empty[rs.slot]);
              rs.next(p.stages);
            }
          umma_commit(&dfull[buf]);
        }
      }
    }
  } else if (warp < 4) {
    // ---------------- group A: logits -> statistics -> digits ----------------
    pdl_wait();  // logits (score kernel), scales / zero points of the newest token
    const int ta = tid;
    VQIter it(i0, i1, n_super);
    int sb = 0;
    constexpr int NP = VQ_SUB / 256;  // token pairs per thread per sub-block
    while (it.next(bg, s0u, s1u)) {
      const int b = bg / p.G, g = bg - b * p.G;
      const int c0 = s0u * SUPER, c1 = min(T_rows, s1u * SUPER);
      const int nt = c1 - c0;
      const int ntok = (nt + TILE_M - 1) / TILE_M * TILE_M;
      const float* lg = p.logits + ((size_t)b * p.n_heads + g * p.s) * p.ld_logits + c0;
      const float* sc = p.scales + (size_t)bg * p.T_cap + c0;
      const float* zp = p.zps + (size_t)bg * p.T_cap + c0;
      float2 x[NP][V_HP], xn[NP][V_HP];
      auto load = [&](int s0, float2 (&dst)[NP][V_HP]) {
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const int t = s0 + 2 * ta + 256 * i;
#pragma unroll
          for (int h = 0; h < V_HP; ++h) {
            float2 v = make_float2(-INFINITY, -INFINITY);
            if (h < p.s && t < nt) {
              v = __ldcg(reinterpret_cast<const float2*>(lg + (size_t)h * p.ld_logits + t));
              if (t + 1 >= nt) v.y = -INFINITY;
            }
            dst[i][h] = v;
          }
        }
      };
      load(0, xn);
      for (int s0 = 0; s0 < ntok; s0 += VQ_SUB, ++sb) {
        const int buf = sb & 1;
#pragma unroll
        for (int i = 0; i < NP; ++i)
#pragma unroll
          for (int h = 0; h < V_HP; ++h) x[i][h] = xn[i][h];
        if (s0 + VQ_SUB < ntok) load(s0 + VQ_SUB, xn);
        float2 sv[NP], zv[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const int t = s0 + 2 * ta + 256 * i;
          sv[i] = make_float2(0.f, 0.f);
          zv[i] = make_float2(0.f, 0.f);
          if (t < nt) {
            sv[i].x = __ldg(sc + t);
            zv[i].x = __ldg(zp + t);
            if (t + 1 < nt) {
              sv[i].y = __ldg(sc + t + 1);
              zv[i].y = __ldg(zp + t + 1);
            }
          }
        }
        // (1) logit maximum of the sub-block
        float m[V_HP];
#pragma unroll
        for (int h = 0; h < V_HP; ++h) {
          m[h] = -INFINITY;
#pragma unroll
          for (int i = 0; i < NP; ++i) m[h] = fmaxf(m[h], fmaxf(x[i][h].x, x[i][h].y));
          m[h] = warp_reduce(m[h], [](float a, float c) { return fmaxf(a, c); });
          if (lane == 0) red_f[0][warp][h] = m[h];
        }
        named_bar_sync(3, 128);
        // (2) p = exp(x - m), q = p s, and max q
        float l[V_HP], mx[V_HP];
        float2 q[NP][V_HP];
#pragma unroll
        for (int h = 0; h < V_HP; ++h) {
          m[h] = fmaxf(fmaxf(red_f[0][0][h], red_f[0][1][h]), fmaxf(red_f[0][2][h], red_f[0][3][h]));
          l[h] = 0.f;
          mx[h] = 0.f;
#pragma unroll
          for (int i = 0; i < NP; ++i) {
            float p0 = 0.f, p1 = 0.f;
            if (h < p.s) {
              p0 = __expf(x[i][h].x - m[h]);
              p1 = __expf(x[i][h].y - m[h]);
            }
            l[h] += p0 + p1;
            q[i][h] = make_float2(p0 * sv[i].x, p1 * sv[i].y);
            mx[h] = fmaxf(mx[h], fmaxf(q[i][h].x, q[i][h].y));
          }
          mx[h] = warp_reduce(mx[h], [](float a, float c) { return fmaxf(a, c); });
          if (lane == 0) red_f[1][warp][h] = mx[h];
        }
        // the digit buffer is free once sub-block sb - 2 was read back
        if (sb >= 2) mbar_wait(&dempty[buf], ((sb >> 1) - 1) & 1);
        named_bar_sync(3, 128);
        // (3) digits w = 254 hi + lo = round(32258 q / max q); exact int64 sum w z
        uint8_t* pb = pbuf + buf * VQ_PBUF;
        long long zw[V_HP];
#pragma unroll
        for (int h = 0; h < V_HP; ++h) {
          mx[h] = fmaxf(fmaxf(red_f[1][0][h], red_f[1][1][h]), fmaxf(red_f[1][2][h], red_f[1][3][h]));
          const float inv = mx[h] > 0.f ? 127.f / mx[h] : 0.f;
          zw[h] = 0;
#pragma unroll
          for (int i = 0; i < NP; ++i) {
            const int tl = 2 * ta + 256 * i;
            if (h < p.s && s0 + tl < ntok) {
              const float v0 = q[i][h].x * inv, v1 = q[i][h].y * inv;
              const float h0 = rintf(v0), h1 = rintf(v1);
              const float l0 = fminf(fmaxf(rintf((v0 - h0) * 254.f), -127.f), 127.f);
              const float l1 = fminf(fmaxf(rintf((v1 - h1) * 254.f), -127.f), 127.f);
              zw[h] += (long long)(254 * (int)h0 + (int)l0) * (long long)zv[i].x +
                       (long long)(254 * (int)h1 + (int)l1) * (long long)zv[i].y;
              // K-major SW128: row r, token tk -> 16-byte chunk (tk / 16) ^ (r & 7)
              const int blk = tl >> 7, tk = tl & 127;
              uint8_t* rb = pb + blk * 2048 + (tk & 15);
              *reinterpret_cast<uint16_t*>(rb + h * 128 + ((((tk >> 4) ^ h) & 7) << 4)) =
                  (uint16_t)((uint8_t)(int)h0 | ((uint32_t)(uint8_t)(int)h1 << 8));
              *reinterpret_cast<uint16_t*>(rb + (h + 4) * 128 + ((((tk >> 4) ^ (h + 4)) & 7) << 4)) =
                  (uint16_t)((uint8_t)(int8_t)(int)l0 | ((uint32_t)(uint8_t)(int8_t)(int)l1 << 8));
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
        for (int h = 0; h < V_HP; ++h) {
          l[h] = warp_reduce(l[h], [](float a, float c) { return a + c; });
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) zw[h] += __shfl_xor_sync(0xffffffffu, zw[h], o);
          if (lane == 0) {
            red_f[0][warp][h] = l[h];
            red_z[warp][h] = zw[h];
          }
        }
        named_bar_sync(3, 128);
        if (ta < V_HP) {
          const int h = ta;
          float mh = m[0], lh = 0.f, sh = 0.f;
          long long zh = 0;
#pragma unroll
          for (int k = 0; k < V_HP; ++k)
            if (k == h) {
              mh = m[k];
              lh = (red_f[0][0][k] + red_f[0][1][k]) + (red_f[0][2][k] + red_f[0][3][k]);
              sh = mx[k] / VQ_W;
              zh = (red_z[0][k] + red_z[1][k]) + (red_z[2][k] + red_z[3][k]);
            }
          stat[(buf * 3 + 0) * V_HP + h] = mh;
          stat[(buf * 3 + 1) * V_HP + h] = lh;
          stat[(buf * 3 + 2) * V_HP + h] = sh;
          statz[buf * V_HP + h] = zh;
        }
        named_bar_sync(3, 128);
        if (ta == 0) mbar_arrive(&pfull[buf]);
      }
    }
  } else {
    // ---------------- group B: integer sub-block sums -> online softmax -> partial ----------------
    const int tb = tid - 128, wb = warp - 4;
    const int mpos = wb * 32 + lane;  // TMEM lane = operand position in a column tile
    const int col_in = vq_column<BITS>(mpos);
    VQIter it(i0, i1, n_super);
    int sb = 0;
    while (it.next(bg, s0u, s1u)) {
      const int b = bg / p.G, g = bg - b * p.G;
      const int c0 = s0u * SUPER, c1 = min(T_rows, s1u * SUPER);
      const int nblk = (c1 - c0 + TILE_M - 1) / TILE_M;
      float acc[4][V_HP], mr[V_HP], lr[V_HP];
#pragma unroll
      for (int h = 0; h < V_HP; ++h) {
        mr[h] = -INFINITY;
        lr[h] = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j][h] = 0.f;
      }
      for (int b0 = 0; b0 < nblk; b0 += VQ_NB, ++sb) {
        const int buf = sb & 1;
        mbar_wait(&dfull[buf], (sb >> 1) & 1);
        fence_after();
        float sc_old[V_HP], sc_new[V_HP], scl[V_HP];
        long long zw[V_HP];
#pragma unroll
        for (int h = 0; h < V_HP; ++h) {
          const float ms = stat[(buf * 3 + 0) * V_HP + h], ls = stat[(buf * 3 + 1) * V_HP + h];
          scl[h] = stat[(buf * 3 + 2) * V_HP + h];
          zw[h] = statz[buf * V_HP + h];
          const float mn = fmaxf(mr[h], ms);
          sc_old[h] = mr[h] == -INFINITY ? 0.f : __expf(mr[h] - mn);
          sc_new[h] = ms == -INFINITY ? 0.f : __expf(ms - mn);
          lr[h] = lr[h] * sc_old[h] + ls * sc_new[h];
          mr[h] = mn;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j < NJ) {
            float v[16];
            tmem_ld16(tmem + ((uint32_t)(wb * 32) << 16) + (uint32_t)((buf * NJ + j) * 16), v);
            tmem_wait_ld();
#pragma unroll
            for (int h = 0; h < V_HP; ++h) {
              const long long r = 254ll * __float_as_int(v[h]) + __float_as_int(v[h + V_HP]) - zw[h];
              acc[j][h] = acc[j][h] * sc_old[h] + __ll2float_rn(r) * scl[h] * sc_new[h];
            }
          }
        }
        fence_before();
        named_bar_sync(4, 128);
        if (tb == 0) mbar_arrive(&dempty[buf]);
      }
      // the unit's partial (value_merge_kernel layout): slot = first super-tile
      for (int j = 0; j < NJ && j < 4; ++j) {
        const int col = j * 128 + col_in;
#pragma unroll
        for (int h = 0; h < V_HP; ++h)
          if (h < p.s)
            p.pctx[(((size_t)b * p.n_heads + g * p.s + h) * p.ns_cap + s0u) * p.Rv_pad + col] = acc[j][h];
      }
#pragma unroll
      for (int h = 0; h < V_HP; ++h)
        if (tb == h && h < p.s) {
          const size_t pi = ((size_t)b * p.n_heads + g * p.s + h) * p.ns_cap + s0u;
          p.pm[pi] = mr[h];
          p.pl[pi] = lr[h];
        }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 9) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(VQ_TMEM));
  }
}
