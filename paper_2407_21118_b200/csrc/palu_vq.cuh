// Packed-V softmax + value kernel on the int8 tensor pipe (sm_100a
// tcgen05.mma.kind::i8).  Included by palu_tc.cu (namespace palu::tc).
//
// Restates attention.py:445 (_softmax) and :350-362 (_value_output up to
// wo_fused) for quantised value latents, dequantised as quant.py:106-107
// x = (c - z) s, without ever materialising x:
//
//   sum_t p_t x_t[c] = sum_t (p_t s_t) (c_t[c] - z_t)
//
// Per 384-token sub-block and head, u_t = p_t s_t / (max_t s_t) in [0, 1] is
// split into two signed 8-bit digits, w_t = 254 hi_t + lo_t = round(32258 u_t)
// (|u_t - w_t / 32258| <= 1.6e-5).  The tensor pipe accumulates EXACT integer
// sums over the sub-block
//   D[c][hi_h] = sum_t hi_t a_t[c],   D[c][lo_h] = sum_t lo_t a_t[c]  (s32, TMEM)
// with B = the digits (K-major SW128, N = 16 rows: 4 heads x {hi, lo}, 8
// zero rows), K = 32 tokens per MMA, and A in the cache's own [token][col]
// order (MN-major SW128): a = the codes c as u8, nibbles / crumbs expanded to
// bytes by 4 converter warps (8-bit codes copied); the zero-point term
// sum_t w_t z_t is an exact int64 sum on the CUDA cores.  So
//   ctx_sub[c] = (254 D_hi + D_lo - sum_t w_t z_t) * max(s) / 32258
// carries only the digit rounding of the weights.  (Subtracting z in the
// converters instead -- s8 operands, no int64 term -- measured slower: the
// per-byte subtraction costs the converters more than the term costs group A.)  An online softmax across sub-blocks and
// the deterministic value_merge_kernel complete the path.
//
// Raw bf16 values (BITS 16) take the same pipeline without converters: the
// producer TMA-loads {64 columns x 128 tokens} SW128 boxes straight into the
// MN-major operand (one 32 KB stage per 128-column tile), the digits are the
// bf16 pair hi = bf16(p), lo = bf16(p - hi) (~16 significant bits), and
// kind::f16 MMAs accumulate fp32 in TMEM.
//
// Bytes streamed: the packed codes (one 1-D bulk copy per 128-token block,
// L2-prefetched ahead), per-token scales and zero points, and the logits: the HBM-bound stream the north star names, with no bf16 staging.
//
// Warps: 0-5 softmax + digits (group A), 6-9 TMEM readback + online softmax
// (group B), 10-13 converters, 14 bulk-copy producer, 15 MMA issuer + TMEM
// owner.  Pipeline units are whole 128-token blocks (all column tiles):
// every mbarrier hand-off costs ~0.1 us of a warp's time, so per-tile
// hand-offs capped the converter at ~1.2 us per block; group A uses one
// named barrier per sub-block and leaves per-warp partial sums for group B.

// 16 warps = 4 per scheduler quadrant: 128 registers per thread (18 warps
// put 5 on two quadrants and capped the kernel at 96, with spills)
constexpr int VQ_A = 6, VQ_B0 = 6, VQ_CV0 = 10, VQ_CONV = 4, VQ_PROD = 14, VQ_MMA = 15;
constexpr int VQ_THREADS = (VQ_MMA + 1) * 32;
constexpr int VQ_SUB = 384;                 // tokens per digit sub-block (one pair per group-A thread)
constexpr int VQ_NB = VQ_SUB / TILE_M;      // 128-token blocks per sub-block
// digits per block: 16 rows x 128 tokens of s8 (2 KB) or bf16 (4 KB)
template <int BITS>
constexpr int vq_pblk() { return BITS == 16 ? 4096 : 2048; }
constexpr int VQ_STAGE = TILE_M * 128;      // one (block, 128-column tile) u8 operand;
                                            // an operand ring slot holds NJ of them
constexpr int VQ_TMEM = 128;                // 2 buffers x up to 4 tiles x 16 columns
constexpr int VQ_PF = 8;                    // L2 prefetch distance of the code stream (blocks)
constexpr float VQ_W = 127.f * 254.f;       // digit weight scale
// D s32, A u8 (codes, MN-major), B s8 (digits, K-major), M 128, N 16
constexpr uint32_t IDESC_Q = (2u << 4) | (0u << 7) | (1u << 10) | (1u << 15) |
                             ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(TILE_M >> 4) << 24);
// raw bf16 values: D f32, A bf16 (MN-major), B bf16 (K-major), M 128, N 16
constexpr uint32_t IDESC_QB = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) |
                              ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(TILE_M >> 4) << 24);
constexpr int VQ_BSTAGE = TILE_M * 256;    // bf16: one (block, 128-column tile) stage, two 64-col boxes

struct VQParams {
  int B, n_heads, s, G, Rv_pad, T_cap, ld_logits;
  int row_bytes, box_bytes;  // packed row; raw-slot row pitch (= row_bytes: 1-D bulk copies)
  const uint8_t* codes;      // [B][G][T_cap][row_bytes] packed codes
  int raw_slots, stages, ns_cap;
  const int* t_dev;
  const float* logits;
  const float* scales;
  const float* zps;
  float *pm, *pl, *pctx;
  unsigned long long* trace;  // diagnostics (PALU_FUSED_TRACE): per-CTA timeline, else null
  int diag;  // diagnostic builds only (results invalid): 1 no MMAs, 2 no converter stores, 4 no converter loads
};

__device__ __forceinline__ void umma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum)
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

// Warps 0-3 of group A: one sub-block's integer accumulators (TMEM lane
// quarter = warp) -> online softmax across the unit's sub-blocks -> the
// unit's partial at its last sub-block (value_merge_kernel layout).
struct VQPend {
  int sb, b, g, s0u;
  bool first, last;
};
template <int BITS>
__device__ __forceinline__ void vq_readback(const VQParams& p, const VQPend& q, int NJ, int warp, int ta,
                                          int col_in, uint32_t tmem, const float* stat_m,
                                          const float* stat_l, const float* stat_z,
                                          uint64_t* pfull, uint64_t* dfull, uint64_t* dempty,
                                          float (&acc)[4][V_HP], float (&mr)[V_HP], float (&lr)[V_HP]) {
    const int buf = q.sb & 1;
    mbar_wait(&pfull[buf], (q.sb >> 1) & 1);  // every warp's partials (acquire)
    mbar_wait(&dfull[buf], (q.sb >> 1) & 1);  // the sub-block's accumulators
    fence_after();
    if (q.first) {
#pragma unroll
      for (int h = 0; h < V_HP; ++h) {
        mr[h] = -INFINITY;
        lr[h] = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j][h] = 0.f;
      }
    }
    float sc_old[V_HP], sc_new[V_HP];
    float zw[V_HP];
    const float scl = stat_m[buf * (V_HP + 1) + V_HP] / VQ_W;
#pragma unroll
    for (int h = 0; h < V_HP; ++h) {
      const float ms = stat_m[buf * (V_HP + 1) + h];
      float ls = 0.f;
      zw[h] = 0.f;
#pragma unroll
      for (int w = 0; w < VQ_A; ++w) {
        ls += stat_l[(buf * VQ_A + w) * V_HP + h];
        zw[h] += stat_z[(buf * VQ_A + w) * V_HP + h];
      }
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
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)((buf * NJ + j) * 16), v);
        tmem_wait_ld();
#pragma unroll
        for (int h = 0; h < V_HP; ++h) {
          if constexpr (BITS == 16) {
            acc[j][h] = acc[j][h] * sc_old[h] + (v[h] + v[h + V_HP]) * sc_new[h];
          } else {
            // exact integer sum of the two digit planes, then the zero-point term
            const long long r = 254ll * __float_as_int(v[h]) + __float_as_int(v[h + V_HP]);
            acc[j][h] = acc[j][h] * sc_old[h] + (__ll2float_rn(r) + zw[h]) * scl * sc_new[h];
          }
        }
      }
    }
    fence_before();
    named_bar_sync(4, 128);
    if (ta == 0) mbar_arrive(&dempty[buf]);
    if (q.last) {
      // the unit's partial (value_merge_kernel layout): slot = first super-tile
      for (int j = 0; j < NJ && j < 4; ++j) {
        const int col = j * 128 + col_in;
#pragma unroll
        for (int h = 0; h < V_HP; ++h)
          if (h < p.s)
            p.pctx[(((size_t)q.b * p.n_heads + q.g * p.s + h) * p.ns_cap + q.s0u) * p.Rv_pad + col] =
                acc[j][h];
      }
#pragma unroll
      for (int h = 0; h < V_HP; ++h)
        if (ta == h && h < p.s) {
          const size_t pi = ((size_t)q.b * p.n_heads + q.g * p.s + h) * p.ns_cap + q.s0u;
          p.pm[pi] = mr[h];
          p.pl[pi] = lr[h];
        }
    }
  }

template <int BITS>
__global__ void __launch_bounds__(VQ_THREADS, 1)
value_q_kernel(const __grid_constant__ CUtensorMap map_c, const VQParams p) {
  // codes of older tokens stream while the score kernel drains; the producer
  // waits before the newest token's block, group A before the logits
  pdl_launch();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int NJ = p.Rv_pad / 128;
  const int RB = TILE_M * p.row_bytes;
  const int RS = RB;                                             // raw slot: the block's codes
  // operand ring slot: a whole block of u8 tiles; bf16: one 32 KB tile
  const int OB = BITS == 16 ? VQ_BSTAGE : NJ * VQ_STAGE;
  uint8_t* ring = smem;                                          // stages x OB
  uint8_t* pbuf = ring + p.stages * OB;                          // 2 x 8 KB digits
  constexpr int PBLK = vq_pblk<BITS>(), PBUF = VQ_NB * PBLK;
  uint8_t* raw = pbuf + 2 * PBUF;                                // raw_slots x RS
  // per sub-block buffer: max logit per head + max scale (group A), and
  // per-warp partial sums of p and of the int64 zero-point term
  float* stat_m = reinterpret_cast<float*>(raw + (size_t)p.raw_slots * RS);  // [2][V_HP + 1]
  float* stat_l = stat_m + 2 * (V_HP + 1) + 2;                               // [2][VQ_A][V_HP]
  float* stat_z = stat_l + 2 * VQ_A * V_HP;                                  // [2][VQ_A][V_HP]
  uint64_t* full = reinterpret_cast<uint64_t*>(stat_z + 2 * VQ_A * V_HP);
  uint64_t* empty = full + p.stages;
  uint64_t* rfull = empty + p.stages;
  uint64_t* rempty = rfull + p.raw_slots;
  uint64_t* pfull = rempty + p.raw_slots;  // [2] digits + statistics written
  uint64_t* dfull = pfull + 2;             // [2] sub-block accumulators complete
  uint64_t* dempty = dfull + 2;            // [2] sub-block accumulators read back
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dempty + 2);
  uint64_t* lgready = reinterpret_cast<uint64_t*>(tslot + 2);  // group A holds its first logits
  __shared__ float red_m[2][VQ_A][V_HP + 1];  // per-warp max logit per head + max scale

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int T_rows = *p.t_dev + 1;  // final: advanced by the previous step's last launch
  const int n_super = (T_rows + SUPER - 1) / SUPER;
  const int total = p.B * p.G * n_super;
  const int per = (total + (int)gridDim.x - 1) / (int)gridDim.x;
  const int i0 = min(total, (int)blockIdx.x * per), i1 = min(total, i0 + per);

  if (tid == 0) {
    for (int st = 0; st < p.stages; ++st) {
      mbar_init(&full[st], BITS == 16 ? 1 : VQ_CONV);  // TMA tx | one arrive per converter warp
      mbar_init(&empty[st], 1);
    }
    for (int r = 0; r < p.raw_slots; ++r) {
      mbar_init(&rfull[r], 1);
      mbar_init(&rempty[r], VQ_CONV);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&pfull[a], VQ_A);  // one arrive per group-A warp
      mbar_init(&dfull[a], 1);
      mbar_init(&dempty[a], 1);
    }
    mbar_init(lgready, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // digit rows 8..15 of every block stay zero (N = 16 > 4 heads x 2 digits)
  // (u8 digits: per block one 1 KB group of 8 rows each; bf16 digits: per
  // 64-token atom of a block)
  for (int i = tid; i < 2 * PBUF / 2048 * 64; i += VQ_THREADS) {
    const int a = i >> 6, w = i & 63;
    reinterpret_cast<uint4*>(pbuf + a * 2048 + 1024)[w] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (warp == VQ_MMA) {
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
  unsigned long long* tr = p.trace ? p.trace + (size_t)blockIdx.x * TRACE_STRIDE : nullptr;
  // SM clock (cheap; %globaltimer reads cost ~0.1 us); slots 0 / 1 keep the
  // global timer for cross-CTA alignment, slot 2 the clock at entry
  auto mark = [&](int slot) {
    if (tr != nullptr && slot < TRACE_STRIDE) tr[slot] = slot < 2 ? gtimer() : (unsigned long long)clock64();
  };
  if (tid == 0 && tr != nullptr) {
    tr[2] = (unsigned long long)clock64();
    mark(0);
  }

  if (warp == VQ_PROD) {
    // ---------------- producer: one 1-D bulk copy per 128-token block ----------------
    if (lane == 0) {
      VQIter it(i0, i1, n_super);
      Ring rg;
      bool waited = false;
      int kblk = 0;
      const uint64_t pol_first = policy_evict_first();  // codes are read once: keep L2 for the logits
      // L2 prefetch cursor VQ_PF blocks ahead of the loads: the HBM latency
      // then overlaps the ring turnaround instead of gating it
      VQIter pit(i0, i1, n_super);
      int pbg = 0, pc = 0, pc1 = 0;
      auto prefetch_next = [&]() {
        if (pc >= pc1) {
          int a, b;
          if (!pit.next(pbg, a, b)) return;
          pc = a * SUPER;
          pc1 = min(T_rows, b * SUPER);
        }
        bulk_prefetch_l2(p.codes + ((size_t)pbg * p.T_cap + pc) * p.row_bytes, RB);
        pc += TILE_M;
      };
      // start-up: every SM's first loads (~30 MB chip-wide with the L2
      // prefetches) queue ahead of group A's logits reads (the score kernel's
      // output, no longer in L2), holding the first digits back by several
      // us; after V_HEAD_START blocks the producer lets the logits through
      int nblk_issued = 0;
      bool released = false;
      auto gate = [&]() {
        if (released) {
          prefetch_next();
        } else if (nblk_issued == V_HEAD_START) {
          mbar_wait(lgready, 0);
          released = true;
          for (int k = 0; k < VQ_PF; ++k) prefetch_next();
        }
        ++nblk_issued;
      };
      if constexpr (BITS == 16) prefetch_map(&map_c);
      while (BITS == 16 && it.next(bg, s0u, s1u)) {
        // raw bf16: per block and 128-column tile two {64 col, 128 token} SW128
        // boxes straight into the MN-major operand stage
        const int c0 = s0u * SUPER, c1 = min(T_rows, s1u * SUPER);
        for (int t0 = c0; t0 < c1; t0 += TILE_M) {
          gate();
          if (!waited && t0 + TILE_M >= T_rows) {
            pdl_wait();
            waited = true;
          }
          mark(8 + min(kblk++, 47));
          for (int j = 0; j < NJ; ++j, rg.next(p.stages)) {
            mbar_wait(&empty[rg.slot], rg.phase ^ 1);
            mbar_expect_tx(&full[rg.slot], VQ_BSTAGE);
            uint8_t* dst = ring + (size_t)rg.slot * OB;
            tma_load_2d(&map_c, &full[rg.slot], dst, j * 128, bg * p.T_cap + t0);
            tma_load_2d(&map_c, &full[rg.slot], dst + VQ_BSTAGE / 2, j * 128 + 64, bg * p.T_cap + t0);
          }
        }
      }
      while (BITS != 16 && it.next(bg, s0u, s1u)) {
        const int c0 = s0u * SUPER, c1 = min(T_rows, s1u * SUPER);
        for (int t0 = c0; t0 < c1; t0 += TILE_M) {
          gate();
          // the newest token (row T_rows - 1) comes from this step's append
          if (!waited && t0 + TILE_M >= T_rows) {
            pdl_wait();
            waited = true;
          }
          mbar_wait(&rempty[rg.slot], rg.phase ^ 1);
          mark(8 + min(kblk++, 47));
          // a block of one (sequence, group) is one contiguous range of the cache
          mbar_expect_tx(&rfull[rg.slot], RB);
          bulk_load_hint(raw + (size_t)rg.slot * RS, p.codes + ((size_t)bg * p.T_cap + t0) * p.row_bytes,
                    (uint32_t)RB, &rfull[rg.slot], pol_first);
          rg.next(p.raw_slots);
        }
      }
    }
  } else if (warp >= VQ_CV0 && warp < VQ_CV0 + VQ_CONV) {
    if constexpr (BITS != 16) {
    // ---------------- converters: packed block -> u8 MN-major SW128 tiles ----------------
    // work item (row, q) = 16-byte raw chunk q of the row's slice of column
    // tile j; RCR consecutive lanes share a row (conflict-free raw reads)
    constexpr int RCR = BITS;                     // raw chunks per row per 128 columns
    constexpr int RC = RCR * TILE_M / (VQ_CONV * 32);  // items per thread per column tile
    constexpr int OC = 8 / BITS;                  // output 16-byte chunks per raw chunk
    const int ct = tid - VQ_CV0 * 32;
    // per-thread item geometry is the same for every block and column tile:
    // raw source offsets and swizzled destination offsets, computed once
    uint32_t src_off[RC], dst_off[RC][OC];
#pragma unroll
    for (int k = 0; k < RC; ++k) {
      const int w = ct + VQ_CONV * 32 * k;
      const int row = w / RCR, q = w % RCR;
      src_off[k] = (uint32_t)(row * p.row_bytes + 16 * q);
#pragma unroll
      for (int e = 0; e < OC; ++e) dst_off[k][e] = (uint32_t)(row * 128 + (((OC * q + e) ^ (row & 7)) << 4));
    }
    VQIter it(i0, i1, n_super);
    Ring rr, rs;
    int kblk = 0;
    while (it.next(bg, s0u, s1u)) {
      const int c0 = s0u * SUPER, c1 = min(T_rows, s1u * SUPER);
      for (int t0 = c0; t0 < c1; t0 += TILE_M, ++kblk) {
        mbar_wait(&rfull[rr.slot], rr.phase);
        mbar_wait(&empty[rs.slot], rs.phase ^ 1);
        if (ct == 0) mark(56 + min(kblk, 47));
        const uint32_t slot = smem_u32(raw + (size_t)rr.slot * RS);
        const uint32_t ob = smem_u32(ring + (size_t)rs.slot * OB);
        for (int j = 0; j < NJ; ++j) {
          // all of this tile's raw chunks first (the stores below are volatile
          // asm: loads issued after them would serialise)
          uint4 vv[RC];
#pragma unroll
          for (int k = 0; k < RC; ++k) vv[k] = lds128(slot + src_off[k] + j * 16 * BITS);
          const uint32_t st = ob + j * VQ_STAGE;
#pragma unroll
          for (int k = 0; k < RC; ++k) {
            const uint4 v = vv[k];
            if constexpr (BITS == 8) {
              asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(st + dst_off[k][0]),
                           "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                           : "memory");
            } else {
              // nibbles / crumbs -> bytes: chunk e holds bits [BITS e, BITS e + BITS) of every byte
              constexpr uint32_t M = BITS == 4 ? 0x0F0F0F0Fu : 0x03030303u;
#pragma unroll
              for (int e = 0; e < OC; ++e)
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(st + dst_off[k][e]),
                             "r"((v.x >> (BITS * e)) & M), "r"((v.y >> (BITS * e)) & M),
                             "r"((v.z >> (BITS * e)) & M), "r"((v.w >> (BITS * e)) & M)
                             : "memory");
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&full[rs.slot]);
          mbar_arrive(&rempty[rr.slot]);
        }
        if (ct == 0) mark(104 + min(kblk, 47));
        rr.next(p.raw_slots);
        rs.next(p.stages);
      }
    }
    }
  } else if (warp == VQ_MMA) {
    // ---------------- MMA issuer ----------------
    // the whole warp runs the loop (descriptors stay warp-uniform); one
    // elected lane issues the tcgen05 instructions
    {
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
          if (lane == 0) mark(152 + min(sb, 15));
          const uint32_t pb = smem_u32(pbuf + buf * PBUF);
          const int b1 = min(nblk, b0 + VQ_NB);
          for (int blk = b0; BITS == 16 && blk < b1; ++blk)
            for (int j = 0; j < NJ; ++j, rs.next(p.stages)) {
              mbar_wait(&full[rs.slot], rs.phase);
              fence_after();
              const uint32_t d = tmem + (uint32_t)((buf * NJ + j) * 16);
              const uint32_t a0 = smem_u32(ring + rs.slot * OB);
              if (elect_one()) {
                if ((p.diag & 1) == 0)
#pragma unroll
                  for (int kk = 0; kk < TILE_M / 16; ++kk)  // K = 16 tokens: 2 KB of A (2 slabs)
                    umma_bf16_id(d, sdesc_mn(a0 + kk * 2048, VQ_BSTAGE / 2, 1024),
                                 sdesc(pb + (blk - b0) * PBLK + (kk >> 2) * 2048 + (kk & 3) * 32), IDESC_QB,
                                 (blk != b0) || (kk != 0));
                umma_commit(&empty[rs.slot]);
              }
              __syncwarp();
            }
          for (int blk = b0; BITS != 16 && blk < b1; ++blk, rs.next(p.stages)) {
            mbar_wait(&full[rs.slot], rs.phase);
            fence_after();
            const uint64_t db = sdesc(pb + (blk - b0) * PBLK);
            if (elect_one()) {
              for (int j = 0; j < NJ; ++j) {
                const uint32_t d = tmem + (uint32_t)((buf * NJ + j) * 16);
                const uint64_t da = sdesc_mn(smem_u32(ring + rs.slot * OB + j * VQ_STAGE), VQ_STAGE, 1024);
                if ((p.diag & 1) == 0)
#pragma unroll
                  for (int kk = 0; kk < TILE_M / 32; ++kk)  // K = 32 tokens: 4 KB of A, 32 B of B
                    umma_i8(d, da + (uint64_t)(kk * 256), db + (uint64_t)(kk * 2), IDESC_Q,
                            (blk != b0) || (kk != 0));
              }
              umma_commit(&empty[rs.slot]);
            }
            __syncwarp();
          }
          if (elect_one()) umma_commit(&dfull[buf]);
          __syncwarp();
          if (lane == 0) mark(168 + min(sb, 15));
        }
      }
    }
  } else if (warp < VQ_A) {
    // ---------------- group A (warps 0-7): logits -> statistics -> digits ----------------
    // thread = one token pair of each 512-token sub-block; one named barrier
    // per sub-block (max logit per head, max scale); the sums of p and of the
    // zero-point term are left as per-warp partials for the readback
    pdl_wait();  // logits (score kernel), scales / zero points of the newest token
    constexpr int NT = VQ_A * 32;
    const int ta = tid;
    VQIter it(i0, i1, n_super);
    int sb = 0;
    while (it.next(bg, s0u, s1u)) {
      const int b = bg / p.G, g = bg - b * p.G;
      const int c0 = s0u * SUPER, c1 = min(T_rows, s1u * SUPER);
      const int nt = c1 - c0;
      const int ntok = (nt + TILE_M - 1) / TILE_M * TILE_M;
      const float* lg = p.logits + ((size_t)b * p.n_heads + g * p.s) * p.ld_logits + c0;
      const float* sc = p.scales + (size_t)bg * p.T_cap + c0;
      const float* zp = p.zps + (size_t)bg * p.T_cap + c0;
      const uint64_t pol_drop = policy_evict_first();  // the logits are dead after this read
      float2 x[V_HP], xn[V_HP], sv, svn, zv, zvn;
      // the sub-block's logits, scales and zero points; the next sub-block's
      // are in flight while this one runs
      // (no value-dependent masking here: any op on a loaded register would
      // wait for the load and turn the prefetch into a synchronous read; the
      // masks are applied where the values are used)
      auto load = [&](int s0, float2 (&dst)[V_HP], float2& sd, float2& zd) {
        const int t = s0 + 2 * ta;
#pragma unroll
        for (int h = 0; h < V_HP; ++h) {
          float2 v = make_float2(0.f, 0.f);
          if (h < p.s && t < nt) v = ldg64_cg_hint(lg + (size_t)h * p.ld_logits + t, pol_drop);
          dst[h] = v;
        }
        sd = make_float2(1.f, 1.f);
        zd = make_float2(0.f, 0.f);
        if (BITS != 16 && t < nt) {
          sd.x = __ldg(sc + t);
          zd.x = __ldg(zp + t);
          if (t + 1 < nt) {
            sd.y = __ldg(sc + t + 1);
            zd.y = __ldg(zp + t + 1);
          }
        }
      };
      load(0, xn, svn, zvn);
      for (int s0 = 0; s0 < ntok; s0 += VQ_SUB, ++sb) {
        const int buf = sb & 1;
        {
          const int t = s0 + 2 * ta;
#pragma unroll
          for (int h = 0; h < V_HP; ++h)
            x[h] = make_float2(h < p.s && t < nt ? xn[h].x : -INFINITY,
                               h < p.s && t + 1 < nt ? xn[h].y : -INFINITY);
        }
        sv = svn;
        zv = zvn;
        if (s0 + VQ_SUB < ntok) load(s0 + VQ_SUB, xn, svn, zvn);
        if (ta == 0) mark(184 + min(sb, 15));
        // (1) max logit per head and max scale of the sub-block (red_m is
        // double-buffered: the next sub-block's writes cannot race these reads)
        float m[V_HP + 1];
#pragma unroll
        for (int h = 0; h < V_HP; ++h) m[h] = fmaxf(x[h].x, x[h].y);
        m[V_HP] = fmaxf(sv.x, sv.y);
#pragma unroll
        for (int h = 0; h <= V_HP; ++h) {
          m[h] = warp_reduce(m[h], [](float a, float c) { return fmaxf(a, c); });
          if (lane == 0) red_m[buf][warp][h] = m[h];
        }
        if (ta == 0) mark(300 + min(sb, 15));
        named_bar_sync(3, NT);
        if (sb == 0 && ta == 0) mbar_arrive(lgready);  // every group-A thread holds its logits
        if (ta == 0) mark(316 + min(sb, 15));
#pragma unroll
        for (int h = 0; h <= V_HP; ++h) {
          float v = red_m[buf][0][h];
#pragma unroll
          for (int w = 1; w < VQ_A; ++w) v = fmaxf(v, red_m[buf][w][h]);
          m[h] = v;
        }
        // the digit buffer and statistics slot are free once sub-block sb - 2
        // was read back (by warps 0-3 of this group, one iteration ago)
        if (sb >= 2) mbar_wait(&dempty[buf], ((sb >> 1) - 1) & 1);
        if (ta == 0) mark(216 + min(sb, 15));
        // (2) p = exp(x - m), u = p s / max s in [0, 1]; digits w = 254 hi + lo
        const float inv = m[V_HP] > 0.f ? 127.f / m[V_HP] : 0.f;
        uint8_t* pb = pbuf + buf * PBUF;
        const int tl = 2 * ta;
        const bool live = s0 + tl < ntok;
        const int blk = tl >> 7, tk = tl & 127;
        uint8_t* rb = pb + blk * PBLK + (tk & 15);
        float l[V_HP];
        float zw[V_HP];
#pragma unroll
        for (int h = 0; h < V_HP; ++h) {
          l[h] = 0.f;
          zw[h] = 0.f;
          float w0 = 0.f, w1 = 0.f;
          if constexpr (BITS == 16) {
            // bf16 digit pair of p (rows h, h + 4; K-major SW128 atoms of 64
            // tokens, 16-byte chunk ((tk % 64) / 8) ^ row)
            uint8_t* ab = pb + blk * PBLK + (tk >> 6) * 2048 + (tk & 7) * 2;
            const int w8 = (tk & 63) >> 3;
            uint32_t hv = 0u, lv = 0u;
            if (h < p.s && live) {
              const float p0 = __expf(x[h].x - m[h]), p1 = __expf(x[h].y - m[h]);
              l[h] = p0 + p1;
              const __nv_bfloat162 hi = __floats2bfloat162_rn(p0, p1);
              const float2 hf = __bfloat1622float2(hi);
              const __nv_bfloat162 lo = __floats2bfloat162_rn(p0 - hf.x, p1 - hf.y);
              hv = *reinterpret_cast<const uint32_t*>(&hi);
              lv = *reinterpret_cast<const uint32_t*>(&lo);
            }
            if (live) {
              *reinterpret_cast<uint32_t*>(ab + h * 128 + (((w8 ^ h) & 7) << 4)) = hv;
              *reinterpret_cast<uint32_t*>(ab + (h + 4) * 128 + (((w8 ^ (h + 4)) & 7) << 4)) = lv;
            }
          } else if (h < p.s && live) {
            // round-to-nearest integers via the 1.5 * 2^23 magic constant: the
            // low byte of the float's bits is the two's-complement digit, so no
            // F2I / rint is needed; |lo| <= 127 since |v - hi| <= 0.5
            constexpr float MAGIC = 12582912.f;
            const float p0 = __expf(x[h].x - m[h]), p1 = __expf(x[h].y - m[h]);
            l[h] = p0 + p1;
            const float v0 = p0 * sv.x * inv, v1 = p1 * sv.y * inv;
            const float th0 = v0 + MAGIC, th1 = v1 + MAGIC;
            const float h0 = th0 - MAGIC, h1 = th1 - MAGIC;
            const float tl0 = fmaf(v0 - h0, 254.f, MAGIC), tl1 = fmaf(v1 - h1, 254.f, MAGIC);
            w0 = fmaf(254.f, h0, tl0 - MAGIC);  // exact integers < 2^15
            w1 = fmaf(254.f, h1, tl1 - MAGIC);
            // K-major SW128: row r, token tk -> 16-byte chunk (tk / 16) ^ (r & 7)
            *reinterpret_cast<uint16_t*>(rb + h * 128 + ((((tk >> 4) ^ h) & 7) << 4)) =
                (uint16_t)__byte_perm(__float_as_uint(th0), __float_as_uint(th1), 0x0040);
            *reinterpret_cast<uint16_t*>(rb + (h + 4) * 128 + ((((tk >> 4) ^ (h + 4)) & 7) << 4)) =
                (uint16_t)__byte_perm(__float_as_uint(tl0), __float_as_uint(tl1), 0x0040);
          } else if (live) {
            *reinterpret_cast<uint16_t*>(rb + h * 128 + ((((tk >> 4) ^ h) & 7) << 4)) = 0;
            *reinterpret_cast<uint16_t*>(rb + (h + 4) * 128 + ((((tk >> 4) ^ (h + 4)) & 7) << 4)) = 0;
          }
          // - sum w z in fp32: relative to the digit sums it carries ~1e-7
          if (BITS != 16) zw[h] = -fmaf(w0, zv.x, w1 * zv.y);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (ta == 0) mark(332 + min(sb, 15));
        // (3) per-warp partial sums; statistics; release this warp's digits
#pragma unroll
        for (int h = 0; h < V_HP; ++h) {
          l[h] = warp_reduce(l[h], [](float a, float c) { return a + c; });
          zw[h] = warp_reduce(zw[h], [](float a, float c) { return a + c; });
        }
        if (lane == 0) {
#pragma unroll
          for (int h = 0; h < V_HP; ++h) {
            stat_l[(buf * VQ_A + warp) * V_HP + h] = l[h];
            stat_z[(buf * VQ_A + warp) * V_HP + h] = zw[h];
          }
          if (warp == 0) {
#pragma unroll
            for (int h = 0; h <= V_HP; ++h) stat_m[buf * (V_HP + 1) + h] = m[h];
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[buf]);  // release: this warp's digits and partials
        if (ta == 0) mark(200 + min(sb, 15));
      }
    }
  } else {
    // ---------------- group B (warps 8-11): readback -> online softmax -> partial ----------------
    const int wq = warp & 3, tb = tid - VQ_B0 * 32;  // TMEM lane quarter = warp % 4
    const int col_in = vq_column<BITS>(wq * 32 + lane);
    float acc[4][V_HP], mr[V_HP], lr[V_HP];
    VQIter it(i0, i1, n_super);
    int sb = 0;
    while (it.next(bg, s0u, s1u)) {
      const int b = bg / p.G, g = bg - b * p.G;
      const int c0 = s0u * SUPER, c1 = min(T_rows, s1u * SUPER);
      const int nblk = (c1 - c0 + TILE_M - 1) / TILE_M;
      for (int b0 = 0; b0 < nblk; b0 += VQ_NB, ++sb) {
        const VQPend q = {sb, b, g, s0u, b0 == 0, b0 + VQ_NB >= nblk};
        vq_readback<BITS>(p, q, NJ, wq, tb, col_in, tmem, stat_m, stat_l, stat_z, pfull, dfull, dempty,
                          acc, mr, lr);
      }
    }
  }
  fence_before();
  __syncthreads();
  if (tid == 0) {
    mark(1);
    if (tr != nullptr) tr[3] = 2000000ull + (unsigned long long)(i1 - i0);
  }
  if (warp == VQ_MMA) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(VQ_TMEM));
  }
}
