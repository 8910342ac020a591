// tcgen05 (sm_100a) RoPE score kernel: online key reconstruction on the
// 5th-gen tensor cores with TMA-staged latents and a TMEM accumulator.
//
// Restates attention.py:433-444 (palu_decode_step_rope, per group and token
// tile: K_tile = H_tile @ B_g, RoPE at absolute positions, q . k / sqrt(d_h))
// in the query-absorbed form of palu_query_absorb:
//
//   logit[t, head] = sum_j cos(t th_j) (H_t . u_j) + sin(t th_j) (H_t . w_j)
//
// so the dense contraction is one GEMM per (sequence, group, head pair):
//   ACC[128 tokens x 256] = H[128 x R] (smem, TMA, 128B swizzle)
//                          x UW[256 x R]^T (smem, resident for the CTA)
// accumulated in TMEM (2 x 256 columns, double buffered across tiles), and
// the RoPE + q-dot collapses to a cos/sin-weighted row reduction in the
// epilogue (tcgen05.ld 32x32b: one thread = one token).
//
// Warp roles (320 threads): warp 0 TMA producer, warp 1 MMA issuer + TMEM
// owner, warps 2..9 epilogue (warp w reads TMEM lane quarter w % 4 and the
// pair half (w - 2) / 4 of the 64 RoPE frequencies).
#include <cuda.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "palu_sm100.cuh"
#include "palu_tmap.cuh"

namespace palu {
namespace tc {

constexpr int PF_DIST = 0;         // L2 prefetch distance (work items); 0 measured best with PDL split (tools/pf_sweep.sh)
constexpr int SUPER = 2 * TILE_M;  // tokens per work item (the CTA pair)
constexpr int HEAD_BYTES = TILE_M * 128;  // one head's 128 UW rows x 64 bf16

struct VParams;  // value role of the fused kernel (below)

struct Params {
  int B, n_heads, s_k, G, R_pad, T_cap, ld_logits, n_tab, stages;
  int score_pairs;  // CTA pairs running the score role (fused kernel); all pairs otherwise
  int* ready;       // fused: per work item, epilogue warps that published its logits
  int mode;     // profiling only (bit flags): 1 epilogue skips math; 2 MMA skips TMA waits; 4 MMA skips TMEM-empty waits
  int pf_dist;  // L2 prefetch distance in work items (0 = off)
  int pdl_split;  // 0: wait for the predecessor at entry (A/B diagnostics)
  const float2* rope_tab;  // [n_tab + 128][64]
  // weights of a later kernel (the layer's output projection) to bring into
  // L2 with an evict-last policy while this tensor-bound kernel leaves HBM
  // bandwidth idle; the latent streams load evict-first
  const uint8_t* l2pf;
  long long l2pf_bytes;
  const int* t_dev;
  float* logits;
  unsigned long long* trace;  // diagnostics only (PALU_FUSED_TRACE): [CTA][TRACE_STRIDE]
  // quantised keys (bits 2/3/4/8): packed LE codes [B][G][T_cap][code_row_bytes]
  // (quant.py:156-169 order) and per-token fp32 scale / zero point
  int bits, code_row_bytes;
  const uint8_t* codes;
  const float* scales;
  const float* zps;
  // replicated-B groups (QH > 1): scale x RoPE(q) rows, float [B][n_heads][128]
  const float* qrot;
};

constexpr int TRACE_STRIDE = 512;
constexpr int SU = 8;  // score trace marks per accumulator unit
// score epilogue shared memory: the cross-warp reduction buffer, then per
// epilogue warp two (cos/sin base half-row 256 B, lane scales 128 B) buffers
// (+ for replicated-B groups two buffers of the QH rotated query slices)
constexpr int EPI_MAXW = SCORE_EPI > EPI_WARPS ? SCORE_EPI : EPI_WARPS;
constexpr int epi_red_bytes(int nout) { return 4 * (EPI_MAXW / 4 - 1) * (nout < 2 ? 2 : nout) * 128 * 4; }
constexpr int epi_stage_bytes(int qh) { return 2 * 256 + 2 * 128 + (qh > 1 ? 2 * qh * 256 : 0); }
constexpr int score_fixed_bytes(int nout, int qh) {
  return 512 + epi_red_bytes(nout) + EPI_MAXW * epi_stage_bytes(qh);
}
constexpr int SCORE_FIXED_BYTES = score_fixed_bytes(2, 1);

// Profiling modes that skip MMAs or barrier waits (results invalid) exist only
// in diagnostic builds (-DPALU_DIAG); the product library ignores the knobs.
#ifdef PALU_TRACE
constexpr bool kTrace = true;   // per-CTA timelines (tools/score_trace.py, fused_trace.py)
#else
constexpr bool kTrace = false;
#endif
#ifdef PALU_DIAG
constexpr bool kDiag = true;
#else
constexpr bool kDiag = false;
#endif
#ifdef PALU_DIAG
static int diag_env(const char* name) { return getenv(name) ? atoi(getenv(name)) : 0; }
#else
static int diag_env(const char*) { return 0; }
#endif
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid_u32() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

constexpr int CONV_WARPS = 2;    // rope-off latent score: code -> bf16 converter warps per SM
// rope-on score: 4 converter warps (one token row per lane).  2 warps (two
// rows per lane) left the int4-key score at 173 us vs 99 us for bf16 keys;
// 12 warps per CTA still fit the 168-register budget (3 per scheduler quadrant)
constexpr int CODE_BIAS = 128;   // bits <= 4: bf16(128 + c) has bit pattern 0x4300 | c

// Unpack this SM's 128-token tile of packed key codes into the SW128 K-major
// bf16 H stages (the layout TMA would produce), one k-block per stage, and
// signal the leader's full barrier.  Lane cl owns rows cl and cl + 64; the
// next k-block's packed bytes are loaded while the current one is written.
// The operand holds c - z (quant.py:106-107 without the scale): for bits <= 4
// bf16(128 + c) is built with the exponent trick and (128 + z) subtracted in
// bf16x2 (exact when |z| <= 128), else c - z goes through fp32 and one bf16
// rounding; the epilogue multiplies by s.  quant.py:156-169 bit order (code
// k at bits [k b, (k + 1) b)).
// Position in an n-deep mbarrier ring (slot, phase parity), advanced
// incrementally: a runtime modulo per step is an integer-division chain
// (~100 dependent clocks) on the issuing thread.
// (sequence x group, super-tile) of consecutive work items without a
// per-item division (the score roles walk their items in order)
struct ItemPos {
  int bg, st, b, g;
  __device__ __forceinline__ ItemPos(int i, int n_super, int G) {
    bg = i / n_super;
    st = i - bg * n_super;
    b = bg / G;
    g = bg - b * G;
  }
  __device__ __forceinline__ void next(int n_super, int G) {
    if (++st == n_super) {
      st = 0;
      ++bg;
      if (++g == G) {
        g = 0;
        ++b;
      }
    }
  }
};


// A converter warp hands its operand rows over with a CTA-local arrive on its
// own SM's full[stage] (release.cta: no memory barrier).  A cluster-scope
// release from the converter itself compiles to MEMBAR.GPU, which waits for
// the warp's in-flight code prefetch loads: it made the prefetch synchronous
// and cost ~30 % of the packed-key score kernel (int4 r 256: 154 -> 110 us).
// On the peer SM, warp 1 (idle: only the leader issues MMAs) relays each
// completed stage to the leader with the cluster-scope release; the leader's
// MMA issuer acquires at cluster scope.
__device__ __forceinline__ void conv_arrive(uint64_t* bar) { mbar_arrive(bar); }

template <int BITS, int RPL, class PP>
__device__ __forceinline__ void convert_tile(const PP& p, uint8_t* s_h, uint64_t* full,
                                             uint64_t* empty, int bg, int tile, int T_rows,
                                             int kblocks, int cl, Ring& rg) {
  constexpr int NW = BITS;  // 8-byte words per row per 64-code k-block
  const int lane = threadIdx.x & 31;
  const uint8_t* rowp[RPL];
  bool ok[RPL];
  float zr[RPL];
#pragma unroll
  for (int rr = 0; rr < RPL; ++rr) {
    const int t = tile * TILE_M + cl + (TILE_M / RPL) * rr;
    ok[rr] = t < T_rows;
    const size_t tok = (size_t)bg * p.T_cap + (ok[rr] ? t : 0);
    rowp[rr] = p.codes + tok * p.code_row_bytes;
    zr[rr] = ok[rr] ? __ldg(p.zps + tok) : 0.f;
  }
  if constexpr (BITS == 2 || BITS == 4) {
    // fast path: rank order inside each group of 32/BITS codes is permuted
    // (UW is written with the same permutation by palu_query_absorb layouts
    // 2/3) so that one 32-bit word yields bf16 pairs (c_k, c_{k+G/2}) with a
    // shift and a LOP3: 0x43004300 | ((w >> BITS k) & mask)
    constexpr uint32_t MASK = BITS == 4 ? 0x000F000Fu : 0x00030003u;
    constexpr int NV = 2 * BITS / 4;  // uint4 loads per row per k-block (32 B int4, 16 B int2)
    const uint64_t pol = policy_evict_first();  // codes are read once: keep L2 for the logits
    uint4 nx[RPL][2], cu[RPL][2];
    auto load4 = [&](int kb) {
#pragma unroll
      for (int rr = 0; rr < RPL; ++rr)
#pragma unroll
        for (int q = 0; q < NV; ++q)
          nx[rr][q] = ok[rr] ? ldg128_hint(reinterpret_cast<const uint4*>(rowp[rr] + kb * 8 * BITS) + q, pol)
                             : make_uint4(0u, 0u, 0u, 0u);
    };
    load4(0);
    for (int kb = 0; kb < kblocks; ++kb, rg.next(p.stages)) {
#pragma unroll
      for (int rr = 0; rr < RPL; ++rr)
#pragma unroll
        for (int q = 0; q < NV; ++q) cu[rr][q] = nx[rr][q];
      if (kb + 1 < kblocks) load4(kb + 1);
      const int stage = rg.slot;
      mbar_wait(&empty[stage], rg.phase ^ 1);
      uint8_t* sb = s_h + stage * H_STAGE_BYTES;
#pragma unroll
      for (int rr = 0; rr < RPL; ++rr) {
        const int row = cl + (TILE_M / RPL) * rr;
        const uint32_t words[8] = {cu[rr][0].x, cu[rr][0].y, cu[rr][0].z, cu[rr][0].w,
                                   cu[rr][1].x, cu[rr][1].y, cu[rr][1].z, cu[rr][1].w};
        // c - z: one bf16x2 subtract of (128 + z) from (128 + c), exact when
        // |z| <= 128; otherwise through fp32 (one bf16 rounding of c - z)
        const bool zsmall = fabsf(zr[rr]) <= 128.f;
        const __nv_bfloat162 zb = __float2bfloat162_rn((float)CODE_BIAS + zr[rr]);
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          // int4: word ch -> pairs k = 0..3; int2: word ch / 2 -> pairs 4 (ch & 1) + 0..3
          const uint32_t w = BITS == 4 ? words[ch] : words[ch >> 1];
          const int k0 = BITS == 4 ? 0 : 4 * (ch & 1);
          uint32_t wv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t cc = (w >> (BITS * (k0 + e))) & MASK;
            __nv_bfloat162 v;
            if (zsmall) {
              const uint32_t biased = 0x43004300u | cc;
              v = __hsub2(*reinterpret_cast<const __nv_bfloat162*>(&biased), zb);
            } else {
              v = __floats2bfloat162_rn((float)(cc & 0xFFFFu) - zr[rr], (float)(cc >> 16) - zr[rr]);
            }
            wv[e] = *reinterpret_cast<const uint32_t*>(&v);
          }
          const uint32_t dst = smem_u32(sb + row * 128 + ((ch ^ (row & 7)) << 4));
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(wv[0]), "r"(wv[1]),
                       "r"(wv[2]), "r"(wv[3])
                       : "memory");
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        conv_arrive(&full[stage]);
    }
    return;
  }
  unsigned long long nxt[RPL][NW], cur[RPL][NW];
  auto load = [&](int kb) {
#pragma unroll
    for (int rr = 0; rr < RPL; ++rr)
#pragma unroll
      for (int q = 0; q < NW; ++q)
        nxt[rr][q] = ok[rr] ? __ldg(reinterpret_cast<const unsigned long long*>(rowp[rr] + kb * 8 * BITS) + q)
                            : 0ull;
  };
  load(0);
  for (int kb = 0; kb < kblocks; ++kb, rg.next(p.stages)) {
#pragma unroll
    for (int rr = 0; rr < RPL; ++rr)
#pragma unroll
      for (int q = 0; q < NW; ++q) cur[rr][q] = nxt[rr][q];
    if (kb + 1 < kblocks) load(kb + 1);
    const int stage = rg.slot;
    mbar_wait(&empty[stage], rg.phase ^ 1);
    uint8_t* sb = s_h + stage * H_STAGE_BYTES;
#pragma unroll
    for (int rr = 0; rr < RPL; ++rr) {
      const int row = cl + (TILE_M / RPL) * rr;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {  // 8 codes -> one 16-byte swizzled chunk
        uint32_t wv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint32_t c2[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int bit = (ch * 8 + 2 * e + h) * BITS;  // within the k-block
            const int wd = bit >> 6, sh = bit & 63;
            unsigned long long v = cur[rr][wd] >> sh;
            if (sh + BITS > 64 && wd + 1 < NW) v |= cur[rr][wd + 1] << (64 - sh);
            c2[h] = (uint32_t)v & ((1u << BITS) - 1u);
          }
          const __nv_bfloat162 b2 =
              __floats2bfloat162_rn((float)c2[0] - zr[rr], (float)c2[1] - zr[rr]);
          wv[e] = *reinterpret_cast<const uint32_t*>(&b2);
        }
        const uint32_t dst = smem_u32(sb + row * 128 + ((ch ^ (row & 7)) << 4));
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(wv[0]), "r"(wv[1]),
                     "r"(wv[2]), "r"(wv[3])
                     : "memory");
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0)
      conv_arrive(&full[stage]);
  }
}

// Work item = (sequence b, key group g, 256-token super-tile) for a CTA pair
// (cluster of 2, cta_group::2).  SM r of the pair loads tokens
// [256 st + 128 r, +128) of H once and the UW rows of head 2h + r for each head
// pair h of the group; the leader SM issues
//   ACC_h[256 tokens x 256] += H[256 x 64] x UW_h[256 x 64]^T   (per k-block)
// whose rows 128 r .. land in SM r's TMEM.  Each SM's epilogue reduces its
// own 128 tokens x 2 heads per head pair.  Every latent byte crosses L2 -> SM
// once and both SMs' tensor pipes run at the 2-SM rate.
// UH = heads per accumulator unit.  UH 2: one M256 x N256 MMA covers a head
// pair (each SM holds the UW rows of one head), 2 TMEM slots of 256 columns.
// UH 1: one M256 x N128 MMA per head (each SM holds half of every head's UW
// rows: u_j on the leader, w_j on the peer), 4 slots of 128 columns -- for
// short ranks (r <= 128: 8 MMAs per unit) the accumulator must be quad-
// buffered to cover the ~1 us from a unit's last MMA issue to its epilogue
// (tools/score_trace.py: 2 slots left the tensor pipe ~45 % idle at r 128).
template <int UH, int NCONV, int EW, int QH = 1>
__device__ __forceinline__ void score_role(const CUtensorMap& map_h, const CUtensorMap& map_uw,
                                           const Params& p, uint8_t* smem) {
  constexpr int NSLOT = UH == 2 ? 2 : 4;
  constexpr int SLOT_COLS = 128 * UH;
  constexpr int UWB = HEAD_BYTES / 2 * UH;               // UW bytes per (k-block, unit) per SM
  constexpr uint32_t IDESC_U = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(SLOT_COLS >> 3) << 17) |
                               ((uint32_t)(256 >> 4) << 24);
  const int kblocks = p.R_pad / KB;
  const int units = p.s_k / UH;                          // accumulator units per item
  uint8_t* s_uw = smem;                                  // [kblocks][units] x UWB
  uint8_t* s_h = smem + kblocks * units * UWB;           // stages x 16 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_h + p.stages * H_STAGE_BYTES);
  uint64_t* full = bars;                                 // [stages]   (leader's used)
  uint64_t* empty = bars + p.stages;                     // [stages]   (each SM's own)
  uint64_t* tfull = bars + 2 * p.stages;                 // [NSLOT]    (each SM's own)
  uint64_t* tempty = tfull + NSLOT;                      // [NSLOT]    (leader's used)
  uint64_t* uw_full = tempty + NSLOT;                    // [1]        (leader's used)
  uint64_t* uw_empty = uw_full + 1;                      // [1]        (each SM's own)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(uw_empty + 1);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);  // [NSLOT][UH heads][128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mode = kDiag ? p.mode : 0;  // profiling modes exist in diagnostic builds only
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair_id = blockIdx.x >> 1, n_pairs = p.score_pairs;
  const int T_rows = *p.t_dev + 1;
  const int n_super = (T_rows + SUPER - 1) / SUPER;
  const int total = p.B * p.G * n_super;
  const int per = (total + n_pairs - 1) / n_pairs;
  const int i0 = min(total, pair_id * per);
  const int i1 = min(total, i0 + per);
  if (kTrace && p.trace != nullptr && p.ready == nullptr && threadIdx.x == 0)
    p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 0] = gtimer();

  if (warp == 0 && lane == 0) {
    prefetch_map(&map_h);
    prefetch_map(&map_uw);
    for (int s = 0; s < p.stages; ++s) {
      // raw bf16: the leader's expect_tx; quantised: both SMs' converter warps
      mbar_init(&full[s], p.bits == 16 ? 1 : NCONV + (leader ? 1 : 0));  // + the peer's relay
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NSLOT; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * EW);
    }
    mbar_init(uw_full, 1);
    mbar_init(uw_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  cluster_sync();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (kTrace && p.trace != nullptr && p.ready == nullptr && threadIdx.x == 0) {
    p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 2] = gtimer();
    p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 511] = clock64();  // per-unit marks are SM clocks
  }

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both SMs) ----------------
      // standalone kernel: warm L2 with the first items' rows (latent append,
      // two launches back) while the query absorb still runs, then wait for
      // it before the first UW load
      if (p.pf_dist > 0 && p.ready == nullptr)
        for (int ip = i0; ip < min(i1, i0 + p.pf_dist); ++ip) {
          const int bgp = ip / n_super, stp = ip - bgp * n_super;
          const int rowp = bgp * p.T_cap + (2 * stp + (int)rank) * TILE_M;
          if (p.bits == 16) {
            for (int kb = 0; kb < kblocks; ++kb) tma_prefetch_l2(&map_h, kb * KB, rowp);
          } else {
            tma_prefetch_l2(&map_h, 0, rowp);
          }
        }
      pdl_wait();
      int cur = -1, nloads = 0, it = 0, pst = 0, pph = 0;
      const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
      // this CTA's slice of the L2 prefetch, one 32 KB piece per item
      constexpr long long PF_PIECE = 32768;
      const long long pf_share = ((p.l2pf_bytes + gridDim.x - 1) / gridDim.x + PF_PIECE - 1) / PF_PIECE * PF_PIECE;
      long long pf_at = (long long)blockIdx.x * pf_share;
      const long long pf_end = min(p.l2pf_bytes, pf_at + pf_share);
      ItemPos ip_(i0, n_super, p.G);
      for (int i = i0; i < i1; ++i, ++it, ip_.next(n_super, p.G)) {
        const int bg = ip_.bg, st = ip_.st;
        if (p.l2pf != nullptr && pf_at < pf_end) {
          bulk_prefetch_l2_hint(p.l2pf + pf_at, (uint32_t)min(PF_PIECE, pf_end - pf_at), pol_last);
          pf_at += PF_PIECE;
        }
        if (bg != cur) {
          if (nloads > 0) mbar_wait(uw_empty, (nloads - 1) & 1);
          if (leader) mbar_expect_tx(uw_full, 2 * kblocks * units * UWB);
          for (int kb = 0; kb < kblocks; ++kb)
            for (int h = 0; h < units; ++h)
              tma_load_2d_pair(&map_uw, uw_full, s_uw + (kb * units + h) * UWB, kb * KB,
                               UH == 2 ? (bg * p.s_k + 2 * h + (int)rank) * 128
                                       : (bg * p.s_k + h) * 128 + 64 * (int)rank);
          ++nloads;
          cur = bg;
        }
        const int tile = 2 * st + (int)rank;  // this SM's 128-token tile
        const int h_row = bg * p.T_cap + tile * TILE_M;
        // warm L2 with this SM's rows of the item PF_DIST ahead: smem holds only
        // ~1.25 items next to the resident UW, so HBM latency must be hidden in L2
        if (p.pf_dist > 0 && i + p.pf_dist < i1) {
          const int ip = i + p.pf_dist;
          const int bgp = ip / n_super, stp = ip - bgp * n_super;
          const int rowp = bgp * p.T_cap + (2 * stp + (int)rank) * TILE_M;
          if (p.bits == 16) {
            for (int kb = 0; kb < kblocks; ++kb) tma_prefetch_l2(&map_h, kb * KB, rowp);
          } else {
            tma_prefetch_l2(&map_h, 0, rowp);  // packed code rows (one box per tile)
          }
        }
        if (p.bits != 16) continue;  // the converter warps fill the H stages
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[pst], pph ^ 1);
          if (leader) mbar_expect_tx(&full[pst], 2 * H_STAGE_BYTES);
          tma_load_2d_pair_hint(&map_h, &full[pst], s_h + pst * H_STAGE_BYTES, kb * KB, h_row, pol_first);
          if (++pst == p.stages) {
            pst = 0;
            pph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ---------------- MMA issuer (leader SM issues for the pair) ----------------
      // The whole warp runs the loop (warp-uniform descriptors stay in uniform
      // registers); one elected lane -- always the same one, so its commits
      // track its own MMAs -- issues the tcgen05 instructions.
      const uint32_t uw_addr = smem_u32(s_uw);
      const uint32_t h_addr = smem_u32(s_h);
      int cur = -1, nloads = 0, unit = 0;
      // stage ring position of the item's first k-block, kept incrementally:
      // a runtime modulo per k-block is an integer-division chain (~100
      // dependent clocks) that the shallow MMA queue cannot hide
      int st0 = 0, ph0 = 0;
      const unsigned long long c_start = clock64(), g_start = gtimer();
      ItemPos ip_(i0, n_super, p.G);
      for (int i = i0; i < i1; ++i, ip_.next(n_super, p.G)) {
        const int bg = ip_.bg;
        if (bg != cur) {
          if (nloads > 0 && elect_one()) umma2_commit_both(uw_empty);  // frees UW in both SMs
          mbar_wait(uw_full, nloads & 1);
          fence_after();
          ++nloads;
          cur = bg;
        }
        for (int h = 0; h < units; ++h, ++unit) {
          const int slot = unit & (NSLOT - 1);
          if ((mode & 4) == 0) mbar_wait(&tempty[slot], ((unit / NSLOT) & 1) ^ 1);
          fence_after();
          if (kTrace && p.trace != nullptr && p.ready == nullptr && SU * unit + 11 < TRACE_STRIDE && lane == 0)
            p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 4 + SU * unit] = clock64();
          const uint32_t d_tmem = tmem_base + slot * SLOT_COLS;
          for (int kb = 0; kb < kblocks; ++kb) {
            int stage = st0 + kb, par = ph0;
            if (stage >= p.stages) {  // kblocks <= stages: at most one wrap
              stage -= p.stages;
              par ^= 1;
            }
            if (h == 0 && (mode & 2) == 0) {
              if (p.bits == 16)
                mbar_wait(&full[stage], par);
              else
                mbar_wait_cluster(&full[stage], par);  // the peer's stages: a cluster-scope release
              fence_after();
            }
            // profile modes 8 / 16 (diagnostics): pin the A / B operand tile
            const uint32_t a0 = h_addr + ((mode & 8) ? 0 : stage) * H_STAGE_BYTES;
            const uint32_t b0 = uw_addr + ((mode & 16) ? 0 : (kb * units + h)) * UWB;
            // K16 steps are 32 B apart: +2 in the descriptor's address field
            // (smem addresses < 256 KB, so the 14-bit field cannot carry)
            const uint64_t da = sdesc(a0), db = sdesc(b0);
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < KB / 16; ++kk)
                umma2_bf16_id(d_tmem, da + 2 * kk, db + 2 * kk, IDESC_U, (kb | kk) != 0);
              if (h == units - 1) umma2_commit_both(&empty[stage]);
            }
            __syncwarp();
          }
          if (elect_one()) umma2_commit_both(&tfull[slot]);
          __syncwarp();
          if (kTrace && p.trace != nullptr && p.ready == nullptr && SU * unit + 11 < TRACE_STRIDE && lane == 0)
            p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 5 + SU * unit] = clock64();
        }
        st0 += kblocks;
        if (st0 >= p.stages) {
          st0 -= p.stages;
          ph0 ^= 1;
        }
      }
      if (kTrace && p.trace != nullptr && p.ready == nullptr && lane == 0) {  // SM clocks vs wall time of the issue loop
        p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 508] = clock64() - c_start;
        p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 509] = gtimer() - g_start;
        p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 510] = (unsigned long long)unit * kblocks * (KB / 16);
      }
    } else if (p.bits != 16 && lane == 0) {
      // ---------------- peer SM, packed keys: stage relay (see conv_arrive) ----------------
      Ring rg;
      for (int i = i0; i < i1; ++i)
        for (int kb = 0; kb < kblocks; ++kb, rg.next(p.stages)) {
          mbar_wait(&full[rg.slot], rg.phase);
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                           smem_u32(&full[rg.slot]) & PEER_MASK)
                       : "memory");
        }
    }
  } else if (warp >= 2 + EW) {
    // ---------------- quantised keys: converter warps (both SMs) ----------------
    if (p.bits != 16) {
      // the newest token's codes and zero point come from this step's latent
      // append: wait for the predecessor chain before the first code load
      pdl_wait();
      const int cl = (warp - 2 - EW) * 32 + lane;  // the SM tile's row(s) of this lane
      // 16 epilogue warps leave ~96 registers: the 2-row converter build is
      // compiled out there (the host sends packed keys to the 4-warp build)
      if constexpr (EW == 16 && NCONV == 2) __trap();
      Ring rg;
      ItemPos ip_(i0, n_super, p.G);
      for (int i = i0; i < i1; ++i, ip_.next(n_super, p.G)) {
        const int bg = ip_.bg, st = ip_.st;
        const int tile = 2 * st + (int)rank;
        switch (p.bits) {
          case 2: convert_tile<2, TILE_M / (NCONV * 32)>(p, s_h, full, empty, bg, tile, T_rows, kblocks, cl, rg); break;
          case 3: convert_tile<3, TILE_M / (NCONV * 32)>(p, s_h, full, empty, bg, tile, T_rows, kblocks, cl, rg); break;
          case 4: convert_tile<4, TILE_M / (NCONV * 32)>(p, s_h, full, empty, bg, tile, T_rows, kblocks, cl, rg); break;
          default: convert_tile<8, TILE_M / (NCONV * 32)>(p, s_h, full, empty, bg, tile, T_rows, kblocks, cl, rg); break;
        }
      }
    }
  } else {
    // ---------------- epilogue (both SMs): cos/sin-weighted row reduction ----------------
    const int q = warp & 3;          // TMEM lane quarter
    constexpr int JH = EW / 4;       // frequency slices
    constexpr int FPW = 64 / JH;     // frequencies per warp
    const int jh = (warp - 2) >> 2;  // which FPW of the 64 frequencies
    const int delta = q * 32 + lane; // token row inside this SM's tile
    constexpr int CH = JH == 2 ? 8 : 4;  // frequencies per epilogue chunk (TMEM loads of CH columns)
    const uint64_t pol_keep = policy_evict_last();
    float2 cd2[FPW / 2], sd2[FPW / 2];  // cos/sin(delta th_j) for j pairs (2i, 2i + 1)
    {
      const float4* off =
          reinterpret_cast<const float4*>(p.rope_tab + (size_t)(p.n_tab + delta) * 64 + jh * FPW);
#pragma unroll
      for (int i = 0; i < FPW / 2; ++i) {
        const float4 v = off[i];
        cd2[i] = make_float2(v.x, v.y);
        sd2[i] = make_float2(v.z, v.w);
      }
    }
    const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
    // Per item the epilogue needs the tile's cos/sin base half-row and (packed
    // keys) its token scales.  Loaded at the item boundary they cost ~1 us per
    // item (L2 latency under the HBM stream; tools/score_trace.py at r_k 128:
    // the tensor pipe idled behind it), so this warp stages them into shared
    // memory with cp.async one item ahead.
    // QH > 1 (replicated-B groups, UH 1): the accumulator holds K = H B of the
    // group's one KV head (cols j: dim j, j + 64: dim j + 64); the epilogue
    // rotates each pair and dots it with the QH query heads' rotated rows
    static_assert(QH == 1 || UH == 1, "replicated-B groups use N128 units");
    constexpr int NOUT = UH * QH;  // logits per lane per unit
    uint8_t* eb = reinterpret_cast<uint8_t*>(red) + epi_red_bytes(NOUT) + (warp - 2) * epi_stage_bytes(QH);
    auto stage_item = [&](int buf, int tile_, int bg_, int qbuf) {
      if (lane < FPW / 2)
        cp_async16(eb + buf * 256 + lane * 16,
                   reinterpret_cast<const float4*>(p.rope_tab + (size_t)tile_ * 64 + jh * FPW) + lane);
      if (p.bits != 16) {
        const int tq = tile_ * TILE_M + delta;
        if (tq < T_rows) cp_async4(eb + 512 + buf * 128 + lane * 4, p.scales + (size_t)bg_ * p.T_cap + tq);
      }
      if (QH > 1 && qbuf >= 0) {
        // [hh][FPW lo dims | FPW hi dims] of this warp's frequency slice
#pragma unroll
        for (int c = lane; c < QH * 2 * FPW / 4; c += 32) {
          const int hh = c / (FPW / 2), part = c % (FPW / 2);
          const int dim = (part < FPW / 4 ? part * 4 : 64 + (part - FPW / 4) * 4) + jh * FPW;
          cp_async16(eb + 768 + qbuf * QH * 256 + c * 16, p.qrot + ((size_t)bg_ * QH + hh) * 128 + dim);
        }
      }
      cp_async_commit();
    };
    // quantised keys: the newest token's scale comes from this step's append
    pdl_wait();
    int unit = 0, it = 0;
    // QH > 1: the query slices change only with (b, g) -- restaged into the
    // idle buffer when the next item moves to another group
    int q_use = 0, q_next = 0, q_bg0 = -1, q_bg1 = -1;
    ItemPos ip_(i0, n_super, p.G), nx(i0, n_super, p.G);
    if (i0 < i1) stage_item(0, 2 * nx.st + (int)rank, nx.bg, 0);
    q_bg0 = nx.bg;
    nx.next(n_super, p.G);
    for (int i = i0; i < i1; ++i, ++it, ip_.next(n_super, p.G)) {
      const int st = ip_.st;
      const int b = ip_.b, g = ip_.g;
      const int tile = 2 * st + (int)rank;
      if (kTrace && p.trace != nullptr && p.ready == nullptr && warp == 2 && lane == 0 && SU * unit + 11 < TRACE_STRIDE)
        p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 10 + SU * unit] = clock64();
      cp_async_wait_all();
      __syncwarp();
      q_use = q_next;
      if (kTrace && p.trace != nullptr && p.ready == nullptr && warp == 2 && lane == 0 && SU * unit + 11 < TRACE_STRIDE)
        p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 11 + SU * unit] = clock64();
      const uint32_t base_addr = smem_u32(eb) + (uint32_t)(it & 1) * 256u;
      // quantised keys: the converter wrote c - z, so logit = s_t x (epilogue sum)
      float sq = 1.f;
      if (p.bits != 16 && tile * TILE_M + delta < T_rows)
        sq = lds32f(smem_u32(eb) + 512u + (uint32_t)(it & 1) * 128u + (uint32_t)lane * 4u);
      if (i + 1 < i1) {  // the other buffer was consumed an item ago
        int qbuf = -1;
        if (QH > 1 && (q_use ? q_bg1 : q_bg0) != nx.bg) {
          qbuf = q_use ^ 1;  // idle since the item before this one
          if (qbuf) q_bg1 = nx.bg; else q_bg0 = nx.bg;
        }
        q_next = qbuf >= 0 ? qbuf : q_use;
        stage_item((it + 1) & 1, 2 * nx.st + (int)rank, nx.bg, qbuf);
        nx.next(n_super, p.G);
      }
      for (int h = 0; h < units; ++h, ++unit) {
        const int slot = unit & (NSLOT - 1);
        const bool tr = kTrace && p.trace != nullptr && p.ready == nullptr && warp == 2 && lane == 0 &&
                        SU * unit + 11 < TRACE_STRIDE;
        if (tr) p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 9 + SU * unit] = clock64();
        mbar_wait(&tfull[slot], (unit / NSLOT) & 1);
        fence_after();
        if (tr) p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 6 + SU * unit] = clock64();
        float2 acc2[NOUT];
#pragma unroll
        for (int o = 0; o < NOUT; ++o) acc2[o] = make_float2(0.f, 0.f);
        if ((mode & 1) == 0)
#pragma unroll
        for (int jc = 0; jc < FPW / CH; ++jc) {
          // this chunk's accumulator columns (u_j at col, w_j at col + 64) for
          // every head of the unit, then cos/sin((t0 + delta) th_j) = base (x)
          // offset for its CH frequencies while the loads are in flight
          // (recomputed per unit: persistent per-item copies do not fit in
          // registers beside the offsets, and spilled values cost an L2 round
          // trip per use)
          float u[UH][CH], w[UH][CH];
#pragma unroll
          for (int hp = 0; hp < UH; ++hp) {
            const uint32_t col = slot * SLOT_COLS + hp * 128 + jh * FPW + jc * CH;
            tmem_ldn<CH>(lane_base + col, u[hp]);
            tmem_ldn<CH>(lane_base + col + 64, w[hp]);
          }
          float2 c2[CH / 2], s2[CH / 2];
#pragma unroll
          for (int k = 0; k < CH / 2; ++k) {
            const float4 bv = lds128f(base_addr + (uint32_t)(jc * (CH / 2) + k) * 16u);
            const float2 bc = make_float2(bv.x, bv.y), bsn = make_float2(bv.z, bv.w);
            const float2 t = fmul2(bsn, sd2[jc * (CH / 2) + k]);
            c2[k] = ffma2(bc, cd2[jc * (CH / 2) + k], make_float2(-t.x, -t.y));
            s2[k] = ffma2(bsn, cd2[jc * (CH / 2) + k], fmul2(bc, sd2[jc * (CH / 2) + k]));
          }
          tmem_wait_ld();
          if (jc == FPW / CH - 1) {
            // every accumulator column this warp reads is in registers: hand
            // the slot back before the last FMAs and the cross-warp exchange
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_leader(&tempty[slot]);
          }
          if constexpr (QH == 1) {
#pragma unroll
            for (int hp = 0; hp < UH; ++hp)
#pragma unroll
              for (int k = 0; k < CH / 2; ++k) {
                acc2[hp] = ffma2(c2[k], make_float2(u[hp][2 * k], u[hp][2 * k + 1]), acc2[hp]);
                acc2[hp] = ffma2(s2[k], make_float2(w[hp][2 * k], w[hp][2 * k + 1]), acc2[hp]);
              }
          } else {
            const uint32_t qb = smem_u32(eb) + 768u + (uint32_t)q_use * (QH * 256u);
            static_assert(CH % 4 == 0, "query slices are read 4 frequencies at a time");
#pragma unroll
            for (int k4 = 0; k4 < CH / 4; ++k4) {
              // RoPE of the key pairs (dims j, j + 64) for frequencies j .. j + 3
              float2 klo[2], khi[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int k = 2 * k4 + e;
                const float2 lo = make_float2(u[0][2 * k], u[0][2 * k + 1]);
                const float2 hi = make_float2(w[0][2 * k], w[0][2 * k + 1]);
                const float2 t = fmul2(s2[k], hi);
                klo[e] = ffma2(c2[k], lo, make_float2(-t.x, -t.y));
                khi[e] = ffma2(s2[k], lo, fmul2(c2[k], hi));
              }
              const uint32_t jo = (uint32_t)(jc * CH + 4 * k4) * 4u;
#pragma unroll
              for (int hh = 0; hh < QH; ++hh) {
                const float4 ql = lds128f(qb + (uint32_t)hh * (2u * FPW * 4u) + jo);
                const float4 qh = lds128f(qb + (uint32_t)hh * (2u * FPW * 4u) + FPW * 4u + jo);
                acc2[hh] = ffma2(klo[0], make_float2(ql.x, ql.y), acc2[hh]);
                acc2[hh] = ffma2(khi[0], make_float2(qh.x, qh.y), acc2[hh]);
                acc2[hh] = ffma2(klo[1], make_float2(ql.z, ql.w), acc2[hh]);
                acc2[hh] = ffma2(khi[1], make_float2(qh.z, qh.w), acc2[hh]);
              }
            }
          }
        }
        if (mode & 1) {  // diagnostics: no math, release the slot at once
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_leader(&tempty[slot]);
        }
        float v[NOUT];
#pragma unroll
        for (int o = 0; o < NOUT; ++o) v[o] = acc2[o].x + acc2[o].y;
        if (tr) p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 7 + SU * unit] = clock64();
        // exchange buffer and named barrier rotate over 4 units: a warp hands
        // the slot back before this exchange, so unit u + 2 may already be
        // in flight, and reuse at u + 4 waits (through the MMA) for every
        // warp's release of u + 2, issued after its reads of u
        const int xb = unit & 3;
        float* r = red + xb * (JH - 1) * NOUT * TILE_M;
        if (jh != 0) {
#pragma unroll
          for (int o = 0; o < NOUT; ++o) r[((jh - 1) * NOUT + o) * TILE_M + delta] = v[o];
          named_bar_arrive(1 + xb, EW * 32);
        } else {
          named_bar_sync(1 + xb, EW * 32);
          if (tr) p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 8 + SU * unit] = clock64();
#pragma unroll
          for (int k = 0; k < JH - 1; ++k)
#pragma unroll
            for (int o = 0; o < NOUT; ++o) v[o] += lds32f(smem_u32(r + (k * NOUT + o) * TILE_M + delta));
          const int t = tile * TILE_M + delta;
          if (t < T_rows) {
            // UH 2: D columns 0..127 = head 2h (leader's UW rows), 128..255 =
            // head 2h + 1; UH 1: columns 0..63 u_j (leader), 64..127 w_j (peer)
            // QH > 1: the group's query heads g QH .. g QH + QH - 1
            const int head0 = (g * p.s_k + UH * h) * QH;
            float* lg = p.logits + ((size_t)b * p.n_heads + head0) * p.ld_logits + t;
#pragma unroll
            for (int o = 0; o < NOUT; ++o)  // read by the value kernel next: keep in L2
              stg_hint(lg + (size_t)o * p.ld_logits, v[o] * sq, pol_keep);
          }
          if (kTrace && p.trace != nullptr && p.ready != nullptr && warp == 2 && lane == 0 && h == units - 1 &&
              it < TRACE_STRIDE - 8)
            p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 4 + it] = gtimer();
          if (p.ready != nullptr && h == units - 1) {
            // publish this warp's logits of the item to the value role
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicAdd(&p.ready[i], 1);
          }
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
  if (kTrace && p.trace != nullptr && threadIdx.x == 0) {
    p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 1] = gtimer();
    p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 3] = i1 - i0;
  }
}

// NCONV converter warps: 2 for raw bf16 keys (idle; 10 warps keep 168
// registers), 4 for packed keys (2 left the int4-key score at 173 us vs 156
// with 4; the 12-warp build gets 128 registers)
template <int UH, int NCONV, int QH = 1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64 + SCORE_EPI * 32 + NCONV * 32, 1)
rope_score_tc_kernel(const __grid_constant__ CUtensorMap map_h,
                     const __grid_constant__ CUtensorMap map_uw, const Params p) {
  // setup overlaps the query absorb; only the UW loads read its output
  // (score_role's producer waits before them)
  pdl_launch();
  if (!p.pdl_split) pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // no static shared memory here: the dynamic window starts 1024-aligned, and
  // the host sizes it without an alignment pad (room for a 6th H stage)
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  score_role<UH, NCONV, SCORE_EPI, QH>(map_h, map_uw, p, smem);
}

// ===========================================================================
// Fused score + softmax + value kernel (grid-level role split).
//
// The reconstruction is tensor-bound and the value stream is HBM-bound, so
// one persistent grid runs both concurrently on disjoint SMs: CTA pairs
// [0, score_pairs) run score_role and publish per-item readiness; the other
// CTAs run value_role.  A value CTA walks its sub-units (VSched) in the order
// the score pairs complete them; per sub-unit its 8 worker warps turn the
// logits into softmax statistics and bf16 probabilities P (written straight
// into a K-major SW128 smem operand), a TMA warp streams H_v as 2-D swizzled
// boxes {64 columns, 128 tokens}, and one thread issues
//   D[128 columns x 16 heads] += H_v^T (MN-major) x P^T     (tcgen05, TMEM)
// per 128-column pair.  The workers read D back (double-buffered) into a
// per-sub-unit partial; the sub-unit that completes a (sequence, group)
// merges its partials in token order (deterministic).  attention.py:433-446.
// ===========================================================================
struct VParams {
  int Rv_pad, vc;     // value row width; score items per value unit window
  int v_stages;       // TMA ring depth of the value role (32 KB stages)
  unsigned* tickets;  // [B*G] super-tiles merged so far
  float *pm, *pl, *pctx;  // partials [B][n][ns] / [B][n][ns][Rv_pad]
  int ns_cap;  // partial slots per head: super-tiles per group at capacity
  const int* ranks_v;
  const int* o_off;
  float* ctx_out;
  int ld_ctx;
  int no_wait;  // standalone value kernel: the logits are complete at launch
  // quantised values (bits 2/3/4/8; 16 = raw bf16 through TMA): packed codes
  // [B][G][T_cap][code_row_bytes] and per-token fp32 scale / zero point
  int bits, code_row_bytes;
  const uint8_t* codes;
  const float* scales;
  const float* zps;
  int raw_slots;  // standalone kernel, packed V: TMA ring of packed code tiles (+ zero points)
};

constexpr int V_STAGE = 32768;
constexpr int V_RAW_BYTES = 65536;  // packed-code ring (tiles of 128 tokens x 128 codes)  // 128 tokens x 128 columns; 2 TMA boxes of 16 KB
constexpr int V_HP = 4;         // heads per group handled by the value role
constexpr uint32_t IDESC_LS = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(16 >> 3) << 17) |
                              ((uint32_t)(128 >> 4) << 24);  // K-major A and B, M 128, N 16
constexpr int V_TMEM_COLS = 128;
constexpr int V_PF = 0;     // L2 prefetch distance of the value stream (128-token blocks)
constexpr int V_SUB = 512;  // tokens per P sub-block (double-buffered)
#ifndef PALU_V_HEAD_START
#define PALU_V_HEAD_START 2
#endif
constexpr int V_HEAD_START = PALU_V_HEAD_START;  // H_v stages issued before the first logits have arrived

__device__ __forceinline__ uint32_t ld_acquire_u32(const int* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct VUnit {
  int bg, st0, st1, item0;
};

// Value units.  The score role gives pair pr the contiguous items
// [pr * per, (pr + 1) * per) and walks them in order, so unit window (pr, w)
// = items [pr * per + w * vc, + vc) clipped to the pair's block becomes ready
// at about (w + 1) / W of the score run.  Windows are handed out w-major
// (round robin over value CTAs) and split at (sequence, group) boundaries;
// a sub-unit's partial lives at slot = its first super-tile within the group.
struct VSched {
  int per, total, pairs, n_super, vc, W;
  __device__ __forceinline__ int win_end(int a) const {
    const int pr = a / per;
    const int w = (a - pr * per) / vc;
    return min(min(pr * per + (w + 1) * vc, (pr + 1) * per), total);
  }
};

// This value CTA's sub-units, in order (every role of the CTA runs its own copy)
struct VIter {
  VSched s;
  int step, u, a, e;
  __device__ VIter(const VSched& sch, int vcta, int n_vctas)
      : s(sch), step(n_vctas), u(vcta - n_vctas), a(0), e(0) {}
  __device__ __forceinline__ bool next(VUnit& o) {
    while (a >= e) {
      u += step;
      if (u >= s.W * s.pairs) return false;
      const int w = u / s.pairs, pr = u - w * s.pairs;
      a = pr * s.per + w * s.vc;
      e = min(min(a + s.vc, (pr + 1) * s.per), s.total);
    }
    const int bg = a / s.n_super;
    const int se = min(e, (bg + 1) * s.n_super);
    o = VUnit{bg, a - bg * s.n_super, se - bg * s.n_super, a};
    a = se;
    return true;
  }
};

// Quantised values: token rows [t0, t0 + 128) (zeros past t1), columns
// [128 j, 128 j + 128) -> two 64-column MN-major SW128 slabs of c - z.  Lane
// cl owns rows cl and cl + 64.  int4 / int2 use the 32-bit word trick (pairs
// (c_k, c_{k + G/2}) per group of 8 / 16 columns, undone on readback).
struct VStage {  // one converter stage: (unit, 128-token block, column pair)
  int bg, t0, t1, j;
};
template <int BITS, int RPL>  // RPL: token rows per converter lane (128 / converter lanes)
struct VCodes {
  uint4 w[RPL][BITS];
  float z[RPL];
};
template <int BITS, int RPL>
__device__ __forceinline__ void load_v_codes(const VParams& vp, int T_cap, const VStage& g, int cl,
                                             VCodes<BITS, RPL>& c) {
#pragma unroll
  for (int rr = 0; rr < RPL; ++rr) {
    const int t = g.t0 + cl + (128 / RPL) * rr;
    const bool ok = g.bg >= 0 && t < g.t1;
    const size_t tok = (size_t)(ok ? g.bg : 0) * T_cap + (ok ? t : 0);
    const uint4* rp = reinterpret_cast<const uint4*>(vp.codes + tok * vp.code_row_bytes +
                                                     (size_t)g.j * 128 * BITS / 8);
    c.z[rr] = ok ? __ldg(vp.zps + tok) : 0.f;
#pragma unroll
    for (int q = 0; q < BITS; ++q) c.w[rr][q] = ok ? __ldg(rp + q) : make_uint4(0u, 0u, 0u, 0u);
  }
}
template <int BITS, int RPL>
__device__ __forceinline__ void convert_v_codes(const VCodes<BITS, RPL>& c, int cl, uint8_t* sb,
                                                int slab = -1) {
#pragma unroll
  for (int rr = 0; rr < RPL; ++rr) {
    const int row = cl + (128 / RPL) * rr;
    const float z = c.z[rr];
    const bool zsmall = fabsf(z) <= 128.f;
    const __nv_bfloat162 zb = __float2bfloat162_rn((float)CODE_BIAS + z);
    uint32_t wd[4 * BITS];
#pragma unroll
    for (int q = 0; q < BITS; ++q) {
      wd[4 * q] = c.w[rr][q].x;
      wd[4 * q + 1] = c.w[rr][q].y;
      wd[4 * q + 2] = c.w[rr][q].z;
      wd[4 * q + 3] = c.w[rr][q].w;
    }
#pragma unroll
    for (int ch = 0; ch < 16; ++ch) {  // 16 chunks of 8 columns; slab = ch / 8
      if (slab >= 0 && (ch >> 3) != slab) continue;
      uint32_t wv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        __nv_bfloat162 v;
        if (BITS == 4 || BITS == 2) {
          constexpr uint32_t MASK = BITS == 4 ? 0x000F000Fu : 0x00030003u;
          const uint32_t w = BITS == 4 ? wd[ch] : wd[ch >> 1];
          const int k0 = BITS == 4 ? 0 : 4 * (ch & 1);
          const uint32_t cc = (w >> (BITS * (k0 + e))) & MASK;
          if (zsmall) {
            const uint32_t biased = 0x43004300u | cc;
            v = __hsub2(*reinterpret_cast<const __nv_bfloat162*>(&biased), zb);
          } else {
            v = __floats2bfloat162_rn((float)(cc & 0xFFFFu) - z, (float)(cc >> 16) - z);
          }
        } else {
          uint32_t c2[2];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int bit = (ch * 8 + 2 * e + hh) * BITS;
            const int w0 = bit >> 5, sh = bit & 31;
            uint32_t x = wd[w0] >> sh;
            if (sh + BITS > 32 && w0 + 1 < 4 * BITS) x |= wd[w0 + 1] << (32 - sh);
            c2[hh] = x & ((1u << BITS) - 1u);
          }
          v = __floats2bfloat162_rn((float)c2[0] - z, (float)c2[1] - z);
        }
        wv[e] = *reinterpret_cast<const uint32_t*>(&v);
      }
      const uint32_t dst =
          smem_u32(sb + (ch >> 3) * (V_STAGE / 2) + row * 128 + (((ch & 7) ^ (row & 7)) << 4));
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(wv[0]), "r"(wv[1]),
                   "r"(wv[2]), "r"(wv[3])
                   : "memory");
    }
  }
}

// Stage cursor over (unit, 128-token block, column pair) in the value
// pipeline's order; the TMA producer and the converter warps each walk a copy.
struct VStageIter {
  VIter it;
  int T_rows, NJ;
  int blk = 0, jj = 0, nblk = 0, c0 = 0, c1 = 0, bgc = -1;
  bool more = true;
  __device__ VStageIter(const VIter& i, int tr, int nj) : it(i), T_rows(tr), NJ(nj) {}
  __device__ __forceinline__ bool next(VStage& g) {
    if (!more) return false;
    if (bgc < 0 || (jj == 0 && blk == nblk)) {
      VUnit u;
      if (!it.next(u)) {
        more = false;
        return false;
      }
      bgc = u.bg;
      c0 = u.st0 * SUPER;
      c1 = min(T_rows, u.st1 * SUPER);
      nblk = (c1 - c0 + TILE_M - 1) / TILE_M;
      blk = 0;
      jj = 0;
    }
    g = VStage{bgc, c0 + blk * TILE_M, c1, jj};
    if (++jj == NJ) {
      jj = 0;
      ++blk;
    }
    return true;
  }
};

// Packed V through the TMA ring (standalone value kernel): converter lane cl
// owns token row cl of each block; the packed bytes and zero point come from
// shared memory, so the loads run up to V_RAW_BYTES ahead of the conversion.
template <int BITS>
__device__ __forceinline__ void value_converter_ring(VStageIter sit, uint8_t* raw, int nslots,
                                                     uint64_t* rfull, uint64_t* rempty,
                                                     uint8_t* ring, uint64_t* full, uint64_t* empty,
                                                     int vs, int cl, int lane,
                                                     unsigned long long* trace) {
  constexpr int RB = TILE_M * 16 * BITS;  // packed bytes of one stage's tile
  // 8 converter warps: lane pair (2 row, 2 row + 1) of converter lane cl owns the
  // two 64-column slabs of token row cl / 2; 4 warps: one lane per row, both slabs
  const int nconv_lanes = (int)(blockDim.x >> 5) * 32 - 320;
  const int split = nconv_lanes / TILE_M;  // 1 or 2
  const int row = cl / split, slab = split == 2 ? (cl & 1) : -1;
  VStage g;
  int k = 0;
  Ring rr_, rs_;  // raw-code ring, operand ring
  const bool tr = trace != nullptr && cl == 0;
  while (sit.next(g)) {
    const int rs = rr_.slot, st = rs_.slot;
    if (tr && 3 * k + 302 < TRACE_STRIDE) trace[300 + 3 * k] = gtimer();
    mbar_wait(&rfull[rs], rr_.phase);
    if (tr && 3 * k + 302 < TRACE_STRIDE) trace[301 + 3 * k] = gtimer();
    const uint8_t* slot = raw + rs * (RB + TILE_M * 4);
    VCodes<BITS, 1> c;
    const uint32_t a = smem_u32(slot + row * 16 * BITS);
#pragma unroll
    for (int q = 0; q < BITS; ++q)
      c.w[0][q] = (slab < 0 || (q >= slab * BITS / 2 && q < (slab + 1) * BITS / 2 + (BITS & 1)))
                      ? lds128(a + 16 * q)
                      : make_uint4(0u, 0u, 0u, 0u);
    c.z[0] = reinterpret_cast<const float*>(slot + RB)[row];
    mbar_wait(&empty[st], rs_.phase ^ 1);
    if (tr && 3 * k + 302 < TRACE_STRIDE) trace[302 + 3 * k] = gtimer();
    convert_v_codes<BITS, 1>(c, row, ring + st * V_STAGE, slab);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&full[st]);
      mbar_arrive(&rempty[rs]);
    }
    ++k;
    rr_.next(nslots);
    rs_.next(vs);
  }
}

// Converter warp loop: codes of stage n + 2 are in flight while stage n is
// written (two register buffers, loop unrolled by two).
template <int BITS, int RPL, class Next>
__device__ __forceinline__ void value_converter(const VParams& vp, int T_cap, Next&& next_stage,
                                                uint8_t* ring, uint64_t* full, uint64_t* empty,
                                                int vs, int cl, int lane) {
  VStage g0, g1, gn;
  VCodes<BITS, RPL> b0, b1;
  pdl_wait();  // codes / zero points of the newest token come from this step's append
  next_stage(g0);
  next_stage(g1);
  load_v_codes<BITS, RPL>(vp, T_cap, g0, cl, b0);
  load_v_codes<BITS, RPL>(vp, T_cap, g1, cl, b1);
  Ring rg;
  auto emit = [&](const VCodes<BITS, RPL>& b) {
    const int st = rg.slot;
    mbar_wait(&empty[st], rg.phase ^ 1);
    convert_v_codes<BITS, RPL>(b, cl, ring + st * V_STAGE);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&full[st]);
    rg.next(vs);
  };
  while (g0.bg >= 0) {
    emit(b0);
    next_stage(gn);
    g0 = gn;
    load_v_codes<BITS, RPL>(vp, T_cap, g0, cl, b0);
    if (g1.bg < 0) break;
    emit(b1);
    next_stage(gn);
    g1 = gn;
    load_v_codes<BITS, RPL>(vp, T_cap, g1, cl, b1);
    if (g0.bg < 0) break;
  }
}

__device__ void value_role(const CUtensorMap& map_v, const Params& p, const VParams& vp,
                           uint8_t* smem, int vcta, int n_vctas) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int T_rows = *p.t_dev + 1;
  const int n_super = (T_rows + SUPER - 1) / SUPER;
  const int total = p.B * p.G * n_super;
  const int per = (total + p.score_pairs - 1) / p.score_pairs;
  const int vc = vp.vc > 0 ? vp.vc : per;  // vc <= 0: one window per pair (standalone)
  const VSched sch{per, total, p.score_pairs, n_super, vc, (per + vc - 1) / vc};
  const int s_v = p.s_k;
  const int NJ = (vp.Rv_pad + 127) / 128;  // 128-column pairs of 64-column boxes
  const int ns = vp.ns_cap;
  const int vs = vp.v_stages;
  constexpr int PB = V_SUB / 64 * 1024;  // P bytes per sub-block buffer: 1 KB per 64 tokens
  // smem: ring | P[2] (+1 KB: rows 8..15 of the last block alias past it) |
  //       barriers | TMEM slot
  uint8_t* ring = smem;
  uint8_t* pbuf = ring + vs * V_STAGE;
  float* stat = reinterpret_cast<float*>(pbuf + 2 * PB + 1024);  // [2][2][V_HP] (m, l) per sub-block
  uint64_t* full = reinterpret_cast<uint64_t*>(stat + 4 * V_HP);
  uint64_t* empty = full + vs;
  uint64_t* pfull = empty + vs;   // [2] P sub-block written (+ its statistics)
  uint64_t* dfull = pfull + 2;    // [2] sub-block accumulator complete (P consumed)
  uint64_t* dempty = dfull + 2;   // [2] sub-block accumulator read back
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dempty + 2);
  // group A holds the first sub-block's logits (the bf16 producer waits for
  // this after its first V_HEAD_START stages)
  uint64_t* lgready = reinterpret_cast<uint64_t*>(tslot + 2);
  // packed V, standalone kernel: TMA ring of code tiles (+ 128 zero points each)
  const int nslots = vp.raw_slots;
  uint64_t* rfull = reinterpret_cast<uint64_t*>(tslot + 4);  // [nslots]
  uint64_t* rempty = rfull + nslots;                         // [nslots]
  uint8_t* raw = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(rempty + nslots) + 127) & ~uintptr_t(127));
  __shared__ float red_m[4][V_HP], red_l[4][V_HP];

  if (tid == 0) {
    for (int st = 0; st < vs; ++st) {
      // TMA expect_tx | one arrive per converter warp
      mbar_init(&full[st], vp.bits == 16 ? 1 : (int)(blockDim.x >> 5) - 10);
      mbar_init(&empty[st], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&pfull[a], 1);
      mbar_init(&dfull[a], 1);
      mbar_init(&dempty[a], 1);
    }
    mbar_init(lgready, 1);
    for (int a = 0; a < nslots; ++a) {
      mbar_init(&rfull[a], 1);
      mbar_init(&rempty[a], (int)(blockDim.x >> 5) - 10);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(V_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  unsigned long long* vtr = p.trace != nullptr ? p.trace + (size_t)blockIdx.x * TRACE_STRIDE : nullptr;
  if (vtr != nullptr && tid == 0) vtr[495] = gtimer();  // setup done
  VIter it(sch, vcta, n_vctas);
  VUnit u;
  if (warp >= 10) {
    // ---------------- quantised values: converter warps write c - z of each
    // stage's 128 tokens x 128 columns into the MN-major SW128 operand (the
    // layout the TMA boxes would give); columns permuted as for the keys
    if (vp.bits == 16) return;
    const int nconv = (int)(blockDim.x >> 5) - 10;  // 2 (fused kernel) or 8 (packed-V value kernel)
    const int cl = (warp - 10) * 32 + lane;  // token rows cl (+ 64) of each block
    // stage cursor over (unit, block, column pair) in the producer's order
    int blk = 0, jj = 0, nblk = 0, c0 = 0, c1 = 0, bgc = -1;
    bool more = true;
    auto next_stage = [&](VStage& g) {
      if (!more) { g = VStage{-1, 0, 0, 0}; return; }
      if (bgc < 0 || (jj == 0 && blk == nblk)) {
        if (!it.next(u)) { more = false; g = VStage{-1, 0, 0, 0}; return; }
        bgc = u.bg;
        c0 = u.st0 * SUPER;
        c1 = min(T_rows, u.st1 * SUPER);
        nblk = (c1 - c0 + TILE_M - 1) / TILE_M;
        blk = 0;
        jj = 0;
      }
      g = VStage{bgc, c0 + blk * TILE_M, c1, jj};
      if (++jj == NJ) { jj = 0; ++blk; }
    };
#define VCONV(B_, R_) value_converter<B_, R_>(vp, p.T_cap, next_stage, ring, full, empty, vs, cl, lane)
#define VRING(B_) value_converter_ring<B_>(VStageIter(it, T_rows, NJ), raw, nslots, rfull, rempty, ring, \
                                           full, empty, vs, cl, lane,                                  \
                                           p.trace ? p.trace + (size_t)blockIdx.x * TRACE_STRIDE : nullptr)
    if (nslots > 0 && (nconv == 4 || nconv == 8)) {
      switch (vp.bits) {
        case 2: VRING(2); break;
        case 3: VRING(3); break;
        case 4: VRING(4); break;
        default: VRING(8); break;
      }
    } else if (nconv >= 4) {
      switch (vp.bits) {
        case 2: VCONV(2, 1); break;
        case 3: VCONV(3, 1); break;
        case 4: VCONV(4, 1); break;
        default: VCONV(8, 1); break;
      }
    } else {
      switch (vp.bits) {
        case 2: VCONV(2, 2); break;
        case 3: VCONV(3, 2); break;
        case 4: VCONV(4, 2); break;
        default: VCONV(8, 2); break;
      }
    }
#undef VCONV
#undef VRING
    return;
  }

  if (warp == 8 && vp.bits != 16 && nslots > 0) {
    // ---------------- TMA producer, packed V: code tiles {16 bits bytes, 128
    // rows} and the tile's 128 zero points into the raw ring
    if (lane == 0) {
      prefetch_map(&map_v);
      const int RB = TILE_M * 16 * vp.bits;
      VStageIter sit(it, T_rows, NJ);
      VStage g;
      Ring rg;
      bool waited = false;
      while (sit.next(g)) {
        const int rs = rg.slot;
        // the tile holding the newest token (row T_rows - 1, written by this
        // step's append) is loaded only after the predecessor chain completed
        if (!waited && g.t0 + TILE_M >= T_rows) {
          pdl_wait();
          waited = true;
        }
        mbar_wait(&rempty[rs], rg.phase ^ 1);
        mbar_expect_tx(&rfull[rs], RB + TILE_M * 4);
        uint8_t* slot = raw + rs * (RB + TILE_M * 4);
        tma_load_2d(&map_v, &rfull[rs], slot, g.j * 16 * vp.bits, g.bg * p.T_cap + g.t0);
        // T_cap is a multiple of 128 (LatentKVCache): the tile's zero points are
        // 512 aligned bytes inside this sequence/group's row range
        bulk_load(slot + RB, vp.zps + (size_t)g.bg * p.T_cap + g.t0, TILE_M * 4, &rfull[rs]);
        rg.next(nslots);
      }
    }
    return;
  }
  if (warp == 8) {
    // ---------------- TMA producer: H_v does not depend on the score role,
    // so it streams every sub-unit back to back, bounded by the ring
    if (lane == 0 && vp.bits == 16) {
      prefetch_map(&map_v);
      const uint64_t pol_first = policy_evict_first();  // H_v is read once; keep L2 for the weights
      int ctr = 0;
      bool waited = false;
      Ring rg;
      while (it.next(u)) {
        const int c0 = u.st0 * SUPER, c1 = min(T_rows, u.st1 * SUPER);
        const int nblk = (c1 - c0 + TILE_M - 1) / TILE_M;
        for (int blk = 0; blk < nblk; ++blk)
          for (int j = 0; j < NJ; ++j, ++ctr, rg.next(vs)) {
            const int st = rg.slot;
            // newest token (this step's append): wait for the predecessor chain
            if (!waited && c0 + (blk + 1) * TILE_M >= T_rows) {
              pdl_wait();
              waited = true;
            }
            // warm L2 with the rows V_PF blocks ahead: the ring turnaround then
            // sees L2 rather than loaded-HBM latency
            if (V_PF > 0 && blk + V_PF < nblk) {
              const int rowp = u.bg * p.T_cap + c0 + (blk + V_PF) * TILE_M;
              tma_prefetch_l2(&map_v, j * 128, rowp);
              tma_prefetch_l2(&map_v, j * 128 + 64, rowp);
            }
            // start-up: every SM's first ring fill (~28 MB chip-wide) queues
            // ahead of group A's logits reads (written by the score kernel,
            // no longer in L2), which held the first P back ~8 us; issue
            // V_HEAD_START stages, then let the logits through first
            if (vp.no_wait && ctr == V_HEAD_START) mbar_wait(lgready, 0);
            mbar_wait(&empty[st], rg.phase ^ 1);
            if (vtr != nullptr && ctr == 0) vtr[496] = gtimer();  // first TMA issue
            mbar_expect_tx(&full[st], V_STAGE);
            const int row = u.bg * p.T_cap + c0 + blk * TILE_M;
            tma_load_2d_hint(&map_v, &full[st], ring + st * V_STAGE, j * 128, row, pol_first);
            tma_load_2d_hint(&map_v, &full[st], ring + st * V_STAGE + V_STAGE / 2, j * 128 + 64, row, pol_first);
          }
      }
    }
    return;
  }
  if (warp == 9) {
    // ---------------- MMA issuer: per V_SUB-token sub-block sb (buffer sb & 1)
    // D[buf][j] = V^T x P^T over the sub-block's 128-token blocks; the whole
    // warp runs the loop, one elected lane issues the tcgen05 instructions
    {
      int ctr = 0, sb = 0;
      Ring rg;
      while (it.next(u)) {
        const int c0 = u.st0 * SUPER, c1 = min(T_rows, u.st1 * SUPER);
        const int nblk = (c1 - c0 + TILE_M - 1) / TILE_M;
        for (int b0 = 0; b0 < nblk; b0 += V_SUB / TILE_M, ++sb) {
          const int buf = sb & 1;
          if ((p.mode & 2) == 0) mbar_wait(&pfull[buf], (sb >> 1) & 1);
          if (sb >= 2) mbar_wait(&dempty[buf], ((sb >> 1) - 1) & 1);
          fence_after();
          const uint32_t pb = smem_u32(pbuf + buf * PB);
          const int b1 = min(nblk, b0 + V_SUB / TILE_M);
          for (int blk = b0; blk < b1; ++blk)
            for (int j = 0; j < NJ; ++j, ++ctr, rg.next(vs)) {
              const int st = rg.slot;
              mbar_wait(&full[st], rg.phase);
              fence_after();
              if (vtr != nullptr && lane == 0 && ctr == 0) vtr[497] = gtimer();  // first stage landed
              if (vtr != nullptr && lane == 0 && ctr == vs) vtr[498] = gtimer();  // ring wrapped
              if (p.mode & 1) {  // diagnostics: release the stage without MMAs
                if (lane == 0) mbar_arrive(&empty[st]);
                continue;
              }
              const uint32_t a0 = smem_u32(ring + st * V_STAGE);
              const uint32_t d = tmem + (uint32_t)((buf * NJ + j) * 16);
              if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < TILE_M / 16; ++kk)
                  umma_bf16_id(d, sdesc_mn(a0 + kk * 2048, V_STAGE / 2, 1024),
                               sdesc(pb + ((blk - b0) * 2 + kk / 4) * 1024 + (kk % 4) * 32), IDESC_V,
                               (blk != b0) || (kk != 0));
                umma_commit(&empty[st]);
              }
              __syncwarp();
            }
          if (p.mode & 1) {
            if ((p.mode & 2) != 0) mbar_wait(&pfull[buf], (sb >> 1) & 1);
            if (lane == 0) mbar_arrive(&dfull[buf]);
          } else {
            if (elect_one()) umma_commit(&dfull[buf]);
            __syncwarp();
          }
        }
      }
    }
    __syncwarp();
    named_bar_sync(2, 288);
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(V_TMEM_COLS));
    return;
  }

  if (warp < 4) {
    // ======== group A (warps 0-3): logits -> statistics -> P operand ========
    pdl_wait();  // the logits come from the preceding score launch
    const int ta = tid;  // 0..127
    int kk_trace = 0;
    auto trace = [&](int slot) {
      if (p.trace != nullptr && ta == 0 && 5 * kk_trace + 8 < TRACE_STRIDE)
        p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 4 + 5 * kk_trace + slot] = gtimer();
    };
    int sb = 0;
    while (it.next(u)) {
      if (ta == 0 && !vp.no_wait) {
        for (int i = u.item0; i < u.item0 + (u.st1 - u.st0); ++i)
          while (ld_acquire_u32(&p.ready[i]) < 2u * (EPI_WARPS / 2)) __nanosleep(64);
      }
      named_bar_sync(3, 128);
      trace(0);
      const int b = u.bg / p.G, g = u.bg - b * p.G;
      const int c0 = u.st0 * SUPER, c1 = min(T_rows, u.st1 * SUPER);
      const int nt = c1 - c0;
      const int ntok = (nt + TILE_M - 1) / TILE_M * TILE_M;  // padded to whole blocks
      const float* lg = p.logits + ((size_t)b * p.n_heads + g * s_v) * p.ld_logits + c0;
      // the sub-block's logits (thread = token pairs 2 ta + 256 i); the next
      // sub-block's are loaded while this one is processed
      constexpr int NP = V_SUB / 256;
      const uint64_t pol_drop = policy_evict_first();  // the logits are dead after this read
      float2 x[NP][V_HP], xn[NP][V_HP];
      // no value-dependent masking in the prefetch (an op on a loaded register
      // waits for the load); the masks are applied where the values are used
      auto load = [&](int s0, float2 (&dst)[NP][V_HP]) {
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const int t = s0 + 2 * ta + 256 * i;
#pragma unroll
          for (int h = 0; h < V_HP; ++h) {
            float2 v = make_float2(0.f, 0.f);
            if (h < s_v && t < nt) v = ldg64_cg_hint(lg + (size_t)h * p.ld_logits + t, pol_drop);
            dst[i][h] = v;
          }
        }
      };
      load(0, xn);
      for (int s0 = 0; s0 < ntok; s0 += V_SUB, ++sb) {
        const int buf = sb & 1;
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const int t = s0 + 2 * ta + 256 * i;
#pragma unroll
          for (int h = 0; h < V_HP; ++h)
            x[i][h] = make_float2(h < s_v && t < nt ? xn[i][h].x : -INFINITY,
                                  h < s_v && t + 1 < nt ? xn[i][h].y : -INFINITY);
        }
        if (s0 + V_SUB < ntok) load(s0 + V_SUB, xn);
        // quantised values: P carries p s_t (the operand holds c - z)
        float2 sv[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          sv[i] = make_float2(1.f, 1.f);
          const int t = s0 + 2 * ta + 256 * i;
          if (vp.bits != 16 && t < nt) {
            const float* sp = vp.scales + (size_t)u.bg * p.T_cap + c0 + t;
            sv[i].x = __ldg(sp);
            if (t + 1 < nt) sv[i].y = __ldg(sp + 1);
          }
        }
        // (1) max of the sub-block
        float m[V_HP];
#pragma unroll
        for (int h = 0; h < V_HP; ++h) m[h] = -INFINITY;
#pragma unroll
        for (int i = 0; i < NP; ++i)
#pragma unroll
          for (int h = 0; h < V_HP; ++h) m[h] = fmaxf(m[h], fmaxf(x[i][h].x, x[i][h].y));
#pragma unroll
        for (int h = 0; h < V_HP; ++h) {
          m[h] = warp_reduce(m[h], [](float a, float c) { return fmaxf(a, c); });
          if (lane == 0) red_m[warp][h] = m[h];
        }
        // buffer `buf` (P operand + statistics) is free once sub-block sb - 2
        // has been read back
        if (sb >= 2) mbar_wait(&dempty[buf], ((sb >> 1) - 1) & 1);
        named_bar_sync(3, 128);
        if (sb == 0 && ta == 0) mbar_arrive(lgready);  // every group-A thread holds its logits
        trace(2);
#pragma unroll
        for (int h = 0; h < V_HP; ++h)
          m[h] = fmaxf(fmaxf(red_m[0][h], red_m[1][h]), fmaxf(red_m[2][h], red_m[3][h]));
        // (2) P = hi + lo bf16 (rows h and h + 4 of the K-major SW128 operand:
        // ~16 mantissa bits of p at no extra tensor work), zeros past the
        // last token; l sums the fp32 probabilities
        uint8_t* pb = pbuf + buf * PB;
        float l[V_HP];
#pragma unroll
        for (int h = 0; h < V_HP; ++h) l[h] = 0.f;
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const int tl = 2 * ta + 256 * i;
          if (s0 + tl < ntok) {
            const int blk = tl >> 6, w = tl & 63;
            const uint32_t rowb = blk * 1024 + (w & 7) * 2;
#pragma unroll
            for (int h = 0; h < V_HP; ++h) {
              if (h < s_v) {
                const float p0 = __expf(x[i][h].x - m[h]), p1 = __expf(x[i][h].y - m[h]);
                l[h] += p0 + p1;
                const float q0 = p0 * sv[i].x, q1 = p1 * sv[i].y;
                const __nv_bfloat162 hi = __floats2bfloat162_rn(q0, q1);
                const float2 hf = __bfloat1622float2(hi);
                const __nv_bfloat162 lo = __floats2bfloat162_rn(q0 - hf.x, q1 - hf.y);
                *reinterpret_cast<__nv_bfloat162*>(pb + rowb + h * 128 + ((((w >> 3) ^ h) & 7) << 4)) = hi;
                *reinterpret_cast<__nv_bfloat162*>(pb + rowb + (h + 4) * 128 +
                                                   ((((w >> 3) ^ (h + 4)) & 7) << 4)) = lo;
              }
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
        for (int h = 0; h < V_HP; ++h) {
          l[h] = warp_reduce(l[h], [](float a, float c) { return a + c; });
          if (lane == 0) red_l[warp][h] = l[h];
        }
        named_bar_sync(3, 128);
        if (ta < V_HP) {
          float mh = m[0], lh = 0.f;
#pragma unroll
          for (int h = 0; h < V_HP; ++h)
            if (ta == h) {
              mh = m[h];
              lh = (red_l[0][h] + red_l[1][h]) + (red_l[2][h] + red_l[3][h]);
            }
          stat[(buf * 2 + 0) * V_HP + ta] = mh;
          stat[(buf * 2 + 1) * V_HP + ta] = lh;
        }
        named_bar_sync(3, 128);
        if (ta == 0) mbar_arrive(&pfull[buf]);
      }
      trace(1);
      if (p.trace != nullptr) ++kk_trace;
    }
  } else {
    // ======== group B (warps 4-7): sub-block accumulators -> unit partial ========
    // online softmax across the unit's sub-blocks in registers: thread = one
    // V column per 128-column pair j, all heads
    const int tb = tid - 128, wb = warp - 4;  // wb = TMEM lane quarter
    int sb = 0;
    while (it.next(u)) {
      const int b = u.bg / p.G, g = u.bg - b * p.G;
      const int c0 = u.st0 * SUPER, c1 = min(T_rows, u.st1 * SUPER);
      const int nblk = (c1 - c0 + TILE_M - 1) / TILE_M;
      float acc[4][V_HP], mr[V_HP], lr[V_HP];
#pragma unroll
      for (int h = 0; h < V_HP; ++h) {
        mr[h] = -INFINITY;
        lr[h] = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j][h] = 0.f;
      }
      for (int b0 = 0; b0 < nblk; b0 += V_SUB / TILE_M, ++sb) {
        const int buf = sb & 1;
        mbar_wait(&dfull[buf], (sb >> 1) & 1);
        fence_after();
        float sc_old[V_HP], sc_new[V_HP];
#pragma unroll
        for (int h = 0; h < V_HP; ++h) {
          const float ms = stat[(buf * 2 + 0) * V_HP + h], ls = stat[(buf * 2 + 1) * V_HP + h];
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
            for (int h = 0; h < V_HP; ++h)
              acc[j][h] = acc[j][h] * sc_old[h] + (v[h] + v[h + V_HP]) * sc_new[h];
          }
        }
        fence_before();
        named_bar_sync(4, 128);
        if (tb == 0) mbar_arrive(&dempty[buf]);
      }
      // the unit's partial: columns of all heads, statistics
      // TMEM lane m of pair j = column j*128 + m, except int4 / int2 values whose
      // converter stores rank k of each 8 / 16 group at position k < G/2 ? 2k : 2k-G+1
      const int m = wb * 32 + lane;
      const int grp = vp.bits == 4 ? 8 : (vp.bits == 2 ? 16 : 0);
      int mc = m;
      if (grp) {
        const int pp = m % grp;
        mc = m - pp + ((pp & 1) ? grp / 2 + pp / 2 : pp / 2);
      }
      for (int j = 0; j < 4; ++j) {
        const int col = j * 128 + mc;
        if (j < NJ && col < vp.Rv_pad) {
#pragma unroll
          for (int h = 0; h < V_HP; ++h)
            if (h < s_v)
              vp.pctx[(((size_t)b * p.n_heads + g * s_v + h) * ns + u.st0) * vp.Rv_pad + col] = acc[j][h];
        }
      }
#pragma unroll
      for (int h = 0; h < V_HP; ++h)
        if (tb == h && h < s_v) {
          const size_t pi = ((size_t)b * p.n_heads + g * s_v + h) * ns + u.st0;
          vp.pm[pi] = mr[h];
          vp.pl[pi] = lr[h];
        }
      if (tb == 0 && !vp.no_wait)
        for (int i = u.item0; i < u.item0 + (u.st1 - u.st0); ++i) p.ready[i] = 0;
    }
  }
  named_bar_sync(2, 288);
  if (p.trace != nullptr && tid == 0) {
    p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 1] = gtimer();
    p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 3] = 1000000ull + 1;
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
rope_attend_tc_kernel(const __grid_constant__ CUtensorMap map_h,
                      const __grid_constant__ CUtensorMap map_uw,
                      const __grid_constant__ CUtensorMap map_v, const Params p,
                      const VParams vp) {
  pdl_enter();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  if (p.trace != nullptr && threadIdx.x == 0) {
    p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 0] = gtimer();
    p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 2] = smid_u32();
  }
  if ((int)(blockIdx.x >> 1) < p.score_pairs) {
    score_role<2, 2, EPI_WARPS>(map_h, map_uw, p, smem);
  } else {
    const int vcta = (int)blockIdx.x - 2 * p.score_pairs;
    value_role(map_v, p, vp, smem, vcta, (int)gridDim.x - 2 * p.score_pairs);
  }
}

// Deterministic merge of the value units' partials (runs after the fused or
// the standalone value kernel): block = (128 columns, head, sequence).  The
// group's unit slots are found in parallel (a slot starts a unit iff it is
// the group's first super-tile or a window start of the VSched), compacted in
// token order, and summed with 8 independent float4 loads in flight.
__global__ void __launch_bounds__(128)
value_merge_kernel(const float* __restrict__ pm, const float* __restrict__ pl,
                   const float* __restrict__ pctx, int ns, int Rv_pad, int n_heads, int s_v, int G,
                   int B, const int* __restrict__ t_dev, int score_pairs, int vc,
                   const int* __restrict__ ranks_v, const int* __restrict__ o_off,
                   float* __restrict__ ctx, int ld_ctx) {
  pdl_enter();
  extern __shared__ float msm[];
  float* w = msm;                                    // [ns]
  int* ulist = reinterpret_cast<int*>(msm + ns);     // [ns]
  __shared__ int wcount[4];
  __shared__ float inv_l_sh;
  const int head = blockIdx.y, b = blockIdx.z, g = head / s_v;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T_rows = *t_dev + 1;
  const int n_super = (T_rows + SUPER - 1) / SUPER;
  const int total = B * G * n_super;
  const int per = (total + score_pairs - 1) / score_pairs;
  const int bg = b * G + g;
  if (vc <= 0) vc = per;  // standalone value kernel: one window per CTA
  // (1) unit starts of this group, compacted in order (chunks of 128 slots)
  int nu = 0;
  for (int x0 = 0; x0 < n_super; x0 += 128) {
    const int x = x0 + tid;
    bool start = false;
    if (x < n_super) {
      const int a = bg * n_super + x;
      const int off = a - (a / per) * per;
      start = x == 0 || off % vc == 0;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, start);
    if (lane == 0) wcount[warp] = __popc(bal);
    __syncthreads();
    int before = nu;
    for (int q = 0; q < warp; ++q) before += wcount[q];
    if (start) ulist[before + __popc(bal & ((1u << lane) - 1u))] = x;
    nu += wcount[0] + wcount[1] + wcount[2] + wcount[3];
    __syncthreads();
  }
  // (2) the partials of this block's columns are independent of the weights:
  // every warp issues its first units' float4 loads before warp 0 computes the
  // weights exp(m_u - M) and 1 / sum_u w_u l_u (one dependent round trip)
  const size_t base = ((size_t)b * n_heads + head) * ns;
  __shared__ float4 part4[4][32];
  const int r = ranks_v[g];
  const int col = blockIdx.x * 128 + 4 * lane;
  const float* src = pctx + base * (size_t)Rv_pad + min(col, Rv_pad - 4);
  constexpr int PRE = 8;  // units preloaded per warp (4 warps: 32 units)
  float4 pre[PRE];
#pragma unroll
  for (int i = 0; i < PRE; ++i) {
    const int q = warp + 4 * i;
    pre[i] = q < nu ? __ldcg(reinterpret_cast<const float4*>(src + (size_t)ulist[q] * Rv_pad))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (warp == 0) {
    // units q = lane + 32 k: the first two per lane stay in registers
    float mv[2] = {-INFINITY, -INFINITY}, lv[2] = {0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int q = lane + 32 * k;
      if (q < nu) {
        mv[k] = __ldcg(pm + base + ulist[q]);
        lv[k] = __ldcg(pl + base + ulist[q]);
      }
    }
    float M = fmaxf(mv[0], mv[1]);
    for (int q = lane + 64; q < nu; q += 32) M = fmaxf(M, __ldcg(pm + base + ulist[q]));
    M = warp_reduce(M, [](float x, float y) { return fmaxf(x, y); });
    float Ls = 0.f;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int q = lane + 32 * k;
      if (q < nu) {
        const float wq = __expf(mv[k] - M);
        w[q] = wq;
        Ls += wq * lv[k];
      }
    }
    for (int q = lane + 64; q < nu; q += 32) {
      const float wq = __expf(__ldcg(pm + base + ulist[q]) - M);
      w[q] = wq;
      Ls += wq * __ldcg(pl + base + ulist[q]);
    }
    Ls = warp_reduce(Ls, [](float x, float y) { return x + y; });
    if (lane == 0) inv_l_sh = 1.f / Ls;
  }
  __syncthreads();
  // (3) lane = 4 columns of this block's 128; warp w sums units w, w + 4, ...
  // in unit order, then the 4 warp sums combine in a fixed order
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int i = 0; i < PRE; ++i) {
    const int q = warp + 4 * i;
    if (q < nu) {
      const float wq = w[q];
      acc.x = fmaf(wq, pre[i].x, acc.x);
      acc.y = fmaf(wq, pre[i].y, acc.y);
      acc.z = fmaf(wq, pre[i].z, acc.z);
      acc.w = fmaf(wq, pre[i].w, acc.w);
    }
  }
#pragma unroll 8
  for (int q = warp + 4 * PRE; q < nu; q += 4) {
    const float wq = w[q];
    const float4 v = __ldcg(reinterpret_cast<const float4*>(src + (size_t)ulist[q] * Rv_pad));
    acc.x = fmaf(wq, v.x, acc.x);
    acc.y = fmaf(wq, v.y, acc.y);
    acc.z = fmaf(wq, v.z, acc.z);
    acc.w = fmaf(wq, v.w, acc.w);
  }
  part4[warp][lane] = acc;
  __syncthreads();
  if (warp != 0 || col >= r) return;
  const float4 a0 = part4[0][lane], a1 = part4[1][lane], a2 = part4[2][lane], a3 = part4[3][lane];
  const float il = inv_l_sh;
  const float av[4] = {((a0.x + a1.x) + (a2.x + a3.x)) * il, ((a0.y + a1.y) + (a2.y + a3.y)) * il,
                       ((a0.z + a1.z) + (a2.z + a3.z)) * il, ((a0.w + a1.w) + (a2.w + a3.w)) * il};
  float* dst = ctx + (size_t)b * ld_ctx + o_off[head] + col;
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (col + e < r) dst[e] = av[e];
}

// Standalone softmax + value pass on tcgen05 (after palu_rope_score_tc): every
// CTA runs value_role over a round-robin share of the (sequence, group)
// units; no readiness protocol.
// bf16 V: value role warps 0-9; packed V: + converter warps 10.. (one token row per lane)
constexpr int VALUE_THREADS_BF16 = 320;
constexpr int VALUE_THREADS_PACKED = 448;  // 4 converter warps (8 spill at 576 threads)

template <int NT>
__global__ void __launch_bounds__(NT, 1)
value_tc_kernel(const __grid_constant__ CUtensorMap map_v, const Params p, const VParams vp) {
  // H_v rows older than this step stream into the ring while the score kernel
  // drains; the producer waits before the tile holding the newest row (this
  // step's latent append, which may still be running), group A before the logits
  pdl_launch();
  if (!p.pdl_split) pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  if (p.trace != nullptr && threadIdx.x == 0) {
    p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 0] = gtimer();
    p.trace[(size_t)blockIdx.x * TRACE_STRIDE + 2] = smid_u32();
  }
  value_role(map_v, p, vp, smem, (int)blockIdx.x, (int)gridDim.x);
}

// ===========================================================================
// Rope-off score on tcgen05 (attention.py:380-388): per (sequence, key group)
//   D[128 tokens x 16] = H_k[tokens x R] (K-major SW128, TMA) x Q^T,
//   Q[16 x R] = rows h < s: scale * q_lat(head g s + h) (bf16, built in smem)
// one CTA per SM over a contiguous range of (group, 128-token tile) items; the
// latent cache streams at HBM rate, the MMA is tiny.  Warps: 0 TMA producer,
// 1 MMA issuer (+ TMEM owner), 2..5 epilogue / Q builders (warp w reads TMEM
// lane quarter w % 4).
// ===========================================================================
struct LSParams {
  int B, n_heads, s, G, R_pad, T_cap, ld_logits, ld_y, stages;
  float scale;
  const float* y;       // [B][ld_y] fp32, q_lat of head i at q_off[i]
  const int* q_off;
  const int* ranks;
  const int* t_dev;
  float* logits;
  // quantised keys (bits 2/3/4/8): converter warps 6-7 write c - z, the
  // epilogue multiplies by the token scale (quant.py:106-107)
  int bits, code_row_bytes;
  const uint8_t* codes;
  const float* scales;
  const float* zps;
};
constexpr int LS_THREADS = 256;

__global__ void __launch_bounds__(LS_THREADS, 1)
latent_score_tc_kernel(const __grid_constant__ CUtensorMap map_h, const LSParams p) {
  pdl_enter();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int kblocks = p.R_pad / KB;
  const int QB = kblocks * 2048;                      // Q bytes: per k-block 16 rows x 128 B
  uint8_t* s_h = smem;                                // stages x 16 KB
  uint8_t* s_q = s_h + p.stages * H_STAGE_BYTES;      // [2] x QB (+1 KB alias slack)
  uint64_t* full = reinterpret_cast<uint64_t*>(s_q + 2 * QB + 1024);
  uint64_t* empty = full + p.stages;
  uint64_t* dfull = empty + p.stages;  // [2] accumulator slot complete
  uint64_t* dempty = dfull + 2;        // [2] accumulator slot read (4 warps)
  uint64_t* qfull = dempty + 2;        // [2] Q buffer written
  uint64_t* qempty = qfull + 2;        // [2] Q buffer's MMAs complete
  uint32_t* tslot = reinterpret_cast<uint32_t*>(qempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T_rows = *p.t_dev + 1;
  const int ntile = (T_rows + TILE_M - 1) / TILE_M;
  const int total = p.B * p.G * ntile;
  const int per = (total + gridDim.x - 1) / gridDim.x;
  const int i0 = min(total, (int)blockIdx.x * per), i1 = min(total, i0 + per);
  if (threadIdx.x == 0) {
    prefetch_map(&map_h);
    for (int st = 0; st < p.stages; ++st) {
      mbar_init(&full[st], p.bits == 16 ? 1 : CONV_WARPS);
      mbar_init(&empty[st], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&dfull[a], 1);
      mbar_init(&dempty[a], 4);
      mbar_init(&qfull[a], 1);
      mbar_init(&qempty[a], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0) {
    if (lane == 0 && p.bits == 16) {
      const uint64_t pol_first = policy_evict_first();  // H_k is read once: keep L2 for the logits
      Ring rg;
      for (int i = i0; i < i1; ++i) {
        const int bg = i / ntile, tile = i - bg * ntile;
        for (int kb = 0; kb < kblocks; ++kb, rg.next(p.stages)) {
          const int st = rg.slot;
          mbar_wait(&empty[st], rg.phase ^ 1);
          mbar_expect_tx(&full[st], H_STAGE_BYTES);
          tma_load_2d_hint(&map_h, &full[st], s_h + st * H_STAGE_BYTES, kb * KB,
                           bg * p.T_cap + tile * TILE_M, pol_first);
        }
      }
    }
  } else if (warp >= 6) {
    // quantised keys: converter warps (rows cl, cl + 64 of each 128-token tile)
    if (p.bits != 16) {
      const int cl = (warp - 6) * 32 + lane;
      Ring rg;
      for (int i = i0; i < i1; ++i) {
        const int bg = i / ntile, tile = i - bg * ntile;
        switch (p.bits) {
          case 2: convert_tile<2, 2>(p, s_h, full, empty, bg, tile, T_rows, kblocks, cl, rg); break;
          case 3: convert_tile<3, 2>(p, s_h, full, empty, bg, tile, T_rows, kblocks, cl, rg); break;
          case 4: convert_tile<4, 2>(p, s_h, full, empty, bg, tile, T_rows, kblocks, cl, rg); break;
          default: convert_tile<8, 2>(p, s_h, full, empty, bg, tile, T_rows, kblocks, cl, rg); break;
        }
      }
    }
  } else if (warp == 1) {
    // MMA issuer: the whole warp runs the loop, one elected lane issues
    int seg = -1, cur = -1;
    Ring rg;
    for (int i = i0; i < i1; ++i) {
      const int bg = i / ntile;
      if (bg != cur) {
        if (seg >= 0 && elect_one()) umma_commit(&qempty[seg & 1]);
        __syncwarp();
        ++seg;
        cur = bg;
        mbar_wait(&qfull[seg & 1], (seg >> 1) & 1);
        fence_after();
      }
      const int k = i - i0, slot = k & 1;
      if (k >= 2) mbar_wait(&dempty[slot], ((k >> 1) - 1) & 1);
      fence_after();
      const uint32_t q0 = smem_u32(s_q + (seg & 1) * QB);
      for (int kb = 0; kb < kblocks; ++kb, rg.next(p.stages)) {
        const int st = rg.slot;
        mbar_wait(&full[st], rg.phase);
        fence_after();
        const uint32_t a0 = smem_u32(s_h + st * H_STAGE_BYTES);
        const uint64_t da = sdesc(a0), dq = sdesc(q0 + kb * 2048);  // +2 per K16 step
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < KB / 16; ++kk)
            umma_bf16_id(tmem + slot * 16, da + 2 * kk, dq + 2 * kk, IDESC_LS, (kb | kk) != 0);
          umma_commit(&empty[st]);
        }
        __syncwarp();
      }
      if (elect_one()) umma_commit(&dfull[slot]);
      __syncwarp();
    }
  } else {
    // ---------------- epilogue / Q builders (warps 2..5) ----------------
    const int q4 = warp & 3;  // TMEM lane quarter
    const int te = threadIdx.x - 64;  // 0..127
    int seg = -1, cur = -1;
    for (int i = i0; i < i1; ++i) {
      const int bg = i / ntile, tile = i - bg * ntile;
      const int b = bg / p.G, g = bg - b * p.G;
      if (bg != cur) {
        ++seg;
        cur = bg;
        const int buf = seg & 1;
        if (seg >= 2) mbar_wait(&qempty[buf], ((seg >> 1) - 1) & 1);
        // Q rows h < s: scale * q_lat (zeros past the group rank); rows >= s are
        // never read back (their D columns are ignored)
        uint8_t* qb = s_q + buf * QB;
        const int r = p.ranks[g];
        for (int idx = te; idx < p.s * p.R_pad / 2; idx += 128) {
          const int h = idx / (p.R_pad / 2), k = 2 * (idx - h * (p.R_pad / 2));
          const float* qv = p.y + (size_t)b * p.ld_y + p.q_off[g * p.s + h];
          const float v0 = k < r ? qv[k] * p.scale : 0.f, v1 = k + 1 < r ? qv[k + 1] * p.scale : 0.f;
          // int4 / int2 keys: rank k sits at the converter's K position
          // (groups of 8 / 16: k < G/2 ? 2k : 2k - G + 1)
          const int grp = p.bits == 4 ? 8 : (p.bits == 2 ? 16 : 0);
          const float vv[2] = {v0, v1};
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            int pos = k + e;
            if (grp) {
              const int ii = pos % grp;
              pos = pos - ii + (ii < grp / 2 ? 2 * ii : 2 * ii - grp + 1);
            }
            const int kb = pos / KB, w = pos % KB;
            const uint32_t off = kb * 2048 + (h >> 3) * 1024 + (h & 7) * 128 +
                                 ((((w >> 3) ^ (h & 7)) & 7) << 4) + (w & 7) * 2;
            *reinterpret_cast<__nv_bfloat16*>(qb + off) = __float2bfloat16_rn(vv[e]);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        named_bar_sync(1, 128);
        if (te == 0) mbar_arrive(&qfull[buf]);
      }
      const int k = i - i0, slot = k & 1;
      mbar_wait(&dfull[slot], (k >> 1) & 1);
      fence_after();
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(q4 * 32) << 16) + slot * 16, v);
      tmem_wait_ld();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dempty[slot]);
      const int t = tile * TILE_M + q4 * 32 + lane;
      if (t < T_rows) {
        const float sq = p.bits == 16 ? 1.f : __ldg(p.scales + (size_t)bg * p.T_cap + t);
#pragma unroll
        for (int h = 0; h < 16; ++h)
          if (h < p.s) p.logits[((size_t)b * p.n_heads + g * p.s + h) * p.ld_logits + t] = v[h] * sq;
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------
// tile bases: cos/sin(t0 * th_j), t0 = 128 * row (fp64 angle reduction);
// offsets: cos/sin(delta * th_j), delta in [0, 128).
// Row layout per frequency pair (2p, 2p + 1): {cos 2p, cos 2p+1, sin 2p, sin 2p+1}
// -- the float2 halves the epilogue's FFMA2s take without register moves.
__global__ void rope_table_kernel(const double* __restrict__ theta, int half, int n_tiles,
                                  float* __restrict__ tab) {
  const int total = (n_tiles + 128) * half;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int row = i / half, j = i - row * half;
    const double pos = row < n_tiles ? 128.0 * row : (double)(row - n_tiles);
    double sn, cs;
    sincos_big(pos * theta[j], &sn, &cs);
    float* e = tab + (size_t)row * 2 * half + 4 * (j >> 1) + (j & 1);
    e[0] = (float)cs;
    e[2] = (float)sn;
  }
}

// packed key codes: uint8 rows, one box = the whole row x 128 rows (L2 prefetch only)
static int make_map_u8(CUtensorMap* m, const void* base, uint64_t row_bytes, uint64_t rows) {
  EncodeTiledFn fn = encode_fn();
  PALU_REQUIRE(fn != nullptr, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {row_bytes, rows};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {(cuuint32_t)row_bytes, 128};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (codes) failed (%d)", (int)r);
    return PALU_ECUDA;
  }
  return PALU_OK;
}

static int make_map_2d(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows,
                       uint32_t box_cols, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  PALU_REQUIRE(fn != nullptr, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return PALU_ECUDA;
  }
  return PALU_OK;
}

#include "palu_vq.cuh"
#include "palu_lsq.cuh"

}  // namespace tc
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
  tc::rope_table_kernel<<<256, 256, 0, (cudaStream_t)stream>>>(theta, half, n_tiles, rope_tab);
  PALU_LAUNCHED();
  return PALU_OK;
}

int palu_rope_score_tc_splits(int s_k, int R_pad) {
  using namespace palu::tc;
  // one rank slice: the 2-SM pair keeps the whole UW operand resident
  return ((s_k == 2 || s_k == 4) && R_pad % KB == 0 && R_pad <= 256) ? 1 : 0;
}

static unsigned long long* g_trace = nullptr;  // diagnostics (PALU_FUSED_TRACE)
static int g_trace_ctas = 0;

int palu_rope_score_tc(int bits, const void* hk, const float* scales, const float* zps, int B,
                       int n_heads, int s_k, int G, int R_pad, int T_cap, const void* uw,
                       const float* rope_tab, const int* t_dev, float* logits, int ld_logits,
                       void* stream) {
  return palu_rope_score_tc_pf(bits, hk, scales, zps, B, n_heads, s_k, G, R_pad, T_cap, uw, rope_tab, t_dev,
                               logits, ld_logits, nullptr, 0, stream);
}

// qh > 1: replicated-B groups (uw = the static K-major B^T of each group's KV
// head, [B][G][128][R_pad]; qrot = scale x RoPE(q) rows), s_k = 1 per group
static int rope_score_impl(int bits, const void* hk, const float* scales, const float* zps, int B,
                           int n_heads, int s_k, int G, int R_pad, int T_cap, const void* uw,
                           const float* rope_tab, const int* t_dev, float* logits, int ld_logits,
                           const void* l2_prefetch, long long l2_prefetch_bytes, const float* qrot, int qh,
                           void* stream) {
  using namespace palu::tc;
  if (bits != 16 && bits != 2 && bits != 3 && bits != 4 && bits != 8) {
    set_error("palu_rope_score_tc: bits %d unsupported", bits);
    return PALU_EUNSUPPORTED;
  }
  if (qh > 1 ? (s_k != 1 || R_pad % KB != 0 || R_pad > 256 || G * qh != n_heads)
             : (!palu_rope_score_tc_splits(s_k, R_pad) || G * s_k != n_heads)) {
    set_error("palu_rope_score_tc: unsupported shape (R_pad %d, s_k %d)", R_pad, s_k);
    return PALU_EUNSUPPORTED;
  }
  const int row_bytes = bits == 16 ? R_pad * 2 : R_pad * bits / 8;
  PALU_REQUIRE(((uintptr_t)hk & 15) == 0 && ((uintptr_t)uw & 15) == 0, "tc: unaligned operands");
  PALU_REQUIRE(bits == 16 || (row_bytes % 16 == 0 && row_bytes <= 256 && scales && zps),
               "palu_rope_score_tc: quantised rows need 16-byte multiples <= 256 B, scales and "
               "zero points");
  CUtensorMap map_h, map_uw;
  int rc = bits == 16 ? make_map_2d(&map_h, hk, R_pad, (uint64_t)B * G * T_cap, KB, TILE_M)
                      : make_map_u8(&map_h, hk, row_bytes, (uint64_t)B * G * T_cap);
  if (rc) return rc;
  const int kblocks = R_pad / KB;
  // heads per accumulator unit: 1 (quad-buffered N128) for short ranks
  // (UH 1 measured slower at r 128: an N128 pair-MMA costs as much as an N256
  // one, tools/score_trace.py; kept as an option)
  const int uh = qh > 1 ? 1 : (getenv("PALU_SCORE_UH") ? atoi(getenv("PALU_SCORE_UH")) : 2);
  PALU_REQUIRE(uh == 1 || uh == 2, "PALU_SCORE_UH must be 1 or 2");
  PALU_REQUIRE(qh == 1 || (qh == 4 && bits == 16 && qrot != nullptr && ((uintptr_t)qrot & 15) == 0),
               "palu_rope_score_tc_rep: 4 query heads per KV head, raw bf16 keys, aligned rotated queries");
  PALU_REQUIRE(SCORE_EPI == 8 || uh == 2 || bits == 16,
               "PALU_SCORE_UH=1 with packed keys needs the 8-warp score epilogue build");
  rc = make_map_2d(&map_uw, uw, R_pad, (uint64_t)B * G * s_k * 128, KB, uh == 2 ? TILE_M : 64);
  if (rc) return rc;
  const int fixed = kblocks * s_k * (HEAD_BYTES / 2) + (qh > 1 ? score_fixed_bytes(qh, qh) : SCORE_FIXED_BYTES);
  int stages = (SMEM_LIMIT - fixed) / H_STAGE_BYTES;
  if (stages > 12) stages = 12;
  PALU_REQUIRE(stages >= kblocks, "tc: not enough shared memory (%d stages)", stages);
  const size_t smem = (size_t)fixed + (size_t)stages * H_STAGE_BYTES;
  static bool attr = false;
  if (!attr) {
    PALU_CK(cudaFuncSetAttribute(rope_score_tc_kernel<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SMEM_LIMIT));
    PALU_CK(cudaFuncSetAttribute(rope_score_tc_kernel<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SMEM_LIMIT));
    PALU_CK(cudaFuncSetAttribute(rope_score_tc_kernel<2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SMEM_LIMIT));
    PALU_CK(cudaFuncSetAttribute(rope_score_tc_kernel<1, 2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SMEM_LIMIT));
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  Params prm = {};
  prm.pdl_split = pdl_split();
  prm.B = B;
  prm.n_heads = n_heads;
  prm.s_k = s_k;
  prm.G = G;
  prm.R_pad = R_pad;
  prm.T_cap = T_cap;
  prm.ld_logits = ld_logits;
  prm.n_tab = (T_cap + 127) / 128 + 1;
  prm.stages = stages;
  prm.score_pairs = (sms & ~1) / 2;
  prm.ready = nullptr;
  prm.mode = diag_env("PALU_TC_PROFILE_MODE");
  // packed keys: the converter warps read code rows with plain loads, which
  // the L2 prefetch 3 items ahead still helps (-0.5 % step, int4); raw keys
  // stream through TMA and do better without it (tools/pf_sweep.sh)
  prm.pf_dist = getenv("PALU_TC_PF") ? atoi(getenv("PALU_TC_PF")) : (bits == 16 ? PF_DIST : 3);
  prm.rope_tab = reinterpret_cast<const float2*>(rope_tab);
  prm.l2pf = reinterpret_cast<const uint8_t*>(l2_prefetch);
  prm.l2pf_bytes = l2_prefetch ? l2_prefetch_bytes : 0;
  prm.t_dev = t_dev;
  prm.logits = logits;
  prm.trace = nullptr;
  prm.bits = bits;
  prm.code_row_bytes = row_bytes;
  prm.codes = reinterpret_cast<const uint8_t*>(hk);
  prm.scales = scales;
  prm.zps = zps;
  prm.qrot = qrot;
  if (getenv("PALU_SCORE_TRACE")) {  // diagnostics: per-head-pair timeline (tools/score_trace.py)
    if (!g_trace) PALU_CK(cudaMalloc(&g_trace, (size_t)1024 * TRACE_STRIDE * 8));
    PALU_CK(cudaMemsetAsync(g_trace, 0, (size_t)1024 * TRACE_STRIDE * 8, (cudaStream_t)stream));
    prm.trace = g_trace;
    g_trace_ctas = sms & ~1;
  }
  if (qh > 1)
    PALU_CK(launch_k(rope_score_tc_kernel<1, 2, 4>, dim3(sms & ~1), dim3(THREADS_S), smem,
                     (cudaStream_t)stream, map_h, map_uw, prm));
  else if (uh == 1)
    PALU_CK(launch_k(rope_score_tc_kernel<1, 2>, dim3(sms & ~1), dim3(THREADS_S), smem, (cudaStream_t)stream,
                     map_h, map_uw, prm));
  else if (bits != 16)
    PALU_CK(launch_k(rope_score_tc_kernel<2, 4>, dim3(sms & ~1), dim3(THREADS_SQ), smem,
                     (cudaStream_t)stream, map_h, map_uw, prm));
  else
    PALU_CK(launch_k(rope_score_tc_kernel<2, 2>, dim3(sms & ~1), dim3(THREADS_S), smem, (cudaStream_t)stream,
                     map_h, map_uw, prm));
  PALU_LAUNCHED();
  return PALU_OK;
}

int palu_rope_score_tc_pf(int bits, const void* hk, const float* scales, const float* zps, int B,
                          int n_heads, int s_k, int G, int R_pad, int T_cap, const void* uw,
                          const float* rope_tab, const int* t_dev, float* logits, int ld_logits,
                          const void* l2_prefetch, long long l2_prefetch_bytes, void* stream) {
  return rope_score_impl(bits, hk, scales, zps, B, n_heads, s_k, G, R_pad, T_cap, uw, rope_tab, t_dev, logits,
                         ld_logits, l2_prefetch, l2_prefetch_bytes, nullptr, 1, stream);
}

int palu_rope_score_tc_rep(const void* hk, int B, int n_heads, int G, int R_pad, int T_cap, const void* bkt,
                           const float* qrot, const float* rope_tab, const int* t_dev, float* logits,
                           int ld_logits, void* stream) {
  return rope_score_impl(16, hk, nullptr, nullptr, B, n_heads, 1, G, R_pad, T_cap, bkt, rope_tab, t_dev, logits,
                         ld_logits, nullptr, 0, qrot, G > 0 ? n_heads / G : 0, stream);
}

// ---- fused score + softmax + value ------------------------------------------

// Copies the last traced fused launch's timeline ([CTA][TRACE_STRIDE] u64:
// start, end, smid, role/count, events...) to host; returns the CTA count.
int palu_fused_trace(unsigned long long* host, size_t max_ctas) {
  using palu::tc::TRACE_STRIDE;
  if (!g_trace) return 0;
  const size_t n = max_ctas < (size_t)g_trace_ctas ? max_ctas : (size_t)g_trace_ctas;
  PALU_CK(cudaDeviceSynchronize());
  PALU_CK(cudaMemcpy(host, g_trace, n * TRACE_STRIDE * 8, cudaMemcpyDeviceToHost));
  return (int)n;
}

// Cluster-of-2 residency of the fused kernel at its launch configuration.
int palu_fused_max_clusters(int smem_bytes) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 2;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(palu::tc::THREADS);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  PALU_CK(cudaFuncSetAttribute(palu::tc::rope_attend_tc_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, palu::tc::SMEM_LIMIT - 2048));
  int n = 0;
  PALU_CK(cudaOccupancyMaxActiveClusters(&n, palu::tc::rope_attend_tc_kernel, &cfg));
  return n;
}

static int fused_ns_cap(int T_cap) {
  using palu::tc::SUPER;
  return (T_cap + SUPER - 1) / SUPER;
}

// Workspace carve-up shared by the fused and standalone value kernels; every
// array starts on a 256-byte boundary (float4 partial loads in the merge).
struct ValueWs {
  unsigned* tickets;
  int* ready;
  float *pm, *pl, *pctx;
  size_t bytes;
};
static ValueWs value_ws(void* base, int B, int n_heads, int G, int Rv_pad, int T_cap) {
  using palu::tc::SUPER;
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t nc = fused_ns_cap(T_cap);
  const size_t items = (size_t)B * G * ((T_cap + SUPER - 1) / SUPER);
  const size_t head = (size_t)B * n_heads * nc;
  uint8_t* p = reinterpret_cast<uint8_t*>(base);
  size_t o = 256;
  ValueWs w;
  w.tickets = reinterpret_cast<unsigned*>(p + o);
  o = up(o + sizeof(unsigned) * (size_t)B * G);
  w.ready = reinterpret_cast<int*>(p + o);
  o = up(o + sizeof(int) * items);
  w.pm = reinterpret_cast<float*>(p + o);
  o = up(o + sizeof(float) * head);
  w.pl = reinterpret_cast<float*>(p + o);
  o = up(o + sizeof(float) * head);
  w.pctx = reinterpret_cast<float*>(p + o);
  o = up(o + sizeof(float) * head * (size_t)Rv_pad);
  w.bytes = o;
  return w;
}

size_t palu_rope_attend_workspace(int B, int n_heads, int G, int Rv_pad, int T_cap) {
  return value_ws(nullptr, B, n_heads, G, Rv_pad, T_cap).bytes;
}

static int launch_value_merge(const float* pm, const float* pl, const float* pctx, int ns, int Rv_pad,
                              int n_heads, int s, int G, int B, const int* t_dev, int score_pairs,
                              int vc, const int* ranks_v, const int* o_off, float* ctx, int ld_ctx,
                              cudaStream_t st) {
  using namespace palu::tc;
  const size_t smem = (size_t)ns * 8;
  static bool attr = false;
  if (!attr) {
    PALU_CK(cudaFuncSetAttribute(value_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 100 * 1024));
    attr = true;
  }
  PALU_REQUIRE(smem <= 100 * 1024, "value merge: too many super-tiles (%d)", ns);
  PALU_CK(launch_k(value_merge_kernel, dim3((Rv_pad + 127) / 128, n_heads, B), dim3(128), smem, st,
                   pm, pl, pctx, ns, Rv_pad, n_heads, s, G, B, t_dev, score_pairs, vc, ranks_v, o_off,
                   ctx, ld_ctx));
  PALU_LAUNCHED();
  return PALU_OK;
}

int palu_rope_attend_tc(const void* hk, const void* hv, int B, int n_heads, int s, int G,
                        int Rk_pad, int Rv_pad, int T_cap, const void* uw, const float* rope_tab,
                        const int* t_dev, float* logits, int ld_logits, const int* ranks_v,
                        const int* o_off, float* ctx, int ld_ctx, void* workspace,
                        int score_sms, void* stream) {
  using namespace palu::tc;
  if (!palu_rope_score_tc_splits(s, Rk_pad) || G * s != n_heads || Rv_pad % KB != 0 ||
      Rv_pad > 512 || s > V_HP) {
    set_error("palu_rope_attend_tc: unsupported shape (Rk %d, Rv %d, s %d)", Rk_pad, Rv_pad, s);
    return PALU_EUNSUPPORTED;
  }
  PALU_REQUIRE(((uintptr_t)hk & 15) == 0 && ((uintptr_t)uw & 15) == 0 && ((uintptr_t)hv & 15) == 0,
               "tc: unaligned operands");
  CUtensorMap map_h, map_uw;
  int rc = make_map_2d(&map_h, hk, Rk_pad, (uint64_t)B * G * T_cap, KB, TILE_M);
  if (rc) return rc;
  rc = make_map_2d(&map_uw, uw, Rk_pad, (uint64_t)B * G * s * 128, KB, TILE_M);
  if (rc) return rc;
  const int kblocks = Rk_pad / KB;
  const int fixed = 1024 + kblocks * (s / 2) * HEAD_BYTES + SCORE_FIXED_BYTES;
  const int dyn_limit = SMEM_LIMIT - 2048;  // the value role has ~1 KB of static smem
  int stages = (dyn_limit - fixed) / H_STAGE_BYTES;
  if (stages > 12) stages = 12;
  PALU_REQUIRE(stages >= kblocks, "tc: not enough shared memory (%d stages)", stages);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  sms &= ~1;
  if (score_sms <= 0) {
    // balance tensor time against value-stream time (per-SM rates measured on B200:
    // ~8.5 TFLOP/s of reconstruction, ~100 GB/s of value streaming per SM)
    const double flops = 2.0 * n_heads * (double)Rk_pad * 128.0;   // per token
    const double bytes = (double)G * Rv_pad * 2.0;                  // per token
    const double ts = flops / 8.5e12, tv = bytes / 1.0e11;
    score_sms = (int)(sms * ts / (ts + tv) + 0.5);
  }
  score_sms &= ~1;
  if (score_sms < 2) score_sms = 2;
  if (score_sms > sms - 2) score_sms = sms - 2;
  const int vc = getenv("PALU_FUSED_VC") ? atoi(getenv("PALU_FUSED_VC")) : 4;  // tuning only
  const int nc_max = fused_ns_cap(T_cap);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  const ValueWs W = value_ws(ws, B, n_heads, G, Rv_pad, T_cap);
  unsigned* tickets = W.tickets;
  int* ready = W.ready;
  float *pm = W.pm, *pl = W.pl, *pctx = W.pctx;
  Params prm = {};
  prm.pdl_split = pdl_split();
  prm.B = B;
  prm.n_heads = n_heads;
  prm.s_k = s;
  prm.G = G;
  prm.R_pad = Rk_pad;
  prm.T_cap = T_cap;
  prm.ld_logits = ld_logits;
  prm.n_tab = (T_cap + 127) / 128 + 1;
  prm.stages = stages;
  prm.score_pairs = score_sms / 2;
  prm.ready = ready;
  prm.mode = 0;
  prm.pf_dist = PF_DIST;
  prm.rope_tab = reinterpret_cast<const float2*>(rope_tab);
  prm.t_dev = t_dev;
  prm.logits = logits;
  prm.trace = nullptr;
  prm.bits = 16;
  if (getenv("PALU_FUSED_TRACE")) {
    if (!g_trace) PALU_CK(cudaMalloc(&g_trace, (size_t)1024 * TRACE_STRIDE * 8));
    PALU_CK(cudaMemsetAsync(g_trace, 0, (size_t)1024 * TRACE_STRIDE * 8, (cudaStream_t)stream));
    prm.trace = g_trace;
    g_trace_ctas = sms;
  }
  CUtensorMap map_v;
  rc = make_map_2d(&map_v, hv, Rv_pad, (uint64_t)B * G * T_cap, KB, TILE_M);
  if (rc) return rc;
  VParams vp = {};
  vp.Rv_pad = Rv_pad;
  vp.vc = vc;
  const size_t side = (size_t)2 * (V_SUB / 64) * 1024 + 1024 + 4 * V_HP * 4 + 16 * 64 + 64;
  // the value role takes whatever the score role leaves: launch at the limit
  const size_t smem_launch = (size_t)dyn_limit;
  vp.v_stages = (int)(((long long)smem_launch - 1024 - (long long)side) / V_STAGE);
  PALU_REQUIRE(vp.v_stages >= 2, "palu_rope_attend_tc: value ring too small (%d)", vp.v_stages);
  if (vp.v_stages > 8) vp.v_stages = 8;  // 32 KB stages
  vp.tickets = tickets;
  vp.pm = pm;
  vp.pl = pl;
  vp.pctx = pctx;
  vp.ns_cap = nc_max;
  vp.ranks_v = ranks_v;
  vp.o_off = o_off;
  vp.ctx_out = ctx;
  vp.ld_ctx = ld_ctx;
  vp.no_wait = 0;
  vp.bits = 16;
  vp.raw_slots = 0;
  vp.code_row_bytes = Rv_pad * 2;
  vp.codes = nullptr;
  vp.scales = vp.zps = nullptr;
  static bool attr = false;
  if (!attr) {
    PALU_CK(cudaFuncSetAttribute(rope_attend_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 dyn_limit));
    attr = true;
  }
  PALU_CK(launch_k(rope_attend_tc_kernel, dim3(sms), dim3(THREADS), smem_launch, (cudaStream_t)stream,
                   map_h, map_uw, map_v, prm, vp));
  PALU_LAUNCHED();
  return launch_value_merge(pm, pl, pctx, nc_max, Rv_pad, n_heads, s, G, B, t_dev, prm.score_pairs,
                            vc, ranks_v, o_off, ctx, ld_ctx, (cudaStream_t)stream);
}


// Packed V (2/4/8-bit codes) on the int8 tensor pipe (palu_vq.cuh), then the
// deterministic merge.  PALU_VALUE_KERNEL=tc_quant_bf16 keeps the earlier
// converter-to-bf16 kernel (A/B timing).
static bool value_q_enabled(int bits) {
  const char* e = getenv("PALU_VALUE_KERNEL");
  // raw bf16 values: the value role (value_tc_kernel) measured faster than
  // value_q_kernel<16> (74 vs 86 us at r 256); PALU_VALUE_KERNEL=tc_bf16_q for A/B
  if (bits == 16) return e && strcmp(e, "tc_bf16_q") == 0;
  return !(e && strcmp(e, "tc_quant_bf16") == 0);
}

static int launch_value_q(int bits, const void* hv, const float* scales, const float* zps, int B,
                          int n_heads, int s, int G, int Rv_pad, int T_cap, const float* logits,
                          int ld_logits, const int* t_dev, const int* ranks_v, const int* o_off,
                          float* ctx, int ld_ctx, void* workspace, cudaStream_t st) {
  using namespace palu::tc;
  PALU_REQUIRE(Rv_pad % 128 == 0 && Rv_pad <= 512 && s <= V_HP,
               "palu_value_tc (int8 pipe): unsupported shape (Rv %d, s %d)", Rv_pad, s);
  PALU_REQUIRE(T_cap % TILE_M == 0, "palu_value_tc: packed V needs T_cap %% 128 == 0 (got %d)", T_cap);
  const int row_bytes = Rv_pad * bits / 8;
  // packed codes move as 1-D bulk copies (the tensor map is unused); raw bf16
  // rows as {64 columns, 128 tokens} SW128 boxes straight into the operand
  CUtensorMap map_c = {};
  if (bits == 16) {
    const int rc = make_map_2d(&map_c, hv, Rv_pad, (uint64_t)B * G * T_cap, KB, TILE_M);
    if (rc) return rc;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const ValueWs W = value_ws(workspace, B, n_heads, G, Rv_pad, T_cap);
  VQParams p = {};
  p.B = B;
  p.n_heads = n_heads;
  p.s = s;
  p.G = G;
  p.Rv_pad = Rv_pad;
  p.T_cap = T_cap;
  p.ld_logits = ld_logits;
  p.row_bytes = row_bytes;
  p.box_bytes = row_bytes;  // raw slots hold [128 rows][row_bytes] (1-D bulk copies)
  p.codes = reinterpret_cast<const uint8_t*>(hv);
  p.ns_cap = fused_ns_cap(T_cap);
  p.t_dev = t_dev;
  p.logits = logits;
  p.scales = scales;
  p.zps = zps;
  p.pm = W.pm;
  p.pl = W.pl;
  p.pctx = W.pctx;
  p.trace = nullptr;
  p.diag = diag_env("PALU_VQ_DIAG");
  if (getenv("PALU_FUSED_TRACE")) {  // diagnostics: per-CTA timeline (tools/vq_trace.py)
    if (!g_trace) PALU_CK(cudaMalloc(&g_trace, (size_t)1024 * TRACE_STRIDE * 8));
    PALU_CK(cudaMemsetAsync(g_trace, 0, (size_t)1024 * TRACE_STRIDE * 8, st));
    p.trace = g_trace;
    g_trace_ctas = sms;
  }
  const int RB = TILE_M * row_bytes;
  const int dyn_limit = SMEM_LIMIT - 2048;
  // operand ring slots hold whole blocks (NJ column tiles); 2-4 of them, the
  // raw code ring (bulk-copy landing zone) takes the rest, at most 6 blocks.
  // bf16: no raw ring, the operand ring holds up to 8 tiles of 32 KB
  const int NJ = Rv_pad / 128;
  const int OB = bits == 16 ? VQ_BSTAGE : NJ * VQ_STAGE;
  const int RS = RB;  // raw slot: the block's codes
  const int pbuf = VQ_NB * (bits == 16 ? 4096 : 2048);
  const int misc = 1024 + 2 * pbuf + (2 * (V_HP + 1) + 2) * 4 + 2 * VQ_A * V_HP * (4 + 4) + 6 * 8 + 16 + 8;
  if (bits == 16) {
    p.raw_slots = 0;
    p.stages = (dyn_limit - misc) / (OB + 16);
    if (p.stages > 8) p.stages = 8;
    PALU_REQUIRE(p.stages >= 2, "palu_value_tc (bf16): operand ring too small (%d)", p.stages);
  } else {
    // two operand blocks (the MMA drains a block in ~0.3 us); the raw ring --
    // bytes in flight per SM -- takes the rest (2 slots left the converters
    // waiting ~1 us per block on bulk-copy latency at r_v 384)
    p.stages = 2;
    p.raw_slots = (dyn_limit - misc - p.stages * (OB + 16)) / (RS + 16);
    if (p.raw_slots > 6) p.raw_slots = 6;
    PALU_REQUIRE(p.raw_slots >= 2, "palu_value_tc (int8 pipe): raw ring too small (%d)", p.raw_slots);
  }
  const size_t smem = (size_t)misc + (size_t)p.raw_slots * (RS + 16) + (size_t)p.stages * (OB + 16);
  static bool attr = false;
  if (!attr) {
    PALU_CK(cudaFuncSetAttribute(value_q_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_limit));
    PALU_CK(cudaFuncSetAttribute(value_q_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_limit));
    PALU_CK(cudaFuncSetAttribute(value_q_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_limit));
    PALU_CK(cudaFuncSetAttribute(value_q_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_limit));
    attr = true;
  }
  if (bits == 2)
    PALU_CK(launch_k(value_q_kernel<2>, dim3(sms), dim3(VQ_THREADS), smem, st, map_c, p));
  else if (bits == 4)
    PALU_CK(launch_k(value_q_kernel<4>, dim3(sms), dim3(VQ_THREADS), smem, st, map_c, p));
  else if (bits == 16)
    PALU_CK(launch_k(value_q_kernel<16>, dim3(sms), dim3(VQ_THREADS), smem, st, map_c, p));
  else
    PALU_CK(launch_k(value_q_kernel<8>, dim3(sms), dim3(VQ_THREADS), smem, st, map_c, p));
  PALU_LAUNCHED();
  return launch_value_merge(W.pm, W.pl, W.pctx, p.ns_cap, Rv_pad, n_heads, s, G, B, t_dev, sms, 0,
                            ranks_v, o_off, ctx, ld_ctx, st);
}

// Standalone tcgen05 softmax + value (the unfused path's second kernel).
int palu_value_tc(int bits, const void* hv, const float* scales, const float* zps, int B,
                  int n_heads, int s, int G, int Rv_pad, int T_cap, const float* logits,
                  int ld_logits, const int* t_dev, const int* ranks_v, const int* o_off, float* ctx,
                  int ld_ctx, void* workspace, void* stream) {
  using namespace palu::tc;
  if (G * s != n_heads || Rv_pad % KB != 0 || Rv_pad > 512 || s > V_HP ||
      (bits != 16 && (Rv_pad % 128 != 0 || (bits != 2 && bits != 3 && bits != 4 && bits != 8)))) {
    set_error("palu_value_tc: unsupported shape (bits %d, Rv %d, s %d)", bits, Rv_pad, s);
    return PALU_EUNSUPPORTED;
  }
  PALU_REQUIRE(((uintptr_t)hv & 15) == 0, "palu_value_tc: unaligned H_v");
  PALU_REQUIRE(bits == 16 || (scales && zps), "palu_value_tc: quantised values need scales/zps");
  if ((bits == 2 || bits == 4 || bits == 8 || (bits == 16 && Rv_pad % 128 == 0)) &&
      value_q_enabled(bits))
    return launch_value_q(bits, hv, scales, zps, B, n_heads, s, G, Rv_pad, T_cap, logits, ld_logits,
                          t_dev, ranks_v, o_off, ctx, ld_ctx, workspace, (cudaStream_t)stream);
  CUtensorMap map_v = {};
  const int row_bytes = bits == 16 ? Rv_pad * 2 : Rv_pad * bits / 8;
  if (bits == 16) {
    int rc = make_map_2d(&map_v, hv, Rv_pad, (uint64_t)B * G * T_cap, KB, TILE_M);
    if (rc) return rc;
  } else {
    // packed V: code tiles {128 codes, 128 rows} and the per-token zero points
    EncodeTiledFn fn = encode_fn();
    PALU_REQUIRE(fn != nullptr, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)row_bytes, (cuuint64_t)B * G * T_cap};
    const cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
    const cuuint32_t box[2] = {(cuuint32_t)(16 * bits), (cuuint32_t)TILE_M}, es[2] = {1, 1};
    CUresult r = fn(&map_v, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(hv), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    PALU_REQUIRE(r == CUDA_SUCCESS, "palu_value_tc: code tensor map failed (%d)", (int)r);
    PALU_REQUIRE(T_cap % TILE_M == 0, "palu_value_tc: packed V needs T_cap %% 128 == 0 (got %d)", T_cap);
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int vc = 0;
  const int nc_max = fused_ns_cap(T_cap);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  const ValueWs W = value_ws(ws, B, n_heads, G, Rv_pad, T_cap);
  unsigned* tickets = W.tickets;
  int* ready = W.ready;
  float *pm = W.pm, *pl = W.pl, *pctx = W.pctx;
  Params prm = {};
  prm.pdl_split = pdl_split();
  prm.B = B;
  prm.n_heads = n_heads;
  prm.s_k = s;
  prm.G = G;
  prm.T_cap = T_cap;
  prm.ld_logits = ld_logits;
  prm.score_pairs = sms;  // one contiguous window of items per CTA (vc = per)
  prm.mode = diag_env("PALU_VALUE_DIAG");  // diagnostic builds only
  prm.ready = ready;
  prm.t_dev = t_dev;
  prm.logits = const_cast<float*>(logits);
  prm.trace = nullptr;
  if (getenv("PALU_FUSED_TRACE")) {
    if (!g_trace) PALU_CK(cudaMalloc(&g_trace, (size_t)1024 * TRACE_STRIDE * 8));
    PALU_CK(cudaMemsetAsync(g_trace, 0, (size_t)1024 * TRACE_STRIDE * 8, (cudaStream_t)stream));
    prm.trace = g_trace;
    g_trace_ctas = sms;
  }
  VParams vp = {};
  vp.Rv_pad = Rv_pad;
  vp.vc = vc;
  const int dyn_limit = SMEM_LIMIT - 2048;
  vp.raw_slots = 0;
  size_t raw_bytes = 0;
  if (bits != 16) {
    const int rb = TILE_M * 16 * bits + TILE_M * 4;
    vp.raw_slots = V_RAW_BYTES / rb;
    raw_bytes = (size_t)vp.raw_slots * rb + 16 * vp.raw_slots + 256;
  }
  const size_t side = (size_t)2 * (V_SUB / 64) * 1024 + 1024 + 4 * V_HP * 4 + 16 * 64 + 64 + raw_bytes;
  vp.v_stages = (int)(((long long)dyn_limit - 1024 - (long long)side) / V_STAGE);
  PALU_REQUIRE(vp.v_stages >= 2, "palu_value_tc: value ring too small (%d)", vp.v_stages);
  if (vp.v_stages > 8) vp.v_stages = 8;  // 32 KB stages
  vp.tickets = tickets;
  vp.pm = pm;
  vp.pl = pl;
  vp.pctx = pctx;
  vp.ns_cap = nc_max;
  vp.ranks_v = ranks_v;
  vp.o_off = o_off;
  vp.ctx_out = ctx;
  vp.ld_ctx = ld_ctx;
  vp.no_wait = 1;
  vp.bits = bits;
  vp.code_row_bytes = row_bytes;
  vp.codes = reinterpret_cast<const uint8_t*>(hv);
  vp.scales = scales;
  vp.zps = zps;
  static bool attr = false;
  if (!attr) {
    PALU_CK(cudaFuncSetAttribute(value_tc_kernel<VALUE_THREADS_BF16>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_limit));
    PALU_CK(cudaFuncSetAttribute(value_tc_kernel<VALUE_THREADS_PACKED>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_limit));
    attr = true;
  }
  if (bits == 16)
    PALU_CK(launch_k(value_tc_kernel<VALUE_THREADS_BF16>, dim3(sms), dim3(VALUE_THREADS_BF16),
                     (size_t)dyn_limit, (cudaStream_t)stream, map_v, prm, vp));
  else
    PALU_CK(launch_k(value_tc_kernel<VALUE_THREADS_PACKED>, dim3(sms), dim3(VALUE_THREADS_PACKED),
                     (size_t)dyn_limit, (cudaStream_t)stream, map_v, prm, vp));
  PALU_LAUNCHED();
  return launch_value_merge(pm, pl, pctx, nc_max, Rv_pad, n_heads, s, G, B, t_dev, sms, vc, ranks_v,
                            o_off, ctx, ld_ctx, (cudaStream_t)stream);
}


// Rope-off score on tcgen05 (bf16 latents, s <= 16, R_pad % 64 == 0, <= 256).
// Rope-off packed keys on the int8 tensor pipe (palu_lsq.cuh).
static int launch_latent_score_q(int bits, const void* hk, const float* scales, const float* zps, int B,
                                 int n_heads, int s, int G, int R_pad, int T_cap, const float* y, int ld_y,
                                 const int* q_off, const int* ranks, float scale, const int* t_dev,
                                 float* logits, int ld_logits, cudaStream_t st) {
  using namespace palu::tc;
  LQParams p = {};
  p.B = B;
  p.n_heads = n_heads;
  p.s = s;
  p.G = G;
  p.R_pad = R_pad;
  p.T_cap = T_cap;
  p.ld_logits = ld_logits;
  p.ld_y = ld_y;
  p.row_bytes = R_pad * bits / 8;
  p.scale = scale;
  p.y = y;
  p.q_off = q_off;
  p.ranks = ranks;
  p.t_dev = t_dev;
  p.logits = logits;
  p.codes = reinterpret_cast<const uint8_t*>(hk);
  p.scales = scales;
  p.zps = zps;
  p.trace = nullptr;
  if (kTrace && getenv("PALU_LSQ_TRACE")) {  // diagnostics (tools/lsq_trace.py)
    int sms_ = 148;
    cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, 0);
    if (!g_trace) PALU_CK(cudaMalloc(&g_trace, (size_t)1024 * TRACE_STRIDE * 8));
    PALU_CK(cudaMemsetAsync(g_trace, 0, (size_t)1024 * TRACE_STRIDE * 8, st));
    p.trace = g_trace;
    g_trace_ctas = sms_;
  }
  const int OB = R_pad / 128 * 16384, DB = R_pad / 128 * 2048, RB = TILE_M * p.row_bytes;
  const int limit = SMEM_LIMIT - 2048;
  const int misc = 1024 + 2 * DB + 256 + 16 * 8 + 64;  // align, digits, scalars, barriers, TMEM slot
  // three operand stages (the converter runs ahead of the MMA's ~0.5 us
  // commit turnaround), the raw ring takes the rest
  p.stages = getenv("PALU_LQ_STAGES") ? atoi(getenv("PALU_LQ_STAGES")) : 3;
  p.raw_slots = (limit - misc - p.stages * (OB + 16)) / (RB + 16);
  const int rmax = getenv("PALU_LQ_RAW") ? atoi(getenv("PALU_LQ_RAW")) : 12;
  if (p.raw_slots > rmax) p.raw_slots = rmax;
  PALU_REQUIRE(p.raw_slots >= 2, "palu_latent_score_tc (int8 pipe): shared memory too small (%d)", p.raw_slots);
  const size_t smem = (size_t)misc + (size_t)p.stages * (OB + 16) + (size_t)p.raw_slots * (RB + 16);
  static bool attr = false;
  if (!attr) {
    PALU_CK(cudaFuncSetAttribute(latent_score_q_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, limit));
    PALU_CK(cudaFuncSetAttribute(latent_score_q_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, limit));
    PALU_CK(cudaFuncSetAttribute(latent_score_q_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, limit));
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (bits == 2)
    PALU_CK(launch_k(latent_score_q_kernel<2>, dim3(sms), dim3(LQ_THREADS), smem, st, p));
  else if (bits == 4)
    PALU_CK(launch_k(latent_score_q_kernel<4>, dim3(sms), dim3(LQ_THREADS), smem, st, p));
  else
    PALU_CK(launch_k(latent_score_q_kernel<8>, dim3(sms), dim3(LQ_THREADS), smem, st, p));
  PALU_LAUNCHED();
  return PALU_OK;
}

int palu_latent_score_tc(int bits, const void* hk, const float* scales, const float* zps, int B,
                         int n_heads, int s, int G, int R_pad, int T_cap, const float* y, int ld_y,
                         const int* q_off, const int* ranks, float scale, const int* t_dev,
                         float* logits, int ld_logits, void* stream) {
  using namespace palu::tc;
  const int row_bytes = bits == 16 ? R_pad * 2 : R_pad * bits / 8;
  if (G * s != n_heads || s > 16 || R_pad % KB != 0 || R_pad > 256 ||
      (bits != 16 && bits != 2 && bits != 3 && bits != 4 && bits != 8) ||
      (bits != 16 && (row_bytes % 16 != 0 || !scales || !zps))) {
    set_error("palu_latent_score_tc: unsupported shape (bits %d, R_pad %d, s %d)", bits, R_pad, s);
    return PALU_EUNSUPPORTED;
  }
  PALU_REQUIRE(((uintptr_t)hk & 15) == 0, "palu_latent_score_tc: unaligned latents");
  static const bool lq_off = getenv("PALU_LS_KERNEL") && strcmp(getenv("PALU_LS_KERNEL"), "bf16") == 0;
  if ((bits == 2 || bits == 4 || bits == 8) && R_pad % 128 == 0 && T_cap % TILE_M == 0 && s <= 4 && !lq_off)
    return launch_latent_score_q(bits, hk, scales, zps, B, n_heads, s, G, R_pad, T_cap, y, ld_y, q_off,
                                 ranks, scale, t_dev, logits, ld_logits, (cudaStream_t)stream);
  CUtensorMap map_h = {};
  if (bits == 16) {
    int rc = make_map_2d(&map_h, hk, R_pad, (uint64_t)B * G * T_cap, KB, TILE_M);
    if (rc) return rc;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  LSParams prm;
  prm.B = B;
  prm.n_heads = n_heads;
  prm.s = s;
  prm.G = G;
  prm.R_pad = R_pad;
  prm.T_cap = T_cap;
  prm.ld_logits = ld_logits;
  prm.ld_y = ld_y;
  prm.scale = scale;
  prm.y = y;
  prm.q_off = q_off;
  prm.ranks = ranks;
  prm.t_dev = t_dev;
  prm.logits = logits;
  prm.bits = bits;
  prm.code_row_bytes = row_bytes;
  prm.codes = reinterpret_cast<const uint8_t*>(hk);
  prm.scales = scales;
  prm.zps = zps;
  const int QB = R_pad / KB * 2048;
  const int fixed = 1024 + 2 * QB + 1024 + 256;
  prm.stages = (SMEM_LIMIT - 2048 - fixed) / H_STAGE_BYTES;
  const int smax = getenv("PALU_LS_STAGES") ? atoi(getenv("PALU_LS_STAGES")) : 10;  // tuning only
  if (prm.stages > smax) prm.stages = smax;
  const size_t smem = (size_t)fixed + (size_t)prm.stages * H_STAGE_BYTES;
  static bool attr = false;
  if (!attr) {
    PALU_CK(cudaFuncSetAttribute(latent_score_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SMEM_LIMIT - 2048));
    attr = true;
  }
  PALU_CK(launch_k(latent_score_tc_kernel, dim3(sms), dim3(LS_THREADS), smem, (cudaStream_t)stream,
                   map_h, prm));
  return PALU_OK;
}

}  // extern "C"
