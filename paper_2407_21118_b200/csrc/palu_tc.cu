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

#include "palu_sm100.cuh"

namespace palu {
namespace tc {

constexpr int BASE_RING = 4;       // tile-base cos/sin rows in flight
constexpr int PF_DIST = 3;         // L2 prefetch distance (work items)
constexpr int BASE_BYTES = 64 * 8; // 64 float2
constexpr int SUPER = 2 * TILE_M;  // tokens per work item (the CTA pair)
constexpr int HEAD_BYTES = TILE_M * 128;  // one head's 128 UW rows x 64 bf16

struct VParams;  // value role of the fused kernel (below)

struct Params {
  int B, n_heads, s_k, G, R_pad, T_cap, ld_logits, n_tab, stages;
  int score_pairs;  // CTA pairs running the score role (fused kernel); all pairs otherwise
  int* ready;       // fused: per work item, epilogue warps that published its logits
  int mode;     // profiling only (bit flags): 1 epilogue skips math; 2 MMA skips TMA waits; 4 MMA skips TMEM-empty waits
  int pf_dist;  // L2 prefetch distance in work items (0 = off)
  const float2* rope_tab;  // [n_tab + 128][64]
  const int* t_dev;
  float* logits;
};

// Work item = (sequence b, key group g, 256-token super-tile) for a CTA pair
// (cluster of 2, cta_group::2).  SM r of the pair loads tokens
// [256 st + 128 r, +128) of H once and the UW rows of head 2h + r for each head
// pair h of the group; the leader SM issues
//   ACC_h[256 tokens x 256] += H[256 x 64] x UW_h[256 x 64]^T   (per k-block)
// whose rows 128 r .. land in SM r's TMEM.  Each SM's epilogue reduces its
// own 128 tokens x 2 heads per head pair.  Every latent byte crosses L2 -> SM
// once and both SMs' tensor pipes run at the 2-SM rate.
__device__ __forceinline__ void score_role(const CUtensorMap& map_h, const CUtensorMap& map_uw,
                                           const Params& p, uint8_t* smem) {
  const int kblocks = p.R_pad / KB;
  const int halves = p.s_k / 2;
  uint8_t* s_uw = smem;                                  // [kblocks][halves] x 16 KB
  uint8_t* s_h = smem + kblocks * halves * HEAD_BYTES;   // stages x 16 KB
  float2* s_base = reinterpret_cast<float2*>(s_h + p.stages * H_STAGE_BYTES);  // ring
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_base + BASE_RING * 64);
  uint64_t* full = bars;                                 // [stages]   (leader's used)
  uint64_t* empty = bars + p.stages;                     // [stages]   (each SM's own)
  uint64_t* tfull = bars + 2 * p.stages;                 // [2]        (each SM's own)
  uint64_t* tempty = tfull + 2;                          // [2]        (leader's used)
  uint64_t* uw_full = tempty + 2;                        // [1]        (leader's used)
  uint64_t* uw_empty = uw_full + 1;                      // [1]        (each SM's own)
  uint64_t* bfull = uw_empty + 1;                        // [BASE_RING] local
  uint64_t* bempty = bfull + BASE_RING;                  // [BASE_RING] local
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bempty + BASE_RING);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);  // [2 slots][2 heads][128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair_id = blockIdx.x >> 1, n_pairs = p.score_pairs;
  const int T_rows = *p.t_dev + 1;
  const int n_super = (T_rows + SUPER - 1) / SUPER;
  const int total = p.B * p.G * n_super;
  const int per = (total + n_pairs - 1) / n_pairs;
  const int i0 = min(total, pair_id * per);
  const int i1 = min(total, i0 + per);

  if (warp == 0 && lane == 0) {
    prefetch_map(&map_h);
    prefetch_map(&map_uw);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * EPI_WARPS);
    }
    for (int a = 0; a < BASE_RING; ++a) {
      mbar_init(&bfull[a], 1);
      mbar_init(&bempty[a], EPI_WARPS);
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

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both SMs) ----------------
      int cur = -1, nloads = 0, kc = 0, it = 0;
      for (int i = i0; i < i1; ++i, ++it) {
        const int bg = i / n_super, st = i - bg * n_super;
        if (bg != cur) {
          if (nloads > 0) mbar_wait(uw_empty, (nloads - 1) & 1);
          if (leader) mbar_expect_tx(uw_full, 2 * kblocks * halves * HEAD_BYTES);
          for (int kb = 0; kb < kblocks; ++kb)
            for (int h = 0; h < halves; ++h)
              tma_load_2d_pair(&map_uw, uw_full, s_uw + (kb * halves + h) * HEAD_BYTES, kb * KB,
                               (bg * p.s_k + 2 * h + (int)rank) * 128);
          ++nloads;
          cur = bg;
        }
        const int tile = 2 * st + (int)rank;  // this SM's 128-token tile
        const int bs = it % BASE_RING;
        mbar_wait(&bempty[bs], ((it / BASE_RING) & 1) ^ 1);
        mbar_expect_tx(&bfull[bs], BASE_BYTES);
        bulk_load(s_base + bs * 64, p.rope_tab + (size_t)tile * 64, BASE_BYTES, &bfull[bs]);
        const int h_row = bg * p.T_cap + tile * TILE_M;
        // warm L2 with this SM's rows of the item PF_DIST ahead: smem holds only
        // ~1.25 items next to the resident UW, so HBM latency must be hidden in L2
        if (p.pf_dist > 0 && i + p.pf_dist < i1) {
          const int ip = i + p.pf_dist;
          const int bgp = ip / n_super, stp = ip - bgp * n_super;
          const int rowp = bgp * p.T_cap + (2 * stp + (int)rank) * TILE_M;
          for (int kb = 0; kb < kblocks; ++kb) tma_prefetch_l2(&map_h, kb * KB, rowp);
        }
        for (int kb = 0; kb < kblocks; ++kb, ++kc) {
          const int stage = kc % p.stages;
          mbar_wait(&empty[stage], ((kc / p.stages) & 1) ^ 1);
          if (leader) mbar_expect_tx(&full[stage], 2 * H_STAGE_BYTES);
          tma_load_2d_pair(&map_h, &full[stage], s_h + stage * H_STAGE_BYTES, kb * KB, h_row);
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ---------------- MMA issuer (leader SM issues for the pair) ----------------
      const uint32_t uw_addr = smem_u32(s_uw);
      const uint32_t h_addr = smem_u32(s_h);
      int cur = -1, nloads = 0, kc = 0, unit = 0;
      for (int i = i0; i < i1; ++i) {
        const int bg = i / n_super;
        if (bg != cur) {
          if (nloads > 0) umma2_commit_both(uw_empty);  // frees UW in both SMs
          mbar_wait(uw_full, nloads & 1);
          fence_after();
          ++nloads;
          cur = bg;
        }
        for (int h = 0; h < halves; ++h, ++unit) {
          const int slot = unit & 1;
          if ((p.mode & 4) == 0) mbar_wait(&tempty[slot], ((unit >> 1) & 1) ^ 1);
          fence_after();
          const uint32_t d_tmem = tmem_base + slot * N_CTA;
          for (int kb = 0; kb < kblocks; ++kb) {
            const int cnt = kc + kb;
            const int stage = cnt % p.stages;
            if (h == 0 && (p.mode & 2) == 0) {
              mbar_wait(&full[stage], (cnt / p.stages) & 1);
              fence_after();
            }
            const uint32_t a0 = h_addr + stage * H_STAGE_BYTES;
            const uint32_t b0 = uw_addr + (kb * halves + h) * HEAD_BYTES;
#pragma unroll
            for (int kk = 0; kk < KB / 16; ++kk)
              umma2_bf16(d_tmem, sdesc(a0 + kk * 32), sdesc(b0 + kk * 32), (kb | kk) != 0);
            if (h == halves - 1) umma2_commit_both(&empty[stage]);
          }
          umma2_commit_both(&tfull[slot]);
        }
        kc += kblocks;
      }
    }
  } else {
    // ---------------- epilogue (both SMs): cos/sin-weighted row reduction ----------------
    const int q = warp & 3;          // TMEM lane quarter
    const int jh = (warp - 2) >> 2;  // which 32 of the 64 frequencies
    const int delta = q * 32 + lane; // token row inside this SM's tile
    float2 cd2[16], sd2[16];         // cos/sin(delta th_j) for j pairs (2i, 2i + 1)
    {
      const float4* off =
          reinterpret_cast<const float4*>(p.rope_tab + (size_t)(p.n_tab + delta) * 64 + jh * 32);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float4 v = off[i];
        cd2[i] = make_float2(v.x, v.z);
        sd2[i] = make_float2(v.y, v.w);
      }
    }
    const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
    int unit = 0, it = 0;
    for (int i = i0; i < i1; ++i, ++it) {
      const int bg = i / n_super, st = i - bg * n_super;
      const int b = bg / p.G, g = bg - b * p.G;
      const int tile = 2 * st + (int)rank;
      const int bs = it % BASE_RING;
      mbar_wait(&bfull[bs], (it / BASE_RING) & 1);
      // cos/sin((t0 + delta) th_j) = base (x) offset, for this thread's 32 frequencies
      float2 c2[16], s2[16];
      {
        const float4* base = reinterpret_cast<const float4*>(s_base + bs * 64 + jh * 32);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float4 bv = base[k];
          const float2 bc = make_float2(bv.x, bv.z), bsn = make_float2(bv.y, bv.w);
          const float2 t = fmul2(bsn, sd2[k]);
          c2[k] = ffma2(bc, cd2[k], make_float2(-t.x, -t.y));
          s2[k] = ffma2(bsn, cd2[k], fmul2(bc, sd2[k]));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bempty[bs]);
      for (int h = 0; h < halves; ++h, ++unit) {
        const int slot = unit & 1;
        mbar_wait(&tfull[slot], (unit >> 1) & 1);
        fence_after();
        float v[2] = {0.f, 0.f};
        if ((p.mode & 1) == 0)
#pragma unroll
        for (int hp = 0; hp < 2; ++hp) {
          float2 acc2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int jc = 0; jc < 2; ++jc) {
            float u[16], w[16];
            const uint32_t col = slot * N_CTA + hp * 128 + jh * 32 + jc * 16;
            tmem_ld16(lane_base + col, u);
            tmem_ld16(lane_base + col + 64, w);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              acc2 = ffma2(c2[jc * 8 + k], make_float2(u[2 * k], u[2 * k + 1]), acc2);
              acc2 = ffma2(s2[jc * 8 + k], make_float2(w[2 * k], w[2 * k + 1]), acc2);
            }
          }
          v[hp] = acc2.x + acc2.y;
        }
        float* r = red + slot * 2 * TILE_M;
        if (jh == 1) {
          r[delta] = v[0];
          r[TILE_M + delta] = v[1];
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_leader(&tempty[slot]);
          named_bar_arrive(1 + slot, EPI_WARPS * 32);
        } else {
          named_bar_sync(1 + slot, EPI_WARPS * 32);
          const float v0 = v[0] + r[delta], v1 = v[1] + r[TILE_M + delta];
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_leader(&tempty[slot]);
          const int t = tile * TILE_M + delta;
          if (t < T_rows) {
            // D columns 0..127 = head 2h (leader's UW rows), 128..255 = head 2h + 1
            const int head0 = g * p.s_k + 2 * h;
            float* lg = p.logits + ((size_t)b * p.n_heads + head0) * p.ld_logits + t;
            lg[0] = v0;
            lg[p.ld_logits] = v1;
          }
          if (p.ready != nullptr && h == halves - 1) {
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
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
rope_score_tc_kernel(const __grid_constant__ CUtensorMap map_h,
                     const __grid_constant__ CUtensorMap map_uw, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  score_role(map_h, map_uw, p, smem);
}

// ===========================================================================
// Fused score + softmax + value kernel (grid-level role split).
//
// The reconstruction is tensor-bound and the value stream is HBM-bound, so
// one persistent grid runs both concurrently on disjoint SMs: CTA pairs
// [0, score_pairs) run score_role and publish per-item readiness; the other
// CTAs run value_role: they walk the value chunks in the order the score
// pairs complete them, wait for their items, and stream the chunk's H_v rows
// through a deep TMA bulk-copy ring while computing the chunk softmax
// statistics and p . H_v partials; the last chunk of each (sequence, group)
// merges them in a fixed order (deterministic).  attention.py:433-446.
// ===========================================================================
struct VParams {
  const uint8_t* hv;  // [B][G][T_cap][Rv_pad] bf16
  int Rv_pad, vc;     // value row width; score items per value chunk
  int v_stages;       // TMA ring depth of the value role
  unsigned* tickets;  // [B*G]
  float *pm, *pl, *pctx;  // partials [B][n][NCmax] / [B][n][NCmax][Rv_pad]
  int nc_max;
  const int* ranks_v;
  const int* o_off;
  float* ctx_out;
  int ld_ctx;
};

constexpr int V_STAGE = 16384;
constexpr int V_HP = 4;

__device__ __forceinline__ uint32_t ld_acquire_u32(const int* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Completion-ordered list of this value CTA's chunks: chunk ends are score
// items L = pr * per + off visited offset-major, so the k-th chunk of the list
// becomes ready at about the k-th fraction of the score role's run.
struct VChunkIter {
  int per, total, pairs, n_super, vc, vcta, n_vctas;
  int off, pr, k;
  __device__ bool next(int& L) {
    for (; off < per; ++off, pr = 0) {
      for (; pr < pairs; ++pr) {
        const int cand = pr * per + off;
        if (cand >= total || cand >= (pr + 1) * per) continue;
        const int st = cand % n_super;
        if ((st + 1) % vc != 0 && st != n_super - 1) continue;
        if ((k++) % n_vctas != vcta) continue;
        L = cand;
        ++pr;
        return true;
      }
    }
    return false;
  }
};

template <int NSEG>
__device__ void value_role(const Params& p, const VParams& vp, uint8_t* smem, int vcta,
                           int n_vctas) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int T_rows = *p.t_dev + 1;
  const int n_super = (T_rows + SUPER - 1) / SUPER;
  const int total = p.B * p.G * n_super;
  const int per = (total + p.score_pairs - 1) / p.score_pairs;
  const int n_vc = (n_super + vp.vc - 1) / vp.vc;  // value chunks per (b, g)
  const int s_v = p.s_k;
  const int row_bytes = vp.Rv_pad * 2;
  const int segs = row_bytes / 16;
  const int stage_rows = V_STAGE / row_bytes;
  const int max_tok = vp.vc * SUPER;
  // smem: ring | red [8][V_HP][Rv_pad] | ps [V_HP][max_tok] | wsm [V_HP][n_vc] | barriers
  uint8_t* ring = smem;
  float* red = reinterpret_cast<float*>(ring + vp.v_stages * V_STAGE);
  float* ps = red + 8 * V_HP * vp.Rv_pad;
  float* wsm = ps + V_HP * max_tok;
  uint64_t* full = reinterpret_cast<uint64_t*>(wsm + V_HP * vp.nc_max);
  uint64_t* empty = full + vp.v_stages;
  __shared__ float red_m[8][V_HP], red_l[8][V_HP], m_sh[V_HP], inv_l[V_HP];
  __shared__ unsigned ticket_sh;

  if (tid == 0) {
    for (int st = 0; st < vp.v_stages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  VChunkIter iter{per, total, p.score_pairs, n_super, vp.vc, vcta, n_vctas, 0, 0, 0};

  if (warp == 8) {
    // ---------------- producer: H_v rows do not depend on the score role, so
    // stream every chunk of the list back to back (bounded by the ring)
    if (lane == 0) {
      int L, ctr = 0;
      while (iter.next(L)) {
        const int bg = L / n_super, st_last = L % n_super, c = st_last / vp.vc;
        const int c0 = c * vp.vc * SUPER, c1 = min(T_rows, (st_last + 1) * SUPER);
        const uint8_t* src0 = vp.hv + ((size_t)bg * p.T_cap + c0) * row_bytes;
        const int n_loads = (c1 - c0 + stage_rows - 1) / stage_rows;
        for (int pass = 0; pass < s_v; pass += V_HP) {
          for (int l = 0; l < n_loads; ++l, ++ctr) {
            const int st = ctr % vp.v_stages;
            mbar_wait(&empty[st], ((ctr / vp.v_stages) & 1) ^ 1);
            const int nr = min(stage_rows, (c1 - c0) - l * stage_rows);
            mbar_expect_tx(&full[st], (uint32_t)(nr * row_bytes));
            bulk_load(ring + st * V_STAGE, src0 + (size_t)l * stage_rows * row_bytes,
                      (uint32_t)(nr * row_bytes), &full[st]);
          }
        }
      }
    }
    return;
  }
  if (warp > 8) return;
  // ---------------- consumers (warps 0..7) ----------------
  int L, ctr = 0;
  while (iter.next(L)) {
    const int bg = L / n_super, b = bg / p.G, g = bg - b * p.G;
    const int st_last = L % n_super, c = st_last / vp.vc;
    const int item0 = bg * n_super + c * vp.vc;
    const int c0 = c * vp.vc * SUPER, c1 = min(T_rows, (st_last + 1) * SUPER);
    const int n_loads = (c1 - c0 + stage_rows - 1) / stage_rows;
    if (tid == 0) {
      for (int it = item0; it <= L; ++it)
        while (ld_acquire_u32(&p.ready[it]) < 2u * (EPI_WARPS / 2)) __nanosleep(128);
    }
    named_bar_sync(1, 256);
    for (int p0 = 0; p0 < s_v; p0 += V_HP) {
      const int hp = min(V_HP, s_v - p0);
      // (1) chunk softmax statistics (logits via L2: written by the score role)
      const float* lg[V_HP];
#pragma unroll
      for (int h = 0; h < V_HP; ++h)
        lg[h] = p.logits + ((size_t)b * p.n_heads + g * s_v + p0 + min(h, hp - 1)) * p.ld_logits;
      float m[V_HP];
#pragma unroll
      for (int h = 0; h < V_HP; ++h) m[h] = -INFINITY;
      for (int t0 = c0 + tid; t0 < c1; t0 += 4 * 256) {
        float v[4][V_HP];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int h = 0; h < V_HP; ++h)
            v[u][h] = (t0 + u * 256 < c1) ? __ldcg(lg[h] + t0 + u * 256) : -INFINITY;
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int h = 0; h < V_HP; ++h) {
            if (t0 + u * 256 < c1) ps[h * max_tok + (t0 + u * 256 - c0)] = v[u][h];
            m[h] = fmaxf(m[h], v[u][h]);
          }
      }
#pragma unroll
      for (int h = 0; h < V_HP; ++h) {
        m[h] = warp_reduce(m[h], [](float x, float y) { return fmaxf(x, y); });
        if (lane == 0) red_m[warp][h] = m[h];
      }
      named_bar_sync(1, 256);
      if (tid < V_HP) {
        float mm = red_m[0][tid];
        for (int w = 1; w < 8; ++w) mm = fmaxf(mm, red_m[w][tid]);
        m_sh[tid] = mm;
      }
      named_bar_sync(1, 256);
      float l[V_HP];
#pragma unroll
      for (int h = 0; h < V_HP; ++h) {
        m[h] = m_sh[h];
        l[h] = 0.f;
      }
      for (int t = c0 + tid; t < c1; t += 256) {
#pragma unroll
        for (int h = 0; h < V_HP; ++h) {
          const float e = __expf(ps[h * max_tok + (t - c0)] - m[h]);
          ps[h * max_tok + (t - c0)] = e;
          l[h] += e;
        }
      }
#pragma unroll
      for (int h = 0; h < V_HP; ++h) {
        l[h] = warp_reduce(l[h], [](float x, float y) { return x + y; });
        if (lane == 0) red_l[warp][h] = l[h];
      }
      named_bar_sync(1, 256);
      if (tid < hp) {
        float ll = 0.f;
        for (int w = 0; w < 8; ++w) ll += red_l[w][tid];
        const size_t pi = ((size_t)b * p.n_heads + g * s_v + p0 + tid) * vp.nc_max + c;
        vp.pm[pi] = m_sh[tid];
        vp.pl[pi] = ll;
      }
      // (2) reduce the staged rows: one row per warp step, lanes over 16-B segments
      float2 acc[V_HP][NSEG][4];
#pragma unroll
      for (int h = 0; h < V_HP; ++h)
#pragma unroll
        for (int q2 = 0; q2 < NSEG; ++q2)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[h][q2][e] = make_float2(0.f, 0.f);
      for (int l2 = 0; l2 < n_loads; ++l2, ++ctr) {
        const int st = ctr % vp.v_stages;
        mbar_wait(&full[st], (ctr / vp.v_stages) & 1);
        const int r0 = l2 * stage_rows;
        const int nr = min(stage_rows, (c1 - c0) - r0);
        const uint8_t* sbase = ring + st * V_STAGE;
        const float* pst = ps + r0;
        for (int r = warp; r < nr; r += 8) {
          const uint8_t* row = sbase + (size_t)r * row_bytes;
          float pv[V_HP];
#pragma unroll
          for (int h = 0; h < V_HP; ++h) pv[h] = pst[h * max_tok + r];
#pragma unroll
          for (int q2 = 0; q2 < NSEG; ++q2) {
            const int sg = lane + q2 * 32;
            if (NSEG == 1 || sg < segs) {
              const uint4 v = *reinterpret_cast<const uint4*>(row + sg * 16);
              float f[8];
              Vec16<bf16>::unpack(v, f);
#pragma unroll
              for (int h = 0; h < V_HP; ++h) {
                const float2 p2 = make_float2(pv[h], pv[h]);
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  acc[h][q2][e] = ffma2(p2, make_float2(f[2 * e], f[2 * e + 1]), acc[h][q2][e]);
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
      // (3) cross-warp reduction -> chunk partial
#pragma unroll
      for (int h = 0; h < V_HP; ++h)
#pragma unroll
        for (int q2 = 0; q2 < NSEG; ++q2) {
          const int sg = lane + q2 * 32;
          if (sg < segs)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              red[((size_t)warp * V_HP + h) * vp.Rv_pad + sg * 8 + 2 * e] = acc[h][q2][e].x;
              red[((size_t)warp * V_HP + h) * vp.Rv_pad + sg * 8 + 2 * e + 1] = acc[h][q2][e].y;
            }
        }
      named_bar_sync(1, 256);
      for (int idx = tid; idx < hp * vp.Rv_pad; idx += 256) {
        const int h = idx / vp.Rv_pad, col = idx - h * vp.Rv_pad;
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) v += red[((size_t)w * V_HP + h) * vp.Rv_pad + col];
        vp.pctx[(((size_t)b * p.n_heads + g * s_v + p0 + h) * vp.nc_max + c) * vp.Rv_pad + col] = v;
      }
      named_bar_sync(1, 256);
    }
    // ---- consume readiness (reset for the next launch) and merge if last
    if (tid == 0)
      for (int it = item0; it <= L; ++it) p.ready[it] = 0;
    __threadfence();
    named_bar_sync(1, 256);
    if (tid == 0) ticket_sh = atomicAdd(&vp.tickets[bg], 1u);
    named_bar_sync(1, 256);
    if (ticket_sh != (unsigned)(n_vc - 1)) continue;
    __threadfence();
    const int r = vp.ranks_v[g];
    for (int p0 = 0; p0 < s_v; p0 += V_HP) {
      const int hp = min(V_HP, s_v - p0);
      if (warp < hp) {
        const size_t base = ((size_t)b * p.n_heads + g * s_v + p0 + warp) * vp.nc_max;
        float M = -INFINITY;
        for (int cc = lane; cc < n_vc; cc += 32) M = fmaxf(M, __ldcg(vp.pm + base + cc));
        M = warp_reduce(M, [](float x, float y) { return fmaxf(x, y); });
        float Ls = 0.f;
        for (int cc = lane; cc < n_vc; cc += 32) {
          const float w = __expf(__ldcg(vp.pm + base + cc) - M);
          wsm[warp * vp.nc_max + cc] = w;
          Ls += w * __ldcg(vp.pl + base + cc);
        }
        Ls = warp_reduce(Ls, [](float x, float y) { return x + y; });
        if (lane == 0) inv_l[warp] = 1.f / Ls;
      }
      named_bar_sync(1, 256);
      // chunk-parallel: warp w sums chunks w, w + 8, ...; lanes over columns
      for (int h = 0; h < hp; ++h) {
        const float* src =
            vp.pctx + ((size_t)b * p.n_heads + g * s_v + p0 + h) * vp.nc_max * (size_t)vp.Rv_pad;
        for (int col0 = 0; col0 < r; col0 += 128) {
          float a4[4] = {0.f, 0.f, 0.f, 0.f};
          for (int cc = warp; cc < n_vc; cc += 8) {
            const float w = wsm[h * vp.nc_max + cc];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int col = col0 + lane + 32 * q;
              if (col < r) a4[q] = fmaf(w, __ldcg(src + (size_t)cc * vp.Rv_pad + col), a4[q]);
            }
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int col = col0 + lane + 32 * q;
            if (col < r) red[((size_t)warp * V_HP + h) * vp.Rv_pad + col] = a4[q];
          }
        }
      }
      named_bar_sync(1, 256);
      for (int idx = tid; idx < hp * r; idx += 256) {
        const int h = idx / r, col = idx - h * r;
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) v += red[((size_t)w * V_HP + h) * vp.Rv_pad + col];
        vp.ctx_out[(size_t)b * vp.ld_ctx + vp.o_off[g * s_v + p0 + h] + col] = v * inv_l[h];
      }
      named_bar_sync(1, 256);
    }
    if (tid == 0) vp.tickets[bg] = 0u;
  }
}

template <int NSEG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
rope_attend_tc_kernel(const __grid_constant__ CUtensorMap map_h,
                      const __grid_constant__ CUtensorMap map_uw, const Params p,
                      const VParams vp) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  if ((int)(blockIdx.x >> 1) < p.score_pairs) {
    score_role(map_h, map_uw, p, smem);
  } else {
    const int vcta = (int)blockIdx.x - 2 * p.score_pairs;
    value_role<NSEG>(p, vp, smem, vcta, (int)gridDim.x - 2 * p.score_pairs);
  }
}

// ---------------------------------------------------------------------------
// tile bases: cos/sin(t0 * th_j), t0 = 128 * row (fp64 angle reduction);
// offsets: cos/sin(delta * th_j), delta in [0, 128).
__global__ void rope_table_kernel(const double* __restrict__ theta, int half, int n_tiles,
                                  float2* __restrict__ tab) {
  const int total = (n_tiles + 128) * half;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int row = i / half, j = i - row * half;
    const double pos = row < n_tiles ? 128.0 * row : (double)(row - n_tiles);
    double sn, cs;
    sincos_big(pos * theta[j], &sn, &cs);
    tab[i] = make_float2((float)cs, (float)sn);
  }
}

// ---- host: tensor maps through the driver entry point (no -lcuda needed) ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
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
  tc::rope_table_kernel<<<256, 256, 0, (cudaStream_t)stream>>>(theta, half, n_tiles,
                                                               reinterpret_cast<float2*>(rope_tab));
  PALU_LAUNCHED();
  return PALU_OK;
}

int palu_rope_score_tc_splits(int s_k, int R_pad) {
  using namespace palu::tc;
  // one rank slice: the 2-SM pair keeps the whole UW operand resident
  return ((s_k == 2 || s_k == 4) && R_pad % KB == 0 && R_pad <= 256) ? 1 : 0;
}

int palu_rope_score_tc(int bits, const void* hk, const float* scales, const float* zps, int B,
                       int n_heads, int s_k, int G, int R_pad, int T_cap, const void* uw,
                       const float* rope_tab, const int* t_dev, float* logits, int ld_logits,
                       size_t plane_stride, void* stream) {
  using namespace palu::tc;
  (void)scales;
  (void)zps;
  (void)plane_stride;
  if (bits != 16) {
    set_error("palu_rope_score_tc: bits %d not on the tensor-core path yet", bits);
    return PALU_EUNSUPPORTED;
  }
  if (!palu_rope_score_tc_splits(s_k, R_pad) || G * s_k != n_heads) {
    set_error("palu_rope_score_tc: unsupported shape (R_pad %d, s_k %d)", R_pad, s_k);
    return PALU_EUNSUPPORTED;
  }
  PALU_REQUIRE(((uintptr_t)hk & 15) == 0 && ((uintptr_t)uw & 15) == 0, "tc: unaligned operands");
  CUtensorMap map_h, map_uw;
  int rc = make_map_2d(&map_h, hk, R_pad, (uint64_t)B * G * T_cap, KB, TILE_M);
  if (rc) return rc;
  rc = make_map_2d(&map_uw, uw, R_pad, (uint64_t)B * G * s_k * 128, KB, TILE_M);
  if (rc) return rc;
  const int kblocks = R_pad / KB;
  const int fixed = 1024 + kblocks * (s_k / 2) * HEAD_BYTES + BASE_RING * BASE_BYTES + 1024 +
                    2 * 2 * TILE_M * 4;
  int stages = (SMEM_LIMIT - fixed) / H_STAGE_BYTES;
  if (stages > 12) stages = 12;
  PALU_REQUIRE(stages >= kblocks, "tc: not enough shared memory (%d stages)", stages);
  const size_t smem = (size_t)fixed + (size_t)stages * H_STAGE_BYTES;
  static bool attr = false;
  if (!attr) {
    PALU_CK(cudaFuncSetAttribute(rope_score_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SMEM_LIMIT));
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  Params prm;
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
  prm.mode = getenv("PALU_TC_PROFILE_MODE") ? atoi(getenv("PALU_TC_PROFILE_MODE")) : 0;
  prm.pf_dist = getenv("PALU_TC_PF") ? atoi(getenv("PALU_TC_PF")) : PF_DIST;
  prm.rope_tab = reinterpret_cast<const float2*>(rope_tab);
  prm.t_dev = t_dev;
  prm.logits = logits;
  rope_score_tc_kernel<<<dim3(sms & ~1), THREADS, smem, (cudaStream_t)stream>>>(map_h, map_uw, prm);
  PALU_LAUNCHED();
  return PALU_OK;
}

// ---- fused score + softmax + value ------------------------------------------
static int fused_nc_max(int T_cap, int vc) {
  using palu::tc::SUPER;
  const int n_super = (T_cap + SUPER - 1) / SUPER;
  return (n_super + vc - 1) / vc;
}

size_t palu_rope_attend_workspace(int B, int n_heads, int G, int Rv_pad, int T_cap) {
  using palu::tc::SUPER;
  const int vc = 4;
  const int nc = fused_nc_max(T_cap, vc);
  const size_t items = (size_t)B * G * ((T_cap + SUPER - 1) / SUPER);
  const size_t head = (size_t)B * n_heads * nc;
  return 256 + sizeof(unsigned) * (size_t)B * G + sizeof(int) * items + sizeof(float) * head * 2 +
         sizeof(float) * head * (size_t)Rv_pad + 1024;
}

int palu_rope_attend_tc(const void* hk, const void* hv, int B, int n_heads, int s, int G,
                        int Rk_pad, int Rv_pad, int T_cap, const void* uw, const float* rope_tab,
                        const int* t_dev, float* logits, int ld_logits, const int* ranks_v,
                        const int* o_off, float* ctx, int ld_ctx, void* workspace,
                        int score_sms, void* stream) {
  using namespace palu::tc;
  if (!palu_rope_score_tc_splits(s, Rk_pad) || G * s != n_heads || (Rv_pad * 2) % 16 != 0 ||
      Rv_pad > 512) {
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
  const int fixed = 1024 + kblocks * (s / 2) * HEAD_BYTES + BASE_RING * BASE_BYTES + 1024 +
                    2 * 2 * TILE_M * 4;
  const int dyn_limit = SMEM_LIMIT - 2048;  // the value role has ~1 KB of static smem
  int stages = (dyn_limit - fixed) / H_STAGE_BYTES;
  if (stages > 12) stages = 12;
  PALU_REQUIRE(stages >= kblocks, "tc: not enough shared memory (%d stages)", stages);
  const size_t smem = (size_t)fixed + (size_t)stages * H_STAGE_BYTES;
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
  const int vc = 4;
  const int nc_max = fused_nc_max(T_cap, vc);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  unsigned* tickets = reinterpret_cast<unsigned*>(ws + 256);
  int* ready = reinterpret_cast<int*>(tickets + (size_t)B * G);
  const size_t items = (size_t)B * G * ((T_cap + SUPER - 1) / SUPER);
  float* pm = reinterpret_cast<float*>(ready + items);
  float* pl = pm + (size_t)B * n_heads * nc_max;
  float* pctx = pl + (size_t)B * n_heads * nc_max;
  Params prm;
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
  VParams vp;
  vp.hv = reinterpret_cast<const uint8_t*>(hv);
  vp.Rv_pad = Rv_pad;
  vp.vc = vc;
  const size_t side = sizeof(float) * ((size_t)8 * V_HP * Rv_pad + (size_t)V_HP * vc * SUPER +
                                       (size_t)V_HP * nc_max) + 64 * 16 + 1024;
  vp.v_stages = (int)(((long long)smem - 1024 - (long long)side) / V_STAGE);
  PALU_REQUIRE(vp.v_stages >= 3, "palu_rope_attend_tc: value ring too small (%d)", vp.v_stages);
  if (vp.v_stages > 32) vp.v_stages = 32;
  vp.tickets = tickets;
  vp.pm = pm;
  vp.pl = pl;
  vp.pctx = pctx;
  vp.nc_max = nc_max;
  vp.ranks_v = ranks_v;
  vp.o_off = o_off;
  vp.ctx_out = ctx;
  vp.ld_ctx = ld_ctx;
  const int nseg = (Rv_pad * 2 / 16 + 31) / 32;
  static bool attr1 = false, attr2 = false;
  if (nseg == 1) {
    if (!attr1) {
      PALU_CK(cudaFuncSetAttribute(rope_attend_tc_kernel<1>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_limit));
      attr1 = true;
    }
    rope_attend_tc_kernel<1><<<dim3(sms), THREADS, smem, (cudaStream_t)stream>>>(map_h, map_uw,
                                                                                 prm, vp);
  } else {
    if (!attr2) {
      PALU_CK(cudaFuncSetAttribute(rope_attend_tc_kernel<2>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_limit));
      attr2 = true;
    }
    rope_attend_tc_kernel<2><<<dim3(sms), THREADS, smem, (cudaStream_t)stream>>>(map_h, map_uw,
                                                                                 prm, vp);
  }
  PALU_LAUNCHED();
  return PALU_OK;
}

}  // extern "C"
