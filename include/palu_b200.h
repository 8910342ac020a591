/*
 * palu_b200.h -- C ABI of the B200-native Palu latent-KV RoPE decode path.
 *
 * The reference (Palu, pkg/src/palu) has no FFI: its boundary is the Python
 * API of palu.attention (attention.py:392-448 palu_decode_step_rope and the
 * functions it calls).  Each entry point below replaces one numpy stage of
 * that function; the Python host mirror (paper_2407_21118_b200/attention.py)
 * binds them with ctypes exactly as INTEGRATION.md shows.
 *
 * Conventions
 *   - plain pointers and sizes only; all pointers are DEVICE pointers unless
 *     named *_host; memory is owned by the caller (torch on the Python side);
 *   - every call is stream-ordered on `stream` (a cudaStream_t, may be NULL);
 *   - the decode position lives on the device (`t_dev`: rows cached BEFORE
 *     this step) so a whole step can be captured once in a CUDA graph;
 *   - return 0 on success, negative PALU_E* codes otherwise (the host shim
 *     maps PALU_EVALIDATION to palu.errors.ValidationError); no C++
 *     exceptions cross this boundary.
 *
 * Cache layout in HBM (one layer):
 *   latent rows  [B][G][T_cap][row]   row = R_pad elements of the storage
 *                                     dtype (bits==16) or R_pad*bits/8 bytes
 *                                     of little-endian packed codes (bits<16,
 *                                     quant.py:156-169 order inside a row)
 *   scales       [B][G][T_cap] float  (quantised sides only)
 *   zero points  [B][G][T_cap] float  (quantised sides only; integral values,
 *                                     exact below 2^24; exact fp64 scales and
 *                                     int64 zero points go to optional export
 *                                     arrays so quantized_latent() stays
 *                                     bit-exact)
 * Columns >= rank(g) are zero (raw) / code 0 (quantised) and meet zero rows
 * of the padded factors, so they never contribute.
 */
#ifndef PALU_B200_H
#define PALU_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PALU_OK 0
#define PALU_EVALIDATION (-1)
#define PALU_ECUDA (-2)
#define PALU_EUNSUPPORTED (-3)

#define PALU_DTYPE_F32 0
#define PALU_DTYPE_BF16 1

/* Library identity and the device check (fails on anything but sm_100). */
const char* palu_version(void);
int palu_device_check(int device);
const char* palu_last_error(void);

/*
 * y[b][n] (+)= sum_k W[n][k] * x[b][k]   W row-major N x K in `dtype`.
 * Replaces the numpy projections of the step: x @ W_q[:, head]
 * (attention.py:430), x @ A_g (attention.py:343-347, _append_latents) and
 * ctx @ wo_fused (attention.py:361, _value_output).
 */
int palu_gemv(int dtype, const void* W, int N, int K, const float* x, int B, int ldx,
              float* y, int ldy, int accumulate, void* stream);

/*
 * Append row t (= *t_dev) of every group's latent store from fp32 latents
 * lat[b][lat_off[g] + c], c < ranks[g] (ranks/lat_off: device int arrays).
 * bits==16 stores raw `dtype` values (attention.py:249-251); bits in
 * {2,3,4,8} quantises per token in fp64 with quant.py:87-99's operation
 * order (round half away from zero, range floor 1e-8) and packs the codes.
 * Replaces _GroupStore.append (attention.py:248-255).
 */
int palu_latent_append(int dtype, int bits, const float* lat, int B, int ld_lat, int G,
                       const int* ranks, const int* lat_off, void* rows, float* scales,
                       float* zps, double* scales64, int64_t* zps64, int R_pad, int T_cap,
                       const int* t_dev, void* stream);

/*
 * Both sides of one layer's append (palu_latent_append for keys and values)
 * in one launch: lat_k / lat_v point at each side's latents inside the same
 * GEMV output row (row stride ld_lat); quantised sides share one dynamic
 * shared-memory size.  Same results as two palu_latent_append calls.
 */
int palu_latent_append_kv(int dtype, int bits_k, int bits_v, const float* lat_k, const float* lat_v,
                          int B, int ld_lat, int G_k, int G_v, const int* ranks_k,
                          const int* lat_off_k, const int* ranks_v, const int* lat_off_v,
                          void* rows_k, float* scales_k, float* zps_k, double* scales64_k,
                          int64_t* zps64_k, void* rows_v, float* scales_v, float* zps_v,
                          double* scales64_v, int64_t* zps64_v, int R_pad_k, int R_pad_v,
                          int T_cap, const int* t_dev, void* stream);

/*
 * Container export of one group's quantised latents (pipeline.py:513-531):
 * pack_codes (quant.py:156-169) of the first `rank` codes of T stored rows
 * (row_bytes apart, as palu_latent_append writes them) into one LSB-first
 * bitstream of out_bytes = ceil(T * rank * bits / 8) bytes.
 */
int palu_pack_code_stream(int bits, const void* rows, int row_bytes, int rank, int T, void* out,
                          long long out_bytes, void* stream);

/*
 * Bit-exact per-token quantiser on fp64 rows (quant.py:87-99): codes (uint8,
 * one per element), scales (fp64) and zero points (int64).  The cache uses
 * the same device function; this entry point exposes it for parity tests.
 */
int palu_quantize_rows(const double* x, int rows, int cols, int bits, uint8_t* codes,
                       double* scales, int64_t* zps, void* stream);

/* LE bit-packing of `rows` x `cols` codes, one byte-aligned packed row each
 * (quant.py:156-169 order); cols*bits must be a multiple of 8. */
int palu_pack_rows(const uint8_t* codes, int rows, int cols, int bits, uint8_t* packed,
                   void* stream);

/*
 * Query absorption for the RoPE score (attention.py:428-444 restated):
 *   q_rot = RoPE(q, t) per head with fp64 angles, then per head p of key
 *   group g and pair j < d_h/2:
 *     u_j = scale * (q_rot[j]   * B_g[:, p*d_h+j] + q_rot[j+h] * B_g[:, p*d_h+j+h])
 *     w_j = scale * (q_rot[j+h] * B_g[:, p*d_h+j] - q_rot[j]   * B_g[:, p*d_h+j+h])
 *   so that  q_rot . RoPE_t'(h B_g[:, head]) = sum_j cos(t' th_j) h.u_j + sin(t' th_j) h.w_j.
 * bk: [G][bk_rows][s_k*d_h] in `dtype` (rows >= rank zero, bk_rows >= R_pad).
 * layout 0: uw fp32 [B][n][R_pad][d_h]  (cols j < h: u_j, j >= h: w_{j-h})
 * layout 1: uw bf16 [B][G][s_k*d_h][R_pad] (K-major rows, tcgen05 B operand)
 * layout 4: uw float [B][n][d_h] = scale x RoPE_t(q) only (replicated-B groups,
 *           palu_rope_score_tc_rep)
 * layouts 2/3: as 1 with the rank order permuted for int4 / int2 keys on the
 *   tcgen05 path (groups of 8 / 16: rank k at position k < G/2 ? 2k : 2k-G+1)
 */
int palu_query_absorb(int dtype, const float* q, int B, int ld_q, int n_heads, int head_dim,
                      int s_k, const void* bk, int bk_rows, int R_pad, const double* theta,
                      float scale, const int* t_dev, void* uw, int layout, void* stream);

/*
 * palu_latent_append_kv and palu_query_absorb of one layer in ONE launch
 * (attention.py:343-347 + :248-255, and :428-431): both read only the GEMV
 * output row and *t_dev, and the RoPE score needs both, so a single grid
 * takes the append off the serial launch chain.  Arguments are those of the
 * two calls (the absorb's R_pad is R_pad_k); results are identical.
 */
int palu_append_absorb(int dtype, int bits_k, int bits_v, const float* lat_k, const float* lat_v, int B,
                       int ld_lat, int G_k, int G_v, const int* ranks_k, const int* lat_off_k,
                       const int* ranks_v, const int* lat_off_v, void* rows_k, float* scales_k,
                       float* zps_k, double* scales64_k, int64_t* zps64_k, void* rows_v, float* scales_v,
                       float* zps_v, double* scales64_v, int64_t* zps64_v, int R_pad_k, int R_pad_v,
                       int T_cap, const float* q, int ld_q, int n_heads, int head_dim, int s_k,
                       const void* bk, int bk_rows, const double* theta, float scale, void* uw, int layout,
                       const int* t_dev, void* stream);

/*
 * RoPE score over the latent key cache (attention.py:433-444):
 *   logits[b][i][t'] = q_rot_i . RoPE_t'( H_k[g(i)][t'] @ B_g[:, head i] ) / sqrt(d_h)
 * for t' in [0, *t_dev], via the absorbed uw (layout 0).  bits 16 reads raw
 * rows; bits < 16 dequantises (code - z) * s on load (attention.py:265-268).
 * logits: [B][n][ld_logits] fp32.
 */
int palu_rope_score(int dtype, int bits, const void* hk, const float* scales, const float* zps,
                    int B, int n_heads, int head_dim, int s_k, int G, int R_pad, int T_cap,
                    const void* uw, const double* theta, const int* t_dev, float* logits,
                    int ld_logits, void* stream);

/*
 * tcgen05 (sm_100a) RoPE score kernel (attention.py:433-444): same math as
 * palu_rope_score with uw in layout 1 (bf16 [B][G][s_k*128][R_pad]); logits
 * [B][n][ld_logits].  Requires d_h 128, s_k in {2, 4}, R_pad a multiple of 64
 * and <= 256 (palu_rope_score_tc_splits != 0); PALU_EUNSUPPORTED otherwise.
 * bits 16: hk is bf16 [B][G][T_cap][R_pad].  bits 2/3/4/8: hk holds the
 * packed codes [B][G][T_cap][R_pad*bits/8] (quant.py:156-169 order) with fp32
 * scales / zero points [B][G][T_cap]; converter warps unpack the codes into
 * the bf16 MMA operand as code - z (exact for |z| <= 128, else one bf16
 * rounding) and the epilogue multiplies by the scale (quant.py:106-107).
 * uw must use palu_query_absorb layout 2 (int4) / 3 (int2) / 1 (others).
 */
int palu_rope_score_tc_splits(int s_k, int R_pad);
int palu_rope_score_tc(int bits, const void* hk, const float* scales, const float* zps, int B,
                       int n_heads, int s_k, int G, int R_pad, int T_cap, const void* uw,
                       const float* rope_tab, const int* t_dev, float* logits, int ld_logits,
                       void* stream);
/*
 * palu_rope_score_tc that also brings l2_prefetch[0, l2_prefetch_bytes) into
 * L2 with an evict-last policy while it runs (the tensor-bound score leaves
 * HBM bandwidth idle): the host passes the layer's wo_fused^T, which the
 * output GEMV then reads from L2.  The latent streams load evict-first.
 */
int palu_rope_score_tc_pf(int bits, const void* hk, const float* scales, const float* zps, int B,
                          int n_heads, int s_k, int G, int R_pad, int T_cap, const void* uw,
                          const float* rope_tab, const int* t_dev, float* logits, int ld_logits,
                          const void* l2_prefetch, long long l2_prefetch_bytes, void* stream);
/*
 * Replicated-B groups (GQA as its MHA-equivalent layer: the s = n_heads / G
 * query heads of a group share one KV head's B_k columns):
 * reconstruct K = H B once per KV head on the tensor pipe, RoPE each key pair
 * in the epilogue and dot it with the group's rotated queries -- the same
 * logits as palu_rope_score_tc with 1/s of the accumulator traffic.
 * bkt: bf16 [B][G][128][R_pad], row c = column c of the group's KV-head B_k
 * (rank order as the cache); qrot: float [B][n_heads][128] = scale x
 * RoPE_t(q) (palu_append_absorb layout 4).  Raw bf16 keys, head_dim 128,
 * n_heads / G == 4, R_pad % 64 == 0 and <= 256.  Replaces the per-head
 * reconstruction of attention.py:433-444 for such groups.
 */
int palu_rope_score_tc_rep(const void* hk, int B, int n_heads, int G, int R_pad, int T_cap, const void* bkt,
                           const float* qrot, const float* rope_tab, const int* t_dev, float* logits,
                           int ld_logits, void* stream);

/*
 * Fused RoPE score + softmax + value path (attention.py:433-446, 350-362 up
 * to wo_fused): one persistent grid whose CTA pairs [0, score_sms/2) run the
 * tcgen05 score pipeline of palu_rope_score_tc and publish per-tile
 * readiness, while the remaining CTAs stream H_v (bf16 [B][G][T_cap][Rv_pad],
 * Rv_pad % 64 == 0, <= 512) as swizzled 2-D TMA boxes and reduce it on
 * tcgen05 (D[128 cols x 16] += H_v^T x P^T, P = hi + lo bf16 probabilities
 * written by CUDA cores), merging per-unit partials in a fixed order.
 * Output as palu_softmax_value (ctx[b][o_off[i] + c]); logits is scratch.  K
 * and V must share the group size s (<= 4).  score_sms <= 0 picks the split
 * from a per-SM throughput model.  workspace: palu_rope_attend_workspace()
 * bytes, zero-initialised once (all counters reset themselves).  Selected
 * only with score_kernel="fused" (the unfused tcgen05 path is faster on
 * B200 at the bench shapes).
 */
size_t palu_rope_attend_workspace(int B, int n_heads, int G, int Rv_pad, int T_cap);
int palu_rope_attend_tc(const void* hk, const void* hv, int B, int n_heads, int s, int G,
                        int Rk_pad, int Rv_pad, int T_cap, const void* uw, const float* rope_tab,
                        const int* t_dev, float* logits, int ld_logits, const int* ranks_v,
                        const int* o_off, float* ctx, int ld_ctx, void* workspace,
                        int score_sms, void* stream);

/*
 * Softmax + value on tcgen05 (attention.py:445-446, _value_output :350-362 up
 * to wo_fused) after palu_rope_score_tc.  bits 16: bf16 latents; bits
 * 2/3/4/8: packed codes (Rv_pad % 128 == 0) with fp32 scales / zero points,
 * unpacked as c - z by converter warps, the scale folded into P (quant.py:
 * 106-107).  Every SM streams
 * its share of H_v units ([B][G][T_cap][Rv_pad], Rv_pad % 64 == 0, <= 512,
 * s <= 4) as swizzled 2-D TMA boxes and reduces D[128 cols x 16] += H_v^T x
 * P^T with P = hi + lo bf16 probabilities; per-unit partials are merged in a
 * fixed order by the unit that completes each (sequence, group).  Output as
 * palu_softmax_value.  workspace: palu_rope_attend_workspace() bytes,
 * zero-initialised once (the counters reset themselves).
 */
int palu_value_tc(int bits, const void* hv, const float* scales, const float* zps, int B,
                  int n_heads, int s, int G, int Rv_pad, int T_cap, const float* logits,
                  int ld_logits, const int* t_dev, const int* ranks_v, const int* o_off, float* ctx,
                  int ld_ctx, void* workspace, void* stream);

/*
 * Rope-off score (attention.py:380-388, both fusions active): logits[b][i][t]
 * = scale * (H_k[g(i)][t] . q_lat_i) for t <= *t_dev, where q_lat_i =
 * y[b][q_off[i] : q_off[i] + ranks[g(i)]] (y = x @ [wq_fused | A_k | A_v]).
 * palu_latent_score: CUDA cores, every dtype / bit width, s_k <= 8.
 * palu_latent_score_tc: tcgen05 streaming kernel (D[128 tokens x 16] = H_k x
 * Q^T per tile), s_k <= 16, R_pad % 64 == 0, <= 256; bits 16 streams bf16
 * rows through TMA, bits 2/3/4/8 unpack packed codes as c - z (converter
 * warps, as palu_rope_score_tc) and scale the logits per token.
 */
int palu_latent_score(int dtype, int bits, const void* hk, const float* scales, const float* zps,
                      int B, int n_heads, int s_k, int G, int R_pad, int T_cap, const float* y,
                      int ld_y, const int* q_off, const int* ranks, float scale, const int* t_dev,
                      float* logits, int ld_logits, void* stream);
int palu_latent_score_tc(int bits, const void* hk, const float* scales, const float* zps, int B,
                         int n_heads, int s, int G, int R_pad, int T_cap, const float* y, int ld_y,
                         const int* q_off, const int* ranks, float scale, const int* t_dev,
                         float* logits, int ld_logits, void* stream);

/* Diagnostics for the fused kernel (not on the product path): with
 * PALU_FUSED_TRACE set, palu_rope_attend_tc records a per-CTA timeline
 * ([CTA][512] u64: start ns, end ns, SM id, role/count, event times) that
 * palu_fused_trace copies to host (returns the CTA count);
 * palu_fused_max_clusters reports how many 2-CTA clusters of the fused
 * kernel can be co-resident at the given dynamic shared memory size. */
int palu_fused_trace(unsigned long long* host, size_t max_ctas);
int palu_fused_max_clusters(int smem_bytes);

/* cos/sin tables for palu_rope_score_tc: [T_cap/128 + 1][64 pairs] tile bases
 * (fp64-reduced) followed by [128][64] in-tile offsets, float2 each. */
int palu_rope_table(const double* theta, int half, int T_cap, float* rope_tab, void* stream);
size_t palu_rope_table_floats(int half, int T_cap);

/*
 * Softmax + fused value path (attention.py:445-446, _value_output :350-362
 * up to the wo_fused product):  ctx[b][o_off[i] + c] = sum_t' p_i[t'] H_v[g(i)][t'][c]
 * with p_i = softmax(sum of the n_planes logit planes [b][i][0..*t_dev]),
 * split over n_chunks token
 * chunks per (b, group) and merged in a fixed order (deterministic) by the
 * last CTA of each (b, group).  workspace: palu_softmax_value_workspace()
 * bytes, zero-initialised once (the arrival tickets reset themselves).
 */
size_t palu_softmax_value_workspace(int B, int n_heads, int R_pad, int n_chunks);
int palu_softmax_value(int dtype, int bits, const void* hv, const float* scales,
                       const float* zps, int B, int n_heads, int s_v, int G, int R_pad,
                       const int* ranks_v, const int* o_off, int T_cap, const float* logits,
                       int ld_logits, int n_planes, size_t plane_stride, const int* t_dev,
                       int n_chunks, void* workspace, float* ctx, int ld_ctx, void* stream);

/* *t_dev += 1 (cache.t += 1, attention.py:447) -- the last node of a step. */
int palu_advance(int* t_dev, void* stream);

/*
 * Uncompressed baseline (K0; semantics of reference_decode,
 * attention.py:133-168): append post-RoPE k and v rows at t, then per head
 * softmax(K q / sqrt(d_h)) V.  kc/vc: [B][n][T_cap][d_h] in `dtype`;
 * qkv: fp32 [B][3*d] (q | k | v, pre-RoPE); out: fp32 [B][d] attention
 * context (before W_o).
 */
int palu_dense_decode(int dtype, const float* qkv, int B, int n_heads, int head_dim,
                      void* kc, void* vc, int T_cap, const double* theta, const int* t_dev,
                      int n_chunks, void* workspace, float* attn, void* stream);
size_t palu_dense_workspace(int B, int n_heads, int head_dim, int n_chunks);

/*
 * Comparator support for the uncompressed step with flashinfer's trtllm-gen
 * decode kernel (bench.py): RoPE + append of row t into an HND paged bf16
 * K/V cache [page][2][n_kv][page_size][d_h] (page = b * pages_per_seq + t /
 * page_size; same semantics as palu_dense_decode's append; qkv fp32
 * [B][n d_h + 2 n_kv d_h], n_kv < n for GQA), rotated q as bf16
 * [B][n][d_h]; and a bf16 -> fp32 cast of the attention output.
 */
int palu_dense_append_paged(const float* qkv, int B, int n_heads, int n_kv, int head_dim,
                            void* kv_pages, int page_size, int pages_per_seq, const double* theta,
                            const int* t_dev, void* q_out, void* stream);
int palu_cast_bf16_f32(const void* src, float* dst, int n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PALU_B200_H */
