/*
 * glad.h — C ABI of libglad: B200 (sm_100a) decode attention for Grouped
 * Latent Attention (GLA), Grouped-Tied Attention (GTA) and an MLA baseline,
 * over a paged cache, with split-KV and a log-sum-exp merge.
 *
 * Paper: arXiv 2505.21487, "Hardware-Efficient Attention for Fast Decoding".
 * Citation key: P:n = line n of the paper text; readings of silent
 * passages are numbered R1..R16 in DESIGN.md ("Readings").
 *
 * Conventions common to every call
 *  - Pointers are DEVICE pointers unless stated.  The caller owns all memory;
 *    the library never allocates on the hot path and never synchronises the
 *    host.  Every kernel-launching call is asynchronous on `stream`
 *    (cudaStream_t passed as void*; NULL = legacy default stream).
 *  - Element types: bf16 for q, cache, out; fp32 for lse and partials;
 *    int32 for block tables and lengths.  All tensors are dense row-major.
 *  - Errors: host-checkable violations return GLAD_ERR_INVALID_ARG (bad
 *    shape/dim/alignment), GLAD_ERR_UNSUPPORTED (valid but no kernel built
 *    for this shape), GLAD_ERR_WORKSPACE (workspace too small) before any
 *    launch; launch failures return GLAD_ERR_CUDA.  glad_last_error() gives a
 *    thread-local message naming the offending argument.  Device-side contract
 *    breaches (page id out of range, seqlens[b] > pages*page_size, a block
 *    table entry < 0 for a page in use) are undefined behaviour.
 *  - Calls are stateless and reentrant.  Concurrent append and decode on the
 *    same pool are forbidden by contract.
 */
#ifndef GLAD_H_
#define GLAD_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GLAD_API __attribute__((visibility("default")))
#else
#define GLAD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GLAD_OK = 0,
  GLAD_ERR_INVALID_ARG = 1,
  GLAD_ERR_UNSUPPORTED = 2,
  GLAD_ERR_WORKSPACE = 3,
  GLAD_ERR_CUDA = 4
} glad_status;

/* Thread-local description of the last error (never NULL). */
GLAD_API const char* glad_last_error(void);
/* Library version string and the compiled target ("sm_100a"). */
GLAD_API const char* glad_version(void);

/*
 * Paged cache layout (one per rank).  P:304 paged KV; P:240 latent heads
 * c_i^KV; P:48 one decoupled RoPE key per token; P:205-213 GTA tied KV +
 * single-head K_RoPE.
 *
 * Row of one token = [head_0 (d_head) | ... | head_{n-1} (d_head) | rope (d_rope) | pad]
 * (reading R6, pinned by the byte counts P:627).
 * Pool = [num_pages][page_size][row_stride] bf16, contiguous.
 *   GLA/MLA: n_heads_kv = latent heads on this rank (h_c / N), d_head = d_c,
 *            d_rope = d_R.   GTA: n_heads_kv = tied KV heads, d_head = d_h,
 *            d_rope = d_h/2 (the K_RoPE half).
 * Requirements: page_size >= 1 (a power of two; page 1 must work),
 * row_stride >= n_heads_kv*d_head + d_rope and a multiple of 8 (16 B),
 * pool 16-byte aligned.
 */
typedef struct {
  int32_t num_pages;
  int32_t page_size;
  int32_t n_heads_kv;
  int32_t d_head;
  int32_t d_rope;
  int32_t _reserved;
  int64_t row_stride;
} glad_cache_layout;

/* Bytes of the pool described by `layout` (host-only, pure). */
GLAD_API size_t glad_pool_bytes(const glad_cache_layout* layout);

/*
 * Paged-cache append.  For b < B and i < n_new, token
 * position p = seqlens_before[b] + i is written to pool row
 *   block_table[b*bt_stride + p/page_size]*page_size + p%page_size
 * with the first n_heads_kv*d_head + d_rope elements of row (b, i) of
 * `rows` [B, n_new, n_heads_kv*d_head + d_rope] bf16 (RoPE part already
 * rotated by the caller).  Padding columns are not touched.  Bit-exact copy.
 * block_table: [B, bt_stride] int32 (device).  seqlens_before: [B] int32
 * (device).  The caller must have allocated the pages.
 */
GLAD_API glad_status glad_cache_append(const glad_cache_layout* layout, void* pool, const int32_t* block_table,
                              int32_t bt_stride, const int32_t* seqlens_before, const void* rows, int32_t B,
                              int32_t n_new, void* stream);

/*
 * Debug/test gather through the same paging arithmetic as the decode
 * producer: dense_out [B, max_len, n_heads_kv*d_head + d_rope] bf16 receives
 * the logical rows 0..seqlens[b]-1 of each sequence; rows >= seqlens[b] are
 * zero.  Bit-exact.
 */
GLAD_API glad_status glad_paged_gather(const glad_cache_layout* layout, const void* pool, const int32_t* block_table,
                              int32_t bt_stride, const int32_t* seqlens, int32_t B, int32_t max_len,
                              void* dense_out, void* stream);

/*
 * Device workspace (bytes) one decode call needs: the schedule plan
 * (per-unit tile prefix sums) and the partial (o, lse) slots of units that
 * the persistent schedule splits between CTAs.  `variant` is GLAD_GLA,
 * GLAD_MLA or GLAD_GTA; num_ctas as in the decode calls.  0 on invalid input.
 * The workspace must be 256-byte aligned; its contents need no
 * initialisation and are overwritten by every call.
 */
GLAD_API size_t glad_decode_workspace_bytes(const glad_cache_layout* layout, int32_t B, int32_t Lq, int32_t H,
                                            int32_t variant, int32_t num_ctas);

/*
 * GLA decode (per rank: O_i = softmax(Q_i (c_i^KV)^T) c_i^KV,
 * with the decoupled-RoPE score term of P:48 added).
 *
 *  q       [B, Lq, H, d_head + d_rope] bf16: absorbed q_nope (d_head = d_c)
 *          || rotated q_rope (d_rope).  Head h attends to latent head
 *          h / (H / n_heads_kv) (contiguous groups).
 *  pool    paged latent cache (layout above).
 *  seqlens [B] int32: KV length of each sequence INCLUDING the Lq new tokens
 *          (already appended).  Lq > 1 is speculative decoding.
 *  causal  1: query t sees keys j <= seqlens[b] - Lq + t (R2); 0: all keys.
 *  softmax_scale  multiplies q.k (the paper writes no scale, R1).
 *  out     [B, Lq, H, d_head] bf16 = sum_j p_j c_j (latent space).
 *  lse     [B, Lq, H] fp32 natural-log LSE (R3); -inf and out = 0 when a
 *          query has no visible key.
 *  workspace / ws_bytes  device workspace (glad_decode_workspace_bytes).
 *  num_ctas  0 = one persistent CTA per SM (the default); k > 0 = exactly k
 *          CTAs.  The KV tiles of all (sequence, head, query block) units are
 *          split evenly across the CTAs (a unit may be cut into split-KV
 *          segments that are LSE-merged); any k gives the same result up to
 *          fp32 rounding order.
 * Launches three kernels on `stream`: plan, decode, merge.
 * Requirements: H % n_heads_kv == 0; (d_head, d_rope) in {(128, 32),
 * (128, 64), (256, 32), (256, 64), (512, 64)}; Lq >= 1; q and out 16-byte
 * aligned.  Other shapes return GLAD_ERR_UNSUPPORTED.
 */
GLAD_API glad_status glad_gla_decode(const void* q, const void* pool, const glad_cache_layout* layout,
                            const int32_t* block_table, int32_t bt_stride, const int32_t* seqlens, int32_t B,
                            int32_t Lq, int32_t H, float softmax_scale, int32_t causal, void* out, float* lse,
                            void* workspace, size_t ws_bytes, int32_t num_ctas, void* stream);

/* MLA baseline: GLA with a single latent head (n_heads_kv == 1). */
GLAD_API glad_status glad_mla_decode(const void* q, const void* pool, const glad_cache_layout* layout,
                            const int32_t* block_table, int32_t bt_stride, const int32_t* seqlens, int32_t B,
                            int32_t Lq, int32_t H, float softmax_scale, int32_t causal, void* out, float* lse,
                            void* workspace, size_t ws_bytes, int32_t num_ctas, void* stream);

/*
 * GTA decode.  q [B, Lq, H, d_head] bf16 = [q_nope (d_head/2) ||
 * rotated q_rope (d_head/2)] (R4).  Pool rows: n_heads_kv tied states of
 * d_head + one rotated K_RoPE of d_rope = d_head/2.  Key of group g =
 * concat(KV_g[:d_head/2], K_RoPE) (tied half never rotated); value = KV_g.
 * out [B, Lq, H, d_head].  Other arguments as glad_gla_decode.
 * Requirements: d_head == 128, d_rope == 64.
 */
GLAD_API glad_status glad_gta_decode(const void* q, const void* pool, const glad_cache_layout* layout,
                            const int32_t* block_table, int32_t bt_stride, const int32_t* seqlens, int32_t B,
                            int32_t Lq, int32_t H, float softmax_scale, int32_t causal, void* out, float* lse,
                            void* workspace, size_t ws_bytes, int32_t num_ctas, void* stream);

/*
 * Split-KV LSE merge (not in the paper; BASELINE north_star):
 *   lse = ln sum_s exp(lse_s),  out = sum_s exp(lse_s - lse) * o_s
 * o_part [S, B, Lq, H, d_v] fp32 (normalised per split), lse_part
 * [S, B, Lq, H] fp32 (-inf for an empty split).  out [B, Lq, H, d_v] bf16,
 * lse [B, Lq, H] fp32.  d_v % 8 == 0.
 */
GLAD_API glad_status glad_splitkv_combine(const float* o_part, const float* lse_part, int32_t S, int32_t B, int32_t Lq,
                                 int32_t H, int32_t d_v, void* out, float* lse, void* stream);

/*
 * Debug only: when device_buf != NULL every subsequent decode launch writes a
 * per-CTA timeline (globaltimer ns; layout in csrc/decode.cuh, kTraceStride
 * uint64 per CTA, CTAs in launch order) into it.  The caller sizes it for
 * the grid.  NULL turns tracing off (the default).  Only a library built
 * with -DGLAD_TRACE=1 (libglad_trace.so, tools/trace.py) records anything.
 * Not thread-safe.
 */
GLAD_API void glad_debug_set_trace(void* device_buf);
/* Debug/benchmark only: bit mask of the decode call's kernels to launch,
 * 1 = plan, 2 = decode, 4 = merge (default 7; used to time the decode kernel
 * alone), plus A/B switches: 8 = cluster multicast for multi-block units,
 * 16 = no rows mode (64-row swap-AB blocks), 32 = cooperative cp.async
 * producer instead of TMA gather4 for pages < 16, 64 = load-only decode
 * (KV tiles streamed and released, no QK / softmax / PV; the output is
 * undefined — measures the memory side alone), 128 = no (head, query
 * block) CTA groups (multi-block units walked in the ((head, b), block)
 * order), 256 = pages < 16 through TMA gather4 alone (default: gather4
 * for most rows of a tile + 16-B cp.async by a second producer warp for the
 * rest).  Not thread-safe. */
GLAD_API void glad_debug_set_phase_mask(int32_t mask);
/* Debug/benchmark only: force the KV tile height (64, 96 or 128 tokens; 0 =
 * library choice).  Results are identical up to fp32 summation order. */
GLAD_API void glad_debug_set_tile(int32_t tokens);

/* ---- tp_shard helpers: host-only, pure (no CUDA) ---- */

/* D = ceil(N * g_q / h_q).  Returns -1 on invalid input. */
GLAD_API int32_t glad_tp_duplication(int32_t N, int32_t g_q, int32_t h_q);

/*
 * Contiguous ownership for rank `rank` of N: KV/latent heads
 * [kv_begin, kv_end) and query heads [q_begin, q_end).  When
 * n_kv_heads < N each KV head is duplicated D = N / n_kv_heads times and its
 * query heads are split across the replicas.  Output pointers are HOST.
 */
GLAD_API glad_status glad_tp_shard(int32_t h_q, int32_t n_kv_heads, int32_t N, int32_t rank, int32_t* kv_begin,
                          int32_t* kv_end, int32_t* q_begin, int32_t* q_end);

/* ---- the upstream step: kernel inputs from raw tensors ---- */

/*
 * Absorbed query formation (P:48 weight absorption; R2 positions, R5 RoPE):
 *   q_out[b,t,h] = [ W_UK[h] q_nope[b,t,h]  ||  RoPE(q_pe[b,t,h], p) ],
 *   p = seqlens[b] - Lq + t  (seqlens include the Lq new tokens, R2).
 * q_nope [B, Lq, H, d_h] bf16, q_pe [B, Lq, H, d_rope] bf16 (unrotated),
 * w_uk [H, d_c, d_h] bf16 (head h's latent -> key up-projection, so the
 * absorbed query is W_UK[h] q_nope), seqlens [B] int32 (device).  q_out
 * [B, Lq, H, d_c + d_rope] bf16 = the q of glad_gla_decode / glad_mla_decode.
 * RoPE: interleaved pairs, theta_i = rope_base^(-2i/d_rope), angle in fp64.
 * fp32 accumulation, bf16 result.  Supported: d_h in {64, 128}, d_c in
 * {128, 256, 512}; q_nope / w_uk 16-byte aligned.
 */
GLAD_API glad_status glad_gla_absorb_query(const void* q_nope, const void* q_pe, const void* w_uk,
                                           const int32_t* seqlens, int32_t B, int32_t Lq, int32_t H, int32_t d_h,
                                           int32_t d_c, int32_t d_rope, float rope_base, void* q_out, void* stream);

/*
 * Cache append with the RoPE key rotated in the same pass (R5): token
 * p = seqlens_before[b] + i gets the row [ latent[b,i] || RoPE(k_pe[b,i], p) ]
 * (paging as glad_cache_append).  latent [B, n_new, n_heads_kv*d_head] bf16,
 * k_pe [B, n_new, d_rope] bf16 unrotated.  The latent part is a bit-exact
 * copy; the RoPE part is rotated in fp64 and rounded to bf16.
 */
GLAD_API glad_status glad_cache_append_rope(const glad_cache_layout* layout, void* pool, const int32_t* block_table,
                                            int32_t bt_stride, const int32_t* seqlens_before, const void* latent,
                                            const void* k_pe, int32_t B, int32_t n_new, float rope_base,
                                            void* stream);

/* ---- prefill: GLA in the materialised form ---- */

/*
 * Causal self-attention over each prompt in the materialised form of P:48,
 * sigma(Q K^T + Q_R K_R^T) V, with per-head keys and values up-projected from
 * the latent (K_h = c_i W_UK[h], V_h = c_i W_UV[h], i = h / (H / h_c)):
 *   out[b,t,h] = sum_{j <= t} softmax_j( scale * (q_nope[b,t,h] . K_h[j]
 *                + RoPE(q_pe[b,t,h], t) . RoPE(k_pe[b,j], j)) ) V_h[j]
 * for t < seqlens[b]; rows t >= seqlens[b] get out = 0, lse = -inf.
 *  q_nope [B, Lmax, H, d_h], q_pe [B, Lmax, H, d_rope] (unrotated),
 *  latent [B, Lmax, h_c, d_c], k_pe [B, Lmax, d_rope] (unrotated),
 *  w_uk, w_uv [H, d_c, d_h] (latent -> per-head key / value), all bf16;
 *  seqlens [B] int32 (device, prompt lengths <= Lmax); out [B, Lmax, H, d_h]
 *  bf16 (head space); lse [B, Lmax, H] fp32 natural log.  RoPE as R5.
 * Steps: two tcgen05 GEMMs materialise [K_h | V_h] rows (+ the rotated
 * RoPE key) in the workspace, the decode kernels run in rows mode over them
 * as a dense pool, the outputs are moved to their positions.  The
 * workspace (glad_gla_prefill_workspace_bytes, 256-byte aligned) holds the
 * materialised rows: B * ceil(Lmax/64)*64 * (2 H d_h + d_rope) bf16 plus q,
 * out and the decode workspace.  Supported: d_h = 128, d_rope = 64,
 * d_c % 64 == 0, H % h_c == 0.
 */
GLAD_API size_t glad_gla_prefill_workspace_bytes(int32_t B, int32_t Lmax, int32_t H, int32_t d_h, int32_t d_rope,
                                                 int32_t num_ctas);
/* The prefill call itself (see above); launches the two up-projection
 * GEMMs, the RoPE / query kernels, plan + decode + merge, the output move. */
GLAD_API glad_status glad_gla_prefill(const void* q_nope, const void* q_pe, const void* latent, const void* k_pe,
                                      const void* w_uk, const void* w_uv, const int32_t* seqlens, int32_t B,
                                      int32_t Lmax, int32_t H, int32_t h_c, int32_t d_c, int32_t d_h, int32_t d_rope,
                                      float softmax_scale, float rope_base, void* out, float* lse, void* workspace,
                                      size_t ws_bytes, int32_t num_ctas, void* stream);

/* ---- sequence split (context-parallel decode, BASELINE
 * north_star "optional sequence-split for long context merged with an LSE
 * all-gather"; the paper itself splits heads only) ---- */

/*
 * Token range [*begin, *end) of a sequence of L keys owned by rank `rank` of
 * the P ranks that hold the same latent / KV heads (host-only, pure).  Ranges
 * are contiguous, page-aligned (except the final end = L), disjoint, ordered
 * by rank and cover [0, L); pages are split as evenly as possible with later
 * ranks taking the extra ones.  Rank P-1 always holds the last
 * min(L, Lq - 1) keys, so it alone decodes with causal = 1 (bottom-right
 * aligned on its local length, R2) and every other rank with causal = 0.
 * An empty range is begin == end.  Output pointers are HOST.
 */
GLAD_API glad_status glad_seq_split_range(int32_t L, int32_t page_size, int32_t Lq, int32_t P, int32_t rank,
                                          int32_t* begin, int32_t* end);

/*
 * LSE all-gather merge step of the sequence split (device).  lse_all
 * [P, rows] fp32: every rank's lse of the same rows (gathered by the caller,
 * e.g. NCCL all-gather; -inf for an empty range).  o [rows, d_v] bf16: this
 * rank's normalised partial output (the decode's bf16 output: one rounding,
 * as in the unsplit path).  Writes o_out [rows, d_v] fp32 (a separate
 * buffer; kept fp32 so the rescale adds no second bf16 rounding: the caller
 * feeds it to the fp32 o_proj GEMM, see tp.seq_split_oproj_allreduce) =
 * o * exp(lse_all[rank] - lse) with lse = ln sum_p exp(lse_all[p]), and
 * lse_out [rows] (may be NULL).  Summing o_out over the P ranks (e.g. inside
 * the o_proj all-reduce, which is linear) gives the attention output over the
 * whole sequence.  d_v % 8 == 0; o, o_out 16-byte aligned.
 */
GLAD_API glad_status glad_seq_split_rescale(const float* lse_all, int32_t P, int32_t rank, const void* o,
                                            int64_t rows, int32_t d_v, void* o_out, float* lse_out, void* stream);

/* Variants for glad_kv_bytes_per_token_per_device. */
enum { GLAD_MHA = 0, GLAD_MQA = 1, GLAD_GQA = 2, GLAD_GTA = 3, GLAD_GLA = 4, GLAD_MLA = 5 };

/*
 * KV-cache bytes per token per device for one layer (P:123-131 extended
 * with the replicated single RoPE head; reproduces P:624-628, P:1000-1004,
 * P:1299-1305).  n_kv_heads: h_q (MHA), 1 (MQA/MLA), h_kv
 * (GQA/GTA), h_c (GLA); d_head: d_h or d_c; d_rope: d_h/2 (GTA) or d_R
 * (GLA/MLA).  Returns -1 on invalid input.
 */
GLAD_API int64_t glad_kv_bytes_per_token_per_device(int32_t variant, int32_t n_kv_heads, int32_t d_head, int32_t d_rope,
                                           int32_t N, int32_t dtype_bytes);

#ifdef __cplusplus
}
#endif
#endif /* GLAD_H_ */
