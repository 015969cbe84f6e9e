// Paged GLA / MLA / GTA decode attention for sm_100a (tcgen05 + TMEM + TMA).
//
// What it computes (per query row n of a (batch b, latent/KV head i) unit):
//   s_j = scale * (q_nope . K_nope_j + q_rope . k_rope_j),  j visible
//   o   = sum_j softmax(s)_j V_j,   lse = ln sum_j exp(s_j)
// GLA/MLA: K_nope = V = latent c_i (d_c), k_rope = the
// token's single decoupled RoPE key.  GTA: K_nope = first half of
// the tied state, V = the full tied state, k_rope = the single K_RoPE head.
//
// B200 design:
//  * "swap-AB": tokens sit on the UMMA M axis (M = 128 = one tile of T
//    tokens), the g_q*Lq query rows that share the latent head sit on N
//    (16/32/64), so every tcgen05.mma is the full-rate M = 128 shape even for
//    g_q = 8.
//  * S^T[T x NQ] = K_tile . Q^T    (A = KV tile, K-major SW128, straight from
//    the TMA-staged paged rows; B = Q, K-major SW128) -> TMEM, double-buffered.
//  * O^T[D_V x NQ] += V^T . P^T    (A = the SAME smem KV tile read MN-major:
//    the latent is loaded once and reused as K and V; B = P^T bf16,
//    MN-major no-swizzle, written by the softmax warps into the tile's RoPE
//    chunk, which is dead once QK is done) -> TMEM accumulator (2 buffers).
//  * Paged loads: one 2-D TMA box of [min(page,128) rows x 64 cols] per
//    (page run, 64-column chunk); the int32 row coordinate comes from the
//    block table (the TMA unit does the per-row address generation that
//    P:301-318 does with cooperative cp.async).
//  * Persistent, tile-balanced ("stream-K") schedule: a plan kernel turns
//    seqlens into per-unit tile prefix sums; CTA c walks the flattened tile
//    range [c*per, (c+1)*per) across units (unit = (b, head, query block)).
//    A unit finished inside one CTA is written directly; a unit cut by a
//    range boundary leaves partials (o/l, lse) in workspace slot 2c or 2c+1 and
//    the combine kernel merges them (split-KV LSE merge).
//  * Warp roles (384 threads): w0 TMA producer, w1 UMMA issuer (warp-uniform
//    scheduler, one elected lane issues), w2-3 Q loader (+ TMEM alloc), w4-7 / w8-11 two
//    softmax warpgroups, each owning half of the query columns for all 128
//    token lanes.
//  * Online softmax with lazy rescaling: the running max only moves when a
//    p exceeds 2^8 (vote via barrier.red.or), so the cross-lane
//    max reduction and the TMEM O rescale run on a handful of tiles per unit.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <type_traits>

#include "ptx.cuh"

namespace glad {

struct DecodeParams {
  const __nv_bfloat16* q;   // [B, Lq, H, DQ]
  const int32_t* block_table;
  const int32_t* seqlens;
  const int32_t* plan;      // [U + 1] exclusive prefix sum of tiles per unit (plan_kernel)
  __nv_bfloat16* out;       // [B, Lq, H, D_V]
  float* lse;               // [B, Lq, H]
  float* o_part;            // [2G][NQ][D_V] partials of split units (first / last segment of a range)
  float* lse_part;          // [2G][NQ]
  int32_t bt_stride;
  int32_t B, Lq, H, g_q;
  int32_t n_heads_kv;       // heads (latent / tied) in the cache
  int32_t d_head;           // column offset between heads in a cache row
  int32_t rope_col;         // column of the RoPE part in a cache row
  int32_t page_size, log2_page, box_rows;
  int32_t n_qblk, n_units;  // query blocks per head, U = n_heads_kv * B * n_qblk (head-major)
  int32_t causal;
  int32_t n_groups;         // > 1: CTAs form n_groups equal groups, one per unit group (see cta_range)
  int32_t seg_cost;         // virtual tiles the plan puts in front of every unit with work (segment-switch
                            // cost: ranges balance tiles + seg_cost x segments); plan[u] + seg_cost = first real tile
  int32_t qb_outer;         // unit order: 1 = ((head, query block), b), 0 = ((head, b), query block)
  const __nv_bfloat16* pool;  // paged cache (cp.async producer path)
  int64_t row_stride;       // elements
  int32_t cp_kv;            // 1: small pages -> cooperative cp.async producer instead of TMA
  int32_t g4;               // small pages -> TMA gather4 of 4 token rows per instruction (lmap = row map, box (64, 1));
                            // 2: + the LSU warp loading part of every tile (hybrid producer), 1: gather4 only
  int32_t q_tma;            // 1: Q via the 3-D tensor map (box (64, q_box_h, q_box_t)); 0: cp.async
  int32_t q_box_h, q_box_t;
  float scale_log2;         // softmax_scale * log2(e)
  int32_t dbg_load_only;    // debug (phase-mask bit 64): stream the KV tiles only (no QK / softmax / PV; output garbage)
  int cl_n;                 // CTAs per cluster = query blocks per (head, sequence); 1 = no cluster.
                            // With cl_n > 1 the plan is over (head, sequence) groups, the CTAs of a
                            // cluster share each KV tile (TMA multicast) and CTA rank r owns query
                            // block r of every group.
  uint64_t* trace;          // debug timeline (nullptr = off): [cta][kTraceStride]
};
// Debug timeline layout per CTA (globaltimer ns): [0] start, [1] first QK,
// [2] end, [3] number of segments, then per tile i < kTraceTiles: [8+8i] load
// issued, [9+8i] QK issued, [10+8i] S seen by softmax, [11+8i] P written (WG0),
// [12+8i] PV issued, [13+8i] stage free seen by the producer (before load i),
// [14+8i] P written by the second softmax warpgroup, [15+8i] epilogue done
// (last tile of a segment only), [16+10i] QK issue returned, [17+10i] PV
// issue returned (per-tile stride 10).
#ifndef GLAD_ROWS_QK_CHUNK
#define GLAD_ROWS_QK_CHUNK 32  // chunked QK issue (4) measured 1.3x slower (0.313 vs 0.236 ms, C3 q_len 2)
#endif
#ifndef GLAD_ROWS_QK_AHEAD
#define GLAD_ROWS_QK_AHEAD 2
#endif
#ifndef GLAD_SOFTMAX_PHASES
#define GLAD_SOFTMAX_PHASES 0
#endif
#ifndef GLAD_PF_MAX_NS
#define GLAD_PF_MAX_NS 2
#endif
// Rows mode, measured slower and off (A/B, decode ms; no-change / QNB2 / QNB2 + defer / defer):
// C6 materialised prefill 2.83 / 2.95 / 2.91 / 2.90, C7 GTA prefill 1.04 / 1.14 / 1.09 / 1.06:
// the early next-Q load stalls the softmax warps on its global loads in the
// first tile of every segment, and the piecewise epilogue adds TMEM reads to
// the per-tile softmax path.
#ifndef GLAD_ROWS_DEFER
#define GLAD_ROWS_DEFER 0
#endif
#ifndef GLAD_ROWS_QNB2
#define GLAD_ROWS_QNB2 0  // two TMEM Q state-part buffers (next segment's Q written during this one)
#endif
#ifndef GLAD_ROWS_DEFER
#define GLAD_ROWS_DEFER 0  // segment epilogue deferred into the next segment's tiles (two O buffers)
#endif
#ifndef GLAD_ROWS_NS_CAP
#define GLAD_ROWS_NS_CAP 4
#endif
#ifndef GLAD_POLY_GTA_ROWS
#define GLAD_POLY_GTA_ROWS 4  // GTA rows mode (A/B, GTA prefill: 0.815 -> 0.798 ms at 4, 0.853 at 2)
#endif
#ifndef GLAD_POLY_EVERY
#define GLAD_POLY_EVERY 0  // every k-th pair of exponentials via exp2_poly2 (0: all on MUFU)
#endif
#ifndef GLAD_ROWS_WG
#define GLAD_ROWS_WG 2  // rows mode: softmax warpgroups splitting each tile's columns (2: C3 q_len 2 0.203 ms vs 0.213 with 1)
#endif
#ifndef GLAD_DBG_NO_TS
#define GLAD_DBG_NO_TS 0
#endif
#ifndef GLAD_NS_CAP
#define GLAD_NS_CAP 4
#endif
#ifndef GLAD_PF_MIN_BOX
#define GLAD_PF_MIN_BOX 64
#endif
#ifndef GLAD_PF_BULK
#define GLAD_PF_BULK 0  // L2 prefetch: 0 = TMA tensor prefetch of the tile's boxes, 1 = bulk page runs, 2 = bulk, head-0 CTAs only
#endif
#ifndef GLAD_PF_EXTRA
#define GLAD_PF_EXTRA 0  // L2 prefetch distance beyond NS tiles
#endif
#ifndef GLAD_SPLIT_STAGES
#define GLAD_SPLIT_STAGES 1
#endif
#ifndef GLAD_TRACE
#define GLAD_TRACE 0
#endif
#ifndef GLAD_REGS_SPLIT
#define GLAD_REGS_SPLIT 0  // measured: warpgroup 0 needs > 100 registers, the split adds spills
#endif
#ifndef GLAD_REGS_LOW
#define GLAD_REGS_LOW 64
#endif
#ifndef GLAD_REGS_HIGH
#define GLAD_REGS_HIGH 224  // 128 x 64 + 256 x 224 = 65536
#endif
#ifndef GLAD_MMA_BACKOFF_NS
#define GLAD_MMA_BACKOFF_NS 0
#endif
#ifndef GLAD_G4_LSU_PCT
#define GLAD_G4_LSU_PCT 62  // pages < 16: % of each tile's rows loaded by the LSU warps next to gather4 (0: gather4 only);
                            // A/B (C2 page 1 / C3 q_len 2 page 1 decode ms), one LSU warp: 0: 0.723 / 0.449,
                            // 31: 0.565 / 0.374, 37: 0.528 / 0.354, 44: 0.510 / 0.316, 50: 0.558 / 0.317;
                            // two LSU warps: 50: 0.444 / 0.291, 56: 0.424 / 0.291, 62: 0.391 / 0.274, 69: 0.448 / 0.294;
                            // warp 0 as a third (after its gather4 issues): 0.510-0.540 / 0.320-0.345 (slower)
#endif
#ifndef GLAD_G4_LSU_WARPS
#define GLAD_G4_LSU_WARPS 2  // LSU warps of the hybrid producer (2: the Q loader warp copies rows too; the LSU
                             // path is per-warp issue-bound, so its rate scales with the warps)
#endif
#ifndef GLAD_G4_LSU_W0
#define GLAD_G4_LSU_W0 0  // hybrid producer: warp 0 copies LSU rows too after its gather4 issues
#endif
#ifndef GLAD_MMA_IDLE_WAIT
#define GLAD_MMA_IDLE_WAIT 0  // swap-AB MMA scheduler: ns suspend hint on the next expected barrier when idle (0: spin)
#endif
constexpr int kTraceTiles = 128;
constexpr int kTraceStride = 8 + 12 * kTraceTiles + 32;  // + 32 per-CTA debug slots at the end

// Rows mode (NQ = 128) fits TMEM: two S buffers [128 x T] + O [128 x D_V] +
// the query state part [128 x D_V / 2 columns].
template <int D_V, int D_KN, int T>
__host__ __device__ constexpr bool rows_fits() {
  return T <= 96 && 2 * T + D_V + D_KN / 2 <= 512;
}

// KV stages of the unsplit (interleaved) stage layout; mirrors the NS
// computation in DecodeCfg with NLO = NCH_V.
template <int D_V, int D_KN, int D_R, int NQ, int T, int D_S = D_V>
__host__ __device__ constexpr int ns_nosplit() {
  constexpr bool rows = (NQ == 128);
  constexpr int nch_v = D_S / 64, nch = nch_v + 1, nqch = D_KN / 64 + 1;
  constexpr int chunk = T * 128, stage = nch * chunk, lgrp = nch_v * 1024, off_r = nch_v * chunk;
  constexpr int qbytes = rows ? NQ * 128 : nqch * NQ * 128;
  constexpr int aux = 3072 + 64 * 32 + T * 4 + (rows ? 1024 : 2 * NQ * 4);
  constexpr int avail = 227 * 1024 - 1024 - aux;
  constexpr int over = rows ? 0 : (16 * lgrp > off_r + 16384 ? 16 * lgrp : off_r + 16384) - stage;
  constexpr int xtra = over - qbytes - aux > 0 ? over - qbytes - aux : 0;
  constexpr int pbuf = rows ? ((T + 63) / 64) * NQ * 128 : 0;
  return (avail - qbytes - 2 * pbuf - xtra) / stage;
}

template <int D_V_, int D_KN_, int D_R_, int NQ_, int T_ = 128, int D_S_ = D_V_>
struct DecodeCfg {
  // Per head, each token's cache row holds a state slice of D_S columns:
  // the key part is its first D_KN columns, the value its last D_V (GLA /
  // MLA: the latent is both, D_KN = D_V = D_S; GTA: the tied state, key =
  // its first half; materialised prefill: [K_h | V_h], D_S = D_KN + D_V).
  static constexpr int D_V = D_V_;    // value width
  static constexpr int D_KN = D_KN_;  // key part taken from the state
  static constexpr int D_S = D_S_;    // state columns loaded per head and token
  static constexpr int V_CH0 = (D_S_ - D_V_) / 64;  // first value chunk (64 columns) of the state
  static constexpr int D_R = D_R_;    // rope width
  static constexpr int NQ = NQ_;      // query rows per unit (UMMA N; UMMA M in rows mode)
  // Rows mode (NQ = 128): query rows on UMMA M, tokens on N (S = Q K^T,
  // O = P V with P kept in TMEM as the A operand of a "TS" MMA).  One CTA
  // then serves 128 query rows of a head (q_len >= 2 speculative decode,
  // P:278) from one read of each KV tile, and a QK MMA reads a 128-row A and
  // a T-row B from shared memory (balanced against the smem operand
  // bandwidth, instead of 6 KB per 32 tensor cycles at N = 64).
  static constexpr bool ROWS = (NQ_ == 128);
  // tokens per tile (64 / 96 / 128).  Swap-AB: the QK UMMA always has
  // M = 128: with T < 128 its rows >= T read whatever follows the tile in
  // shared memory and are discarded by the softmax (a fraction of QK tensor
  // work traded for a third / fourth KV stage).  Rows: N = T.
  static constexpr int T = T_;
  static constexpr int LANES = 32;  // token lanes per warp quarter in S^T
  static constexpr int DQ = D_KN + D_R;
  static constexpr int NCH_V = D_S / 64;  // state chunks in a stage
  static constexpr int NCH = NCH_V + 1;  // + rope chunk
  static constexpr int NCH_QK = D_KN / 64;
  static constexpr int NQCH = NCH_QK + 1;
  static constexpr int RK = D_R / 16;
  static constexpr int CHUNK = T * 128;  // one [T tokens x 64 cols] bf16 box set
  static constexpr int STAGE = NCH * CHUNK;
  // Stage layout.  Swap-AB ("split" stages): the latent columns in two
  // halves, lo = chunks [0, NLO) and hi = chunks [NLO, NCH_V), each
  // [T/8 row groups][NLO chunks][8 rows][128 B] (one 1-KB SW128 atom per
  // (group, chunk): a page run's half slice is one TMA box), then the RoPE
  // chunk [T rows][128 B] (later P^T).  The halves are filled and released
  // separately (kv_full/kv_empty = lo, kv_full_hi/kv_empty_hi = hi + RoPE):
  // PV's first output blocks read only lo, so lo is refilled while PV still
  // runs on hi, and QK(i+2) starts on lo before hi has landed.
  // Rows mode: one interleaved latent [T/8][NCH_V][8][128 B] (its PV reads
  // all d columns as one N = D_V operand with a uniform 1-KB chunk stride).
  // Split only where the stage count is the bottleneck: 128-token tiles with
  // at most two stages (C2 GLA-2 and the GLA-8 shards: 0.2458 -> 0.2362 ms).
  // Measured slower with three or more stages (C4 GTA 0.391 -> 0.421 ms:
  // the extra TMA issues and barrier round trips cost more than the earlier
  // refill gains) and for MLA's 64-token tiles (0.553 -> 0.594 ms).
  static constexpr int NS_NOSPLIT = ns_nosplit<D_V_, D_KN_, D_R_, NQ_, T_, D_S_>();
  static constexpr bool SPLIT = !ROWS && T == 128 && NS_NOSPLIT <= 2 && GLAD_SPLIT_STAGES;
  static constexpr int NLO = SPLIT ? NCH_V / 2 : NCH_V;  // chunks per half (per stage when not split)
  static constexpr int LO_BYTES = NLO * CHUNK;
  static constexpr int LGRP = NLO * 1024;  // latent row-group stride (within a half)
  static constexpr int OFF_R = NCH_V * CHUNK;
  // byte offset of (64-column) latent chunk c within a stage (row group 0)
  static constexpr int chunk_off(int c) { return c < NLO ? c * 1024 : LO_BYTES + (c - NLO) * 1024; }
  // PV output block blk (d in [128 blk, 128 blk + 128)) = chunks 2 blk, 2 blk + 1:
  // distance between them (the MN-major descriptor's LBO)
  static constexpr int PV_LBO = NLO >= 2 ? 1024 : LO_BYTES;
  // last PV output block that reads lo chunks (kv_empty committed after it)
  static constexpr int BLK_LO_LAST = SPLIT && NLO >= 2 ? NLO / 2 - 1 : D_V / 128 - 1;
  static constexpr int QCHUNK = NQ * 128;
  // Rows mode keeps the query's state part (D_KN) in TMEM (A of a TS-mode
  // QK, written by the softmax warps); only its RoPE chunk is staged in
  // shared memory, which leaves room for four KV stages next to it.
  static constexpr int QBYTES = ROWS ? QCHUNK : NQCH * QCHUNK;
  // P^T (bf16, [NQ/8][128 tok][8]) lives in the stage's RoPE chunk, which is
  // dead once QK of that tile has completed: P is thereby multi-buffered with
  // the KV stages at zero extra shared memory.
  // (Rows mode: P lives in TMEM.)
  static constexpr int PBYTES = ROWS ? 0 : T * NQ * 2;
  static constexpr bool P_SW128 = (NQ == 64);  // MN-major SW128 P^T: PV MMA 70 vs 81 cycles (microbench)
  static constexpr int NBLK_O = D_V / 128;
  static constexpr int NWG = 2;
  static constexpr int CW = ROWS ? 32 : NQ / NWG;
  static constexpr int HC = CW;  // columns per softmax thread (one token row)
  static constexpr int MAXSEG = 64;  // per-CTA segment table entries (aux + 3072), 32 B each (ns_nosplit mirrors it)
  // + cp.async row table (+ rows: row-sum exchange; swap-AB: 1/l of the two O buffers for the deferred epilogue)
  static constexpr int AUX = 3072 + MAXSEG * 32 + T * 4 + (ROWS ? 1024 : 2 * NQ * 4);
  static constexpr int AVAIL = 227 * 1024 - 1024 - AUX;
  // bytes the M = 128 QK may read past the end of the last stage (rows >= T)
  static constexpr int OVER_LAT = (SPLIT ? LO_BYTES : 0) + 16 * LGRP;
  static constexpr int OVER_RAW = ROWS ? 0 : (OVER_LAT > OFF_R + 16384 ? OVER_LAT : OFF_R + 16384) - STAGE;
  static constexpr int XTRA = OVER_RAW - QBYTES - AUX > 0 ? OVER_RAW - QBYTES - AUX : 0;
  // Rows mode: P (bf16 [128 rows x T]) in two shared-memory buffers, K-major
  // 128B-swizzled in 64-token chunks (A of an SS PV), so an S buffer is free
  // as soon as the softmax has read it (QK(i+2) does not wait for PV(i)).
  static constexpr int PCH = (T + 63) / 64;
  static constexpr int PBUF = ROWS ? PCH * NQ * 128 : 0;  // one P buffer
  static constexpr int NS_RAW = (AVAIL - QBYTES - 2 * PBUF - XTRA) / STAGE;
  static constexpr int NS_CAP = ROWS ? GLAD_ROWS_NS_CAP : GLAD_NS_CAP;
  static constexpr int NS = NS_RAW > NS_CAP ? NS_CAP : NS_RAW;
  // L2 prefetch of the tile NS ahead by the producer: it shortens the stage
  // refill chain when there are only two stages (C2 GLA-2: 0.277 -> 0.270
  // ms); with three or more the extra TMA issues cost more than they save
  // (C4 GTA 0.573 -> 0.432 ms, C3 rows 0.223 -> 0.213 ms without it).
  static constexpr bool L2PF = NS <= GLAD_PF_MAX_NS;
  // a second Q buffer (next unit's Q prefetched while this one runs) when it
  // costs no KV stage
  static constexpr int NQB = ((AVAIL - 2 * QBYTES - 2 * PBUF - XTRA) / STAGE >= NS) ? 2 : 1;
  static constexpr int OFF_Q = NS * STAGE;
  static constexpr int OFF_P = OFF_Q + NQB * QBYTES;
  static constexpr int OFF_AUX = OFF_P + 2 * PBUF;
  static constexpr int SMEM_BYTES = 1024 + OFF_AUX + AUX + XTRA;
  // TMEM columns.  Swap-AB: two S^T buffers [128 tok x NQ], then O^T [128 d
  // lanes x NBLK_O*NQ].  Rows mode: two S buffers [128 rows x T] (a tile's
  // bf16 P is written over the upper half of its S buffer), then O [128 rows
  // x D_V].
  static constexpr int SCOLS = ROWS ? T : NQ;             // one S buffer
  static constexpr int OCOLS = ROWS ? D_V : NBLK_O * NQ;  // one O accumulator
  static constexpr int TMEM_O = 2 * SCOLS;                // after the two S buffers
  // two O buffers (the next unit's first PV overlaps this unit's epilogue)
  // when TMEM allows, else one (MLA d_c = 512 with 64 rows; rows mode d_c = 256)
  static constexpr int QNCOLS = ROWS ? D_KN / 2 : 0;  // rows mode: Q state part, 2 bf16 per column
  static constexpr int NOB = (2 * SCOLS + 2 * OCOLS + QNCOLS <= 512) ? 2 : 1;
  static constexpr int QN_COL = 2 * SCOLS + NOB * OCOLS;
  // rows mode: two Q state-part buffers when TMEM allows (D_V = 128: the
  // materialised prefill, GTA), so the next segment's Q is written during
  // this segment and its first QK follows this segment's last one at once
  static constexpr int QNB = (ROWS && GLAD_ROWS_QNB2 && QN_COL + 2 * QNCOLS <= 512) ? 2 : 1;
  // rows mode with two O buffers: the segment epilogue is deferred into the
  // next segment's tiles (one 32-column piece per tile) instead of stalling
  // the softmax warps at every segment switch
  static constexpr bool RDEFER = ROWS && NOB == 2 && GLAD_ROWS_DEFER;
  static constexpr int TMEM_USED = QN_COL + QNB * QNCOLS;
  static constexpr int TMEM_COLS =
      TMEM_USED <= 32 ? 32 : TMEM_USED <= 64 ? 64 : TMEM_USED <= 128 ? 128 : TMEM_USED <= 256 ? 256 : 512;
  static constexpr int NTHREADS = 384;
  static_assert(NS >= 1, "a KV stage does not fit in shared memory");
  static_assert(PBYTES <= CHUNK, "P^T must fit in the RoPE chunk");
  static_assert(D_V % 128 == 0 && D_KN % 64 == 0 && D_KN <= D_V, "unsupported head dims");
  static_assert(D_R % 16 == 0 && D_R >= 16 && D_R <= 64, "unsupported rope dim");
  static_assert(NQ == 16 || NQ == 32 || NQ == 64 || NQ == 128, "NQ must be 16/32/64/128");
  static_assert(!ROWS || D_V <= 256, "rows mode: O [128 x D_V] needs D_V <= 256 (one UMMA N)");
  static_assert(TMEM_USED <= 512, "TMEM budget");
  static_assert(QCHUNK % 1024 == 0, "Q chunk alignment");
  static_assert(T == 128 || T == 96 || T == 64, "tile height");
  static_assert(!SPLIT || NCH_V % 2 == 0, "split stages need an even number of latent chunks");
  static_assert(!SPLIT || V_CH0 == 0, "split stages: value = the state's first columns");
  static_assert(D_S % 64 == 0 && D_S >= D_V && D_S >= D_KN && (D_S == D_V || D_S == D_KN + D_V), "state layout");
};

// Column reduction over groups of LANES lanes (32, or 16 for the halves of a
// warp): v[CW] per lane (lane = token) -> every lane returns the reduction
// over its group of column ((lane % LANES) >> (log2 LANES - log2 CW)).
// Halving butterfly: CW-1 shuffles instead of log2(LANES)*CW.
template <int CW, bool MAX, int LANES = 32>
__device__ __forceinline__ float warp_col_reduce(float (&v)[CW], int lane) {
  static_assert(CW >= 2 && CW <= LANES && (CW & (CW - 1)) == 0, "CW");
  int o = LANES / 2;
#pragma unroll
  for (int K = CW; K > 1; K >>= 1, o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < K / 2; ++i) {
      const float send = upper ? v[i] : v[i + K / 2];
      const float keep = upper ? v[i + K / 2] : v[i];
      const float recv = __shfl_xor_sync(0xffffffffu, send, o);
      v[i] = MAX ? fmaxf(keep, recv) : keep + recv;
    }
  }
#pragma unroll
  for (; o >= 1; o >>= 1) {
    const float recv = __shfl_xor_sync(0xffffffffu, v[0], o);
    v[0] = MAX ? fmaxf(v[0], recv) : v[0] + recv;
  }
  return v[0];
}
template <int CW, int LANES = 32>
__device__ __forceinline__ constexpr int col_shift() {
  return (LANES == 32 ? 5 : 4) - (CW == 32 ? 5 : CW == 16 ? 4 : CW == 8 ? 3 : CW == 4 ? 2 : 1);
}

template <class C>
__device__ __forceinline__ void tmem_load_cols(uint32_t taddr, float (&x)[C::CW]) {
  if constexpr (C::CW % 16 == 0) {
#pragma unroll
    for (int cc = 0; cc < C::CW; cc += 16) tmem_ld16(taddr + cc, x + cc);
  } else {
#pragma unroll
    for (int cc = 0; cc < C::CW; cc += 8) tmem_ld8(taddr + cc, x + cc);
  }
}
// S^T columns of this thread (its token row, CW columns).
template <class C>
__device__ __forceinline__ void tmem_load_s(uint32_t taddr, float (&x)[C::HC]) {
  tmem_load_cols<C>(taddr, x);
}
template <class C>
__device__ __forceinline__ void tmem_store_cols(uint32_t taddr, const float (&x)[C::CW]) {
  if constexpr (C::CW % 16 == 0) {
#pragma unroll
    for (int cc = 0; cc < C::CW; cc += 16) tmem_st16(taddr + cc, x + cc);
  } else {
#pragma unroll
    for (int cc = 0; cc < C::CW; cc += 8) tmem_st8(taddr + cc, x + cc);
  }
}

// Unit index -> (head, sequence, query block).  Two orders, both head-major
// (so the RoPE rows a sequence's heads share are read by concurrently running
// CTA groups and hit L2):
//  qb_outer = 0: u = ((head * B) + b) * n_qblk + qb — a sequence's query
//    blocks are consecutive units (clusters: one plan entry per (head, b));
//  qb_outer = 1: u = ((head * n_qblk) + qb) * B + b — every (head, query
//    block) is one CTA group (cta_range), so the n_qblk blocks that read the
//    same KV tiles (MLA's two 64-head blocks, q_len >= 2) stream the same
//    sequence at the same time and the second read of each tile hits L2.
struct UnitIdx {
  int head, b, qb;
};
__device__ __forceinline__ UnitIdx unit_idx(int u, int B, int n_qblk, int qb_outer) {
  UnitIdx r;
  if (qb_outer) {
    r.b = u % B;
    const int g = u / B;
    r.qb = g % n_qblk;
    r.head = g / n_qblk;
  } else {
    r.qb = u % n_qblk;
    const int hb = u / n_qblk;
    r.b = hb % B;
    r.head = hb / B;
  }
  return r;
}

// One unit u and the part of its
// tile range [t0, t1) that falls in this CTA's flattened range.
struct Seg {
  int u, b, head, qb;
  int pi;          // plan entry: the unit (cl_n = 1) or its (head, sequence) group
  int n0, nq;      // query rows [n0, n0 + nq) of the head's Lq*g_q rows
  int L, kv_end;   // keys visible to the block's last query
  int ld_end;      // keys the tile loads cover: kv_end of the group's last block (cluster)
  int t0, t1;      // tile range within the unit
  bool whole;      // unit entirely inside this CTA -> write final output
};

// Keys visible to the last query of rows [n0, n0 + nq) (bottom-right causal).
__device__ __forceinline__ int rows_kv_end(const DecodeParams& p, int L, int n0, int nq) {
  if (!p.causal) return L;
  const int t_last = (n0 + nq - 1) / p.g_q;
  return max(0, min(L, L - p.Lq + t_last + 1));
}
// Unit fields of plan entry pi for this CTA (cluster rank = query block).
template <int NQ>
__device__ __forceinline__ void seg_unit(const DecodeParams& p, int pi, int L, Seg& s) {
  s.pi = pi;
  const int rank = static_cast<int>(blockIdx.x) % p.cl_n;
  s.u = pi * p.cl_n + rank;
  const UnitIdx ui = unit_idx(s.u, p.B, p.n_qblk, p.qb_outer);
  s.qb = ui.qb;
  s.b = ui.b;
  s.head = ui.head;
  const int nq_total = p.Lq * p.g_q;
  s.n0 = s.qb * NQ;
  s.nq = min(NQ, nq_total - s.n0);
  s.L = L;
  s.kv_end = rows_kv_end(p, L, s.n0, s.nq);
  s.ld_end = s.kv_end;
  if (p.cl_n > 1) {  // the group's last query block sees the most keys
    const int n0l = (p.n_qblk - 1) * NQ;
    s.ld_end = rows_kv_end(p, L, n0l, nq_total - n0l);
  }
}

// (noinline: the on-the-fly path after a segment-table overflow is rare;
// its ~20 runtime integer divisions stay out of every warp role's code)
template <int NQ>
__device__ __noinline__ void make_seg(const DecodeParams& p, int u, int cta_t0, int cta_t1, Seg* out) {
  Seg s;
  seg_unit<NQ>(p, u, __ldg(p.seqlens + unit_idx(u * p.cl_n, p.B, p.n_qblk, p.qb_outer).b), s);
  const int pu0 = __ldg(p.plan + u) + p.seg_cost, pu1 = __ldg(p.plan + u + 1);
  s.t0 = max(cta_t0, pu0) - pu0;
  s.t1 = min(cta_t1, pu1) - pu0;
  s.whole = (s.t0 == 0 && s.t1 == pu1 - pu0);
  *out = s;
}

// Flattened tile range of CTA c.  With n_groups > 1 the G CTAs form
// n_groups equal groups over equal unit counts (KV heads, or (head, query
// block) pairs with qb_outer) and group g splits its own tiles [plan[g U/n],
// plan[(g+1) U/n]) evenly, so CTA (g, k) works on the same sequences as
// (g', k) at the same time: the RoPE rows the heads share, and with
// qb_outer the KV tiles the query blocks share, are served from L2.
struct CtaRange {
  int t0, t1;
};
constexpr int kMaxGroups = 64;  // CTA groups (api.cu caps n_groups)
__device__ __forceinline__ CtaRange cta_range(int c, int G, const int32_t* plan, int U, int n_groups) {
  CtaRange r;
  if (n_groups > 1) {
    const int Gh = G / n_groups, upg = U / n_groups;
    const int g = c / Gh, k = c - g * Gh;
    const int gs = __ldg(plan + g * upg), n = __ldg(plan + (g + 1) * upg) - gs;
    const int per = (n + Gh - 1) / Gh;
    r.t0 = gs + min(n, k * per);
    r.t1 = gs + min(n, (k + 1) * per);
  } else {
    const int total = __ldg(plan + U);
    const int per = (total + G - 1) / G;
    r.t0 = min(total, c * per);
    r.t1 = min(total, r.t0 + per);
  }
  return r;
}
// The same from the group boundaries gb[g] = plan[g U/n] (g = 0..n, n >= 1
// groups; n = 1: [0, total]) staged in shared memory (merge kernel).
__device__ __forceinline__ CtaRange cta_range_gb(int c, int G, const int* gb, int ng) {
  const int Gh = G / ng, g = c / Gh, k = c - g * Gh;
  const int gs = gb[g], n = gb[g + 1] - gs, per = (n + Gh - 1) / Gh;
  CtaRange r;
  r.t0 = gs + min(n, k * per);
  r.t1 = gs + min(n, (k + 1) * per);
  return r;
}
__device__ __forceinline__ int cta_of_tile_gb(int t, int G, const int* gb, int ng) {
  const int Gh = G / ng;
  int g = 0;
  while (g + 1 < ng && gb[g + 1] <= t) ++g;
  const int gs = gb[g], n = gb[g + 1] - gs, per = (n + Gh - 1) / Gh;
  return g * Gh + (t - gs) / per;
}

// Segment table entry (32 B, built once in the prologue so that no warp role
// runs the divisions of seg_unit): e0 = (plan entry, t0, t1, L | whole << 30),
// e1 = (b | head << 20, n0, kv_end, ld_end).
template <int NQ>
__device__ __forceinline__ void seg_to_entry(const Seg& s, int4* dst) {
  dst[0] = make_int4(s.pi, s.t0, s.t1, s.L | ((s.whole ? 1 : 0) << 30));
  dst[1] = make_int4(s.b | (s.head << 20), s.n0, s.kv_end, s.ld_end);
}
template <int NQ>
__device__ __forceinline__ Seg seg_from_entry(const DecodeParams& p, const int4* e) {
  const int4 e0 = e[0], e1 = e[1];
  Seg s;
  s.pi = e0.x;
  s.u = e0.x * p.cl_n + static_cast<int>(blockIdx.x) % p.cl_n;
  s.t0 = e0.y;
  s.t1 = e0.z;
  s.L = e0.w & 0x3FFFFFFF;
  s.whole = (e0.w >> 30) & 1;
  s.b = e1.x & 0xFFFFF;
  s.head = e1.x >> 20;
  s.n0 = e1.y;
  s.qb = e1.y / NQ;
  s.nq = min(NQ, p.Lq * p.g_q - e1.y);
  s.kv_end = e1.z;
  s.ld_end = e1.w;
  return s;
}

// SP: producer paths compiled in — 0: page-run TMA boxes only; 1: + pages <
// 16 through gather4 / the hybrid gather4 + LSU producer; 2: + the
// cooperative cp.async producer (phase-mask bit 32).  Separate
// instantiations keep their code (and register pressure) out of each other:
// the hybrid producer's code alone made the page-64 kernel 6 % slower, the
// cp.async producer's added 98 B of spills to the hybrid one.
template <class C, int SP>
__global__ void __launch_bounds__(C::NTHREADS, 1)
    decode_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap lmap,
                  const __grid_constant__ CUtensorMap qmap,
                  const DecodeParams p) {
  constexpr int T = C::T, NQ = C::NQ, CW = C::CW, NS = C::NS;
  constexpr float TAU = 8.0f;  // lazy-rescale threshold (log2 units)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  uint8_t* aux = smem + C::OFF_AUX;
  uint64_t* bars = reinterpret_cast<uint64_t*>(aux);
  uint64_t* kv_full = bars;        // [4] TMA -> MMA      (tx bytes)
  uint64_t* kv_empty = bars + 4;   // [4] PV done -> TMA  (stage incl. its P^T slot is free)
  uint64_t* s_full = bars + 8;     // [2] QK done -> softmax
  uint64_t* s_empty = bars + 10;   // [2] softmax read S -> MMA
  uint64_t* p_full = bars + 12;    // [4] P^T written (per stage) -> MMA
  uint64_t* pv_done = bars + 16;   // [4] PV(j) complete, j % 4 (O rescale / epilogue)
  uint64_t* q_full = bars + 20;    // [2] Q buffer (s % NQB) of segment s loaded (64 arrivals)
  uint64_t* q_empty = bars + 22;   // [2] last QK of segment s done: Q buffer (s % NQB) free
  uint64_t* o_empty = bars + 24;   // [2] epilogue read O buffer (s & 1) (8 arrivals)
  uint64_t* cl_empty = bars + 26;  // [4] cluster: stage free in all cl_n CTAs (leader's copy is used)
  uint64_t* qn_full = bars + 30;   // [2] rows mode: Q state part of segment s written to TMEM buffer s % QNB (8 warps)
  uint64_t* kv_full_hi = reinterpret_cast<uint64_t*>(aux + 2560);   // [4] split stages: hi half + RoPE landed
  uint64_t* kv_empty_hi = reinterpret_cast<uint64_t*>(aux + 2592);  // [4] split stages: hi half + P^T free
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aux + 256);
  int* range_s = reinterpret_cast<int*>(aux + 264);        // [4] cta tile range, #segments, overflow unit
  int4* segtab = reinterpret_cast<int4*>(aux + 3072);      // [MAXSEG][2] (seg_to_entry)
  int* rowtab = reinterpret_cast<int*>(aux + 3072 + C::MAXSEG * 32);  // [T] pool row per tile row (cp path)
  int* vend_s = reinterpret_cast<int*>(aux + 320);         // [NQ] visible-key end per query column
  float* m_run = reinterpret_cast<float*>(aux + 640);      // [NQ] running max (log2 units)
  float* nm_s = reinterpret_cast<float*>(aux + 896);       // [NQ] -m_run (0 while m_run = -inf)
  float* red = reinterpret_cast<float*>(aux + 1280);       // [2 wg][4 warps][32]
  float* alpha_s = reinterpret_cast<float*>(aux + 2304);   // [NQ] rescale factors / 1/l

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  // small pages with TMA-loaded Q: gather4 + LSU hybrid producer (warps 0 + 3)
  constexpr int G4_LSU_ROWS = (C::T * GLAD_G4_LSU_PCT / 100) & ~3;
  const int cp_kv = SP == 2 ? p.cp_kv : 0;  // small-page producer modes (0 in the page-run instantiation)
  const int g4 = SP == 1 ? p.g4 : 0;
  const bool g4_lsu = G4_LSU_ROWS > 0 && g4 == 2 && p.q_tma;
  const bool g4_lsu2 = g4_lsu && GLAD_G4_LSU_WARPS == 2;  // warp 2 (Q loader) copies LSU rows too
  if (GLAD_TRACE && p.trace && threadIdx.x == 0) p.trace[static_cast<size_t>(cta) * kTraceStride + 7] = globaltimer();

  // ------------------------------------------------------------- setup
  // (PDL) barrier init, TMEM alloc and descriptor prefetch below may overlap
  // the plan kernel; everything that reads global memory another kernel
  // wrote (plan, Q, cache, block table) comes after griddep_wait()
  if (warp == 0) {
    griddep_wait();
    griddep_launch();  // the merge kernel may be scheduled as SMs free up
    // Work range of this CTA and its segment table, with warp-parallel loads
    // (a serial search over the plan would cost one L2 round trip per step).
    const int U = p.n_units;
    const CtaRange rg = cta_range(cta / p.cl_n, gridDim.x / p.cl_n, p.plan, U, p.n_groups);
    const int t0 = rg.t0, t1 = rg.t1;
    int lo = 0, hi = U - 1;  // last unit with plan[u] <= t0 (plan[0] = 0)
    while (lo < hi) {
      const int step = (hi - lo + 32) / 32;
      const int idx = lo + lane * step;
      const bool ok = idx <= hi && __ldg(p.plan + idx) <= t0;
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      const int k = 31 - __clz(m);
      lo = lo + k * step;
      hi = min(hi, lo + step - 1);
    }
    int nseg = 0, more = -1;
    if (t0 < t1) {
      for (int base = lo;; base += 32) {
        const int u = base + lane;
        int pr0 = t1, pu1 = t1;
        if (u < U) { pr0 = __ldg(p.plan + u); pu1 = __ldg(p.plan + u + 1); }
        const bool in = u < U && pr0 < t1;
        const int pu0 = pr0 + p.seg_cost;  // first real tile of the unit
        const int st0 = max(t0, pu0) - pu0, st1 = min(t1, pu1) - pu0;
        const bool has = in && st1 > st0;
        int L = 0;
        if (has) L = __ldg(p.seqlens + unit_idx(u * p.cl_n, p.B, p.n_qblk, p.qb_outer).b);
        const unsigned hm = __ballot_sync(0xffffffffu, has);
        const int pos = nseg + __popc(hm & ((1u << lane) - 1));
        const int whole = (st0 == 0 && st1 == pu1 - pu0) ? 1 : 0;
        if (has && pos < C::MAXSEG) {
          Seg sg;
          seg_unit<NQ>(p, u, L, sg);
          sg.t0 = st0;
          sg.t1 = st1;
          sg.whole = whole != 0;
          seg_to_entry<NQ>(sg, segtab + 2 * pos);
        }
        const int cnt = __popc(hm);
        if (nseg + cnt > C::MAXSEG) {  // table full: the rest is walked on the fly
          const unsigned keep = C::MAXSEG - nseg;
          // first unit not stored: the (keep)-th set bit of hm
          unsigned mm = hm;
          for (unsigned i = 0; i < keep; ++i) mm &= mm - 1;
          more = base + __ffs(mm) - 1;
          nseg = C::MAXSEG;
          break;
        }
        nseg += cnt;
        if (__ballot_sync(0xffffffffu, !in) != 0u) break;  // reached the end of the range
      }
    }
    if (lane == 0) {
      range_s[0] = t0;
      range_s[1] = t1;
      range_s[2] = nseg;
      range_s[3] = more;
    }
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      const int nfull = cp_kv ? (p.q_tma ? 64 : 32) : (g4_lsu ? 1 + 32 * (1 + (g4_lsu2 ? 1 : 0) + (GLAD_G4_LSU_W0 ? 1 : 0)) : 1);  // cp.async lanes (+ the expect_tx arrival)
      mbar_init(&kv_full[i], nfull);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&kv_full_hi[i], nfull);
      mbar_init(&kv_empty_hi[i], 1);
      mbar_init(&p_full[i], C::ROWS ? 4 * GLAD_ROWS_WG : 8);  // softmax warps
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], C::ROWS ? 4 * GLAD_ROWS_WG : 8);
      mbar_init(&o_empty[i], C::ROWS ? 4 * GLAD_ROWS_WG : 8);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&pv_done[i], 1);
    for (int i = 0; i < 4; ++i) mbar_init(&cl_empty[i], p.cl_n);
    for (int i = 0; i < 2; ++i) mbar_init(&qn_full[i], 4 * GLAD_ROWS_WG);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], p.q_tma ? 1 : 64);
      mbar_init(&q_empty[i], 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmap);
    if (!cp_kv) tma_prefetch_desc(&lmap);  // latent boxes, or the gather4 row map
    if (p.q_tma) tma_prefetch_desc(&qmap);
  }
  if (warp == 2) { tmem_alloc(tmem_slot, C::TMEM_COLS); tmem_relinquish(); }
  if (warp != 0) griddep_wait();
  if (warp == 3) {
    // While warp 0 searches the plan: touch the block table, Q and the plan
    // so this SM's address translations are warm when the producer and the
    // Q loader start (their first accesses otherwise pay TLB misses, all
    // 148 SMs at once: measured ~5 us before the first KV load).
    if (lane == 0) prefetch_l2(p.block_table);
    if (lane == 1) prefetch_l2(p.q);
    if (lane == 2) prefetch_l2(p.seqlens);
    if (lane == 3) prefetch_l2(p.o_part);
    if (lane == 4) prefetch_l2(p.out);
  }
  tc_fence_before();
  __syncthreads();
  if (p.cl_n > 1) cluster_sync();  // peers' barriers initialised before any remote arrive / multicast
  tc_fence_after();
#if GLAD_REGS_SPLIT
  // 384 threads x 168 registers at launch; warpgroup 0 (producer, MMA
  // issuer, Q loader) needs few, the two softmax warpgroups many.
  if (warp < 4) setmaxnreg_dec<GLAD_REGS_LOW>();
  else setmaxnreg_inc<GLAD_REGS_HIGH>();
#endif
  const uint32_t tmem = *tmem_slot;
  const int cta_t0 = range_s[0], cta_t1 = range_s[1], nseg_tab = range_s[2], u_more = range_s[3];
  // debug timeline: compiled in only with -DGLAD_TRACE=1 (libglad_trace.so, tools/trace.py)
  uint64_t* trace = (GLAD_TRACE && p.trace) ? p.trace + static_cast<size_t>(cta) * kTraceStride : nullptr;
  if (trace && threadIdx.x == 0) {
    trace[0] = globaltimer();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    trace[kTraceStride - 1] = smid;  // (overlaps tile 127's last slot: only CTAs with < 128 tiles)
  }

  // All roles walk the same sequence of segments: entries of the table,
  // then (only if it overflowed) units walked on the fly from u_more.
  // `k` counts segments, `u` is the on-the-fly cursor.
  auto next_seg = [&](int& k, int& u, Seg& s) -> bool {
    if (k < nseg_tab) {
      s = seg_from_entry<NQ>(p, segtab + 2 * k++);
      return true;
    }
    if (u_more < 0) return false;
    if (k == nseg_tab && u < u_more) u = u_more;
    for (;; ++u) {
      if (u >= p.n_units) return false;
      if (__ldg(p.plan + u) >= cta_t1) return false;
      Seg tmp;
      make_seg<NQ>(p, u, cta_t0, cta_t1, &tmp);
      s = tmp;
      if (s.t1 > s.t0) { ++u; ++k; return true; }
    }
  };

  if (cp_kv && (warp == 0 || (warp == 3 && p.q_tma))) {
    // ============ cooperative cp.async producer for small pages ============
    // The paper's distributed offset calculation on B200 terms: each lane
    // resolves the page-table entry of "its" rows (one lookup per token, an
    // int32 pool row kept in a register); for every row the warp broadcasts
    // that row index with one shuffle and copies the row's slices with
    // 16-B cp.async (lanes = consecutive 16-B units, 512 contiguous bytes per
    // warp instruction) into the same 128B-swizzled layout TMA produces.
    // Two producer warps (0 and 3) split the rows when Q arrives by TMA.
    const int npw = p.q_tma ? 2 : 1;
    const int pw = warp == 0 ? 0 : 1;
    named_bar_sync(3, 96);
    constexpr int RPW = T / 32;          // row registers per lane
    const int row_lo = pw * (T / npw), row_hi = row_lo + T / npw;
    int k = 0, u = 0, it = 0;
    Seg s;
    int pk = 0, pu = 0, ptl = 0, pt1 = 0;  // L2 prefetch cursor NS tiles ahead
    bool pvalid = false;
    Seg ps;
    auto pf_advance = [&]() {
      if (pvalid && ptl + 1 < pt1) { ++ptl; return; }
      pvalid = next_seg(pk, pu, ps);
      if (pvalid) { ptl = ps.t0; pt1 = ps.t1; }
    };
    pf_advance();
    for (int i = 0; i < NS && pvalid; ++i) pf_advance();
    while (next_seg(k, u, s)) {
      const int* bt_row = p.block_table + static_cast<size_t>(s.b) * p.bt_stride;
      const __nv_bfloat16* base_h = p.pool + s.head * p.d_head + lane * 8;  // lane's 16-B unit of the latent slice
      const __nv_bfloat16* base_r = p.pool + p.rope_col + (lane & 7) * 8;
      for (int tl = s.t0; tl < s.t1; ++tl, ++it) {
        const int stage = it % NS;
        const int p0 = tl * T;
        int rowreg[RPW];  // pool row of tile row (32 j + lane), -1 if not visible
#pragma unroll
        for (int j = 0; j < RPW; ++j) {
          const int pos = p0 + 32 * j + lane;
          rowreg[j] = pos < s.ld_end ? __ldg(bt_row + (pos >> p.log2_page)) * p.page_size + (pos & (p.page_size - 1))
                                     : -1;
        }
        mbar_wait(&kv_empty[stage], ((it / NS) & 1) ^ 1);
        if (C::SPLIT) mbar_wait(&kv_empty_hi[stage], ((it / NS) & 1) ^ 1);
        if (trace && pw == 0 && lane == 0 && it < kTraceTiles) trace[13 + 12 * it] = globaltimer();
        const uint32_t sdst = sbase + stage * C::STAGE;
#pragma unroll
        for (int j = 0; j < RPW; ++j) {
          if (32 * j + 31 < row_lo || 32 * j >= row_hi) continue;
#pragma unroll 1  // (not unrolled: keeps the kernel's code small; this is the phase-mask-32 fallback path)
          for (int rr = 0; rr < 32; ++rr) {
            const int r = 32 * j + rr;
            const int row = __shfl_sync(0xffffffffu, rowreg[j], rr);
            if (r < row_lo || r >= row_hi || row < 0) continue;
            const int64_t roff = static_cast<int64_t>(row) * p.row_stride;
            const uint32_t ldst = sdst + (r >> 3) * C::LGRP + (r & 7) * 128;
            // latent slice: units lane, lane + 32, ... (NCH_V chunks x 8 units)
#pragma unroll
            for (int u0 = 0; u0 < C::NCH_V * 8; u0 += 32) {
              const int un = u0 + lane;
              if (un < C::NCH_V * 8)
                cp_async16(ldst + C::chunk_off(un >> 3) + (((un & 7) ^ (r & 7)) << 4), base_h + roff + u0 * 8, 16);
            }
            if (lane < C::D_R / 8)  // RoPE chunk
              cp_async16(sdst + C::OFF_R + r * 128 + ((lane ^ (r & 7)) << 4), base_r + roff, 16);
          }
        }
        cp_async_mbar_arrive(&kv_full[stage]);
        if (C::SPLIT) cp_async_mbar_arrive(&kv_full_hi[stage]);
        if (trace && pw == 0 && lane == 0 && it < kTraceTiles) trace[8 + 12 * it] = globaltimer();
        if (pvalid) {  // L2 prefetch of tile it + NS: each row's latent slice and RoPE
          const int* pbt = p.block_table + static_cast<size_t>(ps.b) * p.bt_stride;
          const int pp0 = ptl * T;
          for (int r2 = row_lo + lane; r2 < row_hi; r2 += 32) {
            const int pos = pp0 + r2;
            if (pos < ps.ld_end) {
              const int64_t row =
                  static_cast<int64_t>(__ldg(pbt + (pos >> p.log2_page))) * p.page_size + (pos & (p.page_size - 1));
              prefetch_l2_bulk(p.pool + row * p.row_stride + ps.head * p.d_head, C::NCH_V * 128);
              prefetch_l2_bulk(p.pool + row * p.row_stride + p.rope_col, C::D_R * 2);
            }
          }
          pf_advance();
        }
      }
    }
  } else if (warp == 0 || (warp == 3 && g4 && p.q_tma) || (warp == 2 && g4_lsu2)) {
    // ========================= TMA producer (all 32 lanes issue) =========================
    // (gather4 mode with TMA-loaded Q: warp 3 is a second producer warp that
    // issues half of every tile's row groups)
    // the first Q load is issued first: QK needs Q, not a second tile (with
    // two LSU warps, warp 2 is the Q loader and arrives once it issued Q(0))
    if (warp != 2) named_bar_sync(3, 96);
    if (trace && lane == 0 && warp == 0) trace[4] = globaltimer();
    const int box_rows = p.box_rows;
    // Boxes per page run of a tile: the latent slice (4-D map: NLO chunks
    // per box, so split stages take one box per half, others one for all
    // NCH_V chunks) and the RoPE chunk (2-D map).  Issued into smem
    // (completing on the half's full barrier) or as an L2 prefetch (bar =
    // nullptr).  item: 0 = latent lo (all chunks if not split), 1 = RoPE,
    // 2 = latent hi.
    const uint16_t mc_mask = static_cast<uint16_t>((1u << p.cl_n) - 1u);
    auto issue_item = [&](const Seg& s, int row, int box, int item, uint32_t stage_addr, uint64_t* bar) {
      if (item != 1) {
        const int half = item == 2 ? 1 : 0;
        const int c = s.head * (p.d_head >> 6) + half * C::NLO;
        const uint32_t dst = stage_addr + half * C::LO_BYTES + box * (box_rows >> 3) * C::LGRP;
        if (!bar) tma_prefetch_4d(&lmap, 0, 0, c, row >> 3);
        else if (p.cl_n > 1) tma_load_4d_mc(dst, &lmap, bar, 0, 0, c, row >> 3, mc_mask);
        else tma_load_4d(dst, &lmap, bar, 0, 0, c, row >> 3);
      } else {
        const uint32_t dst = stage_addr + C::OFF_R + box * box_rows * 128;
        if (!bar) tma_prefetch_2d(&tmap, p.rope_col, row);
        else if (p.cl_n > 1) tma_load_2d_mc(dst, &tmap, bar, p.rope_col, row, mc_mask);
        else tma_load_2d(dst, &tmap, bar, p.rope_col, row);
      }
    };
    // Cluster: rank 0 loads every tile for all cl_n CTAs (multicast) once all
    // of them have freed the stage; the others only arm their kv_full.
    const bool loader = (cta % p.cl_n) == 0;
    auto item_row = [&](const int* bt_row, int p0, int box) {
      const int pos = p0 + box * box_rows;
      return __ldg(bt_row + (pos >> p.log2_page)) * p.page_size + (pos & (p.page_size - 1));
    };
    auto issue_tile = [&](const Seg& s, int tl, int stage, bool prefetch, int page0) {
      const int* bt_row = p.block_table + static_cast<size_t>(s.b) * p.bt_stride;
      const int p0 = tl * T;
      const int ntok = min(T, s.ld_end - p0);
      const int nbox = (ntok + box_rows - 1) / box_rows;
      if (GLAD_PF_BULK && prefetch) {
        // L2 prefetch of whole page runs (all heads' columns + RoPE: rows of a
        // page are contiguous), one bulk prefetch per run
        if (GLAD_PF_BULK == 2 && s.head != 0) return nbox;
        for (int bx = lane; bx < nbox; bx += 32)
          prefetch_l2_bulk(p.pool + static_cast<int64_t>(item_row(bt_row, p0, bx)) * p.row_stride,
                           static_cast<uint32_t>(box_rows * p.row_stride * 2));
        return nbox;
      }
      constexpr int NIT = C::SPLIT ? 3 : 2;
      for (int bx = lane; bx < nbox * NIT; bx += 32)
        issue_item(s, item_row(bt_row, p0, bx / NIT), bx / NIT, bx % NIT, sbase + stage * C::STAGE,
                   prefetch ? nullptr : &kv_full[stage]);
      return nbox;
    };
    // L2 prefetch cursor, PF = NS tiles ahead of the load cursor: the tile
    // that will refill a stage once its PV completes is already on its way
    // to L2, so the refill does not pay the full DRAM latency inside the
    // (release -> load -> QK -> softmax -> PV) chain.
    int pk = 0, pu = 0, ptl = 0, pt1 = 0;
    bool pvalid = false;
    Seg ps;
    auto pf_advance = [&]() {
      if (pvalid && ptl + 1 < pt1) { ++ptl; return; }
      pvalid = next_seg(pk, pu, ps);
      if (pvalid) { ptl = ps.t0; pt1 = ps.t1; }
    };
    // the prefetch cursor is positioned after the first stage load is out
    // (kernel start is latency-bound: the first load must not wait for it)
    bool pf_ready = false;
    int k = 0, u = 0, it = 0, seg = 0;
    Seg s;
    while (next_seg(k, u, s)) {
      const int* bt_row = p.block_table + static_cast<size_t>(s.b) * p.bt_stride;
      if (warp == 2) {  // (g4_lsu2) this segment's Q by TMA, as the Q loader does
        const int qbuf = seg % C::NQB;
        if (seg >= C::NQB) mbar_wait(&q_empty[qbuf], ((seg - C::NQB) / C::NQB) & 1);
        if (lane == 0) {
          constexpr int QCH0 = C::ROWS ? C::NCH_QK : 0;
          const uint32_t qdst = sbase + C::OFF_Q + qbuf * C::QBYTES;
          mbar_arrive_expect_tx(&q_full[qbuf], static_cast<uint32_t>(C::QBYTES));
          const int c1 = s.head * p.g_q + (p.q_box_t == 1 ? s.n0 % p.g_q : 0);
          const int c2 = s.b * p.Lq + s.n0 / p.g_q;
#pragma unroll
          for (int ch = QCH0; ch < C::NQCH; ++ch) {
            const int col = ch < C::NCH_QK ? ch * 64 : C::D_KN;
            tma_load_3d(qdst + (ch - QCH0) * C::QCHUNK, &qmap, &q_full[qbuf], col, c1, c2);
          }
        }
        __syncwarp();
        if (seg == 0) named_bar_arrive(3, 96);
      }
      ++seg;
      for (int tl = s.t0; tl < s.t1; ++tl, ++it) {
        const int stage = it % NS;
        const int p0 = tl * T;
        const int ntok = min(T, s.ld_end - p0);
        const int nbox = (ntok + box_rows - 1) / box_rows;
        // the page lookup of this lane's page run is done before the stage
        // wait: after the release only the TMA issue remains on the critical path
        constexpr int NIT0 = C::SPLIT ? 1 : 2;  // first-issue items per page run (split: lo; else latent + RoPE)
        const int row0 = (loader && !g4 && lane < nbox * NIT0) ? item_row(bt_row, p0, lane / NIT0) : 0;
        if (trace && lane == 0 && warp == 0 && it == 0) {
          if (row0 == 0x7fffffff) __nanosleep(1);  // debug: wait for the lookup itself
          trace[6] = globaltimer();
        }
        const uint32_t ph = ((it / NS) & 1) ^ 1;
        mbar_wait(&kv_empty[stage], ph);
        // cluster multicast and gather4 fill the whole stage at once
        const bool whole_stage = !C::SPLIT || p.cl_n > 1 || g4;
        if (C::SPLIT && whole_stage) mbar_wait(&kv_empty_hi[stage], ph);
        if (trace && lane == 0 && warp == 0 && it < kTraceTiles) trace[13 + 12 * it] = globaltimer();
        if (lane == 0 && !g4)
          mbar_arrive_expect_tx(&kv_full[stage], static_cast<uint32_t>(nbox * box_rows * (C::SPLIT ? C::NLO : C::NCH) * 128));
        if (p.cl_n > 1) {  // stage free here -> tell the loader; the loader waits for every CTA
          if (lane == 0) mbar_arrive_cluster(&cl_empty[stage], 0);
          if (loader) mbar_wait(&cl_empty[stage], (it / NS) & 1);
        }
        __syncwarp();
        const uint32_t stage_addr = sbase + stage * C::STAGE;
        if (g4) {
          // small pages: one gather4 per (4 token rows, 64-column chunk) —
          // the TMA unit does the per-row address generation of P:308-314;
          // each lane resolves the block-table entries of its row groups
          // (rows past the visible end repeat the last visible row: they
          // are zeroed / masked by the softmax like any unloaded row)
          const int ngrp = (ntok + 3) >> 2;
          // hybrid producer (g4_lsu): gather4 (warp 0) takes the first row
          // groups, the LSU path (warp 3: 16-B cp.async per lane)
          // the last G4_LSU_ROWS rows — the two run on different units
          // (TMA engine op rate / LSU), so their rates add
          const int ng4 = g4_lsu ? min(ngrp, (T - G4_LSU_ROWS) / 4) : ngrp;
          if (warp == 0 || !g4_lsu) {
            if (lane == 0 && warp == 0) {
              mbar_arrive_expect_tx(&kv_full[stage], static_cast<uint32_t>(ng4 * (C::SPLIT ? C::NLO : C::NCH) * 512));
              if (C::SPLIT) mbar_arrive_expect_tx(&kv_full_hi[stage], static_cast<uint32_t>(ng4 * (C::NCH - C::NLO) * 512));
            }
            __syncwarp();
            uint64_t* bar_hi = C::SPLIT ? &kv_full_hi[stage] : &kv_full[stage];
            const int npw = (p.q_tma && !g4_lsu ? 2 : 1), pw = warp == 0 ? 0 : 1;
            for (int g = lane + 32 * pw; g < ng4; g += 32 * npw) {
              int rr[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int pos = p0 + min(4 * g + j, ntok - 1);
                rr[j] = __ldg(bt_row + (pos >> p.log2_page)) * p.page_size + (pos & (p.page_size - 1));
              }
              const int r = 4 * g;
              const uint32_t ldst = stage_addr + (r >> 3) * C::LGRP + (r & 7) * 128;
              const int c_head = s.head * p.d_head;
#pragma unroll
              for (int ch = 0; ch < C::NCH_V; ++ch)
                tma_gather4(ldst + C::chunk_off(ch), &lmap, ch < C::NLO ? &kv_full[stage] : bar_hi, c_head + ch * 64,
                            rr[0], rr[1], rr[2], rr[3]);
              tma_gather4(stage_addr + C::OFF_R + r * 128, &lmap, bar_hi, p.rope_col, rr[0], rr[1], rr[2], rr[3]);
            }
          }
          if (g4_lsu && (warp != 0 || GLAD_G4_LSU_W0)) {
            // LSU rows [4 ng4, ntok): each lane resolves one row's pool row,
            // then per row the warp copies the latent slice (lane = 16-B unit)
            // and the RoPE part into the same 128B-swizzled layout
            const __nv_bfloat16* base_h = p.pool + s.head * p.d_head + lane * 8;
            const __nv_bfloat16* base_r = p.pool + p.rope_col + (lane & 7) * 8;
            // LSU warps 3 (, 2 with g4_lsu2, 0 with GLAD_G4_LSU_W0 after its
            // gather4 issues) copy equal contiguous parts of the rows
            constexpr int NLW = 1 + (GLAD_G4_LSU_WARPS == 2 ? 1 : 0) + (GLAD_G4_LSU_W0 ? 1 : 0);
            const int li = warp == 3 ? 0 : (warp == 2 ? 1 : NLW - 1);
            const int h = (ntok - 4 * ng4 + NLW - 1) / NLW;
            const int r_lo = min(ntok, 4 * ng4 + li * h), r_hi = min(ntok, r_lo + h);
            for (int rb = r_lo; rb < r_hi; rb += 32) {
              const int myr = rb + lane;
              const int pos = p0 + min(myr, ntok - 1);
              const int myrow = __ldg(bt_row + (pos >> p.log2_page)) * p.page_size + (pos & (p.page_size - 1));
              const int nr = min(32, r_hi - rb);
#pragma unroll 4
              for (int j = 0; j < nr; ++j) {
                const int r = rb + j;
                const int64_t roff = static_cast<int64_t>(__shfl_sync(0xffffffffu, myrow, j)) * p.row_stride;
                const uint32_t ldst = stage_addr + (r >> 3) * C::LGRP + (r & 7) * 128;
#pragma unroll
                for (int u0 = 0; u0 < C::NCH_V * 8; u0 += 32) {
                  const int un = u0 + lane;
                  if (un < C::NCH_V * 8)
                    cp_async16(ldst + C::chunk_off(un >> 3) + (((un & 7) ^ (r & 7)) << 4), base_h + roff + u0 * 8, 16);
                }
                if (lane < C::D_R / 8) cp_async16(stage_addr + C::OFF_R + r * 128 + ((lane ^ (r & 7)) << 4), base_r + roff, 16);
              }
            }
            cp_async_mbar_arrive(&kv_full[stage]);
            if (C::SPLIT) cp_async_mbar_arrive(&kv_full_hi[stage]);
          }
        } else {
          // latent lo (or the whole latent) + (not split) RoPE, one page run per lane
          if (loader) {
            if (lane < nbox * NIT0) issue_item(s, row0, lane / NIT0, lane % NIT0, stage_addr, &kv_full[stage]);
            for (int bx = lane + 32; bx < nbox * NIT0; bx += 32)  // more boxes than lanes
              issue_item(s, item_row(bt_row, p0, bx / NIT0), bx / NIT0, bx % NIT0, stage_addr, &kv_full[stage]);
          }
          if (C::SPLIT) {
            // hi half + RoPE once PV(it - NS) has read them (P^T lives in the RoPE chunk)
            if (!whole_stage) mbar_wait(&kv_empty_hi[stage], ph);
            if (lane == 0)
              mbar_arrive_expect_tx(&kv_full_hi[stage],
                                    static_cast<uint32_t>(nbox * box_rows * (C::NCH - C::NLO) * 128));
            __syncwarp();
            if (loader) {
              if (lane < nbox) {
                issue_item(s, row0, lane, 2, stage_addr, &kv_full_hi[stage]);
                issue_item(s, row0, lane, 1, stage_addr, &kv_full_hi[stage]);
              }
              for (int bx = lane + 32; bx < nbox; bx += 32) {
                const int rw = item_row(bt_row, p0, bx);
                issue_item(s, rw, bx, 2, stage_addr, &kv_full_hi[stage]);
                issue_item(s, rw, bx, 1, stage_addr, &kv_full_hi[stage]);
              }
            }
          }
        }
        if (trace && lane == 0 && warp == 0 && it < kTraceTiles) trace[8 + 12 * it] = globaltimer();
        // (page runs shorter than GLAD_PF_MIN_BOX rows: no L2 prefetch — its
        // TMA ops per tile grow with the run count; C2 page 16 soaked decode
        // 0.323 -> 0.276 ms without it, page 64 within noise)
        const bool l2pf = C::L2PF && !g4 && box_rows >= GLAD_PF_MIN_BOX;
        if (l2pf && loader && !pf_ready) {
          pf_advance();
          for (int i = 0; i < NS + GLAD_PF_EXTRA + it && pvalid; ++i) pf_advance();
          pf_ready = true;
          if (trace && lane == 0 && warp == 0) trace[kTraceStride - 6] = globaltimer();  // debug: prefetch cursor ready
        }
        if (l2pf && pvalid && loader) {  // L2 prefetch of tile it + NS, after the stage load so it never delays it
          issue_tile(ps, ptl, 0, true, -1);
          pf_advance();
        }
      }
    }
    if (warp == 2 && seg == 0) named_bar_arrive(3, 96);  // no work: release the other producer warps
  } else if (warp == 1 && p.dbg_load_only) {
    // debug: the memory side alone — release every stage as soon as it landed
    int k = 0, u = 0, it = 0, seg = 0;
    Seg s;
    while (next_seg(k, u, s)) {
      for (int tl = s.t0; tl < s.t1; ++tl, ++it) {
        const int stage = it % NS;
        mbar_wait(&kv_full[stage], (it / NS) & 1);
        if (C::SPLIT) mbar_wait(&kv_full_hi[stage], (it / NS) & 1);
        if (lane == 0) {
          mbar_arrive(&kv_empty[stage]);
          if (C::SPLIT) mbar_arrive(&kv_empty_hi[stage]);
        }
        __syncwarp();
      }
      mbar_wait(&q_full[seg % C::NQB], (seg / C::NQB) & 1);  // the Q loader's buffer cycle
      if (lane == 0) mbar_arrive(&q_empty[seg % C::NQB]);
      __syncwarp();
      ++seg;
    }
  } else if (warp >= 4 && p.dbg_load_only) {
    // debug load-only mode: no softmax
  } else if (warp == 1) {
    // ========================= UMMA issuer (warp 1, one elected lane issues) =========================
    // The whole warp runs the scheduler with warp-uniform control flow (every
    // barrier probe and cursor value is made uniform with a vote / REDUX), so
    // descriptors live in uniform registers and each tcgen05.mma costs a
    // couple of uniform adds to issue.
    if constexpr (C::ROWS) {
      // Rows mode: S[128 rows x T] = Q . K_tile^T (A = Q, B = the KV tile,
      // both K-major SW128 as TMA wrote them); O[128 x D_V] += P . V (A = the
      // bf16 P the softmax wrote into the upper half of S's TMEM buffer,
      // B = the same KV tile read MN-major).  S buffer sb is reused by
      // QK(i + 2) only after PV(i) (which reads P from it) has completed.
      constexpr uint32_t idesc_qk = make_idesc_bf16(128, T, false, false);
      constexpr uint32_t idesc_pv = make_idesc_bf16(128, C::D_V, false, true);
      const uint32_t tm = static_cast<uint32_t>(warp_uniform(static_cast<int>(tmem)));
      struct Cursor {
        int k, u, seg, tl, t1, t0;
      };
      Cursor cq{0, 0, -1, 0, 0, 0}, cp{0, 0, -1, 0, 0, 0};
      auto advance = [&](Cursor& c) -> bool {
        if (c.seg >= 0 && c.tl + 1 < c.t1) { ++c.tl; return true; }
        Seg s;
        const bool ok = warp_uniform(next_seg(c.k, c.u, s));
        if (!ok) return false;
        c.k = warp_uniform(c.k);
        c.u = warp_uniform(c.u);
        ++c.seg;
        c.tl = c.t0 = warp_uniform(s.t0);
        c.t1 = warp_uniform(s.t1);
        return true;
      };
      auto probe = [&](uint64_t* bar, int parity) { return warp_uniform(mbar_test_wait(smem_u32(bar), parity)); };
      bool qk_left = advance(cq), pv_left = advance(cp);
      int next_qk = 0, next_pv = 0;
      constexpr int NQK = C::NCH_QK * 4 + C::RK;  // MMAs of one QK
      constexpr int QK_CHUNK = GLAD_ROWS_QK_CHUNK;
      int qk_e = 0;                                // MMAs of QK(next_qk) issued so far
      long long t0 = clock64();
      while (pv_left) {
        bool did = false;
        if (next_pv < next_qk && probe(&p_full[next_pv & 1], (next_pv >> 1) & 1)) {
          const bool first = (cp.tl == cp.t0);
          if (!first || cp.seg < C::NOB || probe(&o_empty[cp.seg % C::NOB], ((cp.seg - C::NOB) / C::NOB) & 1)) {
            if (trace && lane == 0 && next_pv < kTraceTiles) trace[12 + 12 * next_pv] = globaltimer();
            tc_fence_after();
            const int j = next_pv;
            const int stage = j % NS;
            const uint64_t bd = desc_mnmajor_sw128(sbase + stage * C::STAGE + C::V_CH0 * 1024, 1024, C::LGRP);
            const uint32_t obuf = tm + C::TMEM_O + (cp.seg % C::NOB) * C::OCOLS;
            const uint64_t pd = desc_kmajor_sw128(sbase + C::OFF_P + (j & 1) * C::PBUF);
#pragma unroll
            for (int k = 0; k < T / 16; ++k)
              umma_f16_ss_warp(obuf, pd + static_cast<uint64_t>(((k >> 2) * NQ * 128 + (k & 3) * 32) >> 4),
                               bd + static_cast<uint64_t>((k * 2 * C::LGRP) >> 4), idesc_pv, (!first || k > 0) ? 1u : 0u);
            umma_commit_warp(&kv_empty[stage]);
            umma_commit_warp(&pv_done[j & 3]);
            if (trace && lane == 0 && next_pv < kTraceTiles) trace[17 + 12 * next_pv] = globaltimer();
            ++next_pv;
            pv_left = advance(cp);
            did = true;
          }
        }
        // QK is issued in chunks of GLAD_ROWS_QK_CHUNK MMAs, the PV check
        // running between chunks: an MMA issue blocks until the tensor pipe
        // takes it, so a whole 20-MMA QK(i+1) issued just before P(i) lands
        // would hold PV(i) (and with it the stage refill chain) ~0.6 us back.
        bool qk_go = qk_e > 0;
        // QK runs up to two tiles ahead of PV: an S buffer is free once the
        // softmax has read it, so S(i + 2) is ready before softmax(i + 1) ends
        if (!qk_go && qk_left && next_qk - next_pv <= GLAD_ROWS_QK_AHEAD && probe(&kv_full[next_qk % NS], (next_qk / NS) & 1) &&
            probe(&s_empty[next_qk & 1], ((next_qk >> 1) & 1) ^ 1)) {
          const bool first = (cq.tl == cq.t0);
          if (trace && first && cq.seg > 0 && cq.seg < 8 && lane == 0) {  // debug: when each Q barrier flips
            const int sl = kTraceStride - 32 + 3 * cq.seg;
            if (trace[sl] == 0 && mbar_test_wait(smem_u32(&q_full[cq.seg % C::NQB]), (cq.seg / C::NQB) & 1)) trace[sl] = globaltimer();
            if (trace[sl + 1] == 0 && mbar_test_wait(smem_u32(&qn_full[cq.seg % C::QNB]), (cq.seg / C::QNB) & 1)) trace[sl + 1] = globaltimer();
            if (trace[sl + 2] == 0) trace[sl + 2] = globaltimer();  // first probe of this segment's first QK
          }
          if (!first || (probe(&q_full[cq.seg % C::NQB], (cq.seg / C::NQB) & 1) &&
                         probe(&qn_full[cq.seg % C::QNB], (cq.seg / C::QNB) & 1))) {
            qk_go = true;
            if (trace && lane == 0 && next_qk == 0) trace[1] = globaltimer();
            if (trace && lane == 0 && next_qk < kTraceTiles) trace[9 + 12 * next_qk] = globaltimer();
            tc_fence_after();
            if (cp_kv || g4_lsu) fence_proxy_async_smem();
          }
        }
        if (qk_go) {
          const int stage = next_qk % NS;
          const uint32_t d = tm + (next_qk & 1) * C::SCOLS;
          const uint64_t qd = desc_kmajor_sw128(sbase + C::OFF_Q + (cq.seg % C::NQB) * C::QBYTES);
          const uint64_t kd = desc_kmajor_sw128(sbase + stage * C::STAGE, C::LGRP);
          const uint64_t rd = desc_kmajor_sw128(sbase + stage * C::STAGE + C::OFF_R);
          // one chunk, fully unrolled per chunk index (a runtime MMA loop
          // loses the uniform-register descriptors and issues 2x slower).
          // State part: A = Q in TMEM (TS), RoPE part: A = Q's RoPE chunk in smem.
          auto chunk = [&](auto ci) {
            constexpr int e0 = decltype(ci)::value * QK_CHUNK;
#pragma unroll
            for (int e = e0; e < (e0 + QK_CHUNK < NQK ? e0 + QK_CHUNK : NQK); ++e) {
              if (e < C::NCH_QK * 4) {
                if (GLAD_DBG_NO_TS) continue;
                umma_f16_ts_warp(d, tm + C::QN_COL + (cq.seg % C::QNB) * C::QNCOLS + e * 8,
                                 kd + static_cast<uint64_t>(((e >> 2) * 1024 + (e & 3) * 32) >> 4), idesc_qk, e != 0);
              } else {
                umma_f16_ss_warp(d, qd + static_cast<uint64_t>(((e - C::NCH_QK * 4) * 32) >> 4),
                                 rd + static_cast<uint64_t>(((e - C::NCH_QK * 4) * 32) >> 4), idesc_qk,
                                 (GLAD_DBG_NO_TS && e == C::NCH_QK * 4) ? 0u : 1u);
              }
            }
          };
          const int ci = qk_e / QK_CHUNK;
          static_assert(NQK <= 6 * QK_CHUNK, "QK chunks");
          if (ci == 0) chunk(std::integral_constant<int, 0>{});
          else if (ci == 1) chunk(std::integral_constant<int, 1>{});
          else if (ci == 2) chunk(std::integral_constant<int, 2>{});
          else if (ci == 3) chunk(std::integral_constant<int, 3>{});
          else if (ci == 4) chunk(std::integral_constant<int, 4>{});
          else chunk(std::integral_constant<int, 5>{});
          const int e1 = min(qk_e + QK_CHUNK, NQK);
          qk_e = e1;
          if (qk_e == NQK) {
            umma_commit_warp(&s_full[next_qk & 1]);
            if (cq.tl + 1 == cq.t1) umma_commit_warp(&q_empty[cq.seg % C::NQB]);
            if (trace && lane == 0 && next_qk < kTraceTiles) trace[16 + 12 * next_qk] = globaltimer();
            ++next_qk;
            qk_left = advance(cq);
            qk_e = 0;
          }
          did = true;
        }
        if (did) {
          t0 = clock64();
        } else if (warp_uniform(clock64() - t0 > (1ll << 34))) {
          if (lane == 0) printf("glad: MMA scheduler watchdog (rows, cta %d qk %d pv %d)\n", cta, next_qk, next_pv);
          __trap();
        }
      }
      if (trace && lane == 0) trace[3] = cp.seg + 1;
    } else {
      constexpr uint32_t idesc_qk = make_idesc_bf16(128, NQ, false, false);
      constexpr uint32_t idesc_pv = make_idesc_bf16(128, NQ, true, true);
      const uint32_t tm = static_cast<uint32_t>(warp_uniform(static_cast<int>(tmem)));
      // The QK stream and the PV stream walk the CTA's tiles with separate
      // cursors (segment, tile within unit).
      struct Cursor {
        int k, u, seg, tl, t1, t0;
      };
      Cursor cq{0, 0, -1, 0, 0, 0}, cp{0, 0, -1, 0, 0, 0};
      auto advance = [&](Cursor& c) -> bool {  // move to the next tile; false when done
        if (c.seg >= 0 && c.tl + 1 < c.t1) { ++c.tl; return true; }
        Seg s;
        const bool ok = warp_uniform(next_seg(c.k, c.u, s));
        if (!ok) return false;
        c.k = warp_uniform(c.k);
        c.u = warp_uniform(c.u);
        ++c.seg;
        c.tl = c.t0 = warp_uniform(s.t0);
        c.t1 = warp_uniform(s.t1);
        return true;
      };
      auto probe = [&](uint64_t* bar, int parity) { return warp_uniform(mbar_test_wait(smem_u32(bar), parity)); };
      bool qk_left = advance(cq), pv_left = advance(cp);
      int next_qk = 0, next_pv = 0;
      int qk_part = 0;  // split stages: 1 = lo part of QK(next_qk) issued, hi part pending
      // Descriptors are built once per stage / Q buffer; each MMA only adds a
      // compile-time byte offset (>> 4) to the start-address field.
      // QK in two parts (split stages): part 0 = the key chunks of the lo
      // half (issued once lo has landed), part 1 = the remaining key chunks
      // + the RoPE chunk (once hi has landed); s_full is committed after part 1.
      constexpr int QK_LO = C::NCH_QK < C::NLO ? C::NCH_QK : C::NLO;  // key chunks in lo
      auto issue_qk = [&](int part) {
        const int stage = next_qk % NS;
        const int sb = next_qk & 1;
        tc_fence_after();
        if (cp_kv || g4_lsu) fence_proxy_async_smem();  // cp.async (generic proxy) writes -> UMMA (async proxy) reads
        const uint32_t d = tm + sb * NQ;
        const uint64_t ad = desc_kmajor_sw128(sbase + stage * C::STAGE, C::LGRP);
        const uint64_t rd = desc_kmajor_sw128(sbase + stage * C::STAGE + C::OFF_R);
        const uint64_t bd = desc_kmajor_sw128(sbase + C::OFF_Q + (cq.seg % C::NQB) * C::QBYTES);
        if (part == 0) {
#pragma unroll
          for (int c = 0; c < QK_LO; ++c) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_f16_ss_warp(d, ad + static_cast<uint64_t>((C::chunk_off(c) + k * 32) >> 4),
                               bd + static_cast<uint64_t>((c * C::QCHUNK + k * 32) >> 4), idesc_qk, (c | k) != 0);
          }
        }
        if (part == 1 || !C::SPLIT) {
#pragma unroll
          for (int c = C::SPLIT ? QK_LO : C::NCH_QK; c < C::NCH_QK; ++c) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_f16_ss_warp(d, ad + static_cast<uint64_t>((C::chunk_off(c) + k * 32) >> 4),
                               bd + static_cast<uint64_t>((c * C::QCHUNK + k * 32) >> 4), idesc_qk, 1u);
          }
#pragma unroll
          for (int k = 0; k < C::RK; ++k)
            umma_f16_ss_warp(d, rd + static_cast<uint64_t>((k * 32) >> 4),
                             bd + static_cast<uint64_t>((C::NCH_QK * C::QCHUNK + k * 32) >> 4), idesc_qk, 1u);
          umma_commit_warp(&s_full[sb]);
          if (cq.tl + 1 == cq.t1) umma_commit_warp(&q_empty[cq.seg % C::NQB]);  // last QK of the segment: Q free
        }
      };
      auto issue_pv = [&]() {
        tc_fence_after();
        const int j = next_pv;
        const int stage = j % NS;
        const uint32_t kv = sbase + stage * C::STAGE;
        const uint64_t ad = desc_mnmajor_sw128(kv, C::PV_LBO, C::LGRP);
        const uint64_t bd = C::P_SW128 ? desc_mnmajor_sw128(kv + C::OFF_R, 0)
                                       : desc_mnmajor_noswz(kv + C::OFF_R, 128, T * 16);
        const uint32_t obuf = tm + C::TMEM_O + (cp.seg % C::NOB) * C::OCOLS;
        const bool first = (cp.tl == cp.t0);
#pragma unroll
        for (int blk = 0; blk < C::NBLK_O; ++blk) {
#pragma unroll
          for (int k = 0; k < T / 16; ++k)
            umma_f16_ss_warp(obuf + blk * NQ, ad + static_cast<uint64_t>((C::chunk_off(C::V_CH0 + 2 * blk) + k * 2 * C::LGRP) >> 4),
                             bd + static_cast<uint64_t>((C::P_SW128 ? k * 2048 : k * 256) >> 4), idesc_pv,
                             (!first || k > 0) ? 1u : 0u);
          // lo half read by every block up to here: the producer may refill it
          if (C::SPLIT && blk == C::BLK_LO_LAST) umma_commit_warp(&kv_empty[stage]);
        }
        umma_commit_warp(C::SPLIT ? &kv_empty_hi[stage] : &kv_empty[stage]);
        umma_commit_warp(&pv_done[j & 3]);
      };
      long long t0 = clock64();
      while (pv_left) {
        bool did = false;
        if (next_pv < next_qk && probe(&p_full[next_pv % NS], (next_pv / NS) & 1)) {
          // first PV of a segment reuses O buffer (seg % NOB): the epilogue of
          // segment seg - NOB must have read it
          const bool first = (cp.tl == cp.t0);
          if (!first || cp.seg < C::NOB || probe(&o_empty[cp.seg % C::NOB], ((cp.seg - C::NOB) / C::NOB) & 1)) {
            if (trace && lane == 0 && next_pv < kTraceTiles) trace[12 + 12 * next_pv] = globaltimer();
            issue_pv();
            if (trace && lane == 0 && next_pv < kTraceTiles) trace[17 + 12 * next_pv] = globaltimer();
            ++next_pv;
            pv_left = advance(cp);
            did = true;
          }
        }
        // With >= 3 stages the QK stream runs at most one tile ahead of the PV
        // stream: the tensor pipe then strictly alternates QK(i+1), PV(i) (an
        // MMA issue blocks until it executes, so a second QK issued ahead
        // would hold PV(i) back and starve the stage refill).  With two
        // stages the refill itself needs PV(i) first, and greedy order wins.
        // (checked right after a PV issue too: PV(i) + QK(i+2) then go out as
        // one block, one scheduler round trip per tile)
        if (qk_left && qk_part == 0 && (NS < 3 || next_qk - next_pv <= 1) &&
            probe(&kv_full[next_qk % NS], (next_qk / NS) & 1) &&
            probe(&s_empty[next_qk & 1], ((next_qk >> 1) & 1) ^ 1)) {
          const bool first = (cq.tl == cq.t0);
          if (!first || probe(&q_full[cq.seg % C::NQB], (cq.seg / C::NQB) & 1)) {
            if (trace && lane == 0 && next_qk == 0) trace[1] = globaltimer();
            if (trace && lane == 0 && next_qk < kTraceTiles) trace[9 + 12 * next_qk] = globaltimer();
            issue_qk(0);
            if (C::SPLIT) {
              qk_part = 1;
            } else {
              if (trace && lane == 0 && next_qk < kTraceTiles) trace[16 + 12 * next_qk] = globaltimer();
              ++next_qk;
              qk_left = advance(cq);
            }
            did = true;
          }
        }
        // second part of a split QK once the hi half + RoPE have landed
        if (C::SPLIT && qk_part == 1 && probe(&kv_full_hi[next_qk % NS], (next_qk / NS) & 1)) {
          issue_qk(1);
          if (trace && lane == 0 && next_qk < kTraceTiles) trace[16 + 12 * next_qk] = globaltimer();
          qk_part = 0;
          ++next_qk;
          qk_left = advance(cq);
          did = true;
        }
        if (did) {
          t0 = clock64();
        } else {
          if (GLAD_MMA_BACKOFF_NS > 0) __nanosleep(GLAD_MMA_BACKOFF_NS);
          if (GLAD_MMA_IDLE_WAIT > 0) {
            // sleep on the barrier that gates the stage-refill chain first
            if (next_pv < next_qk)
              mbar_try_wait_hint(smem_u32(&p_full[next_pv % NS]), (next_pv / NS) & 1, GLAD_MMA_IDLE_WAIT);
            else if (C::SPLIT && qk_part == 1)
              mbar_try_wait_hint(smem_u32(&kv_full_hi[next_qk % NS]), (next_qk / NS) & 1, GLAD_MMA_IDLE_WAIT);
            else if (qk_left)
              mbar_try_wait_hint(smem_u32(&kv_full[next_qk % NS]), (next_qk / NS) & 1, GLAD_MMA_IDLE_WAIT);
            __syncwarp();
          }
          if (warp_uniform(clock64() - t0 > (1ll << 34))) {
            if (lane == 0) printf("glad: MMA scheduler watchdog (cta %d qk %d pv %d)\n", cta, next_qk, next_pv);
            __trap();
          }
        }
      }
      if (trace && lane == 0) trace[3] = cp.seg + 1;
    }
  } else if (warp < 4 && !(warp == 3 && (cp_kv || g4) && p.q_tma) && !(warp == 2 && g4_lsu2)) {
    // ========================= Q loader: TMA (one thread) or cp.async (64 threads) =========================
    const int tid = threadIdx.x - 64;
    constexpr int QCH0 = C::ROWS ? C::NCH_QK : 0;  // first Q chunk staged in shared memory
    int k = 0, u = 0, seg = 0;
    Seg s;
    while (next_seg(k, u, s)) {
      const int qbuf = seg % C::NQB;
      if (seg >= C::NQB) mbar_wait(&q_empty[qbuf], ((seg - C::NQB) / C::NQB) & 1);
      const uint32_t qdst = sbase + C::OFF_Q + qbuf * C::QBYTES;
      if (p.q_tma) {
        if (tid == 0) {
          mbar_arrive_expect_tx(&q_full[qbuf], static_cast<uint32_t>(C::QBYTES));
          // rows n0.. of head s.head: (t, j) = divmod(n, g_q)
          const int c1 = s.head * p.g_q + (p.q_box_t == 1 ? s.n0 % p.g_q : 0);
          const int c2 = s.b * p.Lq + s.n0 / p.g_q;
#pragma unroll
          for (int ch = QCH0; ch < C::NQCH; ++ch) {  // rows mode: the RoPE chunk only
            const int col = ch < C::NCH_QK ? ch * 64 : C::D_KN;
            tma_load_3d(qdst + (ch - QCH0) * C::QCHUNK, &qmap, &q_full[qbuf], col, c1, c2);
          }
        }
        if (seg == 0) {
          if (trace && tid == 0) trace[5] = globaltimer();
          __syncwarp();
          named_bar_arrive(3, 96);
        }
      } else {
        constexpr int NCQ = C::NQCH - QCH0;  // chunks staged in shared memory
        for (int idx = tid; idx < NQ * NCQ * 8; idx += 64) {
          const int n = idx / (NCQ * 8);
          const int uu = idx - n * (NCQ * 8);
          const int ch = QCH0 + (uu >> 3), w = uu & 7;
          const void* src = p.q;
          uint32_t bytes = 0;
          if (n < s.nq) {
            const bool rope = ch >= C::NCH_QK;
            const int col = rope ? C::D_KN + w * 8 : ch * 64 + w * 8;
            if (!rope || w * 8 < C::D_R) {
              const int ng = s.n0 + n, t = ng / p.g_q, h = s.head * p.g_q + (ng - t * p.g_q);
              src = p.q + ((static_cast<size_t>(s.b) * p.Lq + t) * p.H + h) * C::DQ + col;
              bytes = 16;
            }
          }
          cp_async16(qdst + (ch - QCH0) * C::QCHUNK + n * 128 + ((w ^ (n & 7)) << 4), src, bytes);
        }
        if (seg == 0) named_bar_arrive(3, 96);
        cp_async_wait_all();
        fence_proxy_async_smem();
        mbar_arrive(&q_full[qbuf]);
      }
      ++seg;
    }
    if (seg == 0) named_bar_arrive(3, 96);  // no work: release the producer
  } else if constexpr (C::ROWS) {
    // ============ rows mode: softmax / correction / epilogue (two warpgroups) ============
    // Thread = query row n = TMEM lane (32 wq + lane) of S and O.  Warpgroup
    // wg owns S columns [wg T/2, (wg+1) T/2) of every tile and O columns
    // [wg D_V/2, (wg+1) D_V/2).  Warps 4 + wq and 8 + wq hold the same rows:
    // they keep identical copies of the row's running max (both compute it
    // from the same exchanged values), vote the lazy rescale together
    // (bar.red.or over the pair, barrier 4 + wq) and each keeps a partial
    // row sum, combined in the epilogue.
    if (warp < 4 + 4 * GLAD_ROWS_WG) {  // softmax warpgroups (the rest idle)
    constexpr int NWGR = GLAD_ROWS_WG;   // softmax warpgroups (column split)
    constexpr int TH = T / NWGR;         // S columns per thread
    constexpr int NP = TH / 2;           // bf16 pairs of them (TMEM columns of P)
    constexpr int DH = C::D_V / NWGR;    // O columns per thread
    constexpr uint32_t kTrig = 0x4380u;  // bf16 bits of 2^TAU = 256
    static_assert(TAU == 8.f, "kTrig encodes 2^TAU");
    // every POLY-th pair of exponentials on the FMA pipe: only the GTA rows
    // shape (d_v 128, key 64: the least tensor work per exponential) gains
    constexpr int POLY = (C::D_V == 128 && C::D_KN == 64) ? GLAD_POLY_GTA_ROWS : GLAD_POLY_EVERY;
    static_assert(TH % 16 == 0 && NP % 8 == 0 && DH % 32 == 0, "rows mode tile split");
    const int wg = (warp - 4) >> 2;
    const int wq = warp & 3;
    const int n = wq * 32 + lane;
    const uint32_t lane_addr = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t pair_bar = 4 + wq;
    float* mx_x = red;                                                   // [2 wg][128] partial row max
    float* l_x = reinterpret_cast<float*>(aux + 3072 + C::MAXSEG * 32 + T * 4);  // [2 wg][128] partial row sums
    const float sl2 = p.scale_log2;
    // Q state part of segment sq's row n (this WG's half of D_KN) -> TMEM
    // (A operand of the TS-mode QK: lane = row, 2 bf16 per column).  Called
    // once the last QK that read buffer qb has completed (its S was read).
    auto load_q = [&](const Seg& sq, int qb) {
      constexpr int NV = C::D_KN / (8 * NWGR);  // 16-B vectors of this thread's part of the row
      uint4 v[NV];
      if (n < sq.nq) {
        const int ng = sq.n0 + n, tq = ng / p.g_q, hq = sq.head * p.g_q + (ng - tq * p.g_q);
        const uint4* src = reinterpret_cast<const uint4*>(
            p.q + ((static_cast<size_t>(sq.b) * p.Lq + tq) * p.H + hq) * C::DQ + wg * (C::D_KN / NWGR));
#pragma unroll
        for (int i = 0; i < NV; ++i) v[i] = __ldg(src + i);
      } else {
#pragma unroll
        for (int i = 0; i < NV; ++i) v[i] = make_uint4(0u, 0u, 0u, 0u);
      }
      const uint32_t qa = tmem + lane_addr + C::QN_COL + qb * C::QNCOLS + wg * (C::D_KN / (2 * NWGR));
#pragma unroll
      for (int i = 0; i < NV; i += 4) tmem_st16_u32(qa + i * 4, reinterpret_cast<const uint32_t*>(v + i));
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&qn_full[qb]);
    };
    // debug phase timer (warp 4 of a traced launch): cycles spent between
    // softmax checkpoints, summed over tiles, written at the end
    long long ph_t = clock64(), ph_acc[6] = {0, 0, 0, 0, 0, 0};
    auto PH = [&](int i) {
      if (GLAD_SOFTMAX_PHASES && trace) { const long long t = clock64(); ph_acc[i] += t - ph_t; ph_t = t; }
    };
    int k = 0, u = 0, seg = 0, it = 0;
    Seg s;
    bool have = next_seg(k, u, s);
    if (have) load_q(s, 0);
    // pending (deferred) epilogue of the previous segment (RDEFER): O buffer,
    // 1/l, destination row, next 32-column piece (DH = none pending)
    int e_c = DH, e_j = 0, e_seg = 0;
    bool e_valid = false, e_whole = false;
    float e_inv = 0.f;
    uint32_t e_obuf = 0;
    __nv_bfloat16* e_orow = nullptr;
    float* e_prow = nullptr;
    auto epi_piece = [&]() {
      if (e_c == 0) {  // the segment's last PV must have completed
        mbar_wait(&pv_done[e_j & 3], (e_j >> 2) & 1);
        tc_fence_after();
      }
      const int c = e_c;
      float o[32];
      tmem_ld32(e_obuf + c, o);
      tmem_ld_wait();
      if (c + 32 == DH) {  // O consumed: the segment after next may reuse the buffer
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_empty[e_seg % C::NOB]);
      }
      if (e_valid) {
        if (e_whole) {
#pragma unroll
          for (int q = 0; q < 32; q += 8)
            *reinterpret_cast<uint4*>(e_orow + c + q) =
                make_uint4(pack_bf16x2(o[q] * e_inv, o[q + 1] * e_inv), pack_bf16x2(o[q + 2] * e_inv, o[q + 3] * e_inv),
                           pack_bf16x2(o[q + 4] * e_inv, o[q + 5] * e_inv), pack_bf16x2(o[q + 6] * e_inv, o[q + 7] * e_inv));
        } else {
#pragma unroll
          for (int q = 0; q < 32; q += 4)
            *reinterpret_cast<float4*>(e_prow + c + q) =
                make_float4(o[q] * e_inv, o[q + 1] * e_inv, o[q + 2] * e_inv, o[q + 3] * e_inv);
        }
      }
      e_c += 32;
    };
    while (have) {
      int vend = 0, t_row = 0, h_row = 0;
      if (n < s.nq) {
        const int ng = s.n0 + n;
        t_row = ng / p.g_q;
        h_row = s.head * p.g_q + (ng - t_row * p.g_q);
        vend = p.causal ? max(0, min(s.L, s.L - p.Lq + t_row + 1)) : s.L;
      }
      float m = -INFINITY, nm = 0.f;  // running max (log2 units), -m (0 while m = -inf)
      float2 l2 = make_float2(0.f, 0.f);
      const uint32_t obuf = tmem + lane_addr + C::TMEM_O + (seg % C::NOB) * C::OCOLS + wg * DH;
      Seg sn;
      bool have_n = false, peeked = false;
      for (int tl = s.t0; tl < s.t1; ++tl, ++it) {
        const int sb = it & 1;
        const uint32_t sbuf = tmem + lane_addr + sb * C::SCOLS;
        mbar_wait(&s_full[sb], (it >> 1) & 1);
        PH(0);
        tc_fence_after();
        if (trace && threadIdx.x == 128 && it < kTraceTiles) trace[10 + 12 * it] = globaltimer();
        const int c0 = tl * T + wg * TH;  // first token of this thread's columns
        float x[TH];
#pragma unroll
        for (int c = 0; c < TH; c += 16) tmem_ld16(sbuf + wg * TH + c, x + c);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sb]);  // S(sb) read: QK(it + 2) may overwrite it
        PH(1);
        if (c0 + TH > vend) {
#pragma unroll
          for (int j = 0; j < TH; ++j) x[j] = (c0 + j < vend) ? x[j] : -INFINITY;
        }
        uint32_t pk[NP];
        auto exp_pack = [&]() {
#pragma unroll
          for (int j = 0; j < TH; j += 2) {
            const float2 e = ffma2(make_float2(x[j], x[j + 1]), make_float2(sl2, sl2), make_float2(nm, nm));
            if (POLY && ((j / 2) % POLY) == POLY - 1) {
              const float2 y = exp2_poly2(e);  // part of the exponentials on the FMA pipe
              pk[j / 2] = pack_bf16x2(y.x, y.y);
            } else {
              pk[j / 2] = pack_bf16x2(ex2(e.x), ex2(e.y));
            }
          }
        };
        exp_pack();
        uint32_t pmax = pk[0];
#pragma unroll
        for (int j = 1; j < NP; ++j) pmax = max_u16x2(pmax, pk[j]);
        const bool need = (tl == s.t0) || ((pmax & 0xffffu) > kTrig) || ((pmax >> 16) > kTrig);
        PH(2);
        const bool vote = NWGR == 2 ? named_bar_red_or(pair_bar, 64, need) : __any_sync(0xffffffffu, need);
        if (vote) {
          float mt = x[0];
#pragma unroll
          for (int j = 1; j < TH; ++j) mt = fmaxf(mt, x[j]);
          if constexpr (NWGR == 2) {
            mx_x[wg * 128 + n] = mt;
            named_bar_sync(pair_bar, 64);
            mt = fmaxf(mt, mx_x[(wg ^ 1) * 128 + n]);
          }
          const float mn = fmaxf(m, mt * sl2);
          const float alpha = (mn == -INFINITY) ? 1.f : ex2(m - mn);
          m = mn;
          nm = (mn == -INFINITY) ? 0.f : -mn;
          l2.x *= alpha;
          l2.y *= alpha;
          if (tl > s.t0 && __any_sync(0xffffffffu, alpha != 1.f)) {  // rescale this thread's O half-row
            const int j = it - 1;
            mbar_wait(&pv_done[j & 3], (j >> 2) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < DH; c += 32) {
              float o[32];
              tmem_ld32(obuf + c, o);
              tmem_ld_wait();
#pragma unroll
              for (int q = 0; q < 32; ++q) o[q] *= alpha;
              tmem_st16(obuf + c, o);
              tmem_st16(obuf + c + 16, o + 16);
            }
            tmem_st_wait();
          }
          exp_pack();
        }
        PH(3);
        // row sum of the bf16-rounded p the PV multiplies
#pragma unroll
        for (int j = 0; j < NP; ++j)
          l2 = fadd2(l2, make_float2(__uint_as_float(pk[j] << 16), __uint_as_float(pk[j] & 0xffff0000u)));
        // bf16 P row piece into P buffer sb (K-major SW128, 64-token chunks);
        // its previous contents (tile it - 2) must have been read by PV(it - 2)
        if (it >= 2) mbar_wait(&pv_done[(it - 2) & 3], ((it - 2) >> 2) & 1);
        {
          const uint32_t pb = sbase + C::OFF_P + sb * C::PBUF + n * 128;
#pragma unroll
          for (int g = 0; g < NP / 4; ++g) {
            const int tok = wg * TH + g * 8;  // first token of this 16-B piece
            const uint32_t a = pb + (tok >> 6) * (NQ * 128) + ((((tok & 63) >> 3) ^ (n & 7)) << 4);
            st_shared_v4(a, pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
          }
        }
        const int p0 = tl * T;
        if (p0 + T > s.kv_end) {  // never-loaded tile rows: zero V (0 * stale smem != NaN)
          const uint32_t stage_base = sbase + (it % NS) * C::STAGE;
          for (int idx = wg * 128 + n; idx < T * C::NCH_V; idx += 128 * NWGR) {
            const int tr = idx / C::NCH_V, ch = idx - tr * C::NCH_V;
            if (p0 + tr >= s.kv_end) {
              const uint32_t a = stage_base + (tr >> 3) * C::LGRP + C::chunk_off(ch) + (tr & 7) * 128;
#pragma unroll
              for (int uu = 0; uu < 8; ++uu) st_shared_v4(a + uu * 16, 0u, 0u, 0u, 0u);
            }
          }
        }
        fence_proxy_async_smem();  // P (and zeroed V rows): generic-proxy writes -> UMMA reads
        PH(4);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
        PH(5);
        if (trace && threadIdx.x == 128 && it < kTraceTiles) trace[11 + 12 * it] = globaltimer();
        if (trace && threadIdx.x == 256 && it < kTraceTiles) trace[14 + 12 * it] = globaltimer();
        if (trace && lane == 0 && it < kTraceTiles)  // debug: last softmax warp's P arrival
          atomicMax(reinterpret_cast<unsigned long long*>(trace + 19 + 12 * it), globaltimer());
        if (C::QNB == 2 && !peeked) {
          // two Q buffers: the next segment's Q goes into the other one as soon
          // as this segment's first S was seen (every QK of segment seg - 1,
          // the buffer's last reader, has completed: the MMA pipe is in order)
          peeked = true;
          have_n = next_seg(k, u, sn);
          if (have_n) load_q(sn, (seg + 1) & 1);
        }
        if (C::RDEFER && e_c < DH) epi_piece();  // the previous segment's O, one piece per tile
      }
      if (!peeked) {
        // next segment's Q into TMEM now (this segment's last QK is done), so
        // the load overlaps the epilogue below
        have_n = next_seg(k, u, sn);
        if (have_n) load_q(sn, (seg + 1) % C::QNB);
      }
      if (C::RDEFER) while (e_c < DH) epi_piece();  // (a segment with fewer tiles than pieces)
      if (trace && threadIdx.x == 128 && it - 1 < kTraceTiles) trace[18 + 12 * (it - 1)] = globaltimer();  // next Q in TMEM
      // ---- segment epilogue: O / l, lse (natural log); each WG writes its O half
      float ls = l2.x + l2.y;
      if constexpr (NWGR == 2) {
        l_x[wg * 128 + n] = ls;
        named_bar_sync(pair_bar, 64);
        ls = l_x[n] + l_x[128 + n];  // same order in both WGs
      }
      const float inv_l = ls > 0.f ? 1.f / ls : 0.f;
      const int j = it - 1;
      if (!C::RDEFER) {
        mbar_wait(&pv_done[j & 3], (j >> 2) & 1);
        tc_fence_after();
      }
      // partial slot: 2 per range — the range's first segment (2c) or its
      // last one (2c + 1); only those two can be cut by a range boundary
      const int slot = (2 * (cta / p.cl_n) + (seg == 0 ? 0 : 1)) * p.cl_n + cta % p.cl_n;
      const bool valid = n < s.nq;
      if (valid && wg == 0) {
        const float lse = ls > 0.f ? (m + __log2f(ls)) * 0.69314718055994531f : -INFINITY;
        if (s.whole) p.lse[(static_cast<size_t>(s.b) * p.Lq + t_row) * p.H + h_row] = lse;
        else p.lse_part[static_cast<size_t>(slot) * NQ + n] = lse;
      }
      __nv_bfloat16* orow = p.out + ((static_cast<size_t>(s.b) * p.Lq + t_row) * p.H + h_row) * C::D_V + wg * DH;
      float* prow = p.o_part + (static_cast<size_t>(slot) * NQ + n) * C::D_V + wg * DH;
      if (C::RDEFER) {  // written piecewise during the next segment's tiles (epi_piece)
        e_c = 0;
        e_j = j;
        e_seg = seg;
        e_valid = valid;
        e_whole = s.whole;
        e_inv = inv_l;
        e_obuf = obuf;
        e_orow = orow;
        e_prow = prow;
      }
#pragma unroll 1
      for (int c = 0; c < (C::RDEFER ? 0 : DH); c += 32) {
        float o[32];
        tmem_ld32(obuf + c, o);
        tmem_ld_wait();
        if (c + 32 == DH) {  // O consumed: the segment after next may reuse the buffer
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&o_empty[seg % C::NOB]);
        }
        if (valid) {
          if (s.whole) {
#pragma unroll
            for (int q = 0; q < 32; q += 8)
              *reinterpret_cast<uint4*>(orow + c + q) =
                  make_uint4(pack_bf16x2(o[q] * inv_l, o[q + 1] * inv_l), pack_bf16x2(o[q + 2] * inv_l, o[q + 3] * inv_l),
                             pack_bf16x2(o[q + 4] * inv_l, o[q + 5] * inv_l), pack_bf16x2(o[q + 6] * inv_l, o[q + 7] * inv_l));
          } else {
#pragma unroll
            for (int q = 0; q < 32; q += 4)
              *reinterpret_cast<float4*>(prow + c + q) =
                  make_float4(o[q] * inv_l, o[q + 1] * inv_l, o[q + 2] * inv_l, o[q + 3] * inv_l);
          }
        }
      }
      if constexpr (NWGR == 2) named_bar_sync(pair_bar, 64);  // l_x read by both WGs before the next segment rewrites it
      if (trace && threadIdx.x == 128 && it - 1 < kTraceTiles) trace[15 + 12 * (it - 1)] = globaltimer();
      ++seg;
      s = sn;
      have = have_n;
      PH(5);
    }
    if (C::RDEFER) while (e_c < DH) epi_piece();  // the last segment's O
    if (GLAD_SOFTMAX_PHASES && trace && threadIdx.x == 128)
      for (int i = 0; i < 6; ++i) trace[kTraceStride - 14 + i] = static_cast<uint64_t>(ph_acc[i]);
    }
  } else {
    // ========================= softmax / correction / epilogue =========================
    // Thread -> data: token row tr = 32*wq + lane of S^T (rows >= T carry no
    // token: warp-uniform, they only join the barriers), columns [c0, c0 + CW);
    // O^T: one d row per TMEM lane r = tr.
    constexpr int HC = C::HC, LANES = C::LANES;
    const int wg = (warp - 4) >> 2;
    const int wq = warp & 3;
    const int r = wq * 32 + lane;  // TMEM lane of O^T (d row)
    const int tr = r;              // token row of S^T within the tile
    const bool row_ok = (T == 128) || (wq * 32 < T);
    const int c0 = wg * CW;
    const int cb = c0;
    const uint32_t lane_addr = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t bar_id = 1 + wg;
    const uint32_t nm_addr = smem_u32(nm_s + cb);
    const uint32_t a_addr = smem_u32(alpha_s + cb);
    const uint32_t ao_addr = smem_u32(alpha_s + c0);  // O^T rescale: all CW columns of the WG
    const float sl2 = p.scale_log2;
    // Deferred epilogue: a finished segment's O is written one 128-row
    // block per tile of the NEXT segment (after that tile's P is out, where
    // the softmax warps would otherwise wait for S), not in one piece that
    // stalls the pipeline at every segment switch (~5 us measured).  Its
    // 1/l lives in einv_s[seg % NOB] until then.
    float* einv_s = reinterpret_cast<float*>(aux + 3072 + C::MAXSEG * 32 + T * 4);  // [NOB][NQ]
    int e_blk = C::NBLK_O;  // next block of the pending epilogue (NBLK_O = none pending)
    int e_seg = 0, e_j = 0, e_ncols = 0, e_j0 = 0, e_slot = 0;
    bool e_whole = false;
    size_t e_row0 = 0;
    auto epi_block = [&]() {
      if (e_blk == 0) {  // the segment's last PV must have completed
        mbar_wait(&pv_done[e_j & 3], (e_j >> 2) & 1);
        tc_fence_after();
      }
      const int blk = e_blk;
      const uint32_t eo = tmem + C::TMEM_O + (e_seg % C::NOB) * C::OCOLS;
      float o[CW];
      tmem_load_cols<C>(eo + lane_addr + blk * NQ + c0, o);
      tmem_ld_wait();
      if (blk == C::NBLK_O - 1) {  // O buffer consumed: the segment after next may reuse it
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_empty[e_seg % C::NOB]);
      }
      const uint32_t inv_addr = smem_u32(einv_s + (e_seg % C::NOB) * NQ + c0);
      const int d = blk * 128 + r;
      if (e_whole) {
        // bf16 output [row][d]: a register transpose over groups of 8 lanes
        // (8 consecutive d) turns 32 two-byte stores per thread into CW/8
        // 16-byte ones (the epilogue was bound by store-instruction issue)
        static_assert(CW % 8 == 0, "epilogue transpose");
        uint32_t w[CW / 2];  // stage 0: bf16 pairs (d even, d odd) of CW/2 columns
        {
          float v[CW];
#pragma unroll
          for (int n = 0; n < CW; n += 4) {
            const float4 a = ld_shared_f4(inv_addr + n * 4);
            v[n] = o[n] * a.x; v[n + 1] = o[n + 1] * a.y; v[n + 2] = o[n + 2] * a.z; v[n + 3] = o[n + 3] * a.w;
          }
          const bool odd = lane & 1;
#pragma unroll
          for (int i = 0; i < CW / 2; ++i) {
            const float rv = __shfl_xor_sync(0xffffffffu, odd ? v[i] : v[CW / 2 + i], 1);
            w[i] = odd ? pack_bf16x2(rv, v[CW / 2 + i]) : pack_bf16x2(v[i], rv);
          }
        }
        uint2 x[CW / 4];  // stage 1: 4 consecutive d of CW/4 columns
        {
          const bool hi = lane & 2;
#pragma unroll
          for (int i = 0; i < CW / 4; ++i) {
            const uint32_t rv = __shfl_xor_sync(0xffffffffu, hi ? w[i] : w[CW / 4 + i], 2);
            x[i] = hi ? make_uint2(rv, w[CW / 4 + i]) : make_uint2(w[i], rv);
          }
        }
        const bool hi4 = lane & 4;
        const int col_base = (lane & 1) * (CW / 2) + ((lane >> 1) & 1) * (CW / 4) + (hi4 ? CW / 8 : 0);
        const int d8 = blk * 128 + (r & ~7);
#pragma unroll
        for (int i = 0; i < CW / 8; ++i) {  // stage 2: 8 consecutive d of CW/8 columns -> one 16-B store each
          const uint32_t r0 = __shfl_xor_sync(0xffffffffu, hi4 ? x[i].x : x[CW / 8 + i].x, 4);
          const uint32_t r1 = __shfl_xor_sync(0xffffffffu, hi4 ? x[i].y : x[CW / 8 + i].y, 4);
          const uint4 y = hi4 ? make_uint4(r0, r1, x[CW / 8 + i].x, x[CW / 8 + i].y)
                              : make_uint4(x[i].x, x[i].y, r0, r1);
          const int n = col_base + i;
          if (n < e_ncols) {
            const size_t row = e_row0 + n + static_cast<size_t>((e_j0 + n) / p.g_q) * (p.H - p.g_q);
            *reinterpret_cast<uint4*>(p.out + row * C::D_V + d8) = y;
          }
        }
      } else {
        float* dst = p.o_part + (static_cast<size_t>(e_slot) * NQ + c0) * C::D_V + d;
#pragma unroll
        for (int n = 0; n < CW; n += 4) {
          const float4 a = ld_shared_f4(inv_addr + n * 4);
          if (n < e_ncols) dst[n * C::D_V] = o[n] * a.x;
          if (n + 1 < e_ncols) dst[(n + 1) * C::D_V] = o[n + 1] * a.y;
          if (n + 2 < e_ncols) dst[(n + 2) * C::D_V] = o[n + 2] * a.z;
          if (n + 3 < e_ncols) dst[(n + 3) * C::D_V] = o[n + 3] * a.w;
        }
      }
      ++e_blk;
    };
    int k = 0, u = 0, seg = 0, it = 0;
    Seg s;
    while (next_seg(k, u, s)) {
      // ---- segment setup: per-column visibility, running max reset
      if (r < CW) {
        const int n = c0 + r;
        int ve = 0;
        if (n < s.nq) {
          const int t = (s.n0 + n) / p.g_q;
          ve = p.causal ? max(0, min(s.L, s.L - p.Lq + t + 1)) : s.L;
        }
        vend_s[n] = ve;
        m_run[n] = -INFINITY;
        nm_s[n] = 0.f;
      }
      named_bar_sync(bar_id, 128);
      const int min_vend = p.causal ? max(0, min(s.L, s.L - p.Lq + s.n0 / p.g_q + 1)) : s.L;
      const bool all_cols = (s.nq == NQ);
      const uint32_t obuf = tmem + C::TMEM_O + (seg % C::NOB) * C::OCOLS;
      float l[HC];
#pragma unroll
      for (int n = 0; n < HC; ++n) l[n] = 0.f;

      for (int tl = s.t0; tl < s.t1; ++tl, ++it) {
        const int sb = it & 1;
        mbar_wait(&s_full[sb], (it >> 1) & 1);
        tc_fence_after();
        if (trace && threadIdx.x == 128 && it < kTraceTiles) trace[10 + 12 * it] = globaltimer();
        const int p0 = tl * T;
        const int tok = p0 + tr;
        const bool masked = !(p0 + T <= min_vend && all_cols);  // last tile / causal / padded columns
        // Raw scores q.k of this thread's token row, re-read from TMEM where
        // needed instead of kept live across the vote (S(sb) is released only
        // after it).  Rows >= T (warp-uniform) carry no token and skip it.
        const uint32_t vend_addr = smem_u32(vend_s + cb);
        auto load_x = [&](float (&x)[HC]) {
          tmem_load_s<C>(tmem + lane_addr + sb * NQ + c0, x);
          tmem_ld_wait();
          if (masked) {  // vend = 0 for padded columns
#pragma unroll
            for (int n = 0; n < HC; n += 4) {
              const float4 v = ld_shared_f4(vend_addr + n * 4);
              x[n] = tok < __float_as_int(v.x) ? x[n] : -INFINITY;
              x[n + 1] = tok < __float_as_int(v.y) ? x[n + 1] : -INFINITY;
              x[n + 2] = tok < __float_as_int(v.z) ? x[n + 2] : -INFINITY;
              x[n + 3] = tok < __float_as_int(v.w) ? x[n + 3] : -INFINITY;
            }
          }
        };
        // p = 2^(s*c - m) with the lagging running max m (nm = -m, 0 while m is
        // -inf so masked scores give exactly 0 without a select), packed to bf16.
        // Lazy rescale: the max is only moved when some p exceeds 2^TAU (checked
        // on the packed bf16 bits, which order like unsigned ints for p >= 0) or
        // on the first tile of a segment; then p is recomputed.
        uint32_t pk[HC / 2];
        auto exp_pack = [&](const float (&x)[HC]) {
#pragma unroll
          for (int n = 0; n < HC; n += 4) {
            const float4 m4 = ld_shared_f4(nm_addr + n * 4);
            const float2 e0 = ffma2(make_float2(x[n], x[n + 1]), make_float2(sl2, sl2), make_float2(m4.x, m4.y));
            const float2 e1 =
                ffma2(make_float2(x[n + 2], x[n + 3]), make_float2(sl2, sl2), make_float2(m4.z, m4.w));
            const __nv_bfloat162 v0 = __floats2bfloat162_rn(ex2(e0.x), ex2(e0.y));
            __nv_bfloat162 v1;
            if (GLAD_POLY_EVERY && ((n / 4) % GLAD_POLY_EVERY) == GLAD_POLY_EVERY - 1) {
              const float2 y = exp2_poly2(e1);  // part of the exponentials on the FMA pipe
              v1 = __floats2bfloat162_rn(y.x, y.y);
            } else {
              v1 = __floats2bfloat162_rn(ex2(e1.x), ex2(e1.y));
            }
            pk[n / 2] = *reinterpret_cast<const uint32_t*>(&v0);
            pk[n / 2 + 1] = *reinterpret_cast<const uint32_t*>(&v1);
          }
        };
        constexpr uint32_t kTrig = 0x4380u;  // bf16 bits of 2^TAU = 256
        static_assert(TAU == 8.f, "kTrig encodes 2^TAU");
        bool need = (tl == s.t0);
        if (row_ok) {
          float x[HC];
          load_x(x);
          exp_pack(x);
          uint32_t pmax = pk[0];
#pragma unroll
          for (int n = 1; n < HC / 2; ++n) pmax = max_u16x2(pmax, pk[n]);
          need |= ((pmax & 0xffffu) > kTrig) | ((pmax >> 16) > kTrig);
        }
        if (named_bar_red_or(bar_id, 128, need)) {
          // the running max moves by > 2^TAU somewhere: column max over the WG
          // (in pieces of <= 16 columns to bound register pressure)
          float x[HC];
          if (row_ok) {
            load_x(x);
          } else {
#pragma unroll
            for (int n = 0; n < HC; ++n) x[n] = -INFINITY;
          }
          constexpr int HW = HC > 16 ? 16 : HC;
#pragma unroll
          for (int h0 = 0; h0 < HC; h0 += HW) {
            float tmp[HW];
#pragma unroll
            for (int n = 0; n < HW; ++n) tmp[n] = x[h0 + n];
            const float cm = warp_col_reduce<HW, true, LANES>(tmp, lane);
            if ((lane & ((1 << col_shift<HW, LANES>()) - 1)) == 0)
              red[(wg * 4 + wq) * 32 + (cb - c0) + h0 + ((lane & (LANES - 1)) >> col_shift<HW, LANES>())] = cm;
          }
          named_bar_sync(bar_id, 128);
          if (r < CW) {
            const float* rr = red + wg * 128 + r;
            const float mt = fmaxf(fmaxf(rr[0], rr[32]), fmaxf(rr[64], rr[96])) * sl2;
            const float mo = m_run[c0 + r];
            const float mn = fmaxf(mo, mt);
            alpha_s[c0 + r] = (mn == -INFINITY) ? 1.f : ex2(mo - mn);
            m_run[c0 + r] = mn;
            nm_s[c0 + r] = (mn == -INFINITY) ? 0.f : -mn;
          }
          named_bar_sync(bar_id, 128);
          bool any_scale = false;
#pragma unroll
          for (int n = 0; n < CW; n += 4) {
            const float4 a = ld_shared_f4(ao_addr + n * 4);
            any_scale |= (a.x != 1.f) | (a.y != 1.f) | (a.z != 1.f) | (a.w != 1.f);
          }
#pragma unroll
          for (int n = 0; n < HC; n += 4) {
            const float4 a = ld_shared_f4(a_addr + n * 4);
            l[n] *= a.x; l[n + 1] *= a.y; l[n + 2] *= a.z; l[n + 3] *= a.w;
          }
          if (tl > s.t0 && any_scale) {  // rescale this WG's O^T columns in TMEM
            const int j = it - 1;
            mbar_wait(&pv_done[j & 3], (j >> 2) & 1);
            tc_fence_after();
#pragma unroll
            for (int blk = 0; blk < C::NBLK_O; ++blk) {
              float o[CW];
              const uint32_t ta = obuf + lane_addr + blk * NQ + c0;
              tmem_load_cols<C>(ta, o);
              tmem_ld_wait();
#pragma unroll
              for (int n = 0; n < CW; n += 4) {
                const float4 a = ld_shared_f4(ao_addr + n * 4);
                o[n] *= a.x; o[n + 1] *= a.y; o[n + 2] *= a.z; o[n + 3] *= a.w;
              }
              tmem_store_cols<C>(ta, o);
            }
            tmem_st_wait();
          }
          if (row_ok) {  // again: keeps x dead across the O^T rescale (register pressure)
            float x2[HC];
            load_x(x2);
            exp_pack(x2);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sb]);
        // row sum from the bf16-rounded p the PV multiplies (numerator and
        // denominator consistent; the fp32 sum failed the peaked parity case)
        if (row_ok) {
#pragma unroll
          for (int n = 0; n < HC; n += 2) {
            const float2 v =
                make_float2(__uint_as_float(pk[n / 2] << 16), __uint_as_float(pk[n / 2] & 0xffff0000u));
            const float2 acc = fadd2(make_float2(l[n], l[n + 1]), v);
            l[n] = acc.x;
            l[n + 1] = acc.y;
          }
        }
        // bf16 P^T into the tile's (now dead) RoPE chunk.  NQ = 64: MN-major
        // 128B-swizzled rows of 64 queries (token tr at tr*128, 16-B chunk j at
        // j ^ (tr & 7)); else no-swizzle core matrices [NQ/8][T tok][8].
        const uint32_t stage_base = sbase + (it % NS) * C::STAGE;
        const uint32_t pbase = stage_base + C::OFF_R;
        static_assert(HC % 8 == 0, "P^T rows are stored in 16-B pieces");
        if (row_ok) {
#pragma unroll
          for (int g = 0; g < HC / 8; ++g) {
            const int j = cb / 8 + g;
            const uint32_t pa =
                C::P_SW128 ? pbase + tr * 128 + ((j ^ (tr & 7)) << 4) : pbase + j * (T * 16) + tr * 16;
            st_shared_v4(pa, pk[g * 4], pk[g * 4 + 1], pk[g * 4 + 2], pk[g * 4 + 3]);
          }
        }
        if (wg == 0 && row_ok && tok >= s.kv_end) {  // never-visible rows: zero V (0 * garbage != NaN)
          const uint32_t kvrow = stage_base + (tr >> 3) * C::LGRP + (tr & 7) * 128;
#pragma unroll
          for (int ch = 0; ch < C::NCH_V; ++ch)
#pragma unroll
            for (int uu = 0; uu < 8; ++uu) st_shared_v4(kvrow + C::chunk_off(ch) + uu * 16, 0u, 0u, 0u, 0u);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[it % NS]);
        if (trace && threadIdx.x == 128 && it < kTraceTiles) trace[11 + 12 * it] = globaltimer();
        if (trace && threadIdx.x == 256 && it < kTraceTiles) trace[14 + 12 * it] = globaltimer();
        if (e_blk < C::NBLK_O) epi_block();  // the previous segment's O, one block per tile
      }

      // ------------------------------------------------------- segment epilogue
      while (e_blk < C::NBLK_O) epi_block();  // (a segment shorter than NBLK_O tiles)
      const float cs = warp_col_reduce<HC, false, LANES>(l, lane);
      if ((lane & ((1 << col_shift<HC, LANES>()) - 1)) == 0)
        red[(wg * 4 + wq) * 32 + (cb - c0) + ((lane & (LANES - 1)) >> col_shift<HC, LANES>())] = cs;
      named_bar_sync(bar_id, 128);
      // partial slot: 2 per range — the range's first segment (2c) or its
      // last one (2c + 1); only those two can be cut by a range boundary
      const int slot = (2 * (cta / p.cl_n) + (seg == 0 ? 0 : 1)) * p.cl_n + cta % p.cl_n;
      if (r < CW) {  // fold the row sum into alpha_s as 1/l (reused below) and write lse
        const float* rr = red + wg * 128 + r;
        const float ls = (rr[0] + rr[32]) + (rr[64] + rr[96]);
        alpha_s[c0 + r] = ls > 0.f ? 1.f / ls : 0.f;
        if (c0 + r < s.nq) {
          const float lse = ls > 0.f ? (m_run[c0 + r] + __log2f(ls)) * 0.69314718055994531f : -INFINITY;
          if (s.whole) {
            const int ng = s.n0 + c0 + r, t = ng / p.g_q, h = s.head * p.g_q + (ng - t * p.g_q);
            p.lse[(static_cast<size_t>(s.b) * p.Lq + t) * p.H + h] = lse;
          } else {
            p.lse_part[static_cast<size_t>(slot) * NQ + c0 + r] = lse;
          }
        }
      }
      // pending epilogue of this segment: 1/l to einv_s, output addressing
      // (whole units: the output row of column c0; rows advance by one within
      // a query position's g_q heads and jump to the next position's row
      // block after g_q columns, no per-element division)
      if (r < CW) einv_s[(seg % C::NOB) * NQ + c0 + r] = alpha_s[c0 + r];
      e_blk = 0;
      e_seg = seg;
      e_j = it - 1;  // last tile of this segment
      e_whole = s.whole;
      e_slot = slot;
      e_ncols = min(CW, s.nq - c0);
      e_j0 = 0;
      e_row0 = 0;
      if (s.whole) {
        const int ng = s.n0 + c0, t = ng / p.g_q;
        e_j0 = ng - t * p.g_q;
        e_row0 = (static_cast<size_t>(s.b) * p.Lq + t) * p.H + s.head * p.g_q + e_j0;
      }
      named_bar_sync(bar_id, 128);  // alpha_s / m_run / einv_s settled before the next segment resets them
      // one O buffer (MLA): the next segment's first PV needs it, write it now
      if constexpr (C::NOB == 1) {
        while (e_blk < C::NBLK_O) epi_block();
      }
      if (trace && threadIdx.x == 128 && it - 1 < kTraceTiles) trace[15 + 12 * (it - 1)] = globaltimer();
      ++seg;
    }
    while (e_blk < C::NBLK_O) epi_block();  // the last segment's O
  }

  tc_fence_before();
  __syncthreads();
  if (p.cl_n > 1) cluster_sync();  // no CTA leaves while a peer may still signal it
  if (trace && threadIdx.x == 0) trace[2] = globaltimer();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

}  // namespace glad
