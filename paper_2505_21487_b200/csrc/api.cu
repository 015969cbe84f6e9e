// C ABI of libglad (include/glad.h): argument validation, TMA descriptor
// encoding, split planning and launches.  Host-only logic; every step of the
// compute path runs in the kernels of decode.cuh / aux_kernels.cu.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <tuple>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/glad.h"
#include "internal.h"

#ifndef GLAD_SEG_COST
#define GLAD_SEG_COST 0
#endif
#ifndef GLAD_SEG_COST_ROWS
#define GLAD_SEG_COST_ROWS 12  // rows mode, d_v >= 256
#endif
#ifndef GLAD_SEG_COST_ROWS128
#define GLAD_SEG_COST_ROWS128 4  // rows mode, d_v = 128
#endif
#ifndef GLAD_MIN_GROUP_CTAS
#define GLAD_MIN_GROUP_CTAS 8
#endif

namespace {

thread_local char g_err[512] = "no error";
uint64_t* g_trace = nullptr;  // debug timeline buffer (glad_debug_set_trace)
int g_phase_mask = 7;         // debug: which of plan(1) / decode(2) / merge(4) to launch

glad_status fail(glad_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }
int ilog2(int x) {
  int r = 0;
  while ((1 << r) < x) ++r;
  return r;
}
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() { return glad::tensor_map_encoder(); }

glad_status check_layout(const glad_cache_layout* L) {
  if (!L) return fail(GLAD_ERR_INVALID_ARG, "layout is NULL");
  if (L->num_pages < 1) return fail(GLAD_ERR_INVALID_ARG, "layout.num_pages=%d must be >= 1", L->num_pages);
  if (!is_pow2(L->page_size))
    return fail(GLAD_ERR_INVALID_ARG, "layout.page_size=%d must be a power of two >= 1", L->page_size);
  if (L->n_heads_kv < 1 || L->d_head < 8 || L->d_rope < 0 || L->d_head % 8 || L->d_rope % 8)
    return fail(GLAD_ERR_INVALID_ARG, "layout dims n_heads_kv=%d d_head=%d d_rope=%d invalid", L->n_heads_kv,
                L->d_head, L->d_rope);
  const int64_t w = static_cast<int64_t>(L->n_heads_kv) * L->d_head + L->d_rope;
  if (L->row_stride < w || L->row_stride % 8)
    return fail(GLAD_ERR_INVALID_ARG, "layout.row_stride=%lld must be >= %lld and a multiple of 8",
                static_cast<long long>(L->row_stride), static_cast<long long>(w));
  if (static_cast<int64_t>(L->num_pages) * L->page_size >= (int64_t(1) << 31))
    return fail(GLAD_ERR_INVALID_ARG, "pool has >= 2^31 rows");
  return GLAD_OK;
}

int64_t row_width(const glad_cache_layout* L) {
  return static_cast<int64_t>(L->n_heads_kv) * L->d_head + L->d_rope;
}

// kMAT: materialised prefill rows [K_h | V_h] per query head (glad_gla_prefill)
enum Variant { kGLA, kMLA, kGTA, kMAT };

int g_tile_override = 0;  // debug: force 64 / 96 / 128-token tiles (glad_debug_set_tile)

// KV tile height.  128 is the default: 96-token tiles (three GLA-2 stages)
// and 64-token tiles (four) shorten the refill chain but spend more QK tensor
// work and per-tile softmax overhead per token, and measured no faster on any
// BASELINE shape (C2 0.300 / 0.287 ms at T = 96 / 128, C5 equal, MLA 0.62 /
// 0.61 ms at T = 64 / 128).  The others stay available (and tested) through
// glad_debug_set_tile.
int tile_tokens(const glad::DecodeKey& k0) {
  glad::DecodeKey k = k0;
  if (k.nq == 128) {  // rows mode: no 128-token tiles; the largest tile with three KV stages
    if (g_tile_override == 64 || g_tile_override == 96 || g_tile_override == 128) {
      k.t = g_tile_override == 64 ? 64 : 96;
      if (glad::decode_stages(k) >= 1) return k.t;
    }
    for (int t : {96, 64}) {
      k.t = t;
      if (glad::decode_stages(k) >= 3) return t;
    }
    return 64;
  }
  if (g_tile_override == 64 || g_tile_override == 96 || g_tile_override == 128) return g_tile_override;
  k.t = 128;
  // MLA (144 KB tiles) fits one 128-token stage: split into lo / hi halves it
  // still overlaps the refill with PV (C2 MLA 0.572 -> 0.489 ms against two
  // unsplit 64-token stages)
  if (glad::decode_stages(k) >= 2 || (glad::decode_stages(k) >= 1 && glad::decode_split(k))) return 128;
  return 64;
}

// Resident clusters per (kernel, cluster size), queried once.
int max_clusters(const glad::DecodeKey& k, int cl_n) {
  static std::map<std::tuple<int, int, int, int, int, int>, int> cache;
  const auto key = std::make_tuple(k.d_v, k.d_kn, k.d_r, k.nq, k.t * 4096 + k.d_s, cl_n);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const int n = glad::decode_max_clusters(k, cl_n);
  cache[key] = n;
  return n;
}

struct DecodeGeom {
  glad::DecodeKey key;
  int g_q, n_qblk;
};

glad_status decode_geom(Variant v, const glad_cache_layout* L, int32_t Lq, int32_t H, DecodeGeom* g) {
  glad_status s = check_layout(L);
  if (s != GLAD_OK) return s;
  if (Lq < 1) return fail(GLAD_ERR_INVALID_ARG, "Lq=%d must be >= 1", Lq);
  if (H < 1 || H % L->n_heads_kv)
    return fail(GLAD_ERR_INVALID_ARG, "H=%d must be a positive multiple of n_heads_kv=%d", H, L->n_heads_kv);
  if (v == kMLA && L->n_heads_kv != 1)
    return fail(GLAD_ERR_INVALID_ARG, "MLA requires n_heads_kv == 1 (got %d)", L->n_heads_kv);
  if (v == kGTA && L->d_rope * 2 != L->d_head)
    return fail(GLAD_ERR_INVALID_ARG, "GTA requires d_rope == d_head/2 (got d_head=%d d_rope=%d)", L->d_head,
                L->d_rope);
  if (v == kMAT && (L->d_head % 128 || H != L->n_heads_kv))
    return fail(GLAD_ERR_INVALID_ARG, "materialised rows need d_head = 2 d_h and one query head per KV head");
  g->g_q = H / L->n_heads_kv;
  g->key.d_s = L->d_head;
  g->key.d_v = (v == kMAT) ? L->d_head / 2 : L->d_head;
  g->key.d_kn = (v == kGTA || v == kMAT) ? L->d_head / 2 : L->d_head;
  g->key.d_r = L->d_rope;
  const int64_t nq_total = static_cast<int64_t>(Lq) * g->g_q;
  const int maxnq = glad::decode_max_nq(L->d_head);
  g->key.nq = nq_total <= 16 ? 16 : nq_total <= 32 ? 32 : maxnq;
  // More than 64 query rows per head (q_len >= 2 with g_q = 64):
  // rows mode, one CTA per 128 rows reads each KV tile once for all of them
  // (glad_debug_set_phase_mask bit 16 turns it off for A/B runs).
  glad::DecodeKey kr = g->key;
  kr.nq = 128;
  if (nq_total > 64 && !(g_phase_mask & 16) && glad::decode_rows_supported(kr)) g->key.nq = 128;
  if (v == kMAT) g->key.nq = 128;  // materialised rows: rows mode only (shorter prompts pad the block)
  g->key.t = tile_tokens(g->key);
  g->n_qblk = static_cast<int>((nq_total + g->key.nq - 1) / g->key.nq);
  if (!glad::decode_supported(g->key))
    return fail(GLAD_ERR_UNSUPPORTED, "no decode kernel for d_head=%d d_rope=%d (variant %d, rows/CTA %d)",
                L->d_head, L->d_rope, static_cast<int>(v), g->key.nq);
  if (static_cast<int64_t>(L->n_heads_kv) * g->n_qblk > 65535)
    return fail(GLAD_ERR_UNSUPPORTED, "too many head blocks");
  return GLAD_OK;
}

// Workspace of one decode call: [plan (U+1) int32][lse_part 2G*NQ f32]
// [o_part 2G*NQ*D_V f32] (two partial slots per CTA range), each 256-byte aligned.
struct WsLayout {
  size_t plan, lse, opart, total;
};
WsLayout ws_layout(int64_t U, int64_t G, int nq, int d_v) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  WsLayout w;
  w.plan = 0;
  w.lse = al(static_cast<size_t>(U + 1) * 4);
  w.opart = w.lse + al(static_cast<size_t>(2 * G) * nq * 4);
  w.total = w.opart + al(static_cast<size_t>(2 * G) * nq * d_v * 4);
  return w;
}

glad_status decode_common(Variant v, const void* q, const void* pool, const glad_cache_layout* L,
                          const int32_t* block_table, int32_t bt_stride, const int32_t* seqlens, int32_t B,
                          int32_t Lq, int32_t H, float scale, int32_t causal, void* out, float* lse, void* ws,
                          size_t ws_bytes, int32_t num_ctas, void* stream) {
  DecodeGeom g;
  glad_status s = decode_geom(v, L, Lq, H, &g);
  if (s != GLAD_OK) return s;
  if (B < 0) return fail(GLAD_ERR_INVALID_ARG, "B=%d < 0", B);
  if (B == 0) return GLAD_OK;
  if (!q || !pool || !block_table || !seqlens || !out || !lse)
    return fail(GLAD_ERR_INVALID_ARG, "NULL tensor pointer (q=%p pool=%p bt=%p seqlens=%p out=%p lse=%p)", q,
                pool, block_table, seqlens, out, lse);
  if (!aligned16(q) || !aligned16(pool) || !aligned16(out))
    return fail(GLAD_ERR_INVALID_ARG, "q, pool and out must be 16-byte aligned");
  if (bt_stride < 1) return fail(GLAD_ERR_INVALID_ARG, "bt_stride=%d < 1", bt_stride);
  if (!(scale > 0.f) || !std::isfinite(scale))
    return fail(GLAD_ERR_INVALID_ARG, "softmax_scale=%g must be finite and > 0", scale);
  if (num_ctas < 0) return fail(GLAD_ERR_INVALID_ARG, "num_ctas=%d < 0", num_ctas);
  const int64_t U = static_cast<int64_t>(B) * L->n_heads_kv * g.n_qblk;
  if (U >= (int64_t(1) << 30)) return fail(GLAD_ERR_UNSUPPORTED, "too many work units (%lld)", (long long)U);
  const int G0 = num_ctas > 0 ? num_ctas : num_sms();
  // Several query blocks per (head, sequence) (q_len >= 2, MLA): optionally
  // (glad_debug_set_phase_mask bit 8) a cluster of one CTA per block shares
  // every KV tile through TMA multicast, so the tile is read from HBM once
  // instead of once per block.  Measured: DRAM bytes halve (C3 q_len 2: 1.23
  // -> 0.66 GB) but the step is 5-15 % slower — these shapes are bound by the
  // per-tile QK/softmax/PV chain, not by HBM, and the cluster-wide stage
  // handshake lengthens that chain.  Off by default.
  int cl_n = 1;
  if (g.n_qblk >= 2 && g.n_qblk <= 8 && L->page_size >= 16 && (g_phase_mask & 8) && g.key.nq != 128 &&
      (num_ctas == 0 || num_ctas % g.n_qblk == 0)) {
    cl_n = g.n_qblk;
    if (max_clusters(g.key, cl_n) < 1) cl_n = 1;
  }
  // Ranges (one per CTA, or per cluster): one equal group per KV head when
  // there are enough, so the heads of a sequence advance in lockstep and
  // their shared RoPE rows hit L2.  Several query blocks per unit (MLA's two
  // 64-head blocks, q_len >= 2) without clusters: one group per (head, query
  // block) instead (qb_outer unit order), so the blocks reading the same KV
  // tiles run at the same time and the tiles come from HBM once (C2 MLA:
  // ncu DRAM 2.0x -> ~1x algorithmic); skipped when the groups would get
  // fewer than 16 CTAs each (prefill's many query blocks) or with phase-mask
  // bit 128 (A/B).
  int R0 = G0 / cl_n;
  if (cl_n > 1 && num_ctas == 0) R0 = std::min(R0, max_clusters(g.key, cl_n));
  int qb_outer = 0, n_groups = 0;
  const int64_t ngq = static_cast<int64_t>(L->n_heads_kv) * g.n_qblk;
  if (cl_n == 1 && g.n_qblk > 1 && !(g_phase_mask & 128) && ngq <= 16 && R0 >= 16 * ngq) {
    qb_outer = 1;
    n_groups = static_cast<int>(ngq);
  } else if (L->n_heads_kv > 1 && L->n_heads_kv <= glad::kMaxGroups && R0 >= GLAD_MIN_GROUP_CTAS * L->n_heads_kv) {
    // (not with fewer than GLAD_MIN_GROUP_CTAS CTAs per head: the
    // materialised prefill's 128 "heads" would leave 20 of 148 SMs idle)
    n_groups = L->n_heads_kv;
  }
  const int R = n_groups > 1 ? (R0 / n_groups) * n_groups : R0;
  const int G = R * cl_n;
  const int64_t n_plan = U / cl_n;  // plan entries: units, or (head, sequence) groups
  const WsLayout wl = ws_layout(U, G, g.key.nq, g.key.d_v);
  if (ws == nullptr || ws_bytes < wl.total)
    return fail(GLAD_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, wl.total);
  if (reinterpret_cast<uintptr_t>(ws) & 255u) return fail(GLAD_ERR_INVALID_ARG, "workspace must be 256-byte aligned");

  auto enc = encode_fn();
  if (!enc) return fail(GLAD_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  CUtensorMap tmap;
  // page runs inside a tile: a page never crosses a tile edge when T is a
  // multiple of the page or vice versa; T = 96 with pages >= 32 uses 32-row boxes
  int box_rows = L->page_size;
  while (g.key.t % box_rows) box_rows >>= 1;  // gcd(page, T) (pages are powers of two)
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(row_width(L)),
                        static_cast<cuuint64_t>(L->num_pages) * static_cast<cuuint64_t>(L->page_size)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(L->row_stride) * 2};
  cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1u, 1u};
  // (L2 promotion none/128B/256B measured identical DRAM bytes and time)
  const CUtensorMapL2promotion pr = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUresult cr = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(GLAD_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(cr));
  // The latent slice of a page run as ONE box: the pool viewed as
  // [row group of 8][64-col chunk][8 rows][64 cols], box (64, 8, NCH_V,
  // box_rows / 8) -> smem [group][chunk][8 rows][128 B], the interleaved
  // K-major atom layout the kernel's descriptors expect.
  CUtensorMap lmap;
  std::memset(&lmap, 0, sizeof(lmap));
  // pages shorter than 16 tokens: TMA gather4 (4 token rows per instruction)
  // unless glad_debug_set_phase_mask bit 32 selects the cooperative cp.async
  // producer; lmap is then the row map (box 64 cols x 1 row, 128B swizzle)
  const bool g4 = L->page_size < 16 && !(g_phase_mask & 32);
  if (g4) {
    cuuint64_t gd[2] = {static_cast<cuuint64_t>(row_width(L)),
                        static_cast<cuuint64_t>(L->num_pages) * static_cast<cuuint64_t>(L->page_size)};
    cuuint64_t gs[1] = {static_cast<cuuint64_t>(L->row_stride) * 2};
    cuuint32_t gb[2] = {64u, 1u};
    cuuint32_t ge[2] = {1u, 1u};
    cr = enc(&lmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool), gd, gs, gb, ge,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS)
      return fail(GLAD_ERR_CUDA, "cuTensorMapEncodeTiled (gather4 rows) failed (%d)", static_cast<int>(cr));
  } else if (L->page_size >= 16) {
    const cuuint64_t rs = static_cast<cuuint64_t>(L->row_stride) * 2;
    cuuint64_t ld[4] = {64u, 8u, static_cast<cuuint64_t>(L->n_heads_kv) * L->d_head / 64,
                        static_cast<cuuint64_t>(L->num_pages) * static_cast<cuuint64_t>(L->page_size) / 8};
    cuuint64_t ls[3] = {rs, 128u, 8u * rs};
    // split stages (swap-AB, DecodeCfg::SPLIT): one box per latent half
    const int box_chunks = glad::decode_split(g.key) ? g.key.d_s / 128 : g.key.d_s / 64;
    cuuint32_t lbx[4] = {64u, 8u, static_cast<cuuint32_t>(box_chunks), static_cast<cuuint32_t>(box_rows / 8)};
    cuuint32_t le[4] = {1u, 1u, 1u, 1u};
    cr = enc(&lmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(pool), ld, ls, lbx, le,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS)
      return fail(GLAD_ERR_CUDA, "cuTensorMapEncodeTiled (latent boxes) failed (%d)", static_cast<int>(cr));
  }

  // Q as a 3-D tensor [B*Lq][H][d_qk]: a unit's NQ query rows are one box
  // (64 cols, g_q heads, NQ/g_q positions) or (64 cols, NQ heads, 1).
  const int dq = g.key.d_kn + g.key.d_r;
  int q_box_h = 0, q_box_t = 0;
  if (g.g_q % g.key.nq == 0) { q_box_h = g.key.nq; q_box_t = 1; }
  else if (g.key.nq % g.g_q == 0) { q_box_h = g.g_q; q_box_t = g.key.nq / g.g_q; }
  CUtensorMap qmap;
  std::memset(&qmap, 0, sizeof(qmap));
  bool q_tma = q_box_h > 0 && q_box_h <= 256 && q_box_t <= 256 && (reinterpret_cast<uintptr_t>(q) & 15u) == 0;
  if (q_tma) {
    cuuint64_t qd[3] = {static_cast<cuuint64_t>(dq), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(B) * static_cast<cuuint64_t>(Lq)};
    cuuint64_t qs[2] = {static_cast<cuuint64_t>(dq) * 2, static_cast<cuuint64_t>(H) * dq * 2};
    cuuint32_t qbx[3] = {64u, static_cast<cuuint32_t>(q_box_h), static_cast<cuuint32_t>(q_box_t)};
    cuuint32_t qe[3] = {1u, 1u, 1u};
    q_tma = enc(&qmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(q), qd, qs, qbx, qe,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }

  char* wsb = static_cast<char*>(ws);
  glad::DecodeParams p;
  p.q_tma = q_tma ? 1 : 0;
  p.pool = static_cast<const __nv_bfloat16*>(pool);
  p.row_stride = L->row_stride;
  // pages shorter than 16 tokens: one TMA per page run per chunk costs ~100
  // cycles of issue each; the cooperative cp.async producer wins (measured)
  p.cp_kv = (L->page_size < 16 && !g4) ? 1 : 0;
  p.g4 = g4 ? ((g_phase_mask & 256) ? 1 : 2) : 0;  // bit 256: gather4 alone (no LSU rows)
  p.n_groups = n_groups;
  // segment-switch cost in virtual tiles, so that the ranges balance work +
  // switches (trace: ~2.5 tiles per switch in swap-AB, ~9 in rows mode at
  // d_v = 256).  A/B decode ms over rows-mode costs 0 / 4 / 6 / 9 / 12: C3
  // q_len 2 0.173 / 0.172 / 0.172 / 0.170 / 0.170, absorbed prefill (d_v 256)
  // - / 3.25 / 2.84 / 2.49 / 2.46, GTA prefill (d_v 128, cheaper tiles and
  // switches) - / 0.819 / 0.843 / 0.878 / 0.907, materialised prefill flat;
  // swap-AB 0 / 2 / 3: C2 equal, C5 TP8 shard -2 % at 2, C2 page 1 +1 %.
  p.seg_cost = g.key.nq != 128 ? GLAD_SEG_COST : (g.key.d_v >= 256 ? GLAD_SEG_COST_ROWS : GLAD_SEG_COST_ROWS128);
  p.qb_outer = qb_outer;
  p.q_box_h = q_box_h;
  p.q_box_t = q_box_t;
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.block_table = block_table;
  p.seqlens = seqlens;
  p.plan = reinterpret_cast<const int32_t*>(wsb + wl.plan);
  p.out = static_cast<__nv_bfloat16*>(out);
  p.lse = lse;
  p.o_part = reinterpret_cast<float*>(wsb + wl.opart);
  p.lse_part = reinterpret_cast<float*>(wsb + wl.lse);
  p.bt_stride = bt_stride;
  p.B = B;
  p.Lq = Lq;
  p.H = H;
  p.g_q = g.g_q;
  p.n_heads_kv = L->n_heads_kv;
  p.d_head = L->d_head;
  p.rope_col = L->n_heads_kv * L->d_head;
  p.page_size = L->page_size;
  p.log2_page = ilog2(L->page_size);
  p.box_rows = box_rows;
  p.n_qblk = g.n_qblk;
  p.n_units = static_cast<int32_t>(n_plan);
  p.causal = causal ? 1 : 0;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.trace = g_trace;
  p.dbg_load_only = (g_phase_mask & 64) ? 1 : 0;
  p.cl_n = cl_n;

  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t* plan = reinterpret_cast<int32_t*>(wsb + wl.plan);
  cudaError_t e = cudaSuccess;
  if (g_phase_mask & 1) {
    e = glad::launch_plan(seqlens, plan, p.n_units, p.seg_cost, cl_n, B, g.key.t, g.n_qblk, qb_outer, g.key.nq, Lq, g.g_q, p.causal, H,
                          g.key.d_v, out, lse, nullptr, st);
    if (e != cudaSuccess) return fail(GLAD_ERR_CUDA, "plan launch failed: %s", cudaGetErrorString(e));
  }
  if (g_phase_mask & 2) {
    e = glad::launch_decode(g.key, tmap, lmap, qmap, p, G, st);
    if (e != cudaSuccess) return fail(GLAD_ERR_CUDA, "decode launch failed: %s", cudaGetErrorString(e));
  }
  if (g_phase_mask & 4) {
    e = glad::launch_merge_split(plan, p.o_part, p.lse_part, G, cl_n, p.n_units, g.key.nq, g.n_qblk, qb_outer, B,
                                 n_groups, g.g_q, Lq, H, g.key.d_v, p.seg_cost, out, lse, st);
    if (e != cudaSuccess) return fail(GLAD_ERR_CUDA, "merge launch failed: %s", cudaGetErrorString(e));
  }
  return GLAD_OK;
}

}  // namespace

extern "C" {

const char* glad_last_error(void) { return g_err; }

const char* glad_version(void) { return "glad 0.1.0 sm_100a"; }

void glad_debug_set_trace(void* device_buf) { g_trace = static_cast<uint64_t*>(device_buf); }

void glad_debug_set_phase_mask(int32_t mask) { g_phase_mask = mask & 511; }

void glad_debug_set_tile(int32_t tokens) { g_tile_override = tokens; }

size_t glad_pool_bytes(const glad_cache_layout* L) {
  if (check_layout(L) != GLAD_OK) return 0;
  return static_cast<size_t>(L->num_pages) * L->page_size * static_cast<size_t>(L->row_stride) * 2;
}

glad_status glad_cache_append(const glad_cache_layout* L, void* pool, const int32_t* block_table, int32_t bt_stride,
                              const int32_t* seqlens_before, const void* rows, int32_t B, int32_t n_new,
                              void* stream) {
  glad_status s = check_layout(L);
  if (s != GLAD_OK) return s;
  if (B < 0 || n_new < 0) return fail(GLAD_ERR_INVALID_ARG, "B=%d n_new=%d must be >= 0", B, n_new);
  if (B == 0 || n_new == 0) return GLAD_OK;
  if (!pool || !block_table || !seqlens_before || !rows) return fail(GLAD_ERR_INVALID_ARG, "NULL pointer");
  if (!aligned16(pool) || !aligned16(rows)) return fail(GLAD_ERR_INVALID_ARG, "pool/rows must be 16-byte aligned");
  if (bt_stride < 1) return fail(GLAD_ERR_INVALID_ARG, "bt_stride=%d < 1", bt_stride);
  cudaError_t e = glad::launch_append(pool, L->row_stride, L->page_size, block_table, bt_stride, seqlens_before,
                                      rows, B, n_new, static_cast<int32_t>(row_width(L)),
                                      static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(GLAD_ERR_CUDA, "append launch failed: %s", cudaGetErrorString(e));
  return GLAD_OK;
}

glad_status glad_paged_gather(const glad_cache_layout* L, const void* pool, const int32_t* block_table,
                              int32_t bt_stride, const int32_t* seqlens, int32_t B, int32_t max_len, void* dense_out,
                              void* stream) {
  glad_status s = check_layout(L);
  if (s != GLAD_OK) return s;
  if (B < 0 || max_len < 0) return fail(GLAD_ERR_INVALID_ARG, "B=%d max_len=%d must be >= 0", B, max_len);
  if (B == 0 || max_len == 0) return GLAD_OK;
  if (!pool || !block_table || !seqlens || !dense_out) return fail(GLAD_ERR_INVALID_ARG, "NULL pointer");
  if (!aligned16(pool) || !aligned16(dense_out))
    return fail(GLAD_ERR_INVALID_ARG, "pool/dense_out must be 16-byte aligned");
  cudaError_t e = glad::launch_gather(pool, L->row_stride, L->page_size, block_table, bt_stride, seqlens, B, max_len,
                                      static_cast<int32_t>(row_width(L)), dense_out,
                                      static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(GLAD_ERR_CUDA, "gather launch failed: %s", cudaGetErrorString(e));
  return GLAD_OK;
}

size_t glad_decode_workspace_bytes(const glad_cache_layout* L, int32_t B, int32_t Lq, int32_t H, int32_t variant,
                                   int32_t num_ctas) {
  DecodeGeom g;
  Variant v = variant == GLAD_GTA ? kGTA : variant == GLAD_MLA ? kMLA : kGLA;
  if (B <= 0 || decode_geom(v, L, Lq, H, &g) != GLAD_OK) return 0;
  const int64_t U = static_cast<int64_t>(B) * L->n_heads_kv * g.n_qblk;
  const int G = num_ctas > 0 ? num_ctas : num_sms();
  return ws_layout(U, G, g.key.nq, g.key.d_v).total;
}

glad_status glad_gla_decode(const void* q, const void* pool, const glad_cache_layout* layout,
                            const int32_t* block_table, int32_t bt_stride, const int32_t* seqlens, int32_t B,
                            int32_t Lq, int32_t H, float softmax_scale, int32_t causal, void* out, float* lse,
                            void* workspace, size_t ws_bytes, int32_t num_ctas, void* stream) {
  return decode_common(kGLA, q, pool, layout, block_table, bt_stride, seqlens, B, Lq, H, softmax_scale, causal, out,
                       lse, workspace, ws_bytes, num_ctas, stream);
}

glad_status glad_mla_decode(const void* q, const void* pool, const glad_cache_layout* layout,
                            const int32_t* block_table, int32_t bt_stride, const int32_t* seqlens, int32_t B,
                            int32_t Lq, int32_t H, float softmax_scale, int32_t causal, void* out, float* lse,
                            void* workspace, size_t ws_bytes, int32_t num_ctas, void* stream) {
  return decode_common(kMLA, q, pool, layout, block_table, bt_stride, seqlens, B, Lq, H, softmax_scale, causal, out,
                       lse, workspace, ws_bytes, num_ctas, stream);
}

glad_status glad_gta_decode(const void* q, const void* pool, const glad_cache_layout* layout,
                            const int32_t* block_table, int32_t bt_stride, const int32_t* seqlens, int32_t B,
                            int32_t Lq, int32_t H, float softmax_scale, int32_t causal, void* out, float* lse,
                            void* workspace, size_t ws_bytes, int32_t num_ctas, void* stream) {
  return decode_common(kGTA, q, pool, layout, block_table, bt_stride, seqlens, B, Lq, H, softmax_scale, causal, out,
                       lse, workspace, ws_bytes, num_ctas, stream);
}

glad_status glad_splitkv_combine(const float* o_part, const float* lse_part, int32_t S, int32_t B, int32_t Lq,
                                 int32_t H, int32_t d_v, void* out, float* lse, void* stream) {
  if (S < 1 || B < 0 || Lq < 1 || H < 1 || d_v < 8 || d_v % 8)
    return fail(GLAD_ERR_INVALID_ARG, "combine dims S=%d B=%d Lq=%d H=%d d_v=%d invalid", S, B, Lq, H, d_v);
  if (B == 0) return GLAD_OK;
  if (!o_part || !lse_part || !out || !lse) return fail(GLAD_ERR_INVALID_ARG, "NULL pointer");
  if (!aligned16(o_part) || !aligned16(out)) return fail(GLAD_ERR_INVALID_ARG, "o_part/out must be 16-byte aligned");
  cudaError_t e = glad::launch_combine(o_part, lse_part, S, static_cast<int64_t>(B) * Lq * H, d_v, out, lse,
                                       static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(GLAD_ERR_CUDA, "combine launch failed: %s", cudaGetErrorString(e));
  return GLAD_OK;
}

glad_status glad_gla_absorb_query(const void* q_nope, const void* q_pe, const void* w_uk, const int32_t* seqlens,
                                  int32_t B, int32_t Lq, int32_t H, int32_t d_h, int32_t d_c, int32_t d_rope,
                                  float rope_base, void* q_out, void* stream) {
  if (B < 0 || Lq < 1 || H < 1 || d_rope < 2 || d_rope % 2 || !(rope_base > 1.f))
    return fail(GLAD_ERR_INVALID_ARG, "absorb B=%d Lq=%d H=%d d_rope=%d base=%g invalid", B, Lq, H, d_rope, rope_base);
  if (!glad::absorb_supported(d_h, d_c))
    return fail(GLAD_ERR_UNSUPPORTED, "absorb: no kernel for d_h=%d d_c=%d", d_h, d_c);
  if (B == 0) return GLAD_OK;
  if (!q_nope || !q_pe || !w_uk || !seqlens || !q_out) return fail(GLAD_ERR_INVALID_ARG, "NULL pointer");
  if (d_rope % 8) return fail(GLAD_ERR_INVALID_ARG, "absorb: d_rope=%d must be a multiple of 8", d_rope);
  if (!aligned16(q_nope) || !aligned16(w_uk) || !aligned16(q_out) || (reinterpret_cast<uintptr_t>(q_pe) & 3u))
    return fail(GLAD_ERR_INVALID_ARG, "q_nope / w_uk / q_out must be 16-byte aligned, q_pe 4-byte aligned");
  cudaError_t e = glad::launch_absorb_query(q_nope, q_pe, w_uk, seqlens, B, Lq, H, d_h, d_c, d_rope, rope_base, q_out,
                                            static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(GLAD_ERR_CUDA, "absorb launch failed: %s", cudaGetErrorString(e));
  return GLAD_OK;
}

glad_status glad_cache_append_rope(const glad_cache_layout* layout, void* pool, const int32_t* block_table,
                                   int32_t bt_stride, const int32_t* seqlens_before, const void* latent,
                                   const void* k_pe, int32_t B, int32_t n_new, float rope_base, void* stream) {
  glad_status st = check_layout(layout);
  if (st != GLAD_OK) return st;
  if (B < 0 || n_new < 0 || bt_stride < 1 || !(rope_base > 1.f))
    return fail(GLAD_ERR_INVALID_ARG, "append_rope B=%d n_new=%d bt_stride=%d invalid", B, n_new, bt_stride);
  if (layout->d_rope % 2) return fail(GLAD_ERR_INVALID_ARG, "d_rope=%d must be even", layout->d_rope);
  if (B == 0 || n_new == 0) return GLAD_OK;
  if (!pool || !block_table || !seqlens_before || !latent || !k_pe) return fail(GLAD_ERR_INVALID_ARG, "NULL pointer");
  const int w_lat = layout->n_heads_kv * layout->d_head;
  if (w_lat % 8 || !aligned16(pool) || !aligned16(latent) || (reinterpret_cast<uintptr_t>(k_pe) & 3u))
    return fail(GLAD_ERR_INVALID_ARG, "latent width %% 8, pool / latent 16-byte and k_pe 4-byte alignment required");
  cudaError_t e = glad::launch_append_rope(pool, layout->row_stride, layout->page_size, block_table, bt_stride,
                                           seqlens_before, latent, k_pe, B, n_new, w_lat, layout->d_rope, rope_base,
                                           static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(GLAD_ERR_CUDA, "append_rope launch failed: %s", cudaGetErrorString(e));
  return GLAD_OK;
}

// ---- materialised GLA prefill (prefill.cu) ----
namespace {
struct PrefillWs {
  size_t kv, q, out, lse, bt, dec, total;
  int32_t Lpad, npg;
  int64_t row_stride;
  glad_cache_layout layout;
};
bool prefill_ws(int32_t B, int32_t Lmax, int32_t H, int32_t d_h, int32_t d_rope, int32_t num_ctas, PrefillWs* w) {
  if (B < 1 || Lmax < 1 || H < 1 || d_h < 64 || d_rope < 2) return false;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  w->Lpad = (Lmax + 63) / 64 * 64;
  w->npg = w->Lpad / 64;
  w->row_stride = static_cast<int64_t>(H) * 2 * d_h + d_rope;
  w->layout = glad_cache_layout{B * w->npg, 64, H, 2 * d_h, d_rope, 0, w->row_stride};
  const size_t rows = static_cast<size_t>(B) * Lmax;
  w->kv = 0;
  w->q = w->kv + al(static_cast<size_t>(B) * w->Lpad * w->row_stride * 2);
  w->out = w->q + al(rows * H * (d_h + d_rope) * 2);
  w->lse = w->out + al(rows * H * d_h * 2);
  w->bt = w->lse + al(rows * H * 4);
  w->dec = w->bt + al(static_cast<size_t>(B) * w->npg * 4);
  DecodeGeom g;
  if (decode_geom(kMAT, &w->layout, Lmax, H, &g) != GLAD_OK) return false;
  const int64_t U = static_cast<int64_t>(B) * H * g.n_qblk;
  const int G = num_ctas > 0 ? num_ctas : num_sms();
  w->total = w->dec + ws_layout(U, G, g.key.nq, g.key.d_v).total;
  return true;
}
}  // namespace

size_t glad_gla_prefill_workspace_bytes(int32_t B, int32_t Lmax, int32_t H, int32_t d_h, int32_t d_rope,
                                        int32_t num_ctas) {
  PrefillWs w;
  return prefill_ws(B, Lmax, H, d_h, d_rope, num_ctas, &w) ? w.total : 0;
}

glad_status glad_gla_prefill(const void* q_nope, const void* q_pe, const void* latent, const void* k_pe,
                             const void* w_uk, const void* w_uv, const int32_t* seqlens, int32_t B, int32_t Lmax,
                             int32_t H, int32_t h_c, int32_t d_c, int32_t d_h, int32_t d_rope, float softmax_scale,
                             float rope_base, void* out, float* lse, void* workspace, size_t ws_bytes,
                             int32_t num_ctas, void* stream) {
  if (B < 0 || Lmax < 0) return fail(GLAD_ERR_INVALID_ARG, "prefill B=%d Lmax=%d must be >= 0", B, Lmax);
  if (B == 0 || Lmax == 0) return GLAD_OK;
  if (h_c < 1 || H % h_c || d_c % 64 || d_c < 64 || !(d_h == 128) || d_rope != 64)
    return fail(GLAD_ERR_UNSUPPORTED, "prefill: needs H %% h_c == 0, d_c %% 64 == 0, d_h = 128, d_rope = 64 "
                "(got H=%d h_c=%d d_c=%d d_h=%d d_rope=%d)", H, h_c, d_c, d_h, d_rope);
  if (!(softmax_scale > 0.f) || !std::isfinite(softmax_scale) || !(rope_base > 1.f))
    return fail(GLAD_ERR_INVALID_ARG, "prefill: softmax_scale / rope_base invalid");
  if (!q_nope || !q_pe || !latent || !k_pe || !w_uk || !w_uv || !seqlens || !out || !lse)
    return fail(GLAD_ERR_INVALID_ARG, "prefill: NULL pointer");
  if (!aligned16(q_nope) || !aligned16(latent) || !aligned16(w_uk) || !aligned16(w_uv) || !aligned16(out) ||
      (reinterpret_cast<uintptr_t>(q_pe) & 3u) || (reinterpret_cast<uintptr_t>(k_pe) & 3u))
    return fail(GLAD_ERR_INVALID_ARG, "prefill: q_nope / latent / w_uk / w_uv / out 16-byte, q_pe / k_pe 4-byte aligned");
  PrefillWs w;
  if (!prefill_ws(B, Lmax, H, d_h, d_rope, num_ctas, &w)) return fail(GLAD_ERR_UNSUPPORTED, "prefill: no kernel");
  if (workspace == nullptr || ws_bytes < w.total)
    return fail(GLAD_ERR_WORKSPACE, "prefill workspace %zu bytes < required %zu", ws_bytes, w.total);
  if (reinterpret_cast<uintptr_t>(workspace) & 255u) return fail(GLAD_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  char* ws = static_cast<char*>(workspace);
  void* kv = ws + w.kv;
  void* qf = ws + w.q;
  void* of = ws + w.out;
  float* lf = reinterpret_cast<float*>(ws + w.lse);
  int32_t* bt = reinterpret_cast<int32_t*>(ws + w.bt);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const double lb = log2(static_cast<double>(rope_base));
  cudaError_t e = glad::launch_prefill_upproj(latent, w_uk, B, Lmax, w.Lpad, h_c, d_c, H, d_h, kv, w.row_stride, 0, st);
  if (e == cudaSuccess)
    e = glad::launch_prefill_upproj(latent, w_uv, B, Lmax, w.Lpad, h_c, d_c, H, d_h, kv, w.row_stride, d_h, st);
  if (e == cudaSuccess)
    e = glad::launch_prefill_rope_k(k_pe, B, Lmax, w.Lpad, d_rope, lb, kv, w.row_stride,
                                    static_cast<int64_t>(H) * 2 * d_h, st);
  if (e == cudaSuccess) e = glad::launch_prefill_build_q(q_nope, q_pe, seqlens, B, Lmax, H, d_h, d_rope, lb, qf, st);
  if (e == cudaSuccess) e = glad::launch_prefill_identity_bt(bt, B, w.npg, st);
  if (e != cudaSuccess) return fail(GLAD_ERR_CUDA, "prefill launch failed: %s", cudaGetErrorString(e));
  glad_status s = decode_common(kMAT, qf, kv, &w.layout, bt, w.npg, seqlens, B, Lmax, H, softmax_scale, 1, of, lf,
                                ws + w.dec, w.total - w.dec, num_ctas, stream);
  if (s != GLAD_OK) return s;
  e = glad::launch_prefill_shift_out(of, lf, seqlens, B, Lmax, H, d_h, out, lse, st);
  if (e != cudaSuccess) return fail(GLAD_ERR_CUDA, "prefill launch failed: %s", cudaGetErrorString(e));
  return GLAD_OK;
}

glad_status glad_seq_split_rescale(const float* lse_all, int32_t P, int32_t rank, const void* o, int64_t rows,
                                   int32_t d_v, void* o_out, float* lse_out, void* stream) {
  if (P < 1 || rank < 0 || rank >= P || rows < 0 || d_v < 8 || d_v % 8)
    return fail(GLAD_ERR_INVALID_ARG, "seq split rescale P=%d rank=%d rows=%lld d_v=%d invalid", P, rank,
                static_cast<long long>(rows), d_v);
  if (rows == 0) return GLAD_OK;
  if (!lse_all || !o || !o_out) return fail(GLAD_ERR_INVALID_ARG, "NULL pointer");
  if (!aligned16(o) || !aligned16(o_out)) return fail(GLAD_ERR_INVALID_ARG, "o/o_out must be 16-byte aligned");
  cudaError_t e = glad::launch_lse_rescale(lse_all, P, rank, o, rows, d_v, o_out, lse_out,
                                           static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(GLAD_ERR_CUDA, "seq split rescale launch failed: %s", cudaGetErrorString(e));
  return GLAD_OK;
}

glad_status glad_seq_split_range(int32_t L, int32_t page_size, int32_t Lq, int32_t P, int32_t rank, int32_t* begin,
                                 int32_t* end) {
  if (!begin || !end) return fail(GLAD_ERR_INVALID_ARG, "NULL output pointer");
  if (L < 0 || page_size < 1 || Lq < 1 || P < 1 || rank < 0 || rank >= P)
    return fail(GLAD_ERR_INVALID_ARG, "seq split L=%d page=%d Lq=%d P=%d rank=%d invalid", L, page_size, Lq, P, rank);
  // pages split as evenly as possible, the later ranks taking the extra ones
  const int64_t n = (static_cast<int64_t>(L) + page_size - 1) / page_size;
  const int64_t base = n / P, rem = n % P;
  auto first_page = [&](int64_t r) { return r * base + std::max<int64_t>(0, r - (P - rem)); };
  // the last rank holds (at least) the last Lq - 1 keys, so it alone needs the
  // causal mask: every key of an earlier rank is visible to every query
  int64_t last = first_page(P - 1) * page_size;
  const int64_t must = std::max<int64_t>(0, static_cast<int64_t>(L) - (Lq - 1));
  if (last > must) last = (must / page_size) * page_size;
  int64_t b, e;
  if (rank == P - 1) {
    b = last;
    e = L;
  } else {
    b = std::min<int64_t>(first_page(rank) * page_size, last);
    e = std::min<int64_t>(std::min<int64_t>(first_page(rank + 1) * page_size, last), L);
  }
  *begin = static_cast<int32_t>(b);
  *end = static_cast<int32_t>(std::max(b, e));
  return GLAD_OK;
}

int32_t glad_tp_duplication(int32_t N, int32_t g_q, int32_t h_q) {
  if (N < 1 || g_q < 1 || h_q < 1 || g_q > h_q) return -1;
  return static_cast<int32_t>((static_cast<int64_t>(N) * g_q + h_q - 1) / h_q);
}

glad_status glad_tp_shard(int32_t h_q, int32_t n_kv_heads, int32_t N, int32_t rank, int32_t* kv_begin,
                          int32_t* kv_end, int32_t* q_begin, int32_t* q_end) {
  if (!kv_begin || !kv_end || !q_begin || !q_end) return fail(GLAD_ERR_INVALID_ARG, "NULL output pointer");
  if (h_q < 1 || n_kv_heads < 1 || N < 1 || rank < 0 || rank >= N)
    return fail(GLAD_ERR_INVALID_ARG, "h_q=%d n_kv=%d N=%d rank=%d invalid", h_q, n_kv_heads, N, rank);
  if (h_q % n_kv_heads) return fail(GLAD_ERR_INVALID_ARG, "n_kv_heads=%d must divide h_q=%d", n_kv_heads, h_q);
  if (h_q % N) return fail(GLAD_ERR_INVALID_ARG, "N=%d must divide h_q=%d", N, h_q);
  if (n_kv_heads >= N) {
    if (n_kv_heads % N) return fail(GLAD_ERR_INVALID_ARG, "N=%d must divide n_kv_heads=%d", N, n_kv_heads);
    const int per = n_kv_heads / N;
    *kv_begin = rank * per;
    *kv_end = (rank + 1) * per;
  } else {
    if (N % n_kv_heads) return fail(GLAD_ERR_INVALID_ARG, "n_kv_heads=%d must divide N=%d", n_kv_heads, N);
    const int D = N / n_kv_heads;
    *kv_begin = rank / D;
    *kv_end = rank / D + 1;
  }
  const int qp = h_q / N;
  *q_begin = rank * qp;
  *q_end = (rank + 1) * qp;
  return GLAD_OK;
}

int64_t glad_kv_bytes_per_token_per_device(int32_t variant, int32_t n_kv_heads, int32_t d_head, int32_t d_rope,
                                           int32_t N, int32_t dtype_bytes) {
  if (n_kv_heads < 1 || d_head < 1 || d_rope < 0 || N < 1 || dtype_bytes < 1) return -1;
  int m_kv;
  bool rope;
  switch (variant) {
    case GLAD_MHA: case GLAD_MQA: case GLAD_GQA: m_kv = 2; rope = false; break;
    case GLAD_GTA: case GLAD_GLA: case GLAD_MLA: m_kv = 1; rope = true; break;
    default: return -1;
  }
  const int64_t heads = std::max<int64_t>(1, (n_kv_heads + N - 1) / N);
  return (static_cast<int64_t>(m_kv) * heads * d_head + (rope ? d_rope : 0)) * dtype_bytes;
}

}  // extern "C"
