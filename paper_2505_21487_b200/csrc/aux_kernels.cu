// Paged-cache append / gather and the split-KV LSE merge (sm_100a).
// All three are HBM-bound copies/reductions: 16-byte vector accesses, one
// warp per row, grid sized to the row count.
#include <cuda_bf16.h>

#include "internal.h"

namespace glad {

// P:304 paged KV: position p of sequence b -> pool row
// block_table[b][p / page] * page + p % page.
__global__ void append_kernel(uint4* __restrict__ pool, int64_t row_stride_u4, int page_size,
                              const int32_t* __restrict__ block_table, int32_t bt_stride,
                              const int32_t* __restrict__ seqlens_before, const uint4* __restrict__ rows,
                              int32_t B, int32_t n_new, int32_t width_u4) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= B * n_new) return;
  const int b = w / n_new, i = w - b * n_new;
  const int pos = seqlens_before[b] + i;
  const int page = block_table[static_cast<int64_t>(b) * bt_stride + pos / page_size];
  const int64_t prow = static_cast<int64_t>(page) * page_size + pos % page_size;
  uint4* dst = pool + prow * row_stride_u4;
  const uint4* src = rows + static_cast<int64_t>(w) * width_u4;
  for (int u = lane; u < width_u4; u += 32) dst[u] = __ldg(src + u);
}

__global__ void gather_kernel(const uint4* __restrict__ pool, int64_t row_stride_u4, int page_size,
                              const int32_t* __restrict__ block_table, int32_t bt_stride,
                              const int32_t* __restrict__ seqlens, int32_t B, int32_t max_len, int32_t width_u4,
                              uint4* __restrict__ out) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= static_cast<int64_t>(B) * max_len) return;
  const int b = static_cast<int>(w / max_len), j = static_cast<int>(w - static_cast<int64_t>(b) * max_len);
  uint4* dst = out + w * width_u4;
  if (j < seqlens[b]) {
    const int page = block_table[static_cast<int64_t>(b) * bt_stride + j / page_size];
    const uint4* src = pool + (static_cast<int64_t>(page) * page_size + j % page_size) * row_stride_u4;
    for (int u = lane; u < width_u4; u += 32) dst[u] = __ldg(src + u);
  } else {
    for (int u = lane; u < width_u4; u += 32) dst[u] = make_uint4(0u, 0u, 0u, 0u);
  }
}

// lse = ln sum_s exp(lse_s); out = sum_s exp(lse_s - lse) o_s.  One warp per
// (b, t, h) row; splits with lse_s = -inf contribute nothing (their o_s is
// never read, so it may hold anything).
__global__ void combine_kernel(const float* __restrict__ o_part, const float* __restrict__ lse_part, int32_t S,
                               int64_t rows, int32_t d_v, __nv_bfloat16* __restrict__ out,
                               float* __restrict__ lse) {
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  float mx = -INFINITY;
  for (int s = lane; s < S; s += 32) mx = fmaxf(mx, lse_part[s * rows + row]);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float z = 0.f;
  for (int s = lane; s < S; s += 32) {
    const float ls = lse_part[s * rows + row];
    if (ls != -INFINITY) z += __expf(ls - mx);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  if (lane == 0) lse[row] = (z > 0.f) ? mx + __logf(z) : -INFINITY;
  const float inv_z = (z > 0.f) ? 1.f / z : 0.f;
  for (int d0 = lane * 8; d0 < d_v; d0 += 256) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int s = 0; s < S; ++s) {
      const float ls = lse_part[s * rows + row];
      if (ls == -INFINITY) continue;
      const float w = __expf(ls - mx) * inv_z;
      const float4* src = reinterpret_cast<const float4*>(o_part + (s * rows + row) * d_v + d0);
      const float4 a = __ldg(src), b = __ldg(src + 1);
      acc[0] += w * a.x; acc[1] += w * a.y; acc[2] += w * a.z; acc[3] += w * a.w;
      acc[4] += w * b.x; acc[5] += w * b.y; acc[6] += w * b.z; acc[7] += w * b.w;
    }
    uint4 v;
    v.x = pack_bf16x2(acc[0], acc[1]);
    v.y = pack_bf16x2(acc[2], acc[3]);
    v.z = pack_bf16x2(acc[4], acc[5]);
    v.w = pack_bf16x2(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(out + row * d_v + d0) = v;
  }
}

// Decode schedule plan (one CTA): tiles per unit u = (b, head, query block)
// -> exclusive prefix sum plan[0..U]; plan[U] = total tiles.  Also writes
// the output of units with no visible key (zeros, lse = -inf), which no
// decode CTA visits.
__global__ void plan_kernel(const int32_t* __restrict__ seqlens, int32_t* __restrict__ plan,
                            int U, int seg_cost, int cl_n,
                            int B, int tile, int n_qblk, int qb_outer, int nq_blk, int Lq, int g_q,
                            int causal, int H, int d_v, __nv_bfloat16* __restrict__ out, float* __restrict__ lse,
                            uint64_t* trace) {
  if (trace && threadIdx.x == 0) trace[0] = globaltimer();
  griddep_launch();  // (PDL) the decode kernel's prologue may start now; it waits for this grid before reading plan
  __shared__ int warp_sums[32];
  __shared__ int carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < U; base += blockDim.x) {
    const int u = base + threadIdx.x;
    int tiles = 0;
    if (u < U) {
      // plan entry u: unit u, or with clusters the (head, sequence) group of
      // cl_n units whose tiles are those of its last query block (most keys)
      const int ul = u * cl_n + cl_n - 1;
      const UnitIdx ui = unit_idx(ul, B, n_qblk, qb_outer);
      const int qb = ui.qb, b = ui.b;
      const int n0 = qb * nq_blk;
      const int nq = min(nq_blk, Lq * g_q - n0);
      const int L = seqlens[b];
      int kv_end = L;
      if (causal) kv_end = max(0, min(L, L - Lq + (n0 + nq - 1) / g_q + 1));
      tiles = (kv_end + tile - 1) / tile;
      if (tiles == 0) {  // no visible key: no decode CTA visits the unit(s) (rare; one thread per entry)
        const int head = ui.head;
        const int n_first = (qb - (cl_n - 1)) * nq_blk;  // clusters (qb_outer = 0): the entry's first block
        for (int n = n_first; n < n0 + nq; ++n) {
          const int t = n / g_q, h = head * g_q + (n - t * g_q);
          const int64_t row = (static_cast<int64_t>(b) * Lq + t) * H + h;
          uint4* o = reinterpret_cast<uint4*>(out + row * d_v);
          for (int d = 0; d < d_v / 8; ++d) o[d] = make_uint4(0u, 0u, 0u, 0u);
          lse[row] = -INFINITY;
        }
      }
    }
    if (tiles > 0) tiles += seg_cost;  // virtual tiles: the unit's segment-switch cost in the range balance
    int v = tiles;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane == 31) warp_sums[warp] = v;
    __syncthreads();
    if (warp == 0) {
      int w = lane < nwarps ? warp_sums[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_sums[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int excl = carry + (warp > 0 ? warp_sums[warp - 1] : 0) + v - tiles;
    if (u < U) plan[u] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sums[nwarps - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) plan[U] = carry;
  __syncthreads();
  if (trace && threadIdx.x == 0) trace[1] = globaltimer();
}

cudaError_t launch_plan(const int32_t* seqlens, int32_t* plan, int U, int seg_cost, int cl_n, int B, int tile, int n_qblk,
                        int qb_outer, int nq_blk, int Lq, int g_q, int causal, int H, int d_v, void* out, float* lse,
                        uint64_t* trace, cudaStream_t stream) {
  plan_kernel<<<1, 1024, 0, stream>>>(seqlens, plan, U, seg_cost, cl_n, B, tile, n_qblk, qb_outer, nq_blk, Lq, g_q, causal, H, d_v,
                                      static_cast<__nv_bfloat16*>(out), lse, trace);
  return cudaGetLastError();
}

// Split-KV LSE merge of the units that range boundaries cut (
// oracle.attention.merge_partials).  Ranges belong to CTAs, or with
// clusters (cl_n > 1) to clusters whose CTA r owns query block r of each
// plan entry.  Block (b, r) looks at the boundary between ranges b-1 and b:
// if it cuts a plan entry and is its first cut, the block merges the
// partials of unit entry * cl_n + r (workspace slots (c + entry) * cl_n + r,
// c = first..last range of the entry) into out / lse.  All other blocks
// exit at once.
#ifndef GLAD_MERGE_SPLIT
#define GLAD_MERGE_SPLIT 2  // blocks per merged unit
#endif
constexpr int kMergeThreads = 256;
constexpr int kMergeMaxParts = 8;  // weights staged per pass
__global__ void __launch_bounds__(kMergeThreads) merge_split_kernel(
    const int32_t* __restrict__ plan, const float* __restrict__ o_part, const float* __restrict__ lse_part, int G,
    int cl_n, int U, int nq_blk, int n_qblk, int qb_outer, int B, int n_groups, int g_q, int Lq, int H, int d_v,
    int seg_cost, __nv_bfloat16* __restrict__ out, float* __restrict__ lse) {
  __shared__ int u_s;
  __shared__ float w_s[kMergeMaxParts][128];  // nq_blk <= 128 (rows mode)
  __shared__ float mx_s[128], iz_s[128];
  __shared__ int gb_s[kMaxGroups + 1];
  griddep_wait();  // (PDL) the decode grid's partials and plan are complete and visible
  const int GR = G / cl_n;                     // ranges
  const int b_cta = blockIdx.x / cl_n + 1;     // boundary between ranges b-1 and b
  const int rank = blockIdx.x % cl_n;
  // group boundaries in shared memory: one parallel load instead of a chain
  // of dependent L2 reads per range lookup
  const int ng = n_groups > 1 ? n_groups : 1;
  if (threadIdx.x <= ng) gb_s[threadIdx.x] = __ldg(plan + threadIdx.x * (U / ng));
  __syncthreads();
  const CtaRange rg = cta_range_gb(b_cta, GR, gb_s, ng);
  if (rg.t0 >= rg.t1) return;
  const int t = rg.t0;
  // unit containing tile t: 32-ary search by warp 0 (last u with plan[u] <= t)
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int lo = 0, hi = U - 1;
    while (lo < hi) {
      const int step = (hi - lo + 32) / 32;
      const int idx = lo + lane * step;
      const bool ok = idx <= hi && __ldg(plan + idx) <= t;
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      lo = lo + (31 - __clz(m)) * step;
      hi = min(hi, lo + step - 1);
    }
    if (lane == 0) u_s = lo;
  }
  __syncthreads();
  const int pe = u_s;  // plan entry
  const int pr0 = __ldg(plan + pe), pu1 = __ldg(plan + pe + 1);
  const int pu0 = pr0 + seg_cost;  // first real tile (after the entry's virtual segment-cost tiles)
  if (t <= pu0) return;  // the boundary is at or before the entry's first real tile: not cut here
  const int cf = cta_of_tile_gb(pu0, GR, gb_s, ng);
  if (cf != b_cta - 1) return;  // an earlier boundary cuts it: that block merges
  const int cl = cta_of_tile_gb(pu1 - 1, GR, gb_s, ng);
  const int u = pe * cl_n + rank;
  const UnitIdx ui = unit_idx(u, B, n_qblk, qb_outer);
  const int qb = ui.qb, b = ui.b, head = ui.head;
  const int n0 = qb * nq_blk;
  const int nq = min(nq_blk, Lq * g_q - n0);
  if (nq <= 0) return;
  // partial slot of range c (decode epilogue): 2c if the entry is c's first
  // segment, 2c + 1 if it is its last one (only range cf can have earlier
  // segments, when its range starts before the entry)
  const int cf_last = cta_range_gb(cf, GR, gb_s, ng).t0 < pr0 ? 1 : 0;
  auto slot_of = [&](int c) -> int64_t { return static_cast<int64_t>(2 * c + (c == cf ? cf_last : 0)) * cl_n + rank; };
  for (int n = threadIdx.x; n < nq; n += kMergeThreads) {
    float mx = -INFINITY;
    for (int c = cf; c <= cl; ++c) mx = fmaxf(mx, lse_part[slot_of(c) * nq_blk + n]);
    float z = 0.f;
    if (mx != -INFINITY)
      for (int c = cf; c <= cl; ++c) z += __expf(lse_part[slot_of(c) * nq_blk + n] - mx);
    const int ng = n0 + n, tq = ng / g_q, h = head * g_q + (ng - tq * g_q);
    if (blockIdx.y == 0) lse[(static_cast<int64_t>(b) * Lq + tq) * H + h] = z > 0.f ? mx + __logf(z) : -INFINITY;
    mx_s[n] = mx;
    iz_s[n] = z > 0.f ? 1.f / z : 0.f;
  }
  // items (column n, 4 consecutive d): thread-strided, weights staged per
  // pass of <= kMergeMaxParts partials
  const int d4n = d_v / 4;
  const int items = nq * d4n;
  constexpr int kPer = 8;  // items per thread per sweep (loads in flight)
  // the unit's items are interleaved over gridDim.y blocks (more loads in flight per unit)
  for (int base = blockIdx.y * kMergeThreads * kPer; base < items; base += gridDim.y * kMergeThreads * kPer) {
    float4 acc[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c0 = cf; c0 <= cl; c0 += kMergeMaxParts) {
      const int np = min(kMergeMaxParts, cl + 1 - c0);
      __syncthreads();
      for (int k = threadIdx.x; k < np * nq; k += kMergeThreads) {
        const int cc = k / nq, n = k - cc * nq;
        const float mx = mx_s[n];
        w_s[cc][n] = mx == -INFINITY ? 0.f : __expf(lse_part[slot_of(c0 + cc) * nq_blk + n] - mx) * iz_s[n];
      }
      __syncthreads();
      for (int cc = 0; cc < np; ++cc) {
        const float4* src = reinterpret_cast<const float4*>(
            o_part + slot_of(c0 + cc) * nq_blk * d_v);
        float4 v[kPer];
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          const int it = base + i * kMergeThreads + threadIdx.x;
          v[i] = it < items ? __ldg(src + (it / d4n) * d4n + (it % d4n)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          const int it = base + i * kMergeThreads + threadIdx.x;
          const float w = it < items ? w_s[cc][it / d4n] : 0.f;
          acc[i].x += w * v[i].x; acc[i].y += w * v[i].y; acc[i].z += w * v[i].z; acc[i].w += w * v[i].w;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int it = base + i * kMergeThreads + threadIdx.x;
      if (it < items) {
        const int n = it / d4n, d = (it % d4n) * 4;
        const int ng = n0 + n, tq = ng / g_q, h = head * g_q + (ng - tq * g_q);
        *reinterpret_cast<uint2*>(out + ((static_cast<int64_t>(b) * Lq + tq) * H + h) * d_v + d) =
            make_uint2(pack_bf16x2(acc[i].x, acc[i].y), pack_bf16x2(acc[i].z, acc[i].w));
      }
    }
  }
}

cudaError_t launch_merge_split(const int32_t* plan, const float* o_part, const float* lse_part, int G, int cl_n,
                               int U, int nq_blk, int n_qblk, int qb_outer, int B, int n_groups, int g_q, int Lq,
                               int H, int d_v, int seg_cost, void* out, float* lse, cudaStream_t stream) {
  if (G / cl_n < 2) return cudaSuccess;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((G / cl_n - 1) * cl_n, GLAD_MERGE_SPLIT);
  cfg.blockDim = dim3(kMergeThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = GLAD_PDL ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, merge_split_kernel, plan, o_part, lse_part, G, cl_n, U, nq_blk, n_qblk, qb_outer, B,
                            n_groups, g_q, Lq, H, d_v, seg_cost, static_cast<__nv_bfloat16*>(out), lse);
}

cudaError_t launch_append(void* pool, int64_t row_stride, int page_size, const int32_t* block_table,
                          int32_t bt_stride, const int32_t* seqlens_before, const void* rows, int32_t B,
                          int32_t n_new, int32_t width, cudaStream_t stream) {
  const int64_t warps = static_cast<int64_t>(B) * n_new;
  if (warps == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (warps * 32 + threads - 1) / threads;
  append_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
      static_cast<uint4*>(pool), row_stride / 8, page_size, block_table, bt_stride, seqlens_before,
      static_cast<const uint4*>(rows), B, n_new, width / 8);
  return cudaGetLastError();
}

cudaError_t launch_gather(const void* pool, int64_t row_stride, int page_size, const int32_t* block_table,
                          int32_t bt_stride, const int32_t* seqlens, int32_t B, int32_t max_len, int32_t width,
                          void* dense_out, cudaStream_t stream) {
  const int64_t warps = static_cast<int64_t>(B) * max_len;
  if (warps == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (warps * 32 + threads - 1) / threads;
  gather_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
      static_cast<const uint4*>(pool), row_stride / 8, page_size, block_table, bt_stride, seqlens, B, max_len,
      width / 8, static_cast<uint4*>(dense_out));
  return cudaGetLastError();
}

// Sequence split across the P ranks of a head group: one
// warp per row; the row's global lse = ln sum_p exp(lse_all[p][row]) and the
// rank's normalised partial output is scaled by exp(lse_rank - lse), so the
// group sum of the scaled rows (folded into the o_proj all-reduce) is the
// attention output over the whole sequence.
__global__ void lse_rescale_kernel(const float* __restrict__ lse_all, int32_t P, int32_t rank,
                                   const __nv_bfloat16* __restrict__ o, int64_t rows, int32_t d_v,
                                   float* __restrict__ o_out, float* __restrict__ lse_out) {
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  float mx = -INFINITY;
  for (int p = lane; p < P; p += 32) mx = fmaxf(mx, lse_all[p * rows + row]);
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, s));
  float z = 0.f;
  for (int p = lane; p < P; p += 32) {
    const float ls = lse_all[p * rows + row];
    if (ls != -INFINITY) z += __expf(ls - mx);
  }
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) z += __shfl_xor_sync(0xffffffffu, z, s);
  const float lse = (z > 0.f) ? mx + __logf(z) : -INFINITY;
  if (lane == 0 && lse_out) lse_out[row] = lse;
  const float own = lse_all[static_cast<int64_t>(rank) * rows + row];
  const float w = (own == -INFINITY || lse == -INFINITY) ? 0.f : __expf(own - lse);
  for (int d0 = lane * 8; d0 < d_v; d0 += 256) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(o + row * d_v + d0));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
    const float2 f0 = __bfloat1622float2(h[0]), f1 = __bfloat1622float2(h[1]);
    const float2 f2 = __bfloat1622float2(h[2]), f3 = __bfloat1622float2(h[3]);
    float4* dst = reinterpret_cast<float4*>(o_out + row * d_v + d0);
    dst[0] = make_float4(f0.x * w, f0.y * w, f1.x * w, f1.y * w);
    dst[1] = make_float4(f2.x * w, f2.y * w, f3.x * w, f3.y * w);
  }
}

cudaError_t launch_lse_rescale(const float* lse_all, int32_t P, int32_t rank, const void* o, int64_t rows,
                               int32_t d_v, void* o_out, float* lse_out, cudaStream_t stream) {
  if (rows == 0) return cudaSuccess;
  const int threads = 128;
  const int64_t blocks = (rows * 32 + threads - 1) / threads;
  lse_rescale_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
      lse_all, P, rank, static_cast<const __nv_bfloat16*>(o), rows, d_v, static_cast<float*>(o_out),
      lse_out);
  return cudaGetLastError();
}

cudaError_t launch_combine(const float* o_part, const float* lse_part, int32_t S, int64_t rows, int32_t d_v,
                           void* out, float* lse, cudaStream_t stream) {
  if (rows == 0) return cudaSuccess;
  const int threads = 128;
  const int64_t blocks = (rows * 32 + threads - 1) / threads;
  combine_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
      o_part, lse_part, S, rows, d_v, static_cast<__nv_bfloat16*>(out), lse);
  return cudaGetLastError();
}

}  // namespace glad
