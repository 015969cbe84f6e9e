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
// -> exclusive prefix sum plan[0..U]; plan[U] = total tiles.
__global__ void plan_kernel(const int32_t* __restrict__ seqlens, int32_t* __restrict__ plan, int U, int B, int tile,
                            int n_qblk, int nq_blk, int Lq, int g_q, int causal) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < U; base += blockDim.x) {
    const int u = base + threadIdx.x;
    int tiles = 0;
    if (u < U) {
      const int qb = u % n_qblk;
      const int b = (u / n_qblk) % B;  // head-major unit order
      const int n0 = qb * nq_blk;
      const int nq = min(nq_blk, Lq * g_q - n0);
      const int L = seqlens[b];
      int kv_end = L;
      if (causal) kv_end = max(0, min(L, L - Lq + (n0 + nq - 1) / g_q + 1));
      tiles = (kv_end + tile - 1) / tile;
    }
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
}

// Merge the partial segments of units that a CTA range boundary cut (the
// split-KV LSE merge); write zeros / -inf for units with no visible key.
// One warp per output row (b, t, h).  Units finished inside one CTA were
// written by the decode kernel and are skipped.
__global__ void merge_units_kernel(const int32_t* __restrict__ plan, const float* __restrict__ o_part,
                                   const float* __restrict__ lse_part, int G, int U, int nq_blk, int n_qblk,
                                   int B, int n_heads, int head_groups, int g_q, int Lq, int H, int64_t rows, int d_v,
                                   __nv_bfloat16* __restrict__ out, float* __restrict__ lse) {
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int h = static_cast<int>(row % H);
  const int64_t bt = row / H;
  const int t = static_cast<int>(bt % Lq);
  const int b = static_cast<int>(bt / Lq);
  const int head = h / g_q, j = h - head * g_q;
  const int ng = t * g_q + j;
  const int qb = ng / nq_blk, n = ng - qb * nq_blk;
  const int u = (head * B + b) * n_qblk + qb;
  const int pu0 = plan[u], pu1 = plan[u + 1], total = plan[U];
  if (pu1 == pu0) {  // no visible key
    for (int d = lane * 8; d < d_v; d += 256)
      *reinterpret_cast<uint4*>(out + row * d_v + d) = make_uint4(0u, 0u, 0u, 0u);
    if (lane == 0) lse[row] = -INFINITY;
    return;
  }
  const int c_first = cta_of_tile(pu0, G, total, n_heads, head_groups);
  const int c_last = cta_of_tile(pu1 - 1, G, total, n_heads, head_groups);
  if (c_first == c_last) return;
  float mx = -INFINITY;
  for (int c = c_first + lane; c <= c_last; c += 32)
    mx = fmaxf(mx, lse_part[static_cast<int64_t>(c + u) * nq_blk + n]);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float z = 0.f;
  for (int c = c_first + lane; c <= c_last; c += 32) {
    const float ls = lse_part[static_cast<int64_t>(c + u) * nq_blk + n];
    if (ls != -INFINITY) z += __expf(ls - mx);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  if (lane == 0) lse[row] = (z > 0.f) ? mx + __logf(z) : -INFINITY;
  const float inv_z = (z > 0.f) ? 1.f / z : 0.f;
  for (int d0 = lane * 8; d0 < d_v; d0 += 256) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int c = c_first; c <= c_last; ++c) {
      const int64_t slot = static_cast<int64_t>(c + u) * nq_blk + n;
      const float ls = lse_part[slot];
      if (ls == -INFINITY) continue;
      const float w = __expf(ls - mx) * inv_z;
      const float4* src = reinterpret_cast<const float4*>(o_part + slot * d_v + d0);
      const float4 a = __ldg(src), c4 = __ldg(src + 1);
      acc[0] += w * a.x; acc[1] += w * a.y; acc[2] += w * a.z; acc[3] += w * a.w;
      acc[4] += w * c4.x; acc[5] += w * c4.y; acc[6] += w * c4.z; acc[7] += w * c4.w;
    }
    uint4 v;
    v.x = pack_bf16x2(acc[0], acc[1]);
    v.y = pack_bf16x2(acc[2], acc[3]);
    v.z = pack_bf16x2(acc[4], acc[5]);
    v.w = pack_bf16x2(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(out + row * d_v + d0) = v;
  }
}

cudaError_t launch_plan(const int32_t* seqlens, int32_t* plan, int U, int B, int tile, int n_qblk, int nq_blk, int Lq,
                        int g_q, int causal, cudaStream_t stream) {
  plan_kernel<<<1, 1024, 0, stream>>>(seqlens, plan, U, B, tile, n_qblk, nq_blk, Lq, g_q, causal);
  return cudaGetLastError();
}

cudaError_t launch_merge_units(const int32_t* plan, const float* o_part, const float* lse_part, int G, int U,
                               int nq_blk, int n_qblk, int B, int n_heads, int head_groups, int g_q, int Lq, int H,
                               int64_t rows, int d_v, void* out, float* lse, cudaStream_t stream) {
  if (rows == 0) return cudaSuccess;
  const int threads = 128;
  const int64_t blocks = (rows * 32 + threads - 1) / threads;
  merge_units_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
      plan, o_part, lse_part, G, U, nq_blk, n_qblk, B, n_heads, head_groups, g_q, Lq, H, rows, d_v,
      static_cast<__nv_bfloat16*>(out), lse);
  return cudaGetLastError();
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
