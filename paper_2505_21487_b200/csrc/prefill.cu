// GLA prefill in the materialised form (P:48
// sigma(Q K^T + Q_R K_R^T) V with the per-head keys / values materialised):
//
//   K_h = c_i W_UK[h],  V_h = c_i W_UV[h]          (i = h / g_q)
//   o[b,t,h] = sum_{j<=t} softmax_j( scale (q_nope.K_h[j] + RoPE(q_pe,t).RoPE(k_pe,j)) ) V_h[j]
//
// For a prompt the materialised form does 2 H (d_h + d_R + d_h) FLOPs per
// (query, key) pair against 2 H (d_c + d_R + d_c) for the absorbed one
// (0.56x at the DeepSeek-V3 shape), at the price of one up-projection GEMM
// per head.  Steps (all on `stream`, glad_gla_prefill in api.cu):
//   1. K / V up-projection: the tcgen05 GEMM of gemm.cuh (A = the latent
//      rows, B = W_UK[h] / W_UV[h] read MN-major) writes per-token rows
//      [K_0 | V_0 | K_1 | V_1 | ... | RoPE(k_pe)] into the workspace;
//   2. prefill_rope_k_kernel: the RoPE key of each token into those rows;
//   3. prefill_build_q_kernel: q = [q_nope || RoPE(q_pe, t)] per head, right
//      aligned in a block of Lmax rows (so the decode kernel's bottom-right
//      causal mask is plain causal for every prompt length);
//   4. the decode kernels in rows mode over those rows as a paged pool
//      (identity block table, one "KV head" per query head, D_S = 2 d_h);
//   5. prefill_shift_out_kernel: outputs back to the natural (left aligned)
//      positions; rows t >= L_b get out = 0, lse = -inf.
#include <cuda_bf16.h>

#include "gemm.cuh"
#include "internal.h"

namespace glad {

namespace {

// cos / sin of pos * theta_i with the angle reduced mod 2 pi in fp64 (R5).
__device__ __forceinline__ void rope_cs(int pos, int i, int d, double log2_base, float& c, float& s) {
  const double theta = exp2(-2.0 * i / d * log2_base);
  double a = static_cast<double>(pos) * theta;
  a -= rint(a * 0.15915494309189535) * 6.283185307179586;
  double sd, cd;
  sincos(a, &sd, &cd);
  c = static_cast<float>(cd);
  s = static_cast<float>(sd);
}

// One CTA per (sequence b, query row r of the right-aligned block): the
// angles of position t = r - (Lmax - L_b) once (fp64, shared by all heads),
// then every head's [q_nope || RoPE(q_pe)] row.
__global__ void prefill_build_q_kernel(const __nv_bfloat16* __restrict__ q_nope, const __nv_bfloat16* __restrict__ q_pe,
                                       const int32_t* __restrict__ seqlens, int32_t Lmax, int32_t H, int32_t d_h,
                                       int32_t d_R, double log2_base, __nv_bfloat16* __restrict__ q_full) {
  __shared__ float cs_s[64], sn_s[64];
  const int b = blockIdx.y, r = blockIdx.x;
  const int t = r - (Lmax - __ldg(seqlens + b));
  const int dq = d_h + d_R;
  __nv_bfloat16* dst = q_full + (static_cast<int64_t>(b) * Lmax + r) * H * dq;
  if (t < 0) {  // padding row of the right-aligned block: sees no key
    for (int idx = threadIdx.x; idx < H * dq / 8; idx += blockDim.x)
      reinterpret_cast<uint4*>(dst)[idx] = make_uint4(0u, 0u, 0u, 0u);
    return;
  }
  if (threadIdx.x < d_R / 2) rope_cs(t, threadIdx.x, d_R, log2_base, cs_s[threadIdx.x], sn_s[threadIdx.x]);
  __syncthreads();
  const int64_t src_row = static_cast<int64_t>(b) * Lmax + t;
  // q_nope part: 16-B vectors
  const int nv = d_h / 8;
  for (int idx = threadIdx.x; idx < H * nv; idx += blockDim.x) {
    const int h = idx / nv, v = idx - h * nv;
    reinterpret_cast<uint4*>(dst + h * dq)[v] =
        __ldg(reinterpret_cast<const uint4*>(q_nope + (src_row * H + h) * d_h) + v);
  }
  // RoPE part: one pair per thread
  const int np = d_R / 2;
  for (int idx = threadIdx.x; idx < H * np; idx += blockDim.x) {
    const int h = idx / np, i = idx - h * np;
    const uint32_t x = __ldg(reinterpret_cast<const unsigned int*>(q_pe + (src_row * H + h) * d_R) + i);
    const float x0 = __uint_as_float(x << 16), x1 = __uint_as_float(x & 0xffff0000u);
    const float c = cs_s[i], s = sn_s[i];
    *reinterpret_cast<uint32_t*>(dst + h * dq + d_h + 2 * i) = pack_bf16x2(x0 * c - x1 * s, x0 * s + x1 * c);
  }
}

// One warp per token j < Lmax of sequence b: RoPE(k_pe[b, j], j) into the
// materialised row's RoPE columns (rows of sequence b start at b * Lpad).
__global__ void prefill_rope_k_kernel(const __nv_bfloat16* __restrict__ k_pe, int32_t B, int32_t Lmax, int32_t Lpad,
                                      int32_t d_R, double log2_base, __nv_bfloat16* __restrict__ kv,
                                      int64_t row_stride, int64_t rope_col) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= B * Lmax) return;
  const int b = w / Lmax, j = w - b * Lmax;
  __nv_bfloat16* dst = kv + (static_cast<int64_t>(b) * Lpad + j) * row_stride + rope_col;
  const __nv_bfloat16* src = k_pe + static_cast<int64_t>(w) * d_R;
  for (int i = lane; i < d_R / 2; i += 32) {
    float c, s;
    rope_cs(j, i, d_R, log2_base, c, s);
    const uint32_t x = __ldg(reinterpret_cast<const unsigned int*>(src) + i);
    const float x0 = __uint_as_float(x << 16), x1 = __uint_as_float(x & 0xffff0000u);
    *reinterpret_cast<uint32_t*>(dst + 2 * i) = pack_bf16x2(x0 * c - x1 * s, x0 * s + x1 * c);
  }
}

// block table of the materialised rows: sequence b owns pages [b * npg, (b + 1) * npg)
__global__ void prefill_identity_bt_kernel(int32_t* __restrict__ bt, int32_t B, int32_t npg) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < B * npg) bt[idx] = idx;
}

// out[b, t] = out_full[b, Lmax - L_b + t] (t < L_b), else 0 / -inf.
__global__ void prefill_shift_out_kernel(const __nv_bfloat16* __restrict__ out_full, const float* __restrict__ lse_full,
                                         const int32_t* __restrict__ seqlens, int32_t Lmax, int32_t H, int32_t d_h,
                                         __nv_bfloat16* __restrict__ out, float* __restrict__ lse) {
  const int b = blockIdx.y, t = blockIdx.x;
  const int L = __ldg(seqlens + b);
  const int64_t drow = static_cast<int64_t>(b) * Lmax + t;
  const int nv = H * d_h / 8;
  uint4* d = reinterpret_cast<uint4*>(out + drow * H * d_h);
  if (t >= L) {
    for (int idx = threadIdx.x; idx < nv; idx += blockDim.x) d[idx] = make_uint4(0u, 0u, 0u, 0u);
    for (int h = threadIdx.x; h < H; h += blockDim.x) lse[drow * H + h] = -INFINITY;
    return;
  }
  const int64_t srow = static_cast<int64_t>(b) * Lmax + (Lmax - L + t);
  const uint4* s = reinterpret_cast<const uint4*>(out_full + srow * H * d_h);
  for (int idx = threadIdx.x; idx < nv; idx += blockDim.x) d[idx] = __ldg(s + idx);
  for (int h = threadIdx.x; h < H; h += blockDim.x) lse[drow * H + h] = __ldg(lse_full + srow * H + h);
}

}  // namespace

// K_h (col_off = 0) or V_h (col_off = d_h) of every head into the
// materialised rows: D[h][m][n] = sum_k latent[m][h / g_q][k] w[h][k][n]
// (M = B * Lmax tokens, N = d_h, K = d_c; w read MN-major), row m of
// sequence b = m / Lmax at kv row b * Lpad + m % Lmax.
cudaError_t launch_prefill_upproj(const void* latent, const void* w, int32_t B, int32_t Lmax, int32_t Lpad,
                                  int32_t h_c, int32_t d_c, int32_t H, int32_t d_h, void* kv, int64_t row_stride,
                                  int32_t col_off, cudaStream_t s) {
  auto enc = tensor_map_encoder();
  if (!enc) return cudaErrorNotSupported;
  const int64_t rows = static_cast<int64_t>(B) * Lmax;
  CUtensorMap ta, tb;
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(d_c), static_cast<cuuint64_t>(h_c), static_cast<cuuint64_t>(rows)};
    cuuint64_t str[2] = {static_cast<cuuint64_t>(d_c) * 2, static_cast<cuuint64_t>(h_c) * d_c * 2};
    cuuint32_t box[3] = {64u, 1u, 128u};
    cuuint32_t es[3] = {1u, 1u, 1u};
    if (enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(latent), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(d_h), static_cast<cuuint64_t>(d_c), static_cast<cuuint64_t>(H)};
    cuuint64_t str[2] = {static_cast<cuuint64_t>(d_h) * 2, static_cast<cuuint64_t>(d_c) * d_h * 2};
    cuuint32_t box[3] = {64u, 64u, 1u};
    cuuint32_t es[3] = {1u, 1u, 1u};
    if (enc(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(w), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  GemmParams gp{};
  gp.M = static_cast<int32_t>(rows);
  gp.N = d_h;
  gp.K = d_c;
  gp.a_div = H / h_c;
  gp.out = static_cast<__nv_bfloat16*>(kv) + col_off;
  gp.out_ld = row_stride;
  gp.out_bstride = 2 * d_h;
  gp.seg_len = Lmax;
  gp.seg_pad = Lpad;
  const dim3 grid(static_cast<unsigned>((rows + 127) / 128), 1u, static_cast<unsigned>(H));
  if (d_h == 128) return launch_gemm<128, true, 4>(ta, tb, gp, grid, s);
  if (d_h == 64) return launch_gemm<64, true, 4>(ta, tb, gp, grid, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_prefill_build_q(const void* q_nope, const void* q_pe, const int32_t* seqlens, int32_t B,
                                   int32_t Lmax, int32_t H, int32_t d_h, int32_t d_R, double log2_base, void* q_full,
                                   cudaStream_t s) {
  prefill_build_q_kernel<<<dim3(Lmax, B), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(q_nope),
                                                      static_cast<const __nv_bfloat16*>(q_pe), seqlens, Lmax, H, d_h,
                                                      d_R, log2_base, static_cast<__nv_bfloat16*>(q_full));
  return cudaGetLastError();
}

cudaError_t launch_prefill_rope_k(const void* k_pe, int32_t B, int32_t Lmax, int32_t Lpad, int32_t d_R,
                                  double log2_base, void* kv, int64_t row_stride, int64_t rope_col, cudaStream_t s) {
  const int64_t warps = static_cast<int64_t>(B) * Lmax;
  prefill_rope_k_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, s>>>(
      static_cast<const __nv_bfloat16*>(k_pe), B, Lmax, Lpad, d_R, log2_base, static_cast<__nv_bfloat16*>(kv),
      row_stride, rope_col);
  return cudaGetLastError();
}

cudaError_t launch_prefill_identity_bt(int32_t* bt, int32_t B, int32_t npg, cudaStream_t s) {
  prefill_identity_bt_kernel<<<(B * npg + 255) / 256, 256, 0, s>>>(bt, B, npg);
  return cudaGetLastError();
}

cudaError_t launch_prefill_shift_out(const void* out_full, const float* lse_full, const int32_t* seqlens, int32_t B,
                                     int32_t Lmax, int32_t H, int32_t d_h, void* out, float* lse, cudaStream_t s) {
  prefill_shift_out_kernel<<<dim3(Lmax, B), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(out_full), lse_full,
                                                        seqlens, Lmax, H, d_h, static_cast<__nv_bfloat16*>(out), lse);
  return cudaGetLastError();
}

}  // namespace glad
