// The step right before the decode hot path: form the
// kernel's inputs from the model's raw per-step tensors.
//
//  * absorbed query: q = [ W_UK[h] q_nope  ||  RoPE(q_pe, p_t) ]
//    (weight absorption: the per-head key up-projection is folded into
//    the query so keys never materialise; the decoupled RoPE part is rotated
//    at the query's position p_t = L_b - Lq + t, R2/R5): the batched
//    tcgen05 GEMM of gemm.cuh (TMA-staged operands, TMEM accumulator) with
//    the RoPE pairs in its epilogue.
//  * append_rope_kernel: cache row = [ latent || RoPE(k_pe, p) ] written into
//    the paged pool at position p = seqlens_before[b] + i.
//
// RoPE (R5): interleaved pairs (2i, 2i+1), theta_i = base^(-2i/d), angle
// p * theta_i evaluated in fp64 (positions up to 64K make an fp32 angle off by
// ~4e-3 rad).
#include <cuda_bf16.h>

#include "gemm.cuh"
#include "internal.h"

namespace glad {

namespace {

__device__ __forceinline__ void rope_pair(float x0, float x1, int pos, int i, int d, double log_base, float& y0,
                                          float& y1) {
  const double theta = exp(-2.0 * i / d * log_base);
  // reduce mod 2 pi in fp64 first (|angle| <= pi keeps sincos on its fast
  // path; the large-argument reduction used local memory and dominated)
  double a = static_cast<double>(pos) * theta;
  a -= rint(a * 0.15915494309189535) * 6.283185307179586;
  double s, c;
  sincos(a, &s, &c);
  y0 = static_cast<float>(x0 * c - x1 * s);
  y1 = static_cast<float>(x0 * s + x1 * c);
}

// One warp per new token row: latent copied with 16-B vectors, the RoPE key
// rotated at its position (one pair per lane per pass).
__global__ void append_rope_kernel(__nv_bfloat16* __restrict__ pool, int64_t row_stride, int page_size,
                                   const int32_t* __restrict__ block_table, int32_t bt_stride,
                                   const int32_t* __restrict__ seqlens_before, const __nv_bfloat16* __restrict__ latent,
                                   const __nv_bfloat16* __restrict__ k_pe, int32_t B, int32_t n_new, int32_t w_lat,
                                   int32_t d_R, float rope_base) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= B * n_new) return;
  const int b = w / n_new, i = w - b * n_new;
  const int pos = seqlens_before[b] + i;
  const int page = block_table[static_cast<int64_t>(b) * bt_stride + pos / page_size];
  __nv_bfloat16* dst = pool + (static_cast<int64_t>(page) * page_size + pos % page_size) * row_stride;
  const uint4* src = reinterpret_cast<const uint4*>(latent + static_cast<int64_t>(w) * w_lat);
  for (int u = lane; u < w_lat / 8; u += 32) reinterpret_cast<uint4*>(dst)[u] = __ldg(src + u);
  const double lb = log(static_cast<double>(rope_base));
  const __nv_bfloat16* kp = k_pe + static_cast<int64_t>(w) * d_R;
  for (int pi = lane; pi < d_R / 2; pi += 32) {
    float y0, y1;
    rope_pair(__bfloat162float(kp[2 * pi]), __bfloat162float(kp[2 * pi + 1]), pos, pi, d_R, lb, y0, y1);
    *reinterpret_cast<uint32_t*>(dst + w_lat + 2 * pi) = pack_bf16x2(y0, y1);
  }
}

}  // namespace

bool absorb_supported(int d_h, int d_c) {
  return (d_h == 64 || d_h == 128) && (d_c == 128 || d_c == 256 || d_c == 512);
}

// q[b,t,h] = [ W_UK[h] q_nope[b,t,h] || RoPE(q_pe[b,t,h], L_b - Lq + t) ] as
// a batched tcgen05 GEMM over the heads (gemm.cuh): M = B*Lq rows, N = d_c,
// K = d_h, A = q_nope's rows of head h (3-D map [rows][H][d_h]), B = W_UK[h]
// (K-major, 3-D map [H][d_c][d_h]); the RoPE pairs in the same epilogue.
cudaError_t launch_absorb_query(const void* q_nope, const void* q_pe, const void* w_uk, const int32_t* seqlens,
                                int32_t B, int32_t Lq, int32_t H, int32_t d_h, int32_t d_c, int32_t d_R,
                                float rope_base, void* q_out, cudaStream_t stream) {
  const int64_t rows = static_cast<int64_t>(B) * Lq;
  if (rows == 0) return cudaSuccess;
  auto enc = tensor_map_encoder();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap ta, tb;
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(d_h), static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(rows)};
    cuuint64_t str[2] = {static_cast<cuuint64_t>(d_h) * 2, static_cast<cuuint64_t>(H) * d_h * 2};
    cuuint32_t box[3] = {64u, 1u, 128u};
    cuuint32_t es[3] = {1u, 1u, 1u};
    if (enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(q_nope), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int BN = 128;  // two+ N tiles per head: more CTAs in flight, the RoPE pairs split between them
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(d_h), static_cast<cuuint64_t>(d_c), static_cast<cuuint64_t>(H)};
    cuuint64_t str[2] = {static_cast<cuuint64_t>(d_h) * 2, static_cast<cuuint64_t>(d_c) * d_h * 2};
    cuuint32_t box[3] = {64u, static_cast<cuuint32_t>(BN), 1u};
    cuuint32_t es[3] = {1u, 1u, 1u};
    if (enc(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(w_uk), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  GemmParams gp{};
  gp.M = static_cast<int32_t>(rows);
  gp.N = d_c;
  gp.K = d_h;
  gp.a_div = 1;
  gp.out = static_cast<__nv_bfloat16*>(q_out);
  gp.out_ld = static_cast<int64_t>(H) * (d_c + d_R);
  gp.out_bstride = d_c + d_R;
  gp.rope_src = static_cast<const __nv_bfloat16*>(q_pe);
  gp.seqlens = seqlens;
  gp.rope_ld = static_cast<int64_t>(H) * d_R;
  gp.rope_bstride = d_R;
  gp.rope_col = d_c;
  gp.d_rope = d_R;
  gp.Lq = Lq;
  gp.log2_base = log2(static_cast<double>(rope_base));
  const dim3 grid(static_cast<unsigned>((rows + 127) / 128), static_cast<unsigned>(d_c / BN), static_cast<unsigned>(H));
  return d_h == 64 ? launch_gemm<128, false, 1>(ta, tb, gp, grid, stream) : launch_gemm<128, false, 2>(ta, tb, gp, grid, stream);
}

cudaError_t launch_append_rope(void* pool, int64_t row_stride, int page_size, const int32_t* block_table,
                               int32_t bt_stride, const int32_t* seqlens_before, const void* latent,
                               const void* k_pe, int32_t B, int32_t n_new, int32_t w_lat, int32_t d_R,
                               float rope_base, cudaStream_t stream) {
  const int64_t n = static_cast<int64_t>(B) * n_new;
  if (n == 0) return cudaSuccess;
  const int threads = 256;
  append_rope_kernel<<<static_cast<unsigned>((n * 32 + threads - 1) / threads), threads, 0, stream>>>(
      static_cast<__nv_bfloat16*>(pool), row_stride, page_size, block_table, bt_stride, seqlens_before,
      static_cast<const __nv_bfloat16*>(latent), static_cast<const __nv_bfloat16*>(k_pe), B, n_new, w_lat, d_R,
      rope_base);
  return cudaGetLastError();
}

}  // namespace glad
