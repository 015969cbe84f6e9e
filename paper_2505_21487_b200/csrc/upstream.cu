// The step right before the decode hot path: form the
// kernel's inputs from the model's raw per-step tensors.
//
//  * absorb_query_kernel: q = [ W_UK[h] q_nope  ||  RoPE(q_pe, p_t) ]
//    (weight absorption: the per-head key up-projection is folded into
//    the query so keys never materialise; the decoupled RoPE part is rotated
//    at the query's position p_t = L_b - Lq + t, R2/R5).  A small batched
//    GEMM per head (rows = B*Lq, K = d_h, N = d_c) bound by reading W_UK once
//    per step; warp-level bf16 mma.sync with fp32 accumulation is enough for
//    it (0.5 GFLOP at C2 vs 8 MB of weights).
//  * append_rope_kernel: cache row = [ latent || RoPE(k_pe, p) ] written into
//    the paged pool at position p = seqlens_before[b] + i.
//
// RoPE (R5): interleaved pairs (2i, 2i+1), theta_i = base^(-2i/d), angle
// p * theta_i evaluated in fp64 (positions up to 64K make an fp32 angle off by
// ~4e-3 rad).
#include <cuda_bf16.h>

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

__device__ __forceinline__ uint32_t ld_b32(const __nv_bfloat16* p) { return *reinterpret_cast<const uint32_t*>(p); }

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

constexpr int kRowsPerCta = 64;
constexpr int kAbsorbThreads = 256;

// CTA = (head h, 64 query rows).  Shared memory: the rows' q_nope [64][d_h]
// and W_UK[h] [d_c][d_h] (rows padded by 8 elements against bank conflicts).
// Warp w: rows 16 (w & 3) .. +16, output columns (w >> 2) * d_c / 2 .. + d_c / 2.
template <int DH, int DC>
__global__ void __launch_bounds__(kAbsorbThreads) absorb_query_kernel(
    const __nv_bfloat16* __restrict__ q_nope, const __nv_bfloat16* __restrict__ q_pe,
    const __nv_bfloat16* __restrict__ w_uk, const int32_t* __restrict__ seqlens, int32_t B, int32_t Lq, int32_t H,
    int32_t d_R, float rope_base, __nv_bfloat16* __restrict__ q_out) {
  constexpr int LD = DH + 8;  // padded row (elements)
  constexpr int NSUB = DC / 2 / 8;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* sq = reinterpret_cast<__nv_bfloat16*>(smem_raw);  // [64][LD]
  __nv_bfloat16* sw = sq + kRowsPerCta * LD;                       // [DC][LD]
  const int h = blockIdx.y;
  const int r0 = blockIdx.x * kRowsPerCta;
  const int rows = B * Lq;
  const int nrows = min(kRowsPerCta, rows - r0);
  const int tid = threadIdx.x;
  const int DQ = DC + d_R;
  // stage q_nope rows and W_UK[h] (16-B vectors)
  constexpr int VR = DH / 8;
  // (fully unrolled: all of a thread's 16-B loads are in flight at once —
  // a rolled load -> st.shared loop paid one memory latency per iteration)
#pragma unroll
  for (int idx = tid; idx < kRowsPerCta * VR; idx += kAbsorbThreads) {
    const int r = idx / VR, v = idx - r * VR;
    uint4 x = make_uint4(0u, 0u, 0u, 0u);
    if (r < nrows) x = __ldg(reinterpret_cast<const uint4*>(q_nope + (static_cast<int64_t>(r0 + r) * H + h) * DH) + v);
    *reinterpret_cast<uint4*>(sq + r * LD + v * 8) = x;
  }
  const __nv_bfloat16* wh = w_uk + static_cast<int64_t>(h) * DC * DH;
#pragma unroll
  for (int idx = tid; idx < DC * VR; idx += kAbsorbThreads) {
    const int c = idx / VR, v = idx - c * VR;
    *reinterpret_cast<uint4*>(sw + c * LD + v * 8) = __ldg(reinterpret_cast<const uint4*>(wh + c * DH) + v);
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = 16 * (warp & 3);
  const int n0 = (warp >> 2) * (DC / 2);
  float acc[NSUB][4];
#pragma unroll
  for (int j = 0; j < NSUB; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll
  for (int k0 = 0; k0 < DH; k0 += 16) {
    const uint32_t a0 = ld_b32(sq + (m0 + g) * LD + k0 + 2 * t);
    const uint32_t a1 = ld_b32(sq + (m0 + g + 8) * LD + k0 + 2 * t);
    const uint32_t a2 = ld_b32(sq + (m0 + g) * LD + k0 + 2 * t + 8);
    const uint32_t a3 = ld_b32(sq + (m0 + g + 8) * LD + k0 + 2 * t + 8);
#pragma unroll
    for (int j = 0; j < NSUB; ++j) {
      const __nv_bfloat16* wb = sw + (n0 + 8 * j + g) * LD + k0 + 2 * t;
      mma_bf16_16816(acc[j], a0, a1, a2, a3, ld_b32(wb), ld_b32(wb + 8));
    }
  }
  // absorbed part: rows m0 + g and m0 + g + 8, columns n0 + 8 j + 2 t (+1)
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int r = m0 + g + 8 * half;
    if (r < nrows) {
      __nv_bfloat16* dst = q_out + (static_cast<int64_t>(r0 + r) * H + h) * DQ + n0 + 2 * t;
#pragma unroll
      for (int j = 0; j < NSUB; ++j)
        *reinterpret_cast<uint32_t*>(dst + 8 * j) = pack_bf16x2(acc[j][2 * half], acc[j][2 * half + 1]);
    }
  }
  // RoPE part of the same rows of head h
  const double lb = log(static_cast<double>(rope_base));
  const int np = d_R / 2;
  for (int idx = tid; idx < nrows * np; idx += kAbsorbThreads) {
    const int r = idx / np, i = idx - r * np;
    const int row = r0 + r, b = row / Lq, tq = row - b * Lq;
    const int pos = seqlens[b] - Lq + tq;
    const __nv_bfloat16* src = q_pe + (static_cast<int64_t>(row) * H + h) * d_R + 2 * i;
    float y0, y1;
    rope_pair(__bfloat162float(src[0]), __bfloat162float(src[1]), pos, i, d_R, lb, y0, y1);
    *reinterpret_cast<uint32_t*>(q_out + (static_cast<int64_t>(row) * H + h) * DQ + DC + 2 * i) = pack_bf16x2(y0, y1);
  }
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

template <int DH, int DC>
cudaError_t launch_absorb_t(const void* q_nope, const void* q_pe, const void* w_uk, const int32_t* seqlens,
                            int32_t B, int32_t Lq, int32_t H, int32_t d_R, float rope_base, void* q_out,
                            cudaStream_t stream) {
  constexpr int smem = (kRowsPerCta + DC) * (DH + 8) * 2;
  cudaError_t e = set_func_smem_once(reinterpret_cast<const void*>(absorb_query_kernel<DH, DC>), smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((B * Lq + kRowsPerCta - 1) / kRowsPerCta, H);
  absorb_query_kernel<DH, DC><<<grid, kAbsorbThreads, smem, stream>>>(
      static_cast<const __nv_bfloat16*>(q_nope), static_cast<const __nv_bfloat16*>(q_pe),
      static_cast<const __nv_bfloat16*>(w_uk), seqlens, B, Lq, H, d_R, rope_base,
      static_cast<__nv_bfloat16*>(q_out));
  return cudaGetLastError();
}

}  // namespace

bool absorb_supported(int d_h, int d_c) {
  return (d_h == 64 || d_h == 128) && (d_c == 128 || d_c == 256 || d_c == 512);
}

cudaError_t launch_absorb_query(const void* q_nope, const void* q_pe, const void* w_uk, const int32_t* seqlens,
                                int32_t B, int32_t Lq, int32_t H, int32_t d_h, int32_t d_c, int32_t d_R,
                                float rope_base, void* q_out, cudaStream_t stream) {
  if (B * Lq == 0) return cudaSuccess;
#define GLAD_ABS(DH, DC) \
  if (d_h == DH && d_c == DC) return launch_absorb_t<DH, DC>(q_nope, q_pe, w_uk, seqlens, B, Lq, H, d_R, rope_base, q_out, stream);
  GLAD_ABS(64, 128) GLAD_ABS(64, 256) GLAD_ABS(64, 512) GLAD_ABS(128, 128) GLAD_ABS(128, 256) GLAD_ABS(128, 512)
#undef GLAD_ABS
  return cudaErrorInvalidValue;
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
