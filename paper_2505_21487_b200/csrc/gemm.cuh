// Batched bf16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA)
// for the steps around the decode hot path: the query absorption of the
// upstream step (q_abs[h] = W_UK[h] q_nope[h]) and the per-head K / V
// up-projection of the materialised prefill (K_h = c W_UK[h], V_h = c W_UV[h],
// P:48 sigma(Q K^T + Q_R K_R^T) V with K, V materialised).
//
//   D[z][m][n] = sum_k A[z][m][k] * B[z][n][k]      (fp32 accumulation in TMEM)
//
// One CTA per (128-row M tile, BN-column N tile, batch z).  A is K-major
// (k contiguous), loaded as [128 rows][64 k] 128B-swizzled boxes of a 3-D
// tensor map whose coordinates are (k, a1, a2) = (k, z / a_div, m) (batch on
// the middle dimension: per-head slices of [rows][heads][k] tensors); B is
// K-major ([BN rows][64 k] boxes at (k, n, z)) or MN-major ([64 k][64 n]
// boxes at (n, k, z): a weight stored [z][k][n]).  Warp 0 issues TMA into a
// KSTAGES-deep ring, warp 1 issues tcgen05.mma (M = 128, N = BN, K = 16),
// all four warps then read the accumulator (one row per thread) and write
// bf16 rows with 16-byte stores.  An optional RoPE epilogue (absorbed query)
// rotates a second input's pairs at the row's position and writes them next
// to the product.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "internal.h"
#include "ptx.cuh"

namespace glad {

#ifndef GLAD_ROPE_FP32
#define GLAD_ROPE_FP32 0
#endif

struct GemmParams {
  int32_t M, N, K;          // per batch
  int32_t a_div;            // A's batch coordinate = z / a_div
  __nv_bfloat16* out;       // D[z][m][n] at out + z * out_bstride + row(m) * out_ld + n
  int64_t out_ld, out_bstride;
  int32_t seg_len, seg_pad;  // row(m) = (m / seg_len) * seg_pad + m % seg_len (seg_len = 0: row(m) = m)
  // optional RoPE epilogue (absorbed query, R5): rows m = b * Lq + t at position
  // seqlens[b] - Lq + t; pairs of rope_src + (m * rope_ld + z * rope_bstride)
  // rotated into out + z * out_bstride + m * out_ld + rope_col
  const __nv_bfloat16* rope_src;
  const int32_t* seqlens;
  int64_t rope_ld, rope_bstride;
  int32_t rope_col, d_rope, Lq;
  double log2_base;         // log2(rope base), fp64 (an fp32 log shifts the angle by ~1e-5 rad at 1K)
};

template <int BN, bool B_MN, int KS = 4>
struct GemmCfg {
  static constexpr int BK = 64;                        // k per stage (one 128-B swizzle row)
  static constexpr int A_BYTES = 128 * BK * 2;         // 16 KB
  static constexpr int B_BYTES = BN * BK * 2;          // BN x 64 bf16
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int KSTAGES = (200 * 1024) / STAGE > KS ? KS : (200 * 1024) / STAGE;
  static constexpr int SMEM = 1024 + KSTAGES * STAGE + 128 + 64 * 8;  // + barriers, TMEM slot, RoPE table
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static_assert(BN % 64 == 0 && BN <= 256, "BN");
  static_assert(KSTAGES >= 1, "stages");
};

// RoPE pair (R5): angle pos * theta_i, theta_i = base^(-2i/d), reduced mod
// 2 pi and rotated in fp64 (positions up to 64K; the rotation of a pair can
// cancel, so the result is only one bf16 rounding away from the fp64 value
// when sin / cos and the products are fp64).
__device__ __forceinline__ void rope_rotate_pair(float x0, float x1, int pos, double theta, float& y0, float& y1) {
  double a = static_cast<double>(pos) * theta;
  a -= rint(a * 0.15915494309189535) * 6.283185307179586;
#if GLAD_ROPE_FP32
  float s, c;
  sincosf(static_cast<float>(a), &s, &c);
  y0 = x0 * c - x1 * s;
  y1 = x0 * s + x1 * c;
#else
  double s, c;
  sincos(a, &s, &c);
  y0 = static_cast<float>(x0 * c - x1 * s);
  y1 = static_cast<float>(x0 * s + x1 * c);
#endif
}

template <int BN, bool B_MN, int KS>
__global__ void __launch_bounds__(256)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                     const GemmParams p) {
  using C = GemmCfg<BN, B_MN, KS>;
  constexpr int NS = C::KSTAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * C::STAGE);
  uint64_t* empty = full + 4;
  uint64_t* done = full + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(full + 9);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * BN, z = blockIdx.z;
  const int nk = p.K / C::BK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, C::TMEM_COLS);
    tmem_relinquish();
  }
  double* theta_s = reinterpret_cast<double*>(full + 16);  // [d_rope / 2] RoPE frequencies (fp64)
  if (p.rope_src != nullptr && threadIdx.x < p.d_rope / 2)
    theta_s[threadIdx.x] = exp2(-2.0 * threadIdx.x / p.d_rope * p.log2_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer (one lane)
    if (lane == 0) {
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % NS;
        mbar_wait(&empty[s], ((kc / NS) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], C::STAGE);
        const uint32_t sa = sbase + s * C::STAGE, sb = sa + C::A_BYTES;
        tma_load_3d(sa, &tmap_a, &full[s], kc * C::BK, z / p.a_div, m0);
        if constexpr (B_MN) {
#pragma unroll
          for (int j = 0; j < BN / 64; ++j)  // [64 k][64 n] per 64-column block
            tma_load_3d(sb + j * (C::BK * 128), &tmap_b, &full[s], n0 + 64 * j, kc * C::BK, z);
        } else {
          tma_load_3d(sb, &tmap_b, &full[s], kc * C::BK, n0, z);
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer (one elected lane per instruction)
    constexpr uint32_t idesc = make_idesc_bf16(128, BN, false, B_MN);
    for (int kc = 0; kc < nk; ++kc) {
      const int s = kc % NS;
      mbar_wait(&full[s], (kc / NS) & 1);
      tc_fence_after();
      const uint32_t sa = sbase + s * C::STAGE, sb = sa + C::A_BYTES;
      const uint64_t ad = desc_kmajor_sw128(sa);
      const uint64_t bd = B_MN ? desc_mnmajor_sw128(sb, C::BK * 128, 1024) : desc_kmajor_sw128(sb);
#pragma unroll
      for (int k = 0; k < C::BK / 16; ++k)
        umma_f16_ss_warp(tmem, ad + static_cast<uint64_t>((k * 32) >> 4),
                         bd + static_cast<uint64_t>((B_MN ? k * 2048 : k * 32) >> 4), idesc, (kc | k) != 0);
      umma_commit_warp(&empty[s]);
    }
    umma_commit_warp(done);
  }
  __syncwarp();

  // ---- RoPE part (absorbed query): computed while the TMA loads and MMAs of
  // the product are in flight (fp64 angle / rotation, theta_i from a table)
#ifndef GLAD_DBG_NO_ROPE
  if (p.rope_src != nullptr && warp >= 4) {
#else
  if (false) {
#endif
    // ---- RoPE part (absorbed query), warps 4-7, concurrently with the
    // product's loads / MMAs / epilogue (fp64 angle, theta_i from a table).
    // The CTAs of the N tiles of a row block share the pairs; consecutive
    // threads take consecutive pairs of a row (coalesced 4-byte accesses).
    const int np = p.d_rope / 2, per = (np + gridDim.y - 1) / gridDim.y;
    const int i0 = blockIdx.y * per, npl = min(np, i0 + per) - i0;
    const int nrow = min(128, p.M - m0);
    const int tid = threadIdx.x - 128;
#pragma unroll 4  // independent pairs: overlap the load and sincos latencies
    for (int idx = tid; idx < nrow * npl; idx += 128) {
      const int rl = idx / npl, i = i0 + (idx - rl * npl);
      const int row_r = m0 + rl;
      const int b = row_r / p.Lq, t = row_r - b * p.Lq;
      const int pos = __ldg(p.seqlens + b) - p.Lq + t;
      const uint32_t x = __ldg(reinterpret_cast<const unsigned int*>(
          p.rope_src + static_cast<int64_t>(row_r) * p.rope_ld + static_cast<int64_t>(z) * p.rope_bstride + 2 * i));
      float y0, y1;
      rope_rotate_pair(__uint_as_float(x << 16), __uint_as_float(x & 0xffff0000u), pos, theta_s[i], y0, y1);
      *reinterpret_cast<uint32_t*>(p.out + static_cast<int64_t>(z) * p.out_bstride +
                                   static_cast<int64_t>(row_r) * p.out_ld + p.rope_col + 2 * i) = pack_bf16x2(y0, y1);
    }
  }

  // ---- epilogue (warps 0-3): row m0 + threadIdx.x, BN columns
  if (warp < 4) {
  mbar_wait(done, 0);
  tc_fence_after();
  const int row = m0 + threadIdx.x;
  const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  const int64_t orow_idx = p.seg_len ? static_cast<int64_t>(row / p.seg_len) * p.seg_pad + row % p.seg_len : row;
  __nv_bfloat16* orow = p.out + static_cast<int64_t>(z) * p.out_bstride + orow_idx * p.out_ld + n0;
#pragma unroll 1
  for (int c = 0; c < BN; c += 32) {
    float v[32];
    tmem_ld32(taddr + c, v);
    tmem_ld_wait();
    if (row < p.M && n0 + c < p.N) {
#pragma unroll
      for (int q = 0; q < 32; q += 8)
        *reinterpret_cast<uint4*>(orow + c + q) =
            make_uint4(pack_bf16x2(v[q], v[q + 1]), pack_bf16x2(v[q + 2], v[q + 3]),
                       pack_bf16x2(v[q + 4], v[q + 5]), pack_bf16x2(v[q + 6], v[q + 7]));
    }
  }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int BN, bool B_MN, int KS = 4>
cudaError_t launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, dim3 grid,
                        cudaStream_t stream) {
  using C = GemmCfg<BN, B_MN, KS>;
  cudaError_t e = set_func_smem_once(reinterpret_cast<const void*>(gemm_bf16_kernel<BN, B_MN, KS>), C::SMEM);
  if (e != cudaSuccess) return e;
  gemm_bf16_kernel<BN, B_MN, KS><<<grid, p.rope_src ? 256 : 128, C::SMEM, stream>>>(ta, tb, p);
  return cudaGetLastError();
}

}  // namespace glad
