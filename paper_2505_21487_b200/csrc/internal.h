// Internal (C++) interface between the C-ABI layer and the kernel launchers.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>

#include "decode.cuh"

#ifndef GLAD_PDL
#define GLAD_PDL 1  // programmatic dependent launch for plan -> decode -> merge
#endif

namespace glad {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device
// ordinal): the opt-in is a per-context attribute, so a process that drives
// several GPUs sets it on each (benign race: the set is idempotent).
inline cudaError_t set_func_smem_once(const void* func, int bytes) {
  constexpr int kMaxDev = 64;
  struct Flags { bool done[kMaxDev] = {}; };
  static std::mutex mu;
  static std::map<const void*, Flags> seen;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDev) return cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  std::lock_guard<std::mutex> lk(mu);
  bool& done = seen[func].done[dev];
  if (!done) {
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    done = true;
  }
  return cudaSuccess;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }();
  return fn;
}

// Kernel family key: value width, key-from-state width, rope width, query
// rows per CTA.
struct DecodeKey {
  int d_v, d_kn, d_r, nq, t;  // t: tokens per KV tile (64 / 96 / 128)
  int d_s;                    // state columns loaded per head (d_v, or d_kn + d_v for materialised K | V rows)
};

// Returns cudaErrorInvalidValue (and does not launch) if no instantiation
// matches `key`.
cudaError_t launch_decode(const DecodeKey& key, const CUtensorMap& tmap, const CUtensorMap& lmap, const CUtensorMap& qmap, const DecodeParams& p, int grid,
                          cudaStream_t stream);
bool decode_supported(const DecodeKey& key);
int decode_stages(const DecodeKey& key);                   // KV pipeline stages of the instantiation (0: unsupported)
bool decode_split(const DecodeKey& key);                   // split (lo / hi half) stage layout (DecodeCfg::SPLIT)
int decode_max_clusters(const DecodeKey& key, int cl_n);  // resident clusters of cl_n CTAs (0: error)
int decode_max_nq(int d_v);
bool decode_rows_supported(const DecodeKey& key);  // rows mode (nq = 128) exists for these dims (any t)

cudaError_t launch_plan(const int32_t* seqlens, int32_t* plan, int U, int seg_cost, int cl_n, int B, int tile, int n_qblk,
                        int qb_outer, int nq_blk, int Lq, int g_q, int causal, int H, int d_v, void* out, float* lse,
                        uint64_t* trace, cudaStream_t stream);
cudaError_t launch_merge_split(const int32_t* plan, const float* o_part, const float* lse_part, int G, int cl_n,
                               int U, int nq_blk, int n_qblk, int qb_outer, int B, int n_groups, int g_q, int Lq,
                               int H, int d_v, int seg_cost, void* out, float* lse, cudaStream_t stream);
cudaError_t launch_append(void* pool, int64_t row_stride, int page_size, const int32_t* block_table,
                          int32_t bt_stride, const int32_t* seqlens_before, const void* rows, int32_t B,
                          int32_t n_new, int32_t width, cudaStream_t stream);
cudaError_t launch_gather(const void* pool, int64_t row_stride, int page_size, const int32_t* block_table,
                          int32_t bt_stride, const int32_t* seqlens, int32_t B, int32_t max_len, int32_t width,
                          void* dense_out, cudaStream_t stream);
bool absorb_supported(int d_h, int d_c);
cudaError_t launch_absorb_query(const void* q_nope, const void* q_pe, const void* w_uk, const int32_t* seqlens,
                                int32_t B, int32_t Lq, int32_t H, int32_t d_h, int32_t d_c, int32_t d_R,
                                float rope_base, void* q_out, cudaStream_t stream);
cudaError_t launch_append_rope(void* pool, int64_t row_stride, int page_size, const int32_t* block_table,
                               int32_t bt_stride, const int32_t* seqlens_before, const void* latent,
                               const void* k_pe, int32_t B, int32_t n_new, int32_t w_lat, int32_t d_R,
                               float rope_base, cudaStream_t stream);
// materialised GLA prefill helpers (prefill.cu)
cudaError_t launch_prefill_upproj(const void* latent, const void* w, int32_t B, int32_t Lmax, int32_t Lpad,
                                  int32_t h_c, int32_t d_c, int32_t H, int32_t d_h, void* kv, int64_t row_stride,
                                  int32_t col_off, cudaStream_t s);
cudaError_t launch_prefill_build_q(const void* q_nope, const void* q_pe, const int32_t* seqlens, int32_t B,
                                   int32_t Lmax, int32_t H, int32_t d_h, int32_t d_R, double log2_base, void* q_full,
                                   cudaStream_t s);
cudaError_t launch_prefill_rope_k(const void* k_pe, int32_t B, int32_t Lmax, int32_t Lpad, int32_t d_R,
                                  double log2_base, void* kv, int64_t row_stride, int64_t rope_col, cudaStream_t s);
cudaError_t launch_prefill_identity_bt(int32_t* bt, int32_t B, int32_t npg, cudaStream_t s);
cudaError_t launch_prefill_shift_out(const void* out_full, const float* lse_full, const int32_t* seqlens, int32_t B,
                                     int32_t Lmax, int32_t H, int32_t d_h, void* out, float* lse, cudaStream_t s);
cudaError_t launch_lse_rescale(const float* lse_all, int32_t P, int32_t rank, const void* o, int64_t rows,
                               int32_t d_v, void* o_out, float* lse_out, cudaStream_t stream);
cudaError_t launch_combine(const float* o_part, const float* lse_part, int32_t S, int64_t rows, int32_t d_v,
                           void* out, float* lse, cudaStream_t stream);

}  // namespace glad
