// Instantiation helpers shared by the decode_inst_t*.cu translation units
// (one per tile height, compiled in parallel).
#pragma once
#include "internal.h"

namespace glad {

// The > 48 KB dynamic shared memory opt-in is a per-device (per-context)
// function attribute: cached per device ordinal, set on first use on each.
template <class C, int SP>
cudaError_t set_smem_attr() {
  return set_func_smem_once(reinterpret_cast<const void*>(decode_kernel<C, SP>), C::SMEM_BYTES);
}

template <int DV, int DKN, int DR, int NQ, int T, int DS>
cudaError_t launch_one(const CUtensorMap& tmap, const CUtensorMap& lmap, const CUtensorMap& qmap,
                       const DecodeParams& p, int grid, cudaStream_t stream) {
  using C = DecodeCfg<DV, DKN, DR, NQ, T, DS>;
  // pages < 16: the gather4 / hybrid (SP 1) or cp.async (SP 2) instantiation
  const int sp = p.cp_kv ? 2 : (p.g4 ? 1 : 0);
  cudaError_t e = sp == 2 ? set_smem_attr<C, 2>() : sp == 1 ? set_smem_attr<C, 1>() : set_smem_attr<C, 0>();
  if (e != cudaSuccess) return e;
  // PDL: the prologue overlaps the plan kernel's tail (griddep_wait in the kernel)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(C::NTHREADS);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (GLAD_PDL) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (p.cl_n > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = p.cl_n;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return sp == 2   ? cudaLaunchKernelEx(&cfg, decode_kernel<C, 2>, tmap, lmap, qmap, p)
         : sp == 1 ? cudaLaunchKernelEx(&cfg, decode_kernel<C, 1>, tmap, lmap, qmap, p)
                   : cudaLaunchKernelEx(&cfg, decode_kernel<C, 0>, tmap, lmap, qmap, p);
}

// Calls f.template run<C>() for the DecodeCfg matching (key, T); returns
// cudaErrorInvalidValue for an unsupported key.
template <int T, class F>
cudaError_t with_cfg(const DecodeKey& k, F&& f) {
#define GLAD_NQ(DV, DKN, DR)                                                  \
  switch (k.nq) {                                                             \
    case 16: return f.template run<DecodeCfg<DV, DKN, DR, 16, T>>();          \
    case 32: return f.template run<DecodeCfg<DV, DKN, DR, 32, T>>();          \
    case 64: return f.template run<DecodeCfg<DV, DKN, DR, 64, T>>();          \
    default: return cudaErrorInvalidValue;                                    \
  }
  // rows mode (128 query rows per CTA on UMMA M): GLA / MLA with d_c <= 256
#define GLAD_NQ_R(DV, DR)                                                     \
  switch (k.nq) {                                                             \
    case 16: return f.template run<DecodeCfg<DV, DV, DR, 16, T>>();           \
    case 32: return f.template run<DecodeCfg<DV, DV, DR, 32, T>>();           \
    case 64: return f.template run<DecodeCfg<DV, DV, DR, 64, T>>();           \
    case 128:                                                                 \
      if constexpr (rows_fits<DV, DV, T>()) return f.template run<DecodeCfg<DV, DV, DR, 128, T>>(); \
      else return cudaErrorInvalidValue;                                      \
    default: return cudaErrorInvalidValue;                                    \
  }
  if (k.d_s == 2 * k.d_v) {  // materialised [K_h | V_h] rows (prefill): rows mode only
    if (k.d_v == 128 && k.d_kn == 128 && k.d_r == 64 && k.nq == 128) {
      if constexpr (rows_fits<128, 128, T>()) return f.template run<DecodeCfg<128, 128, 64, 128, T, 256>>();
    }
    return cudaErrorInvalidValue;
  }
  if (k.d_kn == k.d_v) {
    if (k.d_v == 128 && k.d_r == 32) { GLAD_NQ_R(128, 32) }
    if (k.d_v == 128 && k.d_r == 64) { GLAD_NQ_R(128, 64) }
    if (k.d_v == 256 && k.d_r == 32) { GLAD_NQ_R(256, 32) }
    if (k.d_v == 256 && k.d_r == 64) { GLAD_NQ_R(256, 64) }
    if (k.d_v == 512 && k.d_r == 64) { GLAD_NQ(512, 512, 64) }
  } else if (k.d_v == 128 && k.d_kn == 64 && k.d_r == 64) {  // GTA (tied state, key = its first half)
    if (k.nq == 128) {
      if constexpr (rows_fits<128, 64, T>()) return f.template run<DecodeCfg<128, 64, 64, 128, T>>();
      return cudaErrorInvalidValue;
    }
    GLAD_NQ(128, 64, 64)
  }
#undef GLAD_NQ
#undef GLAD_NQ_R
  return cudaErrorInvalidValue;
}

struct LaunchF {
  const CUtensorMap &tmap, &lmap, &qmap;
  const DecodeParams& p;
  int grid;
  cudaStream_t s;
  template <class C>
  cudaError_t run() {
    return launch_one<C::D_V, C::D_KN, C::D_R, C::NQ, C::T, C::D_S>(tmap, lmap, qmap, p, grid, s);
  }
};

// How many clusters of `cl_n` decode CTAs can be resident at once (a
// persistent grid must not exceed it: clusters live inside one GPC).
struct ClustersF {
  int cl_n;
  int* out;
  template <class C>
  cudaError_t run() {
    cudaError_t e = set_smem_attr<C, 0>();  // clusters: pages >= 16 only
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cl_n * 64);
    cfg.blockDim = dim3(C::NTHREADS);
    cfg.dynamicSmemBytes = C::SMEM_BYTES;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl_n;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaOccupancyMaxActiveClusters(out, decode_kernel<C, 0>, &cfg);
  }
};

struct StagesF {
  int* ns;
  template <class C>
  cudaError_t run() {
    *ns = C::NS | (C::SPLIT ? 0x100 : 0);
    return cudaSuccess;
  }
};

template <int T>
cudaError_t launch_decode_t(const DecodeKey& k, const CUtensorMap& tmap, const CUtensorMap& lmap,
                            const CUtensorMap& qmap, const DecodeParams& p, int grid, cudaStream_t s);
template <int T>
int decode_stages_t(const DecodeKey& k);
template <int T>
int decode_max_clusters_t(const DecodeKey& k, int cl_n);

#define GLAD_INSTANTIATE_T(T)                                                                              \
  template <>                                                                                              \
  cudaError_t launch_decode_t<T>(const DecodeKey& k, const CUtensorMap& tmap, const CUtensorMap& lmap,     \
                                 const CUtensorMap& qmap, const DecodeParams& p, int grid, cudaStream_t s) { \
    return with_cfg<T>(k, LaunchF{tmap, lmap, qmap, p, grid, s});                                          \
  }                                                                                                        \
  template <>                                                                                              \
  int decode_stages_t<T>(const DecodeKey& k) {                                                             \
    int ns = 0;                                                                                            \
    return with_cfg<T>(k, StagesF{&ns}) == cudaSuccess ? ns : 0; /* NS | SPLIT << 8 */                      \
  }                                                                                                        \
  template <>                                                                                              \
  int decode_max_clusters_t<T>(const DecodeKey& k, int cl_n) {                                             \
    int n = 0;                                                                                             \
    return with_cfg<T>(k, ClustersF{cl_n, &n}) == cudaSuccess ? n : 0;                                     \
  }

}  // namespace glad
