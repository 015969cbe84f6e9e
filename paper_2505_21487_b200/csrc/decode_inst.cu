// Instantiations of the decode kernel family and the launcher.
#include "internal.h"

namespace glad {

namespace {

template <int DV, int DKN, int DR, int NQ, int T>
cudaError_t launch_one(const CUtensorMap& tmap, const CUtensorMap& lmap, const CUtensorMap& qmap, const DecodeParams& p, int grid, cudaStream_t stream) {
  using C = DecodeCfg<DV, DKN, DR, NQ, T>;
  static bool attr_set = false;  // benign race: idempotent attribute set
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  decode_kernel<C><<<grid, C::NTHREADS, C::SMEM_BYTES, stream>>>(tmap, lmap, qmap, p);
  return cudaGetLastError();
}

template <int DV, int DKN, int DR, int T>
cudaError_t launch_nq_t(int nq, const CUtensorMap& tmap, const CUtensorMap& lmap, const CUtensorMap& qmap, const DecodeParams& p, int grid,
                        cudaStream_t s) {
  switch (nq) {
    case 16: return launch_one<DV, DKN, DR, 16, T>(tmap, lmap, qmap, p, grid, s);
    case 32: return launch_one<DV, DKN, DR, 32, T>(tmap, lmap, qmap, p, grid, s);
    case 64: return launch_one<DV, DKN, DR, 64, T>(tmap, lmap, qmap, p, grid, s);
    default: return cudaErrorInvalidValue;
  }
}
template <int DV, int DKN, int DR>
cudaError_t launch_nq(int nq, int t, const CUtensorMap& tmap, const CUtensorMap& lmap, const CUtensorMap& qmap, const DecodeParams& p, int grid,
                      cudaStream_t s) {
  return t == 64 ? launch_nq_t<DV, DKN, DR, 64>(nq, tmap, lmap, qmap, p, grid, s)
                 : launch_nq_t<DV, DKN, DR, 128>(nq, tmap, lmap, qmap, p, grid, s);
}

}  // namespace

int decode_max_nq(int) { return 64; }

bool decode_supported(const DecodeKey& k) {
  if (k.nq != 16 && k.nq != 32 && k.nq != 64) return false;
  if (k.t != 64 && k.t != 128) return false;
  if (k.nq > decode_max_nq(k.d_v)) return false;
  if (k.d_kn == k.d_v) {  // GLA / MLA: key state == value state
    return (k.d_v == 128 && (k.d_r == 32 || k.d_r == 64)) || (k.d_v == 256 && (k.d_r == 32 || k.d_r == 64)) ||
           (k.d_v == 512 && k.d_r == 64);
  }
  return k.d_v == 128 && k.d_kn == 64 && k.d_r == 64;  // GTA, d_h = 128
}

cudaError_t launch_decode(const DecodeKey& k, const CUtensorMap& tmap, const CUtensorMap& lmap, const CUtensorMap& qmap, const DecodeParams& p, int grid,
                          cudaStream_t s) {
  if (!decode_supported(k)) return cudaErrorInvalidValue;
  if (k.d_kn == k.d_v) {
    if (k.d_v == 128 && k.d_r == 32) return launch_nq<128, 128, 32>(k.nq, k.t, tmap, lmap, qmap, p, grid, s);
    if (k.d_v == 128 && k.d_r == 64) return launch_nq<128, 128, 64>(k.nq, k.t, tmap, lmap, qmap, p, grid, s);
    if (k.d_v == 256 && k.d_r == 32) return launch_nq<256, 256, 32>(k.nq, k.t, tmap, lmap, qmap, p, grid, s);
    if (k.d_v == 256 && k.d_r == 64) return launch_nq<256, 256, 64>(k.nq, k.t, tmap, lmap, qmap, p, grid, s);
    if (k.d_v == 512 && k.d_r == 64) return launch_nq<512, 512, 64>(k.nq, k.t, tmap, lmap, qmap, p, grid, s);
  } else {
    return launch_nq<128, 64, 64>(k.nq, k.t, tmap, lmap, qmap, p, grid, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace glad
