// Decode kernel family: supported keys and the launcher (the instantiations
// live in decode_inst_t{64,96,128}.cu).
#include "decode_inst.h"

namespace glad {

int decode_max_nq(int) { return 64; }

bool decode_rows_supported(const DecodeKey& k) {
  if (k.d_s == 2 * k.d_v) return k.d_v == 128 && k.d_kn == 128 && k.d_r == 64;  // materialised prefill rows
  if (k.d_kn == 64 && k.d_v == 128 && k.d_r == 64) return true;                   // GTA
  return k.d_kn == k.d_v && (k.d_v == 128 || k.d_v == 256) && (k.d_r == 32 || k.d_r == 64);
}

bool decode_supported(const DecodeKey& k) {
  if (k.t != 64 && k.t != 96 && k.t != 128) return false;
  // rows mode: 64- and 96-token tiles whose S buffers, O and the query
  // state part fit TMEM (rows_fits; 128-token tiles faulted on the second
  // tile when they still fitted, before Q moved to TMEM)
  if (k.nq == 128) return decode_rows_supported(k) && (k.t == 64 || k.t == 96) && 2 * k.t + k.d_v + k.d_kn / 2 <= 512;
  if (k.d_s != k.d_v) return false;  // materialised rows: rows mode only
  if (k.nq != 16 && k.nq != 32 && k.nq != 64) return false;
  if (k.nq > decode_max_nq(k.d_v)) return false;
  if (k.d_kn == k.d_v) {  // GLA / MLA: key state == value state
    return (k.d_v == 128 && (k.d_r == 32 || k.d_r == 64)) || (k.d_v == 256 && (k.d_r == 32 || k.d_r == 64)) ||
           (k.d_v == 512 && k.d_r == 64);
  }
  return k.d_v == 128 && k.d_kn == 64 && k.d_r == 64;  // GTA, d_h = 128
}

static int stages_and_split(const DecodeKey& k) {
  if (!decode_supported(k)) return 0;
  return k.t == 64 ? decode_stages_t<64>(k) : k.t == 96 ? decode_stages_t<96>(k) : decode_stages_t<128>(k);
}

int decode_stages(const DecodeKey& k) { return stages_and_split(k) & 0xff; }

bool decode_split(const DecodeKey& k) { return (stages_and_split(k) & 0x100) != 0; }

int decode_max_clusters(const DecodeKey& k, int cl_n) {
  if (!decode_supported(k)) return 0;
  return k.t == 64 ? decode_max_clusters_t<64>(k, cl_n)
                   : k.t == 96 ? decode_max_clusters_t<96>(k, cl_n) : decode_max_clusters_t<128>(k, cl_n);
}

cudaError_t launch_decode(const DecodeKey& k, const CUtensorMap& tmap, const CUtensorMap& lmap,
                          const CUtensorMap& qmap, const DecodeParams& p, int grid, cudaStream_t s) {
  if (!decode_supported(k)) return cudaErrorInvalidValue;
  if (k.t == 64) return launch_decode_t<64>(k, tmap, lmap, qmap, p, grid, s);
  if (k.t == 96) return launch_decode_t<96>(k, tmap, lmap, qmap, p, grid, s);
  return launch_decode_t<128>(k, tmap, lmap, qmap, p, grid, s);
}

}  // namespace glad
