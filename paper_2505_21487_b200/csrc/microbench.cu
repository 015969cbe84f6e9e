// Debug microbenchmark: cycles per tcgen05.mma for the operand layouts the
// decode kernel uses (one CTA, one issuing thread, operands resident in smem).
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace glad {

// which: 0 = A K-major SW128 / B K-major SW128            (QK)
//        1 = A MN-major SW128 / B MN-major no-swizzle      (PV, current P^T layout)
//        2 = A MN-major SW128 / B MN-major SW128           (PV with a swizzled P^T)
//        3 = A MN-major SW128 / B K-major SW128            (PV with K-major P^T)
template <int N>
__global__ void __launch_bounds__(128, 1) mma_bench_kernel(int which, int iters, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t sb = smem_u32(smem);
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) st_shared_v4(sb + i * 16, 0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) { tmem_alloc(&tslot, 256); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t A = sb, Bk = sb + 64 * 1024;
    const uint32_t idesc = make_idesc_bf16(128, N, which != 0, which == 1 || which == 2);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        uint64_t a, b;
        if (which == 0) {
          a = desc_kmajor_sw128(A + (k >> 2) * 16384 + (k & 3) * 32);
          b = desc_kmajor_sw128(Bk + (k >> 2) * (N * 128) + (k & 3) * 32);
        } else {
          a = desc_mnmajor_sw128(A + (k & 7) * 2048, 16384);
          if (which == 1) b = desc_mnmajor_noswz(Bk + (k & 7) * 256, 128, 2048);
          else if (which == 2) b = desc_mnmajor_sw128(Bk + (k & 7) * 2048, 16384);
          else b = desc_kmajor_sw128(Bk + (k >> 2 & 1) * (N * 128) + (k & 3) * 32);
        }
        umma_f16_ss(tmem, a, b, idesc, (it | k) != 0);
      }
    }
    const long long ti = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out[0] = t1 - t0;
    out[1] = static_cast<long long>(iters) * 16;
    out[2] = ti - t0;  // time spent issuing (blocks when the MMA queue is full)
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 256); }
}

}  // namespace glad

extern "C" __attribute__((visibility("default"))) int glad_debug_mma_bench(int which, int n, int iters,
                                                                            long long* dev_out) {
  const int smem = 160 * 1024 + 1024;
  cudaError_t e;
  switch (n) {
    case 16:
      cudaFuncSetAttribute(glad::mma_bench_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      glad::mma_bench_kernel<16><<<1, 128, smem>>>(which, iters, dev_out);
      break;
    case 64:
      cudaFuncSetAttribute(glad::mma_bench_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      glad::mma_bench_kernel<64><<<1, 128, smem>>>(which, iters, dev_out);
      break;
    case 128:
      cudaFuncSetAttribute(glad::mma_bench_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      glad::mma_bench_kernel<128><<<1, 128, smem>>>(which, iters, dev_out);
      break;
    default:
      return 1;
  }
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 4;
}
