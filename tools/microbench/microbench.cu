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

// Completion timeline of a burst of n <= 32 MMAs issued into an idle tensor
// pipe (one commit + mbarrier per MMA; warp 1 records when each completes).
// out[0..n) = completion cycle of MMA i relative to the first issue,
// out[32..32+n) = issue-return cycle of MMA i.  gap_mma: an earlier MMA issued
// `gap` cycles before the burst (probes whether an idle pipe "cools down").
__global__ void __launch_bounds__(128, 1) mma_burst_kernel(int which, int n, int gap, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[33];
  __shared__ uint32_t tslot;
  __shared__ long long t_start;
  const uint32_t sb = smem_u32(smem);
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) st_shared_v4(sb + i * 16, 0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { for (int i = 0; i < 33; ++i) mbar_init(&bars[i], 1); fence_barrier_init(); }
  if (threadIdx.x < 32) { tmem_alloc(&tslot, 256); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t A = sb, Bk = sb + 64 * 1024;
  const uint32_t idesc = make_idesc_bf16(128, 64, (which & 1) != 0, (which & 1) != 0);
  auto da = [&](int k) {
    return (which & 1) == 0 ? desc_kmajor_sw128(A + (k >> 2 & 3) * 16384 + (k & 3) * 32)
                      : desc_mnmajor_sw128(A + (k & 7) * 2048, 16384);
  };
  auto db = [&](int k) {
    return (which & 1) == 0 ? desc_kmajor_sw128(Bk + (k >> 2 & 3) * 8192 + (k & 3) * 32)
                      : desc_mnmajor_sw128(Bk + (k & 7) * 2048, 0);
  };
  if (threadIdx.x == 0) {
    if (gap >= 0) {  // one MMA, wait for it, idle `gap` cycles
      umma_f16_ss(tmem + 128, da(0), db(0), idesc, 0u);
      umma_commit(&bars[32]);
      mbar_wait(&bars[32], 0);
      const long long g0 = clock64();
      while (clock64() - g0 < gap) {}
    }
    const long long t0 = clock64();
    t_start = t0;
    __threadfence_block();
    const bool each = which >= 2;  // commit after every MMA (else only after the last)
    for (int i = 0; i < n; ++i) {
      umma_f16_ss(tmem, da(i), db(i), idesc, i != 0);
      if (each || i == n - 1) umma_commit(&bars[each ? i : 0]);
    }
    out[32 + n - 1] = clock64() - t0;
  } else if (threadIdx.x == 32) {
    long long t[32];
    const int nw = which >= 2 ? n : 1;
    for (int i = 0; i < nw; ++i) {
      while (!mbar_test_wait(smem_u32(&bars[i]), 0)) {}
      t[i] = clock64();
    }
    __syncwarp(1);
    for (int i = 0; i < nw; ++i) out[i] = t[i];
  }
  __syncthreads();
  if (threadIdx.x == 32)
    for (int i = 0; i < (which >= 2 ? n : 1); ++i) out[i] -= t_start;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 256); }
}

}  // namespace glad

extern "C" __attribute__((visibility("default"))) int glad_debug_mma_burst(int which, int n, int gap,
                                                                            long long* dev_out) {
  const int smem = 160 * 1024 + 1024;
  if (n < 1 || n > 32) return 1;
  cudaFuncSetAttribute(glad::mma_burst_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  glad::mma_burst_kernel<<<1, 128, smem>>>(which, n, gap, dev_out);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

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
