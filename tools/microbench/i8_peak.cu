// i8_peak.cu -- measured dense int8 tensor-core rate of tcgen05.mma.cta_group::1.kind::i8 on this
// B200 (SURVEY.md App. D "Dense tcgen05.mma.kind::i8 peak"), the denominator of the "dense head"
// design the survey proposed for the local Jaccard kernel (|P_u ∩ P_v| as a 0/1 contraction over
// cluster-local items).  One CTA per SM, one elected thread issues back-to-back
// M=128 x N=256 x K=32 MMAs (s8 x s8 -> s32, accumulator in TMEM, operands in shared memory,
// SWIZZLE_NONE K-major); completion via tcgen05.commit -> mbarrier.  Operand contents are zero (the
// rate does not depend on values).  Also checks that the product of known operands is right on a
// small case (A = 1, B = 1 -> every accumulator = K * iterations), read back with tcgen05.ld.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8_peak i8_peak.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int M = 128, N = 256, KB = 32;  // K = 32 bytes per MMA (int8)

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
  return d;
}

__host__ __device__ constexpr uint32_t idesc_i8() {
  // c_format S32 = 2 at [4,6); a_format S8 = 1 at [7,10); b_format S8 = 1 at [10,13);
  // a/b K-major (0); N >> 3 at [17,23); M >> 4 at [24,29)
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void __launch_bounds__(128, 1) k_i8(int iters, int8_t fill, long long *cycles, int *ok, int *acc_out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *A = sm, *B = sm + M * KB;  // core matrices (8 rows x 16 B) contiguous: [row-block][k-block]
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  for (int i = threadIdx.x; i < (M + N) * KB; i += blockDim.x) sm[i] = (uint8_t)fill;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");  // operand writes visible to the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(A), sb = (uint32_t)__cvta_generic_to_shared(B);
  // K-major, no swizzle: core matrix (8 rows x 16 B) = 128 B; the 2 core matrices along K are 128 B
  // apart (LBO), consecutive 8-row groups 256 B apart (SBO)
  const uint64_t da = smem_desc(sa, 128, 256), db = smem_desc(sb, 128, 256);
  const uint32_t id = idesc_i8();
  long long t0 = 0, t1 = 0;
  int good = 1;
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t accum = it > 0 ? 1u : 0u;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(id), "r"(accum));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&mbar)));
    // bounded wait on phase 0 (a broken MMA must not hang the GPU)
    uint32_t done = 0;
    for (long long spin = 0; spin < 200000000LL && !done; ++spin) {
      asm volatile(
          "{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n\tselp.u32 %0, 1, 0, q;\n\t}\n"
          : "=r"(done)
          : "r"((uint32_t)__cvta_generic_to_shared(&mbar)));
    }
    t1 = clock64();
    good = done ? 1 : 0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // read back accumulator lane (row) = threadIdx.x, first 4 columns
  uint32_t r0, r1, r2, r3;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  if (blockIdx.x == 0 && threadIdx.x < M) acc_out[threadIdx.x] = (int)r0;
  (void)r1, (void)r2, (void)r3;
  if (threadIdx.x == 0) {
    cycles[blockIdx.x] = t1 - t0;
    ok[blockIdx.x] = good;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

int main() {
  int S = 0;
  cudaDeviceGetAttribute(&S, cudaDevAttrMultiProcessorCount, 0);
  long long *cyc;
  int *ok, *acc;
  cudaMalloc(&cyc, S * sizeof(long long));
  cudaMalloc(&ok, S * sizeof(int));
  cudaMalloc(&acc, M * sizeof(int));
  const int smem = (M + N) * KB;
  cudaFuncSetAttribute(k_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // 1. correctness: A = B = 1 (s8), 3 MMAs -> every accumulator = 3 * 32
  k_i8<<<1, 128, smem>>>(3, 1, cyc, ok, acc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 1;
  }
  int hacc[M], hok = 0;
  cudaMemcpy(hacc, acc, sizeof(hacc), cudaMemcpyDeviceToHost);
  cudaMemcpy(&hok, ok, sizeof(int), cudaMemcpyDeviceToHost);
  int right = 0;
  for (int i = 0; i < M; ++i) right += hacc[i] == 3 * KB;
  printf("{\"check\": \"A=B=1, 3 MMAs\", \"completed\": %d, \"rows_equal_96\": %d, \"acc0\": %d}\n", hok, right, hacc[0]);
  // 2. rate: one CTA per SM, back-to-back MMAs
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_i8<<<S, 128, smem>>>(100, 0, cyc, ok, acc);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k_i8<<<S, 128, smem>>>(iters, 0, cyc, ok, acc);
  cudaEventRecord(e1);
  e = cudaEventSynchronize(e1);
  if (e != cudaSuccess) {
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 1;
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long *hc = new long long[S];
  int *hk = new int[S];
  cudaMemcpy(hc, cyc, S * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaMemcpy(hk, ok, S * sizeof(int), cudaMemcpyDeviceToHost);
  long long mc = 0;
  int nok = 0;
  for (int i = 0; i < S; ++i) {
    mc = hc[i] > mc ? hc[i] : mc;
    nok += hk[i];
  }
  const double macs = (double)M * N * KB * iters * S;
  printf("{\"op\": \"tcgen05.mma.cta_group::1.kind::i8 M128 N256 K32\", \"ctas_completed\": %d, \"sms\": %d, "
         "\"ms\": %.3f, \"tops\": %.1f, \"macs_per_sm_per_clk\": %.0f, \"sm_mhz\": %.0f}\n",
         nok, S, ms, 2.0 * macs / (ms * 1e-3) / 1e12, (double)M * N * KB * iters / (double)mc, mc / (ms * 1e3));
  return 0;
}
