// int_peaks.cu -- measured per-SM-clock throughput of the integer / shared-memory instructions the
// local Jaccard kernel (k_local_tile) is built from, on the B200 it runs on.  These are the roofline
// denominators of bench.py's "alu" roofline ("Per-SM-clock throughput of IADD3 /
// LOP3 / POPC / IMAD / LDS"); the nominal CUDA-guide rates are NOT assumed.
//
// Each test runs a long unrolled loop of independent instructions (8 chains per thread, so latency
// is hidden), grid = 148 x 4 CTAs x 512 threads, timed with CUDA events; the SM clock during the run
// is read from clock64() deltas over the same interval.  Result: lane-ops per SM per clock and per
// second (whole chip).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peaks int_peaks.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define ITERS 4096
#define CH 8

__device__ unsigned long long g_sink;
__device__ long long g_cyc[4096];

template <int OP>
__global__ void __launch_bounds__(512) k_alu(uint32_t seed, int iters) {
  uint32_t a[CH], b = seed ^ threadIdx.x, c = seed * 7u + blockIdx.x;
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = seed + i * 0x9E3779B9u + threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b), "r"(c));   // LOP3 (xor3)
        if (OP == 1) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));                     // IADD
        if (OP == 2) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));       // IMAD
        if (OP == 3) {                                                                               // POPC (+IADD)
          uint32_t p;
          asm volatile("popc.b32 %0, %1;" : "=r"(p) : "r"(a[i] ^ u));
          a[i] += p;
        }
        if (OP == 4) asm volatile("shf.r.wrap.b32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));  // SHF
      }
    }
  }
  long long t1 = clock64();
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) x ^= a[i];
  if (x == 0x12345678u) g_sink = x;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

// LDS.32: conflict-free (lane-consecutive) or random (mask-lookup pattern of the probe)
template <bool RANDOM>
__global__ void __launch_bounds__(512) k_lds(uint32_t seed, int iters) {
  __shared__ uint32_t M[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) M[i] = i * 2654435761u;
  __syncthreads();
  uint32_t idx[CH], acc = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) idx[i] = RANDOM ? ((seed + threadIdx.x * 0x9E3779B9u + i * 7919u) & 8191u)
                                               : ((threadIdx.x & 31) + 32 * i + 512 * (threadIdx.x >> 5)) & 8191u;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const uint32_t v = M[idx[i]];
        acc ^= v;
        idx[i] = RANDOM ? ((idx[i] + (v | 1u) * 40503u) & 8191u) : ((idx[i] + 256u) & 8191u);
      }
    }
  }
  long long t1 = clock64();
  if (acc == 0x12345678u) g_sink = acc;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

static int sms() {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0);
  return n;
}

template <class K>
static void run(const char *name, K kern, double ops_per_thread_iter, int iters, int per_sm_blocks = 4) {
  const int S = sms(), blocks = S * per_sm_blocks, threads = 512;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(1u, 8);  // warm-up
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(1u, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long cyc[4096];
  cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(long long) * blocks);
  double mc = 0;
  for (int i = 0; i < blocks; ++i) mc = cyc[i] > mc ? cyc[i] : mc;
  const double ops = ops_per_thread_iter * iters * (double)blocks * threads;
  const double mhz = mc / (ms * 1e3);  // SM clock seen by the kernel (cycles per microsecond)
  const double per_sm_clk = ops / (S * mc / 1.0) / 1.0;  // lane-ops per SM per clock (CTAs run concurrently)
  printf("{\"op\": \"%s\", \"lane_ops_per_sm_per_clk\": %.1f, \"lane_ops_per_s\": %.4e, \"sm_mhz\": %.0f, "
         "\"ms\": %.3f, \"sms\": %d}\n",
         name, per_sm_clk * 1.0, ops / (ms * 1e-3), mhz, ms, S);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
}

int main() {
  // each inner step: 16 unrolled x CH chains; blocks = 4 per SM run concurrently (<= 2048 threads/SM)
  const double per = 16.0 * CH;
  run("LOP3", k_alu<0>, per, ITERS);
  run("IADD", k_alu<1>, per, ITERS);
  run("IMAD", k_alu<2>, per, ITERS);
  run("POPC", k_alu<3>, per, ITERS);  // popc + add: counts the POPC
  run("SHF", k_alu<4>, per, ITERS);
  run("LDS32_conflict_free", k_lds<false>, per, ITERS / 4);
  run("LDS32_random", k_lds<true>, per, ITERS / 4);
  return 0;
}
