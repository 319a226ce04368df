// c2_internal.cuh -- internals of libc2 (B200, sm_100a).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <map>
#include <vector>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "../../include/c2.h"

// NVTX range for the lifetime of a scope (phases of a build, for nsys/ncu timelines)
struct C2Range {
  explicit C2Range(const char *name) { nvtxRangePushA(name); }
  ~C2Range() { nvtxRangePop(); }
};

#define C2_MAX_T 64
#define C2_MAX_K 64
#define C2_SKETCH_D 8
#define C2_ABSENT16 ((uint16_t)0xFFFF)

struct c2_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  size_t smem_optin = 0;
  char err[512] = {0};
  // options
  int sketch_depth = C2_SKETCH_D;
  bool sync_check = false;
  bool timing = false;
  unsigned long long *kstats = nullptr;
  int clustering = 0;
  int func_offset = 0;  // C2_OPT_FUNC_OFFSET
  int solver = 0;       // C2_OPT_LOCAL_SOLVER: 0 brute force everywhere (A12), 1 Alg. 2 hybrid (Hyrec)
  uint64_t hyrec_seed = 0;  // the call's seed (Hyrec's random initial graphs)   // C2_OPT_CLUSTERING: 0 FastRandomHash (Step 1 of C^2), 1 MinHash (N3 variant)
  int surv_qmax = 2048;  // C2_OPT_SURVIVORS: light-row survivor slots per user (0: off; capped to 16 GiB of slots)
  bool gf_tensor = false;  // C2_OPT_GF_TENSOR: GoldFinger big clusters on the tensor cores (k_gf_mma; measured slower, off)
  bool presketched = false;  // c2_build_host: the sketch of the next fastrandomhash call is already in "sketch"
  cudaStream_t side_stream = nullptr;  // Step 2: light rows' merge concurrent with the per-row top-k
  cudaEvent_t side_ev[2] = {};
  cudaStream_t copy_stream = nullptr;  // c2_build_host: chunked H2D upload overlapping validation + sketch
  cudaEvent_t chunk_ev[16] = {};
  bool split_dev = true;  // C2_OPT_SPLIT_DEVICE: device-side split loop (k_split_dev)
  bool relabel = true;  // C2_OPT_RELABEL  (C2_OPT_KSTATS: kstats = dev [80] K7/K8 counters)
  c2_stats stats{};
  // device workspace: name -> (ptr, bytes); grow-only
  std::map<std::string, std::pair<void *, size_t>> ws;
  // pinned host staging for small D2H reads
  int64_t *h_small = nullptr;
  int64_t *d_small = nullptr;
  cudaEvent_t ev[8] = {nullptr};
  std::vector<cudaEvent_t> tile_ev;  // pairs of events around K7 launches (C2_OPT_TIMING)
  int tile_ev_used = 0;
};

namespace c2 {

int set_err(c2_ctx *ctx, int code, const char *fmt, ...);

// Device scratch owned by the ctx.  Contents are NOT preserved across growth.
void *ws_get(c2_ctx *ctx, const char *name, size_t bytes, int *rc);

// Launch bookkeeping: counts launches and, with C2_OPT_SYNC_CHECK, checks each one.
int after_launch(c2_ctx *ctx, const char *what);
// Synchronise the ctx stream (counted) and check errors.
int stream_sync(c2_ctx *ctx, const char *what);

// Hash parameters of the t generative functions + GoldFinger (product-side SplitMix64).
struct HashParams {
  uint64_t a[C2_MAX_T];
  uint64_t c[C2_MAX_T];
  uint64_t ga, gc;
};
// f0: the first function used is function f0 of the stream (C2_OPT_FUNC_OFFSET)
void make_hash_params(uint64_t seed, int t, HashParams *hp, int f0 = 0);

// ---------------------------------------------------------------- primitives (prims.cu)
// out[i] = sum_{j<i} in[j] for i in [0, n]; out has n+1 entries (out[n] = total).
int scan_exclusive(c2_ctx *ctx, const int32_t *in, int32_t *out, int64_t n);
// Stable LSD radix sort of (key, val) pairs by the low `bits` bits of key.  Result in
// keys_out / vals_out.  Scratch from ctx.
int radix_sort_pairs(c2_ctx *ctx, const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                     uint32_t *vals_out, int64_t n, int bits);

// ---------------------------------------------------------------- stages
struct Csr {
  const int32_t *offs;  // dev [n+1]
  const int32_t *items; // dev [nnz]
  int32_t n;
  int64_t nnz;
  int32_t max_item;     // filled by validate()
  int32_t max_len;
  const int32_t *psize; // dev [n], |P_u|
  const uint32_t *gf_words = nullptr;  // GoldFinger mode: fingerprints [n][32] (psize = popcounts)
};
// K0: CSR rules + |P_u| + max item / max row length (one host sync).
int validate_csr(c2_ctx *ctx, Csr *csr);
int validate_begin(c2_ctx *ctx, int32_t n);
int validate_chunk(c2_ctx *ctx, const Csr &csr, int32_t u0, int32_t u1);
int validate_finish(c2_ctx *ctx, Csr *csr, int64_t nnz);

// Step 1 (k_sketch.cu + k_cluster.cu).  htab == nullptr -> hashed with params.
struct Clusters {
  int32_t *offsets, *members, *cluster_of; // dev, canonical
  int32_t n_clusters[C2_MAX_T];            // host
  int32_t max_size;
};
int sketch(c2_ctx *ctx, const Csr &csr, int t, int b, const HashParams *hp, const uint16_t *htab, int32_t m,
           int D, uint16_t *out);
int sketch_range(c2_ctx *ctx, const Csr &csr, int t, int b, const HashParams *hp, int32_t u0, int32_t u1,
                 uint16_t *out);
int fastrandomhash(c2_ctx *ctx, const Csr &csr, int t, int b, int64_t N, const HashParams *hp,
                   const uint16_t *htab, int32_t m, Clusters *out);
// C^2/MinHash variant: one cluster per min-hash item, no splitting (chunk guard
// for clusters > N).
int minhash_clusters(c2_ctx *ctx, const Csr &csr, int t, int64_t N, const HashParams *hp, Clusters *out);

// Step 2 (k_local.cu).
int gf_encode(c2_ctx *ctx, const Csr &csr, const HashParams *hp, Csr *gf);
// fused=false: cand [t][n][k] per-function lists (c2_local_knn).  fused=true: out = the running
// final lists [n][k], updated in place function by function (Alg. 3 fused, c2_build).
int local_knn(c2_ctx *ctx, const Csr &csr, int t, const Clusters &cl, int k, c2_cand *out, bool fused,
              c2_cand **result);
// Alg. 2 else-branch (k_hyrec.cu): Hyrec on the nh clusters listed (global cluster ids) in sval_h.
int hyrec_clusters(c2_ctx *ctx, const Csr &csr, int t, const int32_t *offsets, const int32_t *members,
                   const int32_t *ccum, const uint32_t *sval_h, int64_t nh, const int32_t *hyrec_f_lo, int k,
                   uint64_t seed, c2_cand *out, bool fused);

// Step 3 (k_merge.cu).  copyout: c2_build's final format conversion of the fused running lists.
int copyout(c2_ctx *ctx, int n, int k, const c2_cand *run, int32_t *nbr, uint16_t *inter, uint16_t *uni,
            float *sim);
int merge(c2_ctx *ctx, int t, int n, int k, const c2_cand *cand, int32_t *nbr, uint16_t *inter, uint16_t *uni,
          float *sim);

}  // namespace c2

#define C2_CUDA(ctx, call)                                                                  \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return c2::set_err((ctx), C2_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                         __FILE__, __LINE__);                                               \
  } while (0)

#define C2_TRY(expr)          \
  do {                        \
    int rc_ = (expr);         \
    if (rc_ != C2_OK) return rc_; \
  } while (0)

#define C2_LAUNCHED(ctx, name) C2_TRY(c2::after_launch((ctx), (name)))

// ---------------------------------------------------------------- device helpers
namespace c2d {

__device__ __forceinline__ uint32_t item_hash(uint64_t a, uint64_t c, uint32_t x, uint32_t b) {
  // h(x) = floor(((a*x + c) mod 2^64) * b / 2^64)  (A1): one IMAD.WIDE-style mul-add + UMULHI
  uint64_t z = a * (uint64_t)x + c;
  return (uint32_t)__umul64hi(z, (uint64_t)b);
}

// Candidate order (A13): (i1,U1,id1) before (i2,U2,id2) iff i1*U2 > i2*U1, ties by lower id.
// inter <= 32767 and union <= 65534 (A28), so the products fit in 32 bits.
__device__ __forceinline__ bool better(uint32_t i1, uint32_t U1, int32_t id1, uint32_t i2, uint32_t U2,
                                       int32_t id2) {
  uint32_t l = i1 * U2, r = i2 * U1;
  return l > r || (l == r && id1 < id2);
}

__device__ __forceinline__ int warp_incl_scan(int v) {
  int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// Warp-aggregated counter increment: lanes of `mask` with equal `key` add their count once.
__device__ __forceinline__ void agg_inc(unsigned mask, int32_t *ctr, int32_t key) {
  unsigned peers = __match_any_sync(mask, key);
  if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(ctr, __popc(peers));
}

}  // namespace c2d
