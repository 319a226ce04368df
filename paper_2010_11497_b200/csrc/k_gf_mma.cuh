// k_gf_mma.cuh -- the GoldFinger variant's tensor-core Step 2 (k_gf_mma.cu), called by local_knn.
#pragma once
#include "k_rows.cuh"

namespace c2 {

__device__ __forceinline__ uint32_t smem_u32_gm(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct GfArgs {
  const BigC *bcs;
  int64_t bc_lo, bc_hi;     // the function's big clusters
  const int64_t *wl_off;    // per cluster: first work item (relative to the function)
  const int64_t *cbase;     // per cluster: first count entry (relative to the function's region)
  const int64_t *nwork;     // device: work items of the function
  const int32_t *witem;     // the function's item -> cluster map
  const int32_t *vperm, *vsize;
  const uint8_t *bytes;     // fingerprints expanded to 0/1 bytes [n][1024] (gf_expand)
  int32_t n;
  int k;
  const c2_cand *seed;      // c2_build: running lists (light-row test); else nullptr
  c2_cand *surv;
  int32_t *qn;
  int32_t qmax;
  uint16_t *cnt;            // count rows (k_row_topk's cnt buffer)
  int64_t tc_base;          // this path's region in cnt
  RowRec *recs;
  unsigned long long *nrec;
  int64_t rcap;
  int *err;
};

int gf_prefix(c2_ctx *ctx, const BigC *bcs, const int64_t *bc_rng, int t, int64_t nbig, int64_t *wl_off,
              int64_t *cbase, int64_t *fsum, int32_t *witem, int64_t icap);
int gf_expand(c2_ctx *ctx, const uint32_t *words, int32_t n, uint8_t *bytes);
int launch_gf_mma(c2_ctx *ctx, const GfArgs &ga);

}  // namespace c2
