// k_rows.cuh -- interface between k_local_tile (k_local.cu) and the per-row kernels (k_rows.cu).
#pragma once
#include "c2_internal.cuh"

namespace c2 {

// A cluster processed by the tile kernel: either one big cluster (slot == 0; members in
// vperm[vp_off .. vp_off + s)) or one "mixed" 32-row slice packing 32/slot small clusters of
// 2..32 users, each in its own aligned group of `slot` positions (empty positions are -1).
struct BigC {
  int32_t f, s, vp_off, sl_off, slot;
  int32_t kc;  // relabeled units: size of the unit's local item universe
};
struct Tile {
  int32_t bc, j;
};

// One row handed from a tile to k_row_topk: user u (|P_u| = pr) of a cluster whose s members are
// vperm[vp_off ..) (sizes vsize[vp_off ..)); its counts |P_u ∩ P_v| are cnt[cnt_off + v].  selfr:
// u's own member position.  Mixed slices: candidates are the members of positions
// [slot_lo, slot_lo + slot) only (slot = 0: all s members).  f: the hash function (c2_local_knn's
// output index).
struct RowRec {
  int32_t u, pr, s, vp_off, selfr, slot_lo, slot, f;
  int64_t cnt_off;
};

struct RowArgs {
  const RowRec *recs;
  const int64_t *nrec;  // device: number of records (written by the tile launch)
  const uint16_t *cnt;
  const int32_t *vperm, *vsize;
  const c2_cand *seed;  // c2_build: running lists [n][k] (updated in place through out); else nullptr
  c2_cand *out;
  int32_t n;
  int k;
  unsigned long long *kstats;
};

int launch_row_topk(c2_ctx *ctx, const RowArgs &ra);
int launch_surv_merge(c2_ctx *ctx, const c2_cand *surv, int32_t *qn, int qmax, int32_t n, int k, c2_cand *run,
                      cudaStream_t st = nullptr);

}  // namespace c2
