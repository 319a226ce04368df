// k_cluster.cu -- Step 1 of C^2 on the GPU: Alg. 1 bucketing and the recursive
// split of clusters larger than N, level-synchronously over all functions, then
// the chunk guard (A9) and the canonical cluster arrays (A25).
//
// Representation.  key[f][u] is the id of the node user u currently belongs to under f
// (level 0: f*b + H_f(u)); slot[f][u] >= 0 iff that node is larger than N and is being split
// at the current level (slot = its index among the level's active nodes).  One level:
//   count : for active users, nv = next distinct value (sketch[d+1], or recomputed from the
//           CSR past the sketch depth) and hist[slot][nv]++
//   assign: groups with >= 2 users become child nodes (new ids); groups of one user and
//           users with no next value stay in the parent, which becomes a terminal residual
//           (A6-A8); children larger than N are active at the next level
//   apply : move users to their child node
// The host reads two counters per level (children, next-level active nodes).
#include <algorithm>

#include <cooperative_groups.h>

#include "c2_internal.cuh"

namespace cg = cooperative_groups;

namespace c2 {

struct HashArgs2 {
  uint64_t a[C2_MAX_T];
  uint64_t c[C2_MAX_T];
};

// ------------------------------------------------------------------ level 0
__global__ void k_level0(const uint16_t *__restrict__ sk, int64_t TN, int32_t n, int32_t b,
                         int32_t *__restrict__ key, uint16_t *__restrict__ curval, int32_t *__restrict__ size0) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = q < TN;
  const unsigned mask = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  int32_t f = (int32_t)(q / n);
  uint16_t v = sk[q * C2_SKETCH_D];  // H_f(u)
  int32_t k = f * b + v;
  key[q] = k;
  curval[q] = v;
  c2d::agg_inc(mask, &size0[k], k);
}

// Same as k_level0 with the node sizes counted in a shared-memory histogram over the b buckets
// of the chunk's first function (blocks cover consecutive (f,u)); one global atomic per non-empty
// bucket per block.  Entries of a later function (chunks crossing a function boundary) count
// directly in global memory.
__global__ void __launch_bounds__(512) k_level0h(const uint16_t *__restrict__ sk, int64_t TN, int32_t n, int32_t b,
                                                 int64_t chunk, int32_t *__restrict__ key,
                                                 uint16_t *__restrict__ curval, int32_t *__restrict__ size0) {
  extern __shared__ int32_t hb[];
  const int64_t q0 = (int64_t)blockIdx.x * chunk, q1 = min(q0 + chunk, TN);
  const int32_t f0 = (int32_t)(q0 / n);
  for (int i = threadIdx.x; i < b; i += blockDim.x) hb[i] = 0;
  __syncthreads();
  for (int64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
    const int32_t f = (int32_t)(q / n);
    const uint16_t v = sk[q * C2_SKETCH_D];  // H_f(u)
    const int32_t k = f * b + v;
    key[q] = k;
    curval[q] = v;
    if (f == f0) atomicAdd(&hb[v], 1);
    else atomicAdd(&size0[k], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < b; i += blockDim.x)
    if (hb[i]) atomicAdd(&size0[(int64_t)f0 * b + i], hb[i]);
}

__global__ void k_flag_gt(const int32_t *__restrict__ cnt, int64_t E, int64_t N, int32_t *__restrict__ flag) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < E) flag[e] = cnt[e] > N ? 1 : 0;
}

__global__ void k_slot0(const int32_t *__restrict__ key, const int32_t *__restrict__ size0,
                        const int32_t *__restrict__ ascan, int64_t TN, int64_t N, int32_t *__restrict__ slot) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= TN) return;
  int32_t k = key[q];
  slot[q] = size0[k] > N ? ascan[k] : -1;
}

// ------------------------------------------------------------------ split level
template <bool TABLE>
__device__ __forceinline__ uint16_t next_above(const int32_t *__restrict__ offs, const int32_t *__restrict__ items,
                                               int32_t u, int f, uint32_t eta, uint32_t b, const HashArgs2 &ha,
                                               const uint16_t *__restrict__ htab, int32_t m) {
  // H\eta(u) = min_{i in P_u, h(i) > eta} h(i), recomputed from the CSR
  uint32_t best = C2_ABSENT16;
  for (int32_t p = offs[u]; p < offs[u + 1]; ++p) {
    uint32_t x = (uint32_t)items[p];
    uint32_t v = TABLE ? (uint32_t)htab[(int64_t)f * m + x] : c2d::item_hash(ha.a[f], ha.c[f], x, b);
    if (v > eta && v < best) best = v;
  }
  return (uint16_t)best;
}

// the D smallest distinct values above eta of {h(i) : i in P_u}, ascending, ABSENT padded
template <bool TABLE>
__device__ __noinline__ void refill_above(const int32_t *__restrict__ offs, const int32_t *__restrict__ items,
                                             int32_t u, int f, uint32_t eta, uint32_t b, uint64_t ha_a, uint64_t ha_c,
                                             const uint16_t *__restrict__ htab, int32_t m, int D,
                                             uint16_t *__restrict__ row) {
  uint32_t s[C2_SKETCH_D];
#pragma unroll
  for (int j = 0; j < C2_SKETCH_D; ++j) s[j] = C2_ABSENT16;
  for (int32_t p = offs[u]; p < offs[u + 1]; ++p) {
    const uint32_t x = (uint32_t)items[p];
    const uint32_t v = TABLE ? (uint32_t)htab[(int64_t)f * m + x] : c2d::item_hash(ha_a, ha_c, x, b);
    if (v <= eta || v >= s[D - 1]) continue;
    bool dup = false;
#pragma unroll
    for (int j = 0; j < C2_SKETCH_D; ++j) dup |= j < D && s[j] == v;
    if (dup) continue;
#pragma unroll
    for (int j = C2_SKETCH_D - 1; j >= 1; --j)
      if (j < D) s[j] = (v < s[j - 1]) ? s[j - 1] : ((v < s[j]) ? v : s[j]);
    s[0] = min(s[0], v);
  }
#pragma unroll
  for (int j = 0; j < C2_SKETCH_D; ++j)
    if (j < D) row[j] = (uint16_t)s[j];
}

template <bool TABLE>
__global__ void k_split_count(const int32_t *__restrict__ slot, const uint16_t *__restrict__ sk,
                              const uint16_t *__restrict__ curval, uint16_t *__restrict__ nextval, int64_t TN,
                              int32_t n, int d, int Deff, int32_t a0, int32_t a1, int32_t b,
                              int32_t *__restrict__ hist, const int32_t *__restrict__ offs,
                              const int32_t *__restrict__ items, HashArgs2 ha, const uint16_t *__restrict__ htab,
                              int32_t m) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= TN) return;
  int32_t s = slot[q];
  if (s < a0 || s >= a1) return;
  uint16_t nv;
  if (d + 1 < Deff) nv = sk[q * C2_SKETCH_D + d + 1];
  else nv = next_above<TABLE>(offs, items, (int32_t)(q % n), (int)(q / n), curval[q], (uint32_t)b, ha, htab, m);
  nextval[q] = nv;
  if (nv != C2_ABSENT16) atomicAdd(&hist[(int64_t)(s - a0) * b + nv], 1);  // (spread over b bins)
}

__global__ void k_child_flags(const int32_t *__restrict__ hist, int64_t E, int64_t N, int32_t *__restrict__ fc,
                              int32_t *__restrict__ fa, unsigned long long *__restrict__ folded) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int one = 0;
  if (e < E) {
    int32_t c = hist[e];
    fc[e] = c >= 2;
    fa[e] = c > N;
    one = c == 1;
  }
  unsigned bal = __ballot_sync(0xffffffffu, one);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(folded, (unsigned long long)__popc(bal));
}

__global__ void k_child_assign(const int32_t *__restrict__ hist, const int32_t *__restrict__ cscan,
                               const int32_t *__restrict__ ascan, int64_t E, int64_t N, int32_t id_base,
                               int32_t slot_base, int32_t *__restrict__ child_id, int32_t *__restrict__ child_slot) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  int32_t c = hist[e];
  child_id[e] = c >= 2 ? id_base + cscan[e] : -1;
  child_slot[e] = c > N ? slot_base + ascan[e] : -1;
}

__global__ void k_split_apply(int32_t *__restrict__ slot, int32_t *__restrict__ key, uint16_t *__restrict__ curval,
                              const uint16_t *__restrict__ nextval, int64_t TN, int32_t a0, int32_t a1, int32_t b,
                              const int32_t *__restrict__ child_id, const int32_t *__restrict__ child_slot,
                              int32_t *__restrict__ slot_next) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= TN) return;
  int32_t s = slot[q];
  if (s < a0 || s >= a1) return;
  uint16_t nv = nextval[q];
  int32_t ns = -1;
  if (nv != C2_ABSENT16) {
    int64_t e = (int64_t)(s - a0) * b + nv;
    int32_t c = child_id[e];
    if (c >= 0) {  // >= 2 users share nv: move to the child node
      key[q] = c;
      curval[q] = nv;
      ns = child_slot[e];
    }
  }
  slot_next[q] = ns;  // -1: stays in the parent's residual (terminal) or child <= N
}

// ------------------------------------------------------------------ device-side split loop (N1)
// The whole recursive split in ONE cooperative kernel: no host round trip per level.
// Same rules and the same node numbering as the host-driven loop above (children numbered by an
// exclusive scan over (active node, next value), active children by a scan over the same order),
// but each level touches only its active users, held in a compact list (q, slot):
//   count  : nv = next distinct value of every active user; hist[slot*b + nv]++          | grid sync
//   scan   : over E = n_active*b bins, children (c >= 2) and active children (c > N),
//            two counts packed in one u64 grid-wide exclusive scan (block partials)      | grid sync
//   apply  : users of a child move to it; users of an active child join the next list;
//            the next level's histogram region is zeroed                                 | grid sync
// Every block computes the level totals from the same partials, so all blocks agree on when
// the loop ends.  Level 0's active nodes come from the same scan over the t*b level-0 bins.
struct SplitDev {
  int32_t *hist;        // [hcap]
  int32_t *child_id;    // [hcap]
  int32_t *child_slot;  // [hcap]
  int32_t *act_q[2];    // [TN] active (f,u) indices, ping-pong
  int32_t *act_s[2];    // [TN] their node's slot among the level's active nodes
  uint16_t *nvb;        // [TN] next value per active-list entry
  unsigned long long *part;  // [grid] block partials of the packed scan
  int32_t *act_n;       // [2] list lengths (atomic append)
  long long *out;       // [8]: next_id, split_nodes, max_depth, folded, levels
  int64_t hcap;
};

__device__ __forceinline__ unsigned long long block_excl_scan_u64(unsigned long long v, unsigned long long *sh,
                                                                  unsigned long long *total) {
  // exclusive scan over the block (blockDim.x <= 1024); sh: 32 entries
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned long long s = lane < nw ? sh[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) sh[lane] = s;  // inclusive prefix of warp totals
  }
  __syncthreads();
  const unsigned long long before = (w ? sh[w - 1] : 0ull) + x - v;
  *total = sh[nw - 1];
  __syncthreads();
  return before;
}

template <bool TABLE>
__global__ void __launch_bounds__(256, 4) k_split_dev(SplitDev sd, const uint16_t *__restrict__ skr, uint16_t *sk,
                                                  int32_t *__restrict__ key,
                                                  uint16_t *__restrict__ curval, const int32_t *__restrict__ size0,
                                                  int64_t TB, int64_t TN, int32_t n, int Deff, int32_t b, int64_t N,
                                                  const int32_t *__restrict__ offs, const int32_t *__restrict__ items,
                                                  HashArgs2 ha, const uint16_t *__restrict__ htab, int32_t m) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned long long sh[32];
  __shared__ unsigned long long s_pre, s_tot;
  const int64_t G = gridDim.x;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gstride = G * blockDim.x;
  const unsigned long long LO = 0xffffffffull;

  // ---- packed grid scan over E bins: value(e) -> (lo, hi) counts; returns the totals.  The
  //      callback emit(e, pre_lo, pre_hi) sees every bin's exclusive prefix.
  auto grid_scan = [&](int64_t E, auto value, auto emit) -> unsigned long long {
    const int64_t lo = E * blockIdx.x / G, hi = E * (blockIdx.x + 1) / G;
    unsigned long long acc = 0;
    for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) acc += value(e);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long s = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
      sd.part[blockIdx.x] = s;
    }
    __syncthreads();
    grid.sync();
    // this block's prefix and the grid total from the partials
    unsigned long long pre = 0, tot = 0;
    for (int64_t g = threadIdx.x; g < G; g += blockDim.x) {
      const unsigned long long p = __ldcg(sd.part + g);
      tot += p;
      if (g < blockIdx.x) pre += p;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      pre += __shfl_xor_sync(0xffffffffu, pre, o);
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = pre;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long s = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
      s_pre = s;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = tot;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long s = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
      s_tot = s;
    }
    __syncthreads();
    unsigned long long carry = s_pre;
    const unsigned long long total = s_tot;
    for (int64_t e0 = lo; e0 < hi; e0 += blockDim.x) {
      const int64_t e = e0 + threadIdx.x;
      const unsigned long long v = e < hi ? value(e) : 0ull;
      unsigned long long tsum;
      const unsigned long long ex = block_excl_scan_u64(v, sh, &tsum) + carry;
      if (e < hi) emit(e, (int64_t)(ex & LO), (int64_t)(ex >> 32));
      carry += tsum;
    }
    return total;
  };

  // ---- level 0: active nodes = level-0 bins larger than N, numbered in bin order
  int64_t n_active = (int64_t)grid_scan(
      TB, [&](int64_t e) -> unsigned long long { return size0[e] > N ? 1ull : 0ull; },
      [&](int64_t e, int64_t pre, int64_t) { sd.child_slot[e] = size0[e] > N ? (int32_t)pre : -1; });
  grid.sync();
  // active lists are appended block-chunk by block-chunk in order (one atomic per block and
  // chunk), so they stay in ascending runs of blockDim.x entries and the gathers of the next
  // level (sketch, curval, key by q) stay mostly coalesced
  __shared__ int s_base;
  auto block_append = [&](bool a, int32_t q, int32_t s, int32_t *ctr, int32_t *lq, int32_t *ls) {
    unsigned long long tot;
    const unsigned long long pre = block_excl_scan_u64(a ? 1ull : 0ull, sh, &tot);
    if (threadIdx.x == 0 && tot) s_base = atomicAdd(ctr, (int)tot);
    __syncthreads();
    if (a) {
      lq[s_base + (int)pre] = q;
      ls[s_base + (int)pre] = s;
    }
    __syncthreads();
  };
  for (int64_t q0 = (int64_t)blockIdx.x * blockDim.x; q0 < TN; q0 += gstride) {
    const int64_t q = q0 + threadIdx.x;
    const int32_t s = q < TN ? sd.child_slot[key[q]] : -1;
    block_append(s >= 0, (int32_t)q, s, &sd.act_n[0], sd.act_q[0], sd.act_s[0]);
  }
  // zero the level-0 histogram region
  for (int64_t e = gtid; e < n_active * b; e += gstride) sd.hist[e] = 0;
  grid.sync();

  int64_t next_id = TB, split_nodes = 0, max_depth = 0, folded = 0;
  int cur = 0;
  int d = 0;
  for (; n_active > 0; ++d) {
    if (d > b + 1) break;  // cannot happen (each level consumes one distinct value)
    const int64_t na = __ldcg(sd.act_n + cur);
    const int32_t *aq = sd.act_q[cur], *as = sd.act_s[cur];
    // count
    for (int64_t i = gtid; i < na; i += gstride) {
      const int32_t q = aq[i];
      uint16_t nv;
      if (d + 1 < Deff) {
        nv = skr[(int64_t)q * C2_SKETCH_D + d + 1];
      } else if (d + 1 == Deff) {
        nv = next_above<TABLE>(offs, items, (int32_t)(q % n), (int)(q / n), curval[q], (uint32_t)b, ha, htab, m);
      } else {
        // deeper: every Deff levels one pass over the row refills the user's sketch row with the
        // next Deff distinct values above its current node's value (H\eta applied Deff times,
        // P:463; the sketch is dead scratch once the split has passed it) instead of one pass per
        // level.  Written and read through the coherent pointer only.
        uint16_t *row = sk + (int64_t)q * C2_SKETCH_D;
        const int j = (d - Deff) % Deff;
        if (j == 0) {
          const int f = (int)(q / n);
          refill_above<TABLE>(offs, items, (int32_t)(q % n), f, curval[q], (uint32_t)b, TABLE ? 0ull : ha.a[f],
                              TABLE ? 0ull : ha.c[f], htab, m, Deff, row);
        }
        nv = row[j];
      }
      sd.nvb[i] = nv;
      if (nv != C2_ABSENT16) atomicAdd(&sd.hist[(int64_t)as[i] * b + nv], 1);
    }
    if (gtid == 0) sd.act_n[cur ^ 1] = 0;
    grid.sync();
    // scan: children (c >= 2, low half) and active children (c > N, high half); singletons folded
    const int64_t E = n_active * b;
    const int32_t idb = (int32_t)next_id;
    unsigned long long ones = 0;
    const unsigned long long tot = grid_scan(
        E,
        [&](int64_t e) -> unsigned long long {
          const int32_t c = __ldcg(sd.hist + e);
          return (unsigned long long)(c >= 2) | ((unsigned long long)(c > N) << 32);
        },
        [&](int64_t e, int64_t pc, int64_t pa) {
          const int32_t c = __ldcg(sd.hist + e);
          sd.child_id[e] = c >= 2 ? idb + (int32_t)pc : -1;
          sd.child_slot[e] = c > N ? (int32_t)pa : -1;
          ones += c == 1;
        });
    // folded singletons (statistics): block sums into out[3]
#pragma unroll
    for (int o = 16; o; o >>= 1) ones += __shfl_xor_sync(0xffffffffu, ones, o);
    if ((threadIdx.x & 31) == 0 && ones) atomicAdd((unsigned long long *)&sd.out[3], ones);
    const int64_t n_child = (int64_t)(tot & LO), n_next = (int64_t)(tot >> 32);
    grid.sync();
    // apply
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < na; i0 += gstride) {
      const int64_t i = i0 + threadIdx.x;
      int32_t q = -1, ns = -1;
      if (i < na) {
        q = aq[i];
        const uint16_t nv = sd.nvb[i];
        if (nv != C2_ABSENT16) {
          const int64_t e = (int64_t)as[i] * b + nv;
          const int32_t c = sd.child_id[e];
          if (c >= 0) {
            key[q] = c;
            curval[q] = nv;
            ns = sd.child_slot[e];
          }
        }
      }
      block_append(ns >= 0, q, ns, &sd.act_n[cur ^ 1], sd.act_q[cur ^ 1], sd.act_s[cur ^ 1]);
    }
    for (int64_t e = gtid; e < n_next * b; e += gstride) sd.hist[e] = 0;
    grid.sync();
    next_id += n_child;
    split_nodes += n_active;
    if (n_child > 0) max_depth = d + 1;
    n_active = n_next;
    cur ^= 1;
  }
  if (gtid == 0) {
    sd.out[0] = next_id;
    sd.out[1] = split_nodes;
    sd.out[2] = max_depth;
    sd.out[4] = d;
    sd.out[5] = n_active;  // nonzero only if the level guard tripped
  }
}

// ------------------------------------------------------------------ canonical form

__global__ void __launch_bounds__(256) k_max(const int32_t *__restrict__ x, int64_t E, int32_t *__restrict__ out,
                                             const long long *__restrict__ dE = nullptr) {
  // grid-stride, one atomic per block.  dE (device-side split loop): the actual number of
  // entries, E is only its bound
  __shared__ int sh[8];
  if (dE) E = min(E, (int64_t)*dE);
  int v = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    v = max(v, x[e]);
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) v = max(v, sh[w]);
    if (v) atomicMax(out, v);
  }
}

// node sizes and smallest members in one pass; lanes hold ascending q, so among the lanes of one
// node the lowest carries its smallest user in this warp (nodes never span functions)
__global__ void k_count_rep(const int32_t *__restrict__ key, int64_t TN, int32_t n, int32_t *__restrict__ size,
                            int32_t *__restrict__ rep) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = q < TN;
  const unsigned mask = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  const int32_t k = key[q];
  const unsigned peers = __match_any_sync(mask, k);
  if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) {  // lowest lane: smallest user of the node in this warp
    atomicAdd(&size[k], __popc(peers));
    atomicMin(&rep[k], (int32_t)(q % n));
  }
}


__global__ void k_heads(const int32_t *__restrict__ key, const int32_t *__restrict__ rep, int64_t TN, int32_t n,
                        int32_t *__restrict__ head) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < TN) head[q] = rep[key[q]] == (int32_t)(q % n);
}

__global__ void k_cluster_of(const int32_t *__restrict__ key, const int32_t *__restrict__ rep,
                             const int32_t *__restrict__ hscan, const int32_t *__restrict__ size, int64_t TN,
                             int32_t n, int32_t *__restrict__ cof, int32_t *__restrict__ csize,
                             uint32_t *__restrict__ skey, uint32_t *__restrict__ sval) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= TN) return;
  int64_t f = q / n;
  int32_t u = (int32_t)(q % n);
  int32_t k = key[q];
  int32_t r = rep[k];
  int32_t c = hscan[f * n + r] - hscan[f * n];  // clusters of f ordered by smallest member
  cof[q] = c;
  if (r == u) csize[f * (n + 1) + c] = size[k];
  skey[q] = (uint32_t)(f * n + c);
  sval[q] = (uint32_t)u;
}

__global__ void k_fix_offsets(const int32_t *__restrict__ raw, int64_t E, int32_t n, int32_t *__restrict__ offsets) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  int64_t f = e / (n + 1);
  offsets[e] = raw[e] - (int32_t)(f * n);
}

__global__ void __launch_bounds__(256) k_pairs(const int32_t *__restrict__ csize, int64_t E,
                                               unsigned long long *__restrict__ acc) {
  // P = sum of s(s-1)/2 over the clusters (A21); grid-stride, one atomic per block
  __shared__ unsigned long long sh[8];
  unsigned long long p = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long s = (unsigned long long)csize[e];
    p += s * (s - (s > 0)) / 2;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = p;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) p += sh[w];
    if (p) atomicAdd(acc, p);
  }
}

// chunk guard: sorted (key, f*n+u) pairs; node_start = exclusive scan of sizes
__global__ void k_chunk_count(const int32_t *__restrict__ size, int64_t E, int64_t N, int32_t *__restrict__ mc) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < E) mc[e] = size[e] > N ? (int32_t)((size[e] + N - 1) / N) : 0;
}

__global__ void k_chunk_assign(const uint32_t *__restrict__ skeys, const uint32_t *__restrict__ svals, int64_t TN,
                               const int32_t *__restrict__ size, const int32_t *__restrict__ start,
                               const int32_t *__restrict__ cbase, int64_t N, int32_t id_base,
                               int32_t *__restrict__ key) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= TN) return;
  uint32_t k = skeys[p];
  int64_t s = size[k];
  if (s <= N) return;
  int64_t r = p - start[k];               // rank among the node's members (ascending id)
  int64_t mcount = (s + N - 1) / N;
  int64_t j = ((r + 1) * mcount + s - 1) / s - 1;  // chunk j = [floor(j s/m), floor((j+1) s/m))
  key[svals[p]] = id_base + cbase[k] + (int32_t)j;
}

static inline unsigned nblk(int64_t x, int bs = 256) { return (unsigned)((x + bs - 1) / bs); }
static inline int bits_for(int64_t x) {
  int b = 1;
  while ((1LL << b) < x) ++b;
  return b;
}

// ------------------------------------------------------------------ small helpers
__global__ void k_fill_pairs(const int32_t *__restrict__ key, int64_t TN, uint32_t *__restrict__ k,
                             uint32_t *__restrict__ v) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < TN) {
    k[q] = (uint32_t)key[q];
    v[q] = (uint32_t)q;
  }
}
int fill_key_pairs(c2_ctx *ctx, const int32_t *key, int64_t TN, uint32_t *k, uint32_t *v) {
  k_fill_pairs<<<nblk(TN), 256, 0, ctx->stream>>>(key, TN, k, v);
  C2_LAUNCHED(ctx, "k_fill_pairs");
  return C2_OK;
}

__global__ void k_count_gt(const int32_t *__restrict__ x, int64_t E, int64_t N, int32_t *__restrict__ out) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned bal = __ballot_sync(0xffffffffu, e < E && x[e] > N);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(out, __popc(bal));
}
int count_gt(c2_ctx *ctx, const int32_t *x, int64_t E, int64_t N, int32_t *out) {
  k_count_gt<<<nblk(E), 256, 0, ctx->stream>>>(x, E, N, out);
  C2_LAUNCHED(ctx, "k_count_gt");
  return C2_OK;
}

// ------------------------------------------------------------------ K4: chunk guard + canonical form
// key[f*n+u] = node id in [0, next_id) (at most one node per cluster; a node larger than N is
// cut into balanced chunks, A9); produces the canonical arrays (A25) and the host statistics.
static int canonicalize(c2_ctx *ctx, int32_t n, int t, int64_t N, int32_t *key, int64_t next_id,
                        int64_t split_nodes, int64_t max_depth, Clusters *out, const long long *dev_split = nullptr) {
  int rc;
  const int64_t TN = (int64_t)t * n;
  cudaStream_t st = ctx->stream;
  cudaEvent_t *ev = ctx->ev;
  unsigned long long *acc = (unsigned long long *)ws_get(ctx, "acc", 64, &rc);
  if (rc) return rc;
  int32_t *hsmall = (int32_t *)ctx->h_small;
  // dev_split: the node count is still on the device (device-side split loop); size the node
  // arrays by the bound t*b + t*n (passed as next_id) and read the count at the first sync
  int32_t *size = (int32_t *)ws_get(ctx, "nsize", (size_t)(next_id + TN + 1) * 4, &rc);
  if (rc) return rc;
  C2_CUDA(ctx, cudaMemsetAsync(size, 0, (size_t)next_id * 4, st));
  int32_t *rep = (int32_t *)ws_get(ctx, "rep", (size_t)(next_id + TN + 1) * 4, &rc);
  if (rc) return rc;
  C2_CUDA(ctx, cudaMemsetAsync(rep, 0x7F, (size_t)next_id * 4, st));
  k_count_rep<<<nblk(TN), 256, 0, st>>>(key, TN, n, size, rep);
  C2_LAUNCHED(ctx, "k_count_rep");
  int32_t *mx = (int32_t *)(acc + 2);
  C2_CUDA(ctx, cudaMemsetAsync(mx, 0, 4, st));
  k_max<<<std::min<unsigned>(nblk(next_id), ctx->num_sms * 8), 256, 0, st>>>(size, next_id, mx, dev_split);
  C2_LAUNCHED(ctx, "k_max");
  C2_CUDA(ctx, cudaMemcpyAsync(hsmall, mx, 4, cudaMemcpyDeviceToHost, st));
  if (dev_split) {
    C2_CUDA(ctx, cudaMemcpyAsync(ctx->h_small + 8, dev_split, 8 * 6, cudaMemcpyDeviceToHost, st));
  } else {
    C2_CUDA(ctx, cudaMemcpyAsync(ctx->h_small + 4, acc + 1, 8, cudaMemcpyDeviceToHost, st));
  }
  C2_TRY(stream_sync(ctx, "max size"));
  int64_t chunked = 0;
  int64_t folded = ctx->h_small[4];
  if (dev_split) {
    const long long *o = (const long long *)(ctx->h_small + 8);
    if (o[5] != 0) return set_err(ctx, C2_ECUDA, "split did not terminate");
    next_id = o[0];
    split_nodes = o[1];
    max_depth = o[2];
    folded = o[3];
  }
  uint32_t *skey = (uint32_t *)ws_get(ctx, "skey", (size_t)TN * 4, &rc);
  if (rc) return rc;
  uint32_t *sval = (uint32_t *)ws_get(ctx, "sval", (size_t)TN * 4, &rc);
  if (rc) return rc;
  uint32_t *skey2 = (uint32_t *)ws_get(ctx, "skey2", (size_t)TN * 4, &rc);
  if (rc) return rc;
  uint32_t *sval2 = (uint32_t *)ws_get(ctx, "sval2", (size_t)TN * 4, &rc);
  if (rc) return rc;
  if (hsmall[0] > N) {
    // A9: residuals larger than N -> ceil(s/N) balanced chunks of their ascending members.
    // Stable sort of (node, f*n+u) by node gives every node's members in ascending order.
    int32_t *tmp = (int32_t *)ws_get(ctx, "chunk_tmp", (size_t)(next_id + 1) * 4 * 4, &rc);
    if (rc) return rc;
    int32_t *start = tmp, *mcnt = tmp + (next_id + 1), *cbase = tmp + 2 * (next_id + 1);
    C2_TRY(scan_exclusive(ctx, size, start, next_id));
    k_chunk_count<<<nblk(next_id), 256, 0, st>>>(size, next_id, N, mcnt);
    C2_LAUNCHED(ctx, "k_chunk_count");
    C2_TRY(scan_exclusive(ctx, mcnt, cbase, next_id));
    // flat index -> (key) pairs
    C2_TRY(fill_key_pairs(ctx, key, TN, skey2, sval2));
    C2_TRY(radix_sort_pairs(ctx, skey2, sval2, skey, sval, TN, bits_for(next_id)));
    k_chunk_assign<<<nblk(TN), 256, 0, st>>>(skey, sval, TN, size, start, cbase, N, (int32_t)next_id, key);
    C2_LAUNCHED(ctx, "k_chunk_assign");
    C2_CUDA(ctx, cudaMemcpyAsync(hsmall, cbase + next_id, 4, cudaMemcpyDeviceToHost, st));
    int32_t *nbig = (int32_t *)(acc + 3);
    C2_CUDA(ctx, cudaMemsetAsync(nbig, 0, 4, st));
    C2_TRY(count_gt(ctx, size, next_id, N, nbig));
    C2_CUDA(ctx, cudaMemcpyAsync(hsmall + 1, nbig, 4, cudaMemcpyDeviceToHost, st));
    C2_TRY(stream_sync(ctx, "chunk guard"));
    int64_t nchunks = hsmall[0];
    chunked = hsmall[1];
    next_id += nchunks;
    size = (int32_t *)ws_get(ctx, "nsize", (size_t)(next_id + 1) * 4, &rc);
    if (rc) return rc;
    C2_CUDA(ctx, cudaMemsetAsync(size, 0, (size_t)next_id * 4, st));
    rep = (int32_t *)ws_get(ctx, "rep", (size_t)(next_id + 1) * 4, &rc);
    if (rc) return rc;
    C2_CUDA(ctx, cudaMemsetAsync(rep, 0x7F, (size_t)next_id * 4, st));
    k_count_rep<<<nblk(TN), 256, 0, st>>>(key, TN, n, size, rep);
    C2_LAUNCHED(ctx, "k_count_rep");
  }
  // (rep[node] = smallest member, from k_count_rep); heads; canonical cluster index by scan over users
  int32_t *head = (int32_t *)ws_get(ctx, "head", (size_t)(2 * TN + 2) * 4, &rc);
  if (rc) return rc;
  int32_t *hscan = head + TN + 1;
  k_heads<<<nblk(TN), 256, 0, st>>>(key, rep, TN, n, head);
  C2_LAUNCHED(ctx, "k_heads");
  C2_TRY(scan_exclusive(ctx, head, hscan, TN));
  const int64_t TN1 = (int64_t)t * (n + 1);
  int32_t *csize = (int32_t *)ws_get(ctx, "csize", (size_t)(2 * TN1 + 2) * 4, &rc);
  if (rc) return rc;
  int32_t *craw = csize + TN1 + 1;
  C2_CUDA(ctx, cudaMemsetAsync(csize, 0, (size_t)TN1 * 4, st));
  k_cluster_of<<<nblk(TN), 256, 0, st>>>(key, rep, hscan, size, TN, n, out->cluster_of, csize, skey2, sval2);
  C2_LAUNCHED(ctx, "k_cluster_of");
  C2_TRY(scan_exclusive(ctx, csize, craw, TN1));
  k_fix_offsets<<<nblk(TN1), 256, 0, st>>>(craw, TN1, n, out->offsets);
  C2_LAUNCHED(ctx, "k_fix_offsets");
  // members: stable sort of (f*n + cluster, u) by key -> ascending members per cluster
  C2_TRY(radix_sort_pairs(ctx, skey2, sval2, skey, (uint32_t *)out->members, TN, bits_for(TN)));
  C2_CUDA(ctx, cudaMemsetAsync(acc, 0, 8, st));
  k_pairs<<<std::min<unsigned>(nblk(TN1), ctx->num_sms * 8), 256, 0, st>>>(csize, TN1, acc);
  C2_LAUNCHED(ctx, "k_pairs");
  C2_CUDA(ctx, cudaMemsetAsync(mx, 0, 4, st));
  k_max<<<std::min<unsigned>(nblk(TN1), ctx->num_sms * 8), 256, 0, st>>>(csize, TN1, mx);
  C2_LAUNCHED(ctx, "k_max");
  // host values: n_clusters[f] = hscan[(f+1)n] - hscan[fn], P, max size
  int32_t *hh = (int32_t *)ctx->h_small + 16;
  for (int f = 0; f <= t; ++f)
    C2_CUDA(ctx, cudaMemcpyAsync(hh + f, hscan + (int64_t)f * n, 4, cudaMemcpyDeviceToHost, st));
  C2_CUDA(ctx, cudaMemcpyAsync(ctx->h_small, acc, 8, cudaMemcpyDeviceToHost, st));
  C2_CUDA(ctx, cudaMemcpyAsync(ctx->h_small + 1, mx, 4, cudaMemcpyDeviceToHost, st));
  C2_TRY(stream_sync(ctx, "canonical"));
  int64_t total = 0;
  for (int f = 0; f < t; ++f) {
    out->n_clusters[f] = hh[f + 1] - hh[f];
    total += out->n_clusters[f];
  }
  out->max_size = (int32_t)(ctx->h_small[1] & 0xffffffff);
  ctx->stats.pairs = ctx->h_small[0];
  ctx->stats.clusters = total;
  ctx->stats.max_cluster_size = out->max_size;
  ctx->stats.split_nodes = split_nodes;
  ctx->stats.max_depth = max_depth;
  ctx->stats.folded_singletons = folded;
  ctx->stats.chunked_residuals = chunked;
  if (ctx->timing) cudaEventRecord(ev[3], st);
  return C2_OK;
}


int fastrandomhash(c2_ctx *ctx, const Csr &csr, int t, int b, int64_t N, const HashParams *hp,
                   const uint16_t *htab, int32_t m, Clusters *out) {
  int rc;
  const int32_t n = csr.n;
  const int64_t TN = (int64_t)t * n;
  cudaStream_t st = ctx->stream;
  HashArgs2 ha;
  for (int f = 0; f < t; ++f) {
    ha.a[f] = hp ? hp->a[f] : 0;
    ha.c[f] = hp ? hp->c[f] : 0;
  }
  const int Deff = ctx->sketch_depth;

  // ---- K1 sketch (all t functions, depth 8)
  uint16_t *sk = (uint16_t *)ws_get(ctx, "sketch", (size_t)TN * C2_SKETCH_D * 2, &rc);
  if (rc) return rc;
  cudaEvent_t *ev = ctx->ev;
  if (ctx->timing) cudaEventRecord(ev[0], st);
  if (ctx->presketched && !htab) ctx->presketched = false;  // computed chunk by chunk during the upload
  else C2_TRY(sketch(ctx, csr, t, b, hp, htab, m, C2_SKETCH_D, sk));
  if (ctx->timing) cudaEventRecord(ev[1], st);

  int32_t *key = (int32_t *)ws_get(ctx, "key", (size_t)TN * 4, &rc);
  if (rc) return rc;
  int32_t *slot = (int32_t *)ws_get(ctx, "slot", (size_t)TN * 4, &rc);
  if (rc) return rc;
  int32_t *slot2 = (int32_t *)ws_get(ctx, "slot2", (size_t)TN * 4, &rc);
  if (rc) return rc;
  uint16_t *curval = (uint16_t *)ws_get(ctx, "curval", (size_t)TN * 2, &rc);
  if (rc) return rc;
  uint16_t *nextval = (uint16_t *)ws_get(ctx, "nextval", (size_t)TN * 2, &rc);
  if (rc) return rc;
  const int64_t TB = (int64_t)t * b;
  int32_t *size0 = (int32_t *)ws_get(ctx, "size0", (size_t)TB * 4, &rc);
  if (rc) return rc;
  int32_t *ascan0 = (int32_t *)ws_get(ctx, "ascan0", (size_t)(TB + 1) * 4 * 2, &rc);
  if (rc) return rc;
  int32_t *aflag0 = ascan0 + TB + 1;
  unsigned long long *acc = (unsigned long long *)ws_get(ctx, "acc", 64, &rc);
  if (rc) return rc;
  int32_t *hsmall = (int32_t *)ctx->h_small;

  // ---- K2 level 0: Alg. 1, B_f[H_f(u)] <- B_f[H_f(u)] ∪ {u}
  C2_CUDA(ctx, cudaMemsetAsync(size0, 0, (size_t)TB * 4, st));
  C2_CUDA(ctx, cudaMemsetAsync(acc, 0, 64, st));
  if (b <= 16384) {
    const int64_t chunk = 8192;
    C2_CUDA(ctx, cudaFuncSetAttribute(k_level0h, cudaFuncAttributeMaxDynamicSharedMemorySize, b * 4));
    k_level0h<<<(unsigned)((TN + chunk - 1) / chunk), 512, (size_t)b * 4, st>>>(sk, TN, n, b, chunk, key, curval,
                                                                              size0);
    C2_LAUNCHED(ctx, "k_level0h");
  } else {
    k_level0<<<nblk(TN), 256, 0, st>>>(sk, TN, n, b, key, curval, size0);
    C2_LAUNCHED(ctx, "k_level0");
  }
  // ---- K3 on the device (N1): the whole split loop in one cooperative kernel when its histogram
  //      bound (at most t*n/(N+1) nodes larger than N at any level, b bins each) is moderate
  const int64_t hcap = std::max<int64_t>(TB, (TN / (N + 1)) * (int64_t)b);
  if (ctx->split_dev && hcap <= ((int64_t)1 << 25)) {
    SplitDev sd;
    char *base = (char *)ws_get(ctx, "split_dev", (size_t)hcap * 12 + (size_t)TN * 18 + 4096 * 8 + 256, &rc);
    if (rc) return rc;
    sd.hist = (int32_t *)base;
    sd.child_id = sd.hist + hcap;
    sd.child_slot = sd.child_id + hcap;
    sd.act_q[0] = sd.child_slot + hcap;
    sd.act_q[1] = sd.act_q[0] + TN;
    sd.act_s[0] = sd.act_q[1] + TN;
    sd.act_s[1] = sd.act_s[0] + TN;
    sd.part = (unsigned long long *)(((uintptr_t)(sd.act_s[1] + TN) + 15) & ~(uintptr_t)15);
    sd.act_n = (int32_t *)(sd.part + 4096);
    sd.out = (long long *)(sd.part + 4097);
    sd.nvb = (uint16_t *)(sd.part + 4106);
    sd.hcap = hcap;
    C2_CUDA(ctx, cudaMemsetAsync(sd.act_n, 0, 8 + 9 * 8, st));
    auto kfn = htab ? k_split_dev<true> : k_split_dev<false>;
    int occ = 0;
    C2_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, 256, 0));
    const int grid = std::min(ctx->num_sms * std::max(occ, 1), 4096);
    int64_t TBa = TB, TNa = TN, Na = N;
    int32_t na = n, ba = b, ma = m;
    int Da = Deff;
    const int32_t *oa = csr.offs, *ia = csr.items;
    uint16_t *skw = sk;
    void *args[] = {&sd, &sk, &skw, &key, &curval, &size0, &TBa, &TNa, &na, &Da, &ba, &Na, &oa, &ia, &ha, &htab, &ma};
    C2_CUDA(ctx, cudaLaunchCooperativeKernel((const void *)kfn, grid, 256, args, 0, st));
    C2_LAUNCHED(ctx, "k_split_dev");
    if (ctx->timing) cudaEventRecord(ev[2], st);
    return canonicalize(ctx, n, t, N, key, TB + TN, 0, 0, out, sd.out);
  }
  k_flag_gt<<<nblk(TB), 256, 0, st>>>(size0, TB, N, aflag0);
  C2_LAUNCHED(ctx, "k_flag_gt");
  C2_TRY(scan_exclusive(ctx, aflag0, ascan0, TB));
  k_slot0<<<nblk(TN), 256, 0, st>>>(key, size0, ascan0, TN, N, slot);
  C2_LAUNCHED(ctx, "k_slot0");
  C2_CUDA(ctx, cudaMemcpyAsync(hsmall, ascan0 + TB, 4, cudaMemcpyDeviceToHost, st));
  C2_TRY(stream_sync(ctx, "level0"));
  int64_t n_active = hsmall[0];
  int64_t next_id = TB;
  int64_t split_nodes = 0, max_depth = 0;

  // ---- K3 recursive split, one level per iteration (batched over active nodes)
  const int64_t max_hist = (int64_t)1 << 26;
  int64_t batch = std::max<int64_t>(1, max_hist / b);
  for (int d = 0; n_active > 0; ++d) {
    if (d > b + 1) return set_err(ctx, C2_ECUDA, "split did not terminate");
    int64_t new_active = 0, children_lvl = 0;
    C2_CUDA(ctx, cudaMemsetAsync(slot2, 0xFF, (size_t)TN * 4, st));
    for (int64_t a0 = 0; a0 < n_active; a0 += batch) {
      int64_t a1 = std::min(n_active, a0 + batch);
      int64_t E = (a1 - a0) * b;
      int32_t *hist = (int32_t *)ws_get(ctx, "hist", (size_t)E * 4, &rc);
      if (rc) return rc;
      int32_t *fbuf = (int32_t *)ws_get(ctx, "hflags", (size_t)(E + 1) * 4 * 4, &rc);
      if (rc) return rc;
      int32_t *fc = fbuf, *fa = fbuf + (E + 1), *cscan = fbuf + 2 * (E + 1), *ascan = fbuf + 3 * (E + 1);
      int32_t *cid = (int32_t *)ws_get(ctx, "child_id", (size_t)E * 4 * 2, &rc);
      if (rc) return rc;
      int32_t *cslot = cid + E;
      C2_CUDA(ctx, cudaMemsetAsync(hist, 0, (size_t)E * 4, st));
      if (htab)
        k_split_count<true><<<nblk(TN), 256, 0, st>>>(slot, sk, curval, nextval, TN, n, d, Deff, (int32_t)a0,
                                                      (int32_t)a1, b, hist, csr.offs, csr.items, ha, htab, m);
      else
        k_split_count<false><<<nblk(TN), 256, 0, st>>>(slot, sk, curval, nextval, TN, n, d, Deff, (int32_t)a0,
                                                       (int32_t)a1, b, hist, csr.offs, csr.items, ha, nullptr, 0);
      C2_LAUNCHED(ctx, "k_split_count");
      k_child_flags<<<nblk(E), 256, 0, st>>>(hist, E, N, fc, fa, acc + 1);
      C2_LAUNCHED(ctx, "k_child_flags");
      C2_TRY(scan_exclusive(ctx, fc, cscan, E));
      C2_TRY(scan_exclusive(ctx, fa, ascan, E));
      k_child_assign<<<nblk(E), 256, 0, st>>>(hist, cscan, ascan, E, N, (int32_t)next_id,
                                              (int32_t)new_active, cid, cslot);
      C2_LAUNCHED(ctx, "k_child_assign");
      k_split_apply<<<nblk(TN), 256, 0, st>>>(slot, key, curval, nextval, TN, (int32_t)a0, (int32_t)a1, b, cid,
                                              cslot, slot2);
      C2_LAUNCHED(ctx, "k_split_apply");
      C2_CUDA(ctx, cudaMemcpyAsync(hsmall, cscan + E, 4, cudaMemcpyDeviceToHost, st));
      C2_CUDA(ctx, cudaMemcpyAsync(hsmall + 1, ascan + E, 4, cudaMemcpyDeviceToHost, st));
      C2_TRY(stream_sync(ctx, "split level"));
      next_id += hsmall[0];
      children_lvl += hsmall[0];
      new_active += hsmall[1];
      if (next_id >= (int64_t)INT32_MAX / 2) return set_err(ctx, C2_EINVAL, "too many split nodes");
    }
    split_nodes += n_active;
    if (children_lvl > 0) max_depth = d + 1;
    std::swap(slot, slot2);  // slot2 was reset to -1 before the level; active users rewritten
    n_active = new_active;
  }
  if (ctx->timing) cudaEventRecord(ev[2], st);

  return canonicalize(ctx, n, t, N, key, next_id, split_nodes, max_depth, out);
}

// ------------------------------------------------------------------ C^2/MinHash variant (N3)
// per function, u's cluster is the item of P_u with the smallest full-range hash
// z_f(x) = a_f*x + c_f mod 2^64 (ties: lower item id) -- one cluster per item, no splitting.
// Warp per user; lane f (+32) handles function f; item loads are warp broadcasts.
__global__ void k_minhash_key(const int32_t *__restrict__ offs, const int32_t *__restrict__ items, int32_t n, int t,
                              HashArgs2 ha, int64_t m, int32_t *__restrict__ key) {
  const int lane = threadIdx.x & 31;
  const int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (u >= n) return;
  const int32_t p0 = offs[u], p1 = offs[u + 1];
  for (int f = lane; f < t; f += 32) {
    const uint64_t a = ha.a[f], c = ha.c[f];
    uint64_t best = ~0ull;
    int32_t arg = INT32_MAX;
    for (int32_t p = p0; p < p1; ++p) {
      const int32_t x = __ldg(items + p);
      const uint64_t z = a * (uint64_t)(uint32_t)x + c;
      if (z < best || (z == best && x < arg)) {
        best = z;
        arg = x;
      }
    }
    key[(int64_t)f * n + u] = (int32_t)((int64_t)f * m + arg);
  }
}

int minhash_clusters(c2_ctx *ctx, const Csr &csr, int t, int64_t N, const HashParams *hp, Clusters *out) {
  int rc;
  const int32_t n = csr.n;
  const int64_t TN = (int64_t)t * n;
  const int64_t m = (int64_t)csr.max_item + 1;
  if ((int64_t)t * m + TN + 1 >= (int64_t)INT32_MAX / 2)
    return set_err(ctx, C2_EINVAL, "MinHash clustering needs t * (max item id + 1) < 2^30");
  HashArgs2 ha;
  for (int f = 0; f < t; ++f) {
    ha.a[f] = hp->a[f];
    ha.c[f] = hp->c[f];
  }
  cudaStream_t st = ctx->stream;
  if (ctx->timing) {
    cudaEventRecord(ctx->ev[0], st);
    cudaEventRecord(ctx->ev[1], st);
  }
  int32_t *key = (int32_t *)ws_get(ctx, "key", (size_t)TN * 4, &rc);
  if (rc) return rc;
  unsigned long long *acc = (unsigned long long *)ws_get(ctx, "acc", 64, &rc);
  if (rc) return rc;
  C2_CUDA(ctx, cudaMemsetAsync(acc, 0, 64, st));
  k_minhash_key<<<nblk((int64_t)n * 32), 256, 0, st>>>(csr.offs, csr.items, n, t, ha, m, key);
  C2_LAUNCHED(ctx, "k_minhash_key");
  if (ctx->timing) cudaEventRecord(ctx->ev[2], st);
  return canonicalize(ctx, n, t, N, key, (int64_t)t * m, 0, 0, out);
}

}  // namespace c2
