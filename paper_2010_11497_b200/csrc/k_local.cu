// k_local.cu -- Step 2 of C^2 on the GPU: brute-force Jaccard top-k inside every cluster
// (Alg. 2, brute-force branch; s(s-1)/2 similarities per cluster).
//
// K5 worklist.  Clusters of more than 32 users ("big") are ordered by function, then by size
//    (largest first: the paper's decreasing priority queue) and cut into 32-user
//    slices; clusters of 2..32 users are packed 32/slot per "mixed" slice, each in an aligned
//    group of slot = 2^ceil(log2 s) positions (pairs across groups are ignored).  Then, once
//    per call:
//      vperm   members of the cluster sorted by |P_v| (descending), so the 32 lists of a
//              slice have similar lengths;
//      packed  for every (slice, item window) a block of u16 window-local item ids laid out
//              [p/8][lane][8] and padded to the slice's longest list with W (M[W] == 0).
//    A warp then streams the 32 lists of a slice with one 16-byte coalesced load per lane per
//    8 items, with no divergence and no bounds checks.
// K7 k_local_tile: persistent CTAs (one per SM), one work item = one slice R (32 rows) of cluster
//    C.  For every item window, shared memory holds the transposed membership mask M[x] =
//    {r in R : x in P_r} (bit r).  Each thread owns VPT slices' lanes (one v each) and
//    accumulates the 32 counts |P_r ∩ P_v| bit-sliced with carry-save adders over 16 masks, so
//    one LDS + ~4 LOP3 serve 32 pairs.  A 32x32 bit transpose turns the planes into counts,
//    stored as cnt[row][member] in shared memory aliased onto the dead M.  The next tile's
//    descriptor record, row blocks and running lists arrive by cp.async during this tile.
// K8 (in K7): exact top-k per row under the order i1*U2 > i2*U1, ties by lower id; one warp per
//    row (rows taken dynamically).  A candidate must beat tau = the row's running Alg. 3 k-th
//    best (fused mode; it never decreases, so the pruning is exact) -- a 2-IMAD test; rows
//    without a full running list, or whose tau lets more than 64 through, first get a bound
//    from round 1 (each lane's best two -> the k-th best of those 64).  Survivors go to a
//    private queue, then are inserted one by one (<= 16) or sorted on exact 64-bit keys and
//    merged into the running list in place, duplicate ids dropped.
#include <algorithm>
#include <vector>

#include "c2_internal.cuh"
#include "cand.cuh"
#include "k_rows.cuh"
#include "k_gf_mma.cuh"

#ifndef C2_LIGHT
#define C2_LIGHT 1  // 1: light rows (full running list) filtered in the phase-A epilogue, merged by k_surv_merge
#endif
#ifndef C2_SNAKE
#define C2_SNAKE 1  // 1: warp w probes slices w, 2W-1-w, 2W+w, ... (slices are longest-first: balances warps)
#endif
#ifndef C2_BULK
#define C2_BULK 1  // 1: tile records + staged row blocks by cp.async.bulk on mbarriers (TMA bulk path)
#endif
#ifndef C2_SPLIT
#define C2_SPLIT 1  // 1: tiles of <= 8 slices split each member list over several warps
#endif
#ifndef C2_HSPLIT
#define C2_HSPLIT 0  // tiles of > TILE_WARPS/2 slices with a free counter slot: the C2_HSPLIT longest slices
                     // (members are longest-first) are each probed by TILE_WARPS/C2_HSPLIT warps (0: off)
#endif
#ifndef C2_KSTATS_STEPS
#define C2_KSTATS_STEPS 0  // 1: kstats also count the probe steps of each tile's busiest warp (diagnostic
                           // build: the extra live register costs 0.7 ms per c5 build even with kstats off)
#endif
#ifndef C2_NHI7
#define C2_NHI7 1  // 1: an 11-plane counter instantiation (item lists of <= 2047) beside the 8-, 12- and 15-plane ones
#endif
#ifndef C2_HIPLANES
#define C2_HIPLANES 0  // h > 0: tiles whose rows all hold < 16 * 2^h items skip the probe's carry ripple above plane H[h-1]
#endif
#ifndef C2_RANKMERGE
#define C2_RANKMERGE 1  // 1: rank-based Alg. 3 step for <= 32 survivors; 0: insertion (<= 16)
#endif

namespace c2 {


// cp.async (sm_80+ async global->shared copies; completion by cp.async.wait_all)
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier: any thread can wait for
// bytes another thread requested (unlike cp.async groups, which only the issuing thread can wait on).
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mb))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *mb, uint32_t parity) {
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(mb)), "r"(parity)
        : "memory");
    if (done) break;
  }
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }


#ifndef C2_TILE_T
#define C2_TILE_T 512
#endif
#ifndef C2_TILE_MINB
#define C2_TILE_MINB 1
#endif
#ifndef C2_FILL_COAL
#define C2_FILL_COAL 1  // multi-window packing: k_sl_fill_coal (coalesced CSR reads) instead of k_sl_fill_rows
#endif
#ifndef C2_EPI_BAR
#define C2_EPI_BAR 1  // keep the light epilogue's barrier even when no row can overflow (measured: without
                      // it c5 takes 56.0 vs 52.9 ms -- the warps drift apart before the next tile)
#endif
#ifndef C2_SIDE_MERGE
#define C2_SIDE_MERGE 1  // light rows' merge on a side stream, concurrent with k_row_topk
#endif
#ifndef C2_PACK32
#define C2_PACK32 0  // 1: packed member lists hold 32-bit byte offsets into the mask M (4 per 16-byte row and
                     // lane; the probe's mask loads need no id extraction) instead of 16-bit ids (8 per row).
                     // Measured at c5: the probe loop drops from ~143 to ~67 instructions per 16 items,
                     // yet the tile kernel takes 35.3 vs 34.4 ms and the packing 2.8 vs 2.0 ms (twice
                     // the bytes): the probe is not issue-bound.  Off by default; parity-tested.
#endif
#ifndef C2_SMEM_BUDGET
#define C2_SMEM_BUDGET 0  // bytes of dynamic shared memory per tile CTA (0: the opt-in maximum)
#endif
constexpr int TILE_T = C2_TILE_T;
constexpr int TILE_WARPS = TILE_T / 32;
constexpr int MAX_WIN = 16;

static inline unsigned nblk(int64_t x, int bs = 256) { return (unsigned)((x + bs - 1) / bs); }

// Packed member lists: per (32-member slice, window) block, rows of 512 bytes; row t holds, for
// the member in lane e, its list positions IPR*t .. IPR*t+IPR-1 as PackT: the window-local item
// id (16-bit) or its byte offset in the mask M (32-bit, C2_PACK32).  Pads: enc(W), with M[W] = 0.
constexpr int IPR = C2_PACK32 ? 4 : 8;
typedef std::conditional<C2_PACK32 != 0, uint32_t, uint16_t>::type PackT;
__host__ __device__ __forceinline__ PackT pk_enc(uint32_t id) { return (PackT)(C2_PACK32 ? id * 4u : id); }
__device__ __forceinline__ PackT *pk_row_ptr(PackT *base, int64_t blk_off, int e) {
  return base + blk_off * (32 * IPR) + e * IPR;
}
__device__ __forceinline__ int64_t pk_idx(int pos) { return (int64_t)(pos / IPR) * (32 * IPR) + (pos % IPR); }
// rows of a block holding c items per member; 32-bit packing rounds to whole quads of rows (the
// probe's step) so its loads never need a bounds test
__host__ __device__ __forceinline__ int32_t pk_rows(int32_t c) {
  const int32_t r = (c + IPR - 1) / IPR;
  return C2_PACK32 ? (r + 3) & ~3 : r;
}
constexpr int PK_SLACK_ROWS = 8;  // rows readable past any block (prefetch of the probe's next step)
static inline int bits_for(int64_t x) {
  int b = 1;
  while ((1LL << b) < x) ++b;
  return b;
}

// ------------------------------------------------------------------ K5 worklist
__device__ __forceinline__ int find_f(const int32_t *ccum, int t, int64_t g) {
  int f = 0;
  while (f + 1 < t && ccum[f + 1] <= g) ++f;
  return f;
}

// category of every cluster: big (> 32 users), small (2..32), single.  One 32-bit sort key
// orders them [big: by function, then size descending][small: by function, slot class]
// [single: by function]; counts per (category, f, class) go to cnt_fc.
constexpr int WLC = 16;  // counters per function: 0 big tiles, 1..5 small per class, 6 single, 7 big, 8 hyrec,
                         // 9 members of big clusters
__device__ __forceinline__ int slot_class(int32_t s) {  // slot = 2^class >= s, s in [2, 32]
  int c = 1;
  while ((1 << c) < s) ++c;
  return c;
}

__device__ __forceinline__ void k_wl_classify_one(const int32_t *__restrict__ offsets, const int32_t *__restrict__ ccum,
                                                  int t, int32_t n, int64_t g, uint32_t *__restrict__ key,
                                                  uint32_t *__restrict__ val, uint32_t maxs, int sized,
                                                  int32_t *__restrict__ cnt_fc, uint32_t hyrec_min, int sb) {
  // sort key: class (2 bits) | function (6 bits) | sb bits of size field; only these 8 + sb bits
  // are sorted (radix passes of 5 bits)
  int f = find_f(ccum, t, g);
  const int fs = sb, cs = sb + 6;
  int64_t c = g - ccum[f];
  const int32_t *off = offsets + (int64_t)f * (n + 1);
  uint32_t s = (uint32_t)(off[c + 1] - off[c]);
  uint32_t k;
  if (s >= hyrec_min) {  // Alg. 2 else-branch: Hyrec (C2_SOLVER_HYBRID only; hyrec_min = UINT32_MAX otherwise)
    k = (3u << cs) | ((uint32_t)f << fs);
    atomicAdd(&cnt_fc[f * WLC + 8], 1);
  } else if (s > 32) {
    k = ((uint32_t)f << fs) | (sized ? min(maxs - s, (1u << sb) - 1u) : 0u);
    atomicAdd(&cnt_fc[f * WLC + 0], (int32_t)((s + 31) / 32));  // big tiles of f
    atomicAdd(&cnt_fc[f * WLC + 7], 1);                          // big clusters of f
    atomicAdd(&cnt_fc[f * WLC + 9], (int32_t)s);                 // their members
  } else if (s >= 2) {
    int cl = slot_class((int32_t)s);
    k = (1u << cs) | ((uint32_t)f << fs) | (uint32_t)cl;
    atomicAdd(&cnt_fc[f * WLC + cl], 1);  // small clusters of (f, class), class 1..5
  } else {
    k = (2u << cs) | ((uint32_t)f << fs);
    atomicAdd(&cnt_fc[f * WLC + 6], 1);  // singletons of f
  }
  key[g] = k;
  val[g] = (uint32_t)g;
}

__global__ void k_wl_classify(const int32_t *__restrict__ offsets, const int32_t *__restrict__ ccum, int t,
                              int32_t n, int64_t C, uint32_t *__restrict__ key, uint32_t *__restrict__ val,
                              uint32_t maxs, int sized, int32_t *__restrict__ cnt_fc_g, uint32_t hyrec_min, int sb) {
  // counters summed per block in shared memory, then one global atomic per non-zero counter
  __shared__ int32_t cnt_fc[WLC * C2_MAX_T];
  for (int i = threadIdx.x; i < WLC * t; i += blockDim.x) cnt_fc[i] = 0;
  __syncthreads();
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < C) k_wl_classify_one(offsets, ccum, t, n, g, key, val, maxs, sized, cnt_fc, hyrec_min, sb);
  __syncthreads();
  for (int i = threadIdx.x; i < WLC * t; i += blockDim.x)
    if (cnt_fc[i]) atomicAdd(&cnt_fc_g[i], cnt_fc[i]);
}

__global__ void k_bc_sizes(const uint32_t *__restrict__ sval, int64_t nbig, const int32_t *__restrict__ offsets,
                           const int32_t *__restrict__ ccum, int t, int32_t n, int32_t *__restrict__ ssz,
                           int32_t *__restrict__ nsl) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nbig) return;
  int64_t g = sval[i];
  int f = find_f(ccum, t, g);
  int64_t c = g - ccum[f];
  const int32_t *off = offsets + (int64_t)f * (n + 1);
  int32_t s = off[c + 1] - off[c];
  ssz[i] = s;
  nsl[i] = (s + 31) / 32;
}

__global__ void k_bc_fill(const uint32_t *__restrict__ sval, int64_t nbig, const int32_t *__restrict__ offsets,
                          const int32_t *__restrict__ ccum, int t, int32_t n, const int32_t *__restrict__ vp_scan,
                          const int32_t *__restrict__ sl_scan, BigC *__restrict__ bcs, Tile *__restrict__ tiles,
                          int32_t *__restrict__ bstart) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nbig) return;
  int64_t g = sval[i];
  int f = find_f(ccum, t, g);
  int64_t c = g - ccum[f];
  const int32_t *off = offsets + (int64_t)f * (n + 1);
  int32_t s = off[c + 1] - off[c];
  BigC b{f, s, vp_scan[i], sl_scan[i], 0, 0};
  bcs[i] = b;
  bstart[i] = off[c];
  int ns = (s + 31) / 32;
  for (int j = 0; j < ns; ++j) tiles[b.sl_off + j] = Tile{(int32_t)i, j};
}

// small clusters (sorted by (f, class)): place members into their mixed slice
struct MixGroup {
  int32_t f, cls, first_entry, count, first_slice;  // entries = positions in the sorted small list
};
__global__ void k_mix_fill(const uint32_t *__restrict__ sval_small, int64_t nsmall, const int32_t *__restrict__ offsets,
                           const int32_t *__restrict__ ccum, int t, int32_t n, const int32_t *__restrict__ members,
                           const MixGroup *__restrict__ groups, int ngroups, int32_t vp_base,
                           const int32_t *__restrict__ psize, int32_t *__restrict__ vperm,
                           int32_t *__restrict__ vsize) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsmall) return;
  int gi = 0;
  while (gi + 1 < ngroups && groups[gi + 1].first_entry <= i) ++gi;
  const MixGroup G = groups[gi];
  int64_t g = sval_small[i];
  int f = find_f(ccum, t, g);
  int64_t c = g - ccum[f];
  const int32_t *off = offsets + (int64_t)f * (n + 1);
  int32_t st = off[c], s = off[c + 1] - st;
  int q = (int)(i - G.first_entry);
  int per = 32 >> G.cls;
  int64_t slice = G.first_slice + q / per;
  int pos = (q % per) << G.cls;
  int32_t *dst = vperm + vp_base + slice * 32 + pos;
  int32_t *dsz = vsize + vp_base + slice * 32 + pos;
  for (int j = 0; j < s; ++j) {
    const int32_t v = members[(int64_t)f * n + st + j];
    dst[j] = v;
    dsz[j] = psize[v];
  }
}

__global__ void k_mix_bc(const MixGroup *__restrict__ groups, int ngroups, int64_t nmix, int64_t nbig, int32_t vp_base,
                         int64_t sl_base, BigC *__restrict__ bcs, Tile *__restrict__ tiles) {
  int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= nmix) return;
  int gi = 0;
  while (gi + 1 < ngroups && groups[gi + 1].first_slice <= m) ++gi;
  bcs[nbig + m] = BigC{groups[gi].f, 32, (int32_t)(vp_base + m * 32), (int32_t)(sl_base + m), 1 << groups[gi].cls, 0};
  tiles[sl_base + m] = Tile{(int32_t)(nbig + m), 0};
}

// singletons: no candidates.  local: pad rows; fused: running list carried over unchanged.
__global__ void k_singles(const uint32_t *__restrict__ sval_single, int64_t nsingle, const int32_t *__restrict__ offsets,
                          const int32_t *__restrict__ ccum, int t, int32_t n, const int32_t *__restrict__ members,
                          int k, int64_t lo, int64_t hi, const c2_cand *__restrict__ seed,
                          c2_cand *__restrict__ out) {
  int64_t e = lo * k + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= hi * k) return;
  int64_t i = e / k;
  int j = (int)(e % k);
  int64_t g = sval_single[i];
  int f = find_f(ccum, t, g);
  int64_t c = g - ccum[f];
  int32_t u = members[(int64_t)f * n + offsets[(int64_t)f * (n + 1) + c]];
  if (seed) out[(int64_t)u * k + j] = seed[(int64_t)u * k + j];
  else out[((int64_t)f * n + u) * k + j] = c2_cand{-1, 0, 0};
}

// vperm: members of each big cluster sorted by |P_v| descending (ties by position).  One CTA
// per cluster, bitonic sort in shared memory for s <= 2048 (larger clusters keep the
// canonical order: performance only, results do not depend on it).
__global__ void __launch_bounds__(256) k_sl_sort(const BigC *__restrict__ bcs, const int32_t *__restrict__ bstart,
                                                  const int32_t *__restrict__ members, int32_t n,
                                                  const int32_t *__restrict__ psize, int32_t *__restrict__ vperm,
                                                  int32_t *__restrict__ vsize) {
  __shared__ uint32_t key[2048];
  const BigC b = bcs[blockIdx.x];
  const int32_t *mem = members + (int64_t)b.f * n + bstart[blockIdx.x];
  int32_t *out = vperm + b.vp_off;
  int32_t *osz = vsize + b.vp_off;
  if (b.s > 2048) {
    for (int i = threadIdx.x; i < b.s; i += blockDim.x) {
      out[i] = mem[i];
      osz[i] = psize[mem[i]];
    }
    return;
  }
  int P = 64;
  while (P < b.s) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    uint32_t ps = i < b.s ? (uint32_t)min(psize[mem[i]], 32767) : 0u;
    key[i] = i < b.s ? ((32767u - ps) << 16) | (uint32_t)i : 0xFFFFFFFFu;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool up = ((lo & size) == 0);
        uint32_t a = key[lo], c = key[hi];
        if ((a > c) == up) {
          key[lo] = c;
          key[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < b.s; i += blockDim.x) {
    const int32_t v = mem[key[i] & 0xFFFF];
    out[i] = v;
    osz[i] = psize[v];
  }
}

// Packed operand lists.  One warp per member position (slice sl, lane slot e): lanes stride the
// member's sorted items (coalesced reads); each window is a filter pass with ballot compaction.
// blk_len8[slice][w] = ceil(max over the slice's 32 lists of |list ∩ window w| / 8) (atomicMax;
// zeroed before).
// One 512-byte descriptor record per tile item, so the tile kernel's next-tile fetch is a
// single cp.async instead of a chain of dependent loads: [0,2) Tile, [2,8) BigC, [8,24) rows'
// block lengths per window, [24,40) block offsets, [64,96) row user ids, [96,128) row |P_u|.
constexpr int REC_W = 128;
__global__ void k_tile_rec(const Tile *__restrict__ tiles, int64_t nslices, const BigC *__restrict__ bcs,
                           const int32_t *__restrict__ vperm, const int32_t *__restrict__ vsize,
                           const int32_t *__restrict__ blk_len8, const int32_t *__restrict__ blk_off8, int nwin,
                           int32_t *__restrict__ rec) {
  const int lane = threadIdx.x & 31;
  const int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (it >= nslices) return;
  const Tile T = tiles[it];
  const BigC B = bcs[T.bc];
  int32_t *r = rec + it * REC_W;
  const int vi = T.j * 32 + lane;
  r[64 + lane] = vi < B.s ? vperm[B.vp_off + vi] : -1;
  r[96 + lane] = vi < B.s ? vsize[B.vp_off + vi] : 0;
  const int64_t sb = (int64_t)(B.sl_off + T.j) * nwin;
  if (lane < 16) {
    r[8 + lane] = lane < nwin ? blk_len8[sb + lane] : 0;
    r[24 + lane] = lane < nwin ? blk_off8[sb + lane] : 0;
  }
  if (lane == 0) {
    r[0] = T.bc, r[1] = T.j;
    r[2] = B.f, r[3] = B.s, r[4] = B.vp_off, r[5] = B.sl_off, r[6] = B.slot, r[7] = B.kc;
  }
}

__device__ __forceinline__ int32_t lower_bound_items(const int32_t *__restrict__ items, int32_t lo, int32_t hi,
                                                     int32_t x) {  // first p in [lo,hi) with items[p] >= x
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (items[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Rows are sorted, so window w of a member's list is the contiguous range [lb(wW), lb((w+1)W)):
// one thread per member position finds its window boundaries by binary search (no item walk)
// and folds the lengths into the slice maxima.
// Per user, once per call (not once per function): the inner window boundaries of its sorted row,
// ub[u][w-1] = first position with item >= w*W (w = 1..nwin-1).
__global__ void k_user_bounds(const int32_t *__restrict__ offs, const int32_t *__restrict__ items, int32_t n,
                              int32_t W, int nwin, int32_t *__restrict__ ub) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  int32_t p = offs[u];
  const int32_t pe = offs[u + 1];
  for (int w = 1; w < nwin; ++w) {
    p = lower_bound_items(items, p, pe, w * W);
    ub[u * (nwin - 1) + w - 1] = p;
  }
}

__global__ void k_sl_len(const Tile *__restrict__ tiles, int64_t nslices, const BigC *__restrict__ bcs,
                         const int32_t *__restrict__ vperm, const int32_t *__restrict__ offs,
                         const int32_t *__restrict__ ub, int32_t W, int nwin, int32_t *__restrict__ blk_len8,
                         int32_t *__restrict__ bounds) {
  const int lane = threadIdx.x & 31;
  const int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (sl >= nslices) return;
  const Tile T = tiles[sl];
  const BigC b = bcs[T.bc];
  const int vi = T.j * 32 + lane;
  const int32_t v = vi < b.s ? vperm[b.vp_off + vi] : -1;
  int32_t p = v >= 0 ? offs[v] : 0;
  const int32_t pe = v >= 0 ? offs[v + 1] : 0;
  int32_t *bd = bounds + (sl * 32 + lane) * (nwin + 1);  // window w of this member: [bd[w], bd[w+1])
  bd[0] = p;
  for (int w = 0; w < nwin; ++w) {
    const int32_t q = w + 1 < nwin ? (v >= 0 ? ub[(int64_t)v * (nwin - 1) + w] : 0) : pe;
    bd[w + 1] = q;
    int c = q - p;
    p = q;
#pragma unroll
    for (int o = 16; o; o >>= 1) c = max(c, __shfl_xor_sync(0xffffffffu, c, o));
    if (lane == 0) blk_len8[sl * nwin + w] = pk_rows(c);
  }
}

// Order within a list does not matter to the counts, so each member's window list is laid out
// by bank: key = (x - e) mod 32 for the member in lane e (the mask word of item x sits in bank
// x mod 32).  At any step the 32 lanes then read words of ~32 different banks instead of random
// ones (random: ~3.4 shared-memory wavefronts per mask load, which binds the probe).
__global__ void __launch_bounds__(256) k_sl_fill(int64_t nslices, const int32_t *__restrict__ bounds,
                                                 const int32_t *__restrict__ items, int32_t W, int nwin,
                                                 const int32_t *__restrict__ blk_len8,
                                                 const int32_t *__restrict__ blk_off8, PackT *__restrict__ packedT,
                                                 int bank_order) {
  __shared__ int hist[8][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t sl = g >> 5;
  if (sl >= nslices) return;
  const int e = (int)(g & 31);
  const int32_t *bd = bounds + g * (nwin + 1);
  int *h = hist[wib];
  for (int w = 0; w < nwin; ++w) {
    const int32_t lo = w * W;
    // this window's items: the contiguous range [pb, pe) of the sorted row (from k_sl_len)
    const int32_t pb = bd[w], pe = bd[w + 1];
    const int32_t len = blk_len8[sl * nwin + w] * IPR;
    PackT *dst = pk_row_ptr(packedT, blk_off8[sl * nwin + w], e);
    if (!bank_order) {  // plain order: one pass, ballot compaction
      int cnt = 0;
      for (int32_t p0 = pb; p0 < pe; p0 += 32) {
        const int32_t p = p0 + lane;
        const int32_t r = p < pe ? items[p] - lo : -1;
        const bool in = r >= 0 && r < W;
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        const int pos = cnt + __popc(bal & ((1u << lane) - 1));
        if (in) dst[pk_idx(pos)] = pk_enc((uint32_t)r);
        cnt += __popc(bal);
      }
      for (int pos = cnt + lane; pos < len; pos += 32) dst[pk_idx(pos)] = pk_enc((uint32_t)W);
      continue;
    }
    h[lane] = 0;
    __syncwarp();
    int cnt = 0;
    for (int32_t p0 = pb; p0 < pe; p0 += 32) {
      const int32_t p = p0 + lane;
      const int32_t r = p < pe ? items[p] - lo : -1;
      const bool in = r >= 0 && r < W;
      if (in) atomicAdd(&h[(r - e) & 31], 1);
      cnt += __popc(__ballot_sync(0xffffffffu, in));
    }
    __syncwarp();
    int c = h[lane], x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    __syncwarp();
    h[lane] = x - c;  // bucket starts
    __syncwarp();
    for (int32_t p0 = pb; p0 < pe; p0 += 32) {
      const int32_t p = p0 + lane;
      const int32_t r = p < pe ? items[p] - lo : -1;
      if (r >= 0 && r < W) {
        const int pos = atomicAdd(&h[(r - e) & 31], 1);
        dst[pk_idx(pos)] = pk_enc((uint32_t)r);
      }
    }
    for (int pos = cnt + lane; pos < len; pos += 32) dst[pk_idx(pos)] = pk_enc((uint32_t)W);
    __syncwarp();
  }
}

// Plain order (multi-window runs): the items of member e in window w are the contiguous range
// [bd[w], bd[w+1]) of its sorted row, so position p of its list is item bd[w] + p.  One warp per
// 16-byte row t of a (slice, window) block: lane e gathers positions 8t..8t+7 of member e and the
// warp writes the block's 512-byte row t with one coalesced uint4 store per lane (the per-list
// form wrote 2-byte scattered stores, i.e. partial sectors).
#if !C2_PACK32
__global__ void __launch_bounds__(256) k_sl_fill_rows(int64_t nb, int nwin, const int32_t *__restrict__ bounds,
                                                      const int32_t *__restrict__ items, int32_t W,
                                                      const int32_t *__restrict__ blk_len8,
                                                      const int32_t *__restrict__ blk_off8, uint4 *__restrict__ packed,
                                                      int64_t nnz, int vec) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwg = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // warps walk the blocks' rows in order: block b, row t (the row index space is blk_off8's)
  for (int64_t b = gw >> 3; b < nb; b += nwg >> 3) {
    const int sub = (int)(gw & 7);
    const int64_t sl = b / nwin;
    const int w = (int)(b - sl * nwin);
    const int32_t *bd = bounds + (sl * 32 + lane) * (nwin + 1);
    const int32_t pb = bd[w], pe = bd[w + 1];
    const int32_t lo = w * W;
    const int32_t len8 = blk_len8[b];
    uint4 *out = packed + (int64_t)blk_off8[b] * 32 + lane;
    for (int t = sub; t < len8; t += 8) {
      uint32_t h[8];
      const int32_t p0 = pb + 8 * t;
      if (p0 >= pe) {  // past this member's list: padding only
#pragma unroll
        for (int j = 0; j < 8; ++j) h[j] = (uint32_t)W;
      } else if (vec && ((int64_t)(p0 & ~3) + 12 <= nnz)) {
        // three aligned 16-byte loads cover the 8 items [p0, p0 + 8) (items is 16-byte aligned)
        const int32_t a0 = p0 & ~3, o = p0 & 3;
        const int4 A = __ldg(reinterpret_cast<const int4 *>(items + a0));
        const int4 Bv = __ldg(reinterpret_cast<const int4 *>(items + a0 + 4));
        const int4 Cv = o ? __ldg(reinterpret_cast<const int4 *>(items + a0 + 8)) : make_int4(0, 0, 0, 0);
        const int32_t x[12] = {A.x, A.y, A.z, A.w, Bv.x, Bv.y, Bv.z, Bv.w, Cv.x, Cv.y, Cv.z, Cv.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int32_t v = o == 0 ? x[j] : o == 1 ? x[j + 1] : o == 2 ? x[j + 2] : x[j + 3];
          h[j] = p0 + j < pe ? (uint32_t)(v - lo) : (uint32_t)W;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int32_t p = p0 + j;
          h[j] = p < pe ? (uint32_t)(__ldg(items + p) - lo) : (uint32_t)W;
        }
      }
      out[(int64_t)t * 32] = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
    }
  }
}
#endif

// Same output as k_sl_fill_rows, with the CSR read coalesced: one warp per (slice, window) block
// takes its 32 members one after the other, the lanes reading consecutive items of a member (full
// 128-byte lines), and transposes them through a shared-memory stage of FR_R rows
// ([row][lane][8] u16, pre-filled with the pad W) that it then writes out as whole 512-byte rows.
constexpr int FR_WARPS = 4;
constexpr int FR_R = 8;  // rows (of 8 items per member) staged per pass
__global__ void __launch_bounds__(FR_WARPS * 32) k_sl_fill_coal(int64_t nb, int nwin, const int32_t *__restrict__ bounds,
                                                               const int32_t *__restrict__ items, int32_t W,
                                                               const int32_t *__restrict__ blk_len8,
                                                               const int32_t *__restrict__ blk_off8,
                                                               uint4 *__restrict__ packed) {
  __shared__ __align__(16) PackT stage[FR_WARPS][FR_R * 32 * IPR];
  constexpr int NH = FR_R * IPR / 32;  // loads per member and chunk
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  PackT *stg = stage[wib];
  uint4 *stg4 = reinterpret_cast<uint4 *>(stg);
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwg = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t pw = C2_PACK32 ? (uint32_t)pk_enc((uint32_t)W) : ((uint32_t)W | ((uint32_t)W << 16));
  const uint4 padv = make_uint4(pw, pw, pw, pw);
  for (int64_t b = gw; b < nb; b += nwg) {
    const int64_t sl = b / nwin;
    const int w = (int)(b - sl * nwin);
    const int32_t *bd = bounds + (sl * 32 + lane) * (nwin + 1);
    const int32_t mpb = bd[w], mpe = bd[w + 1];  // lane e's member: window list [mpb, mpe)
    const int32_t lo = w * W;
    const int32_t len8 = blk_len8[b];
    uint4 *out = packed + (int64_t)blk_off8[b] * 32 + lane;
    for (int32_t t0 = 0; t0 < len8; t0 += FR_R) {
      const int nr = min(FR_R, len8 - t0);
      for (int i = lane; i < nr * 32; i += 32) stg4[i] = padv;
      __syncwarp();
      // members in groups of 8: the group's chunk items (FR_R * IPR each) are all requested
      // before any is stored (8 * NH loads in flight per lane)
      for (int e0 = 0; e0 < 32; e0 += 8) {
        int32_t pbv[8], pev[8], xv[8][NH];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          pbv[i] = __shfl_sync(0xffffffffu, mpb, e0 + i) + IPR * t0;
          pev[i] = min(__shfl_sync(0xffffffffu, mpe, e0 + i), pbv[i] + IPR * nr);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const int32_t p = pbv[i] + 32 * h + lane;
            xv[i][h] = p < pev[i] ? __ldg(items + p) : 0;
          }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const int pos = 32 * h + lane;
            if (pbv[i] + pos < pev[i])
              stg[((pos / IPR) * 32 + e0 + i) * IPR + (pos % IPR)] = pk_enc((uint32_t)(xv[i][h] - lo));
          }
        }
      }
      __syncwarp();
      for (int r = 0; r < nr; ++r) out[(int64_t)(t0 + r) * 32] = stg4[r * 32 + lane];
      __syncwarp();
    }
  }
}

// ------------------------------------------------------------------ cluster-local relabeling
// Only items held by >= 2 members of a cluster can contribute to an intersection, so every
// cluster unit (a big cluster, or one mixed slice of small clusters) gets its own dense item
// universe: the items of in-unit degree >= 2, numbered 0..kc-1 in increasing global id.  Each
// member's list is rewritten in local ids (degree-1 items dropped, order kept) straight into the
// packed [p/8][lane][8] u16 layout, padded with the sentinel kc.  The tile kernel then needs a
// mask M of kc+1 words -- one window, far less shared memory than the global item range -- and
// streams shorter lists.  Results are unchanged: |P_u ∩ P_v| is invariant under dropping items
// that no other member of the unit holds and under renaming items injectively (|P_u| and the
// union still come from the original profile sizes).

// allocation bound per slice: ceil(max original |P_v| over its members / 8)
__global__ void k_sl_maxlen(const Tile *__restrict__ tiles, int64_t nslices, const BigC *__restrict__ bcs,
                            const int32_t *__restrict__ vperm, const int32_t *__restrict__ psize,
                            int32_t *__restrict__ len8) {
  const int lane = threadIdx.x & 31;
  const int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (sl >= nslices) return;
  const Tile T = tiles[sl];
  const BigC b = bcs[T.bc];
  const int vi = T.j * 32 + lane;
  const int32_t v = vi < b.s ? vperm[b.vp_off + vi] : -1;
  int c = v >= 0 ? psize[v] : 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) c = max(c, __shfl_xor_sync(0xffffffffu, c, o));
  if (lane == 0) len8[sl] = pk_rows(c);
}

constexpr int RL_T = 256;
constexpr int RL_MAXS = 2048;  // members per unit handled by the relabel kernel

// One CTA per unit (persistent).  Shared memory (nw = ceil(m/32) words each): seen, seen2 (item
// bitmaps; all zero between units), wslot (word -> index in the touched list), touched (words
// with any item of the unit), tbase (local-id base per touched word); slen[RL_MAXS].  Work is
// O(items of the unit + touched words): local ids are numbered per touched word in the order
// words were first touched (any injective numbering gives the same intersections).
__global__ void __launch_bounds__(RL_T) k_relabel(BigC *__restrict__ bcs, int64_t nunits,
                                                 const int32_t *__restrict__ vperm, const int32_t *__restrict__ offs,
                                                 const int32_t *__restrict__ items, int32_t nw,
                                                 const int32_t *__restrict__ blk_off8, int32_t *__restrict__ blk_len8,
                                                 PackT *__restrict__ packedT, int *__restrict__ counter,
                                                 int *__restrict__ max_kc) {
  extern __shared__ __align__(16) uint32_t rsm[];
  uint32_t *seen = rsm, *seen2 = rsm + nw, *wslot = rsm + 2 * nw, *touched = rsm + 3 * nw, *tbase = rsm + 4 * nw;
  int32_t *slen = reinterpret_cast<int32_t *>(rsm + 5 * nw + 1);
  __shared__ int s_unit, s_nt;
  __shared__ uint32_t s_part[RL_T / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NWARP = RL_T / 32;
  for (int i = tid; i < 2 * nw; i += RL_T) rsm[i] = 0;
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      s_unit = atomicAdd(counter, 1);
      s_nt = 0;
    }
    __syncthreads();
    const int64_t unit = s_unit;
    if (unit >= nunits) break;
    const BigC b = bcs[unit];
    const int npos = ((b.s + 31) / 32) * 32;  // member positions incl. the last slice's tail
    const int32_t *vp = vperm + b.vp_off;
    // 1. in-unit degree (saturating at 2) of every item: seen / seen2 bitmaps; touched words
    for (int i = warp; i < b.s; i += NWARP) {
      const int32_t v = vp[i];
      if (v < 0) continue;
      for (int32_t p = offs[v] + lane; p < offs[v + 1]; p += 32) {
        const int32_t x = items[p];
        const uint32_t bit = 1u << (x & 31);
        const uint32_t old = atomicOr(&seen[x >> 5], bit);
        if (old == 0u) touched[atomicAdd(&s_nt, 1)] = (uint32_t)(x >> 5);
        if (old & bit) atomicOr(&seen2[x >> 5], bit);
      }
    }
    __syncthreads();
    const int nt = s_nt;
    // 2. tbase[i] = degree->=2 items in touched words before i (block-wide exclusive scan)
    {
      const int per = (nt + RL_T - 1) / RL_T;
      const int i0 = min(tid * per, nt), i1 = min(i0 + per, nt);
      uint32_t sum = 0;
      for (int i = i0; i < i1; ++i) sum += __popc(seen2[touched[i]]);
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_part[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        uint32_t x = lane < NWARP ? s_part[lane] : 0u, xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
          if (lane >= o) xi += y;
        }
        if (lane < NWARP) s_part[lane] = xi - x;
      }
      __syncthreads();
      uint32_t run = s_part[warp] + incl - sum;
      for (int i = i0; i < i1; ++i) {
        const uint32_t w = touched[i];
        tbase[i] = run;
        wslot[w] = (uint32_t)i;
        run += __popc(seen2[w]);
      }
      if (i1 == nt && i0 < i1) tbase[nt] = run;
      if (nt == 0 && tid == 0) tbase[0] = 0;
    }
    __syncthreads();
    const uint32_t kc = tbase[nt];
    // 3. compacted lists in local ids, written into the packed layout of each slice
    for (int i = warp; i < npos; i += NWARP) {
      const int32_t v = i < b.s ? vp[i] : -1;
      int cnt = 0;
      if (v >= 0) {
        PackT *dst = pk_row_ptr(packedT, blk_off8[b.sl_off + (i >> 5)], i & 31);
        for (int32_t p0 = offs[v]; p0 < offs[v + 1]; p0 += 32) {
          const int32_t p = p0 + lane;
          bool keep = false;
          uint32_t lid = 0;
          if (p < offs[v + 1]) {
            const int32_t x = items[p];
            const uint32_t w2 = seen2[x >> 5], bit = 1u << (x & 31);
            keep = (w2 & bit) != 0;
            if (keep) lid = tbase[wslot[x >> 5]] + __popc(w2 & (bit - 1));
          }
          const unsigned bal = __ballot_sync(0xffffffffu, keep);
          const int pos = cnt + __popc(bal & ((1u << lane) - 1));
          if (keep) dst[pk_idx(pos)] = pk_enc(lid);
          cnt += __popc(bal);
        }
      }
      if (lane == 0) slen[i] = cnt;
    }
    __syncthreads();
    // 4. per slice: actual length (in 8s), pads = kc up to it; clear the touched words
    for (int i = tid; i < npos; i += RL_T) {
      int mx = slen[i];
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const int len8 = pk_rows(mx);
      const int sl = b.sl_off + (i >> 5);
      if ((i & 31) == 0) blk_len8[sl] = len8;
      PackT *dst = pk_row_ptr(packedT, blk_off8[sl], i & 31);
      for (int pos = slen[i]; pos < len8 * IPR; ++pos) dst[pk_idx(pos)] = pk_enc(kc);
    }
    for (int i = tid; i < nt; i += RL_T) {
      const uint32_t w = touched[i];
      seen[w] = 0;
      seen2[w] = 0;
    }
    if (tid == 0) {
      bcs[unit].kc = (int32_t)kc;
      atomicMax(max_kc, (int)kc);
    }
  }
}

// ------------------------------------------------------------------ K7 tile kernel
__device__ __forceinline__ void csa(uint32_t &h, uint32_t &l, uint32_t a, uint32_t b, uint32_t c) {
  uint32_t u = a ^ b;
  h = (a & b) | (u & c);
  l = u ^ c;
}

// in-register 32x32 bit transpose: A[p] bit r -> A[r] bit p
__device__ __forceinline__ void transpose32_body(uint32_t (&A)[32]) {
#pragma unroll
  for (int j = 16, mi = 0; j != 0; j >>= 1, ++mi) {
    const uint32_t m = mi == 0 ? 0x0000FFFFu : mi == 1 ? 0x00FF00FFu : mi == 2 ? 0x0F0F0F0Fu : mi == 3 ? 0x33333333u
                                                                                                  : 0x55555555u;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      if ((q & j) == 0) {
        uint32_t tt = ((A[q] >> j) ^ A[q + j]) & m;
        A[q + j] ^= tt;
        A[q] ^= tt << j;
      }
    }
  }
}

#ifndef C2_TRANSPOSE_NI
#define C2_TRANSPOSE_NI 1  // one out-of-line transpose body instead of VPT inlined copies (i-cache)
#endif
struct U32x32 {
  uint32_t v[32];
};
__device__ __noinline__ U32x32 transpose32_ni(U32x32 a) {
  transpose32_body(a.v);
  return a;
}
__device__ __forceinline__ void transpose32(uint32_t (&A)[32]) {
#if C2_TRANSPOSE_NI
  U32x32 t;
#pragma unroll
  for (int i = 0; i < 32; ++i) t.v[i] = A[i];
  t = transpose32_ni(t);
#pragma unroll
  for (int i = 0; i < 32; ++i) A[i] = t.v[i];
#else
  transpose32_body(A);
#endif
}

struct TileArgs {
  const Tile *tiles;
  int64_t lo, hi;
  int *counter;
  const BigC *bcs;
  const int32_t *vperm;
  const int32_t *vsize;
  const int32_t *rec;   // k_tile_rec records [nslices][REC_W]
  const int32_t *blk_len8;
  const int32_t *blk_off8;
  const uint4 *packed;
  const int32_t *psize;
  int32_t n;
  int32_t W, nwin;
  int k;
  const c2_cand *seed;  // fused: running lists before this function [n][k]; else nullptr
  unsigned long long *kstats;  // C2_OPT_KSTATS counters or nullptr
  int32_t stg_off, stg_cap;  // two staging buffers (word offset, capacity of each in 16-byte groups; 0: off)
  int32_t scr_off;      // split-probe scratch (word offset; 0: M's own words)
  int relabel;          // 1: items are unit-local ids, the tile's window is [0, B.kc) (nwin == 1)
  c2_cand *surv;        // fused light-row path: survivors [n][qmax] (nullptr: no light rows)
  int32_t *qn;          // survivors per user (read and zeroed by k_surv_merge)
  int32_t qmax;
  // rows handed to k_row_topk: count rows (u16) and records, bump-allocated
  uint16_t *hv_cnt;
  int64_t hv_cap;
  unsigned long long *hv_used;
  RowRec *hv_recs;
  int64_t hv_rcap;
  unsigned long long *hv_nrec;
  int *err;             // set to 1 if a buffer above was too small (the host sizes them exactly)
};

// 8 masks of one uint4 of packed u16 item ids
__device__ __forceinline__ void masks8(const uint32_t *__restrict__ M, uint4 d, uint32_t (&m)[8]) {
#ifdef C2_TIMING_NOCONFLICT  // timing experiment only (wrong counts): every lane reads its own bank
  const uint32_t ln = threadIdx.x & 31u;
  m[0] = M[((d.x & 0xFFFFu) & ~31u) | ln];
  m[1] = M[((d.x >> 16) & ~31u) | ln];
  m[2] = M[((d.y & 0xFFFFu) & ~31u) | ln];
  m[3] = M[((d.y >> 16) & ~31u) | ln];
  m[4] = M[((d.z & 0xFFFFu) & ~31u) | ln];
  m[5] = M[((d.z >> 16) & ~31u) | ln];
  m[6] = M[((d.w & 0xFFFFu) & ~31u) | ln];
  m[7] = M[((d.w >> 16) & ~31u) | ln];
  return;
#endif
  m[0] = M[d.x & 0xFFFFu];
  m[1] = M[d.x >> 16];
  m[2] = M[d.y & 0xFFFFu];
  m[3] = M[d.y >> 16];
  m[4] = M[d.z & 0xFFFFu];
  m[5] = M[d.z >> 16];
  m[6] = M[d.w & 0xFFFFu];
  m[7] = M[d.w >> 16];
}

// 4 masks of one uint4 of byte offsets into M (C2_PACK32)
__device__ __forceinline__ void masks4b(const uint32_t *__restrict__ M, uint4 d, uint32_t *m) {
  const char *Mb = reinterpret_cast<const char *>(M);
  m[0] = *reinterpret_cast<const uint32_t *>(Mb + d.x);
  m[1] = *reinterpret_cast<const uint32_t *>(Mb + d.y);
  m[2] = *reinterpret_cast<const uint32_t *>(Mb + d.z);
  m[3] = *reinterpret_cast<const uint32_t *>(Mb + d.w);
}

template <int NHI>
struct Counter {
  uint32_t ones, twos, fours, eights;
  uint32_t H[NHI];  // counts of sixteens, bit-sliced
  __device__ __forceinline__ void zero() {
    ones = twos = fours = eights = 0;
#pragma unroll
    for (int i = 0; i < NHI; ++i) H[i] = 0;
  }
  // add 8 masks; returns the carry of weight 8 (combined in pairs by add16)
  __device__ __forceinline__ uint32_t add8(const uint32_t (&m)[8]) {
    uint32_t tA, tB, fA, fB, e8;
    csa(tA, ones, ones, m[0], m[1]);
    csa(tB, ones, ones, m[2], m[3]);
    csa(fA, twos, twos, tA, tB);
    csa(tA, ones, ones, m[4], m[5]);
    csa(tB, ones, ones, m[6], m[7]);
    csa(fB, twos, twos, tA, tB);
    csa(e8, fours, fours, fA, fB);
    return e8;
  }
  // add16 for tiles whose counts stay below 2^(4 + LO) unless hi (CTA-uniform): the carry out of
  // plane H[LO - 1] is then always zero and the upper planes need no update
  template <int LO>
  __device__ __forceinline__ void add16h(uint32_t e8a, uint32_t e8b, bool hi) {
    uint32_t carry;
    csa(carry, eights, eights, e8a, e8b);
#pragma unroll
    for (int i = 0; i < (LO < NHI ? LO : NHI); ++i) {
      uint32_t tt = H[i] & carry;
      H[i] ^= carry;
      carry = tt;
    }
    if (hi) {
#pragma unroll
      for (int i = LO; i < NHI; ++i) {
        uint32_t tt = H[i] & carry;
        H[i] ^= carry;
        carry = tt;
      }
    }
  }
  __device__ __forceinline__ void add16(uint32_t e8a, uint32_t e8b) {
    uint32_t carry;
    csa(carry, eights, eights, e8a, e8b);
#pragma unroll
    for (int i = 0; i < NHI; ++i) {
      uint32_t tt = H[i] & carry;
      H[i] ^= carry;
      carry = tt;
    }
  }
};

template <int NHI, int VPT>
__global__ void __launch_bounds__(TILE_T, C2_TILE_MINB) k_local_tile(TileArgs a) {
  extern __shared__ __align__(16) uint32_t dyn[];
  uint32_t *M = dyn;  // W + 1 words, M[W] == 0 (all zero between tiles)
  // tile descriptors, double-buffered: the next tile's are fetched during this tile
  __shared__ int64_t s_it[2];
  __shared__ Tile s_T[2];
  __shared__ BigC s_B[2];
  __shared__ int32_t s_ru2[2][32];
  __shared__ uint32_t s_rp2[2][32];
  __shared__ int32_t s_bl[2][MAX_WIN], s_bo[2][MAX_WIN], s_so[2][MAX_WIN];  // rows' blocks; staged offsets
  __shared__ int s_stg[2];  // 1: the rows' blocks of every window are staged in stg
  __shared__ __align__(16) int32_t s_rec[2][REC_W];  // fetched tile records
  __shared__ uint4 s_ref[32];       // light rows: the running k-th best as a Ref (see make_ref)
  __shared__ int s_qn[32];          // light rows: survivors found by the phase-A epilogue
  __shared__ unsigned s_light;      // light rows (running list full, k-th best with i >= 1)
  __shared__ unsigned s_mxst, s_sumst;  // kstats: probe steps of the tile's busiest warp / of all warps
  __shared__ unsigned s_over;       // light rows with more than qmax survivors (handed to k_row_topk)
  __shared__ int64_t s_cbase, s_rbase;  // this tile's first count entry / record for k_row_topk
  __shared__ int s_pre;                 // 1: s_cbase / s_rbase were allocated early (no barrier needed)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < a.W + 1; i += TILE_T) M[i] = 0;
  uint4 *stg0 = reinterpret_cast<uint4 *>(dyn + a.stg_off);  // staged rows' blocks, one buffer per slot
  const int nwin = a.nwin;
  const int kk = a.k;
  // next-tile descriptors in two halves (TMA bulk copies completing on mbarriers): fetch_issue
  // (one thread, at tile start: claim the next tile, bulk-copy its record), fetch_finish (one warp,
  // once this tile's staged blocks are dead: wait for the record, parse it, bulk-copy the rows'
  // packed blocks into the staging buffer).  Every use of a slot's mbarriers gets exactly one
  // arrival (0 bytes when there is no tile), so all threads can track the phases.
  __shared__ __align__(8) uint64_t mb_rec[2], mb_stg[2];
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&mb_rec[i], 1);
      mbar_init(&mb_stg[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t ph_rec = 0, ph_stg = 0;  // bit b: parity of the next completion of slot b
  auto fetch_issue = [&](int b) {    // one thread
    const int64_t it = a.lo + atomicAdd(a.counter, 1);
    s_it[b] = it;
    if (it < a.hi) {
      fence_proxy_async();
      mbar_arrive_tx(&mb_rec[b], REC_W * 4);
      bulk_g2s(s_rec[b], a.rec + it * REC_W, REC_W * 4, &mb_rec[b]);
    } else {
      mbar_arrive_tx(&mb_rec[b], 0);
    }
  };
  auto fetch_finish = [&](int b) {  // one warp
    mbar_wait(&mb_rec[b], (ph_rec >> b) & 1u);
    const int64_t it = s_it[b];
    if (it >= a.hi) {
      if (lane == 0) mbar_arrive_tx(&mb_stg[b], 0);
      return;
    }
    const int32_t *rc = s_rec[b];
    if (lane == 0) {
      s_T[b] = Tile{rc[0], rc[1]};
      s_B[b] = BigC{rc[2], rc[3], rc[4], rc[5], rc[6], rc[7]};
    }
    s_ru2[b][lane] = rc[64 + lane];
    s_rp2[b][lane] = (uint32_t)rc[96 + lane];
    const int32_t bl = lane < nwin ? rc[8 + lane] : 0;
    const int32_t bo = lane < nwin ? rc[24 + lane] : 0;
    int32_t incl = bl * 32;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    const bool staged = tot <= a.stg_cap;
    if (lane < nwin) {
      s_bl[b][lane] = bl;
      s_bo[b][lane] = bo;
      s_so[b][lane] = incl - bl * 32;
    }
    if (lane == 0) {
      s_stg[b] = staged ? 1 : 0;
      fence_proxy_async();
      mbar_arrive_tx(&mb_stg[b], staged ? (uint32_t)tot * 16u : 0u);
    }
    __syncwarp();
    if (staged && lane < nwin && bl > 0)
      bulk_g2s(stg0 + b * a.stg_cap + (incl - bl * 32), a.packed + (int64_t)bo * 32, (uint32_t)bl * 512u, &mb_stg[b]);
  };
  if (tid == 0) fetch_issue(0);
  if (warp == 0) fetch_finish(0);
  // light rows (c2_build; the row's running list full and its k-th best tau has i >= 1): a
  // candidate can only enter the list if it is strictly better than tau.  Right after phase A,
  // while the bit-sliced counts are still in the threads that made them, every light row's
  // candidates are screened against a per-slice bound with a bit-sliced compare (all 32 rows at
  // once, ~2 LOP3 per count bit), the few that pass get the exact test, and the survivors go to
  // global memory for k_surv_merge.  The other rows' counts go to k_row_topk.
  const bool light_on = C2_LIGHT && a.surv != nullptr;
  int cur = 0;
  // light rows' survivor counts of the tile in slot pb (read and reset by k_surv_merge), written
  // by warp 0 after the NEXT tile's top-of-loop barrier: the light epilogue then needs no barrier
  // of its own when no row can overflow its survivor slots
  bool prev_lt = false;
  // count rows of the tile's k8 rows: bump-allocated in the per-function buffers (one thread)
  auto alloc_rows = [&](unsigned k8, int s4v) {
    const int n8 = __popc(k8);
    if (n8 == 0) return;
    const unsigned long long cb = atomicAdd(a.hv_used, (unsigned long long)n8 * s4v);
    const unsigned long long rb = atomicAdd(a.hv_nrec, (unsigned long long)n8);
    const bool fits = cb + (unsigned long long)n8 * s4v <= (unsigned long long)a.hv_cap &&
                      rb + (unsigned long long)n8 <= (unsigned long long)a.hv_rcap;
    if (!fits) atomicExch(a.err, 1);
    s_cbase = fits ? (int64_t)cb : -1;
    s_rbase = (int64_t)rb;
  };
  auto flush_light = [&](int pb) {
    const unsigned lok = s_light & ~s_over;
    const BigC Bp = s_B[pb];
    const int32_t ru = s_ru2[pb][lane];
    if (((lok >> lane) & 1u) && s_qn[lane] > 0) a.qn[ru] = s_qn[lane];
    if (a.kstats && lane == 0) {
      atomicAdd(&a.kstats[71], (unsigned long long)__popc(lok));
      atomicAdd(&a.kstats[73], (unsigned long long)__popc(s_over));
    }
    if (a.kstats && ((lok >> lane) & 1u)) {
      atomicAdd(&a.kstats[72], (unsigned long long)s_qn[lane]);
      int ev = Bp.s - 1;  // pair evaluations of this row: its cluster-mates (debug work accounting)
      if (Bp.slot) {
        const int32_t *vpp = a.vperm + Bp.vp_off;
        const int lo = lane & ~(Bp.slot - 1);
        ev = -1;
        for (int j = 0; j < Bp.slot; ++j) ev += vpp[lo + j] >= 0 ? 1 : 0;
      }
      atomicAdd(&a.kstats[70], (unsigned long long)ev);
    }
  };
  for (;;) {
    mbar_wait(&mb_stg[cur], (ph_stg >> cur) & 1u);  // this tile's staged row blocks
    ph_rec ^= 1u << cur;  // (slot cur's record and staging phases were consumed)
    ph_stg ^= 1u << cur;
    __syncthreads();
    if (prev_lt && warp == 0) flush_light(cur ^ 1);
    const int64_t it = s_it[cur];
    if (it >= a.hi) break;
    uint4 *stg = stg0 + cur * a.stg_cap;
    if (tid == 0) fetch_issue(cur ^ 1);  // next tile's record: claimed and requested now
    const long long ck0 = a.kstats ? clock64() : 0;
    long long ckA = 0, ckE = 0;
    const Tile T = s_T[cur];
    const BigC B = s_B[cur];
    const int32_t *s_ru = s_ru2[cur];
    const uint32_t *s_rp = s_rp2[cur];
    const int s = B.s;
    const int s4 = (s + 3) & ~3;
    const int nsl = (s + 31) >> 5;
    const int r0 = T.j * 32;
    const int nr = min(32, s - r0);
    const int32_t *vp = a.vperm + B.vp_off;
    const uint32_t W = a.relabel ? (uint32_t)B.kc : (uint32_t)a.W;
    if (tid < 32) s_qn[tid] = 0;
    if (tid == 0) {
      s_light = 0u;
      s_over = 0u;
      s_mxst = 0u;
      s_sumst = 0u;
    }
    const unsigned valid = __ballot_sync(0xffffffffu, lane < nr && s_ru[lane] >= 0);
#if C2_HIPLANES
    // every count of the tile is <= its longest row: short rows never carry into the upper planes
    const bool hi_planes = __reduce_max_sync(0xffffffffu, s_rp[lane]) >= (16u << C2_HIPLANES);
#endif
    unsigned k8rows = valid;  // rows handed to k_row_topk
    const bool lt = light_on && nsl <= VPT * TILE_WARPS;  // (one g0 group: counters of all members live)
    // rows handed to k_row_topk known now (no light rows), or after the light rows are known when no
    // row can overflow its survivor slots: their count rows are allocated early, the atomics'
    // latency hidden behind the probe (published by the first window's barriers)
    if (tid == 0) {
      s_pre = 0;
      if (!lt) {
        alloc_rows(valid, s4);
        s_pre = 1;
      }
    }
    // light rows: the running k-th best tau of every row (one global read per row) is requested now
    // by the last warp and turned into its Ref after the first mask build, so the epilogue can start
    // without a barrier after the last window's mask clear
    c2_cand tl_pre = c2_cand{-1, 0, 0};
    if (lt && warp == TILE_WARPS - 1 && ((valid >> lane) & 1u)) tl_pre = a.seed[(int64_t)s_ru[lane] * kk + kk - 1];
    // small tiles (<= TILE_WARPS/2 slices): G warps share a slice, each probing a contiguous part
    // of its member lists; the partial bit-sliced counters are then added (bit-sliced ripple
    // carry), so no warp idles through the probe of a tile with few slices
    // bigger tiles whose whole slices leave the last counter slot free: the profile lengths are
    // heavy-tailed, so the longest slice alone outlasts the mean warp (c5, kstats: busiest warp
    // 31 steps vs 11 mean in clusters of 257-1024); its lists are split over G warps the same way
    int G = 1;   // warps per split slice
    int Hs = 0;  // slices [0, Hs) are split; their (partial) counters live in slot QS
    constexpr int QS = VPT - 1;
    if (C2_HSPLIT && VPT >= 2 && nsl > TILE_WARPS / 2 && nsl - C2_HSPLIT <= TILE_WARPS * (VPT - 1)) {
      Hs = C2_HSPLIT;
      G = TILE_WARPS / C2_HSPLIT;
    }
    if (C2_SPLIT && nsl <= TILE_WARPS / 2) {
      // parts of >= ~4 steps (pairs of 8-item groups; the rows' own lengths stand for the slices')
      int np = 0;
      for (int w = 0; w < nwin; ++w) np += (s_bl[cur][w] + 1) >> 1;
      G = TILE_WARPS;
      while (G > 1 && (G * nsl > TILE_WARPS || 4 * G > np)) G >>= 1;
      if (G > 1) Hs = nsl;
    }
    const int part = warp % G;
    // ================= phase A: counts |P_r ∩ P_v| for the 32 rows x all v of the cluster
    for (int g0 = 0; g0 < nsl; g0 += VPT * TILE_WARPS) {
      // the slice of this warp's q-th counter (nsl: none); after the probe (all = false) a split
      // slice belongs to its part-0 warp only, which holds the added counters
      auto slice_of = [&](int q, bool all = false) -> int {
        if (Hs > 0 && q == QS) return (warp / G < Hs && (all || part == 0)) ? warp / G : nsl;
        const int jj = Hs + g0 + q * TILE_WARPS + ((C2_SNAKE && (q & 1)) ? TILE_WARPS - 1 - warp : warp);
        return jj < nsl ? jj : nsl;
      };
      Counter<NHI> C[VPT];
#pragma unroll
      for (int q = 0; q < VPT; ++q) C[q].zero();
#if C2_KSTATS_STEPS
      unsigned tsteps = 0u;
#endif
      for (int w = 0; w < nwin; ++w) {
        // ---- build M for window w from the tile's own slice (rows), lane r -> bit r (the first
        //      16-byte group of every thread is kept for the clear below)
        const bool stgd = s_stg[cur] != 0;
        const int32_t n4r = s_bl[cur][w] * 32;
        const uint4 *srcr = stgd ? stg + s_so[cur][w] : a.packed + (int64_t)s_bo[cur][w] * 32;
        const uint32_t pw = C2_PACK32 ? (uint32_t)pk_enc(W) : (W | (W << 16));
        const uint4 padv = make_uint4(pw, pw, pw, pw);
        const uint4 dkeep = tid < n4r ? srcr[tid] : padv;
        for (int gi = tid; gi < n4r; gi += TILE_T) {
          const uint4 d = gi == tid ? dkeep : srcr[gi];
          const uint32_t bit = 1u << (gi & 31);
#if C2_PACK32
          const uint32_t xs[4] = {d.x, d.y, d.z, d.w};  // byte offsets into M
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (xs[q] < 4u * W) atomicOr(reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(M) + xs[q]), bit);
#else
          const uint32_t xs[8] = {d.x & 0xFFFFu, d.x >> 16, d.y & 0xFFFFu, d.y >> 16,
                                  d.z & 0xFFFFu, d.z >> 16, d.w & 0xFFFFu, d.w >> 16};
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (xs[q] < W) atomicOr(&M[xs[q]], bit);
#endif
        }
        __syncthreads();
        // the next tile's row blocks go to the other staging buffer as soon as its record is in
        if (g0 == 0 && w == 0 && warp == TILE_WARPS - 1) {
          if (lt) {
            const bool light = tl_pre.id >= 0 && tl_pre.inter >= 1;
            if (light) {
              const Ref R = make_ref(from_out(tl_pre), s_rp[lane], false);
              s_ref[lane] = make_uint4(R.A, R.B, R.iT, R.idlim);
            }
            const unsigned lm = __ballot_sync(0xffffffffu, light);
            if (lane == 0) {
              s_light = lm;
              if (s - 1 <= a.qmax) {
                alloc_rows(valid & ~lm, s4);
                s_pre = 1;
              }
            }
          }
          fetch_finish(cur ^ 1);
        }
        // ---- probe: each warp streams VPT slices of v lists, two 16-byte loads per step with
        //      the next two steps in flight (odd tails padded with the sentinel item W, M[W] = 0)
        const long long ckpb = a.kstats ? clock64() : 0;
        int nsteps = 0;
#pragma unroll
        for (int q = 0; q < VPT; ++q) {
          const int jj = slice_of(q, true);
          if (jj < nsl) {
            const int64_t bi = (int64_t)(B.sl_off + jj) * nwin + w;
            const bool own = stgd && jj == T.j;  // the tile's own slice: staged
            const int32_t len8 = own ? s_bl[cur][w] : a.blk_len8[bi];
            const uint4 *src = (own ? stg + s_so[cur][w] : a.packed + (int64_t)a.blk_off8[bi] * 32) + lane;
            auto ld = [&](int32_t p) { return p < len8 ? src[(int64_t)p * 32] : padv; };
#if C2_PACK32
            // rows of 4 byte offsets per lane; 16 items (4 rows) per step, the next step in flight
            int32_t plo = 0, phi = len8;  // this warp's part of the lists (quads of rows)
            if (G > 1 && q == QS) {
              const int32_t np = (len8 + 3) >> 2;
              plo = 4 * ((part * np) / G);
              phi = 4 * (((part + 1) * np) / G);
            }
            // blocks are whole quads of rows with >= PK_SLACK_ROWS readable rows after them (global:
            // allocation slack; staged: shared-memory slack), so the step loads need no bounds test
            (void)ld;
            const uint4 *sp = src + (int64_t)plo * 32;
            auto step = [&](const uint4 &d0, const uint4 &d1, const uint4 &d2, const uint4 &d3) {
              uint32_t m[8];
              masks4b(M, d0, m);
              masks4b(M, d1, m + 4);
              uint32_t e8a = C[q].add8(m);
              masks4b(M, d2, m);
              masks4b(M, d3, m + 4);
              uint32_t e8b = C[q].add8(m);
              C[q].add16(e8a, e8b);
            };
            uint4 a0 = sp[0], a1 = sp[32], a2 = sp[64], a3 = sp[96];
            int32_t p4 = plo;
            for (; p4 + 4 < phi; p4 += 8) {  // two steps per iteration (ping-pong, no register moves)
              const uint4 b0 = sp[128], b1 = sp[160], b2 = sp[192], b3 = sp[224];
              step(a0, a1, a2, a3);
              a0 = sp[256];
              a1 = sp[288];
              a2 = sp[320];
              a3 = sp[352];
              step(b0, b1, b2, b3);
              sp += 256;
              nsteps += 2;
            }
            if (p4 < phi) {
              step(a0, a1, a2, a3);
              ++nsteps;
            }
#else
            int32_t plo = 0, phi = len8;  // this warp's part of the lists (pairs of 8-item groups)
            if (G > 1 && q == QS) {
              const int32_t np = (len8 + 1) >> 1;
              plo = 2 * ((part * np) / G);
              phi = 2 * (((part + 1) * np) / G);
            }
            uint4 d0 = ld(plo), d1 = ld(plo + 1), n0 = ld(plo + 2), n1 = ld(plo + 3);
            for (int32_t p8 = plo; p8 < phi; p8 += 2) {
              const uint4 f0 = ld(p8 + 4), f1 = ld(p8 + 5);
              uint32_t m[8];
              masks8(M, d0, m);
              uint32_t e8a = C[q].add8(m);
              masks8(M, d1, m);
              uint32_t e8b = C[q].add8(m);
#if C2_HIPLANES
              C[q].template add16h<C2_HIPLANES>(e8a, e8b, hi_planes);
#else
              C[q].add16(e8a, e8b);
#endif
              d0 = n0;
              d1 = n1;
              n0 = f0;
              n1 = f1;
              ++nsteps;
            }
#endif
          }
        }
#if C2_KSTATS_STEPS
        tsteps += (unsigned)nsteps;
        if (a.kstats && lane == 0 && w + 1 == nwin) {
          atomicMax(&s_mxst, tsteps);
          atomicAdd(&s_sumst, tsteps);
        }
#endif
        if (a.kstats && lane == 0 && s > 1024) {  // probe busy time per step (big tiles)
          atomicAdd(&a.kstats[64], (unsigned long long)(clock64() - ckpb));
          atomicAdd(&a.kstats[65], (unsigned long long)nsteps);
        }
        __syncthreads();
        // ---- clear M
        for (int gi = tid; gi < n4r; gi += TILE_T) {
          const uint4 d = gi == tid ? dkeep : srcr[gi];
#if C2_PACK32
          const uint32_t xs[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (xs[q] < 4u * W) *reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(M) + xs[q]) = 0;
#else
          const uint32_t xs[8] = {d.x & 0xFFFFu, d.x >> 16, d.y & 0xFFFFu, d.y >> 16,
                                  d.z & 0xFFFFu, d.z >> 16, d.w & 0xFFFFu, d.w >> 16};
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (xs[q] < W) M[xs[q]] = 0;
#endif
        }
        // (after the last window's clear no barrier is needed unless the split-probe partial
        // counters use M's words as scratch (G > 1): the next mask build follows the next tile's
        // top-of-loop barrier, and s_ref / s_light were published by the probe's barrier)
        if (w + 1 < nwin || G > 1) __syncthreads();
      }
      if (G > 1) {
        // add the G partial counters of each slice into its part-0 warp (scratch: [warp][plane][lane]
        // in M's words when M is big enough -- re-zeroed by the reader -- else a region of its own)
        constexpr int NPL = 4 + NHI;
        uint32_t *scr = a.scr_off ? dyn + a.scr_off : M;
        if (part != 0 && warp / G < Hs) {
          uint32_t *o = scr + warp * NPL * 32 + lane;
          o[0] = C[QS].ones;
          o[32] = C[QS].twos;
          o[64] = C[QS].fours;
          o[96] = C[QS].eights;
#pragma unroll
          for (int i = 0; i < NHI; ++i) o[(4 + i) * 32] = C[QS].H[i];
        }
        __syncthreads();
        if (part == 0 && warp / G < Hs) {
          for (int pw = 1; pw < G; ++pw) {
            uint32_t *o = scr + (warp + pw) * NPL * 32 + lane;
            uint32_t b[NPL];
#pragma unroll
            for (int j = 0; j < NPL; ++j) {
              b[j] = o[j * 32];
              if (!a.scr_off) o[j * 32] = 0u;
            }
            uint32_t *pa[NPL];
            pa[0] = &C[QS].ones;
            pa[1] = &C[QS].twos;
            pa[2] = &C[QS].fours;
            pa[3] = &C[QS].eights;
#pragma unroll
            for (int i = 0; i < NHI; ++i) pa[4 + i] = &C[QS].H[i];
            uint32_t cy = 0u;
#pragma unroll
            for (int j = 0; j < NPL; ++j) {
              const uint32_t x = *pa[j], y = b[j];
              *pa[j] = x ^ y ^ cy;
              cy = (x & y) | (cy & (x ^ y));
            }
          }
        }
      }
      if (a.kstats) ckA = clock64();
      // ---- light rows: bit-sliced prefilter on the counters (count >= imin_r for all 32 rows at
      //      once), the exact test for the few that pass, survivors to global memory (one g0 group)
      if (lt) {
        const unsigned lm = s_light;
        if (lm) {
          constexpr int NPL = 4 + NHI;
          // per row (lane r): the light row's reference tau = (iT, UT) and |P_r|
          const uint4 Rr = s_ref[lane];  // A = UT + iT, B = iT |P_r|, iT
          const bool lr = (lm >> lane) & 1u;
          int32_t idq[VPT];
          uint32_t psq[VPT];  // the members' ids and sizes, all requested at once
#pragma unroll
          for (int q = 0; q < VPT; ++q) {
            const int vi = slice_of(q) * 32 + lane;
            idq[q] = vi < s ? __ldg(vp + vi) : -1;
            psq[q] = vi < s ? (uint32_t)__ldg(a.vsize + B.vp_off + vi) : 0u;
          }
          // pass 1 (all slices of the warp, independent chains): the prefilter hit masks
          uint32_t hitq[VPT];
#pragma unroll
          for (int q = 0; q < VPT; ++q) {
            hitq[q] = 0u;
            const int jj = slice_of(q);
            if (jj >= nsl) continue;  // (warp-uniform: all lanes of a warp share the slice jj)
            const uint32_t psv = idq[q] >= 0 ? psq[q] : 0xFFFFFFFFu;
            // slice bound: every member has |P_v| >= psmin, so a member passes row r only if
            // i (UT + iT) >= iT (|P_r| + psmin), i.e. i >= imin_r; the bit-planes of the 32 imin_r
            const uint32_t psmin = __reduce_min_sync(0xffffffffu, psv);
            uint32_t imin = 0xFFFFFFFFu;
            if (lr && psmin != 0xFFFFFFFFu) imin = (Rr.y + Rr.z * psmin + Rr.x - 1u) / Rr.x;
            const unsigned pm = __ballot_sync(0xffffffffu, imin < (1u << NPL));
            uint32_t gt = 0u, eq = 0xFFFFFFFFu;
#pragma unroll
            for (int j = NPL - 1; j >= 0; --j) {
              const uint32_t plj = j == 0 ? C[q].ones : j == 1 ? C[q].twos : j == 2 ? C[q].fours
                                                         : j == 3 ? C[q].eights : C[q].H[j > 3 ? j - 4 : 0];
              const uint32_t im = __ballot_sync(0xffffffffu, (imin >> j) & 1u);
              gt |= eq & plj & ~im;
              eq &= ~(plj ^ im);
            }
            uint32_t hit = (gt | eq) & pm;
            if (B.slot) {
              const int lo = lane & ~(B.slot - 1);
              hit &= (B.slot >= 32 ? 0xFFFFFFFFu : ((1u << B.slot) - 1u)) << lo;
            }
            if (jj == T.j) hit &= ~(1u << lane);  // the row itself
            if (idq[q] < 0) hit = 0u;
            hitq[q] = hit;
            if (a.kstats) {
              const int nh = __reduce_add_sync(0xffffffffu, __popc(hit));
              if (lane == 0) atomicAdd(&a.kstats[74], (unsigned long long)nh);
            }
          }
          // pass 2: the exact test for every hit, survivors to global memory
#pragma unroll
          for (int q = 0; q < VPT; ++q) {
            uint32_t hit = hitq[q];
            const int32_t idv = idq[q];
            const uint32_t psv = psq[q];
            while (hit) {
              const int r = __ffs(hit) - 1;
              hit &= hit - 1u;
              uint32_t i = ((C[q].ones >> r) & 1u) | (((C[q].twos >> r) & 1u) << 1) | (((C[q].fours >> r) & 1u) << 2) |
                           (((C[q].eights >> r) & 1u) << 3);
#pragma unroll
              for (int j = 0; j < NHI; ++j) i |= ((C[q].H[j] >> r) & 1u) << (4 + j);
              const uint4 R4 = s_ref[r];
              if (passes(i, psv, idv, Ref{R4.x, R4.y, R4.z, R4.w})) {
                const int pq = atomicAdd(&s_qn[r], 1);
                if (pq < a.qmax)
                  a.surv[(int64_t)s_ru[r] * a.qmax + pq] = c2_cand{idv, (uint16_t)i, (uint16_t)(s_rp[r] + psv - i)};
                else if (pq == a.qmax)
                  atomicOr(&s_over, 1u << r);
              }
            }
          }
        }
        if (C2_EPI_BAR || s - 1 > a.qmax) {  // a row may overflow its survivor slots: s_over must be complete
          __syncthreads();
          k8rows = valid & ~(s_light & ~s_over);
        } else {
          k8rows = valid & ~s_light;
        }
      }
      if (a.kstats) ckE = clock64();
      // ---- the other rows: planes -> 32 counts per member (transpose) -> their count rows, and
      //      one RowRec per row, for k_row_topk
      if (k8rows) {
        if (g0 == 0) {
          if (!s_pre) {
            if (tid == 0) alloc_rows(k8rows, s4);
            __syncthreads();
          }
          if (warp == 0 && ((k8rows >> lane) & 1u) && s_cbase >= 0) {
            const int rk = __popc(k8rows & ((1u << lane) - 1u));
            const int slot = B.slot;
            a.hv_recs[s_rbase + rk] = RowRec{s_ru[lane], (int32_t)s_rp[lane], s, B.vp_off, slot ? lane : r0 + lane,
                                             slot ? (lane & ~(slot - 1)) : 0, slot, B.f, s_cbase + (int64_t)rk * s4};
          }
        }
        const int64_t cb = s_cbase;
        const bool few = __popc(k8rows) <= 4;
        if (cb >= 0) {
#pragma unroll
          for (int q = 0; q < VPT; ++q) {
            const int jj = slice_of(q);
            const int vi = jj * 32 + lane;
            if (jj < nsl && few) {
              // a few rows: each row's count read off the bit-planes
              uint16_t *dst = a.hv_cnt + cb + vi;
              int rk = 0;
              for (unsigned rm = k8rows; rm; rm &= rm - 1u, ++rk) {
                const int r = __ffs(rm) - 1;
                uint32_t i = ((C[q].ones >> r) & 1u) | (((C[q].twos >> r) & 1u) << 1) | (((C[q].fours >> r) & 1u) << 2) |
                             (((C[q].eights >> r) & 1u) << 3);
#pragma unroll
                for (int j = 0; j < NHI; ++j) i |= ((C[q].H[j] >> r) & 1u) << (4 + j);
                if (vi < s) dst[(int64_t)rk * s4] = (uint16_t)i;
              }
            } else if (jj < nsl) {
              uint32_t A[32];
              A[0] = C[q].ones;
              A[1] = C[q].twos;
              A[2] = C[q].fours;
              A[3] = C[q].eights;
#pragma unroll
              for (int i = 0; i < NHI; ++i) A[4 + i] = C[q].H[i];
#pragma unroll
              for (int i = 4 + NHI; i < 32; ++i) A[i] = 0;
              transpose32(A);
              if (vi < s) {
                uint16_t *dst = a.hv_cnt + cb + vi;
                int rk = 0;
#pragma unroll
                for (int r = 0; r < 32; ++r)
                  if ((k8rows >> r) & 1u) dst[(int64_t)(rk++) * s4] = (uint16_t)A[r];
              }
            }
          }
        }
      }
    }
    prev_lt = lt;
    if (a.kstats && tid == 0) {  // tile cycles by cluster size class: mixed, 33-256, 257-1024, >1024
      const long long ck3 = clock64();
      const int cls = B.slot ? 0 : s <= 256 ? 1 : s <= 1024 ? 2 : 3;
      atomicAdd(&a.kstats[32 + cls], (unsigned long long)(ck3 - ck0));
      atomicAdd(&a.kstats[36 + cls], 1ull);
      unsigned long long *kc3 = a.kstats + 40 + 3 * cls;  // phase A / light epilogue / count rows
      atomicAdd(&kc3[0], (unsigned long long)(ckA - ck0));
      atomicAdd(&kc3[1], (unsigned long long)(ckE - ckA));
      atomicAdd(&kc3[2], (unsigned long long)(ck3 - ckE));
      if (lt) {  // (the light epilogue's barrier orders the warps' step counts before this read)
        atomicAdd(&a.kstats[52 + cls], (unsigned long long)s_mxst);
        atomicAdd(&a.kstats[56 + cls], (unsigned long long)s_sumst);
        atomicAdd(&a.kstats[60 + cls], 1ull);
      }
    }
    cur ^= 1;
  }
}

typedef void (*TileKernel)(TileArgs);

template <int NHI>
static TileKernel pick_vpt(int vpt) {
  return vpt <= 1 ? k_local_tile<NHI, 1> : vpt <= 2 ? k_local_tile<NHI, 2> : k_local_tile<NHI, 4>;
}
static TileKernel pick_tile(int nhi, int vpt) {
#if C2_NHI7
  if (nhi > 4 && nhi <= 7) return pick_vpt<7>(vpt);  // lists of <= 2047 items (c5: max 2000)
#endif
  return nhi <= 4 ? pick_vpt<4>(vpt) : nhi <= 8 ? pick_vpt<8>(vpt) : pick_vpt<11>(vpt);
}

// Per function: count entries (s * s4 per cluster: every member is a row) and rows the tiles of
// that function can hand to k_row_topk -- the exact sizes of its buffers.
__global__ void k_cnt_need(const BigC *__restrict__ bcs, int64_t ncl, unsigned long long *__restrict__ need, int t) {
  // per-block sums in shared memory (clusters are ordered by function, so a block touches few
  // functions), then one global atomic per non-zero entry
  __shared__ unsigned long long sn[2 * C2_MAX_T];
  for (int i = threadIdx.x; i < 2 * t; i += blockDim.x) sn[i] = 0ull;
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < ncl) {
    const BigC B = bcs[c];
    const unsigned long long s = (unsigned long long)B.s;
    atomicAdd(&sn[B.f], s * ((s + 3) & ~3ull));
    atomicAdd(&sn[t + B.f], s);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * t; i += blockDim.x)
    if (sn[i]) atomicAdd(&need[i], sn[i]);
}

__global__ void k_init_pads(c2_cand *__restrict__ R, int64_t E) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < E) R[e] = c2_cand{-1, 0, 0};
}

// sum over unordered pairs of (|P_u| + |P_v|) = sum over (f,u) of (s_c - 1) * |P_u|
__global__ void __launch_bounds__(256) k_work_steps(const int32_t *__restrict__ offsets, const int32_t *__restrict__ cof,
                                                    const int32_t *__restrict__ psize, int64_t TN, int32_t n,
                                                    unsigned long long *__restrict__ acc) {
  // sum over (f, u) of (s - 1) |P_u| = sum over unordered local pairs of |P_u| + |P_v|; grid-stride,
  // one atomic per block
  __shared__ unsigned long long sh[8];
  unsigned long long w = 0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < TN; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = q / n;
    const int32_t u = (int32_t)(q % n);
    const int32_t c = cof[q];
    const int32_t *off = offsets + f * (n + 1);
    w += (unsigned long long)(off[c + 1] - off[c] - 1) * (unsigned long long)psize[u];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < 8; ++i) w += sh[i];
    if (w) atomicAdd(acc, w);
  }
}

// ------------------------------------------------------------------ item-id compaction
// Step 2 streams window-local item ids; ids beyond MAX_WIN windows are first renamed densely in
// increasing order (rank among the distinct ids present).  An injective renaming leaves every
// |P_u ∩ P_v| unchanged and keeps rows sorted; |P_u| (psize) is untouched.
__global__ void k_mark_items(const int32_t *__restrict__ items, int64_t nnz, uint32_t *__restrict__ bm) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < nnz) {
    const uint32_t x = (uint32_t)items[p];
    atomicOr(&bm[x >> 5], 1u << (x & 31));
  }
}
__global__ void k_word_pop(const uint32_t *__restrict__ bm, int64_t nw, int32_t *__restrict__ wc) {
  int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w < nw) wc[w] = __popc(bm[w]);
}
__global__ void k_remap_items(const int32_t *__restrict__ items, int64_t nnz, const uint32_t *__restrict__ bm,
                              const int32_t *__restrict__ wbase, int32_t *__restrict__ out) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < nnz) {
    const uint32_t x = (uint32_t)items[p];
    out[p] = wbase[x >> 5] + __popc(bm[x >> 5] & ((1u << (x & 31)) - 1u));
  }
}

static int compact_items(c2_ctx *ctx, Csr *csr) {
  int rc;
  cudaStream_t st = ctx->stream;
  const int64_t nw = ((int64_t)csr->max_item + 32) / 32;
  uint32_t *bm = (uint32_t *)ws_get(ctx, "cmp_bitmap", (size_t)nw * 4, &rc);
  if (rc) return rc;
  int32_t *wc = (int32_t *)ws_get(ctx, "cmp_wc", (size_t)(2 * nw + 2) * 4, &rc);
  if (rc) return rc;
  int32_t *wbase = wc + nw + 1;
  int32_t *out = (int32_t *)ws_get(ctx, "cmp_items", (size_t)csr->nnz * 4, &rc);
  if (rc) return rc;
  C2_CUDA(ctx, cudaMemsetAsync(bm, 0, (size_t)nw * 4, st));
  k_mark_items<<<nblk(csr->nnz), 256, 0, st>>>(csr->items, csr->nnz, bm);
  C2_LAUNCHED(ctx, "k_mark_items");
  k_word_pop<<<nblk(nw), 256, 0, st>>>(bm, nw, wc);
  C2_LAUNCHED(ctx, "k_word_pop");
  C2_TRY(scan_exclusive(ctx, wc, wbase, nw));
  k_remap_items<<<nblk(csr->nnz), 256, 0, st>>>(csr->items, csr->nnz, bm, wbase, out);
  C2_LAUNCHED(ctx, "k_remap_items");
  int32_t distinct = 0;
  C2_CUDA(ctx, cudaMemcpyAsync(&distinct, wbase + nw, 4, cudaMemcpyDeviceToHost, st));
  C2_TRY(stream_sync(ctx, "item compaction"));
  csr->items = out;
  csr->max_item = distinct - 1;
  return C2_OK;
}

int local_knn(c2_ctx *ctx, const Csr &csr_in, int t, const Clusters &cl, int k, c2_cand *out, bool fused,
              c2_cand **result) {
  int rc;
  cudaStream_t st = ctx->stream;
  Csr csr = csr_in;
  if ((int64_t)csr.max_item + 1 > (int64_t)MAX_WIN * 50000) {
    C2_TRY(compact_items(ctx, &csr));
    if ((int64_t)csr.max_item + 1 > (int64_t)MAX_WIN * 50000)
      return set_err(ctx, C2_EDATA, "Step 2 supports at most %d distinct item ids (got %d)", MAX_WIN * 50000,
                     csr.max_item + 1);
  }
  const int32_t n = csr.n;
  int32_t hcum[C2_MAX_T + 1];
  hcum[0] = 0;
  for (int f = 0; f < t; ++f) hcum[f + 1] = hcum[f] + cl.n_clusters[f];
  const int64_t C = hcum[t];
  int32_t *ccum = (int32_t *)ws_get(ctx, "wl_ccum", (C2_MAX_T + 1) * 4 + 4 * WLC * C2_MAX_T, &rc);
  if (rc) return rc;
  int32_t *cnt_fc = ccum + C2_MAX_T + 1;  // [f][WLC]
  C2_CUDA(ctx, cudaMemcpyAsync(ccum, hcum, (t + 1) * 4, cudaMemcpyHostToDevice, st));
  C2_CUDA(ctx, cudaMemsetAsync(cnt_fc, 0, 4 * WLC * C2_MAX_T, st));
  uint32_t *kv = (uint32_t *)ws_get(ctx, "wl_kv", (size_t)C * 4 * 4 + 16, &rc);
  if (rc) return rc;
  uint32_t *key = kv, *val = kv + C, *skey = kv + 2 * C, *sval = kv + 3 * C;
  // Alg. 2: with the hybrid solver, clusters of >= rho k^2 users go to Hyrec
  const uint32_t hyrec_min = ctx->solver == 1 ? (uint32_t)(5 * k * k) : 0xFFFFFFFFu;
  const uint32_t maxs = (uint32_t)std::max(std::min<int64_t>(cl.max_size, (int64_t)hyrec_min - 1), (int64_t)1);
  const int sized = maxs < (1u << 24) ? 1 : 0;
  int sb = 3;  // bits of the key's size field: maxs - s (big clusters) or the slot class (<= 5)
  while (sized && sb < 24 && (1u << sb) <= maxs) ++sb;
  k_wl_classify<<<nblk(C), 256, 0, st>>>(cl.offsets, ccum, t, n, C, key, val, maxs, sized, cnt_fc, hyrec_min, sb);
  C2_LAUNCHED(ctx, "k_wl_classify");
  C2_TRY(radix_sort_pairs(ctx, key, val, skey, sval, C, sb + 8));
  unsigned long long *wacc = (unsigned long long *)ws_get(ctx, "work_acc", 16, &rc);
  if (rc) return rc;
  C2_CUDA(ctx, cudaMemsetAsync(wacc, 0, 8, st));
  k_work_steps<<<std::min<unsigned>(nblk((int64_t)t * n), ctx->num_sms * 5), 256, 0, st>>>(cl.offsets, cl.cluster_of, csr.psize, (int64_t)t * n, n, wacc);
  C2_LAUNCHED(ctx, "k_work_steps");
  int32_t hfc[WLC * C2_MAX_T];
  unsigned long long hwork = 0;
  C2_CUDA(ctx, cudaMemcpyAsync(hfc, cnt_fc, 4 * WLC * t, cudaMemcpyDeviceToHost, st));
  C2_CUDA(ctx, cudaMemcpyAsync(&hwork, wacc, 8, cudaMemcpyDeviceToHost, st));
  C2_TRY(stream_sync(ctx, "worklist counts"));
  ctx->stats.work_steps = (int64_t)hwork;
  int64_t nbig = 0, nsmall = 0, nsingle = 0, nbigtiles = 0, nhyrec = 0, nv_big_cnt = 0;
  int32_t hy_lo[C2_MAX_T + 1];
  for (int f = 0; f < t; ++f) {
    hy_lo[f] = (int32_t)nhyrec;
    nhyrec += hfc[f * WLC + 8];
    nbig += hfc[f * WLC + 7];
    nv_big_cnt += hfc[f * WLC + 9];
    nbigtiles += hfc[f * WLC + 0];
    for (int c = 1; c <= 5; ++c) nsmall += hfc[f * WLC + c];
    nsingle += hfc[f * WLC + 6];
  }
  // mixed slices: groups (f, class) in sorted order
  std::vector<MixGroup> groups;
  int64_t nmix = 0, entry = 0;
  std::vector<int64_t> mix_lo(t + 1, 0);
  for (int f = 0; f < t; ++f) {
    mix_lo[f] = nmix;
    for (int c = 1; c <= 5; ++c) {
      int32_t cntc = hfc[f * WLC + c];
      if (!cntc) continue;
      int per = 32 >> c;
      groups.push_back(MixGroup{f, c, (int32_t)entry, cntc, (int32_t)nmix});
      entry += cntc;
      nmix += (cntc + per - 1) / per;
    }
  }
  mix_lo[t] = nmix;

  hy_lo[t] = (int32_t)nhyrec;
  if (fused) {
    k_init_pads<<<nblk((int64_t)n * k), 256, 0, st>>>(out, (int64_t)n * k);
    C2_LAUNCHED(ctx, "k_init_pads");
  }
  // Hyrec clusters (sorted after the singletons): their lists go straight to cand (local mode) or
  // are merged into the running lists (fused), before the tiles (the merge is order-independent)
  C2_TRY(hyrec_clusters(ctx, csr, t, cl.offsets, cl.members, ccum, sval + (C - nhyrec), nhyrec, hy_lo, k,
                        ctx->hyrec_seed, out, fused));

  // ---- tile descriptors: big clusters (length-sorted members) + mixed slices
  const int64_t ncl = nbig + nmix;
  const int64_t nslices = nbigtiles + nmix;
  BigC *bcs = nullptr;
  Tile *tiles = nullptr;
  int32_t *vperm = nullptr, *vsize = nullptr, *blk_len8 = nullptr, *blk_off8 = nullptr;
  uint4 *packed = nullptr;
  bool relabel = false;
  const int32_t m = csr.max_item + 1;
  int32_t nwin = (int32_t)((m + 50000 - 1) / 50000);
  int32_t W = (int32_t)((m + nwin - 1) / nwin);

  unsigned long long *hv_need = nullptr;
  int64_t nv_big_all = 0;  // members of all big clusters (all functions)
  if (nslices > 0) {
    bcs = (BigC *)ws_get(ctx, "bc", (size_t)ncl * sizeof(BigC), &rc);
    if (rc) return rc;
    tiles = (Tile *)ws_get(ctx, "tiles", (size_t)nslices * sizeof(Tile), &rc);
    if (rc) return rc;
    int64_t nv_big = 0;
    int32_t *bsz = (int32_t *)ws_get(ctx, "bc_sz", (size_t)(nbig + 1) * 4 * 5, &rc);
    if (rc) return rc;
    int32_t *bns = bsz + (nbig + 1), *vp_scan = bsz + 2 * (nbig + 1), *sl_scan = bsz + 3 * (nbig + 1);
    int32_t *bstart = bsz + 4 * (nbig + 1);
    if (nbig > 0) {
      k_bc_sizes<<<nblk(nbig), 256, 0, st>>>(sval, nbig, cl.offsets, ccum, t, n, bsz, bns);
      C2_LAUNCHED(ctx, "k_bc_sizes");
      C2_TRY(scan_exclusive(ctx, bsz, vp_scan, nbig));
      C2_TRY(scan_exclusive(ctx, bns, sl_scan, nbig));
      nv_big = nv_big_cnt;  // (= vp_scan[nbig]; counted by k_wl_classify, read at the worklist sync)
      nv_big_all = nv_big;
    }
    vperm = (int32_t *)ws_get(ctx, "vperm", (size_t)(nv_big + nmix * 32 + 1) * 4 * 2, &rc);
    if (rc) return rc;
    vsize = vperm + (nv_big + nmix * 32 + 1);  // |P_v| of every vperm entry (0 for holes)
    if (nbig > 0) {
      k_bc_fill<<<nblk(nbig), 256, 0, st>>>(sval, nbig, cl.offsets, ccum, t, n, vp_scan, sl_scan, bcs, tiles, bstart);
      C2_LAUNCHED(ctx, "k_bc_fill");
      k_sl_sort<<<(unsigned)nbig, 256, 0, st>>>(bcs, bstart, cl.members, n, csr.psize, vperm, vsize);
      C2_LAUNCHED(ctx, "k_sl_sort");
    }
    if (nmix > 0) {
      MixGroup *dgroups = (MixGroup *)ws_get(ctx, "mix_groups", groups.size() * sizeof(MixGroup), &rc);
      if (rc) return rc;
      C2_CUDA(ctx, cudaMemcpyAsync(dgroups, groups.data(), groups.size() * sizeof(MixGroup), cudaMemcpyHostToDevice,
                                   st));
      C2_CUDA(ctx, cudaMemsetAsync(vperm + nv_big, 0xFF, (size_t)nmix * 32 * 4, st));
      C2_CUDA(ctx, cudaMemsetAsync(vsize + nv_big, 0, (size_t)nmix * 32 * 4, st));
      k_mix_fill<<<nblk(nsmall), 256, 0, st>>>(sval + nbig, nsmall, cl.offsets, ccum, t, n, cl.members, dgroups,
                                               (int)groups.size(), (int32_t)nv_big, csr.psize, vperm, vsize);
      C2_LAUNCHED(ctx, "k_mix_fill");
      k_mix_bc<<<nblk(nmix), 256, 0, st>>>(dgroups, (int)groups.size(), nmix, nbig, (int32_t)nv_big, nbigtiles, bcs,
                                           tiles);
      C2_LAUNCHED(ctx, "k_mix_bc");
    }
    // exact sizes of the per-function buffers handed to k_row_topk (read at the next sync)
    hv_need = (unsigned long long *)ws_get(ctx, "hv_need", (size_t)2 * C2_MAX_T * 8, &rc);
    if (rc) return rc;
    C2_CUDA(ctx, cudaMemsetAsync(hv_need, 0, (size_t)2 * t * 8, st));
    k_cnt_need<<<nblk(ncl), 256, 0, st>>>(bcs, ncl, hv_need, t);
    C2_LAUNCHED(ctx, "k_cnt_need");
    C2_CUDA(ctx, cudaMemcpyAsync(ctx->h_small + 256, hv_need, (size_t)2 * t * 8, cudaMemcpyDeviceToHost, st));
    // cluster-local relabeling (one window of kc+1 words per tile) when the unit bitmaps fit
    // in shared memory; otherwise windows over the global item range
    const int32_t nwq = (m + 31) / 32;
    const size_t rl_smem = (size_t)(5 * nwq + 1 + RL_MAXS) * 4;
    // (pays off only when the global range needs several windows: a unit then usually fits one)
    relabel = ctx->relabel && nwin >= 3 && maxs <= (uint32_t)RL_MAXS && rl_smem <= ctx->smem_optin;
    if (relabel) {
      blk_len8 = (int32_t *)ws_get(ctx, "blk_len8", (size_t)(2 * nslices + 2) * 4, &rc);
      if (rc) return rc;
      blk_off8 = blk_len8 + nslices + 1;
      k_sl_maxlen<<<nblk(nslices * 32), 256, 0, st>>>(tiles, nslices, bcs, vperm, csr.psize, blk_len8);
      C2_LAUNCHED(ctx, "k_sl_maxlen");
      C2_TRY(scan_exclusive(ctx, blk_len8, blk_off8, nslices));
      int32_t tot8;
      C2_CUDA(ctx, cudaMemcpyAsync(&tot8, blk_off8 + nslices, 4, cudaMemcpyDeviceToHost, st));
      C2_TRY(stream_sync(ctx, "packed size"));
      packed = (uint4 *)ws_get(ctx, "packed", ((size_t)tot8 + PK_SLACK_ROWS) * 32 * 16 + 16, &rc);
      if (rc) return rc;
      int *rl = (int *)ws_get(ctx, "relabel_ctr", 16, &rc);
      if (rc) return rc;
      C2_CUDA(ctx, cudaMemsetAsync(rl, 0, 16, st));
      C2_CUDA(ctx, cudaFuncSetAttribute(k_relabel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rl_smem));
      int rl_occ = 1;
      C2_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rl_occ, k_relabel, RL_T, rl_smem));
      k_relabel<<<ctx->num_sms * std::max(rl_occ, 1), RL_T, rl_smem, st>>>(bcs, ncl, vperm, csr.offs, csr.items, nwq, blk_off8, blk_len8,
                                                     reinterpret_cast<PackT *>(packed), rl, rl + 1);
      C2_LAUNCHED(ctx, "k_relabel");
      int32_t hkc;
      C2_CUDA(ctx, cudaMemcpyAsync(&hkc, rl + 1, 4, cudaMemcpyDeviceToHost, st));
      C2_TRY(stream_sync(ctx, "unit universes"));
      if (hkc + 1 <= 50000) {
        nwin = 1;
        W = hkc;
      } else {
        relabel = false;  // a unit universe too large for one window: global windows instead
      }
    }
    if (!relabel) {
      const int64_t nb = nslices * nwin;
      blk_len8 = (int32_t *)ws_get(ctx, "blk_len8", (size_t)(2 * nb + 2) * 4, &rc);
      if (rc) return rc;
      blk_off8 = blk_len8 + nb + 1;
      int32_t *bounds = (int32_t *)ws_get(ctx, "sl_bounds", (size_t)nslices * 32 * (nwin + 1) * 4, &rc);
      if (rc) return rc;
      int32_t *ub = nullptr;
      if (nwin > 1) {
        ub = (int32_t *)ws_get(ctx, "user_bounds", (size_t)n * (nwin - 1) * 4, &rc);
        if (rc) return rc;
        k_user_bounds<<<nblk(n), 256, 0, st>>>(csr.offs, csr.items, n, W, nwin, ub);
        C2_LAUNCHED(ctx, "k_user_bounds");
      }
      k_sl_len<<<nblk(nslices * 32), 256, 0, st>>>(tiles, nslices, bcs, vperm, csr.offs, ub, W, nwin, blk_len8,
                                                   bounds);
      C2_LAUNCHED(ctx, "k_sl_len");
      C2_TRY(scan_exclusive(ctx, blk_len8, blk_off8, nb));
      int32_t tot8;
      C2_CUDA(ctx, cudaMemcpyAsync(&tot8, blk_off8 + nb, 4, cudaMemcpyDeviceToHost, st));
      C2_TRY(stream_sync(ctx, "packed size"));
      packed = (uint4 *)ws_get(ctx, "packed", ((size_t)tot8 + PK_SLACK_ROWS) * 32 * 16 + 16, &rc);
      if (rc) return rc;
      // bank-rotated order pays for its second pass only when lists are long (one window)
      if (nwin == 1) {
        k_sl_fill<<<nblk(nslices * 32 * 32), 256, 0, st>>>(nslices, bounds, csr.items, W, nwin, blk_len8, blk_off8,
                                                           reinterpret_cast<PackT *>(packed), 1);
        C2_LAUNCHED(ctx, "k_sl_fill");
      } else {
        if (C2_FILL_COAL) {
          // one resident wave (the grid-stride loop splits the blocks evenly over the warps)
          static int occ_fc = 0;
          if (!occ_fc) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_fc, k_sl_fill_coal, FR_WARPS * 32, 0);
          k_sl_fill_coal<<<ctx->num_sms * std::max(occ_fc, 1), FR_WARPS * 32, 0, st>>>(nb, nwin, bounds, csr.items, W, blk_len8, blk_off8,
                                                                      packed);
          C2_LAUNCHED(ctx, "k_sl_fill_coal");
        } else {
#if !C2_PACK32
          const int vec = ((uintptr_t)csr.items & 15) == 0 ? 1 : 0;
          k_sl_fill_rows<<<ctx->num_sms * 16, 256, 0, st>>>(nb, nwin, bounds, csr.items, W, blk_len8, blk_off8, packed,
                                                            csr.nnz, vec);
          C2_LAUNCHED(ctx, "k_sl_fill_rows");
#endif
        }
      }
    }
  }

  // ---- per-tile descriptor records
  int32_t *trec = nullptr;
  if (nslices > 0) {
    trec = (int32_t *)ws_get(ctx, "tile_rec", (size_t)nslices * REC_W * 4, &rc);
    if (rc) return rc;
    k_tile_rec<<<nblk(nslices * 32), 256, 0, st>>>(tiles, nslices, bcs, vperm, vsize, blk_len8, blk_off8, nwin, trec);
    C2_LAUNCHED(ctx, "k_tile_rec");
  }

  // ---- light-row survivor buffers (fused only): surv [n][qmax], per-user counts zeroed here and
  //      re-zeroed by k_surv_merge after every function
  c2_cand *surv = nullptr;
  int32_t *surv_qn = nullptr;
  // survivor slots: the option's value, but at most 16 GiB of slots (halved until it fits, >= 64); with
  // slots >= N - 1 no light row can overflow and the light epilogue needs no barrier
  int surv_qmax = ctx->surv_qmax;
  while (surv_qmax > 64 && (size_t)n * surv_qmax * sizeof(c2_cand) > ((size_t)16 << 30)) surv_qmax >>= 1;
  if (fused && C2_LIGHT && surv_qmax > 0 && nslices > 0) {
    surv = (c2_cand *)ws_get(ctx, "surv", (size_t)n * surv_qmax * sizeof(c2_cand), &rc);
    if (rc) return rc;
    surv_qn = (int32_t *)ws_get(ctx, "surv_qn", (size_t)n * 4, &rc);
    if (rc) return rc;
    C2_CUDA(ctx, cudaMemsetAsync(surv_qn, 0, (size_t)n * 4, st));
  }
  // ---- tile kernel configuration
  TileKernel tk = nullptr;
  int grid = 0;
  int32_t stg_off = 0, stg_cap = 0, scr_off = 0;
  size_t smem = 0;
  int *counters = nullptr;
  uint16_t *hv_cnt = nullptr;
  RowRec *hv_recs = nullptr;
  unsigned long long *hv_ctr = nullptr;
  int *hv_err = nullptr;
  int64_t hv_cap = 0, hv_rcap = 0;
  bool gfm = false;
  int64_t *gf_wl = nullptr, *gf_cb = nullptr, *gf_sum = nullptr, *gf_rng = nullptr;
  uint8_t *gf_bytes = nullptr;
  int32_t *gf_witem = nullptr;
  int64_t gf_icap = 0;
  int64_t gf_bc[C2_MAX_T + 1] = {0};
  if (nslices > 0) {
    int nbits = bits_for((int64_t)csr.max_len + 1);
    int nhi = std::max(nbits - 4, 1);
    int max_sl = (int)((maxs + 31) / 32);
    int vpt = max_sl <= TILE_WARPS ? 1 : max_sl <= 2 * TILE_WARPS ? 2 : 4;
    const size_t budget = (C2_SMEM_BUDGET ? std::min<size_t>(C2_SMEM_BUDGET, ctx->smem_optin) : ctx->smem_optin) -
                          4096;  // minus the kernel's static shared memory (~2.5 KB)
    const size_t mw = (size_t)((W + 4) & ~3);  // M: W + 1 words
    // split-probe scratch: TILE_WARPS x (4 + nhi) planes x 32 lanes, in M's words when W + 1 allows
    const size_t scrw = (size_t)TILE_WARPS * (4 + (nhi <= 4 ? 4 : (C2_NHI7 && nhi <= 7) ? 7 : nhi <= 8 ? 8 : 11)) * 32;
    const size_t scr_own = (size_t)W + 1 >= scrw ? 0 : scrw;
    scr_off = scr_own ? (int32_t)mw : 0;
    stg_off = (int32_t)(mw + scr_own);
    const int64_t slack_w = C2_PACK32 ? PK_SLACK_ROWS * 32 * 4 : 0;  // words readable past the staging
    stg_cap = (int32_t)std::min<int64_t>(2048, ((int64_t)budget / 4 - stg_off - slack_w) / 8);  // 16-byte groups, each
    if (stg_cap < 64) stg_cap = 0;
    smem = ((size_t)stg_off + (size_t)stg_cap * 8 + (size_t)slack_w) * 4;
    tk = pick_tile(nhi, vpt);
    C2_CUDA(ctx, cudaFuncSetAttribute(tk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    C2_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tk, TILE_T, smem));
    occ = std::max(occ, 1);
    grid = (int)std::min<int64_t>((int64_t)ctx->num_sms * occ, nslices);
    counters = (int *)ws_get(ctx, "tile_counter", 4 * (2 * C2_MAX_T + 2), &rc);
    if (rc) return rc;
    C2_CUDA(ctx, cudaMemsetAsync(counters, 0, 4 * (2 * C2_MAX_T + 2), st));
    // rows handed to k_row_topk, per function (the buffers are reused function after function)
    for (int f = 0; f < t; ++f) {
      hv_cap = std::max<int64_t>(hv_cap, (int64_t)ctx->h_small[256 + f]);
      hv_rcap = std::max<int64_t>(hv_rcap, (int64_t)ctx->h_small[256 + t + f]);
    }
    // GoldFinger on the tensor cores: the big clusters' count rows get a region of their own
    gfm = csr.gf_words != nullptr && ctx->gf_tensor && nbig > 0;
    hv_cnt = (uint16_t *)ws_get(ctx, "hv_cnt", (size_t)hv_cap * (gfm ? 4 : 2) + 16, &rc);
    if (rc) return rc;
    hv_recs = (RowRec *)ws_get(ctx, "hv_recs", (size_t)(hv_rcap + 1) * sizeof(RowRec), &rc);
    if (rc) return rc;
    hv_ctr = (unsigned long long *)ws_get(ctx, "hv_ctr", (size_t)(2 * C2_MAX_T + 2) * 8, &rc);
    if (rc) return rc;
    hv_err = (int *)(hv_ctr + 2 * C2_MAX_T + 1);
    C2_CUDA(ctx, cudaMemsetAsync(hv_ctr, 0, (size_t)(2 * C2_MAX_T + 2) * 8, st));
    if (gfm) {
      // per function: its big clusters [gf_bc[f], gf_bc[f+1]) (bcs is ordered by function), work-item and
      // count-row prefixes over them
      for (int f = 0; f < t; ++f) gf_bc[f + 1] = gf_bc[f] + hfc[f * WLC + 7];
      gf_wl = (int64_t *)ws_get(ctx, "gf_wl", (size_t)(2 * nbig + 2 * C2_MAX_T + 2 + C2_MAX_T + 1) * 8, &rc);
      if (rc) return rc;
      gf_cb = gf_wl + nbig;
      gf_sum = gf_cb + nbig;
      gf_rng = gf_sum + 2 * C2_MAX_T + 2;
      for (int f = 0; f <= t; ++f) ctx->h_small[400 + f] = gf_bc[f];
      C2_CUDA(ctx, cudaMemcpyAsync(gf_rng, ctx->h_small + 400, (size_t)(t + 1) * 8, cudaMemcpyHostToDevice, st));
      // work items per function <= sum over its clusters of (s/128 + 1)^2 <= nbig + 2 rows/128 + maxs rows/128^2
      gf_icap = nbig + 2 * (nv_big_all / 128 + 1) + (int64_t)maxs * (nv_big_all / 16384 + 1) + 16;
      gf_witem = (int32_t *)ws_get(ctx, "gf_witem", (size_t)t * gf_icap * 4, &rc);
      if (rc) return rc;
      C2_TRY(gf_prefix(ctx, bcs, gf_rng, t, nbig, gf_wl, gf_cb, gf_sum, gf_witem, gf_icap));
      gf_bytes = (uint8_t *)ws_get(ctx, "gf_bytes", (size_t)n * 1024, &rc);
      if (rc) return rc;
      C2_TRY(gf_expand(ctx, csr.gf_words, n, gf_bytes));
    }
  }
  // tiles [lo, hi) of function f: counts -> light rows' survivors (c2_build) + count rows for k_row_topk
  auto launch_tiles = [&](int64_t lo, int64_t hi, int ci, int f) -> int {
    if (hi <= lo) return C2_OK;
    TileArgs ta{tiles, lo, hi, counters + ci, bcs, vperm, vsize, trec, blk_len8, blk_off8, packed, csr.psize, n, W, nwin, k,
                fused ? out : nullptr, ctx->kstats, stg_off, stg_cap, scr_off, relabel ? 1 : 0, fused ? surv : nullptr, surv_qn,
                surv_qmax, hv_cnt, hv_cap, hv_ctr + f, hv_recs, hv_rcap, hv_ctr + C2_MAX_T + f, hv_err};
    int g = (int)std::min<int64_t>(grid, hi - lo);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->timing) {
      while ((int)ctx->tile_ev.size() < 2 * (ctx->tile_ev_used + 1)) {
        cudaEvent_t e;
        C2_CUDA(ctx, cudaEventCreate(&e));
        ctx->tile_ev.push_back(e);
      }
      e0 = ctx->tile_ev[2 * ctx->tile_ev_used];
      e1 = ctx->tile_ev[2 * ctx->tile_ev_used + 1];
      ctx->tile_ev_used++;
      C2_CUDA(ctx, cudaEventRecord(e0, st));
    }
    tk<<<g, TILE_T, smem, st>>>(ta);
    C2_LAUNCHED(ctx, "k_local_tile");
    if (ctx->timing) C2_CUDA(ctx, cudaEventRecord(e1, st));
    ctx->stats.tile_launches++;
    if (ctx->sync_check) {
      int herr = 0;
      C2_CUDA(ctx, cudaMemcpy(&herr, hv_err, 4, cudaMemcpyDeviceToHost));
      if (herr) return set_err(ctx, C2_ECUDA, "k_local_tile: row buffers too small (internal sizing error)");
    }
    return C2_OK;
  };
  // the per-row top-k of the rows function f's tiles handed over
  auto launch_rows = [&](int f) -> int {
    if (nslices == 0) return C2_OK;
    RowArgs ra{hv_recs, (const int64_t *)(hv_ctr + C2_MAX_T + f), hv_cnt, vperm, vsize, fused ? out : nullptr, out, n, k,
               ctx->kstats};
    return launch_row_topk(ctx, ra);
  };
  auto launch_singles = [&](int64_t lo, int64_t hi, const c2_cand *seed, c2_cand *dst) -> int {
    if (hi <= lo) return C2_OK;
    k_singles<<<nblk((hi - lo) * k), 256, 0, st>>>(sval + nbig + nsmall, nsingle, cl.offsets, ccum, t, n, cl.members,
                                                   k, lo, hi, seed, dst);
    C2_LAUNCHED(ctx, "k_singles");
    return C2_OK;
  };
  // Alg. 3 order (c2_build): function by function, every user's running list is merged in place
  // with its neighbourhood in that function's cluster (singletons: nothing to merge).
  // c2_local_knn: the same launches write each function's lists cand[f].
  int64_t blo = 0;
  for (int f = 0; f < t; ++f) {
    C2Range rf("hash function (tiles, row top-k, light-row merge)");
    const int64_t bhi = blo + hfc[f * WLC + 0];
    if (gfm) {
      GfArgs ga{bcs, gf_bc[f], gf_bc[f + 1], gf_wl, gf_cb, gf_sum + 2 * f, gf_witem + (int64_t)f * gf_icap, vperm, vsize, gf_bytes, n, k,
                fused ? out : nullptr, fused ? surv : nullptr, surv_qn, surv_qmax, hv_cnt, hv_cap, hv_recs,
                hv_ctr + C2_MAX_T + f, hv_rcap, hv_err};
      C2_TRY(launch_gf_mma(ctx, ga));
    } else {
      C2_TRY(launch_tiles(blo, bhi, 2 * f, f));
    }
    C2_TRY(launch_tiles(nbigtiles + mix_lo[f], nbigtiles + mix_lo[f + 1], 2 * f + 1, f));
    if (surv && C2_SIDE_MERGE) {
      // the light rows' Alg. 3 step and the other rows' top-k update disjoint users' lists: they run
      // concurrently (side stream); the next function's tiles wait for both
      if (!ctx->side_stream) {
        C2_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking));
        for (auto &e : ctx->side_ev) C2_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      }
      C2_CUDA(ctx, cudaEventRecord(ctx->side_ev[0], st));
      C2_CUDA(ctx, cudaStreamWaitEvent(ctx->side_stream, ctx->side_ev[0], 0));
      C2_TRY(launch_surv_merge(ctx, surv, surv_qn, surv_qmax, n, k, out, ctx->side_stream));
      C2_CUDA(ctx, cudaEventRecord(ctx->side_ev[1], ctx->side_stream));
      C2_TRY(launch_rows(f));
      C2_CUDA(ctx, cudaStreamWaitEvent(st, ctx->side_ev[1], 0));
    } else {
      C2_TRY(launch_rows(f));
      if (surv) C2_TRY(launch_surv_merge(ctx, surv, surv_qn, surv_qmax, n, k, out));  // light rows' Alg. 3 step
    }
    blo = bhi;
  }
  if (!fused) C2_TRY(launch_singles(0, nsingle, nullptr, out));
  if (result) *result = out;
  return C2_OK;
}

}  // namespace c2
