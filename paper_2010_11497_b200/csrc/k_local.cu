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

#ifndef C2_EPI
#define C2_EPI 0  // 1: light rows filtered in the phase-A epilogue (measured slower)
#endif
#ifndef C2_SNAKE
#define C2_SNAKE 1  // 1: warp w probes slices w, 2W-1-w, 2W+w, ... (slices are longest-first: balances warps)
#endif
#ifndef C2_BULK
#define C2_BULK 1  // 1: tile records + staged row blocks by cp.async.bulk on mbarriers (TMA bulk path)
#endif
#ifndef C2_RANKMERGE
#define C2_RANKMERGE 1  // 1: rank-based Alg. 3 step for <= 32 survivors; 0: insertion (<= 16)
#endif

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
#ifndef C2_SMEM_BUDGET
#define C2_SMEM_BUDGET 0  // bytes of dynamic shared memory per tile CTA (0: the opt-in maximum)
#endif
constexpr int TILE_T = C2_TILE_T;
constexpr int TILE_WARPS = TILE_T / 32;
constexpr int MAX_WIN = 16;

static inline unsigned nblk(int64_t x, int bs = 256) { return (unsigned)((x + bs - 1) / bs); }
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
constexpr int WLC = 16;  // counters per function: 0 big tiles, 1..5 small per class, 6 single, 7 big, 8 hyrec
__device__ __forceinline__ int slot_class(int32_t s) {  // slot = 2^class >= s, s in [2, 32]
  int c = 1;
  while ((1 << c) < s) ++c;
  return c;
}

__global__ void k_wl_classify(const int32_t *__restrict__ offsets, const int32_t *__restrict__ ccum, int t,
                              int32_t n, int64_t C, uint32_t *__restrict__ key, uint32_t *__restrict__ val,
                              uint32_t maxs, int sized, int32_t *__restrict__ cnt_fc, uint32_t hyrec_min) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= C) return;
  int f = find_f(ccum, t, g);
  int64_t c = g - ccum[f];
  const int32_t *off = offsets + (int64_t)f * (n + 1);
  uint32_t s = (uint32_t)(off[c + 1] - off[c]);
  uint32_t k;
  if (s >= hyrec_min) {  // Alg. 2 else-branch: Hyrec (C2_SOLVER_HYBRID only; hyrec_min = UINT32_MAX otherwise)
    k = (3u << 30) | ((uint32_t)f << 24);
    atomicAdd(&cnt_fc[f * WLC + 8], 1);
  } else if (s > 32) {
    k = ((uint32_t)f << 24) | (sized ? min(maxs - s, 0xFFFFFFu) : 0u);
    atomicAdd(&cnt_fc[f * WLC + 0], (int32_t)((s + 31) / 32));  // big tiles of f
    atomicAdd(&cnt_fc[f * WLC + 7], 1);                          // big clusters of f
  } else if (s >= 2) {
    int cl = slot_class((int32_t)s);
    k = (1u << 30) | ((uint32_t)f << 24) | (uint32_t)cl;
    atomicAdd(&cnt_fc[f * WLC + cl], 1);  // small clusters of (f, class), class 1..5
  } else {
    k = (2u << 30) | ((uint32_t)f << 24);
    atomicAdd(&cnt_fc[f * WLC + 6], 1);  // singletons of f
  }
  key[g] = k;
  val[g] = (uint32_t)g;
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
__global__ void k_sl_len(const Tile *__restrict__ tiles, int64_t nslices, const BigC *__restrict__ bcs,
                         const int32_t *__restrict__ vperm, const int32_t *__restrict__ offs,
                         const int32_t *__restrict__ items, int32_t W, int nwin, int32_t *__restrict__ blk_len8,
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
    const int32_t q = w + 1 < nwin ? lower_bound_items(items, p, pe, (w + 1) * W) : pe;
    bd[w + 1] = q;
    int c = q - p;
    p = q;
#pragma unroll
    for (int o = 16; o; o >>= 1) c = max(c, __shfl_xor_sync(0xffffffffu, c, o));
    if (lane == 0) blk_len8[sl * nwin + w] = (c + 7) / 8;
  }
}

// Order within a list does not matter to the counts, so each member's window list is laid out
// by bank: key = (x - e) mod 32 for the member in lane e (the mask word of item x sits in bank
// x mod 32).  At any step the 32 lanes then read words of ~32 different banks instead of random
// ones (random: ~3.4 shared-memory wavefronts per mask load, which binds the probe).
__global__ void __launch_bounds__(256) k_sl_fill(int64_t nslices, const int32_t *__restrict__ bounds,
                                                 const int32_t *__restrict__ items, int32_t W, int nwin,
                                                 const int32_t *__restrict__ blk_len8,
                                                 const int32_t *__restrict__ blk_off8, uint16_t *__restrict__ packed16,
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
    const int32_t len = blk_len8[sl * nwin + w] * 8;
    uint16_t *dst = packed16 + (int64_t)blk_off8[sl * nwin + w] * 256 + e * 8;
    if (!bank_order) {  // plain order: one pass, ballot compaction
      int cnt = 0;
      for (int32_t p0 = pb; p0 < pe; p0 += 32) {
        const int32_t p = p0 + lane;
        const int32_t r = p < pe ? items[p] - lo : -1;
        const bool in = r >= 0 && r < W;
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        const int pos = cnt + __popc(bal & ((1u << lane) - 1));
        if (in) dst[(pos >> 3) * 256 + (pos & 7)] = (uint16_t)r;
        cnt += __popc(bal);
      }
      for (int pos = cnt + lane; pos < len; pos += 32) dst[(pos >> 3) * 256 + (pos & 7)] = (uint16_t)W;
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
        dst[(pos >> 3) * 256 + (pos & 7)] = (uint16_t)r;
      }
    }
    for (int pos = cnt + lane; pos < len; pos += 32) dst[(pos >> 3) * 256 + (pos & 7)] = (uint16_t)W;
    __syncwarp();
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
  if (lane == 0) len8[sl] = (c + 7) / 8;
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
                                                 uint16_t *__restrict__ packed16, int *__restrict__ counter,
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
        uint16_t *dst = packed16 + (int64_t)blk_off8[b.sl_off + (i >> 5)] * 256 + (i & 31) * 8;
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
          if (keep) dst[(pos >> 3) * 256 + (pos & 7)] = (uint16_t)lid;
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
      const int len8 = (mx + 7) / 8;
      const int sl = b.sl_off + (i >> 5);
      if ((i & 31) == 0) blk_len8[sl] = len8;
      uint16_t *dst = packed16 + (int64_t)blk_off8[sl] * 256 + (i & 31) * 8;
      for (int pos = slen[i]; pos < len8 * 8; ++pos) dst[(pos >> 3) * 256 + (pos & 7)] = (uint16_t)kc;
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

// ------------------------------------------------------------------ candidate lists
// A candidate (v, i, U) is held as {iu = i | U << 16, id}.  The order (A13): a before b iff
// a.i * b.U > b.i * a.U, ties by lower id.  SENT is worse than every real candidate.
struct Cand {
  uint32_t iu;
  int32_t id;
};
__device__ __forceinline__ Cand sent() { return Cand{1u << 16, INT32_MAX}; }
__device__ __forceinline__ bool is_real(Cand a) { return a.id != INT32_MAX; }
__device__ __forceinline__ bool better_c(Cand a, Cand b) {
  uint32_t l = (a.iu & 0xFFFFu) * (b.iu >> 16), r = (b.iu & 0xFFFFu) * (a.iu >> 16);
  return l > r || (l == r && a.id < b.id);
}
__device__ __forceinline__ Cand shfl_c(Cand a, int src) {
  return Cand{__shfl_sync(0xffffffffu, a.iu, src), __shfl_sync(0xffffffffu, a.id, src)};
}
__device__ __forceinline__ Cand shfl_xor_c(Cand a, int m) {
  return Cand{__shfl_xor_sync(0xffffffffu, a.iu, m), __shfl_xor_sync(0xffffffffu, a.id, m)};
}
__device__ __forceinline__ Cand shfl_up_c(Cand a) {
  return Cand{__shfl_up_sync(0xffffffffu, a.iu, 1), __shfl_up_sync(0xffffffffu, a.id, 1)};
}
__device__ __forceinline__ c2_cand to_out(Cand a) {
  return is_real(a) ? c2_cand{a.id, (uint16_t)(a.iu & 0xFFFFu), (uint16_t)(a.iu >> 16)} : c2_cand{-1, 0, 0};
}
__device__ __forceinline__ Cand from_out(c2_cand e) {
  return e.id >= 0 ? Cand{(uint32_t)e.inter | ((uint32_t)e.uni << 16), e.id} : sent();
}

// Sort key of a candidate: K = q32 << 32 | (2^32 - 1 - id), larger = better, where
// q32 = floor(i/U * 2^32) (U >= 1; 2^32 - 1 for i == U) from the IEEE (correctly rounded) f64
// quotient.  K orders candidates exactly as the fraction comparison (A13): equal fractions
// give identical quotients; distinct fractions with U <= 65534 differ by >= 1/65534^2, i.e. by
// >= 1.00006 after scaling by 2^32, far above the f64 rounding error (< 2^-20), so their
// floors differ.  The payload iu = i | U << 16 rides along.  Sentinel: K = 0.
struct KC {
  uint64_t k;
  uint32_t iu;
};
__device__ __forceinline__ KC to_kc(Cand c) {
  if (!is_real(c)) return KC{0ull, 1u << 16};
  const uint32_t i = c.iu & 0xFFFFu, U = c.iu >> 16;
  const double q = (double)i / (double)U;
  const uint32_t q32 = i >= U ? 0xFFFFFFFFu : (uint32_t)(q * 4294967296.0);
  return KC{((uint64_t)q32 << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)c.id), c.iu};
}
__device__ __forceinline__ int32_t kc_id(KC a) { return (int32_t)(0xFFFFFFFFu - (uint32_t)a.k); }
__device__ __forceinline__ bool kc_real(KC a) { return a.k != 0ull; }
__device__ __forceinline__ Cand kc_cand(KC a) { return kc_real(a) ? Cand{a.iu, kc_id(a)} : sent(); }
__device__ __forceinline__ c2_cand kc_out(KC a) {
  return kc_real(a) ? c2_cand{kc_id(a), (uint16_t)(a.iu & 0xFFFFu), (uint16_t)(a.iu >> 16)} : c2_cand{-1, 0, 0};
}
__device__ __forceinline__ bool better_e(KC a, KC b) { return a.k > b.k; }
__device__ __forceinline__ bool better_e(Cand a, Cand b) { return better_c(a, b); }
__device__ __forceinline__ KC shfl_e(KC a, int src) {
  return KC{__shfl_sync(0xffffffffu, a.k, src), __shfl_sync(0xffffffffu, a.iu, src)};
}
__device__ __forceinline__ KC shfl_xor_e(KC a, int m) {
  return KC{__shfl_xor_sync(0xffffffffu, a.k, m), __shfl_xor_sync(0xffffffffu, a.iu, m)};
}
__device__ __forceinline__ KC shfl_up_e(KC a) {
  return KC{__shfl_up_sync(0xffffffffu, a.k, 1), __shfl_up_sync(0xffffffffu, a.iu, 1)};
}
__device__ __forceinline__ Cand shfl_e(Cand a, int src) { return shfl_c(a, src); }
__device__ __forceinline__ Cand shfl_xor_e(Cand a, int m) { return shfl_xor_c(a, m); }
__device__ __forceinline__ Cand shfl_up_e(Cand a) { return shfl_up_c(a); }

// Bitonic sort of the 32R warp-held elements a[j] (position 32j + lane), best first.
template <int R, class E>
__device__ __forceinline__ void warp_sort(E (&a)[R]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32 * R; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const int js = stride >> 5;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          if ((j & js) == 0) {
            const int p = 32 * j + lane;
            const bool desc = (p & size) == 0;  // lower position takes the better element
            E x = a[j], y = a[j + js];
            if (desc ? better_e(y, x) : better_e(x, y)) {
              a[j] = y;
              a[j + js] = x;
            }
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int p = 32 * j + lane;
          E o = shfl_xor_e(a[j], stride);
          const bool lower = (lane & stride) == 0;
          const bool desc = (p & size) == 0;
          // lower position of a descending block keeps the better one
          if ((lower == desc) ? better_e(o, a[j]) : better_e(a[j], o)) a[j] = o;
        }
      }
    }
  }
}

// Bitonic merge of a bitonic sequence of 32R warp-held elements into best-first order.
template <int R, class E>
__device__ __forceinline__ void warp_bitonic_merge(E (&a)[R]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int stride = 16 * R; stride > 0; stride >>= 1) {
    if (stride >= 32) {
      const int js = stride >> 5;
#pragma unroll
      for (int j = 0; j < R; ++j)
        if ((j & js) == 0 && better_e(a[j + js], a[j])) {
          E x = a[j];
          a[j] = a[j + js];
          a[j + js] = x;
        }
    } else {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        E o = shfl_xor_e(a[j], stride);
        const bool lower = (lane & stride) == 0;
        if (lower ? better_e(o, a[j]) : better_e(a[j], o)) a[j] = o;
      }
    }
  }
}

// Insert x into the sorted warp list a (32R positions, best first); the worst drops out.
template <int R, class E>
__device__ __forceinline__ void warp_insert(E (&a)[R], E x) {
  const int lane = threadIdx.x & 31;
  int pos = 0;
#pragma unroll
  for (int j = 0; j < R; ++j) pos += __popc(__ballot_sync(0xffffffffu, better_e(a[j], x)));
  E up[R];
#pragma unroll
  for (int j = 0; j < R; ++j) up[j] = shfl_up_e(a[j]);
#pragma unroll
  for (int j = 1; j < R; ++j) {
    E last = shfl_e(a[j - 1], 31);
    if (lane == 0) up[j] = last;
  }
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int p = 32 * j + lane;
    if (p == pos) a[j] = x;
    else if (p > pos) a[j] = up[j];
  }
}

template <int R, class E>
__device__ __forceinline__ E warp_get(const E (&a)[R], int p) {
  E r = a[0];
#pragma unroll
  for (int j = 1; j < R; ++j)
    if ((p >> 5) == j) r = a[j];
  return shfl_e(r, p & 31);
}

// Out-of-line copies of the K8 sorting networks: one body per size instead of one per call site
// (the fully unrolled networks otherwise dominate the kernel's code and its i-cache misses).
template <int R>
struct KCA {
  KC e[R];
};
template <int R>
__device__ __noinline__ KCA<R> sort_kc_ni(KCA<R> a) {
  warp_sort<R>(a.e);
  return a;
}
template <int R>
__device__ __noinline__ KCA<R> merge_kc_ni(KCA<R> a) {
  warp_bitonic_merge<R>(a.e);
  return a;
}
template <int R>
__device__ __forceinline__ void sort_kc(KC (&x)[R]) {
  KCA<R> t;
#pragma unroll
  for (int j = 0; j < R; ++j) t.e[j] = x[j];
  t = sort_kc_ni<R>(t);
#pragma unroll
  for (int j = 0; j < R; ++j) x[j] = t.e[j];
}
template <int R>
__device__ __forceinline__ void merge_kc(KC (&x)[R]) {
  KCA<R> t;
#pragma unroll
  for (int j = 0; j < R; ++j) t.e[j] = x[j];
  t = merge_kc_ni<R>(t);
#pragma unroll
  for (int j = 0; j < R; ++j) x[j] = t.e[j];
}

// One Alg. 3 step for one row, by ranks: the m <= 32 queued survivors Q (distinct ids, unsorted)
// and the running list S (best first; its real entries are a prefix, pads have id -1) give
// dst[0..kk) = the first kk distinct ids of S ∪ Q under the order (A13, A16).  A survivor whose id
// is already in S carries identical (i, U) and is dropped.  Every element's output position is
// (its rank in S) + (its rank among the kept survivors): O((|S| + m) * m / 32) exact cross-multiplied
// comparisons per lane, all independent (no sorting network, no 64-bit keys).
template <int KS>
__device__ __forceinline__ void rank_merge(const Cand *qr, int m, const c2_cand *S, int kk, c2_cand *dst) {
  const int lane = threadIdx.x & 31;
  Cand sv[KS];
  int nS = 0;
#pragma unroll
  for (int j = 0; j < KS; ++j) {
    sv[j] = (32 * j + lane < kk) ? from_out(S[32 * j + lane]) : sent();
    nS += __popc(__ballot_sync(0xffffffffu, is_real(sv[j])));
  }
  const Cand q = lane < m ? qr[lane] : sent();
  int rs = 0;
  bool dup = false;
  for (int i = 0; i < nS; ++i) {  // rank of q in S (broadcast reads)
    const Cand si = from_out(S[i]);
    dup |= si.id == q.id;
    rs += better_c(si, q) ? 1 : 0;
  }
  const unsigned dm = __ballot_sync(0xffffffffu, lane < m && dup);
  int rq = 0, sh[KS];
#pragma unroll
  for (int j = 0; j < KS; ++j) sh[j] = 0;
  for (int j = 0; j < m; ++j) {
    const Cand o = shfl_c(q, j);
    if ((dm >> j) & 1u) continue;  // (uniform)
    rq += better_c(o, q) ? 1 : 0;
#pragma unroll
    for (int jj = 0; jj < KS; ++jj) sh[jj] += better_c(o, sv[jj]) ? 1 : 0;
  }
  if (lane < m && !dup && rs + rq < kk) dst[rs + rq] = to_out(q);
#pragma unroll
  for (int jj = 0; jj < KS; ++jj) {
    const int i = 32 * jj + lane;
    if (i < nS && i + sh[jj] < kk) dst[i + sh[jj]] = to_out(sv[jj]);
  }
  for (int p = nS + m - __popc(dm) + lane; p < kk; p += 32) dst[p] = c2_cand{-1, 0, 0};
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

// Shared-memory layout of the K8 phase (32-bit words), aliased onto the M region once phase A
// is done (M is dead then).  Depends on the tile's cluster size s:
//   cnt  [32 rows][RS] u16   |P_r ∩ P_v| by (row, member position); RS = 64*ceil(s/64)+4, so a
//                            warp reading 4 consecutive counts per row (LDS.64, lane = row) is
//                            bank-conflict free
//   vid  [s4] int32          member ids (positions >= s: INT32_MAX)
//   vps  [s4] uint32         member |P_v| (positions >= s: 0)
//   que  [32][qcap] Cand     survivors per row (qcap >= 64*KS, as large as shared memory allows)
struct K8Lay {
  int RS, vid, vps, que, words;
  __host__ __device__ __forceinline__ K8Lay(int s, int qcap) {
    RS = ((s + 63) / 64) * 64 + 4;
    const int s4 = (s + 3) & ~3;
    vid = 16 * RS;
    vps = vid + s4;
    que = vps + s4;
    words = que + 32 * qcap * 2;
  }
};

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
  c2_cand *out;         // local: cand [t][n][k]; fused: running lists after this function
  unsigned long long *kstats;  // C2_OPT_KSTATS counters or nullptr
  uint32_t *gscratch;   // !SMEM_CNT only: per CTA K8Lay(smax, qcap).words words
  int32_t smax;
  int32_t qcap;         // survivor queue capacity per row
  int32_t rl_off;       // fused: word offset of the rows' running lists in shared memory
  int32_t stg_off, stg_cap;  // staging buffer (word offset, capacity in 16-byte groups; 0: off)
  int relabel;          // 1: items are unit-local ids, the tile's window is [0, B.kc) (nwin == 1)
};

// 8 masks of one uint4 of packed u16 item ids
__device__ __forceinline__ void masks8(const uint32_t *__restrict__ M, uint4 d, uint32_t (&m)[8]) {
  m[0] = M[d.x & 0xFFFFu];
  m[1] = M[d.x >> 16];
  m[2] = M[d.y & 0xFFFFu];
  m[3] = M[d.y >> 16];
  m[4] = M[d.z & 0xFFFFu];
  m[5] = M[d.z >> 16];
  m[6] = M[d.w & 0xFFFFu];
  m[7] = M[d.w >> 16];
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

// A fixed reference candidate of row r (|P_r| = pr) in the form that makes the order test of a
// candidate (i, |P_v|, id) two multiply-adds: with U = pr + |P_v| - i and the reference (iT, UT),
//   i*UT > iT*U  <=>  i*(UT + iT) > iT*|P_v| + iT*pr.
// Both sides fit in 32 bits (i <= 32767, U <= 65534, A28).  Ties are decided by id < idlim
// (idlim = idT: strictly better; idT + 1: better or the reference itself).  Unsigned id compare:
// an id of -1 (empty position of a mixed slice) never passes a tie.
struct Ref {
  uint32_t A, B, iT, idlim;
};
__device__ __forceinline__ Ref make_ref(Cand t, uint32_t pr, bool or_equal) {
  const uint32_t i = t.iu & 0xFFFFu, U = t.iu >> 16;
  return Ref{U + i, i * pr, i, (uint32_t)t.id + (or_equal ? 1u : 0u)};
}
__device__ __forceinline__ bool passes(uint32_t i, uint32_t ps, int32_t id, const Ref &R) {
  const uint32_t l = i * R.A, r = R.iT * ps + R.B;
  return l > r || (l == r && (uint32_t)id < R.idlim);
}

template <int NHI, int VPT, int KS, bool SMEM_CNT>
__global__ void __launch_bounds__(TILE_T, C2_TILE_MINB) k_local_tile(TileArgs a) {
  constexpr int R1 = 2 * KS;
  const int qcap = a.qcap;
  extern __shared__ __align__(16) uint32_t dyn[];
  uint32_t *M = dyn;  // phase A: W + 1 words, M[W] == 0
  // tile descriptors, double-buffered: the next tile's are fetched during this tile's K8
  __shared__ int64_t s_it[2];
  __shared__ Tile s_T[2];
  __shared__ BigC s_B[2];
  __shared__ int32_t s_ru2[2][32];
  __shared__ uint32_t s_rp2[2][32];
  __shared__ int32_t s_bl[2][MAX_WIN], s_bo[2][MAX_WIN], s_so[2][MAX_WIN];  // rows' blocks; staged offsets
  __shared__ int s_stg[2];  // 1: the rows' blocks of every window are staged in stg
  __shared__ __align__(16) int32_t s_rec[2][REC_W];  // fetched tile records
  __shared__ int s_row;
  __shared__ int s_wq[TILE_WARPS];  // per-warp survivor counters of the K8 scan (0 between scans)
  __shared__ uint4 s_ref[32];       // light rows: the running k-th best as a Ref (see make_ref)
  __shared__ int s_qn[32];          // light rows: survivors queued by the phase-A epilogue
  __shared__ unsigned s_light;      // rows whose running list is full (fused big-cluster tiles)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < TILE_WARPS) s_wq[tid] = 0;
  for (int i = tid; i < a.W + 1; i += TILE_T) M[i] = 0;
  uint32_t *kb = SMEM_CNT ? dyn : a.gscratch + (int64_t)blockIdx.x * K8Lay(a.smax, qcap).words;  // K8 region
  c2_cand *s_run = reinterpret_cast<c2_cand *>(dyn + a.rl_off);  // fused: the rows' running lists [32][k]
  uint4 *stg = reinterpret_cast<uint4 *>(dyn + a.stg_off);       // staged rows' blocks of the next tile
  const int nwin = a.nwin;
  const int kk = a.k;
  // one warp fetches the descriptors of tile item `it` into slot b
#if C2_BULK
  // next-tile descriptors in two halves: fetch_issue (one thread: claim the tile, bulk-copy its
  // record) right when K8 starts, fetch_finish (the first warp out of K8 rows: wait for the record,
  // parse it, bulk-copy the rows' packed blocks into the staging buffer) -- so no warp waits on a
  // global round trip while others still have rows.  Every use of a slot's mbarriers gets exactly
  // one arrival (0 bytes when there is no tile), so all threads can track the phases.
  __shared__ __align__(8) uint64_t mb_rec[2], mb_stg[2];
  __shared__ int s_claim;
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
      bulk_g2s(stg + (incl - bl * 32), a.packed + (int64_t)bo * 32, (uint32_t)bl * 512u, &mb_stg[b]);
  };
  if (tid == 0) fetch_issue(0);
  if (warp == 0) fetch_finish(0);
#else
  auto fetch = [&](int b) {
    int64_t it = 0;
    if (lane == 0) it = a.lo + atomicAdd(a.counter, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (lane == 0) s_it[b] = it;
    if (it >= a.hi) return;
    cp_async16(&s_rec[b][lane * 4], a.rec + it * REC_W + lane * 4);
    cp_async_wait_all();
    __syncwarp();
    const int32_t *rc = s_rec[b];
    if (lane == 0) {
      s_T[b] = Tile{rc[0], rc[1]};
      s_B[b] = BigC{rc[2], rc[3], rc[4], rc[5], rc[6], rc[7]};
    }
    s_ru2[b][lane] = rc[64 + lane];
    s_rp2[b][lane] = (uint32_t)rc[96 + lane];
    // the rows' packed blocks: copied to the staging buffer now (async), used by the build and
    // the probe of the tile's own slice
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
    if (lane == 0) s_stg[b] = staged ? 1 : 0;
    if (staged)
      for (int w = 0; w < nwin; ++w) {
        const int32_t n4 = __shfl_sync(0xffffffffu, bl, w) * 32;
        const int32_t so = __shfl_sync(0xffffffffu, incl - bl * 32, w);
        const uint4 *g = a.packed + (int64_t)__shfl_sync(0xffffffffu, bo, w) * 32;
        for (int i = lane; i < n4; i += 32) cp_async16(stg + so + i, g + i);
      }
  };
#endif
#if !C2_BULK
  if (warp == 0) fetch(0);
#endif
  int cur = 0;
  for (;;) {
#if C2_BULK
    mbar_wait(&mb_stg[cur], (ph_stg >> cur) & 1u);  // this tile's staged row blocks
    ph_rec ^= 1u << cur;  // (slot cur's record and staging phases were consumed)
    ph_stg ^= 1u << cur;
    if (tid == 0) s_claim = 0;
#else
    cp_async_wait_all();
#endif
    __syncthreads();
    const int64_t it = s_it[cur];
    if (it >= a.hi) break;
    long long ck0 = a.kstats ? clock64() : 0, ck_r1 = 0, ck_scan = 0, ckb = 0, ckp = 0;
    const Tile T = s_T[cur];
    const BigC B = s_B[cur];
    const int32_t *s_ru = s_ru2[cur];
    const uint32_t *s_rp = s_rp2[cur];
    const int s = B.s;
    const int nsl = (s + 31) >> 5;
    const int r0 = T.j * 32;
    const int nr = min(32, s - r0);
    const int32_t *vp = a.vperm + B.vp_off;
    const uint32_t W = a.relabel ? (uint32_t)B.kc : (uint32_t)a.W;
    const K8Lay lay(s, qcap);
    uint16_t *cnt = reinterpret_cast<uint16_t *>(kb);
    int32_t *s_vid = reinterpret_cast<int32_t *>(kb + lay.vid);
    uint32_t *s_vps = kb + lay.vps;
    Cand *s_q = reinterpret_cast<Cand *>(kb + lay.que);
    if (tid == 0) s_row = 0;
    if (tid < 32) s_qn[tid] = 0;
    // light rows: fused mode, big cluster (no slot groups), running list already full.  Their
    // candidates are filtered against the running k-th best right after the transpose, while
    // the counts are still in the thread that made them; K8 then skips their scan.
    const bool epi = C2_EPI && a.seed != nullptr && B.slot == 0;
    // the rows' running lists (fused mode): loaded now, first used in K8 after phase A
    if (a.seed)
      for (int r = warp; r < nr; r += TILE_WARPS) {
        const int32_t u = s_ru[r];
        if (u < 0) continue;
        for (int j = lane; j < kk; j += 32) cp_async8(s_run + r * kk + j, a.seed + (int64_t)u * kk + j);
      }
    // ================= phase A: counts |P_r ∩ P_v| for the 32 rows x all v of the cluster
    for (int g0 = 0; g0 < nsl; g0 += VPT * TILE_WARPS) {
      Counter<NHI> C[VPT];
#pragma unroll
      for (int q = 0; q < VPT; ++q) C[q].zero();
      for (int w = 0; w < nwin; ++w) {
        // ---- build M for window w from the tile's own slice (rows), lane r -> bit r (the first
        //      16-byte group of every thread is kept for the clear below)
        const bool stgd = s_stg[cur] != 0;
        const int32_t n4r = s_bl[cur][w] * 32;
        const uint4 *srcr = stgd ? stg + s_so[cur][w] : a.packed + (int64_t)s_bo[cur][w] * 32;
        const uint32_t pw = W | (W << 16);
        const uint4 padv = make_uint4(pw, pw, pw, pw);
        const uint4 dkeep = tid < n4r ? srcr[tid] : padv;
        for (int gi = tid; gi < n4r; gi += TILE_T) {
          const uint4 d = gi == tid ? dkeep : srcr[gi];
          const uint32_t bit = 1u << (gi & 31);
          const uint32_t xs[8] = {d.x & 0xFFFFu, d.x >> 16, d.y & 0xFFFFu, d.y >> 16,
                                  d.z & 0xFFFFu, d.z >> 16, d.w & 0xFFFFu, d.w >> 16};
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (xs[q] < W) atomicOr(&M[xs[q]], bit);
        }
        __syncthreads();
        if (a.kstats) ckb += clock64();
        // ---- probe: each warp streams VPT slices of v lists, two 16-byte loads per step with
        //      the next two steps in flight (odd tails padded with the sentinel item W, M[W] = 0)
        const long long ckpb = a.kstats ? clock64() : 0;
        int nsteps = 0;
#pragma unroll
        for (int q = 0; q < VPT; ++q) {
          const int jj = g0 + q * TILE_WARPS + ((C2_SNAKE && (q & 1)) ? TILE_WARPS - 1 - warp : warp);
          if (jj < nsl) {
            const int64_t bi = (int64_t)(B.sl_off + jj) * nwin + w;
            const bool own = stgd && jj == T.j;  // the tile's own slice: staged
            const int32_t len8 = own ? s_bl[cur][w] : a.blk_len8[bi];
            const uint4 *src = (own ? stg + s_so[cur][w] : a.packed + (int64_t)a.blk_off8[bi] * 32) + lane;
            auto ld = [&](int32_t p) { return p < len8 ? src[(int64_t)p * 32] : padv; };
            uint4 d0 = ld(0), d1 = ld(1), n0 = ld(2), n1 = ld(3);
            for (int32_t p8 = 0; p8 < len8; p8 += 2) {
              const uint4 f0 = ld(p8 + 4), f1 = ld(p8 + 5);
              uint32_t m[8];
              masks8(M, d0, m);
              uint32_t e8a = C[q].add8(m);
              masks8(M, d1, m);
              uint32_t e8b = C[q].add8(m);
              C[q].add16(e8a, e8b);
              d0 = n0;
              d1 = n1;
              n0 = f0;
              n1 = f1;
              ++nsteps;
            }
          }
        }
        if (a.kstats && lane == 0 && s > 1024) {  // probe busy time per step (big tiles)
          atomicAdd(&a.kstats[64], (unsigned long long)(clock64() - ckpb));
          atomicAdd(&a.kstats[65], (unsigned long long)nsteps);
        }
        if (epi && w == nwin - 1) cp_async_wait_all();  // the rows' running lists (issued at tile start)
        __syncthreads();
        if (a.kstats) ckp += clock64();
        // ---- clear M
        for (int gi = tid; gi < n4r; gi += TILE_T) {
          const uint4 d = gi == tid ? dkeep : srcr[gi];
          const uint32_t xs[8] = {d.x & 0xFFFFu, d.x >> 16, d.y & 0xFFFFu, d.y >> 16,
                                  d.z & 0xFFFFu, d.z >> 16, d.w & 0xFFFFu, d.w >> 16};
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (xs[q] < W) M[xs[q]] = 0;
        }
        if (epi && w == nwin - 1 && warp == TILE_WARPS - 1) {
          const int r = lane;
          const bool light = r < nr && s_ru[r] >= 0 && s_run[r * kk + kk - 1].id >= 0;
          if (light) {
            const Ref R = make_ref(from_out(s_run[r * kk + kk - 1]), s_rp[r], false);
            s_ref[r] = make_uint4(R.A, R.B, R.iT, R.idlim);
          }
          const unsigned lm = __ballot_sync(0xffffffffu, light);
          if (lane == 0) s_light = lm;
        }
        __syncthreads();
      }
      // ---- planes -> 32 counts per v (transpose) -> cnt[r][v] (M is dead from here on when
      //      SMEM_CNT: the host guarantees a single g0 group then)
#pragma unroll
      for (int q = 0; q < VPT; ++q) {
        const int jj = g0 + q * TILE_WARPS + ((C2_SNAKE && (q & 1)) ? TILE_WARPS - 1 - warp : warp);
        const int vi = jj * 32 + lane;
        if (jj < nsl) {
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
#pragma unroll
          for (int r = 0; r < 32; ++r)
            if (r < nr) cnt[r * lay.RS + vi] = (uint16_t)A[r];
          if (epi) {
            // light rows: candidate (v, i, |P_v|) survives iff strictly better than the row's
            // running k-th best (passes() with idlim = id_T), i.e. it would enter the list
            const unsigned lm = s_light;
            if (lm && vi < s) {
              const int32_t idv = vp[vi];
              const uint32_t psv = (uint32_t)a.vsize[B.vp_off + vi];
              for (unsigned q2 = lm; q2; q2 &= q2 - 1) {
                const int r = __ffs(q2) - 1;
                const uint32_t i = cnt[r * lay.RS + vi];
                const uint4 R = s_ref[r];
                const uint32_t l = i * R.x, rr = R.z * psv + R.y;
                if (l >= rr && (l > rr || (uint32_t)idv < R.w) && vi != r0 + r) {
                  const int p = atomicAdd(&s_qn[r], 1);
                  if (p < qcap) s_q[r * qcap + p] = Cand{i | ((s_rp[r] + psv - i) << 16), idv};
                }
              }
            }
          }
        }
      }
    }
    const long long ck1 = a.kstats ? clock64() : 0;
    // member ids and sizes (positions s .. s4-1: never-passing pads)
    {
      const int s4 = (s + 3) & ~3;
      for (int i = tid; i < s4; i += TILE_T) {
        s_vid[i] = i < s ? vp[i] : INT32_MAX;
        s_vps[i] = i < s ? (uint32_t)a.vsize[B.vp_off + i] : 0u;
      }
    }
    cp_async_wait_all();  // the running lists
    __syncthreads();
    // ================= K8: exact top-k per row, one warp per row (no CTA barrier inside)
#if C2_BULK
    if (tid == 0) fetch_issue(cur ^ 1);  // next tile's record: claimed and requested now
#else
    if (warp == 0) fetch(cur ^ 1);  // next tile's descriptors, hidden behind this K8
#endif
    const int slot = B.slot;  // mixed slice: candidates only inside the row's own slot group
    uint32_t *zq = nullptr;  // queue words the warp's previous row wrote (re-zeroed: M alias)
    int zn = 0;
    long long tfin = 0, acc_sel = 0, acc_fin = 0, nrow_b = 0;  // kstats: big tiles' per-row split
    // rows are taken dynamically, the expensive ones first: rows without a full running list
    // (round 1 in big clusters), then the others
    const unsigned heavy = __ballot_sync(0xffffffffu, lane < nr && s_ru[lane] >= 0 &&
                                                          !(a.seed && s_run[lane * kk + kk - 1].id >= 0));
    const int nheavy = __popc(heavy);
    for (;;) {
      if (a.kstats && tfin) {
        acc_fin += clock64() - tfin;
        tfin = 0;
      }
      for (int i = lane; i < zn; i += 32) zq[i] = 0u;
      zn = 0;
      int idx = 0;
      if (lane == 0) idx = atomicAdd(&s_row, 1);
      idx = __shfl_sync(0xffffffffu, idx, 0);
      if (idx >= nr) {
#if C2_BULK
        int claim = 0;
        if (lane == 0) claim = atomicExch(&s_claim, 1);
        if (__shfl_sync(0xffffffffu, claim, 0) == 0) fetch_finish(cur ^ 1);  // first warp out of rows
#endif
        break;
      }
      const int r = idx < nheavy ? (int)__fns(heavy, 0, idx + 1) : (int)__fns(~heavy, 0, idx - nheavy + 1);
      const int32_t u = s_ru[r];
      if (u < 0) continue;
      const uint32_t prr = s_rp[r];
      const int selfr = slot ? r : r0 + r;
      const uint16_t *cr = cnt + r * lay.RS;
      Cand *qr = s_q + r * qcap;
      const Cand tau = a.seed ? from_out(s_run[r * kk + kk - 1]) : sent();
      // survivors of T (strictly better than tau, not worse than a round-1 bound) -> qr by
      // ballot compaction; returns their number (only the first qcap are stored)
      auto scan = [&](const Ref &T) -> int {
        int m = 0;
        if (slot) {
          const int lo = r & ~(slot - 1);
          const int vi = lo + lane;
          bool ok = false;
          Cand x = sent();
          if (lane < slot && vi != selfr) {
            const uint32_t i = cr[vi], ps = s_vps[vi];
            const int32_t id = s_vid[vi];
            ok = passes(i, ps, id, T);
            x = Cand{i | ((prr + ps - i) << 16), id};
          }
          const unsigned bal = __ballot_sync(0xffffffffu, ok);
          if (ok) qr[__popc(bal & ((1u << lane) - 1))] = x;
          return __popc(bal);
        }
        for (int base = 0; base < s; base += 128) {
          const int v4 = base + lane * 4;
          uint32_t iv[4] = {0, 0, 0, 0}, pv[4] = {0, 0, 0, 0};
          int32_t dv[4] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MAX};
          if (v4 < s) {
            const uint2 c = *reinterpret_cast<const uint2 *>(cr + v4);
            const uint4 ps = *reinterpret_cast<const uint4 *>(s_vps + v4);
            const int4 id = *reinterpret_cast<const int4 *>(s_vid + v4);
            iv[0] = c.x & 0xFFFFu, iv[1] = c.x >> 16, iv[2] = c.y & 0xFFFFu, iv[3] = c.y >> 16;
            pv[0] = ps.x, pv[1] = ps.y, pv[2] = ps.z, pv[3] = ps.w;
            dv[0] = id.x, dv[1] = id.y, dv[2] = id.z, dv[3] = id.w;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            // survivors are few: a shared counter bumped by the passing lanes only (queue order
            // is irrelevant, the survivors are sorted by the exact key afterwards)
            if (v4 + e != selfr && passes(iv[e], pv[e], dv[e], T)) {
              const int p = atomicAdd(&s_wq[warp], 1);
              if (p < qcap) qr[p] = Cand{iv[e] | ((prr + pv[e] - iv[e]) << 16), dv[e]};
            }
          }
        }
        __syncwarp();
        m = s_wq[warp];
        __syncwarp();
        if (lane == 0) s_wq[warp] = 0;
        __syncwarp();
        return m;
      };
      // k-th best of the first 64*KS queue entries (all distinct real candidates): a valid
      // lower bound of the row's k-th best
      auto kth_of_queue = [&]() -> Ref {
        if (a.kstats && lane == 0) atomicAdd(&a.kstats[15], 1ull);
        KC e[2 * KS];
#pragma unroll
        for (int j = 0; j < 2 * KS; ++j) e[j] = to_kc(qr[32 * j + lane]);
        sort_kc<2 * KS>(e);
        return make_ref(kc_cand(warp_get<2 * KS>(e, kk - 1)), prr, true);
      };
      long long ckr = a.kstats ? clock64() : 0;
      const long long ckr0 = ckr;
      // round 1: every lane's best R1 candidates of its share; T_r = the k-th best of the
      // 32*R1 tops (any k distinct candidates bound the row's k-th best from below)
      auto round1 = [&](Ref &T) {
        Cand t[R1];
#pragma unroll
        for (int j = 0; j < R1; ++j) t[j] = sent();
        Ref wr = make_ref(sent(), prr, false);
        for (int v4 = lane * 4; v4 < s; v4 += 128) {
          const uint2 c = *reinterpret_cast<const uint2 *>(cr + v4);
          const uint4 ps = *reinterpret_cast<const uint4 *>(s_vps + v4);
          const int4 id = *reinterpret_cast<const int4 *>(s_vid + v4);
          const uint32_t iv[4] = {c.x & 0xFFFFu, c.x >> 16, c.y & 0xFFFFu, c.y >> 16};
          const uint32_t pv[4] = {ps.x, ps.y, ps.z, ps.w};
          const int32_t dv[4] = {id.x, id.y, id.z, id.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (v4 + e != selfr && passes(iv[e], pv[e], dv[e], wr)) {
              Cand x{iv[e] | ((prr + pv[e] - iv[e]) << 16), dv[e]};
#pragma unroll
              for (int j = R1 - 1; j > 0; --j) {
                if (better_c(x, t[j - 1])) t[j] = t[j - 1];
                else if (better_c(x, t[j])) t[j] = x;
              }
              if (better_c(x, t[0])) t[0] = x;
              wr = make_ref(t[R1 - 1], prr, false);
            }
          }
        }
        KC e[R1];
#pragma unroll
        for (int j = 0; j < R1; ++j) e[j] = to_kc(t[j]);
        sort_kc<R1>(e);
        const KC Tr = warp_get<R1>(e, kk - 1);
        if (kc_real(Tr) && better_c(kc_cand(Tr), tau)) T = make_ref(kc_cand(Tr), prr, true);
      };
      Ref T = make_ref(tau, prr, false);
      // rows without a running list yet (tau = sentinel) whose candidates cannot all be queued
      // start with round 1; rows whose tau lets too many through get it after the first scan
      bool r1 = !slot && !is_real(tau) && s - 1 > 64 * KS;
      if (r1) round1(T);
      if (a.kstats) {
        const long long c = clock64();
        ck_r1 += c - ckr;
        ckr = c;
      }
      const bool light = epi && ((s_light >> r) & 1u);
      int m = light ? s_qn[r] : 0;
      if (!light || m > qcap) m = scan(T);  // (a light row whose queue overflowed rescans)
      zq = reinterpret_cast<uint32_t *>(qr);
      zn = 2 * min(m, qcap);
      if (a.kstats && lane == 0) atomicAdd(&a.kstats[16 + min(m, 300) / 20], 1ull);
      if (m > 64 * KS && !slot && !r1) {
        if (a.kstats && lane == 0) atomicAdd(&a.kstats[14], 1ull);
        r1 = true;
        round1(T);
        m = scan(T);
        zn = max(zn, 2 * min(m, qcap));
      }
      int rescans = 0;
      for (; rescans < 2 && m > qcap; ++rescans) {
        T = kth_of_queue();
        __syncwarp();
        m = scan(T);
        zn = max(zn, 2 * min(m, qcap));
      }
      // shrink a long queue in place: keep the entries not worse than the k-th best of its
      // first 64*KS (stops when that makes no progress: massive ties)
      while (m > 64 * KS && m <= qcap) {
        const Ref T2 = kth_of_queue();
        __syncwarp();
        int w = 0;
        for (int b0 = 0; b0 < m; b0 += 32) {
          const int j = b0 + lane;
          Cand x = j < m ? qr[j] : sent();
          const uint32_t i = x.iu & 0xFFFFu, ps = (x.iu >> 16) + i - prr;
          const bool ok = j < m && passes(i, ps, x.id, T2);
          __syncwarp();
          const unsigned bal = __ballot_sync(0xffffffffu, ok);
          if (ok) qr[w + __popc(bal & ((1u << lane) - 1))] = x;
          w += __popc(bal);
        }
        __syncwarp();
        if (w == m) break;
        m = w;
      }
      if (a.kstats) {
        const long long c = clock64();
        ck_scan += c - ckr;
        if (s > 1024) {
          acc_sel += c - ckr0;
          tfin = c;
          ++nrow_b;
        }
      }
      if (a.kstats) {  // pair evaluations of this row: its cluster-mates (debug work accounting)
        int ev = s - 1;
        if (slot) {
          const int lo = r & ~(slot - 1);
          ev = __popc(__ballot_sync(0xffffffffu, lane < slot && s_vid[lo + lane] >= 0)) - 1;
        }
        if (lane == 0) atomicAdd(&a.kstats[70], (unsigned long long)ev);
      }
      if (a.kstats && lane == 0) {
        atomicAdd(&a.kstats[0], 1ull);
        atomicAdd(&a.kstats[1], m == 0 ? 1ull : 0ull);
        atomicAdd(&a.kstats[2], (unsigned long long)m);
        atomicAdd(&a.kstats[3], m > 32 * KS ? 1ull : 0ull);
        atomicAdd(&a.kstats[4], (unsigned long long)rescans);
        atomicAdd(&a.kstats[6], r1 ? 1ull : 0ull);
        if (r == 0) {
          atomicAdd(&a.kstats[5], 1ull);
          atomicAdd(&a.kstats[7], (unsigned long long)s);
        }
      }
      if (a.seed && m == 0) continue;
      c2_cand *dst = a.seed ? a.out + (int64_t)u * kk : a.out + ((int64_t)B.f * a.n + u) * kk;
      if (C2_RANKMERGE && a.seed && m <= 32) {
        // few survivors: Alg. 3 step by ranks (no sorting network, no f64 keys)
        rank_merge<KS>(qr, m, s_run + r * kk, kk, dst);
        continue;
      }
      if (!C2_RANKMERGE && a.seed && m <= 16) {
        // few survivors (one insertion ~20 instructions, sort-32 + merge-64 ~320): insert them one
        // by one into the running list (duplicates skipped)
        KC S[KS];
#pragma unroll
        for (int j = 0; j < KS; ++j) S[j] = to_kc((32 * j + lane < kk) ? from_out(s_run[r * kk + 32 * j + lane]) : sent());
        const KC xk = to_kc(lane < m ? qr[lane] : sent());  // all survivors' keys at once
        for (int j = 0; j < m; ++j) {
          const KC x = shfl_e(xk, j);
          bool dup = false;
#pragma unroll
          for (int jj = 0; jj < KS; ++jj) dup |= S[jj].k == x.k;
          if (__any_sync(0xffffffffu, dup)) continue;
          warp_insert<KS>(S, x);
        }
#pragma unroll
        for (int j = 0; j < KS; ++j)
          if (32 * j + lane < kk) dst[32 * j + lane] = kc_out(S[j]);
        continue;
      }
      KC L[KS];  // top-k of this function's survivors (sentinel padded)
      if (m <= 32 * KS) {
        KC q[KS];
#pragma unroll
        for (int j = 0; j < KS; ++j) q[j] = to_kc((32 * j + lane < m) ? qr[32 * j + lane] : sent());
        sort_kc<KS>(q);
#pragma unroll
        for (int j = 0; j < KS; ++j) L[j] = q[j];
      } else if (m <= 64 * KS) {
        KC q[2 * KS];
#pragma unroll
        for (int j = 0; j < 2 * KS; ++j) q[j] = to_kc((32 * j + lane < m) ? qr[32 * j + lane] : sent());
        sort_kc<2 * KS>(q);
#pragma unroll
        for (int j = 0; j < KS; ++j) L[j] = q[j];
      } else {
        // pathological ties: exact insertion over the row's candidates
        if (a.kstats && lane == 0) atomicAdd(&a.kstats[8], 1ull);
        Cand Lc[KS];
#pragma unroll
        for (int j = 0; j < KS; ++j) Lc[j] = sent();
        Cand thr = sent();
        for (int vb = 0; vb < s; vb += 32) {
          const int vi = vb + lane;
          Cand c = sent();
          if (vi < s) {
            int32_t v = s_vid[vi];
            if (v >= 0 && vi != selfr && (slot == 0 || (vi ^ r) < slot)) {
              uint32_t ci = cr[vi];
              c = Cand{ci | ((prr + s_vps[vi] - ci) << 16), v};
            }
          }
          bool bt = is_real(c) && better_c(c, tau) && better_c(c, thr);
          unsigned mask = __ballot_sync(0xffffffffu, bt);
          while (mask) {
            int l = __ffs(mask) - 1;
            mask &= mask - 1;
            Cand x = shfl_c(c, l);
            if (!better_c(x, thr)) continue;
            warp_insert<KS>(Lc, x);
            thr = warp_get<KS>(Lc, kk - 1);
          }
        }
#pragma unroll
        for (int j = 0; j < KS; ++j) L[j] = to_kc(Lc[j]);
      }
      if (!a.seed) {
#pragma unroll
        for (int j = 0; j < KS; ++j)
          if (32 * j + lane < kk) dst[32 * j + lane] = kc_out(L[j]);
        continue;
      }
      // merge with the running list S (best first): bitonic sequence L(first k) ++ reverse(S)
      KC S[KS];
#pragma unroll
      for (int j = 0; j < KS; ++j) S[j] = to_kc((32 * j + lane < kk) ? from_out(s_run[r * kk + 32 * j + lane]) : sent());
      KC mm[2 * KS];
#pragma unroll
      for (int j = 0; j < KS; ++j) mm[j] = (32 * j + lane < kk) ? L[j] : KC{0ull, 1u << 16};
#pragma unroll
      for (int j = 0; j < KS; ++j) mm[KS + j] = shfl_e(S[KS - 1 - j], 31 - lane);
      merge_kc<2 * KS>(mm);
      // drop adjacent duplicates (a repeated id carries identical values, A16); keep k
      int base = 0;
#pragma unroll
      for (int j = 0; j < 2 * KS; ++j) {
        const uint32_t lo = (uint32_t)mm[j].k;
        uint32_t prev = __shfl_up_sync(0xffffffffu, lo, 1);
        uint32_t prevj = j > 0 ? __shfl_sync(0xffffffffu, (uint32_t)mm[j - 1].k, 31) : 0u;
        if (lane == 0) prev = prevj;
        bool keep = kc_real(mm[j]) && (j + lane == 0 || lo != prev);
        unsigned bal = __ballot_sync(0xffffffffu, keep);
        int rank = base + __popc(bal & ((1u << lane) - 1));
        if (keep && rank < kk) dst[rank] = kc_out(mm[j]);
        base += __popc(bal);
      }
      for (int p = base + lane; p < kk; p += 32) dst[p] = c2_cand{-1, 0, 0};
    }
    const long long ck2 = a.kstats ? clock64() : 0;
    __syncthreads();
    if (a.kstats && lane == 0) {
      const long long ck3 = clock64();
      atomicAdd(&a.kstats[9], (unsigned long long)(ck1 - ck0));    // phase A (+ tile head)
      atomicAdd(&a.kstats[10], (unsigned long long)ck_r1);         // K8 round 1
      atomicAdd(&a.kstats[11], (unsigned long long)ck_scan);       // K8 scan + queue shrink
      atomicAdd(&a.kstats[12], (unsigned long long)(ck2 - ck1 - ck_r1 - ck_scan));  // K8 rest
      atomicAdd(&a.kstats[13], (unsigned long long)(ck3 - ck2));   // wait at the K8 barrier
      if (warp == 0) {  // tile wall cycles by cluster size class: mixed, 33-256, 257-1024, >1024
        const int cls = B.slot ? 0 : s <= 256 ? 1 : s <= 1024 ? 2 : 3;
        atomicAdd(&a.kstats[32 + cls], (unsigned long long)(ck3 - ck0));
        atomicAdd(&a.kstats[36 + cls], 1ull);
        if (nrow_b) {
          atomicAdd(&a.kstats[60], (unsigned long long)acc_sel);
          atomicAdd(&a.kstats[61], (unsigned long long)acc_fin);
          atomicAdd(&a.kstats[62], (unsigned long long)nrow_b);
        }
        {  // per class: build (window sum) / probe / rest of phase A / K8 / wait
          unsigned long long *kc5 = a.kstats + 40 + 5 * cls;
          atomicAdd(&kc5[0], (unsigned long long)(ckb - ck0 * nwin));
          atomicAdd(&kc5[1], (unsigned long long)(ckp - ckb));
          atomicAdd(&kc5[2], (unsigned long long)(ck1 - ck0) - (unsigned long long)(ckp - ckb));
          atomicAdd(&kc5[3], (unsigned long long)(ck2 - ck1));
          atomicAdd(&kc5[4], (unsigned long long)(ck3 - ck2));
        }
      }
    }
    // restore the all-zero M words the K8 region overwrote
    // (queues were re-zeroed row by row; here the counts and member arrays)
    if (SMEM_CNT) {
      const int dw = min(lay.que, a.W + 1);
      uint4 *z = reinterpret_cast<uint4 *>(dyn);
      for (int i = tid; i < dw / 4; i += TILE_T) z[i] = make_uint4(0, 0, 0, 0);
      for (int i = (dw & ~3) + tid; i < dw; i += TILE_T) dyn[i] = 0;
    }
    cur ^= 1;
  }
}

typedef void (*TileKernel)(TileArgs);

template <int NHI, int VPT, bool SM>
static TileKernel pick_ks(int k) {
  return k <= 32 ? k_local_tile<NHI, VPT, 1, SM> : k_local_tile<NHI, VPT, 2, SM>;
}
template <int NHI, bool SM>
static TileKernel pick_vpt(int vpt, int k) {
  return vpt <= 1 ? pick_ks<NHI, 1, SM>(k) : vpt <= 2 ? pick_ks<NHI, 2, SM>(k) : pick_ks<NHI, 4, SM>(k);
}
template <bool SM>
static TileKernel pick_nhi(int nhi, int vpt, int k) {
  return nhi <= 4 ? pick_vpt<4, SM>(vpt, k) : nhi <= 8 ? pick_vpt<8, SM>(vpt, k) : pick_vpt<11, SM>(vpt, k);
}
static TileKernel pick_tile(int nhi, int vpt, int k, bool smem_cnt) {
  return smem_cnt ? pick_nhi<true>(nhi, vpt, k) : pick_nhi<false>(nhi, vpt, k);
}

__global__ void k_init_pads(c2_cand *__restrict__ R, int64_t E) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < E) R[e] = c2_cand{-1, 0, 0};
}

// sum over unordered pairs of (|P_u| + |P_v|) = sum over (f,u) of (s_c - 1) * |P_u|
__global__ void k_work_steps(const int32_t *__restrict__ offsets, const int32_t *__restrict__ cof,
                             const int32_t *__restrict__ psize, int64_t TN, int32_t n,
                             unsigned long long *__restrict__ acc) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long w = 0;
  if (q < TN) {
    int64_t f = q / n;
    int32_t u = (int32_t)(q % n);
    int32_t c = cof[q];
    const int32_t *off = offsets + f * (n + 1);
    w = (unsigned long long)(off[c + 1] - off[c] - 1) * (unsigned long long)psize[u];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
  if ((threadIdx.x & 31) == 0 && w) atomicAdd(acc, w);
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
  k_wl_classify<<<nblk(C), 256, 0, st>>>(cl.offsets, ccum, t, n, C, key, val, maxs, sized, cnt_fc, hyrec_min);
  C2_LAUNCHED(ctx, "k_wl_classify");
  C2_TRY(radix_sort_pairs(ctx, key, val, skey, sval, C, 32));
  unsigned long long *wacc = (unsigned long long *)ws_get(ctx, "work_acc", 16, &rc);
  if (rc) return rc;
  C2_CUDA(ctx, cudaMemsetAsync(wacc, 0, 8, st));
  k_work_steps<<<nblk((int64_t)t * n), 256, 0, st>>>(cl.offsets, cl.cluster_of, csr.psize, (int64_t)t * n, n, wacc);
  C2_LAUNCHED(ctx, "k_work_steps");
  int32_t hfc[WLC * C2_MAX_T];
  unsigned long long hwork = 0;
  C2_CUDA(ctx, cudaMemcpyAsync(hfc, cnt_fc, 4 * WLC * t, cudaMemcpyDeviceToHost, st));
  C2_CUDA(ctx, cudaMemcpyAsync(&hwork, wacc, 8, cudaMemcpyDeviceToHost, st));
  C2_TRY(stream_sync(ctx, "worklist counts"));
  ctx->stats.work_steps = (int64_t)hwork;
  int64_t nbig = 0, nsmall = 0, nsingle = 0, nbigtiles = 0, nhyrec = 0;
  int32_t hy_lo[C2_MAX_T + 1];
  for (int f = 0; f < t; ++f) {
    hy_lo[f] = (int32_t)nhyrec;
    nhyrec += hfc[f * WLC + 8];
    nbig += hfc[f * WLC + 7];
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
      int32_t h1;
      C2_CUDA(ctx, cudaMemcpyAsync(&h1, vp_scan + nbig, 4, cudaMemcpyDeviceToHost, st));
      C2_TRY(stream_sync(ctx, "big cluster sizes"));
      nv_big = h1;
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
      packed = (uint4 *)ws_get(ctx, "packed", (size_t)tot8 * 32 * 16 + 16, &rc);
      if (rc) return rc;
      int *rl = (int *)ws_get(ctx, "relabel_ctr", 16, &rc);
      if (rc) return rc;
      C2_CUDA(ctx, cudaMemsetAsync(rl, 0, 16, st));
      C2_CUDA(ctx, cudaFuncSetAttribute(k_relabel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rl_smem));
      int rl_occ = 1;
      C2_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rl_occ, k_relabel, RL_T, rl_smem));
      k_relabel<<<ctx->num_sms * std::max(rl_occ, 1), RL_T, rl_smem, st>>>(bcs, ncl, vperm, csr.offs, csr.items, nwq, blk_off8, blk_len8,
                                                     reinterpret_cast<uint16_t *>(packed), rl, rl + 1);
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
      k_sl_len<<<nblk(nslices * 32), 256, 0, st>>>(tiles, nslices, bcs, vperm, csr.offs, csr.items, W, nwin,
                                                   blk_len8, bounds);
      C2_LAUNCHED(ctx, "k_sl_len");
      C2_TRY(scan_exclusive(ctx, blk_len8, blk_off8, nb));
      int32_t tot8;
      C2_CUDA(ctx, cudaMemcpyAsync(&tot8, blk_off8 + nb, 4, cudaMemcpyDeviceToHost, st));
      C2_TRY(stream_sync(ctx, "packed size"));
      packed = (uint4 *)ws_get(ctx, "packed", (size_t)tot8 * 32 * 16 + 16, &rc);
      if (rc) return rc;
      // bank-rotated order pays for its second pass only when lists are long (one window)
      k_sl_fill<<<nblk(nslices * 32 * 32), 256, 0, st>>>(nslices, bounds, csr.items, W, nwin, blk_len8, blk_off8,
                                                         reinterpret_cast<uint16_t *>(packed), nwin == 1 ? 1 : 0);
      C2_LAUNCHED(ctx, "k_sl_fill");
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

  // ---- tile kernel configuration
  TileKernel tk = nullptr;
  int grid = 0;
  int qcap = 64;
  int32_t rl_off = 0, stg_off = 0, stg_cap = 0;
  size_t smem = 0;
  uint32_t *gscratch = nullptr;
  int *counters = nullptr;
  const int32_t smax = (int32_t)std::max<uint32_t>(maxs, 32);
  if (nslices > 0) {
    int nbits = bits_for((int64_t)csr.max_len + 1);
    int nhi = std::max(nbits - 4, 1);
    int max_sl = (int)((maxs + 31) / 32);
    int vpt = max_sl <= TILE_WARPS ? 1 : max_sl <= 2 * TILE_WARPS ? 2 : 4;
    // survivor queue per row: 256 entries where shared memory allows, at least 64*KS
    const int qmin = k <= 32 ? 64 : 128;
    qcap = 256;
    const size_t budget = (C2_SMEM_BUDGET ? std::min<size_t>(C2_SMEM_BUDGET, ctx->smem_optin) : ctx->smem_optin) -
                          4096;  // minus the kernel's static shared memory (~2.1 KB)
    const size_t rlw = fused ? (size_t)64 * k : 0;  // the rows' running lists (Cand = 2 words)
    const size_t stgw = 4096;  // staging of the next tile's row blocks: at least 16 KB
    while (qcap > qmin && ((size_t)K8Lay(smax, qcap).words + rlw + stgw) * 4 > budget) qcap -= 64;
    const int k8w = K8Lay(smax, qcap).words;
    const size_t mw = (size_t)((W + 4) & ~3);
    // counts in shared memory (aliased onto M) when one g0 group covers the largest cluster
    // and the K8 region fits; else a per-CTA global scratch region
    const bool smem_cnt = max_sl <= 4 * TILE_WARPS && ((size_t)k8w + rlw) * 4 <= budget;
    rl_off = (int32_t)(((smem_cnt ? std::max(mw, (size_t)k8w) : mw) + 3) & ~(size_t)3);
    stg_off = (int32_t)(((size_t)rl_off + rlw + 3) & ~(size_t)3);
    stg_cap = (int32_t)std::min<int64_t>(4096, ((int64_t)budget / 4 - stg_off) / 4);  // 16-byte groups
    if (stg_cap < 64) stg_cap = 0;
    smem = ((size_t)stg_off + (size_t)stg_cap * 4) * 4;
    tk = pick_tile(nhi, vpt, k, smem_cnt);
    C2_CUDA(ctx, cudaFuncSetAttribute(tk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    C2_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tk, TILE_T, smem));
    occ = std::max(occ, 1);
    grid = (int)std::min<int64_t>((int64_t)ctx->num_sms * occ, nslices);
    if (!smem_cnt) {
      gscratch = (uint32_t *)ws_get(ctx, "tile_scratch", (size_t)grid * k8w * 4, &rc);
      if (rc) return rc;
    }
    counters = (int *)ws_get(ctx, "tile_counter", 4 * (2 * C2_MAX_T + 2), &rc);
    if (rc) return rc;
    C2_CUDA(ctx, cudaMemsetAsync(counters, 0, 4 * (2 * C2_MAX_T + 2), st));
  }
  auto launch_tiles = [&](int64_t lo, int64_t hi, int ci, const c2_cand *seed, c2_cand *dst) -> int {
    if (hi <= lo) return C2_OK;
    TileArgs ta{tiles, lo, hi, counters + ci, bcs, vperm, vsize, trec, blk_len8, blk_off8, packed, csr.psize, n, W, nwin, k,
                seed, dst, ctx->kstats, gscratch, smax, qcap, rl_off, stg_off, stg_cap, relabel ? 1 : 0};
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
    return C2_OK;
  };
  auto launch_singles = [&](int64_t lo, int64_t hi, const c2_cand *seed, c2_cand *dst) -> int {
    if (hi <= lo) return C2_OK;
    k_singles<<<nblk((hi - lo) * k), 256, 0, st>>>(sval + nbig + nsmall, nsingle, cl.offsets, ccum, t, n, cl.members,
                                                   k, lo, hi, seed, dst);
    C2_LAUNCHED(ctx, "k_singles");
    return C2_OK;
  };
  if (!fused) {
    C2_TRY(launch_tiles(0, nslices, 0, nullptr, out));
    C2_TRY(launch_singles(0, nsingle, nullptr, out));
    if (result) *result = out;
  } else {
    // Alg. 3 order: function by function, every user's running list is merged in place with
    // its neighbourhood in that function's cluster (singletons: nothing to merge)
    int64_t blo = 0;
    for (int f = 0; f < t; ++f) {
      int64_t bhi = blo + hfc[f * WLC + 0];
      C2_TRY(launch_tiles(blo, bhi, 2 * f, out, out));
      C2_TRY(launch_tiles(nbigtiles + mix_lo[f], nbigtiles + mix_lo[f + 1], 2 * f + 1, out, out));
      blo = bhi;
    }
    if (result) *result = out;
  }
  return C2_OK;
}

}  // namespace c2
