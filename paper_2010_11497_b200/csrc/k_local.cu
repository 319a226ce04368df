// k_local.cu -- Step 2 of C^2 on the GPU: brute-force Jaccard top-k inside every cluster
// (Alg. 2, brute-force branch; s(s-1)/2 similarities per cluster).
//
// K5 worklist.  Clusters of <= 32 users go to k_local_small (one warp per cluster, all
//    unordered pairs by two-pointer merge, exact rank selection).  Larger ("big") clusters
//    are ordered by function, then by size (largest first: the paper's decreasing priority
//    queue), cut into 32-user slices, and repacked once per call:
//      vperm   members of the cluster sorted by |P_v| (descending), so the 32 lists of a
//              slice have similar lengths;
//      packed  for every (slice, item window) a block of u16 window-local item ids laid out
//              [p/8][lane][8] and padded to the slice's longest list with W (M[W] == 0).
//    A warp then streams the 32 lists of a slice with one 16-byte coalesced load per lane per
//    8 items, with no divergence and no bounds checks.
// K7 k_local_tile: persistent CTAs, one work item = one slice R (32 rows) of cluster C.  For
//    every item window, shared memory holds the transposed membership mask M[x] = {r in R :
//    x in P_r} (bit r).  Each thread owns VPT slices' lanes (one v each) and accumulates the
//    32 counts |P_r ∩ P_v| bit-sliced with Harley-Seal carry-save adders over 16 masks, so
//    one LDS + ~3 LOP3 serve 32 pairs.  A 32x32 bit transpose turns the planes into counts.
// K8 (in K7): per row, a warp keeps the k best candidates under the exact order
//    (i1*U2 > i2*U1, ties by lower id) as a warp-distributed sorted list.  In fused mode
//    (c2_build) the list is seeded with the running Alg. 3 result of the earlier functions,
//    so only candidates that can still enter the final k-NN are inserted (exact: the k-th
//    best never decreases), and the result is written back in place of a per-function list.
#include <algorithm>
#include <vector>

#include "c2_internal.cuh"

namespace c2 {

struct SmallItem {
  int32_t f, start, s;
};
struct BigC {
  int32_t f, start, s, vp_off, sl_off;
};
struct Tile {
  int32_t bc, j;
};

constexpr int TILE_T = 512;
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

__global__ void k_wl_classify(const int32_t *__restrict__ offsets, const int32_t *__restrict__ ccum, int t,
                              int32_t n, int64_t C, int32_t *__restrict__ fsmall, uint32_t *__restrict__ key,
                              uint32_t *__restrict__ val, uint32_t maxs, int sized) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= C) return;
  int f = find_f(ccum, t, g);
  int64_t c = g - ccum[f];
  const int32_t *off = offsets + (int64_t)f * (n + 1);
  uint32_t s = (uint32_t)(off[c + 1] - off[c]);
  bool big = s > 32;
  fsmall[g] = !big;
  // big clusters first, by function, then size descending; small ones after all of them
  key[g] = big ? (uint32_t)f * (sized ? (maxs + 1) : 1u) + (sized ? (maxs - s) : 0u) : 0xFFFFFFFFu;
  val[g] = (uint32_t)g;
}

__global__ void k_wl_small(const int32_t *__restrict__ offsets, const int32_t *__restrict__ ccum, int t, int32_t n,
                           int64_t C, const int32_t *__restrict__ fsmall, const int32_t *__restrict__ sscan,
                           SmallItem *__restrict__ out) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= C || !fsmall[g]) return;
  int f = find_f(ccum, t, g);
  int64_t c = g - ccum[f];
  const int32_t *off = offsets + (int64_t)f * (n + 1);
  out[sscan[g]] = SmallItem{f, off[c], off[c + 1] - off[c]};
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
                          int32_t *__restrict__ per_f) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nbig) return;
  int64_t g = sval[i];
  int f = find_f(ccum, t, g);
  int64_t c = g - ccum[f];
  const int32_t *off = offsets + (int64_t)f * (n + 1);
  int32_t s = off[c + 1] - off[c];
  BigC b{f, off[c], s, vp_scan[i], sl_scan[i]};
  bcs[i] = b;
  int ns = (s + 31) / 32;
  for (int j = 0; j < ns; ++j) tiles[b.sl_off + j] = Tile{(int32_t)i, j};
  atomicAdd(&per_f[f], ns);
}

// vperm: members of each big cluster sorted by |P_v| descending (ties by position).  One CTA
// per cluster, bitonic sort in shared memory for s <= 2048 (larger clusters keep the
// canonical order: performance only, results do not depend on it).
__global__ void __launch_bounds__(1024) k_sl_sort(const BigC *__restrict__ bcs, const int32_t *__restrict__ members,
                                                  int32_t n, const int32_t *__restrict__ psize,
                                                  int32_t *__restrict__ vperm) {
  __shared__ uint32_t key[2048];
  const BigC b = bcs[blockIdx.x];
  const int32_t *mem = members + (int64_t)b.f * n + b.start;
  int32_t *out = vperm + b.vp_off;
  if (b.s > 2048) {
    for (int i = threadIdx.x; i < b.s; i += blockDim.x) out[i] = mem[i];
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
  for (int i = threadIdx.x; i < b.s; i += blockDim.x) out[i] = mem[key[i] & 0xFFFF];
}

// blk_len8[slice][w] = ceil(max over the slice's 32 lists of |list ∩ window w| / 8)
__global__ void k_sl_len(const Tile *__restrict__ tiles, int64_t nslices, const BigC *__restrict__ bcs,
                         const int32_t *__restrict__ vperm, const int32_t *__restrict__ offs,
                         const int32_t *__restrict__ items, int32_t W, int nwin, int32_t *__restrict__ blk_len8) {
  int lane = threadIdx.x & 31;
  int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (sl >= nslices) return;
  Tile T = tiles[sl];
  BigC b = bcs[T.bc];
  int vi = T.j * 32 + lane;
  int cnt[MAX_WIN];
#pragma unroll
  for (int w = 0; w < MAX_WIN; ++w) cnt[w] = 0;
  if (vi < b.s) {
    int32_t v = vperm[b.vp_off + vi];
    int32_t p = offs[v], e = offs[v + 1];
    int32_t bound = W;
    int w = 0, run = 0;
    for (; p < e; ++p) {
      int32_t x = items[p];
      while (x >= bound) {
#pragma unroll
        for (int q = 0; q < MAX_WIN; ++q)
          if (q == w) cnt[q] = run;
        ++w;
        run = 0;
        bound += W;
      }
      ++run;
    }
#pragma unroll
    for (int q = 0; q < MAX_WIN; ++q)
      if (q == w) cnt[q] = run;
  }
#pragma unroll
  for (int q = 0; q < MAX_WIN; ++q) {
    if (q >= nwin) break;
    int c = cnt[q];
#pragma unroll
    for (int o = 16; o; o >>= 1) c = max(c, __shfl_xor_sync(0xffffffffu, c, o));
    if (lane == 0) blk_len8[sl * nwin + q] = (c + 7) / 8;
  }
}

__global__ void k_sl_fill(const Tile *__restrict__ tiles, int64_t nslices, const BigC *__restrict__ bcs,
                          const int32_t *__restrict__ vperm, const int32_t *__restrict__ offs,
                          const int32_t *__restrict__ items, int32_t W, int nwin,
                          const int32_t *__restrict__ blk_len8, const int32_t *__restrict__ blk_off8,
                          uint4 *__restrict__ packed) {
  int lane = threadIdx.x & 31;
  int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (sl >= nslices) return;
  Tile T = tiles[sl];
  BigC b = bcs[T.bc];
  int vi = T.j * 32 + lane;
  int32_t p = 0, e = 0;
  if (vi < b.s) {
    int32_t v = vperm[b.vp_off + vi];
    p = offs[v];
    e = offs[v + 1];
  }
  const uint32_t pad = (uint32_t)W;
  for (int w = 0; w < nwin; ++w) {
    const int32_t hi = (w + 1) * W, lo = w * W;
    const int32_t len8 = blk_len8[sl * nwin + w];
    uint4 *dst = packed + (int64_t)blk_off8[sl * nwin + w] * 32 + lane;
    for (int32_t g = 0; g < len8; ++g) {
      uint32_t h[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        int32_t x = p < e ? items[p] : INT32_MAX;
        bool in = x < hi;
        h[q] = in ? (uint32_t)(x - lo) : pad;
        p += in;
      }
      dst[(int64_t)g * 32] = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16),
                                        h[6] | (h[7] << 16));
    }
  }
}

// ------------------------------------------------------------------ K7 small clusters
constexpr int SMALL_WARPS = 8;

__device__ __forceinline__ void fused_insert(c2_cand *__restrict__ R, int k, int32_t xid, uint32_t xi, uint32_t xU) {
  // insert x into the sorted list R[0..k) (pads last) unless present or not better than R[k-1]
  c2_cand last = R[k - 1];
  if (last.id >= 0 && !c2d::better(xi, xU, xid, last.inter, last.uni, last.id)) return;
  int pos = k;
  for (int q = 0; q < k; ++q) {
    c2_cand e = R[q];
    if (e.id == xid) return;
    if (e.id < 0 || c2d::better(xi, xU, xid, e.inter, e.uni, e.id)) {
      pos = q;
      break;
    }
  }
  if (pos >= k) return;
  for (int q = k - 1; q > pos; --q) R[q] = R[q - 1];
  R[pos] = c2_cand{xid, (uint16_t)xi, (uint16_t)xU};
}

__global__ void __launch_bounds__(SMALL_WARPS * 32) k_local_small(
    const SmallItem *__restrict__ work, int64_t lo, int64_t hi, const int32_t *__restrict__ members, int32_t n,
    const int32_t *__restrict__ offs, const int32_t *__restrict__ itm, const int32_t *__restrict__ psize, int k,
    int fused, c2_cand *__restrict__ out) {
  __shared__ uint32_t cnt[SMALL_WARPS][32][33];
  __shared__ int32_t sid[SMALL_WARPS][32], sps[SMALL_WARPS][32], sbeg[SMALL_WARPS][32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = lo + warp; it < hi; it += nwarps) {
    SmallItem I = work[it];
    const int32_t *mem = members + (int64_t)I.f * n + I.start;
    int s = I.s;
    int32_t u = lane < s ? mem[lane] : -1;
    sid[w][lane] = u;
    sps[w][lane] = u >= 0 ? psize[u] : 0;
    sbeg[w][lane] = u >= 0 ? offs[u] : 0;
    __syncwarp();
    // all unordered pairs (a > b), each by a two-pointer merge of the two sorted rows
    int np = s * (s - 1) / 2;
    for (int p = lane; p < np; p += 32) {
      int a = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)p)) * 0.5f);
      while (a * (a - 1) / 2 > p) --a;
      while ((a + 1) * a / 2 <= p) ++a;
      int bb = p - a * (a - 1) / 2;
      const int32_t *A = itm + sbeg[w][a];
      const int32_t *B = itm + sbeg[w][bb];
      int na = sps[w][a], nb = sps[w][bb];
      int i = 0, j = 0, c = 0;
      while (i < na && j < nb) {
        int32_t x = A[i], y = B[j];
        c += x == y;
        i += x <= y;
        j += y <= x;
      }
      cnt[w][a][bb] = c;
      cnt[w][bb][a] = c;
    }
    __syncwarp();
    if (u >= 0) {
      const uint32_t len = (uint32_t)sps[w][lane];
      if (!fused) {
        // exact rank of every candidate among the row's s-1 candidates
        c2_cand *o = out + ((int64_t)I.f * n + u) * k;
        for (int j = 0; j < s; ++j) {
          if (j == lane) continue;
          int32_t vj = sid[w][j];
          uint32_t ij = cnt[w][lane][j], Uj = len + sps[w][j] - ij;
          int rank = 0;
          for (int j2 = 0; j2 < s; ++j2) {
            if (j2 == lane || j2 == j) continue;
            uint32_t i2 = cnt[w][lane][j2], U2 = len + sps[w][j2] - i2;
            rank += c2d::better(i2, U2, sid[w][j2], ij, Uj, vj);
          }
          if (rank < k) o[rank] = c2_cand{vj, (uint16_t)ij, (uint16_t)Uj};
        }
        for (int q = s - 1; q < k; ++q) o[q] = c2_cand{-1, 0, 0};
      } else {
        // fused: insert each candidate into the running final list of u (Alg. 3)
        c2_cand *R = out + (int64_t)u * k;
        for (int j = 0; j < s; ++j) {
          if (j == lane) continue;
          uint32_t ij = cnt[w][lane][j];
          fused_insert(R, k, sid[w][j], ij, len + sps[w][j] - ij);
        }
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ K7 tile kernel
__device__ __forceinline__ void csa(uint32_t &h, uint32_t &l, uint32_t a, uint32_t b, uint32_t c) {
  uint32_t u = a ^ b;
  h = (a & b) | (u & c);
  l = u ^ c;
}

// in-register 32x32 bit transpose: A[p] bit r -> A[r] bit p
__device__ __forceinline__ void transpose32(uint32_t (&A)[32]) {
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

struct TileArgs {
  const Tile *tiles;
  int64_t lo, hi;
  int *counter;
  const BigC *bcs;
  const int32_t *vperm;
  const int32_t *blk_len8;
  const int32_t *blk_off8;
  const uint4 *packed;
  const int32_t *psize;
  int32_t n;
  int32_t W, nwin;
  int k;
  int fused;
  c2_cand *out;       // local: cand [t][n][k]; fused: running final lists [n][k]
  uint16_t *scratch;  // [grid][32][smax]
  int32_t smax;
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
  // add 8 masks; returns the carry of weight 8 (to be combined by add16)
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

template <int NHI, int VPT, int KS>
__global__ void __launch_bounds__(TILE_T, 1) k_local_tile(TileArgs a) {
  extern __shared__ uint32_t M[];  // W + 1 words; M[W] stays 0 (padding id)
  __shared__ int s_item;
  __shared__ int32_t s_ru[32];
  __shared__ uint32_t s_rp[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i <= a.W; i += TILE_T) M[i] = 0;
  uint16_t *cnt = a.scratch + (int64_t)blockIdx.x * 32 * a.smax;
  const int nwin = a.nwin;
  const uint32_t W = (uint32_t)a.W;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_item = atomicAdd(a.counter, 1);
    __syncthreads();
    const int64_t it = a.lo + s_item;
    if (it >= a.hi) break;
    const Tile T = a.tiles[it];
    const BigC B = a.bcs[T.bc];
    const int nsl = (B.s + 31) >> 5;
    const int r0 = T.j * 32;
    const int nr = min(32, B.s - r0);
    const int32_t *vp = a.vperm + B.vp_off;
    if (tid < 32) {
      int32_t u = tid < nr ? vp[r0 + tid] : -1;
      s_ru[tid] = u;
      s_rp[tid] = u >= 0 ? (uint32_t)a.psize[u] : 0u;
    }
    for (int g0 = 0; g0 < nsl; g0 += VPT * TILE_WARPS) {
      Counter<NHI> C[VPT];
#pragma unroll
      for (int q = 0; q < VPT; ++q) C[q].zero();
      for (int w = 0; w < nwin; ++w) {
        // ---- build M for window w from the tile's own slice (rows), lane r -> bit r
        {
          const int64_t bi = (int64_t)(B.sl_off + T.j) * nwin + w;
          const int32_t n4 = a.blk_len8[bi] * 32;
          const uint4 *src = a.packed + (int64_t)a.blk_off8[bi] * 32;
          for (int gi = tid; gi < n4; gi += TILE_T) {
            uint4 d = src[gi];
            uint32_t bit = 1u << (gi & 31);
            uint32_t xs[8] = {d.x & 0xFFFFu, d.x >> 16, d.y & 0xFFFFu, d.y >> 16,
                              d.z & 0xFFFFu, d.z >> 16, d.w & 0xFFFFu, d.w >> 16};
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (xs[q] < W) atomicOr(&M[xs[q]], bit);
          }
        }
        __syncthreads();
        // ---- probe: each warp streams VPT slices of v lists
#pragma unroll
        for (int q = 0; q < VPT; ++q) {
          const int jj = g0 + q * TILE_WARPS + warp;
          if (jj < nsl) {
            const int64_t bi = (int64_t)(B.sl_off + jj) * nwin + w;
            const int32_t len8 = a.blk_len8[bi];
            const uint4 *src = a.packed + (int64_t)a.blk_off8[bi] * 32 + lane;
            int32_t p8 = 0;
            for (; p8 + 1 < len8; p8 += 2) {
              uint4 d0 = __ldg(src + (int64_t)p8 * 32);
              uint4 d1 = __ldg(src + (int64_t)(p8 + 1) * 32);
              uint32_t m[8];
              masks8(M, d0, m);
              uint32_t e8a = C[q].add8(m);
              masks8(M, d1, m);
              uint32_t e8b = C[q].add8(m);
              C[q].add16(e8a, e8b);
            }
            if (p8 < len8) {
              uint4 d0 = __ldg(src + (int64_t)p8 * 32);
              uint32_t m[8];
              masks8(M, d0, m);
              uint32_t e8a = C[q].add8(m);
              C[q].add16(e8a, 0u);
            }
          }
        }
        __syncthreads();
        // ---- clear M
        {
          const int64_t bi = (int64_t)(B.sl_off + T.j) * nwin + w;
          const int32_t n4 = a.blk_len8[bi] * 32;
          const uint4 *src = a.packed + (int64_t)a.blk_off8[bi] * 32;
          for (int gi = tid; gi < n4; gi += TILE_T) {
            uint4 d = src[gi];
            uint32_t xs[8] = {d.x & 0xFFFFu, d.x >> 16, d.y & 0xFFFFu, d.y >> 16,
                              d.z & 0xFFFFu, d.z >> 16, d.w & 0xFFFFu, d.w >> 16};
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (xs[q] < W) M[xs[q]] = 0;
          }
        }
        __syncthreads();
      }
      // ---- counts: planes -> 32 counts per v (transpose), to scratch [row][v]
#pragma unroll
      for (int q = 0; q < VPT; ++q) {
        const int jj = g0 + q * TILE_WARPS + warp;
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
          if (vi < B.s) {
#pragma unroll
            for (int r = 0; r < 32; ++r)
              if (r < nr) cnt[(int64_t)r * a.smax + vi] = (uint16_t)A[r];
          }
        }
      }
    }
    __syncthreads();
    // ---- K8: per-row top-k, warp per row
    const int kk = a.k;
    const int tl = (kk - 1) & 31, ts = (kk - 1) >> 5;
    for (int r = warp; r < nr; r += TILE_WARPS) {
      const int32_t ur = s_ru[r];
      const uint32_t pr = s_rp[r];
      int32_t id0 = INT32_MAX, id1 = INT32_MAX;
      uint32_t i0 = 0, U0 = 1, i1 = 0, U1 = 1;
      c2_cand *dst = a.fused ? a.out + (int64_t)ur * kk : a.out + ((int64_t)B.f * a.n + ur) * kk;
      if (a.fused) {
        if (lane < kk) {
          c2_cand e = dst[lane];
          if (e.id >= 0) { id0 = e.id; i0 = e.inter; U0 = e.uni; }
        }
        if (KS == 2 && 32 + lane < kk) {
          c2_cand e = dst[32 + lane];
          if (e.id >= 0) { id1 = e.id; i1 = e.inter; U1 = e.uni; }
        }
      }
      int32_t tid_ = __shfl_sync(0xffffffffu, ts ? id1 : id0, tl);
      uint32_t ti = __shfl_sync(0xffffffffu, ts ? i1 : i0, tl);
      uint32_t tU = __shfl_sync(0xffffffffu, ts ? U1 : U0, tl);
      const uint16_t *crow = cnt + (int64_t)r * a.smax;
      for (int vb = 0; vb < B.s; vb += 32) {
        const int vi = vb + lane;
        int32_t v = vi < B.s ? vp[vi] : -1;
        bool valid = v >= 0 && v != ur;
        uint32_t ci = valid ? crow[vi] : 0u;
        uint32_t cU = valid ? pr + (uint32_t)a.psize[v] - ci : 1u;
        bool bt = valid && c2d::better(ci, cU, v, ti, tU, tid_);
        unsigned mask = __ballot_sync(0xffffffffu, bt);
        while (mask) {
          int l = __ffs(mask) - 1;
          mask &= mask - 1;
          uint32_t xi = __shfl_sync(0xffffffffu, ci, l);
          uint32_t xU = __shfl_sync(0xffffffffu, cU, l);
          int32_t xid = __shfl_sync(0xffffffffu, v, l);
          if (!c2d::better(xi, xU, xid, ti, tU, tid_)) continue;
          if (a.fused) {
            bool dup = (id0 == xid) || (KS == 2 && id1 == xid);
            if (__any_sync(0xffffffffu, dup)) continue;  // same id from an earlier function (A16)
          }
          int pos = __popc(__ballot_sync(0xffffffffu, c2d::better(i0, U0, id0, xi, xU, xid)));
          int32_t pid0 = __shfl_up_sync(0xffffffffu, id0, 1);
          uint32_t pi0 = __shfl_up_sync(0xffffffffu, i0, 1), pU0 = __shfl_up_sync(0xffffffffu, U0, 1);
          if (KS == 2) {
            pos += __popc(__ballot_sync(0xffffffffu, c2d::better(i1, U1, id1, xi, xU, xid)));
            int32_t pid1 = __shfl_up_sync(0xffffffffu, id1, 1);
            uint32_t pi1 = __shfl_up_sync(0xffffffffu, i1, 1), pU1 = __shfl_up_sync(0xffffffffu, U1, 1);
            int32_t lid0 = __shfl_sync(0xffffffffu, id0, 31);
            uint32_t li0 = __shfl_sync(0xffffffffu, i0, 31), lU0 = __shfl_sync(0xffffffffu, U0, 31);
            if (lane == 0) { pid1 = lid0; pi1 = li0; pU1 = lU0; }
            const int j1 = 32 + lane;
            if (j1 == pos) { id1 = xid; i1 = xi; U1 = xU; }
            else if (j1 > pos) { id1 = pid1; i1 = pi1; U1 = pU1; }
          }
          if (lane == pos) { id0 = xid; i0 = xi; U0 = xU; }
          else if (lane > pos) { id0 = pid0; i0 = pi0; U0 = pU0; }
          tid_ = __shfl_sync(0xffffffffu, ts ? id1 : id0, tl);
          ti = __shfl_sync(0xffffffffu, ts ? i1 : i0, tl);
          tU = __shfl_sync(0xffffffffu, ts ? U1 : U0, tl);
        }
      }
      if (lane < kk) dst[lane] = id0 == INT32_MAX ? c2_cand{-1, 0, 0} : c2_cand{id0, (uint16_t)i0, (uint16_t)U0};
      if (KS == 2 && 32 + lane < kk)
        dst[32 + lane] = id1 == INT32_MAX ? c2_cand{-1, 0, 0} : c2_cand{id1, (uint16_t)i1, (uint16_t)U1};
    }
  }
}

typedef void (*TileKernel)(TileArgs);

template <int NHI, int VPT>
static TileKernel pick_ks(int k) {
  return k <= 32 ? k_local_tile<NHI, VPT, 1> : k_local_tile<NHI, VPT, 2>;
}
template <int NHI>
static TileKernel pick_vpt(int vpt, int k) {
  return vpt <= 1 ? pick_ks<NHI, 1>(k) : vpt <= 2 ? pick_ks<NHI, 2>(k) : pick_ks<NHI, 4>(k);
}
static TileKernel pick_tile(int nhi, int vpt, int k) {
  return nhi <= 4 ? pick_vpt<4>(vpt, k) : nhi <= 8 ? pick_vpt<8>(vpt, k) : pick_vpt<11>(vpt, k);
}

__global__ void k_init_pads(c2_cand *__restrict__ R, int64_t E) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < E) R[e] = c2_cand{-1, 0, 0};
}

__global__ void k_count_small_f(const SmallItem *__restrict__ w, int64_t ns, int32_t *__restrict__ per_f) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ns) atomicAdd(&per_f[w[i].f], 1);
}

// fused: out = running final lists [n][k] (initialised here); local: out = cand [t][n][k]
int local_knn(c2_ctx *ctx, const Csr &csr, int t, const Clusters &cl, int k, c2_cand *out, bool fused) {
  int rc;
  cudaStream_t st = ctx->stream;
  const int32_t n = csr.n;
  int32_t hcum[C2_MAX_T + 1];
  hcum[0] = 0;
  for (int f = 0; f < t; ++f) hcum[f + 1] = hcum[f] + cl.n_clusters[f];
  const int64_t C = hcum[t];
  int32_t *ccum = (int32_t *)ws_get(ctx, "wl_ccum", (C2_MAX_T + 1) * 4 + 4 * (2 * C2_MAX_T + 2), &rc);
  if (rc) return rc;
  int32_t *per_f = ccum + C2_MAX_T + 1;  // [0..t) tiles per f, [t..2t) small per f
  C2_CUDA(ctx, cudaMemcpyAsync(ccum, hcum, (t + 1) * 4, cudaMemcpyHostToDevice, st));
  C2_CUDA(ctx, cudaMemsetAsync(per_f, 0, 4 * 2 * C2_MAX_T, st));
  int32_t *fl = (int32_t *)ws_get(ctx, "wl_flags", (size_t)(C + 1) * 4 * 2, &rc);
  if (rc) return rc;
  int32_t *fsmall = fl, *sscan = fl + (C + 1);
  uint32_t *kv = (uint32_t *)ws_get(ctx, "wl_kv", (size_t)C * 4 * 4 + 16, &rc);
  if (rc) return rc;
  uint32_t *key = kv, *val = kv + C, *skey = kv + 2 * C, *sval = kv + 3 * C;
  const uint32_t maxs = (uint32_t)std::max(cl.max_size, 1);
  const int sized = maxs < (1u << 25) ? 1 : 0;
  k_wl_classify<<<nblk(C), 256, 0, st>>>(cl.offsets, ccum, t, n, C, fsmall, key, val, maxs, sized);
  C2_LAUNCHED(ctx, "k_wl_classify");
  C2_TRY(scan_exclusive(ctx, fsmall, sscan, C));
  C2_TRY(radix_sort_pairs(ctx, key, val, skey, sval, C, 32));
  int32_t hs;
  C2_CUDA(ctx, cudaMemcpyAsync(&hs, sscan + C, 4, cudaMemcpyDeviceToHost, st));
  C2_TRY(stream_sync(ctx, "worklist counts"));
  const int64_t nsmall = hs, nbig = C - hs;
  SmallItem *wsmall = (SmallItem *)ws_get(ctx, "wl_small", (size_t)(nsmall + 1) * sizeof(SmallItem), &rc);
  if (rc) return rc;
  k_wl_small<<<nblk(C), 256, 0, st>>>(cl.offsets, ccum, t, n, C, fsmall, sscan, wsmall);
  C2_LAUNCHED(ctx, "k_wl_small");
  if (nsmall > 0) {
    k_count_small_f<<<nblk(nsmall), 256, 0, st>>>(wsmall, nsmall, per_f + t);
    C2_LAUNCHED(ctx, "k_count_small_f");
  }
  if (fused) {
    k_init_pads<<<nblk((int64_t)n * k), 256, 0, st>>>(out, (int64_t)n * k);
    C2_LAUNCHED(ctx, "k_init_pads");
  }

  // ---- big clusters: descriptors, tiles, length-sorted member order, packed lists
  int64_t nslices = 0;
  BigC *bcs = nullptr;
  Tile *tiles = nullptr;
  int32_t *vperm = nullptr, *blk_len8 = nullptr, *blk_off8 = nullptr;
  uint4 *packed = nullptr;
  const int32_t m = csr.max_item + 1;
  int32_t nwin = (int32_t)((m + 50000 - 1) / 50000);
  int32_t W = (int32_t)((m + nwin - 1) / nwin);
  if (nwin > MAX_WIN) return set_err(ctx, C2_EINVAL, "item ids up to %d need %d windows (max %d)", m, nwin, MAX_WIN);
  if (nbig > 0) {
    int32_t *bsz = (int32_t *)ws_get(ctx, "bc_sz", (size_t)(nbig + 1) * 4 * 4, &rc);
    if (rc) return rc;
    int32_t *bns = bsz + (nbig + 1), *vp_scan = bsz + 2 * (nbig + 1), *sl_scan = bsz + 3 * (nbig + 1);
    k_bc_sizes<<<nblk(nbig), 256, 0, st>>>(sval, nbig, cl.offsets, ccum, t, n, bsz, bns);
    C2_LAUNCHED(ctx, "k_bc_sizes");
    C2_TRY(scan_exclusive(ctx, bsz, vp_scan, nbig));
    C2_TRY(scan_exclusive(ctx, bns, sl_scan, nbig));
    int32_t h2[2];
    C2_CUDA(ctx, cudaMemcpyAsync(h2, vp_scan + nbig, 4, cudaMemcpyDeviceToHost, st));
    C2_CUDA(ctx, cudaMemcpyAsync(h2 + 1, sl_scan + nbig, 4, cudaMemcpyDeviceToHost, st));
    C2_TRY(stream_sync(ctx, "big cluster sizes"));
    const int64_t nv = h2[0];
    nslices = h2[1];
    bcs = (BigC *)ws_get(ctx, "bc", (size_t)nbig * sizeof(BigC), &rc);
    if (rc) return rc;
    tiles = (Tile *)ws_get(ctx, "tiles", (size_t)nslices * sizeof(Tile), &rc);
    if (rc) return rc;
    vperm = (int32_t *)ws_get(ctx, "vperm", (size_t)nv * 4, &rc);
    if (rc) return rc;
    k_bc_fill<<<nblk(nbig), 256, 0, st>>>(sval, nbig, cl.offsets, ccum, t, n, vp_scan, sl_scan, bcs, tiles, per_f);
    C2_LAUNCHED(ctx, "k_bc_fill");
    k_sl_sort<<<(unsigned)nbig, 1024, 0, st>>>(bcs, cl.members, n, csr.psize, vperm);
    C2_LAUNCHED(ctx, "k_sl_sort");
    const int64_t nb = nslices * nwin;
    blk_len8 = (int32_t *)ws_get(ctx, "blk_len8", (size_t)(2 * nb + 2) * 4, &rc);
    if (rc) return rc;
    blk_off8 = blk_len8 + nb + 1;
    k_sl_len<<<nblk(nslices * 32), 256, 0, st>>>(tiles, nslices, bcs, vperm, csr.offs, csr.items, W, nwin, blk_len8);
    C2_LAUNCHED(ctx, "k_sl_len");
    C2_TRY(scan_exclusive(ctx, blk_len8, blk_off8, nb));
    int32_t tot8;
    C2_CUDA(ctx, cudaMemcpyAsync(&tot8, blk_off8 + nb, 4, cudaMemcpyDeviceToHost, st));
    C2_TRY(stream_sync(ctx, "packed size"));
    packed = (uint4 *)ws_get(ctx, "packed", (size_t)tot8 * 32 * 16 + 16, &rc);
    if (rc) return rc;
    k_sl_fill<<<nblk(nslices * 32), 256, 0, st>>>(tiles, nslices, bcs, vperm, csr.offs, csr.items, W, nwin, blk_len8,
                                                  blk_off8, packed);
    C2_LAUNCHED(ctx, "k_sl_fill");
  }
  int32_t hper[2 * C2_MAX_T];
  C2_CUDA(ctx, cudaMemcpyAsync(hper, per_f, 4 * 2 * C2_MAX_T, cudaMemcpyDeviceToHost, st));
  C2_TRY(stream_sync(ctx, "per-function counts"));

  // ---- tile kernel configuration
  TileKernel tk = nullptr;
  int grid = 0;
  size_t smem = (size_t)(W + 1) * 4;
  uint16_t *scratch = nullptr;
  int *counters = nullptr;
  int32_t smax = (int32_t)((maxs + 31) / 32 * 32);
  if (nslices > 0) {
    int nbits = bits_for((int64_t)csr.max_len + 1);
    int nhi = std::max(nbits - 4, 1);
    int max_sl = (int)((maxs + 31) / 32);
    int vpt = max_sl <= TILE_WARPS ? 1 : max_sl <= 2 * TILE_WARPS ? 2 : 4;
    tk = pick_tile(nhi, vpt, k);
    C2_CUDA(ctx, cudaFuncSetAttribute(tk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    C2_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tk, TILE_T, smem));
    occ = std::max(occ, 1);
    grid = (int)std::min<int64_t>((int64_t)ctx->num_sms * occ, nslices);
    scratch = (uint16_t *)ws_get(ctx, "tile_scratch", (size_t)grid * 32 * smax * 2, &rc);
    if (rc) return rc;
    counters = (int *)ws_get(ctx, "tile_counter", 4 * (C2_MAX_T + 1), &rc);
    if (rc) return rc;
    C2_CUDA(ctx, cudaMemsetAsync(counters, 0, 4 * (C2_MAX_T + 1), st));
  }
  auto launch_small = [&](int64_t lo, int64_t hi) -> int {
    if (hi <= lo) return C2_OK;
    int64_t blocks = std::min<int64_t>((hi - lo + SMALL_WARPS - 1) / SMALL_WARPS, (int64_t)ctx->num_sms * 16);
    k_local_small<<<(unsigned)blocks, SMALL_WARPS * 32, 0, st>>>(wsmall, lo, hi, cl.members, n, csr.offs, csr.items,
                                                                 csr.psize, k, fused ? 1 : 0, out);
    C2_LAUNCHED(ctx, "k_local_small");
    return C2_OK;
  };
  auto launch_tiles = [&](int64_t lo, int64_t hi, int ci) -> int {
    if (hi <= lo) return C2_OK;
    TileArgs ta{tiles, lo, hi, counters + ci, bcs, vperm, blk_len8, blk_off8, packed, csr.psize, n, W, nwin, k,
                fused ? 1 : 0, out, scratch, smax};
    int g = (int)std::min<int64_t>(grid, hi - lo);
    tk<<<g, TILE_T, smem, st>>>(ta);
    C2_LAUNCHED(ctx, "k_local_tile");
    return C2_OK;
  };
  if (!fused) {
    C2_TRY(launch_small(0, nsmall));
    C2_TRY(launch_tiles(0, nslices, 0));
  } else {
    // Alg. 3 order: function by function, each row merged into its running final list
    int64_t slo = 0, tlo = 0;
    for (int f = 0; f < t; ++f) {
      int64_t shi = slo + hper[t + f], thi = tlo + hper[f];
      C2_TRY(launch_tiles(tlo, thi, f));
      C2_TRY(launch_small(slo, shi));
      slo = shi;
      tlo = thi;
    }
  }
  return C2_OK;
}

}  // namespace c2
