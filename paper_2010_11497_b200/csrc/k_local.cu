// k_local.cu -- Step 2 of C^2 on the GPU: brute-force Jaccard top-k inside every cluster
// (Alg. 2, brute-force branch; s(s-1)/2 similarities per cluster).
//
// K5 worklist: clusters of <= 32 users go to k_local_small (one warp per cluster, all
//    unordered pairs by two-pointer merge, exact rank selection).  Larger clusters are cut
//    into row tiles of 32 users, sorted by cluster size (largest first: the paper's
//    decreasing priority queue) and consumed by persistent CTAs of k_local_tile.
// K7 k_local_tile: for a row tile R (32 users) of cluster C, shared memory holds the
//    transposed membership mask M[x] = {r in R : x in P_r} (bit r) for the items x of the
//    current id window.  Each thread takes one v in C and streams its items: the 32 counts
//    |P_r ∩ P_v| are accumulated bit-sliced (Harley-Seal carry-save adders over 8 masks,
//    then a ripple into the high planes), so one LDS + ~5 LOP3 serve 32 pairs.  A 32x32 bit
//    transpose turns the planes into 32 counts (u16, L2 scratch).
// K8 (in K7): per row, a warp keeps the k best candidates under the exact order
//    (i1*U2 > i2*U1, ties by lower id) as a warp-distributed sorted list.
#include <algorithm>
#include <vector>

#include "c2_internal.cuh"

namespace c2 {

struct WorkItem {
  int32_t f, start, s, tile;
};

constexpr int TILE_T = 512;       // threads per tile CTA
constexpr int TILE_WARPS = TILE_T / 32;

// ------------------------------------------------------------------ K5 worklist
__global__ void k_wl_classify(const int32_t *__restrict__ offsets, const int32_t *__restrict__ ccum, int t,
                              int32_t n, int64_t C, int32_t *__restrict__ fsmall, int32_t *__restrict__ fbig,
                              uint32_t *__restrict__ bkey, uint32_t *__restrict__ bval, int32_t maxs) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= C) return;
  int f = 0;
  while (f + 1 < t && ccum[f + 1] <= g) ++f;
  int64_t c = g - ccum[f];
  const int32_t *off = offsets + (int64_t)f * (n + 1);
  int32_t s = off[c + 1] - off[c];
  fsmall[g] = s <= 32;
  fbig[g] = s > 32;
  bkey[g] = (uint32_t)(s > 32 ? maxs - s : maxs + 1);  // big clusters first, largest first
  bval[g] = (uint32_t)g;
}

__global__ void k_wl_small(const int32_t *__restrict__ offsets, const int32_t *__restrict__ ccum, int t, int32_t n,
                           int64_t C, const int32_t *__restrict__ fsmall, const int32_t *__restrict__ sscan,
                           WorkItem *__restrict__ out) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= C || !fsmall[g]) return;
  int f = 0;
  while (f + 1 < t && ccum[f + 1] <= g) ++f;
  int64_t c = g - ccum[f];
  const int32_t *off = offsets + (int64_t)f * (n + 1);
  out[sscan[g]] = WorkItem{f, off[c], off[c + 1] - off[c], 0};
}

// sorted big clusters (vals = g) -> number of tiles, then expansion
__global__ void k_wl_ntiles(const uint32_t *__restrict__ sval, int64_t nbig, const int32_t *__restrict__ offsets,
                            const int32_t *__restrict__ ccum, int t, int32_t n, int32_t *__restrict__ ntiles) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nbig) return;
  int64_t g = sval[i];
  int f = 0;
  while (f + 1 < t && ccum[f + 1] <= g) ++f;
  int64_t c = g - ccum[f];
  const int32_t *off = offsets + (int64_t)f * (n + 1);
  ntiles[i] = (off[c + 1] - off[c] + 31) / 32;
}

__global__ void k_wl_tiles(const uint32_t *__restrict__ sval, int64_t nbig, const int32_t *__restrict__ offsets,
                           const int32_t *__restrict__ ccum, int t, int32_t n, const int32_t *__restrict__ tscan,
                           WorkItem *__restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nbig) return;
  int64_t g = sval[i];
  int f = 0;
  while (f + 1 < t && ccum[f + 1] <= g) ++f;
  int64_t c = g - ccum[f];
  const int32_t *off = offsets + (int64_t)f * (n + 1);
  int32_t s = off[c + 1] - off[c];
  int32_t base = tscan[i];
  for (int j = 0; j < (s + 31) / 32; ++j) out[base + j] = WorkItem{f, off[c], s, j};
}

// ------------------------------------------------------------------ K7 small clusters
constexpr int SMALL_WARPS = 8;

__global__ void __launch_bounds__(SMALL_WARPS * 32) k_local_small(
    const WorkItem *__restrict__ work, int64_t n_items, const int32_t *__restrict__ members, int32_t n,
    const int32_t *__restrict__ offs, const int32_t *__restrict__ itm, const int32_t *__restrict__ psize, int k,
    c2_cand *__restrict__ cand) {
  __shared__ uint32_t cnt[SMALL_WARPS][32][33];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = warp; it < n_items; it += nwarps) {
    WorkItem I = work[it];
    const int32_t *mem = members + (int64_t)I.f * n + I.start;
    int s = I.s;
    int32_t u = lane < s ? mem[lane] : -1;
    int32_t beg = u >= 0 ? offs[u] : 0;
    int32_t len = u >= 0 ? psize[u] : 0;
    // all unordered pairs (a > b), each by a two-pointer merge of the sorted rows
    int np = s * (s - 1) / 2;
    for (int p = lane; p < np; p += 32) {
      int a = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)p)) * 0.5f);
      while (a * (a - 1) / 2 > p) --a;
      while ((a + 1) * a / 2 <= p) ++a;
      int bb = p - a * (a - 1) / 2;
      int32_t ua = mem[a], ub = mem[bb];
      const int32_t *A = itm + offs[ua];
      const int32_t *B = itm + offs[ub];
      int na = psize[ua], nb = psize[ub];
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
    // exact rank of every candidate of row `lane` among the row's s-1 candidates
    if (u >= 0) {
      c2_cand *out = cand + ((int64_t)I.f * n + u) * k;
      for (int j = 0; j < s; ++j) {
        if (j == lane) continue;
        int32_t vj = mem[j];
        uint32_t ij = cnt[w][lane][j], Uj = len + psize[vj] - ij;
        int rank = 0;
        for (int j2 = 0; j2 < s; ++j2) {
          if (j2 == lane || j2 == j) continue;
          int32_t v2 = mem[j2];
          uint32_t i2 = cnt[w][lane][j2], U2 = len + psize[v2] - i2;
          rank += c2d::better(i2, U2, v2, ij, Uj, vj);
        }
        if (rank < k) out[rank] = c2_cand{vj, (uint16_t)ij, (uint16_t)Uj};
      }
      for (int q = s - 1; q < k; ++q) out[q] = c2_cand{-1, 0, 0};
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
    const uint32_t m = mi == 0 ? 0x0000FFFFu : mi == 1 ? 0x00FF00FFu : mi == 2 ? 0x0F0F0F0Fu : mi == 3 ? 0x33333333u : 0x55555555u;
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
  const WorkItem *work;
  int64_t n_items;
  int *counter;
  const int32_t *members;
  int32_t n;
  const int32_t *offs;
  const int32_t *itm;
  const int32_t *psize;
  int32_t W, nwin;
  int k;
  c2_cand *cand;
  uint16_t *scratch;  // [grid][32][smax]
  int32_t smax;
};

template <int NH>
__global__ void __launch_bounds__(TILE_T, 2) k_local_tile(TileArgs a) {
  extern __shared__ uint32_t M[];
  __shared__ int s_item;
  __shared__ int32_t s_ru[32], s_rb[32], s_re[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < a.W; i += TILE_T) M[i] = 0;
  uint16_t *cnt = a.scratch + (int64_t)blockIdx.x * 32 * a.smax;
  const bool single = a.nwin == 1;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_item = atomicAdd(a.counter, 1);
    __syncthreads();
    const int64_t it = s_item;
    if (it >= a.n_items) break;
    const WorkItem I = a.work[it];
    const int32_t *mem = a.members + (int64_t)I.f * a.n + I.start;
    const int r0 = I.tile * 32;
    const int nr = min(32, I.s - r0);
    if (tid < 32) {
      int32_t u = tid < nr ? mem[r0 + tid] : -1;
      s_ru[tid] = u;
      s_rb[tid] = u >= 0 ? a.offs[u] : 0;
      s_re[tid] = u >= 0 ? a.offs[u + 1] : 0;
    }
    __syncthreads();
    // build / clear M for window [lo, lo + W): warp per row, lanes over the row's items
    auto build = [&](int32_t lo, bool set) {
      for (int r = warp; r < nr; r += TILE_WARPS) {
        for (int32_t p = s_rb[r] + lane; p < s_re[r]; p += 32) {
          int32_t x = a.itm[p] - lo;
          if ((uint32_t)x < (uint32_t)a.W) {
            if (set) atomicOr(&M[x], 1u << r);
            else M[x] = 0;
          }
        }
      }
    };
    if (single) {
      build(0, true);
      __syncthreads();
    }
    for (int vg = 0; vg < I.s; vg += TILE_T) {
      const int vi = vg + tid;
      const bool has = vi < I.s;
      const int32_t v = has ? mem[vi] : 0;
      int32_t cur = has ? a.offs[v] : 0;
      const int32_t vend = has ? a.offs[v + 1] : 0;
      uint32_t ones = 0, twos = 0, fours = 0;
      uint32_t H[NH];
#pragma unroll
      for (int i = 0; i < NH; ++i) H[i] = 0;
      for (int w = 0; w < a.nwin; ++w) {
        const int32_t lo = w * a.W, hi = lo + a.W;
        if (!single) {
          build(lo, true);
          __syncthreads();
        }
        if (has) {
          for (;;) {
            uint32_t mm[8];
            int nvalid = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              int32_t p = cur + j;
              int32_t x = p < vend ? __ldg(a.itm + p) : INT32_MAX;
              bool ok = x < hi;
              mm[j] = ok ? M[x - lo] : 0u;
              nvalid += ok;
            }
            uint32_t tA, tB, fA, fB, e8;
            csa(tA, ones, ones, mm[0], mm[1]);
            csa(tB, ones, ones, mm[2], mm[3]);
            csa(fA, twos, twos, tA, tB);
            csa(tA, ones, ones, mm[4], mm[5]);
            csa(tB, ones, ones, mm[6], mm[7]);
            csa(fB, twos, twos, tA, tB);
            csa(e8, fours, fours, fA, fB);
            uint32_t carry = e8;
#pragma unroll
            for (int i = 0; i < NH; ++i) {
              uint32_t tt = H[i] & carry;
              H[i] ^= carry;
              carry = tt;
            }
            cur += nvalid;
            if (nvalid < 8) break;
          }
        }
        if (!single) {
          __syncthreads();
          build(lo, false);
          __syncthreads();
        }
      }
      if (has) {
        uint32_t A[32];
        A[0] = ones;
        A[1] = twos;
        A[2] = fours;
#pragma unroll
        for (int i = 0; i < NH; ++i) A[3 + i] = H[i];
#pragma unroll
        for (int i = 3 + NH; i < 32; ++i) A[i] = 0;
        transpose32(A);
#pragma unroll
        for (int r = 0; r < 32; ++r)
          if (r < nr) cnt[(int64_t)r * a.smax + vi] = (uint16_t)A[r];
      }
    }
    __syncthreads();
    if (single) {
      build(0, false);
    }
    // ---- K8: per-row top-k (warp per row) over the s candidates of the row
    for (int r = warp; r < nr; r += TILE_WARPS) {
      const int32_t ur = s_ru[r];
      const uint32_t pr = (uint32_t)(s_re[r] - s_rb[r]);
      int32_t id0 = INT32_MAX, id1 = INT32_MAX;
      uint32_t i0 = 0, U0 = 1, i1 = 0, U1 = 1;
      const int kk = a.k;
      const int tl = (kk - 1) & 31, ts = (kk - 1) >> 5;
      int32_t tid_ = INT32_MAX;
      uint32_t ti = 0, tU = 1;
      const uint16_t *crow = cnt + (int64_t)r * a.smax;
      for (int vb = 0; vb < I.s; vb += 32) {
        const int vi = vb + lane;
        int32_t v = vi < I.s ? mem[vi] : -1;
        bool valid = v >= 0 && v != ur;
        uint32_t ci = valid ? crow[vi] : 0;
        uint32_t cU = valid ? pr + (uint32_t)a.psize[v] - ci : 1;
        bool bt = valid && c2d::better(ci, cU, v, ti, tU, tid_);
        unsigned mask = __ballot_sync(0xffffffffu, bt);
        while (mask) {
          int l = __ffs(mask) - 1;
          mask &= mask - 1;
          uint32_t xi = __shfl_sync(0xffffffffu, ci, l);
          uint32_t xU = __shfl_sync(0xffffffffu, cU, l);
          int32_t xid = __shfl_sync(0xffffffffu, v, l);
          if (!c2d::better(xi, xU, xid, ti, tU, tid_)) continue;
          unsigned g0 = __ballot_sync(0xffffffffu, c2d::better(i0, U0, id0, xi, xU, xid));
          unsigned g1 = kk > 32 ? __ballot_sync(0xffffffffu, c2d::better(i1, U1, id1, xi, xU, xid)) : 0u;
          int pos = __popc(g0) + __popc(g1);
          // shift right by one from pos, insert x at pos
          int32_t pid0 = __shfl_up_sync(0xffffffffu, id0, 1);
          uint32_t pi0 = __shfl_up_sync(0xffffffffu, i0, 1), pU0 = __shfl_up_sync(0xffffffffu, U0, 1);
          int32_t pid1 = __shfl_up_sync(0xffffffffu, id1, 1);
          uint32_t pi1 = __shfl_up_sync(0xffffffffu, i1, 1), pU1 = __shfl_up_sync(0xffffffffu, U1, 1);
          int32_t lid0 = __shfl_sync(0xffffffffu, id0, 31);
          uint32_t li0 = __shfl_sync(0xffffffffu, i0, 31), lU0 = __shfl_sync(0xffffffffu, U0, 31);
          if (lane == 0) { pid1 = lid0; pi1 = li0; pU1 = lU0; }
          const int j0 = lane, j1 = 32 + lane;
          if (j0 == pos) { id0 = xid; i0 = xi; U0 = xU; }
          else if (j0 > pos) { id0 = pid0; i0 = pi0; U0 = pU0; }
          if (j1 == pos) { id1 = xid; i1 = xi; U1 = xU; }
          else if (j1 > pos) { id1 = pid1; i1 = pi1; U1 = pU1; }
          // threshold = entry k-1
          int32_t a_id = ts ? id1 : id0;
          uint32_t a_i = ts ? i1 : i0, a_U = ts ? U1 : U0;
          tid_ = __shfl_sync(0xffffffffu, a_id, tl);
          ti = __shfl_sync(0xffffffffu, a_i, tl);
          tU = __shfl_sync(0xffffffffu, a_U, tl);
        }
      }
      c2_cand *out = a.cand + ((int64_t)I.f * a.n + ur) * kk;
      if (lane < kk) out[lane] = id0 == INT32_MAX ? c2_cand{-1, 0, 0} : c2_cand{id0, (uint16_t)i0, (uint16_t)U0};
      if (32 + lane < kk)
        out[32 + lane] = id1 == INT32_MAX ? c2_cand{-1, 0, 0} : c2_cand{id1, (uint16_t)i1, (uint16_t)U1};
    }
  }
}

template <int NH>
static int launch_tile(c2_ctx *ctx, TileArgs &ta, size_t smem, int grid) {
  cudaFuncSetAttribute(k_local_tile<NH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_local_tile<NH><<<grid, TILE_T, smem, ctx->stream>>>(ta);
  C2_LAUNCHED(ctx, "k_local_tile");
  return C2_OK;
}

template <int NH>
static int tile_occupancy(size_t smem) {
  cudaFuncSetAttribute(k_local_tile<NH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_local_tile<NH>, TILE_T, smem);
  return nb;
}

static inline unsigned nblk(int64_t x, int bs = 256) { return (unsigned)((x + bs - 1) / bs); }
static inline int bits_for(int64_t x) {
  int b = 1;
  while ((1LL << b) < x) ++b;
  return b;
}

int local_knn(c2_ctx *ctx, const Csr &csr, int t, const Clusters &cl, int k, c2_cand *cand) {
  int rc;
  cudaStream_t st = ctx->stream;
  const int32_t n = csr.n;
  int64_t C = 0;
  int32_t hcum[C2_MAX_T + 1];
  hcum[0] = 0;
  for (int f = 0; f < t; ++f) hcum[f + 1] = hcum[f] + cl.n_clusters[f];
  C = hcum[t];
  int32_t *ccum = (int32_t *)ws_get(ctx, "wl_ccum", (C2_MAX_T + 1) * 4, &rc);
  if (rc) return rc;
  C2_CUDA(ctx, cudaMemcpyAsync(ccum, hcum, (t + 1) * 4, cudaMemcpyHostToDevice, st));
  int32_t *fl = (int32_t *)ws_get(ctx, "wl_flags", (size_t)(C + 1) * 4 * 4, &rc);
  if (rc) return rc;
  int32_t *fsmall = fl, *fbig = fl + (C + 1), *sscan = fl + 2 * (C + 1), *bscan = fl + 3 * (C + 1);
  uint32_t *kv = (uint32_t *)ws_get(ctx, "wl_kv", (size_t)C * 4 * 4 + 16, &rc);
  if (rc) return rc;
  uint32_t *bkey = kv, *bval = kv + C, *skey = kv + 2 * C, *sval = kv + 3 * C;
  const int32_t maxs = std::max(cl.max_size, 1);
  k_wl_classify<<<nblk(C), 256, 0, st>>>(cl.offsets, ccum, t, n, C, fsmall, fbig, bkey, bval, maxs);
  C2_LAUNCHED(ctx, "k_wl_classify");
  C2_TRY(scan_exclusive(ctx, fsmall, sscan, C));
  C2_TRY(scan_exclusive(ctx, fbig, bscan, C));
  C2_TRY(radix_sort_pairs(ctx, bkey, bval, skey, sval, C, bits_for(maxs + 2)));
  int32_t h2[2];
  C2_CUDA(ctx, cudaMemcpyAsync(h2, sscan + C, 4, cudaMemcpyDeviceToHost, st));
  C2_CUDA(ctx, cudaMemcpyAsync(h2 + 1, bscan + C, 4, cudaMemcpyDeviceToHost, st));
  C2_TRY(stream_sync(ctx, "worklist counts"));
  const int64_t nsmall = h2[0], nbig = h2[1];
  WorkItem *wsmall = (WorkItem *)ws_get(ctx, "wl_small", (size_t)(nsmall + 1) * sizeof(WorkItem), &rc);
  if (rc) return rc;
  k_wl_small<<<nblk(C), 256, 0, st>>>(cl.offsets, ccum, t, n, C, fsmall, sscan, wsmall);
  C2_LAUNCHED(ctx, "k_wl_small");
  int64_t ntiles_total = 0;
  WorkItem *wtile = nullptr;
  if (nbig > 0) {
    int32_t *nt = (int32_t *)ws_get(ctx, "wl_nt", (size_t)(nbig + 1) * 4 * 2, &rc);
    if (rc) return rc;
    int32_t *tscan = nt + nbig + 1;
    k_wl_ntiles<<<nblk(nbig), 256, 0, st>>>(sval, nbig, cl.offsets, ccum, t, n, nt);
    C2_LAUNCHED(ctx, "k_wl_ntiles");
    C2_TRY(scan_exclusive(ctx, nt, tscan, nbig));
    int32_t ht;
    C2_CUDA(ctx, cudaMemcpyAsync(&ht, tscan + nbig, 4, cudaMemcpyDeviceToHost, st));
    C2_TRY(stream_sync(ctx, "worklist tiles"));
    ntiles_total = ht;
    wtile = (WorkItem *)ws_get(ctx, "wl_tiles", (size_t)(ntiles_total + 1) * sizeof(WorkItem), &rc);
    if (rc) return rc;
    k_wl_tiles<<<nblk(nbig), 256, 0, st>>>(sval, nbig, cl.offsets, ccum, t, n, tscan, wtile);
    C2_LAUNCHED(ctx, "k_wl_tiles");
  }
  // ---- small clusters
  if (nsmall > 0) {
    int64_t blocks = std::min<int64_t>((nsmall + SMALL_WARPS - 1) / SMALL_WARPS, (int64_t)ctx->num_sms * 16);
    k_local_small<<<(unsigned)blocks, SMALL_WARPS * 32, 0, st>>>(wsmall, nsmall, cl.members, n, csr.offs, csr.items,
                                                                 csr.psize, k, cand);
    C2_LAUNCHED(ctx, "k_local_small");
  }
  // ---- tiles
  if (ntiles_total > 0) {
    const int32_t m = csr.max_item + 1;
    const int64_t wmax = 28 * 1024;  // 112 KB of masks -> two CTAs per SM
    int32_t nwin = (int32_t)((m + wmax - 1) / wmax);
    int32_t W = (int32_t)(((m + nwin - 1) / nwin + 31) / 32 * 32);
    size_t smem = (size_t)W * 4;
    int bits = bits_for((int64_t)csr.max_len + 1);
    int nh = std::max(bits - 3, 1);
    int occ;
    if (nh <= 5) occ = tile_occupancy<5>(smem);
    else if (nh <= 8) occ = tile_occupancy<8>(smem);
    else if (nh <= 9) occ = tile_occupancy<9>(smem);
    else occ = tile_occupancy<12>(smem);
    occ = std::max(occ, 1);
    int grid = (int)std::min<int64_t>((int64_t)ctx->num_sms * occ, ntiles_total);
    int32_t smax = (maxs + 31) / 32 * 32;
    uint16_t *scratch = (uint16_t *)ws_get(ctx, "tile_scratch", (size_t)grid * 32 * smax * 2, &rc);
    if (rc) return rc;
    int *counter = (int *)ws_get(ctx, "tile_counter", 64, &rc);
    if (rc) return rc;
    C2_CUDA(ctx, cudaMemsetAsync(counter, 0, 4, st));
    TileArgs ta{wtile, ntiles_total, counter, cl.members, n, csr.offs, csr.items, csr.psize, W, nwin, k, cand,
                scratch, smax};
    if (nh <= 5) C2_TRY(launch_tile<5>(ctx, ta, smem, grid));
    else if (nh <= 8) C2_TRY(launch_tile<8>(ctx, ta, smem, grid));
    else if (nh <= 9) C2_TRY(launch_tile<9>(ctx, ta, smem, grid));
    else C2_TRY(launch_tile<12>(ctx, ta, smem, grid));
  }
  return C2_OK;
}

}  // namespace c2
