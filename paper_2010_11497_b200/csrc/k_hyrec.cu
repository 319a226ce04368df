// k_hyrec.cu -- Alg. 2's else-branch: Hyrec on clusters with |C| >= rho k^2
// (rho = 5), selected by C2_OPT_LOCAL_SOLVER = C2_SOLVER_HYBRID (the default is brute force for
// every cluster, reading A12).  Hyrec: start from a random k-degree graph over C and
// repeatedly compare every user with the neighbours of its neighbours, keeping the k best; stop when
// fewer than delta*k*|C| neighbourhood entries changed in an iteration (delta = 0.001) or after 30
// iterations.  Iterations are synchronous (every user reads the previous iteration's graph),
// so the result is deterministic and reproducible by the test oracle (reading A34).
//
// Layout: the members of all Hyrec clusters concatenated (hmem, global ids; cluster of member a =
// hcl[a]); neighbour graphs nb[2][S][k] (cluster-local indices, ping-pong by iteration), lists
// nl[2][S][k] (c2_cand, global ids).  One warp per member per iteration: the member's profile as an
// item bitmap in shared memory, the <= k + k^2 candidates deduplicated in a shared hash set, one
// lane per candidate for the intersection, then k rounds of exact warp argmax.  All 30 iterations
// are launched; a cluster that converged is skipped (device-side flag, no host synchronisation).
#include <algorithm>
#include <vector>

#include "c2_internal.cuh"

namespace c2 {

constexpr uint64_t HYREC_SALT = 0x4879726563526e67ULL;  // "HyrecRng" (as the oracle's)
constexpr int HYREC_RHO = 5, HYREC_DELTA_INV = 1000, HYREC_MAX_ITERS = 30;
constexpr int HY_WARPS = 4;

static inline unsigned nblk_h(int64_t x, int bs = 256) { return (unsigned)((x + bs - 1) / bs); }

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

struct HyCl {
  int32_t f, start, s, base;  // function, offset in members[f], size, first member position in hmem
};

__global__ void k_hy_clusters(const uint32_t *__restrict__ sval, int64_t nh, const int32_t *__restrict__ offsets,
                              const int32_t *__restrict__ ccum, int t, int32_t n, HyCl *__restrict__ hc,
                              int32_t *__restrict__ sz) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nh) return;
  const int64_t g = sval[i];
  int f = 0;
  while (f + 1 < t && ccum[f + 1] <= g) ++f;
  const int64_t c = g - ccum[f];
  const int32_t *off = offsets + (int64_t)f * (n + 1);
  hc[i] = HyCl{f, off[c], off[c + 1] - off[c], 0};
  sz[i] = off[c + 1] - off[c];
}

__global__ void k_hy_members(HyCl *__restrict__ hc, int64_t nh, const int32_t *__restrict__ sbase,
                             const int32_t *__restrict__ members, int32_t n, int32_t *__restrict__ hmem,
                             int32_t *__restrict__ hcl) {
  const int64_t i = blockIdx.x;
  if (i >= nh) return;
  HyCl h = hc[i];
  h.base = sbase[i];
  if (threadIdx.x == 0) hc[i] = h;
  for (int j = threadIdx.x; j < h.s; j += blockDim.x) {
    hmem[h.base + j] = members[(int64_t)h.f * n + h.start + j];
    hcl[h.base + j] = (int32_t)i;
  }
}

// random initial graph: k distinct cluster-local indices != a, drawn from mixed counters
__global__ void k_hy_init(const HyCl *__restrict__ hc, const int32_t *__restrict__ hmem,
                          const int32_t *__restrict__ hcl, int32_t S, int k, uint64_t seed, int32_t *__restrict__ nb0,
                          int32_t *__restrict__ done) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= S) return;
  const HyCl h = hc[hcl[a]];
  const int32_t al = (int32_t)(a - h.base);
  if (al == 0) done[hcl[a]] = -1;
  const uint64_t key = mix64(mix64((seed ^ HYREC_SALT) + (uint64_t)h.f) + (uint64_t)hmem[a]);
  int32_t *nb = nb0 + a * k;
  int got = 0;
  for (uint64_t j = 0; got < k; ++j) {
    const uint64_t r = mix64(key + j + 1);
    const int32_t b = (int32_t)__umul64hi(r, (uint64_t)h.s);
    if (b == al) continue;
    bool dup = false;
    for (int q = 0; q < got; ++q) dup |= nb[q] == b;
    if (!dup) nb[got++] = b;
  }
}

struct HyArgs {
  const int32_t *offs, *items, *psize;
  const HyCl *hc;
  const int32_t *hmem, *hcl;
  int32_t S;
  int k;
  const int32_t *nb_prev;
  int32_t *nb_next;
  c2_cand *nl_out;
  unsigned long long *upd;
  const int32_t *done;
  int32_t nwords;  // item bitmap words per warp
  int hcap;        // hash-set slots per warp (power of two >= 2 (k + k^2))
  int ccap;        // candidate capacity per warp (k + k^2)
};

__device__ __forceinline__ bool hy_better(uint32_t iu1, int32_t id1, uint32_t iu2, int32_t id2) {
  return c2d::better(iu1 & 0xFFFFu, iu1 >> 16, id1, iu2 & 0xFFFFu, iu2 >> 16, id2);
}

__global__ void __launch_bounds__(HY_WARPS * 32) k_hy_iter(HyArgs a) {
  extern __shared__ __align__(16) uint32_t hsm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int per_warp = a.nwords + a.hcap + 3 * a.ccap + 2 * a.k + 1;
  uint32_t *bm = hsm + w * per_warp;
  int32_t *hset = reinterpret_cast<int32_t *>(bm + a.nwords);
  int32_t *cloc = hset + a.hcap;                                   // candidate local index
  int32_t *cid = cloc + a.ccap;                                    // candidate global id
  uint32_t *ciu = reinterpret_cast<uint32_t *>(cid + a.ccap);     // inter | union << 16
  int32_t *prevN = reinterpret_cast<int32_t *>(ciu + a.ccap);      // this member's previous neighbours
  int32_t *newN = prevN + a.k;
  int *cnt = newN + a.k;
  for (int i = lane; i < a.nwords; i += 32) bm[i] = 0;
  for (int i = lane; i < a.hcap; i += 32) hset[i] = -1;
  const int k = a.k;
  for (int64_t m = (int64_t)blockIdx.x * HY_WARPS + w; m < a.S; m += (int64_t)gridDim.x * HY_WARPS) {
    const int32_t c = a.hcl[m];
    if (a.done[c] >= 0) continue;  // converged: its lists are final
    const HyCl h = a.hc[c];
    const int32_t al = (int32_t)(m - h.base);
    const int32_t u = a.hmem[m];
    if (lane == 0) *cnt = 0;
    for (int j = lane; j < k; j += 32) prevN[j] = a.nb_prev[m * k + j];
    // the member's profile as a bitmap
    const int32_t p0 = a.offs[u], p1 = a.offs[u + 1];
    for (int32_t p = p0 + lane; p < p1; p += 32) {
      const uint32_t x = (uint32_t)a.items[p];
      atomicOr(&bm[x >> 5], 1u << (x & 31));
    }
    __syncwarp();
    // candidates: N(u) and the neighbours of its neighbours, deduplicated, u excluded
    const int tot = k + k * k;
    for (int e = lane; e < tot; e += 32) {
      int32_t b;
      if (e < k) b = prevN[e];
      else b = a.nb_prev[(int64_t)(h.base + prevN[(e - k) / k]) * k + (e - k) % k];
      if (b == al) continue;
      uint32_t slot = ((uint32_t)b * 0x9E3779B1u) & (uint32_t)(a.hcap - 1);
      for (;;) {
        const int32_t old = atomicCAS(&hset[slot], -1, b);
        if (old == -1) {
          cloc[atomicAdd(cnt, 1)] = b;
          break;
        }
        if (old == b) break;
        slot = (slot + 1) & (uint32_t)(a.hcap - 1);
      }
    }
    __syncwarp();
    const int nc = *cnt;
    // exact (inter, union) of every candidate: one lane per candidate walks its profile
    const uint32_t pu = (uint32_t)(p1 - p0);
    for (int q = lane; q < nc; q += 32) {
      const int32_t v = a.hmem[h.base + cloc[q]];
      uint32_t i = 0;
      for (int32_t p = a.offs[v]; p < a.offs[v + 1]; ++p) {
        const uint32_t x = (uint32_t)a.items[p];
        i += (bm[x >> 5] >> (x & 31)) & 1u;
      }
      const uint32_t U = pu + (uint32_t)(a.offs[v + 1] - a.offs[v]) - i;
      cid[q] = v;
      ciu[q] = i | (U << 16);
    }
    __syncwarp();
    // k rounds of exact warp argmax (candidates taken are marked id = INT32_MAX)
    const int kk = min(k, nc);
    for (int r = 0; r < kk; ++r) {
      uint32_t biu = 0;
      int32_t bid = INT32_MAX, bq = -1;
      for (int q = lane; q < nc; q += 32) {
        const int32_t id = cid[q];
        if (id == INT32_MAX) continue;
        if (bq < 0 || hy_better(ciu[q], id, biu, bid)) {
          biu = ciu[q];
          bid = id;
          bq = q;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const uint32_t oiu = __shfl_xor_sync(0xffffffffu, biu, o);
        const int32_t oid = __shfl_xor_sync(0xffffffffu, bid, o);
        const int32_t oq = __shfl_xor_sync(0xffffffffu, bq, o);
        if (oq >= 0 && (bq < 0 || hy_better(oiu, oid, biu, bid))) {
          biu = oiu;
          bid = oid;
          bq = oq;
        }
      }
      if (lane == 0) {
        a.nl_out[m * k + r] = c2_cand{bid, (uint16_t)(biu & 0xFFFFu), (uint16_t)(biu >> 16)};
        newN[r] = cloc[bq];
        cid[bq] = INT32_MAX;
      }
      __syncwarp();
    }
    for (int r = kk + lane; r < k; r += 32) {  // (|C| - 1 >= k for Hyrec clusters: not reached)
      a.nl_out[m * k + r] = c2_cand{-1, 0, 0};
      newN[r] = -1;
    }
    __syncwarp();
    // updates: new neighbours not in the previous graph
    int up = 0;
    for (int r = lane; r < kk; r += 32) {
      bool found = false;
      for (int j = 0; j < k; ++j) found |= prevN[j] == newN[r];
      up += found ? 0 : 1;
      a.nb_next[m * k + r] = newN[r];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) up += __shfl_xor_sync(0xffffffffu, up, o);
    if (lane == 0 && up) atomicAdd(&a.upd[c], (unsigned long long)up);
    // restore the per-warp structures
    for (int32_t p = p0 + lane; p < p1; p += 32) bm[(uint32_t)a.items[p] >> 5] = 0;
    for (int i = lane; i < a.hcap; i += 32) hset[i] = -1;
    __syncwarp();
  }
}

__global__ void k_hy_check(const HyCl *__restrict__ hc, int64_t nh, int k, int it,
                           unsigned long long *__restrict__ upd, int32_t *__restrict__ done) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nh) return;
  if (done[c] < 0) {
    const unsigned long long u = upd[c];
    if (u * HYREC_DELTA_INV < (unsigned long long)k * (unsigned long long)hc[c].s || it + 1 >= HYREC_MAX_ITERS)
      done[c] = it;
  }
  upd[c] = 0;
}

// final lists -> cand[f][u] (local mode) or merged into the running Alg. 3 lists (fused mode,
// members of function f only: a user is in one cluster per function)
__global__ void k_hy_out(const HyCl *__restrict__ hc, const int32_t *__restrict__ hmem, const int32_t *__restrict__ hcl,
                         int32_t S, int k, int32_t n, const c2_cand *__restrict__ nl0, const c2_cand *__restrict__ nl1,
                         const int32_t *__restrict__ done, int f_only, c2_cand *__restrict__ out, int fused) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= S) return;
  const int32_t c = hcl[a];
  const HyCl h = hc[c];
  if (fused && h.f != f_only) return;
  const c2_cand *L = ((done[c] & 1) ? nl1 : nl0) + a * k;
  const int32_t u = hmem[a];
  if (!fused) {
    for (int j = 0; j < k; ++j) out[((int64_t)h.f * n + u) * k + j] = L[j];
    return;
  }
  // Alg. 3 step: running list R (best first, pads last) merged with L, duplicates dropped (A16)
  c2_cand *R = out + (int64_t)u * k;
  c2_cand res[C2_MAX_K];
  int i = 0, j = 0, cntr = 0;
  int32_t last = -1;
  while (cntr < k) {
    const bool ri = i < k && R[i].id >= 0, lj = j < k && L[j].id >= 0;
    if (!ri && !lj) break;
    c2_cand x;
    if (ri && (!lj || c2d::better(R[i].inter, R[i].uni, R[i].id, L[j].inter, L[j].uni, L[j].id))) x = R[i++];
    else x = L[j++];
    if (x.id == last) continue;
    last = x.id;
    res[cntr++] = x;
  }
  for (int q = 0; q < k; ++q) R[q] = q < cntr ? res[q] : c2_cand{-1, 0, 0};
}

int hyrec_clusters(c2_ctx *ctx, const Csr &csr, int t, const int32_t *offsets, const int32_t *members,
                   const int32_t *ccum, const uint32_t *sval_h, int64_t nh, const int32_t *hyrec_f_lo, int k,
                   uint64_t seed, c2_cand *out, bool fused) {
  if (nh <= 0) return C2_OK;
  int rc;
  cudaStream_t st = ctx->stream;
  const int32_t n = csr.n;
  HyCl *hc = (HyCl *)ws_get(ctx, "hy_cl", (size_t)nh * sizeof(HyCl), &rc);
  if (rc) return rc;
  int32_t *sz = (int32_t *)ws_get(ctx, "hy_sz", (size_t)(2 * nh + 2) * 4, &rc);
  if (rc) return rc;
  int32_t *sbase = sz + nh + 1;
  k_hy_clusters<<<nblk_h(nh), 256, 0, st>>>(sval_h, nh, offsets, ccum, t, n, hc, sz);
  C2_LAUNCHED(ctx, "k_hy_clusters");
  C2_TRY(scan_exclusive(ctx, sz, sbase, nh));
  int32_t S = 0;
  C2_CUDA(ctx, cudaMemcpyAsync(&S, sbase + nh, 4, cudaMemcpyDeviceToHost, st));
  C2_TRY(stream_sync(ctx, "hyrec members"));
  int32_t *hmem = (int32_t *)ws_get(ctx, "hy_mem", (size_t)S * 4 * 2, &rc);
  if (rc) return rc;
  int32_t *hcl = hmem + S;
  k_hy_members<<<(unsigned)nh, 256, 0, st>>>(hc, nh, sbase, members, n, hmem, hcl);
  C2_LAUNCHED(ctx, "k_hy_members");
  int32_t *nb = (int32_t *)ws_get(ctx, "hy_nb", (size_t)S * k * 4 * 2, &rc);
  if (rc) return rc;
  c2_cand *nl = (c2_cand *)ws_get(ctx, "hy_nl", (size_t)S * k * sizeof(c2_cand) * 2, &rc);
  if (rc) return rc;
  unsigned long long *upd = (unsigned long long *)ws_get(ctx, "hy_upd", (size_t)nh * 8 + 8, &rc);
  if (rc) return rc;
  int32_t *done = (int32_t *)ws_get(ctx, "hy_done", (size_t)nh * 4 + 4, &rc);
  if (rc) return rc;
  C2_CUDA(ctx, cudaMemsetAsync(upd, 0, (size_t)nh * 8, st));
  k_hy_init<<<nblk_h(S), 256, 0, st>>>(hc, hmem, hcl, S, k, seed, nb, done);
  C2_LAUNCHED(ctx, "k_hy_init");
  HyArgs ha;
  ha.offs = csr.offs;
  ha.items = csr.items;
  ha.psize = csr.psize;
  ha.hc = hc;
  ha.hmem = hmem;
  ha.hcl = hcl;
  ha.S = S;
  ha.k = k;
  ha.upd = upd;
  ha.done = done;
  ha.nwords = (int32_t)(((int64_t)csr.max_item + 32) / 32);
  ha.ccap = k + k * k;
  int hcap = 64;
  while (hcap < 2 * ha.ccap) hcap <<= 1;
  ha.hcap = hcap;
  const size_t per_warp = ((size_t)ha.nwords + hcap + 3 * ha.ccap + 2 * k + 1) * 4;
  const size_t smem = per_warp * HY_WARPS;
  if (smem > ctx->smem_optin)
    return set_err(ctx, C2_EINVAL, "Hyrec needs %zu B of shared memory per block (item ids too large)", smem);
  C2_CUDA(ctx, cudaFuncSetAttribute(k_hy_iter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 1;
  C2_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hy_iter, HY_WARPS * 32, smem));
  const int grid = std::max(1, std::min<int>(ctx->num_sms * std::max(occ, 1), (S + HY_WARPS - 1) / HY_WARPS));
  for (int it = 0; it < HYREC_MAX_ITERS; ++it) {
    ha.nb_prev = nb + (size_t)(it & 1) * S * k;
    ha.nb_next = nb + (size_t)((it + 1) & 1) * S * k;
    ha.nl_out = nl + (size_t)(it & 1) * S * k;
    k_hy_iter<<<grid, HY_WARPS * 32, smem, st>>>(ha);
    C2_LAUNCHED(ctx, "k_hy_iter");
    k_hy_check<<<nblk_h(nh), 256, 0, st>>>(hc, nh, k, it, upd, done);
    C2_LAUNCHED(ctx, "k_hy_check");
  }
  if (!fused) {
    k_hy_out<<<nblk_h(S), 256, 0, st>>>(hc, hmem, hcl, S, k, n, nl, nl + (size_t)S * k, done, 0, out, 0);
    C2_LAUNCHED(ctx, "k_hy_out");
  } else {
    for (int f = 0; f < t; ++f) {
      if (hyrec_f_lo[f + 1] == hyrec_f_lo[f]) continue;
      k_hy_out<<<nblk_h(S), 256, 0, st>>>(hc, hmem, hcl, S, k, n, nl, nl + (size_t)S * k, done, f, out, 1);
      C2_LAUNCHED(ctx, "k_hy_out");
    }
  }
  return C2_OK;
}

}  // namespace c2
