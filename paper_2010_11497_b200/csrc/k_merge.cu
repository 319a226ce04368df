// k_merge.cu -- Step 3 of C^2 on the GPU: Alg. 3.  Each user's t partial
// neighbourhoods (sorted best-first by c2_local_knn) are merged keeping the k best; the
// similarity values are reused, never recomputed.  Because the lists are sorted under
// one strict total order and a repeated id carries identical (inter, uni) (A16), a head-
// comparison t-way merge that skips an id equal to the last one emitted yields exactly the
// first k distinct ids of the union.  k_merge_w (t <= 32, below) is the warp-cooperative version;
// k_merge (one thread per user, heads in registers) serves t > 32.
#include <algorithm>

#include "c2_internal.cuh"

namespace c2 {

template <int TMAX>
__global__ void __launch_bounds__(128) k_merge(const c2_cand *__restrict__ cand, int t, int32_t n, int k,
                                               int32_t *__restrict__ nbr, uint16_t *__restrict__ inter,
                                               uint16_t *__restrict__ uni, float *__restrict__ sim) {
  int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  int pos[TMAX];
  int32_t hid[TMAX];
  uint32_t hi[TMAX], hU[TMAX];
#pragma unroll
  for (int f = 0; f < TMAX; ++f) {
    pos[f] = 0;
    hid[f] = -1;
    hi[f] = 0;
    hU[f] = 1;
    if (f < t) {
      c2_cand e = cand[((int64_t)f * n + u) * k];
      hid[f] = e.id;
      hi[f] = e.inter;
      hU[f] = e.uni;
    }
  }
  int cnt = 0;
  int32_t last = -1;
  int32_t *onb = nbr + u * k;
  uint16_t *oi = inter + u * k, *ou = uni + u * k;
  float *os = sim ? sim + u * k : nullptr;
  while (cnt < k) {
    int bf = -1;
    int32_t bid = -1;
    uint32_t bi = 0, bU = 1;
#pragma unroll
    for (int f = 0; f < TMAX; ++f) {
      if (f < t && hid[f] >= 0 && (bf < 0 || c2d::better(hi[f], hU[f], hid[f], bi, bU, bid))) {
        bf = f;
        bid = hid[f];
        bi = hi[f];
        bU = hU[f];
      }
    }
    if (bf < 0) break;  // all lists exhausted
#pragma unroll
    for (int f = 0; f < TMAX; ++f) {
      if (f == bf) {
        int p = ++pos[f];
        if (p < k) {
          c2_cand e = cand[((int64_t)f * n + u) * k + p];
          hid[f] = e.id;
          hi[f] = e.inter;
          hU[f] = e.uni;
        } else {
          hid[f] = -1;
        }
      }
    }
    if (bid == last) continue;  // same id from another function: identical values (A16)
    last = bid;
    onb[cnt] = bid;
    oi[cnt] = (uint16_t)bi;
    ou[cnt] = (uint16_t)bU;
    if (os) os[cnt] = __fdiv_rn((float)bi, (float)bU);
    ++cnt;
  }
  for (; cnt < k; ++cnt) {
    onb[cnt] = -1;
    oi[cnt] = 0;
    ou[cnt] = 0;
    if (os) os[cnt] = 0.0f;
  }
}

// c2_build's final step: the fused path's running lists are already Alg. 3's result (sorted
// best-first, distinct ids, pads last), so the outputs are an element-wise format conversion
// (coalesced; the same IEEE division for sim as k_merge).
__global__ void k_copyout(const c2_cand *__restrict__ run, int64_t E, int32_t *__restrict__ nbr,
                          uint16_t *__restrict__ inter, uint16_t *__restrict__ uni, float *__restrict__ sim) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const c2_cand c = run[e];
  const bool real = c.id >= 0;
  nbr[e] = real ? c.id : -1;
  inter[e] = real ? c.inter : 0;
  uni[e] = real ? c.uni : 0;
  if (sim) sim[e] = real ? __fdiv_rn((float)c.inter, (float)c.uni) : 0.0f;
}

int copyout(c2_ctx *ctx, int n, int k, const c2_cand *run, int32_t *nbr, uint16_t *inter, uint16_t *uni,
            float *sim) {
  const int64_t E = (int64_t)n * k;
  k_copyout<<<(unsigned)((E + 255) / 256), 256, 0, ctx->stream>>>(run, E, nbr, inter, uni, sim);
  C2_LAUNCHED(ctx, "k_copyout");
  return C2_OK;
}

// Warp-cooperative Alg. 3 (t <= 32): L = next power of two >= t lanes per user, 32/L users per warp.
// The warp stages its users' t*k candidates in shared memory with coalesced loads (each list is k
// consecutive 8-byte records), then every user's L lanes run a head-comparison merge: lane f holds
// list f's head; each round a shuffle argmax over the L lanes picks the best head under the exact
// order, every lane whose head carries that id advances (a repeated id has identical values, A16:
// duplicates are consumed together), and the winner is recorded.  Outputs are staged per warp and
// written as consecutive rows (users of a warp are consecutive), i.e. coalesced.
constexpr int MW_WARPS = 4;
template <int L>
__global__ void __launch_bounds__(MW_WARPS * 32) k_merge_w(const c2_cand *__restrict__ cand, int t, int32_t n, int k,
                                                           int32_t *__restrict__ nbr, uint16_t *__restrict__ inter,
                                                           uint16_t *__restrict__ uni, float *__restrict__ sim) {
  constexpr int UP = 32 / L;  // users per warp
  extern __shared__ __align__(16) c2_cand msm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  c2_cand *buf = msm + (size_t)w * (UP * t * k + UP * k);  // [UP][t][k] inputs, then [UP][k] outputs
  c2_cand *obuf = buf + UP * t * k;
  const int j = lane / L, f = lane % L;  // this lane: user j of the warp, list f
  for (int64_t u0 = ((int64_t)blockIdx.x * MW_WARPS + w) * UP; u0 < n; u0 += (int64_t)gridDim.x * MW_WARPS * UP) {
    const int nu = (n - u0 < UP) ? (int)(n - u0) : UP;
    // coalesced staging: entry e = (user jj, list ff, position p)
    const int tot = nu * t * k;
    for (int e = lane; e < tot; e += 32) {
      const int jj = e / (t * k), r = e % (t * k), ff = r / k, p = r % k;
      buf[e] = cand[((int64_t)ff * n + u0 + jj) * k + p];
    }
    __syncwarp();
    const bool act = j < nu && f < t;
    const c2_cand *mylist = buf + ((size_t)j * t + f) * k;
    int pos = 0;
    c2_cand h = act ? mylist[0] : c2_cand{-1, 0, 0};
    int cnt = 0;
    for (int r = 0; r < k; ++r) {
      // best head of the group (pads have id -1: never best)
      int32_t bid = h.id;
      uint32_t bi = h.inter, bU = h.uni;
#pragma unroll
      for (int o = L / 2; o >= 1; o >>= 1) {
        const int32_t oid = __shfl_xor_sync(0xffffffffu, bid, o);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const uint32_t oU = __shfl_xor_sync(0xffffffffu, bU, o);
        if (oid >= 0 && (bid < 0 || c2d::better(oi, oU, oid, bi, bU, bid))) {
          bid = oid;
          bi = oi;
          bU = oU;
        }
      }
      if (bid < 0) continue;  // this group's lists are exhausted (rounds stay warp-uniform)
      if (act && h.id == bid) {  // consume the winner from every list holding it
        ++pos;
        h = pos < k ? mylist[pos] : c2_cand{-1, 0, 0};
      }
      if (f == 0 && j < nu) obuf[j * k + r] = c2_cand{bid, (uint16_t)bi, (uint16_t)bU};
      ++cnt;
    }
    if (f == 0 && j < nu)
      for (int r = cnt; r < k; ++r) obuf[j * k + r] = c2_cand{-1, 0, 0};
    __syncwarp();
    // coalesced row writes
    const int64_t base = u0 * k;
    for (int e = lane; e < nu * k; e += 32) {
      const c2_cand c = obuf[e];
      const bool real = c.id >= 0;
      nbr[base + e] = real ? c.id : -1;
      inter[base + e] = real ? c.inter : 0;
      uni[base + e] = real ? c.uni : 0;
      if (sim) sim[base + e] = real ? __fdiv_rn((float)c.inter, (float)c.uni) : 0.0f;
    }
    __syncwarp();
  }
}

template <int L>
static int launch_merge_w(c2_ctx *ctx, int t, int n, int k, const c2_cand *cand, int32_t *nbr, uint16_t *inter,
                          uint16_t *uni, float *sim) {
  constexpr int UP = 32 / L;
  const size_t smem = (size_t)MW_WARPS * (UP * t * k + UP * k) * sizeof(c2_cand);
  C2_CUDA(ctx, cudaFuncSetAttribute(k_merge_w<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 1;
  C2_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_merge_w<L>, MW_WARPS * 32, smem));
  const int64_t groups = ((int64_t)n + (int64_t)MW_WARPS * UP - 1) / ((int64_t)MW_WARPS * UP);
  const int grid = (int)std::min<int64_t>(groups, (int64_t)ctx->num_sms * std::max(occ, 1) * 4);
  k_merge_w<L><<<grid, MW_WARPS * 32, smem, ctx->stream>>>(cand, t, n, k, nbr, inter, uni, sim);
  C2_LAUNCHED(ctx, "k_merge_w");
  return C2_OK;
}

int merge(c2_ctx *ctx, int t, int n, int k, const c2_cand *cand, int32_t *nbr, uint16_t *inter, uint16_t *uni,
          float *sim) {
  if (t <= 32) {
    if (t <= 1) return launch_merge_w<1>(ctx, t, n, k, cand, nbr, inter, uni, sim);
    if (t <= 2) return launch_merge_w<2>(ctx, t, n, k, cand, nbr, inter, uni, sim);
    if (t <= 4) return launch_merge_w<4>(ctx, t, n, k, cand, nbr, inter, uni, sim);
    if (t <= 8) return launch_merge_w<8>(ctx, t, n, k, cand, nbr, inter, uni, sim);
    if (t <= 16) return launch_merge_w<16>(ctx, t, n, k, cand, nbr, inter, uni, sim);
    return launch_merge_w<32>(ctx, t, n, k, cand, nbr, inter, uni, sim);
  }
  unsigned blocks = (unsigned)((n + 127) / 128);
  if (t <= 8) k_merge<8><<<blocks, 128, 0, ctx->stream>>>(cand, t, n, k, nbr, inter, uni, sim);
  else if (t <= 16) k_merge<16><<<blocks, 128, 0, ctx->stream>>>(cand, t, n, k, nbr, inter, uni, sim);
  else k_merge<64><<<blocks, 128, 0, ctx->stream>>>(cand, t, n, k, nbr, inter, uni, sim);
  C2_LAUNCHED(ctx, "k_merge");
  return C2_OK;
}

}  // namespace c2
