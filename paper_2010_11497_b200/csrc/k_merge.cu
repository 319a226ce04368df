// k_merge.cu -- Step 3 of C^2 on the GPU: Alg. 3.  Each user's t partial
// neighbourhoods (sorted best-first by c2_local_knn) are merged keeping the k best; the
// similarity values are reused, never recomputed.  Because the lists are sorted under
// one strict total order and a repeated id carries identical (inter, uni) (A16), a head-
// comparison t-way merge that skips an id equal to the last one emitted yields exactly the
// first k distinct ids of the union.  One thread per user; heads held in registers.  (A warp-
// cooperative variant -- coalesced staging in shared memory, L lanes per user, shuffle argmax per
// round -- measured slower at c5, 2.18 vs 1.35 ms: its 30 rounds of dependent shuffles are
// latency-bound.)
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

constexpr int MG_T = 128;  // users per k_merge2 block
// Even k: the same merge with each list read as 16-byte pairs of entries (rows start 16-byte
// aligned: k * 8 bytes per row), the pair's second entry held in registers until its turn, so
// every byte of cand is loaded once and the load count halves; outputs leave through shared
// memory as coalesced stores.
template <int TMAX>
__global__ void __launch_bounds__(MG_T) k_merge2(const c2_cand *__restrict__ cand, int t, int32_t n, int k,
                                                 int32_t *__restrict__ nbr, uint16_t *__restrict__ inter,
                                                 uint16_t *__restrict__ uni, float *__restrict__ sim) {
  // outputs of the block's MG_T users staged in shared memory ([user][k], the global layout), then
  // written with coalesced stores: nbr | sim (4 B) and inter | uni (2 B) per entry
  extern __shared__ __align__(16) uint32_t msm[];
  uint32_t *s_nb = msm, *s_sim = msm + MG_T * k;
  uint16_t *s_i = reinterpret_cast<uint16_t *>(msm + 2 * MG_T * k), *s_u = s_i + MG_T * k;
  const int64_t u0 = (int64_t)blockIdx.x * MG_T;
  const int64_t u = u0 + threadIdx.x;
  if (u < n) {
    int pos[TMAX];
    int32_t hid[TMAX];
    uint32_t hiu[TMAX];  // head inter | uni << 16
    uint2 nxt[TMAX];     // the entry after the head when pos is even
#pragma unroll
    for (int f = 0; f < TMAX; ++f) {
      pos[f] = 0;
      hid[f] = -1;
      hiu[f] = 1u << 16;
      nxt[f] = make_uint2(0xFFFFFFFFu, 0u);
      if (f < t) {
        const uint4 q = __ldg(reinterpret_cast<const uint4 *>(cand + ((int64_t)f * n + u) * k));
        hid[f] = (int32_t)q.x;
        hiu[f] = q.y;
        nxt[f] = make_uint2(q.z, q.w);
      }
    }
    int cnt = 0;
    int32_t last = -1;
    const int ob = threadIdx.x * k;
    while (cnt < k) {
      int bf = -1;
      int32_t bid = -1;
      uint32_t bi = 0, bU = 1;
#pragma unroll
      for (int f = 0; f < TMAX; ++f) {
        const uint32_t fi = hiu[f] & 0xFFFFu, fU = hiu[f] >> 16;
        if (f < t && hid[f] >= 0 && (bf < 0 || c2d::better(fi, fU, hid[f], bi, bU, bid))) {
          bf = f;
          bid = hid[f];
          bi = fi;
          bU = fU;
        }
      }
      if (bf < 0) break;  // all lists exhausted
#pragma unroll
      for (int f = 0; f < TMAX; ++f) {
        if (f == bf) {
          const int p = ++pos[f];
          if (p >= k) {
            hid[f] = -1;
          } else if (p & 1) {
            hid[f] = (int32_t)nxt[f].x;
            hiu[f] = nxt[f].y;
          } else {
            const uint4 q = __ldg(reinterpret_cast<const uint4 *>(cand + ((int64_t)f * n + u) * k + p));
            hid[f] = (int32_t)q.x;
            hiu[f] = q.y;
            nxt[f] = make_uint2(q.z, q.w);
          }
        }
      }
      if (bid == last) continue;  // same id from another function: identical values (A16)
      last = bid;
      s_nb[ob + cnt] = (uint32_t)bid;
      s_i[ob + cnt] = (uint16_t)bi;
      s_u[ob + cnt] = (uint16_t)bU;
      s_sim[ob + cnt] = __float_as_uint(__fdiv_rn((float)bi, (float)bU));
      ++cnt;
    }
    for (; cnt < k; ++cnt) {
      s_nb[ob + cnt] = 0xFFFFFFFFu;
      s_i[ob + cnt] = 0;
      s_u[ob + cnt] = 0;
      s_sim[ob + cnt] = 0u;
    }
  }
  __syncthreads();
  const int64_t nu = (int64_t)n - u0 < MG_T ? (int64_t)n - u0 : (int64_t)MG_T;
  const int64_t E = nu * k, e0 = u0 * k;
  for (int64_t e = threadIdx.x; e < E; e += MG_T) {
    nbr[e0 + e] = (int32_t)s_nb[e];
    inter[e0 + e] = s_i[e];
    uni[e0 + e] = s_u[e];
    if (sim) sim[e0 + e] = __uint_as_float(s_sim[e]);
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

int merge(c2_ctx *ctx, int t, int n, int k, const c2_cand *cand, int32_t *nbr, uint16_t *inter, uint16_t *uni,
          float *sim) {
  unsigned blocks = (unsigned)((n + 127) / 128);
  if ((k & 1) == 0 && ((uintptr_t)cand & 15) == 0) {
    const size_t sm = (size_t)MG_T * k * 12;
    auto kern = t <= 8 ? k_merge2<8> : t <= 16 ? k_merge2<16> : k_merge2<64>;
    C2_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<(unsigned)((n + MG_T - 1) / MG_T), MG_T, sm, ctx->stream>>>(cand, t, n, k, nbr, inter, uni, sim);
    C2_LAUNCHED(ctx, "k_merge2");
    return C2_OK;
  }
  if (t <= 8) k_merge<8><<<blocks, 128, 0, ctx->stream>>>(cand, t, n, k, nbr, inter, uni, sim);
  else if (t <= 16) k_merge<16><<<blocks, 128, 0, ctx->stream>>>(cand, t, n, k, nbr, inter, uni, sim);
  else k_merge<64><<<blocks, 128, 0, ctx->stream>>>(cand, t, n, k, nbr, inter, uni, sim);
  C2_LAUNCHED(ctx, "k_merge");
  return C2_OK;
}

}  // namespace c2
