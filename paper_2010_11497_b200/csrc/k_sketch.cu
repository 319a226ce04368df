// k_sketch.cu -- K1 FastRandomHash sketch and K6 GoldFinger encode.
//
// K1: for every user u and function f, the D smallest DISTINCT values of {h_f(x) : x in P_u}
// (ascending, C2_ABSENT padded).  Element 0 is H_f(u) = min_{i in P_u} h_f(i); element
// d+1 is H\eta(u) with eta = element d (reading A5), so the recursive split never has to
// revisit the CSR while its depth stays below D (A29).  k_sketch_w (hashed, the product path):
// one warp per user, bitmap windows (below); k_sketch (an injected hash table, the paper's worked
// examples): G lanes per user, a sorted distinct top-8 per (user, function) in registers.
#include <algorithm>

#include "c2_internal.cuh"

namespace c2 {

struct HashArgs {
  uint64_t a[C2_MAX_T];
  uint64_t c[C2_MAX_T];
};

// G consecutive lanes share one user (its items are loaded once, broadcast to the group) and
// lane g of the group handles function f0 + g, so a warp covers 32/G users.
template <int G, bool TABLE, bool POW2>
__global__ void __launch_bounds__(256) k_sketch(const int32_t *__restrict__ offs, const int32_t *__restrict__ items,
                                                int32_t n, int t, int f0, uint32_t b, HashArgs ha,
                                                const uint16_t *__restrict__ htab, int32_t m, int D,
                                                uint16_t *__restrict__ out) {
  int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t u = gt / G;
  int f = f0 + (int)(gt % G);
  if (u >= n) return;
  const bool active = f < t;
  const uint64_t ca = active ? ha.a[f] : 0, cc = active ? ha.c[f] : 0;
  uint32_t s[C2_SKETCH_D];
#pragma unroll
  for (int j = 0; j < C2_SKETCH_D; ++j) s[j] = C2_ABSENT16;
  const int32_t p0 = offs[u], p1 = offs[u + 1];
  auto insert = [&](uint32_t v) {
    if (v < s[C2_SKETCH_D - 1]) {
      bool dup = false;
#pragma unroll
      for (int j = 0; j < C2_SKETCH_D - 1; ++j) dup |= (s[j] == v);
      if (!dup) {  // insert v into the sorted distinct list
#pragma unroll
        for (int j = C2_SKETCH_D - 1; j >= 1; --j) s[j] = (v < s[j - 1]) ? s[j - 1] : ((v < s[j]) ? v : s[j]);
        s[0] = min(s[0], v);
      }
    }
  };
  auto hash = [&](uint32_t x) -> uint32_t {
    if (TABLE) return active ? (uint32_t)__ldg(htab + (int64_t)f * m + x) : C2_ABSENT16;
    // h(x) = floor(z * b / 2^64): for b = 2^M (every config) the top M bits of z = a*x + c
    if (POW2) return (uint32_t)((ca * (uint64_t)x + cc) >> (65 - __ffs(b)));  // b >= 2
    return c2d::item_hash(ca, cc, x, b);
  };
  // eight items in flight per step (the loads do not depend on the insertions)
  int32_t p = p0;
  for (; p + 8 <= p1; p += 8) {
    uint32_t x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = (uint32_t)__ldg(items + p + q);
    uint32_t v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = hash(x[q]);
#pragma unroll
    for (int q = 0; q < 8; ++q) insert(v[q]);
  }
  for (; p < p1; ++p) insert(hash((uint32_t)__ldg(items + p)));
  if (!active) return;
  uint16_t *o = out + ((int64_t)f * n + u) * D;
  if (D == C2_SKETCH_D) {
    *reinterpret_cast<uint4 *>(o) = make_uint4(s[0] | (s[1] << 16), s[2] | (s[3] << 16), s[4] | (s[5] << 16),
                                               s[6] | (s[7] << 16));
  } else {
#pragma unroll
    for (int j = 0; j < C2_SKETCH_D; ++j)
      if (j < D) o[j] = (uint16_t)s[j];
  }
}

// Hashed sketch (no injected table): one warp per user, lanes striding the user's items with
// coalesced loads; all functions of a group of SK_FG are hashed from each loaded item.  The D
// smallest distinct values of function f are found with a shared-memory bitmap over a value
// window [base_f, base_f + Wv): every hash in the window sets its bit (atomicOr, so duplicates
// merge), then the warp reads the window's words in order (ballot-free: popc + warp scan) and
// takes the first D set bits.  Wv is sized from |P_u| so ~SK_K values fall in the first window
// (E = |P_u| * Wv / b); a function that finds fewer than D values there (and has values left
// above the window) slides its window up and re-reads the items -- exact for every (b, |P_u|).
// Per item and function: one 64-bit multiply-add, a compare, and for ~SK_K/|P_u| of them one
// shared atomic; no per-lane sorted inserts (the divergence of the thread-per-(user, f) form).
#ifndef C2_SK_NOBR
#define C2_SK_NOBR 0  // 1: no per-function branch in the item loops (finished functions' windows moved out of range)
#endif
constexpr int SK_WARPS = 8;
constexpr int SK_FG = 8;      // functions per pass over the items
constexpr int SK_CAPW = 128;  // window words per function (4096 values)
#ifndef C2_SK_MINB
#define C2_SK_MINB 3
#endif
#ifndef C2_SK_K
#define C2_SK_K 12  // (c5: 16 -> 1.80 ms, 12 -> 1.72, 10 -> 1.75, 20 -> 1.87)
#endif
constexpr int SK_K = C2_SK_K;  // target number of hashed values inside the first window

template <bool POW2>
__global__ void __launch_bounds__(SK_WARPS * 32, C2_SK_MINB) k_sketch_w(const int32_t *__restrict__ offs,
                                                            const int32_t *__restrict__ items, int32_t n, int t,
                                                            uint32_t b, HashArgs ha, int D,
                                                            uint16_t *__restrict__ out, int64_t u0 = 0,
                                                            int64_t n_total = -1, int32_t nnz = INT32_MAX) {
  // users [u0, u0 + n) of a CSR of n_total users (offs points at user u0); out is [t][n_total][D]
  if (n_total < 0) n_total = n;
  __shared__ __align__(16) uint32_t bm[SK_WARPS][SK_FG * SK_CAPW];
  __shared__ __align__(16) uint16_t sv[SK_WARPS][SK_FG][C2_SKETCH_D];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // extraction and output: the 4 lanes 4f..4f+3 own function f of the group
  const int myf = lane >> 2, sub = lane & 3;
  uint32_t *B = bm[w];
  for (int i = lane; i < SK_FG * SK_CAPW; i += 32) B[i] = 0;
  __syncwarp();
  const int sh = POW2 ? 65 - __ffs(b) : 0;
  const int64_t nwarps = (int64_t)gridDim.x * SK_WARPS;
  const float kb = (float)SK_K * (float)b;
  for (int f0 = 0; f0 < t; f0 += SK_FG) {
    const int nf = min(SK_FG, t - f0);
    uint64_t fa[SK_FG], fc[SK_FG];
#pragma unroll
    for (int f = 0; f < SK_FG; ++f) {
      fa[f] = f < nf ? ha.a[f0 + f] : 0;
      fc[f] = f < nf ? ha.c[f0 + f] : 0;
    }
    for (int64_t u = (int64_t)blockIdx.x * SK_WARPS + w; u < n; u += nwarps) {
      // (clamped: the chunked upload path hashes rows before their validation result is read)
      const int32_t p0 = max(__ldg(offs + u), 0), p1 = max(min(__ldg(offs + u + 1), nnz), p0);
      // first window: ~SK_K of the |P_u| hashes (uniform over [0, b)) expected inside; a multiple
      // of 512 values, so every lane's quarter of the words is a whole number of uint4
      const float wf = kb / (float)max(p1 - p0, 1);
      const uint32_t W0 = wf >= (float)(SK_CAPW * 32 - 512) ? SK_CAPW * 32 : ((uint32_t)wf + 512u) & ~511u;
      uint32_t mybase = 0;  // window start of function myf
      int mycnt = 0;        // values of function myf found so far
      unsigned need = (1u << nf) - 1u;
      uint32_t Wv = W0;
      while (need) {
        uint32_t base[SK_FG];
        // a function that needs no more values gets a window start no hash reaches (v < b <= 2^16,
        // so v - base >= 2^31 > Wv): the item loops test every function without a per-function branch
#pragma unroll
        for (int f = 0; f < SK_FG; ++f) {
          base[f] = __shfl_sync(0xffffffffu, mybase, 4 * f);
          if (C2_SK_NOBR && !((need >> f) & 1u)) base[f] = 0x80000000u;
        }
        // ---- hash pass: set the bits of the values inside each needing function's window
        auto hset = [&](int f, uint32_t x) {
          const uint64_t z = fa[f] * (uint64_t)x + fc[f];
          const uint32_t v = POW2 ? (uint32_t)(z >> sh) : (uint32_t)__umul64hi(z, (uint64_t)b);
          const uint32_t d = v - base[f];
          if (d < Wv) atomicOr(&B[f * SK_CAPW + (d >> 5)], 1u << (d & 31));
        };
        const bool all = need == (1u << SK_FG) - 1u;  // (every function of a full group: round 1)
        int32_t bq = p0;
        for (; bq + 128 <= p1; bq += 128) {  // four items per lane, no bounds checks (warp-uniform trip count)
          uint32_t x[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) x[q] = (uint32_t)__ldg(items + bq + lane + 32 * q);
          if (all || C2_SK_NOBR) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
              for (int f = 0; f < SK_FG; ++f) hset(f, x[q]);
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
              for (int f = 0; f < SK_FG; ++f)
                if ((need >> f) & 1u) hset(f, x[q]);
          }
        }
        for (int32_t p = bq + lane; p < p1; p += 32) {
          const uint32_t x = (uint32_t)__ldg(items + p);
#pragma unroll
          for (int f = 0; f < SK_FG; ++f)
            if (C2_SK_NOBR || ((need >> f) & 1u)) hset(f, x);
        }
        __syncwarp();
        // ---- extraction, all functions at once: lane sub of function myf reads its quarter of the
        //      window's words (uint4), a 4-lane prefix places its set bits, the first D - mycnt
        //      are kept; the words are cleared as they are read
        const int nq = (int)(Wv >> 9);  // uint4 per lane
        const bool act = (need >> myf) & 1u;
        uint4 *Bq = reinterpret_cast<uint4 *>(B + myf * SK_CAPW) + sub * nq;
        int pc = 0;
        if (act)
          for (int j = 0; j < nq; ++j) {
            const uint4 q = Bq[j];
            pc += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
          }
        int incl = pc;
        {
          const int y1 = __shfl_up_sync(0xffffffffu, incl, 1, 4);
          if (sub >= 1) incl += y1;
          const int y2 = __shfl_up_sync(0xffffffffu, incl, 2, 4);
          if (sub >= 2) incl += y2;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 3, 4);
        if (act) {
          int r = mycnt + incl - pc;
          const uint32_t vb = mybase + (uint32_t)(sub * nq * 128);
          for (int j = 0; j < nq && r < D; ++j) {
            const uint4 q = Bq[j];
            const uint32_t ws[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              uint32_t word = ws[e];
              while (word && r < D) {
                const int bp = __ffs(word) - 1;
                word &= word - 1;
                sv[w][myf][r++] = (uint16_t)(vb + (uint32_t)(j * 128 + e * 32 + bp));
              }
            }
          }
          for (int j = 0; j < nq; ++j) Bq[j] = make_uint4(0u, 0u, 0u, 0u);
          mycnt = min(D, mycnt + tot);
          mybase += Wv;
        }
        const unsigned done = __ballot_sync(0xffffffffu, sub == 0 && (mycnt >= D || mybase >= b));
        unsigned dn = 0;
#pragma unroll
        for (int f = 0; f < SK_FG; ++f) dn |= ((done >> (4 * f)) & 1u) << f;
        need &= ~dn;
        __syncwarp();
        Wv = SK_CAPW * 32;  // later windows (rare): the full capacity
      }
      // ---- out[f][u][0..D): lane 4f writes function f0+f's row (ABSENT past the values found)
      if (sub == 0 && myf < nf) {
        const uint4 q = *reinterpret_cast<const uint4 *>(sv[w][myf]);
        uint32_t s[C2_SKETCH_D] = {q.x & 0xFFFFu, q.x >> 16, q.y & 0xFFFFu, q.y >> 16,
                                   q.z & 0xFFFFu, q.z >> 16, q.w & 0xFFFFu, q.w >> 16};
#pragma unroll
        for (int j = 0; j < C2_SKETCH_D; ++j) s[j] = j < mycnt ? s[j] : C2_ABSENT16;
        uint16_t *o = out + ((int64_t)(f0 + myf) * n_total + u0 + u) * D;
        if (D == C2_SKETCH_D) {
          *reinterpret_cast<uint4 *>(o) = make_uint4(s[0] | (s[1] << 16), s[2] | (s[3] << 16), s[4] | (s[5] << 16),
                                                     s[6] | (s[7] << 16));
        } else {
#pragma unroll
          for (int j = 0; j < C2_SKETCH_D; ++j)
            if (j < D) o[j] = (uint16_t)s[j];
        }
      }
      __syncwarp();
    }
  }
}

template <int G>
static int launch_sketch(c2_ctx *ctx, const Csr &csr, int t, int f0, int b, const HashArgs &ha,
                         const uint16_t *htab, int32_t m, int D, uint16_t *out) {
  unsigned blocks = (unsigned)(((int64_t)csr.n * G + 255) / 256);
  if (htab)
    k_sketch<G, true, false><<<blocks, 256, 0, ctx->stream>>>(csr.offs, csr.items, csr.n, t, f0, (uint32_t)b, ha, htab, m,
                                                       D, out);
  else if (b >= 2 && (b & (b - 1)) == 0)
    k_sketch<G, false, true><<<blocks, 256, 0, ctx->stream>>>(csr.offs, csr.items, csr.n, t, f0, (uint32_t)b, ha,
                                                              nullptr, 0, D, out);
  else
    k_sketch<G, false, false><<<blocks, 256, 0, ctx->stream>>>(csr.offs, csr.items, csr.n, t, f0, (uint32_t)b, ha,
                                                               nullptr, 0, D, out);
  C2_LAUNCHED(ctx, "k_sketch");
  return C2_OK;
}

// users [u0, u1) of the hashed (no table) sketch, depth C2_SKETCH_D, into out [t][csr.n][D]
int sketch_range(c2_ctx *ctx, const Csr &csr, int t, int b, const HashParams *hp, int32_t u0, int32_t u1,
                 uint16_t *out) {
  HashArgs ha;
  for (int f = 0; f < t; ++f) {
    ha.a[f] = hp->a[f];
    ha.c[f] = hp->c[f];
  }
  const int32_t nloc = u1 - u0;
  if (nloc <= 0) return C2_OK;
  const bool pow2 = b >= 2 && (b & (b - 1)) == 0;
  auto kern = pow2 ? k_sketch_w<true> : k_sketch_w<false>;
  static int occ[2] = {0, 0};
  if (!occ[pow2]) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[pow2], kern, SK_WARPS * 32, 0);
  const unsigned grid = (unsigned)std::min<int64_t>((int64_t)ctx->num_sms * std::max(occ[pow2], 1),
                                                    ((int64_t)nloc + SK_WARPS - 1) / SK_WARPS);
  kern<<<grid, SK_WARPS * 32, 0, ctx->stream>>>(csr.offs + u0, csr.items, nloc, t, (uint32_t)b, ha, C2_SKETCH_D, out,
                                                 (int64_t)u0, (int64_t)csr.n, (int32_t)csr.nnz);
  C2_LAUNCHED(ctx, "k_sketch_w");
  return C2_OK;
}

int sketch(c2_ctx *ctx, const Csr &csr, int t, int b, const HashParams *hp, const uint16_t *htab, int32_t m, int D,
           uint16_t *out) {
  HashArgs ha;
  for (int f = 0; f < t; ++f) {
    ha.a[f] = hp ? hp->a[f] : 0;
    ha.c[f] = hp ? hp->c[f] : 0;
  }
  if (!htab && csr.n > 0) {
    // persistent grid: every block resident (users are taken in a grid-stride loop)
    const bool pow2 = b >= 2 && (b & (b - 1)) == 0;
    auto kern = pow2 ? k_sketch_w<true> : k_sketch_w<false>;
    static int occ[2] = {0, 0};
    if (!occ[pow2]) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[pow2], kern, SK_WARPS * 32, 0);
    const unsigned grid = (unsigned)std::min<int64_t>((int64_t)ctx->num_sms * std::max(occ[pow2], 1),
                                                      ((int64_t)csr.n + SK_WARPS - 1) / SK_WARPS);
    kern<<<grid, SK_WARPS * 32, 0, ctx->stream>>>(csr.offs, csr.items, csr.n, t, (uint32_t)b, ha, D, out, (int64_t)0,
                                                   (int64_t)csr.n, csr.nnz > 0 ? (int32_t)csr.nnz : INT32_MAX);
    C2_LAUNCHED(ctx, "k_sketch_w");
    return C2_OK;
  }
  for (int f0 = 0; f0 < t; f0 += 8) {
    int rem = t - f0;
    if (rem <= 2) C2_TRY(launch_sketch<2>(ctx, csr, t, f0, b, ha, htab, m, D, out));
    else if (rem <= 4) C2_TRY(launch_sketch<4>(ctx, csr, t, f0, b, ha, htab, m, D, out));
    else C2_TRY(launch_sketch<8>(ctx, csr, t, f0, b, ha, htab, m, D, out));
  }
  return C2_OK;
}

// ---------------------------------------------------------------- K6 GoldFinger encode
// F_u = OR over x in P_u of bit g(x), g(x) = floor(((a_g*x + c_g) mod 2^64) * 1024 / 2^64)
// (reading A19).  The fingerprint is materialised as the ascending list of its set
// bit positions, so the local kernel runs unchanged on it: |F_u AND F_v| is the size of the
// intersection of the two lists, pc(F_u) the list length.  Warp per user; word w of the
// 1024-bit vector is owned by lane w.
__global__ void __launch_bounds__(256) k_gf_bits(const int32_t *__restrict__ offs, const int32_t *__restrict__ items,
                                                 int32_t n, uint64_t ga, uint64_t gc, uint32_t *__restrict__ words,
                                                 int32_t *__restrict__ pc) {
  __shared__ uint32_t bm[8][32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (u >= n) return;
  bm[w][lane] = 0;
  __syncwarp();
  for (int32_t p = offs[u] + lane; p < offs[u + 1]; p += 32) {
    uint32_t bit = c2d::item_hash(ga, gc, (uint32_t)items[p], 1024u);
    atomicOr(&bm[w][bit >> 5], 1u << (bit & 31));
  }
  __syncwarp();
  uint32_t word = bm[w][lane];
  words[u * 32 + lane] = word;
  int c = __popc(word);
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) pc[u] = c;
}

__global__ void __launch_bounds__(256) k_gf_list(const uint32_t *__restrict__ words, const int32_t *__restrict__ goffs,
                                                 int32_t n, int32_t *__restrict__ gitems) {
  int lane = threadIdx.x & 31;
  int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (u >= n) return;
  uint32_t word = words[u * 32 + lane];
  int c = __popc(word);
  int pos = c2d::warp_incl_scan(c) - c + goffs[u];
  while (word) {
    int bpos = __ffs(word) - 1;
    word &= word - 1;
    gitems[pos++] = lane * 32 + bpos;
  }
}

int gf_encode(c2_ctx *ctx, const Csr &csr, const HashParams *hp, Csr *gf) {
  int rc;
  int n = csr.n;
  uint32_t *words = (uint32_t *)ws_get(ctx, "gf_words", (size_t)n * 128, &rc);
  if (rc) return rc;
  int32_t *pc = (int32_t *)ws_get(ctx, "gf_pc", (size_t)n * 4, &rc);
  if (rc) return rc;
  int32_t *goffs = (int32_t *)ws_get(ctx, "gf_offs", (size_t)(n + 1) * 4, &rc);
  if (rc) return rc;
  unsigned blocks = (unsigned)(((int64_t)n * 32 + 255) / 256);
  k_gf_bits<<<blocks, 256, 0, ctx->stream>>>(csr.offs, csr.items, n, hp->ga, hp->gc, words, pc);
  C2_LAUNCHED(ctx, "k_gf_bits");
  C2_TRY(scan_exclusive(ctx, pc, goffs, n));
  int32_t total;
  C2_CUDA(ctx, cudaMemcpyAsync(&total, goffs + n, 4, cudaMemcpyDeviceToHost, ctx->stream));
  C2_TRY(stream_sync(ctx, "gf_encode"));
  int32_t *gitems = (int32_t *)ws_get(ctx, "gf_items", (size_t)total * 4 + 16, &rc);
  if (rc) return rc;
  k_gf_list<<<blocks, 256, 0, ctx->stream>>>(words, goffs, n, gitems);
  C2_LAUNCHED(ctx, "k_gf_list");
  gf->offs = goffs;
  gf->items = gitems;
  gf->n = n;
  gf->nnz = total;
  gf->psize = pc;
  gf->max_item = 1023;
  gf->gf_words = words;
  gf->max_len = csr.max_len < 1024 ? csr.max_len : 1024;
  return C2_OK;
}

}  // namespace c2
