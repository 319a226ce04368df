// k_sketch.cu -- K1 FastRandomHash sketch and K6 GoldFinger encode.
//
// K1: for every user u and function f, the D smallest DISTINCT values of {h_f(x) : x in P_u}
// (ascending, C2_ABSENT padded).  Element 0 is H_f(u) = min_{i in P_u} h_f(i); element
// d+1 is H\eta(u) with eta = element d (reading A5), so the recursive split never has to
// revisit the CSR while its depth stays below D (A29).  One pass over the item list computes
// all t functions (TF per pass), keeping a sorted distinct top-8 per function in registers.
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

int sketch(c2_ctx *ctx, const Csr &csr, int t, int b, const HashParams *hp, const uint16_t *htab, int32_t m, int D,
           uint16_t *out) {
  HashArgs ha;
  for (int f = 0; f < t; ++f) {
    ha.a[f] = hp ? hp->a[f] : 0;
    ha.c[f] = hp ? hp->c[f] : 0;
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
  gf->max_len = csr.max_len < 1024 ? csr.max_len : 1024;
  return C2_OK;
}

}  // namespace c2
