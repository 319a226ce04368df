// prims.cu -- ctx plumbing, device-wide scan, stable LSD radix sort, CSR validation (K0).
#include "c2_internal.cuh"

namespace c2 {

int set_err(c2_ctx *ctx, int code, const char *fmt, ...) {
  if (ctx) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(ctx->err, sizeof(ctx->err), fmt, ap);
    va_end(ap);
  }
  return code;
}

void *ws_get(c2_ctx *ctx, const char *name, size_t bytes, int *rc) {
  *rc = C2_OK;
  if (bytes == 0) bytes = 16;
  auto it = ctx->ws.find(name);
  if (it != ctx->ws.end() && it->second.second >= bytes) return it->second.first;
  if (it != ctx->ws.end()) {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(it->second.first);
    ctx->ws.erase(it);
  }
  void *p = nullptr;
  size_t want = bytes + bytes / 8;  // headroom so slowly growing inputs do not reallocate
  if (cudaMalloc(&p, want) != cudaSuccess) {
    cudaGetLastError();
    *rc = set_err(ctx, C2_ENOMEM, "cudaMalloc(%zu) failed for workspace '%s'", want, name);
    return nullptr;
  }
  ctx->ws[name] = {p, want};
  return p;
}

int after_launch(c2_ctx *ctx, const char *what) {
  ctx->stats.launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(ctx, C2_ECUDA, "launch of %s failed: %s", what, cudaGetErrorString(e));
  if (ctx->sync_check) {
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return set_err(ctx, C2_ECUDA, "%s failed: %s", what, cudaGetErrorString(e));
  }
  return C2_OK;
}

int stream_sync(c2_ctx *ctx, const char *what) {
  ctx->stats.host_syncs++;
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return set_err(ctx, C2_ECUDA, "sync after %s: %s", what, cudaGetErrorString(e));
  return C2_OK;
}

static uint64_t splitmix64(uint64_t *s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

void make_hash_params(uint64_t seed, int t, HashParams *hp, int f0) {
  uint64_t s = seed;  // A2: (a_0, c_0, a_1, c_1, ...) from one stream
  for (int f = 0; f < f0; ++f) {  // functions before the first one used (multi-GPU shards, N2)
    splitmix64(&s);
    splitmix64(&s);
  }
  for (int f = 0; f < t; ++f) {
    hp->a[f] = splitmix64(&s);
    hp->c[f] = splitmix64(&s);
  }
  uint64_t g = seed ^ C2_GF_SALT;
  hp->ga = splitmix64(&g);
  hp->gc = splitmix64(&g);
}

// ------------------------------------------------------------------ scan
constexpr int SCAN_T = 1024, SCAN_I = 4, SCAN_TILE = SCAN_T * SCAN_I;

// Block-wide exclusive scan of SCAN_I consecutive values per thread; returns the block total.
__device__ __forceinline__ int block_scan_excl(int (&v)[SCAN_I], int *sm_warp) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int sum = 0;
#pragma unroll
  for (int j = 0; j < SCAN_I; ++j) { int x = v[j]; v[j] = sum; sum += x; }
  int incl = c2d::warp_incl_scan(sum);
  if (lane == 31) sm_warp[w] = incl;
  __syncthreads();
  if (w == 0) {
    int x = lane < (SCAN_T / 32) ? sm_warp[lane] : 0;
    int y = c2d::warp_incl_scan(x);
    if (lane < SCAN_T / 32) sm_warp[lane] = y - x;
    if (lane == 31) sm_warp[32] = y;
  }
  __syncthreads();
  int base = sm_warp[w] + incl - sum;
#pragma unroll
  for (int j = 0; j < SCAN_I; ++j) v[j] += base;
  int total = sm_warp[32];
  __syncthreads();
  return total;
}

__global__ void k_scan_reduce(const int32_t *__restrict__ in, int64_t n, int32_t *__restrict__ part) {
  __shared__ int sm[33];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_I;
  int v[SCAN_I];
#pragma unroll
  for (int j = 0; j < SCAN_I; ++j) v[j] = base + j < n ? in[base + j] : 0;
  int tot = block_scan_excl(v, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void k_scan_down(const int32_t *__restrict__ in, int64_t n, const int32_t *__restrict__ part_scan,
                            int32_t *__restrict__ out) {
  __shared__ int sm[33];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_I;
  int v[SCAN_I];
#pragma unroll
  for (int j = 0; j < SCAN_I; ++j) v[j] = base + j < n ? in[base + j] : 0;
  block_scan_excl(v, sm);
  int off = part_scan ? part_scan[blockIdx.x] : 0;  // (nullptr: a single tile)
#pragma unroll
  for (int j = 0; j < SCAN_I; ++j)
    if (base + j <= n) out[base + j] = v[j] + off;  // out has n+1 entries
}

int scan_exclusive(c2_ctx *ctx, const int32_t *in, int32_t *out, int64_t n) {
  // out[n] is produced by the tile that contains index n (value = total).
  int64_t nb = (n + 1 + SCAN_TILE - 1) / SCAN_TILE;
  if (nb == 1) {  // one tile: one launch
    k_scan_down<<<1, SCAN_T, 0, ctx->stream>>>(in, n, nullptr, out);
    C2_LAUNCHED(ctx, "k_scan_down");
    return C2_OK;
  }
  int rc;
  // scratch names depend on depth so recursion does not alias
  static const char *names[4] = {"scan_p0", "scan_p1", "scan_p2", "scan_p3"};
  static thread_local int depth = 0;
  if (depth >= 4) return set_err(ctx, C2_EINVAL, "scan too large");
  int32_t *part = (int32_t *)ws_get(ctx, names[depth], (size_t)(2 * nb + 2) * 4, &rc);
  if (rc) return rc;
  int32_t *part_scan = part + nb + 1;
  k_scan_reduce<<<(unsigned)nb, SCAN_T, 0, ctx->stream>>>(in, n, part);
  C2_LAUNCHED(ctx, "k_scan_reduce");
  if (nb == 1) {
    C2_CUDA(ctx, cudaMemsetAsync(part_scan, 0, 4, ctx->stream));
  } else {
    depth++;
    int r = scan_exclusive(ctx, part, part_scan, nb);
    depth--;
    if (r) return r;
  }
  k_scan_down<<<(unsigned)nb, SCAN_T, 0, ctx->stream>>>(in, n, part_scan, out);
  C2_LAUNCHED(ctx, "k_scan_down");
  return C2_OK;
}

// ------------------------------------------------------------------ radix sort
constexpr int RS_T = 256, RS_I = 8, RS_TILE = RS_T * RS_I, RS_BITS = 5, RS_BINS = 1 << RS_BITS;

__global__ void k_radix_hist(const uint32_t *__restrict__ keys, int64_t n, int shift, int32_t *__restrict__ hist,
                             int nblocks) {
  __shared__ int cnt[RS_BINS];
  if (threadIdx.x < RS_BINS) cnt[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * RS_TILE;
  for (int j = threadIdx.x; j < RS_TILE; j += RS_T) {
    int64_t i = base + j;
    if (i < n) atomicAdd(&cnt[(keys[i] >> shift) & (RS_BINS - 1)], 1);
  }
  __syncthreads();
  if (threadIdx.x < RS_BINS) hist[(int64_t)threadIdx.x * nblocks + blockIdx.x] = cnt[threadIdx.x];
}

// Stable scatter: thread i owns tile elements [RS_I*i, RS_I*i + RS_I); counts per (digit,
// thread) are scanned digit-major then thread-major, which preserves input order.
__global__ void __launch_bounds__(RS_T) k_radix_scatter(const uint32_t *__restrict__ kin,
                                                        const uint32_t *__restrict__ vin, uint32_t *__restrict__ kout,
                                                        uint32_t *__restrict__ vout, int64_t n, int shift,
                                                        const int32_t *__restrict__ gbase, int nblocks) {
  __shared__ int cnt[RS_BINS * RS_T];
  __shared__ int sm_warp[RS_T / 32 + 1];
  for (int j = threadIdx.x; j < RS_BINS * RS_T; j += RS_T) cnt[j] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * RS_TILE + (int64_t)threadIdx.x * RS_I;
  uint32_t k[RS_I], v[RS_I];
  int loc[RS_I];
#pragma unroll
  for (int j = 0; j < RS_I; ++j) {
    bool ok = base + j < n;
    k[j] = ok ? kin[base + j] : 0;
    v[j] = ok ? vin[base + j] : 0;
    int d = (k[j] >> shift) & (RS_BINS - 1);
    loc[j] = ok ? cnt[d * RS_T + threadIdx.x]++ : 0;
  }
  __syncthreads();
  // exclusive scan over cnt[d*RS_T + i] (RS_BINS*RS_T entries; thread q owns RS_BINS consecutive)
  int run[RS_BINS];
  int s = 0;
#pragma unroll
  for (int j = 0; j < RS_BINS; ++j) { run[j] = s; s += cnt[threadIdx.x * RS_BINS + j]; }
  int incl = c2d::warp_incl_scan(s);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 31) sm_warp[w] = incl;
  __syncthreads();
  if (w == 0) {
    int x = lane < RS_T / 32 ? sm_warp[lane] : 0;
    int y = c2d::warp_incl_scan(x);
    if (lane < RS_T / 32) sm_warp[lane] = y - x;
  }
  __syncthreads();
  int off = sm_warp[w] + incl - s;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < RS_BINS; ++j) cnt[threadIdx.x * RS_BINS + j] = run[j] + off;
  __syncthreads();
  // per-digit start of this block's slice inside the digit's global range
  __shared__ int dstart[RS_BINS];
  if (threadIdx.x < RS_BINS) dstart[threadIdx.x] = gbase[(int64_t)threadIdx.x * nblocks + blockIdx.x] - cnt[threadIdx.x * RS_T];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < RS_I; ++j) {
    if (base + j < n) {
      int d = (k[j] >> shift) & (RS_BINS - 1);
      int64_t dst = (int64_t)dstart[d] + cnt[d * RS_T + threadIdx.x] + loc[j];
      kout[dst] = k[j];
      vout[dst] = v[j];
    }
  }
}

// One tile (n <= RS_TILE): every pass in one CTA, keys and values ping-ponging in shared memory;
// the same stable digit-major / thread-major ranking as k_radix_scatter.
__global__ void __launch_bounds__(RS_T) k_radix_small(const uint32_t *__restrict__ kin, const uint32_t *__restrict__ vin,
                                                      uint32_t *__restrict__ kout, uint32_t *__restrict__ vout, int n,
                                                      int passes) {
  extern __shared__ __align__(16) uint32_t rsm[];
  uint32_t *sk0 = rsm, *sv0 = rsm + RS_TILE, *sk1 = rsm + 2 * RS_TILE, *sv1 = rsm + 3 * RS_TILE;
  int *cnt = reinterpret_cast<int *>(rsm + 4 * RS_TILE);  // [RS_BINS][RS_T]
  __shared__ int sm_warp[RS_T / 32 + 1];
  for (int i = threadIdx.x; i < n; i += RS_T) {
    sk0[i] = kin[i];
    sv0[i] = vin[i];
  }
  const int base = threadIdx.x * RS_I;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int p = 0; p < passes; ++p) {
    const int shift = p * RS_BITS;
    for (int j = threadIdx.x; j < RS_BINS * RS_T; j += RS_T) cnt[j] = 0;
    __syncthreads();
    uint32_t k[RS_I], v[RS_I];
    int loc[RS_I];
#pragma unroll
    for (int j = 0; j < RS_I; ++j) {
      const bool ok = base + j < n;
      k[j] = ok ? sk0[base + j] : 0u;
      v[j] = ok ? sv0[base + j] : 0u;
      const int d = (k[j] >> shift) & (RS_BINS - 1);
      loc[j] = ok ? cnt[d * RS_T + threadIdx.x]++ : 0;
    }
    __syncthreads();
    int run[RS_BINS];
    int s = 0;
#pragma unroll
    for (int j = 0; j < RS_BINS; ++j) {
      run[j] = s;
      s += cnt[threadIdx.x * RS_BINS + j];
    }
    const int incl = c2d::warp_incl_scan(s);
    if (lane == 31) sm_warp[w] = incl;
    __syncthreads();
    if (w == 0) {
      const int x = lane < RS_T / 32 ? sm_warp[lane] : 0;
      const int y = c2d::warp_incl_scan(x);
      if (lane < RS_T / 32) sm_warp[lane] = y - x;
    }
    __syncthreads();
    const int off = sm_warp[w] + incl - s;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < RS_BINS; ++j) cnt[threadIdx.x * RS_BINS + j] = run[j] + off;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < RS_I; ++j) {
      if (base + j < n) {
        const int d = (k[j] >> shift) & (RS_BINS - 1);
        const int dst = cnt[d * RS_T + threadIdx.x] + loc[j];
        sk1[dst] = k[j];
        sv1[dst] = v[j];
      }
    }
    __syncthreads();
    uint32_t *t = sk0; sk0 = sk1; sk1 = t;
    t = sv0; sv0 = sv1; sv1 = t;
  }
  for (int i = threadIdx.x; i < n; i += RS_T) {
    kout[i] = sk0[i];
    vout[i] = sv0[i];
  }
}

int radix_sort_pairs(c2_ctx *ctx, const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                     uint32_t *vals_out, int64_t n, int bits) {
  if (n == 0) return C2_OK;
  if (n <= RS_TILE) {
    const int passes = std::max(1, (bits + RS_BITS - 1) / RS_BITS);
    const size_t sm = (size_t)(4 * RS_TILE + RS_BINS * RS_T) * 4;
    C2_CUDA(ctx, cudaFuncSetAttribute(k_radix_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_radix_small<<<1, RS_T, sm, ctx->stream>>>(keys_in, vals_in, keys_out, vals_out, (int)n, passes);
    C2_LAUNCHED(ctx, "k_radix_small");
    return C2_OK;
  }
  int passes = (bits + RS_BITS - 1) / RS_BITS;
  if (passes < 1) passes = 1;
  int nblocks = (int)((n + RS_TILE - 1) / RS_TILE);
  int rc;
  int32_t *hist = (int32_t *)ws_get(ctx, "rs_hist", (size_t)(RS_BINS * nblocks + 1) * 4 * 2, &rc);
  if (rc) return rc;
  int32_t *hscan = hist + RS_BINS * nblocks + 1;
  uint32_t *tk = (uint32_t *)ws_get(ctx, "rs_tk", (size_t)n * 4, &rc);
  if (rc) return rc;
  uint32_t *tv = (uint32_t *)ws_get(ctx, "rs_tv", (size_t)n * 4, &rc);
  if (rc) return rc;
  // ping-pong so that the final pass writes keys_out / vals_out
  const uint32_t *ki = keys_in, *vi = vals_in;
  for (int p = 0; p < passes; ++p) {
    bool last_to_out = ((passes - 1 - p) % 2) == 0;
    uint32_t *ko = last_to_out ? keys_out : tk;
    uint32_t *vo = last_to_out ? vals_out : tv;
    int shift = p * RS_BITS;
    k_radix_hist<<<nblocks, RS_T, 0, ctx->stream>>>(ki, n, shift, hist, nblocks);
    C2_LAUNCHED(ctx, "k_radix_hist");
    C2_TRY(scan_exclusive(ctx, hist, hscan, (int64_t)RS_BINS * nblocks));
    k_radix_scatter<<<nblocks, RS_T, 0, ctx->stream>>>(ki, vi, ko, vo, n, shift, hscan, nblocks);
    C2_LAUNCHED(ctx, "k_radix_scatter");
    ki = ko;
    vi = vo;
  }
  return C2_OK;
}

// ------------------------------------------------------------------ K0: validate CSR
// flags[0] = first bad row (INT32_MAX if none), flags[1] = max item, flags[2] = max length,
// flags[3] = nnz consistency (offsets[0] must be 0).
__global__ void k_validate(const int32_t *__restrict__ offs, const int32_t *__restrict__ items, int32_t n,
                           int32_t *__restrict__ psize, int32_t *__restrict__ flags, int32_t u_base,
                           const int32_t *__restrict__ last, int32_t nnz_known) {
  // users [u_base, u_base + n) of the CSR; offs and psize point at user u_base; nnz = nnz_known
  // if >= 0 (host entry point), else *last (the device CSR's final offset).  A row reaching
  // outside [0, nnz) is flagged before any of its items is read.
  const int32_t nnz = nnz_known >= 0 ? nnz_known : *last;
  int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int32_t mx_item = -1, mx_len = 0;
  for (int64_t u = warp; u < n; u += nwarps) {  // warp per user, coalesced row reads
    int32_t s = offs[u], e = offs[u + 1];
    int32_t len = e - s;
    bool bad = len <= 0 || len > 32767 || (u + u_base == 0 && s != 0) || s < 0 || e > nnz;
    for (int32_t p = s + lane; p < e && !bad; p += 32) {
      int32_t x = items[p];
      int32_t prev = p > s ? items[p - 1] : -1;
      bool b = x < 0 || x <= prev;
      if (__any_sync(__activemask(), b)) bad = true;
      mx_item = max(mx_item, x);
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      psize[u] = len;
      if (bad) atomicMin(&flags[0], (int32_t)(u + u_base));
    }
    mx_len = max(mx_len, len);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx_item = max(mx_item, __shfl_xor_sync(0xffffffffu, mx_item, o));
    mx_len = max(mx_len, __shfl_xor_sync(0xffffffffu, mx_len, o));
  }
  if (lane == 0) {
    atomicMax(&flags[1], mx_item);
    atomicMax(&flags[2], mx_len);
  }
}

__global__ void k_init_flags(int32_t *flags) {
  flags[0] = INT32_MAX;
  flags[1] = -1;
  flags[2] = 0;
  flags[3] = 0;
}

// Chunked form (c2_build_host overlaps the CSR upload with validation): validate_begin once,
// validate_chunk per user range as its rows arrive, validate_finish reads the flags (one sync).
int validate_begin(c2_ctx *ctx, int32_t n) {
  int rc;
  ws_get(ctx, "psize", (size_t)n * 4, &rc);
  if (rc) return rc;
  int32_t *flags = (int32_t *)ws_get(ctx, "vflags", 64, &rc);
  if (rc) return rc;
  k_init_flags<<<1, 1, 0, ctx->stream>>>(flags);
  C2_LAUNCHED(ctx, "k_init_flags");
  return C2_OK;
}
int validate_chunk(c2_ctx *ctx, const Csr &csr, int32_t u0, int32_t u1) {
  int rc;
  int32_t *psize = (int32_t *)ws_get(ctx, "psize", (size_t)csr.n * 4, &rc);
  if (rc) return rc;
  int32_t *flags = (int32_t *)ws_get(ctx, "vflags", 64, &rc);
  if (rc) return rc;
  k_validate<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(csr.offs + u0, csr.items, u1 - u0, psize + u0, flags, u0,
                                                         csr.offs + csr.n, (int32_t)csr.nnz);
  C2_LAUNCHED(ctx, "k_validate");
  return C2_OK;
}
int validate_finish(c2_ctx *ctx, Csr *csr, int64_t nnz) {
  int rc;
  int32_t *psize = (int32_t *)ws_get(ctx, "psize", (size_t)csr->n * 4, &rc);
  if (rc) return rc;
  int32_t *flags = (int32_t *)ws_get(ctx, "vflags", 64, &rc);
  if (rc) return rc;
  int32_t h[4];
  C2_CUDA(ctx, cudaMemcpyAsync(h, flags, 16, cudaMemcpyDeviceToHost, ctx->stream));
  C2_TRY(stream_sync(ctx, "validate"));
  if (h[0] != INT32_MAX)
    return set_err(ctx, C2_EDATA, "CSR row %d violates the input rules (empty, unsorted, duplicate, negative id or "
                   "|P_u| > 32767)", h[0]);
  csr->nnz = nnz;
  csr->max_item = h[1];
  csr->max_len = h[2];
  csr->psize = psize;
  return C2_OK;
}

int validate_csr(c2_ctx *ctx, Csr *csr) {
  int rc;
  int32_t *psize = (int32_t *)ws_get(ctx, "psize", (size_t)csr->n * 4, &rc);
  if (rc) return rc;
  int32_t *flags = (int32_t *)ws_get(ctx, "vflags", 64, &rc);
  if (rc) return rc;
  k_init_flags<<<1, 1, 0, ctx->stream>>>(flags);
  C2_LAUNCHED(ctx, "k_init_flags");
  int blocks = ctx->num_sms * 8;
  k_validate<<<blocks, 256, 0, ctx->stream>>>(csr->offs, csr->items, csr->n, psize, flags, 0, csr->offs + csr->n, -1);
  C2_LAUNCHED(ctx, "k_validate");
  int32_t h[5];
  C2_CUDA(ctx, cudaMemcpyAsync(h, flags, 16, cudaMemcpyDeviceToHost, ctx->stream));
  C2_CUDA(ctx, cudaMemcpyAsync(h + 4, csr->offs + csr->n, 4, cudaMemcpyDeviceToHost, ctx->stream));
  C2_TRY(stream_sync(ctx, "validate"));
  if (h[0] != INT32_MAX)
    return set_err(ctx, C2_EDATA, "CSR row %d violates the input rules (empty, unsorted, duplicate, negative id or "
                   "|P_u| > 32767)", h[0]);
  csr->nnz = h[4];
  csr->max_item = h[1];
  csr->max_len = h[2];
  csr->psize = psize;
  return C2_OK;
}

}  // namespace c2
