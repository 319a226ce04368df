// c2_api.cu -- the extern "C" entry points declared in include/c2.h.
#include <algorithm>
#include <cstring>

#include "c2_internal.cuh"

using namespace c2;

namespace {

int check_common(c2_ctx *ctx, const void *offs, const void *items, int32_t n, int32_t t) {
  if (!ctx) return C2_EINVAL;
  if (!offs || !items) return set_err(ctx, C2_EINVAL, "NULL CSR pointer");
  if (n < 1 || n >= (1 << 29)) return set_err(ctx, C2_EINVAL, "n_users=%d out of [1, 2^29)", n);
  if (t < 1 || t > C2_MAX_T) return set_err(ctx, C2_EINVAL, "t=%d out of [1, 64]", t);
  if ((int64_t)t * n >= INT32_MAX) return set_err(ctx, C2_EINVAL, "t*n_users must be < 2^31");
  return C2_OK;
}

int check_b_N(c2_ctx *ctx, int32_t b, int64_t N) {
  if (b < 1 || b > 32768) return set_err(ctx, C2_EINVAL, "b=%d out of [1, 32768]", b);
  if (N < 2) return set_err(ctx, C2_EINVAL, "max_cluster_N=%lld must be >= 2", (long long)N);
  return C2_OK;
}

int check_k(c2_ctx *ctx, int32_t k, int32_t sim_mode) {
  if (k < 1 || k > C2_MAX_K) return set_err(ctx, C2_EINVAL, "k=%d out of [1, 64]", k);
  if (sim_mode != C2_SIM_EXACT && sim_mode != C2_SIM_GF1024) return set_err(ctx, C2_EINVAL, "bad sim_mode");
  return C2_OK;
}

void begin(c2_ctx *ctx) {
  ctx->stats.launches = 0;
  ctx->stats.host_syncs = 0;
  ctx->stats.tile_launches = 0;
  ctx->stats.ms_tile = 0;
  ctx->tile_ev_used = 0;
  ctx->err[0] = 0;
  ctx->presketched = false;
  cudaSetDevice(ctx->device);
}

int cluster_buffers(c2_ctx *ctx, int t, int n, Clusters *cl) {
  int rc;
  cl->offsets = (int32_t *)ws_get(ctx, "cl_offsets", (size_t)t * (n + 1) * 4, &rc);
  if (rc) return rc;
  cl->members = (int32_t *)ws_get(ctx, "cl_members", (size_t)t * n * 4, &rc);
  if (rc) return rc;
  cl->cluster_of = (int32_t *)ws_get(ctx, "cl_cof", (size_t)t * n * 4, &rc);
  return rc;
}

__global__ void k_cl_maxsize(const int32_t *__restrict__ offsets, int t, int32_t n, const int32_t *__restrict__ ncl,
                             int32_t *__restrict__ out) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int v = 0;
  if (e < (int64_t)t * n) {
    int64_t f = e / n, c = e % n;
    if (c < ncl[f]) v = offsets[f * (n + 1) + c + 1] - offsets[f * (n + 1) + c];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, v);
}

__global__ void k_u16_max(const uint16_t *__restrict__ x, int64_t E, int32_t *__restrict__ out) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int v = e < E ? (int)x[e] : 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, v);
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// Steps 1-3 on device data.  ev[6] validation start, ev[0..3] step 1, ev[4] step 2, ev[5] step 3.
int build_device(c2_ctx *ctx, const int32_t *offs, const int32_t *items, int32_t n, int32_t t, int32_t b, int32_t N,
                 int32_t k, int32_t sim_mode, uint64_t seed, int32_t *nbr, uint16_t *inter, uint16_t *uni,
                 float *sim, const Csr *prevalidated = nullptr) {
  cudaStream_t st = ctx->stream;
  C2Range r_build("c2_build");
  if (ctx->timing && !prevalidated) cudaEventRecord(ctx->ev[6], st);
  Csr csr{offs, items, n, -1, 0, 0, nullptr};
  if (prevalidated) {
    csr = *prevalidated;  // c2_build_host: validated (and sketched) chunk by chunk during the upload
  } else {
    C2Range r("validate");
    C2_TRY(validate_csr(ctx, &csr));
  }
  HashParams hp;
  make_hash_params(seed, t, &hp, ctx->func_offset);
  Clusters cl;
  C2_TRY(cluster_buffers(ctx, t, n, &cl));
  {
    C2Range r("step1 clustering (FastRandomHash / MinHash)");
    if (ctx->clustering == 1) C2_TRY(minhash_clusters(ctx, csr, t, N, &hp, &cl));
    else C2_TRY(fastrandomhash(ctx, csr, t, b, N, &hp, nullptr, 0, &cl));
  }
  Csr sims = csr;
  if (sim_mode == C2_SIM_GF1024) C2_TRY(gf_encode(ctx, csr, &hp, &sims));
  ctx->hyrec_seed = seed;
  int rc;
  // Steps 2+3 fused: function by function, every local neighbourhood is merged into the
  // running Alg. 3 result; the final lists equal merge(local lists) exactly.
  c2_cand *run = (c2_cand *)ws_get(ctx, "runlist", (size_t)n * k * sizeof(c2_cand), &rc);
  if (rc) return rc;
  c2_cand *fin = nullptr;
  {
    C2Range r("step2+3 local top-k and Alg. 3 merge");
    C2_TRY(local_knn(ctx, sims, t, cl, k, run, true, &fin));
  }
  if (ctx->timing) cudaEventRecord(ctx->ev[4], st);
  C2Range r_out("copy-out");
  C2_TRY(copyout(ctx, n, k, fin, nbr, inter, uni, sim));
  if (ctx->timing) cudaEventRecord(ctx->ev[5], st);
  return C2_OK;
}

void collect_timing(c2_ctx *ctx) {
  if (!ctx->timing) return;
  cudaEventSynchronize(ctx->ev[5]);
  ctx->stats.ms_sketch = ev_ms(ctx->ev[0], ctx->ev[1]);
  ctx->stats.ms_cluster = ev_ms(ctx->ev[1], ctx->ev[3]);
  ctx->stats.ms_local = ev_ms(ctx->ev[3], ctx->ev[4]);
  ctx->stats.ms_merge = ev_ms(ctx->ev[4], ctx->ev[5]);
  ctx->stats.ms_total = ev_ms(ctx->ev[6], ctx->ev[5]);
  double mt = 0;
  for (int i = 0; i < ctx->tile_ev_used; ++i) mt += ev_ms(ctx->tile_ev[2 * i], ctx->tile_ev[2 * i + 1]);
  ctx->stats.ms_tile = mt;
}

}  // namespace

extern "C" {

int c2_ctx_create(c2_ctx **out, int device, void *cuda_stream) {
  if (!out) return C2_EINVAL;
  *out = nullptr;
  c2_ctx *ctx = new (std::nothrow) c2_ctx();
  if (!ctx) return C2_ENOMEM;
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    delete ctx;
    return C2_ECUDA;
  }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  ctx->smem_optin = optin;
  if (cuda_stream) {
    ctx->stream = (cudaStream_t)cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete ctx;
      return C2_ECUDA;
    }
    ctx->own_stream = true;
  }
  if (cudaMallocHost(&ctx->h_small, 4096) != cudaSuccess) {
    delete ctx;
    return C2_ENOMEM;
  }
  for (auto &e : ctx->ev) cudaEventCreate(&e);
  *out = ctx;
  return C2_OK;
}

void c2_ctx_destroy(c2_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto &kv : ctx->ws) cudaFree(kv.second.first);
  for (auto &e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto &e : ctx->tile_ev) cudaEventDestroy(e);
  if (ctx->side_stream) {
    cudaStreamSynchronize(ctx->side_stream);
    cudaStreamDestroy(ctx->side_stream);
    for (auto &e : ctx->side_ev)
      if (e) cudaEventDestroy(e);
  }
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
    for (auto &e : ctx->chunk_ev)
      if (e) cudaEventDestroy(e);
  }
  if (ctx->h_small) cudaFreeHost(ctx->h_small);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char *c2_last_error(const c2_ctx *ctx) { return ctx ? ctx->err : "NULL ctx"; }

int c2_ctx_set_option(c2_ctx *ctx, int key, int64_t value) {
  if (!ctx) return C2_EINVAL;
  switch (key) {
    case C2_OPT_SKETCH_DEPTH:
      if (value < 1 || value > C2_SKETCH_D) return set_err(ctx, C2_EINVAL, "sketch depth must be in [1, 8]");
      ctx->sketch_depth = (int)value;
      return C2_OK;
    case C2_OPT_SYNC_CHECK: ctx->sync_check = value != 0; return C2_OK;
    case C2_OPT_TIMING: ctx->timing = value != 0; return C2_OK;
    case C2_OPT_KSTATS: ctx->kstats = (unsigned long long *)(intptr_t)value; return C2_OK;
    case C2_OPT_RELABEL: ctx->relabel = value != 0; return C2_OK;
    case C2_OPT_SPLIT_DEVICE: ctx->split_dev = value != 0; return C2_OK;
    case C2_OPT_GF_TENSOR: ctx->gf_tensor = value != 0; return C2_OK;
    case C2_OPT_SURVIVORS:
      if (value < 0 || value > 4096) return set_err(ctx, C2_EINVAL, "survivor slots must be in [0, 4096]");
      ctx->surv_qmax = (int)value;
      return C2_OK;
    case C2_OPT_LOCAL_SOLVER:
      if (value != C2_SOLVER_BRUTE && value != C2_SOLVER_HYBRID) return set_err(ctx, C2_EINVAL, "bad local solver");
      ctx->solver = (int)value;
      return C2_OK;
    case C2_OPT_FUNC_OFFSET:
      if (value < 0 || value > (1 << 20)) return set_err(ctx, C2_EINVAL, "bad function offset");
      ctx->func_offset = (int)value;
      return C2_OK;
    case C2_OPT_CLUSTERING:
      if (value != C2_CLUSTER_FRH && value != C2_CLUSTER_MINHASH) return set_err(ctx, C2_EINVAL, "bad clustering");
      ctx->clustering = (int)value;
      return C2_OK;
    default: return set_err(ctx, C2_EINVAL, "unknown option %d", key);
  }
}

int c2_sketch(c2_ctx *ctx, const int32_t *csr_offsets, const int32_t *item_ids, int32_t n_users, int32_t t,
              int32_t b, uint64_t seed, int32_t D, uint16_t *sketch_out) {
  C2_TRY(check_common(ctx, csr_offsets, item_ids, n_users, t));
  C2_TRY(check_b_N(ctx, b, 2));
  if (D < 1 || D > C2_SKETCH_D || !sketch_out) return set_err(ctx, C2_EINVAL, "bad D or NULL output");
  begin(ctx);
  Csr csr{csr_offsets, item_ids, n_users, -1, 0, 0, nullptr};
  C2_TRY(validate_csr(ctx, &csr));
  HashParams hp;
  make_hash_params(seed, t, &hp, ctx->func_offset);
  return sketch(ctx, csr, t, b, &hp, nullptr, 0, D, sketch_out);
}

static int frh_common(c2_ctx *ctx, const int32_t *offs, const int32_t *items, int32_t n, int32_t t, int32_t b,
                      int32_t N, uint64_t seed, const uint16_t *htab, int32_t m, c2_clusters *out) {
  C2_TRY(check_common(ctx, offs, items, n, t));
  C2_TRY(check_b_N(ctx, b, N));
  if (!out || !out->offsets || !out->members || !out->cluster_of || !out->n_clusters)
    return set_err(ctx, C2_EINVAL, "NULL cluster output");
  begin(ctx);
  Csr csr{offs, items, n, -1, 0, 0, nullptr};
  C2_TRY(validate_csr(ctx, &csr));
  if (htab && csr.max_item >= m) return set_err(ctx, C2_EDATA, "item id %d >= table width m=%d", csr.max_item, m);
  if (htab) {  // every table value must be a bucket in [0, b) (it indexes per-bucket histograms)
    int rc;
    int32_t *mx = (int32_t *)ws_get(ctx, "htab_max", 4, &rc);
    if (rc) return rc;
    C2_CUDA(ctx, cudaMemsetAsync(mx, 0, 4, ctx->stream));
    const int64_t E = (int64_t)t * m;
    k_u16_max<<<(unsigned)((E + 255) / 256), 256, 0, ctx->stream>>>(htab, E, mx);
    C2_LAUNCHED(ctx, "k_u16_max");
    int32_t hmx = 0;
    C2_CUDA(ctx, cudaMemcpyAsync(&hmx, mx, 4, cudaMemcpyDeviceToHost, ctx->stream));
    C2_TRY(stream_sync(ctx, "table check"));
    if (hmx >= b) return set_err(ctx, C2_EINVAL, "hash table value %d >= b=%d", hmx, b);
  }
  HashParams hp;
  make_hash_params(seed, t, &hp, ctx->func_offset);
  Clusters cl;
  cl.offsets = out->offsets;
  cl.members = out->members;
  cl.cluster_of = out->cluster_of;
  if (ctx->clustering == 1 && !htab) C2_TRY(minhash_clusters(ctx, csr, t, N, &hp, &cl));
  else C2_TRY(fastrandomhash(ctx, csr, t, b, N, htab ? nullptr : &hp, htab, m, &cl));
  for (int f = 0; f < t; ++f) out->n_clusters[f] = cl.n_clusters[f];
  return C2_OK;
}

int c2_fastrandomhash(c2_ctx *ctx, const int32_t *csr_offsets, const int32_t *item_ids, int32_t n_users, int32_t t,
                      int32_t b, int32_t max_cluster_N, uint64_t seed, c2_clusters *out) {
  return frh_common(ctx, csr_offsets, item_ids, n_users, t, b, max_cluster_N, seed, nullptr, 0, out);
}

int c2_fastrandomhash_table(c2_ctx *ctx, const int32_t *csr_offsets, const int32_t *item_ids, int32_t n_users,
                            int32_t t, int32_t b, int32_t max_cluster_N, const uint16_t *htab, int32_t m,
                            c2_clusters *out) {
  if (!htab || m < 1) return set_err(ctx, C2_EINVAL, "NULL table or m < 1");
  return frh_common(ctx, csr_offsets, item_ids, n_users, t, b, max_cluster_N, 0, htab, m, out);
}

int c2_local_knn(c2_ctx *ctx, const int32_t *csr_offsets, const int32_t *item_ids, int32_t n_users, int32_t t,
                 const c2_clusters *clusters, int32_t k, int32_t sim_mode, uint64_t seed, c2_cand *cand) {
  C2_TRY(check_common(ctx, csr_offsets, item_ids, n_users, t));
  C2_TRY(check_k(ctx, k, sim_mode));
  if (!clusters || !clusters->offsets || !clusters->members || !clusters->cluster_of || !clusters->n_clusters || !cand)
    return set_err(ctx, C2_EINVAL, "NULL clusters (offsets, members, cluster_of, n_clusters) or cand");
  begin(ctx);
  Csr csr{csr_offsets, item_ids, n_users, -1, 0, 0, nullptr};
  C2_TRY(validate_csr(ctx, &csr));
  HashParams hp;
  make_hash_params(seed, t, &hp, ctx->func_offset);
  Clusters cl;
  cl.offsets = clusters->offsets;
  cl.members = clusters->members;
  cl.cluster_of = clusters->cluster_of;
  int rc;
  int32_t *ncl = (int32_t *)ws_get(ctx, "api_ncl", (C2_MAX_T + 2) * 4, &rc);
  if (rc) return rc;
  int32_t *mx = ncl + C2_MAX_T;
  for (int f = 0; f < t; ++f) {
    cl.n_clusters[f] = clusters->n_clusters[f];
    if (cl.n_clusters[f] < 1 || cl.n_clusters[f] > n_users) return set_err(ctx, C2_EINVAL, "bad n_clusters[%d]", f);
  }
  C2_CUDA(ctx, cudaMemcpyAsync(ncl, cl.n_clusters, t * 4, cudaMemcpyHostToDevice, ctx->stream));
  C2_CUDA(ctx, cudaMemsetAsync(mx, 0, 4, ctx->stream));
  int64_t TN = (int64_t)t * n_users;
  k_cl_maxsize<<<(unsigned)((TN + 255) / 256), 256, 0, ctx->stream>>>(cl.offsets, t, n_users, ncl, mx);
  C2_LAUNCHED(ctx, "k_cl_maxsize");
  int32_t hmx;
  C2_CUDA(ctx, cudaMemcpyAsync(&hmx, mx, 4, cudaMemcpyDeviceToHost, ctx->stream));
  C2_TRY(stream_sync(ctx, "cluster max size"));
  cl.max_size = hmx;
  Csr sims = csr;
  if (sim_mode == C2_SIM_GF1024) C2_TRY(gf_encode(ctx, csr, &hp, &sims));
  ctx->hyrec_seed = seed;
  return local_knn(ctx, sims, t, cl, k, cand, false, nullptr);
}

int c2_merge(c2_ctx *ctx, int32_t t, int32_t n_users, int32_t k, const c2_cand *cand, int32_t *nbr,
             uint16_t *inter, uint16_t *uni, float *sim) {
  if (!ctx) return C2_EINVAL;
  if (t < 1 || t > C2_MAX_T || n_users < 1 || (int64_t)t * n_users >= INT32_MAX)
    return set_err(ctx, C2_EINVAL, "bad t or n_users");
  C2_TRY(check_k(ctx, k, 0));
  if (!cand || !nbr || !inter || !uni) return set_err(ctx, C2_EINVAL, "NULL pointer");
  begin(ctx);
  return merge(ctx, t, n_users, k, cand, nbr, inter, uni, sim);
}

int c2_build(c2_ctx *ctx, const int32_t *csr_offsets, const int32_t *item_ids, int32_t n_users, int32_t t, int32_t b,
             int32_t max_cluster_N, int32_t k, int32_t sim_mode, uint64_t seed, int32_t *nbr, uint16_t *inter,
             uint16_t *uni, float *sim) {
  C2_TRY(check_common(ctx, csr_offsets, item_ids, n_users, t));
  C2_TRY(check_b_N(ctx, b, max_cluster_N));
  C2_TRY(check_k(ctx, k, sim_mode));
  if (!nbr || !inter || !uni) return set_err(ctx, C2_EINVAL, "NULL output");
  begin(ctx);
  C2_TRY(build_device(ctx, csr_offsets, item_ids, n_users, t, b, max_cluster_N, k, sim_mode, seed, nbr, inter, uni,
                      sim));
  collect_timing(ctx);
  return C2_OK;
}

int c2_build_host(c2_ctx *ctx, const int32_t *csr_offsets, const int32_t *item_ids, int32_t n_users, int32_t t,
                  int32_t b, int32_t max_cluster_N, int32_t k, int32_t sim_mode, uint64_t seed, int32_t *nbr,
                  uint16_t *inter, uint16_t *uni, float *sim) {
  C2_TRY(check_common(ctx, csr_offsets, item_ids, n_users, t));
  C2_TRY(check_b_N(ctx, b, max_cluster_N));
  C2_TRY(check_k(ctx, k, sim_mode));
  if (!nbr || !inter || !uni) return set_err(ctx, C2_EINVAL, "NULL output");
  begin(ctx);
  int64_t nnz = csr_offsets[n_users];
  if (nnz < 1 || csr_offsets[0] != 0) return set_err(ctx, C2_EDATA, "bad offsets");
  int rc;
  cudaStream_t st = ctx->stream;
  int32_t *d_offs = (int32_t *)ws_get(ctx, "host_offs", (size_t)(n_users + 1) * 4, &rc);
  if (rc) return rc;
  int32_t *d_items = (int32_t *)ws_get(ctx, "host_items", (size_t)nnz * 4, &rc);
  if (rc) return rc;
  size_t nk = (size_t)n_users * k;
  char *d_out = (char *)ws_get(ctx, "host_out", nk * (4 + 2 + 2 + 4), &rc);
  if (rc) return rc;
  int32_t *d_nbr = (int32_t *)d_out;
  float *d_sim = (float *)(d_out + nk * 4);
  uint16_t *d_inter = (uint16_t *)(d_out + nk * 8);
  uint16_t *d_uni = (uint16_t *)(d_out + nk * 10);
  // Upload in user chunks of ~equal item counts on a copy stream; each chunk is validated and
  // (FastRandomHash path) sketched on the compute stream as soon as it has arrived, so the PCIe
  // transfer overlaps Step 1's first kernels.  The validation result is read once at the end.
  if (!ctx->copy_stream) {
    C2_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (auto &e : ctx->chunk_ev) C2_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t cs = ctx->copy_stream;
  if (ctx->timing) cudaEventRecord(ctx->ev[6], st);
  C2_CUDA(ctx, cudaEventRecord(ctx->chunk_ev[15], st));  // earlier work on these buffers is done first
  C2_CUDA(ctx, cudaStreamWaitEvent(cs, ctx->chunk_ev[15], 0));
  const int nch = (int)std::min<int64_t>(8, n_users);
  HashParams hp;
  make_hash_params(seed, t, &hp, ctx->func_offset);
  const bool frh = ctx->clustering == 0;
  uint16_t *skb = nullptr;
  if (frh) {
    skb = (uint16_t *)ws_get(ctx, "sketch", (size_t)t * n_users * C2_SKETCH_D * 2, &rc);
    if (rc) return rc;
  }
  Csr csr{d_offs, d_items, n_users, nnz, -1, 0, nullptr};
  C2_TRY(validate_begin(ctx, n_users));
  int32_t u0 = 0;
  for (int c = 0; c < nch; ++c) {
    int32_t u1 = n_users;
    if (c + 1 < nch) {  // first user whose row starts at or after the chunk's share of the items
      const int64_t target = nnz * (c + 1) / nch;
      u1 = (int32_t)(std::lower_bound(csr_offsets + u0, csr_offsets + n_users, (int32_t)target) - csr_offsets);
      u1 = std::max(u1, u0 + 1);
    }
    const int64_t p0 = std::max<int64_t>(csr_offsets[u0], 0), p1 = std::min<int64_t>(csr_offsets[u1], nnz);
    C2_CUDA(ctx, cudaMemcpyAsync(d_offs + u0, csr_offsets + u0, (size_t)(u1 - u0 + 1) * 4, cudaMemcpyHostToDevice,
                                 cs));  // (offsets u0..u1: the chunk's rows and the end of its last row)
    if (p1 > p0)
      C2_CUDA(ctx, cudaMemcpyAsync(d_items + p0, item_ids + p0, (size_t)(p1 - p0) * 4, cudaMemcpyHostToDevice, cs));
    C2_CUDA(ctx, cudaEventRecord(ctx->chunk_ev[c], cs));
    C2_CUDA(ctx, cudaStreamWaitEvent(st, ctx->chunk_ev[c], 0));
    C2_TRY(validate_chunk(ctx, csr, u0, u1));
    if (frh) C2_TRY(sketch_range(ctx, csr, t, b, &hp, u0, u1, skb));
    if (u1 >= n_users) break;
    u0 = u1;
  }
  C2_TRY(validate_finish(ctx, &csr, nnz));
  ctx->presketched = frh;
  C2_TRY(build_device(ctx, d_offs, d_items, n_users, t, b, max_cluster_N, k, sim_mode, seed, d_nbr, d_inter, d_uni,
                      sim ? d_sim : nullptr, &csr));
  C2_CUDA(ctx, cudaMemcpyAsync(nbr, d_nbr, nk * 4, cudaMemcpyDeviceToHost, st));
  C2_CUDA(ctx, cudaMemcpyAsync(inter, d_inter, nk * 2, cudaMemcpyDeviceToHost, st));
  C2_CUDA(ctx, cudaMemcpyAsync(uni, d_uni, nk * 2, cudaMemcpyDeviceToHost, st));
  if (sim) C2_CUDA(ctx, cudaMemcpyAsync(sim, d_sim, nk * 4, cudaMemcpyDeviceToHost, st));
  C2_TRY(stream_sync(ctx, "build_host outputs"));
  collect_timing(ctx);
  return C2_OK;
}

int c2_get_stats(const c2_ctx *ctx, c2_stats *out) {
  if (!ctx || !out) return C2_EINVAL;
  *out = ctx->stats;
  return C2_OK;
}

}  // extern "C"
