/* include/c2.h -- C ABI of the B200 (sm_100a) Cluster-and-Conquer (C^2) hot path.
 *
 * Problem (paper P:133-172, "P:n" = line n of PAPER.md, arXiv 2010.11497): users U with
 * item sets P_u; build an approximate KNN graph where each user gets k neighbours under
 * Jaccard similarity J(u,v) = |P_u ∩ P_v| / |P_u ∪ P_v|.  C^2 computes it in three
 * steps, one entry point each:
 *   c2_fastrandomhash  Step 1: FastRandomHash clustering, t configurations of b buckets,
 *                      H(u) = min_{i in P_u} h(i) (Alg. 1), clusters
 *                      larger than N recursively split with H\eta.
 *   c2_local_knn       Step 2: brute-force KNN inside every cluster (Alg. 2 brute branch,
 *                      P:549-577), s(s-1)/2 similarities per cluster.
 *   c2_merge           Step 3: Alg. 3, per user merge of the t partial
 *                      neighbourhoods keeping the k best, similarity values reused.
 * c2_build runs all three.  The readings of the paper (numbered A#) are listed in DESIGN.md.
 *
 * CONVENTIONS (all entry points)
 *  - Pointers marked "dev" are CUDA device memory on the ctx's device, OWNED BY THE CALLER;
 *    "host" pointers are ordinary host memory.  The library never frees caller memory; its
 *    scratch lives in the ctx (grown on demand, reused, freed by c2_ctx_destroy).
 *  - Work is enqueued on the ctx stream in order.  Entry points return after the work is
 *    enqueued, except where a host value is produced (n_clusters, stats), which costs one
 *    stream synchronisation; the recursive split also synchronises once per level.
 *  - CSR input: csr_offsets dev int32[n_users+1] (offsets[0] = 0), item_ids dev int32[nnz],
 *    each row non-empty, strictly ascending, ids >= 0, |P_u| <= 32767 (A17, A18, A28).
 *    Rows violating this make the call return C2_EDATA (first bad row in c2_last_error).
 *    Any id in [0, 2^31) is accepted; Step 2 renames ids densely (order-preserving, which leaves
 *    every intersection unchanged) when they exceed its 800,000-id window range, and returns
 *    C2_EDATA if the CSR holds more than 800,000 DISTINCT item ids.
 *  - Scalars: 1 <= t <= 64; 1 <= b <= 32768 (A26); N >= 2 (A27); 1 <= k <= 64;
 *    1 <= n_users < 2^29; t * n_users < 2^31.  Otherwise C2_EINVAL, nothing enqueued.
 *  - Errors: integer codes below; c2_last_error() describes the last failure of that ctx.
 *    On a non-OK return the outputs are unspecified.  No exceptions cross the ABI.
 *  - Determinism: outputs are a pure function of (CSR, t, b, N, k, seed, sim_mode), bit
 *    exact with the CPU oracle (tests/), independent of launch configuration.
 *  - One ctx per host thread; contexts are independent.
 */
#ifndef C2_H
#define C2_H
#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define C2_API __attribute__((visibility("default")))
#else
#define C2_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct c2_ctx c2_ctx;

/* One neighbour candidate: id, |P_u ∩ P_v|, |P_u ∪ P_v|.  Padding = {-1, 0, 0}.  8 bytes. */
typedef struct {
  int32_t id;
  uint16_t inter;
  uint16_t uni;
} c2_cand;

enum {
  C2_OK = 0,
  C2_EINVAL = -1, /* bad scalar parameter or NULL pointer */
  C2_EDATA = -2,  /* CSR rule violated */
  C2_ENOMEM = -3, /* device allocation failed */
  C2_ECUDA = -4   /* CUDA runtime error */
};

enum {
  C2_SIM_EXACT = 0,  /* exact set Jaccard */
  C2_SIM_GF1024 = 1  /* GoldFinger: 1024-bit fingerprint, bit = multiply-add-shift of the item
                        with the GF seed; J = popc(A&B)/(pc(A)+pc(B)-popc(A&B)) (A19) */
};

/* Hash parameters (A1, A2): h_f(x) = floor(((a_f*x + c_f) mod 2^64) * b / 2^64), where
 * (a_0,c_0,a_1,c_1,...) are consecutive outputs of SplitMix64 seeded with `seed`; the
 * GoldFinger function uses the stream seeded with seed ^ C2_GF_SALT and b = 1024. */
#define C2_GF_SALT 0x476f6c6446696e67ULL
#define C2_ABSENT 0xFFFFu /* sketch padding: no further distinct value */

/* ---------------------------------------------------------------- context */
/* Create a context on CUDA device `device`, enqueueing on `cuda_stream` (a cudaStream_t;
 * NULL -> the ctx creates and owns a non-blocking stream, NOT ordered with the legacy default
 * stream; pass cudaStreamLegacy, i.e. (void *)1, to enqueue on the legacy default stream).
 * *out receives the ctx. */
C2_API int c2_ctx_create(c2_ctx **out, int device, void *cuda_stream);
C2_API void c2_ctx_destroy(c2_ctx *ctx);
/* Message for the last non-OK return of this ctx (static storage owned by the ctx). */
C2_API const char *c2_last_error(const c2_ctx *ctx);

enum {
  C2_OPT_SKETCH_DEPTH = 1, /* 1..8: sketch values kept per (function,user); deeper split
                              levels recompute from the CSR (A29).  Default 8. */
  C2_OPT_SYNC_CHECK = 2,   /* nonzero: synchronise + check errors after every launch */
  C2_OPT_TIMING = 3,       /* nonzero: record per-phase CUDA-event times into c2_stats */
  C2_OPT_KSTATS = 4,       /* diagnostics: value = address of a dev uint64[80] the local kernel adds
                              counters to (rows, survivors, sort sizes, overflows; 0 = off) */
  C2_OPT_RELABEL = 5,      /* nonzero (default): when the item range needs >= 3 shared-memory windows,
                              Step 2 renumbers each cluster's shared items densely (one window per
                              tile); 0: always windows over the global item range.  Results are
                              identical either way. */
  C2_OPT_CLUSTERING = 6,   /* Step 1 of c2_fastrandomhash / c2_build: C2_CLUSTER_FRH (default) or
                              C2_CLUSTER_MINHASH (the paper's C^2/MinHash ablation) */
  C2_OPT_FUNC_OFFSET = 7,  /* f0 >= 0 (default 0): the t functions used are functions f0 .. f0+t-1 of the
                              seed's stream (A2), so G processes that each run t/G consecutive functions
                              together run exactly the functions of one t-function run (multi-GPU by
                              hash function; their merged lists equal the single run's, A16) */
  C2_OPT_LOCAL_SOLVER = 8, /* Step 2's per-cluster solver: C2_SOLVER_BRUTE (default, every cluster, A12) or
                              C2_SOLVER_HYBRID (Alg. 2: brute force if |C| < 5k^2, else Hyrec) */
  C2_OPT_GF_TENSOR = 10,   /* nonzero: in GoldFinger mode the intersections of clusters of more than 32
                              users are 0/1 contractions of the 1024-bit fingerprints on the tensor
                              cores (tcgen05.mma kind::i8, k_gf_mma); 0 (default, measured faster at c4):
                              the bit-sliced list kernel.  Results are identical either way. */
  C2_OPT_SPLIT_DEVICE = 11, /* nonzero (default): the recursive split runs as ONE cooperative
                              kernel looping over the levels on the device (no host synchronisation
                              per level) whenever its histogram bound (t*n/(N+1) * b bins) is at most
                              2^25; 0: one host-driven pass per level.  Results are identical. */
  C2_OPT_SURVIVORS = 9     /* c2_build only, 0..4096 (default 2048; halved while n*slots*8 B > 16 GiB): slots per user of the
                              light-row path (a row whose running list is full is screened in the
                              local kernel's epilogue and merged by a separate kernel; a row with more
                              survivors than slots gets its full count row and k_row_topk instead).  0: no
                              light rows.  Results are identical for every value. */
};
enum {
  C2_SOLVER_BRUTE = 0,
  C2_SOLVER_HYBRID = 1 /* Hyrec: random initial k-graph (SplitMix64-mixed counters from the call's
                          seed), synchronous neighbours-of-neighbours rounds until fewer than 0.001*k*|C|
                          entries change or 30 rounds; item ids must fit a shared-memory bitmap */
};
enum {
  C2_CLUSTER_FRH = 0,    /* FastRandomHash + recursive split */
  C2_CLUSTER_MINHASH = 1 /* per function, u's cluster = the item of P_u with the smallest full-range hash
                            z_f(x) = a_f*x + c_f mod 2^64 (ties: lower id): t x m clusters, no split; b is
                            ignored; clusters larger than N are cut into balanced chunks (A9; pass
                            N >= n_users for the paper's unbounded clusters).  Needs t*(max id+1) < 2^30. */
};
C2_API int c2_ctx_set_option(c2_ctx *ctx, int key, int64_t value);

/* ---------------------------------------------------------------- step 1 */
/* Canonical cluster assignment (A25): for function f, clusters are ordered by their
 * smallest member and members are ascending. */
typedef struct {
  int32_t *offsets;    /* dev [t][n_users+1]; cluster c of f = members[f][offsets[f][c] ..
                          offsets[f][c+1]), c < n_clusters[f]; offsets[f][c] = n_users for
                          c >= n_clusters[f] */
  int32_t *members;    /* dev [t][n_users] */
  int32_t *cluster_of; /* dev [t][n_users]: c such that u is in cluster c of f */
  int32_t *n_clusters; /* HOST [t]; written before return (one stream synchronisation) */
} c2_clusters;

/* Step 1: FastRandomHash clustering with recursive splitting.  Every cluster
 * ends with at most N users: a residual larger than N is cut into ceil(s/N) balanced chunks
 * of its ascending members (A9). */
C2_API int c2_fastrandomhash(c2_ctx *ctx, const int32_t *csr_offsets, const int32_t *item_ids, int32_t n_users,
                      int32_t t, int32_t b, int32_t max_cluster_N, uint64_t seed, c2_clusters *out);

/* As c2_fastrandomhash but h_f(x) = htab[f*m + x] (dev uint16 [t][m], values < b), for the
 * paper's worked examples.  Item ids must be < m (else C2_EDATA); a table
 * value >= b returns C2_EINVAL (checked on the device, one extra stream synchronisation). */
C2_API int c2_fastrandomhash_table(c2_ctx *ctx, const int32_t *csr_offsets, const int32_t *item_ids, int32_t n_users,
                            int32_t t, int32_t b, int32_t max_cluster_N, const uint16_t *htab, int32_t m,
                            c2_clusters *out);

/* Stage hook: sketch[f][u][0..D) = the D smallest DISTINCT values of {h_f(x) : x in P_u},
 * ascending, padded with C2_ABSENT (dev uint16 [t][n_users][D], 1 <= D <= 8).
 * sketch[f][u][0] = H_f(u); sketch[f][u][d+1] = H\sketch[f][u][d](u). */
C2_API int c2_sketch(c2_ctx *ctx, const int32_t *csr_offsets, const int32_t *item_ids, int32_t n_users, int32_t t,
              int32_t b, uint64_t seed, int32_t D, uint16_t *sketch);

/* ---------------------------------------------------------------- step 2 */
/* Step 2: for every cluster C of every function and every u in C, the first min(k,|C|-1)
 * users v in C \ {u} under the order "v1 before v2 iff i1*U2 > i2*U1, ties by lower id"
 * (i = |P_u ∩ P_v|, U = |P_u ∪ P_v|; A13-A15), padded with {-1,0,0}.
 * cand: dev [t][n_users][k], list of (f,u) at cand[(f*n_users + u)*k].  `clusters` must be
 * a canonical assignment of the same CSR (e.g. from c2_fastrandomhash; n_clusters host); all
 * four of its pointers are required (NULL -> C2_EINVAL).
 * sim_mode C2_SIM_GF1024 uses the fingerprints derived from `seed` (A19). */
C2_API int c2_local_knn(c2_ctx *ctx, const int32_t *csr_offsets, const int32_t *item_ids, int32_t n_users, int32_t t,
                 const c2_clusters *clusters, int32_t k, int32_t sim_mode, uint64_t seed, c2_cand *cand);

/* ---------------------------------------------------------------- step 3 */
/* Step 3 (Alg. 3): per user the first k distinct ids of the union of its t lists under the
 * same order; a repeated id always carries the same (inter, uni) (A16).  cand as produced
 * by c2_local_knn (each list sorted best-first, pads last).  Outputs dev [n_users][k]:
 * nbr (id or -1), inter, uni; sim (nullable) = (float)inter/(float)uni (IEEE div.rn), 0 for
 * pads. */
C2_API int c2_merge(c2_ctx *ctx, int32_t t, int32_t n_users, int32_t k, const c2_cand *cand, int32_t *nbr,
             uint16_t *inter, uint16_t *uni, float *sim);

/* ---------------------------------------------------------------- whole path */
/* Steps 1-3 on device-resident inputs; outputs as c2_merge.  Cluster arrays and candidate
 * lists live in ctx scratch. */
C2_API int c2_build(c2_ctx *ctx, const int32_t *csr_offsets, const int32_t *item_ids, int32_t n_users, int32_t t,
             int32_t b, int32_t max_cluster_N, int32_t k, int32_t sim_mode, uint64_t seed, int32_t *nbr,
             uint16_t *inter, uint16_t *uni, float *sim);

/* As c2_build with HOST inputs and outputs (nnz = csr_offsets[n_users]).  The CSR is uploaded
 * in up to 8 user chunks on a ctx-owned copy stream; each chunk is validated and (FastRandomHash
 * clustering) sketched on the ctx stream as soon as it has arrived, so the transfer overlaps
 * Step 1; the outputs come back on the ctx stream.  Host buffers may be pageable or pinned
 * (pinned: full PCIe rate); sim may be NULL.  A rule violation in any chunk returns C2_EDATA
 * with that row's index.  Returns after the outputs are in host memory. */
C2_API int c2_build_host(c2_ctx *ctx, const int32_t *csr_offsets, const int32_t *item_ids, int32_t n_users, int32_t t,
                  int32_t b, int32_t max_cluster_N, int32_t k, int32_t sim_mode, uint64_t seed, int32_t *nbr,
                  uint16_t *inter, uint16_t *uni, float *sim);

/* ---------------------------------------------------------------- stats */
typedef struct {
  int64_t pairs;             /* P = sum over functions and clusters of s(s-1)/2 (A21) */
  int64_t clusters;          /* total clusters over all functions */
  int64_t max_cluster_size;
  int64_t split_nodes;       /* nodes split by H\eta */
  int64_t max_depth;         /* deepest split level that created a cluster */
  int64_t folded_singletons; /* users alone in their new cluster, kept in the parent (A7) */
  int64_t chunked_residuals; /* residuals larger than N cut by the chunk guard (A9) */
  int64_t launches;          /* kernels launched by the last entry point */
  int64_t host_syncs;        /* stream synchronisations in the last entry point */
  double ms_sketch, ms_cluster, ms_local, ms_merge, ms_total; /* with C2_OPT_TIMING */
  int64_t work_steps;    /* sum over unordered local pairs of |P_u|+|P_v|: the element comparisons of
                            a two-pointer intersection (algorithmic work unit of Step 2) */
  int64_t tile_launches; /* launches of the local tile kernel (K7) in the last call */
  double ms_tile;        /* with C2_OPT_TIMING: summed CUDA-event duration of those launches */
} c2_stats;
/* Statistics of the last c2_fastrandomhash / c2_local_knn / c2_merge / c2_build call. */
C2_API int c2_get_stats(const c2_ctx *ctx, c2_stats *out);

#ifdef __cplusplus
}
#endif
#endif
