/* oracle/c2o.h -- CPU oracle for the Cluster-and-Conquer (C^2) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2010_11497_b200/, include/c2.h) never includes, links or calls it, and
 * this file shares no code, header, table or constant generator with it.
 *
 * Citations: "P:n" = line n of the paper text (arXiv 2010.11497, PAPER.md);
 * "A#" = reading number in DESIGN.md "Readings of the paper".
 *
 * Parity pins: see DESIGN.md "Oracle pins".  One function is "parity unpinned"
 * against the paper: the item hash h_f (the paper's Jenkins variant and seeds are
 * unspecified); it is pinned by definition (SplitMix64 reference vectors,
 * closed forms) and statistically (uniformity, Theorem 1).
 */
#ifndef C2O_H
#define C2O_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One candidate of a local or final neighbourhood: (v, |P_u ∩ P_v|, |P_u ∪ P_v|). Pad = {-1,0,0}. */
typedef struct {
  int32_t id;
  uint16_t inter;
  uint16_t uni;
} c2o_cand;

#define C2O_ABSENT 0xFFFFu
#define C2O_GF_BITS 1024
#define C2O_GF_SALT 0x476f6c6446696e67ULL /* "GoldFing" */
/* Alg. 2 hybrid: Hyrec for clusters with |C| >= rho k^2, rho = 5; delta = 0.001 and at
 * most 30 iterations; the initial random graph is drawn from SplitMix64-mixed counters
 * seeded with seed ^ C2O_HYREC_SALT (reading A34). */
#define C2O_HYREC_RHO 5
#define C2O_HYREC_DELTA_INV 1000
#define C2O_HYREC_MAX_ITERS 30
#define C2O_HYREC_SALT 0x4879726563526e67ULL /* "HyrecRng" */

/* SplitMix64 generator step (A2). */
uint64_t c2o_splitmix64_next(uint64_t *state);
/* Hash parameters of the t generative functions: draws a_0, c_0, a_1, c_1, ... (A2). */
void c2o_hash_params(uint64_t seed, int t, uint64_t *a, uint64_t *c);
/* GoldFinger hash parameters: SplitMix64 stream seeded with seed ^ C2O_GF_SALT (A19). */
void c2o_gf_params(uint64_t seed, uint64_t *a, uint64_t *c);
/* Generative hash h(x) = floor(((a*x + c) mod 2^64) * b / 2^64) in [0,b) (A1, A3). */
uint32_t c2o_item_hash(uint64_t a, uint64_t c, uint64_t x, uint32_t b);
/* htab[f][x] = h_f(x) for x in [0,m). */
int c2o_hash_table(uint64_t seed, int t, uint32_t b, int64_t m, uint16_t *htab);
/* gtab[x] = GoldFinger bit of item x in [0,1024). */
int c2o_gf_table(uint64_t seed, int64_t m, uint16_t *gtab);

/* H_f(u) = min_{i in P_u} h_f(i).  H is [t][n]. */
int c2o_frh(int64_t n, const int32_t *offs, const int32_t *items, int t, int64_t m, const uint16_t *htab,
            int32_t *H);
/* First D values of the ascending list of DISTINCT h_f values of P_u, padded with 0xFFFF.  [t][n][D]. */
int c2o_sketch(int64_t n, const int32_t *offs, const int32_t *items, int t, int64_t m, const uint16_t *htab,
               int D, uint16_t *sk);

/* Step 1 (Alg. 1 + recursive splitting) followed by the chunk guard (A9) and
 * the canonical form (A25).  formulation 0 = recursive H\eta split,
 * 1 = sorted-distinct-prefix trie (second formulation).
 * Outputs: offsets [t][n+1], members [t][n], cluster_of [t][n], n_clusters [t],
 * stats [8] = {clusters, max_depth, split_nodes, folded_singletons, chunked_residuals,
 *              pairs P, max_cluster_size, residual_clusters}. */
int c2o_cluster(int64_t n, const int32_t *offs, const int32_t *items, int t, int64_t m, const uint16_t *htab,
                int64_t N, int formulation, int32_t *offsets, int32_t *members, int32_t *cluster_of,
                int32_t *n_clusters, int64_t *stats);

/* C^2/MinHash variant: per function, users grouped by the item of their profile
 * with the smallest full-range hash z_f(x) = a_f*x + c_f mod 2^64 (ties: lower item id), i.e.
 * t x m clusters, no splitting.  N >= n keeps them whole (the paper's variant); a smaller N
 * applies the chunk guard (A9, reading A33).  Outputs and stats as c2o_cluster. */
int c2o_minhash_cluster(int64_t n, const int32_t *offs, const int32_t *items, int t, uint64_t seed, int64_t N,
                        int32_t *offsets, int32_t *members, int32_t *cluster_of, int32_t *n_clusters,
                        int64_t *stats);

/* Step 2, brute-force branch of Alg. 2: per cluster, all s(s-1)/2 similarities
 * (P:555), then per user the first min(k, s-1) candidates under the order (A13/A14), padded.
 * sim_mode 0 = exact sets, 1 = GoldFinger-1024 (gtab != NULL).  cand is [t][n][k]. */
int c2o_local_knn(int64_t n, const int32_t *offs, const int32_t *items, int t, const int32_t *offsets,
                  const int32_t *members, const int32_t *n_clusters, int k, int sim_mode, const uint16_t *gtab,
                  int64_t m, int nthreads, c2o_cand *cand);
/* As c2o_local_knn with the local solver selectable: solver 0 = brute force everywhere (A12),
 * 1 = Alg. 2 hybrid: brute force if |C| < rho k^2, else Hyrec; 2 = test hook: Hyrec for
 * every cluster with |C| > k.  hyrec_iters (nullable)
 * receives the total number of Hyrec iterations run. */
int c2o_local_knn2(int64_t n, const int32_t *offs, const int32_t *items, int t, const int32_t *offsets,
                   const int32_t *members, const int32_t *n_clusters, int k, int sim_mode, const uint16_t *gtab,
                   int64_t m, int nthreads, int solver, uint64_t seed, c2o_cand *cand, int64_t *hyrec_iters);

/* Step 3, Alg. 3: per user, add the t partial neighbourhoods into a set bounded
 * to k keeping the best, reusing similarity values; output sorted best-first, padded.
 * sim (nullable) = (float)inter / (float)uni, 0 for pads. */
int c2o_merge(int64_t n, int t, int k, const c2o_cand *cand, int nthreads, int32_t *nbr, uint16_t *inter,
              uint16_t *uni, float *sim);

/* Second formulation of Step 2+3: top-k of V(u) = U_f cluster_f(u) \ {u}. */
int c2o_knn_union(int64_t n, const int32_t *offs, const int32_t *items, int t, const int32_t *offsets,
                  const int32_t *members, const int32_t *cluster_of, int k, int sim_mode, const uint16_t *gtab,
                  int64_t m, int nthreads, int32_t *nbr, uint16_t *inter, uint16_t *uni);

/* Same for the users listed in `users` only (sampled parity at full size); outputs [n_sub][k]. */
int c2o_knn_union_users(int64_t n, const int32_t *offs, const int32_t *items, int t, const int32_t *offsets,
                        const int32_t *members, const int32_t *cluster_of, int k, int sim_mode,
                        const uint16_t *gtab, int64_t m, int64_t n_sub, const int32_t *users, int nthreads,
                        int32_t *nbr, uint16_t *inter, uint16_t *uni);

/* Exact KNN (brute force over all users) for the users listed in `users`
 * (n_sub of them); outputs are [n_sub][k]. */
int c2o_exact_knn(int64_t n, const int32_t *offs, const int32_t *items, int k, int sim_mode,
                  const uint16_t *gtab, int64_t m, int64_t n_sub, const int32_t *users, int nthreads,
                  int32_t *nbr, uint16_t *inter, uint16_t *uni);

/* Exact (inter, union) of explicit pairs, for quality (Eq. 1-2, A30). */
int c2o_pair_counts(int64_t n, const int32_t *offs, const int32_t *items, int64_t npairs, const int32_t *u,
                    const int32_t *v, int32_t *inter, int32_t *uni);

#ifdef __cplusplus
}
#endif
#endif
