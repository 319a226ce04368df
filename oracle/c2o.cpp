// oracle/c2o.cpp -- plain, slow, obviously-correct CPU oracle of the C^2 hot path.
//
// TEST INFRASTRUCTURE ONLY (see c2o.h).  Written from the paper (PAPER.md, "P:n")
// and the readings listed in DESIGN.md ("A#").  No blocking, fusion or reordering
// beyond what the paper's definitions and algorithms state; std::sort / std::map are
// used as library steps.  std::thread is used only to run independent clusters/users
// concurrently (the paper's own thread pool over clusters); results do not
// depend on the thread count.
#include "c2o.h"

#include <algorithm>
#include <atomic>
#include <bitset>
#include <cstring>
#include <functional>
#include <map>
#include <thread>
#include <vector>

namespace {

// ---------------------------------------------------------------- helpers
inline bool row_ok(const int32_t *offs, const int32_t *items, int64_t n, int64_t m) {
  for (int64_t u = 0; u < n; ++u) {
    if (offs[u + 1] <= offs[u]) return false;  // empty profile (A17)
    for (int32_t p = offs[u]; p < offs[u + 1]; ++p) {
      if (items[p] < 0 || (m > 0 && items[p] >= m)) return false;
      if (p > offs[u] && items[p] <= items[p - 1]) return false;  // unsorted / duplicate (A18)
    }
  }
  return true;
}

template <class F>
void parallel_for(int64_t count, int nthreads, F fn) {
  if (nthreads < 1) nthreads = 1;
  std::atomic<int64_t> next(0);
  auto worker = [&]() {
    for (;;) {
      int64_t i = next.fetch_add(1);
      if (i >= count) break;
      fn(i);
    }
  };
  if (nthreads == 1) { worker(); return; }
  std::vector<std::thread> th;
  for (int q = 0; q < nthreads; ++q) th.emplace_back(worker);
  for (auto &x : th) x.join();
}

// |P_u ∩ P_v| by a two-pointer merge of the two sorted profiles.
int64_t intersect_sorted(const int32_t *a, int64_t na, const int32_t *b, int64_t nb) {
  int64_t i = 0, j = 0, c = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j]) ++i;
    else if (b[j] < a[i]) ++j;
    else { ++c; ++i; ++j; }
  }
  return c;
}

// The order of candidates (A13/A14): (v1,i1,U1) before (v2,i2,U2) iff i1/U1 > i2/U2,
// compared exactly as i1*U2 > i2*U1, ties broken by the lower id (BJ.north_star).
inline bool better(const c2o_cand &x, const c2o_cand &y) {
  int64_t l = (int64_t)x.inter * (int64_t)y.uni, r = (int64_t)y.inter * (int64_t)x.uni;
  if (l != r) return l > r;
  return x.id < y.id;
}

const c2o_cand PAD = {-1, 0, 0};

// Similarity "profiles": exact mode uses the item sets; GF mode the 1024-bit fingerprint
// F_u = OR of bits gtab[x] over x in P_u (A19).
struct Profiles {
  int64_t n;
  const int32_t *offs, *items;
  int mode;
  std::vector<std::bitset<C2O_GF_BITS>> fp;
  std::vector<int32_t> pc;
  Profiles(int64_t n_, const int32_t *o, const int32_t *it, int mode_, const uint16_t *gtab)
      : n(n_), offs(o), items(it), mode(mode_) {
    if (mode == 1) {
      fp.resize(n);
      pc.resize(n);
      for (int64_t u = 0; u < n; ++u) {
        for (int32_t p = offs[u]; p < offs[u + 1]; ++p) fp[u].set(gtab[items[p]]);
        pc[u] = (int32_t)fp[u].count();
      }
    }
  }
  int32_t size(int64_t u) const { return mode == 1 ? pc[u] : offs[u + 1] - offs[u]; }
  int32_t inter(int64_t u, int64_t v) const {
    if (mode == 1) return (int32_t)(fp[u] & fp[v]).count();
    return (int32_t)intersect_sorted(items + offs[u], offs[u + 1] - offs[u], items + offs[v], offs[v + 1] - offs[v]);
  }
  c2o_cand cand(int64_t u, int64_t v) const {
    int32_t i = inter(u, v);
    c2o_cand c;
    c.id = (int32_t)v;
    c.inter = (uint16_t)i;
    c.uni = (uint16_t)(size(u) + size(v) - i);  // |A ∪ B| = |A| + |B| - |A ∩ B|
    return c;
  }
};

// First min(k, cands.size()) candidates under the order, then padding (A14).
void write_topk(std::vector<c2o_cand> &cands, int k, c2o_cand *out) {
  std::sort(cands.begin(), cands.end(), better);
  for (int j = 0; j < k; ++j) out[j] = j < (int)cands.size() ? cands[j] : PAD;
}

// ---------------------------------------------------------------- clustering
struct ClusterSet {
  std::vector<std::vector<int32_t>> clusters;
  int64_t max_depth = 0, split_nodes = 0, folded = 0, residuals = 0;
};

// Formulation 0: the paper's recursive split.  A node C with index eta of size > N is
// split by H\eta(u) = min_{i in P_u, h(i) > eta} h(i); users for whom it is
// undefined (A6) and users alone in their new cluster (A7) stay in C, which is then
// emitted as a terminal residual (A8); new clusters larger than N are split again.
struct RecursiveSplit {
  const int32_t *offs, *items;
  const uint16_t *h;  // h_f row of the hash table
  int64_t N;
  ClusterSet *out;
  uint32_t h_excl(int32_t u, uint32_t eta) const {  // H\eta(u), C2O_ABSENT if undefined
    uint32_t best = C2O_ABSENT;
    for (int32_t p = offs[u]; p < offs[u + 1]; ++p) {
      uint32_t v = h[items[p]];
      if (v > eta && v < best) best = v;
    }
    return best;
  }
  void split(const std::vector<int32_t> &C, uint32_t eta, int64_t depth) {
    if ((int64_t)C.size() <= N) {  // strict "larger than N" trigger (A4)
      out->clusters.push_back(C);
      out->max_depth = std::max(out->max_depth, depth);
      return;
    }
    out->split_nodes++;
    std::map<uint32_t, std::vector<int32_t>> groups;
    std::vector<int32_t> residual;
    for (int32_t u : C) {
      uint32_t v = h_excl(u, eta);
      if (v == C2O_ABSENT) residual.push_back(u);
      else groups[v].push_back(u);
    }
    for (auto &g : groups) {
      if (g.second.size() == 1) { residual.push_back(g.second[0]); out->folded++; }
      else split(g.second, g.first, depth + 1);
    }
    if (!residual.empty()) {  // empty residual -> no cluster (A10)
      out->clusters.push_back(residual);
      out->residuals++;
      out->max_depth = std::max(out->max_depth, depth);
    }
  }
};

void cluster_recursive(int64_t n, const int32_t *offs, const int32_t *items, const uint16_t *h, int64_t N,
                       ClusterSet &cs) {
  // Alg. 1: B[H(u)] <- B[H(u)] ∪ {u}, H(u) = min_i h(i).
  std::map<uint32_t, std::vector<int32_t>> B;
  for (int64_t u = 0; u < n; ++u) {
    uint32_t H = C2O_ABSENT;
    for (int32_t p = offs[u]; p < offs[u + 1]; ++p) H = std::min<uint32_t>(H, h[items[p]]);
    B[H].push_back((int32_t)u);
  }
  RecursiveSplit rs{offs, items, h, N, &cs};
  for (auto &bk : B) rs.split(bk.second, bk.first, 0);  // root singletons emitted as-is (A11)
}

// Formulation 1: sorted-distinct-prefix trie.  S(u) = ascending distinct h values of P_u.
// A depth-d node is the set of users sharing (S[0..d]) minus ancestors' residuals; the
// next value inside a node of value S[d] is S[d+1] (second formulation).
void cluster_trie(int64_t n, const int32_t *offs, const int32_t *items, const uint16_t *h, int64_t N,
                  ClusterSet &cs) {
  std::vector<std::vector<uint32_t>> S(n);
  for (int64_t u = 0; u < n; ++u) {
    for (int32_t p = offs[u]; p < offs[u + 1]; ++p) S[u].push_back(h[items[p]]);
    std::sort(S[u].begin(), S[u].end());
    S[u].erase(std::unique(S[u].begin(), S[u].end()), S[u].end());
  }
  std::vector<int32_t> order(n);
  for (int64_t u = 0; u < n; ++u) order[u] = (int32_t)u;
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return S[a] < S[b]; });
  // value of user u at depth d, C2O_ABSENT past the end
  auto val = [&](int32_t u, int64_t d) -> uint32_t { return d < (int64_t)S[u].size() ? S[u][d] : C2O_ABSENT; };
  // process range [lo,hi) of `order` whose users share S[0..d]
  std::function<void(int64_t, int64_t, int64_t)> rec = [&](int64_t lo, int64_t hi, int64_t d) {
    if (hi - lo <= N) {
      cs.clusters.emplace_back(order.begin() + lo, order.begin() + hi);
      cs.max_depth = std::max(cs.max_depth, d);
      return;
    }
    cs.split_nodes++;
    std::vector<int32_t> residual;
    int64_t i = lo;
    while (i < hi) {
      uint32_t v = val(order[i], d + 1);
      int64_t j = i;
      while (j < hi && val(order[j], d + 1) == v) ++j;
      if (v == C2O_ABSENT) residual.insert(residual.end(), order.begin() + i, order.begin() + j);
      else if (j - i == 1) { residual.push_back(order[i]); cs.folded++; }
      else rec(i, j, d + 1);
      i = j;
    }
    if (!residual.empty()) {
      cs.clusters.push_back(residual);
      cs.residuals++;
      cs.max_depth = std::max(cs.max_depth, d);
    }
  };
  int64_t i = 0;
  while (i < n) {
    uint32_t v = val(order[i], 0);
    int64_t j = i;
    while (j < n && val(order[j], 0) == v) ++j;
    rec(i, j, 0);
    i = j;
  }
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

uint64_t c2o_splitmix64_next(uint64_t *state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

void c2o_hash_params(uint64_t seed, int t, uint64_t *a, uint64_t *c) {
  uint64_t st = seed;
  for (int f = 0; f < t; ++f) {
    a[f] = c2o_splitmix64_next(&st);
    c[f] = c2o_splitmix64_next(&st);
  }
}

void c2o_gf_params(uint64_t seed, uint64_t *a, uint64_t *c) {
  uint64_t st = seed ^ C2O_GF_SALT;
  *a = c2o_splitmix64_next(&st);
  *c = c2o_splitmix64_next(&st);
}

uint32_t c2o_item_hash(uint64_t a, uint64_t c, uint64_t x, uint32_t b) {
  uint64_t z = a * x + c;  // mod 2^64
  return (uint32_t)(((unsigned __int128)z * (unsigned __int128)b) >> 64);
}

int c2o_hash_table(uint64_t seed, int t, uint32_t b, int64_t m, uint16_t *htab) {
  if (t < 1 || b < 1 || b > 32768 || m < 0) return -1;
  std::vector<uint64_t> a(t), c(t);
  c2o_hash_params(seed, t, a.data(), c.data());
  for (int f = 0; f < t; ++f)
    for (int64_t x = 0; x < m; ++x) htab[f * m + x] = (uint16_t)c2o_item_hash(a[f], c[f], (uint64_t)x, b);
  return 0;
}

int c2o_gf_table(uint64_t seed, int64_t m, uint16_t *gtab) {
  uint64_t a, c;
  c2o_gf_params(seed, &a, &c);
  for (int64_t x = 0; x < m; ++x) gtab[x] = (uint16_t)c2o_item_hash(a, c, (uint64_t)x, C2O_GF_BITS);
  return 0;
}

int c2o_frh(int64_t n, const int32_t *offs, const int32_t *items, int t, int64_t m, const uint16_t *htab,
            int32_t *H) {
  if (!row_ok(offs, items, n, m)) return -2;
  for (int f = 0; f < t; ++f)
    for (int64_t u = 0; u < n; ++u) {
      uint32_t best = C2O_ABSENT;
      for (int32_t p = offs[u]; p < offs[u + 1]; ++p) best = std::min<uint32_t>(best, htab[f * m + items[p]]);
      H[f * n + u] = (int32_t)best;
    }
  return 0;
}

int c2o_sketch(int64_t n, const int32_t *offs, const int32_t *items, int t, int64_t m, const uint16_t *htab,
               int D, uint16_t *sk) {
  if (!row_ok(offs, items, n, m)) return -2;
  for (int f = 0; f < t; ++f)
    for (int64_t u = 0; u < n; ++u) {
      std::vector<uint16_t> s;
      for (int32_t p = offs[u]; p < offs[u + 1]; ++p) s.push_back(htab[f * m + items[p]]);
      std::sort(s.begin(), s.end());
      s.erase(std::unique(s.begin(), s.end()), s.end());
      for (int d = 0; d < D; ++d) sk[(f * n + u) * D + d] = d < (int)s.size() ? s[d] : (uint16_t)C2O_ABSENT;
    }
  return 0;
}

// Chunk guard (A9) + canonical form (A25) of one function's clusters; accumulates stats.
static void emit_canonical(int64_t n, ClusterSet &cs, int64_t N, int f, int32_t *offsets, int32_t *members,
                           int32_t *cluster_of, int32_t *n_clusters, int64_t *st) {
  // An emitted cluster larger than N is replaced by ceil(s/N) balanced chunks of its
  // ascending members.
  std::vector<std::vector<int32_t>> final_;
  for (auto &C : cs.clusters) {
    std::sort(C.begin(), C.end());
    int64_t s = (int64_t)C.size();
    if (s <= N) { final_.push_back(C); continue; }
    int64_t mc = (s + N - 1) / N;
    st[4]++;
    for (int64_t j = 0; j < mc; ++j)
      final_.emplace_back(C.begin() + (j * s) / mc, C.begin() + ((j + 1) * s) / mc);
  }
  // Canonical form (A25): clusters ordered by smallest member, members ascending.
  std::sort(final_.begin(), final_.end(),
            [](const std::vector<int32_t> &x, const std::vector<int32_t> &y) { return x[0] < y[0]; });
  int32_t *off = offsets + f * (n + 1);
  int32_t *mem = members + f * n;
  int32_t *cof = cluster_of + f * n;
  int64_t pos = 0;
  for (size_t c = 0; c < final_.size(); ++c) {
    off[c] = (int32_t)pos;
    for (int32_t u : final_[c]) { mem[pos++] = u; cof[u] = (int32_t)c; }
    int64_t s = (int64_t)final_[c].size();
    st[5] += s * (s - 1) / 2;  // P counts unordered pairs (A21)
    st[6] = std::max(st[6], s);
  }
  for (size_t c = final_.size(); c <= (size_t)n; ++c) off[c] = (int32_t)pos;
  n_clusters[f] = (int32_t)final_.size();
  st[0] += (int64_t)final_.size();
  st[1] = std::max(st[1], cs.max_depth);
  st[2] += cs.split_nodes;
  st[3] += cs.folded;
  st[7] += cs.residuals;
}

int c2o_cluster(int64_t n, const int32_t *offs, const int32_t *items, int t, int64_t m, const uint16_t *htab,
                int64_t N, int formulation, int32_t *offsets, int32_t *members, int32_t *cluster_of,
                int32_t *n_clusters, int64_t *stats) {
  if (N < 2 || t < 1) return -1;
  if (!row_ok(offs, items, n, m)) return -2;
  int64_t st[8] = {0};
  for (int f = 0; f < t; ++f) {
    ClusterSet cs;
    if (formulation == 0) cluster_recursive(n, offs, items, htab + f * m, N, cs);
    else cluster_trie(n, offs, items, htab + f * m, N, cs);
    emit_canonical(n, cs, N, f, offsets, members, cluster_of, n_clusters, st);
  }
  if (stats) std::memcpy(stats, st, sizeof(st));
  return 0;
}

int c2o_minhash_cluster(int64_t n, const int32_t *offs, const int32_t *items, int t, uint64_t seed, int64_t N,
                        int32_t *offsets, int32_t *members, int32_t *cluster_of, int32_t *n_clusters,
                        int64_t *stats) {
  if (N < 2 || t < 1) return -1;
  if (!row_ok(offs, items, n, 0)) return -2;
  std::vector<uint64_t> a(t), c(t);
  c2o_hash_params(seed, t, a.data(), c.data());
  int64_t st[8] = {0};
  for (int f = 0; f < t; ++f) {
    // MinHash: the full-range hash z_f(x) = a_f*x + c_f mod 2^64 (the
    // A1 family before range reduction) simulates a random permutation of the items; u's
    // cluster is the item of P_u that comes first, i.e. one cluster per item, no splitting.
    std::map<int32_t, std::vector<int32_t>> byitem;
    for (int64_t u = 0; u < n; ++u) {
      uint64_t best = ~0ULL;
      int32_t arg = -1;
      for (int32_t p = offs[u]; p < offs[u + 1]; ++p) {
        uint64_t z = a[f] * (uint64_t)items[p] + c[f];
        if (arg < 0 || z < best || (z == best && items[p] < arg)) { best = z; arg = items[p]; }
      }
      byitem[arg].push_back((int32_t)u);
    }
    ClusterSet cs;
    for (auto &g : byitem) cs.clusters.push_back(g.second);
    emit_canonical(n, cs, N, f, offsets, members, cluster_of, n_clusters, st);
  }
  if (stats) std::memcpy(stats, st, sizeof(st));
  return 0;
}

// SplitMix64 finalizer (the mixing function of c2o_splitmix64_next) used as a counter-based
// generator for Hyrec's random initial graph.
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// Hyrec on one cluster (Alg. 2 else-branch; reading A34 in DESIGN.md):
// start from a random k-degree graph over C, then repeatedly compare every user with the
// neighbours of its neighbours and keep the k best (synchronous iterations: all users read the
// previous iteration's graph); stop when fewer than delta*k*|C| neighbourhood entries changed
// (delta = 0.001) or after 30 iterations.  Output: k best-first lists.
static void hyrec_cluster(const Profiles &P, const int32_t *C, int64_t s, int f, int k, uint64_t seed,
                          c2o_cand *out_base, int64_t n, int64_t *iters_out) {
  std::map<int32_t, int64_t> local;
  for (int64_t a = 0; a < s; ++a) local[C[a]] = a;
  std::vector<std::vector<int32_t>> N(s);  // local indices
  for (int64_t a = 0; a < s; ++a) {
    const uint64_t key = mix64(mix64((seed ^ C2O_HYREC_SALT) + (uint64_t)f) + (uint64_t)C[a]);
    for (uint64_t j = 0; (int)N[a].size() < k; ++j) {
      const uint64_t r = mix64(key + j + 1);
      const int64_t b = (int64_t)(((unsigned __int128)r * (unsigned __int128)(uint64_t)s) >> 64);
      if (b == a || std::find(N[a].begin(), N[a].end(), (int32_t)b) != N[a].end()) continue;
      N[a].push_back((int32_t)b);
    }
  }
  std::vector<std::vector<c2o_cand>> L(s);
  int64_t it = 0;
  for (;;) {
    int64_t updates = 0;
    std::vector<std::vector<int32_t>> Nn(s);
    for (int64_t a = 0; a < s; ++a) {
      std::vector<int32_t> cand(N[a].begin(), N[a].end());
      for (int32_t b : N[a]) cand.insert(cand.end(), N[b].begin(), N[b].end());  // neighbours' neighbours
      std::sort(cand.begin(), cand.end());
      cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
      std::vector<c2o_cand> cs;
      for (int32_t b : cand)
        if (b != a) cs.push_back(P.cand(C[a], C[b]));
      std::sort(cs.begin(), cs.end(), better);
      cs.resize(std::min<size_t>(cs.size(), (size_t)k));
      for (const c2o_cand &x : cs) {
        const int32_t b = (int32_t)local[x.id];
        Nn[a].push_back(b);
        if (std::find(N[a].begin(), N[a].end(), b) == N[a].end()) ++updates;
      }
      L[a] = cs;
    }
    N.swap(Nn);
    ++it;
    if (updates * C2O_HYREC_DELTA_INV < (int64_t)k * s || it >= C2O_HYREC_MAX_ITERS) break;
  }
  for (int64_t a = 0; a < s; ++a)
    for (int j = 0; j < k; ++j) out_base[(int64_t)C[a] * k + j] = j < (int)L[a].size() ? L[a][j] : PAD;
  if (iters_out) *iters_out = it;
}

int c2o_local_knn2(int64_t n, const int32_t *offs, const int32_t *items, int t, const int32_t *offsets,
                   const int32_t *members, const int32_t *n_clusters, int k, int sim_mode, const uint16_t *gtab,
                   int64_t m, int nthreads, int solver, uint64_t seed, c2o_cand *cand, int64_t *hyrec_iters) {
  if (k < 1 || t < 1) return -1;
  if (!row_ok(offs, items, n, m)) return -2;
  Profiles P(n, offs, items, sim_mode, gtab);
  // work list of (f, cluster), largest first (the paper's decreasing priority queue)
  std::vector<std::pair<int64_t, std::pair<int, int32_t>>> work;
  for (int f = 0; f < t; ++f)
    for (int32_t c = 0; c < n_clusters[f]; ++c) {
      int64_t s = offsets[f * (n + 1) + c + 1] - offsets[f * (n + 1) + c];
      work.push_back({-s, {f, c}});
    }
  std::sort(work.begin(), work.end());
  std::atomic<int64_t> hit(0);
  parallel_for((int64_t)work.size(), nthreads, [&](int64_t w) {
    int f = work[w].second.first;
    int32_t c = work[w].second.second;
    const int32_t *C = members + f * n + offsets[f * (n + 1) + c];
    int64_t s = -work[w].first;
    // Alg. 2: brute force if |C| < rho k^2, else Hyrec -- with solver = 1 only; the
    // default (solver = 0) is brute force for every cluster (A12, BASELINE.json north_star).
    const bool hyrec = (solver == 1 && s >= (int64_t)C2O_HYREC_RHO * k * k) || (solver == 2 && s > k);
    if (hyrec) {
      int64_t its = 0;
      hyrec_cluster(P, C, s, f, k, seed, cand + (int64_t)f * n * k, n, &its);
      hit += its;
      return;
    }
    // Brute force: the s(s-1)/2 similarities of the cluster, each computed once.
    std::vector<c2o_cand> sims((size_t)(s * s));
    for (int64_t a = 0; a < s; ++a)
      for (int64_t b = a + 1; b < s; ++b) {
        c2o_cand x = P.cand(C[a], C[b]);
        sims[a * s + b] = x;
        x.id = C[a];
        sims[b * s + a] = x;
      }
    for (int64_t a = 0; a < s; ++a) {
      std::vector<c2o_cand> cands;
      for (int64_t b = 0; b < s; ++b)
        if (b != a) cands.push_back(sims[a * s + b]);  // self excluded (A15)
      write_topk(cands, k, cand + ((int64_t)f * n + C[a]) * k);
    }
  });
  if (hyrec_iters) *hyrec_iters = hit.load();
  return 0;
}

int c2o_local_knn(int64_t n, const int32_t *offs, const int32_t *items, int t, const int32_t *offsets,
                  const int32_t *members, const int32_t *n_clusters, int k, int sim_mode, const uint16_t *gtab,
                  int64_t m, int nthreads, c2o_cand *cand) {
  return c2o_local_knn2(n, offs, items, t, offsets, members, n_clusters, k, sim_mode, gtab, m, nthreads, 0, 0,
                        cand, nullptr);
}

int c2o_merge(int64_t n, int t, int k, const c2o_cand *cand, int nthreads, int32_t *nbr, uint16_t *inter,
              uint16_t *uni, float *sim) {
  if (k < 1 || t < 1) return -1;
  parallel_for(n, nthreads, [&](int64_t u) {
    // knn(u): a set bounded to k, keeping the k best seen (Alg. 3 line "heap bounded to k").
    std::vector<c2o_cand> knn;
    for (int f = 0; f < t; ++f) {          // for each hash function
      const c2o_cand *L = cand + ((int64_t)f * n + u) * k;
      for (int j = 0; j < k; ++j) {        // for (v, s) in knn'(u)
        const c2o_cand &e = L[j];
        if (e.id < 0) break;               // padding
        bool dup = false;                  // "reuse similarity values" (A16)
        for (auto &x : knn) if (x.id == e.id) dup = true;
        if (dup) continue;
        if ((int)knn.size() < k) { knn.push_back(e); continue; }
        size_t worst = 0;
        for (size_t q = 1; q < knn.size(); ++q) if (better(knn[worst], knn[q])) worst = q;
        if (better(e, knn[worst])) knn[worst] = e;
      }
    }
    std::sort(knn.begin(), knn.end(), better);
    for (int j = 0; j < k; ++j) {
      c2o_cand e = j < (int)knn.size() ? knn[j] : PAD;
      nbr[u * k + j] = e.id;
      inter[u * k + j] = e.inter;
      uni[u * k + j] = e.uni;
      if (sim) sim[u * k + j] = e.id < 0 ? 0.0f : (float)e.inter / (float)e.uni;
    }
  });
  return 0;
}

int c2o_knn_union_users(int64_t n, const int32_t *offs, const int32_t *items, int t, const int32_t *offsets,
                        const int32_t *members, const int32_t *cluster_of, int k, int sim_mode,
                        const uint16_t *gtab, int64_t m, int64_t n_sub, const int32_t *users, int nthreads,
                        int32_t *nbr, uint16_t *inter, uint16_t *uni) {
  if (!row_ok(offs, items, n, m)) return -2;
  Profiles P(n, offs, items, sim_mode, gtab);
  parallel_for(n_sub, nthreads, [&](int64_t q) {
    int64_t u = users[q];
    std::vector<int32_t> V;  // V(u) = U_f cluster_f(u) \ {u}
    for (int f = 0; f < t; ++f) {
      int32_t c = cluster_of[f * n + u];
      for (int32_t p = offsets[f * (n + 1) + c]; p < offsets[f * (n + 1) + c + 1]; ++p)
        if (members[f * n + p] != u) V.push_back(members[f * n + p]);
    }
    std::sort(V.begin(), V.end());
    V.erase(std::unique(V.begin(), V.end()), V.end());
    std::vector<c2o_cand> cands;
    for (int32_t v : V) cands.push_back(P.cand(u, v));
    std::vector<c2o_cand> out(k);
    write_topk(cands, k, out.data());
    for (int j = 0; j < k; ++j) { nbr[q * k + j] = out[j].id; inter[q * k + j] = out[j].inter; uni[q * k + j] = out[j].uni; }
  });
  return 0;
}

int c2o_knn_union(int64_t n, const int32_t *offs, const int32_t *items, int t, const int32_t *offsets,
                  const int32_t *members, const int32_t *cluster_of, int k, int sim_mode, const uint16_t *gtab,
                  int64_t m, int nthreads, int32_t *nbr, uint16_t *inter, uint16_t *uni) {
  std::vector<int32_t> all(n);
  for (int64_t u = 0; u < n; ++u) all[u] = (int32_t)u;
  return c2o_knn_union_users(n, offs, items, t, offsets, members, cluster_of, k, sim_mode, gtab, m, n, all.data(),
                             nthreads, nbr, inter, uni);
}

int c2o_exact_knn(int64_t n, const int32_t *offs, const int32_t *items, int k, int sim_mode,
                  const uint16_t *gtab, int64_t m, int64_t n_sub, const int32_t *users, int nthreads,
                  int32_t *nbr, uint16_t *inter, uint16_t *uni) {
  if (!row_ok(offs, items, n, m)) return -2;
  Profiles P(n, offs, items, sim_mode, gtab);
  parallel_for(n_sub, nthreads, [&](int64_t q) {
    int64_t u = users[q];
    std::vector<c2o_cand> cands;
    for (int64_t v = 0; v < n; ++v)
      if (v != u) cands.push_back(P.cand(u, v));
    std::vector<c2o_cand> out(k);
    write_topk(cands, k, out.data());
    for (int j = 0; j < k; ++j) { nbr[q * k + j] = out[j].id; inter[q * k + j] = out[j].inter; uni[q * k + j] = out[j].uni; }
  });
  return 0;
}

int c2o_pair_counts(int64_t n, const int32_t *offs, const int32_t *items, int64_t npairs, const int32_t *u,
                    const int32_t *v, int32_t *inter, int32_t *uni) {
  (void)n;
  for (int64_t q = 0; q < npairs; ++q) {
    int64_t a = u[q], b = v[q];
    int64_t i = intersect_sorted(items + offs[a], offs[a + 1] - offs[a], items + offs[b], offs[b + 1] - offs[b]);
    inter[q] = (int32_t)i;
    uni[q] = (int32_t)((offs[a + 1] - offs[a]) + (offs[b + 1] - offs[b]) - i);
  }
  return 0;
}

}  // extern "C"
