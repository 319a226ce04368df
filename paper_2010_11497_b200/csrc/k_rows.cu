// k_rows.cu -- Step 2's per-row exact top-k (K8) and the light rows' Alg. 3 step, as kernels of
// their own, run after each k_local_tile launch.
//
// k_local_tile computes every tile's intersection counts |P_r ∩ P_v| (phase A) and splits its rows:
//   light rows (c2_build, running list full): screened in the tile's epilogue; the few cluster-mates
//       strictly better than the row's running k-th best are left in surv[u][..] -> k_surv_merge;
//   the other rows: their count row cnt[v] (u16, one entry per cluster member) and a RowRec go to
//       global memory -> k_row_topk.
// Both kernels are one warp per row/user with many warps per SM, so the latency-bound selection
// and merge steps of one row overlap other rows' instead of holding the tile's CTA barrier.
#include "cand.cuh"
#include "k_rows.cuh"

namespace c2 {

// ---------------------------------------------------------------- K8: exact top-k of one row
// Candidates of row u: the members v != u of its cluster (or of its slot group in a mixed slice),
// with i = cnt[v] = |P_u ∩ P_v| and U = |P_u| + |P_v| - i.  Output: the k best under the
// order (A13) -- written as the function's list (c2_local_knn) or merged with the row's running
// Alg. 3 list in place (c2_build).  Exactness: a candidate is queued only if it is not
// worse than a valid lower bound of the k-th best (the running k-th best, or the k-th best of any
// k distinct candidates); the queue is then sorted on exact keys (cand.cuh).
#ifndef C2_RM_KEYS
#define C2_RM_KEYS 1  // k <= 32: the <= 32-survivor Alg. 3 step by ranks on exact 64-bit keys (rank_merge_k1;
                      // c5: 51.3 vs 51.5 ms without)
#endif
#ifndef C2_R1_KO
#define C2_R1_KO 0  // 1: round 1's bound by a key-only sort, the payload fetched afterwards (measured at c5:
                    // 51.6 vs 51.3 ms with the payload carried through the sort -- off)
#endif
#ifndef C2_R1MUL
#define C2_R1MUL 2  // round 1 keeps C2_R1MUL * KS best candidates per lane
#endif
constexpr int RT_WARPS = 8;
constexpr int RT_QCAP = 256;  // survivor queue per warp (>= 64 * KS)

template <int KS>
#ifndef C2_RT_MINB
#define C2_RT_MINB 4
#endif
__global__ void __launch_bounds__(RT_WARPS * 32, C2_RT_MINB) k_row_topk(RowArgs a) {
  constexpr int R1 = C2_R1MUL * KS;
  __shared__ __align__(16) Cand s_q[RT_WARPS][RT_QCAP];
  __shared__ __align__(16) c2_cand s_run[RT_WARPS][C2_MAX_K];
  __shared__ int s_wq[RT_WARPS];
  __shared__ __align__(16) uint64_t s_kb[RT_WARPS][32];  // rank_merge_k1's key buffers
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kk = a.k;
  const int qcap = RT_QCAP;
  Cand *qr = s_q[warp];
  if (lane == 0) s_wq[warp] = 0;
  __syncwarp();
  const int64_t nrec = *a.nrec;
  for (int64_t ri = (int64_t)blockIdx.x * RT_WARPS + warp; ri < nrec; ri += (int64_t)gridDim.x * RT_WARPS) {
    const RowRec rec = a.recs[ri];
    const int32_t u = rec.u;
    const uint32_t prr = (uint32_t)rec.pr;
    const int s = rec.s;
    const int slot = rec.slot;
    const int selfr = rec.selfr;
    const uint16_t *cr = a.cnt + rec.cnt_off;
    const int32_t *vid = a.vperm + rec.vp_off;
    const int32_t *vps = a.vsize + rec.vp_off;
    // running list (fused): staged in shared memory, the output overwrites it in place
    if (a.seed) {
      for (int j = lane; j < kk; j += 32) s_run[warp][j] = a.seed[(int64_t)u * kk + j];
      __syncwarp();
    }
    const c2_cand *run = s_run[warp];
    const Cand tau = a.seed ? from_out(run[kk - 1]) : sent();
    // survivors of T (strictly better than tau, not worse than a round-1 bound) -> qr; returns
    // their number (only the first qcap are stored)
    auto scan = [&](const Ref &T) -> int {
      if (slot) {
        const int vi = rec.slot_lo + lane;
        bool ok = false;
        Cand x = sent();
        if (lane < slot && vi != selfr) {
          const int32_t id = vid[vi];
          if (id >= 0) {
            const uint32_t i = cr[vi], ps = (uint32_t)vps[vi];
            ok = passes(i, ps, id, T);
            x = Cand{i | ((prr + ps - i) << 16), id};
          }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (ok) qr[__popc(bal & ((1u << lane) - 1))] = x;
        return __popc(bal);
      }
      for (int base = 0; base < s; base += 128) {
        uint32_t iv[4], pv[4];
        int32_t dv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int v = base + 32 * e + lane;
          iv[e] = v < s ? cr[v] : 0u;
          pv[e] = v < s ? (uint32_t)vps[v] : 0u;
          dv[e] = v < s && v != selfr ? vid[v] : INT32_MAX;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (dv[e] != INT32_MAX && passes(iv[e], pv[e], dv[e], T)) {
            const int p = atomicAdd(&s_wq[warp], 1);
            if (p < qcap) qr[p] = Cand{iv[e] | ((prr + pv[e] - iv[e]) << 16), dv[e]};
          }
        }
      }
      __syncwarp();
      const int m = s_wq[warp];
      __syncwarp();
      if (lane == 0) s_wq[warp] = 0;
      __syncwarp();
      return m;
    };
    // k-th best of the first 64*KS queue entries (all distinct real candidates): a valid lower
    // bound of the row's k-th best
    auto kth_of_queue = [&]() -> Ref {
      KC e[2 * KS];
#pragma unroll
      for (int j = 0; j < 2 * KS; ++j) e[j] = to_kc(qr[32 * j + lane]);
      sort_kc<2 * KS>(e);
      return make_ref(kc_cand(warp_get<2 * KS>(e, kk - 1)), prr, true);
    };
    // round 1: every lane's best R1 candidates of its share; T_r = the k-th best of the 32*R1
    // tops (any k distinct candidates bound the row's k-th best from below)
    auto round1 = [&](Ref &T) {
      Cand t[R1];
#pragma unroll
      for (int j = 0; j < R1; ++j) t[j] = sent();
      Ref wr = make_ref(sent(), prr, false);
      for (int base = 0; base < s; base += 128) {  // four candidates per lane in flight
        uint32_t iv[4], pv[4];
        int32_t dv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int v = base + 32 * e + lane;
          iv[e] = v < s ? cr[v] : 0u;
          pv[e] = v < s ? (uint32_t)vps[v] : 0u;
          dv[e] = v < s && v != selfr ? vid[v] : INT32_MAX;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (dv[e] != INT32_MAX && passes(iv[e], pv[e], dv[e], wr)) {
            const Cand x{iv[e] | ((prr + pv[e] - iv[e]) << 16), dv[e]};
#pragma unroll
            for (int j = R1 - 1; j > 0; --j) {
              if (better_c(x, t[j - 1])) t[j] = t[j - 1];
              else if (better_c(x, t[j])) t[j] = x;
            }
            if (better_c(x, t[0])) t[0] = x;
            wr = make_ref(t[R1 - 1], prr, false);
          }
        }
      }
#if C2_R1_KO
      // the k-th best of the 32*R1 tops by a key-only sort; its (i, U) is then fetched from the
      // lane that holds it (keys are distinct for distinct ids)
      KO e[R1], e0[R1];
#pragma unroll
      for (int j = 0; j < R1; ++j) e0[j] = e[j] = KO{to_kc(t[j]).k};
      sort_ko<R1>(e);
      const uint64_t kT = warp_get<R1>(e, kk - 1).k;
      uint32_t iuT = 1u << 16;
#pragma unroll
      for (int j = 0; j < R1; ++j) {
        const unsigned hb = __ballot_sync(0xffffffffu, kT != 0ull && e0[j].k == kT);
        if (hb) iuT = __shfl_sync(0xffffffffu, t[j].iu, __ffs(hb) - 1);
      }
      const Cand Tc = kT != 0ull ? Cand{iuT, (int32_t)(0xFFFFFFFFu - (uint32_t)kT)} : sent();
      if (is_real(Tc) && better_c(Tc, tau)) T = make_ref(Tc, prr, true);
#else
      KC e[R1];
#pragma unroll
      for (int j = 0; j < R1; ++j) e[j] = to_kc(t[j]);
      sort_kc<R1>(e);
      const KC Tr = warp_get<R1>(e, kk - 1);
      if (kc_real(Tr) && better_c(kc_cand(Tr), tau)) T = make_ref(kc_cand(Tr), prr, true);
#endif
    };
    Ref T = make_ref(tau, prr, false);
    // rows without a running list yet (tau = sentinel) whose candidates cannot all be queued
    // start with round 1; rows whose tau lets too many through get it after the first scan
    bool r1 = !slot && !is_real(tau) && s - 1 > 64 * KS;
    if (r1) round1(T);
    int m = scan(T);
    int zn = min(m, qcap);
    if (a.kstats && lane == 0) atomicAdd(&a.kstats[16 + min(m, 300) / 20], 1ull);
    if (m > 64 * KS && !slot && !r1) {
      if (a.kstats && lane == 0) atomicAdd(&a.kstats[14], 1ull);
      r1 = true;
      round1(T);
      m = scan(T);
    }
    int rescans = 0;
    for (; rescans < 2 && m > qcap; ++rescans) {
      T = kth_of_queue();
      __syncwarp();
      m = scan(T);
    }
    // shrink a long queue in place: keep the entries not worse than the k-th best of its first
    // 64*KS (stops when that makes no progress: massive ties)
    while (m > 64 * KS && m <= qcap) {
      const Ref T2 = kth_of_queue();
      __syncwarp();
      int w = 0;
      for (int b0 = 0; b0 < m; b0 += 32) {
        const int j = b0 + lane;
        Cand x = j < m ? qr[j] : sent();
        const uint32_t i = x.iu & 0xFFFFu, ps = (x.iu >> 16) + i - prr;
        const bool ok = j < m && passes(i, ps, x.id, T2);
        __syncwarp();
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (ok) qr[w + __popc(bal & ((1u << lane) - 1))] = x;
        w += __popc(bal);
      }
      __syncwarp();
      if (w == m) break;
      m = w;
    }
    (void)zn;
    if (a.kstats && lane == 0) {
      atomicAdd(&a.kstats[0], 1ull);
      atomicAdd(&a.kstats[1], m == 0 ? 1ull : 0ull);
      atomicAdd(&a.kstats[2], (unsigned long long)m);
      atomicAdd(&a.kstats[3], m > 32 * KS ? 1ull : 0ull);
      atomicAdd(&a.kstats[4], (unsigned long long)rescans);
      atomicAdd(&a.kstats[6], r1 ? 1ull : 0ull);
      int ev = s - 1;  // pair evaluations of this row: its cluster-mates (debug work accounting)
      if (slot) {
        ev = -1;
        for (int j = 0; j < slot; ++j) ev += vid[rec.slot_lo + j] >= 0 ? 1 : 0;
      }
      atomicAdd(&a.kstats[70], (unsigned long long)ev);
    }
    c2_cand *dst = a.seed ? a.out + (int64_t)u * kk : a.out + ((int64_t)rec.f * a.n + u) * kk;
    if (a.seed && m == 0) continue;
    if (a.seed && m <= 32) {
      // few survivors: Alg. 3 step by ranks (no sorting network, no f64 keys)
#if C2_RM_KEYS
      if (KS == 1) rank_merge_k1(qr, m, run, kk, dst, s_kb[warp]);
      else rank_merge<KS>(qr, m, run, kk, dst);
#else
      rank_merge<KS>(qr, m, run, kk, dst);
#endif
      __syncwarp();
      continue;
    }
    KC L[KS];  // top-k of this function's survivors (sentinel padded)
    if (m <= 32 * KS) {
      KC q[KS];
#pragma unroll
      for (int j = 0; j < KS; ++j) q[j] = to_kc((32 * j + lane < m) ? qr[32 * j + lane] : sent());
      sort_kc<KS>(q);
#pragma unroll
      for (int j = 0; j < KS; ++j) L[j] = q[j];
    } else if (m <= 64 * KS) {
      KC q[2 * KS];
#pragma unroll
      for (int j = 0; j < 2 * KS; ++j) q[j] = to_kc((32 * j + lane < m) ? qr[32 * j + lane] : sent());
      sort_kc<2 * KS>(q);
#pragma unroll
      for (int j = 0; j < KS; ++j) L[j] = q[j];
    } else {
      // pathological ties: exact insertion over the row's candidates
      if (a.kstats && lane == 0) atomicAdd(&a.kstats[8], 1ull);
      Cand Lc[KS];
#pragma unroll
      for (int j = 0; j < KS; ++j) Lc[j] = sent();
      Cand thr = sent();
      for (int vb = 0; vb < s; vb += 32) {
        const int vi = vb + lane;
        Cand c = sent();
        if (vi < s) {
          const int32_t v = vid[vi];
          if (v >= 0 && vi != selfr && (slot == 0 || (vi - rec.slot_lo >= 0 && vi - rec.slot_lo < slot))) {
            const uint32_t ci = cr[vi];
            c = Cand{ci | ((prr + (uint32_t)vps[vi] - ci) << 16), v};
          }
        }
        const bool bt = is_real(c) && better_c(c, tau) && better_c(c, thr);
        unsigned mask = __ballot_sync(0xffffffffu, bt);
        while (mask) {
          const int l = __ffs(mask) - 1;
          mask &= mask - 1;
          const Cand x = shfl_c(c, l);
          if (!better_c(x, thr)) continue;
          warp_insert<KS>(Lc, x);
          thr = warp_get<KS>(Lc, kk - 1);
        }
      }
#pragma unroll
      for (int j = 0; j < KS; ++j) L[j] = to_kc(Lc[j]);
    }
    if (!a.seed || run[0].id < 0) {  // no running list (c2_local_knn, or a row's first cluster): L is the result
#pragma unroll
      for (int j = 0; j < KS; ++j)
        if (32 * j + lane < kk) dst[32 * j + lane] = kc_out(L[j]);
      __syncwarp();
      continue;
    }
    // merge with the running list S (best first): bitonic sequence L(first k) ++ reverse(S)
    KC S[KS];
#pragma unroll
    for (int j = 0; j < KS; ++j) S[j] = to_kc((32 * j + lane < kk) ? from_out(run[32 * j + lane]) : sent());
    KC mm[2 * KS];
#pragma unroll
    for (int j = 0; j < KS; ++j) mm[j] = (32 * j + lane < kk) ? L[j] : KC{0ull, 1u << 16};
#pragma unroll
    for (int j = 0; j < KS; ++j) mm[KS + j] = shfl_e(S[KS - 1 - j], 31 - lane);
    merge_kc<2 * KS>(mm);
    // drop adjacent duplicates (a repeated id carries identical values, A16); keep k
    int base = 0;
#pragma unroll
    for (int j = 0; j < 2 * KS; ++j) {
      const uint32_t lo = (uint32_t)mm[j].k;
      uint32_t prev = __shfl_up_sync(0xffffffffu, lo, 1);
      const uint32_t prevj = j > 0 ? __shfl_sync(0xffffffffu, (uint32_t)mm[j - 1].k, 31) : 0u;
      if (lane == 0) prev = prevj;
      const bool keep = kc_real(mm[j]) && (j + lane == 0 || lo != prev);
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      const int rank = base + __popc(bal & ((1u << lane) - 1));
      if (keep && rank < kk) dst[rank] = kc_out(mm[j]);
      base += __popc(bal);
    }
    for (int p = base + lane; p < kk; p += 32) dst[p] = c2_cand{-1, 0, 0};
    __syncwarp();
  }
}

// One Alg. 3 step on warp-held lists: S (best first, 32*KS positions, sentinel padded) becomes the
// first k distinct ids of S ∪ X, X = one candidate (or sentinel) per lane, by a bitonic sort of X on
// exact keys, a bitonic merge with S reversed and an adjacent-duplicate drop (A13, A16).
template <int KS>
__device__ __forceinline__ void sort_merge_step(Cand (&S)[KS], Cand x, int k, c2_cand *sbuf) {
  const int lane = threadIdx.x & 31;
  KC q[KS];
  q[0] = to_kc(x);
#pragma unroll
  for (int j = 1; j < KS; ++j) q[j] = KC{0ull, 1u << 16};
  sort_kc<KS>(q);
  KC mm[2 * KS];
#pragma unroll
  for (int j = 0; j < KS; ++j) mm[j] = (32 * j + lane < k) ? q[j] : KC{0ull, 1u << 16};
#pragma unroll
  for (int j = 0; j < KS; ++j) mm[KS + j] = shfl_e(to_kc(S[KS - 1 - j]), 31 - lane);
  merge_kc<2 * KS>(mm);
  int base = 0;
#pragma unroll
  for (int j = 0; j < 2 * KS; ++j) {
    const uint32_t lo = (uint32_t)mm[j].k;
    uint32_t prev = __shfl_up_sync(0xffffffffu, lo, 1);
    const uint32_t prevj = j > 0 ? __shfl_sync(0xffffffffu, (uint32_t)mm[j - 1].k, 31) : 0u;
    if (lane == 0) prev = prevj;
    const bool keep = kc_real(mm[j]) && (j + lane == 0 || lo != prev);
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    const int rank = base + __popc(bal & ((1u << lane) - 1));
    if (keep && rank < k) sbuf[rank] = kc_out(mm[j]);
    base += __popc(bal);
  }
  for (int p = base + lane; p < k; p += 32) sbuf[p] = c2_cand{-1, 0, 0};
  __syncwarp();
#pragma unroll
  for (int j = 0; j < KS; ++j) S[j] = (32 * j + lane < k) ? from_out(sbuf[32 * j + lane]) : sent();
  __syncwarp();
}

// ---------------------------------------------------------------- light rows' Alg. 3 step
// k_local_tile's phase-A epilogue left each light user's survivors -- its cluster-mates strictly
// better than its running k-th best -- in surv[u][0..qn[u]).  One warp per user with survivors:
// the running list S (full, best first) sits in registers (lane j holds S[32*jj + j]); survivors
// are read 32 at a time and those still strictly better than the current k-th best are merged in:
// a few by insertion (a duplicate id carries the same (i, U) and is skipped, A16), more by one
// sort-and-merge step.  The result is the first k distinct ids of S ∪ Q under the order (A13),
// whatever the survivors' order.
constexpr int SM_INSERT_MAX = 32;  // survivors of a chunk merged by insertion (more: sort + merge; at 6 the
                                   // sort-and-merge step measured slower at c5: 6.6 vs 5.9 ms over 8 launches)
#ifndef C2_SM_MERGE_MIN
#define C2_SM_MERGE_MIN 16
#endif
#ifndef C2_SM_RANK
#define C2_SM_RANK 2  // k <= 32: every survivor chunk merged by ranks (2: on exact 64-bit keys, 1: cross products;
                      // 0: insertion / bitonic merge below)
#endif
constexpr int SM_MERGE_MIN = C2_SM_MERGE_MIN;  // k <= 32: chunks with more survivors take the bitonic merge
                                               // (c5: threshold 4 57.6 ms, 8 56.3, 16 55.4, off 55.5)

template <int KS>
__global__ void __launch_bounds__(256) k_surv_merge(const c2_cand *__restrict__ surv, int32_t *__restrict__ qn,
                                                    int qmax, int32_t n, int k, c2_cand *__restrict__ run,
                                                    unsigned long long *kstats = nullptr) {
  __shared__ c2_cand s_buf[8][32 * KS];
  __shared__ __align__(16) uint64_t s_key[8][32];  // C2_SM_RANK == 2: kept survivors' keys
  const int lane = threadIdx.x & 31;
  c2_cand *sbuf = s_buf[threadIdx.x >> 5];
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwg = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // one user per warp and iteration (small configs: every user with survivors gets its own warp)
  for (int64_t u = gw; u < n; u += nwg) {
    const int m = qn[u];
    if (m <= 0) continue;
    __syncwarp();
    if (lane == 0) qn[u] = 0;
    if (m > qmax) continue;  // the row was handed to k_row_topk by its producer
    {
      c2_cand *Rw = run + u * k;
      Cand S[KS];
#pragma unroll
      for (int jj = 0; jj < KS; ++jj) S[jj] = (32 * jj + lane < k) ? from_out(Rw[32 * jj + lane]) : sent();
      Cand tau = warp_get<KS>(S, k - 1);
      const c2_cand *Q = surv + u * qmax;
      bool changed = false;
      for (int c0 = 0; c0 < m; c0 += 32) {
        Cand x = c0 + lane < m ? from_out(Q[c0 + lane]) : sent();
        bool ok = is_real(x) && better_c(x, tau);
        unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (!bal) continue;
        changed = true;
        if (KS == 1 && C2_SM_RANK) {
          // k <= 32, every chunk by ranks (independent comparisons, no serial insertion chain):
          // rs = the survivor's rank in S (binary search; a repeated id carries the same (i, U),
          // so its twin sits exactly at rs, A16), then over the kept survivors o: rq = the
          // survivor's rank among them, sh = lane's S entry's; new positions rs + rq and lane + sh
#if C2_SM_RANK == 2
          // exact 64-bit keys (cand.cuh to_kc: larger = better, distinct for distinct ids): the
          // binary search and the pairwise ranks are plain 64-bit compares; the kept survivors'
          // keys are compacted into shared memory and read back as broadcasts
          const uint64_t xk = to_kc(ok ? x : sent()).k, sk = to_kc(S[0]).k;
          int r = 0;
#pragma unroll
          for (int st = 16; st >= 1; st >>= 1) {
            const uint64_t o = __shfl_sync(0xffffffffu, sk, min(r + st - 1, 31));
            if (r + st <= 32 && o > xk) r += st;
          }
          const int32_t at_id = __shfl_sync(0xffffffffu, S[0].id, min(r, 31));
          ok = ok && !(r < 32 && at_id == x.id);
          const unsigned km = __ballot_sync(0xffffffffu, ok);
#ifdef C2_KSTATS_SURV  // diagnostic build: survivors still better than tau / of those, not yet in the list
          if (kstats && lane == 0) {
            atomicAdd(&kstats[75], (unsigned long long)__popc(bal));
            atomicAdd(&kstats[76], (unsigned long long)__popc(km));
          }
#endif
          const int nS = __popc(__ballot_sync(0xffffffffu, lane < k && is_real(S[0])));
          const int mk = __popc(km);
          uint64_t *kb = s_key[threadIdx.x >> 5];
          if (ok) kb[__popc(km & ((1u << lane) - 1u))] = xk;  // positions < mk
          if (lane >= mk) kb[lane] = 0ull;  // padding read by the last group of 4 (0: better than nothing)
          __syncwarp();
          int rq = 0, sh = 0;
          for (int j = 0; j < mk; j += 4) {
            const ulonglong2 k01 = *reinterpret_cast<const ulonglong2 *>(kb + j);
            const ulonglong2 k23 = *reinterpret_cast<const ulonglong2 *>(kb + j + 2);
            rq += (k01.x > xk) + (k01.y > xk) + (k23.x > xk) + (k23.y > xk);
            sh += (k01.x > sk) + (k01.y > sk) + (k23.x > sk) + (k23.y > sk);
          }
          __syncwarp();
#else
          int r = 0;
#pragma unroll
          for (int st = 16; st >= 1; st >>= 1) {
            const Cand o = shfl_c(S[0], min(r + st - 1, 31));
            if (r + st <= 32 && better_c(o, x)) r += st;
          }
          const Cand at = shfl_c(S[0], min(r, 31));
          ok = ok && !(r < 32 && at.id == x.id);
          const unsigned km = __ballot_sync(0xffffffffu, ok);
          const int nS = __popc(__ballot_sync(0xffffffffu, lane < k && is_real(S[0])));
          const uint32_t xi = x.iu & 0xFFFFu, xU = x.iu >> 16;
          const uint32_t si = S[0].iu & 0xFFFFu, sU = S[0].iu >> 16;
          int rq = 0, sh = 0;
          for (unsigned mm = km; mm; mm &= mm - 1u) {
            const int j = __ffs(mm) - 1;
            const uint32_t oiu = __shfl_sync(0xffffffffu, x.iu, j);
            const int32_t oid = __shfl_sync(0xffffffffu, x.id, j);
            const uint32_t oi = oiu & 0xFFFFu, oU = oiu >> 16;
            const uint32_t l1 = oi * xU, r1 = xi * oU;  // o before x?
            rq += (l1 > r1 || (l1 == r1 && oid < x.id)) ? 1 : 0;
            const uint32_t l2 = oi * sU, r2 = si * oU;  // o before lane's S entry?
            sh += (l2 > r2 || (l2 == r2 && oid < S[0].id)) ? 1 : 0;
          }
#endif
          if (ok && r + rq < k) sbuf[r + rq] = to_out(x);
          if (lane < nS && lane + sh < k) sbuf[lane + sh] = to_out(S[0]);
          for (int p = nS + __popc(km) + lane; p < k; p += 32) sbuf[p] = c2_cand{-1, 0, 0};
          __syncwarp();
          S[0] = lane < k ? from_out(sbuf[lane]) : sent();
          __syncwarp();
          tau = warp_get<KS>(S, k - 1);
          continue;
        }
        if (KS == 1 && __popc(bal) > SM_MERGE_MIN) {
          // k <= 32: drop the survivors already in S (binary search of S, best first: a repeated id
          // carries the same (i, U), so it sits exactly where the search ends, A16), sort the rest
          // best first, reverse them against S and keep the better of each pair (the 32 best of
          // S and Q as a bitonic sequence), then one bitonic merge
          int r = 0;
#pragma unroll
          for (int st = 16; st >= 1; st >>= 1) {
            const Cand o = shfl_c(S[0], min(r + st - 1, 31));
            if (r + st <= 32 && better_c(o, x)) r += st;
          }
          const Cand at = shfl_c(S[0], min(r, 31));
          ok = ok && !(r < 32 && at.id == x.id);
          Cand q[1] = {ok ? x : sent()};
          warp_sort<1>(q);
          const Cand qr = shfl_c(q[0], 31 - lane);  // worst first
          Cand mrg[1] = {better_c(qr, S[0]) ? qr : S[0]};
          warp_bitonic_merge<1>(mrg);
          S[0] = (lane < k) ? mrg[0] : sent();
          tau = warp_get<KS>(S, k - 1);
          continue;
        }
        if (__popc(bal) > SM_INSERT_MAX) {
          sort_merge_step<KS>(S, ok ? x : sent(), k, sbuf);
          tau = warp_get<KS>(S, k - 1);
          continue;
        }
        while (bal) {
          const int l = __ffs(bal) - 1;
          bal &= bal - 1u;
          const Cand y = shfl_c(x, l);
          if (!better_c(y, tau)) continue;  // (uniform)
          bool dup = false;
#pragma unroll
          for (int jj = 0; jj < KS; ++jj) dup |= S[jj].id == y.id;
          if (__any_sync(0xffffffffu, dup)) continue;
          warp_insert<KS>(S, y);
          tau = warp_get<KS>(S, k - 1);
        }
      }
      if (changed) {
#pragma unroll
        for (int jj = 0; jj < KS; ++jj)
          if (32 * jj + lane < k) Rw[32 * jj + lane] = to_out(S[jj]);
      }
    }
  }
}

int launch_row_topk(c2_ctx *ctx, const RowArgs &ra) {
  static int occ[2] = {0, 0};
  const int ks = ra.k <= 32 ? 0 : 1;
  auto kern = ks ? k_row_topk<2> : k_row_topk<1>;
  if (!occ[ks]) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[ks], kern, RT_WARPS * 32, 0);
  kern<<<ctx->num_sms * std::max(occ[ks], 1), RT_WARPS * 32, 0, ctx->stream>>>(ra);
  C2_LAUNCHED(ctx, "k_row_topk");
  return C2_OK;
}

int launch_surv_merge(c2_ctx *ctx, const c2_cand *surv, int32_t *qn, int qmax, int32_t n, int k, c2_cand *run,
                      cudaStream_t st) {
  // one resident wave: the grid-stride loop gives every block the same share of users, so blocks
  // beyond the resident ones would run as a second, partial wave
  static int occ[2] = {0, 0};
  const int ks = k <= 32 ? 0 : 1;
  auto kern = ks ? k_surv_merge<2> : k_surv_merge<1>;
  if (!occ[ks]) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[ks], kern, 256, 0);
  const int g = ctx->num_sms * std::max(occ[ks], 1);
  if (!st) st = ctx->stream;
#ifdef C2_KSTATS_SURV
  kern<<<g, 256, 0, st>>>(surv, qn, qmax, n, k, run, ctx->kstats);
#else
  kern<<<g, 256, 0, st>>>(surv, qn, qmax, n, k, run, nullptr);
#endif
  C2_LAUNCHED(ctx, "k_surv_merge");
  return C2_OK;
}

}  // namespace c2
