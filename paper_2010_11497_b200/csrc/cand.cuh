// cand.cuh -- candidate lists of the local top-k (K8) and the Alg. 3 merge: the exact order of
// candidates (A13: i1*U2 > i2*U1, ties by lower id), warp-held sorted lists, sorting networks on
// exact 64-bit keys, insertion and rank-based merges.  Shared by k_local.cu (the tile kernel's
// phase-A epilogue) and k_rows.cu (per-row top-k and the light-row merge).
#pragma once
#include "c2_internal.cuh"

namespace c2 {

// ------------------------------------------------------------------ candidate lists
// A candidate (v, i, U) is held as {iu = i | U << 16, id}.  The order (A13): a before b iff
// a.i * b.U > b.i * a.U, ties by lower id.  SENT is worse than every real candidate.
struct Cand {
  uint32_t iu;
  int32_t id;
};
__device__ __forceinline__ Cand sent() { return Cand{1u << 16, INT32_MAX}; }
__device__ __forceinline__ bool is_real(Cand a) { return a.id != INT32_MAX; }
__device__ __forceinline__ bool better_c(Cand a, Cand b) {
  uint32_t l = (a.iu & 0xFFFFu) * (b.iu >> 16), r = (b.iu & 0xFFFFu) * (a.iu >> 16);
  return l > r || (l == r && a.id < b.id);
}
__device__ __forceinline__ Cand shfl_c(Cand a, int src) {
  return Cand{__shfl_sync(0xffffffffu, a.iu, src), __shfl_sync(0xffffffffu, a.id, src)};
}
__device__ __forceinline__ Cand shfl_xor_c(Cand a, int m) {
  return Cand{__shfl_xor_sync(0xffffffffu, a.iu, m), __shfl_xor_sync(0xffffffffu, a.id, m)};
}
__device__ __forceinline__ Cand shfl_up_c(Cand a) {
  return Cand{__shfl_up_sync(0xffffffffu, a.iu, 1), __shfl_up_sync(0xffffffffu, a.id, 1)};
}
__device__ __forceinline__ c2_cand to_out(Cand a) {
  return is_real(a) ? c2_cand{a.id, (uint16_t)(a.iu & 0xFFFFu), (uint16_t)(a.iu >> 16)} : c2_cand{-1, 0, 0};
}
__device__ __forceinline__ Cand from_out(c2_cand e) {
  return e.id >= 0 ? Cand{(uint32_t)e.inter | ((uint32_t)e.uni << 16), e.id} : sent();
}

// Sort key of a candidate: K = q32 << 32 | (2^32 - 1 - id), larger = better, where
// q32 = floor(i/U * 2^32) (U >= 1; 2^32 - 1 for i == U) from the IEEE (correctly rounded) f64
// quotient.  K orders candidates exactly as the fraction comparison (A13): equal fractions
// give identical quotients; distinct fractions with U <= 65534 differ by >= 1/65534^2, i.e. by
// >= 1.00006 after scaling by 2^32, far above the f64 rounding error (< 2^-20), so their
// floors differ.  The payload iu = i | U << 16 rides along.  Sentinel: K = 0.
struct KC {
  uint64_t k;
  uint32_t iu;
};
__device__ __forceinline__ KC to_kc(Cand c) {
  if (!is_real(c)) return KC{0ull, 1u << 16};
  const uint32_t i = c.iu & 0xFFFFu, U = c.iu >> 16;
  const double q = (double)i / (double)U;
  const uint32_t q32 = i >= U ? 0xFFFFFFFFu : (uint32_t)(q * 4294967296.0);
  return KC{((uint64_t)q32 << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)c.id), c.iu};
}
__device__ __forceinline__ int32_t kc_id(KC a) { return (int32_t)(0xFFFFFFFFu - (uint32_t)a.k); }
__device__ __forceinline__ bool kc_real(KC a) { return a.k != 0ull; }
__device__ __forceinline__ Cand kc_cand(KC a) { return kc_real(a) ? Cand{a.iu, kc_id(a)} : sent(); }
__device__ __forceinline__ c2_cand kc_out(KC a) {
  return kc_real(a) ? c2_cand{kc_id(a), (uint16_t)(a.iu & 0xFFFFu), (uint16_t)(a.iu >> 16)} : c2_cand{-1, 0, 0};
}
__device__ __forceinline__ bool better_e(KC a, KC b) { return a.k > b.k; }
__device__ __forceinline__ bool better_e(Cand a, Cand b) { return better_c(a, b); }
__device__ __forceinline__ KC shfl_e(KC a, int src) {
  return KC{__shfl_sync(0xffffffffu, a.k, src), __shfl_sync(0xffffffffu, a.iu, src)};
}
__device__ __forceinline__ KC shfl_xor_e(KC a, int m) {
  return KC{__shfl_xor_sync(0xffffffffu, a.k, m), __shfl_xor_sync(0xffffffffu, a.iu, m)};
}
__device__ __forceinline__ KC shfl_up_e(KC a) {
  return KC{__shfl_up_sync(0xffffffffu, a.k, 1), __shfl_up_sync(0xffffffffu, a.iu, 1)};
}
// Key-only element (the key's payload looked up afterwards): one 64-bit shuffle per exchange
struct KO {
  uint64_t k;
};
__device__ __forceinline__ bool better_e(KO a, KO b) { return a.k > b.k; }
__device__ __forceinline__ KO shfl_e(KO a, int src) { return KO{__shfl_sync(0xffffffffu, a.k, src)}; }
__device__ __forceinline__ KO shfl_xor_e(KO a, int m) { return KO{__shfl_xor_sync(0xffffffffu, a.k, m)}; }
__device__ __forceinline__ KO shfl_up_e(KO a) { return KO{__shfl_up_sync(0xffffffffu, a.k, 1)}; }
__device__ __forceinline__ Cand shfl_e(Cand a, int src) { return shfl_c(a, src); }
__device__ __forceinline__ Cand shfl_xor_e(Cand a, int m) { return shfl_xor_c(a, m); }
__device__ __forceinline__ Cand shfl_up_e(Cand a) { return shfl_up_c(a); }

// Bitonic sort of the 32R warp-held elements a[j] (position 32j + lane), best first.
template <int R, class E>
__device__ __forceinline__ void warp_sort(E (&a)[R]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32 * R; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const int js = stride >> 5;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          if ((j & js) == 0) {
            const int p = 32 * j + lane;
            const bool desc = (p & size) == 0;  // lower position takes the better element
            E x = a[j], y = a[j + js];
            if (desc ? better_e(y, x) : better_e(x, y)) {
              a[j] = y;
              a[j + js] = x;
            }
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int p = 32 * j + lane;
          E o = shfl_xor_e(a[j], stride);
          const bool lower = (lane & stride) == 0;
          const bool desc = (p & size) == 0;
          // lower position of a descending block keeps the better one
          if ((lower == desc) ? better_e(o, a[j]) : better_e(a[j], o)) a[j] = o;
        }
      }
    }
  }
}

// Bitonic merge of a bitonic sequence of 32R warp-held elements into best-first order.
template <int R, class E>
__device__ __forceinline__ void warp_bitonic_merge(E (&a)[R]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int stride = 16 * R; stride > 0; stride >>= 1) {
    if (stride >= 32) {
      const int js = stride >> 5;
#pragma unroll
      for (int j = 0; j < R; ++j)
        if ((j & js) == 0 && better_e(a[j + js], a[j])) {
          E x = a[j];
          a[j] = a[j + js];
          a[j + js] = x;
        }
    } else {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        E o = shfl_xor_e(a[j], stride);
        const bool lower = (lane & stride) == 0;
        if (lower ? better_e(o, a[j]) : better_e(a[j], o)) a[j] = o;
      }
    }
  }
}

// Insert x into the sorted warp list a (32R positions, best first); the worst drops out.
template <int R, class E>
__device__ __forceinline__ void warp_insert(E (&a)[R], E x) {
  const int lane = threadIdx.x & 31;
  int pos = 0;
#pragma unroll
  for (int j = 0; j < R; ++j) pos += __popc(__ballot_sync(0xffffffffu, better_e(a[j], x)));
  E up[R];
#pragma unroll
  for (int j = 0; j < R; ++j) up[j] = shfl_up_e(a[j]);
#pragma unroll
  for (int j = 1; j < R; ++j) {
    E last = shfl_e(a[j - 1], 31);
    if (lane == 0) up[j] = last;
  }
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int p = 32 * j + lane;
    if (p == pos) a[j] = x;
    else if (p > pos) a[j] = up[j];
  }
}

template <int R, class E>
__device__ __forceinline__ E warp_get(const E (&a)[R], int p) {
  E r = a[0];
#pragma unroll
  for (int j = 1; j < R; ++j)
    if ((p >> 5) == j) r = a[j];
  return shfl_e(r, p & 31);
}

// Out-of-line copies of the K8 sorting networks: one body per size instead of one per call site
// (the fully unrolled networks otherwise dominate the kernel's code and its i-cache misses).
template <int R>
struct KCA {
  KC e[R];
};
template <int R>
__device__ __noinline__ KCA<R> sort_kc_ni(KCA<R> a) {
  warp_sort<R>(a.e);
  return a;
}
template <int R>
__device__ __noinline__ KCA<R> merge_kc_ni(KCA<R> a) {
  warp_bitonic_merge<R>(a.e);
  return a;
}
template <int R>
struct KOA {
  KO e[R];
};
template <int R>
__device__ __noinline__ KOA<R> sort_ko_ni(KOA<R> a) {
  warp_sort<R>(a.e);
  return a;
}
template <int R>
__device__ __forceinline__ void sort_ko(KO (&x)[R]) {
  KOA<R> t;
#pragma unroll
  for (int j = 0; j < R; ++j) t.e[j] = x[j];
  t = sort_ko_ni<R>(t);
#pragma unroll
  for (int j = 0; j < R; ++j) x[j] = t.e[j];
}
template <int R>
__device__ __forceinline__ void sort_kc(KC (&x)[R]) {
  KCA<R> t;
#pragma unroll
  for (int j = 0; j < R; ++j) t.e[j] = x[j];
  t = sort_kc_ni<R>(t);
#pragma unroll
  for (int j = 0; j < R; ++j) x[j] = t.e[j];
}
template <int R>
__device__ __forceinline__ void merge_kc(KC (&x)[R]) {
  KCA<R> t;
#pragma unroll
  for (int j = 0; j < R; ++j) t.e[j] = x[j];
  t = merge_kc_ni<R>(t);
#pragma unroll
  for (int j = 0; j < R; ++j) x[j] = t.e[j];
}

// One Alg. 3 step for one row, by ranks: the m <= 32 queued survivors Q (distinct ids, unsorted)
// and the running list S (best first; its real entries are a prefix, pads have id -1) give
// dst[0..kk) = the first kk distinct ids of S ∪ Q under the order (A13, A16).  A survivor whose id
// is already in S carries identical (i, U) and is dropped.  Every element's output position is
// (its rank in S) + (its rank among the kept survivors): O((|S| + m) * m / 32) exact cross-multiplied
// comparisons per lane, all independent (no sorting network, no 64-bit keys).
template <int KS>
__device__ __forceinline__ void rank_merge(const Cand *qr, int m, const c2_cand *S, int kk, c2_cand *dst) {
  const int lane = threadIdx.x & 31;
  Cand sv[KS];
  int nS = 0;
#pragma unroll
  for (int j = 0; j < KS; ++j) {
    sv[j] = (32 * j + lane < kk) ? from_out(S[32 * j + lane]) : sent();
    nS += __popc(__ballot_sync(0xffffffffu, is_real(sv[j])));
  }
  const Cand q = lane < m ? qr[lane] : sent();
  int rs = 0;
  bool dup = false;
  for (int i = 0; i < nS; ++i) {  // rank of q in S (broadcast reads)
    const Cand si = from_out(S[i]);
    dup |= si.id == q.id;
    rs += better_c(si, q) ? 1 : 0;
  }
  const unsigned dm = __ballot_sync(0xffffffffu, lane < m && dup);
  int rq = 0, sh[KS];
#pragma unroll
  for (int j = 0; j < KS; ++j) sh[j] = 0;
  for (int j = 0; j < m; ++j) {
    const Cand o = shfl_c(q, j);
    if ((dm >> j) & 1u) continue;  // (uniform)
    rq += better_c(o, q) ? 1 : 0;
#pragma unroll
    for (int jj = 0; jj < KS; ++jj) sh[jj] += better_c(o, sv[jj]) ? 1 : 0;
  }
  if (lane < m && !dup && rs + rq < kk) dst[rs + rq] = to_out(q);
#pragma unroll
  for (int jj = 0; jj < KS; ++jj) {
    const int i = 32 * jj + lane;
    if (i < nS && i + sh[jj] < kk) dst[i + sh[jj]] = to_out(sv[jj]);
  }
  for (int p = nS + m - __popc(dm) + lane; p < kk; p += 32) dst[p] = c2_cand{-1, 0, 0};
}

// rank_merge for k <= 32 on exact 64-bit keys (to_kc): the rank of a queued survivor in S by a
// binary search over the warp-held keys of S, the pairwise ranks by 64-bit compares against the
// kept survivors' keys compacted into kb (a per-warp shared buffer of 32 keys, read as
// broadcasts); no S-side ranks when S is empty (a row's first cluster).  Same result as rank_merge.
__device__ __forceinline__ void rank_merge_k1(const Cand *qr, int m, const c2_cand *S, int kk, c2_cand *dst,
                                              uint64_t *kb) {
  const int lane = threadIdx.x & 31;
  const Cand sv = lane < kk ? from_out(S[lane]) : sent();
  const int nS = __popc(__ballot_sync(0xffffffffu, is_real(sv)));
  const Cand q = lane < m ? qr[lane] : sent();
  const uint64_t qk = to_kc(q).k, sk = to_kc(sv).k;
  int rs = 0;
  bool keep = lane < m;
  if (nS > 0) {
#pragma unroll
    for (int st = 16; st >= 1; st >>= 1) {
      const uint64_t o = __shfl_sync(0xffffffffu, sk, min(rs + st - 1, 31));
      if (rs + st <= 32 && o > qk) rs += st;
    }
    const int32_t at_id = __shfl_sync(0xffffffffu, sv.id, min(rs, 31));
    keep = keep && !(rs < 32 && at_id == q.id);  // a repeated id carries identical (i, U) (A16)
  }
  const unsigned km = __ballot_sync(0xffffffffu, keep);
  const int mk = __popc(km);
  if (keep) kb[__popc(km & ((1u << lane) - 1u))] = qk;
  if (lane >= mk) kb[lane] = 0ull;
  __syncwarp();
  int rq = 0, sh = 0;
  if (nS > 0) {
    for (int j = 0; j < mk; j += 4) {
      const ulonglong2 a = *reinterpret_cast<const ulonglong2 *>(kb + j);
      const ulonglong2 b = *reinterpret_cast<const ulonglong2 *>(kb + j + 2);
      rq += (a.x > qk) + (a.y > qk) + (b.x > qk) + (b.y > qk);
      sh += (a.x > sk) + (a.y > sk) + (b.x > sk) + (b.y > sk);
    }
  } else {
    for (int j = 0; j < mk; j += 4) {
      const ulonglong2 a = *reinterpret_cast<const ulonglong2 *>(kb + j);
      const ulonglong2 b = *reinterpret_cast<const ulonglong2 *>(kb + j + 2);
      rq += (a.x > qk) + (a.y > qk) + (b.x > qk) + (b.y > qk);
    }
  }
  __syncwarp();
  if (keep && rs + rq < kk) dst[rs + rq] = to_out(q);
  if (lane < nS && lane + sh < kk) dst[lane + sh] = to_out(sv);
  for (int p = nS + mk + lane; p < kk; p += 32) dst[p] = c2_cand{-1, 0, 0};
}

// A fixed reference candidate of row r (|P_r| = pr) in the form that makes the order test of a
// candidate (i, |P_v|, id) two multiply-adds: with U = pr + |P_v| - i and the reference (iT, UT),
//   i*UT > iT*U  <=>  i*(UT + iT) > iT*|P_v| + iT*pr.
// Both sides fit in 32 bits (i <= 32767, U <= 65534, A28).  Ties are decided by id < idlim
// (idlim = idT: strictly better; idT + 1: better or the reference itself).  Unsigned id compare:
// an id of -1 (empty position of a mixed slice) never passes a tie.
struct Ref {
  uint32_t A, B, iT, idlim;
};
__device__ __forceinline__ Ref make_ref(Cand t, uint32_t pr, bool or_equal) {
  const uint32_t i = t.iu & 0xFFFFu, U = t.iu >> 16;
  return Ref{U + i, i * pr, i, (uint32_t)t.id + (or_equal ? 1u : 0u)};
}
__device__ __forceinline__ bool passes(uint32_t i, uint32_t ps, int32_t id, const Ref &R) {
  const uint32_t l = i * R.A, r = R.iT * ps + R.B;
  return l > r || (l == r && (uint32_t)id < R.idlim);
}

}  // namespace c2
