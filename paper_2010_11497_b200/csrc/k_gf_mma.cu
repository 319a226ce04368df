// k_gf_mma.cu -- Step 2 of the GoldFinger variant (c4, reading A19) on the 5th-generation
// tensor cores: with 1024-bit fingerprints, |F_u AND F_v| is a dense 0/1 contraction of length 1024,
// so a 128-row x 128-member block of one cluster is two chains of 16 tcgen05.mma.kind::i8 (K = 32
// bytes each) into a 128 x 128 s32 accumulator in tensor memory.
//
// One CTA (4 warps) per (cluster, 128-row block, 128-member block) of a function's big clusters:
//   1. each thread expands one row's and one member's fingerprint words (half of the 1024 bits per
//      pass) into 0/1 bytes in shared memory, K-major core matrices (8 rows x 16 B, no swizzle);
//   2. one thread issues the MMAs, tcgen05.commit -> mbarrier;
//   3. warp w reads TMEM lanes 32w..32w+31 (its rows) with tcgen05.ld 32x32b.x16: each thread holds
//      16 consecutive members' counts i = popc(F_r AND F_v) at a time, writes them to its row's count
//      row (for k_row_topk) and, for a light row (c2_build, running list full), tests every member
//      exactly against the running k-th best (A13) and appends the survivors to surv[u] (global
//      counter qn[u]; the thread that takes slot qmax hands the row to k_row_topk instead).
// Rows without a full running list (and all rows in c2_local_knn) get a RowRec from the member-block-0
// CTA.  Counts and tests are integers, so the result is bit-exact to the list kernel's.
#include <algorithm>

#include "cand.cuh"
#include "k_gf_mma.cuh"

namespace c2 {

constexpr int GM_M = 128, GM_N = 128, GM_KC = 256;  // rows, members, fingerprint bits per pass
constexpr int GM_T = 128;

__device__ __forceinline__ uint64_t gm_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100); base offset 0, SWIZZLE_NONE
  return d;
}
__host__ __device__ constexpr uint32_t gm_idesc() {
  // D s32 [4,6) = 2; A s8 [7,10) = 1; B s8 [10,13) = 1; both K-major; N>>3 [17,23); M>>4 [24,29)
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(GM_N >> 3) << 17) | ((uint32_t)(GM_M >> 4) << 24);
}
// 4 bits -> 4 bytes of 0/1 (byte j = bit j)
__device__ __forceinline__ uint32_t nib4(uint32_t x) { return ((x & 0xFu) * 0x00204081u) & 0x01010101u; }

// Fingerprints expanded once per call to 0/1 bytes, [n][1024] int8 (bit x of F_u -> byte x).
__global__ void k_gf_expand(const uint32_t *__restrict__ words, int64_t nw, uint4 *__restrict__ bytes) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one word -> 32 bytes
  if (i >= nw) return;
  const uint32_t x = words[i];
  bytes[2 * i] = make_uint4(nib4(x), nib4(x >> 4), nib4(x >> 8), nib4(x >> 12));
  bytes[2 * i + 1] = make_uint4(nib4(x >> 16), nib4(x >> 20), nib4(x >> 24), nib4(x >> 28));
}

// One operand row (a user's GM_KC bytes of pass `pass`) into the K-major core-matrix layout: byte
// (row, k) at ((row / 8) * (GM_KC / 16) + k / 16) * 128 + (row % 8) * 16 + k % 16 (cp.async, 16 B).
__device__ __forceinline__ void stage_row(uint8_t *op, int row, const uint8_t *src) {
  uint8_t *base = op + (row >> 3) * (GM_KC / 16) * 128 + (row & 7) * 16;
  if (src) {
#pragma unroll
    for (int kb = 0; kb < GM_KC / 16; ++kb)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32_gm(base + kb * 128)), "l"(src + kb * 16));
  } else {
#pragma unroll
    for (int kb = 0; kb < GM_KC / 16; ++kb) *reinterpret_cast<uint4 *>(base + kb * 128) = make_uint4(0, 0, 0, 0);
  }
}

__global__ void __launch_bounds__(GM_T, 3) k_gf_mma(GfArgs a) {
  extern __shared__ __align__(1024) uint8_t gsm[];
  uint8_t *A = gsm, *Bm = gsm + GM_M * GM_KC;
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t s_mbar;
  __shared__ int32_t s_mid[GM_N];
  __shared__ uint32_t s_mpc[GM_N];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32_gm(&s_tmem)),
                 "n"(GM_N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32_gm(&s_mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  const uint32_t sa = smem_u32_gm(A), sb = smem_u32_gm(Bm);
  constexpr uint32_t SBO = (GM_KC / 16) * 128;  // next 8-row group
  const uint32_t id = gm_idesc();
  uint32_t phase = 0;
  const int kk = a.k;
  const int64_t nwork = *a.nwork;
  for (int64_t wi = blockIdx.x; wi < nwork; wi += gridDim.x) {
    // work item -> (cluster c, row block rb, member block mb); CTAs stride the items, so the CTAs of
    // the SM array share a cluster's member fingerprints in L2
    const int64_t c = a.witem[wi];
    const BigC B = a.bcs[c];
    const int s = B.s, s4 = (s + 3) & ~3;
    const int nb = (s + GM_M - 1) / GM_M;
    const int rem = (int)(wi - a.wl_off[c]);
    const int rb = rem / nb, mb = rem - rb * nb;
    const int32_t *vp = a.vperm + B.vp_off;
    const int32_t *vs = a.vsize + B.vp_off;
    const int ri = rb * GM_M + tid, mi = mb * GM_N + tid;  // this thread's row and member (expansion)
    const int32_t ru = ri < s ? vp[ri] : -1, mu = mi < s ? vp[mi] : -1;
    s_mid[tid] = mu;
    s_mpc[tid] = mu >= 0 ? (uint32_t)vs[mi] : 0xFFFFFFFFu;
    for (int pass = 0; pass < 1024 / GM_KC; ++pass) {
      stage_row(A, tid, ru >= 0 ? a.bytes + (int64_t)ru * 1024 + pass * GM_KC : nullptr);
      stage_row(Bm, tid, mu >= 0 ? a.bytes + (int64_t)mu * 1024 + pass * GM_KC : nullptr);
      asm volatile("cp.async.wait_all;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
      __syncthreads();
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int k8 = 0; k8 < GM_KC / 32; ++k8) {
          const uint64_t da = gm_desc(sa + k8 * 256, 128, SBO), db = gm_desc(sb + k8 * 256, 128, SBO);
          const uint32_t acc = (pass > 0 || k8 > 0) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
              "l"(da), "l"(db), "r"(id), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32_gm(&s_mbar)));
      }
      // all threads: the MMAs are done (shared operands reusable, accumulator final after the last)
      for (;;) {
        uint32_t done;
        asm volatile(
            "{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}\n"
            : "=r"(done)
            : "r"(smem_u32_gm(&s_mbar)), "r"(phase));
        if (done) break;
      }
      phase ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;");
    }
    // ---- epilogue: thread = row (TMEM lane), 16 members per tcgen05.ld
    const int r = rb * GM_M + warp * 32 + lane;  // this thread's row
    const bool rv = r < s;
    const int32_t u = rv ? vp[r] : -1;
    const uint32_t pr = rv ? (uint32_t)vs[r] : 0u;
    bool light = false;
    Ref R{0, 0, 0, 0};
    uint32_t imin = 0xFFFFFFFFu;  // a member of this block can pass only with i >= imin
    if (rv && a.seed) {
      const c2_cand tl = a.seed[(int64_t)u * kk + kk - 1];
      light = a.surv != nullptr && tl.id >= 0 && tl.inter >= 1;
      if (light) {
        R = make_ref(from_out(tl), pr, false);
        uint32_t psmin = 0xFFFFFFFFu;
        for (int j = 0; j < GM_N; ++j) psmin = min(psmin, s_mpc[j]);
        if (psmin != 0xFFFFFFFFu) imin = (R.B + R.iT * psmin + R.A - 1u) / R.A;
      }
    }
    const int64_t coff = a.tc_base + a.cbase[c] + (int64_t)r * s4;  // this row's count row
    if (rv && !light && mb == 0) {  // handed to k_row_topk
      const unsigned long long ri2 = atomicAdd(a.nrec, 1ull);
      if (ri2 < (unsigned long long)a.rcap) a.recs[ri2] = RowRec{u, (int32_t)pr, s, B.vp_off, r, 0, 0, B.f, coff};
      else atomicExch(a.err, 1);
    }
    __syncwarp();
#pragma unroll 1
    for (int g = 0; g < GM_N / 16; ++g) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
          "%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(g * 16)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const int m0 = mb * GM_N + g * 16;
      if (!rv || m0 >= s) continue;
      // count row entries m0 .. m0+15 (4 at a time: the row is 8-byte aligned)
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        if (m0 + j < s) {
          const uint2 pk = make_uint2(v[j] | (v[j + 1] << 16), v[j + 2] | (v[j + 3] << 16));
          *reinterpret_cast<uint2 *>(a.cnt + coff + m0 + j) = pk;
        }
      }
      if (light) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int m = m0 + j;
          if (m >= s || m == r || v[j] < imin) continue;
          const int32_t idv = s_mid[g * 16 + j];
          const uint32_t psv = s_mpc[g * 16 + j];
          if (passes(v[j], psv, idv, R)) {
            const int pq = atomicAdd(a.qn + u, 1);
            if (pq < a.qmax) {
              a.surv[(int64_t)u * a.qmax + pq] = c2_cand{idv, (uint16_t)v[j], (uint16_t)(pr + psv - v[j])};
            } else if (pq == a.qmax) {  // too many survivors: the full count row goes to k_row_topk
              const unsigned long long ri2 = atomicAdd(a.nrec, 1ull);
              if (ri2 < (unsigned long long)a.rcap) a.recs[ri2] = RowRec{u, (int32_t)pr, s, B.vp_off, r, 0, 0, B.f, coff};
              else atomicExch(a.err, 1);
            }
          }
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // TMEM and the member arrays are rewritten by the next work item
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(GM_N));
}

// Per function (one block each): exclusive prefixes over its big clusters [bc_lo, bc_hi) of the
// work items ceil(s/128)^2 (wl_off, global over all functions) and of the count-row sizes s * s4
// (cbase, relative to the function's region).
__global__ void k_gf_prefix(const BigC *__restrict__ bcs, const int64_t *__restrict__ bc_rng, int t,
                            int64_t *__restrict__ wl_off, int64_t *__restrict__ cbase, int64_t *__restrict__ fsum) {
  __shared__ int64_t sw[1024], sc[1024];
  const int f = blockIdx.x;
  const int64_t b0 = bc_rng[f], b1 = bc_rng[f + 1];
  int64_t wcarry = 0, ccarry = 0;
  for (int64_t base = b0; base < b1; base += blockDim.x) {
    const int64_t c = base + threadIdx.x;
    int64_t w = 0, cc = 0;
    if (c < b1) {
      const int64_t s = bcs[c].s, nb = (s + GM_M - 1) / GM_M;
      w = nb * nb;
      cc = s * ((s + 3) & ~3ll);
    }
    sw[threadIdx.x] = w;
    sc[threadIdx.x] = cc;
    __syncthreads();
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {  // inclusive Hillis-Steele scan
      const int64_t aw = threadIdx.x >= o ? sw[threadIdx.x - o] : 0, ac = threadIdx.x >= o ? sc[threadIdx.x - o] : 0;
      __syncthreads();
      sw[threadIdx.x] += aw;
      sc[threadIdx.x] += ac;
      __syncthreads();
    }
    if (c < b1) {
      wl_off[c] = wcarry + sw[threadIdx.x] - w;
      cbase[c] = ccarry + sc[threadIdx.x] - cc;
    }
    wcarry += sw[blockDim.x - 1];
    ccarry += sc[blockDim.x - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    fsum[2 * f] = wcarry;       // work items of function f
    fsum[2 * f + 1] = ccarry;   // count entries of function f
  }
}

// item -> cluster map: witem[f * icap + w] = c for the work items w of cluster c (function f)
__global__ void k_gf_items(const BigC *__restrict__ bcs, int64_t nbig, const int64_t *__restrict__ wl_off,
                           int64_t icap, int32_t *__restrict__ witem) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nbig) return;
  const BigC B = bcs[c];
  const int64_t nb = (B.s + GM_M - 1) / GM_M, w0 = wl_off[c];
  int32_t *o = witem + (int64_t)B.f * icap;
  for (int64_t w = w0; w < w0 + nb * nb && w < icap; ++w) o[w] = (int32_t)c;
}

int gf_prefix(c2_ctx *ctx, const BigC *bcs, const int64_t *bc_rng, int t, int64_t nbig, int64_t *wl_off,
              int64_t *cbase, int64_t *fsum, int32_t *witem, int64_t icap) {
  k_gf_prefix<<<t, 1024, 0, ctx->stream>>>(bcs, bc_rng, t, wl_off, cbase, fsum);
  C2_LAUNCHED(ctx, "k_gf_prefix");
  k_gf_items<<<(unsigned)((nbig + 255) / 256), 256, 0, ctx->stream>>>(bcs, nbig, wl_off, icap, witem);
  C2_LAUNCHED(ctx, "k_gf_items");
  return C2_OK;
}

int gf_expand(c2_ctx *ctx, const uint32_t *words, int32_t n, uint8_t *bytes) {
  const int64_t nw = (int64_t)n * 32;
  k_gf_expand<<<(unsigned)((nw + 255) / 256), 256, 0, ctx->stream>>>(words, nw, reinterpret_cast<uint4 *>(bytes));
  C2_LAUNCHED(ctx, "k_gf_expand");
  return C2_OK;
}

int launch_gf_mma(c2_ctx *ctx, const GfArgs &ga) {
  if (ga.bc_hi <= ga.bc_lo) return C2_OK;
  const int smem = (GM_M + GM_N) * GM_KC;
  static bool attr = false;
  if (!attr) {
    C2_CUDA(ctx, cudaFuncSetAttribute(k_gf_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  k_gf_mma<<<ctx->num_sms * 3, GM_T, smem, ctx->stream>>>(ga);
  C2_LAUNCHED(ctx, "k_gf_mma");
  return C2_OK;
}

}  // namespace c2
