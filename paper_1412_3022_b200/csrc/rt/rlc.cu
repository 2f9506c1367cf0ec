// Runtime-coefficient region-linear-combination kernel (sm_100a): the GF(2^8) coefficients are
// DATA (per-plan tables in device memory), not code, so a new failure pattern costs only the host
// inversion (decode/repair initialisation "depends on the failure pattern") and no NVRTC.
//
// It computes the same plans as the generated bitsliced kernels (plan.hpp): for every stripe t and
// byte position p
//     in_i[t][p]  = XOR_terms  mu * block(slot, blk)[t][p]          (derived inputs: the helper
//                                                                    projection, P:53 footnote)
//     out_r[t][p] = XOR_i      A[r][i] * in_i[t][p]
// on bytes in their natural layout (no bit transposes), with the north star's table formulation:
// a GF(2^8) product c*x is split on the bits of x as 3+3+2,
//     c*x = T0[x & 7] ^ T1[(x >> 3) & 7] ^ T2[x >> 6],   T0[j] = c*j, T1[j] = c*(j<<3), T2[j] = c*(j<<6)
// (multiplication by c is GF(2)-linear in x), and each lookup is ONE byte permute (PRMT) for four
// bytes at once: an 8-entry table is two registers, the 4-entry one is one.  Per 32-bit word and
// coefficient: 3 PRMT + 2 LOP3 (ALU pipe).  The PRMT selectors of a word are shared by every row
// that reads it: 3 LOP3 (ALU) + 5 IMAD.HI (FMA pipe) per input word.
//
// Selector trick: PRMT reads 4 selector nibbles from bits 0..15.  For u = w & 0x07070707 (the low
// 3 bits of bytes b0..b3 at bit offsets 0, 8, 16, 24), u + (u >> 12) holds b0, b2, b1, b3 in
// nibbles 0..3 (the fields are disjoint: no carries), one IMAD.HI with addend.  The products come
// out in byte order (0, 2, 1, 3) -- the same fixed permutation for every table -- and are
// accumulated in that order; one PRMT per output word restores the order.
//
// Work decomposition (B200: 148 SMs; measured, profiles/r02):
//   * item = (stripe t, tile of TP = GT * V * 4 bytes of every block); CTA b walks a contiguous
//     range of items (static split; 1 CTA per SM, or 2 for single-group plans).
//   * G row groups of GT consumer threads: thread j of group g owns V consecutive 32-bit words of
//     the tile and R rows (rows g R .. g R + R - 1 of the pass) of accumulators in registers; a pass
//     covers G R rows, more rows run as further passes over the tile.  All groups read the same
//     staged input words (more warps per SM for the same shared-memory traffic: the ALU latency
//     of the dependent PRMT -> LOP3 chains is hidden by 16-32 warps instead of 8).
//   * 1 producer warp streams the tile of every term's block (the flattened sequence item ->
//     pass -> term, which the consumers walk in the same order) into a ring of D shared-memory
//     slots of TPS terms each with TMA 1-D bulk copies (cp.async.bulk ... mbarrier::complete_tx),
//     TPS lanes per slot in parallel, FULL/EMPTY mbarrier pairs per slot: up to D x TPS x TP bytes
//     in flight per CTA, no registers held, one barrier round trip per TPS terms.
//   * Zero coefficients are skipped with warp-uniform branches on a per-input row mask (the
//     paper's sparsity, applied at run time; the mask is broadcast with a shuffle so the
//     compiler emits plain uniform branches), with the next row's tables loaded before the branch
//     (software pipelining of the shared-memory table loads); outputs leave with 16-B evict-first
//     stores.
//   * The plan (tables, masks, wiring; <= 160 KB) is copied to shared memory when the stripe's plan
//     changes, so config 4's per-stripe failure patterns run in ONE launch (stripe_plan[t]); the
//     coefficient tables of larger plans (k = 16 decode: 1.1 MB) are read from device memory (TG).
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "rlc.hpp"

namespace pmrc_rt {

typedef uint32_t u32;
typedef unsigned long long u64;

constexpr int D = 4;    // ring slots
constexpr int TPS = 4;  // terms (block tiles) per slot

static __device__ __forceinline__ u32 prmt(u32 a, u32 b, u32 s) {
  u32 d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}
// ((a * b) >> 32) + c on the FMA pipe (IMAD.HI): a right shift with an addend
static __device__ __forceinline__ u32 madhi(u32 a, u32 b, u32 c) {
  u32 d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
static __device__ __forceinline__ u32 xor3(u32 a, u32 b, u32 c) {
  u32 d;
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

struct Sel {
  u32 s0, s1, s2;
};
struct Shifts {
  u32 sh3, sh6, sh12;  // 2^29, 2^26, 2^20 (kernel parameters, see RlcArgs)
};
// Per word: 3 LOP3 (masks) + 3 LEA.HI (u + (u >> 12): a literal power of two makes ptxas emit
// one LEA.HI, where a run-time multiplier with an addend costs IMAD.HI + a MOV of the zero half of
// its 64-bit addend) + 2 IMAD.HI (the plain shifts, run-time multipliers: FMA pipe, RZ addend).
static __device__ __forceinline__ Sel make_sel(u32 w, const Shifts &k) {
  Sel s;
  const u32 u0 = w & 0x07070707u;
  s.s0 = madhi(u0, 1u << 20, u0);                    // u0 + (u0 >> 12)
  const u32 u1 = madhi(w, k.sh3, 0u) & 0x07070707u;  // (w >> 3) & 7 per byte
  s.s1 = madhi(u1, 1u << 20, u1);
  const u32 u2 = madhi(w, k.sh6, 0u) & 0x03030303u;  // (w >> 6) & 3 per byte
  s.s2 = madhi(u2, 1u << 20, u2);
  return s;
}
// acc ^= c * w (permuted byte order); c's tables t = (T0a, T0b, T1a, T1b), t2 = T2
static __device__ __forceinline__ void mac(u32 &acc, const uint4 &t, u32 t2, const Sel &s) {
  acc = xor3(acc, prmt(t.x, t.y, s.s0), prmt(t.z, t.w, s.s1));
  acc ^= prmt(t2, t2, s.s2);
}
// the same with a pending operand carried between consecutive products of one sum (3 LOP3 per 2
// products instead of 4): acc ^= pend ^ c*w, and the product's last lookup becomes the new pend
static __device__ __forceinline__ void mac_pend(u32 &acc, u32 &pend, const uint4 &t, u32 t2, const Sel &s) {
  acc = xor3(acc, pend, prmt(t.x, t.y, s.s0));
  acc ^= prmt(t.z, t.w, s.s1);
  pend = prmt(t2, t2, s.s2);
}
static __device__ __forceinline__ u32 unperm(u32 a) { return prmt(a, 0u, 0x3120u); }

// ---- mbarrier / bulk-copy primitives (shared::cta addresses) ----
static __device__ __forceinline__ u32 smem_addr(const void *p) { return (u32)__cvta_generic_to_shared(p); }
static __device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
static __device__ __forceinline__ void mbar_arrive(u32 bar) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(bar) : "memory");
}
static __device__ __forceinline__ void mbar_expect_tx(u32 bar, u32 bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
static __device__ __forceinline__ void mbar_wait(u32 bar, u32 parity) {
  asm volatile(
      "{ .reg .pred p;\n"
      "WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=; }" ::"r"(bar),
      "r"(parity)
      : "memory");
}
static __device__ __forceinline__ void bulk_g2s(u32 dst, const void *src, u32 bytes, u32 bar, u64 policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}
static __device__ __forceinline__ void named_sync(u32 id, u32 n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int V>
static __device__ __forceinline__ void store_vec(unsigned char *p, const u32 *w) {
  if (V == 4) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(w[0]), "r"(w[1 % V]), "r"(w[2 % V]),
                 "r"(w[3 % V])
                 : "memory");
  } else {
    asm volatile("st.global.cs.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(w[0]), "r"(w[1 % V]) : "memory");
  }
}

size_t rlc_smem_bytes(int V, int GT, unsigned max_words) {
  const size_t plan = ((size_t)max_words * 4 + 127) & ~(size_t)127;
  return plan + (size_t)D * TPS * GT * V * 4 + 2 * D * 8;
}

template <int R, int V, int G, int GT, bool TG>
__global__ void __launch_bounds__(GT * G + 32, G == 1 ? 2 : 1) rlc_kernel(const RlcArgs a) {
  extern __shared__ __align__(128) u32 sm[];
  constexpr u32 TP = GT * V * 4;           // tile bytes per block
  constexpr u32 SLOT = TPS * TP;
  constexpr u32 NCW = G * GT / 32;         // consumer warps
  constexpr u32 NCT = G * GT;              // consumer threads
  const u32 plan_bytes = ((a.max_words * 4u) + 127u) & ~127u;
  unsigned char *ring = (unsigned char *)sm + plan_bytes;
  const u32 bar_full = smem_addr(ring + D * SLOT), bar_empty = bar_full + 8 * D;
  const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const u64 tiles = (a.S + TP - 1) / TP;
  const u64 items = tiles * a.stripes;
  const u64 per = items / gridDim.x, rem = items % gridDim.x;
  const u64 b = blockIdx.x;
  // per-stripe patterns of unequal cost (config 4: a parity-node repair costs ~3.6x a systematic
  // one): the host splits the items by estimated cost; otherwise equal item counts
  const u64 i0 = a.item_bounds ? a.item_bounds[b] : b * per + (b < rem ? b : rem);
  const u64 i1 = a.item_bounds ? a.item_bounds[b + 1] : i0 + per + (b < rem ? 1 : 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < D; s++) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NCW) {
    // ---------------- producer warp: TPS lanes fill one slot per round ----------------
    // Lane j of a round issues term q = TPS k + j of the flattened sequence (item -> pass -> term)
    // into slot k % D; lane 0 arrives on FULL after all of the round's copies are registered.
    u64 pol_first, pol_normal;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_normal));
    // terms of item `it` (0 for stripes without work) and its plan
    auto item_terms = [&](u64 it, const u32 *&pb) -> u32 {
      const u64 t = it / tiles;
      const u32 pi = a.stripe_plan ? (u32)a.stripe_plan[t] : 0u;
      if (pi == 0xFFFFu) return 0u;
      pb = a.stripe_plan ? (const u32 *)a.plan_ptrs[pi] : a.plan0;
      return __ldg(pb + offsetof(RlcHdr, seq_len) / 4);
    };
    u64 it = i0;   // walk position (uniform): item and offset within it
    u32 e = 0;
    for (u32 k = 0;; k++) {
      // this lane's term: `lane` positions after (it, e)
      u64 itj = it;
      u32 ej = e + lane;
      const u32 *pb = nullptr;
      u32 tot = 0;
      while (itj < i1 && ej >= (tot = item_terms(itj, pb))) {
        ej -= tot;
        itj++;
      }
      const bool mine = lane < (u32)TPS && itj < i1;
      if (!__any_sync(0xffffffffu, mine)) break;
      const u32 s = k % D;
      if (k >= (u32)D) mbar_wait(bar_empty + 8 * s, ((k / D) - 1) & 1);
      if (mine) {
        const u64 t = itj / tiles, tile = itj - t * tiles;
        const u32 n_pass = __ldg(pb + offsetof(RlcHdr, n_pass) / 4), off_terms = __ldg(pb + offsetof(RlcHdr, off_terms) / 4);
        const u32 j = __ldg(pb + __ldg(pb + offsetof(RlcHdr, off_seq) / 4) + ej);
        const u64 p0 = tile * TP;
        const u32 bytes = (u32)((a.S - p0) < TP ? (a.S - p0) : TP);
        // single-pass plans read each tile once: stream it (evict-first); multi-pass plans may
        // re-read it in a later pass, from L2
        const u64 pol = n_pass == 1 ? pol_first : pol_normal;
        const u32 w0 = __ldg(pb + off_terms + 2 * j), w1 = __ldg(pb + off_terms + 2 * j + 1);
        const u32 slot = w0 & 0xFFFFu, blk = w1 & 0xFFFFu;
        const unsigned char *src =
            (const unsigned char *)(a.slot_ptr[slot] + t * a.slot_stride[slot] + (u64)blk * a.S + p0);
        mbar_expect_tx(bar_full + 8 * s, bytes);
        bulk_g2s(smem_addr(ring + s * SLOT + lane * TP), src, bytes, bar_full + 8 * s, pol);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_full + 8 * s);
      // advance the walk by TPS terms
      u32 n = TPS;
      while (it < i1) {
        const u32 tt = item_terms(it, pb);
        if (e + n < tt) {
          e += n;
          break;
        }
        n -= tt - e;
        e = 0;
        it++;
      }
    }
    return;
  }

  // ---------------- G groups of GT consumer threads ----------------
  const Shifts ks = {a.sh3, a.sh6, a.sh12};
  const u32 g = threadIdx.x / GT, tid = threadIdx.x % GT;
  int cur = -1;
  RlcHdr h;
  const u32 *tabs = sm;  // coefficient tables: shared memory, or the plan in device memory (TG)
  u32 q = 0;
  for (u64 it = i0; it < i1; it++) {
    const u64 t = it / tiles, tile = it - t * tiles;
    const int pl = a.stripe_plan ? (int)a.stripe_plan[t] : 0;
    if (pl == 0xFFFF) continue;  // nothing to compute in this stripe
    if (pl != cur) {             // (re)load the stripe's plan into shared memory
      named_sync(1, NCT);
      const u32 *src = a.stripe_plan ? (const u32 *)a.plan_ptrs[pl] : a.plan0;
      const u32 words = __ldg(src + offsetof(RlcHdr, smem_words) / 4);
      for (u32 e = threadIdx.x * 4; e < words; e += NCT * 4) {
        if (e + 4 <= words) *(uint4 *)(sm + e) = __ldg((const uint4 *)(src + e));
        else
          for (u32 f = e; f < words; f++) sm[f] = __ldg(src + f);
      }
      named_sync(1, NCT);
      cur = pl;
      h = *(const RlcHdr *)sm;
      tabs = TG ? src : sm;
    }
    const u32 n_rb = h.n_rb, passes = h.n_pass;
    const u64 p = tile * TP + (u64)tid * (V * 4);
    const bool act = p < a.S;
    for (u32 pass = 0; pass < passes; pass++) {
      const u32 rb = pass * G + g;  // this group's row block
      const bool rows_here = rb < n_rb;
      // rows of the block that exist (the last block may be short: repair has alpha = 7 rows)
      const u32 nvalid = rows_here ? min((u32)R, h.n_out - rb * R) : 0u;
      const u32 vmask = nvalid >= 32u ? 0xFFFFFFFFu : (1u << nvalid) - 1u;
      u32 acc[R][V];
#pragma unroll
      for (int r = 0; r < R; r++)
#pragma unroll
        for (int v = 0; v < V; v++) acc[r][v] = 0u;
      // the term stream of this pass: slot wait, this thread's words, slot release
      auto fetch = [&](u32 e, u32 (&x)[V]) -> u32 {
        const u32 j = sm[h.off_seq + e];
        const u32 k = q / TPS, sub = q - k * TPS, s = k % D;
        if (sub == 0) mbar_wait(bar_full + 8 * s, (k / D) & 1);
        if (V == 4) {
          const uint4 v4 = *(const uint4 *)(ring + s * SLOT + sub * TP + tid * 16);
          x[0] = v4.x; x[1 % V] = v4.y; x[2 % V] = v4.z; x[3 % V] = v4.w;
        } else {
          const uint2 v2 = *(const uint2 *)(ring + s * SLOT + sub * TP + tid * 8);
          x[0] = v2.x; x[1 % V] = v2.y;
        }
        if (sub == TPS - 1) {
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_empty + 8 * s);
        }
        return j;
      };
      // a complete (derived) input i, natural byte order: apply it to this group's rows
      auto apply = [&](u32 i, const u32 (&win)[V]) {
        const u32 mask = __shfl_sync(0xffffffffu, rows_here ? sm[h.off_masks + i * n_rb + rb] : 0u, 0);
        if (!mask) return;
        Sel sl[V];
#pragma unroll
        for (int v = 0; v < V; v++) sl[v] = make_sel(win[v], ks);
        const u32 *tA = tabs + h.off_tabA + 4 * (i * h.n_out + rb * R);
        const u32 *tB = tabs + h.off_tabB + i * h.n_out + rb * R;
        if (mask == vmask) {
          // every row of the block reads this input (the host clusters rows of equal support, so
          // this is the common case): no branches, all R rows' tables loaded up front, and the
          // R x V independent MAC chains interleave freely (rows past n_out of a short last block
          // compute garbage that is never stored)
          constexpr int RB = R < 8 ? R : 8;  // tables loaded 8 rows at a time (registers)
#pragma unroll
          for (int r0 = 0; r0 < R; r0 += RB) {
            uint4 tb[RB];
            u32 t2[RB];
#pragma unroll
            for (int r = 0; r < RB; r++) {
              tb[r] = *(const uint4 *)(tA + 4 * (r0 + r));
              t2[r] = tB[r0 + r];
            }
#pragma unroll
            for (int r = 0; r < RB; r++)
#pragma unroll
              for (int v = 0; v < V; v++) mac(acc[r0 + r][v], tb[r], t2[r], sl[v]);
          }
          return;
        }
        uint4 tbn = *(const uint4 *)tA;
        u32 t2n = tB[0];
#pragma unroll
        for (int r = 0; r < R; r++) {
          const uint4 tb = tbn;
          const u32 t2 = t2n;
          if (r + 1 < R) {  // next row's tables before this row's branch (loads overlap the MACs)
            tbn = *(const uint4 *)(tA + 4 * (r + 1));
            t2n = tB[r + 1];
          }
          if (mask & (1u << r)) {
#pragma unroll
            for (int v = 0; v < V; v++) mac(acc[r][v], tb, t2, sl[v]);
          }
        }
      };
      const u32 e0 = sm[h.off_pstart + pass], e1 = sm[h.off_pstart + pass + 1];
      // the plan's term structure (uniform per plan) picks one of three loops, so that no loop
      // carries state it does not need (a mixed loop's branch joins cost register moves)
      const u32 mode = h.flags & (kRlcDirect | kRlcNoPlain);
      if (mode == kRlcDirect) {
        // every input is one plain term (encode, decode, systematic repair)
        for (u32 e = e0; e < e1; e++, q++) {
          u32 x[V];
          const u32 j = fetch(e, x);
          apply(sm[h.off_terms + 2 * j + 1] >> 16, x);
        }
      } else if (mode == kRlcNoPlain) {
        // every term carries a coefficient (parity-node repair: the helpers' projections)
        u32 wp[V], pe[V];
#pragma unroll
        for (int v = 0; v < V; v++) wp[v] = pe[v] = 0u;
        for (u32 e = e0; e < e1; e++, q++) {
          u32 x[V];
          const u32 j = fetch(e, x);
          const uint4 tb = *(const uint4 *)(sm + h.off_ttabA + 4 * j);
          const u32 t2 = sm[h.off_ttabB + j];
#pragma unroll
          for (int v = 0; v < V; v++) mac_pend(wp[v], pe[v], tb, t2, make_sel(x[v], ks));
          const u32 w0 = __shfl_sync(0xffffffffu, sm[h.off_terms + 2 * j], 0);
          if (!(w0 & 0x40000000u)) continue;  // more terms of this input follow
          u32 win[V];
#pragma unroll
          for (int v = 0; v < V; v++) {
            win[v] = unperm(wp[v] ^ pe[v]);
            wp[v] = pe[v] = 0u;
          }
          apply(sm[h.off_terms + 2 * j + 1] >> 16, win);
        }
      } else {
        u32 wn[V], wp[V], pe[V];
#pragma unroll
        for (int v = 0; v < V; v++) wn[v] = wp[v] = pe[v] = 0u;
        for (u32 e = e0; e < e1; e++, q++) {
          u32 x[V];
          const u32 j = fetch(e, x);
          // the term word is the same for the whole warp: broadcast it so the plain / last tests
          // below compile to uniform branches (no BSSY/BSYNC reconvergence per term)
          const u32 w0 = __shfl_sync(0xffffffffu, sm[h.off_terms + 2 * j], 0);
          if (w0 & 0x80000000u) {  // plain term (coefficient 1)
#pragma unroll
            for (int v = 0; v < V; v++) wn[v] ^= x[v];
          } else {
            const uint4 tb = *(const uint4 *)(sm + h.off_ttabA + 4 * j);
            const u32 t2 = sm[h.off_ttabB + j];
#pragma unroll
            for (int v = 0; v < V; v++) mac_pend(wp[v], pe[v], tb, t2, make_sel(x[v], ks));
          }
          if (!(w0 & 0x40000000u)) continue;  // more terms of this input follow
          u32 win[V];
#pragma unroll
          for (int v = 0; v < V; v++) {
            win[v] = wn[v] ^ unperm(wp[v] ^ pe[v]);
            wn[v] = wp[v] = pe[v] = 0u;
          }
          apply(sm[h.off_terms + 2 * j + 1] >> 16, win);
        }
      }
      if (act && rows_here) {
#pragma unroll
        for (int r = 0; r < R; r++) {
          const u32 row = rb * R + r;
          if (row < h.n_out) {
            const u32 slot = sm[h.off_outs + 2 * row], blk = sm[h.off_outs + 2 * row + 1];
            u32 o[V];
#pragma unroll
            for (int v = 0; v < V; v++) o[v] = unperm(acc[r][v]);
            store_vec<V>((unsigned char *)(a.slot_ptr[slot] + t * a.slot_stride[slot] + (u64)blk * a.S + p), o);
          }
        }
      }
    }
  }
}

template <int R, int V, int G, int GT, bool TG>
static int launch_one(const RlcArgs &a, int grid, cudaStream_t st) {
  const size_t smem = rlc_smem_bytes(V, GT, a.max_words);
  auto k = rlc_kernel<R, V, G, GT, TG>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
  k<<<grid, GT * G + 32, smem, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template <int R, int V, int G, int GT, bool TG>
static int occ_one(unsigned max_words) {
  const size_t smem = rlc_smem_bytes(V, GT, max_words);
  auto k = rlc_kernel<R, V, G, GT, TG>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, GT * G + 32, smem) != cudaSuccess) return 0;
  return n;
}

// the instantiated shapes (rlc.hpp)
#define RLC_SHAPES(X)                                                                                \
  X(8, 4, 1, 256, false) X(8, 4, 2, 256, false) X(8, 4, 1, 256, true) X(8, 4, 2, 256, true)          \
  X(7, 4, 1, 256, false) X(7, 4, 2, 256, false) X(7, 4, 1, 256, true) X(7, 4, 2, 256, true)

int rlc_launch(const RlcArgs &a, const RlcShape &sh, int grid, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
#define X(r, v, gg, gt, tgv) \
  if (sh.R == r && sh.V == v && sh.G == gg && sh.GT == gt && sh.tg == tgv) return launch_one<r, v, gg, gt, tgv>(a, grid, st);
  RLC_SHAPES(X)
#undef X
  return -2;
}

int rlc_ctas_per_sm(const RlcShape &sh, unsigned max_words) {
#define X(r, v, gg, gt, tgv) \
  if (sh.R == r && sh.V == v && sh.G == gg && sh.GT == gt && sh.tg == tgv) return occ_one<r, v, gg, gt, tgv>(max_words);
  RLC_SHAPES(X)
#undef X
  return 0;
}

bool rlc_shape_ok(const RlcShape &sh) {
#define X(r, v, gg, gt, tgv) \
  if (sh.R == r && sh.V == v && sh.G == gg && sh.GT == gt && sh.tg == tgv) return true;
  RLC_SHAPES(X)
#undef X
  return false;
}

}  // namespace pmrc_rt
