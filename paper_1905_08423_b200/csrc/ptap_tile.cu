// ptap_tile.cu -- deterministic owner-computes numeric pass of the
// all-at-once / merged triple product (one-rank structure: no A_o, no P_o).
//
// The reference fixes the value of every C entry by its summation order
// (src/_kernels.py:446-515, src/tripleproduct.py:12-16):
//
//   AP(i,g)  = fold over the pairs (A entry k ascending, P entry of row k) in
//              order, the first product setting the slot (hm_add,
//              src/_kernels.py:116-147);
//   C(J,g)   = ((0 + P(i1,J) AP(i1,g)) + P(i2,J) AP(i2,g)) + ...  over the
//              contributing fine rows i1 < i2 < ... (C zeroed, then `+=` in
//              the local row loop, src/_kernels.py:498-514).
//
// k_tile_numeric reproduces both orders exactly, so C is bit-identical to the
// reference at one rank and bitwise repeatable, with no atomics on C:
//
//   * The fine rows are cut into blocks of TR = 64 consecutive rows ("items"),
//     handed out in ascending order by an atomic ticket to a persistent grid.
//   * Fold: the item's A rows (one contiguous CSR range) are staged into
//     shared memory by a TMA bulk copy (cp.async.bulk + mbarrier); two warps
//     fold the even and the odd rows, one row per lane (on a lexicographic
//     grid each warp then holds rows of one structural class, so the
//     per-row slot maps are read as broadcasts), into a [slot][lane]
//     accumulator (bank-conflict free).  The AP rows go to an L2-resident
//     ring of AP blocks and the item publishes them (release flag).
//   * Gather: C row J is computed by the item that folded J's LAST
//     contributing row, after acquiring the publication flags of the blocks
//     of its other contributors (all earlier items): one warp per C row walks
//     the contributors in ascending row order (P_d^T, sorted in the plan),
//     and lane s adds P(i,J) * AP(i,s) into position pmap(i,J,s) of a shared
//     accumulator row.  Each C entry is written once, with a plain store.
//   * A ring slot is reused only after every item that reads the block it
//     holds has signalled (per-block reader counts, epoch-coded so nothing is
//     reset between passes).
//
// Deadlock freedom: an item waits only on items with smaller tickets (the
// blocks of its contributors, and the readers of the block its ring slot last
// held, which is more than the contributor span behind it), and tickets are
// taken in order by running CTAs.
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <cstdint>
#include <cstdlib>

#include "ptap_device.cuh"
#include "ptap_kernels.cuh"

namespace ptapdev {

namespace {

constexpr int TW = 2;              // fold warps per CTA (even / odd rows of a block)
#ifndef PTAP_TILE_GW
#define PTAP_TILE_GW 2
#endif
constexpr int GW = PTAP_TILE_GW;   // gather warps per CTA (run concurrently with the fold warps)
constexpr int NT = (TW + GW) * 32;
constexpr int TR = TILE_ROWS;      // rows per block (item)
constexpr int AST = 33;            // accumulator stride per slot (doubles): conflict-free both ways
constexpr int GCAP = TILE_GCAP;    // contributor entries staged per gather chunk
constexpr int MAXRUN = TILE_MAXRUN;

// Dynamic shared memory (offsets in TileArgs, sized from the plan):
//   aval[acap] | acol[acap + 4] | pstage[pvcap] | prp[prcap] | union{acc[TW][napc][AST], gather meta} | tail
struct TileTail {
  unsigned long long bar;
  int item, next, jb, nrun;
  int zero;  // a zero word: lanes without a fold program read Q[0] through it
  int rk0[MAXRUN], rk1[MAXRUN], rvoff[MAXRUN], rpoff[MAXRUN];
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TILE_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TILE_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// one contiguous global -> shared copy through the TMA unit (bulk, non-tensor)
__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// the same with an L2 eviction-priority hint: A is streamed once, so its
// lines go first and leave L2 to P's rows and the AP ring
__device__ __forceinline__ void tma_bulk_g2s_stream(void *dst, const void *src, uint32_t bytes,
                                                    unsigned long long *bar) {
  asm volatile(
      "{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      " cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n}"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Flags are polled with relaxed (strong, L2) loads: an acquire load at gpu
// scope is followed by CCTL.IVALL on sm_100a (the SM's whole L1 is
// invalidated on every poll, which evicted the fold's P rows and slot maps:
// 110 -> 30 ms).  The data guarded by a flag is read with
// ld.global.cg (L2, the coherence point) only after the polling loop exits.
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// reader signals: the item's reads of the ring returned their values before
// the CTA barrier that precedes the signal, so a relaxed add suffices (WAR)
__device__ __forceinline__ void red_relaxed_add_u32(uint32_t *p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// predicated loads (no divergent branch around them)
__device__ __forceinline__ double ld_cg_f64_if(bool p, const double *ptr) {
  double v = 0.0;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.cg.f64 %0, [%1];\n}"
               : "+d"(v) : "l"(ptr), "r"((int)p));
  return v;
}
__device__ __forceinline__ uint32_t ldg_u8_or(bool p, const uint8_t *ptr, uint32_t dflt) {
  uint32_t v = dflt;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.nc.u8 %0, [%1];\n}"
               : "+r"(v) : "l"(ptr), "r"((int)p));
  return v;
}
__device__ __forceinline__ bool before(uint32_t have, uint32_t want) { return (int32_t)(have - want) < 0; }
// named barriers: 1 = the fold warps, 2 = the gather warps
__device__ __forceinline__ void bar_fold() { asm volatile("bar.sync 1, %0;" ::"n"(TW * 32) : "memory"); }
__device__ __forceinline__ void bar_gather() { asm volatile("bar.sync 2, %0;" ::"n"(GW * 32) : "memory"); }

// Stage block b's inputs: its A rows (one CSR range) and the P rows its
// columns reference (the plan's runs of consecutive P rows), by TMA bulk
// copies completing on `bar`.  Warp 0 issues; a block without runs (too
// many / too large) reads P from global memory in the fold.
__device__ __forceinline__ void stage_block(const Ops &op, const TileArgs &ta, int b, TileTail &T, double *aval,
                                            int32_t *acol, double *pstage, int64_t *prp, int lane) {
  const int r0 = b * TR, r1 = min(r0 + TR, ta.nloc);
  const int64_t a0 = __ldg(op.ad_rp + r0), a1 = __ldg(op.ad_rp + r1);
  const int64_t c0 = a0 & ~3ll, v0 = a0 & ~1ll;
  const int64_t cend = a1 & ~3ll, vend = a1 & ~1ll;
  const int nrun = ta.pstage ? ta.pr_n[b] : 0;
  int k0 = 0, k1 = 0, k0a = 0, kcnt = 0;
  int64_t pv0 = 0, pcnt = 0;
  if (lane < nrun) {
    const int2 kr = ta.pr_k[(int64_t)b * MAXRUN + lane];
    k0 = kr.x;
    k1 = kr.y;
    k0a = k0 & ~1;
    kcnt = ((k1 + 1 - k0a) + 1) & ~1;  // row offsets k0a .. k1 (inclusive), even count
    pv0 = __ldg(op.pd_rp + k0) & ~1ll;
    pcnt = ((__ldg(op.pd_rp + k1) - pv0) + 1) & ~1ll;
  }
  int off = (int)pcnt, roff = kcnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, off, o), z = __shfl_up_sync(FULL, roff, o);
    if (lane >= o) { off += y; roff += z; }
  }
  const int ptot = __shfl_sync(FULL, off, 31), rtot = __shfl_sync(FULL, roff, 31);
  off -= (int)pcnt;
  roff -= kcnt;
  if (lane == 0) {
    T.nrun = nrun;
    fence_proxy_async();
    mbar_arrive_expect_tx(&T.bar,
                          (uint32_t)((cend - c0) * 4 + (vend - v0) * 8 + (int64_t)ptot * 8 + (int64_t)rtot * 8));
    if (ta.a_evict_first) {
      if (cend > c0) tma_bulk_g2s_stream(acol, op.ad_col + c0, (uint32_t)((cend - c0) * 4), &T.bar);
      if (vend > v0) tma_bulk_g2s_stream(aval, op.ad_val + v0, (uint32_t)((vend - v0) * 8), &T.bar);
    } else {
      if (cend > c0) tma_bulk_g2s(acol, op.ad_col + c0, (uint32_t)((cend - c0) * 4), &T.bar);
      if (vend > v0) tma_bulk_g2s(aval, op.ad_val + v0, (uint32_t)((vend - v0) * 8), &T.bar);
    }
  }
  __syncwarp();
  if (lane < nrun) {
    T.rk0[lane] = k0;
    T.rk1[lane] = k1;
    T.rvoff[lane] = off - (int)pv0;   // shared value index = global value index + rvoff
    T.rpoff[lane] = roff - k0a;       // shared row-offset index = row + rpoff
    if (pcnt) tma_bulk_g2s(pstage + off, op.pd_val + pv0, (uint32_t)(pcnt * 8), &T.bar);
    tma_bulk_g2s(prp + roff, op.pd_rp + k0a, (uint32_t)(kcnt * 8), &T.bar);
  }
  // tails of the A range (< 16 bytes) by plain loads
  if (lane < a1 - cend) acol[cend - c0 + lane] = __ldg(op.ad_col + cend + lane);
  if (lane < a1 - vend) aval[vend - v0 + lane] = __ldg(op.ad_val + vend + lane);
}

}  // namespace

// ---------------------------------------------------------------------------
// the numeric kernel
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT, 12 / (TW + GW) > 4 ? 5 : 4) k_tile_numeric(Ops op, MapArgs mp, TileArgs ta, LockArgs la, const int64_t *c_rp,
                                                          double *c_val, int blk_lo, int blk_hi, int item_hi) {
  extern __shared__ __align__(16) unsigned char tile_smem_raw[];
  double *aval = (double *)(tile_smem_raw + ta.sm_aval);
  int32_t *acol = (int32_t *)(tile_smem_raw + ta.sm_acol);
  double *pstage = (double *)(tile_smem_raw + ta.sm_pstage);
  int64_t *prp = (int64_t *)(tile_smem_raw + ta.sm_prp);
  double *accall = (double *)(tile_smem_raw + ta.sm_acc);
  double *g_pv = (double *)(tile_smem_raw + ta.sm_meta);
  int32_t *g_apb = (int32_t *)(g_pv + GCAP);
  int32_t *g_blk = g_apb + GCAP;
  TileTail &T = *(TileTail *)(tile_smem_raw + ta.sm_tail);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t epoch = *(volatile const uint32_t *)(ta.ctl + 1);
  const int R = ta.ring_blocks;
  if (tid == 0) {
    mbar_init(&T.bar, 1);
    T.zero = 0;
    T.item = blk_lo + (int)atomicAdd(ta.ctl, 1u);
  }
  __syncthreads();
  uint32_t phase = 0;
  int b = T.item;
  if (warp == 0 && b < blk_hi) stage_block(op, ta, b, T, aval, acol, pstage, prp, lane);
  while (b < item_hi) {
    if (warp < TW) {
    if (b < blk_hi) {  // items past the last block only gather (the ownership delay)
      const int r0 = b * TR, r1 = min(r0 + TR, ta.nloc);
      const int64_t c0 = __ldg(op.ad_rp + r0) & ~3ll, v0 = __ldg(op.ad_rp + r0) & ~1ll;
      // ---- per-lane row setup (overlaps the copy) ----------------------------
      const int i = r0 + 2 * lane + warp;
      int len = 0, nap = 0, apo = 0;
      const uint8_t *smp = mp.smap;
      int64_t arow = 0;
      if (i < r1) {
        const int pd0 = (int)__ldg(op.pd_rp + i);
        if ((int)__ldg(op.pd_rp + i + 1) > pd0) {  // rows without P entries contribute nothing
          arow = __ldg(op.ad_rp + i);
          len = (int)(__ldg(op.ad_rp + i + 1) - arow);
          smp += (int64_t)(__ldg((const unsigned long long *)mp.smap_rp + i) & SMAP_OFF_MASK);
          nap = __ldg(mp.nap + i);
          apo = __ldg(ta.ap_off + i);
        }
      }
      mbar_wait(&T.bar, phase);
      phase ^= 1u;
      bar_fold();
      // ---- fold: one row per lane, [slot][lane] accumulators ------------------
      double *acc = accall + warp * ta.napc * AST;
      if (la.cls != nullptr && !(ta.dbg & 8)) {
        // The class-lockstep fold (ptap_lock.cu): the lane walks its class's
        // slot-major program -- per pair an A value and a Q row start from the
        // staged block, a P value from the class-major copy Q -- with the
        // reference's arithmetic: the first product of a slot sets it, the
        // others are added in fold order, each multiply and add rounded on its
        // own (src/_kernels.py:116-147), so AP rows keep the reference's bits.
        uint4 k0 = make_uint4(0u, 0u, 0u, 0u), k1 = k0;
        if (i < r1) {
          const uint4 *kp = (const uint4 *)(la.cls + __ldg(la.rowcls + i));
          k0 = __ldg(kp);
          k1 = __ldg(kp + 1);
        }
        const int K_alen = (int)(k0.x & 0xffu);
        const unsigned long long K_sub = ((unsigned long long)k1.y << 32) | k1.x;
        const unsigned long long K_s0 = ((unsigned long long)k1.w << 32) | k1.z;
        const bool prog = (int)(K_sub >> 56) > 0;
        const int tc = (int)(arow - c0), tv = (int)(arow - v0);
        if (prog)
#pragma unroll 4
          for (int j = 0; j < K_alen; ++j) acol[tc + j] = (int32_t)__ldg(la.pq + acol[tc + j]);
        __syncwarp();
        const uint32_t a_sa = smem_u32(aval) + (prog ? (uint32_t)tv * 8u : 0u);
        const uint32_t c_sa = prog ? smem_u32(acol) + (uint32_t)tc * 4u : smem_u32(&T.zero);
        const uint2 *zchunk = la.fold + la.fold_zero;
#pragma unroll 1
        for (int sw = 0; sw < la.lw; ++sw) {  // the sub-programs one after the other (each ends on a slot boundary)
          const int c_lo = (int)((K_sub >> (8 * sw)) & 0xffu), c_hi = (int)((K_sub >> (8 * (sw + 1))) & 0xffu);
          const int nch = c_hi - c_lo;
          const int nchmax = __reduce_max_sync(FULL, nch);
          const uint2 *fp = la.fold + k0.z + (size_t)c_lo * 8;
          uint32_t o_sa = smem_u32(acc) + (uint32_t)((int)((K_s0 >> (8 * sw)) & 0xffu) * AST + lane) * 8u;
          double a = 0.0;
          bool fresh = true;
#pragma unroll 1
          for (int c = 0; c < nchmax; ++c) {
            const uint4 *src = (const uint4 *)(c < nch ? fp + c * 8 : zchunk);
            uint2 e[8];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const uint4 v = __ldg(src + u);
              e[2 * u] = make_uint2(v.x, v.y);
              e[2 * u + 1] = make_uint2(v.z, v.w);
            }
            double av[8], pv[8];
            uint32_t qi[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              asm volatile("ld.shared.f64 %0, [%1];" : "=d"(av[u]) : "r"(a_sa + (e[u].x & 0xffu)));
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(qi[u]) : "r"(c_sa + (e[u].x >> 16)));
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) pv[u] = __ldg(la.Q + (qi[u] + e[u].y));
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const double prod = __dmul_rn(av[u], pv[u]);
              a = fresh ? prod : __dadd_rn(a, prod);
              fresh = false;
              if (e[u].x & 0x8000u) {
                asm volatile("st.shared.f64 [%0], %1;" ::"r"(o_sa), "d"(a) : "memory");
                o_sa += (uint32_t)AST * 8u;
                fresh = true;
              }
            }
          }
        }
        __syncwarp();
      } else {
      const int nrun = T.nrun;
      const double *pbase = nrun ? pstage : op.pd_val;  // staged P rows, or global memory
      const int tc = (int)(arow - c0), tv = (int)(arow - v0);
      const int maxlen = (ta.dbg & 8) ? 0 : __reduce_max_sync(FULL, len);
      int run = 0, r = 0;
      // entry e's A value, P row (offset into pbase) and length; the next
      // entry's are loaded while this one's updates run
      int nps = 0, npl = 0;
      double na = 0.0;
      auto fetch = [&](int e) {
        npl = 0;
        if (e < len) {
          const int k = acol[tc + e];
          na = aval[tv + e];
          if (nrun) {
            while (k >= T.rk1[r]) ++r;  // a row's columns ascend: the run index only moves forward
            const int x = k + T.rpoff[r];
            const int pk0 = (int)prp[x];
            npl = (int)prp[x + 1] - pk0;
            nps = pk0 + T.rvoff[r];
          } else {
            const int pk0 = (int)__ldg(op.pd_rp + k);
            npl = (int)__ldg(op.pd_rp + k + 1) - pk0;
            nps = pk0;
          }
        }
      };
      fetch(0);
#pragma unroll 1
      for (int e = 0; e < maxlen; ++e) {
        const double ae = na;
        const int pse = nps, ple = npl;
        fetch(e + 1);
        const int maxpl = __reduce_max_sync(FULL, ple);
#pragma unroll 1
        for (int u0 = 0; u0 < maxpl; u0 += 4) {
          double pv[4], old[4];
          uint32_t sb[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool act = u0 + q < ple;
            pv[q] = act ? pbase[pse + u0 + q] : 0.0;
            sb[q] = ldg_u8_or(act, smp + run + u0 + q, 0x80u);
          }
          // the slots of one entry's P row are distinct: load, then store
#pragma unroll
          for (int q = 0; q < 4; ++q) old[q] = (sb[q] & 0x80) ? 0.0 : acc[(sb[q] & 0x7f) * AST + lane];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (u0 + q < ple) {
              const double prod = __dmul_rn(ae, pv[q]);
              acc[(sb[q] & 0x7f) * AST + lane] = (sb[q] & 0x80) ? prod : __dadd_rn(old[q], prod);
            }
          }
        }
        run += ple;
      }
      }
      __syncwarp();
      // ---- the ring slot must have been read by every reader of its previous
      //      occupant (this pass), then AP rows -> ring, publish ---------------
      if (tid == 0 && b >= R && !(ta.dbg & 1)) {
        const int q = b - R;
        const uint32_t want = epoch * ta.expect[q];
        while (before(ld_relaxed_u32(ta.readcnt + q), want)) __nanosleep(64);
      }
      bar_fold();
      double *ringb = ta.ring + (size_t)(b % R) * (size_t)ta.blkcap;
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        const int nj = __shfl_sync(FULL, nap, j), oj = __shfl_sync(FULL, apo, j);
        if (lane < nj) ringb[oj + lane] = acc[lane * AST + j];
      }
      bar_fold();
      if (tid == 0) st_release_u32(ta.flags + b, epoch);  // cumulative over the CTA's ring stores (bar.sync)
    }
    // ---- next item: its copies overlap the rest of this item's gather --------
    if (tid == 0) T.next = blk_lo + (int)atomicAdd(ta.ctl, 1u);
    bar_fold();
    const int bn = T.next;
    if (warp == 0 && bn < blk_hi) stage_block(op, ta, bn, T, aval, acol, pstage, prp, lane);
    } else {
    // ---- gather: the item's C rows (contiguous; owner >= last block + delay) --
    {
      const int gt = tid - TW * 32, gw = warp - TW;
      const int j1 = (ta.dbg & 4) ? ta.own_rp[b] : ta.own_rp[b + 1];
      for (int ja = ta.own_rp[b]; ja < j1;) {
        // chunk [ja, jb) of C rows whose contributor entries fit the stage
        if (gt == 0) {
          int jb = ja + 1;
          const int tA = ta.t_rp[ja];
          while (jb < j1 && ta.t_rp[jb + 1] - tA <= GCAP) ++jb;
          T.jb = jb;
        }
        bar_gather();
        const int jb = T.jb, tA = ta.t_rp[ja], tB = ta.t_rp[jb];
        // contributor metadata of the whole chunk at once (coalesced, one
        // latency for all of them), then wait for their blocks' flags
        for (int t = tA + gt; t < tB; t += GW * 32) {
          const int ii = ta.t_row[t];
          const int bk = ii / TR;
          g_pv[t - tA] = __ldg(op.pd_val + ta.t_pidx[t]);
          g_apb[t - tA] = (bk % R) * ta.blkcap + __ldg(ta.ap_off + ii);
          g_blk[t - tA] = bk;
        }
        bar_gather();
        if (!(ta.dbg & 2))
          for (int t = gt; t < tB - tA; t += GW * 32) {
            const int bk = g_blk[t];
            if (bk != b)
              while (before(ld_relaxed_u32(ta.flags + bk), epoch)) __nanosleep(32);
          }
        bar_gather();
        for (int J = ja + gw; J < jb; J += GW) {
          const int t0 = ta.t_rp[J] - tA, nk = ta.t_rp[J + 1] - tA - t0;
          const int64_t cb0 = c_rp[J];
          const int w = (int)(c_rp[J + 1] - cb0);
          const uint8_t *qm = ta.qmap + ta.qmap_rp[J];
          // lane c owns positions c and c + 32 of C row J; contributors in
          // ascending row order: slot bytes, then AP values, then the sums
          double acc0 = 0.0, acc1 = 0.0;
          if (w <= 32) {  // one position per lane, 16 contributors in flight
#pragma unroll 1
            for (int k0 = 0; k0 < nk; k0 += 16) {
              uint32_t s0[16];
              double v0[16];
#pragma unroll
              for (int u = 0; u < 16; ++u) s0[u] = ldg_u8_or(k0 + u < nk && lane < w, qm + (k0 + u) * w + lane, 0xffu);
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const int ab = g_apb[t0 + min(k0 + u, nk - 1)];
                v0[u] = ld_cg_f64_if(s0[u] != 0xffu, ta.ring + ab + (s0[u] & 0xff));
              }
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                // an absent entry adds pk * 0 = +-0: the running sum starts at
                // +0 and a round-to-nearest sum of +0-started terms is never
                // -0, so adding a signed zero leaves its bits unchanged
                const double pk = (k0 + u < nk) ? g_pv[t0 + k0 + u] : 0.0;
                acc0 = __dadd_rn(acc0, __dmul_rn(pk, v0[u]));
              }
            }
          } else {
#pragma unroll 1
            for (int k0 = 0; k0 < nk; k0 += 8) {
              uint32_t s0[8], s1[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int kk = k0 + u;
                s0[u] = ldg_u8_or(kk < nk, qm + kk * w + lane, 0xffu);
                s1[u] = ldg_u8_or(kk < nk && lane + 32 < w, qm + kk * w + lane + 32, 0xffu);
              }
              double v0[8], v1[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int ab = g_apb[t0 + min(k0 + u, nk - 1)];
                v0[u] = ld_cg_f64_if(s0[u] != 0xffu, ta.ring + ab + (s0[u] & 0xff));
                v1[u] = ld_cg_f64_if(s1[u] != 0xffu, ta.ring + ab + (s1[u] & 0xff));
              }
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const double pk = (k0 + u < nk) ? g_pv[t0 + k0 + u] : 0.0;
                acc0 = __dadd_rn(acc0, __dmul_rn(pk, v0[u]));
                acc1 = __dadd_rn(acc1, __dmul_rn(pk, v1[u]));
              }
            }
          }
          if (lane < w) c_val[cb0 + lane] = acc0;
          if (lane + 32 < w) c_val[cb0 + lane + 32] = acc1;
        }
        bar_gather();
        ja = jb;
      }
    }
    }
    // ---- item end: signal the blocks this item read ---------------------------
    __syncthreads();
    for (int q = ta.rd_rp[b] + tid; q < ta.rd_rp[b + 1]; q += NT) red_relaxed_add_u32(ta.readcnt + ta.rd_blk[q], 1u);
    b = T.next;
    __syncthreads();
  }
}

// one numeric pass: new epoch, ticket reset (graph-capturable, no host sync)
__global__ void k_tile_begin(uint32_t *ctl) {
  ctl[0] = 0u;
  ctl[1] += 1u;
}
// range launches of one pass share its epoch: only the ticket is reset
__global__ void k_tile_ticket_reset(uint32_t *ctl) { ctl[0] = 0u; }

// dynamic shared memory layout of k_tile_numeric for a plan (offsets in ta)
size_t tile_smem_layout(TileArgs &ta, int amax_blk, int pvmax, int prmax) {
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  size_t o = 0;
  ta.sm_aval = (int32_t)o;
  o = al(o + 8 * (size_t)(amax_blk + 2));
  ta.sm_acol = (int32_t)o;
  o = al(o + 4 * (size_t)(amax_blk + 4));
  ta.sm_pstage = (int32_t)o;
  o = al(o + 8 * (size_t)std::max(pvmax, 2));
  ta.sm_prp = (int32_t)o;
  o = al(o + 8 * (size_t)std::max(prmax, 2));
  ta.sm_acc = (int32_t)o;
  o = al(o + (size_t)TW * ta.napc * AST * 8);
  ta.sm_meta = (int32_t)o;
  o = al(o + (size_t)GCAP * 16);
  ta.sm_tail = (int32_t)o;
  o = al(o + sizeof(TileTail));
  ta.sm_total = (int32_t)o;
  return o;
}

cudaError_t launch_tile_numeric(const Ops &op, const MapArgs &mp, const TileArgs &ta, const LockArgs &la,
                                const int64_t *c_rp, double *c_val, int blk_lo, int blk_hi, bool new_pass,
                                cudaStream_t st) {
  if (new_pass) k_tile_begin<<<1, 1, 0, st>>>(ta.ctl);
  else k_tile_ticket_reset<<<1, 1, 0, st>>>(ta.ctl);
  // the lockstep fold reads P's values class-major: refresh the copy once per pass
  if (new_pass && la.cls != nullptr) {
    cudaError_t pe = launch_lock_permute_f64(la.nloc, op.pd_rp, la.pq, la.ltab, op.pd_val, la.Q, st);
    if (pe != cudaSuccess) return pe;
  }
  // the last range of a pass also runs the gather-only items of the delay
  const int item_hi = blk_hi >= ta.nblk ? ta.nitems : blk_hi;
  if (item_hi <= blk_lo) return cudaGetLastError();
  cudaError_t e = cudaFuncSetAttribute(k_tile_numeric, cudaFuncAttributeMaxDynamicSharedMemorySize, ta.sm_total);
  if (e != cudaSuccess) return e;
  const int grid = std::min(ta.grid, item_hi - blk_lo);
  k_tile_numeric<<<grid, NT, ta.sm_total, st>>>(op, mp, ta, la, c_rp, c_val, blk_lo, std::min(blk_hi, ta.nblk),
                                                     item_hi);
  return cudaGetLastError();
}

int tile_grid(const TileArgs &ta) {
  int dev = 0, nsm = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(k_tile_numeric, cudaFuncAttributeMaxDynamicSharedMemorySize, ta.sm_total);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tile_numeric, NT, ta.sm_total) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  return nsm * per_sm;
}

// ---------------------------------------------------------------------------
// plan construction (symbolic)
// ---------------------------------------------------------------------------

// P_d^T counts: contributors of each local C row
__global__ void k_tile_tcount(int64_t nnz, const int32_t *pd_col, int32_t *cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + pd_col[e], 1);
}

// P_d^T scatter: (fine row, index of the entry in its P row)
__global__ void k_tile_tscatter(int64_t n, const int64_t *pd_rp, const int32_t *pd_col, const int32_t *t_rp,
                                int32_t *cursor, int32_t *t_row, uint8_t *t_jx, int *status) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p0 = pd_rp[i], p1 = pd_rp[i + 1];
    if (p1 - p0 > 255) atomicOr(status, ST_ROW_TOO_WIDE);
    for (int64_t e = p0; e < p1; ++e) {
      const int32_t J = pd_col[e];
      const int pos = t_rp[J] + atomicAdd(cursor + J, 1);
      t_row[pos] = (int32_t)i;
      t_jx[pos] = (uint8_t)(e - p0);
    }
  }
}

// sort each C row's contributors by row (ascending: the reference's order),
// write its P value index, and the key of the balanced owner assignment:
// owner(J) = floor(O_J / ncl) with O_J = J * nblk + max_{J' <= J} ((L_J' + delay) * ncl - J' * nblk),
// L = block of the last contributor.  This is the smallest non-decreasing
// assignment with owner(J) >= L_J + delay that hands out C rows at the
// average rate of ncl / nblk rows per item, so gathers are spread evenly
// over the items (a lexicographic grid concentrates the last contributors of
// C in one block of four) and each item owns a contiguous range of C rows.
__global__ void k_tile_tsort(int64_t ncl, int nblk, int delay, const int64_t *pd_rp, const int32_t *t_rp,
                             int32_t *t_row, uint8_t *t_jx, int32_t *t_pidx, long long *key,
                             unsigned long long *stats) {
  for (int64_t J = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; J < ncl; J += (int64_t)gridDim.x * blockDim.x) {
    const int t0 = t_rp[J], t1 = t_rp[J + 1];
    for (int a = t0 + 1; a < t1; ++a) {
      const int32_t r = t_row[a];
      const uint8_t x = t_jx[a];
      int b = a - 1;
      while (b >= t0 && t_row[b] > r) {
        t_row[b + 1] = t_row[b];
        t_jx[b + 1] = t_jx[b];
        --b;
      }
      t_row[b + 1] = r;
      t_jx[b + 1] = x;
    }
    for (int a = t0; a < t1; ++a) t_pidx[a] = (int32_t)pd_rp[t_row[a]] + t_jx[a];
    const long long L = t1 > t0 ? (long long)(t_row[t1 - 1] / TR) : -(1ll << 40);
    key[J] = (L + delay) * (long long)ncl - (long long)J * nblk;
    if (t1 > t0) atomicMax(stats + 1, (unsigned long long)(t1 - t0));
  }
}

struct MaxLL {
  __device__ __forceinline__ long long operator()(long long a, long long b) const { return a > b ? a : b; }
};

// owner of every C row from the scanned keys; contributor span in items
__global__ void k_tile_owner(int64_t ncl, int nblk, const long long *scanned, const int32_t *t_rp,
                             const int32_t *t_row, int32_t *owner, unsigned long long *stats) {
  for (int64_t J = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; J < ncl; J += (int64_t)gridDim.x * blockDim.x) {
    const long long o = ((long long)J * nblk + scanned[J]) / (long long)ncl;
    const int ob = (int)(o > 0 ? o : 0);
    owner[J] = ob;
    const int t0 = t_rp[J], t1 = t_rp[J + 1];
    if (t1 > t0) atomicMax(stats + 0, (unsigned long long)(ob - t_row[t0] / TR));
    atomicMax(stats + 3, (unsigned long long)ob);
  }
}

// own_rp[i] = first C row owned by an item >= i (owners are non-decreasing)
__global__ void k_tile_own_rp(int nitems, int64_t ncl, const int32_t *owner, int32_t *own_rp) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= nitems; i += gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = ncl;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (owner[mid] < i) lo = mid + 1; else hi = mid;
    }
    own_rp[i] = (int32_t)lo;
  }
}

// AP offsets inside each block (rows in natural order, lengths rounded up to
// 2 doubles), and the largest block
__global__ void k_tile_apoff(int64_t n, const int64_t *ad_rp, const int64_t *pd_rp, const uint8_t *nap,
                             uint16_t *ap_off, unsigned long long *stats) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t r0 = w * TR;
  if (r0 >= n) return;
  int v[2], s = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t i = r0 + 2 * lane + h;
    v[h] = (i < n && pd_rp[i + 1] > pd_rp[i]) ? ((nap[i] + 1) & ~1) : 0;
    s += v[h];
  }
  int incl = s;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  int off = incl - s;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t i = r0 + 2 * lane + h;
    if (i < n) ap_off[i] = (uint16_t)off;
    off += v[h];
  }
  if (lane == 31) {
    atomicMax(stats + 2, (unsigned long long)incl);
    const int64_t r1 = (r0 + TR < n ? r0 + TR : n);
    atomicMax(stats + 4, (unsigned long long)(ad_rp[r1] - ad_rp[r0]));
  }
}

// distinct blocks read by each item's gathers (bitmap over [b - span, b]);
// pass 0 counts, pass 1 writes the lists and the per-block reader counts
__global__ void k_tile_reads(int pass, int nblk, int delay, int span, const int32_t *own_rp,
                             const int32_t *t_rp, const int32_t *t_row, int32_t *rd_cnt, const int32_t *rd_rp,
                             int32_t *rd_blk, uint32_t *expect) {
  extern __shared__ uint32_t bits_all[];
  const int wpb = blockDim.x >> 5, lane = threadIdx.x & 31;
  const int nw = (span + 1 + 31) >> 5;
  uint32_t *bits = bits_all + (threadIdx.x >> 5) * nw;
  const int b = blockIdx.x * wpb + (threadIdx.x >> 5);
  if (b >= nblk) return;
  for (int x = lane; x < nw; x += 32) bits[x] = 0;
  __syncwarp();
  for (int J = own_rp[b]; J < own_rp[b + 1]; ++J) {
    for (int t = t_rp[J] + lane; t < t_rp[J + 1]; t += 32) {
      const int d = b - delay - t_row[t] / TR;
      atomicOr(bits + (d >> 5), 1u << (d & 31));
    }
  }
  __syncwarp();
  if (pass == 0) {
    int c = 0;
    for (int x = lane; x < nw; x += 32) c += __popc(bits[x]);
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
    if (lane == 0) rd_cnt[b] = c;
  } else if (lane == 0) {
    int pos = rd_rp[b];
    for (int x = nw - 1; x >= 0; --x) {  // ascending block order
      uint32_t m = bits[x];
      while (m) {
        const int hb = 31 - __clz(m);
        m &= ~(1u << hb);
        const int q = b - delay - (x * 32 + hb);
        rd_blk[pos++] = q;
        atomicAdd(expect + q, 1u);
      }
    }
  }
}

// per C row: byte length of its gather map (contributors x row width)
__global__ void k_tile_qlen(int64_t ncl, const int32_t *t_rp, const int64_t *c_rp, int64_t *qlen) {
  for (int64_t J = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; J < ncl; J += (int64_t)gridDim.x * blockDim.x)
    qlen[J] = (int64_t)(t_rp[J + 1] - t_rp[J]) * (c_rp[J + 1] - c_rp[J]);
}

// gather map of C row J: qm[k * w + c] = slot of C(J,:)'s c-th column in the
// AP row of J's k-th contributor (ascending rows), 0xff when that row has no
// such column -- the inverse of the contributors' position maps
__global__ void k_tile_qmap(int64_t ncl, const int32_t *t_rp, const int32_t *t_row, const uint8_t *t_jx,
                            const int64_t *c_rp, const int64_t *qm_rp, const uint8_t *nap, const int64_t *pmap_rp,
                            const uint8_t *pmap, uint8_t *qm) {
  const int lane = threadIdx.x & 31;
  for (int64_t J = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; J < ncl;
       J += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int t0 = t_rp[J], nk = t_rp[J + 1] - t0;
    const int w = (int)(c_rp[J + 1] - c_rp[J]);
    uint8_t *out = qm + qm_rp[J];
    for (int x = lane; x < nk * w; x += 32) out[x] = 0xff;
    __syncwarp();
    for (int k = 0; k < nk; ++k) {
      const int ii = t_row[t0 + k], jx = t_jx[t0 + k];
      const int na = nap[ii];
      const uint8_t *pm = pmap + pmap_rp[ii] + (int64_t)jx * na;
      for (int sl = lane; sl < na; sl += 32) out[k * w + pm[sl]] = (uint8_t)sl;
    }
    __syncwarp();
  }
}

// C row J is final once the item owning it ran: report the last fine row of
// that item's range (the streamed host pass downloads rows by this)
__global__ void k_tile_c_last(int64_t ncl, int nblk, int nitems, int nloc, const int32_t *own_rp, int32_t *last) {
  for (int64_t J = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; J < ncl; J += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = nitems;  // owner: last item i with own_rp[i] <= J
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (own_rp[mid] <= J) lo = mid; else hi = mid;
    }
    last[J] = lo >= nblk ? nloc - 1 : min(nloc - 1, (lo + 1) * TR - 1);
  }
}

// Runs of consecutive P rows referenced by each block's A columns (the P rows
// the fold stages into shared memory).  One warp per block: a bitmap of the
// block's columns over [kmin, kmax], run starts and ends counted per lane on
// contiguous word ranges and placed by a warp scan.  Blocks whose columns
// span more than the bitmap, or need more than MAXRUN runs or more than
// pvcap staged values, get no runs (their fold reads P from global memory).
constexpr int PRUN_BITS = 1 << 18;
__global__ void k_tile_pruns(int nblk, int64_t nloc, const int64_t *ad_rp, const int32_t *ad_col,
                             const int64_t *pd_rp, int64_t pnnz, int pvcap, int prcap, uint8_t *pr_n, int2 *pr_k,
                             unsigned long long *stats) {
  extern __shared__ uint32_t pbits[];
  const int lane = threadIdx.x & 31;
  for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
    const int64_t r0 = (int64_t)b * TR, r1 = (r0 + TR < nloc ? r0 + TR : nloc);
    int kmin = INT32_MAX, kmax = -1;
    for (int64_t i = r0 + lane; i < r1; i += 32) {
      const int64_t x0 = ad_rp[i], x1 = ad_rp[i + 1];
      if (x1 > x0) { kmin = min(kmin, ad_col[x0]); kmax = max(kmax, ad_col[x1 - 1]); }
    }
    kmin = __reduce_min_sync(FULL, kmin);
    kmax = __reduce_max_sync(FULL, kmax);
    int nrun = 0;
    if (kmax >= kmin && kmax - kmin < PRUN_BITS) {
      const int nw = (kmax - kmin + 32) >> 5;
      for (int x = lane; x < nw; x += 32) pbits[x] = 0u;
      __syncwarp();
      for (int64_t e = ad_rp[r0] + lane; e < ad_rp[r1]; e += 32) {
        const int d = ad_col[e] - kmin;
        atomicOr(pbits + (d >> 5), 1u << (d & 31));
      }
      __syncwarp();
      const int per = (nw + 31) / 32, w0 = min(nw, lane * per), w1 = min(nw, w0 + per);
      int ns = 0, ne = 0;
      for (int x = w0; x < w1; ++x) {
        const uint32_t w = pbits[x];
        const uint32_t prev = x > 0 ? (pbits[x - 1] >> 31) : 0u, next = x + 1 < nw ? (pbits[x + 1] & 1u) : 0u;
        ns += __popc(w & ~((w << 1) | prev));
        ne += __popc(w & ~((w >> 1) | (next << 31)));
      }
      int is = ns, ie = ne;
      for (int o = 1; o < 32; o <<= 1) {
        const int ys = __shfl_up_sync(FULL, is, o), ye = __shfl_up_sync(FULL, ie, o);
        if (lane >= o) { is += ys; ie += ye; }
      }
      nrun = __shfl_sync(FULL, is, 31);
      if (nrun <= MAXRUN) {
        int ps = is - ns, pe = ie - ne;
        int2 *out = pr_k + (int64_t)b * MAXRUN;
        for (int x = w0; x < w1; ++x) {
          const uint32_t w = pbits[x];
          const uint32_t prev = x > 0 ? (pbits[x - 1] >> 31) : 0u, next = x + 1 < nw ? (pbits[x + 1] & 1u) : 0u;
          uint32_t st = w & ~((w << 1) | prev), en = w & ~((w >> 1) | (next << 31));
          while (st) { const int bt = __ffs(st) - 1; st &= st - 1; out[ps++].x = kmin + x * 32 + bt; }
          while (en) { const int bt = __ffs(en) - 1; en &= en - 1; out[pe++].y = kmin + x * 32 + bt + 1; }
        }
        __syncwarp();
        // staged values (even-aligned per run, as k_tile_numeric copies them)
        int64_t tot = 0, rtot = 0;
        bool ok = true;
        if (lane < nrun) {
          const int2 kr = out[lane];
          const int64_t v0 = pd_rp[kr.x] & ~1ll, cnt = ((pd_rp[kr.y] - v0) + 1) & ~1ll;
          const int64_t k0a = kr.x & ~1, kcnt = ((kr.y + 1 - k0a) + 1) & ~1ll;
          tot = cnt;
          rtot = kcnt;
          ok = v0 + cnt <= pnnz && k0a + kcnt <= nloc + 1;  // the copies may not read past the arrays
        }
        for (int o = 16; o; o >>= 1) {
          tot += __shfl_xor_sync(FULL, tot, o);
          rtot += __shfl_xor_sync(FULL, rtot, o);
        }
        ok = __all_sync(FULL, ok);
        if (!ok || tot > pvcap || rtot > prcap) {
          nrun = 0;
        } else if (lane == 0) {
          atomicMax(stats + 5, (unsigned long long)tot);
          atomicMax(stats + 7, (unsigned long long)rtot);
        }
      } else {
        nrun = 0;
      }
      __syncwarp();
    }
    if (lane == 0) {
      pr_n[b] = (uint8_t)nrun;
      if (nrun) atomicAdd(stats + 6, 1ull);
    }
  }
}

cudaError_t launch_tile_pruns(int nblk, int64_t nloc, const int64_t *ad_rp, const int32_t *ad_col,
                              const int64_t *pd_rp, int64_t pnnz, int pvcap, int prcap, uint8_t *pr_n, int2 *pr_k,
                              unsigned long long *stats, cudaStream_t st) {
  if (nblk <= 0) return cudaSuccess;
  const size_t sm = PRUN_BITS / 8;
  cudaError_t e = cudaFuncSetAttribute(k_tile_pruns, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k_tile_pruns<<<std::min(nblk, 148 * 6), 32, sm, st>>>(nblk, nloc, ad_rp, ad_col, pd_rp, pnnz, pvcap, prcap, pr_n,
                                                       pr_k, stats);
  return cudaGetLastError();
}

static inline int gblocks(int64_t n, int t) {
  int64_t g = (n + t - 1) / t;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 64));
}

cudaError_t launch_tile_transpose(int64_t n, int64_t ncl, const int64_t *pd_rp, const int32_t *pd_col,
                                  int64_t pnnz, int32_t *cnt, int32_t *t_rp, int32_t *cursor, int32_t *t_row,
                                  uint8_t *t_jx, void *scratch, size_t scratch_bytes, int *status,
                                  cudaStream_t st) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (ncl + 1), st)) != cudaSuccess) return e;
  if (pnnz > 0) k_tile_tcount<<<gblocks(pnnz, 256), 256, 0, st>>>(pnnz, pd_col, cnt);
  size_t bytes = scratch_bytes;
  if ((e = cub::DeviceScan::ExclusiveSum(scratch, bytes, cnt, t_rp, (int)(ncl + 1), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(cursor, 0, sizeof(int32_t) * (ncl + 1), st)) != cudaSuccess) return e;
  if (n > 0) k_tile_tscatter<<<gblocks(n, 256), 256, 0, st>>>(n, pd_rp, pd_col, t_rp, cursor, t_row, t_jx, status);
  return cudaGetLastError();
}

size_t tile_scan_scratch(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int32_t *)nullptr, (int32_t *)nullptr, (int)(n + 1));
  return bytes;
}

size_t tile_owner_scratch(int64_t ncl) {
  size_t bytes = 0;
  cub::DeviceScan::InclusiveScan(nullptr, bytes, (long long *)nullptr, (long long *)nullptr, MaxLL(), (int)ncl);
  return bytes;
}

cudaError_t launch_tile_owners(int64_t ncl, int nblk, int delay, const int64_t *pd_rp, const int32_t *t_rp,
                               int32_t *t_row, uint8_t *t_jx, int32_t *t_pidx, long long *key, int32_t *owner,
                               unsigned long long *stats, void *scratch, size_t scratch_bytes, cudaStream_t st) {
  if (ncl <= 0) return cudaSuccess;
  k_tile_tsort<<<gblocks(ncl, 128), 128, 0, st>>>(ncl, nblk, delay, pd_rp, t_rp, t_row, t_jx, t_pidx, key, stats);
  size_t bytes = scratch_bytes;
  cudaError_t e = cub::DeviceScan::InclusiveScan(scratch, bytes, key, key, MaxLL(), (int)ncl, st);
  if (e != cudaSuccess) return e;
  k_tile_owner<<<gblocks(ncl, 256), 256, 0, st>>>(ncl, nblk, key, t_rp, t_row, owner, stats);
  return cudaGetLastError();
}

cudaError_t launch_tile_own_rp(int nitems, int64_t ncl, const int32_t *owner, int32_t *own_rp, cudaStream_t st) {
  k_tile_own_rp<<<gblocks(nitems + 1, 256), 256, 0, st>>>(nitems, ncl, owner, own_rp);
  return cudaGetLastError();
}

cudaError_t launch_tile_apoff(int64_t n, const int64_t *ad_rp, const int64_t *pd_rp, const uint8_t *nap,
                              uint16_t *ap_off, unsigned long long *stats, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t nblk = (n + TR - 1) / TR;
  k_tile_apoff<<<(int)((nblk * 32 + 255) / 256), 256, 0, st>>>(n, ad_rp, pd_rp, nap, ap_off, stats);
  return cudaGetLastError();
}

cudaError_t launch_tile_reads(int pass, int nitems, int delay, int span, const int32_t *own_rp,
                              const int32_t *t_rp, const int32_t *t_row, int32_t *rd_cnt,
                              const int32_t *rd_rp, int32_t *rd_blk, uint32_t *expect, cudaStream_t st) {
  const int nblk = nitems;
  if (nblk <= 0) return cudaSuccess;
  const int wpb = 4;
  const size_t sm = (size_t)wpb * ((span + 1 + 31) / 32) * 4;
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_tile_reads, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  k_tile_reads<<<(nblk + wpb - 1) / wpb, wpb * 32, sm, st>>>(pass, nblk, delay, span, own_rp, t_rp, t_row,
                                                             rd_cnt, rd_rp, rd_blk, expect);
  return cudaGetLastError();
}

cudaError_t launch_tile_qmap(int64_t ncl, const TileArgs &ta, const int64_t *c_rp, int64_t *qlen, int64_t *qm_rp,
                             const uint8_t *nap, const int64_t *pmap_rp, const uint8_t *pmap, uint8_t *qm, int pass,
                             cudaStream_t st) {
  if (ncl <= 0) return cudaSuccess;
  if (pass == 0) k_tile_qlen<<<gblocks(ncl, 256), 256, 0, st>>>(ncl, ta.t_rp, c_rp, qlen);
  else k_tile_qmap<<<gblocks(ncl * 32, 256), 256, 0, st>>>(ncl, ta.t_rp, ta.t_row, ta.t_jx, c_rp, qm_rp, nap, pmap_rp,
                                                           pmap, qm);
  return cudaGetLastError();
}

cudaError_t launch_tile_c_last(int64_t ncl, const TileArgs &ta, int32_t *last, cudaStream_t st) {
  if (ncl > 0)
    k_tile_c_last<<<gblocks(ncl, 256), 256, 0, st>>>(ncl, ta.nblk, ta.nitems, ta.nloc, ta.own_rp, last);
  return cudaGetLastError();
}

cudaError_t launch_tile_scan32(const int32_t *in, int32_t *out, int n, void *scratch, size_t scratch_bytes,
                               cudaStream_t st) {
  size_t bytes = scratch_bytes;
  return cub::DeviceScan::ExclusiveSum(scratch, bytes, in, out, n + 1, st);
}

}  // namespace ptapdev
