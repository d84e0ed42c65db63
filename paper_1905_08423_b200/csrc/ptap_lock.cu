// ptap_lock.cu -- class-lockstep numeric pass of the all-at-once / merged
// triple product (one-rank structure: no A_o, no P_o; the q4a plan).
//
// The reference folds one fine row at a time (src/_kernels.py:446-515):
// AP(i,:) = sum_k A(i,k) P(k,:) into a hash, then C(J,:) += P(i,J) AP(i,:)
// for every J of P(i,:).  The plan's interned maps (ptap_mapped.cu) already
// say that rows of one structural class -- same A row length, same P row
// lengths of its columns, same slot map, same position map -- run the same
// sequence of multiply-adds on different data.  This kernel runs 32 rows of
// one class in lockstep, one row per lane:
//
//   * rows are cut into tiles of 64 consecutive fine rows; the plan sorts
//     each tile's rows by class and cuts the classes into groups of <= 32 rows
//     (on a lexicographic grid: the even-x and the odd-x rows of a line);
//   * a tile's A rows (one contiguous CSR range) come into shared memory by
//     TMA bulk copies (cp.async.bulk + mbarrier), A is read exactly once;
//   * P's values are read from a class-major copy Q (k_lock_permute, once per
//     pass): rows of P with L entries are stored entry-major, Q_L[t][rank],
//     in ascending row order, so the 32 lanes of a group, whose neighbours of
//     one role are consecutive rows of one length, load consecutive doubles;
//   * the class's fold program lists its (A entry, P entry) pairs SLOT-MAJOR,
//     so a lane accumulates one AP slot at a time in a register (no
//     read-modify-write of a shared accumulator, no per-pair slot byte) and
//     stores it once into the warp's AP buffer;
//   * the outer products run transposed: for each row of the group the lanes
//     take the (target row, AP slot) items of the class's outer program, so
//     the fp64 reductions of one instruction fall into a few C rows.
//
// Every index in the inner loops is warp-uniform (the program) or a lane
// register (the row's staging offset).  The result differs from the
// reference only in summation order (fused multiply-adds, slot-major fold,
// atomic C updates): the default pass's parity gate (row-scaled 1e-12)
// applies; the deterministic pass (ptap_tile.cu) keeps the reference order.
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <cstdint>
#include <cstdlib>

#include "ptap_device.cuh"
#include "ptap_kernels.cuh"

namespace ptapdev {

namespace {

constexpr int LT = LOCK_TILE;  // fine rows per tile
constexpr int TGS = 33;              // stride of the per-target arrays (bank-conflict free both ways)
constexpr unsigned FULLM = 0xffffffffu;

__device__ __forceinline__ uint32_t sm_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void lk_mbar_init(unsigned long long *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void lk_mbar_expect(unsigned long long *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void lk_mbar_wait(unsigned long long *bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "LOCK_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LOCK_WAIT_%=;\n}" ::"r"(sm_u32(bar)),
      "r"(phase)
      : "memory");
}
// A is streamed once: evict-first in L2, which stays with Q, C and the programs
__device__ __forceinline__ void lk_bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
  asm volatile(
      "{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      " cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n}"
      ::"r"(sm_u32(dst)), "l"(src), "r"(bytes), "r"(sm_u32(bar))
      : "memory");
}
__device__ __forceinline__ double lk_lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lk_lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void lk_sts_f64(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

__device__ __forceinline__ unsigned long long lk_mix(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

}  // namespace

// ---------------------------------------------------------------------------
// The numeric kernel: one CTA per tile, W warps per group of 32 rows.
// Dynamic shared memory: aval[acap] | acol[acap] | rs[LT + 4] | per group
// { ap[32 * aps], tgv[8 * TGS], tgc[8 * TGS] } | mbarrier
// ---------------------------------------------------------------------------
constexpr int LG = LT / 32;  // groups per tile
template <int LW>
__device__ __forceinline__ void lk_group_bar(int g) {
  if (g == 0)
    asm volatile("bar.sync 1, %0;" ::"n"(LW * 32) : "memory");
  else
    asm volatile("bar.sync 2, %0;" ::"n"(LW * 32) : "memory");
}

template <int LW>
__global__ void __launch_bounds__(LG * LW * 32) k_lock_numeric(Ops op, LockArgs la, double *__restrict__ c_val,
                                                               int tile0, int *status) {
  extern __shared__ __align__(16) unsigned char lsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = warp / LW, w = warp - g * LW;
  double *aval = (double *)lsm;
  uint32_t *acol = (uint32_t *)(aval + la.acap);
  int32_t *rs = (int32_t *)(acol + la.acap);
  unsigned char *wbase = (unsigned char *)(rs + LT + 4);
  const int wbytes = (32 * la.aps + 8 * TGS) * 8 + 8 * TGS * 4 + 8;
  unsigned long long *bar = (unsigned long long *)(wbase + (size_t)LG * wbytes);
  double *ap = (double *)(wbase + (size_t)g * wbytes);
  double *tgv = ap + 32 * la.aps;
  int32_t *tgc = (int32_t *)(tgv + 8 * TGS);

  const int tile = tile0 + blockIdx.x;
  const int r0 = tile * LT, r1 = min(r0 + LT, la.nloc);
  const int64_t a0 = __ldg(op.ad_rp + r0), a1 = __ldg(op.ad_rp + r1);
  const int64_t c0 = a0 & ~3ll, cend = a1 & ~3ll;
  if (a1 < a0 || a1 - c0 > (int64_t)la.acap) {  // A's row offsets are not the symbolic ones
    if (tid == 0) atomicOr(status, ST_DRIFT);
    return;
  }
  if (tid == 0) lk_mbar_init(bar, 1);
  __syncthreads();
  if (tid == 0) {
    const uint32_t n = (uint32_t)(cend - c0);
    lk_mbar_expect(bar, n * 12u);
    if (n) {
      lk_bulk_g2s(acol, op.ad_col + c0, n * 4u, bar);
      lk_bulk_g2s(aval, op.ad_val + c0, n * 8u, bar);
    }
  }
  // tails of the range (< 16 bytes each) and the rows' staging offsets
  if (tid < (int)(a1 - cend)) {
    acol[cend - c0 + tid] = (uint32_t)__ldg(op.ad_col + cend + tid);
    aval[cend - c0 + tid] = __ldg(op.ad_val + cend + tid);
  }
  if (tid <= r1 - r0) rs[tid] = (int32_t)(__ldg(op.ad_rp + r0 + tid) - c0);
  if (tid == 0) rs[LT + 2] = 0;
  // the lane's row (sorted position 32 g + lane of the tile) and its class
  const int cnt = min(32, r1 - r0 - 32 * g);
  const bool active = lane < cnt;
  uint4 k0 = make_uint4(0u, 0u, 0u, 0u), k1 = k0;  // the class header, field by field (no local-memory struct)
  int q = 0;
  if (active) {
    const uint32_t info = __ldg(la.rowinfo + r0 + 32 * g + lane);
    q = (int)(info & 0xffu);
    const uint4 *kp = (const uint4 *)(la.cls + (info >> 8));
    k0 = __ldg(kp);
    k1 = __ldg(kp + 1);
  }
  __syncthreads();
  lk_mbar_wait(bar, 0);
  if (cnt <= 0) return;
  const int i = r0 + q, rsl = rs[q];
  if (active && rs[q + 1] - rsl != (int)(k0.x & 0xffu)) {  // not the row its class was built from
    atomicOr(status, ST_DRIFT);
    k0 = k1 = make_uint4(0u, 0u, 0u, 0u);
  }
  const int K_alen = (int)(k0.x & 0xffu), K_ntg = (int)((k0.x >> 16) & 0xffu), K_niter = (int)(k0.x >> 24);
  const uint32_t K_tstride = k0.y, K_fold_off = k0.z, K_outer_off = k0.w;
  const unsigned long long K_sub = ((unsigned long long)k1.y << 32) | k1.x, K_s0 = ((unsigned long long)k1.w << 32) | k1.z;
  const int sub_lo = (int)((K_sub >> (8 * w)) & 0xffu), sub_hi = (int)((K_sub >> (8 * (w + 1))) & 0xffu);
  const int sub_all = (int)(K_sub >> 56), slot0 = (int)((K_s0 >> (8 * w)) & 0xffu);
  const uint32_t aval_sa = sm_u32(aval), acol_sa = sm_u32(acol);
  const uint32_t ap_sa0 = sm_u32(ap), tgv_sa = sm_u32(tgv), tgc_sa = sm_u32(tgc);

  // columns -> Q index of the column's P row.  The raw tile keeps rows of one
  // parity an even number of words apart (2-way bank conflicts for a lane per
  // row), so the converted indices are written back transposed: sorted row r
  // of group g at the odd stride la.ast, conflict-free for the fold.  All raw
  // columns are read (into registers) before any converted one is written.
  constexpr int CQ = (32 + LW - 1) / LW;
  uint32_t cq[CQ];
  const bool conv = sub_all > 0 && !(la.dbg & 4);
#pragma unroll
  for (int jj = 0; jj < CQ; ++jj) {
    const int j = w + jj * LW;
    cq[jj] = 0u;
    if (conv && j < K_alen) cq[jj] = __ldg(la.pq + acol[rsl + j]);
  }
  __syncthreads();
  const uint32_t c_row_sa = acol_sa + (uint32_t)((g * 32 + lane) * la.ast) * 4u;
#pragma unroll
  for (int jj = 0; jj < CQ; ++jj) {
    const int j = w + jj * LW;
    if (conv && j < K_alen)
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(c_row_sa + (uint32_t)j * 4u), "r"(cq[jj]) : "memory");
  }
  if (conv) {
    const uint32_t pqi = __ldg(la.pq + i);
    for (int jt = w; jt < K_ntg; jt += LW) {
      const size_t x = (size_t)pqi + (size_t)jt * K_tstride;
      tgv[jt * TGS + lane] = __ldg(la.Q + x);
      tgc[jt * TGS + lane] = __ldg(la.cbQ + x);
    }
  }
  lk_group_bar<LW>(g);

  // fold, slot-major: warp w folds the slots of its range of the lane's class
  // program; one register accumulator, stored once per slot.  Entries past a
  // lane's sub-program are zero: they read the row's first A entry and Q
  // value and accumulate into a register that is never stored (a lane with
  // no program reads Q[0] through a zero word of shared memory).
  {
    const int nch = sub_hi - sub_lo;
    const int nchmax = __reduce_max_sync(FULLM, nch);
    const uint2 *fp = la.fold + K_fold_off + (size_t)sub_lo * 8;
    const uint32_t a_sa = sub_all > 0 ? aval_sa + (uint32_t)rsl * 8u : aval_sa;
    const uint32_t c_sa = sub_all > 0 ? c_row_sa : sm_u32(rs + LT + 2);
    uint32_t o_sa = ap_sa0 + (uint32_t)(lane * la.aps + slot0) * 8u;
    double acc = 0.0;
    const uint2 *zchunk = la.fold + la.fold_zero;  // eight zero entries
    auto load = [&](uint2(&e)[8], int c) {
      const uint4 *src = (const uint4 *)(c < nch ? fp + c * 8 : zchunk);  // chunks are 64-byte aligned
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint4 v = __ldg(src + u);
        e[2 * u] = make_uint2(v.x, v.y);
        e[2 * u + 1] = make_uint2(v.z, v.w);
      }
    };
    auto process = [&](const uint2(&e)[8]) {
      double av[8], pv[8];
      uint32_t qi[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        av[u] = lk_lds_f64(a_sa + (e[u].x & 0xffu));
        qi[u] = lk_lds_u32(c_sa + (e[u].x >> 16));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) pv[u] = __ldg(la.Q + (qi[u] + e[u].y));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc = fma(av[u], pv[u], acc);
        if (e[u].x & 0x8000u) {
          lk_sts_f64(o_sa, acc);
          o_sa += 8u;
          acc = 0.0;
        }
      }
    };
    // two chunks per round, the next chunk's entries loaded while one folds
    uint2 ea[8], eb[8];
    load(ea, 0);
#pragma unroll 1
    for (int c = 0; c < ((la.dbg & 2) ? 0 : nchmax); c += 2) {
      load(eb, c + 1);
      process(ea);
      if (c + 1 < nchmax) {
        load(ea, c + 2);
        process(eb);
      }
    }
  }
  lk_group_bar<LW>(g);

  // outer products, transposed: the lanes take the (target, slot) items of
  // row r's class; warp w takes rows w, w + LW, ...  The decoded program words
  // of the first two rounds stay in registers while the class does not change.
  {
    const uint32_t rstride = (uint32_t)la.aps * 8u;
    uint32_t cached = 0xffffffffu;
    uint32_t s0a = 0, tv0 = 0, tc0 = 0, ps0 = 0, s1a = 0, tv1 = 0, tc1 = 0, ps1 = 0;
    bool ok0 = false, ok1 = false;
    auto decode = [&](uint32_t off, int nit) {
      const uint32_t wd0 = nit > 0 ? __ldg(la.outer + off + lane) : 0xffffffffu;
      const uint32_t wd1 = nit > 1 ? __ldg(la.outer + off + 32 + lane) : 0xffffffffu;
      ok0 = wd0 != 0xffffffffu;
      ok1 = wd1 != 0xffffffffu;
      s0a = ap_sa0 + (wd0 & 0xffu);
      tv0 = tgv_sa + ((wd0 >> 8) & 0xffu) * (TGS * 8u);
      tc0 = tgc_sa + ((wd0 >> 8) & 0xffu) * (TGS * 4u);
      ps0 = wd0 >> 16;
      s1a = ap_sa0 + (wd1 & 0xffu);
      tv1 = tgv_sa + ((wd1 >> 8) & 0xffu) * (TGS * 8u);
      tc1 = tgc_sa + ((wd1 >> 8) & 0xffu) * (TGS * 4u);
      ps1 = wd1 >> 16;
      cached = off;
    };
    auto tail = [&](uint32_t off, int nit, int r) {  // rounds past the two cached ones (classes with > 64 items)
      const uint32_t ro = (uint32_t)r * rstride, r8 = (uint32_t)r * 8u, r4 = (uint32_t)r * 4u;
      for (int u = 2; u < nit; ++u) {
        const uint32_t wd = __ldg(la.outer + off + u * 32 + lane);
        if (wd != 0xffffffffu) {
          const uint32_t jt = (wd >> 8) & 0xffu;
          const double apv = lk_lds_f64(ap_sa0 + ro + (wd & 0xffu));
          const double tv = lk_lds_f64(tgv_sa + jt * (TGS * 8u) + r8);
          const uint32_t cb = lk_lds_u32(tgc_sa + jt * (TGS * 4u) + r4);
          atomicAdd(c_val + (cb + (wd >> 16)), tv * apv);
        }
      }
    };
    // two rows per step (all their operands loaded before the reductions)
    // while both are of the cached class; otherwise one row at a time
    for (int r = w; r < ((la.dbg & 1) ? 0 : cnt); r += 2 * LW) {
      const int rb = r + LW;
      const bool hasb = rb < cnt;
      const uint32_t off = __shfl_sync(FULLM, K_outer_off, r);
      const int nit = __shfl_sync(FULLM, K_niter, r);
      const uint32_t offb = __shfl_sync(FULLM, K_outer_off, hasb ? rb : r);
      const int nitb = __shfl_sync(FULLM, K_niter, hasb ? rb : r);
      if (off != cached) decode(off, nit);
      const bool pair = hasb && offb == off;
      const uint32_t ro = (uint32_t)r * rstride, r8 = (uint32_t)r * 8u, r4 = (uint32_t)r * 4u;
      const uint32_t rob = (uint32_t)rb * rstride, rb8 = (uint32_t)rb * 8u, rb4 = (uint32_t)rb * 4u;
      double apv[4], tv[4];
      uint32_t cb[4];
      const bool on[4] = {ok0, ok1, ok0 && pair, ok1 && pair};
      if (on[0]) { apv[0] = lk_lds_f64(s0a + ro); tv[0] = lk_lds_f64(tv0 + r8); cb[0] = lk_lds_u32(tc0 + r4); }
      if (on[1]) { apv[1] = lk_lds_f64(s1a + ro); tv[1] = lk_lds_f64(tv1 + r8); cb[1] = lk_lds_u32(tc1 + r4); }
      if (on[2]) { apv[2] = lk_lds_f64(s0a + rob); tv[2] = lk_lds_f64(tv0 + rb8); cb[2] = lk_lds_u32(tc0 + rb4); }
      if (on[3]) { apv[3] = lk_lds_f64(s1a + rob); tv[3] = lk_lds_f64(tv1 + rb8); cb[3] = lk_lds_u32(tc1 + rb4); }
      if (on[0]) atomicAdd(c_val + (cb[0] + ps0), tv[0] * apv[0]);
      if (on[1]) atomicAdd(c_val + (cb[1] + ps1), tv[1] * apv[1]);
      if (on[2]) atomicAdd(c_val + (cb[2] + ps0), tv[2] * apv[2]);
      if (on[3]) atomicAdd(c_val + (cb[3] + ps1), tv[3] * apv[3]);
      if (nit > 2) tail(off, nit, r);
      if (pair) {
        if (nitb > 2) tail(offb, nitb, rb);
      } else if (hasb) {  // the second row is of another class
        decode(offb, nitb);
        if (ok0) {
          const double a = lk_lds_f64(s0a + rob), t = lk_lds_f64(tv0 + rb8);
          const uint32_t c = lk_lds_u32(tc0 + rb4);
          atomicAdd(c_val + (c + ps0), t * a);
        }
        if (ok1) {
          const double a = lk_lds_f64(s1a + rob), t = lk_lds_f64(tv1 + rb8);
          const uint32_t c = lk_lds_u32(tc1 + rb4);
          atomicAdd(c_val + (c + ps1), t * a);
        }
        if (nitb > 2) tail(offb, nitb, rb);
      }
    }
  }
}

size_t lock_smem_bytes(const LockArgs &la) {
  const size_t wbytes = (size_t)(32 * la.aps + 8 * TGS) * 8 + 8 * TGS * 4 + 8;
  return (size_t)la.acap * 12 + (LT + 4) * 4 + (size_t)LG * wbytes + 16;
}

cudaError_t launch_lock_numeric(const Ops &op, const LockArgs &la, double *c_val, int tile_lo, int tile_hi,
                                int *status, cudaStream_t st) {
  if (tile_hi <= tile_lo) return cudaSuccess;
  const size_t sm = lock_smem_bytes(la);
  static size_t opted[LOCK_WMAX + 1] = {0};
  const int lw = la.lw == 3 ? 3 : 2;
  if (sm > opted[lw]) {
    cudaError_t e = lw == 3 ? cudaFuncSetAttribute(k_lock_numeric<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)
                            : cudaFuncSetAttribute(k_lock_numeric<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    opted[lw] = sm;
  }
  if (lw == 3)
    k_lock_numeric<3><<<tile_hi - tile_lo, LG * 3 * 32, sm, st>>>(op, la, c_val, tile_lo, status);
  else
    k_lock_numeric<2><<<tile_hi - tile_lo, LG * 2 * 32, sm, st>>>(op, la, c_val, tile_lo, status);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Q: P's values (and the C row starts of P's entries) in class-major order.
// ---------------------------------------------------------------------------
// pass 0: per 256-row block, rows per length (0..8) -> blkcnt[L * nb + blk]
__global__ void __launch_bounds__(256) k_lock_plen(int64_t n, const int64_t *pd_rp, uint8_t *plen8, int32_t *blkcnt,
                                                   int nb, unsigned long long *bad) {
  __shared__ int hist[LOCK_NLEN];
  if (threadIdx.x < LOCK_NLEN) hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t k = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (k < n) {
    int64_t L = __ldg(pd_rp + k + 1) - __ldg(pd_rp + k);
    if (L > 8) {
      atomicAdd(bad, 1ull);
      L = 0;
    }
    plen8[k] = (uint8_t)L;
    atomicAdd(&hist[(int)L], 1);
  }
  __syncthreads();
  if (threadIdx.x < LOCK_NLEN) blkcnt[(int64_t)threadIdx.x * nb + blockIdx.x] = hist[threadIdx.x];
}

// exclusive scan of each length's block counts (one CTA per length), totals -> ltab[L]
__global__ void __launch_bounds__(1024) k_lock_scan9(int nb, int32_t *blkcnt, int32_t *ltab) {
  typedef cub::BlockScan<int, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  int32_t *row = blkcnt + (int64_t)blockIdx.x * nb;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += 1024) {
    const int idx = base + threadIdx.x;
    const int v = idx < nb ? row[idx] : 0;
    int ex, tot;
    Scan(tmp).ExclusiveSum(v, ex, tot);
    const int c = carry;
    if (idx < nb) row[idx] = c + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry = c + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) ltab[blockIdx.x] = carry;
}

// ltab: [0, NLEN) rows per length N_L, [NLEN, 2 NLEN) first Q index of length L
__global__ void k_lock_ltab(int32_t *ltab, unsigned long long *bad) {
  long long off = 0;
  for (int L = 0; L < LOCK_NLEN; ++L) {
    ltab[LOCK_NLEN + L] = (int32_t)off;
    off += (long long)L * ltab[L];
  }
  if (off >= (1ll << 31)) atomicAdd(bad, 1ull);
}

// pq[k] = Q index of P row k's first entry (entry t sits t * N_L further)
__global__ void __launch_bounds__(256) k_lock_pq(int64_t n, const uint8_t *plen8, const int32_t *blkbase, int nb,
                                                 const int32_t *ltab, uint32_t *pq) {
  __shared__ int wcnt[8][LOCK_NLEN];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 8 * LOCK_NLEN) (&wcnt[0][0])[threadIdx.x] = 0;
  __syncthreads();
  const int64_t k = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const bool in = k < n;
  const int L = in ? plen8[k] : LOCK_NLEN;  // out-of-range lanes match each other only
  const unsigned m = __match_any_sync(FULLM, L);
  const int rank = __popc(m & ((1u << lane) - 1u));
  if (in && rank == 0) wcnt[warp][L] = __popc(m);
  __syncthreads();
  if (in) {
    int base = 0;
    for (int w = 0; w < warp; ++w) base += wcnt[w][L];
    pq[k] = (uint32_t)(ltab[LOCK_NLEN + L] + blkbase[(int64_t)L * nb + blockIdx.x] + base + rank);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_lock_permute(int64_t n, const int64_t *pd_rp, const uint32_t *pq,
                                                      const int32_t *ltab, const T *__restrict__ src,
                                                      T *__restrict__ dst) {
  const int64_t k = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (k >= n) return;
  const int64_t b = __ldg(pd_rp + k);
  const int L = (int)(__ldg(pd_rp + k + 1) - b);
  if (L <= 0 || L > 8) return;
  const size_t N = (size_t)__ldg(ltab + L);
  size_t x = __ldg(pq + k);
  for (int t = 0; t < L; ++t, x += N) dst[x] = __ldg(src + b + t);
}

cudaError_t launch_lock_qlayout(int64_t n, const int64_t *pd_rp, uint8_t *plen8, int32_t *blkcnt, int32_t *ltab,
                                uint32_t *pq, unsigned long long *bad, cudaStream_t st) {
  const int nb = (int)((n + 255) / 256);
  if (nb == 0) return cudaSuccess;
  k_lock_plen<<<nb, 256, 0, st>>>(n, pd_rp, plen8, blkcnt, nb, bad);
  k_lock_scan9<<<LOCK_NLEN, 1024, 0, st>>>(nb, blkcnt, ltab);
  k_lock_ltab<<<1, 1, 0, st>>>(ltab, bad);
  k_lock_pq<<<nb, 256, 0, st>>>(n, plen8, blkcnt, nb, ltab, pq);
  return cudaGetLastError();
}

cudaError_t launch_lock_permute_f64(int64_t n, const int64_t *pd_rp, const uint32_t *pq, const int32_t *ltab,
                                    const double *src, double *dst, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_lock_permute<double><<<(int)((n + 255) / 256), 256, 0, st>>>(n, pd_rp, pq, ltab, src, dst);
  return cudaGetLastError();
}
cudaError_t launch_lock_permute_i32(int64_t n, const int64_t *pd_rp, const uint32_t *pq, const int32_t *ltab,
                                    const int32_t *src, int32_t *dst, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_lock_permute<int32_t><<<(int)((n + 255) / 256), 256, 0, st>>>(n, pd_rp, pq, ltab, src, dst);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Row classes.  key(i) = hash(A row length, own P row length, P row lengths of
// the row's columns in order, interned slot map, interned position map).  A
// row claims or finds its key's slot in an open-addressed table; the smallest
// row of a slot is the class representative; k_lock_verify then compares
// every row with its representative field by field, so the classes are exact
// (a hash collision marks the plan ineligible instead of merging two classes).
// 8 lanes per row.
// ---------------------------------------------------------------------------
constexpr int CG = 8;

__device__ __forceinline__ unsigned long long lock_row_key(const Ops &op, const uint8_t *plen8, const int64_t *smap_rp,
                                                           const int64_t *pmap_rp, int64_t i, int gl, int &alen) {
  const int64_t a0 = __ldg(op.ad_rp + i), a1 = __ldg(op.ad_rp + i + 1);
  alen = (int)(a1 - a0);
  unsigned long long h = 0;
  for (int j = gl; j < alen; j += CG)
    h += lk_mix(((unsigned long long)j << 8) | plen8[__ldg(op.ad_col + a0 + j)]);
#pragma unroll
  for (int o = CG / 2; o; o >>= 1) h += __shfl_xor_sync(FULLM, h, o, CG);
  h ^= lk_mix((unsigned long long)__ldg(smap_rp + i));
  h ^= lk_mix((unsigned long long)__ldg(pmap_rp + i) * 0x9E3779B97F4A7C15ull + 0x51ull);
  h = lk_mix(h ^ ((unsigned long long)alen << 8) ^ plen8[i]);
  return h ? h : 1ull;
}

__global__ void __launch_bounds__(256) k_lock_claim(Ops op, const uint8_t *plen8, const int64_t *smap_rp,
                                                    const int64_t *pmap_rp, unsigned long long *keys, uint32_t *rep,
                                                    uint32_t mask, uint16_t *slot_of, unsigned long long *nclaim,
                                                    unsigned long long *bad, const uint8_t *pure) {
  const int gl = threadIdx.x & (CG - 1);
  const int64_t i = ((int64_t)blockIdx.x * 256 + threadIdx.x) / CG;
  const bool in = i < op.nloc;
  int alen = 0;
  unsigned long long h = lock_row_key(op, plen8, smap_rp, pmap_rp, in ? i : 0, gl, alen);
  if (!in || gl) return;
  if (pure && !pure[i]) h = 2ull;  // rows with A_o / P_o parts (several ranks) never run here: one empty class
  uint32_t s = (uint32_t)(h >> 17) & mask;
  for (int probe = 0; probe < 128; ++probe, s = (s + 1) & mask) {
    unsigned long long cur = *(volatile unsigned long long *)(keys + s);
    if (cur == 0) {
      cur = atomicCAS(keys + s, 0ull, h);
      if (cur == 0) {
        atomicAdd(nclaim, 1ull);
        cur = h;
      }
    }
    if (cur == h) {
      if ((uint32_t)i < *(volatile uint32_t *)(rep + s)) atomicMin(rep + s, (uint32_t)i);
      slot_of[i] = (uint16_t)s;
      return;
    }
  }
  slot_of[i] = 0;
  atomicAdd(bad, 1ull);
}

__global__ void __launch_bounds__(256) k_lock_verify(Ops op, const uint8_t *plen8, const int64_t *smap_rp,
                                                     const int64_t *pmap_rp, const uint32_t *rep,
                                                     const uint16_t *slot_of, unsigned long long *bad,
                                                     const uint8_t *pure) {
  const int gl = threadIdx.x & (CG - 1);
  const int64_t i = ((int64_t)blockIdx.x * 256 + threadIdx.x) / CG;
  if (i >= op.nloc || (pure && !pure[i])) return;
  const int64_t r = rep[slot_of[i]];
  if (r == i) return;
  bool ok = r < op.nloc;
  if (ok) {
    const int64_t a0 = __ldg(op.ad_rp + i), b0 = __ldg(op.ad_rp + r);
    const int alen = (int)(__ldg(op.ad_rp + i + 1) - a0);
    ok = alen == (int)(__ldg(op.ad_rp + r + 1) - b0) && plen8[i] == plen8[r] &&
         __ldg(smap_rp + i) == __ldg(smap_rp + r) && __ldg(pmap_rp + i) == __ldg(pmap_rp + r);
    if (ok)
      for (int j = gl; j < alen; j += CG)
        ok = ok && plen8[__ldg(op.ad_col + a0 + j)] == plen8[__ldg(op.ad_col + b0 + j)];
  }
  if (!ok) atomicAdd(bad, 1ull);
}

// dense class ids in table-slot order; representatives; class count -> out[0]
__global__ void __launch_bounds__(1024) k_lock_compact(int tbl, const unsigned long long *keys, const uint32_t *rep,
                                                       int32_t *slot2cls, uint32_t *reps, unsigned long long *out) {
  typedef cub::BlockScan<int, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < tbl; base += 1024) {
    const int s = base + threadIdx.x;
    const int v = (s < tbl && keys[s] != 0) ? 1 : 0;
    int ex, tot;
    Scan(tmp).ExclusiveSum(v, ex, tot);
    const int c = carry;
    if (s < tbl) slot2cls[s] = v ? c + ex : -1;
    if (v) reps[c + ex] = rep[s];
    __syncthreads();
    if (threadIdx.x == 0) carry = c + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = (unsigned long long)carry;
}

// pairs per AP slot of the class represented by row r, and the cut of the
// slots into lw contiguous ranges of about equal pair counts
__device__ void lock_class_split(const Ops &op, const uint8_t *plen8, const uint8_t *sm, int64_t a0, int alen, int nap,
                                 int lw, int *cnt, int *first, int *pairs) {
  for (int s = 0; s < 32; ++s) cnt[s] = 0;
  int p = 0;
  for (int j = 0; j < alen; ++j) {
    const int L = plen8[__ldg(op.ad_col + a0 + j)];
    for (int t = 0; t < L; ++t) cnt[sm[p++] & 0x1f]++;
  }
  const int np = p;
  int s = 0, cum = 0;
  for (int w = 0; w < lw; ++w) {
    first[w] = s;
    int mine = 0;
    const int want = (int)(((long long)np * (w + 1)) / lw);
    while (s < nap && (w == lw - 1 || cum + cnt[s] <= want || mine == 0)) {
      mine += cnt[s];
      cum += cnt[s];
      ++s;
    }
    pairs[w] = mine;
  }
  first[lw] = nap;
}

// class headers and program offsets (one CTA): out[1] fold entries, out[2] outer words
__global__ void __launch_bounds__(1024) k_lock_headers(int ncls, Ops op, const uint8_t *plen8, const int64_t *smap_rp,
                                                       const uint8_t *smap, const uint8_t *nap, const uint32_t *reps,
                                                       const int32_t *ltab, LockClass *cls, unsigned long long *out,
                                                       unsigned long long *bad, const uint8_t *pure, int lw) {
  typedef cub::BlockScan<unsigned, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned carry_f, carry_o;
  if (threadIdx.x == 0) carry_f = carry_o = 0;
  __syncthreads();
  for (int base = 0; base < ncls; base += 1024) {
    const int c = base + threadIdx.x;
    LockClass K{};
    unsigned fsz = 0, osz = 0;
    if (c < ncls && !(pure && !pure[reps[c]])) {
      const int64_t r = reps[c];
      const int64_t a0 = __ldg(op.ad_rp + r);
      const int alen = (int)(__ldg(op.ad_rp + r + 1) - a0), napr = nap[r], ntg = plen8[r];
      int np = 0;
      for (int j = 0; j < min(alen, 32); ++j) np += plen8[__ldg(op.ad_col + a0 + j)];
      const int slen = (int)((unsigned long long)__ldg(smap_rp + r) >> 40);
      if (np != slen || alen > 32 || napr > 32) {
        atomicAdd(bad, 1ull);
      } else {
        K.alen = (uint8_t)alen;
        K.nap = (uint8_t)napr;
        K.ntg = (uint8_t)ntg;
        K.tstride = ltab[ntg];
        if (ntg > 0 && napr > 0 && np > 0) {  // a row without targets contributes nothing
          int cnt[32], first[LOCK_WMAX + 1], pairs[LOCK_WMAX];
          const uint8_t *sm = smap + ((unsigned long long)__ldg(smap_rp + r) & SMAP_OFF_MASK);
          lock_class_split(op, plen8, sm, a0, alen, napr, lw, cnt, first, pairs);
          int ch = 0;
          for (int w = 0; w < lw; ++w) {
            K.sub[w] = (uint8_t)ch;
            K.s0[w] = (uint8_t)first[w];
            ch += (pairs[w] + 7) / 8;
          }
          for (int w = lw; w < 8; ++w) K.sub[w] = (uint8_t)ch;
          if (ch > 255) atomicAdd(bad, 1ull);
          fsz = (unsigned)ch * 8u;
          const int items = ntg * napr;
          K.niter = (uint8_t)((items + 31) / 32);
          osz = (unsigned)K.niter * 32u;
        }
      }
    }
    unsigned fex, ftot, oex, otot;
    Scan(tmp).ExclusiveSum(fsz, fex, ftot);
    __syncthreads();
    Scan(tmp).ExclusiveSum(osz, oex, otot);
    const unsigned cf = carry_f, co = carry_o;
    if (c < ncls) {
      K.fold_off = cf + fex;
      K.outer_off = co + oex;
      cls[c] = K;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      carry_f = cf + ftot;
      carry_o = co + otot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[1] = carry_f;
    out[2] = carry_o;
  }
}

// the programs, one thread per class: pairs bucketed by AP slot (stable: fold
// order inside a slot), the last pair of a slot flagged, each sub-program
// padded to 8 entries with invalid ones; outer items in (target, slot) order
__global__ void __launch_bounds__(128) k_lock_programs(int ncls, Ops op, const uint8_t *plen8, const int64_t *smap_rp,
                                                       const uint8_t *smap, const int64_t *pmap_rp,
                                                       const uint8_t *pmap, const uint32_t *reps, const int32_t *ltab,
                                                       const LockClass *cls, uint2 *fold, uint32_t *outer, int lw) {
  const int c = blockIdx.x * 128 + threadIdx.x;
  if (c >= ncls) return;
  const LockClass K = cls[c];
  if (K.sub[7] == 0) return;
  const int64_t r = reps[c];
  const int64_t a0 = __ldg(op.ad_rp + r);
  const uint8_t *sm = smap + ((unsigned long long)__ldg(smap_rp + r) & SMAP_OFF_MASK);
  uint2 *fp = fold + K.fold_off;
  int cnt[32], pos[32], first[LOCK_WMAX + 1], pairs[LOCK_WMAX];
  lock_class_split(op, plen8, sm, a0, K.alen, K.nap, lw, cnt, first, pairs);
  for (int q = 0; q < (int)K.sub[7] * 8; ++q) fp[q] = make_uint2(0u, 0u);
  for (int w = 0; w < lw; ++w) {
    int run = (int)K.sub[w] * 8;
    for (int s = first[w]; s < first[w + 1]; ++s) {
      pos[s] = run;
      run += cnt[s];
      cnt[s] = run;  // end of the slot's bucket
    }
  }
  int p = 0;
  for (int j = 0; j < K.alen; ++j) {
    const int L = plen8[__ldg(op.ad_col + a0 + j)];
    const uint32_t N = (uint32_t)ltab[L];
    for (int t = 0; t < L; ++t) {
      const int s = sm[p++] & 0x1f;
      const int at = pos[s]++;
      const uint32_t last = at + 1 == cnt[s] ? 0x8000u : 0u;
      fp[at] = make_uint2((uint32_t)(j * 8) | ((uint32_t)(j * 4) << 16) | last, (uint32_t)t * N);
    }
  }
  uint32_t *ow = outer + K.outer_off;
  const int items = (int)K.ntg * K.nap;
  const uint8_t *pm = pmap + __ldg(pmap_rp + r);
  for (int it = 0; it < (int)K.niter * 32; ++it) {
    uint32_t wd = 0xffffffffu;
    if (it < items) {
      const int jt = it / K.nap, s = it - jt * K.nap;
      wd = (uint32_t)(s * 8) | ((uint32_t)jt << 8) | ((uint32_t)pm[jt * K.nap + s] << 16);
    }
    ow[it] = wd;
  }
}

// a tile's rows sorted by class (stable): rowinfo[tile start + sorted position]
// = class << 8 | row - tile start; the largest tile (A entries) -> amax
__global__ void __launch_bounds__(LOCK_TILE) k_lock_rowinfo(int64_t n, const int64_t *ad_rp, const uint16_t *slot_of,
                                                            const int32_t *slot2cls, uint32_t *rowinfo,
                                                            uint32_t *rowcls, unsigned long long *amax) {
  __shared__ int key[LT];
  const int q = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * LT;
  const int nr = (int)min((int64_t)LT, n - r0);
  key[q] = q < nr ? ((slot2cls[slot_of[r0 + q]] << 6) | q) : 0x7fffffff;
  __syncthreads();
  const int mine = key[q];
  int rank = 0;
  for (int k = 0; k < LT; ++k) rank += key[k] < mine;
  if (q < nr) rowinfo[r0 + rank] = ((uint32_t)(mine >> 6) << 8) | (uint32_t)q;
  if (q < nr && rowcls) rowcls[r0 + q] = (uint32_t)(mine >> 6);
  if (q == 0) atomicMax(amax, (unsigned long long)(ad_rp[r0 + nr] - ad_rp[r0]));
  // the longest A row -> amax[1]
  const int alen = q < nr ? (int)(ad_rp[r0 + q + 1] - ad_rp[r0 + q]) : 0;
  const int wmax = __reduce_max_sync(FULLM, alen);
  if ((q & 31) == 0) atomicMax(amax + 1, (unsigned long long)wmax);
}

cudaError_t launch_lock_classes(const Ops &op, const uint8_t *plen8, const int64_t *smap_rp, const int64_t *pmap_rp,
                                unsigned long long *keys, uint32_t *rep, int tbl, uint16_t *slot_of,
                                int32_t *slot2cls, uint32_t *reps, unsigned long long *out, unsigned long long *bad,
                                const uint8_t *pure, cudaStream_t st) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(keys, 0, sizeof(unsigned long long) * tbl, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(rep, 0xff, sizeof(uint32_t) * tbl, st)) != cudaSuccess) return e;
  const int64_t threads = op.nloc * CG;
  const int nb = (int)((threads + 255) / 256);
  if (nb == 0) return cudaSuccess;
  k_lock_claim<<<nb, 256, 0, st>>>(op, plen8, smap_rp, pmap_rp, keys, rep, (uint32_t)(tbl - 1), slot_of, out + 3, bad,
                                   pure);
  k_lock_verify<<<nb, 256, 0, st>>>(op, plen8, smap_rp, pmap_rp, rep, slot_of, bad, pure);
  k_lock_compact<<<1, 1024, 0, st>>>(tbl, keys, rep, slot2cls, reps, out);
  return cudaGetLastError();
}

cudaError_t launch_lock_headers(int ncls, const Ops &op, const uint8_t *plen8, const MapArgs &mp,
                                const uint32_t *reps, const int32_t *ltab, LockClass *cls,
                                unsigned long long *out, unsigned long long *bad, const uint8_t *pure, int lw,
                                cudaStream_t st) {
  k_lock_headers<<<1, 1024, 0, st>>>(ncls, op, plen8, mp.smap_rp, mp.smap, mp.nap, reps, ltab, cls, out, bad, pure,
                                     lw);
  return cudaGetLastError();
}

cudaError_t launch_lock_programs(int ncls, const Ops &op, const uint8_t *plen8, const MapArgs &mp,
                                 const uint32_t *reps, const int32_t *ltab, const LockClass *cls, uint2 *fold,
                                 uint32_t *outer, int lw, cudaStream_t st) {
  if (ncls == 0) return cudaSuccess;
  k_lock_programs<<<(ncls + 127) / 128, 128, 0, st>>>(ncls, op, plen8, mp.smap_rp, mp.smap, mp.pmap_rp, mp.pmap, reps,
                                                      ltab, cls, fold, outer, lw);
  return cudaGetLastError();
}

cudaError_t launch_lock_rowinfo(int64_t n, const int64_t *ad_rp, const uint16_t *slot_of, const int32_t *slot2cls,
                                uint32_t *rowinfo, uint32_t *rowcls, unsigned long long *amax, cudaStream_t st) {
  const int nt = (int)((n + LT - 1) / LT);
  if (nt == 0) return cudaSuccess;
  k_lock_rowinfo<<<nt, LT, 0, st>>>(n, ad_rp, slot_of, slot2cls, rowinfo, rowcls, amax);
  return cudaGetLastError();
}

}  // namespace ptapdev
