// ptap_device.cuh -- shared device-side pieces of the B200 PtAP library.
//
// Layout conventions:
//   row offsets int64, column indices int32, values fp64; rows of every CSR
//   keep ascending columns.  The C produced by the library is one CSR of the
//   rank's coarse rows with GLOBAL columns (the diag/offdiag split of the
//   reference's LocalMatrix is a host-side view taken on export).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ptap_b200.h"

namespace ptapdev {

constexpr unsigned FULL = 0xffffffffu;
constexpr int32_t EMPTY32 = -1;
constexpr unsigned long long EMPTY64 = 0xffffffffffffffffull;

// Status bits set by kernels (read back by ptap_plan_check / symbolic).
enum : int { ST_DRIFT = 1, ST_ARENA_FULL = 2, ST_TABLE_FULL = 4, ST_ROW_TOO_WIDE = 8 };

// The operands one rank sees, flattened for kernels (see ptap_operands).
struct Ops {
  int64_t nloc, m, c_lo, c_hi;
  const int64_t *ad_rp; const int32_t *ad_col; const double *ad_val;
  const int64_t *ao_rp; const int32_t *ao_col; const double *ao_val;
  const int64_t *pd_rp; const int32_t *pd_col; const double *pd_val;
  const int64_t *po_rp; const int32_t *po_col; const double *po_val;
  const int32_t *p_colmap;
  const int64_t *pr_rp; const int32_t *pr_col; const double *pr_val;
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ uint32_t hash32(uint32_t g, int log2t) {
  return (g * 0x9E3779B1u) >> (32 - log2t);
}
__device__ __forceinline__ unsigned long long hash64(unsigned long long k) {
  k ^= k >> 33; k *= 0xff51afd7ed558ccdull; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ull; k ^= k >> 33;
  return k;
}

// first index in [lo,hi) with col[idx] >= g
__device__ __forceinline__ int64_t lower_bound32(const int32_t *__restrict__ col, int64_t lo, int64_t hi, int32_t g) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(col + mid) < g) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <int GROUP>
__device__ __forceinline__ int group_sum(int v) {
#pragma unroll
  for (int o = GROUP / 2; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o, GROUP);
  return v;
}

// Insert / accumulate into an open-addressing table (keys int32, values
// fp64) owned by one lane group.  Within one call of a step every lane of a
// group carries a distinct key, so only the slot *claim* needs an atomic;
// the value update is a plain read-modify-write.  The first product for a
// key SETS the slot, later ones ADD (the reference's hm_add semantics,
// src/_kernels.py:116-147), and products are rounded before the add.
template <bool NUM>
__device__ __forceinline__ bool table_put(int32_t *keys, double *vals, int log2t, int32_t g, double v, int &nnew) {
  const uint32_t mask = (1u << log2t) - 1u;
  uint32_t h = hash32((uint32_t)g, log2t);
  for (uint32_t probe = 0; probe <= mask; ++probe) {
    int32_t k = keys[h];
    if (k == g) {
      if (NUM) vals[h] = __dadd_rn(vals[h], v);
      return true;
    }
    if (k == EMPTY32) {
      int32_t old = atomicCAS(keys + h, EMPTY32, g);
      if (old == EMPTY32) {
        if (NUM) vals[h] = v;
        ++nnew;
        return true;
      }
      if (old == g) {  // cannot happen within a step (distinct keys); kept for safety
        if (NUM) vals[h] = __dadd_rn(vals[h], v);
        return true;
      }
    }
    h = (h + 1) & mask;
  }
  return false;
}

__device__ __forceinline__ int table_find(const int32_t *keys, int log2t, int32_t g) {
  const uint32_t mask = (1u << log2t) - 1u;
  uint32_t h = hash32((uint32_t)g, log2t);
  for (uint32_t probe = 0; probe <= mask; ++probe) {
    int32_t k = keys[h];
    if (k == g) return (int)h;
    if (k == EMPTY32) return -1;
    h = (h + 1) & mask;
  }
  return -1;
}

// Pairs (A entry, P entry) of one batch of A entries, flattened in the
// reference's fold order and staged in shared memory per lane group.
// The hash-table row kernels broadcast each A entry by shuffle and never read
// this window, so it is sized 0: its 12 bytes per pair per group only cost
// resident warps (config 5 hash numeric at 2 M points: 8 -> 6.40 ms,
// 0 -> 4.48 ms).
#ifndef PTAP_PAIRS_PER_LANE
#define PTAP_PAIRS_PER_LANE 0
#endif
constexpr int PAIRS_PER_LANE = PTAP_PAIRS_PER_LANE;  // window = PAIRS_PER_LANE * GROUP pairs

struct PStage {
  int32_t *desc;  // [window] P entry index; bit 31 set = P_o entry
  double *a;      // [window] the A value of the pair (numeric only)
};

__device__ __forceinline__ unsigned lanemask_lt() { return (1u << lane_id()) - 1u; }

// Find g in the table or claim an empty slot for it; returns the slot and
// sets `existed`.  Only keys distinct within the calling lanes may race.
__device__ __forceinline__ int table_find_or_claim(int32_t *keys, int log2t, int32_t g, bool &existed) {
  const uint32_t mask = (1u << log2t) - 1u;
  uint32_t h = hash32((uint32_t)g, log2t);
  for (uint32_t probe = 0; probe <= mask; ++probe) {
    int32_t k = keys[h];
    if (k == g) { existed = true; return (int)h; }
    if (k == EMPTY32) {
      int32_t old = atomicCAS(keys + h, EMPTY32, g);
      if (old == EMPTY32) { existed = false; return (int)h; }
      if (old == g) { existed = true; return (int)h; }
    }
    h = (h + 1) & mask;
  }
  existed = false;
  return -1;
}

// Row i of A*P accumulated by one lane group of GROUP lanes, in the
// reference's fold order (src/_kernels.py:205-227): the A_d entries of row i
// in ascending order, then the A_o entries.  One A entry per step: the
// group's lanes scatter its P row (P_d entries, then P_o; columns distinct, so
// a step is conflict-free) and a __syncwarp orders the steps.  The first
// product for a key sets the slot, later ones add (hm_add, :116-147), each
// rounded before the add.  Per chunk of GROUP A entries every lane loads one
// entry and its P row bounds; the step then broadcasts them by shuffle.
// i < 0 marks an idle group (it still joins every warp-collective).  Returns
// (per lane) the number of new keys this lane created.
template <int GROUP, bool NUM>
__device__ __forceinline__ int ap_row_accumulate(const Ops &op, int64_t i, int32_t *keys, double *vals,
                                                 int log2t, const PStage &ps, int *status) {
  const int gl = threadIdx.x & (GROUP - 1);
  int nnew = 0;
  bool ok = true;
  const bool has_po = op.po_rp != nullptr;
#pragma unroll 1
  for (int src = 0; src < 2; ++src) {
    const int64_t *arp = src ? op.ao_rp : op.ad_rp;
    if (arp == nullptr) continue;  // uniform
    const int32_t *acol = src ? op.ao_col : op.ad_col;
    const double *aval = src ? op.ao_val : op.ad_val;
    const int64_t *qrp = src ? op.pr_rp : op.pd_rp;
    const int32_t *qcol = src ? op.pr_col : op.pd_col;
    const double *qval = src ? op.pr_val : op.pd_val;
    const int32_t coff = src ? 0 : (int32_t)op.c_lo;
    const bool po_here = has_po && src == 0;
    int64_t t0 = 0, t1 = 0;
    if (i >= 0) { t0 = __ldg(arp + i); t1 = __ldg(arp + i + 1); }
    int len = (int)(t1 - t0);
    int maxlen = __reduce_max_sync(FULL, len);
#pragma unroll 1
    for (int tb = 0; tb < maxlen; tb += GROUP) {
      int t = tb + gl;
      double a = 0.0;
      int32_t d0 = 0, o0 = 0;
      uint32_t pk = 0;  // nd (16 bits) | plen << 16
      if (t < len) {
        int32_t k = __ldg(acol + t0 + t);
        if (NUM) a = __ldg(aval + t0 + t);
        int64_t x0 = __ldg(qrp + k);
        d0 = (int32_t)x0;
        int nd = (int)(__ldg(qrp + k + 1) - x0), plen = nd;
        if (po_here) {
          int64_t y0 = __ldg(op.po_rp + k);
          o0 = (int32_t)y0;
          plen += (int)(__ldg(op.po_rp + k + 1) - y0);
        }
        pk = (uint32_t)nd | ((uint32_t)plen << 16);
      }
      int steps = min(GROUP, maxlen - tb);
#pragma unroll 1
      for (int j = 0; j < steps; ++j) {
        uint32_t pkj = __shfl_sync(FULL, pk, j, GROUP);
        int32_t d0j = __shfl_sync(FULL, d0, j, GROUP);
        double aj = NUM ? __shfl_sync(FULL, a, j, GROUP) : 0.0;
        int32_t o0j = po_here ? __shfl_sync(FULL, o0, j, GROUP) : 0;
        int ndj = (int)(pkj & 0xffff), plj = (int)(pkj >> 16);
        for (int u = gl; u < plj; u += GROUP) {
          int32_t g;
          double p = 0.0;
          if (u < ndj) {
            g = __ldg(qcol + d0j + u) + coff;
            if (NUM) p = __ldg(qval + d0j + u);
          } else {
            int32_t e = o0j + (u - ndj);
            g = __ldg(op.p_colmap + __ldg(op.po_col + e));
            if (NUM) p = __ldg(op.po_val + e);
          }
          ok &= table_put<NUM>(keys, vals, log2t, g, NUM ? __dmul_rn(aj, p) : 0.0, nnew);
        }
        __syncwarp();
      }
    }
  }
  if (!ok) atomicOr(status, ST_TABLE_FULL);
  return nnew;
}

// Second walk over row i's pairs in the same fold order as ap_row_accumulate,
// writing the slot byte of every pair (symbolic map building).  slot_of maps
// a table position to the key's rank; the first pair of each slot (in fold
// order) is flagged with 0x80 when flag_first.  `seen` has one int per slot.
template <int GROUP>
__device__ __forceinline__ void ap_row_write_smap(const Ops &op, int64_t i, const int32_t *keys, int log2t,
                                                  const int32_t *slot_of, int32_t *seen, const PStage &ps,
                                                  uint8_t *smap_row, bool flag_first) {
  const int gl = threadIdx.x & (GROUP - 1);
  const bool has_po = op.po_rp != nullptr;
  int run = 0;
#pragma unroll 1
  for (int src = 0; src < 2; ++src) {
    const int64_t *arp = src ? op.ao_rp : op.ad_rp;
    if (arp == nullptr) continue;
    const int32_t *acol = src ? op.ao_col : op.ad_col;
    const int64_t *qrp = src ? op.pr_rp : op.pd_rp;
    const int32_t *qcol = src ? op.pr_col : op.pd_col;
    const int32_t coff = src ? 0 : (int32_t)op.c_lo;
    const bool po_here = has_po && src == 0;
    int64_t t0 = 0, t1 = 0;
    if (i >= 0) { t0 = arp[i]; t1 = arp[i + 1]; }
    int len = (int)(t1 - t0);
    int maxlen = __reduce_max_sync(FULL, len);
#pragma unroll 1
    for (int tb = 0; tb < maxlen; tb += GROUP) {
      int t = tb + gl;
      int32_t d0 = 0, o0 = 0;
      uint32_t pk = 0;
      if (t < len) {
        int32_t k = acol[t0 + t];
        int64_t x0 = qrp[k];
        d0 = (int32_t)x0;
        int nd = (int)(qrp[k + 1] - x0), plen = nd;
        if (po_here) { o0 = (int32_t)op.po_rp[k]; plen += (int)(op.po_rp[k + 1] - op.po_rp[k]); }
        pk = (uint32_t)nd | ((uint32_t)plen << 16);
      }
      int steps = min(GROUP, maxlen - tb);
      for (int j = 0; j < steps; ++j) {
        uint32_t pkj = __shfl_sync(FULL, pk, j, GROUP);
        int32_t d0j = __shfl_sync(FULL, d0, j, GROUP);
        int32_t o0j = po_here ? __shfl_sync(FULL, o0, j, GROUP) : 0;
        int ndj = (int)(pkj & 0xffff), plj = (int)(pkj >> 16);
        for (int u = gl; u < plj; u += GROUP) {
          int32_t g = u < ndj ? qcol[d0j + u] + coff : op.p_colmap[op.po_col[o0j + (u - ndj)]];
          int h = table_find(keys, log2t, g);
          int sl = h >= 0 ? slot_of[h] : 0;
          bool first = flag_first && seen[sl] == 0;  // slots of one P row are distinct
          smap_row[run + u] = (uint8_t)(sl | (first ? 0x80 : 0));
          seen[sl] = 1;
        }
        __syncwarp();
        run += plj;
      }
    }
  }
}

// Compact a group's table into (key, value) lists; returns the entry count
// (uniform within the group).  Order is slot order (irrelevant downstream).
template <int GROUP, bool NUM>
__device__ __forceinline__ int table_compact(const int32_t *keys, const double *vals, int tsize,
                                             int32_t *lk, double *lv) {
  const int lane = lane_id();
  const int gl = lane & (GROUP - 1);
  const unsigned gmask = (GROUP == 32) ? FULL : (((1u << GROUP) - 1u) << (lane & ~(GROUP - 1)));
  int n = 0;
  for (int s0 = 0; s0 < tsize; s0 += GROUP) {
    int s = s0 + gl;
    int32_t k = keys[s];
    bool occ = k != EMPTY32;
    unsigned b = __ballot_sync(FULL, occ) & gmask;
    int before = __popc(b & ((1u << lane) - 1u));
    if (occ) {
      lk[n + before] = k;
      if (NUM) lv[n + before] = vals[s];
    }
    n += __popc(b);
  }
  __syncwarp();
  return n;
}

template <int GROUP>
__device__ __forceinline__ void table_clear(int32_t *keys, int tsize) {
  const int gl = threadIdx.x & (GROUP - 1);
  for (int s = gl; s < tsize; s += GROUP) keys[s] = EMPTY32;
  __syncwarp();
}

}  // namespace ptapdev
