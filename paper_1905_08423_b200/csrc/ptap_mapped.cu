// ptap_mapped.cu -- plan-mapped numeric pass of the all-at-once / merged
// triple product.
//
// The symbolic phase (k_outer_symbolic + k_build_pmap) records, for every fine row i it will
// process, two byte maps that make the numeric pass free of hashing and of
// searches in C -- the "caching intermediate data" mode of the paper
// (Table 6) applied to the outer-product algorithm:
//
//   smap[i]: for each (A entry, P entry) pair of row i, in the reference's
//            fold order (A_d entries ascending, for each its P_d then P_o row;
//            then A_o entries with the gathered rows, src/_kernels.py:205-227),
//            the slot of the pair's column in AP(i,:) (slots = the row's
//            columns in ascending order);
//   pmap[i]: for each entry J of P(i,:) (P_d entries, then P_o entries) and
//            each slot s, the position of AP(i,:)'s s-th column inside the
//            target row (the local C row J, or the staging row of J).
//
// The numeric kernel (k_outer_numeric_mapped) then folds AP(i,:) into a dense
// per-row accumulator in the reference's order (one A entry per step, lanes
// over its P row: conflict-free), and scatters P(i,J)*AP(i,s) to
// C[row_start(J) + pmap] with fp64 atomics -- the outer product of
// src/_kernels.py:446-515 without the per-entry binary searches (_c_slot,
// :421-443).  Both maps are one byte per entry (rows with more than 255 AP
// columns or C rows longer than 256 use the hash path instead).
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdlib>

#include "ptap_device.cuh"
#include "ptap_kernels.cuh"

namespace ptapdev {

// lengths of the per-row maps (selected rows: P(i,:) nonempty)
__global__ void k_map_lengths(int64_t n, const int64_t *pd_rp, const int64_t *po_rp, const int64_t *apub,
                              const int64_t *ap_nnz, int64_t *slen, int64_t *plen) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t np_ = pd_rp[i + 1] - pd_rp[i];
  if (po_rp) np_ += po_rp[i + 1] - po_rp[i];
  bool sel = np_ > 0;
  slen[i] = sel ? apub[i] : 0;
  plen[i] = sel ? np_ * ap_nnz[i] : 0;
}

// staging row of every P_o entry (global coarse column -> staging row index)
__global__ void k_po_srow(int64_t nnz, const int32_t *po_col, const int32_t *colmap, int64_t s_nrows,
                          const int32_t *s_rows, int32_t *po_srow, int *status) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  int32_t Jg = colmap[po_col[e]];
  int64_t r = lower_bound32(s_rows, 0, s_nrows, Jg);
  if (r >= s_nrows || s_rows[r] != Jg) { po_srow[e] = -1; atomicOr(status, ST_DRIFT); }
  else po_srow[e] = (int32_t)r;
}

__global__ void k_max_i64(int64_t n, const int64_t *v, unsigned long long *mx) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long x = i < n ? (unsigned long long)v[i] : 0;
  for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(FULL, x, o));
  if (lane_id() == 0 && x) atomicMax(mx, x);
}

__global__ void k_max_rowlen(int64_t n, const int64_t *rp, unsigned long long *mx) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long x = i < n ? (unsigned long long)(rp[i + 1] - rp[i]) : 0;
  for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(FULL, x, o));
  if (lane_id() == 0 && x) atomicMax(mx, x);
}

struct __align__(16) StepEntry {
  double a;        // A value of the entry
  int32_t d0;      // start of its P_d (or remote) row
  uint32_t pk;     // pair offset (16 bits) | nd (8 bits) << 16 | plen (8 bits) << 24
};

// resident CTAs per SM requested from ptxas: the kernel is bound by load
// latency, so the 4-lane instantiation trades a few spilled registers for
// 48 resident warps (measured: 6 -> 8.55 ms, 5 -> 8.66 ms, 7 -> 9.57 ms)
#ifndef PTAP_MINB
#define PTAP_MINB 6
#endif
#ifndef PTAP_PF
#define PTAP_PF 1
#endif
// resident CTAs requested for the 16-lane wide-row kernel (cfg4: 1 -> 16.8,
// 4 -> 14.0, 5 -> 13.1, 6 -> 12.7, 7 -> 12.7 ms)
#ifndef PTAP_MINB16
#define PTAP_MINB16 6
#endif
#ifndef PTAP_MINB_Q4A
#define PTAP_MINB_Q4A 4
#endif
#ifndef PTAP_QA_PF
#define PTAP_QA_PF 1
#endif
#ifndef PTAP_QA_PRED
#define PTAP_QA_PRED 1
#endif
#ifndef PTAP_QA_PRED_OUTER
#define PTAP_QA_PRED_OUTER 0
#endif
#ifndef PTAP_QA_OUTER1
#define PTAP_QA_OUTER1 1
#endif
#ifndef PTAP_QA_PERM
#define PTAP_QA_PERM 1
#endif
// per-group shared region: accumulator (NAPCAP + 1 slots), then G step
// entries and G P_o row starts (group stride 352 B for <4,32>: successive
// groups start 12 bank pairs apart -- the best of the strides measured)
__host__ __device__ constexpr size_t acc_region_bytes(int napcap) {
  return (((size_t)(napcap + 1) * 8 + 15) & ~(size_t)15);
}
__host__ __device__ constexpr size_t group_bytes(int g, int napcap) {
  return (acc_region_bytes(napcap) + (size_t)g * 16 + (size_t)g * 4 + 15) & ~(size_t)15;
}

// Outer-product phase shared by the mapped kernels: the target rows of
// P(i,:) are fetched G at a time (lane gl of the group loads target jb+gl:
// column, value and row start) so the dependent loads of all targets are in
// flight together; the group then walks them in order, lane gl scattering
// slots gl, gl+G, ... of AP(i,:) with fp64 atomics.
template <int G, int NREG>
__device__ __forceinline__ void outer_scatter(const Ops &op, const MapArgs &mp, const OuterTargets &tg, int64_t i,
                                              int64_t pd0, int64_t pd1, int64_t po0, int64_t po1, bool wl, bool ws,
                                              int nap, const double (&accr)[NREG], int gl) {
  const int ndP = (int)(pd1 - pd0);
  const int nP = ndP + (int)(po1 - po0);
  const int maxj = __reduce_max_sync(FULL, i >= 0 ? nP : 0);
  const int64_t pbase = i >= 0 ? __ldg(mp.pmap_rp + i) : 0;
  for (int jb = 0; jb < maxj; jb += G) {
    const int jm = jb + gl;
    double pij = 0.0;
    int64_t base = -1;  // -1: nothing to scatter for this target
    if (i >= 0 && jm < nP) {
      if (jm < ndP) {
        if (wl) {
          int32_t J = __ldg(op.pd_col + pd0 + jm);
          pij = __ldg(op.pd_val + pd0 + jm);
          base = __ldg(tg.c_rp + J);
        }
      } else if (ws) {
        int64_t e = po0 + (jm - ndP);
        pij = __ldg(op.po_val + e);
        base = __ldg(tg.s_rp + __ldg(mp.po_srow + e));
      }
    }
    const int cnt = min(G, maxj - jb);
    for (int q = 0; q < cnt; ++q) {
      const int64_t b = __shfl_sync(FULL, base, q, G);
      const double pv = __shfl_sync(FULL, pij, q, G);
      if (b >= 0) {
        double *cval = (jb + q < ndP) ? tg.c_val : tg.s_val;
        const uint8_t *pm = mp.pmap + pbase + (int64_t)(jb + q) * nap;
#pragma unroll
        for (int k = 0; k < NREG; ++k) {
          int s = gl + G * k;
          if (s < nap) atomicAdd(cval + b + __ldg(pm + s), __dmul_rn(pv, accr[k]));
        }
      }
    }
  }
}

template <int G, int NAPCAP>
__global__ void __launch_bounds__(256, G <= 8 ? PTAP_MINB : (G == 16 ? PTAP_MINB16 : 1)) k_outer_numeric_mapped(Ops op, const int32_t *rows, unsigned long long nrows,
                                                              MapArgs mp, OuterTargets tg, int do_send, int do_local,
                                                              int *status) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NREG = NAPCAP / G;  // accumulator slots owned per lane in the outer phase
  const int lane = lane_id(), gl = lane & (G - 1);
  const int gpw = 32 / G;
  const int gpc = (blockDim.x >> 5) * gpw;
  const int gid = (threadIdx.x >> 5) * gpw + lane / G;
  // per group: acc[NAPCAP + 1] (f64, +1 pad spreads groups over banks), ent[G], o0[G]
  constexpr size_t gbytes = group_bytes(G, NAPCAP);
  unsigned char *gbase = smem + (size_t)gid * gbytes;
  double *acc = (double *)gbase;
  StepEntry *ent = (StepEntry *)(gbase + acc_region_bytes(NAPCAP));
  int32_t *ent_o0 = (int32_t *)(ent + G);
  const bool has_po = op.po_rp != nullptr;
  for (unsigned long long r0 = (unsigned long long)blockIdx.x * gpc + (threadIdx.x >> 5) * gpw; r0 < nrows;
       r0 += (unsigned long long)gridDim.x * gpc) {
    unsigned long long ridx = r0 + lane / G;
    int64_t i = ridx < nrows ? (rows ? (int64_t)rows[ridx] : (int64_t)ridx) : -1;
    int64_t pd0 = 0, pd1 = 0, po0 = 0, po1 = 0;
    if (i >= 0) {
      pd0 = __ldg(op.pd_rp + i); pd1 = __ldg(op.pd_rp + i + 1);
      if (has_po) { po0 = __ldg(op.po_rp + i); po1 = __ldg(op.po_rp + i + 1); }
    }
    bool wl = do_local && pd1 > pd0, ws = do_send && po1 > po0;
    if (!(wl || ws)) i = -1;
    if (__all_sync(FULL, i < 0)) continue;
    int nap = i >= 0 ? (int)__ldg(mp.nap + i) : 0;
    if (nap > 127)  // no first-touch flags in the map: zero-fill
      for (int s = gl; s < nap; s += G) acc[s] = 0.0;
    int64_t sbase = i >= 0 ? (int64_t)(__ldg(mp.smap_rp + i) & SMAP_OFF_MASK) : 0;
    const uint8_t *smap = mp.smap + sbase;
    int run = 0;
    __syncwarp();
#pragma unroll 1
    for (int src = 0; src < 2; ++src) {
      const int64_t *arp = src ? op.ao_rp : op.ad_rp;
      if (arp == nullptr) continue;
      const int32_t *acol = src ? op.ao_col : op.ad_col;
      const double *aval = src ? op.ao_val : op.ad_val;
      const int64_t *qrp = src ? op.pr_rp : op.pd_rp;
      const double *qval = src ? op.pr_val : op.pd_val;
      const bool po_here = has_po && src == 0;
      int64_t t0 = 0, t1 = 0;
      if (i >= 0) { t0 = __ldg(arp + i); t1 = __ldg(arp + i + 1); }
      int len = (int)(t1 - t0);
      int maxlen = __reduce_max_sync(FULL, len);
#pragma unroll 1
      for (int tb = 0; tb < maxlen; tb += G) {
        int t = tb + gl;
        StepEntry en;
        en.a = 0.0; en.d0 = 0;
        int nd = 0, plen = 0;
        int32_t o0 = 0;
        if (t < len) {
          int32_t k = __ldg(acol + t0 + t);
          en.a = __ldg(aval + t0 + t);
          int64_t x0 = __ldg(qrp + k);
          en.d0 = (int32_t)x0;
          nd = plen = (int)(__ldg(qrp + k + 1) - x0);
          if (po_here) {
            int64_t y0 = __ldg(op.po_rp + k);
            o0 = (int32_t)y0;
            plen += (int)(__ldg(op.po_rp + k + 1) - y0);
          }
        }
        int incl = plen;
#pragma unroll
        for (int o = 1; o < G; o <<= 1) {
          int y = __shfl_up_sync(FULL, incl, o, G);
          if (gl >= o) incl += y;
        }
        en.pk = (uint32_t)(run + incl - plen) | ((uint32_t)nd << 16) | ((uint32_t)plen << 24);
        ent[gl] = en;
        if (po_here) ent_o0[gl] = o0;
        int ctot = __shfl_sync(FULL, incl, G - 1, G);
        __syncwarp();
        int steps = min(G, maxlen - tb);
#if PTAP_PF
        if constexpr (G <= 8) {
          // the P values and slots of all G steps are loaded before the
          // folds (independent loads in flight together); the folds stay in
          // step order
          double pv[G];
          int sv[G];
#pragma unroll
          for (int j = 0; j < G; ++j) {
            pv[j] = 0.0; sv[j] = 0;
            if (j < steps) {
              const StepEntry ej = ent[j];
              const int plj = (int)(ej.pk >> 24), ndj = (int)((ej.pk >> 16) & 0xff);
              if (gl < plj) {
                pv[j] = gl < ndj ? __ldg(qval + ej.d0 + gl) : __ldg(op.po_val + ent_o0[j] + (gl - ndj));
                sv[j] = __ldg(smap + (ej.pk & 0xffff) + gl);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < G; ++j) {
            if (j < steps) {
              const StepEntry ej = ent[j];
              const int plj = (int)(ej.pk >> 24);
              if (gl < plj) {
                int s = sv[j], sl = (nap > 127) ? s : (s & 0x7f);
                double prod = __dmul_rn(ej.a, pv[j]);
                acc[sl] = (nap <= 127 && (s & 0x80)) ? prod : __dadd_rn(acc[sl], prod);
                const int ndj = (int)((ej.pk >> 16) & 0xff);
                for (int u = gl + G; u < plj; u += G) {
                  double p = u < ndj ? __ldg(qval + ej.d0 + u) : __ldg(op.po_val + ent_o0[j] + (u - ndj));
                  int s2 = __ldg(smap + (ej.pk & 0xffff) + u), sl2 = (nap > 127) ? s2 : (s2 & 0x7f);
                  double pr2 = __dmul_rn(ej.a, p);
                  acc[sl2] = (nap <= 127 && (s2 & 0x80)) ? pr2 : __dadd_rn(acc[sl2], pr2);
                }
              }
              __syncwarp();
            }
          }
        } else
#endif
#pragma unroll 1
        for (int j = 0; j < steps; ++j) {
          const StepEntry ej = ent[j];  // one 16-byte shared load per step
          int plj = (int)(ej.pk >> 24);
          if (gl < plj) {
            int ndj = (int)((ej.pk >> 16) & 0xff);
            const uint8_t *sm = smap + (ej.pk & 0xffff);
            for (int u = gl; u < plj; u += G) {
              double p = u < ndj ? __ldg(qval + ej.d0 + u) : __ldg(op.po_val + ent_o0[j] + (u - ndj));
              int s = __ldg(sm + u);
              double prod = __dmul_rn(ej.a, p);
              int sl = s & 0x7f;
              if (nap > 127) sl = s;
              acc[sl] = (nap <= 127 && (s & 0x80)) ? prod : __dadd_rn(acc[sl], prod);
            }
          }
          __syncwarp();
        }
        run += ctot;
      }
    }
    // accumulator slots of this lane into registers (slot = gl + G*r)
    double accr[NREG];
#pragma unroll
    for (int r = 0; r < NREG; ++r) accr[r] = (gl + G * r < nap) ? acc[gl + G * r] : 0.0;
    // outer products into C (local rows) and the staging (send rows)
    outer_scatter<G, NREG>(op, mp, tg, i, pd0, pd1, po0, po1, wl, ws, nap, accr, gl);
    __syncwarp();
  }
}

// Bin-0 kernel (AP rows of at most 32 slots): 8 fine rows per warp, 4 lanes
// per row.  Same fold order, rounding and scatter as k_outer_numeric_mapped,
// with the shared-memory traffic cut down (the kernel is bound by the L1
// data pipe): the slot maps of a batch of consecutive rows are copied into
// shared memory with one coalesced sweep instead of 8 row-strided byte
// gathers per step, and the step entries live in [step][row] arrays so each
// per-step broadcast is a single conflict-free 8-byte load.
#ifndef PTAP_Q4_ACC
#define PTAP_Q4_ACC 36
#endif
constexpr int Q4_RPW = 8, Q4_G = 4, Q4_CAP = 32, Q4_ACC = PTAP_Q4_ACC, Q4_SMW = 264;
struct __align__(16) Q4Warp {
  double a[Q4_G][Q4_RPW];     // A value of step j, row r
  int2 dp[Q4_G][Q4_RPW];      // start of its P row, packed offsets/lengths
  int32_t o0[Q4_G][Q4_RPW];   // start of its P_o row
  uint32_t sm[Q4_SMW];        // slot maps of the batch
};
static inline size_t q4_smem(int warps) {
  return (size_t)warps * (Q4_RPW * Q4_ACC * sizeof(double) + sizeof(Q4Warp));
}

// fold of one A block (SRC 0: A_d with P_d/P_o rows, 1: A_o with the
// gathered remote rows) for the 8 rows of a q4 batch; a template so that the
// block's arrays are kernel parameters, not registers
template <int SRC>
__device__ __forceinline__ void q4_fold(const Ops &op, Q4Warp &W, double *acc, const uint8_t *smb, int sbo, int i,
                                        int gl, int r, int &run) {
  constexpr int G = Q4_G;
  const int64_t *arp = SRC ? op.ao_rp : op.ad_rp;
  const int32_t *acol = SRC ? op.ao_col : op.ad_col;
  const double *aval = SRC ? op.ao_val : op.ad_val;
  const int64_t *qrp = SRC ? op.pr_rp : op.pd_rp;
  const double *qval = SRC ? op.pr_val : op.pd_val;
  const bool po_here = SRC == 0 && op.po_rp != nullptr;
  int t0 = 0, len = 0;
  if (i >= 0) { t0 = (int)__ldg(arp + i); len = (int)__ldg(arp + i + 1) - t0; }
  const int maxlen = __reduce_max_sync(FULL, len);
#pragma unroll 1
  for (int tb = 0; tb < maxlen; tb += G) {
    const int t = tb + gl;
    double a = 0.0;
    int d0 = 0, o0 = 0, nd = 0, plen = 0;
    if (t < len) {
      const int k = __ldg(acol + t0 + t);
      a = __ldg(aval + t0 + t);
      d0 = (int)__ldg(qrp + k);
      nd = plen = (int)__ldg(qrp + k + 1) - d0;
      if (po_here) {
        o0 = (int)__ldg(op.po_rp + k);
        plen += (int)__ldg(op.po_rp + k + 1) - o0;
      }
    }
    int incl = plen;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o, G);
      if (gl >= o) incl += y;
    }
    W.a[gl][r] = a;
    W.dp[gl][r] = make_int2(d0, (int)((uint32_t)(run + incl - plen) | ((uint32_t)nd << 16) | ((uint32_t)plen << 24)));
    if (po_here) W.o0[gl][r] = o0;
    run += __shfl_sync(FULL, incl, G - 1, G);
    __syncwarp();
    const int steps = min(G, maxlen - tb);
    // P values and slots of all steps first (independent loads in flight
    // together), then the folds in step order
    double pv[G];
    int sv[G];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      pv[j] = 0.0; sv[j] = 0;
      if (j < steps) {
        const int2 e = W.dp[j][r];
        const int plj = (int)((uint32_t)e.y >> 24), ndj = (e.y >> 16) & 0xff;
        if (gl < plj) {
          pv[j] = gl < ndj ? __ldg(qval + e.x + gl) : __ldg(op.po_val + W.o0[j][r] + (gl - ndj));
          sv[j] = smb[sbo + (e.y & 0xffff) + gl];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
      if (j < steps) {
        const int2 e = W.dp[j][r];
        const int plj = (int)((uint32_t)e.y >> 24);
        if (gl < plj) {
          const double aj = W.a[j][r];
          const int s = sv[j], sl = s & 0x7f;
          const double prod = __dmul_rn(aj, pv[j]);
          acc[sl] = (s & 0x80) ? prod : __dadd_rn(acc[sl], prod);
          if (plj > G) {  // P rows longer than the group
            const int ndj = (e.y >> 16) & 0xff, off = sbo + (e.y & 0xffff);
            for (int u = gl + G; u < plj; u += G) {
              const double p = u < ndj ? __ldg(qval + e.x + u) : __ldg(op.po_val + W.o0[j][r] + (u - ndj));
              const int s2 = smb[off + u], sl2 = s2 & 0x7f;
              const double pr2 = __dmul_rn(aj, p);
              acc[sl2] = (s2 & 0x80) ? pr2 : __dadd_rn(acc[sl2], pr2);
            }
          }
        }
        __syncwarp();
      }
    }
  }
}

__global__ void __launch_bounds__(256, PTAP_MINB) k_outer_numeric_q4(Ops op, const int32_t *rows,
                                                                      unsigned long long nrows, MapArgs mp,
                                                                      OuterTargets tg, int do_send, int do_local,
                                                                      int *status, int row0) {
  // 32-bit offsets throughout (the plan checks every array fits): 64-bit
  // live values would spill
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int G = Q4_G, NREG = Q4_CAP / Q4_G;
  const int lane = lane_id(), gl = lane & (G - 1), r = lane / G;
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double *acc = (double *)smem + (warp * Q4_RPW + r) * Q4_ACC;
  Q4Warp &W = ((Q4Warp *)((double *)smem + nwarps * Q4_RPW * Q4_ACC))[warp];
  const uint8_t *smb = (const uint8_t *)W.sm;
  const bool has_po = op.po_rp != nullptr;
  const int total = (int)nrows;
  for (int r0 = (blockIdx.x * nwarps + warp) * Q4_RPW; r0 < total; r0 += gridDim.x * nwarps * Q4_RPW) {
    const int ridx = r0 + r;
    int i = ridx < total ? (rows ? rows[ridx] : row0 + ridx) : -1;
    bool wl = false, ws = false;
    if (i >= 0) {
      wl = do_local && __ldg(op.pd_rp + i + 1) > __ldg(op.pd_rp + i);
      ws = do_send && has_po && __ldg(op.po_rp + i + 1) > __ldg(op.po_rp + i);
    }
    // slot maps -> shared, row by row (interned maps: <= 128 bytes per row at
    // its pool offset; 33 words per row cover any 4-byte misalignment)
    int sbo;
    __syncwarp();
    {
      const unsigned long long sx = i >= 0 ? __ldg(mp.smap_rp + i) : 0ull;
      const int sb = (int)(sx & SMAP_OFF_MASK), slen = (int)(sx >> 40);
      if (i >= 0) {
        const int wb = sb >> 2, we = (sb + slen + 3) >> 2;
        const uint32_t *src = (const uint32_t *)mp.smap + wb;
        for (int q = gl; q < we - wb; q += G) W.sm[r * 33 + q] = __ldg(src + q);
      }
      sbo = r * 132 + (sb & 3);
    }
    if (!(wl || ws)) i = -1;
    __syncwarp();
    if (__all_sync(FULL, i < 0)) continue;
    int run = 0;
    q4_fold<0>(op, W, acc, smb, sbo, i, gl, r, run);
    if (op.ao_rp != nullptr) q4_fold<1>(op, W, acc, smb, sbo, i, gl, r, run);
    int64_t pd0 = 0, pd1 = 0, po0 = 0, po1 = 0;
    int nap = 0;
    if (i >= 0) {
      pd0 = __ldg(op.pd_rp + i); pd1 = __ldg(op.pd_rp + i + 1);
      if (has_po) { po0 = __ldg(op.po_rp + i); po1 = __ldg(op.po_rp + i + 1); }
      nap = (int)__ldg(mp.nap + i);  // <= 32: first-touch flags valid
    }
    double accr[NREG];
#pragma unroll
    for (int q = 0; q < NREG; ++q) accr[q] = (gl + G * q < nap) ? acc[gl + G * q] : 0.0;
    outer_scatter<G, NREG>(op, mp, tg, i, pd0, pd1, po0, po1, wl, ws, nap, accr, gl);
  }
}

// Grid size of the grid-stride numeric kernels: PTAP_GRID_RESIDENT=1 caps the
// grid at the resident CTA count (one contiguous band of rows in flight);
// the default oversubscribes the grid (148 x 64 CTAs).
template <typename K>
static unsigned long long grid_cap(K kern, int threads, size_t smem) {
  static int mode = -1;
  if (mode < 0) mode = getenv("PTAP_GRID_RESIDENT") ? 1 : 0;
  if (!mode) {
    // CTAs per SM in the grid (PTAP_GRID_MULT): enough that each CTA folds
    // one or two row chunks, so the rows in flight advance as one band in
    // launch order (cfg3 L1: 64 -> 7.16 ms, 256 -> 7.09, 1024 -> 6.92,
    // 2048 -> 6.95; cfg4 12.70 -> 12.35 ms)
    static const int mult = getenv("PTAP_GRID_MULT") ? atoi(getenv("PTAP_GRID_MULT")) : 1024;
    return 148ull * (unsigned long long)(mult > 0 ? mult : 1024);
  }
  int dev = 0, nsm = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  return (unsigned long long)nsm * per_sm;
}

template <typename K>
static cudaError_t opt_in(K kern, size_t bytes) {
  if (bytes > 48 * 1024) return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return cudaSuccess;
}

// no more CTAs than can be resident: the rows in flight form one contiguous
// band, so the gathered P rows and the touched C rows stay in L2
template <typename K>
static unsigned long long resident(K kern, int threads, size_t smem) {
  int dev = 0, nsm = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  return (unsigned long long)nsm * per_sm;
}

static inline int nb(int64_t n, int t) { return (int)((n + t - 1) / t > 0 ? (n + t - 1) / t : 1); }

// 32-bit shared-window accesses and predicated loads/stores for the q4a
// fold: without them ptxas rematerialises the accumulator's shared-window
// base (S2R SR_CgaCtaId) and a global-memory descriptor for every step under
// the 64-register budget, and wraps each conditional access in a divergent
// region (BSSY/BSYNC)
__device__ __forceinline__ uint32_t sh_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int2 lds_v2s32(uint32_t a) {
  int2 v;
  asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f64_if(bool p, uint32_t a) {
  double v = 0.0;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.f64 %0, [%1];\n}" : "+d"(v) : "r"(a), "r"((int)p));
  return v;
}
__device__ __forceinline__ uint32_t lds_u8_if(bool p, uint32_t a) {
  uint32_t v = 0;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.u8 %0, [%1];\n}" : "+r"(v) : "r"(a), "r"((int)p));
  return v;
}
__device__ __forceinline__ void sts_f64_if(bool p, uint32_t a, double v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.shared.f64 [%0], %1;\n}" ::"r"(a), "d"(v), "r"((int)p)
               : "memory");
}
__device__ __forceinline__ uint32_t ldg_u8_if(bool p, const uint8_t *ptr) {
  uint32_t v = 0;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.nc.u8 %0, [%1];\n}" : "+r"(v) : "l"(ptr), "r"((int)p));
  return v;
}
__device__ __forceinline__ void red_add_f64_if(bool p, double *ptr, double v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q red.global.add.f64 [%0], %1;\n}" ::"l"(ptr), "d"(v), "r"((int)p)
               : "memory");
}
__device__ __forceinline__ double ldg_f64_if(bool p, const double *ptr) {
  double v = 0.0;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.nc.f64 %0, [%1];\n}" : "+d"(v) : "l"(ptr), "r"((int)p));
  return v;
}

// q4a outer phase with the C-row-start map: every lane of a row's group reads
// each target's (C row start, P value) directly (one broadcast load each, two
// targets in flight), no shuffles, no column -> row-pointer chain
template <int G, int NREG>
__device__ __forceinline__ void outer_scatter_cb(const Ops &op, const MapArgs &mp, const OuterTargets &tg, int i,
                                                 int pd0, int pd1, int nap, const double (&accr)[NREG], int gl) {
  const int nP = i >= 0 ? pd1 - pd0 : 0;
  const int maxj = __reduce_max_sync(FULL, nP);
  const int64_t pbase = i >= 0 ? __ldg(mp.pmap_rp + i) : 0;
#if PTAP_QA_OUTER1
  // one target per round: fewer live registers than the two-target rounds
  // below (7.18 -> 7.14 ms; predicating the slot rounds instead: 7.23)
  for (int jj = 0; jj < maxj; ++jj) {
    if (jj < nP) {
      const int b0 = __ldg(mp.cbase + pd0 + jj);
      const double v0 = __ldg(op.pd_val + pd0 + jj);
      const uint8_t *pm = mp.pmap + pbase + (int64_t)jj * nap;
      double *cv = tg.c_val + b0;
#pragma unroll
      for (int k = 0; k < NREG; ++k) {
        const int s = gl + G * k;
        if (s < nap) atomicAdd(cv + __ldg(pm + s), __dmul_rn(v0, accr[k]));
      }
    }
  }
  return;
#endif
  for (int jj = 0; jj < maxj; jj += 2) {
    int b0 = -1, b1 = -1;
    double v0 = 0.0, v1 = 0.0;
    if (jj < nP) { b0 = __ldg(mp.cbase + pd0 + jj); v0 = __ldg(op.pd_val + pd0 + jj); }
    if (jj + 1 < nP) { b1 = __ldg(mp.cbase + pd0 + jj + 1); v1 = __ldg(op.pd_val + pd0 + jj + 1); }
#if PTAP_QA_PRED_OUTER
    // predicated, branch-free: per slot one byte load and one reduction
    // (measured slower: 7.35 vs 7.21 ms; off)
    {
      const uint8_t *pm0 = mp.pmap + pbase + (int64_t)jj * nap;
      const uint8_t *pm1 = pm0 + nap;
      double *c0 = tg.c_val + (b0 >= 0 ? b0 : 0), *c1 = tg.c_val + (b1 >= 0 ? b1 : 0);
#pragma unroll
      for (int k = 0; k < NREG; ++k) {
        const int s = gl + G * k;
        const bool p0 = b0 >= 0 && s < nap, p1 = b1 >= 0 && s < nap;
        const uint32_t q0 = ldg_u8_if(p0, pm0 + s), q1 = ldg_u8_if(p1, pm1 + s);
        red_add_f64_if(p0, c0 + q0, __dmul_rn(v0, accr[k]));
        red_add_f64_if(p1, c1 + q1, __dmul_rn(v1, accr[k]));
      }
    }
#else
    if (b0 >= 0) {
      const uint8_t *pm = mp.pmap + pbase + (int64_t)jj * nap;
#pragma unroll
      for (int k = 0; k < NREG; ++k) {
        const int s = gl + G * k;
        if (s < nap) atomicAdd(tg.c_val + b0 + __ldg(pm + s), __dmul_rn(v0, accr[k]));
      }
    }
    if (b1 >= 0) {
      const uint8_t *pm = mp.pmap + pbase + (int64_t)(jj + 1) * nap;
#pragma unroll
      for (int k = 0; k < NREG; ++k) {
        const int s = gl + G * k;
        if (s < nap) atomicAdd(tg.c_val + b1 + __ldg(pm + s), __dmul_rn(v1, accr[k]));
      }
    }
#endif
  }
}

// ---------------------------------------------------------------------------
// q4a: the bin-0 kernel for one-rank structure (identity rows, no A_o/P_o,
// A rows <= 32 entries) with the next batch's A columns and slot maps copied
// into shared memory by cp.async while the current batch scatters its outer
// products: the fold starts its dependent chain (column -> P row bounds -> P
// values) from shared memory, and the copy latency hides behind the atomics.
// A's values stay in global memory (staging them too costs resident warps:
// 8.37 vs 8.02 ms measured).
// ---------------------------------------------------------------------------
constexpr int QA_ACAP = 256;  // A entries of a batch of 8 rows (<= 32 each)
#ifndef PTAP_QA_VALS
#define PTAP_QA_VALS 0
#endif
struct __align__(16) QaStage {
#if PTAP_QA_VALS
  double val[QA_ACAP];
#endif
  int32_t col[QA_ACAP];
};
static inline size_t q4a_smem(int warps) {
  return (size_t)warps * (Q4_RPW * Q4_ACC * sizeof(double) + sizeof(Q4Warp) + sizeof(QaStage));
}

__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// row of a batch handled by lane group g: with PTAP_QA_PERM the first
// half-warp takes the batch's even rows and the second its odd rows, so on a
// lexicographic grid (x parity alternating) each half-warp folds rows of one
// structural class, whose same-step slots sit at fixed bank offsets
__device__ __forceinline__ int qa_row(int g) {
#if PTAP_QA_PERM
  return ((g & 3) << 1) | (g >> 2);
#else
  return g;
#endif
}

// issue the copies of batch [r0, r0 + 8) (rows are consecutive)
__device__ __forceinline__ void qa_stage(const Ops &op, const MapArgs &mp, Q4Warp &W, QaStage &S, int r0, int total,
                                         int lane) {
  const int r1 = min(r0 + Q4_RPW, total);
  const int a0 = (int)__ldg(op.ad_rp + r0), a1 = (int)__ldg(op.ad_rp + r1);
  const int32_t *csrc = mp.poff ? mp.poff : op.ad_col;  // packed P row bounds, or A's columns
  for (int q = lane; q < a1 - a0; q += 32) {
    cp_async4(&S.col[q], csrc + a0 + q);
#if PTAP_QA_VALS
    cp_async8(&S.val[q], op.ad_val + a0 + q);
#endif
  }
  // slot maps row by row: rows of one class share an interned map, so a
  // batch's maps are not one contiguous run
  const int i = r0 + qa_row(lane >> 2);
  if (i < r1) {
    const unsigned long long sx = __ldg(mp.smap_rp + i);
    const int sb = (int)(sx & SMAP_OFF_MASK), slen = (int)(sx >> 40);
    const int wb = sb >> 2, nw = ((sb + slen + 3) >> 2) - wb;
    const uint32_t *src = (const uint32_t *)mp.smap + wb;
    for (int q = lane & 3; q < nw; q += 4) cp_async4(&W.sm[(lane >> 2) * 33 + q], src + q);
  }
  cp_async_commit();
}

__global__ void __launch_bounds__(256, PTAP_MINB_Q4A) k_outer_numeric_q4a(Ops op, unsigned long long nrows, MapArgs mp,
                                                                          OuterTargets tg, int *status, int row0) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int G = Q4_G, NREG = Q4_CAP / Q4_G;
  const int lane = lane_id(), gl = lane & (G - 1), r = lane / G;
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double *acc = (double *)smem + (warp * Q4_RPW + r) * Q4_ACC;
  Q4Warp &W = ((Q4Warp *)((double *)smem + nwarps * Q4_RPW * Q4_ACC))[warp];
  QaStage &S = ((QaStage *)((unsigned char *)smem + nwarps * (Q4_RPW * Q4_ACC * sizeof(double) + sizeof(Q4Warp))))[warp];
  const uint8_t *smb = (const uint8_t *)W.sm;
#if PTAP_QA_PRED
  const uint32_t acc_sa = sh_addr(acc), smb_sa = sh_addr(smb), dp_sa = sh_addr(&W.dp[0][r]), a_sa = sh_addr(&W.a[0][r]);
#endif
  const int total = row0 + (int)nrows;
  const int stride = gridDim.x * nwarps * Q4_RPW;
  int r0 = row0 + (blockIdx.x * nwarps + warp) * Q4_RPW;
  if (r0 < total) qa_stage(op, mp, W, S, r0, total, lane);
  for (; r0 < total; r0 += stride) {
    const int i_all = r0 + qa_row(r);
    int i = i_all < total ? i_all : -1;
    int pd0 = 0, pd1 = 0;
    if (i >= 0) { pd0 = (int)__ldg(op.pd_rp + i); pd1 = (int)__ldg(op.pd_rp + i + 1); }
    const bool wl = pd1 > pd0;
    const int a0 = (int)__ldg(op.ad_rp + r0);
    int t0 = 0, len = 0, sbo = 0;
    if (i >= 0) {
      t0 = (int)__ldg(op.ad_rp + i) - a0;
      len = (int)__ldg(op.ad_rp + i + 1) - a0 - t0;
      sbo = r * 132 + (int)(__ldg(mp.smap_rp + i) & 3);
    }
    if (!wl) i = -1;
    if (i < 0) len = 0;
    cp_async_wait_all();
    __syncwarp();
    // fold: A entries from shared memory, P values and row bounds from global
    int run = 0;
    const int maxlen = __reduce_max_sync(FULL, len);
#if PTAP_QA_PF
    // the next chunk's A value and P row bounds are loaded while this
    // chunk's steps run (the column -> row-bounds chain is the top stall)
    int nd0 = 0, nd1 = 0;
    double na = 0.0;
    auto fetch = [&](int tt) {
      nd0 = nd1 = 0;
      na = 0.0;
      if (tt < len) {
        const int k = S.col[t0 + tt];
        na = __ldg(op.ad_val + a0 + t0 + tt);
        if (mp.poff) {
          nd0 = k & 0x0fffffff;
          nd1 = nd0 + (int)((unsigned)k >> 28);
        } else {
          nd0 = (int)__ldg(op.pd_rp + k);
          nd1 = (int)__ldg(op.pd_rp + k + 1);
        }
      }
    };
    fetch(gl);
#endif
#pragma unroll 1
    for (int tb = 0; tb < maxlen; tb += G) {
      const int t = tb + gl;
#if PTAP_QA_PF
      const double a = na;
      const int d0 = nd0, plen = nd1 - nd0;
      fetch(t + G);
#else
      double a = 0.0;
      int d0 = 0, plen = 0;
      if (t < len) {
        const int k = S.col[t0 + t];
#if PTAP_QA_VALS
        a = S.val[t0 + t];
#else
        a = __ldg(op.ad_val + a0 + t0 + t);
#endif
        if (mp.poff) {
          d0 = k & 0x0fffffff;
          plen = (int)((unsigned)k >> 28);
        } else {
          d0 = (int)__ldg(op.pd_rp + k);
          plen = (int)__ldg(op.pd_rp + k + 1) - d0;
        }
      }
#endif
      int incl = plen;
#pragma unroll
      for (int o = 1; o < G; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o, G);
        if (gl >= o) incl += y;
      }
      W.a[gl][r] = a;
      W.dp[gl][r] = make_int2(d0, (int)((uint32_t)(run + incl - plen) | ((uint32_t)plen << 24)));
      run += __shfl_sync(FULL, incl, G - 1, G);
      __syncwarp();
      const int steps = min(G, maxlen - tb);
#if PTAP_QA_PRED
      double pv[G];
      uint32_t sv[G];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int2 e = lds_v2s32(dp_sa + j * (Q4_RPW * 8));
        const bool act = j < steps && gl < (int)((uint32_t)e.y >> 24);
        pv[j] = ldg_f64_if(act, op.pd_val + (uint32_t)(e.x + gl));
        sv[j] = lds_u8_if(act, smb_sa + (uint32_t)(sbo + (e.y & 0xffff) + gl));
      }
#pragma unroll
      for (int j = 0; j < G; ++j) {
        if (j < steps) {
          const int2 e = lds_v2s32(dp_sa + j * (Q4_RPW * 8));
          const int plj = (int)((uint32_t)e.y >> 24);
          const bool act = gl < plj;
          const double aj = lds_f64(a_sa + j * (Q4_RPW * 8));
          const uint32_t s = sv[j], ad = acc_sa + (s & 0x7f) * 8;
          const double prod = __dmul_rn(aj, pv[j]);
          const double old = lds_f64_if(act && !(s & 0x80), ad);
          sts_f64_if(act, ad, (s & 0x80) ? prod : __dadd_rn(old, prod));
          if (plj > G) {  // P rows longer than the group (rare)
            const uint32_t off = smb_sa + (uint32_t)(sbo + (e.y & 0xffff));
            for (int u = gl + G; u < plj; u += G) {
              const double pu = __ldg(op.pd_val + (uint32_t)(e.x + u));
              const uint32_t s2 = lds_u8_if(true, off + u), ad2 = acc_sa + (s2 & 0x7f) * 8;
              const double pr2 = __dmul_rn(aj, pu);
              const double old2 = lds_f64_if(!(s2 & 0x80), ad2);
              sts_f64_if(true, ad2, (s2 & 0x80) ? pr2 : __dadd_rn(old2, pr2));
            }
          }
          __syncwarp();
        }
      }
#else
      double pv[G];
      int sv[G];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        pv[j] = 0.0; sv[j] = 0;
        if (j < steps) {
          const int2 e = W.dp[j][r];
          const int plj = (int)((uint32_t)e.y >> 24);
          if (gl < plj) {
            pv[j] = __ldg(op.pd_val + e.x + gl);
            sv[j] = smb[sbo + (e.y & 0xffff) + gl];
          }
        }
      }
#pragma unroll
      for (int j = 0; j < G; ++j) {
        if (j < steps) {
          const int2 e = W.dp[j][r];
          const int plj = (int)((uint32_t)e.y >> 24);
          if (gl < plj) {
            const double aj = W.a[j][r];
            const int s = sv[j], sl = s & 0x7f;
            const double prod = __dmul_rn(aj, pv[j]);
            acc[sl] = (s & 0x80) ? prod : __dadd_rn(acc[sl], prod);
            if (plj > G) {
              const int off = sbo + (e.y & 0xffff);
              for (int u = gl + G; u < plj; u += G) {
                const double pu = __ldg(op.pd_val + e.x + u);
                const int s2 = smb[off + u], sl2 = s2 & 0x7f;
                const double pr2 = __dmul_rn(aj, pu);
                acc[sl2] = (s2 & 0x80) ? pr2 : __dadd_rn(acc[sl2], pr2);
              }
            }
          }
          __syncwarp();
        }
      }
#endif
    }
    __syncwarp();
    // the next batch's A entries and slot maps stream in behind the scatter
    if (r0 + stride < total) qa_stage(op, mp, W, S, r0 + stride, total, lane);
    const int nap = i >= 0 ? (int)__ldg(mp.nap + i) : 0;
    double accr[NREG];
#pragma unroll
#if PTAP_QA_PRED_OUTER
    for (int q = 0; q < NREG; ++q) accr[q] = lds_f64_if(gl + G * q < nap, acc_sa + (gl + G * q) * 8);
#else
    for (int q = 0; q < NREG; ++q) accr[q] = (gl + G * q < nap) ? acc[gl + G * q] : 0.0;
#endif
#ifdef PTAP_QA_ABLATE_OUTER  // timing experiments only: C is not written
    if (accr[0] == 1.2345e-300) tg.c_val[0] = accr[1];
#else
    if (mp.cbase)
      outer_scatter_cb<G, NREG>(op, mp, tg, i, pd0, pd1, nap, accr, gl);
    else
      outer_scatter<G, NREG>(op, mp, tg, i, pd0, pd1, 0, 0, wl, false, nap, accr, gl);
#endif
  }
  cp_async_wait_all();
}

cudaError_t launch_outer_numeric_q4a(const Ops &op, unsigned long long nrows, const MapArgs &mp,
                                     const OuterTargets &tg, int *status, cudaStream_t st, int row0) {
  if (nrows == 0) return cudaSuccess;
  const int warps = 8;
  const size_t sm = q4a_smem(warps);
  cudaError_t e;
  if ((e = opt_in(k_outer_numeric_q4a, sm)) != cudaSuccess) return e;
  const unsigned long long rpc = (unsigned long long)warps * Q4_RPW;
  unsigned long long grid = (nrows + rpc - 1) / rpc;
  grid = std::min(grid, grid_cap(k_outer_numeric_q4a, warps * 32, sm));
  k_outer_numeric_q4a<<<(int)grid, warps * 32, sm, st>>>(op, nrows, mp, tg, status, row0);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Map interning.  The per-row slot and position maps depend only on the
// row's structure relative to its own AP row and target rows, so rows of the
// same structural class (every interior row of a stencil's parity class, every
// node of an aggregate position in smoothed aggregation) carry byte-identical
// maps.  k_intern stores each distinct byte string once: a warp hashes its
// row's string, probes an open-addressed table of (hash -> pool offset); the
// first warp to claim a hash copies the string into the pool and publishes its
// offset, later warps with the same hash wait for the publication and compare
// the bytes (a collision keeps probing).  Rows whose probe sequence runs out
// get a private copy, so the result is exact whatever the table holds.
// out[i] = pool offset (| length << 40 when pack_len).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

constexpr int INTERN_PROBES = 64, INTERN_G = 8;

// 32-bit word w of a string of len bytes starting at byte address s (any
// alignment), zero past the end: pool entries are word aligned, zero padded
__device__ __forceinline__ uint32_t intern_word(const uint8_t *s, int len, int w) {
  const uintptr_t a = (uintptr_t)s + 4 * w;
  const uint32_t *p = (const uint32_t *)(a & ~(uintptr_t)3);
  const int sh = (int)(a & 3) * 8;
  uint32_t x = p[0];
  if (sh) x = __funnelshift_r(x, p[1], sh);
  const int rem = len - 4 * w;
  return rem >= 4 ? x : (x & ((1u << (8 * rem)) - 1u));
}

// Three passes, no waiting between warps: (1) claim: each row hashes its
// string and finds or claims the table slot of that hash (the claiming row
// becomes the class representative); (2) resolve: each row compares its bytes
// with its representative's (both in the source maps) and keeps the
// representative as owner when equal, itself otherwise (a hash collision or
// no slot: a private copy); (3) after a scan of the owners' word counts,
// owners copy their strings into the pool and every row records its owner's
// pool offset.  INTERN_G lanes per row, 4 rows per warp.
__device__ __forceinline__ unsigned long long intern_hash(const uint8_t *s, int len, int gl, unsigned gmask) {
  constexpr int G = INTERN_G;
  const int nwords = (len + 3) >> 2;
  unsigned long long h = 0;
  for (int w = gl; w < nwords; w += G) h += mix64(((unsigned long long)w << 32) | intern_word(s, len, w));
#pragma unroll
  for (int o = G / 2; o; o >>= 1) h += __shfl_xor_sync(gmask, h, o, G);
  h = mix64(h ^ ((unsigned long long)len << 40));
  return h ? h : 1;
}

__global__ void __launch_bounds__(256) k_intern_claim(int64_t n, const uint8_t *src, const int64_t *src_rp,
                                                      unsigned long long *keys, int64_t *vals,
                                                      unsigned long long mask, int64_t *slot_of,
                                                      unsigned long long *claims) {
  constexpr int G = INTERN_G;
  const int lane = lane_id(), gl = lane & (G - 1);
  const unsigned gmask = 0xffu << (lane & ~(G - 1));
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / G;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; i < n; i += ng) {
    const int64_t s0 = src_rp[i];
    const int len = (int)(src_rp[i + 1] - s0);
    if (len == 0) {
      if (gl == 0) slot_of[i] = -1;
      continue;
    }
    const unsigned long long h = intern_hash(src + s0, len, gl, gmask);
    if (gl == 0) {
      unsigned long long slot = h & mask;
      int64_t found = -1;
      for (int probe = 0; probe < INTERN_PROBES; ++probe) {
        unsigned long long k = keys[slot];  // a stale 0 only costs a CAS
        if (k == 0) {
          // claims stop at half the table (rows that do not repeat -- an
          // unstructured input -- must not fill it): later new strings
          // stay private
          if (*(volatile unsigned long long *)claims > (mask >> 1)) break;
          k = atomicCAS(keys + slot, 0ull, h);
          if (k == 0) {
            vals[slot] = i;  // the representative; read after this kernel
            atomicAdd(claims, 1ull);
          }
        }
        if (k == 0 || k == h) { found = (int64_t)slot; break; }
        slot = (slot + 1) & mask;
      }
      slot_of[i] = found;
    }
  }
}

__global__ void __launch_bounds__(256) k_intern_resolve(int64_t n, const uint8_t *src, const int64_t *src_rp,
                                                        const int64_t *vals, const int64_t *slot_of,
                                                        int64_t *owner, int64_t *words) {
  constexpr int G = INTERN_G;
  const int lane = lane_id(), gl = lane & (G - 1);
  const unsigned gmask = 0xffu << (lane & ~(G - 1));
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / G;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; i < n; i += ng) {
    const int64_t s0 = __ldg(src_rp + i);
    const int len = (int)(__ldg(src_rp + i + 1) - s0);
    const int64_t sl = __ldg(slot_of + i);
    int64_t own = i;
    if (len > 0 && sl >= 0) {
      const int64_t rep = __ldg(vals + sl);
      if (rep != i) {
        const int64_t r0 = __ldg(src_rp + rep);
        bool eq = __ldg(src_rp + rep + 1) - r0 == len;
        if (eq) {
          const int nwords = (len + 3) >> 2;
          for (int w = gl; w < nwords; w += G) eq &= intern_word(src + s0, len, w) == intern_word(src + r0, len, w);
        }
        if (__all_sync(gmask, eq)) own = rep;
      }
    }
    if (gl == 0) {
      owner[i] = own;
      words[i] = own == i ? (int64_t)((len + 3) >> 2) : 0;
    }
  }
}

__global__ void __launch_bounds__(256) k_intern_copy(int64_t n, const uint8_t *src, const int64_t *src_rp,
                                                     const int64_t *owner, const int64_t *wpos, uint8_t *pool,
                                                     int64_t *out, int pack_len) {
  constexpr int G = INTERN_G;
  const int lane = lane_id(), gl = lane & (G - 1);
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / G;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; i < n; i += ng) {
    const int64_t s0 = src_rp[i];
    const int len = (int)(src_rp[i + 1] - s0);
    const int64_t own = owner[i];
    const int64_t off = wpos[own] * 4;
    if (own == i) {
      uint32_t *pw = (uint32_t *)(pool + off);
      for (int w = gl; w < ((len + 3) >> 2); w += G) pw[w] = intern_word(src + s0, len, w);
    }
    if (gl == 0) out[i] = pack_len ? (off | ((int64_t)len << 40)) : off;
  }
}

// ---------------------------------------------------------------------------
// Do the rows repeat?  A fine row's slot map is fixed by its A row length, the
// P row lengths of its columns and the relative order of the pairs' coarse
// columns, so rows whose (length, P row lengths, column - row minimum)
// sequences agree share their slot map.  k_struct_sample hashes that
// signature for a pseudo-random sample of rows (a warp per row) and counts the
// distinct ones in a table; the plan keeps interned maps only when the sample
// repeats (structured operators), and unstructured operators take the hash
// numeric path, which stores nothing per row.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void sig_row_block(const Ops &op, int src, int64_t i, int &lo, unsigned long long &h,
                                              bool hash_pass) {
  const int lane = lane_id();
  const int64_t *arp = src ? op.ao_rp : op.ad_rp;
  if (arp == nullptr) return;
  const int32_t *acol = src ? op.ao_col : op.ad_col;
  const int64_t *qrp = src ? op.pr_rp : op.pd_rp;
  const int32_t *qcol = src ? op.pr_col : op.pd_col;
  const int32_t coff = src ? 0 : (int32_t)op.c_lo;
  const bool po_here = src == 0 && op.po_rp != nullptr;
  const int64_t t0 = arp[i], t1 = arp[i + 1];
  for (int64_t t = t0 + lane; t < t1; t += 32) {
    const int32_t k = acol[t];
    const int64_t d0 = qrp[k], d1 = qrp[k + 1];
    const int64_t o0 = po_here ? op.po_rp[k] : 0, o1 = po_here ? op.po_rp[k + 1] : 0;
    unsigned long long he = 0;
    for (int64_t q = d0; q < d1 + (o1 - o0); ++q) {
      const int32_t g = q < d1 ? qcol[q] + coff : op.p_colmap[op.po_col[o0 + (q - d1)]];
      if (!hash_pass) lo = min(lo, g);
      else he += mix64(((unsigned long long)(q - d0) << 32) | (uint32_t)(g - lo));
    }
    if (hash_pass)
      h += mix64(he ^ ((unsigned long long)(src * 4096 + (t - t0)) << 40) ^ ((unsigned long long)(d1 - d0 + o1 - o0) << 56));
  }
}

__global__ void __launch_bounds__(256) k_struct_sample(Ops op, int64_t nsample, unsigned long long *keys,
                                                       unsigned long long mask, unsigned long long *distinct) {
  const int lane = lane_id();
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < nsample; j += nw) {
    const int64_t i = nsample >= op.nloc ? j : (int64_t)(mix64((unsigned long long)j) % (unsigned long long)op.nloc);
    int lo = INT_MAX;
    unsigned long long h = 0;
    for (int src = 0; src < 2; ++src) sig_row_block(op, src, i, lo, h, false);
    lo = __reduce_min_sync(FULL, lo);
    for (int src = 0; src < 2; ++src) sig_row_block(op, src, i, lo, h, true);
#pragma unroll
    for (int o = 16; o; o >>= 1) h += __shfl_xor_sync(FULL, h, o);
    const int64_t alen = (op.ad_rp[i + 1] - op.ad_rp[i]) + (op.ao_rp ? op.ao_rp[i + 1] - op.ao_rp[i] : 0);
    h = mix64(h ^ (unsigned long long)alen);
    if (h == 0) h = 1;
    if (lane == 0) {
      unsigned long long slot = h & mask;
      for (int probe = 0; probe <= (int)mask; ++probe) {
        const unsigned long long k = atomicCAS(keys + slot, 0ull, h);
        if (k == 0) { atomicAdd(distinct, 1ull); break; }
        if (k == h) break;
        slot = (slot + 1) & mask;
      }
    }
  }
}

cudaError_t launch_struct_sample(const Ops &op, int64_t nsample, unsigned long long *keys, unsigned long long mask,
                                 unsigned long long *distinct, cudaStream_t st) {
  if (nsample <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((nsample + 7) / 8, 148 * 16);
  k_struct_sample<<<blocks, 256, 0, st>>>(op, nsample, keys, mask, distinct);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Locality order of a plan without maps.  The hash numeric pass visits its
// rows in bin-list order; on an operator in a random numbering (config 5:
// points in natural order) consecutive rows share no neighbours, so every
// gathered P row and every touched C row is a DRAM miss (ncu: 312 GB read per
// pass against 8 GB of operands).  Sorting each bin's rows by the first
// coarse column of P(i,:) -- the aggregate, for smoothed aggregation -- puts
// the rows of one aggregate, which share most neighbours and targets, next to
// each other.  Only the visiting order changes; C and the reference's
// per-entry summation order do not (fp64 atomics already leave the latter
// free).
// ---------------------------------------------------------------------------
__global__ void k_row_order_keys(int64_t n, const int32_t *rows, const int64_t *pd_rp, const int32_t *pd_col,
                                 uint32_t *key, int32_t *val) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int32_t i = rows ? rows[q] : (int32_t)q;
  const int64_t e0 = pd_rp[i];
  key[q] = pd_rp[i + 1] > e0 ? (uint32_t)pd_col[e0] : 0xffffffffu;
  val[q] = i;
}

size_t row_order_scratch_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, (int)n);
  return bytes + 2 * (size_t)n * sizeof(uint32_t) + (size_t)n * sizeof(int32_t) + 256;
}

// rows_out[0..n) = rows_in (identity when null) stably sorted by the first
// coarse column of their P_d row (rows without one last)
cudaError_t launch_row_order(int64_t n, const int32_t *rows_in, int32_t *rows_out, const int64_t *pd_rp,
                             const int32_t *pd_col, void *scratch, size_t scratch_bytes, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  uint32_t *key_in = (uint32_t *)scratch, *key_out = key_in + n;
  int32_t *val_in = (int32_t *)(key_out + n);
  void *tmp = (void *)(((uintptr_t)(val_in + n) + 255) & ~(uintptr_t)255);
  size_t tmp_bytes = scratch_bytes - ((char *)tmp - (char *)scratch);
  k_row_order_keys<<<nb(n, 256), 256, 0, st>>>(n, rows_in, pd_rp, pd_col, key_in, val_in);
  return cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key_in, key_out, val_in, rows_out, (int)n, 0, 32, st);
}

__global__ void k_pack_offsets(int64_t n, const int64_t *rp, int64_t *out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = rp[i] | ((rp[i + 1] - rp[i]) << 40);
}

// out[i] = in[i] - sub (plain offsets) or, with add_packed >= 0, packed
// entries (offset | len << 40) with add_packed added to the offset part
__global__ void k_offsets_shift(int64_t n, const int64_t *in, int64_t sub, int64_t add_packed, int64_t *out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (add_packed < 0) {
    out[i] = in[i] - sub;
  } else {
    const unsigned long long x = (unsigned long long)in[i];
    out[i] = (int64_t)(((x & SMAP_OFF_MASK) + (unsigned long long)add_packed) | (x & ~SMAP_OFF_MASK));
  }
}
cudaError_t launch_offsets_shift(int64_t n, const int64_t *in, int64_t sub, int64_t add_packed, int64_t *out,
                                 cudaStream_t st) {
  if (n > 0) k_offsets_shift<<<nb(n, 256), 256, 0, st>>>(n, in, sub, add_packed, out);
  return cudaGetLastError();
}

cudaError_t launch_pack_offsets(int64_t n, const int64_t *rp, int64_t *out, cudaStream_t st) {
  if (n > 0) k_pack_offsets<<<nb(n, 256), 256, 0, st>>>(n, rp, out);
  return cudaGetLastError();
}

cudaError_t launch_intern(int pass, int64_t n, const uint8_t *src, const int64_t *src_rp, unsigned long long *keys,
                          int64_t *vals, unsigned long long mask, int64_t *slot_of, int64_t *owner, int64_t *words,
                          uint8_t *pool, int64_t *out, int pack_len, unsigned long long *claims, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((n + 31) / 32, 148 * 32);
  if (pass == 0) k_intern_claim<<<blocks, 256, 0, st>>>(n, src, src_rp, keys, vals, mask, slot_of, claims);
  else if (pass == 1) k_intern_resolve<<<blocks, 256, 0, st>>>(n, src, src_rp, vals, slot_of, owner, words);
  else k_intern_copy<<<blocks, 256, 0, st>>>(n, src, src_rp, owner, words, pool, out, pack_len);
  return cudaGetLastError();
}

// flag[i] = 1 for the listed rows that the q4a kernel can fold on its own:
// an A_d row of at most 32 entries, no A_o entries, no P_o entries of its
// own, and none in the P rows of its neighbours (q4a folds P_d rows only)
__global__ void k_pure_rows(int64_t n, const int32_t *rows, Ops op, uint8_t *flag) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int32_t i = rows ? rows[q] : (int32_t)q;
  const bool ao = op.ao_rp && op.ao_rp[i + 1] > op.ao_rp[i];
  bool po = op.po_rp && op.po_rp[i + 1] > op.po_rp[i];
  const int64_t t0 = op.ad_rp[i], t1 = op.ad_rp[i + 1];
  if (op.po_rp && !po)
    for (int64_t t = t0; t < t1; ++t) {
      const int32_t k = op.ad_col[t];
      if (op.po_rp[k + 1] > op.po_rp[k]) { po = true; break; }
    }
  flag[i] = (!ao && !po && t1 - t0 <= 32) ? 1 : 0;
}

cudaError_t launch_pure_rows(int64_t n, const int32_t *rows, const Ops &op, uint8_t *flag, cudaStream_t st) {
  if (n > 0) k_pure_rows<<<nb(n, 256), 256, 0, st>>>(n, rows, op, flag);
  return cudaGetLastError();
}

// poff[e] = P_rp[k] | (P_rp[k+1] - P_rp[k]) << 28 for A entry e with column k
// (the plan checks nnz(P_d) < 2^28 and P rows <= 15): the q4a fold reads this
// instead of A's column and P's row bounds, one dependent load less per chunk
__global__ void k_build_poff(int64_t nnz, const int32_t *ad_col, const int64_t *pd_rp, int32_t *poff) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  const int32_t k = ad_col[e];
  const int64_t x0 = pd_rp[k];
  poff[e] = (int32_t)(x0 | ((pd_rp[k + 1] - x0) << 28));
}

cudaError_t launch_build_poff(int64_t nnz, const int32_t *ad_col, const int64_t *pd_rp, int32_t *poff,
                              cudaStream_t st) {
  if (nnz > 0) k_build_poff<<<nb(nnz, 256), 256, 0, st>>>(nnz, ad_col, pd_rp, poff);
  return cudaGetLastError();
}

// cbase[e] = C row start of the row P_d entry e targets (the outer phase of
// q4a reads it instead of the column -> C row pointer chain)
__global__ void k_build_cbase(int64_t nnz, const int32_t *pd_col, const int64_t *c_rp, int32_t *cbase) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nnz) cbase[e] = (int32_t)c_rp[pd_col[e]];
}

cudaError_t launch_build_cbase(int64_t nnz, const int32_t *pd_col, const int64_t *c_rp, int32_t *cbase,
                               cudaStream_t st) {
  if (nnz > 0) k_build_cbase<<<nb(nnz, 256), 256, 0, st>>>(nnz, pd_col, c_rp, cbase);
  return cudaGetLastError();
}

// last[J] = largest local fine row i with P_d(i, J) != 0 (-1: none): C row
// J holds its final value once every fine row <= last[J] is folded
__global__ void k_c_last_row(int64_t n, const int64_t *pd_rp, const int32_t *pd_col, int32_t *last) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int64_t e = pd_rp[i]; e < pd_rp[i + 1]; ++e) atomicMax(last + pd_col[e], (int32_t)i);
}

cudaError_t launch_c_last_row(int64_t n, const int64_t *pd_rp, const int32_t *pd_col, int64_t ncl, int32_t *last,
                              cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(last, 0xff, sizeof(int32_t) * (ncl > 0 ? ncl : 1), st);
  if (e != cudaSuccess) return e;
  if (n > 0) k_c_last_row<<<nb(n, 256), 256, 0, st>>>(n, pd_rp, pd_col, last);
  return cudaGetLastError();
}


cudaError_t launch_map_lengths(int64_t n, const int64_t *pd_rp, const int64_t *po_rp, const int64_t *apub,
                               const int64_t *ap_nnz, int64_t *slen, int64_t *plen, cudaStream_t st) {
  if (n > 0) k_map_lengths<<<nb(n, 256), 256, 0, st>>>(n, pd_rp, po_rp, apub, ap_nnz, slen, plen);
  return cudaGetLastError();
}

cudaError_t launch_po_srow(int64_t nnz, const int32_t *po_col, const int32_t *colmap, int64_t s_nrows,
                           const int32_t *s_rows, int32_t *po_srow, int *status, cudaStream_t st) {
  if (nnz > 0) k_po_srow<<<nb(nnz, 256), 256, 0, st>>>(nnz, po_col, colmap, s_nrows, s_rows, po_srow, status);
  return cudaGetLastError();
}

cudaError_t launch_max_i64(int64_t n, const int64_t *v, unsigned long long *mx, cudaStream_t st) {
  if (n > 0) k_max_i64<<<nb(n, 256), 256, 0, st>>>(n, v, mx);
  return cudaGetLastError();
}

cudaError_t launch_max_rowlen(int64_t n, const int64_t *rp, unsigned long long *mx, cudaStream_t st) {
  if (n > 0) k_max_rowlen<<<nb(n, 256), 256, 0, st>>>(n, rp, mx);
  return cudaGetLastError();
}

cudaError_t launch_outer_numeric_mapped(int bin, const Ops &op, const int32_t *rows, unsigned long long nrows,
                                        const MapArgs &mp, const OuterTargets &tg, int do_send, int do_local,
                                        int *status, cudaStream_t st, int row0) {
  if (nrows == 0) return cudaSuccess;
  const int warps = 8;
  cudaError_t e;
  if (bin == 3) {  // bin 0 through the 32-bit q4 kernel (eligibility checked by the plan)
    const size_t sm = q4_smem(warps);
    if ((e = opt_in(k_outer_numeric_q4, sm)) != cudaSuccess) return e;
    const unsigned long long rpc = (unsigned long long)warps * Q4_RPW;
    unsigned long long grid = (nrows + rpc - 1) / rpc;
    grid = std::min(grid, grid_cap(k_outer_numeric_q4, warps * 32, sm));
    k_outer_numeric_q4<<<(int)grid, warps * 32, sm, st>>>(op, rows, nrows, mp, tg, do_send, do_local, status,
                                                          row0);
  } else if (bin == 0) {
    constexpr int G = 4, CAP = 32;
    const int gpc = warps * (32 / G);
    size_t sm = (size_t)gpc * group_bytes(G, CAP);
    if ((e = opt_in(k_outer_numeric_mapped<G, CAP>, sm)) != cudaSuccess) return e;
    unsigned long long grid = (nrows + gpc - 1) / gpc;
    grid = std::min(grid, grid_cap(k_outer_numeric_mapped<G, CAP>, warps * 32, sm));
    k_outer_numeric_mapped<G, CAP><<<(int)grid, warps * 32, sm, st>>>(op, rows, nrows, mp, tg, do_send, do_local,
                                                                    status);
  } else if (bin == 2) {  // AP rows of 33..128 slots: 16 lanes per row, two rows per warp
    constexpr int G = 16, CAP = 128;
    const int gpc = warps * (32 / G);
    size_t sm = (size_t)gpc * group_bytes(G, CAP);
    if ((e = opt_in(k_outer_numeric_mapped<G, CAP>, sm)) != cudaSuccess) return e;
    unsigned long long grid = (nrows + gpc - 1) / gpc;
    grid = std::min(grid, grid_cap(k_outer_numeric_mapped<G, CAP>, warps * 32, sm));
    k_outer_numeric_mapped<G, CAP><<<(int)grid, warps * 32, sm, st>>>(op, rows, nrows, mp, tg, do_send, do_local,
                                                                    status);
  } else {
    constexpr int G = 32, CAP = 256;
    const int gpc = warps;
    size_t sm = (size_t)gpc * group_bytes(G, CAP);
    if ((e = opt_in(k_outer_numeric_mapped<G, CAP>, sm)) != cudaSuccess) return e;
    unsigned long long grid = (nrows + gpc - 1) / gpc;
    grid = std::min(grid, grid_cap(k_outer_numeric_mapped<G, CAP>, warps * 32, sm));
    k_outer_numeric_mapped<G, CAP><<<(int)grid, warps * 32, sm, st>>>(op, rows, nrows, mp, tg, do_send, do_local,
                                                                    status);
  }
  return cudaGetLastError();
}

}  // namespace ptapdev
