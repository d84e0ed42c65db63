// ptap_kernels.cu -- sm_100a kernels of the B200 PtAP library.
//
// Kernel map (reference function each one replaces, /root/reference/pkg/src/ptap):
//   k_row_work            work estimates for binning (AP-row upper bound)    (new)
//   k_bin_rows            rows -> work bins                                  (new)
//   k_ap_count<G>         exact nnz of AP rows                               _kernels.py:178-202 row_ap_symbolic
//   k_outer_symbolic<G>   structural outer products into combined-key arenas _kernels.py:361-418 outer_symbolic_driver
//   k_arena_*             sorted drain of an arena into CSR rows             tripleproduct.py:165-212
//   k_sort_rows*          per-row sort of columns (optionally with payload)  hs_drain / np.sort
//   k_outer_numeric<G>    fused AP row + outer-product scatter               _kernels.py:446-515 outer_numeric_driver
//   k_merge_slots/add     received batches -> C in ascending source order    _kernels.py:528-548 scatter_add_rows
//   k_ct_fill/numeric<G>  two-step C~ = A P rows                             _kernels.py:248-349 ap_{symbolic,numeric}_driver
//   k_transpose_*         stable transpose of P blocks with permutation      sparse.py:165-178
//   k_ptc_symbolic        two-step P^T C~ structure                          _kernels.py:558-580
//   k_ptc_numeric<G>      two-step P^T C~ values (staging or C)              _kernels.py:583-677
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "ptap_device.cuh"
#include "ptap_kernels.cuh"

namespace ptapdev {

// ---------------------------------------------------------------------------
// work estimates: apub(i) = sum over A row i of nnz(P row k); mac_ap total
// ---------------------------------------------------------------------------
__global__ void k_row_work(Ops op, int64_t *apub, unsigned long long *mac_total) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long mine = 0;
  if (i < op.nloc) {
    int64_t s = 0;
    for (int64_t t = op.ad_rp[i]; t < op.ad_rp[i + 1]; ++t) {
      int32_t k = op.ad_col[t];
      s += op.pd_rp[k + 1] - op.pd_rp[k];
      if (op.po_rp) s += op.po_rp[k + 1] - op.po_rp[k];
    }
    if (op.ao_rp)
      for (int64_t t = op.ao_rp[i]; t < op.ao_rp[i + 1]; ++t) {
        int32_t k = op.ao_col[t];
        s += op.pr_rp[k + 1] - op.pr_rp[k];
      }
    apub[i] = s;
    mine = (unsigned long long)s;
  }
  unsigned long long w = mine;
  for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(FULL, w, o);
  if (lane_id() == 0 && w) atomicAdd(mac_total, w);
}

// rows -> bins by estimated distinct keys; mode selects rows like the
// reference's loop predicates (0 all, 1 P_o nonempty, 2 P_d nonempty, 3 either)
__global__ void k_bin_rows(int64_t nrows, const int64_t *est, const int64_t *pd_rp, const int64_t *po_rp,
                           int mode, BinLists bl, unsigned long long *selected) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int b = -1;
  if (i < nrows) {
    bool pd = pd_rp && pd_rp[i + 1] > pd_rp[i];
    bool po = po_rp && po_rp[i + 1] > po_rp[i];
    bool want = mode == 0 || (mode == 1 && po) || (mode == 2 && pd) || (mode == 3 && (po || pd)) ||
                (mode == 4 && est[i] >= 0);
    if (want) {
      int64_t n = est[i];
      b = NBINS - 1;
      for (int q = 0; q < NBINS - 1; ++q)
        if (n <= bin_capacity(q)) { b = q; break; }
    }
  }
  // block-level aggregation: one global atomic per bin per block
  __shared__ unsigned scnt[NBINS + 1];
  __shared__ unsigned long long sbase[NBINS + 1];
  const int lane = lane_id();
  if (threadIdx.x <= NBINS) scnt[threadIdx.x] = 0;
  __syncthreads();
  unsigned woff[NBINS];
  unsigned any = __ballot_sync(FULL, b >= 0);
  if (lane == 0 && any) atomicAdd(scnt + NBINS, (unsigned)__popc(any));
#pragma unroll
  for (int q = 0; q < NBINS; ++q) {
    unsigned bits = __ballot_sync(FULL, b == q);
    unsigned w = 0;
    if (bits && lane == 0) w = atomicAdd(scnt + q, (unsigned)__popc(bits));
    woff[q] = __shfl_sync(FULL, w, 0);
  }
  __syncthreads();
  if (threadIdx.x < NBINS) {
    sbase[threadIdx.x] = scnt[threadIdx.x] ? atomicAdd(bl.count + threadIdx.x, (unsigned long long)scnt[threadIdx.x]) : 0;
  } else if (threadIdx.x == NBINS && scnt[NBINS]) {
    atomicAdd(selected, (unsigned long long)scnt[NBINS]);
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NBINS; ++q) {
    unsigned bits = __ballot_sync(FULL, b == q);
    if (b == q && bl.rows[q]) bl.rows[q][sbase[q] + woff[q] + __popc(bits & ((1u << lane) - 1u))] = (int32_t)i;
  }
}

// max estimate inside the last (global-table) bin
__global__ void k_max_est(const int32_t *rows, unsigned long long nrows, const int64_t *est, unsigned long long *mx) {
  unsigned long long r = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long v = 0;
  if (r < nrows) v = (unsigned long long)est[rows ? rows[r] : (int32_t)r];
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
  if (lane_id() == 0 && v) atomicMax(mx, v);
}

// ---------------------------------------------------------------------------
// group-table addressing shared by the row kernels
// ---------------------------------------------------------------------------
struct GroupTables {
  int32_t *keys; double *vals; int32_t *lk;
  PStage ps;
  int32_t *slot_of; int32_t *sb;  // symbolic only
};
// per-group footprint: 8-byte items first (vals[T], a[WIN]) then 4-byte
// items (keys[T], lk[T/2], desc[WIN]); WIN = PAIRS_PER_LANE * GROUP
__host__ __device__ inline size_t group_bytes(int log2t, bool num, int group) {
  size_t T = (size_t)1 << log2t;
  size_t W = (size_t)PAIRS_PER_LANE * group;
  size_t b8 = num ? (T + W) * 8 : 0;
  size_t b4 = T * 4 + (T / 2) * 4 + W * 4 + (num ? 0 : T * 4 + (T / 2) * 4);  // symbolic: slot_of[T], sb[T/2]
  return (b8 + b4 + 15) & ~(size_t)15;
}
template <int GROUP, bool NUM, bool GT>
__device__ __forceinline__ GroupTables group_tables(unsigned char *gtables, int log2t) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int gpw = 32 / GROUP;
  const int gid = (threadIdx.x >> 5) * gpw + lane_id() / GROUP;
  const int gpc = (blockDim.x >> 5) * gpw;
  size_t gb = group_bytes(log2t, NUM, GROUP);
  unsigned char *base = GT ? gtables + ((size_t)blockIdx.x * gpc + gid) * gb : smem + (size_t)gid * gb;
  const int T = 1 << log2t;
  const int W = PAIRS_PER_LANE * GROUP;
  GroupTables t;
  unsigned char *q = base;
  if (NUM) {
    t.vals = (double *)q; q += (size_t)T * 8;
    t.ps.a = (double *)q; q += (size_t)W * 8;
  } else {
    t.vals = nullptr; t.ps.a = nullptr;
  }
  t.keys = (int32_t *)q; q += (size_t)T * 4;
  t.lk = (int32_t *)q; q += (size_t)(T / 2) * 4;
  t.ps.desc = (int32_t *)q; q += (size_t)W * 4;
  t.slot_of = NUM ? nullptr : (int32_t *)q; q += NUM ? 0 : (size_t)T * 4;
  t.sb = NUM ? nullptr : (int32_t *)q;
  return t;
}

// ---------------------------------------------------------------------------
// exact AP row sizes
// ---------------------------------------------------------------------------
template <int GROUP, bool GT>
__global__ void __launch_bounds__(256) k_ap_count(Ops op, const int32_t *rows, unsigned long long nrows, int log2t,
                                                  unsigned char *gtables, int64_t *ap_nnz, int *status) {
  GroupTables tb = group_tables<GROUP, false, GT>(gtables, log2t);
  const int gpw = 32 / GROUP;
  const int gpc = (blockDim.x >> 5) * gpw;
  const int T = 1 << log2t;
  for (unsigned long long r0 = (unsigned long long)blockIdx.x * gpc + (threadIdx.x >> 5) * gpw; r0 < nrows;
       r0 += (unsigned long long)gridDim.x * gpc) {
    unsigned long long ridx = r0 + lane_id() / GROUP;
    int64_t i = ridx < nrows ? (rows ? (int64_t)rows[ridx] : (int64_t)ridx) : -1;
    table_clear<GROUP>(tb.keys, T);
    int nnew = ap_row_accumulate<GROUP, false>(op, i, tb.keys, nullptr, log2t, tb.ps, status);
    nnew = group_sum<GROUP>(nnew);
    if (i >= 0 && (lane_id() & (GROUP - 1)) == 0) ap_nnz[i] = nnew;
    __syncwarp();
  }
}

// Optimistic AP row count: 4 lanes and one 64-slot shared table per row, 8
// rows per warp, over every row of the block.  A row whose distinct columns
// do not fit (or whose pair count exceeds 256) gets -1 and is recounted by
// the binned k_ap_count; on stencil-like inputs no row is.
constexpr int APC_G = 4, APC_LOG2T = 6;
__global__ void __launch_bounds__(256) k_ap_count_small(Ops op, int64_t nrows, const int64_t *apub,
                                                        int64_t *ap_nnz) {
  constexpr int T = 1 << APC_LOG2T, GPC = 256 / APC_G;
  __shared__ int32_t keys_all[GPC][T];
  __shared__ int fail_all[GPC];
  const int gid = threadIdx.x / APC_G;
  int32_t *keys = keys_all[gid];
  int *fail = fail_all + gid;
  PStage ps{nullptr, nullptr};
  for (int64_t r0 = (int64_t)blockIdx.x * GPC; r0 < nrows; r0 += (int64_t)gridDim.x * GPC) {
    int64_t i = r0 + gid;
    if (i >= nrows || __ldg(apub + i) > 256) i = -1;
    table_clear<APC_G>(keys, T);
    if ((lane_id() & (APC_G - 1)) == 0) *fail = 0;
    __syncwarp();
    int nnew = ap_row_accumulate<APC_G, false>(op, i, keys, nullptr, APC_LOG2T, ps, fail);
    nnew = group_sum<APC_G>(nnew);
    __syncwarp();
    if ((lane_id() & (APC_G - 1)) == 0) {
      const int64_t r = r0 + gid;
      if (r < nrows) ap_nnz[r] = (i < 0 || *fail) ? -1 : nnew;
    }
    __syncwarp();
  }
}

// est2[i] = apub[i] for rows the optimistic count left at -1, else -1
__global__ void k_retry_est(int64_t n, const int64_t *ap_nnz, const int64_t *apub, int64_t *est2,
                            unsigned long long *nretry) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool r = i < n && ap_nnz[i] < 0;
  if (i < n) est2[i] = r ? apub[i] : -1;
  unsigned b = __ballot_sync(FULL, r);
  if (lane_id() == 0 && b) atomicAdd(nretry, (unsigned long long)__popc(b));
}

cudaError_t launch_ap_count_small(const Ops &op, int64_t nrows, const int64_t *apub, int64_t *ap_nnz,
                                  cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  int64_t blocks = (nrows + 63) / 64;
  int grid = (int)std::min<int64_t>(blocks, 148 * 32);
  k_ap_count_small<<<grid, 256, 0, st>>>(op, nrows, apub, ap_nnz);
  return cudaGetLastError();
}

cudaError_t launch_retry_est(int64_t n, const int64_t *ap_nnz, const int64_t *apub, int64_t *est2,
                             unsigned long long *nretry, cudaStream_t st) {
  if (n > 0) k_retry_est<<<(int)((n + 255) / 256), 256, 0, st>>>(n, ap_nnz, apub, est2, nretry);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// arenas
// ---------------------------------------------------------------------------
// Insert key = row * m + col.  Row-bucketed arenas (log2b > 0, the local
// C arenas) place row r's keys in its own run of 2^log2b slots (the column
// hashed inside it): the ~13 inserts per C entry then hit the same few lines,
// which neighbouring fine rows (processed together) keep hot in L2, instead
// of one random DRAM line per insert.  Overflow probes linearly, as in the
// hashed mode.
__device__ __forceinline__ void arena_insert(const Arena &a, unsigned long long row, unsigned long long col,
                                             int *status) {
  const unsigned long long key = row * a.m + col;
  unsigned long long *ar = a.keys;
  if (a.log2b > 0) {
    // inside the row's own run first (wrapping within it); a row longer than
    // its run continues at a hashed position, so overflow never cascades
    // into the neighbouring rows' runs
    const unsigned long long bm = (1ull << a.log2b) - 1ull;
    const unsigned long long b0 = (row << a.log2b) & a.mask;
    unsigned long long o = (unsigned long long)hash32((uint32_t)col, a.log2b) & bm;
    for (unsigned long long probe = 0; probe <= bm; ++probe) {
      const unsigned long long hh = b0 | o;
      const unsigned long long k = ar[hh];
      if (k == key) return;
      if (k == EMPTY64) {
        const unsigned long long old = atomicCAS(ar + hh, EMPTY64, key);
        if (old == EMPTY64 || old == key) return;
      }
      o = (o + 1) & bm;
    }
  }
  unsigned long long h = hash64(key) & a.mask;
  for (int probe = 0; probe < 8192; ++probe) {
    unsigned long long k = ar[h];
    if (k == key) return;
    if (k == EMPTY64) {
      unsigned long long old = atomicCAS(ar + h, EMPTY64, key);
      if (old == EMPTY64 || old == key) return;
    }
    h = (h + 1) & a.mask;
  }
  atomicOr(status, ST_ARENA_FULL);
}

// The same insertion returning the key's slot (single-shot pass: the slot
// indexes a value array beside the keys); ~0 when the arena is full.
__device__ __forceinline__ unsigned long long arena_insert_slot(const Arena &a, unsigned long long row,
                                                                unsigned long long col, int *status) {
  const unsigned long long key = row * a.m + col;
  unsigned long long *ar = a.keys;
  if (a.log2b > 0) {
    const unsigned long long bm = (1ull << a.log2b) - 1ull;
    const unsigned long long b0 = (row << a.log2b) & a.mask;
    unsigned long long o = (unsigned long long)hash32((uint32_t)col, a.log2b) & bm;
    for (unsigned long long probe = 0; probe <= bm; ++probe) {
      const unsigned long long hh = b0 | o;
      const unsigned long long k = ar[hh];
      if (k == key) return hh;
      if (k == EMPTY64) {
        const unsigned long long old = atomicCAS(ar + hh, EMPTY64, key);
        if (old == EMPTY64 || old == key) return hh;
      }
      o = (o + 1) & bm;
    }
  }
  unsigned long long h = hash64(key) & a.mask;
  for (int probe = 0; probe < 8192; ++probe) {
    unsigned long long k = ar[h];
    if (k == key) return h;
    if (k == EMPTY64) {
      unsigned long long old = atomicCAS(ar + h, EMPTY64, key);
      if (old == EMPTY64 || old == key) return h;
    }
    h = (h + 1) & a.mask;
  }
  atomicOr(status, ST_ARENA_FULL);
  return ~0ull;
}

// Single-shot pass: symbolic and numeric together (BASELINE north_star (3);
// SURVEY 3.2 "an additional single-shot fast path").  One walk over the fine
// rows: AP(i,:) with values in the group's hash table (row_ap_numeric,
// src/_kernels.py:203-227), then every outer product P(i,J) * AP(i,g) goes
// into the local C arena, key and value at once (the key's slot indexes a
// value array): no second pass over A, no maps.  The arena is drained into
// sorted CSR with the values as payload (k_arena_scatter_vals, k_sort_rows).
template <int GROUP, bool GT>
__global__ void __launch_bounds__(256) k_outer_oneshot(Ops op, const int32_t *rows, unsigned long long nrows,
                                                       int log2t, unsigned char *gtables, Arena local, double *avals,
                                                       int *status) {
  GroupTables tb = group_tables<GROUP, true, GT>(gtables, log2t);
  const int gpw = 32 / GROUP;
  const int gpc = (blockDim.x >> 5) * gpw;
  const int T = 1 << log2t;
  const int gl = lane_id() & (GROUP - 1);
  for (unsigned long long r0 = (unsigned long long)blockIdx.x * gpc + (threadIdx.x >> 5) * gpw; r0 < nrows;
       r0 += (unsigned long long)gridDim.x * gpc) {
    unsigned long long ridx = r0 + lane_id() / GROUP;
    int64_t i = ridx < nrows ? (rows ? (int64_t)rows[ridx] : (int64_t)ridx) : -1;
    int64_t pd0 = 0, pd1 = 0;
    if (i >= 0) { pd0 = op.pd_rp[i]; pd1 = op.pd_rp[i + 1]; }
    if (pd1 <= pd0) i = -1;
    if (__all_sync(FULL, i < 0)) continue;
    table_clear<GROUP>(tb.keys, T);
    ap_row_accumulate<GROUP, true>(op, i, tb.keys, tb.vals, log2t, tb.ps, status);
    if (i >= 0) {
      for (int64_t jj = pd0; jj < pd1; ++jj) {
        const unsigned long long J = (unsigned long long)__ldg(op.pd_col + jj);
        const double pij = __ldg(op.pd_val + jj);
        for (int s = gl; s < T; s += GROUP) {
          const int32_t g = tb.keys[s];
          if (g != EMPTY32) {
            const unsigned long long slot = arena_insert_slot(local, J, (unsigned long long)g, status);
            if (slot != ~0ull) atomicAdd(avals + slot, __dmul_rn(pij, tb.vals[s]));
          }
        }
      }
    }
    __syncwarp();
  }
}

// structural outer products P(i,:) (x) AP(i,:) (src/_kernels.py:361-418):
// local rows go to the local arena keyed (J - c_lo)*m + g, send rows to the
// send arena keyed J*m + g.
template <int GROUP, bool GT>
__global__ void __launch_bounds__(256) k_outer_symbolic(Ops op, const int32_t *rows, unsigned long long nrows,
                                                        int log2t, unsigned char *gtables, int do_send,
                                                        int do_local, Arena local, Arena send, MapOut mo,
                                                        int *status) {
  GroupTables tb = group_tables<GROUP, false, GT>(gtables, log2t);
  const int gpw = 32 / GROUP;
  const int gpc = (blockDim.x >> 5) * gpw;
  const int T = 1 << log2t;
  const int gl = lane_id() & (GROUP - 1);
  const bool maps = mo.smap != nullptr;
  for (unsigned long long r0 = (unsigned long long)blockIdx.x * gpc + (threadIdx.x >> 5) * gpw; r0 < nrows;
       r0 += (unsigned long long)gridDim.x * gpc) {
    unsigned long long ridx = r0 + lane_id() / GROUP;
    int64_t i = ridx < nrows ? (rows ? (int64_t)rows[ridx] : (int64_t)ridx) : -1;
    int64_t pd0 = 0, pd1 = 0, po0 = 0, po1 = 0;
    if (i >= 0) {
      pd0 = op.pd_rp[i]; pd1 = op.pd_rp[i + 1];
      if (op.po_rp) { po0 = op.po_rp[i]; po1 = op.po_rp[i + 1]; }
    }
    bool wl = do_local && pd1 > pd0, ws = do_send && po1 > po0;
    if (!(wl || ws)) i = -1;
    table_clear<GROUP>(tb.keys, T);
    ap_row_accumulate<GROUP, false>(op, i, tb.keys, nullptr, log2t, tb.ps, status);
    int n = table_compact<GROUP, false>(tb.keys, nullptr, T, tb.lk, nullptr);
    if (maps) {
      // sorted pattern of the row (slot = rank), then the slot map of its pairs
      int P2 = 1;
      while (P2 < n) P2 <<= 1;
      int maxP2 = __reduce_max_sync(FULL, i >= 0 ? P2 : 1);
      if (maxP2 <= 64) {
        // short rows: rank of every key = number of smaller keys (no sort)
        if (i >= 0) {
          int32_t *pat = mo.pat + mo.pat_rp[i];
          for (int x = gl; x < n; x += GROUP) {
            const int32_t g = tb.lk[x];
            int rk = 0;
            for (int y = 0; y < n; ++y) rk += tb.lk[y] < g;
            pat[rk] = g;
            tb.slot_of[table_find(tb.keys, log2t, g)] = rk;
          }
          if (gl == 0) mo.nap[i] = (uint8_t)n;
        }
        __syncwarp();
      } else {
        for (int x = gl; x < maxP2; x += GROUP) tb.sb[x] = (i >= 0 && x < n) ? tb.lk[x] : INT32_MAX;
        __syncwarp();
        for (int k = 2; k <= maxP2; k <<= 1)
          for (int j = k >> 1; j > 0; j >>= 1) {
            for (int x = gl; x < maxP2; x += GROUP) {
              int y = x ^ j;
              if (y > x) {
                bool up = (x & k) == 0;
                int32_t kx = tb.sb[x], ky = tb.sb[y];
                if ((kx > ky) == up) { tb.sb[x] = ky; tb.sb[y] = kx; }
              }
            }
            __syncwarp();
          }
        if (i >= 0) {
          int32_t *pat = mo.pat + mo.pat_rp[i];
          for (int x = gl; x < n; x += GROUP) {
            int32_t g = tb.sb[x];
            pat[x] = g;
            tb.slot_of[table_find(tb.keys, log2t, g)] = x;
          }
          if (gl == 0) mo.nap[i] = (uint8_t)n;
        }
        __syncwarp();
      }
      for (int x = gl; x < maxP2; x += GROUP) tb.sb[x] = 0;  // seen[slot]
      __syncwarp();
      ap_row_write_smap<GROUP>(op, i, tb.keys, log2t, tb.slot_of, tb.sb, tb.ps,
                               mo.smap + (i >= 0 ? mo.smap_rp[i] : 0), n <= 127);
    }
    if (i >= 0 && n > 0) {
      if (wl && local.keys)
        for (int64_t jj = pd0; jj < pd1; ++jj) {
          const unsigned long long J = (unsigned long long)__ldg(op.pd_col + jj);
          for (int e = gl; e < n; e += GROUP) arena_insert(local, J, (unsigned long long)tb.lk[e], status);
        }
      if (ws && send.keys)
        for (int64_t jj = po0; jj < po1; ++jj) {
          const unsigned long long J = (unsigned long long)op.p_colmap[op.po_col[jj]];
          for (int e = gl; e < n; e += GROUP) arena_insert(send, J, (unsigned long long)tb.lk[e], status);
        }
    }
    __syncwarp();
  }
}

// Position maps: for every target row J of P(i,:) (local C row or staging
// row), the position of each AP slot of row i inside row J, found by a
// binary search of the row's sorted pattern.  8-lane groups, 4 rows per warp.
__global__ void __launch_bounds__(256) k_build_pmap(Ops op, unsigned long long nrows, MapArgs mp, MapOut mo,
                                                    OuterTargets tg, int *status, int64_t row0) {
  constexpr int G = 8;
  // the row's sorted AP pattern (<= 255 columns) is searched from shared memory
  __shared__ int32_t spat_all[256 / G][256];
  const int gl = lane_id() & (G - 1);
  const int gpc = (blockDim.x >> 5) * (32 / G);
  int32_t *pat = spat_all[threadIdx.x / G];
  const unsigned gmask = 0xffu << (lane_id() & ~(G - 1));
  for (unsigned long long r0 = (unsigned long long)blockIdx.x * gpc + (threadIdx.x >> 5) * (32 / G); r0 < nrows;
       r0 += (unsigned long long)gridDim.x * gpc) {
    unsigned long long ridx = r0 + lane_id() / G;
    if (ridx >= nrows) continue;
    int64_t i = row0 + (int64_t)ridx;
    int64_t pd0 = op.pd_rp[i], pd1 = op.pd_rp[i + 1], po0 = 0, po1 = 0;
    if (op.po_rp) { po0 = op.po_rp[i]; po1 = op.po_rp[i + 1]; }
    int ndP = (int)(pd1 - pd0), nP = ndP + (int)(po1 - po0);
    if (nP == 0) continue;
    int n = mp.nap[i];
    const int32_t *gpat = mo.pat + mo.pat_rp[i];
    __syncwarp(gmask);
    for (int x = gl; x < n; x += G) pat[x] = gpat[x];
    __syncwarp(gmask);
    uint8_t *pm = mp.pmap + mp.pmap_rp[i];
    for (int jj = 0; jj < nP; ++jj) {
      int64_t c0, c1;
      const int32_t *ccol;
      if (jj < ndP) {
        int32_t J = op.pd_col[pd0 + jj];
        c0 = tg.c_rp[J]; c1 = tg.c_rp[J + 1]; ccol = tg.c_col;
      } else {
        int32_t sr = mp.po_srow[po0 + (jj - ndP)];
        if (sr < 0) { if (gl == 0) atomicOr(status, ST_DRIFT); continue; }
        c0 = tg.s_rp[sr]; c1 = tg.s_rp[sr + 1]; ccol = tg.s_col;
      }
      for (int64_t e = c0 + gl; e < c1; e += G) {
        int32_t g = ccol[e];
        int lo = 0, hi = n;
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (pat[mid] < g) lo = mid + 1; else hi = mid;
        }
        if (lo < n && pat[lo] == g) pm[(int64_t)jj * n + lo] = (uint8_t)(e - c0);
      }
    }
  }
}

__global__ void k_arena_fill_empty(unsigned long long *ar, unsigned long long cap) {
  unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < cap) ar[s] = EMPTY64;
}

// received (row, col) structure into the local arena (src/_kernels.py:518-525)
__global__ void k_arena_insert_batch(Arena ar, int64_t nrows, const int32_t *rows, const int64_t *rp,
                                     const int32_t *col, int64_t m, int64_t c_lo, int64_t c_hi, int *status) {
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nrows) return;
  int32_t J = rows[w];
  if (J < c_lo || J >= c_hi) { if (lane_id() == 0) atomicOr(status, ST_DRIFT); return; }
  const unsigned long long r = (unsigned long long)(J - c_lo);
  for (int64_t e = rp[w] + lane_id(); e < rp[w + 1]; e += 32) arena_insert(ar, r, (unsigned long long)col[e], status);
}

__global__ void k_arena_rowcount(Arena ar, unsigned long long m, int64_t *cnt) {
  unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (s > ar.mask) return;
  unsigned long long k = ar.keys[s];
  if (k != EMPTY64) atomicAdd((unsigned long long *)(cnt + k / m), 1ull);
}

__global__ void k_arena_scatter(Arena ar, unsigned long long m, const int64_t *rp, int64_t *cursor, int32_t *col) {
  unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (s > ar.mask) return;
  unsigned long long k = ar.keys[s];
  if (k == EMPTY64) return;
  unsigned long long r = k / m;
  unsigned long long pos = (unsigned long long)rp[r] + atomicAdd((unsigned long long *)(cursor + r), 1ull);
  col[pos] = (int32_t)(k - r * m);
}

__global__ void k_arena_scatter_vals(Arena ar, unsigned long long m, const int64_t *rp, int64_t *cursor, int32_t *col,
                                     const double *avals, int64_t *payload) {
  unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (s > ar.mask) return;
  unsigned long long k = ar.keys[s];
  if (k == EMPTY64) return;
  unsigned long long r = k / m;
  unsigned long long pos = (unsigned long long)rp[r] + atomicAdd((unsigned long long *)(cursor + r), 1ull);
  col[pos] = (int32_t)(k - r * m);
  payload[pos] = __double_as_longlong(avals[s]);
}

// ---------------------------------------------------------------------------
// per-row sorts (warp per row, bitonic in shared memory, <= 1024 entries;
// block per row up to 8192 entries for the rare wide rows)
// ---------------------------------------------------------------------------
template <bool PAIRS>
__global__ void __launch_bounds__(256) k_sort_rows(int64_t nrows, const int64_t *rp, int32_t *keys,
                                                   int64_t *payload, int32_t *wide_rows,
                                                   unsigned long long *nwide) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int wpc = blockDim.x >> 5;
  int32_t *sk = (int32_t *)(smem + (size_t)warp * 1024 * 4);
  int64_t *sp = (int64_t *)(smem + (size_t)wpc * 1024 * 4 + (size_t)warp * 1024 * 8);
  for (int64_t r = (int64_t)blockIdx.x * wpc + warp; r < nrows; r += (int64_t)gridDim.x * wpc) {
    int64_t b = rp[r];
    int L = (int)(rp[r + 1] - b);
    if (L <= 1) continue;
    if (L > 1024) {
      if (lane == 0) wide_rows[atomicAdd(nwide, 1ull)] = (int32_t)r;
      continue;
    }
    int P2 = 1;
    while (P2 < L) P2 <<= 1;
    for (int x = lane; x < P2; x += 32) {
      sk[x] = x < L ? keys[b + x] : INT32_MAX;
      if (PAIRS) sp[x] = x < L ? payload[b + x] : 0;
    }
    __syncwarp();
    for (int k = 2; k <= P2; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int x = lane; x < P2; x += 32) {
          int y = x ^ j;
          if (y > x) {
            bool up = (x & k) == 0;
            int32_t kx = sk[x], ky = sk[y];
            if ((kx > ky) == up) {
              sk[x] = ky; sk[y] = kx;
              if (PAIRS) { int64_t t = sp[x]; sp[x] = sp[y]; sp[y] = t; }
            }
          }
        }
        __syncwarp();
      }
    for (int x = lane; x < L; x += 32) {
      keys[b + x] = sk[x];
      if (PAIRS) payload[b + x] = sp[x];
    }
    __syncwarp();
  }
}

template <bool PAIRS>
__global__ void __launch_bounds__(1024) k_sort_rows_block(const int32_t *rows, const int64_t *rp, int32_t *keys,
                                                          int64_t *payload, int *status) {
  extern __shared__ __align__(16) unsigned char smem[];
  int64_t r = rows[blockIdx.x];
  int64_t b = rp[r];
  int L = (int)(rp[r + 1] - b);
  if (L > 8192) { if (threadIdx.x == 0) atomicOr(status, ST_ROW_TOO_WIDE); return; }
  int P2 = 1;
  while (P2 < L) P2 <<= 1;
  int32_t *sk = (int32_t *)smem;
  int64_t *sp = (int64_t *)(smem + 8192 * 4);
  for (int x = threadIdx.x; x < P2; x += blockDim.x) {
    sk[x] = x < L ? keys[b + x] : INT32_MAX;
    if (PAIRS) sp[x] = x < L ? payload[b + x] : 0;
  }
  __syncthreads();
  for (int k = 2; k <= P2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int x = threadIdx.x; x < P2; x += blockDim.x) {
        int y = x ^ j;
        if (y > x) {
          bool up = (x & k) == 0;
          int32_t kx = sk[x], ky = sk[y];
          if ((kx > ky) == up) {
            sk[x] = ky; sk[y] = kx;
            if (PAIRS) { int64_t t = sp[x]; sp[x] = sp[y]; sp[y] = t; }
          }
        }
      }
      __syncthreads();
    }
  for (int x = threadIdx.x; x < L; x += blockDim.x) {
    keys[b + x] = sk[x];
    if (PAIRS) payload[b + x] = sp[x];
  }
}

// ---------------------------------------------------------------------------
// fused numeric all-at-once / merged (src/_kernels.py:446-515)
// ---------------------------------------------------------------------------
template <int GROUP, bool GT>
__global__ void __launch_bounds__(256) k_outer_numeric(Ops op, const int32_t *rows, unsigned long long nrows,
                                                       int log2t, unsigned char *gtables, int do_send,
                                                       int do_local, OuterTargets tg, int *status) {
  GroupTables tb = group_tables<GROUP, true, GT>(gtables, log2t);
  const int gpw = 32 / GROUP;
  const int gpc = (blockDim.x >> 5) * gpw;
  const int T = 1 << log2t;
  const int gl = lane_id() & (GROUP - 1);
  for (unsigned long long r0 = (unsigned long long)blockIdx.x * gpc + (threadIdx.x >> 5) * gpw; r0 < nrows;
       r0 += (unsigned long long)gridDim.x * gpc) {
    unsigned long long ridx = r0 + lane_id() / GROUP;
    int64_t i = ridx < nrows ? (rows ? (int64_t)rows[ridx] : (int64_t)ridx) : -1;
    int64_t pd0 = 0, pd1 = 0, po0 = 0, po1 = 0;
    if (i >= 0) {
      pd0 = op.pd_rp[i]; pd1 = op.pd_rp[i + 1];
      if (op.po_rp) { po0 = op.po_rp[i]; po1 = op.po_rp[i + 1]; }
    }
    bool wl = do_local && pd1 > pd0, ws = do_send && po1 > po0;
    if (!(wl || ws)) i = -1;
    if (__all_sync(FULL, i < 0)) continue;
    table_clear<GROUP>(tb.keys, T);
    int n = group_sum<GROUP>(ap_row_accumulate<GROUP, true>(op, i, tb.keys, tb.vals, log2t, tb.ps, status));
    // outer product P(i,:) (x) AP(i,:): for each target row J, the lanes walk
    // C's stored row J (coalesced columns) and pull the matching AP value
    // from the group's table; every AP key must be found in every row J.
    int nj_l = wl ? (int)(pd1 - pd0) : 0;
    int nj_s = ws ? (int)(po1 - po0) : 0;
    int maxj = __reduce_max_sync(FULL, nj_l + nj_s);
    for (int jj = 0; jj < maxj; ++jj) {
      int found = 0;
      bool live = i >= 0 && jj < nj_l + nj_s;
      if (live) {
        int64_t c0, c1;
        double pij;
        const int32_t *ccol;
        double *cval;
        bool row_ok = true;
        if (jj < nj_l) {
          int32_t J = __ldg(op.pd_col + pd0 + jj);
          pij = __ldg(op.pd_val + pd0 + jj);
          c0 = __ldg(tg.c_rp + J); c1 = __ldg(tg.c_rp + J + 1);
          ccol = tg.c_col; cval = tg.c_val;
        } else {
          int64_t e = po0 + (jj - nj_l);
          int32_t Jg = __ldg(op.p_colmap + __ldg(op.po_col + e));
          pij = __ldg(op.po_val + e);
          int64_t sr = lower_bound32(tg.s_rows, 0, tg.s_nrows, Jg);
          row_ok = sr < tg.s_nrows && __ldg(tg.s_rows + sr) == Jg;
          c0 = row_ok ? __ldg(tg.s_rp + sr) : 0; c1 = row_ok ? __ldg(tg.s_rp + sr + 1) : 0;
          ccol = tg.s_col; cval = tg.s_val;
        }
        for (int64_t e = c0 + gl; e < c1; e += GROUP) {
          int sl = table_find(tb.keys, log2t, __ldg(ccol + e));
          if (sl >= 0) {
            ++found;
            atomicAdd(cval + e, __dmul_rn(pij, tb.vals[sl]));
          }
        }
      }
      found = group_sum<GROUP>(found);
      if (live && found != n && gl == 0) atomicOr(status, ST_DRIFT);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// received batches: slot map (symbolic) and ordered adds (numeric)
// ---------------------------------------------------------------------------
__global__ void k_merge_slots(int64_t nrows, const int32_t *rows, const int64_t *rp, const int32_t *col,
                              int64_t c_lo, const int64_t *c_rp, const int32_t *c_col, int64_t *slot, int *status) {
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nrows) return;
  int64_t J = rows[w] - c_lo;
  int64_t c0 = c_rp[J], c1 = c_rp[J + 1];
  for (int64_t e = rp[w] + lane_id(); e < rp[w + 1]; e += 32) {
    int64_t pos = lower_bound32(c_col, c0, c1, col[e]);
    if (pos < c1 && c_col[pos] == col[e]) slot[e] = pos;
    else { slot[e] = -1; atomicOr(status, ST_DRIFT); }
  }
}

__global__ void k_merge_add(int64_t n, const int64_t *slot, const double *vals, double *c_val) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) {
    int64_t s = slot[e];
    if (s >= 0) c_val[s] = __dadd_rn(c_val[s], vals[e]);
  }
}

// ---------------------------------------------------------------------------
// two-step: C~ = A P rows (structure sorted later), values onto structure
// ---------------------------------------------------------------------------
template <int GROUP, bool GT>
__global__ void __launch_bounds__(256) k_ct_fill(Ops op, const int32_t *rows, unsigned long long nrows, int log2t,
                                                 unsigned char *gtables, const int64_t *ct_rp, int32_t *ct_col,
                                                 int *status) {
  GroupTables tb = group_tables<GROUP, false, GT>(gtables, log2t);
  const int gpw = 32 / GROUP;
  const int gpc = (blockDim.x >> 5) * gpw;
  const int T = 1 << log2t;
  const int gl = lane_id() & (GROUP - 1);
  for (unsigned long long r0 = (unsigned long long)blockIdx.x * gpc + (threadIdx.x >> 5) * gpw; r0 < nrows;
       r0 += (unsigned long long)gridDim.x * gpc) {
    unsigned long long ridx = r0 + lane_id() / GROUP;
    int64_t i = ridx < nrows ? (rows ? (int64_t)rows[ridx] : (int64_t)ridx) : -1;
    table_clear<GROUP>(tb.keys, T);
    ap_row_accumulate<GROUP, false>(op, i, tb.keys, nullptr, log2t, tb.ps, status);
    int n = table_compact<GROUP, false>(tb.keys, nullptr, T, tb.lk, nullptr);
    if (i >= 0) {
      int64_t b = ct_rp[i];
      if (ct_rp[i + 1] - b != n) { if (gl == 0) atomicOr(status, ST_DRIFT); }
      else for (int e = gl; e < n; e += GROUP) ct_col[b + e] = tb.lk[e];
    }
    __syncwarp();
  }
}

template <int GROUP, bool GT>
__global__ void __launch_bounds__(256) k_ct_numeric(Ops op, const int32_t *rows, unsigned long long nrows,
                                                    int log2t, unsigned char *gtables, const int64_t *ct_rp,
                                                    const int32_t *ct_col, double *ct_val, int *status) {
  GroupTables tb = group_tables<GROUP, true, GT>(gtables, log2t);
  const int gpw = 32 / GROUP;
  const int gpc = (blockDim.x >> 5) * gpw;
  const int T = 1 << log2t;
  const int gl = lane_id() & (GROUP - 1);
  for (unsigned long long r0 = (unsigned long long)blockIdx.x * gpc + (threadIdx.x >> 5) * gpw; r0 < nrows;
       r0 += (unsigned long long)gridDim.x * gpc) {
    unsigned long long ridx = r0 + lane_id() / GROUP;
    int64_t i = ridx < nrows ? (rows ? (int64_t)rows[ridx] : (int64_t)ridx) : -1;
    table_clear<GROUP>(tb.keys, T);
    int nnew = ap_row_accumulate<GROUP, true>(op, i, tb.keys, tb.vals, log2t, tb.ps, status);
    nnew = group_sum<GROUP>(nnew);
    if (i >= 0) {
      int64_t b = ct_rp[i], L = ct_rp[i + 1] - b;
      if (L != nnew) { if (gl == 0) atomicOr(status, ST_DRIFT); }
      else
        for (int64_t e = gl; e < L; e += GROUP) {
          int s = table_find(tb.keys, log2t, ct_col[b + e]);
          if (s < 0) atomicOr(status, ST_DRIFT);
          else ct_val[b + e] = tb.vals[s];
        }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// stable transpose of a P block (src/sparse.py:165-178)
// ---------------------------------------------------------------------------
__global__ void k_count_cols(int64_t nnz, const int32_t *col, int64_t *cnt) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nnz) atomicAdd((unsigned long long *)(cnt + col[e]), 1ull);
}

__global__ void k_transpose_scatter(int64_t nrows, const int64_t *rp, const int32_t *col, const int64_t *t_rp,
                                    int64_t *cursor, int32_t *t_row, int64_t *t_perm) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
    int32_t q = col[e];
    int64_t pos = t_rp[q] + (int64_t)atomicAdd((unsigned long long *)(cursor + q), 1ull);
    t_row[pos] = (int32_t)i;
    if (t_perm) t_perm[pos] = e;
  }
}

__global__ void k_gather(int64_t n, const int64_t *perm, const double *src, double *dst) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) dst[e] = src[perm[e]];
}

// two-step structure of P^T C~ rows into an arena; target_map maps the
// transposed row id to the arena row (local J, or global J for the send side)
__global__ void k_ptc_symbolic(int64_t nrows, const int64_t *t_rp, const int32_t *t_row, const int32_t *target_map,
                               int64_t target_offset, const int64_t *ct_rp, const int32_t *ct_col, Arena ar,
                               unsigned long long m, int *status) {
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nrows) return;
  unsigned long long tgt = target_map ? (unsigned long long)target_map[w] : (unsigned long long)(w + target_offset);
  for (int64_t t = t_rp[w]; t < t_rp[w + 1]; ++t) {
    int32_t i = t_row[t];
    for (int64_t e = ct_rp[i] + lane_id(); e < ct_rp[i + 1]; e += 32)
      arena_insert(ar, tgt, (unsigned long long)ct_col[e], status);
  }
}

// two-step numeric rows of P^T C~ (src/_kernels.py:583-677): fold over the
// transposed row's entries (ascending fine row) with C~ rows scattered per
// step; then written onto the target structure (staging: set; C: 0 + acc).
template <int GROUP, bool GT>
__global__ void __launch_bounds__(256) k_ptc_numeric(const int32_t *rows, unsigned long long nrows, int log2t,
                                                     unsigned char *gtables, const int64_t *t_rp,
                                                     const int32_t *t_row, const double *t_val,
                                                     const int32_t *target_map, int64_t target_offset,
                                                     const int64_t *ct_rp, const int32_t *ct_col,
                                                     const double *ct_val, PtcTarget tg, int *status) {
  GroupTables tb = group_tables<GROUP, true, GT>(gtables, log2t);
  const int gpw = 32 / GROUP;
  const int gpc = (blockDim.x >> 5) * gpw;
  const int T = 1 << log2t;
  const int gl = lane_id() & (GROUP - 1);
  for (unsigned long long r0 = (unsigned long long)blockIdx.x * gpc + (threadIdx.x >> 5) * gpw; r0 < nrows;
       r0 += (unsigned long long)gridDim.x * gpc) {
    unsigned long long ridx = r0 + lane_id() / GROUP;
    int64_t q = ridx < nrows ? (rows ? (int64_t)rows[ridx] : (int64_t)ridx) : -1;
    table_clear<GROUP>(tb.keys, T);
    int64_t t0 = 0, t1 = 0;
    if (q >= 0) { t0 = t_rp[q]; t1 = t_rp[q + 1]; }
    int len = (int)(t1 - t0);
    int maxlen = __reduce_max_sync(FULL, len);
    bool ok = true;
    int nnew = 0;
    for (int t = 0; t < maxlen; ++t) {
      int64_t e0 = 0, e1 = 0;
      double lv = 0.0;
      if (t < len) {
        int32_t i = t_row[t0 + t];
        lv = t_val[t0 + t];
        e0 = ct_rp[i]; e1 = ct_rp[i + 1];
      }
      for (int64_t e = e0 + gl; e < e1; e += GROUP)
        ok &= table_put<true>(tb.keys, tb.vals, log2t, ct_col[e], __dmul_rn(lv, ct_val[e]), nnew);
      __syncwarp();
    }
    if (!ok) atomicOr(status, ST_TABLE_FULL);
    nnew = group_sum<GROUP>(nnew);
    int found = 0;
    bool checked = false;
    if (q >= 0) {
      int64_t tgt = target_map ? (int64_t)target_map[q] : q + target_offset;
      int64_t r = tgt;
      if (tg.is_staging) {
        r = lower_bound32(tg.rows, 0, tg.nrows, (int32_t)tgt);
        if (r >= tg.nrows || tg.rows[r] != (int32_t)tgt) r = -1;
      }
      if (r < 0) {
        if (nnew > 0 && gl == 0) atomicOr(status, ST_DRIFT);
      } else {
        checked = true;
        int64_t c0 = tg.rp[r], c1 = tg.rp[r + 1];
        for (int64_t e = c0 + gl; e < c1; e += GROUP) {
          int s = table_find(tb.keys, log2t, tg.col[e]);
          if (s >= 0) {
            ++found;
            tg.val[e] = tg.is_staging ? tb.vals[s] : __dadd_rn(0.0, tb.vals[s]);
          } else {
            tg.val[e] = 0.0;  // C slot fed only by received batches (or drift on staging)
            if (tg.is_staging) atomicOr(status, ST_DRIFT);
          }
        }
      }
    }
    found = group_sum<GROUP>(found);  // warp-collective: outside the per-group branches
    if (checked && found != nnew && gl == 0) atomicOr(status, ST_DRIFT);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// scans (exclusive, int64), compaction helpers
// ---------------------------------------------------------------------------
constexpr int SCAN_THREADS = 256, SCAN_ITEMS = 8, SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_tiles(const int64_t *in, int64_t *out, int64_t n,
                                                             int64_t *tile_sums) {
  __shared__ int64_t warp_tot[SCAN_THREADS / 32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int64_t v[SCAN_ITEMS];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    v[k] = (base + k < n) ? in[base + k] : 0;
    s += v[k];
  }
  int64_t incl = s;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t wt = lane < SCAN_THREADS / 32 ? warp_tot[lane] : 0;
    int64_t wi = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(FULL, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < SCAN_THREADS / 32) warp_tot[lane] = wi - wt;
    if (lane == SCAN_THREADS / 32 - 1) tile_sums[blockIdx.x] = wi;
  }
  __syncthreads();
  int64_t run = warp_tot[warp] + incl - s;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
}

__global__ void k_scan_add(int64_t *out, int64_t n, const int64_t *tile_off) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) out[e] += tile_off[e / SCAN_TILE];
}

__global__ void k_set_total(int64_t *out, int64_t n, const int64_t *in) {
  // out[n] = out[n-1] + in[n-1]
  if (n == 0) out[0] = 0;
  else out[n] = out[n - 1] + in[n - 1];
}

// flags[i] = cnt[i] > 0 ; used to compact the nonempty send rows in order
__global__ void k_nonzero_flags(int64_t n, const int64_t *cnt, int64_t *flags) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flags[i] = cnt[i] > 0 ? 1 : 0;
}

__global__ void k_compact_rows(int64_t n, const int64_t *cnt, const int64_t *pos, const int64_t *dense_rp,
                               int32_t *rows, int64_t *rp) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && cnt[i] > 0) {
    rows[pos[i]] = (int32_t)i;
    rp[pos[i]] = dense_rp[i];
  }
}

__global__ void k_fill_i64(int64_t *p, int64_t n, int64_t v) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void k_iota32(int32_t *p, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = (int32_t)i;
}

__global__ void k_colmap_targets(int64_t n, const int32_t *colmap, int32_t *out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = colmap[i];
}

__global__ void k_row_lengths(int64_t n, const int64_t *rp, int64_t *len) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) len[i] = rp[i + 1] - rp[i];
}

// outer-product bounds: out[0] = sum nnz(P_d(i,:))*ap_nnz(i), out[1] = sum
// nnz(P_o(i,:))*ap_nnz(i), out[2] = sum ap_nnz(i)
__global__ void k_outer_bounds(int64_t n, const int64_t *pd_rp, const int64_t *po_rp, const int64_t *ap_nnz,
                               unsigned long long *out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long a = 0, b = 0, c = 0;
  if (i < n) {
    c = (unsigned long long)ap_nnz[i];
    a = (unsigned long long)(pd_rp[i + 1] - pd_rp[i]) * c;
    if (po_rp) b = (unsigned long long)(po_rp[i + 1] - po_rp[i]) * c;
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(FULL, a, o); b += __shfl_xor_sync(FULL, b, o); c += __shfl_xor_sync(FULL, c, o);
  }
  if (lane_id() == 0) {
    if (a) atomicAdd(out, a);
    if (b) atomicAdd(out + 1, b);
    if (c) atomicAdd(out + 2, c);
  }
}

// rehash the keys of an arena into a larger one (growth on overflow)
__global__ void k_arena_rehash(Arena from, Arena to, int *status) {
  unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (s > from.mask) return;
  unsigned long long k = from.keys[s];
  if (k != EMPTY64) arena_insert(to, k / to.m, k % to.m, status);
}

// Bin-0 structural outer products with the slot maps (AP rows <= 32 slots,
// <= 128 fold pairs per row, every offset within 32 bits -- the plan's q4
// condition): 8 fine rows per warp, 4 lanes each, one 64-slot table per row.
// A single walk over the pairs in fold order inserts the AP columns; the pair
// that inserts a key is that key's first in fold order, so recording the
// table position (and an inserted bit) per pair gives the slot map once the
// row's pattern is ranked -- no second walk and no per-pair probe.  The map
// bytes are assembled in shared memory and stored as aligned 32-bit words.
constexpr int SQ_R = 8, SQ_G = 4, SQ_LOG2T = 6, SQ_T = 64, SQ_SMB = 132;
// keys/lk rows padded to 68 words: the 8 row groups of a warp read the same
// index of their own rows at once, and a 64-word stride put all 8 in one bank
constexpr int SQ_TP = SQ_T + 4;
struct __align__(16) SqWarp {
  int32_t keys[SQ_R][SQ_TP];
  int32_t lk[SQ_R][SQ_TP];      // compacted keys, INT32_MAX-padded to a multiple of 4
  uint8_t lpos[SQ_R][SQ_T];     // their table positions
  uint8_t slot_of[SQ_R][SQ_T];  // table position -> slot (rank)
  uint32_t sm[SQ_R][SQ_SMB / 4];  // slot bytes of the row, at (start & 3) + pair
  int2 dp[SQ_G][SQ_R];          // step entries: P row start, packed offsets/lengths
  int32_t o0[SQ_G][SQ_R];       // P_o row start of the step entry
};

template <int SRC>
__device__ __forceinline__ void sq_walk(const Ops &op, SqWarp &W, int i, int gl, int r, int sbo, int &run) {
  constexpr int G = SQ_G;
  const int64_t *arp = SRC ? op.ao_rp : op.ad_rp;
  const int32_t *acol = SRC ? op.ao_col : op.ad_col;
  const int64_t *qrp = SRC ? op.pr_rp : op.pd_rp;
  const int32_t *qcol = SRC ? op.pr_col : op.pd_col;
  const int32_t coff = SRC ? 0 : (int32_t)op.c_lo;
  const bool po_here = SRC == 0 && op.po_rp != nullptr;
  int32_t *keys = W.keys[r];
  uint8_t *smb = (uint8_t *)W.sm[r];
  int t0 = 0, len = 0;
  if (i >= 0) { t0 = (int)__ldg(arp + i); len = (int)__ldg(arp + i + 1) - t0; }
  const int maxlen = __reduce_max_sync(FULL, len);
#pragma unroll 1
  for (int tb = 0; tb < maxlen; tb += G) {
    const int t = tb + gl;
    int d0 = 0, o0 = 0, nd = 0, plen = 0;
    if (t < len) {
      const int k = __ldg(acol + t0 + t);
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
    W.dp[gl][r] = make_int2(d0, (int)((uint32_t)(run + incl - plen) | ((uint32_t)nd << 16) | ((uint32_t)plen << 24)));
    if (po_here) W.o0[gl][r] = o0;
    run += __shfl_sync(FULL, incl, G - 1, G);
    __syncwarp();
    const int steps = min(G, maxlen - tb);
    // the AP columns of all steps first (independent loads), then the inserts
    // in step order
    int32_t gv[G];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      gv[j] = EMPTY32;
      if (j < steps) {
        const int2 e = W.dp[j][r];
        const int plj = (int)((uint32_t)e.y >> 24), ndj = (e.y >> 16) & 0xff;
        if (gl < plj)
          gv[j] = gl < ndj ? __ldg(qcol + e.x + gl) + coff
                           : op.p_colmap[op.po_col[W.o0[j][r] + (gl - ndj)]];
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
      if (j < steps) {
        const int2 e = W.dp[j][r];
        const int plj = (int)((uint32_t)e.y >> 24), ndj = (e.y >> 16) & 0xff, off = sbo + (e.y & 0xffff);
        for (int u = gl; u < plj; u += G) {
          const int32_t g = u == gl ? gv[j] : (u < ndj ? __ldg(qcol + e.x + u) + coff
                                                       : op.p_colmap[op.po_col[W.o0[j][r] + (u - ndj)]]);
          uint32_t h = hash32((uint32_t)g, SQ_LOG2T);
          uint8_t rec = 0xff;
          for (int probe = 0; probe < SQ_T; ++probe) {
            const int32_t kk = keys[h];
            if (kk == g) { rec = (uint8_t)h; break; }
            if (kk == EMPTY32) {
              const int32_t old = atomicCAS(keys + h, EMPTY32, g);
              if (old == EMPTY32) { rec = (uint8_t)(h | 0x80); break; }
              if (old == g) { rec = (uint8_t)h; break; }
            }
            h = (h + 1) & (SQ_T - 1);
          }
          smb[off + u] = rec;  // 0xff: table full (cannot happen for <= 32 keys)
        }
        __syncwarp();
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_outer_symbolic_q4(Ops op, const int32_t *rows, unsigned long long nrows,
                                                           int do_send, int do_local, Arena local, Arena send,
                                                           MapOut mo, int *status, int row0) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int G = SQ_G;
  const int lane = lane_id(), gl = lane & (G - 1), r = lane / G;
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  SqWarp &W = ((SqWarp *)smem)[warp];
  const int total = (int)nrows;
  for (int r0 = (blockIdx.x * nwarps + warp) * SQ_R; r0 < total; r0 += gridDim.x * nwarps * SQ_R) {
    const int ridx = r0 + r;
    int i = ridx < total ? (rows ? rows[ridx] : row0 + ridx) : -1;
    int pd0 = 0, pd1 = 0, po0 = 0, po1 = 0;
    if (i >= 0) {
      pd0 = (int)__ldg(op.pd_rp + i); pd1 = (int)__ldg(op.pd_rp + i + 1);
      if (op.po_rp) { po0 = (int)__ldg(op.po_rp + i); po1 = (int)__ldg(op.po_rp + i + 1); }
    }
    const bool wl = do_local && pd1 > pd0, ws = do_send && po1 > po0;
    if (!(wl || ws)) i = -1;
    if (__all_sync(FULL, i < 0)) continue;
    const int sb = i >= 0 ? (int)mo.smap_rp[i] : 0;
    const int sbo = sb & 3;
    for (int x = gl; x < SQ_T; x += G) W.keys[r][x] = EMPTY32;
    __syncwarp();
    int run = 0;
    sq_walk<0>(op, W, i, gl, r, sbo, run);
    if (op.ao_rp != nullptr) sq_walk<1>(op, W, i, gl, r, sbo, run);
    // compact the row's keys with their table positions
    int n = 0;
    const unsigned gmask = 0xfu << (lane & ~(G - 1));
    for (int s0 = 0; s0 < SQ_T; s0 += G) {
      const int sidx = s0 + gl;
      const int32_t k = W.keys[r][sidx];
      const bool occ = k != EMPTY32;
      const unsigned b = __ballot_sync(FULL, occ) & gmask;
      if (occ) {
        const int at = n + __popc(b & ((1u << lane) - 1u));
        W.lk[r][at] = k;
        W.lpos[r][at] = (uint8_t)sidx;
      }
      n += __popc(b);
    }
    if (gl < 4) W.lk[r][n + gl] = INT32_MAX;  // n <= SQ_T: the pad fits the row
    __syncwarp();
    // slot = rank of the key in the row (sorted pattern), no sort needed: the
    // lane's keys stay in registers and the row streams past them 4 at a time
    {
      constexpr int KPL = SQ_T / G;
      const int nmax = __reduce_max_sync(FULL, i >= 0 ? n : 0);
      int32_t mine[KPL];
      int rk[KPL];
#pragma unroll
      for (int q = 0; q < KPL; ++q) {
        mine[q] = gl + G * q < n ? W.lk[r][gl + G * q] : INT32_MAX;
        rk[q] = 0;
      }
      for (int y0 = 0; y0 < n; y0 += 4) {
        const int4 v = *reinterpret_cast<const int4 *>(&W.lk[r][y0]);
#pragma unroll
        for (int q = 0; q < KPL; ++q)
          if (G * q < nmax) rk[q] += (v.x < mine[q]) + (v.y < mine[q]) + (v.z < mine[q]) + (v.w < mine[q]);
      }
      if (i >= 0) {
        int32_t *pat = mo.pat + mo.pat_rp[i];
#pragma unroll
        for (int q = 0; q < KPL; ++q) {
          const int x = gl + G * q;
          if (x < n) {
            pat[rk[q]] = mine[q];
            W.slot_of[r][W.lpos[r][x]] = (uint8_t)rk[q];
          }
        }
        if (gl == 0) mo.nap[i] = (uint8_t)n;
      }
    }
    __syncwarp();
    // slot bytes: table position -> slot, keeping the first-product bit; then
    // store them (aligned interior as 32-bit words, the two ends as bytes)
    if (i >= 0) {
      const int npairs = run;
      uint8_t *smb = (uint8_t *)W.sm[r];
      for (int q = gl; q < npairs; q += G) {
        const uint8_t b = smb[sbo + q];
        smb[sbo + q] = (uint8_t)(W.slot_of[r][b & 0x7f] | (b & 0x80));
      }
      __syncwarp(0xfu << (lane & ~(G - 1)));
      uint8_t *dst = mo.smap + (int64_t)sb - sbo;  // 4-byte aligned
      const int nbytes = sbo + npairs, nw = (nbytes + 3) >> 2;
      for (int w = gl; w < nw; w += G) {
        const bool edge = (w == 0 && sbo != 0) || (w == nw - 1 && (nbytes & 3) != 0);
        if (!edge) {
          ((uint32_t *)dst)[w] = W.sm[r][w];
        } else {
          for (int c = 0; c < 4; ++c) {
            const int q = 4 * w + c;
            if (q >= sbo && q < nbytes) dst[q] = smb[q];
          }
        }
      }
    }
    // structural outer products into the arenas
    if (i >= 0 && n > 0) {
      if (wl && local.keys)
        for (int jj = pd0; jj < pd1; ++jj) {
          const unsigned long long J = (unsigned long long)__ldg(op.pd_col + jj);
          for (int e = gl; e < n; e += G) arena_insert(local, J, (unsigned long long)W.lk[r][e], status);
        }
      if (ws && send.keys)
        for (int jj = po0; jj < po1; ++jj) {
          const unsigned long long J = (unsigned long long)op.p_colmap[op.po_col[jj]];
          for (int e = gl; e < n; e += G) arena_insert(send, J, (unsigned long long)W.lk[r][e], status);
        }
    }
    __syncwarp();
  }
}

cudaError_t launch_outer_symbolic_q4(const Ops &op, const int32_t *rows, unsigned long long nrows, int do_send,
                                     int do_local, Arena local, Arena send, const MapOut &mo, int *status,
                                     cudaStream_t stream, int row0) {
  if (nrows == 0) return cudaSuccess;
  const int warps = 8;
  const size_t sm = (size_t)warps * sizeof(SqWarp);
  cudaError_t e;
  if (sm > 48 * 1024 &&
      (e = cudaFuncSetAttribute(k_outer_symbolic_q4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)) != cudaSuccess)
    return e;
  const unsigned long long rpc = (unsigned long long)warps * SQ_R;
  unsigned long long grid = (nrows + rpc - 1) / rpc;
  grid = std::min<unsigned long long>(grid, 148ull * 64);
  k_outer_symbolic_q4<<<(int)grid, warps * 32, sm, stream>>>(op, rows, nrows, do_send, do_local, local, send, mo,
                                                             status, row0);
  return cudaGetLastError();
}

// C's pattern row by row (one rank, nothing received): C(J,:) is the union of
// the AP rows of the fine rows i with P_d(i,J) != 0 -- a per-row hash set in
// shared memory, one warp per C row, instead of ~13 global-arena inserts per
// entry (SURVEY §8(a) a6/a7 restated row-wise).  FILL = false counts (and
// flags rows whose union does not fit the table), FILL = true writes the
// sorted columns.
constexpr int CU_LOG2T = 9, CU_T = 1 << CU_LOG2T, CU_MAX = 384;

// the contributors' AP entries of C row J, flattened over the warp's lanes
// 32 contributors at a time; f(g, c_base_pm, s) is called for every entry
// (g = column, s = its slot in the contributor's AP row)
template <typename F>
__device__ __forceinline__ void cu_sweep(int64_t J, const int64_t *t_rp, const int32_t *t_row, const int64_t *pat_rp,
                                         const int32_t *pat, const uint8_t *nap, const int64_t *pd_rp,
                                         const int32_t *pd_col, const int64_t *pmap_rp, F f) {
  const int lane = lane_id();
  for (int64_t tb = t_rp[J]; tb < t_rp[J + 1]; tb += 32) {
    const int nc = (int)min((int64_t)32, t_rp[J + 1] - tb);
    int my_n = 0;
    int64_t my_base = 0, my_pm = -1;
    if (lane < nc) {
      const int32_t i = t_row[tb + lane];
      my_base = pat_rp[i];
      my_n = (int)(pat_rp[i + 1] - my_base);  // pattern rows are a CSR (AP rows or C~ rows)
      if (pmap_rp) {  // where row i's positions for target J go: jj-th block of its map
        const int64_t e0 = pd_rp[i], e1 = pd_rp[i + 1];
        int64_t jj = 0;
        for (int64_t e = e0; e < e1; ++e)
          if (pd_col[e] == (int32_t)J) { jj = e - e0; break; }
        my_pm = pmap_rp[i] + jj * my_n;
      }
    }
    int incl = my_n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int tot = __shfl_sync(FULL, incl, 31);
    const int excl = incl - my_n;
    for (int q0 = 0; q0 < tot; q0 += 32) {
      const int q = q0 + lane;
      int c = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int cand = c + step;
        const int ex = __shfl_sync(FULL, excl, cand < 32 ? cand : 31);
        if (cand < nc && ex <= q) c = cand;
      }
      const int64_t base = __shfl_sync(FULL, my_base, c);
      const int64_t pm = __shfl_sync(FULL, my_pm, c);
      const int exc = __shfl_sync(FULL, excl, c);
      if (q < tot) f(__ldg(pat + base + (q - exc)), pm, q - exc);
    }
  }
}

// C's pattern row by row (one rank, nothing received): C(J,:) is the union of
// the AP rows of the fine rows i with P_d(i,J) != 0 -- a per-row hash set in
// shared memory, one warp per C row, instead of ~13 global-arena inserts per
// entry (SURVEY §8(a) a6/a7 restated row-wise).  FILL = false counts (and
// flags rows whose union does not fit the table), FILL = true writes the
// sorted columns and, when pmap is given, the position map of every
// contributor (the byte position of each of its AP slots in C row J).
template <bool FILL>
__global__ void __launch_bounds__(256) k_c_union(int64_t ncl, const int64_t *t_rp, const int32_t *t_row,
                                                 const int64_t *pat_rp, const int32_t *pat, const uint8_t *nap,
                                                 int64_t *cnt, const int64_t *c_rp, int32_t *c_col,
                                                 const int64_t *pd_rp, const int32_t *pd_col,
                                                 const int64_t *pmap_rp, uint8_t *pmap, int *status) {
  // compacted keys need only CU_MAX entries (a longer union fails the row
  // anyway): 38 KB per CTA instead of 44, one more resident CTA per SM
  __shared__ int32_t keys_all[8][CU_T];
  __shared__ int32_t lk_all[8][CU_MAX];
  __shared__ uint16_t lpos_all[8][CU_MAX];
  __shared__ uint8_t rank_all[8][CU_T];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  int32_t *keys = keys_all[warp], *lk = lk_all[warp];
  uint16_t *lpos = lpos_all[warp];
  uint8_t *srank = rank_all[warp];
  for (int64_t J = (int64_t)blockIdx.x * 8 + warp; J < ncl; J += (int64_t)gridDim.x * 8) {
    for (int x = lane; x < CU_T; x += 32) keys[x] = EMPTY32;
    __syncwarp();
    bool full = false;
    cu_sweep(J, t_rp, t_row, pat_rp, pat, nap, nullptr, nullptr, nullptr, [&](int32_t g, int64_t, int) {
      uint32_t h = hash32((uint32_t)g, CU_LOG2T);
      int probe = 0;
      for (; probe < CU_T; ++probe) {
        const int32_t k = keys[h];
        if (k == g) break;
        if (k == EMPTY32) {
          const int32_t old = atomicCAS(keys + h, EMPTY32, g);
          if (old == EMPTY32 || old == g) break;
        }
        h = (h + 1) & (CU_T - 1);
      }
      full |= probe == CU_T;
    });
    __syncwarp();
    // compact
    int n = 0;
    for (int s0 = 0; s0 < CU_T; s0 += 32) {
      const int32_t k = keys[s0 + lane];
      const unsigned b = __ballot_sync(FULL, k != EMPTY32);
      if (k != EMPTY32) {
        const int at = n + __popc(b & ((1u << lane) - 1u));
        if (at < CU_MAX) {
          lk[at] = k;
          lpos[at] = (uint16_t)(s0 + lane);
        }
      }
      n += __popc(b);
    }
    __syncwarp();
    full = __any_sync(FULL, full) || n > CU_MAX;
    if (!FILL) {
      if (lane == 0) {
        cnt[J] = n;
        if (full) atomicOr(status, ST_TABLE_FULL);
      }
    } else {
      int32_t *out = c_col + c_rp[J];
      for (int x = lane; x < n; x += 32) {
        const int32_t g = lk[x];
        int rk = 0;
        for (int y = 0; y < n; ++y) rk += lk[y] < g;
        out[rk] = g;
        srank[lpos[x]] = (uint8_t)rk;
      }
      __syncwarp();
      if (pmap)
        cu_sweep(J, t_rp, t_row, pat_rp, pat, nap, pd_rp, pd_col, pmap_rp, [&](int32_t g, int64_t pm, int sl) {
          uint32_t h = hash32((uint32_t)g, CU_LOG2T);
          for (int probe = 0; probe < CU_T && keys[h] != g; ++probe) h = (h + 1) & (CU_T - 1);
          pmap[pm + sl] = srank[h];
        });
    }
    __syncwarp();
  }
}

cudaError_t launch_c_union(bool fill, int64_t ncl, const int64_t *t_rp, const int32_t *t_row, const int64_t *pat_rp,
                           const int32_t *pat, const uint8_t *nap, int64_t *cnt, const int64_t *c_rp, int32_t *c_col,
                           const int64_t *pd_rp, const int32_t *pd_col, const int64_t *pmap_rp, uint8_t *pmap,
                           int *status, cudaStream_t st) {
  if (ncl <= 0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>((ncl + 7) / 8, 148 * 16);
  if (fill)
    k_c_union<true><<<grid, 256, 0, st>>>(ncl, t_rp, t_row, pat_rp, pat, nap, cnt, c_rp, c_col, pd_rp, pd_col,
                                          pmap_rp, pmap, status);
  else
    k_c_union<false><<<grid, 256, 0, st>>>(ncl, t_rp, t_row, pat_rp, pat, nap, cnt, c_rp, c_col, pd_rp, pd_col,
                                           pmap_rp, pmap, status);
  return cudaGetLastError();
}

// exact table sizes for the two-step P^T C~ rows: the length of the target
// row of the allocated structure (C row, or staging row when present)
__global__ void k_ptc_est(int64_t nrows, const int32_t *target_map, int64_t target_offset, int is_staging,
                          int64_t t_nrows, const int32_t *t_rows, const int64_t *t_rp, int64_t *est) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nrows) return;
  int64_t tgt = target_map ? (int64_t)target_map[q] : q + target_offset;
  int64_t r = tgt;
  if (is_staging) {
    r = lower_bound32(t_rows, 0, t_nrows, (int32_t)tgt);
    if (r >= t_nrows || t_rows[r] != (int32_t)tgt) { est[q] = 0; return; }
  }
  est[q] = t_rp[r + 1] - t_rp[r];
}

// L2 flush: stream through a buffer larger than L2
__global__ void k_touch(int4 *buf, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int4 v = buf[i];
    v.x += 1;
    buf[i] = v;
  }
}

// ---------------------------------------------------------------------------
// explicit instantiations via launch helpers
// ---------------------------------------------------------------------------
static int grid_for(unsigned long long groups, int groups_per_cta, int max_ctas) {
  unsigned long long g = (groups + groups_per_cta - 1) / groups_per_cta;
  if (g > (unsigned long long)max_ctas) g = max_ctas;
  if (g < 1) g = 1;
  return (int)g;
}

template <typename K>
static cudaError_t set_smem(K kern, size_t bytes) {
  if (bytes > 48 * 1024) return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return cudaSuccess;
}

#define PTAP_ROWKERNEL_DISPATCH(KERNEL, NUM, ...)                                                         \
  do {                                                                                                     \
    if (gtables) {                                                                                         \
      KERNEL<32, true><<<max_ctas, warps * 32, 0, stream>>>(__VA_ARGS__);                                  \
    } else if (group == 8) {                                                                               \
      int gpc = warps * 4;                                                                                 \
      size_t sm = group_bytes(log2t, NUM, 8) * gpc;                                                        \
      if ((e = set_smem(KERNEL<8, false>, sm)) != cudaSuccess) return e;                                   \
      KERNEL<8, false><<<grid_for(nrows, gpc, max_ctas), warps * 32, sm, stream>>>(__VA_ARGS__);           \
    } else {                                                                                               \
      int gpc = warps;                                                                                     \
      size_t sm = group_bytes(log2t, NUM, 32) * gpc;                                                       \
      if ((e = set_smem(KERNEL<32, false>, sm)) != cudaSuccess) return e;                                  \
      KERNEL<32, false><<<grid_for(nrows, gpc, max_ctas), warps * 32, sm, stream>>>(__VA_ARGS__);          \
    }                                                                                                      \
    return cudaGetLastError();                                                                             \
  } while (0)

cudaError_t launch_ap_count(const LaunchShape &s, const Ops &op, const int32_t *rows, unsigned long long nrows,
                            int64_t *ap_nnz, int *status, cudaStream_t stream) {
  const int group = s.group, warps = s.warps, log2t = s.log2t, max_ctas = s.max_ctas;
  unsigned char *gtables = s.gtables;
  cudaError_t e;
  PTAP_ROWKERNEL_DISPATCH(k_ap_count, false, op, rows, nrows, log2t, gtables, ap_nnz, status);
}

cudaError_t launch_outer_symbolic(const LaunchShape &s, const Ops &op, const int32_t *rows, unsigned long long nrows,
                                  int do_send, int do_local, Arena local, Arena send, const MapOut &mo, int *status,
                                  cudaStream_t stream) {
  const int group = s.group, warps = s.warps, log2t = s.log2t, max_ctas = s.max_ctas;
  unsigned char *gtables = s.gtables;
  cudaError_t e;
  static const bool g16 = !getenv("PTAP_NO_SYM16");
  if (g16 && s.bin == 1 && !gtables) {
    // AP rows of 33..128 keys (config 4): 16 lanes per row, two rows per warp
    const int gpc = warps * 2;
    const size_t sm = group_bytes(log2t, false, 16) * gpc;
    if ((e = set_smem(k_outer_symbolic<16, false>, sm)) != cudaSuccess) return e;
    k_outer_symbolic<16, false><<<grid_for(nrows, gpc, max_ctas), warps * 32, sm, stream>>>(
        op, rows, nrows, log2t, gtables, do_send, do_local, local, send, mo, status);
    return cudaGetLastError();
  }
  PTAP_ROWKERNEL_DISPATCH(k_outer_symbolic, false, op, rows, nrows, log2t, gtables, do_send, do_local, local, send,
                          mo, status);
}

cudaError_t launch_outer_oneshot(const LaunchShape &s, const Ops &op, const int32_t *rows, unsigned long long nrows,
                                 Arena local, double *avals, int *status, cudaStream_t stream) {
  const int group = s.group, warps = s.warps, log2t = s.log2t, max_ctas = s.max_ctas;
  unsigned char *gtables = s.gtables;
  cudaError_t e;
  PTAP_ROWKERNEL_DISPATCH(k_outer_oneshot, true, op, rows, nrows, log2t, gtables, local, avals, status);
}

cudaError_t launch_outer_numeric(const LaunchShape &s, const Ops &op, const int32_t *rows, unsigned long long nrows,
                                 int do_send, int do_local, const OuterTargets &tg, int *status,
                                 cudaStream_t stream) {
  const int group = s.group, warps = s.warps, log2t = s.log2t, max_ctas = s.max_ctas;
  unsigned char *gtables = s.gtables;
  cudaError_t e;
  PTAP_ROWKERNEL_DISPATCH(k_outer_numeric, true, op, rows, nrows, log2t, gtables, do_send, do_local, tg, status);
}

cudaError_t launch_ct_fill(const LaunchShape &s, const Ops &op, const int32_t *rows, unsigned long long nrows,
                           const int64_t *ct_rp, int32_t *ct_col, int *status, cudaStream_t stream) {
  const int group = s.group, warps = s.warps, log2t = s.log2t, max_ctas = s.max_ctas;
  unsigned char *gtables = s.gtables;
  cudaError_t e;
  PTAP_ROWKERNEL_DISPATCH(k_ct_fill, false, op, rows, nrows, log2t, gtables, ct_rp, ct_col, status);
}

cudaError_t launch_ct_numeric(const LaunchShape &s, const Ops &op, const int32_t *rows, unsigned long long nrows,
                              const int64_t *ct_rp, const int32_t *ct_col, double *ct_val, int *status,
                              cudaStream_t stream) {
  const int group = s.group, warps = s.warps, log2t = s.log2t, max_ctas = s.max_ctas;
  unsigned char *gtables = s.gtables;
  cudaError_t e;
  PTAP_ROWKERNEL_DISPATCH(k_ct_numeric, true, op, rows, nrows, log2t, gtables, ct_rp, ct_col, ct_val, status);
}

cudaError_t launch_ptc_numeric(const LaunchShape &s, const int32_t *rows, unsigned long long nrows,
                               const int64_t *t_rp, const int32_t *t_row, const double *t_val,
                               const int32_t *target_map, int64_t target_offset, const int64_t *ct_rp,
                               const int32_t *ct_col, const double *ct_val, const PtcTarget &tg, int *status,
                               cudaStream_t stream) {
  const int group = s.group, warps = s.warps, log2t = s.log2t, max_ctas = s.max_ctas;
  unsigned char *gtables = s.gtables;
  cudaError_t e;
  PTAP_ROWKERNEL_DISPATCH(k_ptc_numeric, true, rows, nrows, log2t, gtables, t_rp, t_row, t_val, target_map,
                          target_offset, ct_rp, ct_col, ct_val, tg, status);
}

size_t row_kernel_group_bytes(int log2t, bool num, int group) { return group_bytes(log2t, num, group); }

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t > 0 ? (n + t - 1) / t : 1); }

cudaError_t launch_row_work(const Ops &op, int64_t *apub, unsigned long long *mac, cudaStream_t st) {
  if (op.nloc > 0) k_row_work<<<nblk(op.nloc, 256), 256, 0, st>>>(op, apub, mac);
  return cudaGetLastError();
}

cudaError_t launch_bin_rows(int64_t nrows, const int64_t *est, const int64_t *pd_rp, const int64_t *po_rp, int mode,
                            const BinLists &bl, unsigned long long *selected, cudaStream_t st) {
  if (nrows > 0) k_bin_rows<<<nblk(nrows, 256), 256, 0, st>>>(nrows, est, pd_rp, po_rp, mode, bl, selected);
  return cudaGetLastError();
}

cudaError_t launch_max_est(const int32_t *rows, unsigned long long nrows, const int64_t *est, unsigned long long *mx,
                           cudaStream_t st) {
  if (nrows > 0) k_max_est<<<nblk((int64_t)nrows, 256), 256, 0, st>>>(rows, nrows, est, mx);
  return cudaGetLastError();
}

cudaError_t launch_arena_fill_empty(Arena ar, cudaStream_t st) {
  unsigned long long cap = ar.mask + 1;
  k_arena_fill_empty<<<nblk((int64_t)cap, 256), 256, 0, st>>>(ar.keys, cap);
  return cudaGetLastError();
}

cudaError_t launch_arena_insert_batch(Arena ar, int64_t nrows, const int32_t *rows, const int64_t *rp,
                                      const int32_t *col, int64_t m, int64_t c_lo, int64_t c_hi, int *status,
                                      cudaStream_t st) {
  if (nrows > 0) k_arena_insert_batch<<<nblk(nrows * 32, 256), 256, 0, st>>>(ar, nrows, rows, rp, col, m, c_lo, c_hi, status);
  return cudaGetLastError();
}

cudaError_t launch_arena_rowcount(Arena ar, int64_t m, int64_t *cnt, cudaStream_t st) {
  unsigned long long cap = ar.mask + 1;
  k_arena_rowcount<<<nblk((int64_t)cap, 256), 256, 0, st>>>(ar, (unsigned long long)m, cnt);
  return cudaGetLastError();
}

cudaError_t launch_arena_scatter(Arena ar, int64_t m, const int64_t *rp, int64_t *cursor, int32_t *col,
                                 cudaStream_t st) {
  unsigned long long cap = ar.mask + 1;
  k_arena_scatter<<<nblk((int64_t)cap, 256), 256, 0, st>>>(ar, (unsigned long long)m, rp, cursor, col);
  return cudaGetLastError();
}

cudaError_t launch_arena_scatter_vals(Arena ar, int64_t m, const int64_t *rp, int64_t *cursor, int32_t *col,
                                      const double *avals, int64_t *payload, cudaStream_t st) {
  unsigned long long cap = ar.mask + 1;
  k_arena_scatter_vals<<<nblk((int64_t)cap, 256), 256, 0, st>>>(ar, (unsigned long long)m, rp, cursor, col, avals,
                                                                payload);
  return cudaGetLastError();
}

cudaError_t launch_sort_rows(int64_t nrows, const int64_t *rp, int32_t *keys, int64_t *payload, int32_t *wide_rows,
                             unsigned long long *nwide, cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  const int warps = 8;
  int grid = (int)((nrows + warps - 1) / warps);
  if (grid > 148 * 16) grid = 148 * 16;
  cudaError_t e;
  if (payload) {
    size_t sm = (size_t)warps * 1024 * 12;
    if ((e = set_smem(k_sort_rows<true>, sm)) != cudaSuccess) return e;
    k_sort_rows<true><<<grid, warps * 32, sm, st>>>(nrows, rp, keys, payload, wide_rows, nwide);
  } else {
    size_t sm = (size_t)warps * 1024 * 4;
    k_sort_rows<false><<<grid, warps * 32, sm, st>>>(nrows, rp, keys, payload, wide_rows, nwide);
  }
  return cudaGetLastError();
}

cudaError_t launch_sort_rows_block(int64_t nwide, const int32_t *rows, const int64_t *rp, int32_t *keys,
                                   int64_t *payload, int *status, cudaStream_t st) {
  if (nwide <= 0) return cudaSuccess;
  cudaError_t e;
  size_t sm = 8192 * 4 + (payload ? 8192 * 8 : 0);
  if (payload) {
    if ((e = set_smem(k_sort_rows_block<true>, sm)) != cudaSuccess) return e;
    k_sort_rows_block<true><<<(int)nwide, 1024, sm, st>>>(rows, rp, keys, payload, status);
  } else {
    if ((e = set_smem(k_sort_rows_block<false>, sm)) != cudaSuccess) return e;
    k_sort_rows_block<false><<<(int)nwide, 1024, sm, st>>>(rows, rp, keys, payload, status);
  }
  return cudaGetLastError();
}

cudaError_t launch_merge_slots(int64_t nrows, const int32_t *rows, const int64_t *rp, const int32_t *col, int64_t c_lo,
                               const int64_t *c_rp, const int32_t *c_col, int64_t *slot, int *status,
                               cudaStream_t st) {
  if (nrows > 0) k_merge_slots<<<nblk(nrows * 32, 256), 256, 0, st>>>(nrows, rows, rp, col, c_lo, c_rp, c_col, slot, status);
  return cudaGetLastError();
}

// values-only refresh of the gathered P rows, owner side (reference
// update_remote_rows_numeric with its gather_idx, src/comm.py:590-594,
// 625-649): out[t] = value idx[t] of the concatenation [P_d.val, P_o.val],
// read in place (no concatenated copy); an index past the structure sets
// ST_DRIFT (the structure changed since the symbolic gather)
__global__ void k_pack_values(const double *d_val, int64_t nd, const double *o_val, int64_t no, const int64_t *idx,
                              int64_t n, double *out, int *status) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = idx[t];
    double v = 0.0;
    if (x >= 0 && x < nd) v = d_val[x];
    else if (x >= nd && x < nd + no) v = o_val[x - nd];
    else atomicOr(status, ST_DRIFT);
    out[t] = v;
  }
}
cudaError_t launch_pack_values(const double *d_val, int64_t nd, const double *o_val, int64_t no, const int64_t *idx,
                               int64_t n, double *out, int *status, cudaStream_t st) {
  if (n > 0) k_pack_values<<<nblk(n, 256), 256, 0, st>>>(d_val, nd, o_val, no, idx, n, out, status);
  return cudaGetLastError();
}

cudaError_t launch_merge_add(int64_t n, const int64_t *slot, const double *vals, double *c_val, cudaStream_t st) {
  if (n > 0) k_merge_add<<<nblk(n, 256), 256, 0, st>>>(n, slot, vals, c_val);
  return cudaGetLastError();
}

cudaError_t launch_count_cols(int64_t nnz, const int32_t *col, int64_t *cnt, cudaStream_t st) {
  if (nnz > 0) k_count_cols<<<nblk(nnz, 256), 256, 0, st>>>(nnz, col, cnt);
  return cudaGetLastError();
}

cudaError_t launch_transpose_scatter(int64_t nrows, const int64_t *rp, const int32_t *col, const int64_t *t_rp,
                                     int64_t *cursor, int32_t *t_row, int64_t *t_perm, cudaStream_t st) {
  if (nrows > 0) k_transpose_scatter<<<nblk(nrows, 256), 256, 0, st>>>(nrows, rp, col, t_rp, cursor, t_row, t_perm);
  return cudaGetLastError();
}

cudaError_t launch_gather(int64_t n, const int64_t *perm, const double *src, double *dst, cudaStream_t st) {
  if (n > 0) k_gather<<<nblk(n, 256), 256, 0, st>>>(n, perm, src, dst);
  return cudaGetLastError();
}

cudaError_t launch_ptc_symbolic(int64_t nrows, const int64_t *t_rp, const int32_t *t_row, const int32_t *target_map,
                                int64_t target_offset, const int64_t *ct_rp, const int32_t *ct_col, Arena ar,
                                int64_t m, int *status, cudaStream_t st) {
  if (nrows > 0)
    k_ptc_symbolic<<<nblk(nrows * 32, 256), 256, 0, st>>>(nrows, t_rp, t_row, target_map, target_offset, ct_rp,
                                                          ct_col, ar, (unsigned long long)m, status);
  return cudaGetLastError();
}

cudaError_t scan_exclusive(const int64_t *in, int64_t *out, int64_t n, int64_t *scratch, cudaStream_t st) {
  // out has n+1 entries; scratch must hold scan_scratch_elems(n) int64
  if (n <= 0) {
    cudaMemsetAsync(out, 0, sizeof(int64_t), st);
    return cudaGetLastError();
  }
  int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  int64_t *tile_sums = scratch;
  int64_t *tile_off = scratch + tiles;
  k_scan_tiles<<<(int)tiles, SCAN_THREADS, 0, st>>>(in, out, n, tile_sums);
  if (tiles > 1) {
    cudaError_t e = scan_exclusive(tile_sums, tile_off, tiles, scratch + 2 * tiles + 1, st);
    if (e != cudaSuccess) return e;
    k_scan_add<<<nblk(n, 256), 256, 0, st>>>(out, n, tile_off);
  }
  k_set_total<<<1, 1, 0, st>>>(out, n, in);
  return cudaGetLastError();
}

int64_t scan_scratch_elems(int64_t n) {
  int64_t tot = 0;
  while (n > 1) {
    int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    tot += 2 * tiles + 1;
    n = tiles;
  }
  return tot + 4;
}

cudaError_t launch_nonzero_flags(int64_t n, const int64_t *cnt, int64_t *flags, cudaStream_t st) {
  if (n > 0) k_nonzero_flags<<<nblk(n, 256), 256, 0, st>>>(n, cnt, flags);
  return cudaGetLastError();
}

cudaError_t launch_compact_rows(int64_t n, const int64_t *cnt, const int64_t *pos, const int64_t *dense_rp,
                                int32_t *rows, int64_t *rp, cudaStream_t st) {
  if (n > 0) k_compact_rows<<<nblk(n, 256), 256, 0, st>>>(n, cnt, pos, dense_rp, rows, rp);
  return cudaGetLastError();
}

cudaError_t launch_iota32(int32_t *p, int64_t n, cudaStream_t st) {
  if (n > 0) k_iota32<<<nblk(n, 256), 256, 0, st>>>(p, n);
  return cudaGetLastError();
}

cudaError_t launch_row_lengths(int64_t n, const int64_t *rp, int64_t *len, cudaStream_t st) {
  if (n > 0) k_row_lengths<<<nblk(n, 256), 256, 0, st>>>(n, rp, len);
  return cudaGetLastError();
}

cudaError_t launch_outer_bounds(int64_t n, const int64_t *pd_rp, const int64_t *po_rp, const int64_t *ap_nnz,
                                unsigned long long *out, cudaStream_t st) {
  if (n > 0) k_outer_bounds<<<nblk(n, 256), 256, 0, st>>>(n, pd_rp, po_rp, ap_nnz, out);
  return cudaGetLastError();
}

cudaError_t launch_arena_rehash(Arena from, Arena to, int *status, cudaStream_t st) {
  unsigned long long cap = from.mask + 1;
  k_arena_rehash<<<nblk((int64_t)cap, 256), 256, 0, st>>>(from, to, status);
  return cudaGetLastError();
}

cudaError_t launch_ptc_est(int64_t nrows, const int32_t *target_map, int64_t target_offset, int is_staging,
                           int64_t t_nrows, const int32_t *t_rows, const int64_t *t_rp, int64_t *est,
                           cudaStream_t st) {
  if (nrows > 0)
    k_ptc_est<<<nblk(nrows, 256), 256, 0, st>>>(nrows, target_map, target_offset, is_staging, t_nrows, t_rows, t_rp, est);
  return cudaGetLastError();
}

cudaError_t launch_build_pmap(const Ops &op, unsigned long long nrows, const MapArgs &mp, const MapOut &mo,
                              const OuterTargets &tg, int *status, cudaStream_t st, int64_t row0) {
  if (nrows == 0) return cudaSuccess;
  unsigned long long grid = (nrows + 31) / 32;
  if (grid > 148ull * 64) grid = 148ull * 64;
  k_build_pmap<<<(int)grid, 256, 0, st>>>(op, nrows, mp, mo, tg, status, row0);
  return cudaGetLastError();
}

// order-independent digest of an index array (position-sensitive): sum of
// mix(salt, i, v) over the entries, wrapping
__device__ __forceinline__ unsigned long long dg_mix(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
template <typename T>
__global__ void k_digest(const T *a, int64_t n, unsigned long long salt, unsigned long long *out) {
  unsigned long long h = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    h += dg_mix((salt << 58) ^ ((unsigned long long)i << 24) ^ dg_mix((unsigned long long)(long long)a[i]));
  for (int o = 16; o; o >>= 1) h += __shfl_xor_sync(FULL, h, o);
  if ((threadIdx.x & 31) == 0 && h) atomicAdd(out, h);
}
cudaError_t launch_digest_i64(const int64_t *a, int64_t n, unsigned long long salt, unsigned long long *out,
                              cudaStream_t st) {
  if (n > 0 && a) k_digest<int64_t><<<148 * 8, 256, 0, st>>>(a, n, salt, out);
  return cudaGetLastError();
}
cudaError_t launch_digest_i32(const int32_t *a, int64_t n, unsigned long long salt, unsigned long long *out,
                              cudaStream_t st) {
  if (n > 0 && a) k_digest<int32_t><<<148 * 8, 256, 0, st>>>(a, n, salt, out);
  return cudaGetLastError();
}

cudaError_t launch_touch(void *buf, int64_t bytes, cudaStream_t st) {
  int64_t n = bytes / 16;
  k_touch<<<148 * 8, 256, 0, st>>>((int4 *)buf, n);
  return cudaGetLastError();
}

}  // namespace ptapdev
