// ptap_capi.cu -- extern "C" entry points (include/ptap_b200.h) and the
// device-resident TripleProductPlan.
//
// The plan owns every device buffer it allocates (cudaMallocAsync on the
// caller's stream) and books each under one of the reference's ledger
// categories (src/ledger.py:23-34):
//   output_matrix        C (row offsets, columns, values)
//   auxiliary_matrices   two-step only: C~ = A P, the transposes of P, its staging
//   transient_hash_peak  arenas, work estimates, count arrays (freed by the end of symbolic)
//   plan_cache           bin row lists, all-at-once staging, received-slot map, transpose permutations
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/ptap_b200.h"
#include "ptap_kernels.cuh"

using namespace ptapdev;

namespace {

thread_local std::string g_err;

ptap_status fail(ptap_status s, const std::string &msg) {
  g_err = msg;
  return s;
}

enum Cat { CAT_INPUT = 0, CAT_OUTPUT = 1, CAT_AUX = 2, CAT_TRANSIENT = 3, CAT_PLAN = 4 };

cudaMemPool_t lib_pool();

// PTAP_TRACE=1: synchronise and print the wall time of each symbolic step
struct Tracer {
  bool on = getenv("PTAP_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(cudaStream_t st, const char *what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    auto t1 = std::chrono::steady_clock::now();
    unsigned long long reserved = 0, used = 0;
    cudaMemPool_t pool = lib_pool();
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    fprintf(stderr, "[ptap] %-28s %9.3f ms   pool reserved %.2f GB used %.2f GB\n", what,
            std::chrono::duration<double, std::milli>(t1 - t0).count(), reserved / 1e9, used / 1e9);
    t0 = t1;
  }
};

#define CK(x)                                                                                            \
  do {                                                                                                   \
    cudaError_t _e = (x);                                                                                \
    if (_e != cudaSuccess)                                                                               \
      return fail(_e == cudaErrorMemoryAllocation ? PTAP_ERR_OOM : PTAP_ERR_CUDA,                        \
                  std::string(#x) + ": " + cudaGetErrorString(_e));                                      \
  } while (0)

#define CKS(x)                                   \
  do {                                                 \
    ptap_status _s = (x);                              \
    if (_s != PTAP_OK) return _s;                      \
  } while (0)

struct Alloc {
  size_t bytes;
  int cat;
};

struct BinSet {
  int32_t *rows[NBINS] = {nullptr, nullptr, nullptr, nullptr};
  int64_t count[NBINS] = {0, 0, 0, 0};
  int log2t_global = 0;             // table size of the global-memory bin
  unsigned char *gtables = nullptr; // global tables for the heavy bin
  int64_t selected = 0;             // rows selected (reference row-kernel calls)
  bool identity0 = false;           // bin 0 holds every row in order (rows[0] == nullptr)
};

struct Transpose {
  int64_t nrows = 0, nnz = 0;
  int64_t *rp = nullptr;
  int32_t *row = nullptr;
  int64_t *perm = nullptr;
  double *val = nullptr;
};

}  // namespace

struct ptap_plan {
  int alg = 0;
  int64_t nloc = 0, m = 0, c_lo = 0, c_hi = 0, ncl = 0, colmap_len = 0;
  std::map<void *, Alloc> allocs;
  int64_t cur[5] = {0, 0, 0, 0, 0}, peak[5] = {0, 0, 0, 0, 0};
  int64_t prod_cur = 0, prod_peak = 0, total_cur = 0, total_peak = 0;
  int *d_status = nullptr;
  int *h_status = nullptr;          // pinned: status of the last pass, copied asynchronously
  cudaEvent_t status_ev = nullptr;
  bool status_pending = false;
  bool status_graph = false;        // a pass captured into a CUDA graph writes h_status on replay
  unsigned long long *d_u64 = nullptr;  // 24 scratch counters
  bool released = false;
  bool symbolic_done = false;
  BinSet bins_send, bins_local, bins_all, bins_ptd, bins_pto;
  // transient state carried from symbolic_send to symbolic_local
  int64_t *ap_nnz = nullptr;
  int64_t *apub = nullptr;
  Arena local_arena{nullptr, 0};
  // plan-mapped numeric (all-at-once / merged)
  bool mapped = false;
  bool q4 = false;                  // bin 0 runs k_outer_numeric_q4
  bool q4_sym = false;              // ... and k_outer_symbolic_q4
  bool pmap_ready = false;          // position maps written by the row-union pass
  bool smap_interned = false;       // slot maps already interned (row-union path)
  bool rows_unstructured = false;   // sampled row structures do not repeat
  bool q4a = false;                 // identity bin 0 runs k_outer_numeric_q4a
  bool tile = false;                // ... and the deterministic owner-computes kernel replaces it
  bool deterministic = false;       // plan option: bitwise-repeatable numeric passes (tile kernel)
  int maps_opt = -1;                // plan option: -1 row-sample policy, 0 no plan maps (hash path), 1 keep maps
  // symbolic-time image of the operands' structure (drift detection)
  int64_t img_shape[11] = {0};
  const void *img_ptr[11] = {nullptr};
  unsigned long long img_digest = 0;
  TileArgs ta{};
  LockArgs la{};
  bool lock = false;                // class-lockstep numeric kernel (ptap_lock.cu) replaces q4a
  int lock_opt = -1;                // plan option "lockstep": -1 when eligible, 0 never, 1 same as -1
  int lock_classes = 0;
  bool single_shot = false;         // plan option: symbolic_local also computes C's values (one pass over A)
  bool values_ready = false;        // ... and did: C holds the product of the symbolic-time operands
  int64_t max_nap = 0;              // widest AP row
  int64_t qmap_bytes = 0;           // tile gather maps (interned)
  bool smap_deferred = false;       // slot-map buffer not allocated yet (chunked or allocated on first use)
  bool pmap_interned = false;       // position maps built and interned chunk by chunk
  std::vector<std::pair<int64_t, int64_t>> qa_runs;  // several ranks: runs of rows without A_o/P_o (q4a)
  int32_t *qa_rest = nullptr;       // ... and the other bin-0 rows (q4)
  int64_t qa_rest_n = 0;
  bool merged_deferred = false;     // merged plan without send rows: local structure built in symbolic_local
  double avg_p_row = 4.0;           // P entries per local fine row (arena sizing)
  bool want_maps = false;
  MapArgs maps{};
  MapOut mo{};           // symbolic map outputs (smap, nap) + transient sorted patterns
  int64_t *pat_rp = nullptr;
  int32_t *pat = nullptr;
  int64_t smap_bytes = 0, pmap_bytes = 0;
  unsigned long long bound_local = 0, bound_send = 0, sum_ap = 0;
  // C
  int64_t c_nnz = 0;
  int64_t *c_rp = nullptr;
  int32_t *c_col = nullptr;
  double *c_val = nullptr;
  // staging
  int64_t s_nrows = 0, s_nnz = 0;
  int32_t *s_rows = nullptr;
  int64_t *s_rp = nullptr;
  int32_t *s_col = nullptr;
  double *s_val = nullptr;
  // received merge map
  int64_t r_nnz = 0;
  int64_t *r_slot = nullptr;
  std::vector<int64_t> r_src_nnz_off;
  // two-step
  int64_t ct_nnz = 0;
  int64_t *ct_rp = nullptr;
  int32_t *ct_col = nullptr;
  double *ct_val = nullptr;
  Transpose ptd, pto;
  ptap_counters cnt{0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, -1};
};

namespace {

// The library's own stream-ordered pool (not the device default pool, which
// torch and NCCL may use): freed plan memory is kept for the next symbolic
// phase, and release_cache / plan destroy trim it back to the driver.
// PTAP_POOL_RESERVE_GB maps a block up front (opt-in).
cudaMemPool_t lib_pool() {
  static cudaMemPool_t pool = nullptr;
  static int pool_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (pool && pool_dev == dev) return pool;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
    cudaGetLastError();
    cudaDeviceGetDefaultMemPool(&pool, dev);
  }
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  pool_dev = dev;
  const char *rv = getenv("PTAP_POOL_RESERVE_GB");
  const double gb = rv ? atof(rv) : 0.0;
  if (gb > 0) {
    void *ptr = nullptr;
    if (cudaMallocFromPoolAsync(&ptr, (size_t)(gb * 1073741824.0), pool, 0) == cudaSuccess) {
      cudaFreeAsync(ptr, 0);
      cudaStreamSynchronize(0);
    }
    cudaGetLastError();
  }
  return pool;
}

void trim_pool() {
  cudaMemPoolTrimTo(lib_pool(), 0);
}

int g_live_plans = 0;

// Map the pool's memory up front for a plan of this size (about the
// symbolic phase's peak: 10 B per nonzero of A and P), so the large
// transient buffers of every symbolic phase come out of memory the pool
// already holds instead of new driver mappings (measured: warm symbolic
// phases of config 3 at 44 ms with outliers of 131 and 217 ms while the pool
// grew).  PTAP_POOL_RESERVE_GB overrides the size (0: off).  The pool is the
// library's own; the memory goes back when the last plan is destroyed.
void reserve_pool(const ptap_operands *o) {
  double want = 10.0 * (double)(o->a_diag.nnz + o->a_off.nnz + o->p_diag.nnz + o->p_off.nnz + o->p_remote.nnz);
  if (const char *rv = getenv("PTAP_POOL_RESERVE_GB")) want = atof(rv) * 1073741824.0;
  if (want < (double)(256 << 20)) return;
  cudaMemPool_t pool = lib_pool();
  unsigned long long reserved = 0;
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
  if ((double)reserved >= want) return;
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) { cudaGetLastError(); return; }
  const double cap = 0.5 * (double)fr;  // never more than half of what is free
  if (want > cap) want = cap;
  if ((double)reserved >= want) return;
  void *ptr = nullptr;
  if (cudaMallocFromPoolAsync(&ptr, (size_t)want, pool, 0) == cudaSuccess) {
    cudaFreeAsync(ptr, 0);
    cudaStreamSynchronize(0);
  }
  cudaGetLastError();
}

ptap_status palloc_raw(ptap_plan *p, void **out, size_t bytes, int cat, cudaStream_t st) {
  if (bytes == 0) bytes = 16;
  bytes = (bytes + 255) & ~size_t(255);
  void *ptr = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync(&ptr, bytes, lib_pool(), st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? PTAP_ERR_OOM : PTAP_ERR_CUDA,
                std::string("cudaMallocAsync(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  }
  p->allocs[ptr] = Alloc{bytes, cat};
  p->cur[cat] += bytes;
  if (p->cur[cat] > p->peak[cat]) p->peak[cat] = p->cur[cat];
  if (cat != CAT_INPUT) {
    p->prod_cur += bytes;
    if (p->prod_cur > p->prod_peak) p->prod_peak = p->prod_cur;
  }
  p->total_cur += bytes;
  if (p->total_cur > p->total_peak) p->total_peak = p->total_cur;
  *out = ptr;
  return PTAP_OK;
}

template <typename T>
ptap_status palloc(ptap_plan *p, T **out, int64_t count, int cat, cudaStream_t st) {
  void *v = nullptr;
  ptap_status s = palloc_raw(p, &v, (size_t)(count > 0 ? count : 1) * sizeof(T), cat, st);
  *out = (T *)v;
  return s;
}

template <typename T>
void pfree(ptap_plan *p, T *&ptr, cudaStream_t st) {
  if (!ptr) return;
  auto it = p->allocs.find((void *)ptr);
  if (it != p->allocs.end()) {
    p->cur[it->second.cat] -= it->second.bytes;
    if (it->second.cat != CAT_INPUT) p->prod_cur -= it->second.bytes;
    p->total_cur -= it->second.bytes;
    p->allocs.erase(it);
  }
  cudaFreeAsync((void *)ptr, st);
  ptr = nullptr;
}

Ops make_ops(const ptap_operands *o) {
  Ops op;
  op.nloc = o->n_local; op.m = o->m_global; op.c_lo = o->c_lo; op.c_hi = o->c_hi;
  op.ad_rp = o->a_diag.row_ptr; op.ad_col = o->a_diag.col; op.ad_val = o->a_diag.val;
  op.ao_rp = o->a_off.nnz > 0 ? o->a_off.row_ptr : nullptr; op.ao_col = o->a_off.col; op.ao_val = o->a_off.val;
  op.pd_rp = o->p_diag.row_ptr; op.pd_col = o->p_diag.col; op.pd_val = o->p_diag.val;
  op.po_rp = o->p_off.nnz > 0 ? o->p_off.row_ptr : nullptr; op.po_col = o->p_off.col; op.po_val = o->p_off.val;
  op.p_colmap = o->p_colmap;
  op.pr_rp = o->p_remote.row_ptr; op.pr_col = o->p_remote.col; op.pr_val = o->p_remote.val;
  return op;
}

ptap_status validate(const ptap_operands *o) {
  if (!o) return fail(PTAP_ERR_VALUE, "null operands");
  if (o->a_diag.nrows != o->n_local || o->p_diag.nrows != o->n_local)
    return fail(PTAP_ERR_PARTITION, "A and P must share the rank's row block");
  if (o->a_diag.ncols != o->n_local)
    return fail(PTAP_ERR_PARTITION, "the column partition of A must equal the row partition of P");
  if (o->c_lo < 0 || o->c_hi < o->c_lo || o->c_hi > o->m_global || o->p_diag.ncols != o->c_hi - o->c_lo)
    return fail(PTAP_ERR_PARTITION, "P's diagonal block does not match the owned coarse range");
  if (o->m_global > 0 && (double)o->m_global * (double)o->m_global >= 4.611686018427388e18)
    return fail(PTAP_ERR_PARTITION, "output dimension too large for combined row/col keys");
  if (o->m_global >= (int64_t)INT32_MAX) return fail(PTAP_ERR_VALUE, "coarse dimension exceeds int32 columns");
  if (o->a_off.nnz > 0 && (o->a_off.nrows != o->n_local || o->a_off.ncols != o->p_remote.nrows))
    return fail(PTAP_ERR_DRIFT, "gathered rows do not match A's off-diagonal columns");
  if (o->p_off.nnz > 0 && (o->p_off.nrows != o->n_local || o->p_off.ncols != o->p_colmap_len))
    return fail(PTAP_ERR_PARTITION, "P's off-diagonal block does not match its column map");
  return PTAP_OK;
}

void op_shape(const ptap_operands *o, int64_t *sh, const void **pt) {
  const int64_t v[11] = {o->n_local, o->m_global, o->c_lo, o->c_hi, o->a_diag.nnz, o->a_off.nnz, o->p_diag.nnz,
                         o->p_off.nnz, o->p_colmap_len, o->p_remote.nrows, o->p_remote.nnz};
  for (int k = 0; k < 11; ++k) sh[k] = v[k];
  const void *q[11] = {o->a_diag.row_ptr, o->a_diag.col, o->a_off.row_ptr, o->a_off.col, o->p_diag.row_ptr,
                       o->p_diag.col, o->p_off.row_ptr, o->p_off.col, o->p_colmap, o->p_remote.row_ptr,
                       o->p_remote.col};
  if (pt)
    for (int k = 0; k < 11; ++k) pt[k] = q[k];
}

// digest of every structure array of the operands (row offsets, columns,
// column map): one pass over 1.9 GB on config 3 level 1, synchronous
ptap_status op_digest(ptap_plan *p, const ptap_operands *o, cudaStream_t st, unsigned long long *out) {
  unsigned long long *d = p->d_u64 + 23;
  CK(cudaMemsetAsync(d, 0, sizeof(unsigned long long), st));
  const ptap_csr *blocks[5] = {&o->a_diag, &o->a_off, &o->p_diag, &o->p_off, &o->p_remote};
  for (int k = 0; k < 5; ++k) {
    const ptap_csr &c = *blocks[k];
    if (c.nnz > 0) {
      CK(launch_digest_i64(c.row_ptr, c.nrows + 1, 2 * k + 1, d, st));
      CK(launch_digest_i32(c.col, c.nnz, 2 * k + 2, d, st));
    }
  }
  if (o->p_colmap_len > 0) CK(launch_digest_i32(o->p_colmap, o->p_colmap_len, 11, d, st));
  CK(cudaMemcpyAsync(out, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return PTAP_OK;
}

ptap_status record_image(ptap_plan *p, const ptap_operands *o, cudaStream_t st) {
  op_shape(o, p->img_shape, p->img_ptr);
  return op_digest(p, o, st, &p->img_digest);
}

// every numeric call: the operands' shape must be the symbolic one (the
// kernels trust the plan's maps); when the structure arrays were swapped
// for other buffers, their contents must digest to the symbolic image
// (reference: CRC32 structure token, src/comm.py:517-524, and the fill
// checks of src/spgemm.py:54-68)
ptap_status check_image(ptap_plan *p, const ptap_operands *o, cudaStream_t st) {
  int64_t sh[11];
  const void *pt[11];
  op_shape(o, sh, pt);
  for (int k = 0; k < 11; ++k)
    if (sh[k] != p->img_shape[k])
      return fail(PTAP_ERR_DRIFT, "operand structure changed since the symbolic phase (sizes differ)");
  bool same = true;
  for (int k = 0; k < 11; ++k) same = same && pt[k] == p->img_ptr[k];
  if (same) return PTAP_OK;
  unsigned long long dg = 0;
  CKS(op_digest(p, o, st, &dg));
  if (dg != p->img_digest) return fail(PTAP_ERR_DRIFT, "operand structure changed since the symbolic phase");
  for (int k = 0; k < 11; ++k) p->img_ptr[k] = pt[k];
  return PTAP_OK;
}

ptap_status read_status(ptap_plan *p, cudaStream_t st, int *out) {
  CK(cudaStreamSynchronize(st));
  CK(cudaMemcpy(out, p->d_status, sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemset(p->d_status, 0, sizeof(int)));
  return PTAP_OK;
}

ptap_status status_to_error(int s, const char *where) {
  if (s & ST_ROW_TOO_WIDE) return fail(PTAP_ERR_VALUE, std::string(where) + ": a row exceeds 8192 entries");
  if (s & ST_DRIFT)
    return fail(PTAP_ERR_DRIFT, std::string(where) + ": numeric data does not match the symbolic structure");
  if (s & ST_TABLE_FULL) return fail(PTAP_ERR_DRIFT, std::string(where) + ": a row outgrew its symbolic size");
  return PTAP_OK;
}

int ceil_log2(unsigned long long v) {
  int l = 0;
  while ((1ull << l) < v) ++l;
  return l;
}

// ---- bins -------------------------------------------------------------------
LaunchShape shape_for(int q, const BinSet &bs) {
  LaunchShape s{};
  s.bin = q;
  s.gtables = nullptr;
  s.max_ctas = 148 * 64;
  switch (q) {
    case 0: s.group = 8; s.warps = 8; s.log2t = 6; break;   // <= 32 keys
    case 1: s.group = 8; s.warps = 8; s.log2t = 8; break;   // <= 128 keys
    case 2: s.group = 32; s.warps = 2; s.log2t = 11; break; // <= 1024 keys
    default:
      s.group = 32; s.warps = 4; s.log2t = bs.log2t_global; s.max_ctas = 148 * 2; s.gtables = bs.gtables;
  }
  return s;
}

void free_bins(ptap_plan *p, BinSet &bs, cudaStream_t st) {
  for (int q = 0; q < NBINS; ++q) pfree(p, bs.rows[q], st);
  pfree(p, bs.gtables, st);
  bs = BinSet{};
}

// mode: 0 all rows, 1 rows with P_o, 2 rows with P_d, 3 either
ptap_status build_bins(ptap_plan *p, BinSet &bs, int64_t nrows, const int64_t *est, const int64_t *pd_rp,
                       const int64_t *po_rp, int mode, bool num, int cat, cudaStream_t st) {
  bs = BinSet{};
  unsigned long long *cnt = p->d_u64;  // [0..3] counts, [4] selected
  CK(cudaMemsetAsync(cnt, 0, 8 * sizeof(unsigned long long), st));
  BinLists bl{};
  bl.count = cnt;
  CK(launch_bin_rows(nrows, est, pd_rp, po_rp, mode, bl, cnt + 4, st));
  p->cnt.kernel_launches++;
  unsigned long long h[8];
  CK(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  bs.selected = (int64_t)h[4];
  // every row selected and in bin 0: the bin is the identity list
  bool identity = (int64_t)h[0] == nrows;
  if (identity) {
    bs.identity0 = true;
    bs.count[0] = nrows;
  } else {
    for (int q = 0; q < NBINS; ++q) {
      bs.count[q] = (int64_t)h[q];
      if (h[q]) CKS(palloc(p, &bs.rows[q], (int64_t)h[q], cat, st));
    }
    CK(cudaMemsetAsync(cnt, 0, 8 * sizeof(unsigned long long), st));
    for (int q = 0; q < NBINS; ++q) bl.rows[q] = bs.rows[q];
    CK(launch_bin_rows(nrows, est, pd_rp, po_rp, mode, bl, cnt + 4, st));
    p->cnt.kernel_launches++;
  }
  if (bs.count[NBINS - 1] > 0) {
    CK(cudaMemsetAsync(cnt + 5, 0, sizeof(unsigned long long), st));
    CK(launch_max_est(bs.rows[NBINS - 1], (unsigned long long)bs.count[NBINS - 1], est, cnt + 5, st));
    unsigned long long mx = 0;
    CK(cudaMemcpyAsync(&mx, cnt + 5, sizeof(mx), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    bs.log2t_global = ceil_log2(2 * (mx > 0 ? mx : 1));
    LaunchShape s = shape_for(NBINS - 1, bs);
    size_t bytes = (size_t)s.max_ctas * s.warps * row_kernel_group_bytes(bs.log2t_global, num, s.group);
    CKS(palloc(p, &bs.gtables, (int64_t)bytes, cat, st));
  }
  return PTAP_OK;
}

template <typename F>
ptap_status for_bins(ptap_plan *p, BinSet &bs, F launch) {
  for (int q = 0; q < NBINS; ++q) {
    if (bs.count[q] == 0) continue;
    LaunchShape s = shape_for(q, bs);
    const int32_t *rows = (q == 0 && bs.identity0) ? nullptr : bs.rows[q];
    CK(launch(s, rows, (unsigned long long)bs.count[q]));
    p->cnt.kernel_launches++;
  }
  return PTAP_OK;
}

// ---- arenas ------------------------------------------------------------------
// bucket_rows > 0: the keys' rows are [0, bucket_rows) (a local C arena) and
// each row gets its own run of slots when the capacity allows >= 8 per row
ptap_status arena_alloc(ptap_plan *p, Arena &ar, unsigned long long min_keys, cudaStream_t st,
                        unsigned long long bucket_rows = 0) {
  unsigned long long cap = 1024;
  while (cap * 3 < min_keys * 4) cap <<= 1;  // <= 75% load at the estimate
  CKS(palloc(p, &ar.keys, (int64_t)cap, CAT_TRANSIENT, st));
  ar.mask = cap - 1;
  ar.m = (unsigned long long)p->m;
  ar.log2b = 0;
  // row buckets suit operators whose rows repeat; on an unstructured one
  // (config 5) bucket runs overflow and chain (4 M points: 535 vs 20 ms), so
  // its arena is hashed
  if (bucket_rows > 0 && !getenv("PTAP_HASHED_ARENA") && !p->rows_unstructured) {
    unsigned long long r = 1;
    while (r < bucket_rows) r <<= 1;
    int lb = 0;
    while ((r << (lb + 1)) <= cap) ++lb;
    ar.log2b = lb >= 3 ? lb : 0;
  }
  CK(launch_arena_fill_empty(ar, st));
  p->cnt.kernel_launches++;
  return PTAP_OK;
}

ptap_status arena_grow(ptap_plan *p, Arena &ar, cudaStream_t st) {
  Arena big{nullptr, 0};
  CKS(arena_alloc(p, big, 2 * (ar.mask + 1), st, ar.log2b > 0 ? (ar.mask + 1) >> ar.log2b : 0));
  CK(launch_arena_rehash(ar, big, p->d_status, st));
  p->cnt.kernel_launches++;
  pfree(p, ar.keys, st);
  ar = big;
  return PTAP_OK;
}

// Arena -> CSR over `nrows_dense` rows (row id = key / m), columns sorted.
// avals / val_out: the single-shot pass's value array beside the keys, drained
// as the sort's payload into the rows' values
ptap_status arena_to_csr(ptap_plan *p, Arena ar, int64_t nrows_dense, int cat, int64_t **rp_out, int32_t **col_out,
                         int64_t *nnz_out, int64_t **cnt_keep, cudaStream_t st, const double *avals = nullptr,
                         double **val_out = nullptr) {
  int64_t *cnt = nullptr, *rp = nullptr, *scratch = nullptr;
  Tracer tr;
  tr.on = tr.on && getenv("PTAP_TRACE")[0] == '2';
  CKS(palloc(p, &cnt, nrows_dense, CAT_TRANSIENT, st));
  CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (nrows_dense > 0 ? nrows_dense : 1), st));
  CK(launch_arena_rowcount(ar, p->m, cnt, st));
  tr.mark(st, "  drain: rowcount");
  CKS(palloc(p, &rp, nrows_dense + 1, cat, st));
  CKS(palloc(p, &scratch, scan_scratch_elems(nrows_dense), CAT_TRANSIENT, st));
  CK(scan_exclusive(cnt, rp, nrows_dense, scratch, st));
  int64_t nnz = 0;
  CK(cudaMemcpyAsync(&nnz, rp + nrows_dense, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  tr.mark(st, "  drain: scan");
  int32_t *col = nullptr;
  CKS(palloc(p, &col, nnz, cat, st));
  int64_t *cursor = scratch;  // reuse: needs nrows_dense entries
  pfree(p, scratch, st);
  CKS(palloc(p, &cursor, nrows_dense, CAT_TRANSIENT, st));
  CK(cudaMemsetAsync(cursor, 0, sizeof(int64_t) * (nrows_dense > 0 ? nrows_dense : 1), st));
  int64_t *payload = nullptr;
  if (avals) {
    CKS(palloc(p, &payload, nnz, cat, st));
    CK(launch_arena_scatter_vals(ar, p->m, rp, cursor, col, avals, payload, st));
  } else {
    CK(launch_arena_scatter(ar, p->m, rp, cursor, col, st));
  }
  pfree(p, cursor, st);
  tr.mark(st, "  drain: scatter");
  int32_t *wide = nullptr;
  CKS(palloc(p, &wide, nnz / 1024 + 2, CAT_TRANSIENT, st));
  CK(cudaMemsetAsync(p->d_u64 + 6, 0, sizeof(unsigned long long), st));
  CK(launch_sort_rows(nrows_dense, rp, col, payload, wide, p->d_u64 + 6, st));
  unsigned long long nwide = 0;
  CK(cudaMemcpyAsync(&nwide, p->d_u64 + 6, sizeof(nwide), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  tr.mark(st, "  drain: sort rows");
  CK(launch_sort_rows_block((int64_t)nwide, wide, rp, col, payload, p->d_status, st));
  tr.mark(st, "  drain: sort wide");
  if (val_out) *val_out = (double *)payload;  // the payload holds the doubles' bits
  pfree(p, wide, st);
  p->cnt.kernel_launches += 6;
  if (cnt_keep) *cnt_keep = cnt; else pfree(p, cnt, st);
  *rp_out = rp;
  *col_out = col;
  *nnz_out = nnz;
  return PTAP_OK;
}

// send arena -> staging rows (global coarse ids, ascending) + CSR
ptap_status arena_to_staging(ptap_plan *p, Arena ar, int cat, cudaStream_t st) {
  int64_t *dense_rp = nullptr, *cnt = nullptr;
  int32_t *col = nullptr;
  int64_t nnz = 0;
  CKS(arena_to_csr(p, ar, p->m, cat, &dense_rp, &col, &nnz, &cnt, st));
  int64_t *flags = nullptr, *pos = nullptr, *scratch = nullptr;
  CKS(palloc(p, &flags, p->m, CAT_TRANSIENT, st));
  CKS(palloc(p, &pos, p->m + 1, CAT_TRANSIENT, st));
  CKS(palloc(p, &scratch, scan_scratch_elems(p->m), CAT_TRANSIENT, st));
  CK(launch_nonzero_flags(p->m, cnt, flags, st));
  CK(scan_exclusive(flags, pos, p->m, scratch, st));
  int64_t nrows = 0;
  CK(cudaMemcpyAsync(&nrows, pos + p->m, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  CKS(palloc(p, &p->s_rows, nrows, cat, st));
  CKS(palloc(p, &p->s_rp, nrows + 1, cat, st));
  CK(launch_compact_rows(p->m, cnt, pos, dense_rp, p->s_rows, p->s_rp, st));
  CK(cudaMemcpyAsync(p->s_rp + nrows, dense_rp + p->m, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  p->cnt.kernel_launches += 3;
  pfree(p, flags, st);
  pfree(p, pos, st);
  pfree(p, scratch, st);
  pfree(p, cnt, st);
  pfree(p, dense_rp, st);
  p->s_nrows = nrows;
  p->s_nnz = nnz;
  p->s_col = col;
  CKS(palloc(p, &p->s_val, nnz, cat, st));
  CK(cudaMemsetAsync(p->s_val, 0, sizeof(double) * (nnz > 0 ? nnz : 1), st));
  return PTAP_OK;
}

ptap_status build_transpose(ptap_plan *p, Transpose &t, int64_t ntrows, const int64_t *rp, const int32_t *col,
                            int64_t nnz, cudaStream_t st) {
  t.nrows = ntrows;
  t.nnz = nnz;
  int64_t *cnt = nullptr, *scratch = nullptr;
  CKS(palloc(p, &cnt, ntrows, CAT_TRANSIENT, st));
  CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (ntrows > 0 ? ntrows : 1), st));
  if (nnz > 0) CK(launch_count_cols(nnz, col, cnt, st));
  CKS(palloc(p, &t.rp, ntrows + 1, CAT_AUX, st));
  CKS(palloc(p, &scratch, scan_scratch_elems(ntrows), CAT_TRANSIENT, st));
  CK(scan_exclusive(cnt, t.rp, ntrows, scratch, st));
  CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (ntrows > 0 ? ntrows : 1), st));
  CKS(palloc(p, &t.row, nnz, CAT_AUX, st));
  CKS(palloc(p, &t.perm, nnz, CAT_PLAN, st));
  CKS(palloc(p, &t.val, nnz, CAT_AUX, st));
  if (nnz > 0) {
    CK(launch_transpose_scatter(p->nloc, rp, col, t.rp, cnt, t.row, t.perm, st));
    int32_t *wide = nullptr;
    CKS(palloc(p, &wide, nnz / 1024 + 2, CAT_TRANSIENT, st));
    CK(cudaMemsetAsync(p->d_u64 + 6, 0, sizeof(unsigned long long), st));
    CK(launch_sort_rows(ntrows, t.rp, t.row, t.perm, wide, p->d_u64 + 6, st));
    unsigned long long nwide = 0;
    CK(cudaMemcpyAsync(&nwide, p->d_u64 + 6, sizeof(nwide), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(launch_sort_rows_block((int64_t)nwide, wide, t.rp, t.row, t.perm, p->d_status, st));
    pfree(p, wide, st);
  }
  p->cnt.kernel_launches += 5;
  pfree(p, cnt, st);
  pfree(p, scratch, st);
  return PTAP_OK;
}

ptap_status ap_sizes(ptap_plan *p, const Ops &op, int64_t **ap_nnz_out, cudaStream_t st, int64_t **apub_out = nullptr) {
  int64_t *apub = nullptr, *ap_nnz = nullptr;
  CKS(palloc(p, &apub, op.nloc, CAT_TRANSIENT, st));
  CK(cudaMemsetAsync(p->d_u64 + 7, 0, sizeof(unsigned long long), st));
  CK(launch_row_work(op, apub, p->d_u64 + 7, st));
  unsigned long long mac_ap = 0;
  CK(cudaMemcpyAsync(&mac_ap, p->d_u64 + 7, sizeof(mac_ap), cudaMemcpyDeviceToHost, st));
  p->cnt.mac_ap = (int64_t)mac_ap;
  CKS(palloc(p, &ap_nnz, op.nloc, CAT_TRANSIENT, st));
  CK(cudaMemsetAsync(ap_nnz, 0, sizeof(int64_t) * (op.nloc > 0 ? op.nloc : 1), st));
  // optimistic small-table count first; rows that do not fit are recounted
  // through the work bins
  const int64_t *est = apub;
  int64_t *est2 = nullptr;
  int mode = 0;
  if (!getenv("PTAP_NO_FASTCOUNT")) {
    CK(launch_ap_count_small(op, op.nloc, apub, ap_nnz, st));
    CKS(palloc(p, &est2, op.nloc, CAT_TRANSIENT, st));
    CK(cudaMemsetAsync(p->d_u64 + 16, 0, sizeof(unsigned long long), st));
    CK(launch_retry_est(op.nloc, ap_nnz, apub, est2, p->d_u64 + 16, st));
    p->cnt.kernel_launches += 2;
    est = est2;
    mode = 4;
  }
  BinSet tmp;
  CKS(build_bins(p, tmp, op.nloc, est, op.pd_rp, op.po_rp, mode, false, CAT_TRANSIENT, st));
  CKS(for_bins(p, tmp, [&](const LaunchShape &s, const int32_t *rows, unsigned long long n) {
    return launch_ap_count(s, op, rows, n, ap_nnz, p->d_status, st);
  }));
  free_bins(p, tmp, st);
  pfree(p, est2, st);
  if (apub_out) *apub_out = apub; else pfree(p, apub, st);
  // bounds of the outer products
  CK(cudaMemsetAsync(p->d_u64 + 8, 0, 3 * sizeof(unsigned long long), st));
  CK(launch_outer_bounds(op.nloc, op.pd_rp, op.po_rp, ap_nnz, p->d_u64 + 8, st));
  unsigned long long b[3];
  CK(cudaMemcpyAsync(b, p->d_u64 + 8, sizeof(b), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  p->bound_local = b[0];
  p->bound_send = b[1];
  p->sum_ap = b[2];
  p->cnt.mac_outer = (int64_t)(b[0] + b[1]);
  p->cnt.kernel_launches += 3;
  *ap_nnz_out = ap_nnz;
  return PTAP_OK;
}

unsigned long long local_arena_estimate(const ptap_plan *p, int64_t extra) {
  // a C row unions the AP rows of its contributors; the wider P's rows, the
  // more the union outgrows one AP row (27-pt/trilinear: ~1.8x, smoothed
  // aggregation: ~6x), so scale the average AP row by 1 + (P entries/row)/2
  double avg = p->nloc > 0 ? (double)p->sum_ap / (double)p->nloc : 1.0;
  double est = (double)p->ncl * (avg * (1.0 + 0.5 * p->avg_p_row) + 8.0) + (double)extra;
  double bound = (double)p->bound_local + (double)extra;
  if (est > bound) est = bound;
  // test hook: an undersized first arena, so the growth path runs
  if (const char *sh = getenv("PTAP_ARENA_SHRINK")) est /= std::max(1.0, atof(sh));
  if (est < 64) est = 64;
  return (unsigned long long)est;
}

// run `pass` until it completes without arena overflow (growing the arena)
template <typename F>
ptap_status with_arena_retry(ptap_plan *p, Arena &ar, cudaStream_t st, F pass) {
  for (int attempt = 0; attempt < 8; ++attempt) {
    CKS(pass());
    int s = 0;
    CKS(read_status(p, st, &s));
    if (!(s & ST_ARENA_FULL)) {
      if (s) return status_to_error(s, "symbolic");
      return PTAP_OK;
    }
    CKS(arena_grow(p, ar, st));
  }
  return fail(PTAP_ERR_OOM, "symbolic arena kept overflowing");
}

// Do the operator's rows repeat structurally?  k_struct_sample counts the
// distinct row signatures of 65,536 sampled rows; more than one in four
// distinct marks the operator unstructured (maps are skipped, rows are
// visited in aggregate order).
ptap_status sample_row_structures(ptap_plan *p, const Ops &op, cudaStream_t st) {
  if (p->nloc <= 0) return PTAP_OK;
  const int64_t nsample = std::min<int64_t>(p->nloc, 65536);
  const int64_t ent = int64_t(1) << 17;
  unsigned long long *keys = nullptr, *cnt = p->d_u64 + 21;
  CKS(palloc(p, &keys, ent, CAT_TRANSIENT, st));
  CK(cudaMemsetAsync(keys, 0, sizeof(unsigned long long) * ent, st));
  CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
  CK(launch_struct_sample(op, nsample, keys, (unsigned long long)(ent - 1), cnt, st));
  unsigned long long distinct = 0;
  CK(cudaMemcpyAsync(&distinct, cnt, sizeof(distinct), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  pfree(p, keys, st);
  p->cnt.kernel_launches++;
  p->cnt.row_structures_ppm = (int64_t)(1e6 * (double)distinct / (double)nsample);
  p->rows_unstructured = (int64_t)distinct * 4 > nsample;
  return PTAP_OK;
}

// Plan-mapped numeric: byte maps of slots (AP row) and positions (target rows)
// computed once here so numeric passes do no hashing and no searching.
// Plan-mapped numeric, part 1 (before the outer-product symbolic pass): the
// slot maps are written by that pass itself, so allocate them here.
ptap_status prepare_maps(ptap_plan *p, const Ops &op, const ptap_operands *ops, cudaStream_t st) {
  p->want_maps = false;
  Tracer tr;
  tr.on = tr.on && getenv("PTAP_TRACE")[0] == '2';
  if (getenv("PTAP_NO_MAPS") || p->maps_opt == 0) return PTAP_OK;
  unsigned long long *mx = p->d_u64 + 12;
  CK(cudaMemsetAsync(mx, 0, 3 * sizeof(unsigned long long), st));
  CK(launch_max_i64(p->nloc, p->ap_nnz, mx, st));      // AP row width  (slot byte)
  CK(launch_max_i64(p->nloc, p->apub, mx + 1, st));    // pairs per row (16-bit offsets)
  CK(launch_max_rowlen(p->nloc, op.pd_rp, mx + 2, st)); // P row length (8-bit counts)
  unsigned long long h[3];
  CK(cudaMemcpyAsync(h, mx, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  p->cnt.kernel_launches += 3;
  tr.mark(st, "  maps: maxima");
  p->max_nap = (int64_t)h[0];
  if (h[0] > 255 || h[1] > 65535 || h[2] > 255) return PTAP_OK;  // hash path for this plan
  // maps pay for themselves when rows repeat (interned, a small pool); on an
  // operator whose rows do not repeat they would cost about as much memory as
  // the two-step's auxiliary matrices, so such a plan keeps no maps and
  // numeric runs the hash path (PTAP_MAPS=1 keeps them regardless)
  if (!getenv("PTAP_MAPS") && p->maps_opt != 1 && p->rows_unstructured) return PTAP_OK;  // rows do not repeat: hash path
  {
    // bin 0 through k_outer_numeric_q4: <= 128 map bytes per row and every
    // offset it touches within 32 bits
    const int64_t lim = INT32_MAX;
    const int64_t nnz_max = std::max<int64_t>({ops->a_diag.nnz, ops->a_off.nnz, ops->p_diag.nnz, ops->p_off.nnz,
                                      ops->p_remote.nnz});
    p->q4 = h[1] <= 128 && p->nloc < lim && nnz_max < lim && !getenv("PTAP_NO_Q4");
    p->q4_sym = p->q4 && !getenv("PTAP_NO_Q4_SYMBOLIC");
    // q4a (A staged by cp.async): one-rank structure, A rows <= 32 entries
    if (p->q4 && ops->a_off.nnz == 0 && ops->p_off.nnz == 0 && !getenv("PTAP_NO_Q4A")) {
      CK(cudaMemsetAsync(mx, 0, sizeof(unsigned long long), st));
      CK(launch_max_rowlen(p->nloc, op.ad_rp, mx, st));
      unsigned long long amax = 0;
      CK(cudaMemcpyAsync(&amax, mx, sizeof(amax), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      p->q4a = amax <= 32;
      // packed P row bounds per A entry (one dependent load less in the fold):
      // opt-in, it trades 4 B of plan memory per A entry (+1.8 GB on cfg3,
      // aux 3.94 -> 5.74 GB) for ~3% (8.13 -> 7.89 ms)
      if (p->q4a && ops->p_diag.nnz < (int64_t(1) << 28) && h[2] <= 15 && getenv("PTAP_POFF")) {
        CKS(palloc(p, &p->maps.poff, ops->a_diag.nnz, CAT_PLAN, st));
        CK(launch_build_poff(ops->a_diag.nnz, op.ad_col, op.pd_rp, p->maps.poff, st));
        p->cnt.kernel_launches++;
      }
    }
  }
  int64_t *slen = nullptr, *scratch = nullptr;
  CKS(palloc(p, &slen, p->nloc, CAT_TRANSIENT, st));
  CKS(palloc(p, &scratch, scan_scratch_elems(p->nloc), CAT_TRANSIENT, st));
  int64_t *unused = nullptr;
  CKS(palloc(p, &unused, p->nloc, CAT_TRANSIENT, st));
  tr.mark(st, "  maps: alloc 1");
  CK(launch_map_lengths(p->nloc, op.pd_rp, op.po_rp, p->apub, p->ap_nnz, slen, unused, st));
  CKS(palloc(p, &p->maps.smap_rp, p->nloc + 1, CAT_PLAN, st));
  CK(scan_exclusive(slen, p->maps.smap_rp, p->nloc, scratch, st));
  CKS(palloc(p, &p->pat_rp, p->nloc + 1, CAT_TRANSIENT, st));
  CK(scan_exclusive(p->ap_nnz, p->pat_rp, p->nloc, scratch, st));
  int64_t tot[2];
  CK(cudaMemcpyAsync(&tot[0], p->maps.smap_rp + p->nloc, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&tot[1], p->pat_rp + p->nloc, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  tr.mark(st, "  maps: lengths + scans");
  pfree(p, slen, st);
  pfree(p, unused, st);
  pfree(p, scratch, st);
  p->smap_bytes = tot[0];
  // a rank that sends nothing writes its slot maps in symbolic_local, which
  // builds them chunk by chunk when it can: the full buffer is deferred
  p->smap_deferred = ops->p_off.nnz == 0 && !getenv("PTAP_NO_MAP_CHUNKS");
  if (!p->smap_deferred) CKS(palloc(p, &p->maps.smap, tot[0] + 16, CAT_PLAN, st));  // padded: staged word-wise
  CKS(palloc(p, &p->maps.nap, p->nloc, CAT_PLAN, st));
  CKS(palloc(p, &p->pat, tot[1], CAT_TRANSIENT, st));
  tr.mark(st, "  maps: alloc 2");
  p->mo = MapOut{p->maps.smap_rp, p->maps.smap, p->maps.nap, p->pat_rp, p->pat};
  p->want_maps = true;
  return PTAP_OK;
}

// position-map storage (C rows and staging rows must fit a byte)
ptap_status alloc_pmap(ptap_plan *p, const Ops &op, const ptap_operands *ops, cudaStream_t st, bool *ok_out) {
  unsigned long long *mx = p->d_u64 + 12;
  CK(cudaMemsetAsync(mx, 0, 2 * sizeof(unsigned long long), st));
  CK(launch_max_rowlen(p->ncl, p->c_rp, mx, st));
  if (p->s_nrows) CK(launch_max_rowlen(p->s_nrows, p->s_rp, mx + 1, st));
  unsigned long long h[2];
  CK(cudaMemcpyAsync(h, mx, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *ok_out = h[0] <= 256 && h[1] <= 256;
  if (!*ok_out) return PTAP_OK;
  int64_t *plen = nullptr, *scratch = nullptr, *unused = nullptr;
  CKS(palloc(p, &plen, p->nloc, CAT_TRANSIENT, st));
  CKS(palloc(p, &unused, p->nloc, CAT_TRANSIENT, st));
  CKS(palloc(p, &scratch, scan_scratch_elems(p->nloc), CAT_TRANSIENT, st));
  CK(launch_map_lengths(p->nloc, op.pd_rp, op.po_rp, p->apub, p->ap_nnz, unused, plen, st));
  CKS(palloc(p, &p->maps.pmap_rp, p->nloc + 1, CAT_PLAN, st));
  CK(scan_exclusive(plen, p->maps.pmap_rp, p->nloc, scratch, st));
  int64_t tot = 0;
  CK(cudaMemcpyAsync(&tot, p->maps.pmap_rp + p->nloc, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  pfree(p, plen, st);
  pfree(p, unused, st);
  pfree(p, scratch, st);
  p->pmap_bytes = tot;
  CKS(palloc(p, &p->maps.pmap, tot + 16, CAT_PLAN, st));  // padded: interned word-wise
  int64_t po_nnz = ops->p_off.nnz;
  CKS(palloc(p, &p->maps.po_srow, po_nnz, CAT_PLAN, st));
  if (po_nnz > 0)
    CK(launch_po_srow(po_nnz, op.po_col, op.p_colmap, p->s_nrows, p->s_rows, p->maps.po_srow, p->d_status, st));
  p->cnt.kernel_launches += 4;
  return PTAP_OK;
}

// Interns a per-row byte map (src at monotone offsets src_rp[0..n]) into a
// pool holding each distinct row map once (word aligned); src and src_rp are
// replaced by the pool and the per-row pool offsets (| length << 40 with
// pack_len).  Three kernels (claim, resolve, copy) around one scan; see
// k_intern_claim.
ptap_status intern_map(ptap_plan *p, uint8_t *&src, int64_t *&src_rp, int64_t n, int64_t total, bool pack_len,
                       int64_t *pool_bytes, cudaStream_t st) {
  if (getenv("PTAP_NO_INTERN")) {
    if (pack_len) {  // same packed layout without sharing: offset | length << 40
      int64_t *out = nullptr;
      CKS(palloc(p, &out, n + 1, CAT_PLAN, st));
      CK(launch_pack_offsets(n, src_rp, out, st));
      p->cnt.kernel_launches++;
      pfree(p, src_rp, st);
      src_rp = out;
    }
    *pool_bytes = total;
    return PTAP_OK;
  }
  int64_t ent = 1024;
  while (ent < 2 * n && ent < (int64_t(1) << 22)) ent <<= 1;
  unsigned long long *keys = nullptr;
  int64_t *vals = nullptr, *slot_of = nullptr, *owner = nullptr, *words = nullptr, *wpos = nullptr,
          *scratch = nullptr, *out = nullptr;
  CKS(palloc(p, &keys, ent, CAT_TRANSIENT, st));
  CKS(palloc(p, &vals, ent, CAT_TRANSIENT, st));
  CKS(palloc(p, &slot_of, n, CAT_TRANSIENT, st));
  CKS(palloc(p, &owner, n, CAT_TRANSIENT, st));
  CKS(palloc(p, &words, n, CAT_TRANSIENT, st));
  CKS(palloc(p, &wpos, n + 1, CAT_TRANSIENT, st));
  CKS(palloc(p, &scratch, scan_scratch_elems(n), CAT_TRANSIENT, st));
  unsigned long long *claims = p->d_u64 + 20;
  CK(cudaMemsetAsync(keys, 0, sizeof(unsigned long long) * ent, st));
  CK(cudaMemsetAsync(claims, 0, sizeof(unsigned long long), st));
  CK(launch_intern(0, n, src, src_rp, keys, vals, (unsigned long long)(ent - 1), slot_of, owner, words, nullptr,
                   nullptr, 0, claims, st));
  CK(launch_intern(1, n, src, src_rp, keys, vals, 0, slot_of, owner, words, nullptr, nullptr, 0, claims, st));
  pfree(p, keys, st);
  pfree(p, vals, st);
  pfree(p, slot_of, st);
  CK(scan_exclusive(words, wpos, n, scratch, st));
  int64_t nw = 0;
  CK(cudaMemcpyAsync(&nw, wpos + n, sizeof(nw), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  p->cnt.kernel_launches += 3;
  if (nw * 4 > total / 2) {
    // the rows hardly repeat (unstructured input): keep the per-row maps as
    // they are rather than hold a second copy of most of them
    pfree(p, owner, st);
    pfree(p, words, st);
    pfree(p, wpos, st);
    pfree(p, scratch, st);
    if (pack_len) {
      CKS(palloc(p, &out, n + 1, CAT_PLAN, st));
      CK(launch_pack_offsets(n, src_rp, out, st));
      p->cnt.kernel_launches++;
      pfree(p, src_rp, st);
      src_rp = out;
    }
    *pool_bytes = total;
    return PTAP_OK;
  }
  uint8_t *pool = nullptr;
  CKS(palloc(p, &pool, nw * 4 + 16, CAT_PLAN, st));  // +16: the numeric kernels stage maps as words
  CKS(palloc(p, &out, n + 1, CAT_PLAN, st));
  CK(launch_intern(2, n, src, src_rp, nullptr, nullptr, 0, nullptr, owner, wpos, pool, out, pack_len ? 1 : 0,
                   nullptr, st));
  p->cnt.kernel_launches++;
  pfree(p, owner, st);
  pfree(p, words, st);
  pfree(p, wpos, st);
  pfree(p, scratch, st);
  pfree(p, src, st);
  pfree(p, src_rp, st);
  src = pool;
  src_rp = out;
  *pool_bytes = nw * 4;
  return PTAP_OK;
}

// ---- deterministic owner-computes numeric plan (ptap_tile.cu) ----------------
void free_tile(ptap_plan *p, cudaStream_t st) {
  TileArgs &t = p->ta;
  pfree(p, t.ap_off, st); pfree(p, t.ring, st); pfree(p, t.own_rp, st); pfree(p, t.t_pidx, st);
  pfree(p, t.t_rp, st); pfree(p, t.t_row, st); pfree(p, t.t_jx, st); pfree(p, t.rd_rp, st);
  pfree(p, t.rd_blk, st); pfree(p, t.expect, st); pfree(p, t.flags, st); pfree(p, t.readcnt, st);
  pfree(p, t.ctl, st);
  pfree(p, t.qmap, st); pfree(p, t.qmap_rp, st); pfree(p, t.pr_n, st); pfree(p, t.pr_k, st);
  pfree(p, t.t_jx, st);
  t = TileArgs{};
  p->tile = false;
}

// Eligible: one-rank structure (the q4a plan: no A_o / P_o, A rows <= 32),
// interned maps, AP rows <= 32 slots, C rows <= 64 entries with <= 32
// contributors, and a contributor span that keeps the AP ring small.
ptap_status build_tile(ptap_plan *p, const Ops &op, const ptap_operands *ops, cudaStream_t st) {
  p->tile = false;
  if (!(p->deterministic || getenv("PTAP_DETERMINISTIC")) || getenv("PTAP_NO_TILE")) return PTAP_OK;
  if (!p->mapped || !p->q4a || p->alg == PTAP_TWO_STEP || p->max_nap > 32) return PTAP_OK;
  const int64_t n = p->nloc, ncl = p->ncl, pnnz = ops->p_diag.nnz;
  if (n <= 0 || ncl <= 0 || pnnz >= INT32_MAX || ops->a_diag.nnz >= INT32_MAX || n >= INT32_MAX - 2 * TILE_ROWS)
    return PTAP_OK;
  unsigned long long *stats = nullptr;  // span, max contributors, largest block, largest owner, A per block,
  CKS(palloc(p, &stats, 8, CAT_TRANSIENT, st));  // staged P values, staged blocks
  CK(cudaMemsetAsync(stats, 0, 8 * sizeof(unsigned long long), st));
  unsigned long long *cmax_d = p->d_u64 + 12;
  CK(cudaMemsetAsync(cmax_d, 0, sizeof(unsigned long long), st));
  CK(launch_max_rowlen(ncl, p->c_rp, cmax_d, st));
  TileArgs &t = p->ta;
  t = TileArgs{};
  const int nblk = (int)((n + TILE_ROWS - 1) / TILE_ROWS);
  t.nloc = (int32_t)n;
  t.nblk = nblk;
  t.napc = (int32_t)std::max<int64_t>(1, p->max_nap);
  // per-block AP offsets, the largest block, and the P rows each block stages
  uint16_t *ap_off = nullptr;
  uint8_t *pr_n = nullptr;
  int2 *pr_k = nullptr;
  CKS(palloc(p, &ap_off, n, CAT_PLAN, st));
  CKS(palloc(p, &pr_n, nblk, CAT_PLAN, st));
  CKS(palloc(p, &pr_k, (int64_t)nblk * TILE_MAXRUN, CAT_PLAN, st));
  t.ap_off = ap_off; t.pr_n = pr_n; t.pr_k = pr_k;
  CK(launch_tile_apoff(n, op.ad_rp, op.pd_rp, p->maps.nap, ap_off, stats, st));
  // P runs staged in shared memory: measured slower (17.4 vs 13.9 ms on
  // config 3: the extra shared memory costs resident CTAs), so opt-in
  const bool pstage = getenv("PTAP_TILE_PSTAGE") != nullptr;
  const int pvcap = pstage ? 3072 : 0;
  t.pstage = pstage ? 1 : 0;
  t.a_evict_first = getenv("PTAP_TILE_NO_EVICT") ? 0 : 1;
  if (pstage)
    CK(launch_tile_pruns(nblk, n, op.ad_rp, op.ad_col, op.pd_rp, pnnz, pvcap, 1024, pr_n, pr_k, stats, st));
  else
    CK(cudaMemsetAsync(pr_n, 0, nblk, st));
  unsigned long long hs[8], cmax = 0;
  CK(cudaMemcpyAsync(hs, stats, sizeof(hs), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&cmax, cmax_d, sizeof(cmax), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (cmax > (unsigned long long)TILE_MAX_CROW || hs[4] > 64 * 32) {
    pfree(p, stats, st);
    free_tile(p, st);
    return PTAP_OK;
  }
  const int64_t blkcap = std::max<int64_t>(2, (int64_t)hs[2]);
  tile_smem_layout(t, (int)hs[4], pstage ? (int)hs[5] : 0, pstage ? (int)hs[7] : 0);
  const int grid = tile_grid(t);
  // ownership delay: C row J is gathered at least `delay` items after the
  // block of its last contributor, so its contributors were published a
  // full grid of items earlier and the gather practically never waits
  const int delay = getenv("PTAP_TILE_DELAY") ? atoi(getenv("PTAP_TILE_DELAY")) : grid;
  const int64_t wide = std::max<int64_t>(ncl, nblk + delay + 2);
  const size_t sbytes = std::max(tile_scan_scratch(wide), tile_owner_scratch(ncl));
  uint8_t *scratch = nullptr;
  int32_t *cnt = nullptr, *cursor = nullptr, *owner = nullptr;
  long long *key = nullptr;
  CKS(palloc(p, &scratch, (int64_t)sbytes, CAT_TRANSIENT, st));
  CKS(palloc(p, &cnt, wide + 1, CAT_TRANSIENT, st));
  CKS(palloc(p, &cursor, wide + 1, CAT_TRANSIENT, st));
  int32_t *t_rp = nullptr, *t_row = nullptr, *t_pidx = nullptr, *own_rp = nullptr;
  uint8_t *t_jx = nullptr;
  CKS(palloc(p, &t_rp, ncl + 1, CAT_PLAN, st));
  CKS(palloc(p, &t_row, pnnz, CAT_PLAN, st));
  CKS(palloc(p, &t_pidx, pnnz, CAT_PLAN, st));
  CKS(palloc(p, &t_jx, pnnz, CAT_TRANSIENT, st));
  t.t_rp = t_rp; t.t_row = t_row; t.t_pidx = t_pidx; t.t_jx = t_jx;
  CK(launch_tile_transpose(n, ncl, op.pd_rp, op.pd_col, pnnz, cnt, t_rp, cursor, t_row, t_jx, scratch, sbytes,
                           p->d_status, st));
  CKS(palloc(p, &owner, ncl, CAT_TRANSIENT, st));
  CKS(palloc(p, &key, ncl, CAT_TRANSIENT, st));
  CK(launch_tile_owners(ncl, nblk, delay, op.pd_rp, t_rp, t_row, t_jx, t_pidx, key, owner, stats, scratch, sbytes,
                        st));
  pfree(p, key, st);
  CK(cudaMemcpyAsync(hs, stats, sizeof(hs), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  p->cnt.kernel_launches += 10;
  const int64_t span = (int64_t)hs[0], kmax = (int64_t)hs[1];
  const int nitems = std::max<int>(nblk, (int)hs[3] + 1);
  t.nitems = nitems;
  const int64_t R = std::min<int64_t>(nblk, span + 2 * (int64_t)grid + 64);
  if (kmax > 32 || span > 32768 || R * blkcap >= INT32_MAX || R * blkcap * 8 > (int64_t(512) << 20)) {
    pfree(p, scratch, st); pfree(p, cnt, st); pfree(p, cursor, st); pfree(p, owner, st); pfree(p, stats, st);
    free_tile(p, st);
    return PTAP_OK;
  }
  const unsigned long long staged_blocks = hs[6];
  pfree(p, stats, st);
  CKS(palloc(p, &own_rp, nitems + 1, CAT_PLAN, st));
  t.own_rp = own_rp;
  CK(launch_tile_own_rp(nitems, ncl, owner, own_rp, st));
  pfree(p, owner, st);
  // reader lists
  int32_t *rd_rp = nullptr, *rd_blk = nullptr;
  uint32_t *expect = nullptr;
  CKS(palloc(p, &rd_rp, nitems + 1, CAT_PLAN, st));
  CKS(palloc(p, &expect, nblk, CAT_PLAN, st));
  t.rd_rp = rd_rp; t.expect = expect;
  CK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nitems + 1), st));
  CK(cudaMemsetAsync(expect, 0, sizeof(uint32_t) * nblk, st));
  CK(launch_tile_reads(0, nitems, 0, (int)span, own_rp, t_rp, t_row, cnt, nullptr, nullptr, nullptr, st));
  CK(launch_tile_scan32(cnt, rd_rp, nitems, scratch, sbytes, st));
  int32_t nrd = 0;
  CK(cudaMemcpyAsync(&nrd, rd_rp + nitems, sizeof(nrd), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  CKS(palloc(p, &rd_blk, nrd, CAT_PLAN, st));
  t.rd_blk = rd_blk;
  CK(launch_tile_reads(1, nitems, 0, (int)span, own_rp, t_rp, t_row, nullptr, rd_rp, rd_blk, expect, st));
  pfree(p, scratch, st); pfree(p, cnt, st); pfree(p, cursor, st);
  // gather maps (inverse position maps per C row), interned like the others
  {
    int64_t *qlen = nullptr, *qrp = nullptr, *sc = nullptr;
    uint8_t *qm = nullptr;
    CKS(palloc(p, &qlen, ncl, CAT_TRANSIENT, st));
    CKS(palloc(p, &qrp, ncl + 1, CAT_PLAN, st));
    CKS(palloc(p, &sc, scan_scratch_elems(ncl), CAT_TRANSIENT, st));
    CK(launch_tile_qmap(ncl, t, p->c_rp, qlen, nullptr, nullptr, nullptr, nullptr, nullptr, 0, st));
    CK(scan_exclusive(qlen, qrp, ncl, sc, st));
    int64_t qtot = 0;
    CK(cudaMemcpyAsync(&qtot, qrp + ncl, sizeof(qtot), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    pfree(p, qlen, st);
    pfree(p, sc, st);
    CKS(palloc(p, &qm, qtot + 16, CAT_PLAN, st));
    CK(launch_tile_qmap(ncl, t, p->c_rp, nullptr, qrp, p->maps.nap, p->maps.pmap_rp, p->maps.pmap, qm, 1, st));
    int64_t pool = 0;
    CKS(intern_map(p, qm, qrp, ncl, qtot, false, &pool, st));
    pfree(p, t_jx, st);
    t.t_jx = nullptr;
    t.qmap = qm;
    t.qmap_rp = qrp;
    p->qmap_bytes = pool;
    p->cnt.kernel_launches += 2;
  }
  uint32_t *flags = nullptr, *readcnt = nullptr, *ctl = nullptr;
  CKS(palloc(p, &flags, nblk, CAT_PLAN, st));
  CKS(palloc(p, &readcnt, nblk, CAT_PLAN, st));
  CKS(palloc(p, &ctl, 4, CAT_PLAN, st));
  CK(cudaMemsetAsync(flags, 0, sizeof(uint32_t) * nblk, st));
  CK(cudaMemsetAsync(readcnt, 0, sizeof(uint32_t) * nblk, st));
  CK(cudaMemsetAsync(ctl, 0, sizeof(uint32_t) * 4, st));
  t.flags = flags; t.readcnt = readcnt; t.ctl = ctl;
  double *ring = nullptr;
  CKS(palloc(p, &ring, R * blkcap, CAT_PLAN, st));
  t.ring = ring;
  t.ring_blocks = (int32_t)R;
  t.blkcap = (int32_t)blkcap;
  t.grid = grid;
  t.dbg = getenv("PTAP_TILE_DBG") ? atoi(getenv("PTAP_TILE_DBG")) : 0;
  p->cnt.kernel_launches += 3;
  int s = 0;
  CKS(read_status(p, st, &s));
  if (s) {
    free_tile(p, st);
    return status_to_error(s, "tile plan");
  }
  p->tile = true;
  if (getenv("PTAP_TRACE"))
    fprintf(stderr,
            "[ptap] tile plan: %d blocks (%llu stage P), %d items (delay %d), span %lld, ring %lld x %lld doubles, "
            "grid %d, smem %d B, %d reads, gather maps %lld B\n",
            nblk, staged_blocks, nitems, delay, (long long)span, (long long)R, (long long)blkcap, grid, t.sm_total, nrd, (long long)p->qmap_bytes);
  return PTAP_OK;
}

// ---- class-lockstep numeric plan (ptap_lock.cu) ------------------------------
void free_lock(ptap_plan *p, cudaStream_t st) {
  LockArgs &l = p->la;
  pfree(p, l.pq, st); pfree(p, l.Q, st); pfree(p, l.cbQ, st); pfree(p, l.rowinfo, st); pfree(p, l.rowcls, st);
  pfree(p, l.cls, st); pfree(p, l.fold, st); pfree(p, l.outer, st); pfree(p, l.ltab, st);
  l = LockArgs{};
  p->lock = false;
}

// Eligible: the q4a plan (one-rank structure, A rows <= 32 entries) with
// interned maps, AP rows <= 32 slots, P rows <= 8 entries, fewer than 32768
// row classes, the C-row-start map, and a tile that fits shared memory.
// `pure` (several ranks): device flags of the rows without A_o / P_o parts (own
// or neighbours'); only tiles inside runs of such rows are launched
// (build_q4a_runs), the other rows share one empty class.
ptap_status build_lock(ptap_plan *p, const Ops &op, const ptap_operands *ops, cudaStream_t st,
                       const uint8_t *pure = nullptr) {
  p->lock = false;
  if (getenv("PTAP_NO_LOCK") || p->lock_opt == 0) return PTAP_OK;
  const bool for_tile = p->tile;  // the deterministic kernel takes the classes, programs and Q for its fold
  if (!p->mapped || !(p->q4a || pure) || p->alg == PTAP_TWO_STEP || p->max_nap > 32 ||
      (!for_tile && !p->maps.cbase) || getenv("PTAP_TILE_NO_LOCKFOLD") && for_tile)
    return PTAP_OK;
  const int64_t n = p->nloc, pnnz = ops->p_diag.nnz;
  if (n <= 0 || p->ncl <= 0 || pnnz <= 0 || pnnz >= INT32_MAX || ops->a_diag.nnz >= INT32_MAX ||
      n >= INT32_MAX - 2 * LOCK_TILE || p->c_nnz >= INT32_MAX - 256)
    return PTAP_OK;
  LockArgs &l = p->la;
  l = LockArgs{};
  const int ntiles = (int)((n + LOCK_TILE - 1) / LOCK_TILE);
  const int nb = (int)((n + 255) / 256);
  unsigned long long *st8 = nullptr;  // [0] classes, [1] fold entries, [2] outer words, [3] claims, [4] bad, [5] largest tile
  uint8_t *plen8 = nullptr;
  int32_t *blkcnt = nullptr, *ltab = nullptr, *slot2cls = nullptr;
  uint32_t *pq = nullptr, *rep = nullptr, *reps = nullptr, *rowinfo = nullptr;
  unsigned long long *keys = nullptr;
  uint16_t *slot_of = nullptr;
  auto drop_transient = [&]() {
    pfree(p, st8, st); pfree(p, plen8, st); pfree(p, blkcnt, st); pfree(p, slot2cls, st);
    pfree(p, rep, st); pfree(p, reps, st); pfree(p, keys, st); pfree(p, slot_of, st);
  };
  CKS(palloc(p, &st8, 8, CAT_TRANSIENT, st));
  CK(cudaMemsetAsync(st8, 0, 8 * sizeof(unsigned long long), st));
  CKS(palloc(p, &plen8, n, CAT_TRANSIENT, st));
  CKS(palloc(p, &blkcnt, (int64_t)LOCK_NLEN * nb, CAT_TRANSIENT, st));
  CKS(palloc(p, &ltab, 2 * LOCK_NLEN, CAT_PLAN, st));
  CKS(palloc(p, &pq, n, CAT_PLAN, st));
  l.ltab = ltab; l.pq = pq;
  CK(launch_lock_qlayout(n, op.pd_rp, plen8, blkcnt, ltab, pq, st8 + 4, st));
  pfree(p, blkcnt, st);
  CKS(palloc(p, &keys, LOCK_TABLE, CAT_TRANSIENT, st));
  CKS(palloc(p, &rep, LOCK_TABLE, CAT_TRANSIENT, st));
  CKS(palloc(p, &reps, LOCK_TABLE, CAT_TRANSIENT, st));
  CKS(palloc(p, &slot2cls, LOCK_TABLE, CAT_TRANSIENT, st));
  CKS(palloc(p, &slot_of, n, CAT_TRANSIENT, st));
  CK(launch_lock_classes(op, plen8, p->maps.smap_rp, p->maps.pmap_rp, keys, rep, LOCK_TABLE, slot_of, slot2cls, reps,
                         st8, st8 + 4, pure, st));
  unsigned long long h[8];
  CK(cudaMemcpyAsync(h, st8, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  p->cnt.kernel_launches += 7;
  if (h[4] != 0 || h[3] > LOCK_TABLE / 2 || h[0] == 0) {
    if (getenv("PTAP_TRACE"))
      fprintf(stderr, "[ptap] lockstep plan: not eligible (%llu classes, %llu flagged)\n", h[0], h[4]);
    drop_transient();
    free_lock(p, st);
    return PTAP_OK;
  }
  const int ncls = (int)h[0];
  LockClass *cls = nullptr;
  CKS(palloc(p, &cls, ncls, CAT_PLAN, st));
  l.cls = cls;
  // warps per group: long programs (27-point stencils: ~90 pairs per row) split three ways, short ones two
  l.lw = p->nloc > 0 && (double)p->cnt.mac_ap / (double)p->nloc >= 48.0 ? 3 : 2;
  if (const char *lwv = getenv("PTAP_LOCK_WARPS")) l.lw = atoi(lwv) == 3 ? 3 : 2;
  CK(launch_lock_headers(ncls, op, plen8, p->maps, reps, ltab, cls, st8, st8 + 4, pure, l.lw, st));
  CKS(palloc(p, &rowinfo, n, CAT_PLAN, st));
  l.rowinfo = rowinfo;
  uint32_t *rowcls = nullptr;
  if (for_tile) {
    CKS(palloc(p, &rowcls, n, CAT_PLAN, st));
    l.rowcls = rowcls;
  }
  CK(launch_lock_rowinfo(n, op.ad_rp, slot_of, slot2cls, rowinfo, rowcls, st8 + 5, st));
  CK(cudaMemcpyAsync(h, st8, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  p->cnt.kernel_launches += 2;
  l.nloc = (int32_t)n;
  l.ntiles = ntiles;
  l.ast = (int32_t)(std::max<unsigned long long>(1, h[6]) | 1);
  // the staged column region also holds the transposed converted rows (2 groups x 32 rows x ast)
  l.acap = (int32_t)((std::max<unsigned long long>(h[5] + 4, (unsigned long long)LOCK_TILE * l.ast) + 3) & ~3ull);
  l.aps = (int32_t)(std::max<int64_t>(1, p->max_nap) | 1);
  l.dbg = getenv("PTAP_LOCK_DBG") ? atoi(getenv("PTAP_LOCK_DBG")) : 0;
  if (h[4] != 0 || lock_smem_bytes(l) > 200 * 1024 || h[1] >= (1ull << 31) || h[2] >= (1ull << 31)) {
    if (getenv("PTAP_TRACE"))
      fprintf(stderr, "[ptap] lockstep plan: not eligible (%llu flagged, tile of %llu entries)\n", h[4], h[5]);
    drop_transient();
    free_lock(p, st);
    return PTAP_OK;
  }
  uint2 *fold = nullptr;
  uint32_t *outer = nullptr;
  CKS(palloc(p, &fold, (int64_t)h[1] + 8, CAT_PLAN, st));
  CK(cudaMemsetAsync(fold + h[1], 0, 8 * sizeof(uint2), st));
  l.fold_zero = (uint32_t)h[1];
  CKS(palloc(p, &outer, (int64_t)h[2] + 32, CAT_PLAN, st));
  l.fold = fold; l.outer = outer;
  CK(launch_lock_programs(ncls, op, plen8, p->maps, reps, ltab, cls, fold, outer, l.lw, st));
  drop_transient();
  // the C row starts in Q order replace the per-entry map of the q4a kernel
  int32_t *cbq = nullptr;
  double *Q = nullptr;
  if (!for_tile) {
    CKS(palloc(p, &cbq, pnnz, CAT_PLAN, st));
    CK(launch_lock_permute_i32(n, op.pd_rp, pq, ltab, p->maps.cbase, cbq, st));
    l.cbQ = cbq;
    if (!pure) pfree(p, p->maps.cbase, st);  // several ranks: the runs' unaligned edges keep the per-row kernel
  }
  CKS(palloc(p, &Q, pnnz, CAT_PLAN, st));
  l.Q = Q;
  p->cnt.kernel_launches += 3;
  p->lock = true;
  p->lock_classes = ncls;
  if (getenv("PTAP_TRACE"))
    fprintf(stderr,
            "[ptap] lockstep plan: %d tiles, %d classes, programs %llu + %llu entries, tile <= %d A entries, "
            "smem %zu B\n",
            ntiles, ncls, h[1], h[2], l.acap, lock_smem_bytes(l));
  return PTAP_OK;
}

// the lockstep kernel stages A by TMA bulk copies: 16-byte aligned arrays
static bool lock_usable(const ptap_plan *p, const Ops &op) {
  return p->lock && (((uintptr_t)op.ad_col | (uintptr_t)op.ad_val) & 15) == 0;
}

// Part 2 (C and the staging allocated): position maps (unless the row-union
// pass already wrote them), then drop the transient patterns.  Falls back to
// the hash path if a target row is wider than a byte can address.
ptap_status build_maps(ptap_plan *p, const Ops &op, const ptap_operands *ops, cudaStream_t st) {
  p->mapped = false;
  if (!p->want_maps) return PTAP_OK;
  bool ok = p->pmap_ready;
  if (!ok) {
    CKS(alloc_pmap(p, op, ops, st, &ok));
    if (ok) {
      OuterTargets tg{p->c_rp, p->c_col, p->c_val, p->s_nrows, p->s_rows, p->s_rp, p->s_col, p->s_val};
      CK(launch_build_pmap(op, (unsigned long long)p->nloc, p->maps, p->mo, tg, p->d_status, st));
      p->cnt.kernel_launches++;
    }
  }
  p->mapped = ok;
  pfree(p, p->pat, st);
  pfree(p, p->pat_rp, st);
  p->mo = MapOut{};
  if (ok) {
    if (!p->smap_interned)
      CKS(intern_map(p, p->maps.smap, p->maps.smap_rp, p->nloc, p->smap_bytes, true, &p->smap_bytes, st));
    p->smap_interned = true;
    if (!p->pmap_interned)
      CKS(intern_map(p, p->maps.pmap, p->maps.pmap_rp, p->nloc, p->pmap_bytes, false, &p->pmap_bytes, st));
    p->pmap_interned = true;
    p->cnt.numeric_path = 1;
    p->cnt.map_bytes = p->smap_bytes + p->pmap_bytes;
    CKS(build_tile(p, op, ops, st));
    if (p->tile) {
      p->cnt.numeric_path = 2;
      CKS(build_lock(p, op, ops, st));  // its fold walks the class programs when the plan is eligible
    }
  }
  // C row start per P_d entry for the q4a outer phase (4 B per P entry)
  if (ok && p->q4a && !p->tile && p->c_nnz < INT32_MAX && !getenv("PTAP_NO_CBASE")) {
    CKS(palloc(p, &p->maps.cbase, ops->p_diag.nnz, CAT_PLAN, st));
    CK(launch_build_cbase(ops->p_diag.nnz, op.pd_col, p->c_rp, p->maps.cbase, st));
    p->cnt.kernel_launches++;
    CKS(build_lock(p, op, ops, st));
    if (p->lock) p->cnt.numeric_path = 3;
  }
  if (!ok) {
    pfree(p, p->maps.smap_rp, st);
    pfree(p, p->maps.smap, st);
    pfree(p, p->maps.nap, st);
    pfree(p, p->maps.poff, st);
  }
  return PTAP_OK;
}

ptap_status free_maps(ptap_plan *p, cudaStream_t st) {
  free_tile(p, st);
  free_lock(p, st);
  pfree(p, p->maps.smap_rp, st); pfree(p, p->maps.pmap_rp, st);
  pfree(p, p->maps.smap, st); pfree(p, p->maps.pmap, st);
  pfree(p, p->maps.nap, st); pfree(p, p->maps.po_srow, st);
  pfree(p, p->maps.poff, st); pfree(p, p->maps.cbase, st);
  pfree(p, p->qa_rest, st);
  p->qa_rest_n = 0;
  p->qa_runs.clear();
  p->mapped = false;
  return PTAP_OK;
}

// C rows as unions of pattern rows (CSR pat_rp/pat: AP rows, or the two-step
// C~ rows) over each C row's contributors (t_rp/t_row: P_d^T).  With pm_op,
// the fill pass also writes the all-at-once position maps.  PTAP_ERR_VALUE:
// some union outgrew the per-row table (the caller takes the arena path).
ptap_status c_rows_by_union(ptap_plan *p, const int64_t *t_rp, const int32_t *t_row, const int64_t *pat_rp,
                            const int32_t *pat, const Ops *pm_op, const ptap_operands *pm_ops, cudaStream_t st) {
  const int64_t ncl = p->ncl;
  int64_t *cnt = nullptr, *scratch = nullptr;
  CKS(palloc(p, &cnt, ncl, CAT_TRANSIENT, st));
  CKS(palloc(p, &scratch, scan_scratch_elems(ncl), CAT_TRANSIENT, st));
  CK(launch_c_union(false, ncl, t_rp, t_row, pat_rp, pat, nullptr, cnt, nullptr, nullptr, nullptr, nullptr, nullptr,
                    nullptr, p->d_status, st));
  int s1 = 0;
  CKS(read_status(p, st, &s1));
  ptap_status ret = PTAP_OK;
  if (s1 & ST_TABLE_FULL) {
    ret = PTAP_ERR_VALUE;
  } else {
    CKS(palloc(p, &p->c_rp, ncl + 1, CAT_OUTPUT, st));
    CK(scan_exclusive(cnt, p->c_rp, ncl, scratch, st));
    int64_t nnz = 0;
    CK(cudaMemcpyAsync(&nnz, p->c_rp + ncl, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    p->c_nnz = nnz;
    CKS(palloc(p, &p->c_col, nnz, CAT_OUTPUT, st));
    bool pm_ok = false;
    if (pm_op) CKS(alloc_pmap(p, *pm_op, pm_ops, st, &pm_ok));
    CK(launch_c_union(true, ncl, t_rp, t_row, pat_rp, pat, nullptr, nullptr, p->c_rp, p->c_col,
                      pm_ok ? pm_op->pd_rp : nullptr, pm_ok ? pm_op->pd_col : nullptr,
                      pm_ok ? p->maps.pmap_rp : nullptr, pm_ok ? p->maps.pmap : nullptr, p->d_status, st));
    p->pmap_ready = pm_ok;
    p->cnt.kernel_launches += 1;
  }
  p->cnt.kernel_launches += 2;
  pfree(p, cnt, st);
  pfree(p, scratch, st);
  return ret;
}

// C's structure without an arena (all-at-once, a rank that neither sends nor
// receives): maps-only outer pass over the local rows, P_d^T, then the row
// unions of the contributors' sorted AP rows, which also write the position
// maps.
// the deferred slot-map buffer, full size, for the unchunked passes
ptap_status ensure_smap(ptap_plan *p, cudaStream_t st) {
  if (!p->smap_deferred) return PTAP_OK;
  CKS(palloc(p, &p->maps.smap, p->smap_bytes + 16, CAT_PLAN, st));
  p->mo.smap = p->maps.smap;
  p->smap_deferred = false;
  return PTAP_OK;
}

// The maps-only outer-product pass over row chunks, each chunk's slot maps
// interned as soon as they are written, so the per-row maps (1.5 GB on
// config 3) never exist at once: every row of the plan is in the identity
// bin 0 (one-rank structure).  The chunk pools are concatenated (a row class
// recurs in every chunk, at ~10 KB per chunk on config 3).
ptap_status chunked_slot_maps(ptap_plan *p, const Ops &op, cudaStream_t st, bool *done) {
  *done = false;
  BinSet &bs = p->bins_local;
  const int64_t n = p->nloc;
  if (!p->smap_deferred || !p->q4_sym || !bs.identity0 || bs.count[0] != n || bs.count[1] || bs.count[2] ||
      bs.count[3] || n < 4 * 65536 || getenv("PTAP_NO_INTERN"))
    return PTAP_OK;
  p->smap_deferred = false;
  const int K = std::max<int64_t>(2, std::min<int64_t>(16, p->smap_bytes >> 27));  // ~128 MB chunks
  std::vector<int64_t> rb(K + 1), off(K + 1);
  for (int c = 0; c <= K; ++c) rb[c] = n * c / K;
  for (int c = 0; c <= K; ++c)
    CK(cudaMemcpyAsync(&off[c], p->maps.smap_rp + rb[c], sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  int64_t *gout = nullptr;
  CKS(palloc(p, &gout, n + 1, CAT_PLAN, st));
  std::vector<uint8_t *> pools(K, nullptr);
  std::vector<int64_t> pbytes(K, 0);
  int64_t cum = 0;
  Arena none{nullptr, 0};
  for (int c = 0; c < K; ++c) {
    const int64_t r0 = rb[c], r1 = rb[c + 1], nc = r1 - r0;
    const int64_t base = off[c] & ~int64_t(3), total = off[c + 1] - base;
    uint8_t *chunk = nullptr;
    int64_t *crp = nullptr;
    CKS(palloc(p, &chunk, total + 16, CAT_TRANSIENT, st));
    MapOut mc = p->mo;
    mc.smap = chunk - base;  // the kernel writes at smap_rp[i]
    CK(launch_outer_symbolic_q4(op, nullptr, (unsigned long long)nc, 0, 1, none, none, mc, p->d_status, st,
                                (int)r0));
    CKS(palloc(p, &crp, nc + 1, CAT_TRANSIENT, st));
    CK(launch_offsets_shift(nc + 1, p->maps.smap_rp + r0, base, -1, crp, st));
    int64_t pb = 0;
    CKS(intern_map(p, chunk, crp, nc, total, true, &pb, st));
    pb = (pb + 3) & ~int64_t(3);
    CK(launch_offsets_shift(nc, crp, 0, cum, gout + r0, st));
    pfree(p, crp, st);
    pools[c] = chunk;
    pbytes[c] = pb;
    cum += pb;
    p->cnt.kernel_launches += 3;
  }
  uint8_t *pool = nullptr;
  CKS(palloc(p, &pool, cum + 16, CAT_PLAN, st));
  int64_t at = 0;
  for (int c = 0; c < K; ++c) {
    if (pbytes[c]) CK(cudaMemcpyAsync(pool + at, pools[c], pbytes[c], cudaMemcpyDeviceToDevice, st));
    at += pbytes[c];
    pfree(p, pools[c], st);
  }
  CK(cudaMemsetAsync(pool + cum, 0, 16, st));
  pfree(p, p->maps.smap_rp, st);
  p->maps.smap = pool;
  p->maps.smap_rp = gout;
  p->smap_bytes = cum;
  p->mo.smap = nullptr;
  p->mo.smap_rp = nullptr;
  p->smap_interned = true;
  *done = true;
  return PTAP_OK;
}

// Position maps chunk by chunk once C's pattern is known: each fine-row
// window's maps are found by binary search in its target C rows
// (k_build_pmap) and interned at once, so the per-row maps (0.87 GB on
// config 3) never exist together with the AP patterns they are built from.
ptap_status chunked_pos_maps(ptap_plan *p, const Ops &op, cudaStream_t st, bool *done) {
  *done = false;
  const int64_t n = p->nloc;
  if (getenv("PTAP_NO_MAP_CHUNKS") || getenv("PTAP_NO_INTERN") || op.po_rp != nullptr || n < 4 * 65536) return PTAP_OK;
  unsigned long long *mx = p->d_u64 + 12;
  CK(cudaMemsetAsync(mx, 0, sizeof(unsigned long long), st));
  CK(launch_max_rowlen(p->ncl, p->c_rp, mx, st));
  unsigned long long cmax = 0;
  CK(cudaMemcpyAsync(&cmax, mx, sizeof(cmax), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (cmax > 256) return PTAP_OK;  // positions must fit a byte: the caller takes the hash path
  int64_t *plen = nullptr, *scratch = nullptr, *unused = nullptr, *prp = nullptr;
  CKS(palloc(p, &plen, n, CAT_TRANSIENT, st));
  CKS(palloc(p, &unused, n, CAT_TRANSIENT, st));
  CKS(palloc(p, &scratch, scan_scratch_elems(n), CAT_TRANSIENT, st));
  CK(launch_map_lengths(n, op.pd_rp, op.po_rp, p->apub, p->ap_nnz, unused, plen, st));
  CKS(palloc(p, &prp, n + 1, CAT_TRANSIENT, st));
  CK(scan_exclusive(plen, prp, n, scratch, st));
  pfree(p, plen, st);
  pfree(p, unused, st);
  pfree(p, scratch, st);
  int64_t tot = 0;
  CK(cudaMemcpyAsync(&tot, prp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const int K = (int)std::max<int64_t>(2, std::min<int64_t>(16, tot >> 27));
  std::vector<int64_t> rb(K + 1), off(K + 1);
  for (int c = 0; c <= K; ++c) rb[c] = n * c / K;
  for (int c = 0; c <= K; ++c) CK(cudaMemcpyAsync(&off[c], prp + rb[c], sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  int64_t *gout = nullptr;
  CKS(palloc(p, &gout, n + 1, CAT_PLAN, st));
  std::vector<uint8_t *> pools(K, nullptr);
  std::vector<int64_t> pbytes(K, 0);
  int64_t cum = 0;
  OuterTargets tg{p->c_rp, p->c_col, nullptr, 0, nullptr, nullptr, nullptr, nullptr};
  for (int c = 0; c < K; ++c) {
    const int64_t r0 = rb[c], r1 = rb[c + 1], nc = r1 - r0;
    const int64_t base = off[c] & ~int64_t(3), total = off[c + 1] - base;
    uint8_t *chunk = nullptr;
    int64_t *crp = nullptr;
    CKS(palloc(p, &chunk, total + 16, CAT_TRANSIENT, st));
    MapArgs mc = p->maps;
    mc.pmap = chunk - base;
    mc.pmap_rp = prp;
    CK(launch_build_pmap(op, (unsigned long long)nc, mc, p->mo, tg, p->d_status, st, r0));
    CKS(palloc(p, &crp, nc + 1, CAT_TRANSIENT, st));
    CK(launch_offsets_shift(nc + 1, prp + r0, base, -1, crp, st));
    int64_t pb = 0;
    CKS(intern_map(p, chunk, crp, nc, total, false, &pb, st));
    pb = (pb + 3) & ~int64_t(3);
    CK(launch_offsets_shift(nc, crp, 0, cum, gout + r0, st));
    pfree(p, crp, st);
    pools[c] = chunk;
    pbytes[c] = pb;
    cum += pb;
    p->cnt.kernel_launches += 3;
  }
  pfree(p, prp, st);
  uint8_t *pool = nullptr;
  CKS(palloc(p, &pool, cum + 16, CAT_PLAN, st));
  int64_t at = 0;
  for (int c = 0; c < K; ++c) {
    if (pbytes[c]) CK(cudaMemcpyAsync(pool + at, pools[c], pbytes[c], cudaMemcpyDeviceToDevice, st));
    at += pbytes[c];
    pfree(p, pools[c], st);
  }
  CK(cudaMemsetAsync(pool + cum, 0, 16, st));
  p->maps.pmap = pool;
  p->maps.pmap_rp = gout;
  p->pmap_bytes = cum;
  CKS(palloc(p, &p->maps.po_srow, 1, CAT_PLAN, st));  // no P_o entries
  p->pmap_ready = true;
  p->pmap_interned = true;
  *done = true;
  return PTAP_OK;
}

ptap_status c_by_unions(ptap_plan *p, const Ops &op, const ptap_operands *ops, cudaStream_t st, Tracer *tr) {
  Arena none{nullptr, 0};
  bool chunked = false;
  CKS(chunked_slot_maps(p, op, st, &chunked));
  if (!chunked) CKS(ensure_smap(p, st));
  if (!chunked)
    CKS(for_bins(p, p->bins_local, [&](const LaunchShape &s, const int32_t *rows, unsigned long long n) {
      if (s.bin == 0 && p->q4_sym && p->mo.smap)
        return launch_outer_symbolic_q4(op, rows, n, 0, 1, none, none, p->mo, p->d_status, st);
      return launch_outer_symbolic(s, op, rows, n, 0, 1, none, none, p->mo, p->d_status, st);
    }));
  p->cnt.symbolic_row_kernel_calls += p->bins_local.selected;
  int s0 = 0;
  CKS(read_status(p, st, &s0));
  CKS(status_to_error(s0, "symbolic"));
  tr->mark(st, "local outer symbolic (maps)");
  if (p->mo.smap) {  // the slot maps are complete: intern them before C's pass
    CKS(intern_map(p, p->maps.smap, p->maps.smap_rp, p->nloc, p->smap_bytes, true, &p->smap_bytes, st));
    p->mo.smap = nullptr;
    p->mo.smap_rp = nullptr;
    p->smap_interned = true;
    tr->mark(st, "slot maps interned");
  }
  // P_d^T structure: fine rows contributing to each local C row
  const int64_t ncl = p->ncl, pnnz = ops->p_diag.nnz;
  int64_t *cnt = nullptr, *t_rp = nullptr, *scratch = nullptr;
  int32_t *t_row = nullptr;
  CKS(palloc(p, &cnt, ncl, CAT_TRANSIENT, st));
  CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (ncl > 0 ? ncl : 1), st));
  if (pnnz > 0) CK(launch_count_cols(pnnz, op.pd_col, cnt, st));
  CKS(palloc(p, &t_rp, ncl + 1, CAT_TRANSIENT, st));
  CKS(palloc(p, &scratch, scan_scratch_elems(ncl), CAT_TRANSIENT, st));
  CK(scan_exclusive(cnt, t_rp, ncl, scratch, st));
  CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (ncl > 0 ? ncl : 1), st));
  CKS(palloc(p, &t_row, pnnz, CAT_TRANSIENT, st));
  CK(launch_transpose_scatter(p->nloc, op.pd_rp, op.pd_col, t_rp, cnt, t_row, nullptr, st));
  p->cnt.kernel_launches += 3;
  pfree(p, cnt, st);
  pfree(p, scratch, st);
  tr->mark(st, "P_d^T");
  // position maps: chunked after the unions (bounded memory), or written by
  // the unions' fill pass
  const bool chunk_pm = !getenv("PTAP_NO_MAP_CHUNKS") && !getenv("PTAP_NO_INTERN") && op.po_rp == nullptr &&
                        p->nloc >= 4 * 65536;
  ptap_status ret = c_rows_by_union(p, t_rp, t_row, p->mo.pat_rp, p->mo.pat, chunk_pm ? nullptr : &op, ops, st);
  pfree(p, t_rp, st);
  pfree(p, t_row, st);
  tr->mark(st, "C rows by unions");
  if (ret == PTAP_OK && chunk_pm) {
    bool done = false;
    CKS(chunked_pos_maps(p, op, st, &done));
    tr->mark(st, "position maps (chunked)");
  }
  return ret;
}

// each bin's row list in locality order (launch_row_order); an identity bin
// becomes an explicit list
ptap_status order_bins(ptap_plan *p, BinSet &bs, const Ops &op, cudaStream_t st) {
  for (int q = 0; q < NBINS; ++q) {
    const int64_t n = bs.count[q];
    if (n < 2) continue;
    const bool ident = q == 0 && bs.identity0;
    int32_t *out = nullptr;
    CKS(palloc(p, &out, n, CAT_PLAN, st));
    const size_t bytes = row_order_scratch_bytes(n);
    uint8_t *scratch = nullptr;
    CKS(palloc(p, &scratch, (int64_t)bytes, CAT_TRANSIENT, st));
    CK(launch_row_order(n, ident ? nullptr : bs.rows[q], out, op.pd_rp, op.pd_col, scratch, bytes, st));
    p->cnt.kernel_launches += 2;
    pfree(p, scratch, st);
    if (!ident) pfree(p, bs.rows[q], st);
    bs.rows[q] = out;
    if (ident) bs.identity0 = false;
  }
  return PTAP_OK;
}

// Several ranks: the q4a kernel reads only A_d and P_d, so the local bin-0
// rows whose A_o and P_o rows are empty -- the interior of a row block --
// can run it; this finds their runs of consecutive rows (>= 256 rows, at
// most 64 runs) and keeps the other bin-0 rows as a list for the q4 kernel.
ptap_status build_q4a_runs(ptap_plan *p, const Ops &op, const ptap_operands *ops, cudaStream_t st) {
  BinSet &bs = p->bins_local;
  if (!p->mapped || !p->q4 || p->q4a || p->alg != PTAP_ALLATONCE || bs.count[0] == 0 ||
      getenv("PTAP_NO_Q4A_RUNS") || p->c_nnz >= INT32_MAX)
    return PTAP_OK;
  const int64_t n = p->nloc, nb0 = bs.count[0];
  uint8_t *flag = nullptr;
  CKS(palloc(p, &flag, n, CAT_TRANSIENT, st));
  CK(cudaMemsetAsync(flag, 0, n > 0 ? n : 1, st));
  const int32_t *b0 = bs.identity0 ? nullptr : bs.rows[0];  // identity bin: rows 0..n-1
  CK(launch_pure_rows(nb0, b0, op, flag, st));
  std::vector<uint8_t> hf(n);
  std::vector<int32_t> rows(nb0);
  CK(cudaMemcpyAsync(hf.data(), flag, n, cudaMemcpyDeviceToHost, st));
  if (b0) CK(cudaMemcpyAsync(rows.data(), b0, nb0 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  else for (int64_t i = 0; i < nb0; ++i) rows[i] = (int32_t)i;
  CK(cudaStreamSynchronize(st));
  p->cnt.kernel_launches++;
  struct FlagGuard {
    ptap_plan *p; uint8_t *&f; cudaStream_t st;
    ~FlagGuard() { pfree(p, f, st); }
  } guard{p, flag, st};
  std::vector<std::pair<int64_t, int64_t>> runs;
  for (int64_t i = 0; i < n;) {
    if (!hf[i]) { ++i; continue; }
    int64_t j = i;
    while (j < n && hf[j]) ++j;
    if (j - i >= 256) runs.emplace_back(i, j - i);
    i = j;
  }
  if (runs.empty() || runs.size() > 64) return PTAP_OK;
  std::vector<uint8_t> in_run(n, 0);
  for (auto &r : runs) std::fill(in_run.begin() + r.first, in_run.begin() + r.first + r.second, 1);
  std::vector<int32_t> rest;
  rest.reserve(nb0);
  for (int32_t i : rows)
    if (!in_run[i]) rest.push_back(i);
  if (!rest.empty()) {
    CKS(palloc(p, &p->qa_rest, (int64_t)rest.size(), CAT_PLAN, st));
    CK(cudaMemcpyAsync(p->qa_rest, rest.data(), rest.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  p->qa_rest_n = (int64_t)rest.size();
  if (!p->maps.cbase) {
    CKS(palloc(p, &p->maps.cbase, ops->p_diag.nnz, CAT_PLAN, st));
    CK(launch_build_cbase(ops->p_diag.nnz, op.pd_col, p->c_rp, p->maps.cbase, st));
    p->cnt.kernel_launches++;
  }
  p->qa_runs = runs;
  // the runs' whole 64-row tiles take the class-lockstep pass
  CKS(build_lock(p, op, ops, st, flag));
  if (p->lock) p->cnt.numeric_path = 3;
  if (getenv("PTAP_TRACE")) {
    int64_t in = 0;
    for (auto &r : runs) in += r.second;
    fprintf(stderr, "[ptap] q4a runs: %zu covering %lld rows, %lld bin-0 rows through q4\n", runs.size(), (long long)in,
            (long long)p->qa_rest_n);
  }
  return PTAP_OK;
}

ptap_status run_outer_numeric(ptap_plan *p, const Ops &op, BinSet &bs, int do_send, int do_local, cudaStream_t st) {
  OuterTargets tg{p->c_rp, p->c_col, p->c_val, p->s_nrows, p->s_rows, p->s_rp, p->s_col, p->s_val};
  if (p->mapped) {
    for (int q = 0; q < NBINS; ++q) {
      if (bs.count[q] == 0) continue;
      const int32_t *rows = (q == 0 && bs.identity0) ? nullptr : bs.rows[q];
      if (q == 0 && !p->qa_runs.empty() && &bs == &p->bins_local && do_local && !do_send) {
        const bool lk = lock_usable(p, op);
        if (lk) {
          CK(launch_lock_permute_f64(p->nloc, op.pd_rp, p->la.pq, p->la.ltab, op.pd_val, p->la.Q, st));
          p->cnt.kernel_launches++;
        }
        for (auto &r : p->qa_runs) {
          int64_t lo = r.first, hi = r.first + r.second;
          if (lk) {  // whole tiles inside the run in lockstep, its edges row by row
            const int64_t t0 = (lo + LOCK_TILE - 1) / LOCK_TILE, t1 = hi / LOCK_TILE;
            if (t1 > t0) {
              if (t0 * LOCK_TILE > lo) {
                CK(launch_outer_numeric_q4a(op, (unsigned long long)(t0 * LOCK_TILE - lo), p->maps, tg, p->d_status, st,
                                            (int)lo));
                p->cnt.kernel_launches++;
              }
              CK(launch_lock_numeric(op, p->la, p->c_val, (int)t0, (int)t1, p->d_status, st));
              p->cnt.kernel_launches++;
              lo = t1 * LOCK_TILE;
            }
          }
          if (hi > lo) {
            CK(launch_outer_numeric_q4a(op, (unsigned long long)(hi - lo), p->maps, tg, p->d_status, st, (int)lo));
            p->cnt.kernel_launches++;
          }
        }
        if (p->qa_rest_n > 0) {
          CK(launch_outer_numeric_mapped(3, op, p->qa_rest, (unsigned long long)p->qa_rest_n, p->maps, tg, do_send,
                                         do_local, p->d_status, st));
          p->cnt.kernel_launches++;
        }
        continue;
      }
      // q4a plans have no P_o (one-rank structure), so a merged pass's send
      // half is empty and its fused loop is the local loop
      if (q == 0 && p->q4a && bs.identity0 && do_local && (!do_send || op.po_rp == nullptr)) {
        if (p->tile) {  // deterministic owner-computes pass: writes every C entry once
          CK(launch_tile_numeric(op, p->maps, p->ta, p->lock ? p->la : LockArgs{}, p->c_rp, p->c_val, 0, p->ta.nblk, true,
                                 st));
          p->cnt.kernel_launches += 2;
          continue;
        }
        if (lock_usable(p, op)) {  // rows of one class in lockstep; P's values class-major first
          CK(launch_lock_permute_f64(p->nloc, op.pd_rp, p->la.pq, p->la.ltab, op.pd_val, p->la.Q, st));
          CK(launch_lock_numeric(op, p->la, p->c_val, 0, p->la.ntiles, p->d_status, st));
          p->cnt.kernel_launches += 2;
          continue;
        }
        CK(launch_outer_numeric_q4a(op, (unsigned long long)bs.count[q], p->maps, tg, p->d_status, st, 0));
        p->cnt.kernel_launches++;
        continue;
      }
      const int kb = q == 0 ? (p->q4 ? 3 : 0) : (q == 1 && !getenv("PTAP_NO_MAPPED16") ? 2 : 1);
      CK(launch_outer_numeric_mapped(kb, op, rows, (unsigned long long)bs.count[q], p->maps, tg, do_send,
                                     do_local, p->d_status, st));
      p->cnt.kernel_launches++;
    }
    return PTAP_OK;
  }
  return for_bins(p, bs, [&](const LaunchShape &s, const int32_t *rows, unsigned long long n) {
    return launch_outer_numeric(s, op, rows, n, do_send, do_local, tg, p->d_status, st);
  });
}

}  // namespace

// ============================================================================
extern "C" {

const char *ptap_last_error(void) { return g_err.c_str(); }
const char *ptap_version(void) { return "ptap_b200 0.1 (sm_100a)"; }

ptap_status ptap_plan_create(int algorithm, const ptap_operands *ops, ptap_plan **out) {
  if (!out) return fail(PTAP_ERR_VALUE, "null output");
  if (algorithm < 0 || algorithm > 2) return fail(PTAP_ERR_VALUE, "unknown algorithm");
  CKS(validate(ops));
  reserve_pool(ops);
  ptap_plan *p = new ptap_plan();
  ++g_live_plans;
  p->alg = algorithm;
  p->nloc = ops->n_local;
  p->m = ops->m_global;
  p->c_lo = ops->c_lo;
  p->c_hi = ops->c_hi;
  p->ncl = ops->c_hi - ops->c_lo;
  p->colmap_len = ops->p_colmap_len;
  cudaError_t e = cudaMalloc(&p->d_status, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&p->d_u64, 24 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(p->d_status, 0, sizeof(int));
  if (e != cudaSuccess) {
    delete p;
    --g_live_plans;
    return fail(PTAP_ERR_CUDA, std::string("plan create: ") + cudaGetErrorString(e));
  }
  *out = p;
  return PTAP_OK;
}

ptap_status ptap_plan_set_option(ptap_plan *p, const char *key, int64_t value) {
  if (!p || !key) return fail(PTAP_ERR_VALUE, "null argument");
  if (!strcmp(key, "deterministic")) {
    p->deterministic = value != 0;
    return PTAP_OK;
  }
  if (!strcmp(key, "single_shot")) {
    p->single_shot = value != 0;
    if (p->single_shot) p->maps_opt = 0;  // nothing kept per row: later passes run the hash numeric path
    return PTAP_OK;
  }
  if (!strcmp(key, "lockstep")) {
    p->lock_opt = value < 0 ? -1 : (value ? 1 : 0);
    return PTAP_OK;
  }
  if (!strcmp(key, "maps")) {
    p->maps_opt = value < 0 ? -1 : (value ? 1 : 0);
    return PTAP_OK;
  }
  return fail(PTAP_ERR_VALUE, std::string("unknown plan option '") + key + "'");
}

ptap_status ptap_plan_values_ready(ptap_plan *p, int *ready) {
  if (!p || !ready) return fail(PTAP_ERR_VALUE, "null argument");
  *ready = p->values_ready ? 1 : 0;
  return PTAP_OK;
}

ptap_status ptap_plan_destroy(ptap_plan *p) {
  if (!p) return PTAP_OK;
  cudaDeviceSynchronize();
  for (auto &kv : p->allocs) cudaFreeAsync(kv.first, 0);
  cudaStreamSynchronize(0);
  cudaFree(p->d_status);
  cudaFree(p->d_u64);
  if (p->h_status) cudaFreeHost(p->h_status);
  if (p->status_ev) cudaEventDestroy(p->status_ev);
  delete p;
  // the last plan gone: give the pool's memory back to the driver (torch,
  // NCCL), unless PTAP_POOL_KEEP asks to keep it for the next plan
  if (--g_live_plans <= 0 && !getenv("PTAP_POOL_KEEP")) trim_pool();
  return PTAP_OK;
}

ptap_status ptap_symbolic_send(ptap_plan *p, const ptap_operands *ops, void *stream) {
  if (!p) return fail(PTAP_ERR_VALUE, "null plan");
  CKS(validate(ops));
  cudaStream_t st = (cudaStream_t)stream;
  CKS(record_image(p, ops, st));
  Ops op = make_ops(ops);
  Tracer tr;
  if (p->nloc > 0) p->avg_p_row = (double)(ops->p_diag.nnz + ops->p_off.nnz) / (double)p->nloc;
  CKS(ap_sizes(p, op, &p->ap_nnz, st, &p->apub));
  tr.mark(st, "ap_sizes");
  CKS(sample_row_structures(p, op, st));
  tr.mark(st, "row-structure sample");
  if (p->alg != PTAP_TWO_STEP) CKS(prepare_maps(p, op, ops, st));
  tr.mark(st, "prepare_maps");
  if (p->alg == PTAP_TWO_STEP) {
    // C~ = A P (src/spgemm.py:184-202), booked as auxiliary
    CKS(palloc(p, &p->ct_rp, p->nloc + 1, CAT_AUX, st));
    int64_t *scratch = nullptr;
    CKS(palloc(p, &scratch, scan_scratch_elems(p->nloc), CAT_TRANSIENT, st));
    CK(scan_exclusive(p->ap_nnz, p->ct_rp, p->nloc, scratch, st));
    pfree(p, scratch, st);
    CK(cudaMemcpyAsync(&p->ct_nnz, p->ct_rp + p->nloc, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CKS(palloc(p, &p->ct_col, p->ct_nnz, CAT_AUX, st));
    CKS(palloc(p, &p->ct_val, p->ct_nnz, CAT_AUX, st));
    CKS(build_bins(p, p->bins_all, p->nloc, p->ap_nnz, op.pd_rp, op.po_rp, 0, true, CAT_PLAN, st));
    CKS(for_bins(p, p->bins_all, [&](const LaunchShape &s, const int32_t *rows, unsigned long long n) {
      return launch_ct_fill(s, op, rows, n, p->ct_rp, p->ct_col, p->d_status, st);
    }));
    int32_t *wide = nullptr;
    CKS(palloc(p, &wide, p->ct_nnz / 1024 + 2, CAT_TRANSIENT, st));
    CK(cudaMemsetAsync(p->d_u64 + 6, 0, sizeof(unsigned long long), st));
    CK(launch_sort_rows(p->nloc, p->ct_rp, p->ct_col, nullptr, wide, p->d_u64 + 6, st));
    unsigned long long nwide = 0;
    CK(cudaMemcpyAsync(&nwide, p->d_u64 + 6, sizeof(nwide), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(launch_sort_rows_block((int64_t)nwide, wide, p->ct_rp, p->ct_col, nullptr, p->d_status, st));
    pfree(p, wide, st);
    // explicit local transposes of P_d and P_o (src/tripleproduct.py:393-399)
    CKS(build_transpose(p, p->ptd, p->ncl, op.pd_rp, op.pd_col, ops->p_diag.nnz, st));
    CKS(build_transpose(p, p->pto, p->colmap_len, ops->p_off.row_ptr, ops->p_off.col, ops->p_off.nnz, st));
    // send structure C_s = P_o^T C~ (no remote rows of C~ needed)
    Arena send{nullptr, 0};
    CKS(arena_alloc(p, send, p->bound_send + 16, st));
    CKS(with_arena_retry(p, send, st, [&]() -> ptap_status {
      CK(launch_ptc_symbolic(p->pto.nrows, p->pto.rp, p->pto.row, ops->p_colmap, 0, p->ct_rp, p->ct_col, send, p->m,
                             p->d_status, st));
      p->cnt.kernel_launches++;
      return PTAP_OK;
    }));
    CKS(arena_to_staging(p, send, CAT_AUX, st));
    pfree(p, send.keys, st);
    p->cnt.symbolic_row_kernel_calls += p->nloc;
  } else {
    bool merged = p->alg == PTAP_MERGED;
    // merged with nothing to send: the fused loop is the local loop, whose
    // structure is then built in symbolic_local exactly as for all-at-once
    p->merged_deferred = merged && ops->p_off.nnz == 0 && !getenv("PTAP_NO_UNION");
    if (p->merged_deferred) {
      CKS(build_bins(p, p->bins_all, p->nloc, p->ap_nnz, op.pd_rp, op.po_rp, 3, true, CAT_PLAN, st));
      CKS(build_bins(p, p->bins_local, p->nloc, p->ap_nnz, op.pd_rp, op.po_rp, 2, true, CAT_PLAN, st));
      merged = false;  // the send pass below has no rows
    } else if (merged) {
      CKS(build_bins(p, p->bins_all, p->nloc, p->ap_nnz, op.pd_rp, op.po_rp, 3, true, CAT_PLAN, st));
      p->cnt.symbolic_row_kernel_calls += p->bins_all.selected;
    } else {
      CKS(build_bins(p, p->bins_send, p->nloc, p->ap_nnz, op.pd_rp, op.po_rp, 1, true, CAT_PLAN, st));
      CKS(build_bins(p, p->bins_local, p->nloc, p->ap_nnz, op.pd_rp, op.po_rp, 2, true, CAT_PLAN, st));
      p->cnt.symbolic_row_kernel_calls += p->bins_send.selected;
    }
    Arena send{nullptr, 0};
    CKS(arena_alloc(p, send, p->bound_send + 16, st));
    if (merged) CKS(arena_alloc(p, p->local_arena, local_arena_estimate(p, 0), st, (unsigned long long)p->ncl));
    BinSet empty_bins{};
    BinSet &bs = merged ? p->bins_all : (p->merged_deferred ? empty_bins : p->bins_send);
    auto pass = [&]() -> ptap_status {
      return for_bins(p, bs, [&](const LaunchShape &s, const int32_t *rows, unsigned long long n) {
        if (s.bin == 0 && p->q4_sym && p->mo.smap)
          return launch_outer_symbolic_q4(op, rows, n, 1, merged ? 1 : 0, p->local_arena, send, p->mo, p->d_status, st);
        return launch_outer_symbolic(s, op, rows, n, 1, merged ? 1 : 0, p->local_arena, send, p->mo, p->d_status, st);
      });
    };
    if (merged) {
      // the fused pass inserts into both arenas; grow the local one on overflow
      for (int attempt = 0;; ++attempt) {
        CKS(pass());
        int s = 0;
        CKS(read_status(p, st, &s));
        if (!(s & ST_ARENA_FULL)) {
          if (s) return status_to_error(s, "merged symbolic");
          break;
        }
        if (attempt > 8) return fail(PTAP_ERR_OOM, "symbolic arena kept overflowing");
        CKS(arena_grow(p, p->local_arena, st));
        CKS(arena_grow(p, send, st));
      }
    } else {
      CKS(with_arena_retry(p, send, st, pass));
    }
    tr.mark(st, "outer symbolic (send/merged)");
    CKS(arena_to_staging(p, send, CAT_PLAN, st));
    pfree(p, send.keys, st);
    tr.mark(st, "staging drain");
  }
  int s = 0;
  CKS(read_status(p, st, &s));
  if (s) return status_to_error(s, "symbolic send");
  p->cnt.nnz_staging = p->s_nnz;
  return PTAP_OK;
}

ptap_status ptap_plan_staging(ptap_plan *p, ptap_staging *out) {
  if (!p || !out) return fail(PTAP_ERR_VALUE, "null argument");
  out->nrows = p->s_nrows;
  out->nnz = p->s_nnz;
  out->rows = p->s_rows;
  out->row_ptr = p->s_rp;
  out->col = p->s_col;
  out->val = p->s_val;
  return PTAP_OK;
}

ptap_status ptap_symbolic_local(ptap_plan *p, const ptap_operands *ops, const ptap_received *recv, void *stream) {
  if (!p) return fail(PTAP_ERR_VALUE, "null plan");
  CKS(validate(ops));
  cudaStream_t st = (cudaStream_t)stream;
  Ops op = make_ops(ops);
  int64_t rnnz = recv ? recv->nnz : 0;
  Tracer tr;
  // nothing received and nothing sent (every target row local): C row by
  // row as unions of the contributors' AP rows, no global arena
  const bool local_loop_here = p->alg == PTAP_ALLATONCE || p->merged_deferred;
  bool use_union = local_loop_here && p->want_maps && !(recv && recv->nrows > 0) && ops->p_off.nnz == 0 &&
                   !getenv("PTAP_NO_UNION");
  if (use_union) {
    ptap_status us = c_by_unions(p, op, ops, st, &tr);
    if (us == PTAP_OK) goto c_allocated;
    if (us != PTAP_ERR_VALUE) return us;  // PTAP_ERR_VALUE: a union outgrew the table -> arena path
  }
  if (p->alg == PTAP_TWO_STEP && !(recv && recv->nrows > 0) && ops->p_off.nnz == 0 && !getenv("PTAP_NO_UNION")) {
    // C = P_d^T C~ row by row: unions of the C~ rows of each C row's contributors
    ptap_status us = c_rows_by_union(p, p->ptd.rp, p->ptd.row, p->ct_rp, p->ct_col, nullptr, nullptr, st);
    tr.mark(st, "C rows by unions");
    if (us == PTAP_OK) goto c_allocated;
    if (us != PTAP_ERR_VALUE) return us;
  }
  if (p->alg != PTAP_MERGED || p->merged_deferred)
    CKS(arena_alloc(p, p->local_arena, local_arena_estimate(p, rnnz), st, (unsigned long long)p->ncl));
  tr.mark(st, "local arena alloc");
  // single-shot: the same arena takes keys and values in one pass over A
  p->values_ready = false;
  if (p->single_shot && local_loop_here && !p->want_maps && !(recv && recv->nrows > 0) && ops->p_off.nnz == 0) {
    Arena &la = p->local_arena;
    double *avals = nullptr;
    for (int attempt = 0;; ++attempt) {
      if (attempt >= 8) return fail(PTAP_ERR_OOM, "single-shot arena kept overflowing");
      CKS(palloc(p, &avals, (int64_t)(la.mask + 1), CAT_TRANSIENT, st));
      CK(cudaMemsetAsync(avals, 0, sizeof(double) * (la.mask + 1), st));
      CKS(for_bins(p, p->bins_local, [&](const LaunchShape &s, const int32_t *rows, unsigned long long n) {
        return launch_outer_oneshot(s, op, rows, n, la, avals, p->d_status, st);
      }));
      int s = 0;
      CKS(read_status(p, st, &s));
      if (!(s & ST_ARENA_FULL)) {
        if (s) return status_to_error(s, "single-shot pass");
        break;
      }
      pfree(p, avals, st);  // a grown arena keeps the keys; the values are recomputed
      CKS(arena_grow(p, la, st));
    }
    p->cnt.symbolic_row_kernel_calls += p->bins_local.selected;
    p->cnt.numeric_row_kernel_calls += p->bins_local.selected;
    p->r_src_nnz_off.clear();
    p->r_nnz = 0;
    tr.mark(st, "single-shot outer pass");
    CKS(arena_to_csr(p, la, p->ncl, CAT_OUTPUT, &p->c_rp, &p->c_col, &p->c_nnz, nullptr, st, avals, &p->c_val));
    tr.mark(st, "C drain + sort (values)");
    pfree(p, avals, st);
    pfree(p, la.keys, st);
    la = Arena{nullptr, 0};
    p->values_ready = true;
    goto c_allocated;
  }
  {
  Arena &la = p->local_arena;
  if (local_loop_here) {
    CKS(ensure_smap(p, st));
    CKS(with_arena_retry(p, la, st, [&]() -> ptap_status {
      return for_bins(p, p->bins_local, [&](const LaunchShape &s, const int32_t *rows, unsigned long long n) {
        Arena none{nullptr, 0};
        if (s.bin == 0 && p->q4_sym && p->mo.smap)
          return launch_outer_symbolic_q4(op, rows, n, 0, 1, la, none, p->mo, p->d_status, st);
        return launch_outer_symbolic(s, op, rows, n, 0, 1, la, none, p->mo, p->d_status, st);
      });
    }));
    p->cnt.symbolic_row_kernel_calls += p->bins_local.selected;
  } else if (p->alg == PTAP_TWO_STEP) {
    CKS(with_arena_retry(p, la, st, [&]() -> ptap_status {
      CK(launch_ptc_symbolic(p->ptd.nrows, p->ptd.rp, p->ptd.row, nullptr, 0, p->ct_rp, p->ct_col, la, p->m,
                             p->d_status, st));
      p->cnt.kernel_launches++;
      return PTAP_OK;
    }));
  }
  // received structure (src/tripleproduct.py:191-200): owner rows only
  p->r_src_nnz_off.clear();
  p->r_nnz = rnnz;
  if (recv && recv->nrows > 0) {
    for (int k = 0; k <= recv->nsrc; ++k) p->r_src_nnz_off.push_back(recv->src_nnz_off[k]);
    CKS(with_arena_retry(p, la, st, [&]() -> ptap_status {
      CK(launch_arena_insert_batch(la, recv->nrows, recv->rows, recv->row_ptr, recv->col, p->m, p->c_lo, p->c_hi,
                                   p->d_status, st));
      p->cnt.kernel_launches++;
      return PTAP_OK;
    }));
  }
  tr.mark(st, "local outer symbolic + recv");
  // allocate C (src/tripleproduct.py:203-212, src/spgemm.py:71-104)
  CKS(arena_to_csr(p, la, p->ncl, CAT_OUTPUT, &p->c_rp, &p->c_col, &p->c_nnz, nullptr, st));
  tr.mark(st, "C drain + sort");
  pfree(p, la.keys, st);
  la = Arena{nullptr, 0};
  }
c_allocated:
  if (recv && recv->nrows > 0) {
    CKS(palloc(p, &p->r_slot, rnnz, CAT_PLAN, st));
    CK(launch_merge_slots(recv->nrows, recv->rows, recv->row_ptr, recv->col, p->c_lo, p->c_rp, p->c_col, p->r_slot,
                          p->d_status, st));
    p->cnt.kernel_launches++;
  }
  if (p->alg == PTAP_TWO_STEP) {
    int64_t *est = nullptr;
    CKS(palloc(p, &est, p->ncl > p->colmap_len ? p->ncl : p->colmap_len, CAT_TRANSIENT, st));
    CK(launch_ptc_est(p->ptd.nrows, nullptr, 0, 0, p->ncl, nullptr, p->c_rp, est, st));
    CKS(build_bins(p, p->bins_ptd, p->ptd.nrows, est, nullptr, nullptr, 0, true, CAT_PLAN, st));
    CK(launch_ptc_est(p->pto.nrows, ops->p_colmap, 0, 1, p->s_nrows, p->s_rows, p->s_rp, est, st));
    CKS(build_bins(p, p->bins_pto, p->pto.nrows, est, nullptr, nullptr, 0, true, CAT_PLAN, st));
    pfree(p, est, st);
    p->cnt.kernel_launches += 2;
  }
  tr.mark(st, "merge slots / two-step bins");
  if (p->alg != PTAP_TWO_STEP) CKS(build_maps(p, op, ops, st));
  tr.mark(st, "position maps");
  CKS(build_q4a_runs(p, op, ops, st));
  // C's values last: the position maps' transient peak is over by now
  if (!p->values_ready) {
    CKS(palloc(p, &p->c_val, p->c_nnz, CAT_OUTPUT, st));
    CK(cudaMemsetAsync(p->c_val, 0, sizeof(double) * (p->c_nnz > 0 ? p->c_nnz : 1), st));
  }
  if (p->rows_unstructured && !(p->alg != PTAP_TWO_STEP && p->mapped) && !getenv("PTAP_NO_ROW_ORDER")) {
    // an operator whose rows do not repeat: visit rows in aggregate order
    // (k_row_order_keys) -- the hash numeric path, and two-step's C~ = A P
    CKS(order_bins(p, p->bins_local, op, st));
    CKS(order_bins(p, p->bins_all, op, st));
    CKS(order_bins(p, p->bins_send, op, st));
    tr.mark(st, "row order");
  }
  pfree(p, p->ap_nnz, st);
  pfree(p, p->apub, st);
  int s = 0;
  CKS(read_status(p, st, &s));
  if (s & ST_DRIFT) {
    if (recv && recv->nrows > 0)
      return fail(PTAP_ERR_DRIFT, "received contribution rows outside the owned range or not in the structure");
  }
  if (s) return status_to_error(s, "symbolic local");
  p->cnt.nnz_c = p->c_nnz;
  p->cnt.symbolic_runs++;
  p->symbolic_done = true;
  return PTAP_OK;
}

// the tile pass is the whole local loop and stores every C entry: no zero fill
static bool tile_writes_all(const ptap_plan *p, const BinSet &bs, const Ops &op) {
  return p->tile && p->q4a && bs.identity0 && op.po_rp == nullptr && p->r_nnz == 0;
}

static ptap_status numeric_ready(ptap_plan *p) {
  if (!p) return fail(PTAP_ERR_VALUE, "null plan");
  if (p->released) return fail(PTAP_ERR_DRIFT, "plan internals were released (free-after-solve); rebuild the plan");
  if (!p->symbolic_done) return fail(PTAP_ERR_VALUE, "numeric called before symbolic");
  return PTAP_OK;
}

ptap_status ptap_numeric_send(ptap_plan *p, const ptap_operands *ops, void *stream) {
  CKS(numeric_ready(p));
  CKS(validate(ops));
  cudaStream_t st = (cudaStream_t)stream;
  CKS(check_image(p, ops, st));
  Ops op = make_ops(ops);
  if (p->alg == PTAP_TWO_STEP) {
    CKS(for_bins(p, p->bins_all, [&](const LaunchShape &s, const int32_t *rows, unsigned long long n) {
      return launch_ct_numeric(s, op, rows, n, p->ct_rp, p->ct_col, p->ct_val, p->d_status, st);
    }));
    CK(launch_gather(p->ptd.nnz, p->ptd.perm, ops->p_diag.val, p->ptd.val, st));
    CK(launch_gather(p->pto.nnz, p->pto.perm, ops->p_off.val, p->pto.val, st));
    p->cnt.kernel_launches += 2;
    PtcTarget tg{1, p->s_nrows, p->s_rows, p->s_rp, p->s_col, p->s_val};
    CKS(for_bins(p, p->bins_pto, [&](const LaunchShape &s, const int32_t *rows, unsigned long long n) {
      return launch_ptc_numeric(s, rows, n, p->pto.rp, p->pto.row, p->pto.val, ops->p_colmap, 0, p->ct_rp,
                                p->ct_col, p->ct_val, tg, p->d_status, st);
    }));
    return PTAP_OK;
  }
  bool merged = p->alg == PTAP_MERGED;
  if (p->s_nnz > 0) CK(cudaMemsetAsync(p->s_val, 0, sizeof(double) * p->s_nnz, st));
  BinSet &bs = merged ? p->bins_all : p->bins_send;
  if (merged && p->c_nnz > 0 && !tile_writes_all(p, bs, op))
    CK(cudaMemsetAsync(p->c_val, 0, sizeof(double) * p->c_nnz, st));
  CKS(run_outer_numeric(p, op, bs, 1, merged ? 1 : 0, st));
  p->cnt.numeric_row_kernel_calls += bs.selected;
  return PTAP_OK;
}

ptap_status ptap_numeric_local(ptap_plan *p, const ptap_operands *ops, void *stream) {
  CKS(numeric_ready(p));
  CKS(validate(ops));
  cudaStream_t st = (cudaStream_t)stream;
  CKS(check_image(p, ops, st));
  Ops op = make_ops(ops);
  if (p->alg == PTAP_TWO_STEP) {
    PtcTarget tg{0, p->ncl, nullptr, p->c_rp, p->c_col, p->c_val};
    CKS(for_bins(p, p->bins_ptd, [&](const LaunchShape &s, const int32_t *rows, unsigned long long n) {
      return launch_ptc_numeric(s, rows, n, p->ptd.rp, p->ptd.row, p->ptd.val, nullptr, 0, p->ct_rp, p->ct_col,
                                p->ct_val, tg, p->d_status, st);
    }));
    p->cnt.numeric_row_kernel_calls += p->nloc;
  } else if (p->alg == PTAP_ALLATONCE) {
    if (p->c_nnz > 0 && !tile_writes_all(p, p->bins_local, op))
      CK(cudaMemsetAsync(p->c_val, 0, sizeof(double) * p->c_nnz, st));
    CKS(run_outer_numeric(p, op, p->bins_local, 0, 1, st));
    p->cnt.numeric_row_kernel_calls += p->bins_local.selected;
  }
  p->cnt.numeric_runs++;
  return PTAP_OK;
}

ptap_status ptap_numeric_local_rows(ptap_plan *p, const ptap_operands *ops, int64_t row_lo, int64_t row_hi,
                                    int flags, void *stream) {
  CKS(numeric_ready(p));
  CKS(validate(ops));
  if (p->alg != PTAP_ALLATONCE || !p->mapped || !p->q4 || !p->bins_local.identity0)
    return fail(PTAP_ERR_VALUE, "plan has no range-addressable local rows");
  if (row_lo < 0 || row_hi > p->nloc || row_lo > row_hi) return fail(PTAP_ERR_VALUE, "row range");
  cudaStream_t st = (cudaStream_t)stream;
  CKS(check_image(p, ops, st));
  Ops op = make_ops(ops);
  if (p->tile) {
    // block-aligned ranges (the last may end at nloc); the first call of a
    // pass opens a new epoch
    if (row_lo % TILE_ROWS || (row_hi % TILE_ROWS && row_hi != p->nloc))
      return fail(PTAP_ERR_VALUE, "row range must be aligned to the plan's 64-row blocks");
    const int b0 = (int)(row_lo / TILE_ROWS), b1 = (int)((row_hi + TILE_ROWS - 1) / TILE_ROWS);
    CK(launch_tile_numeric(op, p->maps, p->ta, p->lock ? p->la : LockArgs{}, p->c_rp, p->c_val, b0, b1,
                           (flags & 1) != 0, st));
    p->cnt.kernel_launches += 2;
    p->cnt.numeric_row_kernel_calls += row_hi - row_lo;
    if (flags & 2) p->cnt.numeric_runs++;
    return PTAP_OK;
  }
  if ((flags & 1) && p->c_nnz > 0) CK(cudaMemsetAsync(p->c_val, 0, sizeof(double) * p->c_nnz, st));
  OuterTargets tg{p->c_rp, p->c_col, p->c_val, p->s_nrows, p->s_rows, p->s_rp, p->s_col, p->s_val};
  if (p->q4a && lock_usable(p, op) && row_lo % LOCK_TILE == 0 && (row_hi % LOCK_TILE == 0 || row_hi == p->nloc)) {
    if (flags & 1) {
      CK(launch_lock_permute_f64(p->nloc, op.pd_rp, p->la.pq, p->la.ltab, op.pd_val, p->la.Q, st));
      p->cnt.kernel_launches++;
    }
    CK(launch_lock_numeric(op, p->la, p->c_val, (int)(row_lo / LOCK_TILE),
                           (int)((row_hi + LOCK_TILE - 1) / LOCK_TILE), p->d_status, st));
    p->cnt.kernel_launches++;
    p->cnt.numeric_row_kernel_calls += row_hi - row_lo;
  } else if (row_hi > row_lo) {
    if (p->q4a)
      CK(launch_outer_numeric_q4a(op, (unsigned long long)(row_hi - row_lo), p->maps, tg, p->d_status, st,
                                  (int)row_lo));
    else
      CK(launch_outer_numeric_mapped(3, op, nullptr, (unsigned long long)(row_hi - row_lo), p->maps, tg, 0, 1,
                                     p->d_status, st, (int)row_lo));
    p->cnt.kernel_launches++;
    p->cnt.numeric_row_kernel_calls += row_hi - row_lo;
  }
  if (flags & 2) p->cnt.numeric_runs++;
  return PTAP_OK;
}

ptap_status ptap_plan_c_last_row(ptap_plan *p, const ptap_operands *ops, int32_t *last, void *stream) {
  CKS(numeric_ready(p));
  CKS(validate(ops));
  if (!last && p->ncl > 0) return fail(PTAP_ERR_VALUE, "null output");
  if (p->tile) CK(launch_tile_c_last(p->ncl, p->ta, last, (cudaStream_t)stream));
  else CK(launch_c_last_row(p->nloc, ops->p_diag.row_ptr, ops->p_diag.col, p->ncl, last, (cudaStream_t)stream));
  return PTAP_OK;
}

ptap_status ptap_numeric_merge(ptap_plan *p, const double *recv_vals, void *stream) {
  CKS(numeric_ready(p));
  cudaStream_t st = (cudaStream_t)stream;
  if (p->r_nnz == 0) return PTAP_OK;
  // ascending source rank, one launch per source (src/tripleproduct.py:215-229)
  for (size_t k = 0; k + 1 < p->r_src_nnz_off.size(); ++k) {
    int64_t a = p->r_src_nnz_off[k], b = p->r_src_nnz_off[k + 1];
    if (b > a) {
      CK(launch_merge_add(b - a, p->r_slot + a, recv_vals + a, p->c_val, st));
      p->cnt.kernel_launches++;
    }
  }
  return PTAP_OK;
}

ptap_status ptap_pack_values(ptap_plan *p, const ptap_operands *ops, const int64_t *idx, int64_t n, double *out,
                             void *stream) {
  if (!p || !ops) return fail(PTAP_ERR_VALUE, "null argument");
  if (n > 0 && (!idx || !out)) return fail(PTAP_ERR_VALUE, "null buffer");
  CK(launch_pack_values(ops->p_diag.val, ops->p_diag.nnz, ops->p_off.val, ops->p_off.nnz, idx, n, out, p->d_status,
                        (cudaStream_t)stream));
  p->cnt.kernel_launches++;
  return PTAP_OK;
}

// Non-blocking status: the device status word of this pass is copied to
// pinned host memory behind the pass (and reset on the device); the result
// is read by ptap_plan_status_poll, which waits only for that copy.
ptap_status ptap_plan_status_async(ptap_plan *p, void *stream) {
  if (!p) return fail(PTAP_ERR_VALUE, "null plan");
  cudaStream_t st = (cudaStream_t)stream;
  if (!p->h_status) {
    CK(cudaMallocHost(&p->h_status, sizeof(int)));
    *p->h_status = 0;
    CK(cudaEventCreateWithFlags(&p->status_ev, cudaEventDisableTiming));
  }
  if (p->status_pending) {  // fold the previous pass's status in first
    CK(cudaEventSynchronize(p->status_ev));
    const int prev = *p->h_status;
    if (prev) {
      p->status_pending = false;
      return status_to_error(prev, "numeric");
    }
  }
  CK(cudaMemcpyAsync(p->h_status, p->d_status, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemsetAsync(p->d_status, 0, sizeof(int), st));
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(st, &cap));
  if (cap != cudaStreamCaptureStatusNone) {
    // captured: each replay writes the status to h_status; the caller
    // synchronises before ptap_plan_status_poll reads it
    p->status_graph = true;
    return PTAP_OK;
  }
  CK(cudaEventRecord(p->status_ev, st));
  p->status_pending = true;
  return PTAP_OK;
}

ptap_status ptap_plan_status_poll(ptap_plan *p) {
  if (!p) return fail(PTAP_ERR_VALUE, "null plan");
  if (!p->status_pending) {
    if (p->status_graph && p->h_status) {  // replays of a captured pass (caller synchronised)
      const int s = *p->h_status;
      *p->h_status = 0;
      return status_to_error(s, "numeric");
    }
    return PTAP_OK;
  }
  CK(cudaEventSynchronize(p->status_ev));
  p->status_pending = false;
  const int s = *p->h_status;
  *p->h_status = 0;
  return status_to_error(s, "numeric");
}

ptap_status ptap_plan_check(ptap_plan *p, void *stream) {
  if (!p) return fail(PTAP_ERR_VALUE, "null plan");
  int s = 0;
  CKS(read_status(p, (cudaStream_t)stream, &s));
  return status_to_error(s, "numeric");
}

ptap_status ptap_plan_verify(ptap_plan *p, const ptap_operands *ops, void *stream) {
  CKS(numeric_ready(p));
  CKS(validate(ops));
  cudaStream_t st = (cudaStream_t)stream;
  int64_t sh[11];
  op_shape(ops, sh, nullptr);
  for (int k = 0; k < 11; ++k)
    if (sh[k] != p->img_shape[k])
      return fail(PTAP_ERR_DRIFT, "operand structure changed since the symbolic phase (sizes differ)");
  unsigned long long dg = 0;
  CKS(op_digest(p, ops, st, &dg));
  if (dg != p->img_digest) return fail(PTAP_ERR_DRIFT, "operand structure changed since the symbolic phase");
  int s = 0;
  CKS(read_status(p, st, &s));
  return status_to_error(s, "numeric");
}

ptap_status ptap_plan_get_ctilde(ptap_plan *p, ptap_c_view *out) {
  if (!p || !out) return fail(PTAP_ERR_VALUE, "null argument");
  if (p->alg != PTAP_TWO_STEP) return fail(PTAP_ERR_VALUE, "only a two-step plan stores C~ = A P");
  if (p->released) return fail(PTAP_ERR_DRIFT, "plan internals were released (free-after-solve); rebuild the plan");
  out->nrows = p->nloc;
  out->ncols = p->m;
  out->nnz = p->ct_nnz;
  out->row_ptr = p->ct_rp;
  out->col = p->ct_col;
  out->val = p->ct_val;
  return PTAP_OK;
}

ptap_status ptap_plan_get_c(ptap_plan *p, ptap_c_view *out) {
  if (!p || !out) return fail(PTAP_ERR_VALUE, "null argument");
  out->nrows = p->ncl;
  out->ncols = p->m;
  out->nnz = p->c_nnz;
  out->row_ptr = p->c_rp;
  out->col = p->c_col;
  out->val = p->c_val;
  return PTAP_OK;
}

ptap_status ptap_plan_release_cache(ptap_plan *p) {
  if (!p) return fail(PTAP_ERR_VALUE, "null plan");
  if (p->released) return PTAP_OK;
  cudaStream_t st = 0;
  cudaDeviceSynchronize();
  free_bins(p, p->bins_send, st);
  free_bins(p, p->bins_local, st);
  free_bins(p, p->bins_all, st);
  free_bins(p, p->bins_ptd, st);
  free_bins(p, p->bins_pto, st);
  pfree(p, p->s_rows, st); pfree(p, p->s_rp, st); pfree(p, p->s_col, st); pfree(p, p->s_val, st);
  pfree(p, p->r_slot, st);
  free_maps(p, st);
  pfree(p, p->ct_rp, st); pfree(p, p->ct_col, st); pfree(p, p->ct_val, st);
  for (Transpose *t : {&p->ptd, &p->pto}) {
    pfree(p, t->rp, st); pfree(p, t->row, st); pfree(p, t->perm, st); pfree(p, t->val, st);
  }
  cudaStreamSynchronize(st);
  trim_pool();
  p->released = true;
  return PTAP_OK;
}

ptap_status ptap_plan_memory(ptap_plan *p, ptap_memory *out) {
  if (!p || !out) return fail(PTAP_ERR_VALUE, "null argument");
  for (int c = 0; c < 5; ++c) {
    out->current[c] = p->cur[c];
    out->peak[c] = p->peak[c];
  }
  out->product_peak = p->prod_peak;
  out->device_high_water = p->total_peak;
  return PTAP_OK;
}

ptap_status ptap_plan_counters(ptap_plan *p, ptap_counters *out) {
  if (!p || !out) return fail(PTAP_ERR_VALUE, "null argument");
  *out = p->cnt;
  return PTAP_OK;
}

// ---- standalone C~ = A P ------------------------------------------------------
ptap_status ptap_spgemm_ap_symbolic(const ptap_operands *ops, int64_t *nnz_out, int64_t **row_ptr_out,
                                    int32_t **col_out, void *stream) {
  CKS(validate(ops));
  cudaStream_t st = (cudaStream_t)stream;
  ptap_plan tmp;
  tmp.nloc = ops->n_local; tmp.m = ops->m_global; tmp.c_lo = ops->c_lo; tmp.c_hi = ops->c_hi;
  if (cudaMalloc(&tmp.d_status, sizeof(int)) != cudaSuccess ||
      cudaMalloc(&tmp.d_u64, 24 * sizeof(unsigned long long)) != cudaSuccess)
    return fail(PTAP_ERR_CUDA, "alloc");
  cudaMemset(tmp.d_status, 0, sizeof(int));
  Ops op = make_ops(ops);
  ptap_status rc = PTAP_OK;
  int64_t *ap_nnz = nullptr, *rp = nullptr, *scratch = nullptr;
  int32_t *col = nullptr, *wide = nullptr;
  int64_t nnz = 0;
  BinSet bs;
  do {
    if ((rc = ap_sizes(&tmp, op, &ap_nnz, st)) != PTAP_OK) break;
    if (cudaMalloc(&rp, sizeof(int64_t) * (tmp.nloc + 1)) != cudaSuccess) { rc = fail(PTAP_ERR_OOM, "alloc"); break; }
    if ((rc = palloc(&tmp, &scratch, scan_scratch_elems(tmp.nloc), CAT_TRANSIENT, st)) != PTAP_OK) break;
    scan_exclusive(ap_nnz, rp, tmp.nloc, scratch, st);
    cudaMemcpyAsync(&nnz, rp + tmp.nloc, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (cudaMalloc(&col, sizeof(int32_t) * (nnz > 0 ? nnz : 1)) != cudaSuccess) { rc = fail(PTAP_ERR_OOM, "alloc"); break; }
    if ((rc = build_bins(&tmp, bs, tmp.nloc, ap_nnz, op.pd_rp, op.po_rp, 0, false, CAT_TRANSIENT, st)) != PTAP_OK) break;
    rc = for_bins(&tmp, bs, [&](const LaunchShape &s, const int32_t *rows, unsigned long long n) {
      return launch_ct_fill(s, op, rows, n, rp, col, tmp.d_status, st);
    });
    if (rc != PTAP_OK) break;
    if ((rc = palloc(&tmp, &wide, nnz / 1024 + 2, CAT_TRANSIENT, st)) != PTAP_OK) break;
    cudaMemsetAsync(tmp.d_u64 + 6, 0, sizeof(unsigned long long), st);
    launch_sort_rows(tmp.nloc, rp, col, nullptr, wide, tmp.d_u64 + 6, st);
    unsigned long long nwide = 0;
    cudaMemcpyAsync(&nwide, tmp.d_u64 + 6, sizeof(nwide), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    launch_sort_rows_block((int64_t)nwide, wide, rp, col, nullptr, tmp.d_status, st);
    int s = 0;
    if ((rc = read_status(&tmp, st, &s)) != PTAP_OK) break;
    if (s) rc = status_to_error(s, "spgemm symbolic");
  } while (0);
  cudaStreamSynchronize(st);
  for (auto &kv : tmp.allocs) cudaFree(kv.first);
  tmp.allocs.clear();
  cudaFree(tmp.d_status);
  cudaFree(tmp.d_u64);
  tmp.d_status = nullptr;
  tmp.d_u64 = nullptr;
  if (rc != PTAP_OK) {
    cudaFree(rp);
    cudaFree(col);
    return rc;
  }
  *nnz_out = nnz;
  *row_ptr_out = rp;
  *col_out = col;
  return PTAP_OK;
}

ptap_status ptap_spgemm_ap_numeric(const ptap_operands *ops, const int64_t *row_ptr, const int32_t *col, double *val,
                                   void *stream) {
  CKS(validate(ops));
  cudaStream_t st = (cudaStream_t)stream;
  ptap_plan tmp;
  tmp.nloc = ops->n_local; tmp.m = ops->m_global;
  if (cudaMalloc(&tmp.d_status, sizeof(int)) != cudaSuccess ||
      cudaMalloc(&tmp.d_u64, 24 * sizeof(unsigned long long)) != cudaSuccess)
    return fail(PTAP_ERR_CUDA, "alloc");
  cudaMemset(tmp.d_status, 0, sizeof(int));
  Ops op = make_ops(ops);
  ptap_status rc = PTAP_OK;
  int64_t *est = nullptr;
  BinSet bs;
  do {
    if ((rc = palloc(&tmp, &est, tmp.nloc, CAT_TRANSIENT, st)) != PTAP_OK) break;
    launch_row_lengths(tmp.nloc, row_ptr, est, st);
    if ((rc = build_bins(&tmp, bs, tmp.nloc, est, nullptr, nullptr, 0, true, CAT_TRANSIENT, st)) != PTAP_OK) break;
    rc = for_bins(&tmp, bs, [&](const LaunchShape &s, const int32_t *rows, unsigned long long n) {
      return launch_ct_numeric(s, op, rows, n, row_ptr, col, val, tmp.d_status, st);
    });
    if (rc != PTAP_OK) break;
    int s = 0;
    if ((rc = read_status(&tmp, st, &s)) != PTAP_OK) break;
    if (s) rc = status_to_error(s, "spgemm numeric");
  } while (0);
  cudaStreamSynchronize(st);
  for (auto &kv : tmp.allocs) cudaFree(kv.first);
  tmp.allocs.clear();
  cudaFree(tmp.d_status);
  cudaFree(tmp.d_u64);
  tmp.d_status = nullptr;
  tmp.d_u64 = nullptr;
  return rc;
}

// ---- standalone transpose (reference transpose_with_permutation) ------------
ptap_status ptap_transpose(int64_t nrows, int64_t ncols, const int64_t *rp, const int32_t *col, const double *val,
                           int64_t nnz, int64_t *t_rp, int32_t *t_col, int64_t *perm, double *t_val, void *stream) {
  if (nrows < 0 || ncols < 0 || nnz < 0 || !rp || !t_rp || (nnz > 0 && (!col || !t_col || !perm)))
    return fail(PTAP_ERR_VALUE, "transpose: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  ptap_plan tmp;
  tmp.nloc = nrows;
  if (cudaMalloc(&tmp.d_status, sizeof(int)) != cudaSuccess ||
      cudaMalloc(&tmp.d_u64, 24 * sizeof(unsigned long long)) != cudaSuccess)
    return fail(PTAP_ERR_CUDA, "alloc");
  cudaMemset(tmp.d_status, 0, sizeof(int));
  ptap_status rc = PTAP_OK;
  int64_t *cnt = nullptr, *scratch = nullptr;
  int32_t *wide = nullptr;
  do {
    if ((rc = palloc(&tmp, &cnt, ncols, CAT_TRANSIENT, st)) != PTAP_OK) break;
    if ((rc = palloc(&tmp, &scratch, scan_scratch_elems(ncols), CAT_TRANSIENT, st)) != PTAP_OK) break;
    cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (ncols > 0 ? ncols : 1), st);
    if (nnz > 0) launch_count_cols(nnz, col, cnt, st);
    scan_exclusive(cnt, t_rp, ncols, scratch, st);
    cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (ncols > 0 ? ncols : 1), st);
    if (nnz > 0) {
      launch_transpose_scatter(nrows, rp, col, t_rp, cnt, t_col, perm, st);
      // rows of the transpose in ascending source row (a stable transpose:
      // perm is the stable argsort of the columns, as in the reference)
      if ((rc = palloc(&tmp, &wide, nnz / 1024 + 2, CAT_TRANSIENT, st)) != PTAP_OK) break;
      cudaMemsetAsync(tmp.d_u64 + 6, 0, sizeof(unsigned long long), st);
      launch_sort_rows(ncols, t_rp, t_col, perm, wide, tmp.d_u64 + 6, st);
      unsigned long long nwide = 0;
      cudaMemcpyAsync(&nwide, tmp.d_u64 + 6, sizeof(nwide), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      launch_sort_rows_block((int64_t)nwide, wide, t_rp, t_col, perm, tmp.d_status, st);
      if (val && t_val) launch_gather(nnz, perm, val, t_val, st);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { rc = fail(PTAP_ERR_CUDA, std::string("transpose: ") + cudaGetErrorString(e)); break; }
    int s = 0;
    if ((rc = read_status(&tmp, st, &s)) != PTAP_OK) break;
    if (s) rc = status_to_error(s, "transpose");
  } while (0);
  cudaStreamSynchronize(st);
  for (auto &kv : tmp.allocs) cudaFree(kv.first);
  tmp.allocs.clear();
  cudaFree(tmp.d_status);
  cudaFree(tmp.d_u64);
  tmp.d_status = nullptr;
  tmp.d_u64 = nullptr;
  return rc;
}

ptap_status ptap_device_free(void *ptr, void *stream) {
  // buffers handed out by ptap_spgemm_ap_symbolic come from cudaMalloc
  if (ptr) {
    cudaStreamSynchronize((cudaStream_t)stream);
    cudaFree(ptr);
  }
  return PTAP_OK;
}

ptap_status ptap_l2_flush(void *stream) {
  static void *buf = nullptr;
  const int64_t bytes = 512ll << 20;
  if (!buf && cudaMalloc(&buf, bytes) != cudaSuccess) return fail(PTAP_ERR_OOM, "l2 flush buffer");
  cudaError_t e = launch_touch(buf, bytes, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(PTAP_ERR_CUDA, cudaGetErrorString(e));
  return PTAP_OK;
}

}  // extern "C"
