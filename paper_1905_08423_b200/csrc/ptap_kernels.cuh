// ptap_kernels.cuh -- host-callable launchers of the kernels in ptap_kernels.cu
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ptap_device.cuh"

namespace ptapdev {

// Work bins: estimated distinct AP-row keys n -> table shape.
//   bin 0: n <= 32    4 rows per warp (8-lane groups), 64-slot shared tables
//   bin 1: n <= 128   4 rows per warp, 256-slot shared tables
//   bin 2: n <= 1024  1 row per warp, 2048-slot shared tables
//   bin 3: larger     1 row per warp, global-memory tables (heavy rows)
constexpr int NBINS = 4;
__host__ __device__ inline int64_t bin_capacity(int q) { return q == 0 ? 32 : (q == 1 ? 128 : 1024); }

struct BinLists {
  int32_t *rows[NBINS];
  unsigned long long *count;  // device, NBINS entries
};

struct Arena {
  unsigned long long *keys;
  unsigned long long mask;  // capacity - 1 (power of two)
  int log2b = 0;            // > 0: row-bucketed placement (2^log2b slots per row), 0: hashed
  unsigned long long m = 0; // key = row * m + col
};

struct OuterTargets {
  const int64_t *c_rp; const int32_t *c_col; double *c_val;     // local C rows (global columns)
  int64_t s_nrows; const int32_t *s_rows; const int64_t *s_rp; const int32_t *s_col; double *s_val;  // staging
};

struct PtcTarget {
  int is_staging;
  int64_t nrows;
  const int32_t *rows;  // staging row ids (global), for lookup
  const int64_t *rp;
  const int32_t *col;
  double *val;
};

// plan-mapped numeric (ptap_mapped.cu)
struct MapOut {  // symbolic outputs of the outer-product pass (null: no maps)
  const int64_t *smap_rp;
  uint8_t *smap;
  uint8_t *nap;
  const int64_t *pat_rp;  // sorted AP row patterns (transient, for the position maps)
  int32_t *pat;
};

struct MapArgs {
  int64_t *smap_rp;  // [nloc] pool offset | map length << 40 (interned maps)
  uint8_t *smap;     // slot of every (A entry, P entry) pair, fold order
  int64_t *pmap_rp;  // [nloc] pool offset of the row's position map (interned)
  uint8_t *pmap;     // position of every slot in every target row of P(i,:)
  uint8_t *nap;      // [nloc] AP row sizes
  int32_t *po_srow;  // [nnz(P_o)] staging row of every P_o entry
  int32_t *poff;     // [nnz(A_d)] q4a: start of the entry's P row | (its length << 28); null: unused
  int32_t *cbase;    // [nnz(P_d)] q4a: start of the C row each P_d entry targets; null: unused
};

struct LaunchShape {
  int bin;       // work bin of the rows
  int group;     // 8 or 32 lanes per row
  int warps;     // warps per CTA
  int log2t;     // table slots = 1 << log2t
  int max_ctas;  // grid cap (grid-stride loops)
  unsigned char *gtables;  // non-null: tables in global memory (one per group of the capped grid)
};

size_t row_kernel_group_bytes(int log2t, bool num, int group);

cudaError_t launch_row_work(const Ops &op, int64_t *apub, unsigned long long *mac, cudaStream_t st);
cudaError_t launch_bin_rows(int64_t nrows, const int64_t *est, const int64_t *pd_rp, const int64_t *po_rp, int mode,
                            const BinLists &bl, unsigned long long *selected, cudaStream_t st);
cudaError_t launch_max_est(const int32_t *rows, unsigned long long nrows, const int64_t *est, unsigned long long *mx,
                           cudaStream_t st);
cudaError_t launch_ap_count_small(const Ops &op, int64_t nrows, const int64_t *apub, int64_t *ap_nnz,
                                  cudaStream_t st);
cudaError_t launch_retry_est(int64_t n, const int64_t *ap_nnz, const int64_t *apub, int64_t *est2,
                             unsigned long long *nretry, cudaStream_t st);
cudaError_t launch_outer_symbolic_q4(const Ops &op, const int32_t *rows, unsigned long long nrows, int do_send,
                                     int do_local, Arena local, Arena send, const MapOut &mo, int *status,
                                     cudaStream_t stream, int row0 = 0);
cudaError_t launch_offsets_shift(int64_t n, const int64_t *in, int64_t sub, int64_t add_packed, int64_t *out,
                                 cudaStream_t st);
cudaError_t launch_c_union(bool fill, int64_t ncl, const int64_t *t_rp, const int32_t *t_row, const int64_t *pat_rp,
                           const int32_t *pat, const uint8_t *nap, int64_t *cnt, const int64_t *c_rp, int32_t *c_col,
                           const int64_t *pd_rp, const int32_t *pd_col, const int64_t *pmap_rp, uint8_t *pmap,
                           int *status, cudaStream_t st);
cudaError_t launch_ap_count(const LaunchShape &s, const Ops &op, const int32_t *rows, unsigned long long nrows,
                            int64_t *ap_nnz, int *status, cudaStream_t stream);
cudaError_t launch_outer_symbolic(const LaunchShape &s, const Ops &op, const int32_t *rows, unsigned long long nrows,
                                  int do_send, int do_local, Arena local, Arena send, const MapOut &mo, int *status,
                                  cudaStream_t stream);
cudaError_t launch_build_pmap(const Ops &op, unsigned long long nrows, const MapArgs &mp, const MapOut &mo,
                              const OuterTargets &tg, int *status, cudaStream_t st, int64_t row0 = 0);
cudaError_t launch_outer_numeric(const LaunchShape &s, const Ops &op, const int32_t *rows, unsigned long long nrows,
                                 int do_send, int do_local, const OuterTargets &tg, int *status,
                                 cudaStream_t stream);
cudaError_t launch_outer_oneshot(const LaunchShape &s, const Ops &op, const int32_t *rows, unsigned long long nrows,
                                 Arena local, double *avals, int *status, cudaStream_t stream);
cudaError_t launch_arena_scatter_vals(Arena ar, int64_t m, const int64_t *rp, int64_t *cursor, int32_t *col,
                                      const double *avals, int64_t *payload, cudaStream_t st);
cudaError_t launch_ct_fill(const LaunchShape &s, const Ops &op, const int32_t *rows, unsigned long long nrows,
                           const int64_t *ct_rp, int32_t *ct_col, int *status, cudaStream_t stream);
cudaError_t launch_ct_numeric(const LaunchShape &s, const Ops &op, const int32_t *rows, unsigned long long nrows,
                              const int64_t *ct_rp, const int32_t *ct_col, double *ct_val, int *status,
                              cudaStream_t stream);
cudaError_t launch_ptc_numeric(const LaunchShape &s, const int32_t *rows, unsigned long long nrows,
                               const int64_t *t_rp, const int32_t *t_row, const double *t_val,
                               const int32_t *target_map, int64_t target_offset, const int64_t *ct_rp,
                               const int32_t *ct_col, const double *ct_val, const PtcTarget &tg, int *status,
                               cudaStream_t stream);
cudaError_t launch_arena_fill_empty(Arena ar, cudaStream_t st);
cudaError_t launch_arena_insert_batch(Arena ar, int64_t nrows, const int32_t *rows, const int64_t *rp,
                                      const int32_t *col, int64_t m, int64_t c_lo, int64_t c_hi, int *status,
                                      cudaStream_t st);
cudaError_t launch_arena_rowcount(Arena ar, int64_t m, int64_t *cnt, cudaStream_t st);
cudaError_t launch_arena_scatter(Arena ar, int64_t m, const int64_t *rp, int64_t *cursor, int32_t *col,
                                 cudaStream_t st);
cudaError_t launch_sort_rows(int64_t nrows, const int64_t *rp, int32_t *keys, int64_t *payload, int32_t *wide_rows,
                             unsigned long long *nwide, cudaStream_t st);
cudaError_t launch_sort_rows_block(int64_t nwide, const int32_t *rows, const int64_t *rp, int32_t *keys,
                                   int64_t *payload, int *status, cudaStream_t st);
cudaError_t launch_merge_slots(int64_t nrows, const int32_t *rows, const int64_t *rp, const int32_t *col, int64_t c_lo,
                               const int64_t *c_rp, const int32_t *c_col, int64_t *slot, int *status,
                               cudaStream_t st);
cudaError_t launch_merge_add(int64_t n, const int64_t *slot, const double *vals, double *c_val, cudaStream_t st);
cudaError_t launch_pack_values(const double *d_val, int64_t nd, const double *o_val, int64_t no, const int64_t *idx,
                               int64_t n, double *out, int *status, cudaStream_t st);
cudaError_t launch_count_cols(int64_t nnz, const int32_t *col, int64_t *cnt, cudaStream_t st);
cudaError_t launch_transpose_scatter(int64_t nrows, const int64_t *rp, const int32_t *col, const int64_t *t_rp,
                                     int64_t *cursor, int32_t *t_row, int64_t *t_perm, cudaStream_t st);
cudaError_t launch_gather(int64_t n, const int64_t *perm, const double *src, double *dst, cudaStream_t st);
cudaError_t launch_ptc_symbolic(int64_t nrows, const int64_t *t_rp, const int32_t *t_row, const int32_t *target_map,
                                int64_t target_offset, const int64_t *ct_rp, const int32_t *ct_col, Arena ar,
                                int64_t m, int *status, cudaStream_t st);
cudaError_t scan_exclusive(const int64_t *in, int64_t *out, int64_t n, int64_t *scratch, cudaStream_t st);
int64_t scan_scratch_elems(int64_t n);
cudaError_t launch_nonzero_flags(int64_t n, const int64_t *cnt, int64_t *flags, cudaStream_t st);
cudaError_t launch_compact_rows(int64_t n, const int64_t *cnt, const int64_t *pos, const int64_t *dense_rp,
                                int32_t *rows, int64_t *rp, cudaStream_t st);
cudaError_t launch_iota32(int32_t *p, int64_t n, cudaStream_t st);
cudaError_t launch_row_lengths(int64_t n, const int64_t *rp, int64_t *len, cudaStream_t st);
cudaError_t launch_outer_bounds(int64_t n, const int64_t *pd_rp, const int64_t *po_rp, const int64_t *ap_nnz,
                                unsigned long long *out, cudaStream_t st);
cudaError_t launch_arena_rehash(Arena from, Arena to, int *status, cudaStream_t st);
cudaError_t launch_ptc_est(int64_t nrows, const int32_t *target_map, int64_t target_offset, int is_staging,
                           int64_t t_nrows, const int32_t *t_rows, const int64_t *t_rp, int64_t *est,
                           cudaStream_t st);
cudaError_t launch_touch(void *buf, int64_t bytes, cudaStream_t st);
cudaError_t launch_digest_i64(const int64_t *a, int64_t n, unsigned long long salt, unsigned long long *out,
                              cudaStream_t st);
cudaError_t launch_digest_i32(const int32_t *a, int64_t n, unsigned long long salt, unsigned long long *out,
                              cudaStream_t st);
cudaError_t launch_map_lengths(int64_t n, const int64_t *pd_rp, const int64_t *po_rp, const int64_t *apub,
                               const int64_t *ap_nnz, int64_t *slen, int64_t *plen, cudaStream_t st);
cudaError_t launch_po_srow(int64_t nnz, const int32_t *po_col, const int32_t *colmap, int64_t s_nrows,
                           const int32_t *s_rows, int32_t *po_srow, int *status, cudaStream_t st);
cudaError_t launch_max_i64(int64_t n, const int64_t *v, unsigned long long *mx, cudaStream_t st);
cudaError_t launch_max_rowlen(int64_t n, const int64_t *rp, unsigned long long *mx, cudaStream_t st);

cudaError_t launch_outer_numeric_mapped(int bin, const Ops &op, const int32_t *rows, unsigned long long nrows,
                                        const MapArgs &mp, const OuterTargets &tg, int do_send, int do_local,
                                        int *status, cudaStream_t st, int row0 = 0);
cudaError_t launch_outer_numeric_q4a(const Ops &op, unsigned long long nrows, const MapArgs &mp,
                                     const OuterTargets &tg, int *status, cudaStream_t st, int row0 = 0);
cudaError_t launch_struct_sample(const Ops &op, int64_t nsample, unsigned long long *keys, unsigned long long mask,
                                 unsigned long long *distinct, cudaStream_t st);
size_t row_order_scratch_bytes(int64_t n);
cudaError_t launch_row_order(int64_t n, const int32_t *rows_in, int32_t *rows_out, const int64_t *pd_rp,
                             const int32_t *pd_col, void *scratch, size_t scratch_bytes, cudaStream_t st);
cudaError_t launch_pack_offsets(int64_t n, const int64_t *rp, int64_t *out, cudaStream_t st);
cudaError_t launch_intern(int pass, int64_t n, const uint8_t *src, const int64_t *src_rp, unsigned long long *keys,
                          int64_t *vals, unsigned long long mask, int64_t *slot_of, int64_t *owner, int64_t *words,
                          uint8_t *pool, int64_t *out, int pack_len, unsigned long long *claims, cudaStream_t st);
// packed smap_rp entries of an interned plan: pool offset | map length << 40
constexpr unsigned long long SMAP_OFF_MASK = (1ull << 40) - 1;
cudaError_t launch_pure_rows(int64_t n, const int32_t *rows, const Ops &op, uint8_t *flag, cudaStream_t st);
cudaError_t launch_build_poff(int64_t nnz, const int32_t *ad_col, const int64_t *pd_rp, int32_t *poff,
                              cudaStream_t st);
cudaError_t launch_build_cbase(int64_t nnz, const int32_t *pd_col, const int64_t *c_rp, int32_t *cbase,
                               cudaStream_t st);
cudaError_t launch_c_last_row(int64_t n, const int64_t *pd_rp, const int32_t *pd_col, int64_t ncl, int32_t *last,
                              cudaStream_t st);

// deterministic owner-computes numeric pass (ptap_tile.cu)
constexpr int TILE_ROWS = 64;      // fine rows per block (work item)
constexpr int TILE_MAX_CROW = 64;  // widest C row the gather handles
constexpr int TILE_GCAP = 512;     // contributor entries staged per gather chunk
constexpr int TILE_MAXRUN = 16;    // runs of P rows staged per block
struct TileArgs {
  int32_t nloc, nblk, nitems, ring_blocks, blkcap, grid;  // nitems = nblk + ownership delay
  int32_t napc;             // accumulator slots per row (>= widest AP row)
  int32_t pstage;           // 1: stage the blocks' P runs in shared memory
  int32_t a_evict_first;    // 1: A's copies carry an L2 evict-first hint
  int32_t sm_aval, sm_acol, sm_pstage, sm_prp, sm_acc, sm_meta, sm_tail, sm_total;  // dynamic shared memory layout (bytes)
  const uint8_t *pr_n;      // [nblk] runs of P rows staged per block (0: read P from global memory)
  const int2 *pr_k;         // [nblk * TILE_MAXRUN] run [k0, k1) of P rows
  int32_t dbg;              // timing experiments only (PTAP_TILE_DBG): 1 no ring wait, 2 no flag wait, 4 no gather, 8 no fold
  const uint16_t *ap_off;   // [nloc] AP row offset inside its block's ring slot (doubles)
  double *ring;             // [ring_blocks * blkcap] AP rows of the blocks in flight
  const int32_t *own_rp;    // [nitems + 1] first C row owned by each item (owners are non-decreasing)
  const int64_t *qmap_rp;   // [ncl] gather map of each C row (interned pool offset)
  const uint8_t *qmap;      // [contributor][position] -> AP slot, 0xff: none
  const int32_t *t_rp;      // [ncl + 1] P_d^T: contributors of each C row
  const int32_t *t_row;     // [nnz(P_d)] contributing fine rows, ascending per C row
  const int32_t *t_pidx;    // [nnz(P_d)] index of P(i,J) in P_d's values
  const uint8_t *t_jx;      // symbolic only: index of the entry inside the fine row's P row
  const int32_t *rd_rp;     // [nblk + 1] distinct blocks each item's gathers read
  const int32_t *rd_blk;
  const uint32_t *expect;   // [nblk] readers of each block per pass
  uint32_t *flags;          // [nblk] epoch in which the block's AP rows were published
  uint32_t *readcnt;        // [nblk] reader signals, cumulative over passes
  uint32_t *ctl;            // [0] ticket, [1] epoch
};
size_t tile_smem_layout(TileArgs &ta, int amax_blk, int pvmax, int prmax);
int tile_grid(const TileArgs &ta);
cudaError_t launch_tile_pruns(int nblk, int64_t nloc, const int64_t *ad_rp, const int32_t *ad_col,
                              const int64_t *pd_rp, int64_t pnnz, int pvcap, int prcap, uint8_t *pr_n, int2 *pr_k,
                              unsigned long long *stats, cudaStream_t st);
size_t tile_scan_scratch(int64_t n);
struct LockArgs;
cudaError_t launch_tile_numeric(const Ops &op, const MapArgs &mp, const TileArgs &ta, const LockArgs &la,
                                const int64_t *c_rp, double *c_val, int blk_lo, int blk_hi, bool new_pass,
                                cudaStream_t st);
cudaError_t launch_tile_transpose(int64_t n, int64_t ncl, const int64_t *pd_rp, const int32_t *pd_col,
                                  int64_t pnnz, int32_t *cnt, int32_t *t_rp, int32_t *cursor, int32_t *t_row,
                                  uint8_t *t_jx, void *scratch, size_t scratch_bytes, int *status,
                                  cudaStream_t st);
size_t tile_owner_scratch(int64_t ncl);
cudaError_t launch_tile_owners(int64_t ncl, int nblk, int delay, const int64_t *pd_rp, const int32_t *t_rp,
                               int32_t *t_row, uint8_t *t_jx, int32_t *t_pidx, long long *key, int32_t *owner,
                               unsigned long long *stats, void *scratch, size_t scratch_bytes, cudaStream_t st);
cudaError_t launch_tile_own_rp(int nitems, int64_t ncl, const int32_t *owner, int32_t *own_rp, cudaStream_t st);
cudaError_t launch_tile_apoff(int64_t n, const int64_t *ad_rp, const int64_t *pd_rp, const uint8_t *nap,
                              uint16_t *ap_off, unsigned long long *stats, cudaStream_t st);
cudaError_t launch_tile_reads(int pass, int nitems, int delay, int span, const int32_t *own_rp,
                              const int32_t *t_rp, const int32_t *t_row, int32_t *rd_cnt,
                              const int32_t *rd_rp, int32_t *rd_blk, uint32_t *expect, cudaStream_t st);
cudaError_t launch_tile_qmap(int64_t ncl, const TileArgs &ta, const int64_t *c_rp, int64_t *qlen, int64_t *qm_rp,
                             const uint8_t *nap, const int64_t *pmap_rp, const uint8_t *pmap, uint8_t *qm, int pass,
                             cudaStream_t st);
cudaError_t launch_tile_c_last(int64_t ncl, const TileArgs &ta, int32_t *last, cudaStream_t st);
cudaError_t launch_tile_scan32(const int32_t *in, int32_t *out, int n, void *scratch, size_t scratch_bytes,
                               cudaStream_t st);

// class-lockstep numeric pass (ptap_lock.cu)
constexpr int LOCK_TILE = 64;  // fine rows per tile
constexpr int LOCK_NLEN = 9;   // P row lengths 0..8
constexpr int LOCK_TABLE = 65536;  // class table slots (a plan with more than half as many classes is not eligible)
constexpr int LOCK_WMAX = 4;  // most warps per group of 32 rows (the plan picks 2 or 3: LockArgs.lw)
struct __align__(16) LockClass {  // one structural class of fine rows (32 bytes)
  uint8_t alen, nap, ntg, niter;  // A row length, AP slots, own P entries (targets), outer-program words / 32
  int32_t tstride;                // rows of P with ntg entries: stride of the row's own entries in Q
  uint32_t fold_off, outer_off;   // program offsets (entries / words)
  uint8_t sub[8];                 // fold sub-program w = chunks [sub[w], sub[w+1]) of 8 entries (slot ranges, balanced); sub[7] = all chunks
  uint8_t s0[8];                  // first AP slot of sub-program w
};
struct LockArgs {
  int32_t nloc, ntiles, acap, aps;  // acap: staged A entries per tile, aps: AP buffer stride (doubles, odd)
  int32_t lw;                       // warps per group of 32 rows: they split the fold by slot ranges, the outer products by rows
  uint32_t fold_zero;               // index of eight zero entries behind the fold programs
  int32_t ast;                      // odd stride (words) of the converted column rows, >= the longest A row
  int32_t dbg;                      // timing experiments only (PTAP_LOCK_DBG): 1 no outer products, 2 no fold, 4 no column conversion
  const uint32_t *pq;       // [nloc] Q index of the first entry of P row k
  double *Q;                // [nnz(P_d)] P's values, class-major (rewritten every pass)
  const int32_t *cbQ;       // [nnz(P_d)] C row start of every P entry, same order
  const uint32_t *rowinfo;  // [nloc] per tile, rows sorted by class: class << 8 | row - tile start
  const uint32_t *rowcls;   // [nloc] class of every row (the deterministic kernel's lockstep fold)
  const LockClass *cls;
  const uint2 *fold;        // x: A entry*8 | last-of-slot << 15 | A entry*4 << 16, y: Q offset of the P entry
  const uint32_t *outer;    // slot*8 | target << 8 | position in the C row << 16
  const int32_t *ltab;      // [0, NLEN) rows of P per length, [NLEN, 2 NLEN) first Q index per length
};
size_t lock_smem_bytes(const LockArgs &la);
cudaError_t launch_lock_numeric(const Ops &op, const LockArgs &la, double *c_val, int tile_lo, int tile_hi,
                                int *status, cudaStream_t st);
cudaError_t launch_lock_qlayout(int64_t n, const int64_t *pd_rp, uint8_t *plen8, int32_t *blkcnt, int32_t *ltab,
                                uint32_t *pq, unsigned long long *bad, cudaStream_t st);
cudaError_t launch_lock_permute_f64(int64_t n, const int64_t *pd_rp, const uint32_t *pq, const int32_t *ltab,
                                    const double *src, double *dst, cudaStream_t st);
cudaError_t launch_lock_permute_i32(int64_t n, const int64_t *pd_rp, const uint32_t *pq, const int32_t *ltab,
                                    const int32_t *src, int32_t *dst, cudaStream_t st);
cudaError_t launch_lock_classes(const Ops &op, const uint8_t *plen8, const int64_t *smap_rp, const int64_t *pmap_rp,
                                unsigned long long *keys, uint32_t *rep, int tbl, uint16_t *slot_of,
                                int32_t *slot2cls, uint32_t *reps, unsigned long long *out, unsigned long long *bad,
                                const uint8_t *pure, cudaStream_t st);
cudaError_t launch_lock_headers(int ncls, const Ops &op, const uint8_t *plen8, const MapArgs &mp,
                                const uint32_t *reps, const int32_t *ltab, LockClass *cls,
                                unsigned long long *out, unsigned long long *bad, const uint8_t *pure, int lw,
                                cudaStream_t st);
cudaError_t launch_lock_programs(int ncls, const Ops &op, const uint8_t *plen8, const MapArgs &mp,
                                 const uint32_t *reps, const int32_t *ltab, const LockClass *cls, uint2 *fold,
                                 uint32_t *outer, int lw, cudaStream_t st);
cudaError_t launch_lock_rowinfo(int64_t n, const int64_t *ad_rp, const uint16_t *slot_of, const int32_t *slot2cls,
                                uint32_t *rowinfo, uint32_t *rowcls, unsigned long long *amax, cudaStream_t st);

}  // namespace ptapdev
