/*
 * ptap_b200.h -- C ABI of the B200-native Galerkin triple product C = P^T A P.
 *
 * This is the drop-in boundary under the Python operator API
 * (paper_1905_08423_b200.tripleproduct), which mirrors the reference's
 * ptap / run_symbolic / run_numeric / {aao,merged,two_step}_{symbolic,numeric}
 * (reference src/tripleproduct.py:358-529).  The reference is pure Python +
 * numba, so its "FFI" is the kernel seam in src/_kernels.py; the entry points
 * below replace the *phases* of the reference drivers rather than its
 * CPU-shaped per-row kernels:
 *
 *   ptap_plan_create / ptap_plan_destroy        TripleProductPlan            src/tripleproduct.py:105-145
 *   ptap_symbolic_send                          send loop + _build_staging   src/tripleproduct.py:241-279, 380-416
 *   ptap_symbolic_local                         local loop + merge + alloc   src/tripleproduct.py:280-300, 418-437
 *   ptap_numeric_send                           numeric send loop           src/tripleproduct.py:303-341, 440-470
 *   ptap_numeric_local                          numeric local loop          src/tripleproduct.py:342-348, 472-486
 *   ptap_numeric_merge                          _merge_numeric_batches      src/tripleproduct.py:215-229
 *   ptap_numeric_local_rows, ptap_plan_c_last_row  the local loop over a row  src/tripleproduct.py:342-348
 *                                               range (streamed uploads)
 *   ptap_plan_release_cache                     release_cache (cache=free)  src/tripleproduct.py:127-139
 *   ptap_plan_memory                            MemoryLedger categories     src/ledger.py:23-34
 *   ptap_plan_counters                          PlanCounters                src/ledger.py:149-156
 *   ptap_spgemm_ap_* (C~ = A P alone)           symbolic_ap / numeric_ap    src/spgemm.py:184-234
 *
 * Conventions
 *   - All pointers in the operand structs are DEVICE pointers borrowed from
 *     the caller (torch tensors); sizes are element counts.
 *   - Row offsets are int64, column indices int32, values fp64.
 *   - Every call takes a cudaStream_t (passed as void*) and is asynchronous
 *     unless documented; all device memory a plan owns is allocated in the
 *     symbolic calls (numeric calls never allocate).
 *   - Every call returns a ptap_status; on failure ptap_last_error() returns
 *     a thread-local message.  Status -> Python exception mapping:
 *        PTAP_ERR_PARTITION -> PartitionMismatchError
 *        PTAP_ERR_DRIFT     -> StructuralDriftError
 *        PTAP_ERR_OWNERSHIP -> OwnershipError
 *        PTAP_ERR_VALUE     -> ValueError
 *        PTAP_ERR_CUDA, PTAP_ERR_OOM -> DeviceError
 *   - Communication (the P~_r gather and the C_s -> owner exchange) is done
 *     by the caller over NCCL (torch.distributed); the library exposes the
 *     staging buffers and consumes received batches.
 */
#ifndef PTAP_B200_H
#define PTAP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PTAP_OK = 0,
    PTAP_ERR_VALUE = 1,
    PTAP_ERR_PARTITION = 2,
    PTAP_ERR_DRIFT = 3,
    PTAP_ERR_OWNERSHIP = 4,
    PTAP_ERR_CUDA = 5,
    PTAP_ERR_OOM = 6
} ptap_status;

typedef enum { PTAP_TWO_STEP = 0, PTAP_ALLATONCE = 1, PTAP_MERGED = 2 } ptap_algorithm;

/* Device CSR block (int64 row offsets, int32 columns, fp64 values). */
typedef struct {
    int64_t nrows;
    int64_t ncols;
    int64_t nnz;
    const int64_t *row_ptr;
    const int32_t *col;
    const double *val; /* may be NULL in symbolic calls */
} ptap_csr;

/* One rank's operands, the device image of two reference LocalMatrix objects
 * (src/partition.py:70-97) plus the gathered remote rows of P
 * (RemoteRows, src/comm.py:494-514). */
typedef struct {
    int64_t n_local;   /* fine rows owned (A and P row block)            */
    int64_t m_global;  /* global coarse dimension                        */
    int64_t c_lo;      /* owned coarse range [c_lo, c_hi) of C           */
    int64_t c_hi;
    ptap_csr a_diag;   /* columns: local fine rows                        */
    ptap_csr a_off;    /* columns: compact, index rows of p_remote        */
    ptap_csr p_diag;   /* columns: local coarse (global = col + c_lo)     */
    ptap_csr p_off;    /* columns: compact, global = p_colmap[col]        */
    const int32_t *p_colmap;
    int64_t p_colmap_len;
    ptap_csr p_remote; /* gathered P rows, columns global                 */
} ptap_operands;

/* Send-side staging of C_s (reference SendStaging, src/tripleproduct.py:59-102):
 * rows are global coarse rows owned elsewhere, ascending; dest_row_off[d] ..
 * dest_row_off[d+1] are the rows owned by rank d. Device pointers owned by
 * the plan. */
typedef struct {
    int64_t nrows;
    int64_t nnz;
    const int32_t *rows;     /* global coarse row ids           */
    const int64_t *row_ptr;  /* nrows+1                          */
    const int32_t *col;      /* global coarse columns, sorted    */
    double *val;             /* numeric values (after numeric_send) */
} ptap_staging;

/* Received contribution batches, concatenated in ascending source rank. */
typedef struct {
    int32_t nsrc;
    const int32_t *src_rank;     /* host array, nsrc entries              */
    const int64_t *src_row_off;  /* host array, nsrc+1 (rows per source)  */
    const int64_t *src_nnz_off;  /* host array, nsrc+1 (entries)          */
    int64_t nrows;
    int64_t nnz;
    const int32_t *rows;     /* device: global coarse rows              */
    const int64_t *row_ptr;  /* device: nrows+1, relative to the batch  */
    const int32_t *col;      /* device: global coarse columns           */
} ptap_received;

/* The output C (unified local rows with global columns, sorted). */
typedef struct {
    int64_t nrows;
    int64_t ncols;
    int64_t nnz;
    const int64_t *row_ptr;
    const int32_t *col;
    double *val;
} ptap_c_view;

typedef struct {
    int64_t current[5]; /* input, output, auxiliary, transient, plan_cache */
    int64_t peak[5];
    int64_t product_peak;
    int64_t device_high_water; /* bytes: max over the plan's life of all library allocations */
} ptap_memory;

typedef struct {
    int64_t symbolic_runs;
    int64_t numeric_runs;
    int64_t symbolic_row_kernel_calls; /* AP rows computed, reference meaning */
    int64_t numeric_row_kernel_calls;
    int64_t kernel_launches;           /* launches issued by this plan so far */
    int64_t nnz_c;
    int64_t nnz_staging;
    int64_t mac_ap;                    /* multiply-adds of the A*P rows       */
    int64_t mac_outer;                 /* multiply-adds of the outer products */
    int64_t numeric_path;              /* all-at-once/merged numeric: 3 plan maps, class-lockstep kernel; 2 deterministic owner-computes; 1 plan maps; 0 hash tables */
    int64_t map_bytes;                 /* plan maps kept (slot + position pools, interned) */
    int64_t row_structures_ppm;        /* distinct row structures per 1e6 sampled rows, -1: not sampled */
} ptap_counters;

typedef struct ptap_plan ptap_plan;

const char *ptap_last_error(void);
const char *ptap_version(void);

ptap_status ptap_plan_create(int algorithm, const ptap_operands *ops, ptap_plan **out);
ptap_status ptap_plan_destroy(ptap_plan *plan);
/* Plan options, set between create and the symbolic calls.
 *   "deterministic" (0/1): numeric passes bitwise repeatable and, at one rank,
 *     bit-identical to the reference's summation order (src/tripleproduct.py:12-16,
 *     src/_kernels.py:446-515): the owner-computes kernel of ptap_tile.cu
 *     replaces the fp64-atomic scatter when the plan's local loop has
 *     one-rank structure (counters.numeric_path == 2 when it is in use).
 *   "maps" (-1/0/1): plan maps of the all-at-once / merged numeric pass:
 *     -1 (default) kept when sampled rows repeat, 0 never (hash numeric path,
 *     nothing stored per row), 1 always.
 *   "lockstep" (-1/0/1): the class-lockstep numeric kernel (ptap_lock.cu:
 *     32 rows of one structural class in lockstep, A tiles staged by TMA,
 *     P's values class-major) for plans with maps and one-rank structure:
 *     -1/1 (default) when the plan is eligible, 0 never (the per-row mapped
 *     kernels run instead).  counters.numeric_path == 3 when it is in use.
 *   "single_shot" (0/1): symbolic and numeric in one pass (BASELINE north_star
 *     (3); SURVEY 3.2's additional single-shot fast path): when the rank neither
 *     sends nor receives, ptap_symbolic_local walks A's rows once, computing
 *     every AP row with values and adding its outer products, keys and values
 *     together, into the C arena, which is drained into sorted CSR with the
 *     values as payload; C then holds the product of the symbolic-time operands
 *     (ptap_plan_values_ready) and no numeric call is needed.  No maps are
 *     kept: later numeric passes on the plan run the hash path. */
ptap_status ptap_plan_set_option(ptap_plan *plan, const char *key, int64_t value);
/* 1 when the last symbolic phase also computed C's values (single_shot). */
ptap_status ptap_plan_values_ready(ptap_plan *plan, int *ready);

/* Symbolic, phase 1: AP-row binning and the send-side structure C_s (all
 * variants), plus (two-step) C~ and the local transposes. */
ptap_status ptap_symbolic_send(ptap_plan *plan, const ptap_operands *ops, void *stream);
ptap_status ptap_plan_staging(ptap_plan *plan, ptap_staging *out);
/* Symbolic, phase 2: local structure, merge of received structure (may be
 * NULL when nothing was received), allocation of C and of the merge slot map.
 * Synchronises the stream. */
ptap_status ptap_symbolic_local(ptap_plan *plan, const ptap_operands *ops,
                                const ptap_received *recv, void *stream);

/* Numeric phases.  numeric_send fills staging values; numeric_local zeroes C
 * and adds the local contributions (merged: numeric_send does both loops
 * in one fused pass and numeric_local only zero-fills when needed);
 * numeric_merge adds received values (same concatenated layout as the
 * symbolic ptap_received) in ascending source order. */
ptap_status ptap_numeric_send(ptap_plan *plan, const ptap_operands *ops, void *stream);
ptap_status ptap_numeric_local(ptap_plan *plan, const ptap_operands *ops, void *stream);
ptap_status ptap_numeric_merge(ptap_plan *plan, const double *recv_vals, void *stream);
/* All-at-once local loop over the fine rows [row_lo, row_hi) only, so a
 * caller can fold row blocks as their A values arrive (flags bit 0: first
 * block of the pass -- zero C / open a new epoch; bit 1: last block of the
 * pass, counted as one numeric run).  Ranges are aligned to 64-row blocks
 * (the last may end at n_local).  Returns PTAP_ERR_VALUE when the plan's
 * local rows are not one range-addressable bin (callers then use
 * ptap_numeric_local). */
ptap_status ptap_numeric_local_rows(ptap_plan *plan, const ptap_operands *ops, int64_t row_lo, int64_t row_hi,
                                    int flags, void *stream);
/* last[J] (device, int32, one per local C row) = the largest local fine row
 * contributing to C row J, -1 for none: C row J is final once rows <= last[J]
 * are folded. */
ptap_status ptap_plan_c_last_row(ptap_plan *plan, const ptap_operands *ops, int32_t *last, void *stream);
/* Synchronise and report device-side drift detected by the last numeric pass. */
ptap_status ptap_plan_check(ptap_plan *plan, void *stream);
/* Non-blocking variant: enqueue the copy of the pass's status word to pinned
 * host memory (no host synchronisation; reports a failure of the PREVIOUS
 * pass if one was pending), and read it later with ptap_plan_status_poll.
 * Inside CUDA-graph capture the copy becomes part of the graph: synchronise
 * after a replay, then poll. */
ptap_status ptap_plan_status_async(ptap_plan *plan, void *stream);
ptap_status ptap_plan_status_poll(ptap_plan *plan);
/* Owner side of the per-pass values-only refresh of the gathered P rows
 * (update_remote_rows_numeric, src/comm.py:625-649): out[t] = value idx[t] of
 * [P_d.val, P_o.val] (the symbolic gather's serve index), device buffers,
 * asynchronous; an index past the structure flags drift in the plan status. */
ptap_status ptap_pack_values(ptap_plan *plan, const ptap_operands *ops, const int64_t *idx, int64_t n,
                             double *out, void *stream);
/* Full structural check (reference verify_filled, src/spgemm.py:58-68, and the
 * CRC32 token of src/comm.py:517-524): digest of every structure array of the
 * operands against the symbolic-time digest; PTAP_ERR_DRIFT on mismatch.
 * (Every numeric call already checks sizes, and re-digests when a structure
 * array was replaced by another buffer.)  Synchronises. */
ptap_status ptap_plan_verify(ptap_plan *plan, const ptap_operands *ops, void *stream);
/* Two-step only: the stored auxiliary C~ = A P (reference plan.ctilde,
 * src/tripleproduct.py:105-145), rows of the rank, global columns. */
ptap_status ptap_plan_get_ctilde(ptap_plan *plan, ptap_c_view *out);

ptap_status ptap_plan_get_c(ptap_plan *plan, ptap_c_view *out);
ptap_status ptap_plan_release_cache(ptap_plan *plan);
ptap_status ptap_plan_memory(ptap_plan *plan, ptap_memory *out);
ptap_status ptap_plan_counters(ptap_plan *plan, ptap_counters *out);

/* Row-wise SpGEMM C~ = A P on its own (reference symbolic_ap / numeric_ap,
 * src/spgemm.py:184-234): output rows keep global columns. */
ptap_status ptap_spgemm_ap_symbolic(const ptap_operands *ops, int64_t *nnz_out,
                                    int64_t **row_ptr_out, int32_t **col_out, void *stream);
ptap_status ptap_spgemm_ap_numeric(const ptap_operands *ops, const int64_t *row_ptr,
                                   const int32_t *col, double *val, void *stream);
ptap_status ptap_device_free(void *ptr, void *stream);

/* Transpose of a device CSR block with the value permutation (reference
 * CsrMatrix.transpose_with_permutation, src/sparse.py:165-178): t_rp
 * (ncols+1), t_col (nnz: source rows, ascending within each row), perm (nnz:
 * t entry -> source entry, the stable argsort of the columns), t_val (nnz,
 * optional: val[perm]).  Caller-owned device buffers.  Synchronises. */
ptap_status ptap_transpose(int64_t nrows, int64_t ncols, const int64_t *row_ptr, const int32_t *col,
                           const double *val, int64_t nnz, int64_t *t_row_ptr, int32_t *t_col, int64_t *perm,
                           double *t_val, void *stream);

/* Device generators of the BASELINE configurations (bit-identical to the
 * host generators in problems.py). Row block [row_lo, row_hi) of an n^3 grid.
 * Two-call protocol: row_ptr first (nnz returned), then col/val. */
ptap_status ptap_gen_stencil_rowptr(int points, int64_t n, int64_t row_lo, int64_t row_hi,
                                    int64_t *row_ptr, int64_t *nnz_out, void *stream);
ptap_status ptap_gen_stencil_fill(int points, int kind, uint64_t seed, int64_t n, int64_t row_lo,
                                  int64_t row_hi, const int64_t *row_ptr, int32_t *col,
                                  double *val, void *stream);
ptap_status ptap_gen_trilinear_rowptr(int64_t nc, int64_t row_lo, int64_t row_hi,
                                      int64_t *row_ptr, int64_t *nnz_out, void *stream);
ptap_status ptap_gen_trilinear_fill(int64_t nc, int64_t row_lo, int64_t row_hi,
                                    const int64_t *row_ptr, int32_t *col, double *val,
                                    void *stream);

/* Config 4 (block transport, problems_amg.block_transport): nn^3 nodes x ncomp
 * components, 7-point coupling per component plus a dense in-node block;
 * P = (I - omega D^-1 A) P_tent over agg^3 node aggregates with scipy's
 * operation order (bit-identical to the host generator for the same omega).
 * row_ptr of A and P first, then A, then (omega from the caller's power
 * iteration, ptap_gen_spmv_dinv: w = D^-1 A v) P from A's values. */
ptap_status ptap_gen_block_transport_rowptr(int64_t nn, int ncomp, int64_t agg, int64_t row_lo, int64_t row_hi,
                                            int64_t *a_row_ptr, int64_t *a_nnz_out, int64_t *p_row_ptr,
                                            int64_t *p_nnz_out, void *stream);
ptap_status ptap_gen_block_transport_a(int64_t nn, int ncomp, uint64_t seed, int64_t row_lo, int64_t row_hi,
                                       const int64_t *row_ptr, int32_t *col, double *val, void *stream);
ptap_status ptap_gen_spmv_dinv(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *val,
                               const double *v, double *w, void *stream);
ptap_status ptap_gen_block_transport_p(int64_t nn, int ncomp, int64_t agg, double omega, int64_t row_lo,
                                       int64_t row_hi, const int64_t *a_row_ptr, const double *a_val,
                                       const int64_t *p_row_ptr, int32_t *p_col, double *p_val, void *stream);

/* Config 5 (problems_amg.knn_laplacian): the K nearest neighbours (K <= 32) of
 * n points of the unit cube, given sorted by cell of a G^3 grid with the
 * cells' offsets (G^3 + 1); neighbours in sorted-index space, ascending
 * squared distance.  The rest of the generator (symmetrised graph, greedy
 * distance-2 aggregation, smoothed P) is device tensor plumbing in devgen.py. */
ptap_status ptap_gen_knn(int64_t n, const double *pts, const int64_t *cell_start, int G, int K,
                         int32_t *out_idx, double *out_d2, void *stream);

/* Device L2 flush helper for benchmarking (writes a buffer larger than L2). */
ptap_status ptap_l2_flush(void *stream);

#ifdef __cplusplus
}
#endif
#endif /* PTAP_B200_H */
