/*
 * ptap_oracle.c -- CPU restatement of the reference PtAP algorithms.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker, not product
 * code: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load it.  The product path (the CUDA library
 * under paper_1905_08423_b200/csrc) never links or calls it.
 *
 * What it restates (reference = /root/reference/pkg/src/ptap, "src/" below):
 *   - make_partition               src/partition.py:51-60
 *   - diag/offdiag row split        src/partition.py:123-154
 *   - remote-row gather of P        src/comm.py:527-622 (the served row is the
 *                                   owner's row merged and sorted by global
 *                                   column, i.e. the global row of P)
 *   - AP row fold                   src/_kernels.py:205-227 (A_d entries in
 *                                   ascending local column, then A_o entries in
 *                                   ascending compact = ascending global column;
 *                                   first product *sets* the slot, later ones
 *                                   add, hm_add :116-147)
 *   - all-at-once / merged numeric  src/_kernels.py:446-515 and
 *                                   src/tripleproduct.py:303-355
 *   - all-at-once / merged symbolic src/_kernels.py:361-418 and
 *                                   src/tripleproduct.py:241-300 (combined-key
 *                                   arena, Fibonacci hash, 75% growth)
 *   - two-step symbolic / numeric   src/tripleproduct.py:380-490,
 *                                   src/_kernels.py:248-349, 558-677,
 *                                   src/sparse.py:165-178 (stable transpose)
 *   - contribution merge order      src/tripleproduct.py:215-229: local
 *                                   contributions first, then received batches
 *                                   in ascending source rank.
 *
 * Arithmetic: every multiply is rounded before the add (no FMA contraction;
 * build with -ffp-contract=off), matching numba's default IEEE semantics.
 * The per-entry summation order is exactly the reference's, so the output is
 * bit-identical to the reference at the same rank count (pinned against
 * fixtures generated from the reference itself: tests/golden/).
 *
 * Ranks are simulated in one process (as the reference's thread harness
 * does); when built with OpenMP, per-rank local work runs one rank per
 * thread, which changes nothing in the arithmetic.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ALG_TWO_STEP 0
#define ALG_ALLATONCE 1
#define ALG_MERGED 2

typedef struct {
    int64_t rows_sym;     /* AP-row kernel calls in symbolic (reference counter) */
    int64_t rows_num;     /* AP-row kernel calls in numeric  */
    int64_t nnz_c;
    int64_t mac_ap;       /* sum over (i,k) in A of nnz(P(k,:)) restricted to processed rows */
    int64_t mac_outer;    /* sum over processed rows of nnz(P(i,:)) * nnz(AP(i,:)) */
    int64_t staged_entries; /* total send-side staging entries over ranks */
} oracle_stats;

/* ------------------------------------------------------------------ */
/* partition (src/partition.py:51-60)                                   */
/* ------------------------------------------------------------------ */
static void block_rows(int64_t n, int np, int64_t *off) {
    int64_t base = n / np, extra = n % np;
    off[0] = 0;
    for (int r = 0; r < np; r++) off[r + 1] = off[r] + base + (r < extra ? 1 : 0);
}

/* ------------------------------------------------------------------ */
/* combined-key arena: open addressing, linear probing, pow2 capacity,  */
/* growth at 75% load, empty = -1 (src/_kernels.py:42-108)              */
/* ------------------------------------------------------------------ */
typedef struct { int64_t *keys; int64_t cap, size; } arena_t;
static const uint64_t FIB = 0x9E3779B97F4A7C15ull;

static void arena_init(arena_t *a, int64_t cap) {
    a->cap = cap; a->size = 0;
    a->keys = (int64_t *)malloc(sizeof(int64_t) * cap);
    for (int64_t s = 0; s < cap; s++) a->keys[s] = -1;
}
static void arena_put_raw(int64_t *keys, int64_t cap, int64_t k) {
    uint64_t mask = (uint64_t)cap - 1, h = ((uint64_t)k * FIB) & mask;
    while (keys[h] >= 0) h = (h + 1) & mask;
    keys[h] = k;
}
static void arena_insert(arena_t *a, int64_t k) {
    if ((a->size + 1) * 4 > 3 * a->cap) {
        int64_t ncap = a->cap * 2;
        int64_t *nk = (int64_t *)malloc(sizeof(int64_t) * ncap);
        for (int64_t s = 0; s < ncap; s++) nk[s] = -1;
        for (int64_t s = 0; s < a->cap; s++) if (a->keys[s] >= 0) arena_put_raw(nk, ncap, a->keys[s]);
        free(a->keys); a->keys = nk; a->cap = ncap;
    }
    uint64_t mask = (uint64_t)a->cap - 1, h = ((uint64_t)k * FIB) & mask;
    for (;;) {
        int64_t cur = a->keys[h];
        if (cur == k) return;
        if (cur < 0) { a->keys[h] = k; a->size++; return; }
        h = (h + 1) & mask;
    }
}
static int cmp_i64(const void *x, const void *y) {
    int64_t a = *(const int64_t *)x, b = *(const int64_t *)y;
    return (a > b) - (a < b);
}
/* sorted occupied keys (src/tripleproduct.py:165-168) */
static int64_t *arena_drain(arena_t *a, int64_t *count) {
    int64_t *out = (int64_t *)malloc(sizeof(int64_t) * (a->size ? a->size : 1));
    int64_t n = 0;
    for (int64_t s = 0; s < a->cap; s++) if (a->keys[s] >= 0) out[n++] = a->keys[s];
    qsort(out, n, sizeof(int64_t), cmp_i64);
    *count = n;
    return out;
}
static void arena_free(arena_t *a) { free(a->keys); a->keys = NULL; }

/* ------------------------------------------------------------------ */
/* sparse accumulator for one row (plays the RowSet/RowAccumulator role) */
/* ------------------------------------------------------------------ */
typedef struct { int64_t *stamp; double *val; int64_t *list; int64_t len, epoch; } spa_t;
static void spa_init(spa_t *s, int64_t m, int64_t maxlen) {
    s->stamp = (int64_t *)calloc(m ? m : 1, sizeof(int64_t));
    s->val = (double *)calloc(m ? m : 1, sizeof(double));
    s->list = (int64_t *)malloc(sizeof(int64_t) * (maxlen ? maxlen : 1));
    s->len = 0; s->epoch = 0;
}
static void spa_free(spa_t *s) { free(s->stamp); free(s->val); free(s->list); }
static inline void spa_clear(spa_t *s) { s->epoch++; s->len = 0; }
/* hm_add semantics: first write sets, later writes add (src/_kernels.py:116-147) */
static inline void spa_add(spa_t *s, int64_t g, double v) {
    if (s->stamp[g] != s->epoch) { s->stamp[g] = s->epoch; s->val[g] = v; s->list[s->len++] = g; }
    else s->val[g] = s->val[g] + v;
}
static inline void spa_mark(spa_t *s, int64_t g) {
    if (s->stamp[g] != s->epoch) { s->stamp[g] = s->epoch; s->list[s->len++] = g; }
}

/* ------------------------------------------------------------------ */
/* the global problem and one rank's view                               */
/* ------------------------------------------------------------------ */
typedef struct {
    int64_t n, m;
    const int64_t *a_ip, *a_j; const double *a_v;
    const int64_t *p_ip, *p_j; const double *p_v;
    int np;
    int64_t *roff, *coff;          /* row partition of A/P, partition of C */
} prob_t;

/* Row i of A in the rank's fold order: A_d entries (columns owned by the
 * rank, ascending), then A_o entries (the rest, ascending global column).
 * Calls body(k, a) for each entry. */
#define FOR_A_ROW_RANK_ORDER(pr, lo, hi, i, K, AV, BODY)                         \
    do {                                                                          \
        for (int64_t _t = (pr)->a_ip[i]; _t < (pr)->a_ip[(i) + 1]; _t++) {        \
            int64_t K = (pr)->a_j[_t];                                            \
            if (K < (lo) || K >= (hi)) continue;                                  \
            double AV = (pr)->a_v ? (pr)->a_v[_t] : 0.0; (void)AV;                \
            BODY                                                                  \
        }                                                                         \
        for (int64_t _t = (pr)->a_ip[i]; _t < (pr)->a_ip[(i) + 1]; _t++) {        \
            int64_t K = (pr)->a_j[_t];                                            \
            if (K >= (lo) && K < (hi)) continue;                                  \
            double AV = (pr)->a_v ? (pr)->a_v[_t] : 0.0; (void)AV;                \
            BODY                                                                  \
        }                                                                         \
    } while (0)

/* AP row i (src/_kernels.py:205-227); values folded in rank order. */
static void ap_row_numeric(const prob_t *pr, int64_t lo, int64_t hi, int64_t i, spa_t *s) {
    spa_clear(s);
    FOR_A_ROW_RANK_ORDER(pr, lo, hi, i, k, a, {
        for (int64_t u = pr->p_ip[k]; u < pr->p_ip[k + 1]; u++) {
            double prod = a * pr->p_v[u];
            spa_add(s, pr->p_j[u], prod);
        }
    });
}
static void ap_row_symbolic(const prob_t *pr, int64_t lo, int64_t hi, int64_t i, spa_t *s) {
    spa_clear(s);
    FOR_A_ROW_RANK_ORDER(pr, lo, hi, i, k, a, {
        for (int64_t u = pr->p_ip[k]; u < pr->p_ip[k + 1]; u++) spa_mark(s, pr->p_j[u]);
    });
}

/* binary search of global column g in row J of the assembled C pattern */
static inline int64_t c_slot(const int64_t *c_ip, const int64_t *c_j, int64_t J, int64_t g) {
    int64_t lo = c_ip[J], hi = c_ip[J + 1];
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (c_j[mid] < g) lo = mid + 1; else hi = mid;
    }
    return (lo < c_ip[J + 1] && c_j[lo] == g) ? lo : -1;
}

/* ------------------------------------------------------------------ */
/* per-rank local transpose of the P row block (src/sparse.py:165-178): */
/* rows = columns of P restricted to [c0,c1) (diag) or outside (offdiag)*/
/* entries ascending in local row i (stable).                          */
/* ------------------------------------------------------------------ */
typedef struct { int64_t nrows; int64_t *rowid; int64_t *ip; int64_t *i; double *v; } ptrans_t;

static void local_transpose(const prob_t *pr, int64_t lo, int64_t hi, int64_t c0, int64_t c1,
                            int offdiag, ptrans_t *t) {
    /* collect the distinct target columns first (diag: all of [c0,c1); offdiag: col_map) */
    int64_t m = pr->m;
    int64_t *cnt = (int64_t *)calloc(m + 1, sizeof(int64_t));
    for (int64_t i = lo; i < hi; i++)
        for (int64_t u = pr->p_ip[i]; u < pr->p_ip[i + 1]; u++) {
            int64_t J = pr->p_j[u];
            int inside = (J >= c0 && J < c1);
            if (inside != !offdiag) continue;
            cnt[J]++;
        }
    int64_t nrows = 0;
    if (!offdiag) nrows = c1 - c0;
    else for (int64_t J = 0; J < m; J++) if (cnt[J]) nrows++;
    t->nrows = nrows;
    t->rowid = (int64_t *)malloc(sizeof(int64_t) * (nrows ? nrows : 1));
    t->ip = (int64_t *)calloc(nrows + 1, sizeof(int64_t));
    int64_t *rowof = (int64_t *)malloc(sizeof(int64_t) * (m ? m : 1));
    int64_t r = 0;
    if (!offdiag) { for (int64_t J = c0; J < c1; J++) { rowof[J] = r; t->rowid[r] = J; t->ip[r + 1] = cnt[J]; r++; } }
    else for (int64_t J = 0; J < m; J++) if (cnt[J]) { rowof[J] = r; t->rowid[r] = J; t->ip[r + 1] = cnt[J]; r++; }
    for (int64_t q = 0; q < nrows; q++) t->ip[q + 1] += t->ip[q];
    int64_t tot = t->ip[nrows];
    t->i = (int64_t *)malloc(sizeof(int64_t) * (tot ? tot : 1));
    t->v = (double *)malloc(sizeof(double) * (tot ? tot : 1));
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (nrows ? nrows : 1));
    for (int64_t q = 0; q < nrows; q++) cur[q] = t->ip[q];
    for (int64_t i = lo; i < hi; i++)
        for (int64_t u = pr->p_ip[i]; u < pr->p_ip[i + 1]; u++) {
            int64_t J = pr->p_j[u];
            int inside = (J >= c0 && J < c1);
            if (inside != !offdiag) continue;
            int64_t q = rowof[J];
            t->i[cur[q]] = i;
            t->v[cur[q]] = pr->p_v ? pr->p_v[u] : 0.0;
            cur[q]++;
        }
    free(cnt); free(rowof); free(cur);
}
static void ptrans_free(ptrans_t *t) { free(t->rowid); free(t->ip); free(t->i); free(t->v); }

/* C~ = A*P rows of one rank, sorted structure + values (two-step,
 * src/spgemm.py:184-234, src/_kernels.py:248-349) */
typedef struct { int64_t lo, hi; int64_t *ip, *j; double *v; } ctilde_t;

static void build_ctilde(const prob_t *pr, int64_t lo, int64_t hi, spa_t *s, int with_values, ctilde_t *ct) {
    int64_t nr = hi - lo;
    ct->lo = lo; ct->hi = hi;
    ct->ip = (int64_t *)calloc(nr + 1, sizeof(int64_t));
    for (int64_t i = lo; i < hi; i++) { ap_row_symbolic(pr, lo, hi, i, s); ct->ip[i - lo + 1] = ct->ip[i - lo] + s->len; }
    int64_t tot = ct->ip[nr];
    ct->j = (int64_t *)malloc(sizeof(int64_t) * (tot ? tot : 1));
    ct->v = with_values ? (double *)malloc(sizeof(double) * (tot ? tot : 1)) : NULL;
    for (int64_t i = lo; i < hi; i++) {
        if (with_values) ap_row_numeric(pr, lo, hi, i, s); else ap_row_symbolic(pr, lo, hi, i, s);
        int64_t base = ct->ip[i - lo];
        memcpy(ct->j + base, s->list, sizeof(int64_t) * s->len);
        qsort(ct->j + base, s->len, sizeof(int64_t), cmp_i64);
        if (with_values) for (int64_t q = 0; q < s->len; q++) ct->v[base + q] = s->val[ct->j[base + q]];
    }
}
static void ctilde_free(ctilde_t *ct) { free(ct->ip); free(ct->j); free(ct->v); }

/* ------------------------------------------------------------------ */
/* SYMBOLIC: per-rank send arena (global row keys) and local arena      */
/* (local row keys), then owner merge and assembly.                     */
/* ------------------------------------------------------------------ */
typedef struct { arena_t send, local; int64_t rows_processed; } rank_sym_t;

static void symbolic_outer_rank(const prob_t *pr, int r, int alg, spa_t *s, rank_sym_t *rs) {
    int64_t lo = pr->roff[r], hi = pr->roff[r + 1];
    int64_t c0 = pr->coff[r], c1 = pr->coff[r + 1];
    int64_t m = pr->m;
    arena_init(&rs->send, 64); arena_init(&rs->local, 64);
    rs->rows_processed = 0;
    int passes = (alg == ALG_MERGED) ? 1 : 2;
    for (int pass = 0; pass < passes; pass++) {
        int do_send = (alg == ALG_MERGED) || pass == 0;
        int do_local = (alg == ALG_MERGED) || pass == 1;
        for (int64_t i = lo; i < hi; i++) {
            int pd = 0, po = 0;
            for (int64_t u = pr->p_ip[i]; u < pr->p_ip[i + 1]; u++) {
                int64_t J = pr->p_j[u];
                if (J >= c0 && J < c1) pd = 1; else po = 1;
            }
            int ws = do_send && po, wl = do_local && pd;
            if (!(ws || wl)) continue;
            rs->rows_processed++;
            ap_row_symbolic(pr, lo, hi, i, s);
            for (int64_t u = pr->p_ip[i]; u < pr->p_ip[i + 1]; u++) {
                int64_t J = pr->p_j[u];
                int inside = (J >= c0 && J < c1);
                if (inside && wl) { for (int64_t q = 0; q < s->len; q++) arena_insert(&rs->local, (J - c0) * m + s->list[q]); }
                else if (!inside && ws) { for (int64_t q = 0; q < s->len; q++) arena_insert(&rs->send, J * m + s->list[q]); }
            }
        }
    }
}

static void symbolic_two_step_rank(const prob_t *pr, int r, spa_t *s, rank_sym_t *rs) {
    int64_t lo = pr->roff[r], hi = pr->roff[r + 1];
    int64_t c0 = pr->coff[r], c1 = pr->coff[r + 1];
    int64_t m = pr->m;
    arena_init(&rs->send, 64); arena_init(&rs->local, 64);
    rs->rows_processed = hi - lo;
    ctilde_t ct; build_ctilde(pr, lo, hi, s, 0, &ct);
    for (int part = 0; part < 2; part++) {      /* 0: Pt_o (send), 1: Pt_d (local) */
        ptrans_t t; local_transpose(pr, lo, hi, c0, c1, part == 0, &t);
        for (int64_t q = 0; q < t.nrows; q++) {
            if (t.ip[q] == t.ip[q + 1]) continue;
            int64_t J = t.rowid[q];
            int64_t base = (part == 0 ? J : (J - c0)) * m;
            for (int64_t e = t.ip[q]; e < t.ip[q + 1]; e++) {
                int64_t li = t.i[e] - lo;
                for (int64_t x = ct.ip[li]; x < ct.ip[li + 1]; x++)
                    arena_insert(part == 0 ? &rs->send : &rs->local, base + ct.j[x]);
            }
        }
        ptrans_free(&t);
    }
    ctilde_free(&ct);
}

/* builds the global C pattern; returns nnz */
static int64_t run_symbolic(const prob_t *pr, int alg, int64_t **c_ip_out, int64_t **c_j_out,
                            oracle_stats *st) {
    int np = pr->np;
    int64_t m = pr->m;
    rank_sym_t *rs = (rank_sym_t *)calloc(np, sizeof(rank_sym_t));
    int64_t rows_total = 0;
#pragma omp parallel
    {
        spa_t s; spa_init(&s, m, m);
#pragma omp for schedule(dynamic, 1)
        for (int r = 0; r < np; r++) {
            if (alg == ALG_TWO_STEP) symbolic_two_step_rank(pr, r, &s, &rs[r]);
            else symbolic_outer_rank(pr, r, alg, &s, &rs[r]);
        }
        spa_free(&s);
    }
    int64_t staged = 0;
    /* owner merge: received send-arena keys (global row) in ascending source
     * order (src/tripleproduct.py:195-200) -- order is irrelevant for a set */
    for (int src = 0; src < np; src++) {
        rows_total += rs[src].rows_processed;
        int64_t cnt; int64_t *keys = arena_drain(&rs[src].send, &cnt);
        staged += cnt;
        for (int64_t q = 0; q < cnt; q++) {
            int64_t J = keys[q] / m, g = keys[q] % m;
            int o = 0;
            while (!(J >= pr->coff[o] && J < pr->coff[o + 1])) o++;
            arena_insert(&rs[o].local, (J - pr->coff[o]) * m + g);
        }
        free(keys);
        arena_free(&rs[src].send);
    }
    int64_t *c_ip = (int64_t *)calloc(m + 1, sizeof(int64_t));
    int64_t total = 0;
    int64_t **dr = (int64_t **)calloc(np, sizeof(int64_t *));
    int64_t *dn = (int64_t *)calloc(np, sizeof(int64_t));
    for (int o = 0; o < np; o++) {
        dr[o] = arena_drain(&rs[o].local, &dn[o]);
        arena_free(&rs[o].local);
        for (int64_t q = 0; q < dn[o]; q++) c_ip[pr->coff[o] + dr[o][q] / m + 1]++;
        total += dn[o];
    }
    for (int64_t J = 0; J < m; J++) c_ip[J + 1] += c_ip[J];
    int64_t *c_j = (int64_t *)malloc(sizeof(int64_t) * (total ? total : 1));
    int64_t pos = 0;
    for (int o = 0; o < np; o++) {         /* drained keys are sorted by (row, col) */
        for (int64_t q = 0; q < dn[o]; q++) c_j[pos++] = dr[o][q] % m;
        free(dr[o]);
    }
    free(dr); free(dn); free(rs);
    *c_ip_out = c_ip; *c_j_out = c_j;
    if (st) { st->rows_sym = rows_total; st->nnz_c = total; st->staged_entries = staged; }
    return total;
}

/* ------------------------------------------------------------------ */
/* NUMERIC                                                              */
/* ------------------------------------------------------------------ */
/* all-at-once / merged (src/_kernels.py:446-515): staging[r] and C share */
/* the global C pattern's slot numbering.                                */
static void numeric_outer_rank(const prob_t *pr, int r, int alg, const int64_t *c_ip, const int64_t *c_j,
                               double *cvals, double *stage, spa_t *s, int64_t *rows_out,
                               int64_t *mac_ap, int64_t *mac_outer) {
    int64_t lo = pr->roff[r], hi = pr->roff[r + 1];
    int64_t c0 = pr->coff[r], c1 = pr->coff[r + 1];
    int64_t rows = 0, mapc = 0, moc = 0;
    int passes = (alg == ALG_MERGED) ? 1 : 2;
    for (int pass = 0; pass < passes; pass++) {
        int do_send = (alg == ALG_MERGED) || pass == 0;
        int do_local = (alg == ALG_MERGED) || pass == 1;
        for (int64_t i = lo; i < hi; i++) {
            int pd = 0, po = 0;
            for (int64_t u = pr->p_ip[i]; u < pr->p_ip[i + 1]; u++) {
                int64_t J = pr->p_j[u];
                if (J >= c0 && J < c1) pd = 1; else po = 1;
            }
            int ws = do_send && po, wl = do_local && pd;
            if (!(ws || wl)) continue;
            rows++;
            ap_row_numeric(pr, lo, hi, i, s);
            for (int64_t t = pr->a_ip[i]; t < pr->a_ip[i + 1]; t++) {
                int64_t k = pr->a_j[t];
                mapc += pr->p_ip[k + 1] - pr->p_ip[k];
            }
            for (int64_t u = pr->p_ip[i]; u < pr->p_ip[i + 1]; u++) {
                int64_t J = pr->p_j[u];
                double pv = pr->p_v[u];
                int inside = (J >= c0 && J < c1);
                double *tgt;
                if (inside && wl) tgt = cvals;
                else if (!inside && ws) tgt = stage;
                else continue;
                moc += s->len;
                for (int64_t q = 0; q < s->len; q++) {
                    int64_t g = s->list[q];
                    int64_t slot = c_slot(c_ip, c_j, J, g);
                    double prod = pv * s->val[g];
                    tgt[slot] = tgt[slot] + prod;
                }
            }
        }
    }
    *rows_out = rows; *mac_ap = mapc; *mac_outer = moc;
}

/* two-step numeric (src/tripleproduct.py:440-490) */
static void numeric_two_step_rank(const prob_t *pr, int r, const int64_t *c_ip, const int64_t *c_j,
                                  double *cvals, double *stage, spa_t *s) {
    int64_t lo = pr->roff[r], hi = pr->roff[r + 1];
    int64_t c0 = pr->coff[r], c1 = pr->coff[r + 1];
    ctilde_t ct; build_ctilde(pr, lo, hi, s, 1, &ct);
    for (int part = 0; part < 2; part++) {      /* 0: Pt_o -> staging, 1: Pt_d -> C */
        ptrans_t t; local_transpose(pr, lo, hi, c0, c1, part == 0, &t);
        for (int64_t q = 0; q < t.nrows; q++) {
            if (t.ip[q] == t.ip[q + 1]) continue;
            int64_t J = t.rowid[q];
            spa_clear(s);
            for (int64_t e = t.ip[q]; e < t.ip[q + 1]; e++) {
                int64_t li = t.i[e] - lo;
                double lv = t.v[e];
                for (int64_t x = ct.ip[li]; x < ct.ip[li + 1]; x++) {
                    double prod = lv * ct.v[x];
                    spa_add(s, ct.j[x], prod);
                }
            }
            for (int64_t x = 0; x < s->len; x++) {
                int64_t g = s->list[x];
                int64_t slot = c_slot(c_ip, c_j, J, g);
                if (part == 0) stage[slot] = s->val[g];              /* staging set */
                else cvals[slot] = cvals[slot] + s->val[g];          /* C += acc    */
            }
        }
        ptrans_free(&t);
    }
    ctilde_free(&ct);
}

static void run_numeric(const prob_t *pr, int alg, const int64_t *c_ip, const int64_t *c_j, int64_t nnz,
                        double *cvals, oracle_stats *st) {
    int np = pr->np;
    int64_t m = pr->m;
    double **stage = (double **)calloc(np, sizeof(double *));
    int64_t *rows = (int64_t *)calloc(np, sizeof(int64_t));
    int64_t *mapc = (int64_t *)calloc(np, sizeof(int64_t));
    int64_t *moc = (int64_t *)calloc(np, sizeof(int64_t));
    for (int64_t q = 0; q < nnz; q++) cvals[q] = 0.0;
#pragma omp parallel
    {
        spa_t s; spa_init(&s, m, m);
#pragma omp for schedule(dynamic, 1)
        for (int r = 0; r < np; r++) {
            stage[r] = (np > 1) ? (double *)calloc(nnz ? nnz : 1, sizeof(double)) : NULL;
            if (alg == ALG_TWO_STEP) numeric_two_step_rank(pr, r, c_ip, c_j, cvals, stage[r], &s);
            else numeric_outer_rank(pr, r, alg, c_ip, c_j, cvals, stage[r], &s, &rows[r], &mapc[r], &moc[r]);
        }
        spa_free(&s);
    }
    /* merge: per owner, received staging in ascending source rank, after
     * all local contributions (src/tripleproduct.py:215-229) */
    if (np > 1) {
#pragma omp parallel for schedule(dynamic, 1)
        for (int o = 0; o < np; o++) {
            for (int src = 0; src < np; src++) {
                if (src == o) continue;
                for (int64_t J = pr->coff[o]; J < pr->coff[o + 1]; J++)
                    for (int64_t q = c_ip[J]; q < c_ip[J + 1]; q++) cvals[q] = cvals[q] + stage[src][q];
            }
        }
    }
    if (st) {
        st->rows_num = 0; st->mac_ap = 0; st->mac_outer = 0;
        for (int r = 0; r < np; r++) { st->rows_num += rows[r]; st->mac_ap += mapc[r]; st->mac_outer += moc[r]; }
    }
    for (int r = 0; r < np; r++) free(stage[r]);
    free(stage); free(rows); free(mapc); free(moc);
}

/* ------------------------------------------------------------------ */
/* exported entry points (ctypes)                                       */
/* ------------------------------------------------------------------ */
typedef struct {
    int64_t *c_ip, *c_j; int64_t nnz; int64_t m;
    int64_t *roff, *coff;
    prob_t pr;
    int alg;
} oracle_plan;

/* Symbolic phase: returns an opaque plan holding the assembled C pattern. */
void *ptap_oracle_symbolic(int64_t n, int64_t m,
                           const int64_t *a_ip, const int64_t *a_j,
                           const int64_t *p_ip, const int64_t *p_j,
                           int nranks, int algorithm, oracle_stats *st) {
    oracle_plan *pl = (oracle_plan *)calloc(1, sizeof(oracle_plan));
    pl->roff = (int64_t *)malloc(sizeof(int64_t) * (nranks + 1));
    pl->coff = (int64_t *)malloc(sizeof(int64_t) * (nranks + 1));
    block_rows(n, nranks, pl->roff);
    block_rows(m, nranks, pl->coff);
    prob_t pr = {n, m, a_ip, a_j, NULL, p_ip, p_j, NULL, nranks, pl->roff, pl->coff};
    pl->pr = pr; pl->m = m; pl->alg = algorithm;
    pl->nnz = run_symbolic(&pl->pr, algorithm, &pl->c_ip, &pl->c_j, st);
    return pl;
}

int64_t ptap_oracle_nnz(void *plan) { return ((oracle_plan *)plan)->nnz; }

void ptap_oracle_pattern(void *plan, int64_t *c_ip, int64_t *c_j) {
    oracle_plan *pl = (oracle_plan *)plan;
    memcpy(c_ip, pl->c_ip, sizeof(int64_t) * (pl->m + 1));
    memcpy(c_j, pl->c_j, sizeof(int64_t) * pl->nnz);
}

/* Numeric phase on the plan's pattern; A/P structure must be the one given
 * to the symbolic phase (the reference raises StructuralDriftError otherwise). */
int ptap_oracle_numeric(void *plan, const int64_t *a_ip, const int64_t *a_j, const double *a_v,
                        const int64_t *p_ip, const int64_t *p_j, const double *p_v,
                        double *c_vals, oracle_stats *st) {
    oracle_plan *pl = (oracle_plan *)plan;
    prob_t pr = pl->pr;
    pr.a_ip = a_ip; pr.a_j = a_j; pr.a_v = a_v;
    pr.p_ip = p_ip; pr.p_j = p_j; pr.p_v = p_v;
    run_numeric(&pr, pl->alg, pl->c_ip, pl->c_j, pl->nnz, c_vals, st);
    return 0;
}

void ptap_oracle_free(void *plan) {
    oracle_plan *pl = (oracle_plan *)plan;
    if (!pl) return;
    free(pl->c_ip); free(pl->c_j); free(pl->roff); free(pl->coff); free(pl);
}

int ptap_oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
