/*
 * oracle/ref_scan.c -- TEST INFRASTRUCTURE ONLY (parity checker + CPU
 * baseline).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this; the product path never
 * does.
 *
 * Plain-C restatement of the reference kmerscan scan path
 * (/root/reference/pkg/src/kmerscan), function by function:
 *   ref_scan_from       <- _kernels.py:18-29   scan_from
 *   ref_match_chunk     <- _kernels.py:43-113  match_chunk_kernel (+ _push_location :32-40)
 *   ref_pss             <- engine.py:80-91     possible_starting_states (np.unique image)
 *   plan                <- ingest.py:78-94     plan_chunks (floor split, remainder last)
 *   ref_run             <- engine.py:137-237   run + reduce (chain walk, splice, lexsort)
 * Threads: one pthread per chunk, like the reference's ThreadPoolExecutor
 * (engine.py:223-232).  Pinned against the reference's golden vectors and
 * against fixtures produced by the real reference (tests/golden/).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OTHER_SYMS 5

typedef struct {
    const int32_t* trans; /* nq x 5 */
    int32_t nq;
    const int32_t* out_off;
    const int32_t* out_ids;
    int32_t ne;
} RefDfa;

typedef struct {
    int64_t* rows; /* pairs */
    int64_t n, cap;
} Rows;

static int rows_push(Rows* r, int64_t off, int64_t id) {
    if (r->n == r->cap) {
        int64_t cap = 2 * r->cap + 64;
        int64_t* p = (int64_t*)realloc(r->rows, (size_t)cap * 16);
        if (!p) return -1;
        r->rows = p;
        r->cap = cap;
    }
    r->rows[2 * r->n] = off;
    r->rows[2 * r->n + 1] = id;
    r->n++;
    return 0;
}

/* _kernels.py:18-29 */
int64_t ref_scan_from(const int32_t* trans, const int32_t* out_off, const int32_t* out_ids,
                      const uint8_t* sym, int64_t start, int64_t end, int64_t state, int64_t* counts) {
    int64_t s = state;
    for (int64_t j = start; j < end; ++j) {
        s = trans[s * OTHER_SYMS + sym[j]];
        for (int32_t k = out_off[s]; k < out_off[s + 1]; ++k) counts[out_ids[k]] += 1;
    }
    return s;
}

/* _kernels.py:43-113.  Per run i: counts[i*ne..], last[i], conv[i];
 * rows[i] (locate) for the run's own emitted locations. */
typedef struct {
    int64_t nr;
    int64_t* counts; /* nr x ne */
    int64_t* last;
    int64_t* conv;
    Rows* rows; /* nr, or NULL */
} ChunkOut;

static int ref_match_chunk(const RefDfa* d, const uint8_t* sym, int64_t c_start, int64_t c_end,
                           int64_t g_off, const int64_t* pss, int64_t nr, int64_t window, int locate,
                           ChunkOut* out) {
    const int64_t m = c_end - c_start;
    const int64_t ne = d->ne;
    const int64_t weff = window < m ? window : m;
    int64_t* fr_states = (int64_t*)malloc((size_t)(weff > 0 ? weff : 1) * 8);
    int64_t* fr_counts = (int64_t*)calloc((size_t)((weff > 0 ? weff : 1) * (ne > 0 ? ne : 1)), 8);
    if (!fr_states || !fr_counts) return -1;
    memset(out->counts, 0, (size_t)(nr * ne) * 8);

    /* full run R0 records the convergence window */
    int64_t s = pss[0];
    int64_t* c0 = out->counts;
    for (int64_t j = 0; j < m; ++j) {
        s = d->trans[s * OTHER_SYMS + sym[c_start + j]];
        for (int32_t k = d->out_off[s]; k < d->out_off[s + 1]; ++k) {
            int32_t e = d->out_ids[k];
            c0[e] += 1;
            if (locate && rows_push(&out->rows[0], g_off + j + 1, e)) return -1;
        }
        if (j < weff) {
            fr_states[j] = s;
            memcpy(&fr_counts[j * ne], c0, (size_t)ne * 8);
        }
    }
    out->last[0] = s;
    out->conv[0] = -1;

    /* speculative runs stop at the first state shared with R0 and reconcile */
    for (int64_t i = 1; i < nr; ++i) {
        int64_t* ci = &out->counts[i * ne];
        s = pss[i];
        out->conv[i] = -1;
        for (int64_t j = 0; j < m; ++j) {
            s = d->trans[s * OTHER_SYMS + sym[c_start + j]];
            for (int32_t k = d->out_off[s]; k < d->out_off[s + 1]; ++k) {
                int32_t e = d->out_ids[k];
                ci[e] += 1;
                if (locate && rows_push(&out->rows[i], g_off + j + 1, e)) return -1;
            }
            if (j < weff && s == fr_states[j]) {
                out->conv[i] = j;
                for (int64_t e = 0; e < ne; ++e) ci[e] += c0[e] - fr_counts[j * ne + e];
                s = out->last[0];
                break;
            }
        }
        out->last[i] = s;
    }
    free(fr_states);
    free(fr_counts);
    return 0;
}

/* engine.py:80-91: sorted unique image of column `prev_last` */
static int64_t ref_pss(const RefDfa* d, int prev_last, int64_t* out, uint8_t* seen) {
    memset(seen, 0, (size_t)d->nq);
    for (int32_t q = 0; q < d->nq; ++q) seen[d->trans[q * OTHER_SYMS + prev_last]] = 1;
    int64_t n = 0;
    for (int32_t q = 0; q < d->nq; ++q)
        if (seen[q]) out[n++] = q;
    return n;
}

typedef struct {
    const RefDfa* d;
    const uint8_t* sym;
    int64_t lo, hi, window;
    int locate;
    const int64_t* pss;
    int64_t nr;
    ChunkOut out;
    int rc;
} Job;

static void* job_main(void* p) {
    Job* j = (Job*)p;
    j->rc = ref_match_chunk(j->d, j->sym, j->lo, j->hi, j->lo, j->pss, j->nr, j->window, j->locate, &j->out);
    return NULL;
}

static int cmp_rows(const void* a, const void* b) {
    const int64_t* x = (const int64_t*)a;
    const int64_t* y = (const int64_t*)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
    return 0;
}

/* engine.py:207-237 (+ reduce :137-204).  Returns 0, -1 (alloc), -3 (chain).
 * conv_hist (nullable, window+1 entries) / n_spec / n_conv feed metadata. */
int ref_run(const int32_t* trans, int32_t nq, const int32_t* out_off, const int32_t* out_ids, int32_t ne,
            const uint8_t* sym, int64_t n, int64_t workers, int64_t window, int locate, int64_t* counts_out,
            int64_t** rows_out, int64_t* n_rows, int64_t* pss_sizes, int64_t* n_spec, int64_t* n_conv,
            int64_t* conv_hist) {
    RefDfa d = {trans, nq, out_off, out_ids, ne};
    int64_t w = workers < (n > 1 ? n : 1) ? workers : (n > 1 ? n : 1);
    if (w < 1) w = 1;
    const int64_t q = n / w;
    Job* jobs = (Job*)calloc((size_t)w, sizeof(Job));
    int64_t* pss_all = (int64_t*)malloc((size_t)(w * nq) * 8);
    uint8_t* seen = (uint8_t*)malloc((size_t)nq);
    pthread_t* th = (pthread_t*)malloc((size_t)w * sizeof(pthread_t));
    if (!jobs || !pss_all || !seen || !th) return -1;
    int rc = 0;
    for (int64_t i = 0; i < w; ++i) {
        Job* j = &jobs[i];
        j->d = &d;
        j->sym = sym;
        j->lo = i * q;
        j->hi = i < w - 1 ? (i + 1) * q : n;
        j->window = window;
        j->locate = locate;
        j->pss = &pss_all[i * nq];
        if (i == 0) {
            pss_all[0] = 0; /* START */
            j->nr = 1;
        } else {
            j->nr = ref_pss(&d, sym[j->lo - 1], &pss_all[i * nq], seen);
        }
        if (pss_sizes) pss_sizes[i] = j->nr;
        j->out.nr = j->nr;
        j->out.counts = (int64_t*)malloc((size_t)(j->nr * (ne > 0 ? ne : 1)) * 8);
        j->out.last = (int64_t*)malloc((size_t)j->nr * 8);
        j->out.conv = (int64_t*)malloc((size_t)j->nr * 8);
        j->out.rows = locate ? (Rows*)calloc((size_t)j->nr, sizeof(Rows)) : NULL;
        if (!j->out.counts || !j->out.last || !j->out.conv || (locate && !j->out.rows)) return -1;
    }
    if (w == 1) {
        job_main(&jobs[0]);
    } else {
        for (int64_t i = 0; i < w; ++i) pthread_create(&th[i], NULL, job_main, &jobs[i]);
        for (int64_t i = 0; i < w; ++i) pthread_join(th[i], NULL);
    }
    for (int64_t i = 0; i < w; ++i)
        if (jobs[i].rc) rc = -1;

    /* reduce: chain walk, counts, location splice, sort */
    memset(counts_out, 0, (size_t)ne * 8);
    Rows all = {NULL, 0, 0};
    int64_t want = 0, spec = 0, conv = 0;
    for (int64_t i = 0; i < w && rc == 0; ++i) {
        Job* j = &jobs[i];
        int64_t sel = -1;
        for (int64_t r = 0; r < j->nr; ++r)
            if (j->pss[r] == want) {
                sel = r;
                break;
            }
        if (sel < 0) {
            rc = -3;
            break;
        }
        for (int64_t e = 0; e < ne; ++e) counts_out[e] += j->out.counts[sel * ne + e];
        if (locate) {
            Rows* rs = &j->out.rows[sel];
            for (int64_t k = 0; k < rs->n; ++k)
                if (rows_push(&all, rs->rows[2 * k], rs->rows[2 * k + 1])) rc = -1;
            if (j->out.conv[sel] >= 0) {
                Rows* r0 = &j->out.rows[0];
                const int64_t border = j->lo + j->out.conv[sel] + 1;
                for (int64_t k = 0; k < r0->n; ++k)
                    if (r0->rows[2 * k] > border && rows_push(&all, r0->rows[2 * k], r0->rows[2 * k + 1])) rc = -1;
            }
        }
        want = j->out.last[sel];
        for (int64_t r = 1; r < j->nr; ++r) {
            ++spec;
            if (j->out.conv[r] >= 0) {
                ++conv;
                if (conv_hist && j->out.conv[r] <= window) conv_hist[j->out.conv[r]] += 1;
            }
        }
    }
    if (locate && rc == 0) {
        if (all.n > 1) qsort(all.rows, (size_t)all.n, 16, cmp_rows);
        *rows_out = all.rows;
        *n_rows = all.n;
    } else {
        free(all.rows);
    }
    if (n_spec) *n_spec = spec;
    if (n_conv) *n_conv = conv;
    for (int64_t i = 0; i < w; ++i) {
        free(jobs[i].out.counts);
        free(jobs[i].out.last);
        free(jobs[i].out.conv);
        if (jobs[i].out.rows) {
            for (int64_t r = 0; r < jobs[i].nr; ++r) free(jobs[i].out.rows[r].rows);
            free(jobs[i].out.rows);
        }
    }
    free(jobs);
    free(pss_all);
    free(seen);
    free(th);
    return rc;
}

/* scan_from with location rows (_kernels.py:18-40): rows [g_off + j + 1, e]. */
int64_t ref_scan_rows(const int32_t* trans, const int32_t* out_off, const int32_t* out_ids, const uint8_t* sym,
                      int64_t start, int64_t end, int64_t state, int64_t g_off, int64_t* counts, int64_t** rows_out,
                      int64_t* n_rows) {
    Rows r = {NULL, 0, 0};
    int64_t s = state;
    for (int64_t j = start; j < end; ++j) {
        s = trans[s * OTHER_SYMS + sym[j]];
        for (int32_t k = out_off[s]; k < out_off[s + 1]; ++k) {
            counts[out_ids[k]] += 1;
            if (rows_push(&r, g_off + j + 1, out_ids[k])) return -1;
        }
    }
    *rows_out = r.rows;
    *n_rows = r.n;
    return s;
}

int64_t ref_effective_workers(int64_t n, int64_t workers) {
    int64_t cap = n > 1 ? n : 1;
    return workers < cap ? workers : cap;
}

void ref_free(void* p) { free(p); }
