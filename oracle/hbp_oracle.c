/*
 * hbp_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker and the CPU
 * baseline arm).  Nothing in paper_2504_08860_b200/ links, loads or calls this
 * file; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may.
 *
 * A plain-C restatement of the reference's compiled CPU loops (numba
 * @njit kernels in /root/reference/pkg/src/hbp_spmv/_kernels.py) plus the
 * per-block Python loops that are too slow to run as Python at bench scale
 * (build_hbp, hbp.py:150-238; the fixed+ticket executor, engine.py:137-193;
 * combine, engine.py:196-201).  All arrays use the reference's DENSE layout
 * (rows x column-blocks slot arrays, bc-major block order).
 *
 * Floating point: compiled with -ffp-contract=off so `s += a*b` is a separate
 * multiply and add, like the numba kernels.
 *
 * Parity: pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py) -- see tests/test_oracle_golden.py.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORC_OK 0
#define ORC_E_PERM 1      /* "permutation of block (br, bc) is not a bijection" */
#define ORC_E_EMITTED 2   /* "emitted element count disagrees with matrix nnz" */
#define ORC_E_NOMEM 3
#define ORC_E_WORKERS 4

/* _kernels.py:13-19  csr_kernel: per row, left-to-right in storage order. */
void orc_csr_kernel(const int64_t *row_ptr, const int64_t *col_idx,
                    const double *values, const double *x, double *out,
                    int64_t rows) {
    for (int64_t i = 0; i < rows; ++i) {
        double s = 0.0;
        for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; ++j)
            s += values[j] * x[col_idx[j]];
        out[i] = s;
    }
}

/* The reference's y for selected rows without its dense layout: per row,
 * each column block's run is summed left to right from 0.0 exactly as
 * hbp_block_kernel (_kernels.py:22-47) chases the row's add_sign chain (a
 * row's elements in a block are its CSR run, step order), and the blocks'
 * partials are folded in ascending bc as combine (engine.py:196-201) does.
 * Empty blocks contribute the dense partial's +0.0, which never changes a
 * sum that started from 0.0 (partials are never -0.0), so they are skipped.
 * rows_sel[k] names the k-th row; out[k] gets its y.  Used for parity at
 * sizes where the dense rows x ncb arrays do not fit host memory. */
void orc_rows_blocked(const int64_t *row_ptr, const int64_t *col_idx,
                      const double *values, const double *x, int64_t C,
                      const int64_t *rows_sel, int64_t nsel, double *out) {
    for (int64_t k = 0; k < nsel; ++k) {
        const int64_t i = rows_sel[k];
        double y = 0.0;
        int first = 1;
        int64_t j = row_ptr[i];
        while (j < row_ptr[i + 1]) {
            const int64_t bc = col_idx[j] / C;
            double s = 0.0;
            for (; j < row_ptr[i + 1] && col_idx[j] / C == bc; ++j)
                s += values[j] * x[col_idx[j]];
            if (first) y = s, first = 0;
            else y += s;
        }
        out[k] = y;
    }
}

/* reorder.py:112-136 build_block_permutation: rows claim slots in ascending
 * local-row order; preliminary slot = hash_slot (reorder.py:106-109) mod n;
 * +1 linear probing with wraparound.  Returns the probe count (inspections of
 * an already-claimed slot).  `taken` is caller scratch of >= n bytes. */
static uint64_t probe_block(const int32_t *row_nnz, int64_t n, int64_t a,
                            int64_t b, int64_t c, int64_t d, int64_t bmax,
                            uint8_t *taken, uint32_t *out) {
    uint64_t probes = 0;
    memset(taken, 0, (size_t)n);
    for (int64_t r = 0; r < n; ++r) {
        int64_t g = ((int64_t)row_nnz[r]) >> a;
        if (g > bmax) g = bmax;
        int64_t pos = (g * b + (r * c) % d) % n;
        while (taken[pos]) {
            ++probes;
            if (++pos == n) pos = 0;
        }
        taken[pos] = 1;
        out[pos] = (uint32_t)r;
    }
    return probes;
}

uint64_t orc_hash_perm_block(const int32_t *row_nnz, int64_t n, int64_t a,
                             int64_t b, int64_t c, int64_t d, int64_t bmax,
                             uint32_t *out) {
    uint8_t *taken = (uint8_t *)malloc((size_t)(n > 0 ? n : 1));
    uint64_t p = probe_block(row_nnz, n, a, b, c, d, bmax, taken, out);
    free(taken);
    return p;
}

/* _kernels.py:62-92 hash_perm_kernel: every block (empty ones included),
 * bc-major; slot_nnz is row_counts flattened [bc][global row]. */
uint64_t orc_hash_perm(const int32_t *slot_nnz, int64_t rows, int64_t R,
                       int64_t nrb, int64_t ncb, int64_t a, int64_t b,
                       int64_t c, int64_t d, int64_t bmax, uint32_t *out) {
    uint8_t *taken = (uint8_t *)malloc((size_t)R);
    uint64_t probes = 0;
    for (int64_t bc = 0; bc < ncb; ++bc)
        for (int64_t br = 0; br < nrb; ++br) {
            int64_t base = bc * rows + br * R;
            int64_t n = rows - br * R;
            if (n > R) n = R;
            probes += probe_block(slot_nnz + base, n, a, b, c, d, bmax, taken,
                                  out + base);
        }
    free(taken);
    return probes;
}

/* hbp.py:138-147 _zero_row_for: -1 for an empty slot, else the number of
 * empty slots at lower lanes of the same W-lane group. */
static void zero_row_for(const int64_t *slot_nnz, int64_t n, int64_t W,
                         int32_t *out) {
    for (int64_t g0 = 0; g0 < n; g0 += W) {
        int32_t empties = 0;
        for (int64_t s = g0; s < g0 + W && s < n; ++s) {
            if (slot_nnz[s] == 0) {
                out[s] = -1;
                ++empties;
            } else {
                out[s] = empties;
            }
        }
    }
}

/* hbp.py:150-238 build_hbp, one block at a time in bc-major order.  Within a
 * W-lane group, elements are emitted column-major: step t emits the (t+1)-th
 * element of every lane still holding one, lanes ascending (hbp.py:194-206).
 * add_sign links consecutive elements of one slot (hbp.py:208-213).
 * group_start = block element base + exclusive prefix of group counts
 * (hbp.py:215-216); an empty block repeats its base (hbp.py:190-192). */
int orc_build_hbp(const int64_t *col_idx, const double *values,
                  const int32_t *row_counts, const int64_t *row_starts,
                  const int64_t *block_elem_start, const uint32_t *perms,
                  int64_t rows, int64_t nnz, int64_t R, int64_t W, int64_t nrb,
                  int64_t ncb, uint32_t *col_out, double *data_out,
                  int32_t *add_out, int32_t *zero_row_out, int64_t *gs_out,
                  int64_t *bad_block /* [2]: br, bc on ORC_E_PERM */) {
    int64_t *slot_nnz = (int64_t *)malloc(sizeof(int64_t) * (size_t)R);
    int64_t *last = (int64_t *)malloc(sizeof(int64_t) * (size_t)R);
    int64_t *src = (int64_t *)malloc(sizeof(int64_t) * (size_t)R);
    uint8_t *seen = (uint8_t *)malloc((size_t)R);
    if (!slot_nnz || !last || !src || !seen) return ORC_E_NOMEM;
    int64_t gpc = (nrb - 1) * (R / W) + ((rows - (nrb - 1) * R) + W - 1) / W;
    int64_t emitted = 0;
    int rc = ORC_OK;
    for (int64_t bc = 0; bc < ncb && rc == ORC_OK; ++bc) {
        for (int64_t br = 0; br < nrb; ++br) {
            int64_t n = rows - br * R;
            if (n > R) n = R;
            int64_t base = bc * rows + br * R;
            int64_t r0 = br * R;
            memset(seen, 0, (size_t)n);
            for (int64_t s = 0; s < n; ++s) {
                uint32_t p = perms[base + s];
                if (p >= (uint32_t)n || seen[p]) {
                    bad_block[0] = br;
                    bad_block[1] = bc;
                    rc = ORC_E_PERM;
                    break;
                }
                seen[p] = 1;
                slot_nnz[s] = row_counts[bc * rows + r0 + p];
                src[s] = row_starts[bc * rows + r0 + p];
            }
            if (rc != ORC_OK) break;
            zero_row_for(slot_nnz, n, W, zero_row_out + base);
            int64_t ng = (n + W - 1) / W;
            int64_t gb = bc * gpc + br * (R / W);
            int64_t pos = block_elem_start[br * ncb + bc];
            for (int64_t g = 0; g < ng; ++g) {
                gs_out[gb + g] = pos;
                int64_t q0 = g * W, q1 = q0 + W < n ? q0 + W : n;
                int64_t maxlen = 0;
                for (int64_t q = q0; q < q1; ++q)
                    if (slot_nnz[q] > maxlen) maxlen = slot_nnz[q];
                for (int64_t t = 0; t < maxlen; ++t)
                    for (int64_t q = q0; q < q1; ++q) {
                        if (slot_nnz[q] <= t) continue;
                        int64_t j = src[q] + t;
                        col_out[pos] = (uint32_t)col_idx[j];
                        data_out[pos] = values[j];
                        add_out[pos] = -1;
                        if (t > 0) add_out[last[q]] = (int32_t)(pos - last[q]);
                        last[q] = pos;
                        ++pos;
                        ++emitted;
                    }
            }
        }
    }
    if (rc == ORC_OK) {
        gs_out[ncb * gpc] = nnz;
        if (emitted != nnz) rc = ORC_E_EMITTED;
    }
    free(slot_nnz);
    free(last);
    free(src);
    free(seen);
    return rc;
}

/* _kernels.py:22-47 hbp_block_kernel: chase add_sign chains lane by lane;
 * accumulate-then-test. */
void orc_block_kernel(const uint32_t *col, const double *data,
                      const int32_t *add_sign, const int32_t *zero_row,
                      const uint32_t *output_hash, const int64_t *group_start,
                      int64_t group_base, int64_t n_groups, int64_t slot_base,
                      int64_t rows_in_block, int64_t warp, const double *x,
                      int64_t col_offset, double *partial,
                      int64_t partial_base) {
    for (int64_t gl = 0; gl < n_groups; ++gl) {
        int64_t start = group_start[group_base + gl];
        int64_t lanes = rows_in_block - gl * warp;
        if (lanes > warp) lanes = warp;
        for (int64_t q = 0; q < lanes; ++q) {
            int64_t slot = slot_base + gl * warp + q;
            int64_t zr = zero_row[slot];
            if (zr < 0) continue;
            int64_t j = start + q - zr;
            double s = 0.0;
            for (;;) {
                s += data[j] * x[(int64_t)col[j] - col_offset];
                int32_t step = add_sign[j];
                if (step < 0) break;
                j += step;
            }
            partial[partial_base + output_hash[slot]] = s;
        }
    }
}

/* engine.py:137-193 _run_plan / run_spmv: fixed contiguous chunks per worker,
 * then a shared ticket (the reference uses a threading.Lock; an atomic
 * fetch-add is the same claim order semantics).  The partial is zero-filled
 * inside the call like np.zeros at engine.py:185-186. */
typedef struct {
    const uint32_t *col;
    const double *data;
    const int32_t *add_sign;
    const int32_t *zero_row;
    const uint32_t *output_hash;
    const int64_t *group_start;
    const int32_t *block_order; /* [nblocks][2] = (br, bc) */
    const int64_t *ranges;      /* [workers][2] */
    int64_t nblocks, rows, cols, C, R, W, gpc;
    const double *x;
    double *partial;
    int64_t ticket;
    int32_t *log_worker;
    int8_t *log_kind;
    int64_t *log_start, *log_end;
} plan_ctx;

typedef struct {
    plan_ctx *ctx;
    int64_t wid;
} worker_arg;

static int64_t now_ns(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec;
}

static void run_block(plan_ctx *c, int64_t idx, int64_t wid, int8_t kind) {
    int64_t br = c->block_order[2 * idx], bc = c->block_order[2 * idx + 1];
    int64_t n = c->rows - br * c->R;
    if (n > c->R) n = c->R;
    int64_t ng = (n + c->W - 1) / c->W;
    int64_t t0 = c->log_start ? now_ns() : 0;
    orc_block_kernel(c->col, c->data, c->add_sign, c->zero_row, c->output_hash,
                     c->group_start, bc * c->gpc + br * (c->R / c->W), ng,
                     bc * c->rows + br * c->R, n, c->W, c->x, 0, c->partial,
                     bc * c->rows + br * c->R);
    if (c->log_start) {
        c->log_start[idx] = t0;
        c->log_end[idx] = now_ns();
        c->log_worker[idx] = (int32_t)wid;
        c->log_kind[idx] = kind;
    }
}

static void *worker_main(void *p) {
    worker_arg *wa = (worker_arg *)p;
    plan_ctx *c = wa->ctx;
    int64_t lo = c->ranges[2 * wa->wid], hi = c->ranges[2 * wa->wid + 1];
    for (int64_t i = lo; i < hi; ++i) run_block(c, i, wa->wid, 0);
    for (;;) {
        int64_t i = __atomic_fetch_add(&c->ticket, 1, __ATOMIC_SEQ_CST);
        if (i >= c->nblocks) break;
        run_block(c, i, wa->wid, 1);
    }
    return NULL;
}

int orc_run_spmv(const uint32_t *col, const double *data,
                 const int32_t *add_sign, const int32_t *zero_row,
                 const uint32_t *output_hash, const int64_t *group_start,
                 int64_t rows, int64_t cols, int64_t C, int64_t R, int64_t W,
                 int64_t nrb, int64_t ncb, const int32_t *block_order,
                 int64_t nblocks, int64_t fixed_count, const int64_t *ranges,
                 int64_t workers, const double *x, double *partial,
                 int32_t *log_worker, int8_t *log_kind, int64_t *log_start,
                 int64_t *log_end) {
    if (workers < 1) return ORC_E_WORKERS;
    plan_ctx c;
    c.col = col;
    c.data = data;
    c.add_sign = add_sign;
    c.zero_row = zero_row;
    c.output_hash = output_hash;
    c.group_start = group_start;
    c.block_order = block_order;
    c.ranges = ranges;
    c.nblocks = nblocks;
    c.rows = rows;
    c.cols = cols;
    c.C = C;
    c.R = R;
    c.W = W;
    c.gpc = (nrb - 1) * (R / W) + ((rows - (nrb - 1) * R) + W - 1) / W;
    c.x = x;
    c.partial = partial;
    c.ticket = fixed_count;
    c.log_worker = log_worker;
    c.log_kind = log_kind;
    c.log_start = log_start;
    c.log_end = log_end;
    memset(partial, 0, sizeof(double) * (size_t)(ncb * rows));
    if (workers == 1) {
        worker_arg wa = {&c, 0};
        worker_main(&wa);
        return ORC_OK;
    }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)workers);
    worker_arg *wa = (worker_arg *)malloc(sizeof(worker_arg) * (size_t)workers);
    for (int64_t w = 0; w < workers; ++w) {
        wa[w].ctx = &c;
        wa[w].wid = w;
        pthread_create(&th[w], NULL, worker_main, &wa[w]);
    }
    for (int64_t w = 0; w < workers; ++w) pthread_join(th[w], NULL);
    free(th);
    free(wa);
    return ORC_OK;
}

/* engine.py:196-201 combine: out = segment(0); out += segment(bc), bc
 * ascending. */
void orc_combine(const double *partial, int64_t rows, int64_t ncb,
                 double *out) {
    memcpy(out, partial, sizeof(double) * (size_t)rows);
    for (int64_t bc = 1; bc < ncb; ++bc) {
        const double *seg = partial + bc * rows;
        for (int64_t i = 0; i < rows; ++i) out[i] += seg[i];
    }
}

/* _kernels.py:50-59 block2d_kernel (engine.py:204-225): per block row, its
 * run in CSR order, into partial[bc*rows + row]; blocks in bc-major order. */
void orc_block2d(const int64_t *col_idx, const double *values, const int32_t *row_counts,
                 const int64_t *row_starts, const int64_t *block_nnz, int64_t rows,
                 int64_t R, int64_t nrb, int64_t ncb, const double *x, double *partial) {
    memset(partial, 0, sizeof(double) * (size_t)(ncb * rows));
    for (int64_t bc = 0; bc < ncb; ++bc)
        for (int64_t br = 0; br < nrb; ++br) {
            if (block_nnz[br * ncb + bc] == 0) continue;
            int64_t r0 = br * R, n = rows - r0 < R ? rows - r0 : R;
            for (int64_t r = 0; r < n; ++r) {
                int64_t gr = r0 + r, j = row_starts[bc * rows + gr];
                double s = 0.0;
                for (int64_t k = 0; k < row_counts[bc * rows + gr]; ++k)
                    s += values[j + k] * x[col_idx[j + k]];
                partial[bc * rows + gr] = s;
            }
        }
}
