/*
 * hbp.h -- C ABI of libhbp.so, the sm_100a (B200) implementation of the
 * Hash-based Partition (HBP) SpMV hot path (arXiv 2504.08860).
 *
 * The reference package (`hbp_spmv`, /root/reference/pkg/src/hbp_spmv) binds
 * its native code through numba-compiled kernels called from Python with
 * caller-allocated, C-contiguous buffers and no error path inside kernels
 * (SURVEY.md §8b).  This ABI keeps those conventions on the GPU:
 *
 *   - every entry point takes raw DEVICE pointers, 64-bit sizes and a
 *     cudaStream_t (passed as `hbp_stream_t`, NULL = legacy default stream);
 *   - nothing allocates: outputs and scratch are caller-provided; functions
 *     that need CUB scratch take (temp, temp_bytes) and report the size when
 *     called with temp == NULL (CUB convention);
 *   - no mutable state on the data path: the work ticket, partials and
 *     per-SpMV scratch live in caller memory, so calls are re-entrant per
 *     stream and per device.  Process-wide state is limited to (a) a
 *     per-device cache of kernel launch attributes (idempotent) and (b) the
 *     A/B tuning selectors hbp_stream_set_variant / HBP_STREAM_VARIANT /
 *     HBP_ROWBLOCK_VARIANT, read once; every variant computes the same y;
 *   - return value: HBP_OK, an HBP_E_* code, or a cudaError_t (< 1000).
 *     hbp_status_string() maps it to the reference's error vocabulary.
 *
 * Each function cites the reference interface it replaces (file:line under
 * /root/reference/pkg/src/hbp_spmv/).  Layout vocabulary:
 *   - "block"   = one (br, bc) tile of row_height x col_width;
 *   - "nzb"     = number of NONZERO blocks, listed bc-major (engine.py:86-93);
 *   - "slot"    = one (block, local row) entry; compact slot arrays hold
 *                 row_height entries per nonzero block (short last row block
 *                 padded with zeros);
 *   - "group"   = warp_size consecutive slots (hbp.py:17-19); compact group
 *                 arrays hold gpb = row_height / warp_size groups per nonzero
 *                 block (missing groups of a short block have size 0).
 */
#ifndef HBP_H
#define HBP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *hbp_stream_t; /* cudaStream_t */

enum {
    HBP_OK = 0,
    HBP_E_ARG = 1001,         /* invalid argument ("config", "length", ...) */
    HBP_E_PERM = 1002,        /* "permutation of block (br, bc) is not a bijection" */
    HBP_E_DUP = 1003,         /* "duplicate (row, col) entries; canonicalize first" */
    HBP_E_UNSUPPORTED = 1004, /* geometry outside what the kernels support */
    HBP_E_FORMAT = 1005       /* structurally invalid HBP arrays */
};

enum { HBP_F32 = 0, HBP_F64 = 1 };

const char *hbp_status_string(int status);
/* The CUDA runtime's pending (non-sticky) error of this library, cleared on
 * read (cudaGetLastError) -- for tests that check no call left one behind. */
int hbp_last_error(void);
int hbp_abi_version(void);
/* sizeof hbp_format_t, hbp_schedule_t, hbp_balanced_t, hbp_seg_t (bindings
 * check their struct mirrors against it); no device needed. */
int hbp_struct_sizes(int64_t *sizes);

/* Device facts for sizing persistent grids (replaces the worker-count
 * argument of engine.py:96 / cli.py:59-60 with a device-derived default). */
int hbp_device_sm_count(int *sms);
int hbp_spmv_default_workers(int dtype, int64_t warp_size, int64_t *workers);

/* ---------------------------------------------------------------- utils */
/* CUB device-wide primitives used by the host pipeline (temp == NULL -> size). */
int hbp_exclusive_sum_i64(const int64_t *in, int64_t *out, int64_t n, void *temp,
                          size_t *temp_bytes, hbp_stream_t stream);
int hbp_inclusive_sum_i64(const int64_t *in, int64_t *out, int64_t n, void *temp,
                          size_t *temp_bytes, hbp_stream_t stream);
/* Stable LSD radix sort of (u32 key, u32 value) pairs on bits [0, end_bit). */
int hbp_sort_pairs_u32(const uint32_t *keys_in, uint32_t *keys_out, const uint32_t *vals_in,
                       uint32_t *vals_out, int64_t n, int end_bit, void *temp,
                       size_t *temp_bytes, hbp_stream_t stream);
/* Stable LSD radix sort of (u64 key, u64 value) pairs on bits [0, end_bit). */
int hbp_sort_pairs_u64(const uint64_t *keys_in, uint64_t *keys_out, const uint64_t *vals_in,
                       uint64_t *vals_out, int64_t n, int end_bit, void *temp,
                       size_t *temp_bytes, hbp_stream_t stream);

/* L2 residency of the gathered x vector (B200: 126 MB L2): persisting
 * set-aside plus an access-policy window on `stream`. */
int hbp_l2_persist(const void *base, size_t bytes, float hit_ratio, hbp_stream_t stream);
int hbp_l2_persist_reset(hbp_stream_t stream);
int hbp_l2_info(int *l2_bytes, int *max_persist, int *max_window);

/* ------------------------------------------------------- formats (COO/CSR) */
/* formats.py:243-258 coo_to_csr, after the caller sorted keys = row*cols+col
 * (stable, values carried by the original index `order`):
 * gathers col/val, rejects duplicates (HBP_E_DUP) and builds row_ptr. */
int hbp_coo_finish_csr(const uint64_t *sorted_keys, const uint64_t *order, const void *val_in,
                       int64_t nnz, int64_t rows, int64_t cols, int dtype, int64_t *row_ptr,
                       int32_t *col_idx, void *val_out, int32_t *dup_flag,
                       hbp_stream_t stream);
/* formats.py:87-97 TripletMatrix.canonicalized: given keys sorted stably,
 * marks run heads (head[i] = 1 if key[i] != key[i-1]) ... */
int hbp_coo_run_heads(const uint64_t *sorted_keys, int64_t n, int64_t *head,
                      hbp_stream_t stream);
/* ... and sums each duplicate run left to right in sorted order (np.add.reduceat). */
int hbp_coo_reduce_runs(const uint64_t *sorted_keys, const uint64_t *order, const double *val_in,
                        const int64_t *head_incl, int64_t n, int64_t cols, int64_t *row_out,
                        int64_t *col_out, double *val_out, hbp_stream_t stream);

/* ----------------------------------------------------- make_grid (compact) */
/* partition.py:100-127 make_grid, without its dense rows x ncb arrays.
 * A "run" is the maximal piece of one CSR row inside one column block. */
int hbp_grid_count_runs(const int64_t *row_ptr, const int32_t *col_idx, int64_t rows,
                        int64_t cols, int64_t col_width, int64_t *runs_per_row,
                        hbp_stream_t stream);
/* Writes every run (bc, row, csr start, count), row-major order, at
 * run_offset[row] (exclusive prefix of runs_per_row). */
int hbp_grid_emit_runs(const int64_t *row_ptr, const int32_t *col_idx, int64_t rows,
                       int64_t cols, int64_t col_width, const int64_t *run_offset,
                       int64_t nruns, uint32_t *run_bc, uint32_t *run_row, int64_t *run_start,
                       int32_t *run_count, hbp_stream_t stream);
/* After the runs are ordered bc-major (order = stable sort by bc, NULL when
 * ncb == 1), flags the first run of every nonzero block. */
int hbp_grid_block_heads(const uint32_t *sorted_bc, const uint32_t *order,
                         const uint32_t *run_row, int64_t nruns, int64_t row_height,
                         int64_t *head, hbp_stream_t stream);
/* Scatters runs into the compact per-block slot arrays: blk_br/blk_bc
 * (nonzero block directory, bc-major), len_local[blk*R + local_row] (the
 * reference's BlockGrid.row_counts restricted to nonzero blocks) and
 * start_local (BlockGrid.row_starts).  len_local must be zero-filled. */
int hbp_grid_fill_slots(const uint32_t *sorted_bc, const uint32_t *order,
                        const uint32_t *run_row, const int64_t *run_start,
                        const int32_t *run_count, const int64_t *block_incl, int64_t nruns,
                        int64_t row_height, int32_t *blk_br, int32_t *blk_bc,
                        uint32_t *len_local, int64_t *start_local, hbp_stream_t stream);
/* partition.py:118-124 block_nnz over nonzero blocks. */
int hbp_block_nnz(const uint32_t *len_local, int64_t nzb, int64_t row_height, int64_t *block_nnz,
                  hbp_stream_t stream);

/* ------------------------------------------------------- hash reordering */
/* reorder.py:80-85: row_counts[bc, row] at sampled flat indices
 * (flat = bc*rows + row), by binary search in the CSR row. */
int hbp_sample_counts(const int64_t *row_ptr, const int32_t *col_idx, int64_t rows,
                      int64_t col_width, const int64_t *flat_idx, int64_t k, int32_t *counts,
                      hbp_stream_t stream);
/* reorder.py:174-184 hash_permutations -> _kernels.py:62-92
 * hash_perm_kernel, for nonzero blocks: FCFS linear probing with an
 * occupancy bitmap (first free slot at or after the preliminary slot,
 * cyclic), bit-exact with the reference's literal probe loop.
 * perm[blk*R + slot] = local row; *probes += reference OpCounter.probes. */
int hbp_hash_perm(const uint32_t *len_local, const int32_t *blk_br, int64_t nzb, int64_t rows,
                  int64_t row_height, int64_t a, int64_t b, int64_t c, int64_t d,
                  int64_t bucket_max, uint32_t *perm, unsigned long long *probes,
                  hbp_stream_t stream);
/* The permutation every EMPTY block of height n gets (all counts zero):
 * needed only to expand to the reference's dense output_hash. */
int hbp_hash_perm_empty(int64_t n, int64_t a, int64_t b, int64_t c, int64_t d,
                        int64_t bucket_max, uint32_t *perm, hbp_stream_t stream);
/* reorder.py:187-219 sort_permutations (stable ascending nnz) for nonzero
 * blocks, and reorder.py:222-225 identity_permutations. */
int hbp_sort_perm(const uint32_t *len_local, const int32_t *blk_br, int64_t nzb, int64_t rows,
                  int64_t row_height, uint32_t *perm, hbp_stream_t stream);
/* reorder.py:139-157 _counting_merge_sort: the number of key comparisons the
 * reference's instrumented top-down merge sort makes on keys[0..n) (split at
 * len//2, merge with `<=`); *out += that count (sort_permutation(counter=)). */
int hbp_merge_comparisons(const int64_t *keys, int64_t n, unsigned long long *out,
                          hbp_stream_t stream);
/* Gathers nonzero blocks' slices of a dense [ncb*rows] permutation table and
 * checks every block (empty ones too) is a bijection (hbp.py:179-181):
 * *bad = smallest bc-major block index that is not, or -1. */
int hbp_gather_dense_perm(const uint32_t *dense, int64_t rows, int64_t ncb, int64_t row_height,
                          const int32_t *blk_br, const int32_t *blk_bc, int64_t nzb,
                          uint32_t *perm, long long *bad, hbp_stream_t stream);
/* (`bad` must hold LLONG_MAX on entry; it is atomically lowered.) */

/* ------------------------------------------------------------- build_hbp */
/* hbp.py:183-185,215: permuted slot lengths, zero_row (nullable) and per
 * group nnz (group_nnz has nzb*gpb + 1 entries; the last is set to 0 so an
 * exclusive sum yields group_start with the nnz sentinel).  Checks the
 * compact permutation is a bijection: *bad = first bad nonzero block or -1. */
int hbp_slot_lengths(const uint32_t *len_local, const uint32_t *perm, const int32_t *blk_br,
                     int64_t nzb, int64_t rows, int64_t row_height, int64_t warp_size,
                     uint32_t *slot_len, int32_t *zero_row, int64_t *group_nnz,
                     long long *bad, hbp_stream_t stream);
/* hbp.py:194-213: column-major-within-group emission of col/data and the
 * add_sign stride chain (nullable), computed from slot lengths. */
int hbp_emit(const uint32_t *slot_len, const uint32_t *perm, const int64_t *start_local,
             const int64_t *group_start, const int32_t *blk_br, int64_t nzb, int64_t rows,
             int64_t row_height, int64_t warp_size, const int32_t *col_idx, const void *values,
             int dtype, uint32_t *col, void *data, int32_t *add_sign, hbp_stream_t stream);
/* Per row block, the number of its nonzero blocks (rb_count zero-filled by
 * the caller; its exclusive sum is rb_ptr, and a stable sort of the block
 * indices by br lists each row block's blocks in ascending bc). */
int hbp_row_block_counts(const int32_t *blk_br, int64_t nzb, int64_t *rb_count,
                         hbp_stream_t stream);

/* Dense (reference-layout) view of the slot and group arrays:
 * zero_row[ncb*rows], output_hash[ncb*rows], group_start[ncb*gpc+1]
 * (hbp.py:51-62 HbpMatrix fields).  empty_perm_full / empty_perm_last are
 * hbp_hash_perm_empty() for heights R and the last block's height. */
int hbp_expand_reference(const int32_t *blk_br, const int32_t *blk_bc, int64_t nzb, int64_t rows,
                         int64_t cols, int64_t nnz, int64_t col_width, int64_t row_height,
                         int64_t warp_size,
                         const uint32_t *perm, const int32_t *zero_row_c,
                         const int64_t *group_start_c, const uint32_t *empty_perm_full,
                         const uint32_t *empty_perm_last, int32_t *zero_row, uint32_t *output_hash,
                         int64_t *group_start, hbp_stream_t stream);

/* ----------------------------------------------- the paper's baselines */
/* formats.py:266-273 csr_spmv -> _kernels.py:13-19 csr_kernel (PAPER Alg. 1):
 * one thread per row, left to right, unfused (f64 bitwise with the
 * reference; f32 values accumulate in f64). */
int hbp_csr_spmv(const int64_t *row_ptr, const int32_t *col_idx, const void *values, int dtype,
                 int64_t rows, const void *x, void *y, hbp_stream_t stream);
/* engine.py:204-225 block2d_spmv_baseline -> _kernels.py:50-59
 * block2d_kernel: each nonzero block's row runs in CSR order into the
 * compact partial [nzb*R] (combine with hbp_combine). */
int hbp_block2d_spmv(const uint32_t *len_local, const int64_t *start_local, const int32_t *blk_br,
                     int64_t nzb, int64_t rows, int64_t row_height, const int32_t *col_idx,
                     const void *values, int dtype, const void *x, double *partial,
                     hbp_stream_t stream);

/* metrics.py:26-79 group_stats (GroupStats.from_lanes) over the nonzero
 * blocks: per lane group g = bc*groups_per_col + br*(R/W) + gi, the lane
 * counts in slot order (perm: compact slot -> local row tables [nzb*R], or
 * NULL for the unordered grid) into lanes[g*W + q], and mean / population
 * std_dev (numpy pairwise float64, bitwise) / max / utilization.  Groups of
 * empty blocks are not written (caller initialises 0, 0, 0, 1.0). */
int hbp_group_stats(const int32_t *blk_br, const int32_t *blk_bc, int64_t nzb,
                    const int32_t *len_local, const uint32_t *perm, int64_t rows,
                    int64_t row_height, int64_t warp_size, int64_t groups_per_col,
                    int32_t *lanes, double *mean, double *std_dev, int32_t *max_nnz,
                    double *utilization, hbp_stream_t stream);

/* hbp.py:241-315 hbp_to_triplets: follows every slot's add_sign chain over
 * the reference-layout arrays; row_out[j] = row of element j, seen[j] =
 * visit count (zero-filled by the caller), *err |= 1 (lane start outside its
 * group), 2 (column outside its block), 4 (invalid stride), 8 (chain escapes
 * its group). */
int hbp_walk_chains(int64_t rows, int64_t cols, int64_t col_width, int64_t row_height,
                    int64_t warp_size, const int32_t *zero_row, const uint32_t *output_hash,
                    const int64_t *group_start, const uint32_t *col, const int32_t *add_sign,
                    int64_t nnz, int64_t *row_out, int32_t *seen, int32_t *err,
                    hbp_stream_t stream);

/* deserialize_hbp (hbp.py:349-381) support: per dense slot [ncb*rows] the
 * length of its add_sign chain (0 for empty slots, zero_row < 0), walked as
 * hbp_block_kernel walks it (_kernels.py:35-46) but bounded to the slot's
 * group range.  Validation is the caller's (hbp.py:102-135 first). */
int hbp_chain_lengths(int64_t rows, int64_t cols, int64_t col_width, int64_t row_height,
                      int64_t warp_size, const int32_t *zero_row, const int64_t *group_start,
                      const int32_t *add_sign, int64_t nnz, int32_t *len_out,
                      hbp_stream_t stream);

/* ------------------------------------------------------------------ SpMV */
typedef struct {
    int64_t rows, cols, col_width, row_height, warp_size;
    int64_t nrb, ncb, nzb, nnz;
    int32_t dtype; /* HBP_F32 or HBP_F64 (element values, x and y) */
    int32_t exact; /* 1: reference summation order, bitwise for f64 */
    const int32_t *blk_br;       /* [nzb] */
    const int32_t *blk_bc;       /* [nzb] */
    const uint32_t *slot_len;    /* [nzb*R] permuted in-block row lengths */
    const uint32_t *perm;        /* [nzb*R] output_hash (slot -> local row) */
    const int64_t *group_start;  /* [nzb*gpb + 1] */
    const uint32_t *col;         /* [nnz] global column */
    const void *data;            /* [nnz] */
    const int64_t *rb_ptr;       /* [nrb+1] combine lists, ascending bc */
    const int32_t *rb_blk;       /* [nzb] */
    const int64_t *phase_ptr;    /* [nzb*gpb + 1] phase stream index (W = 32), nullable */
    const void *phases;          /* uint2 (live mask, group offset) per phase (+32 pad), nullable */
    /* Hot-column staging (hbp_spmv_stream only; all nullable / 0 = off):
     * scol[e] = HBP_HOT_FLAG | s when col[e] == hot_cols[s], else col[e]. */
    const uint32_t *scol;        /* [nnz] (+16 pad) staged column stream */
    const uint32_t *hot_cols;    /* [n_hot + n_warm] column of hot slot s, then of warm slot w */
    int64_t n_hot;               /* multiple of 4, see hbp_hot_capacity */
    int64_t n_warm;              /* warm tier: scol = HBP_WARM_FLAG | w (cols < 2^30) */
    int32_t cold_last;           /* 1: cold columns gathered L2 evict-last too (x fits L2) */
    int32_t reserved;            /* flags: HBP_FLAG_DIRECT_SINGLE */
    /* nullable: the staged slots in ascending column order (refresh_cols[i] =
     * hot_cols[refresh_slots[i]]) -- hbp_spmv_stream then refreshes x_hot by
     * reading x in column order and scattering into the slots, instead of
     * gathering it in slot (degree) order */
    const uint32_t *refresh_cols;
    const uint32_t *refresh_slots;
} hbp_format_t;
/* hbp_spmv_stream with a partial AND y: rows of row blocks that have exactly
 * one nonzero block are written to y directly (there is nothing to combine;
 * bitwise the same), and hbp_combine skips those row blocks. */
#define HBP_FLAG_DIRECT_SINGLE 4
/* Packed x (hbp_spmv_stream with hot staging): every column the matrix uses
 * is in hot_cols (heaviest first); scol holds HBP_HOT_FLAG | s for the n_hot
 * staged ones and the PLAIN index w < n_warm of the packed copy
 * x_hot[n_hot + w] for the rest, which the kernel gathers instead of x
 * (degree-ordered: the heavy columns share L2 lines).  n_warm is then the
 * packed count and no warm tier is used. */
#define HBP_FLAG_PACKED_X 8
#define HBP_HOT_FLAG 0x80000000u
#define HBP_WARM_FLAG 0x40000000u
/* peer copies of y a stream launch can write (hbp_balanced_t.y_peer): 8 GPUs */
#define HBP_MAX_PEERS 7

/* Phase stream (runtime index used by hbp_spmv_stream, W = 32): a group's
 * phases are its maximal step ranges with a fixed live-lane set; phase j is
 * (live mask, element offset within the group).  nph[ngroups] is set to 0
 * so an exclusive sum of nph gives phase_ptr. */
int hbp_phase_counts(const uint32_t *slot_len, int64_t ngroups, int64_t *nph,
                     hbp_stream_t stream);
int hbp_phase_emit(const uint32_t *slot_len, int64_t ngroups, const int64_t *phase_ptr,
                   void *phases, hbp_stream_t stream);

typedef struct {
    int64_t workers;     /* persistent warps (paper: one warp per worker) */
    int64_t fixed_count; /* engine.py:107 int(f * nzb + 0.5) */
    uint32_t *ticket;    /* device scratch, 1 word; reset by the call */
    int32_t *log_worker; /* nullable ExecutionLog (engine.py:71-83) */
    int8_t *log_kind;
    int64_t *log_start_ns;
    int64_t *log_end_ns;
} hbp_schedule_t;

/* engine.py:179-193 run_spmv -> _run_plan (engine.py:137-176) ->
 * block_spmv (engine.py:123-134) -> _kernels.py:22-47 hbp_block_kernel.
 * Fixed contiguous chunks per worker, then an atomic ticket.  Writes either
 * the compact partial [nzb*R] (per block, indexed by ORIGINAL local row),
 * or -- when y_direct != NULL and ncb == 1 -- y directly. */
int hbp_spmv_blocks(const hbp_format_t *f, const hbp_schedule_t *sched, const void *x,
                    double *partial, void *y_direct, hbp_stream_t stream);
/* Element-balanced SpMV (B200 schedule for warp_size == 32): the element
 * array is cut into `workers` equal ranges, one per persistent warp.  Exact
 * mode (f64 or fmt->exact) rounds cuts to group boundaries -- every row is
 * summed in reference order by one lane; otherwise cuts fall on step
 * boundaries and split groups are combined by the last-arriving warp from
 * per-warp partials (deterministic, f64 accumulation).  Scratch (fast mode):
 * part_head/part_tail f64[workers*32], cut_end i64[workers], counters
 * u32[nzb*gpb] zero-filled once (the kernel leaves them zeroed). */
typedef struct {
    int64_t workers;
    double *part_head;
    double *part_tail;
    int64_t *cut_end;
    uint32_t *counters;
    void *x_hot; /* [n_hot + n_warm] scratch: x at hot_cols (hot, then warm tier) */
    int64_t *slice_lo; /* nullable [workers + 1]: stream slice bounds (hbp_stream_slices) */
    int64_t *slice_g;  /* nullable [workers]: first group of each stream slice */
    uint32_t *rb_done; /* nullable [nrb], zero-filled once: fused combine (stream
                          kernel with partial AND y; the kernel leaves it zeroed) */
    const double *y_sumsq; /* nullable: rows written straight to y are multiplied by
                              1 / sqrt(*y_sumsq) (iterated SpMV: y = A (x / ||x||)) */
    int64_t hub_min;       /* exact mode only; 0 = off.  Groups longer than hub_min
                              elements (hub rows) are cut across warps and summed as
                              in fast mode (deterministic, not the reference's order:
                              within ~1e-14 relative for f64); every other row stays
                              bitwise the reference.  Needs the fast-mode scratch. */
    /* Stream kernel, competitive pieces (engine.py:137-176 applied to element
     * slices): with pieces > workers, the first fixed_elems elements are cut
     * into `workers` equal pieces (warp w starts on piece w, its fixed chunk)
     * and the rest into pieces - workers equal pieces that warps claim with
     * an atomic ticket (ticket: u32[2], zero-filled once; the kernel leaves
     * it zeroed).  slice_lo/slice_g and part_head/part_tail are then sized
     * by pieces.  0 (or == workers): one static slice per warp. */
    int64_t pieces;
    int64_t fixed_elems;
    uint32_t *ticket;
    int64_t *warp_ns; /* nullable [2*workers]: %globaltimer at each warp's start
                         and end (load-balance diagnostics) */
    /* nullable [ngroups + 1]: exclusive prefix of per-group costs
     * (hbp_group_costs); hbp_stream_slices then cuts equal COST instead of
     * equal elements (a group's fixed cost sits at its start). */
    const int64_t *cost_prefix;
    /* 0: CTA c runs slices c*warps_per_cta .. (contiguous ranges per SM);
     * 1: slice w runs on CTA w % ctas (each SM gets slices from all over the
     * element array).  Results do not depend on it. */
    int64_t warp_map;
    /* Tail pieces (with pieces > workers): instead of a ticket, pieces
     * workers..pieces-1 run as a second launch of the static kernel (one warp
     * per piece) that depends programmatically on the first: its CTAs take
     * SMs as the first launch's CTAs finish, so the imbalance of the static
     * slices is filled in by the hardware's CTA scheduler.  With a cost
     * prefix, fixed_elems is then a cost (the first fixed_elems cost units
     * form the `workers` static pieces).  piece_base: first piece of this
     * launch (set by the library for the second launch; 0 for callers). */
    int64_t tail;
    int64_t piece_base;
    /* Peer copies of y (SURVEY §8(e) fused variant: the iterated SpMV's
     * all-gather folded into its stores).  Every value the stream kernel
     * writes to y[r] (one column block, no partial) is also written to
     * y_peer[p][r] for p < n_peers: device pointers, normally other GPUs'
     * next-x buffers mapped with hbp_ipc_open, stored over NVLink as the
     * rows finish; each warp ends with a system-scope fence.  0: off. */
    int64_t n_peers;
    void *y_peer[HBP_MAX_PEERS];
} hbp_balanced_t;

int hbp_balanced_workers(const hbp_format_t *f, int64_t *workers);
/* Same slices and combine rule, but each warp streams its slice's col/data
 * through shared memory with cp.async.bulk (TMA bulk copies, two chunks in
 * flight), gathers x for a whole chunk at once and sums rows from shared
 * memory via the group's phase table (hbp_spmv_stream.cu).  Slices are cut
 * at arbitrary element offsets in fast mode (no cut_end needed).  col and
 * data must be readable 16 bytes past nnz (the builder pads them). */
int hbp_stream_workers(const hbp_format_t *f, int64_t *workers);
/* Precomputes the stream kernel's per-worker slice bounds and first groups
 * (otherwise every warp binary-searches group_start at launch -- ~20
 * dependent loads, visible on small matrices). */
int hbp_stream_slices(const hbp_format_t *f, const hbp_balanced_t *b, hbp_stream_t stream);
/* Stream-kernel cost of every group in element units (the per-warp cost
 * model fitted to measured warp times, tools/warp_cost.py): its elements -
 * (w_hot / 64) per element staged in shared memory (HBP_HOT_FLAG in scol;
 * cheaper gathers) + w_group + w_short per one- / two-step phase + w_step
 * per step-loop phase + w_modular per modular-pass phase (fewer than 12 live
 * lanes, more than 4 steps).  cost[ngroups]. */
int hbp_group_costs(const hbp_format_t *f, int64_t w_group, int64_t w_short, int64_t w_step,
                    int64_t w_modular, int64_t w_hot, int64_t *cost, hbp_stream_t stream);
/* Tuning: kernel variant of hbp_spmv_stream for later calls (0 = default;
 * the others are measured alternatives and diagnostics).
 * Not thread-safe; for benchmarks. */
int hbp_stream_set_variant(int variant);
int hbp_spmv_stream(const hbp_format_t *f, const hbp_balanced_t *b, const void *x, void *y,
                    double *partial, hbp_stream_t stream);
/* Hot-column staging for power-law column degrees (R-MAT): the n_hot
 * columns with the most nonzeros have their x entries copied into every
 * SM's shared memory at the start of hbp_spmv_stream, so their gathers are
 * shared-memory loads instead of L1->L2 sector requests (the bound of a
 * random-gather SpMV).  Results are unchanged: the same x
 * values are multiplied in the same order.  Not a reference interface; the
 * reference reads x[col] directly (_kernels.py:41-46).
 *   hbp_col_degree:  deg[c] += #{e = i * stride : col[e] == c} (deg zero-filled;
 *                    stride 1 = exact degrees, larger = a deterministic sample).
 *   hbp_hot_capacity: largest n_hot the stream kernel can stage for dtype
 *                    (mode 0: hot tier only; 1: with a warm tier; 2: with a
 *                    packed x, HBP_FLAG_PACKED_X -- its L2-resident gathers
 *                    leave L1 room for a larger tier).
 *   hbp_hot_slots:   slot_of[hot_cols[s]] = s (slot_of filled with -1).
 *   hbp_hot_remap:   scol[e] = slot s = slot_of[col[e]]: s < n_hot -> HBP_HOT_FLAG | s,
 *                    n_hot <= s -> HBP_WARM_FLAG | (s - n_hot), none -> col[e].
 *   hbp_hot_remap_packed: the same with n_hot <= s -> (s - n_hot) (HBP_FLAG_PACKED_X;
 *                    every column must have a slot).
 *   hbp_hot_gather:  x_hot[s] = x[hot_cols[s]] (run inside hbp_spmv_stream).
 * The warm tier (next-heaviest columns after the hot ones) is a compact copy
 * of x that the kernel gathers with an L2 evict-last policy while the other
 * ("cold") columns are gathered evict-first: on matrices whose x exceeds L2
 * (cfg5: 256 MB) the heavy columns stay L2-resident in a dense array. */
int hbp_col_degree(const uint32_t *col, int64_t nnz, int64_t stride, uint32_t *deg,
                   hbp_stream_t stream);
int hbp_hot_capacity(int dtype, int mode, int64_t *n_hot_max);
int hbp_hot_slots(const uint32_t *hot_cols, int64_t n_hot, int32_t *slot_of,
                  hbp_stream_t stream);
int hbp_hot_remap(const uint32_t *col, int64_t nnz, const int32_t *slot_of, int64_t n_hot,
                  uint32_t *scol, hbp_stream_t stream);
int hbp_hot_remap_packed(const uint32_t *col, int64_t nnz, const int32_t *slot_of, int64_t n_hot,
                         uint32_t *scol, hbp_stream_t stream);
int hbp_hot_gather(const void *x, int dtype, const uint32_t *hot_cols, int64_t n_hot,
                   void *x_hot, hbp_stream_t stream);
int hbp_spmv_balanced(const hbp_format_t *f, const hbp_balanced_t *b, const void *x, void *y,
                      double *partial, hbp_stream_t stream);

/* Column-segment schedule (warp_size == 32, several column blocks):
 * engine.py:123-134 block_spmv per nonzero block, with the block's
 * x-segment x[bc*C, (bc+1)*C) (engine.py:127-134) staged in shared memory --
 * only the window [win_lo, win_hi) its columns touch (hbp_seg_windows), one
 * TMA bulk copy per block, double-buffered.  One persistent CTA per worker
 * runs engine.py:96-176's plan: its fixed contiguous chunk of the bc-major
 * nonzero blocks, then blocks [fixed_count, nzb) drawn from an atomic
 * ticket.  The CTA's warps walk the block's groups lane-per-row in step
 * order (exact mode: bitwise _kernels.py:41-46).  Outputs as
 * hbp_spmv_stream: y when ncb == 1, else the compact partial (and y for
 * single-block row blocks with HBP_FLAG_DIRECT_SINGLE). */
typedef struct {
    int64_t ctas;           /* persistent CTAs (hbp_seg_workers) */
    int64_t fixed_count;    /* engine.py:107 int(f * nzb + 0.5) */
    uint32_t *ticket;       /* [2] device words, zeroed once by the caller; left zeroed */
    const int32_t *win_lo;  /* [nzb] first column the block touches */
    const int32_t *win_hi;  /* [nzb] one past the last */
    int64_t win_cap;        /* max(win_hi - win_lo): shared buffer size */
} hbp_seg_t;
/* Per nonzero block column window; *win_cap (device int64) = max width. */
int hbp_seg_windows(const hbp_format_t *f, int32_t *win_lo, int32_t *win_hi, int64_t *win_cap,
                    hbp_stream_t stream);
/* Resident CTAs for a window capacity (SMs x occupancy, at most nzb). */
int hbp_seg_workers(const hbp_format_t *f, int64_t win_cap, int64_t *ctas);
int hbp_spmv_seg(const hbp_format_t *f, const hbp_seg_t *s, const void *x, void *y,
                 double *partial, hbp_stream_t stream);
/* A/B tuning selector of the launch shape (HBP_SEG_VARIANT); 0 = default. */
int hbp_seg_set_variant(int v);

/* Row-block owner with TMA-staged elements (hbp_spmv_rowstage.cu; W = 32):
 * a persistent CTA per row block bulk-copies the col/data ranges of all the
 * row block's nonzero blocks -- and, with windows, each block's touched x
 * window -- into shared memory with one mbarrier, walks them there and folds
 * the block partials in ascending bc: y bitwise that of hbp_spmv_blocks +
 * hbp_combine.  hbp_rowstage_plan fills the per-block staging descriptors
 * desc (i64[4*nzb], rb_blk order) and caps (device u64[3]: largest staged
 * element span of a row block, most nonzero blocks in a row block, largest
 * staged x span); win_lo / win_hi are hbp_seg_windows' per-block column
 * windows (nullable: no x staging).  Pass ecap / kmax / xcap (xcap 0: x
 * gathered from global memory; > 0 needs a 16-byte aligned x); kmax <= 32,
 * shared memory ecap * (4 + sizeof V) + kmax * R * 8 + xcap * sizeof V must
 * fit one CTA. */
int hbp_rowstage_plan(const hbp_format_t *f, const int32_t *win_lo, const int32_t *win_hi,
                      int64_t *desc, unsigned long long *caps, hbp_stream_t stream);
int hbp_spmv_rowstage(const hbp_format_t *f, const int64_t *desc, const void *x, void *y,
                      int64_t ecap, int64_t kmax, int64_t xcap, hbp_stream_t stream);
/* engine.py:196-201 combine over nonzero blocks only, ascending bc
 * (bitwise equal to the dense combine); rows of row blocks with
 * no nonzero block get +0.0. */
int hbp_combine(const hbp_format_t *f, const double *partial, void *y, hbp_stream_t stream);
/* Row-block-owner SpMV + combine in one launch (small matrices with several
 * column blocks): one CTA per row block runs block_spmv (engine.py:123-134)
 * over its nonzero blocks in ascending bc and folds them as combine does
 * (engine.py:196-201), then writes y (+0.0 for empty row blocks).  Bitwise
 * equal to hbp_spmv_blocks + hbp_combine.  row_height <= 3072. */
int hbp_spmv_rowblock(const hbp_format_t *f, const void *x, void *y, hbp_stream_t stream);
/* engine.py:196-201 combine of a caller-made dense PartialVector
 * partial[bc*rows + row] (PartialVector(values, rows, ncb)): y = seg 0, then
 * y += seg bc for bc = 1..ncb-1 (__dadd_rn), f64 out. */
int hbp_combine_dense(const double *partial, int64_t rows, int64_t ncb, double *y,
                      hbp_stream_t stream);
/* Zero y for row blocks with no nonzero block (direct mode companion). */
int hbp_zero_empty_rows(const hbp_format_t *f, void *y, hbp_stream_t stream);
/* Dense PartialVector view (engine.py:59-68): partial_dense[bc*rows + row]. */
int hbp_expand_partial(const hbp_format_t *f, const double *partial, double *partial_dense,
                       hbp_stream_t stream);

/* hbp.py:241-315 hbp_to_triplets: invert the layout (per element row, col,
 * value) from slot lengths; integrity checks live in the host wrapper. */
int hbp_to_triplets(const hbp_format_t *f, int64_t *row_out, int64_t *col_out, void *val_out,
                    hbp_stream_t stream);

/* ------------------------------------------------ iterated SpMV (cfg5) */
/* Power iteration x <- A x / ||A x||_2 (the reference has no iterated path;
 * SURVEY.md §8(e) config 5).  hbp_sumsq: out[0] = sum y_i^2 in f64,
 * deterministic; scratch holds hbp_sumsq_scratch() doubles.  hbp_scale:
 * out_i = y_i * (V)(1 / sqrt(sumsq[0])), sumsq read on the device (after an
 * optional all-reduce), out may alias y. */
int hbp_sumsq(const void *y, int dtype, int64_t n, double *scratch, double *out,
              hbp_stream_t stream);
/* y_i += a_i (the two column parts of a row stripe in the overlapped power
 * iteration: own columns while the all-gather runs, the rest after it). */
int hbp_add(void *y, const void *a, int dtype, int64_t n, hbp_stream_t stream);
int hbp_sumsq_scratch(int64_t *doubles);
int hbp_scale(const void *y, int dtype, int64_t n, const double *sumsq, void *out,
              hbp_stream_t stream);

/* Peer mappings for the fused power iteration (hbp_balanced_t.y_peer): one
 * process per GPU exports the device buffer its next x lives in and maps the
 * other ranks' (CUDA IPC over NVLink / NVSwitch; the handles travel through
 * torch.distributed).  hbp_ipc_export: handle[HBP_IPC_HANDLE_BYTES] of the
 * allocation holding ptr and ptr's byte offset in it (device allocations
 * from a caching allocator start below ptr).  hbp_ipc_open: the exporter's
 * allocation mapped into this process, plus offset (*ptr is then the
 * exporter's ptr).  hbp_ipc_close: unmap (ptr as returned minus offset). */
#define HBP_IPC_HANDLE_BYTES 64
int hbp_ipc_export(const void *ptr, void *handle, int64_t *offset);
int hbp_ipc_open(const void *handle, int64_t offset, void **ptr);
int hbp_ipc_close(void *base);
#ifdef __cplusplus
}
#endif
#endif /* HBP_H */
