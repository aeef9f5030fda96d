// hbp_build.cu -- GPU preprocessing for the HBP format (sm_100a).
//
// Replaces the reference's CPU preprocessing:
//   make_grid          partition.py:100-127   -> count/emit runs, block heads, fill slots
//   sample_hash_params reorder.py:69-103       -> sampled counts (the (a, c) arithmetic
//                                                 stays on the host, same numpy calls)
//   hash_permutations  reorder.py:174-184 -> hbp_reorder.cu
//   build_hbp          hbp.py:150-238          -> slot lengths, group sizes, emission
// The reference's arrays are dense in rows x column-blocks; here every
// per-slot array is compact over NONZERO blocks and
// hbp_expand_reference() rebuilds the dense view for parity.
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

#include "hbp.h"
#include "hbp_common.cuh"

using namespace hbp;

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ int64_t rows_in_block(int64_t rows, int64_t R, int64_t br) {
    int64_t n = rows - br * R;
    return n < R ? n : R;
}

// ------------------------------------------------------------- make_grid
// A run head is the row's first element or an element whose column block
// differs from its predecessor's (partition.py:109-112).  A warp takes 32
// consecutive rows: each lane walks its own row when it is short (<= kShortRow
// elements: a row then costs one lane, not a warp with a dependent row_ptr
// load per row -- cfg3's 33.5M rows of 33 elements), and
// rows longer than that are walked by the whole warp, 32 elements per step.
// Column blocks by 32-bit division: C < cols < 2^31 off the single-block path.
constexpr int64_t kShortRow = 64;

__global__ void k_count_runs(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                             int64_t rows, int64_t C, int single_block,
                             int64_t *__restrict__ out) {
    const uint32_t Cu = (uint32_t)(C < 0xffffffffLL ? C : 0xffffffffLL);
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * 32; base < rows; base += nwarps * 32) {
        const int64_t r = base + lane;
        int64_t lo = 0, hi = 0;
        if (r < rows) lo = row_ptr[r], hi = row_ptr[r + 1];
        if (single_block) {
            if (r < rows) out[r] = hi > lo ? 1 : 0;
            continue;
        }
        const bool shortr = hi - lo <= kShortRow;
        if (r < rows && shortr) {
            int64_t cnt = 0;
            uint32_t prev = 0xffffffffu;
            for (int64_t j = lo; j < hi; ++j) {
                const uint32_t bc = (uint32_t)col[j] / Cu;
                cnt += bc != prev;
                prev = bc;
            }
            out[r] = cnt;
        }
        unsigned longm = __ballot_sync(0xffffffffu, r < rows && !shortr);
        while (longm) {
            const int l = __ffs(longm) - 1;
            longm &= longm - 1;
            const int64_t lo_l = __shfl_sync(0xffffffffu, lo, l), hi_l = __shfl_sync(0xffffffffu, hi, l);
            int64_t cnt = 0;
            for (int64_t b = lo_l; b < hi_l; b += 32) {
                const int64_t j = b + lane;
                bool head = false;
                if (j < hi_l)
                    head = (j == lo_l) || ((uint32_t)col[j] / Cu != (uint32_t)col[j - 1] / Cu);
                cnt += __popc(__ballot_sync(0xffffffffu, head));
            }
            if (lane == l) out[r] = cnt;
        }
    }
}

__global__ void k_emit_runs(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                            int64_t rows, int64_t C, int single_block,
                            const int64_t *__restrict__ run_offset, uint32_t *__restrict__ run_bc,
                            uint32_t *__restrict__ run_row, int64_t *__restrict__ run_start) {
    const uint32_t Cu = (uint32_t)(C < 0xffffffffLL ? C : 0xffffffffLL);
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t base = warp * 32; base < rows; base += nwarps * 32) {
        const int64_t r = base + lane;
        int64_t lo = 0, hi = 0, off = 0;
        if (r < rows) lo = row_ptr[r], hi = row_ptr[r + 1], off = run_offset[r];
        if (single_block) {
            if (r < rows && hi > lo) {
                run_bc[off] = 0;
                run_row[off] = (uint32_t)r;
                run_start[off] = lo;
            }
            continue;
        }
        const bool shortr = hi - lo <= kShortRow;
        if (r < rows && shortr) {
            uint32_t prev = 0xffffffffu;
            for (int64_t j = lo; j < hi; ++j) {
                const uint32_t bc = (uint32_t)col[j] / Cu;
                if (bc != prev) {
                    run_bc[off] = bc;
                    run_row[off] = (uint32_t)r;
                    run_start[off] = j;
                    ++off;
                }
                prev = bc;
            }
        }
        unsigned longm = __ballot_sync(0xffffffffu, r < rows && !shortr);
        while (longm) {
            const int l = __ffs(longm) - 1;
            longm &= longm - 1;
            const int64_t lo_l = __shfl_sync(0xffffffffu, lo, l), hi_l = __shfl_sync(0xffffffffu, hi, l);
            int64_t off_l = __shfl_sync(0xffffffffu, off, l);
            const int64_t r_l = base + l;
            for (int64_t b = lo_l; b < hi_l; b += 32) {
                const int64_t j = b + lane;
                bool head = false;
                uint32_t bc = 0;
                if (j < hi_l) {
                    bc = (uint32_t)col[j] / Cu;
                    head = (j == lo_l) || (bc != (uint32_t)col[j - 1] / Cu);
                }
                const unsigned m = __ballot_sync(0xffffffffu, head);
                if (head) {
                    const int64_t i = off_l + __popc(m & lt);
                    run_bc[i] = bc;
                    run_row[i] = (uint32_t)r_l;
                    run_start[i] = j;
                }
                off_l += __popc(m);
            }
        }
    }
}

// count = next run start of the same row (or the row end) - this start
__global__ void k_run_counts(const int64_t *__restrict__ row_ptr,
                             const int64_t *__restrict__ run_offset,
                             const uint32_t *__restrict__ run_row,
                             const int64_t *__restrict__ run_start, int64_t nruns,
                             int32_t *__restrict__ run_count) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nruns;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t r = run_row[i];
        int64_t end = (i + 1 < run_offset[r + 1]) ? run_start[i + 1] : row_ptr[r + 1];
        run_count[i] = (int32_t)(end - run_start[i]);
    }
}

__global__ void k_block_heads(const uint32_t *__restrict__ sbc, const uint32_t *__restrict__ order,
                              const uint32_t *__restrict__ run_row, int64_t nruns, int64_t R,
                              int64_t *__restrict__ head) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nruns;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t h = 1;
        if (i > 0) {
            uint32_t ri = run_row[order ? order[i] : i];
            uint32_t rp = run_row[order ? order[i - 1] : i - 1];
            uint32_t bi = sbc ? sbc[i] : 0, bp = sbc ? sbc[i - 1] : 0;
            h = (bi != bp) || (ri / R != rp / R);
        }
        head[i] = h;
    }
}

__global__ void k_fill_slots(const uint32_t *__restrict__ sbc, const uint32_t *__restrict__ order,
                             const uint32_t *__restrict__ run_row,
                             const int64_t *__restrict__ run_start,
                             const int32_t *__restrict__ run_count,
                             const int64_t *__restrict__ block_incl, int64_t nruns, int64_t R,
                             int32_t *__restrict__ blk_br, int32_t *__restrict__ blk_bc,
                             uint32_t *__restrict__ len_local, int64_t *__restrict__ start_local) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nruns;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t src = order ? order[i] : (uint32_t)i;
        uint32_t r = run_row[src];
        int64_t blk = block_incl[i] - 1;
        int64_t br = r / R;
        if (i == 0 || block_incl[i - 1] != block_incl[i]) {
            blk_br[blk] = (int32_t)br;
            blk_bc[blk] = sbc ? (int32_t)sbc[i] : 0;
        }
        int64_t s = blk * R + (r - br * R);
        len_local[s] = (uint32_t)run_count[src];
        start_local[s] = run_start[src];
    }
}

// warp per nonzero block
__global__ void k_block_nnz(const uint32_t *__restrict__ len_local, int64_t nzb, int64_t R,
                            int64_t *__restrict__ out) {
    int lane = threadIdx.x & 31;
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = warp; b < nzb; b += nwarps) {
        unsigned long long s = 0;
        for (int64_t i = lane; i < R; i += 32) s += len_local[b * R + i];
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[b] = (int64_t)s;
    }
}

// --------------------------------------------------------- sampled counts
// reorder.py:80-85 reads row_counts[flat] at numpy-drawn flat indices; the
// count of row r inside column block bc is found by binary search.
__device__ __forceinline__ int64_t lower_bound_col(const int32_t *col, int64_t lo, int64_t hi,
                                                   int64_t v) {
    while (lo < hi) {
        int64_t m = (lo + hi) >> 1;
        if ((int64_t)col[m] < v) lo = m + 1;
        else hi = m;
    }
    return lo;
}

__global__ void k_sample_counts(const int64_t *__restrict__ row_ptr,
                                const int32_t *__restrict__ col, int64_t rows, int64_t C,
                                const int64_t *__restrict__ flat, int64_t k,
                                int32_t *__restrict__ counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t f = flat[i];
        int64_t bc = f / rows, r = f - bc * rows;
        int64_t lo = row_ptr[r], hi = row_ptr[r + 1];
        int64_t a = lower_bound_col(col, lo, hi, bc * C);
        int64_t b = lower_bound_col(col, a, hi, (bc + 1) * C);
        counts[i] = (int32_t)(b - a);
    }
}

// Bijection check, warp per block with a per-warp bitmap in shared memory.
// dense == true: every (br, bc) block of a [ncb*rows] table (hbp.py:179-181);
// otherwise the compact [nzb*R] table.  *bad = min offending block index.
__global__ void k_check_perm(const uint32_t *__restrict__ tab, int64_t rows, int64_t R,
                             int64_t nrb, int64_t nblocks, const int32_t *__restrict__ blk_br,
                             int dense, long long *__restrict__ bad) {
    extern __shared__ uint32_t bits[];
    int lane = threadIdx.x & 31;
    int wib = threadIdx.x >> 5;
    int nw = (int)((R + 31) >> 5);
    uint32_t *my = bits + wib * nw;
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t blk = warp; blk < nblocks; blk += nwarps) {
        int64_t br, base;
        if (dense) {
            int64_t bc = blk / nrb;
            br = blk - bc * nrb;
            base = bc * rows + br * R;
        } else {
            br = blk_br[blk];
            base = blk * R;
        }
        int64_t n = rows_in_block(rows, R, br);
        for (int w = lane; w < nw; w += 32) my[w] = 0u;
        __syncwarp();
        bool ok = true;
        for (int64_t s = lane; s < n; s += 32) {
            uint32_t v = tab[base + s];
            if (v >= (uint64_t)n) {
                ok = false;
            } else {
                uint32_t old = atomicOr(&my[v >> 5], 1u << (v & 31));
                if (old & (1u << (v & 31))) ok = false;
            }
        }
        if (!__all_sync(0xffffffffu, ok) && lane == 0) atomicMin(bad, (long long)blk);
        __syncwarp();
    }
}

__global__ void k_gather_perm(const uint32_t *__restrict__ dense, int64_t rows, int64_t R,
                              const int32_t *__restrict__ blk_br,
                              const int32_t *__restrict__ blk_bc, int64_t nzb,
                              uint32_t *__restrict__ perm) {
    int64_t total = nzb * R;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t blk = i / R, s = i - blk * R;
        int64_t br = blk_br[blk];
        int64_t n = rows_in_block(rows, R, br);
        perm[i] = s < n ? dense[(int64_t)blk_bc[blk] * rows + br * R + s] : 0u;
    }
}

// ----------------------------------------------------------- build_hbp
// One lane-group (segment) per HBP warp group.
__global__ void k_slot_lengths(const uint32_t *__restrict__ len_local,
                               const uint32_t *__restrict__ perm,
                               const int32_t *__restrict__ blk_br, int64_t nzb, int64_t rows,
                               int64_t R, int W, uint32_t *__restrict__ slot_len,
                               int32_t *__restrict__ zero_row, int64_t *__restrict__ group_nnz) {
    Seg sg = make_seg(W);
    if (sg.idle()) return;
    const int64_t gpb = R / W;
    const int64_t ngroups = nzb * gpb;
    int64_t seg_id = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * sg.spw + sg.seg;
    int64_t nseg = (((int64_t)gridDim.x * blockDim.x) >> 5) * sg.spw;
    if (seg_id == 0 && sg.q == 0) group_nnz[ngroups] = 0;
    for (int64_t gg = seg_id; gg < ngroups; gg += nseg) {
        int64_t blk = gg / gpb, g = gg - blk * gpb;
        int64_t n = rows_in_block(rows, R, blk_br[blk]);
        int64_t slot = g * W + sg.q;
        bool valid = slot < n;
        uint32_t len = 0;
        if (valid) {
            uint32_t r = perm[blk * R + slot];
            len = r < (uint32_t)n ? len_local[blk * R + r] : 0u;  // bad tables caught by k_check_perm
        }
        slot_len[blk * R + slot] = len;
        unsigned empt = seg_ballot(sg, valid && len == 0);
        if (zero_row) {
            int32_t zr = (valid && len == 0) ? -1 : __popc(empt & ((1u << sg.q) - 1u));
            zero_row[blk * R + slot] = valid ? zr : -1;
        }
        long long tot = seg_add_i64(sg, (long long)len);
        if (sg.q == 0) group_nnz[gg] = tot;
    }
}

// Column-major emission within a group (hbp.py:194-213).  Within a "phase"
// (a maximal step range with a fixed live-lane set of size k) the element
// of live lane `rank` at step t sits at base + (t - t0) * k + rank, so all
// addresses come from the slot lengths.
template <typename V>
__global__ void k_emit(const uint32_t *__restrict__ slot_len, const uint32_t *__restrict__ perm,
                       const int64_t *__restrict__ start_local,
                       const int64_t *__restrict__ group_start,
                       const int32_t *__restrict__ blk_br, int64_t nzb, int64_t rows, int64_t R,
                       int W, const int32_t *__restrict__ col_idx, const V *__restrict__ vals,
                       uint32_t *__restrict__ col_out, V *__restrict__ data_out,
                       int32_t *__restrict__ add_out) {
    __shared__ int64_t tab_src[kThreads / 32][32];
    __shared__ int32_t tab_nx[kThreads / 32][32];  // rank in the next phase, or -1
    Seg sg = make_seg(W);
    if (sg.idle()) return;
    const int wib = threadIdx.x >> 5;
    const int64_t gpb = R / W;
    const int64_t ngroups = nzb * gpb;
    const unsigned lt = (1u << sg.q) - 1u;
    int64_t seg_id = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * sg.spw + sg.seg;
    int64_t nseg = (((int64_t)gridDim.x * blockDim.x) >> 5) * sg.spw;
    for (int64_t gg = seg_id; gg < ngroups; gg += nseg) {
        int64_t blk = gg / gpb, g = gg - blk * gpb;
        int64_t slot = blk * R + g * W + sg.q;
        uint32_t len = slot_len[slot];
        int64_t src = len ? start_local[blk * R + perm[slot]] : 0;
        int64_t base = group_start[gg];
        uint32_t t0 = 0;
        bool live = len > 0;
        unsigned mask = seg_ballot(sg, live);
        while (mask) {
            const int k = __popc(mask);
            const int rank = __popc(mask & lt);
            const uint32_t t1 = seg_min_u32(sg, live ? len : 0xffffffffu);
            const bool live_n = len > t1;
            const unsigned mask_n = seg_ballot(sg, live_n);
            const int rank_n = __popc(mask_n & lt);
            const int64_t M = (int64_t)(t1 - t0);
            if (2 * k >= W || M < 4) {
                if (live) {
                    int64_t p = base + rank;
                    int64_t j = src + t0;
                    for (int64_t t = 0; t < M; ++t, p += k, ++j) {
                        col_out[p] = (uint32_t)col_idx[j];
                        data_out[p] = vals[j];
                        if (add_out)
                            add_out[p] = (t + 1 < M) ? k : (live_n ? k + rank_n - rank : -1);
                    }
                }
            } else {
                // few live lanes over many steps: the segment writes the
                // phase's positions cooperatively (coalesced)
                if (live) {
                    tab_src[wib][sg.shift + rank] = src + t0;
                    tab_nx[wib][sg.shift + rank] = live_n ? (k + rank_n - rank) : -1;
                }
                __syncwarp(sg.mask);
                const int64_t total = M * k;
                for (int64_t off = sg.q; off < total; off += W) {
                    int64_t t = off / k;
                    int r = (int)(off - t * k);
                    int64_t j = tab_src[wib][sg.shift + r] + t;
                    int64_t p = base + off;
                    col_out[p] = (uint32_t)col_idx[j];
                    data_out[p] = vals[j];
                    if (add_out) add_out[p] = (t + 1 < M) ? k : tab_nx[wib][sg.shift + r];
                }
                __syncwarp(sg.mask);
            }
            base += M * k;
            t0 = t1;
            live = live_n;
            mask = mask_n;
        }
    }
}

// Element-balanced emission for W = 32.  k_emit gives a warp whole groups,
// so the few groups holding hot rows serialise the tail (measured: 23 % of
// warps active on R-MAT).  Here warp w owns the output range
// [w E / N, (w+1) E / N), enters the group and phase containing its start,
// and writes every phase it overlaps cooperatively: 32 consecutive output
// positions per pass (coalesced stores); position off of a phase with k
// live lanes is step t = off / k of rank r = off mod k, read from the rank's
// source row (a shared-memory table built at phase entry).
__constant__ uint32_t c_emit_magic[33] = {
    0u,          0u,          2147483648u, 1431655766u, 1073741824u, 858993460u,  715827883u,
    613566757u,  536870912u,  477218589u,  429496730u,  390451573u,  357913942u,  330382100u,
    306783379u,  286331154u,  268435456u,  252645136u,  238609295u,  226050911u,  214748365u,
    204522253u,  195225787u,  186737709u,  178956971u,  171798692u,  165191050u,  159072863u,
    153391690u,  148102321u,  143165577u,  138547333u,  134217728u};

__device__ __forceinline__ int64_t div_k(int64_t n, int k) {  // n >= 0, 1 <= k <= 32
    if (k == 1) return n;
    if (n < (1 << 26)) return (int64_t)(((uint64_t)n * c_emit_magic[k]) >> 32);
    return n / k;
}

template <typename V>
__global__ void __launch_bounds__(kThreads)
    k_emit_sliced(const uint32_t *__restrict__ slot_len, const uint32_t *__restrict__ perm,
                  const int64_t *__restrict__ start_local, const int64_t *__restrict__ gs,
                  int64_t nzb, int64_t R, const int32_t *__restrict__ col_idx,
                  const V *__restrict__ vals, uint32_t *__restrict__ col_out,
                  V *__restrict__ data_out, int32_t *__restrict__ add_out) {
    __shared__ int64_t tab_src[kThreads / 32][32];
    __shared__ int32_t tab_nx[kThreads / 32][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t gpb = R / 32, ngroups = nzb * gpb;
    const int64_t E = gs[ngroups];
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t lo = (int64_t)((__int128)w * E / nw), hi = (int64_t)((__int128)(w + 1) * E / nw);
    if (lo >= hi) return;
    // group containing lo: largest g with gs[g] <= lo
    int64_t a = 0, b = ngroups;
    while (b - a > 1) {
        const int64_t m = (a + b) >> 1;
        if (gs[m] <= lo) a = m;
        else b = m;
    }
    for (int64_t g = a; g < ngroups; ++g) {
        const int64_t g0 = gs[g], g1 = gs[g + 1];
        if (g0 >= hi) break;
        if (g1 <= lo) continue;
        const int64_t blk = g / gpb;
        const int64_t slot = blk * R + (g - blk * gpb) * 32 + lane;
        const uint32_t len = slot_len[slot];
        const int64_t src = len ? start_local[blk * R + perm[slot]] : 0;
        int64_t pbase = g0;
        uint32_t t0 = 0;
        bool live = len > 0;
        unsigned mask = __ballot_sync(0xffffffffu, live);
        while (mask) {
            const int k = __popc(mask);
            const int rank = __popc(mask & lt);
            const uint32_t t1 = __reduce_min_sync(0xffffffffu, live ? len : 0xffffffffu);
            const bool live_n = len > t1;
            const unsigned mask_n = __ballot_sync(0xffffffffu, live_n);
            const int rank_n = __popc(mask_n & lt);
            const int64_t M = (int64_t)(t1 - t0);
            const int64_t pend = pbase + M * k;
            if (pend > lo) {
                __syncwarp();
                if (live) {
                    tab_src[wib][rank] = src + t0;
                    tab_nx[wib][rank] = live_n ? (k + rank_n - rank) : -1;
                }
                __syncwarp();
                const int64_t o0 = (lo > pbase ? lo : pbase) - pbase;
                const int64_t o1 = (hi < pend ? hi : pend) - pbase;
                for (int64_t off = o0 + lane; off < o1; off += 32) {
                    const int64_t t = div_k(off, k);
                    const int r = (int)(off - t * k);
                    const int64_t j = tab_src[wib][r] + t;
                    const int64_t p = pbase + off;
                    col_out[p] = (uint32_t)__ldg(col_idx + j);
                    data_out[p] = __ldg(vals + j);
                    if (add_out) add_out[p] = (t + 1 < M) ? k : tab_nx[wib][r];
                }
                if (pend >= hi) return;
            }
            pbase = pend;
            t0 = t1;
            live = live_n;
            mask = mask_n;
        }
    }
}

// ---- phase stream (runtime index for the streaming SpMV, W = 32) --------
// A group's "phases" are its maximal step ranges with a fixed live-lane set
// (one per distinct nonzero slot length).  Phase j is stored as
// (live mask, group-relative element offset); k = popc(mask), its step count
// is (next offset - offset) / k.  Warp per group.
__global__ void k_phase_counts(const uint32_t *__restrict__ slot_len, int64_t ngroups,
                               int64_t *__restrict__ nph) {
    const int lane = threadIdx.x & 31;
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t g = warp; g < ngroups; g += nwarps) {
        const uint32_t len = slot_len[g * 32 + lane];
        // distinct nonzero lengths: lane counts if no lower lane has the same length
        const unsigned same = __match_any_sync(0xffffffffu, len);
        const bool first = len > 0 && (same & ((1u << lane) - 1u)) == 0u;
        const int n = __popc(__ballot_sync(0xffffffffu, first));
        if (lane == 0) nph[g] = n;
    }
    if (warp == 0 && lane == 0) nph[ngroups] = 0;
}

__global__ void k_phase_emit(const uint32_t *__restrict__ slot_len, int64_t ngroups,
                             const int64_t *__restrict__ phase_ptr, uint2 *__restrict__ phases) {
    const int lane = threadIdx.x & 31;
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t g = warp; g < ngroups; g += nwarps) {
        const uint32_t len = slot_len[g * 32 + lane];
        uint2 *out = phases + phase_ptr[g];
        uint32_t t0 = 0, off = 0;
        int j = 0;
        bool live = len > 0;
        unsigned mask = __ballot_sync(0xffffffffu, live);
        while (mask) {
            const uint32_t t1 = __reduce_min_sync(0xffffffffu, live ? len : 0xffffffffu);
            if (lane == (j & 31)) out[j] = make_uint2(mask, off);
            off += (t1 - t0) * (uint32_t)__popc(mask);
            ++j;
            t0 = t1;
            live = len > t0;
            mask = __ballot_sync(0xffffffffu, live);
        }
    }
}

__global__ void k_rb_counts(const int32_t *__restrict__ blk_br, int64_t nzb,
                            int64_t *__restrict__ cnt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nzb;
         i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long *)&cnt[blk_br[i]], 1ull);
}

// ------------------------------------------------------ dense expansion
__global__ void k_expand_slots(int64_t rows, int64_t ncb, int64_t R,
                               const uint32_t *__restrict__ ep_full,
                               const uint32_t *__restrict__ ep_last,
                               uint32_t *__restrict__ output_hash, int32_t *__restrict__ zero_row) {
    int64_t total = ncb * rows;
    int64_t nrb = (rows + R - 1) / R;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i % rows;
        int64_t br = r / R, s = r - br * R;
        bool last_short = (br == nrb - 1) && (rows - br * R) < R;
        output_hash[i] = last_short ? ep_last[s] : ep_full[s];
        zero_row[i] = -1;
    }
}

__global__ void k_scatter_slots(const int32_t *__restrict__ blk_br,
                                const int32_t *__restrict__ blk_bc, int64_t nzb, int64_t rows,
                                int64_t R, const uint32_t *__restrict__ perm,
                                const int32_t *__restrict__ zr_c,
                                uint32_t *__restrict__ output_hash, int32_t *__restrict__ zero_row) {
    int64_t total = nzb * R;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t blk = i / R, s = i - blk * R;
        int64_t br = blk_br[blk];
        if (s >= rows_in_block(rows, R, br)) continue;
        int64_t d = (int64_t)blk_bc[blk] * rows + br * R + s;
        output_hash[d] = perm[i];
        zero_row[d] = zr_c[i];
    }
}

__global__ void k_expand_groups(const int32_t *__restrict__ blk_br,
                                const int32_t *__restrict__ blk_bc, int64_t nzb, int64_t nrb,
                                int64_t ncb, int64_t gpc, int64_t gpb, int64_t nnz,
                                const int64_t *__restrict__ gs_c, int64_t *__restrict__ gs) {
    int64_t total = ncb * gpc;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= total;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (e == total) {
            gs[e] = nnz;
            continue;
        }
        int64_t bc = e / gpc, rem = e - bc * gpc;
        int64_t br = rem / gpb, g = rem - br * gpb;
        int64_t key = bc * nrb + br;
        int64_t lo = 0, hi = nzb;
        while (lo < hi) {
            int64_t m = (lo + hi) >> 1;
            int64_t km = (int64_t)blk_bc[m] * nrb + blk_br[m];
            if (km < key) lo = m + 1;
            else hi = m;
        }
        int64_t v;
        if (lo < nzb && (int64_t)blk_bc[lo] * nrb + blk_br[lo] == key) v = gs_c[lo * gpb + g];
        else v = lo < nzb ? gs_c[lo * gpb] : nnz;
        gs[e] = v;
    }
}

// hbp.py:241-315 hbp_to_triplets: walk every slot's add_sign chain over the
// reference-layout arrays (dense zero_row / output_hash / group_start), one
// thread per slot.  err bits: 1 lane start outside its group, 2 column
// outside the block, 4 invalid stride, 8 chain escapes its group.
__global__ void k_walk_chains(int64_t rows, int64_t cols, int64_t C, int64_t R, int64_t W,
                              int64_t ncb, int64_t gpc, const int32_t *__restrict__ zero_row,
                              const uint32_t *__restrict__ output_hash,
                              const int64_t *__restrict__ group_start,
                              const uint32_t *__restrict__ col, const int32_t *__restrict__ add,
                              int64_t nnz, int64_t *__restrict__ row_out,
                              int32_t *__restrict__ seen, int32_t *__restrict__ err) {
    int64_t total = ncb * rows;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t zr = zero_row[i];
        if (zr < 0) continue;
        int64_t bc = i / rows, row = i - bc * rows;
        int64_t br = row / R, s = row - br * R, g = s / W, q = s - g * W;
        int64_t gb = bc * gpc + br * (R / W) + g;
        int64_t gs = group_start[gb], ge = group_start[gb + 1];
        int64_t j = gs + q - zr;
        if (j < gs || j >= ge || j >= nnz || j < 0) {
            atomicOr(err, 1);
            continue;
        }
        int64_t out_row = br * R + (int64_t)output_hash[i];
        int64_t lo = bc * C, hi = lo + C < cols ? lo + C : cols;
        for (;;) {
            int64_t c = col[j];
            if (c < lo || c >= hi) {
                atomicOr(err, 2);
                break;
            }
            atomicAdd(&seen[j], 1);
            row_out[j] = out_row;
            int32_t step = add[j];
            if (step == 0 || (step < 0 && step != -1)) {
                atomicOr(err, 4);
                break;
            }
            if (step < 0) break;
            j += step;
            if (j >= ge || j >= nnz) {
                atomicOr(err, 8);
                break;
            }
        }
    }
}

// Slot lengths of a reference-layout matrix (deserialize_hbp): per dense slot
// the number of elements on its add_sign chain, walked as hbp_block_kernel
// walks it (_kernels.py:35-46) but bounded to the group's element range, so a
// corrupt chain ends instead of running away (validation is separate).
__global__ void k_chain_lengths(int64_t rows, int64_t R, int64_t W, int64_t ncb, int64_t gpc,
                                const int32_t *__restrict__ zero_row,
                                const int64_t *__restrict__ group_start,
                                const int32_t *__restrict__ add, int64_t nnz,
                                int32_t *__restrict__ len_out) {
    int64_t total = ncb * rows;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t zr = zero_row[i];
        int32_t k = 0;
        if (zr >= 0) {
            int64_t bc = i / rows, row = i - bc * rows;
            int64_t br = row / R, s = row - br * R, g = s / W, q = s - g * W;
            int64_t gb = bc * gpc + br * (R / W) + g;
            int64_t gs = group_start[gb], ge = group_start[gb + 1];
            int64_t j = gs + q - zr;
            for (;;) {
                ++k;
                int32_t st = (j >= 0 && j < nnz) ? add[j] : -1;
                if (st < 0 || j + st >= ge) break;
                j += st;
            }
        }
        len_out[i] = k;
    }
}

}  // namespace

// ====================================================================== ABI
extern "C" {

int hbp_grid_count_runs(const int64_t *row_ptr, const int32_t *col_idx, int64_t rows,
                        int64_t cols, int64_t col_width, int64_t *runs_per_row,
                        hbp_stream_t stream) {
    if (rows < 1 || col_width < 1) return HBP_E_ARG;
    k_count_runs<<<grid_for(rows * 32, kThreads), kThreads, 0, as_stream(stream)>>>(
        row_ptr, col_idx, rows, col_width, col_width >= cols, runs_per_row);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_grid_emit_runs(const int64_t *row_ptr, const int32_t *col_idx, int64_t rows,
                       int64_t cols, int64_t col_width, const int64_t *run_offset,
                       int64_t nruns, uint32_t *run_bc, uint32_t *run_row, int64_t *run_start,
                       int32_t *run_count, hbp_stream_t stream) {
    if (rows < 1 || col_width < 1) return HBP_E_ARG;
    cudaStream_t s = as_stream(stream);
    k_emit_runs<<<grid_for(rows * 32, kThreads), kThreads, 0, s>>>(
        row_ptr, col_idx, rows, col_width, col_width >= cols, run_offset, run_bc, run_row,
        run_start);
    HBP_LAUNCH_CHECK();
    if (nruns > 0) {
        k_run_counts<<<grid_for(nruns, kThreads), kThreads, 0, s>>>(row_ptr, run_offset, run_row,
                                                                    run_start, nruns, run_count);
        HBP_LAUNCH_CHECK();
    }
    return HBP_OK;
}

int hbp_grid_block_heads(const uint32_t *sorted_bc, const uint32_t *order,
                         const uint32_t *run_row, int64_t nruns, int64_t row_height,
                         int64_t *head, hbp_stream_t stream) {
    if (nruns <= 0) return HBP_OK;
    k_block_heads<<<grid_for(nruns, kThreads), kThreads, 0, as_stream(stream)>>>(
        sorted_bc, order, run_row, nruns, row_height, head);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_grid_fill_slots(const uint32_t *sorted_bc, const uint32_t *order,
                        const uint32_t *run_row, const int64_t *run_start,
                        const int32_t *run_count, const int64_t *block_incl, int64_t nruns,
                        int64_t row_height, int32_t *blk_br, int32_t *blk_bc,
                        uint32_t *len_local, int64_t *start_local, hbp_stream_t stream) {
    if (nruns <= 0) return HBP_OK;
    k_fill_slots<<<grid_for(nruns, kThreads), kThreads, 0, as_stream(stream)>>>(
        sorted_bc, order, run_row, run_start, run_count, block_incl, nruns, row_height, blk_br,
        blk_bc, len_local, start_local);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_block_nnz(const uint32_t *len_local, int64_t nzb, int64_t row_height, int64_t *block_nnz,
                  hbp_stream_t stream) {
    if (nzb <= 0) return HBP_OK;
    k_block_nnz<<<grid_for(nzb * 32, kThreads), kThreads, 0, as_stream(stream)>>>(
        len_local, nzb, row_height, block_nnz);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_sample_counts(const int64_t *row_ptr, const int32_t *col_idx, int64_t rows,
                      int64_t col_width, const int64_t *flat_idx, int64_t k, int32_t *counts,
                      hbp_stream_t stream) {
    if (k <= 0) return HBP_OK;
    k_sample_counts<<<grid_for(k, kThreads), kThreads, 0, as_stream(stream)>>>(
        row_ptr, col_idx, rows, col_width, flat_idx, k, counts);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

static int check_perm(const uint32_t *tab, int64_t rows, int64_t R, int64_t nrb, int64_t nblocks,
                      const int32_t *blk_br, int dense, long long *bad, cudaStream_t s) {
    if (nblocks <= 0) return HBP_OK;
    int64_t nw = (R + 31) / 32;
    int warps = 8;
    while (warps > 1 && nw * 4 * warps > 48 * 1024) warps >>= 1;
    if (nw * 4 * warps > 48 * 1024) return HBP_E_UNSUPPORTED;
    k_check_perm<<<grid_for(nblocks * 32, warps * 32), warps * 32, (size_t)(nw * 4 * warps), s>>>(
        tab, rows, R, nrb, nblocks, blk_br, dense, bad);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_gather_dense_perm(const uint32_t *dense, int64_t rows, int64_t ncb, int64_t row_height,
                          const int32_t *blk_br, const int32_t *blk_bc, int64_t nzb,
                          uint32_t *perm, long long *bad, hbp_stream_t stream) {
    cudaStream_t s = as_stream(stream);
    int64_t nrb = (rows + row_height - 1) / row_height;
    int st = check_perm(dense, rows, row_height, nrb, ncb * nrb, nullptr, 1, bad, s);
    if (st) return st;
    if (nzb > 0) {
        k_gather_perm<<<grid_for(nzb * row_height, kThreads), kThreads, 0, s>>>(
            dense, rows, row_height, blk_br, blk_bc, nzb, perm);
        HBP_LAUNCH_CHECK();
    }
    return HBP_OK;
}

int hbp_slot_lengths(const uint32_t *len_local, const uint32_t *perm, const int32_t *blk_br,
                     int64_t nzb, int64_t rows, int64_t row_height, int64_t warp_size,
                     uint32_t *slot_len, int32_t *zero_row, int64_t *group_nnz,
                     long long *bad, hbp_stream_t stream) {
    if (warp_size < 1 || warp_size > 32 || row_height % warp_size) return HBP_E_UNSUPPORTED;
    cudaStream_t s = as_stream(stream);
    int64_t nrb = (rows + row_height - 1) / row_height;
    if (bad) {
        int st = check_perm(perm, rows, row_height, nrb, nzb, blk_br, 0, bad, s);
        if (st) return st;
    }
    int64_t ngroups = nzb * (row_height / warp_size);
    int64_t spw = 32 / warp_size;
    int64_t warps = (ngroups + spw - 1) / spw;
    k_slot_lengths<<<grid_for((warps > 0 ? warps : 1) * 32, kThreads), kThreads, 0, s>>>(
        len_local, perm, blk_br, nzb, rows, row_height, (int)warp_size, slot_len, zero_row,
        group_nnz);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_emit(const uint32_t *slot_len, const uint32_t *perm, const int64_t *start_local,
             const int64_t *group_start, const int32_t *blk_br, int64_t nzb, int64_t rows,
             int64_t row_height, int64_t warp_size, const int32_t *col_idx, const void *values,
             int dtype, uint32_t *col, void *data, int32_t *add_sign, hbp_stream_t stream) {
    if (warp_size < 1 || warp_size > 32 || row_height % warp_size) return HBP_E_UNSUPPORTED;
    if (nzb <= 0) return HBP_OK;
    int64_t ngroups = nzb * (row_height / warp_size);
    int64_t spw = 32 / warp_size;
    unsigned grid = grid_for(((ngroups + spw - 1) / spw) * 32, kThreads);
    cudaStream_t s = as_stream(stream);
    if (warp_size == 32) {  // element-balanced emission
        int dev = 0, sms = 0;
        HBP_CUDA_TRY(cudaGetDevice(&dev));
        HBP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const unsigned g2 = (unsigned)sms * 8;  // 64 warps per SM
        if (dtype == HBP_F64)
            k_emit_sliced<double><<<g2, kThreads, 0, s>>>(
                slot_len, perm, start_local, group_start, nzb, row_height, col_idx,
                (const double *)values, col, (double *)data, add_sign);
        else if (dtype == HBP_F32)
            k_emit_sliced<float><<<g2, kThreads, 0, s>>>(
                slot_len, perm, start_local, group_start, nzb, row_height, col_idx,
                (const float *)values, col, (float *)data, add_sign);
        else
            return HBP_E_ARG;
        HBP_LAUNCH_CHECK();
        return HBP_OK;
    }
    if (dtype == HBP_F64)
        k_emit<double><<<grid, kThreads, 0, s>>>(slot_len, perm, start_local, group_start, blk_br,
                                                 nzb, rows, row_height, (int)warp_size, col_idx,
                                                 (const double *)values, col, (double *)data,
                                                 add_sign);
    else if (dtype == HBP_F32)
        k_emit<float><<<grid, kThreads, 0, s>>>(slot_len, perm, start_local, group_start, blk_br,
                                                nzb, rows, row_height, (int)warp_size, col_idx,
                                                (const float *)values, col, (float *)data,
                                                add_sign);
    else
        return HBP_E_ARG;
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_phase_counts(const uint32_t *slot_len, int64_t ngroups, int64_t *nph,
                     hbp_stream_t stream) {
    if (ngroups < 0) return HBP_E_ARG;
    k_phase_counts<<<grid_for((ngroups + 1) * 32, kThreads), kThreads, 0, as_stream(stream)>>>(
        slot_len, ngroups, nph);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_phase_emit(const uint32_t *slot_len, int64_t ngroups, const int64_t *phase_ptr,
                   void *phases, hbp_stream_t stream) {
    if (ngroups <= 0) return HBP_OK;
    k_phase_emit<<<grid_for(ngroups * 32, kThreads), kThreads, 0, as_stream(stream)>>>(
        slot_len, ngroups, phase_ptr, (uint2 *)phases);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_row_block_counts(const int32_t *blk_br, int64_t nzb, int64_t *rb_count,
                         hbp_stream_t stream) {
    if (nzb <= 0) return HBP_OK;
    k_rb_counts<<<grid_for(nzb, kThreads), kThreads, 0, as_stream(stream)>>>(blk_br, nzb,
                                                                             rb_count);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_expand_reference(const int32_t *blk_br, const int32_t *blk_bc, int64_t nzb, int64_t rows,
                         int64_t cols, int64_t nnz, int64_t col_width, int64_t row_height,
                         int64_t warp_size, const uint32_t *perm, const int32_t *zero_row_c,
                         const int64_t *group_start_c, const uint32_t *empty_perm_full,
                         const uint32_t *empty_perm_last, int32_t *zero_row, uint32_t *output_hash,
                         int64_t *group_start, hbp_stream_t stream) {
    if (warp_size < 1 || row_height % warp_size) return HBP_E_ARG;
    cudaStream_t s = as_stream(stream);
    int64_t R = row_height, W = warp_size;
    int64_t nrb = (rows + R - 1) / R, ncb = (cols + col_width - 1) / col_width;
    int64_t last = rows - (nrb - 1) * R;
    int64_t gpc = (nrb - 1) * (R / W) + (last + W - 1) / W;
    k_expand_slots<<<grid_for(ncb * rows, kThreads), kThreads, 0, s>>>(
        rows, ncb, R, empty_perm_full, empty_perm_last, output_hash, zero_row);
    HBP_LAUNCH_CHECK();
    if (nzb > 0) {
        k_scatter_slots<<<grid_for(nzb * R, kThreads), kThreads, 0, s>>>(
            blk_br, blk_bc, nzb, rows, R, perm, zero_row_c, output_hash, zero_row);
        HBP_LAUNCH_CHECK();
    }
    k_expand_groups<<<grid_for(ncb * gpc + 1, kThreads), kThreads, 0, s>>>(
        blk_br, blk_bc, nzb, nrb, ncb, gpc, R / W, nnz, group_start_c, group_start);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_walk_chains(int64_t rows, int64_t cols, int64_t col_width, int64_t row_height,
                    int64_t warp_size, const int32_t *zero_row, const uint32_t *output_hash,
                    const int64_t *group_start, const uint32_t *col, const int32_t *add_sign,
                    int64_t nnz, int64_t *row_out, int32_t *seen, int32_t *err,
                    hbp_stream_t stream) {
    if (warp_size < 1 || row_height % warp_size) return HBP_E_ARG;
    int64_t R = row_height, W = warp_size;
    int64_t nrb = (rows + R - 1) / R, ncb = (cols + col_width - 1) / col_width;
    int64_t last = rows - (nrb - 1) * R;
    int64_t gpc = (nrb - 1) * (R / W) + (last + W - 1) / W;
    k_walk_chains<<<grid_for(ncb * rows, kThreads), kThreads, 0, as_stream(stream)>>>(
        rows, cols, col_width, R, W, ncb, gpc, zero_row, output_hash, group_start, col, add_sign,
        nnz, row_out, seen, err);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_chain_lengths(int64_t rows, int64_t cols, int64_t col_width, int64_t row_height,
                      int64_t warp_size, const int32_t *zero_row, const int64_t *group_start,
                      const int32_t *add_sign, int64_t nnz, int32_t *len_out,
                      hbp_stream_t stream) {
    if (warp_size < 1 || row_height < 1 || row_height % warp_size || col_width < 1)
        return HBP_E_ARG;
    if (rows < 1 || cols < 1) return HBP_OK;
    int64_t R = row_height, W = warp_size;
    int64_t nrb = (rows + R - 1) / R, ncb = (cols + col_width - 1) / col_width;
    int64_t last = rows - (nrb - 1) * R;
    int64_t gpc = (nrb - 1) * (R / W) + (last + W - 1) / W;
    k_chain_lengths<<<grid_for(ncb * rows, kThreads), kThreads, 0, as_stream(stream)>>>(
        rows, R, W, ncb, gpc, zero_row, group_start, add_sign, nnz, len_out);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

}  // extern "C"
