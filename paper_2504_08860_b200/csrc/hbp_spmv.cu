// hbp_spmv.cu -- the HBP SpMV and the combine on sm_100a.
//
// Reference path: hbp_spmv (engine.py:228-232) ->
// plan_execution (engine.py:96-115) -> run_spmv (engine.py:179-193) ->
// _run_plan (engine.py:137-176: fixed chunks, then a ticket) -> block_spmv
// (engine.py:123-134) -> hbp_block_kernel (_kernels.py:22-47) -> combine
// (engine.py:196-201).
//
// GPU mapping ("each block being computed by a warp"): one
// persistent warp per worker; a worker runs its fixed contiguous chunk of
// nonzero blocks, then claims blocks with an atomic ticket.  Inside a block
// each W-lane segment owns one HBP group and each lane one slot (= one row).
// Instead of chasing add_sign (a serial dependent-load chain) the lane
// derives element addresses from the group's slot lengths: within a phase
// where k lanes are live, lane `rank` reads base + t*k + rank -- the same
// elements in the same order, coalesced across the
// k live lanes, with loads of several steps in flight.  Each row's sum is
// accumulated in step order, so:
//   f64: __dmul_rn / __dadd_rn, bitwise identical to the reference;
//   f32: products are exact in f64, sums in f64, one rounding at the end.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "hbp.h"
#include "hbp_common.cuh"

using namespace hbp;

namespace {

constexpr int kSpmvThreads = 256;
constexpr int kSpmvWarps = kSpmvThreads / 32;

template <typename V, bool EXACT>
__device__ __forceinline__ double fmadd(double acc, V v, V xv) {
    if (EXACT) return __dadd_rn(acc, __dmul_rn((double)v, (double)xv));
    return fma((double)v, (double)xv, acc);  // exact product for f32 inputs
}

// Sum of one slot's elements in step order.  All segment lanes must call it.
template <typename V, bool EXACT, int U = 4>
__device__ __forceinline__ double group_dot(const Seg &sg, const uint32_t *__restrict__ col,
                                            const V *__restrict__ data,
                                            const V *__restrict__ x, uint32_t len,
                                            int64_t base, uint64_t pe, uint64_t pl) {
    const unsigned lt = (1u << sg.q) - 1u;
    double acc = 0.0;
    uint32_t t0 = 0;
    bool live = len > 0;
    unsigned mask = seg_ballot(sg, live);
    while (mask) {
        const int k = __popc(mask);
        const uint32_t t1 = seg_min_u32(sg, live ? len : 0xffffffffu);
        if (live) {
            const int rank = __popc(mask & lt);
            const uint32_t *cp = col + base + rank;
            const V *dp = data + base + rank;
            const uint32_t M = t1 - t0;
            uint32_t t = 0;
            for (; U == 4 && t + 4 <= M; t += 4) {
                uint32_t c0 = ld_stream_u32(cp, pe), c1 = ld_stream_u32(cp + k, pe),
                         c2 = ld_stream_u32(cp + 2 * k, pe), c3 = ld_stream_u32(cp + 3 * k, pe);
                V v0 = ld_stream(dp, pe), v1 = ld_stream(dp + k, pe), v2 = ld_stream(dp + 2 * k, pe),
                  v3 = ld_stream(dp + 3 * k, pe);
                V x0 = ld_x(x + c0, pl), x1 = ld_x(x + c1, pl), x2 = ld_x(x + c2, pl), x3 = ld_x(x + c3, pl);
                acc = fmadd<V, EXACT>(acc, v0, x0);
                acc = fmadd<V, EXACT>(acc, v1, x1);
                acc = fmadd<V, EXACT>(acc, v2, x2);
                acc = fmadd<V, EXACT>(acc, v3, x3);
                cp += 4 * k;
                dp += 4 * k;
            }
            for (; U == 2 && t + 2 <= M; t += 2) {
                uint32_t c0 = ld_stream_u32(cp, pe), c1 = ld_stream_u32(cp + k, pe);
                V v0 = ld_stream(dp, pe), v1 = ld_stream(dp + k, pe);
                V x0 = ld_x(x + c0, pl), x1 = ld_x(x + c1, pl);
                acc = fmadd<V, EXACT>(acc, v0, x0);
                acc = fmadd<V, EXACT>(acc, v1, x1);
                cp += 2 * k;
                dp += 2 * k;
            }
            for (; t < M; ++t) {
                uint32_t c0 = ld_stream_u32(cp, pe);
                V v0 = ld_stream(dp, pe);
                acc = fmadd<V, EXACT>(acc, v0, ld_x(x + c0, pl));
                cp += k;
                dp += k;
            }
        }
        base += (int64_t)(t1 - t0) * k;
        t0 = t1;
        live = len > t0;
        mask = seg_ballot(sg, live);
    }
    return acc;
}

template <typename V, bool EXACT, bool DIRECT, bool LOG>
__global__ void __launch_bounds__(kSpmvThreads)
    k_spmv(const hbp_format_t f, const hbp_schedule_t sch, const V *__restrict__ x,
           double *__restrict__ partial, V *__restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int64_t worker = (int64_t)blockIdx.x * kSpmvWarps + (threadIdx.x >> 5);
    if (worker >= sch.workers) return;  // whole warps exit together
    const Seg sg = make_seg((int)f.warp_size);
    const int64_t R = f.row_height, W = f.warp_size, gpb = R / W;
    const V *__restrict__ data = (const V *)f.data;
    const uint64_t pe = policy_evict_first(), pl = policy_evict_last();

    auto run_block = [&](int64_t idx, int8_t kind) {
        int64_t t_start = 0;
        if (LOG && lane == 0) t_start = globaltimer_ns();
        const int64_t br = f.blk_br[idx];
        int64_t n = f.rows - br * R;
        if (n > R) n = R;
        const int64_t ng = (n + W - 1) / W;
        if (!sg.idle()) {
            for (int64_t g = sg.seg; g < ng; g += sg.spw) {
                const int64_t slot = g * W + sg.q;
                const bool valid = slot < n;
                const uint32_t len = valid ? f.slot_len[idx * R + slot] : 0u;
                const double acc = group_dot<V, EXACT>(sg, f.col, data, x, len,
                                                       f.group_start[idx * gpb + g], pe, pl);
                if (valid) {
                    const uint32_t row = f.perm[idx * R + slot];
                    if (DIRECT) y[br * R + row] = (V)acc;
                    else partial[idx * R + row] = acc;
                }
            }
        }
        __syncwarp();
        if (LOG && lane == 0) {
            sch.log_start_ns[idx] = t_start;
            sch.log_end_ns[idx] = globaltimer_ns();
            sch.log_worker[idx] = (int32_t)worker;
            sch.log_kind[idx] = kind;
        }
    };

    // engine.py:107-115: contiguous chunks, the first `rem` one block longer
    const int64_t per = sch.fixed_count / sch.workers, rem = sch.fixed_count % sch.workers;
    const int64_t lo = worker * per + (worker < rem ? worker : rem);
    const int64_t hi = lo + per + (worker < rem ? 1 : 0);
    for (int64_t idx = lo; idx < hi; ++idx) run_block(idx, 0);
    // engine.py:159-165: ticket acquisition over [fixed_count, nzb)
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(sch.ticket, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        const int64_t idx = sch.fixed_count + (int64_t)t;
        if (idx >= f.nzb) break;
        run_block(idx, 1);
    }
}

// Row-block-owner schedule (small matrices with several column blocks): one
// CTA (8 warps) per row block computes the block partials of its nonzero blocks into
// shared memory -- up to `kmax` blocks at once, one (block, group) task per
// warp segment, so the blocks' load chains overlap -- and folds them in
// ascending bc exactly as combine does (engine.py:196-201: s = p_first;
// s += p_next ...), carrying the running sum across chunks of kmax blocks.
// The per-slot sums are k_spmv's (group_dot), so results are bitwise those
// of hbp_spmv_blocks + hbp_combine, without the partial array, the combine
// launch or the empty-row pass.
constexpr int kRowThreadsMax = 512;
constexpr int64_t kRowSmem = 48 * 1024;                  // no opt-in needed
constexpr int64_t kRowBlockMaxR = kRowSmem / 16;         // kmax >= 1 plus the running sum

template <typename V, bool EXACT, int NT, int MINB, int U>
__global__ void __launch_bounds__(NT, MINB)
    k_spmv_rowblock(const hbp_format_t f, const V *__restrict__ x, V *__restrict__ y, int kmax) {
    extern __shared__ double sm[];  // pl[kmax][R], then the running sum ys[R]
    const Seg sg = make_seg((int)f.warp_size);
    const int64_t R = f.row_height, W = f.warp_size, gpb = R / W;
    const int64_t nrb = (f.rows + R - 1) / R;
    double *ys = sm + (int64_t)kmax * R;
    const V *__restrict__ data = (const V *)f.data;
    const uint64_t pe = policy_evict_first(), pl = policy_evict_last();
    const int seg0 = (threadIdx.x >> 5) * sg.spw + sg.seg;
    const int nseg = (blockDim.x >> 5) * sg.spw;
    for (int64_t br = blockIdx.x; br < nrb; br += gridDim.x) {
        const int64_t lo = f.rb_ptr[br], hi = f.rb_ptr[br + 1];
        int64_t n64 = f.rows - br * R;
        const int n = (int)(n64 > R ? R : n64);
        const int ng = (int)((n + W - 1) / W);
        V *yb = y + br * R;
        if (lo == hi) {
            for (int r = threadIdx.x; r < n; r += blockDim.x) yb[r] = (V)0;
            continue;
        }
        for (int64_t c0 = lo; c0 < hi; c0 += kmax) {
            const int cnt = (int)(hi - c0 < kmax ? hi - c0 : kmax);
            if (!sg.idle()) {
                for (int t = seg0; t < cnt * ng; t += nseg) {
                    const int j = t / ng, g = t - j * ng;
                    const int64_t idx = f.rb_blk[c0 + j];
                    const int slot = g * (int)W + sg.q;
                    const bool valid = slot < n;
                    const uint32_t len = valid ? f.slot_len[idx * R + slot] : 0u;
                    const uint32_t row = valid ? f.perm[idx * R + slot] : 0u;
                    const int64_t gs = f.group_start[idx * gpb + g];
                    const double acc = group_dot<V, EXACT, U>(sg, f.col, data, x, len, gs, pe, pl);
                    if (valid) sm[(int64_t)j * R + row] = acc;
                }
            }
            __syncthreads();
            const bool last = c0 + kmax >= hi;
            for (int r = threadIdx.x; r < n; r += blockDim.x) {
                double v = c0 == lo ? sm[r] : __dadd_rn(ys[r], sm[r]);
                for (int j = 1; j < cnt; ++j) v = __dadd_rn(v, sm[(int64_t)j * R + r]);
                if (last) yb[r] = (V)v;
                else ys[r] = v;
            }
            __syncthreads();
        }
    }
}

// combine over nonzero blocks, ascending bc (engine.py:196-201).  Each warp
// scans 32 row blocks with one coalesced rb_ptr load and a ballot, skips the
// single-block row blocks the SpMV kernel wrote itself, and sums the rows of
// the others four rows per lane at a time (independent loads in flight).  No
// per-row 64-bit division remains: the earlier thread-per-row form spent
// 112 us of cfg3's 2.7 ms step on divisions and rb_ptr chains.
template <typename V>
__device__ __forceinline__ double combine_row(const hbp_format_t &f,
                                              const double *__restrict__ partial, int64_t lo,
                                              int64_t hi, int64_t R, int64_t local) {
    double s = 0.0;
    if (lo < hi) {
        // the reference's left-to-right sum
        s = partial[(int64_t)f.rb_blk[lo] * R + local];
        int64_t i = lo + 1;
        for (; i + 4 <= hi; i += 4) {
            const int32_t b0 = f.rb_blk[i], b1 = f.rb_blk[i + 1], b2 = f.rb_blk[i + 2],
                          b3 = f.rb_blk[i + 3];
            const double p0 = partial[(int64_t)b0 * R + local];
            const double p1 = partial[(int64_t)b1 * R + local];
            const double p2 = partial[(int64_t)b2 * R + local];
            const double p3 = partial[(int64_t)b3 * R + local];
            s = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(s, p0), p1), p2), p3);
        }
        for (; i < hi; ++i) s = __dadd_rn(s, partial[(int64_t)f.rb_blk[i] * R + local]);
    }
    return s;
}

template <typename V>
__global__ void k_combine(const hbp_format_t f, const double *__restrict__ partial,
                          V *__restrict__ y, int64_t nrb) {
    const int64_t R = f.row_height;
    const bool skip_single = (f.reserved & HBP_FLAG_DIRECT_SINGLE) != 0;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nseg = (R + 127) / 128;  // 128-row segments: one warp task each
    const int64_t ntask = (nrb + 31) / 32 * nseg;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntask;
         t += nwarps) {
        const int64_t c = t / nseg, seg = t - c * nseg;
        const int64_t br = c * 32 + lane;
        int64_t lo = 0, hi = 0;
        bool need = false;
        if (br < nrb) {
            lo = f.rb_ptr[br];
            hi = f.rb_ptr[br + 1];
            need = !(skip_single && hi - lo == 1);
        }
        unsigned mask = __ballot_sync(0xffffffffu, need);
        while (mask) {
            const int b = __ffs(mask) - 1;
            mask &= mask - 1;
            const int64_t rb = c * 32 + b;
            const int64_t blo = __shfl_sync(0xffffffffu, lo, b);
            const int64_t bhi = __shfl_sync(0xffffffffu, hi, b);
            int64_t n = f.rows - rb * R;
            if (n > R) n = R;
            if (n > (seg + 1) * 128) n = (seg + 1) * 128;
            V *yb = y + rb * R;
            int64_t local = seg * 128 + lane;
            if (local + 96 < n) {
                const double s0 = combine_row<V>(f, partial, blo, bhi, R, local);
                const double s1 = combine_row<V>(f, partial, blo, bhi, R, local + 32);
                const double s2 = combine_row<V>(f, partial, blo, bhi, R, local + 64);
                const double s3 = combine_row<V>(f, partial, blo, bhi, R, local + 96);
                yb[local] = (V)s0;
                yb[local + 32] = (V)s1;
                yb[local + 64] = (V)s2;
                yb[local + 96] = (V)s3;
                local += 128;
            }
            for (; local < n; local += 32) yb[local] = (V)combine_row<V>(f, partial, blo, bhi, R, local);
        }
    }
}

// Row-block-parallel combine for matrices with many nonzero blocks per row
// block (few row blocks, many column blocks): the scan above gives each warp
// 32 row blocks in series, so with nrb = 512 only 64 warps would run.  Here
// one warp task = (row block, 32-row segment), a lane per row, summed in
// ascending bc by combine_row (bitwise the same).
template <typename V>
__global__ void k_combine_rows(const hbp_format_t f, const double *__restrict__ partial,
                               V *__restrict__ y, int64_t nrb) {
    const int64_t R = f.row_height;
    const bool skip_single = (f.reserved & HBP_FLAG_DIRECT_SINGLE) != 0;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nseg = (R + 31) / 32;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < nrb * nseg;
         t += nwarps) {
        const int64_t rb = t / nseg, seg = t - rb * nseg;
        const int64_t lo = f.rb_ptr[rb], hi = f.rb_ptr[rb + 1];
        if (skip_single && hi - lo == 1) continue;
        int64_t n = f.rows - rb * R;
        if (n > R) n = R;
        const int64_t local = seg * 32 + lane;
        if (local < n) y[rb * R + local] = (V)combine_row<V>(f, partial, lo, hi, R, local);
    }
}

template <typename V>
__global__ void k_zero_empty(const hbp_format_t f, V *__restrict__ y, int64_t nrb) {
    // same warp scan as k_combine: one rb_ptr load + ballot per 32 row blocks
    const int64_t R = f.row_height;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c * 32 < nrb;
         c += nwarps) {
        const int64_t br = c * 32 + lane;
        const bool empty = br < nrb && f.rb_ptr[br] == f.rb_ptr[br + 1];
        unsigned mask = __ballot_sync(0xffffffffu, empty);
        while (mask) {
            const int b = __ffs(mask) - 1;
            mask &= mask - 1;
            const int64_t rb = c * 32 + b;
            int64_t n = f.rows - rb * R;
            if (n > R) n = R;
            for (int64_t local = lane; local < n; local += 32) y[rb * R + local] = (V)0;
        }
    }
}

__global__ void k_expand_partial(const hbp_format_t f, const double *__restrict__ partial,
                                 double *__restrict__ dense) {
    const int64_t R = f.row_height;
    const int64_t total = f.nzb * R;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t blk = i / R, s = i - blk * R;
        const int64_t br = f.blk_br[blk];
        if (br * R + s >= f.rows) continue;
        dense[(int64_t)f.blk_bc[blk] * f.rows + br * R + s] = partial[i];
    }
}

// hbp.py:241-315: every element's (row, col, value), by position.
template <typename V>
__global__ void k_to_triplets(const hbp_format_t f, int64_t *__restrict__ row_out,
                              int64_t *__restrict__ col_out, V *__restrict__ val_out) {
    const Seg sg = make_seg((int)f.warp_size);
    if (sg.idle()) return;
    const int64_t R = f.row_height, W = f.warp_size, gpb = R / W;
    const int64_t ngroups = f.nzb * gpb;
    const unsigned lt = (1u << sg.q) - 1u;
    const V *data = (const V *)f.data;
    int64_t seg_id = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * sg.spw + sg.seg;
    int64_t nseg = (((int64_t)gridDim.x * blockDim.x) >> 5) * sg.spw;
    for (int64_t gg = seg_id; gg < ngroups; gg += nseg) {
        const int64_t blk = gg / gpb, g = gg - blk * gpb;
        const int64_t slot = blk * R + g * W + sg.q;
        const uint32_t len = f.slot_len[slot];
        const int64_t row = (int64_t)f.blk_br[blk] * R + (len ? f.perm[slot] : 0);
        int64_t base = f.group_start[gg];
        uint32_t t0 = 0;
        bool live = len > 0;
        unsigned mask = seg_ballot(sg, live);
        while (mask) {
            const int k = __popc(mask);
            const uint32_t t1 = seg_min_u32(sg, live ? len : 0xffffffffu);
            if (live) {
                int64_t p = base + __popc(mask & lt);
                for (uint32_t t = t0; t < t1; ++t, p += k) {
                    row_out[p] = row;
                    col_out[p] = f.col[p];
                    val_out[p] = data[p];
                }
            }
            base += (int64_t)(t1 - t0) * k;
            t0 = t1;
            live = len > t0;
            mask = seg_ballot(sg, live);
        }
    }
}

template <typename V, bool EXACT, bool DIRECT, bool LOG>
void launch_spmv(const hbp_format_t *f, const hbp_schedule_t *s, const void *x, double *partial,
                 void *y, cudaStream_t st) {
    unsigned grid = (unsigned)((s->workers + kSpmvWarps - 1) / kSpmvWarps);
    k_spmv<V, EXACT, DIRECT, LOG><<<grid, kSpmvThreads, 0, st>>>(*f, *s, (const V *)x, partial,
                                                                 (V *)y);
}

template <typename V, bool EXACT>
void dispatch_spmv(const hbp_format_t *f, const hbp_schedule_t *s, const void *x,
                   double *partial, void *y, cudaStream_t st) {
    const bool direct = y != nullptr, log = s->log_worker != nullptr;
    if (direct) {
        if (log) launch_spmv<V, EXACT, true, true>(f, s, x, partial, y, st);
        else launch_spmv<V, EXACT, true, false>(f, s, x, partial, y, st);
    } else {
        if (log) launch_spmv<V, EXACT, false, true>(f, s, x, partial, y, st);
        else launch_spmv<V, EXACT, false, false>(f, s, x, partial, y, st);
    }
}

// engine.py:196-201 combine over a caller-made dense PartialVector
// [ncb][rows] (reference layout): y = seg0; y += seg_bc, ascending bc.
__global__ void k_combine_dense(const double *__restrict__ p, int64_t rows, int64_t ncb,
                                double *__restrict__ y) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        double s = p[r];
        for (int64_t bc = 1; bc < ncb; ++bc) s = __dadd_rn(s, p[bc * rows + r]);
        y[r] = s;
    }
}

}  // namespace

extern "C" {

int hbp_spmv_default_workers(int dtype, int64_t warp_size, int64_t *workers) {
    int dev = 0, sms = 0, per_sm = 0;
    HBP_CUDA_TRY(cudaGetDevice(&dev));
    HBP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (dtype == HBP_F64)
        HBP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, k_spmv<double, true, true, false>, kSpmvThreads, 0));
    else
        HBP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, k_spmv<float, false, true, false>, kSpmvThreads, 0));
    (void)warp_size;
    *workers = (int64_t)sms * per_sm * kSpmvWarps;
    return HBP_OK;
}

int hbp_spmv_blocks(const hbp_format_t *f, const hbp_schedule_t *s, const void *x,
                    double *partial, void *y_direct, hbp_stream_t stream) {
    if (!f || !s || s->workers < 1) return HBP_E_ARG;
    if (f->warp_size < 1 || f->warp_size > 32 || f->row_height % f->warp_size)
        return HBP_E_UNSUPPORTED;
    if (y_direct && f->ncb != 1) return HBP_E_ARG;
    cudaStream_t st = as_stream(stream);
    HBP_CUDA_TRY(cudaMemsetAsync(s->ticket, 0, sizeof(uint32_t), st));
    if (f->nzb == 0) return HBP_OK;
    if (!y_direct && !partial) return HBP_E_ARG;
    if (f->dtype == HBP_F64) dispatch_spmv<double, true>(f, s, x, partial, y_direct, st);
    else if (f->dtype == HBP_F32) dispatch_spmv<float, false>(f, s, x, partial, y_direct, st);
    else return HBP_E_ARG;
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_spmv_rowblock(const hbp_format_t *f, const void *x, void *y, hbp_stream_t stream) {
    if (!f || f->rows < 0 || (f->rows > 0 && !y)) return HBP_E_ARG;
    if (f->warp_size < 1 || f->warp_size > 32 || f->row_height % f->warp_size ||
        f->row_height > kRowBlockMaxR)
        return HBP_E_UNSUPPORTED;
    if (f->rows == 0) return HBP_OK;
    if (f->nzb > 0 && !x) return HBP_E_ARG;
    const int64_t R = f->row_height, spw = 32 / f->warp_size;
    const int64_t warps = (R / f->warp_size + spw - 1) / spw;
    const int64_t nrb = (f->rows + R - 1) / R;
    const unsigned grid = (unsigned)(nrb < (1 << 30) ? nrb : (1 << 30));
    cudaStream_t st = as_stream(stream);
    if (f->dtype != HBP_F64 && f->dtype != HBP_F32) return HBP_E_ARG;
    static const int variant =  // tuning A/B only
        getenv("HBP_ROWBLOCK_VARIANT") ? atoi(getenv("HBP_ROWBLOCK_VARIANT")) : 0;
    const int nt = variant == 1 || variant == 2 ? kRowThreadsMax : variant == 3 ? 128 : 256;
    const int kcap = variant == 1 || variant == 2 ? 8 : variant == 3 ? 2 : 4;
    const int threads = (int)(warps * 32 < nt ? warps * 32 : nt);
    int kmax = (int)(kRowSmem / (8 * R)) - 1;
    if (kmax > kcap) kmax = kcap;
    const size_t smem = sizeof(double) * (size_t)R * (size_t)(kmax + 1);
#define HBP_RB_LAUNCH(NT, MINB, U)                                                                    \
    do {                                                                                         \
        if (f->dtype == HBP_F64)                                                                 \
            k_spmv_rowblock<double, true, NT, MINB, U><<<grid, threads, smem, st>>>(                 \
                *f, (const double *)x, (double *)y, kmax);                                       \
        else                                                                                     \
            k_spmv_rowblock<float, false, NT, MINB, U><<<grid, threads, smem, st>>>(                 \
                *f, (const float *)x, (float *)y, kmax);                                         \
    } while (0)
    // cfg1 (same box, L2 flushed, tools/prof_spmv.py --flush): 8 CTAs x 8 warps
    // x 32 regs, two-step unroll, 4 blocks per chunk 37.6 us; 16 x 4 warps 38.1;
    // 4 x 16 warps 41.6 (warps idle at the barrier when a row block has 1.5
    // blocks x 16 groups); 3 x 16 warps x 40 regs 48.6 (unroll 4) / 49.8
    // (unroll 2) / 48.4 us (no unroll); 2 x 16 x 64 regs 53.6 us.  A
    // step-batched walk (positions of 4 or 8 steps from per-step ballots, then
    // all loads) was slower: 51.6 / 66 us.
    // f32 spills 68 B at 32 registers; 4 CTAs x 64 registers (no spill) is
    // slower where the auto schedule picks this kernel (banded 35M / 138M nnz:
    // 0.106 / 0.349 vs 0.102 / 0.320 ms), so both dtypes use 8 x 32.
    if (variant == 1) HBP_RB_LAUNCH(512, 3, 4);
    else if (variant == 2) HBP_RB_LAUNCH(512, 4, 2);
    else if (variant == 3) HBP_RB_LAUNCH(128, 16, 2);
    else HBP_RB_LAUNCH(256, 8, 2);
#undef HBP_RB_LAUNCH
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_combine(const hbp_format_t *f, const double *partial, void *y, hbp_stream_t stream) {
    if (!f || f->rows < 1) return HBP_E_ARG;
    cudaStream_t st = as_stream(stream);
    if (f->row_height < 1) return HBP_E_ARG;
    const int64_t nrb = (f->rows + f->row_height - 1) / f->row_height;
    int dev = 0, sms = 0;
    HBP_CUDA_TRY(cudaGetDevice(&dev));
    HBP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // one warp per (32 row blocks, 128-row segment), at most 64 warps per SM
    const int64_t warps = (nrb + 31) / 32 * ((f->row_height + 127) / 128),
                  cap = (int64_t)sms * 8 * 8;
    const int threads = 256;
    if (f->nzb >= 4 * nrb) {  // many blocks per row block: a task per (row block, 32 rows)
        const int64_t tasks = nrb * ((f->row_height + 31) / 32);
        const unsigned g2 = (unsigned)(((tasks < cap ? tasks : cap) + 7) / 8);
        if (f->dtype == HBP_F64)
            k_combine_rows<double><<<g2, threads, 0, st>>>(*f, partial, (double *)y, nrb);
        else if (f->dtype == HBP_F32)
            k_combine_rows<float><<<g2, threads, 0, st>>>(*f, partial, (float *)y, nrb);
        else return HBP_E_ARG;
        HBP_LAUNCH_CHECK();
        return HBP_OK;
    }
    const unsigned grid = (unsigned)(((warps < cap ? warps : cap) + 7) / 8);
    if (f->dtype == HBP_F64)
        k_combine<double><<<grid, threads, 0, st>>>(*f, partial, (double *)y, nrb);
    else if (f->dtype == HBP_F32)
        k_combine<float><<<grid, threads, 0, st>>>(*f, partial, (float *)y, nrb);
    else return HBP_E_ARG;
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_combine_dense(const double *partial, int64_t rows, int64_t ncb, double *y,
                      hbp_stream_t stream) {
    if (rows < 0 || ncb < 1) return HBP_E_ARG;
    if (rows == 0) return HBP_OK;
    k_combine_dense<<<grid_for(rows, 256), 256, 0, as_stream(stream)>>>(partial, rows, ncb, y);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_zero_empty_rows(const hbp_format_t *f, void *y, hbp_stream_t stream) {
    if (!f || f->rows < 1) return HBP_E_ARG;
    cudaStream_t st = as_stream(stream);
    if (f->row_height < 1) return HBP_E_ARG;
    const int64_t nrb = (f->rows + f->row_height - 1) / f->row_height;
    const unsigned grid = grid_for((nrb + 31) / 32 * 32, 256);
    if (f->dtype == HBP_F64) k_zero_empty<double><<<grid, 256, 0, st>>>(*f, (double *)y, nrb);
    else if (f->dtype == HBP_F32) k_zero_empty<float><<<grid, 256, 0, st>>>(*f, (float *)y, nrb);
    else return HBP_E_ARG;
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_expand_partial(const hbp_format_t *f, const double *partial, double *partial_dense,
                       hbp_stream_t stream) {
    if (!f) return HBP_E_ARG;
    cudaStream_t st = as_stream(stream);
    HBP_CUDA_TRY(cudaMemsetAsync(partial_dense, 0, sizeof(double) * (size_t)(f->ncb * f->rows), st));
    if (f->nzb == 0) return HBP_OK;
    k_expand_partial<<<grid_for(f->nzb * f->row_height, 256), 256, 0, st>>>(*f, partial,
                                                                           partial_dense);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_to_triplets(const hbp_format_t *f, int64_t *row_out, int64_t *col_out, void *val_out,
                    hbp_stream_t stream) {
    if (!f || f->warp_size < 1 || f->warp_size > 32) return HBP_E_ARG;
    if (f->nzb == 0) return HBP_OK;
    cudaStream_t st = as_stream(stream);
    int64_t spw = 32 / f->warp_size;
    int64_t warps = (f->nzb * (f->row_height / f->warp_size) + spw - 1) / spw;
    unsigned grid = grid_for(warps * 32, 256);
    if (f->dtype == HBP_F64)
        k_to_triplets<double><<<grid, 256, 0, st>>>(*f, row_out, col_out, (double *)val_out);
    else
        k_to_triplets<float><<<grid, 256, 0, st>>>(*f, row_out, col_out, (float *)val_out);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

}  // extern "C"
