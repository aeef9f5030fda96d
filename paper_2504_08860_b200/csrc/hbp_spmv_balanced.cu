// hbp_spmv_balanced.cu -- element-balanced HBP SpMV for B200 (W = 32).
//
// The reference's scheduler (engine.py:96-176) balances BLOCKS (fixed chunks
// + a ticket); on skewed matrices (R-MAT: rows of 10^5 nonzeros) one block,
// one group, even one row can exceed the whole SpMV's budget when a single
// warp walks it.  This kernel keeps the HBP format and per-row arithmetic
// but partitions the ELEMENT array [0, nnz) into equal contiguous ranges, one
// per persistent warp:
//
//   * exact mode (f64, bitwise with the reference): every cut is rounded up
//     to a group boundary, so each row is summed by one lane in step order;
//   * fast mode (f32 values, f64 accumulation): cuts are rounded up to a STEP
//     boundary inside a group; a group split over several warps leaves one
//     per-lane partial per piece, and the warp that completes the group's
//     element count (atomic, last arriver) adds the pieces in warp order --
//     deterministic, one rounding to f32 at the end.
//
// Inside a piece the lane-serial phases of hbp_spmv.cu are used while many
// lanes are live; phases with few live lanes over many steps (the tails of
// hot rows) are read cooperatively: S = 32/k sub-streams per live lane, so
// every warp load is 32 consecutive elements.
//
// Group g of the compact layout owns slots [g*32, g*32+32) (R = gpb*32), and
// E_g(t) = sum over lanes of min(len, t) is one warp reduction, which makes
// step <-> element-offset conversion a short binary search.
#include <cuda_runtime.h>
#include <stdint.h>

#include "hbp.h"
#include "hbp_common.cuh"

using namespace hbp;

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr unsigned FULL = 0xffffffffu;

template <typename V, bool EXACT>
__device__ __forceinline__ double fma_acc(double acc, V v, V xv) {
    if (EXACT) return __dadd_rn(acc, __dmul_rn((double)v, (double)xv));
    return fma((double)v, (double)xv, acc);
}

// largest g in [0, n] with gs[g] <= e
__device__ __forceinline__ int64_t upper_group(const int64_t *__restrict__ gs, int64_t n,
                                               int64_t e) {
    int64_t lo = 0, hi = n + 1;  // answer in [0, n]
    while (hi - lo > 1) {
        int64_t m = (lo + hi) >> 1;
        if (gs[m] <= e) lo = m;
        else hi = m;
    }
    return lo;
}

// smallest g in [0, n] with gs[g] >= e
__device__ __forceinline__ int64_t lower_group(const int64_t *__restrict__ gs, int64_t n,
                                               int64_t e) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t m = (lo + hi) >> 1;
        if (gs[m] < e) lo = m + 1;
        else hi = m;
    }
    return lo;
}

// elements of the group before step t
__device__ __forceinline__ uint32_t elems_before(uint32_t len, uint32_t t) {
    return __reduce_add_sync(FULL, len < t ? len : t);
}

// smallest step t with E(t) >= o  (o <= E(maxlen))
__device__ __forceinline__ uint32_t step_at(uint32_t len, uint32_t o) {
    uint32_t hi = __reduce_max_sync(FULL, len), lo = 0;
    while (lo < hi) {
        uint32_t m = lo + ((hi - lo) >> 1);
        if (elems_before(len, m) >= o) hi = m;
        else lo = m + 1;
    }
    return lo;
}

// Rounds an element offset up to the cut the balanced schedule uses.
template <bool EXACT>
__device__ __forceinline__ int64_t snap_cut(const hbp_format_t &f, int64_t ngroups, int64_t e) {
    if (e <= 0) return 0;
    if (e >= f.nnz) return f.nnz;
    const int64_t *gs = f.group_start;
    int64_t g = upper_group(gs, ngroups, e);
    int64_t g0 = gs[g];
    if (g0 == e) return e;
    if (EXACT) return gs[g + 1];
    uint32_t len = ((const uint32_t *)f.slot_len)[g * 32 + (threadIdx.x & 31)];
    uint32_t t = step_at(len, (uint32_t)(e - g0));
    return g0 + elems_before(len, t);
}

// Sum of this lane's row over steps [ta, tb) of its group; base = position of step ta.
template <typename V, bool EXACT>
__device__ __forceinline__ double piece_dot(const uint32_t *__restrict__ col,
                                            const V *__restrict__ data, const V *__restrict__ x,
                                            uint32_t len, int64_t base, uint32_t ta, uint32_t tb,
                                            uint64_t pe, uint64_t pl) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    double acc = 0.0;
    uint32_t t0 = ta;
    bool live = len > t0;
    unsigned mask = __ballot_sync(FULL, live);
    while (mask && t0 < tb) {
        const int k = __popc(mask);
        uint32_t t1 = __reduce_min_sync(FULL, live ? len : 0xffffffffu);
        if (t1 > tb) t1 = tb;
        const uint32_t M = t1 - t0;
        const int rank = __popc(mask & lt);
        if (EXACT || k >= 12 || M < 8) {
            if (live) {
                const uint32_t *cp = col + base + rank;
                const V *dp = data + base + rank;
                uint32_t t = 0;
                for (; t + 4 <= M; t += 4) {
                    uint32_t c0 = ld_stream_u32(cp, pe), c1 = ld_stream_u32(cp + k, pe),
                             c2 = ld_stream_u32(cp + 2 * k, pe),
                             c3 = ld_stream_u32(cp + 3 * k, pe);
                    V v0 = ld_stream(dp, pe), v1 = ld_stream(dp + k, pe),
                      v2 = ld_stream(dp + 2 * k, pe), v3 = ld_stream(dp + 3 * k, pe);
                    V x0 = ld_x(x + c0, pl), x1 = ld_x(x + c1, pl), x2 = ld_x(x + c2, pl),
                      x3 = ld_x(x + c3, pl);
                    acc = fma_acc<V, EXACT>(acc, v0, x0);
                    acc = fma_acc<V, EXACT>(acc, v1, x1);
                    acc = fma_acc<V, EXACT>(acc, v2, x2);
                    acc = fma_acc<V, EXACT>(acc, v3, x3);
                    cp += 4 * k;
                    dp += 4 * k;
                }
                for (; t < M; ++t) {
                    uint32_t c0 = ld_stream_u32(cp, pe);
                    acc = fma_acc<V, EXACT>(acc, ld_stream(dp, pe), ld_x(x + c0, pl));
                    cp += k;
                    dp += k;
                }
            }
        } else {
            // few live lanes, many steps: S sub-streams per live lane
            int S = 32 / k;
            S = 1 << (31 - __clz(S));  // power of two, k*S <= 32
            const int r = lane % k, s = lane / k;
            double v = 0.0;
            if (s < S) {
                const int64_t stride = (int64_t)S * k;
                const uint32_t *cp = col + base + (int64_t)s * k + r;
                const V *dp = data + base + (int64_t)s * k + r;
                uint32_t t = s;
                for (; t + 3 * S < M; t += 4 * S) {
                    uint32_t c0 = ld_stream_u32(cp, pe), c1 = ld_stream_u32(cp + stride, pe),
                             c2 = ld_stream_u32(cp + 2 * stride, pe),
                             c3 = ld_stream_u32(cp + 3 * stride, pe);
                    V v0 = ld_stream(dp, pe), v1 = ld_stream(dp + stride, pe),
                      v2 = ld_stream(dp + 2 * stride, pe), v3 = ld_stream(dp + 3 * stride, pe);
                    V x0 = ld_x(x + c0, pl), x1 = ld_x(x + c1, pl), x2 = ld_x(x + c2, pl),
                      x3 = ld_x(x + c3, pl);
                    v = fma_acc<V, false>(v, v0, x0);
                    v = fma_acc<V, false>(v, v1, x1);
                    v = fma_acc<V, false>(v, v2, x2);
                    v = fma_acc<V, false>(v, v3, x3);
                    cp += 4 * stride;
                    dp += 4 * stride;
                }
                for (; t < M; t += S) {
                    uint32_t c0 = ld_stream_u32(cp, pe);
                    v = fma_acc<V, false>(v, ld_stream(dp, pe), ld_x(x + c0, pl));
                    cp += stride;
                    dp += stride;
                }
            }
            for (int off = S >> 1; off >= 1; off >>= 1) v += __shfl_down_sync(FULL, v, off * k);
            const double tot = __shfl_sync(FULL, v, live ? rank : 0);
            if (live) acc += tot;
        }
        base += (int64_t)M * k;
        t0 = t1;
        live = len > t0;
        mask = __ballot_sync(FULL, live);
    }
    return acc;
}

template <typename V, bool EXACT>
__global__ void __launch_bounds__(kThreads)
    k_spmv_balanced(const hbp_format_t f, const hbp_balanced_t b, const V *__restrict__ x,
                    V *__restrict__ y, double *__restrict__ partial) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int64_t Nw = b.workers;
    if (w >= Nw) return;
    const int64_t R = f.row_height, gpb = R / 32;
    const int64_t ngroups = f.nzb * gpb;
    const int64_t E = f.nnz;
    const int64_t *__restrict__ gs = f.group_start;
    const uint32_t *__restrict__ slot_len = (const uint32_t *)f.slot_len;
    const uint32_t *__restrict__ perm = (const uint32_t *)f.perm;
    const V *__restrict__ data = (const V *)f.data;
    const uint64_t pe = policy_evict_first(), pl = policy_evict_last();

    const int64_t c_lo = snap_cut<EXACT>(f, ngroups, (int64_t)((__int128)w * E / Nw));
    const int64_t c_hi = snap_cut<EXACT>(f, ngroups, (int64_t)((__int128)(w + 1) * E / Nw));
    if (!EXACT && lane == 0) b.cut_end[w] = c_hi;

    int64_t g = upper_group(gs, ngroups, c_lo);  // gs[g] <= c_lo < gs[g+1] when g < ngroups
    if (!(g < ngroups && gs[g] < c_lo)) g = lower_group(gs, ngroups, c_lo);
    const bool last_warp = (w == Nw - 1);
    for (; g < ngroups && (gs[g] < c_hi || last_warp); ++g) {
        const int64_t g0 = gs[g], g1 = gs[g + 1];
        const int64_t ea = g0 > c_lo ? g0 : c_lo;
        const int64_t eb = g1 < c_hi ? g1 : c_hi;
        const bool full = (ea == g0) && (eb == g1);
        const uint32_t len = slot_len[g * 32 + lane];
        const uint32_t ta = (ea == g0) ? 0u : step_at(len, (uint32_t)(ea - g0));
        const uint32_t tb = (eb == g1) ? 0xffffffffu : step_at(len, (uint32_t)(eb - g0));
        const double acc = piece_dot<V, EXACT>(f.col, data, x, len, ea, ta, tb, pe, pl);

        const int64_t blk = g / gpb;
        const int64_t local = (g - blk * gpb) * 32 + lane;
        const int64_t br = f.blk_br[blk];
        const bool valid = local < f.rows - br * R;
        if (full) {
            if (valid) {
                const uint32_t row = perm[g * 32 + lane];
                if (partial) partial[blk * R + row] = acc;
                else y[br * R + row] = (V)acc;
            }
            continue;
        }
        if (EXACT) continue;  // unreachable: exact cuts never split a group
        // piece of a split group: publish, then the last arriver combines
        double *slotp = (ea > g0) ? b.part_head + w * 32 : b.part_tail + w * 32;
        __stcg(slotp + lane, acc);
        __threadfence();
        __syncwarp();
        uint32_t done = 0;
        if (lane == 0) {
            const uint32_t n = (uint32_t)(eb - ea);
            const uint32_t old = atomicAdd(b.counters + g, n);
            done = (old + n == (uint32_t)(g1 - g0));
        }
        done = __shfl_sync(FULL, done, 0);
        if (!done) continue;
        __threadfence();
        // first piece: the warp whose range holds g0 (its tail slot)
        int64_t wa = (int64_t)((__int128)g0 * Nw / E);
        while (wa + 1 < Nw && (int64_t)((__int128)(wa + 1) * E / Nw) <= g0) ++wa;
        while (wa > 0 && (int64_t)((__int128)wa * E / Nw) > g0) --wa;
        double s = __ldcg(b.part_tail + wa * 32 + lane);
        for (int64_t v = wa + 1; v < Nw; ++v) {
            s += __ldcg(b.part_head + v * 32 + lane);
            if (__ldcg(b.cut_end + v) >= g1) break;
        }
        if (valid) {
            const uint32_t row = perm[g * 32 + lane];
            if (partial) partial[blk * R + row] = s;
            else y[br * R + row] = (V)s;
        }
        if (lane == 0) b.counters[g] = 0u;  // self-cleaning for the next launch
    }
}

template <typename V, bool EXACT>
int launch(const hbp_format_t *f, const hbp_balanced_t *b, const void *x, void *y,
           double *partial, cudaStream_t st) {
    unsigned grid = (unsigned)((b->workers + kWarps - 1) / kWarps);
    k_spmv_balanced<V, EXACT><<<grid, kThreads, 0, st>>>(*f, *b, (const V *)x, (V *)y, partial);
    return (int)cudaGetLastError();
}

}  // namespace

extern "C" {

int hbp_balanced_workers(const hbp_format_t *f, int64_t *workers) {
    if (!f) return HBP_E_ARG;
    int dev = 0, sms = 0, per_sm = 0;
    HBP_CUDA_TRY(cudaGetDevice(&dev));
    HBP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (f->dtype == HBP_F64)
        HBP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, k_spmv_balanced<double, true>, kThreads, 0));
    else
        HBP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, k_spmv_balanced<float, false>, kThreads, 0));
    int64_t wmax = (int64_t)sms * per_sm * kWarps;
    // at least ~512 elements per warp so cuts stay far apart
    int64_t wcap = f->nnz / 512;
    if (wcap < 1) wcap = 1;
    *workers = wmax < wcap ? wmax : wcap;
    return HBP_OK;
}

int hbp_spmv_balanced(const hbp_format_t *f, const hbp_balanced_t *b, const void *x, void *y,
                      double *partial, hbp_stream_t stream) {
    if (!f || !b || b->workers < 1) return HBP_E_ARG;
    if (f->warp_size != 32 || f->row_height % 32) return HBP_E_UNSUPPORTED;
    if (!partial && (!y || f->ncb != 1)) return HBP_E_ARG;
    if (f->nzb == 0) return HBP_OK;
    cudaStream_t st = as_stream(stream);
    const bool exact = f->exact != 0 || f->dtype == HBP_F64;
    if (!exact && (!b->part_head || !b->part_tail || !b->cut_end || !b->counters))
        return HBP_E_ARG;
    int rc;
    if (f->dtype == HBP_F64) {
        rc = exact ? launch<double, true>(f, b, x, y, partial, st)
                   : launch<double, false>(f, b, x, y, partial, st);
    } else if (f->dtype == HBP_F32) {
        rc = exact ? launch<float, true>(f, b, x, y, partial, st)
                   : launch<float, false>(f, b, x, y, partial, st);
    } else {
        return HBP_E_ARG;
    }
    return rc;
}

}  // extern "C"
