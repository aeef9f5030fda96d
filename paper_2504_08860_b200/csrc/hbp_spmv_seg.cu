// hbp_spmv_seg.cu -- column-segment HBP SpMV (W = 32, several column blocks).
//
// The reference runs each nonzero block against its x-segment
// x[bc*C : (bc+1)*C] (engine.py:127-134 block_spmv -> _kernels.py:22-47).
// Here a persistent CTA owns one block at a time:
//
//   1. the part of the segment the block's columns touch, x[win_lo, win_hi)
//      (hbp_seg_windows, once per operator), is bulk-copied into shared memory
//      with cp.async.bulk (TMA, mbarrier completion), double-buffered so the
//      next block's segment lands while the current one is walked;
//   2. the CTA's warps take the block's groups; lane q walks its row in step
//      order (positions from per-step ballots of the slot lengths, the
//      closed form of build_hbp's layout), loading U steps of
//      col / data at once (coalesced: a step's live lanes are consecutive
//      elements) and reading x from shared memory -- every gather is a
//      shared-memory load, none goes through the L1 miss path;
//   3. blocks are scheduled as the reference plans them (engine.py:96-176):
//      CTA w runs its fixed contiguous chunk of the bc-major block list, then
//      draws blocks [fixed_count, nzb) from an atomic ticket (competitive
//      pool).  The ticket pair lives in caller memory and is left zeroed.
//
// Exact mode (f64) sums each row as _kernels.py:41-46 does (products
// __dmul_rn, then __dadd_rn in step order): bitwise the reference.  f32 data
// forms f32 products and sums them in f64 in step order (deterministic).
#include <cuda_runtime.h>

#include <atomic>
#include <stdint.h>
#include <stdlib.h>

#include "hbp.h"
#include "hbp_common.cuh"

using namespace hbp;

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kMaxDevices = 64;

__device__ __forceinline__ unsigned lanemask_lt_() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename V>
__device__ __forceinline__ V lds_x(uint32_t a) {
    V v;
    if constexpr (sizeof(V) == 4) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    else asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

// per-block column window [min col, max col + 1): one CTA per nonzero block
__global__ void k_seg_windows(const int64_t *__restrict__ gs, int64_t gpb, int64_t nzb,
                              const uint32_t *__restrict__ col, int32_t *__restrict__ win_lo,
                              int32_t *__restrict__ win_hi,
                              unsigned long long *__restrict__ cap) {
    __shared__ uint32_t s_lo[32], s_hi[32];
    for (int64_t blk = blockIdx.x; blk < nzb; blk += gridDim.x) {
        const int64_t e0 = gs[blk * gpb], e1 = gs[(blk + 1) * gpb];
        uint32_t lo = 0xffffffffu, hi = 0u;
        for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
            const uint32_t c = __ldcs(col + e);
            lo = c < lo ? c : lo;
            hi = c > hi ? c : hi;
        }
        lo = __reduce_min_sync(FULL, lo);
        hi = __reduce_max_sync(FULL, hi);
        const int wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
        if ((threadIdx.x & 31) == 0) s_lo[wid] = lo, s_hi[wid] = hi;
        __syncthreads();
        if (threadIdx.x < 32) {
            lo = threadIdx.x < nw ? s_lo[threadIdx.x] : 0xffffffffu;
            hi = threadIdx.x < nw ? s_hi[threadIdx.x] : 0u;
            lo = __reduce_min_sync(FULL, lo);
            hi = __reduce_max_sync(FULL, hi);
            if (threadIdx.x == 0) {
                if (e1 <= e0) lo = hi = 0u;  // (nonzero blocks are never empty)
                else hi += 1u;
                win_lo[blk] = (int32_t)lo;
                win_hi[blk] = (int32_t)hi;
                atomicMax(cap, (unsigned long long)(hi - lo));
            }
        }
        __syncthreads();
    }
}

// shared layout of one CTA: two window buffers, two mbarriers, two block ids
struct SegCtl {
    uint64_t mbar[2];
    int32_t blk[2];
};

template <typename V>
__host__ __device__ constexpr size_t buf_bytes(int64_t cap) {
    return (size_t)((cap * (int64_t)sizeof(V) + 16 + 15) & ~(int64_t)15);
}

// L2 bulk prefetch of [p, p + bytes) (16-byte aligned span covering it)
__device__ __forceinline__ void prefetch_l2(const void *p, size_t bytes) {
    const uintptr_t a = (uintptr_t)p & ~(uintptr_t)15;
    const uintptr_t b = ((uintptr_t)p + bytes + 15) & ~(uintptr_t)15;
    if (b > a)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(b - a))
                     : "memory");
}

// PF: 0 none; 1 each group's element range is bulk-prefetched into L2 when
// its walk starts (the default: the batched loads then hit L2 while the
// prefetch streams the group from HBM in full lines); 2 the warp's next
// group of the block is prefetched instead
template <typename V, bool EXACT, int NW, int MINB, int U, int PF = 0>
__global__ void __launch_bounds__(NW * 32, MINB)
    k_spmv_seg(const hbp_format_t f, const hbp_seg_t s, const V *__restrict__ x,
               V *__restrict__ y, double *__restrict__ partial) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const size_t bb = buf_bytes<V>(s.win_cap);
    SegCtl &ctl = *reinterpret_cast<SegCtl *>(smem_raw + 2 * bb);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int32_t R = (int32_t)f.row_height, gpb = R / 32;
    const int64_t nzb = f.nzb;
    const int64_t w = blockIdx.x;
    // engine.py:107-115: contiguous fixed chunks, the first `rem` one longer
    const int64_t per = s.fixed_count / s.ctas, rem = s.fixed_count % s.ctas;
    int64_t fx = w * per + (w < rem ? w : rem);
    const int64_t fx_hi = fx + per + (w < rem ? 1 : 0);
    const uint64_t pol_el = policy_evict_last();  // x: reused by neighbouring row blocks
    const uint64_t pol_ef = policy_evict_first(); // element stream

    // thread 0: next block of this worker (fixed chunk, then the ticket)
    auto draw = [&]() -> int32_t {
        if (fx < fx_hi) return (int32_t)fx++;
        const int64_t idx = s.fixed_count + (int64_t)atomicAdd(s.ticket, 1u);
        return idx < nzb ? (int32_t)idx : -1;
    };
    // thread 0: bring x[win_lo, win_hi) of block b into buffer i.  Byte layout:
    // element c sits at (addr(x + c) - P), P = addr(x + win_lo) rounded down to
    // 16 B; the 16-byte-aligned interior is one bulk copy, the (< 16 B) head
    // and tail are plain loads.
    auto stage = [&](int32_t b, int i) {
        unsigned char *buf = smem_raw + (size_t)i * bb;
        const int64_t lo = s.win_lo[b], hi = s.win_hi[b];
        const uintptr_t xa = (uintptr_t)x;
        const uintptr_t P = (xa + (uintptr_t)lo * sizeof(V)) & ~(uintptr_t)15;
        const uintptr_t pa = (xa + (uintptr_t)lo * sizeof(V) + 15) & ~(uintptr_t)15;
        const uintptr_t pb = (xa + (uintptr_t)hi * sizeof(V)) & ~(uintptr_t)15;
        fence_proxy_async();  // earlier generic accesses of this buffer before the bulk write
        if (pb > pa) {
            mbar_expect_tx(&ctl.mbar[i], (uint32_t)(pb - pa));
            bulk_g2s(buf + (pa - P), (const void *)pa, (uint32_t)(pb - pa), &ctl.mbar[i], pol_el);
        } else {
            mbar_expect_tx(&ctl.mbar[i], 0u);
        }
        const int64_t ea = pb > pa ? (int64_t)((pa - xa) / sizeof(V)) : hi;
        const int64_t eb = pb > pa ? (int64_t)((pb - xa) / sizeof(V)) : hi;
        for (int64_t c = lo; c < ea; ++c)
            *reinterpret_cast<V *>(buf + (xa + (uintptr_t)c * sizeof(V) - P)) = __ldg(x + c);
        for (int64_t c = eb; c < hi; ++c)
            *reinterpret_cast<V *>(buf + (xa + (uintptr_t)c * sizeof(V) - P)) = __ldg(x + c);
    };

    if (threadIdx.x == 0) {
        mbar_init(&ctl.mbar[0], 1);
        mbar_init(&ctl.mbar[1], 1);
        fence_mbar_init();
        const int32_t b0 = draw();
        ctl.blk[0] = b0;
        if (b0 >= 0) stage(b0, 0);
    }
    __syncthreads();

    const unsigned lt = lanemask_lt_();
    const bool direct_single = partial != nullptr && (f.reserved & HBP_FLAG_DIRECT_SINGLE);
    for (uint32_t j = 0;; ++j) {
        const int i = (int)(j & 1u);
        const int32_t blk = ctl.blk[i];
        if (blk < 0) break;
        if (threadIdx.x == 0) {  // next block into the other buffer (free since the last barrier)
            const int32_t nb = draw();
            ctl.blk[i ^ 1] = nb;
            if (nb >= 0) stage(nb, i ^ 1);
        }
        mbar_wait(&ctl.mbar[i], (j >> 1) & 1u);
        // shared address of x[c] is xs + c * sizeof(V) (mod 2^32)
        const int64_t lo = s.win_lo[blk];
        const uintptr_t xa = (uintptr_t)x;
        const uintptr_t P = (xa + (uintptr_t)lo * sizeof(V)) & ~(uintptr_t)15;
        const uint32_t xs = smem_addr(smem_raw + (size_t)i * bb) + (uint32_t)(xa - P);
        const int64_t br = f.blk_br[blk];
        const int64_t left = f.rows - br * R;
        const int32_t nrows = (int32_t)(left < R ? left : R);
        const int32_t ngb = (nrows + 31) >> 5;
        bool to_partial = partial != nullptr;
        if (direct_single && f.rb_ptr[br + 1] - f.rb_ptr[br] == 1) to_partial = false;

        for (int32_t gi = wib; gi < ngb; gi += NW) {
            const int32_t slot = gi * 32 + lane;
            const bool valid = slot < nrows;
            const int64_t sidx = (int64_t)blk * R + slot;
            const uint32_t len = valid ? __ldcs(f.slot_len + sidx) : 0u;
            const int64_t g0 = __ldcs(f.group_start + (int64_t)blk * gpb + gi);
            if constexpr (PF != 0) {
                const int32_t gp = PF == 1 ? gi : gi + NW;
                if (lane == 0 && (PF == 1 || gp < ngb)) {
                    const int64_t a0 = PF == 1 ? g0 : f.group_start[(int64_t)blk * gpb + gp];
                    const int64_t a1 = f.group_start[(int64_t)blk * gpb + gp + 1];
                    if (a1 > a0) {
                        prefetch_l2(f.col + a0, (size_t)(a1 - a0) * 4);
                        prefetch_l2((const V *)f.data + a0, (size_t)(a1 - a0) * sizeof(V));
                    }
                }
            }
            const uint32_t maxlen = __reduce_max_sync(FULL, len);
            double acc = 0.0;
            int64_t off = g0;  // element index where the next batch's first step starts
            // software pipeline: the loads of batch t + U are in flight while
            // batch t is summed (each batch: U steps of col / data)
            uint32_t ca[U], cb[U];
            V da[U], db[U];
            uint32_t la = 0u, lb = 0u;  // live bits of the batch's steps
            auto load_batch = [&](uint32_t t, uint32_t(&cc)[U], V(&dv)[U], uint32_t &lvb) {
                lvb = 0u;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool lv = len > t + (uint32_t)u;
                    const unsigned m = __ballot_sync(FULL, lv);
                    const int64_t pos = off + __popc(m & lt);
                    off += __popc(m);
                    cc[u] = 0u;
                    dv[u] = (V)0;
                    if (lv) {
                        cc[u] = ld_stream_u32(f.col + pos, pol_ef);
                        dv[u] = ld_stream((const V *)f.data + pos, pol_ef);
                        lvb |= 1u << u;
                    }
                }
            };
            auto sum_batch = [&](const uint32_t(&cc)[U], const V(&dv)[U], uint32_t lvb) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if ((lvb >> u) & 1u) {
                        const V xv = lds_x<V>(xs + cc[u] * (uint32_t)sizeof(V));
                        V p;
                        if constexpr (EXACT) p = (V)__dmul_rn((double)dv[u], (double)xv);
                        else p = dv[u] * xv;
                        acc = __dadd_rn(acc, (double)p);
                    }
                }
            };
            if (maxlen > 0) load_batch(0u, ca, da, la);
            for (uint32_t t = 0; t < maxlen; t += 2 * U) {
                if (t + U < maxlen) load_batch(t + U, cb, db, lb);
                sum_batch(ca, da, la);
                if (t + U >= maxlen) break;
                if (t + 2 * U < maxlen) load_batch(t + 2 * U, ca, da, la);
                sum_batch(cb, db, lb);
            }
            if (valid) {
                const uint32_t row = __ldcs(f.perm + sidx);
                if (to_partial) partial[(int64_t)blk * R + row] = acc;
                else __stcs(y + br * R + row, (V)acc);
            }
        }
        __syncthreads();  // buffer i and ctl.blk[i] are free again
    }
    // the last CTA out resets the ticket pair for the next call
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(s.ticket + 1, 1u) == gridDim.x - 1) {
            s.ticket[0] = 0u;
            s.ticket[1] = 0u;
            __threadfence();
        }
    }
}

// launch shapes (warps per CTA, min CTAs per SM, steps loaded per batch);
// HBP_SEG_VARIANT selects one for A/B sweeps, 0 is the default
struct Shape {
    int nw, minb, u;
};
// cfg3 (banded, 1.1B nnz, f64, same box): 0 = 4 warps x 8 CTAs, 4-step
// batches, each group's element range bulk-prefetched into L2 as its walk
// starts: 2.15-2.18 ms (0.97 of the measured HBM peak); without the prefetch
// 2.54 (variant 5); 16 x 1 CTAs 4.6 ms (variant 1); the per-warp stream
// kernel 2.65 ms
constexpr Shape kShapes[] = {{4, 8, 4}, {16, 1, 4}, {8, 3, 8}, {16, 2, 4}, {8, 2, 8}, {4, 8, 4},
                             {2, 16, 4}, {4, 6, 8}, {2, 12, 8}, {4, 8, 4}, {4, 8, 4},
                             {2, 16, 4}, {8, 4, 4}, {4, 6, 8}, {4, 8, 2}, {16, 2, 4}, {8, 4, 4}};
constexpr int kNShapes = sizeof(kShapes) / sizeof(kShapes[0]);
std::atomic<int> g_seg_variant{-1};  // A/B tuning selector (process-wide, read once)
int seg_variant() {
    int v = g_seg_variant.load(std::memory_order_relaxed);
    if (v < 0) {
        const char *e = getenv("HBP_SEG_VARIANT");
        v = e ? atoi(e) : 0;
        if (v < 0 || v >= kNShapes) v = 0;
        g_seg_variant.store(v, std::memory_order_relaxed);
    }
    return v;
}

#define HBP_SEG_SWITCH(FN, V, EXACT, ...)                        \
    switch (seg_variant()) {                                     \
        case 1: return FN<V, EXACT, 16, 1, 4>(__VA_ARGS__);      \
        case 2: return FN<V, EXACT, 8, 3, 8>(__VA_ARGS__);       \
        case 3: return FN<V, EXACT, 16, 2, 4>(__VA_ARGS__);      \
        case 4: return FN<V, EXACT, 8, 2, 8>(__VA_ARGS__);       \
        case 5: return FN<V, EXACT, 4, 8, 4>(__VA_ARGS__);       \
        case 6: return FN<V, EXACT, 2, 16, 4>(__VA_ARGS__);      \
        case 7: return FN<V, EXACT, 4, 6, 8>(__VA_ARGS__);       \
        case 8: return FN<V, EXACT, 2, 12, 8>(__VA_ARGS__);      \
        case 9: return FN<V, EXACT, 4, 8, 4, 1>(__VA_ARGS__);    \
        case 10: return FN<V, EXACT, 4, 8, 4, 2>(__VA_ARGS__);   \
        case 11: return FN<V, EXACT, 2, 16, 4, 1>(__VA_ARGS__);  \
        case 12: return FN<V, EXACT, 8, 4, 4, 1>(__VA_ARGS__);   \
        case 13: return FN<V, EXACT, 4, 6, 8, 1>(__VA_ARGS__);   \
        case 14: return FN<V, EXACT, 4, 8, 2, 1>(__VA_ARGS__);   \
        case 15: return FN<V, EXACT, 16, 2, 4, 1>(__VA_ARGS__);  \
        case 16: return FN<V, EXACT, 8, 4, 4>(__VA_ARGS__);      \
        default: return FN<V, EXACT, 4, 8, 4, 1>(__VA_ARGS__);   \
    }

template <typename V, bool EXACT, int NW, int MINB, int U, int PF = 0>
int prepare(int64_t win_cap, size_t *smem) {
    *smem = 2 * buf_bytes<V>(win_cap) + sizeof(SegCtl);
    static std::atomic<size_t> attr[kMaxDevices];
    int dev = 0;
    HBP_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= kMaxDevices) return HBP_E_ARG;
    if (attr[dev].load(std::memory_order_relaxed) < *smem) {
        HBP_CUDA_TRY(cudaFuncSetAttribute(k_spmv_seg<V, EXACT, NW, MINB, U, PF>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem));
        attr[dev].store(*smem, std::memory_order_relaxed);
    }
    return HBP_OK;
}

template <typename V, bool EXACT, int NW, int MINB, int U, int PF = 0>
int occupancy_of(int64_t win_cap, int *per_sm) {
    size_t smem = 0;
    const int rc = prepare<V, EXACT, NW, MINB, U, PF>(win_cap, &smem);
    if (rc) return rc;
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        per_sm, k_spmv_seg<V, EXACT, NW, MINB, U, PF>, NW * 32, smem);
}

template <typename V, bool EXACT>
int occupancy(int64_t win_cap, int *per_sm) {
    HBP_SEG_SWITCH(occupancy_of, V, EXACT, win_cap, per_sm)
}

template <typename V, bool EXACT, int NW, int MINB, int U, int PF = 0>
int launch_of(const hbp_format_t *f, const hbp_seg_t *s, const void *x, void *y, double *partial,
              cudaStream_t st) {
    size_t smem = 0;
    const int rc = prepare<V, EXACT, NW, MINB, U, PF>(s->win_cap, &smem);
    if (rc) return rc;
    k_spmv_seg<V, EXACT, NW, MINB, U, PF><<<(unsigned)s->ctas, NW * 32, smem, st>>>(
        *f, *s, (const V *)x, (V *)y, partial);
    return (int)cudaGetLastError();
}

template <typename V, bool EXACT>
int launch(const hbp_format_t *f, const hbp_seg_t *s, const void *x, void *y, double *partial,
           cudaStream_t st) {
    HBP_SEG_SWITCH(launch_of, V, EXACT, f, s, x, y, partial, st)
}

bool exact_of(const hbp_format_t *f) { return f->exact != 0 || f->dtype == HBP_F64; }

}  // namespace

extern "C" {

int hbp_seg_windows(const hbp_format_t *f, int32_t *win_lo, int32_t *win_hi,
                    int64_t *win_cap, hbp_stream_t stream) {
    if (!f || !win_lo || !win_hi || !win_cap) return HBP_E_ARG;
    if (f->warp_size != 32 || f->row_height % 32) return HBP_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    HBP_CUDA_TRY(cudaMemsetAsync(win_cap, 0, sizeof(int64_t), st));
    if (f->nzb == 0) return HBP_OK;
    if (f->cols > ((int64_t)1 << 31) - 1) return HBP_E_UNSUPPORTED;
    const int64_t gpb = f->row_height / 32;
    const unsigned grid = (unsigned)(f->nzb < 148 * 16 ? f->nzb : 148 * 16);
    k_seg_windows<<<grid, 256, 0, st>>>(f->group_start, gpb, f->nzb, f->col, win_lo, win_hi,
                                         (unsigned long long *)win_cap);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_seg_workers(const hbp_format_t *f, int64_t win_cap, int64_t *ctas) {
    if (!f || !ctas || win_cap < 0) return HBP_E_ARG;
    int dev = 0, sms = 0, per_sm = 0;
    HBP_CUDA_TRY(cudaGetDevice(&dev));
    HBP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int rc;
    if (f->dtype == HBP_F64)
        rc = exact_of(f) ? occupancy<double, true>(win_cap, &per_sm)
                         : occupancy<double, false>(win_cap, &per_sm);
    else if (f->dtype == HBP_F32)
        rc = exact_of(f) ? occupancy<float, true>(win_cap, &per_sm)
                         : occupancy<float, false>(win_cap, &per_sm);
    else return HBP_E_ARG;
    if (rc) return rc;
    if (per_sm < 1) return HBP_E_UNSUPPORTED;  // window beyond shared memory
    int64_t n = (int64_t)sms * per_sm;
    if (f->nzb > 0 && n > f->nzb) n = f->nzb;
    *ctas = n < 1 ? 1 : n;
    return HBP_OK;
}

int hbp_seg_set_variant(int v) {
    if (v < 0 || v >= kNShapes) return HBP_E_ARG;
    g_seg_variant.store(v, std::memory_order_relaxed);
    return HBP_OK;
}

int hbp_spmv_seg(const hbp_format_t *f, const hbp_seg_t *s, const void *x, void *y,
                 double *partial, hbp_stream_t stream) {
    if (!f || !s || s->ctas < 1 || !s->ticket || !s->win_lo || !s->win_hi) return HBP_E_ARG;
    if (f->warp_size != 32 || f->row_height % 32) return HBP_E_UNSUPPORTED;
    if (s->fixed_count < 0 || s->fixed_count > f->nzb || s->win_cap < 0) return HBP_E_ARG;
    if (!partial && (!y || f->ncb != 1)) return HBP_E_ARG;
    if ((f->reserved & HBP_FLAG_DIRECT_SINGLE) && partial && (!y || !f->rb_ptr)) return HBP_E_ARG;
    if (f->nzb == 0) return HBP_OK;
    if (f->nzb >= ((int64_t)1 << 31) - 1 || s->ctas >= ((int64_t)1 << 31)) return HBP_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    if (f->dtype == HBP_F64)
        return exact_of(f) ? launch<double, true>(f, s, x, y, partial, st)
                           : launch<double, false>(f, s, x, y, partial, st);
    if (f->dtype == HBP_F32)
        return exact_of(f) ? launch<float, true>(f, s, x, y, partial, st)
                           : launch<float, false>(f, s, x, y, partial, st);
    return HBP_E_ARG;
}

}  // extern "C"
