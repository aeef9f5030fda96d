// hbp_spmv_rowstage.cu -- row-block-owner HBP SpMV with TMA-staged elements
// (W = 32; small matrices with several column blocks, e.g. cfg1).
//
// Same work split and arithmetic as hbp_spmv_rowblock (one CTA per row
// block computes the partials of the row block's nonzero blocks, then folds
// them in ascending bc exactly as combine does, engine.py:196-201), but the
// dependent global-load chain of each (block, group) task is cut:
//
//   1. a per-operator descriptor table (hbp_rowstage_plan) holds every
//      nonzero block's 16-byte-aligned element span and its offset in the
//      row block's staging buffer, so thread j of the CTA bulk-copies
//      (cp.async.bulk) block j's col/data straight away -- one DRAM round
//      trip for the whole row block, issued in parallel, no registers held;
//   2. the CTA is persistent and loads the next row block's rb_ptr entries
//      and descriptors into registers behind the current walk; several CTAs
//      per SM overlap one row block's copies with another's walk (a
//      double-buffered form -- row block i+1's copies in flight while i is
//      walked -- halved the CTAs per SM and measured slower, 32.8 vs 28.7 us);
//   3. every lane loads its tasks' slot length, output row and group start
//      one task ahead (block indices from shared memory, no division);
//   4. the walk reads col/data from shared memory (positions from per-step
//      ballots of the slot lengths, the closed form of build_hbp's layout);
//      only the x gathers go to global memory, four steps in flight.
//
// Per-slot sums are group_dot's (hbp_spmv.cu): f64 products __dmul_rn, then
// __dadd_rn in step order -- bitwise the reference; f32 products exact in f64,
// f64 sums.  So y is bitwise that of hbp_spmv_blocks + hbp_combine.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "hbp.h"
#include "hbp_common.cuh"

using namespace hbp;

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kMaxBlocks = 32;  // nonzero blocks per row block (staging table)

template <typename V, bool EXACT>
__device__ __forceinline__ double fmadd_rs(double acc, V v, V xv) {
    if (EXACT) return __dadd_rn(acc, __dmul_rn((double)v, (double)xv));
    return fma((double)v, (double)xv, acc);
}

__device__ __forceinline__ void mbar_expect_only(uint64_t *m, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(m)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive1(uint64_t *m) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(m)) : "memory");
}

__host__ __device__ constexpr int64_t staged_span(int64_t e0, int64_t e1) {
    return ((e1 - (e0 & ~(int64_t)3)) + 3) & ~(int64_t)3;  // 16-byte granules of u32 / V
}

// Descriptor of the block at row-block position i (rb_blk order), 4 x i64:
// desc[4i]   = a0 (first staged element, e0 rounded down to a multiple of 4),
// desc[4i+1] = m (staged elements, a multiple of 4) << 32 | offset of a0 in
//              the row block's element buffer;
// desc[4i+2] = xa (first staged column of the block's x window, rounded down
//              to a 16-byte multiple), or -1 without windows;
// desc[4i+3] = xn (columns staged from xa: up to the window end) << 32 |
//              offset of xa in the row block's x buffer.
// caps[0] = largest element buffer, caps[1] = most blocks in a row block,
// caps[2] = largest x buffer (in columns, 16-byte granules).
__global__ void k_rowstage_plan(const hbp_format_t f, const int32_t *__restrict__ win_lo,
                                const int32_t *__restrict__ win_hi, int64_t *__restrict__ desc,
                                unsigned long long *__restrict__ caps) {
    const int64_t R = f.row_height, gpb = R / 32, nrb = (f.rows + R - 1) / R;
    const int64_t A = f.dtype == HBP_F64 ? 2 : 4;  // x elements per 16 bytes
    for (int64_t br = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; br < nrb;
         br += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = f.rb_ptr[br], hi = f.rb_ptr[br + 1];
        int64_t off = 0, xoff = 0;
        for (int64_t i = lo; i < hi; ++i) {
            const int64_t b = f.rb_blk[i];
            const int64_t e0 = f.group_start[b * gpb], e1 = f.group_start[(b + 1) * gpb];
            const int64_t m = staged_span(e0, e1);
            desc[4 * i] = e0 & ~(int64_t)3;
            desc[4 * i + 1] = (m << 32) | off;
            off += m;
            if (win_lo) {
                const int64_t xa = (int64_t)win_lo[b] / A * A;
                const int64_t xn = (int64_t)win_hi[b] - xa;
                desc[4 * i + 2] = xa;
                desc[4 * i + 3] = (xn << 32) | xoff;
                xoff += (xn + A - 1) / A * A;
            } else {
                desc[4 * i + 2] = -1;
                desc[4 * i + 3] = 0;
            }
        }
        atomicMax(caps, (unsigned long long)off);
        atomicMax(caps + 1, (unsigned long long)(hi - lo));
        atomicMax(caps + 2, (unsigned long long)xoff);
    }
}

template <typename V, bool EXACT, int NT, bool XW>
__global__ void __launch_bounds__(NT)
    k_spmv_rowstage(const hbp_format_t f, const int64_t *__restrict__ desc,
                    const V *__restrict__ x, V *__restrict__ y, int32_t ecap, int32_t xcap,
                    int32_t kmax) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ int64_t s_base[kMaxBlocks];  // staged index of element 0 of block j
    __shared__ int32_t s_blk[kMaxBlocks];   // block j's index (rb_blk order)
    __shared__ int32_t s_xbase[kMaxBlocks]; // XW: staged x index of column 0 of block j
    uint32_t *col_s = reinterpret_cast<uint32_t *>(sm);
    V *dat_s = reinterpret_cast<V *>(sm + (int64_t)ecap * 4);
    double *part = reinterpret_cast<double *>(sm + (int64_t)ecap * (4 + sizeof(V)));
    // XW: the row block's x windows after the partials
    V *x_s = reinterpret_cast<V *>(sm + (int64_t)ecap * (4 + sizeof(V)) +
                                   (int64_t)kmax * f.row_height * 8);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int nwarps = NT / 32;
    const unsigned lt = (1u << lane) - 1u;
    const int32_t R = (int32_t)f.row_height, gpb = R / 32;
    const int64_t nrb = (f.rows + R - 1) / R;
    const V *__restrict__ data = (const V *)f.data;
    const uint64_t pe = policy_evict_first(), pl = policy_evict_last();
    if (threadIdx.x == 0) {
        mbar_init(&mbar, 1);
        fence_mbar_init();
    }
    __syncthreads();

    // The next row block's rb_ptr entries, and (threads j < its block count)
    // block j's descriptor and index, are loaded into registers while the
    // current row block is walked, so staging issues without a round trip.
    int64_t br = blockIdx.x;
    int64_t lo = 0, hi = 0, d_a0 = 0, d_mo = 0, d_xa = 0, d_xo = 0;
    int32_t d_blk = 0;
    auto fetch_desc = [&](int64_t l, int64_t h) {
        if ((int64_t)threadIdx.x < h - l) {
            d_a0 = desc[4 * (l + threadIdx.x)];
            d_mo = desc[4 * (l + threadIdx.x) + 1];
            if (XW) {
                d_xa = desc[4 * (l + threadIdx.x) + 2];
                d_xo = desc[4 * (l + threadIdx.x) + 3];
            }
            d_blk = f.rb_blk[l + threadIdx.x];
        }
    };
    if (br < nrb) {
        lo = f.rb_ptr[br];
        hi = f.rb_ptr[br + 1];
        fetch_desc(lo, hi);
    }
    uint32_t phase = 0u;
    for (; br < nrb; br += gridDim.x) {
        const int64_t n64 = f.rows - br * R;
        const int32_t n = (int32_t)(n64 > R ? R : n64);
        const int32_t cnt = (int32_t)(hi - lo);
        if ((int)threadIdx.x < cnt) {  // thread j stages block j
            const int32_t m = (int32_t)(d_mo >> 32), off = (int32_t)(d_mo & 0xffffffff);
            s_base[threadIdx.x] = (int64_t)off - d_a0;
            s_blk[threadIdx.x] = d_blk;
            fence_proxy_async();  // the CTA's generic accesses of the buffers (barrier-ordered) first
            if (m > 0) {
                mbar_expect_only(&mbar, (uint32_t)m * (4u + (uint32_t)sizeof(V)));
                bulk_g2s(col_s + off, f.col + d_a0, (uint32_t)m * 4u, &mbar, pe);
                bulk_g2s(dat_s + off, data + d_a0, (uint32_t)m * (uint32_t)sizeof(V), &mbar, pe);
            }
            if (XW) {  // the block's x window: 16-byte granules by TMA, the rest by hand
                constexpr int32_t A = 16 / (int32_t)sizeof(V);
                const int32_t xn = (int32_t)(d_xo >> 32), xo = (int32_t)(d_xo & 0xffffffff);
                s_xbase[threadIdx.x] = xo - (int32_t)d_xa;
                const int32_t nb = xn / A * A;
                if (nb > 0) {
                    mbar_expect_only(&mbar, (uint32_t)nb * (uint32_t)sizeof(V));
                    bulk_g2s(x_s + xo, x + d_xa, (uint32_t)nb * (uint32_t)sizeof(V), &mbar, pl);
                }
                for (int32_t i = nb; i < xn; ++i) x_s[xo + i] = x[d_xa + i];
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) mbar_arrive1(&mbar);
        const int64_t nx = br + gridDim.x;
        int64_t nlo = 0, nhi = 0;
        if (nx < nrb) {
            nlo = f.rb_ptr[nx];
            nhi = f.rb_ptr[nx + 1];
        }
        V *yb = y + br * R;
        const int32_t ng = (n + 31) >> 5;
        const int32_t ntask = cnt * ng;
        // task t = (block j, group g), t = j * ng + g; advanced without division
        int32_t tj = 0, tg = wid;
        while (tg >= ng && tj < cnt) tg -= ng, ++tj;
        uint32_t len_n = 0u, row_n = 0u;
        int32_t base_n = 0, j_n = 0, g_n = 0;
        auto load = [&]() {
            const int64_t b = s_blk[tj];
            const int32_t slot = tg * 32 + lane;
            len_n = slot < n ? __ldcs(f.slot_len + b * R + slot) : 0u;
            row_n = slot < n ? __ldcs(f.perm + b * R + slot) : 0u;
            base_n = (int32_t)(f.group_start[b * gpb + tg] + s_base[tj]);
            j_n = tj;
            g_n = tg;
            tg += nwarps;
            while (tg >= ng) tg -= ng, ++tj;
        };
        if (wid < ntask) load();
        mbar_wait(&mbar, phase);
        phase ^= 1u;
        for (int32_t t = wid; t < ntask; t += nwarps) {
            const uint32_t len = len_n, row = row_n;
            int32_t base = base_n;
            const int32_t j = j_n;
            const bool valid = g_n * 32 + lane < n;
            const int32_t xb = XW ? s_xbase[j] : 0;
            // x of column c: the staged window (XW) or global memory
            auto X = [&](uint32_t c) -> V { return XW ? x_s[(int32_t)c + xb] : ld_x(x + c, pl); };
            if (t + nwarps < ntask) load();
            double acc = 0.0;
            uint32_t t0 = 0;
            bool live = len > 0;
            unsigned mask = __ballot_sync(FULL, live);
            while (mask) {
                const int k = __popc(mask);
                const uint32_t t1 = __reduce_min_sync(FULL, live ? len : 0xffffffffu);
                if (live) {
                    int32_t p = base + __popc(mask & lt);
                    const uint32_t M = t1 - t0;
                    uint32_t s = 0;
                    for (; s + 4 <= M; s += 4) {
                        const uint32_t c0 = col_s[p], c1 = col_s[p + k], c2 = col_s[p + 2 * k],
                                       c3 = col_s[p + 3 * k];
                        const V x0 = X(c0), x1 = X(c1), x2 = X(c2), x3 = X(c3);
                        acc = fmadd_rs<V, EXACT>(acc, dat_s[p], x0);
                        acc = fmadd_rs<V, EXACT>(acc, dat_s[p + k], x1);
                        acc = fmadd_rs<V, EXACT>(acc, dat_s[p + 2 * k], x2);
                        acc = fmadd_rs<V, EXACT>(acc, dat_s[p + 3 * k], x3);
                        p += 4 * k;
                    }
                    if (s + 2 <= M) {
                        const uint32_t c0 = col_s[p], c1 = col_s[p + k];
                        const V x0 = X(c0), x1 = X(c1);
                        acc = fmadd_rs<V, EXACT>(acc, dat_s[p], x0);
                        acc = fmadd_rs<V, EXACT>(acc, dat_s[p + k], x1);
                        p += 2 * k;
                        s += 2;
                    }
                    if (s < M) acc = fmadd_rs<V, EXACT>(acc, dat_s[p], X(col_s[p]));
                }
                base += (int32_t)(t1 - t0) * k;
                t0 = t1;
                live = len > t0;
                mask = __ballot_sync(FULL, live);
            }
            if (valid) part[(int64_t)j * R + row] = acc;
        }
        fetch_desc(nlo, nhi);  // the next row block's descriptors, behind the walk
        __syncthreads();
        // fold in ascending bc: s = p_first; s += p_next ... (combine's order);
        // a row block without nonzero blocks gets +0.0
        for (int32_t r = threadIdx.x; r < n; r += NT) {
            double v = cnt ? part[r] : 0.0;
            for (int32_t j = 1; j < cnt; ++j) v = __dadd_rn(v, part[(int64_t)j * R + r]);
            __stcs(yb + r, (V)v);
        }
        lo = nlo;
        hi = nhi;
        __syncthreads();
    }
}

template <typename V, bool EXACT, int NT, bool XW>
int launch_rowstage(const hbp_format_t *f, const int64_t *desc, const void *x, void *y,
                    int32_t ecap, int32_t kmax, int32_t xcap, cudaStream_t st) {
    const size_t smem = (size_t)ecap * (4 + sizeof(V)) + (size_t)kmax * f->row_height * 8 +
                        (XW ? (size_t)xcap * sizeof(V) : 0);
    auto kern = k_spmv_rowstage<V, EXACT, NT, XW>;
    HBP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 0, per_sm = 0;
    HBP_CUDA_TRY(cudaGetDevice(&dev));
    HBP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    HBP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
    if (per_sm < 1) return HBP_E_UNSUPPORTED;
    const int64_t nrb = (f->rows + f->row_height - 1) / f->row_height;
    const int64_t want = (int64_t)sms * per_sm;
    const unsigned grid = (unsigned)(nrb < want ? nrb : want);
    kern<<<grid, NT, smem, st>>>(*f, desc, (const V *)x, (V *)y, ecap, xcap, kmax);
    return (int)cudaGetLastError();
}

}  // namespace

extern "C" {

int hbp_rowstage_plan(const hbp_format_t *f, const int32_t *win_lo, const int32_t *win_hi,
                      int64_t *desc, unsigned long long *caps, hbp_stream_t stream) {
    if (!f || !caps || !f->rb_ptr || (f->nzb > 0 && (!f->rb_blk || !desc))) return HBP_E_ARG;
    if (!win_lo != !win_hi) return HBP_E_ARG;
    if (f->warp_size != 32 || f->row_height % 32) return HBP_E_UNSUPPORTED;
    cudaStream_t st = as_stream(stream);
    HBP_CUDA_TRY(cudaMemsetAsync(caps, 0, 3 * sizeof(unsigned long long), st));
    const int64_t nrb = (f->rows + f->row_height - 1) / f->row_height;
    if (nrb == 0 || f->nzb == 0) return HBP_OK;
    k_rowstage_plan<<<grid_for(nrb, 256), 256, 0, st>>>(*f, win_lo, win_hi, desc, caps);
    return (int)cudaGetLastError();
}

int hbp_spmv_rowstage(const hbp_format_t *f, const int64_t *desc, const void *x, void *y,
                      int64_t ecap, int64_t kmax, int64_t xcap, hbp_stream_t stream) {
    if (!f || f->rows < 0 || (f->rows > 0 && !y)) return HBP_E_ARG;
    if (f->warp_size != 32 || f->row_height % 32) return HBP_E_UNSUPPORTED;
    if (f->rows == 0) return HBP_OK;
    if (!f->rb_ptr || (f->nzb > 0 && (!x || !f->rb_blk || !desc))) return HBP_E_ARG;
    if (ecap < 4 || kmax < 1 || (ecap & 3) || xcap < 0) return HBP_E_ARG;
    if (kmax > kMaxBlocks || ecap > (1 << 24) || xcap > (1 << 24)) return HBP_E_UNSUPPORTED;
    // x windows staged by TMA need a 16-byte aligned x (and a plan with windows)
    if (xcap > 0 && ((uintptr_t)x & 15)) return HBP_E_ARG;
    cudaStream_t st = as_stream(stream);
    // tuning A/B only: threads per CTA (256 default: cfg1 24.1-25.0 us vs 28.2-28.7 at
    // 512, ncu kernel times, caches flushed)
    static const int nt =
        getenv("HBP_ROWSTAGE_THREADS") ? atoi(getenv("HBP_ROWSTAGE_THREADS")) : 256;
    const int32_t e = (int32_t)ecap, k = (int32_t)kmax, xc = (int32_t)xcap;
    const bool xw = xcap > 0;
#define HBP_RS(V, EX)                                                                            \
    return nt == 512 ? (xw ? launch_rowstage<V, EX, 512, true>(f, desc, x, y, e, k, xc, st)     \
                           : launch_rowstage<V, EX, 512, false>(f, desc, x, y, e, k, xc, st))   \
                     : (xw ? launch_rowstage<V, EX, 256, true>(f, desc, x, y, e, k, xc, st)     \
                           : launch_rowstage<V, EX, 256, false>(f, desc, x, y, e, k, xc, st))
    if (f->dtype == HBP_F64) HBP_RS(double, true);
    if (f->dtype == HBP_F32) HBP_RS(float, false);
#undef HBP_RS
    return HBP_E_ARG;
}

}  // extern "C"
