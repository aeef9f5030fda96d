// hbp_spmv_stream.cu -- TMA-streamed, element-balanced HBP SpMV (W = 32).
//
// Why: in the HBP layout a group's elements are step-major (all lanes' first
// elements, then the second ...).  On skewed matrices a group has ~10
// "phases" (step ranges with a fixed live-lane set) and few live lanes, so a
// lane-per-row walk over global memory pays two dependent DRAM round trips
// (col, then x) per phase.  Here memory and the irregular walk are decoupled:
//
//   1. each persistent warp owns an equal slice [c_lo, c_hi) of the element
//      array (exact mode: slice ends rounded up to group boundaries);
//   2. lane 0 streams the slice's col/data through shared memory in chunks of
//      CH elements with cp.async.bulk (TMA bulk copies, mbarrier completion),
//      two chunks in flight;
//   3. per chunk the warp gathers x for all CH elements at once (CH/32
//      independent loads per lane) and stores the products (f64) in shared
//      memory;
//   4. the group's phase table (offset, live count k, live mask, steps) is
//      built once per group from the 32 slot lengths with ballots, and the
//      products are summed per row from shared memory:
//        exact (f64): each lane adds its own elements in step order --
//                     bitwise identical to the reference (_kernels.py:41-46);
//        fast  (f32 data, f64 sums): phases with k < 16 live lanes use
//                     S = 32/k sub-streams per lane and a shuffle tree.
//   5. a group cut by a slice boundary (fast mode only) leaves per-lane
//      partials; the warp whose piece completes the group's element count
//      (atomic) adds the pieces in slice order (deterministic).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "hbp.h"
#include "hbp_common.cuh"

using namespace hbp;

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr unsigned FULL = 0xffffffffu;

template <typename V, int CH>
struct __align__(16) WarpSmem {
    uint32_t col[2][CH + 8];
    V val[2][CH + 8];
    double prod[CH];
    int32_t ph_off[33];
    int32_t ph_k[32];
    uint32_t ph_mask[32];
    uint64_t mbar[2];
};

// ---- PTX helpers: mbarrier + bulk async copy (sm_90+ / sm_100a) ------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *m, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(m)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(m)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(m)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *m, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(m)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// per live-lane count k (1..32): sub-streams S = largest power of two with
// k*S <= 32, and the 16-bit reciprocal ceil(2^16/k) (exact lane / k for lane < 32)
__constant__ int c_streams[33] = {0,  32, 16, 8, 8, 4, 4, 4, 4, 2, 2, 2, 2, 2, 2, 2, 2,
                                  1,  1,  1,  1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};
__constant__ uint32_t c_magic16[33] = {
    0,    65536, 32768, 21846, 16384, 13108, 10923, 9363, 8192, 7282, 6554,
    5958, 5462,  5042,  4682,  4370,  4096,  3856,  3641, 3450, 3277, 3121,
    2979, 2850,  2731,  2622,  2521,  2428,  2341,  2260, 2185, 2115, 2048};

// ceil(2^32 / k): floor(n / k) = (n * m) >> 32 exactly for n < 2^27
__constant__ uint64_t c_magic32[33] = {
    0ull,          4294967296ull, 2147483648ull, 1431655766ull, 1073741824ull, 858993460ull,
    715827883ull,  613566757ull,  536870912ull,  477218589ull,  429496730ull,  390451573ull,
    357913942ull,  330382100ull,  306783379ull,  286331154ull,  268435456ull,  252645136ull,
    238609295ull,  226050911ull,  214748365ull,  204522253ull,  195225787ull,  186737709ull,
    178956971ull,  171798692ull,  165191050ull,  159072863ull,  153391690ull,  148102321ull,
    143165577ull,  138547333ull,  134217728ull};

// ceil(n / k) for 0 < n < 2^20, 1 <= k <= 32
__device__ __forceinline__ int32_t ceil_div_small(int32_t n, int k) {
    return (int32_t)((((uint64_t)(uint32_t)(n + k - 1)) * c_magic32[k]) >> 32);
}

template <typename V, bool EXACT>
__device__ __forceinline__ double mul(V v, V xv) {
    if (EXACT) return __dmul_rn((double)v, (double)xv);
    return (double)v * (double)xv;  // exact for f32 inputs
}

// largest g in [0, n] with gs[g] <= e
__device__ __forceinline__ int64_t upper_group(const int64_t *__restrict__ gs, int64_t n,
                                               int64_t e) {
    int64_t lo = 0, hi = n + 1;
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

__device__ __forceinline__ int64_t cut_at(int64_t w, int64_t E, int64_t Nw) {
    return (int64_t)((__int128)w * E / Nw);
}

template <typename V, bool EXACT, int CH, bool XNA>
struct Streamer {
    const hbp_format_t &f;
    WarpSmem<V, CH> &S;
    const V *__restrict__ x;
    int64_t c_lo, c_hi, nchunks;
    int lane;
    uint64_t pe, pl;
    // current chunk window
    int64_t cur = -1, a = 0, bnd = 0;

    // chunk c covers elements [base + c*CH, min(base + (c+1)*CH, c_hi)),
    // base = c_lo rounded down to 4 elements (16-byte aligned for col and
    // data); elements before c_lo belong to the previous slice and are
    // gathered but never summed.
    int64_t base;

    __device__ void chunk_bounds(int64_t c, int64_t &ca, int64_t &cb) const {
        ca = base + c * CH;
        cb = ca + CH < c_hi ? ca + CH : c_hi;
    }

    __device__ void issue(int64_t c) {  // lane 0 only
        int64_t ca, cb;
        chunk_bounds(c, ca, cb);
        const int buf = (int)(c & 1);
        const uint32_t bc = (uint32_t)(((cb - ca) * 4 + 15) & ~(int64_t)15);
        const uint32_t bv = (uint32_t)(((cb - ca) * (int64_t)sizeof(V) + 15) & ~(int64_t)15);
        mbar_expect_tx(&S.mbar[buf], bc + bv);
        bulk_g2s(S.col[buf], f.col + ca, bc, &S.mbar[buf], pe);
        bulk_g2s(S.val[buf], (const V *)f.data + ca, bv, &S.mbar[buf], pe);
    }

    // make chunk c the current one: wait, gather x, products -> S.prod.
    // Chunks are 16-byte aligned in element space (a = base + c*CH), so each
    // lane reads 4 consecutive cols / values with one vector LDS.
    __device__ void prepare(int64_t c) {
        chunk_bounds(c, a, bnd);
        cur = c;
        const int buf = (int)(c & 1);
        mbar_wait(&S.mbar[buf], (uint32_t)((c >> 1) & 1));
        const int n = (int)(bnd - a);
        constexpr int U = CH / 128;
        uint4 cl[U];
        V xv[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = 4 * lane + 128 * u;
            cl[u] = *reinterpret_cast<const uint4 *>(&S.col[buf][i]);
            if (i + 3 >= n) {  // tail of the last chunk: never gather past the slice
                if (i >= n) cl[u].x = 0u;
                if (i + 1 >= n) cl[u].y = 0u;
                if (i + 2 >= n) cl[u].z = 0u;
                cl[u].w = 0u;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t cc[4] = {cl[u].x, cl[u].y, cl[u].z, cl[u].w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
                xv[u][e] = XNA ? ld_x_na(x + cc[e], pl) : ld_x(x + cc[e], pl);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = 4 * lane + 128 * u;
            V vv[4];
            if (sizeof(V) == 4) {
                const float4 t = *reinterpret_cast<const float4 *>(&S.val[buf][i]);
                vv[0] = t.x, vv[1] = t.y, vv[2] = t.z, vv[3] = t.w;
            } else {
                const double2 t0 = *reinterpret_cast<const double2 *>(&S.val[buf][i]);
                const double2 t1 = *reinterpret_cast<const double2 *>(&S.val[buf][i + 2]);
                vv[0] = t0.x, vv[1] = t0.y, vv[2] = t1.x, vv[3] = t1.y;
            }
            double2 p0, p1;
            p0.x = mul<V, EXACT>(vv[0], xv[u][0]);
            p0.y = mul<V, EXACT>(vv[1], xv[u][1]);
            p1.x = mul<V, EXACT>(vv[2], xv[u][2]);
            p1.y = mul<V, EXACT>(vv[3], xv[u][3]);
            *reinterpret_cast<double2 *>(&S.prod[i]) = p0;
            *reinterpret_cast<double2 *>(&S.prod[i + 2]) = p1;
        }
        fence_proxy_async();  // generic reads of this buffer precede the next bulk write
        __syncwarp();
        if (lane == 0 && c + 2 < nchunks) issue(c + 2);
    }
};

template <typename V, bool EXACT, int CH, int MINB, bool XNA>
__global__ void __launch_bounds__(kThreads, MINB)
    k_spmv_stream(const hbp_format_t f, const hbp_balanced_t b, const V *__restrict__ x,
                  V *__restrict__ y, double *__restrict__ partial) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WarpSmem<V, CH> &S = reinterpret_cast<WarpSmem<V, CH> *>(smem_raw)[wib];
    const int64_t w = (int64_t)blockIdx.x * kWarps + wib;
    const int64_t Nw = b.workers;
    if (w >= Nw) return;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t R = f.row_height, gpb = R / 32;
    const int64_t ngroups = f.nzb * gpb;
    const int64_t E = f.nnz;
    const int64_t *__restrict__ gs = f.group_start;
    const uint32_t *__restrict__ slot_len = (const uint32_t *)f.slot_len;
    const uint32_t *__restrict__ permp = (const uint32_t *)f.perm;

    Streamer<V, EXACT, CH, XNA> st{f, S, x};
    st.lane = lane;
    st.pe = policy_evict_first();
    st.pl = policy_evict_last();

    int64_t c_lo = cut_at(w, E, Nw), c_hi = cut_at(w + 1, E, Nw);
    if (EXACT) {  // round slice ends up to group boundaries
        if (c_lo > 0 && c_lo < E) {
            int64_t g = upper_group(gs, ngroups, c_lo);
            if (gs[g] != c_lo) c_lo = gs[g + 1];
        }
        if (c_hi > 0 && c_hi < E) {
            int64_t g = upper_group(gs, ngroups, c_hi);
            if (gs[g] != c_hi) c_hi = gs[g + 1];
        }
    }
    st.c_lo = c_lo;
    st.c_hi = c_hi;
    st.base = c_lo & ~(int64_t)3;
    st.nchunks = c_hi > c_lo ? (c_hi - st.base + CH - 1) / CH : 0;

    if (lane == 0) {
        mbar_init(&S.mbar[0], 1);
        mbar_init(&S.mbar[1], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (lane == 0) {
        if (st.nchunks > 0) st.issue(0);
        if (st.nchunks > 1) st.issue(1);
    }

    int64_t g = upper_group(gs, ngroups, c_lo);
    if (!(g < ngroups && gs[g] < c_lo)) g = lower_group(gs, ngroups, c_lo);
    const bool last_warp = (w == Nw - 1);

    // prefetched metadata of group g
    int64_t gs0 = g < ngroups ? gs[g] : E;
    int64_t gs1 = g < ngroups ? gs[g + 1] : E;
    uint32_t len_n = g < ngroups ? slot_len[g * 32 + lane] : 0u;
    uint32_t perm_n = g < ngroups ? permp[g * 32 + lane] : 0u;

    for (; g < ngroups && (gs0 < c_hi || last_warp); ++g) {
        const uint32_t len = len_n, row_local = perm_n;
        const int64_t g0 = gs0, g1 = gs1;
        if (g + 1 < ngroups) {  // prefetch the next group's metadata
            gs0 = g1;
            gs1 = gs[g + 2];
            len_n = slot_len[(g + 1) * 32 + lane];
            perm_n = permp[(g + 1) * 32 + lane];
        }
        const int64_t lo = g0 > c_lo ? g0 : c_lo;
        const int64_t hi = g1 < c_hi ? g1 : c_hi;
        const bool piece = (lo > g0) || (hi < g1);

        double acc = 0.0;
        if (lo < hi) {
            // ---- phase table of the group
            int nph = 0;
            {
                uint32_t t0 = 0;
                int32_t off = 0;
                bool live = len > 0;
                unsigned mask = __ballot_sync(FULL, live);
                while (mask) {
                    const int k = __popc(mask);
                    const uint32_t t1 = __reduce_min_sync(FULL, live ? len : 0xffffffffu);
                    if (lane == nph) {
                        S.ph_off[nph] = off;
                        S.ph_k[nph] = k;
                        S.ph_mask[nph] = mask;
                    }
                    off += (int32_t)(t1 - t0) * k;
                    ++nph;
                    t0 = t1;
                    live = len > t0;
                    mask = __ballot_sync(FULL, live);
                }
                if (lane == 0) S.ph_off[nph] = off;
                __syncwarp();
            }
            // phase containing group-relative offset lo - g0
            int j = 0;
            const int32_t o_lo = (int32_t)(lo - g0);
            while (j + 1 < nph && S.ph_off[j + 1] <= o_lo) ++j;

            int64_t pos = lo;
            while (pos < hi) {
                if (pos >= st.bnd) st.prepare(st.cur + 1);
                const int64_t seg_end = hi < st.bnd ? hi : st.bnd;
                const int32_t wa = (int32_t)(pos - g0), wb = (int32_t)(seg_end - g0);
                const double *pr = S.prod + (g0 - st.a);  // pr[o] = product at group offset o
                // walk phases overlapping [wa, wb)
                for (;;) {
                    const int32_t po = S.ph_off[j], pn = S.ph_off[j + 1];
                    const int32_t plo = wa > po ? wa : po, phi = wb < pn ? wb : pn;
                    const int k = S.ph_k[j];
                    const unsigned pm = S.ph_mask[j];
                    const bool live = (pm >> lane) & 1u;
                    const int rank = __popc(pm & lt);
                    // lane-serial unless the phase is long with few live lanes
                    if (EXACT || k >= 16 || pn - po <= 8 * k) {
                        if (live && plo < phi) {
                            // first own step at or after plo (plo == po: step 0)
                            int32_t p = po + rank;
                            if (plo != po) {
                                const int32_t rel = plo - p;
                                if (rel > 0) p += ceil_div_small(rel, k) * k;
                            }
                            for (; p < phi; p += k)
                                acc = EXACT ? __dadd_rn(acc, pr[p]) : acc + pr[p];
                        }
                    } else {
                        const int SS = c_streams[k];
                        const int s = (int)(((uint32_t)lane * c_magic16[k]) >> 16);  // lane / k
                        const int r = lane - s * k;
                        double v = 0.0;
                        if (s < SS && plo < phi) {
                            const int32_t rel = plo - po - r;
                            int32_t t = rel > 0 ? ceil_div_small(rel, k) : 0;
                            t += (s - t) & (SS - 1);  // next step of sub-stream s
                            const int32_t stride = SS * k;
                            int32_t p = po + t * k + r;
                            double v1 = 0.0;
                            for (; p + stride < phi; p += 2 * stride) {
                                v += pr[p];
                                v1 += pr[p + stride];
                            }
                            if (p < phi) v += pr[p];
                            v += v1;
                        }
                        for (int d = SS >> 1; d >= 1; d >>= 1) v += __shfl_down_sync(FULL, v, d * k);
                        const double tot = __shfl_sync(FULL, v, live ? rank : 0);
                        if (live) acc += tot;
                    }
                    if (pn <= wb && j + 1 < nph) ++j;
                    else break;
                }
                pos = seg_end;
            }
        }

        // ---- outputs
        const int64_t blk = g / gpb;
        const int64_t local = (g - blk * gpb) * 32 + lane;
        const int64_t br = f.blk_br[blk];
        const bool valid = local < f.rows - br * R;
        if (!piece) {
            if (valid) {
                if (partial) partial[blk * R + row_local] = acc;
                else y[br * R + row_local] = (V)acc;
            }
            continue;
        }
        // fast mode only: a piece of a group cut by slice boundaries
        double *slotp = (lo > g0) ? b.part_head + w * 32 : b.part_tail + w * 32;
        __stcg(slotp + lane, acc);
        __threadfence();
        __syncwarp();
        uint32_t done = 0;
        if (lane == 0) {
            const uint32_t n = (uint32_t)(hi - lo);
            const uint32_t old = atomicAdd(b.counters + g, n);
            done = (old + n == (uint32_t)(g1 - g0));
        }
        done = __shfl_sync(FULL, done, 0);
        if (!done) continue;
        __threadfence();
        int64_t wa = (int64_t)((__int128)g0 * Nw / E);
        while (wa + 1 < Nw && cut_at(wa + 1, E, Nw) <= g0) ++wa;
        while (wa > 0 && cut_at(wa, E, Nw) > g0) --wa;
        double s = __ldcg(b.part_tail + wa * 32 + lane);
        for (int64_t v = wa + 1; v < Nw; ++v) {
            s += __ldcg(b.part_head + v * 32 + lane);
            if (cut_at(v + 1, E, Nw) >= g1) break;
        }
        if (valid) {
            if (partial) partial[blk * R + row_local] = s;
            else y[br * R + row_local] = (V)s;
        }
        if (lane == 0) b.counters[g] = 0u;
    }
}

template <typename V, bool EXACT, int CH, int MINB, bool XNA>
int launch(const hbp_format_t *f, const hbp_balanced_t *b, const void *x, void *y,
           double *partial, cudaStream_t st) {
    const size_t smem = sizeof(WarpSmem<V, CH>) * kWarps;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_spmv_stream<V, EXACT, CH, MINB, XNA>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    unsigned grid = (unsigned)((b->workers + kWarps - 1) / kWarps);
    k_spmv_stream<V, EXACT, CH, MINB, XNA><<<grid, kThreads, smem, st>>>(*f, *b, (const V *)x,
                                                                      (V *)y, partial);
    return (int)cudaGetLastError();
}

template <typename V, bool EXACT, int CH, int MINB, bool XNA>
int occupancy_of(int *per_sm) {
    const size_t smem = sizeof(WarpSmem<V, CH>) * kWarps;
    cudaFuncSetAttribute(k_spmv_stream<V, EXACT, CH, MINB, XNA>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        per_sm, k_spmv_stream<V, EXACT, CH, MINB, XNA>, kThreads, smem);
}

// Tile / occupancy variants (chunk CH, min CTAs per SM), chosen with the
// environment variable HBP_STREAM_VARIANT for sweeps; 0 is the default.
constexpr int kVariants = 9;
int variant() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("HBP_STREAM_VARIANT");
        v = e ? atoi(e) : 0;
        if (v < 0 || v >= kVariants) v = 0;
    }
    return v;
}

#define HBP_STREAM_VARIANTS(FN, V, EXACT, ...)          \
    switch (variant()) {                                 \
        case 1: return FN<V, EXACT, 256, 4, false>(__VA_ARGS__); \
        case 5: return FN<V, EXACT, 256, 3, false>(__VA_ARGS__); \
        case 6: return FN<V, EXACT, 256, 4, true>(__VA_ARGS__); \
        case 7: return FN<V, EXACT, 128, 4, true>(__VA_ARGS__); \
        case 8: return FN<V, EXACT, 512, 2, true>(__VA_ARGS__); \
        case 2: return FN<V, EXACT, 128, 4, false>(__VA_ARGS__); \
        case 3: return FN<V, EXACT, 512, 2, false>(__VA_ARGS__); \
        case 4: return FN<V, EXACT, 128, 6, false>(__VA_ARGS__); \
        default: return FN<V, EXACT, 256, 3, true>(__VA_ARGS__); \
    }

template <typename V, bool EXACT>
int occupancy(int *per_sm) {
    HBP_STREAM_VARIANTS(occupancy_of, V, EXACT, per_sm)
}

template <typename V, bool EXACT>
int run(const hbp_format_t *f, const hbp_balanced_t *b, const void *x, void *y, double *partial,
        cudaStream_t st) {
    HBP_STREAM_VARIANTS(launch, V, EXACT, f, b, x, y, partial, st)
}

}  // namespace

extern "C" {

int hbp_stream_workers(const hbp_format_t *f, int64_t *workers) {
    if (!f) return HBP_E_ARG;
    int dev = 0, sms = 0, per_sm = 0;
    HBP_CUDA_TRY(cudaGetDevice(&dev));
    HBP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const bool exact = f->exact != 0 || f->dtype == HBP_F64;
    int rc;
    if (f->dtype == HBP_F64) rc = exact ? occupancy<double, true>(&per_sm) : occupancy<double, false>(&per_sm);
    else rc = exact ? occupancy<float, true>(&per_sm) : occupancy<float, false>(&per_sm);
    if (rc) return rc;
    int64_t wmax = (int64_t)sms * per_sm * kWarps;
    int64_t wcap = f->nnz / 1024;
    if (wcap < 1) wcap = 1;
    *workers = wmax < wcap ? wmax : wcap;
    return HBP_OK;
}

int hbp_spmv_stream(const hbp_format_t *f, const hbp_balanced_t *b, const void *x, void *y,
                    double *partial, hbp_stream_t stream) {
    if (!f || !b || b->workers < 1) return HBP_E_ARG;
    if (f->warp_size != 32 || f->row_height % 32) return HBP_E_UNSUPPORTED;
    if (!partial && (!y || f->ncb != 1)) return HBP_E_ARG;
    if (f->nzb == 0) return HBP_OK;
    const bool exact = f->exact != 0 || f->dtype == HBP_F64;
    if (!exact && (!b->part_head || !b->part_tail || !b->counters)) return HBP_E_ARG;
    cudaStream_t st = as_stream(stream);
    if (f->dtype == HBP_F64)
        return exact ? run<double, true>(f, b, x, y, partial, st)
                     : run<double, false>(f, b, x, y, partial, st);
    if (f->dtype == HBP_F32)
        return exact ? run<float, true>(f, b, x, y, partial, st)
                     : run<float, false>(f, b, x, y, partial, st);
    return HBP_E_ARG;
}

}  // extern "C"
