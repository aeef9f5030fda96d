// hbp_spmv_stream.cu -- TMA-streamed, element-balanced HBP SpMV (W = 32).
//
// Why: in the HBP layout a group's elements are step-major (all live lanes'
// t-th elements, then the (t+1)-th ...).  On skewed matrices a group has ~10
// "phases" (step ranges with a fixed live-lane set) and few live lanes, so a
// lane-per-row walk over global memory pays dependent DRAM round trips (col,
// then x) per phase.  Here memory and the irregular walk are decoupled:
//
//   1. each persistent warp owns an equal slice [c_lo, c_hi) of the element
//      array (exact mode: slice ends rounded up to group boundaries);
//   2. lane 0 streams the slice's col/data into a shared-memory ring of NB
//      chunks of CH elements with cp.async.bulk (TMA bulk copies completing
//      on per-slot mbarriers), NB-2 chunks ahead of the walk;
//   3. the x gathers of chunk c+1 are issued (registers) before the walk of
//      chunk c needs them; when the walk reaches chunk c+1 the products are
//      written over its values (f32 data: f32 products; exact f64 data:
//      __dmul_rn products), so products of the chunks the walk can touch are
//      always resident.  f32 lanes own 4 consecutive elements of a chunk,
//      f64 lanes 2L, 2L+1, 2L+64, 2L+65 (conflict-free 16-byte accesses).
//      With hot-column staging (hbp_hot.cu) the gathers of the heaviest
//      columns read the SM's shared copy of x, and past L2 a warm tier reads
//      a compact evict-last copy;
//   4. each group's phases come precomputed from the phase stream (live mask
//      and element offset per phase, hbp_phase_emit), one phase per lane
//      register; the walk is
//        - exact mode: a step-uniform loop, every live lane adds its element
//          of the step -- each row is summed in step order, bitwise identical
//          to _kernels.py:41-46 for f64;
//        - fast mode: per phase of k live lanes, passes of S*k consecutive
//          elements (S = floor(32/k)); lane i always meets rank i mod k, keeps
//          a register sum over the phase, and one shuffle tree per phase
//          folds the S sums of each rank into the row owner's accumulator;
//   5. a group cut by a slice boundary (fast mode only) leaves per-lane
//      partials; the warp whose piece completes the group's element count
//      (atomic) adds the pieces in slice order -- deterministic.
//
// Precision (fast mode): f32 products (relative error <= u = 2^-24 each),
// consecutive pairs of a row's products added in f32 (one more rounding of
// at most u of the pair's magnitude), everything else summed in f64, one
// final rounding to f32: componentwise error <= ~3u |A||x| (1.8e-7).
#include <cuda_runtime.h>

#include <atomic>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "hbp.h"
#include "hbp_common.cuh"

constexpr int kMaxDevices = 64;

using namespace hbp;

namespace {

constexpr unsigned FULL = 0xffffffffu;
// Hot-column staging (hbp_hot.cu): one CTA per SM holds one copy
// of x at the hot columns after the warps' rings; shared memory per SM is
// capped at kHotBudget so L1 keeps room to stage the remaining x gathers.
constexpr int kHotThreads = 896;   // 28 warps at 72 registers (measured best)
constexpr int kWarmThreads = 768;  // warm-tier launches (x beyond L2): 24 warps measured best
constexpr size_t kHotBudgetDefault = 155 * 1024;   // hot tier only -> 164 KB carveout
constexpr size_t kWarmBudgetDefault = 131 * 1024;  // with a warm tier -> 132 KB carveout
constexpr size_t kPackedBudgetDefault = 185 * 1024;  // packed x -> 196 KB carveout

// Column slots: a chunk's columns are needed only until its gathers are
// issued; while chunk ready+1 is started, chunks up to ready+NB-2 are in
// flight, so NB-2 slots (rounded up to a power of two, >= 2) suffice.
// Column slots: a chunk's columns are needed only until its gathers are
// issued; while chunk ready+1 is started, chunks up to ready+NB-2 are in
// flight, so NB-2 slots (rounded up to a power of two, >= 2) suffice.
template <int NB>
struct ColSlots {
    static constexpr int value = NB <= 4 ? 2 : (NB <= 6 ? 4 : NB);
};

template <typename V, int CH, int NB>
struct __align__(16) WarpSmem {
    uint32_t col[ColSlots<NB>::value * CH];
    V val[NB * CH];  // values, then products in place
    uint32_t ph_mask[33];
    int32_t ph_off[33];
    uint64_t mbar[NB];
    // cold ring state, touched once per chunk (kept out of registers)
    const uint32_t *colg;  // f.col + base
    const V *valg;         // f.data + base
    int32_t len32;         // c_hi - base
    int32_t nchunks;
    int32_t ready;         // chunks <= ready hold products
    int32_t pending;       // chunk whose x gathers are in flight (-1: none)
    uint64_t pol_stream;   // L2 evict-first policy (element stream)
    uint64_t pol_x;        // L2 evict-last policy (x gathers; warm tier when staged)
    uint64_t pol_cold;     // L2 evict-normal policy (cold columns when staged)
};

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ceil(2^16 / k): floor(n / k) = (n * m) >> 16 exactly for n <= 32
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

__device__ __forceinline__ int32_t div_small(int32_t n, int k) {  // 0 <= n < 2^30
    if (n < (1 << 26)) return (int32_t)(((uint64_t)(uint32_t)n * c_magic32[k]) >> 32);
    return n / k;
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

// Cut v of the slicing: equal ranges of the element array per worker, or,
// with competitive pieces (np > nw), nw equal pieces of the first F
// elements (the workers' fixed chunks) followed by np - nw equal pieces of
// the rest (the ticket pool; engine.py:38-56 plan_execution on elements).
__device__ __forceinline__ int64_t piece_cut(int64_t v, int64_t E, int64_t nw, int64_t np,
                                             int64_t F) {
    if (np <= nw) return cut_at(v, E, nw);
    if (v <= nw) return (int64_t)((__int128)v * F / nw);
    return F + (int64_t)((__int128)(v - nw) * (E - F) / (np - nw));
}

// Slice of worker (or piece) w: [cut(w), cut(w+1)); exact mode rounds both
// ends up to group boundaries (every row summed by one lane in step order).
// g = the first group whose elements the slice touches.
// With hub_min > 0 (exact mode), a cut inside a group longer than hub_min
// elements stays where it is: that group is split over warps like a
// fast-mode group (the thresholded hub-row path).
__device__ __forceinline__ void stream_slice_at(const int64_t *__restrict__ gs, int64_t ngroups,
                                                int64_t E, int64_t c_lo, int64_t c_hi, bool exact,
                                                int64_t hub_min, int64_t *lo, int64_t *hi,
                                                int64_t *g0) {
    if (exact) {
        if (c_lo > 0 && c_lo < E) {
            int64_t g = upper_group(gs, ngroups, c_lo);
            if (gs[g] != c_lo && !(hub_min > 0 && gs[g + 1] - gs[g] > hub_min)) c_lo = gs[g + 1];
        }
        if (c_hi > 0 && c_hi < E) {
            int64_t g = upper_group(gs, ngroups, c_hi);
            if (gs[g] != c_hi && !(hub_min > 0 && gs[g + 1] - gs[g] > hub_min)) c_hi = gs[g + 1];
        }
    }
    int64_t g = upper_group(gs, ngroups, c_lo);
    if (!(g < ngroups && gs[g] < c_lo)) g = lower_group(gs, ngroups, c_lo);
    *lo = c_lo;
    *hi = c_hi;
    *g0 = g;
}
__device__ __forceinline__ void stream_slice(const int64_t *__restrict__ gs, int64_t ngroups,
                                             int64_t E, int64_t w, int64_t Nw, bool exact,
                                             int64_t hub_min, int64_t *lo, int64_t *hi,
                                             int64_t *g0, int64_t np = 0, int64_t F = 0) {
    stream_slice_at(gs, ngroups, E, piece_cut(w, E, Nw, np, F), piece_cut(w + 1, E, Nw, np, F),
                    exact, hub_min, lo, hi, g0);
}

// Element offset of the cost-balanced cut v of Nw: the cost prefix cp
// (exclusive, per group; a group's fixed cost sits at its start, then one
// unit per element) reaches v * total / Nw.
__device__ __forceinline__ int64_t cost_cut(const int64_t *__restrict__ gs,
                                            const int64_t *__restrict__ cp, int64_t ngroups,
                                            int64_t E, int64_t v, int64_t Nw, int64_t np = 0,
                                            int64_t Fc = 0) {
    const int64_t n = np > Nw ? np : Nw;
    if (v <= 0) return 0;
    if (v >= n) return E;
    const int64_t tot = cp[ngroups];
    int64_t T;
    if (np > Nw) {  // Nw pieces of the first Fc cost units, then np - Nw of the rest
        const int64_t F = Fc < 0 ? 0 : (Fc > tot ? tot : Fc);
        T = v <= Nw ? (int64_t)((__int128)v * F / Nw)
                    : F + (int64_t)((__int128)(v - Nw) * (tot - F) / (np - Nw));
    } else {
        T = (int64_t)((__int128)v * tot / Nw);
    }
    int64_t lo = 0, hi = ngroups;  // largest g < ngroups with cp[g] <= T
    while (hi - lo > 1) {
        const int64_t m = (lo + hi) >> 1;
        if (cp[m] <= T) lo = m;
        else hi = m;
    }
    const int64_t len = gs[lo + 1] - gs[lo];
    const int64_t fixed = (cp[lo + 1] - cp[lo]) - len;
    int64_t off = T - cp[lo] - fixed;
    off = off < 0 ? 0 : (off > len ? len : off);
    return gs[lo] + off;
}

// one thread per slice (per piece when np > Nw); cost-balanced cuts when a
// cost prefix is given
__global__ void k_stream_slices(const int64_t *__restrict__ gs, int64_t ngroups, int64_t E,
                                int64_t Nw, bool exact, int64_t hub_min,
                                int64_t *__restrict__ slice_lo, int64_t *__restrict__ slice_g,
                                int64_t np, int64_t F, const int64_t *__restrict__ cp) {
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = np > Nw ? np : Nw;
    if (w >= n) return;
    int64_t lo, hi, g;
    if (cp) {
        const int64_t c_lo = cost_cut(gs, cp, ngroups, E, w, Nw, np, F);
        const int64_t c_hi = cost_cut(gs, cp, ngroups, E, w + 1, Nw, np, F);
        stream_slice_at(gs, ngroups, E, c_lo, c_hi, exact, hub_min, &lo, &hi, &g);
    } else {
        stream_slice(gs, ngroups, E, w, Nw, exact, hub_min, &lo, &hi, &g, np, F);
    }
    slice_lo[w] = lo;
    slice_g[w] = g;
    if (w == n - 1) slice_lo[n] = hi;
}

// hbp_group_costs: one warp per group -- lanes count the group's staged (hot)
// elements, lane 0 classifies its phases as the walk does (one- / two-step,
// modular passes for k < 12 live lanes over more than 4 steps, step loop)
__global__ void k_group_costs(const int64_t *__restrict__ gs, const int64_t *__restrict__ pptr,
                              const uint2 *__restrict__ phs, const uint32_t *__restrict__ scol,
                              int64_t ngroups, int64_t wg, int64_t ws, int64_t wt, int64_t wm,
                              int64_t wh, int64_t *__restrict__ cost) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < ngroups;
         g += nwarps) {
        const int64_t e0 = gs[g], len = gs[g + 1] - e0;
        int64_t hot = 0;
        if (scol && wh)
            for (int64_t e = lane; e < len; e += 32) hot += (__ldcs(scol + e0 + e) & HBP_HOT_FLAG) != 0;
        for (int o = 16; o; o >>= 1) hot += __shfl_xor_sync(0xffffffffu, hot, o);
        if (lane == 0) {
            const int64_t p0 = pptr[g], p1 = pptr[g + 1];
            int64_t nshort = 0, nstep = 0, nmod = 0;
            for (int64_t j = p0; j < p1; ++j) {
                const uint2 ph = phs[j];
                const int64_t end = j + 1 < p1 ? (int64_t)phs[j + 1].y : len;
                const int k = __popc(ph.x);
                const int64_t n = end - (int64_t)ph.y;
                if (n <= 2 * k) ++nshort;
                else if (k < 12 && n > 4 * k) ++nmod;
                else ++nstep;
            }
            cost[g] = len - ((hot * wh) >> 6) + wg + ws * nshort + wt * nstep + wm * nmod;
        }
    }
}

template <typename V, bool EXACT>
__device__ __forceinline__ V product(V v, V xv) {
    if (EXACT) return (V)__dmul_rn((double)v, (double)xv);
    return v * xv;
}

// Streams one warp's slice through the shared-memory ring.  All positions
// are 32-bit offsets relative to `base` (slice start rounded down to 16 B).
// Only res32 and the in-flight gathers live in registers; the rest of the
// ring state sits in the warp's shared block and is read once per chunk.
// x gather of a staged column: HBP_HOT_FLAG | s reads the CTA's shared copy
// of x at hot slot s, anything else x[c] from global memory (no L1 line).
__device__ __forceinline__ float ld_x_staged(const float *x, uint32_t hot_base, uint32_t c,
                                             uint64_t pol) {
    float v;
    asm volatile(
        "{\n.reg .pred p;\n"
        "setp.lt.s32 p, %3, 0;\n"
        "@p ld.shared.f32 %0, [%4];\n"
        "@!p ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;\n}"
        : "=f"(v)
        : "l"(x + c), "l"(pol), "r"(c), "r"(hot_base + ((c & 0x7fffffffu) << 2)));
    return v;
}
__device__ __forceinline__ double ld_x_staged(const double *x, uint32_t hot_base, uint32_t c,
                                              uint64_t pol) {
    double v;
    asm volatile(
        "{\n.reg .pred p;\n"
        "setp.lt.s32 p, %3, 0;\n"
        "@p ld.shared.f64 %0, [%4];\n"
        "@!p ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;\n}"
        : "=d"(v)
        : "l"(x + c), "l"(pol), "r"(c), "r"(hot_base + ((c & 0x7fffffffu) << 3)));
    return v;
}

// Staged gather (hot + warm tiers, hbp_hot.cu): HBP_HOT_FLAG | s reads the
// CTA's shared copy, HBP_WARM_FLAG | w the compact warm copy xw[w] (L2
// evict-last), anything else x[c] (L2 evict-normal); global loads skip L1.
template <typename V>
__device__ __forceinline__ V ld_x_tiered(const V *x, const V *xw, uint32_t hot_base, uint32_t c,
                                         uint64_t pol_warm, uint64_t pol_cold) {
    const bool warm = (c & HBP_WARM_FLAG) != 0;
    const V *g = warm ? xw + (c & 0x3fffffffu) : x + c;
    const uint64_t pol = warm ? pol_warm : pol_cold;
    const uint32_t hs = hot_base + ((c & 0x7fffffffu) * (uint32_t)sizeof(V));
    V v;
    if constexpr (sizeof(V) == 4)
        asm volatile(
            "{\n.reg .pred p;\n"
            "setp.lt.s32 p, %3, 0;\n"
            "@p ld.shared.f32 %0, [%4];\n"
            "@!p ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;\n}"
            : "=f"(v)
            : "l"(g), "l"(pol), "r"(c), "r"(hs));
    else
        asm volatile(
            "{\n.reg .pred p;\n"
            "setp.lt.s32 p, %3, 0;\n"
            "@p ld.shared.f64 %0, [%4];\n"
            "@!p ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;\n}"
            : "=d"(v)
            : "l"(g), "l"(pol), "r"(c), "r"(hs));
    return v;
}

template <typename V, bool EXACT, int CH, int NB, int XM, bool HOT>
struct Ring {
    static_assert((NB & (NB - 1)) == 0 && (CH & (CH - 1)) == 0, "NB, CH: powers of two");
    static constexpr int RMASK = NB * CH - 1;
    static constexpr int EPL = CH / 32;  // elements per lane per chunk
    static constexpr int NCOL = ColSlots<NB>::value;
    // f64 (XM & 2048): lane L owns elements 2L, 2L+1, 2L+64, 2L+65 of a chunk,
    // so the product pass's 16-byte shared accesses are contiguous across lanes
    // (4 instead of 8 wavefronts each); f32 keeps 4 consecutive per lane
    static constexpr bool PAIR = sizeof(V) == 8 && EPL == 4 && (XM & 2048) != 0;
    __device__ __forceinline__ int elem_of(int e) const {
        return PAIR ? 2 * lane + (e & 1) + 64 * (e >> 1) : EPL * lane + e;
    }
    WarpSmem<V, CH, NB> &S;
    const V *__restrict__ x;
    uint32_t hot_base = 0;  // shared address of the staged x (HOT)
    const V *xw = nullptr;  // warm tier (HOT)
    int32_t res32 = 0;  // products resident for offsets < res32
    int lane;
    V xr[EPL];          // gathered x of the pending chunk

    // lane 0: bulk-copy chunk c (< nchunks) into its slot
    __device__ __forceinline__ void issue(int32_t c, int32_t nchunks, int32_t len32) {
        const int slot = c & (NB - 1);
        uint32_t bc = CH * 4, bv = CH * (uint32_t)sizeof(V);
        if (c == nchunks - 1) {
            const int32_t n = len32 - c * CH;
            bc = (uint32_t)((n * 4 + 15) & ~15);
            bv = (uint32_t)((n * (int)sizeof(V) + 15) & ~15);
        }
        const uint64_t pe = policy_evict_first();  // created in place: no smem load + R2UR
        mbar_expect_tx(&S.mbar[slot], bc + bv);
        bulk_g2s(&S.col[(c & (NCOL - 1)) * CH], S.colg + (int64_t)c * CH, bc, &S.mbar[slot], pe);
        bulk_g2s(&S.val[slot * CH], S.valg + (int64_t)c * CH, bv, &S.mbar[slot], pe);
    }

    // chunk c: wait for its bytes, issue its x gathers into xr
    __device__ __forceinline__ void start(int32_t c, int32_t nchunks, int32_t len32) {
        const int slot = c & (NB - 1);
        mbar_wait(&S.mbar[slot], (uint32_t)((c / NB) & 1));
        uint32_t cc[EPL];
        const uint32_t *cs = &S.col[(c & (NCOL - 1)) * CH + EPL * lane];
        if constexpr (PAIR) {  // elements 2L, 2L+1, 2L+64, 2L+65
            const uint32_t *cp = &S.col[(c & (NCOL - 1)) * CH + 2 * lane];
            const uint2 t0 = *reinterpret_cast<const uint2 *>(cp);
            const uint2 t1 = *reinterpret_cast<const uint2 *>(cp + 64);
            cc[0] = t0.x, cc[1] = t0.y, cc[2] = t1.x, cc[3] = t1.y;
        } else if constexpr (EPL % 4 == 0) {
#pragma unroll
            for (int e = 0; e < EPL; e += 4) {
                const uint4 t = *reinterpret_cast<const uint4 *>(cs + e);
                cc[e] = t.x, cc[e + 1] = t.y, cc[e + 2] = t.z, cc[e + 3] = t.w;
            }
        } else if constexpr (EPL == 2) {
            const uint2 t = *reinterpret_cast<const uint2 *>(cs);
            cc[0] = t.x, cc[1] = t.y;
        } else {
#pragma unroll
            for (int e = 0; e < EPL; ++e) cc[e] = cs[e];
        }
        if (c == nchunks - 1) {  // never gather past the slice
            const int32_t n = len32 - c * CH;
#pragma unroll
            for (int e = 0; e < EPL; ++e)
                if (elem_of(e) >= n) cc[e] = 0u;
        }
        const uint64_t pl = policy_evict_last();
        {
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
                constexpr int XG = XM & 3;
                if constexpr ((XM & 8) != 0) {  // diagnostic: no global gathers (wrong y)
                    V hv;
                    const uint32_t a = hot_base + ((cc[e] & 4095u) * (uint32_t)sizeof(V));
                    if constexpr (sizeof(V) == 4) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(hv) : "r"(a));
                    else asm volatile("ld.shared.f64 %0, [%1];" : "=d"(hv) : "r"(a));
                    xr[e] = hv;
                } else if constexpr (HOT && (XM & 32) != 0) {  // + warm tier
                    xr[e] = ld_x_tiered(x, xw, hot_base, cc[e], pl, S.pol_cold);
                } else if constexpr (HOT) xr[e] = ld_x_staged(x, hot_base, cc[e], pl);
                else xr[e] = XG ? ld_x_na(x + cc[e], pl) : ld_x(x + cc[e], pl);
            }
        }
    }

    // chunk c (pending): values -> products (in place)
    __device__ __forceinline__ void finish(int32_t c) {
        if constexpr (PAIR) {  // two conflict-free 16-byte accesses per lane
            V *v = &S.val[(c & (NB - 1)) * CH + 2 * lane];
            double2 t0 = *reinterpret_cast<double2 *>(v);
            double2 t1 = *reinterpret_cast<double2 *>(v + 64);
            t0.x = (double)product<V, EXACT>((V)t0.x, xr[0]);
            t0.y = (double)product<V, EXACT>((V)t0.y, xr[1]);
            t1.x = (double)product<V, EXACT>((V)t1.x, xr[2]);
            t1.y = (double)product<V, EXACT>((V)t1.y, xr[3]);
            *reinterpret_cast<double2 *>(v) = t0;
            *reinterpret_cast<double2 *>(v + 64) = t1;
            return;
        }
        V *v = &S.val[(c & (NB - 1)) * CH + EPL * lane];
        if constexpr (sizeof(V) == 4 && EPL % 4 == 0) {
#pragma unroll
            for (int e = 0; e < EPL; e += 4) {
                float4 t = *reinterpret_cast<float4 *>(v + e);
                t.x = (float)product<V, EXACT>((V)t.x, xr[e]);
                t.y = (float)product<V, EXACT>((V)t.y, xr[e + 1]);
                t.z = (float)product<V, EXACT>((V)t.z, xr[e + 2]);
                t.w = (float)product<V, EXACT>((V)t.w, xr[e + 3]);
                *reinterpret_cast<float4 *>(v + e) = t;
            }
        } else if constexpr (sizeof(V) == 4 && EPL == 2) {
            float2 t = *reinterpret_cast<float2 *>(v);
            t.x = (float)product<V, EXACT>((V)t.x, xr[0]);
            t.y = (float)product<V, EXACT>((V)t.y, xr[1]);
            *reinterpret_cast<float2 *>(v) = t;
        } else if constexpr (sizeof(V) == 8 && EPL % 2 == 0) {
#pragma unroll
            for (int e = 0; e < EPL; e += 2) {
                double2 t = *reinterpret_cast<double2 *>(v + e);
                t.x = (double)product<V, EXACT>((V)t.x, xr[e]);
                t.y = (double)product<V, EXACT>((V)t.y, xr[e + 1]);
                *reinterpret_cast<double2 *>(v + e) = t;
            }
        } else {
#pragma unroll
            for (int e = 0; e < EPL; ++e) v[e] = product<V, EXACT>(v[e], xr[e]);
        }
    }

    // make offsets < need resident (warp-uniform); refills the ring
    __device__ __forceinline__ void advance(int32_t need) {
        if (need <= res32) return;
        const int32_t nchunks = S.nchunks, len32 = S.len32;
        int32_t ready = S.ready, pending = S.pending;
        while (need > res32) {
            if (pending < 0) {
                if (ready + 1 >= nchunks) break;
                start(ready + 1, nchunks, len32);
                pending = ready + 1;
            }
            __syncwarp();  // the walk's reads of the oldest slot are done
            finish(pending);
            ready = pending;
            pending = -1;
            res32 = (ready * CH + CH < len32 ? ready * CH + CH : len32);
            fence_proxy_async();  // generic ring accesses precede later bulk writes
            __syncwarp();
            if (ready + 1 < nchunks) {
                start(ready + 1, nchunks, len32);
                pending = ready + 1;
            }
            // the slot of chunk ready - 2 is free (the walk may still read
            // ready - 1 for a step straddling the boundary)
            if (lane == 0 && ready + NB - 2 < nchunks) issue(ready + NB - 2, nchunks, len32);
        }
        __syncwarp();
        if (lane == 0) {
            S.ready = ready;
            S.pending = pending;
        }
        __syncwarp();
    }

    __device__ __forceinline__ double at(int32_t o) const { return (double)S.val[o & RMASK]; }
    __device__ __forceinline__ V raw(int32_t o) const { return S.val[o & RMASK]; }
    // two products added in the value type (f32: one extra rounding), then widened
    __device__ __forceinline__ double at2(int32_t o1, int32_t o2) const {
        return (double)(S.val[o1 & RMASK] + S.val[o2 & RMASK]);
    }
};

// Fast-mode walk of one group (or the piece [lo_r, hi_r) of it).  Phase j's
// live mask and start offset sit in lane j's `ph`.  Per phase of k live lanes:
//   - k < KT and more than LMIN steps: passes of stride = S*k consecutive
//     elements (S = floor(32/k)); lane i takes element q + i, whose rank is
//     i mod k in every pass, so each lane keeps one register sum for the phase;
//     a deterministic shuffle tree folds the S sums of a rank and the row's
//     owner lane takes its rank's total;
//   - otherwise step by step: each live lane adds its element of the step.
template <bool PIECE, int KT, int LMIN, bool SHORT, class RingT>
__device__ __forceinline__ double walk_fast(RingT &ring, const uint2 ph, const int np,
                                            const int32_t gb, const int32_t gend,
                                            const int32_t lo_r, const int32_t hi_r,
                                            const int lane) {
    const unsigned lt = lanemask_lt();
    double acc = 0.0;
    int j = 0;
    if (PIECE)  // phase containing lo
        j = __popc(__ballot_sync(FULL, lane < np && (int32_t)ph.y <= lo_r - gb)) - 1;
    int32_t ps = gb + (int32_t)__shfl_sync(FULL, ph.y, j);
    for (;;) {
        const unsigned pm = __shfl_sync(FULL, ph.x, j);
        const int32_t pe_o = (int32_t)__shfl_sync(FULL, ph.y, (j + 1) & 31);
        const int32_t pe = gb + (j + 1 < np ? pe_o : gend);
        const int k = __popc(pm);
        const int32_t stop = PIECE ? (pe < hi_r ? pe : hi_r) : pe;
        if (SHORT && !PIECE && pe - ps <= 2 * k) {
            // one- or two-step phase (most phases on skewed rows, few
            // elements): each live lane adds its one or two elements; same
            // arithmetic as the step loop below (pair added in f32)
            if (pe > ring.res32) ring.advance(pe);
            if ((pm >> lane) & 1u) {
                const int32_t P = ps + __popc(pm & lt);
                if (pe - ps > k) acc += ring.at2(P, P + k);
                else acc += ring.at(P);
            }
        } else if (k < KT && pe - ps > LMIN * k) {
            const uint32_t mk = c_magic16[k];
            const int SS = (int)((32u * mk) >> 16);  // floor(32 / k)
            const int32_t stride = SS * k;
            int32_t q = ps;
            if (PIECE && lo_r > ps) q = ps + ((lo_r - ps) / stride) * stride;
            const bool act = lane < stride;
            double v0 = 0.0, v1 = 0.0;
            if constexpr (!PIECE) {
                // whole phase: tight double passes over the resident window, the
                // ring advance outside the inner loop (same sums as below)
                for (;;) {
                    const int32_t lim = ring.res32 < stop ? ring.res32 : stop;
                    for (; q + 2 * stride <= lim; q += 2 * stride)
                        if (act) v0 += ring.at2(q + lane, q + stride + lane);
                    if (q >= stop) break;
                    const int32_t need = q + 2 * stride < stop ? q + 2 * stride : stop;
                    if (need > ring.res32) {
                        ring.advance(need);
                        continue;
                    }
                    const int32_t P0 = q + lane, P1 = q + stride + lane;  // last, partial
                    if (act && P1 < stop) v0 += ring.at2(P0, P1);
                    else if (act && P0 < stop) v0 += ring.at(P0);
                    break;
                }
            }
            for (; PIECE && q < stop; q += 2 * stride) {
                const int32_t q2 = q + stride;
                const int32_t need = q2 + stride < stop ? q2 + stride : stop;
                if (need > ring.res32) ring.advance(need);
                const int32_t P0 = q + lane, P1 = q2 + lane;
                if (!PIECE && P1 < stop) {
                    if (act) v0 += ring.at2(P0, P1);
                } else {
                    if (act && P0 < stop && (!PIECE || P0 >= lo_r)) v0 += ring.at(P0);
                    if (act && P1 < stop && (!PIECE || P1 >= lo_r)) v1 += ring.at(P1);
                }
            }
            double v = v0 + v1;
            if (SS > 1) {
                const int s = (int)(((uint32_t)lane * mk) >> 16);  // lane / k
                for (int d = 1; d < SS; d <<= 1) {
                    const double o = __shfl_down_sync(FULL, v, d * k);
                    if ((s & (2 * d - 1)) == 0 && s + d < SS) v += o;
                }
            }
            const double tot = __shfl_sync(FULL, v, __popc(pm & lt));
            if ((pm >> lane) & 1u) acc += tot;
        } else if (!PIECE) {
            // whole phase, steps end exactly at pe: bound checks merged with
            // the residency limit, two steps per iteration
            const bool live = (pm >> lane) & 1u;
            const int32_t P0 = ps + __popc(pm & lt);
            int32_t pb = 0;  // element offset of the step within the phase
            const int32_t plen = pe - ps;
            for (;;) {
                int32_t lim = ring.res32 - ps;
                lim = lim < plen ? lim : plen;
                for (; pb + 2 * k <= lim; pb += 2 * k) {
                    if (live) acc += ring.at2(P0 + pb, P0 + pb + k);
                }
                if (pb + k <= lim) {
                    if (live) acc += ring.at(P0 + pb);
                    pb += k;
                }
                if (pb >= plen) break;
                ring.advance(ps + pb + k);
            }
        } else {
            const bool live = (pm >> lane) & 1u;
            const int32_t rank = __popc(pm & lt);
            int32_t pb = ps;
            if (lo_r > ps) pb = ps + div_small(lo_r - ps, k) * k;
            for (; pb < stop; pb += k) {
                const int32_t need = pb + k < stop ? pb + k : stop;
                if (need > ring.res32) ring.advance(need);
                const int32_t P = pb + rank;
                if (live && P < stop && P >= lo_r) acc += ring.at(P);
            }
        }
        if ((PIECE && stop < pe) || ++j == np) break;  // reached hi, or the group's end
        ps = pe;
    }
    return acc;
}

template <typename V, bool EXACT, int CH, int NB, int MINB, int XM, int KT, int LMIN, int NT,
          bool HOT>
__global__ void __launch_bounds__(NT, MINB)
    k_spmv_stream(const hbp_format_t f, const hbp_balanced_t b, const V *__restrict__ x,
                  V *__restrict__ y, double *__restrict__ partial) {
    constexpr int kWarps = NT / 32;
    // XM & 4: group metadata and y are touched once -> L2 evict-first, so
    // they do not displace x (evict-last) from L2
    constexpr bool MS = (XM & 4) != 0;
    constexpr bool SHORT = (XM & 16) != 0;  // fast path for 1-2 step phases
    constexpr bool FC = (XM & 512) != 0;     // fused combine (b.rb_done; partial mode)
    constexpr bool HUBT = EXACT && (XM & 4096) != 0;  // exact mode with the hub-row path
    auto ldm = [](const auto *p) { return MS ? __ldcs(p) : *p; };
    auto stm = [](auto *p, auto v) {
        if constexpr (MS) __stcs(p, v);
        else *p = v;
    };
    // a row of y, and its copies in the peers' buffers (hbp_balanced_t.y_peer:
    // the fused power iteration's all-gather; plain stores over NVLink)
    auto sty = [&](V *yrow, int64_t r, V v) {
        stm(yrow, v);
        if (b.n_peers) {
#pragma unroll
            for (int p = 0; p < HBP_MAX_PEERS; ++p)
                if (p < b.n_peers) stm(static_cast<V *>(b.y_peer[p]) + r, v);
        }
    };
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    using Smem = WarpSmem<V, CH, NB>;
    Smem &S = reinterpret_cast<Smem *>(smem_raw)[wib];
    V *const hot = reinterpret_cast<V *>(smem_raw + sizeof(Smem) * kWarps);
    if constexpr (HOT) {  // stage x at the hot columns (b.x_hot, hbp_hot_gather)
        // launched as a programmatic dependent of k_hot_gather: everything
        // above ran while the gather finished; its x_hot is visible after this
        // (a tail launch, piece_base > 0, depends on the main launch, which only
        // triggers it after this wait -- so it must not wait for that launch)
        if (b.piece_base == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
        const int32_t nv = (int32_t)(f.n_hot * (int64_t)sizeof(V) / 16);
        const uint4 *src = (const uint4 *)b.x_hot;
        for (int32_t i = threadIdx.x; i < nv; i += NT) reinterpret_cast<uint4 *>(hot)[i] = __ldcg(src + i);
        __syncthreads();
    }
    // the tail launch (if any) may be scheduled now: its CTAs take the SMs
    // this launch's CTAs free
    if (b.tail && b.piece_base == 0) asm volatile("griddepcontrol.launch_dependents;");
    const int64_t w0 = b.warp_map ? (int64_t)wib * gridDim.x + blockIdx.x
                                  : (int64_t)blockIdx.x * kWarps + wib;
    const int64_t Nw = b.workers;
    if (w0 >= Nw) return;
    if (b.warp_ns && lane == 0) b.warp_ns[2 * w0] = globaltimer_ns();
    // XM & 8192: competitive pieces -- warp w0 runs piece w0 (its fixed chunk),
    // then claims pieces Nw.. with the ticket (engine.py:155-165 on slices)
    constexpr bool TK = (XM & 8192) != 0;
    // total pieces (the slice table's size): competitive (TK) or tail pieces
    const int64_t Np = (TK || b.pieces > Nw) ? b.pieces : Nw;
    const int32_t R = (int32_t)f.row_height, gpb = R / 32;
    const int64_t ngroups = f.nzb * gpb;
    const int64_t E = f.nnz;
    const int64_t *__restrict__ gs = f.group_start;
    const int64_t *__restrict__ pptr = f.phase_ptr;
    const uint2 *__restrict__ phs = (const uint2 *)f.phases;
    const uint32_t *__restrict__ permp = (const uint32_t *)f.perm;

    for (int64_t w = w0 + (TK ? 0 : b.piece_base), np_done = 0;; ++np_done) {
    int64_t c_lo, c_hi, g;
    if (b.slice_lo) {  // precomputed (hbp_stream_slices): no binary searches here
        c_lo = b.slice_lo[w];
        c_hi = b.slice_lo[w + 1];
        g = b.slice_g[w];
    } else {
        stream_slice(gs, ngroups, E, w, Nw, EXACT, EXACT ? b.hub_min : 0, &c_lo, &c_hi, &g);
    }
    const int64_t base = c_lo & ~(int64_t)3;
    Ring<V, EXACT, CH, NB, XM, HOT> ring{S, x};
    ring.lane = lane;
    if constexpr (HOT) {
        ring.hot_base = smem_addr(hot);
        ring.xw = (const V *)b.x_hot + f.n_hot;
    }
    const int32_t len32 = (int32_t)(c_hi - base);
    const int32_t lo_s = (int32_t)(c_lo - base);  // slice start (0..3)
    if (TK && np_done) {  // the previous piece's ring is drained (every chunk waited)
        fence_proxy_async();
        __syncwarp();
    }
    if (lane == 0) {
        const int32_t nchunks = c_hi > c_lo ? (len32 + CH - 1) / CH : 0;
        if (TK && np_done)
            for (int i = 0; i < NB; ++i) mbar_inval(&S.mbar[i]);
        S.colg = (HOT ? f.scol : f.col) + base;
        S.valg = (const V *)f.data + base;
        S.len32 = len32;
        S.nchunks = nchunks;
        S.ready = -1;
        S.pending = -1;
        S.pol_stream = policy_evict_first();
        S.pol_x = policy_evict_last();
        S.pol_cold = f.cold_last ? policy_evict_last() : policy_evict_normal();
        for (int i = 0; i < NB; ++i) mbar_init(&S.mbar[i], 1);
        fence_mbar_init();
        for (int c = 0; c <= NB - 3 && c < nchunks; ++c) ring.issue(c, nchunks, len32);
    }
    __syncwarp();

    const bool last_warp = (w == Np - 1);
    // y written directly is scaled by 1 / sqrt(*b.y_sumsq) when given (the
    // power iteration folds x / ||x|| into the next SpMV); 1.0 is exact
    const double ys = b.y_sumsq ? 1.0 / sqrt(*b.y_sumsq) : 1.0;
    // output position of group g: nonzero block blk, group gi within it
    int32_t blk = (int32_t)(g / gpb), gi = (int32_t)(g - (int64_t)blk * gpb);
    // the group loop in 32 bits (hbp_spmv_stream rejects >= 2^31 groups)
    const int32_t ng32 = (int32_t)ngroups;
    int32_t gq = (int32_t)g;
    int32_t rows_left = 0;  // rows of block blk (<= R)
    int32_t br_cur = 0;     // its row block
    bool to_partial = false;  // outputs of block blk go to the partial (else y)
    // (output addresses are formed at the store from blk / br_cur: two 64-bit
    // pointers fewer live across the walk)
    auto enter_block = [&]() {
        if (blk < f.nzb) {
            const int64_t br = f.blk_br[blk];
            const int64_t left = f.rows - br * R;
            rows_left = (int32_t)(left < R ? left : R);
            br_cur = (int32_t)br;
            to_partial = partial != nullptr;
            // a row block with a single nonzero block needs no combine: its
            // rows go straight to y (hbp_combine then skips the row block)
            if (to_partial && !FC && (f.reserved & HBP_FLAG_DIRECT_SINGLE) &&
                f.rb_ptr[br + 1] - f.rb_ptr[br] == 1)
                to_partial = false;
        }
    };
    // Fused combine (engine.py:196-201; b.rb_done set, partial and y given):
    // every finished group counts toward its row block; the warp that
    // completes a row block's nb * gpb groups sums its partials in ascending
    // bc (the rb_blk order, as hbp_combine does -- bitwise the same) and
    // writes y, then resets the counter.
    // Groups are counted locally and published once per row block the warp
    // leaves (one fence per block, not per group).
    int32_t pend_br = -1, pend_rows = 0;
    uint32_t pend_n = 0;
    auto flush_done = [&](int32_t br, uint32_t n, int32_t nrows) {
        __syncwarp();
        __threadfence();  // this warp's partials before the count
        const int64_t lo = f.rb_ptr[br], hi = f.rb_ptr[br + 1];
        uint32_t last = 0;
        if (lane == 0) {
            const uint32_t total = (uint32_t)((hi - lo) * gpb);
            last = (atomicAdd(b.rb_done + br, n) + n == total);
        }
        if (!__shfl_sync(FULL, last, 0)) return;
        __threadfence();
        V *yr = y + (int64_t)br * R;
        // four rows per lane at a time (independent loads in flight), each
        // summed left to right over the row block's blocks
        for (int32_t r0 = 0; r0 < nrows; r0 += 128) {
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            for (int64_t i = lo; i < hi; ++i) {
                const double *pp = partial + (int64_t)f.rb_blk[i] * R + r0 + lane;
                // rows past the row block's end belong to the next block's
                // partial (or lie past the allocation for the last one)
                const int32_t r = r0 + lane;
                const double p0 = r < nrows ? __ldcg(pp) : 0.0,
                             p1 = r + 32 < nrows ? __ldcg(pp + 32) : 0.0,
                             p2 = r + 64 < nrows ? __ldcg(pp + 64) : 0.0,
                             p3 = r + 96 < nrows ? __ldcg(pp + 96) : 0.0;
                if (i == lo) a0 = p0, a1 = p1, a2 = p2, a3 = p3;
                else a0 = __dadd_rn(a0, p0), a1 = __dadd_rn(a1, p1), a2 = __dadd_rn(a2, p2),
                     a3 = __dadd_rn(a3, p3);
            }
            const int32_t r = r0 + lane;
            if (r < nrows) stm(yr + r, (V)a0);
            if (r + 32 < nrows) stm(yr + r + 32, (V)a1);
            if (r + 64 < nrows) stm(yr + r + 64, (V)a2);
            if (r + 96 < nrows) stm(yr + r + 96, (V)a3);
        }
        if (lane == 0) b.rb_done[br] = 0u;
    };
    auto group_done = [&](int32_t br, int32_t nrows) {
        if constexpr (!FC) return;
        if (br != pend_br) {
            if (pend_n) flush_done(pend_br, pend_n, pend_rows);
            pend_br = br, pend_rows = nrows, pend_n = 0;
        }
        ++pend_n;
    };
    enter_block();

    // prefetched metadata of group g: element range (base-relative), output
    // rows, phases
    int32_t gr0 = gq < ng32 ? (int32_t)(gs[gq] - base) : len32;
    int32_t gr1 = gq < ng32 ? (int32_t)(gs[gq + 1] - base) : len32;
    uint32_t perm_n = gq < ng32 ? permp[(int64_t)gq * 32 + lane] : 0u;
    // phase-stream offsets fit 32 bits (hbp_spmv_stream checks the total)
    int32_t pp0 = gq < ng32 ? (int32_t)pptr[gq] : 0;
    int32_t pp1 = gq < ng32 ? (int32_t)pptr[gq + 1] : 0;
    uint2 ph_n = make_uint2(0u, 0u);
    if (gq < ng32 && lane < pp1 - pp0) ph_n = phs[pp0 + lane];

    for (; gq < ng32 && (gr0 < len32 || last_warp); ++gq) {
        const uint32_t row_local = perm_n;
        const int32_t g0 = gr0, g1 = gr1;
        const int np = (int)(pp1 - pp0);
        const uint2 ph = ph_n;
        if (gq + 1 < ng32) {  // prefetch the next group's metadata
            gr0 = g1;
            gr1 = (int32_t)(ldm(gs + gq + 2) - base);
            perm_n = ldm(permp + (int64_t)(gq + 1) * 32 + lane);
            pp0 = pp1;
            pp1 = (int32_t)ldm(pptr + gq + 2);
            // address known now (no wait on pp1); lanes >= the phase count
            // read the next group's phases (padded stream) and are ignored
            ph_n = ldm(phs + pp0 + lane);
        }
        const int32_t lo = g0 > lo_s ? g0 : lo_s;
        const int32_t hi = g1 < len32 ? g1 : len32;
        const bool piece = (lo > g0) || (hi < g1);

        double acc = 0.0;
        // exact mode with the hub-row path: groups longer than b.hub_min are
        // walked (and split over warps) as in fast mode
        const bool hub = HUBT && (int64_t)(g1 - g0) > b.hub_min;
        if ((!EXACT || hub) && lo < hi) {
            acc = piece ? walk_fast<true, KT, LMIN, SHORT>(ring, ph, np, g0, g1 - g0, lo, hi, lane)
                        : walk_fast<false, KT, LMIN, SHORT>(ring, ph, np, g0, g1 - g0, lo, hi, lane);
        } else if (lo < hi) {
            __syncwarp();  // previous group's table reads are done
            if (lane < np) {
                S.ph_mask[lane] = ph.x;
                S.ph_off[lane] = (int32_t)ph.y;
            }
            if (lane == 0) S.ph_off[np] = g1 - g0;
            __syncwarp();
            const unsigned lt = lanemask_lt();
            // exact mode: whole groups only (slices end on group boundaries)
            int j = 0;
            unsigned pm = S.ph_mask[0];
            int k = __popc(pm);
            int32_t pend_j = g0 + S.ph_off[1];  // ring offset where phase j ends
            int32_t pb = g0;
            bool live = (pm >> lane) & 1u;
            int rank = __popc(pm & lt);

            // ---- exact mode: step-uniform lane walk, each row in step order
            while (pb < hi) {
                for (; pb < pend_j; pb += k) {
                    if (pb + k > ring.res32) ring.advance(pb + k);
                    if (live) acc = __dadd_rn(acc, ring.at(pb + rank));
                }
                if (++j == np) break;
                pm = S.ph_mask[j];
                k = __popc(pm);
                pend_j = g0 + S.ph_off[j + 1];
                live = (pm >> lane) & 1u;
                rank = __popc(pm & lt);
            }
        }

        // ---- outputs
        const int32_t gi_now = gi;
        const bool valid = gi_now * 32 + lane < rows_left;
        const int32_t br_now = br_cur, rows_now = rows_left, blk_now = blk;
        double *const pb_now = to_partial ? partial + (int64_t)blk_now * R : nullptr;
        V *const yb_now = y + (int64_t)br_now * R;
        if (++gi == gpb) {
            gi = 0;
            ++blk;
            enter_block();
        }
        if (!piece) {
            if (valid) {
                if (pb_now) pb_now[row_local] = acc;
                else sty(yb_now + row_local, (int64_t)br_now * R + row_local, (V)(acc * ys));
            }
            if (FC && pb_now) group_done(br_now, rows_now);
            continue;
        }
        // fast mode only: a piece of a group cut by slice boundaries
        const int64_t ga0 = base + g0, ga1 = base + g1;  // absolute element range
        double *slotp = (lo > g0) ? b.part_head + w * 32 : b.part_tail + w * 32;
        __stcg(slotp + lane, acc);
        __threadfence();
        __syncwarp();
        uint32_t done = 0;
        if (lane == 0) {
            const uint32_t n = (uint32_t)(hi - lo);
            const uint32_t old = atomicAdd(b.counters + gq, n);
            done = (old + n == (uint32_t)(g1 - g0));
        }
        done = __shfl_sync(FULL, done, 0);
        if (!done) continue;
        __threadfence();
        int64_t wa;
        const bool by_table = TK || b.slice_lo != nullptr;  // cuts need not be equal
        if (by_table) {  // last piece starting at or before ga0 (slice_lo sorted)
            int64_t l = 0, h = Np;
            while (h - l > 1) {
                const int64_t m = (l + h) >> 1;
                if (b.slice_lo[m] <= ga0) l = m;
                else h = m;
            }
            wa = l;
        } else {
            wa = (int64_t)((__int128)ga0 * Nw / E);
            while (wa + 1 < Nw && cut_at(wa + 1, E, Nw) <= ga0) ++wa;
            while (wa > 0 && cut_at(wa, E, Nw) > ga0) --wa;
        }
        double s = __ldcg(b.part_tail + wa * 32 + lane);
        for (int64_t v = wa + 1; v < Np; ++v) {
            s += __ldcg(b.part_head + v * 32 + lane);
            if ((by_table ? b.slice_lo[v + 1] : cut_at(v + 1, E, Nw)) >= ga1) break;
        }
        if (valid) {
            if (pb_now) pb_now[row_local] = s;
            else sty(yb_now + row_local, (int64_t)br_now * R + row_local, (V)(s * ys));
        }
        if (lane == 0) b.counters[gq] = 0u;
        if (FC && pb_now) group_done(br_now, rows_now);
    }
    if (FC && pend_n) flush_done(pend_br, pend_n, pend_rows);
    if constexpr (!TK) break;
    else {
        int64_t nxt = 0;
        if (lane == 0) {
            const uint32_t t = atomicAdd(b.ticket, 1u);
            nxt = Nw + (int64_t)t;
            // every warp draws exactly one ticket past the pool; the last such
            // draw resets the counters for the next launch
            if (nxt >= Np && atomicAdd(b.ticket + 1, 1u) + 1u == (uint32_t)Nw) {
                b.ticket[0] = 0u;
                b.ticket[1] = 0u;
            }
        }
        nxt = __shfl_sync(FULL, nxt, 0);
        if (nxt >= Np) break;
        w = nxt;
    }
    }
    if (b.n_peers) __threadfence_system();  // peer stores before the next collective
    if (b.warp_ns && lane == 0) b.warp_ns[2 * w0 + 1] = globaltimer_ns();
}

// Shared memory per SM is kept to what MINB CTAs need: the rest of the
// 256 KB unified L1/shared array stays L1, which stages the in-flight x
// gathers (measured: more shared memory -> fewer gathers in flight -> slower).
// HBP_CARVEOUT (percent of the maximum shared capacity) overrides.
template <class K>
void set_attributes(K kernel, size_t smem, int minb) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int pct = -1;
    if (const char *e = getenv("HBP_CARVEOUT")) pct = atoi(e);
    if (pct < 0) {
        int dev = 0, max_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&max_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        const size_t need = (smem + 1024) * (size_t)minb;  // + per-CTA reservation
        pct = max_sm > 0 ? (int)((need * 100 + max_sm - 1) / max_sm) : 100;
        if (pct > 100) pct = 100;
    }
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

template <typename V, int CH, int NB, int NT>
constexpr size_t ring_smem() {
    return sizeof(WarpSmem<V, CH, NB>) * (NT / 32);
}

// Kernel attributes are per device and per instantiation: the shared-memory
// size each instantiation was last configured for on each device.  Both the
// occupancy query and the launch go through here (a staged launch's size
// depends on n_hot, so a query for another matrix re-sets it).  Idempotent,
// so a lost race only repeats the call.
template <typename V, bool EXACT, int CH, int NB, int MINB, int XM, int KT, int LMIN, int NT,
          bool HOT>
int ensure_attributes(size_t smem) {
    static std::atomic<size_t> attr[kMaxDevices];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return HBP_E_ARG;
    if (attr[dev].load(std::memory_order_relaxed) != smem) {
        set_attributes(k_spmv_stream<V, EXACT, CH, NB, MINB, XM, KT, LMIN, NT, HOT>, smem, MINB);
        attr[dev].store(smem, std::memory_order_relaxed);
    }
    return HBP_OK;
}

template <typename V, bool EXACT, int CH, int NB, int MINB, int XM, int KT, int LMIN, int NT,
          bool HOT>
int launch_one(const hbp_format_t *f, const hbp_balanced_t *b, const void *x, void *y,
               double *partial, cudaStream_t st, bool pdl);

template <typename V, bool EXACT, int CH, int NB, int MINB, int XM, int KT, int LMIN, int NT,
          bool HOT>
int launch(const hbp_format_t *f, const hbp_balanced_t *b, const void *x, void *y,
           double *partial, cudaStream_t st) {
    // staged launches follow k_hot_gather as programmatic dependents
    const int r = launch_one<V, EXACT, CH, NB, MINB, XM, KT, LMIN, NT, HOT>(f, b, x, y, partial,
                                                                           st, HOT);
    if (r || !(b->tail && b->pieces > b->workers)) return r;
    // tail pieces: a second launch, one warp per piece, depending on the main
    // one programmatically (it triggers once its own dependencies are met)
    hbp_balanced_t b2 = *b;
    b2.piece_base = b->workers;
    b2.workers = b->pieces - b->workers;
    b2.warp_ns = nullptr;
    return launch_one<V, EXACT, CH, NB, MINB, XM, KT, LMIN, NT, HOT>(f, &b2, x, y, partial, st,
                                                                     true);
}

template <typename V, bool EXACT, int CH, int NB, int MINB, int XM, int KT, int LMIN, int NT,
          bool HOT>
int launch_one(const hbp_format_t *f, const hbp_balanced_t *b, const void *x, void *y,
               double *partial, cudaStream_t st, bool pdl) {
    const size_t smem = ring_smem<V, CH, NB, NT>() + (HOT ? (size_t)f->n_hot * sizeof(V) : 0);
    const int ra = ensure_attributes<V, EXACT, CH, NB, MINB, XM, KT, LMIN, NT, HOT>(smem);
    if (ra) return ra;
    unsigned grid = (unsigned)((b->workers + NT / 32 - 1) / (NT / 32));
    if (pdl) {
        // programmatic dependent launch after k_hot_gather (which triggers its
        // dependents on entry): this kernel's launch and CTA setup overlap the
        // gather's tail; griddepcontrol.wait orders the x_hot reads (a tail
        // launch depends on the main launch the same way)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(NT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return (int)cudaLaunchKernelEx(&cfg, k_spmv_stream<V, EXACT, CH, NB, MINB, XM, KT, LMIN, NT, HOT>,
                                       *f, *b, (const V *)x, (V *)y, partial);
    }
    k_spmv_stream<V, EXACT, CH, NB, MINB, XM, KT, LMIN, NT, HOT><<<grid, NT, smem, st>>>(
        *f, *b, (const V *)x, (V *)y, partial);
    return (int)cudaGetLastError();
}

template <typename V, bool EXACT, int CH, int NB, int MINB, int XM, int KT, int LMIN, int NT,
          bool HOT>
int occupancy_of(const hbp_format_t *f, int *per_sm, int *warps_per_cta) {
    const size_t smem = ring_smem<V, CH, NB, NT>() + (HOT ? (size_t)f->n_hot * sizeof(V) : 0);
    const int ra = ensure_attributes<V, EXACT, CH, NB, MINB, XM, KT, LMIN, NT, HOT>(smem);
    if (ra) return ra;
    *warps_per_cta = NT / 32;
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        per_sm, k_spmv_stream<V, EXACT, CH, NB, MINB, XM, KT, LMIN, NT, HOT>, NT, smem);
}

// Tile / occupancy variants (chunk CH, ring slots NB, min CTAs per SM,
// threads per CTA), chosen with HBP_STREAM_VARIANT for sweeps; 0 is the
// default.  Earlier sweeps (CH 64/128, L1 allocation of x, KT/LMIN of the
// modular passes) are in the git history; 128/4/3x256 with L1::no_allocate x
// gathers and KT=12, LMIN=4 won on cfg2 and H.
constexpr int kVariants = 4;
// tuning knob for A/B sweeps only (HBP_STREAM_VARIANT / hbp_stream_set_variant):
// process-wide by design, read once; every variant computes the same y
std::atomic<int> g_variant{-1};
int variant() {
    int v = g_variant.load(std::memory_order_relaxed);
    if (v < 0) {
        const char *e = getenv("HBP_STREAM_VARIANT");
        v = e ? atoi(e) : 0;
        if (v < 0 || v >= kVariants) v = 0;
        g_variant.store(v, std::memory_order_relaxed);
    }
    return v;
}

bool staged(const hbp_format_t *f) { return f->n_hot > 0 && f->scol && f->hot_cols; }
bool packed(const hbp_format_t *f) { return staged(f) && (f->reserved & HBP_FLAG_PACKED_X); }
// a warm tier (its own instantiation) -- not with a packed x, whose n_warm
// counts the packed columns gathered like plain ones
bool warm(const hbp_format_t *f) { return f->n_warm > 0 && !packed(f); }

// One variant = (chunk CH, ring slots NB, threads NT, CTAs per SM MINB, the
// XM feature bits).  f64 data always uses CH 128, NB 4.  Every launch is one CTA per SM (staged ones need one shared
// copy of x per SM): 28 warps, or 24 with a warm tier.
#define HBP_VARIANT(FN, V, EXACT, HOT, CH, NB, NT, MINB, ...)                              \
    HBP_VARIANT_X(FN, V, EXACT, HOT, CH, NB, NT, MINB, 21 | 2048, __VA_ARGS__)
#define HBP_VARIANT_X(FN, V, EXACT, HOT, CH, NB, NT, MINB, XM, ...)                         \
    return FN<V, EXACT, (sizeof(V) == 4 ? CH : 128), (sizeof(V) == 4 ? NB : 4), MINB, XM,   \
              12, 4, NT, HOT>(__VA_ARGS__)

#define HBP_VARIANTS(FN, V, EXACT, HOT, NTD, MINBD, ...)                                     \
    switch (variant()) {                                                                    \
        case 1: HBP_VARIANT_X(FN, V, EXACT, HOT, 128, 4, NTD, MINBD, 29, __VA_ARGS__);      \
        case 2: HBP_VARIANT_X(FN, V, EXACT, HOT, 128, 4, 768, 1, 21 | 2048, __VA_ARGS__);   \
        case 3: HBP_VARIANT_X(FN, V, EXACT, HOT, 128, 4, NTD, MINBD, 5, __VA_ARGS__);       \
        default: HBP_VARIANT(FN, V, EXACT, HOT, 128, 4, NTD, MINBD, __VA_ARGS__);           \
    }

// a warm tier (XM | 32) costs an address/policy select per gather, so it has
// its own instantiation
// The fused combine (XM | 512) and the warm tier (XM | 32) each have their
// own instantiation of the default variant: their bookkeeping would cost the
// direct-mode kernel registers (spills) it does not need.
// exact mode with the hub-row path (b->hub_min > 0) is its own instantiation
// (XM | 4096): the fast-mode walk it adds would cost the plain exact kernel
// registers
// competitive pieces (b->pieces > b->workers, XM | 8192) have their own
// instantiations of the default, warm and unstaged kernels
#define HBP_STREAM_DISPATCH(FN, V, EXACT, FUSED, HUB, TICKET, ...)                          \
    if (TICKET && !HUB && !FUSED) {                                                         \
        if (staged(f) && warm(f)) {                                                         \
            HBP_VARIANT_X(FN, V, EXACT, true, 128, 4, kWarmThreads, 1, 53 | 2048 | 8192, __VA_ARGS__); \
        }                                                                                   \
        if (staged(f)) {                                                                    \
            HBP_VARIANT_X(FN, V, EXACT, true, 128, 4, kHotThreads, 1, 21 | 2048 | 8192, __VA_ARGS__); \
        }                                                                                   \
        HBP_VARIANT_X(FN, V, EXACT, false, 128, 4, kHotThreads, 1, 21 | 2048 | 8192, __VA_ARGS__); \
    }                                                                                       \
    if (EXACT && HUB) {                                                                     \
        if (staged(f) && warm(f)) {                                                         \
            HBP_VARIANT_X(FN, V, EXACT, true, 128, 4, kWarmThreads, 1, 53 | 2048 | 4096, __VA_ARGS__); \
        }                                                                                   \
        if (staged(f)) {                                                                    \
            HBP_VARIANT_X(FN, V, EXACT, true, 128, 4, kHotThreads, 1, 21 | 2048 | 4096, __VA_ARGS__); \
        }                                                                                   \
        HBP_VARIANT_X(FN, V, EXACT, false, 128, 4, kHotThreads, 1, 21 | 2048 | 4096, __VA_ARGS__); \
    }                                                                                       \
    if (staged(f)) {                                                                        \
        if (FUSED && warm(f)) {                                                             \
            HBP_VARIANT_X(FN, V, EXACT, true, 128, 4, kWarmThreads, 1, 53 | 512 | 2048, __VA_ARGS__); \
        }                                                                                   \
        if (FUSED) {                                                                        \
            HBP_VARIANT_X(FN, V, EXACT, true, 128, 4, kHotThreads, 1, 21 | 512 | 2048, __VA_ARGS__); \
        }                                                                                   \
        if (warm(f)) {                                                                      \
            HBP_VARIANT_X(FN, V, EXACT, true, 128, 4, kWarmThreads, 1, 53 | 2048, __VA_ARGS__); \
        }                                                                                   \
        HBP_VARIANTS(FN, V, EXACT, true, kHotThreads, 1, __VA_ARGS__)                       \
    }                                                                                       \
    if (FUSED) {                                                                            \
        HBP_VARIANT_X(FN, V, EXACT, false, 128, 4, kHotThreads, 1, 21 | 512 | 2048, __VA_ARGS__); \
    }                                                                                       \
    HBP_VARIANTS(FN, V, EXACT, false, kHotThreads, 1, __VA_ARGS__)

template <typename V, int CH, int NB, int MINB, int NT>
int ring_bytes(size_t *out) {
    *out = ring_smem<V, (sizeof(V) == 4 ? CH : 128), (sizeof(V) == 4 ? NB : 4), NT>();
    return 0;
}
#define HBP_RING_BYTES(V, CH, NB, NT) ring_bytes<V, CH, NB, 1, NT>(out)
template <typename V>
int hot_ring_bytes(size_t *out, bool warm) {  // shared memory of the staged launch's rings
    if (warm) return HBP_RING_BYTES(V, 128, 4, kWarmThreads);
    if (variant() == 2) return HBP_RING_BYTES(V, 128, 4, 768);
    return HBP_RING_BYTES(V, 128, 4, kHotThreads);
}

template <typename V, bool EXACT>
int occupancy(const hbp_format_t *f, int *per_sm, int *warps_per_cta) {
    HBP_STREAM_DISPATCH(occupancy_of, V, EXACT, false, false, false, f, per_sm, warps_per_cta)
}

// x_hot[s] = x[hot_cols[s]]: four slots per thread (one 16-byte load of
// hot_cols, four independent gathers in flight); hot_cols / x_hot are
// 16-byte aligned (torch allocations), a tail of < 4 slots is done singly
template <typename V>
__global__ void k_hot_gather(const V *__restrict__ x, const uint32_t *__restrict__ hot_cols,
                             int64_t n_hot, V *__restrict__ x_hot) {
    // the stream kernel (a programmatic dependent) may launch now; it waits
    // for this grid's completion before reading x_hot
    asm volatile("griddepcontrol.launch_dependents;");
    const int64_t n4 = n_hot >> 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint4 c = __ldcs(reinterpret_cast<const uint4 *>(hot_cols) + i);
        const V v0 = __ldg(x + c.x), v1 = __ldg(x + c.y), v2 = __ldg(x + c.z), v3 = __ldg(x + c.w);
        V *o = x_hot + 4 * i;
        o[0] = v0, o[1] = v1, o[2] = v2, o[3] = v3;
    }
    const int64_t t = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_hot && t < (n4 << 2) + 4) x_hot[t] = __ldg(x + hot_cols[t]);
}

// x_hot[slots[i]] = x[cols[i]] with cols ascending: x is read in column
// order (coalesced runs) and the copy written by scatter (it is L2-resident)
template <typename V>
__global__ void k_hot_refresh(const V *__restrict__ x, const uint32_t *__restrict__ cols,
                              const uint32_t *__restrict__ slots, int64_t n,
                              V *__restrict__ x_hot) {
    asm volatile("griddepcontrol.launch_dependents;");
    const int64_t n4 = n >> 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint4 c = __ldcs(reinterpret_cast<const uint4 *>(cols) + i);
        const uint4 s = __ldcs(reinterpret_cast<const uint4 *>(slots) + i);
        const V v0 = __ldg(x + c.x), v1 = __ldg(x + c.y), v2 = __ldg(x + c.z), v3 = __ldg(x + c.w);
        x_hot[s.x] = v0, x_hot[s.y] = v1, x_hot[s.z] = v2, x_hot[s.w] = v3;
    }
    const int64_t t = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n && t < (n4 << 2) + 4) x_hot[slots[t]] = __ldg(x + cols[t]);
}

template <typename V>
int hot_refresh(const void *x, const uint32_t *cols, const uint32_t *slots, int64_t n,
                void *x_hot, cudaStream_t st) {
    if (n == 0) return HBP_OK;
    if (((uintptr_t)cols & 15) || ((uintptr_t)slots & 15)) return HBP_E_ARG;
    k_hot_refresh<V><<<grid_for((n + 3) / 4, 256), 256, 0, st>>>((const V *)x, cols, slots, n,
                                                                  (V *)x_hot);
    return (int)cudaGetLastError();
}

template <typename V>
int hot_gather(const void *x, const uint32_t *hot_cols, int64_t n_hot, void *x_hot,
               cudaStream_t st) {
    if (n_hot == 0) return HBP_OK;
    if (((uintptr_t)hot_cols & 15) || ((uintptr_t)x_hot & 15)) return HBP_E_ARG;
    k_hot_gather<V><<<grid_for((n_hot + 3) / 4, 256), 256, 0, st>>>((const V *)x, hot_cols,
                                                                    n_hot, (V *)x_hot);
    return (int)cudaGetLastError();
}

template <typename V, bool EXACT>
int run(const hbp_format_t *f, const hbp_balanced_t *b, const void *x, void *y, double *partial,
        cudaStream_t st) {
    if (staged(f)) {
        const int rc =
            f->refresh_cols
                ? hot_refresh<V>(x, f->refresh_cols, f->refresh_slots, f->n_hot + f->n_warm,
                                 b->x_hot, st)
                : hot_gather<V>(x, f->hot_cols, f->n_hot + f->n_warm, b->x_hot, st);
        if (rc) return rc;
        if (packed(f)) x = (const V *)b->x_hot + f->n_hot;  // gathers read the packed copy
    }
    HBP_STREAM_DISPATCH(launch, V, EXACT, (b->rb_done != nullptr), (b->hub_min > 0),
                        (b->pieces > b->workers && !b->tail), f, b, x, y, partial, st)
}

}  // namespace

extern "C" {

int hbp_stream_workers(const hbp_format_t *f, int64_t *workers) {
    if (!f) return HBP_E_ARG;
    int dev = 0, sms = 0, per_sm = 0, wpc = 0;
    HBP_CUDA_TRY(cudaGetDevice(&dev));
    HBP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const bool exact = f->exact != 0 || f->dtype == HBP_F64;
    int rc;
    if (f->dtype == HBP_F64)
        rc = exact ? occupancy<double, true>(f, &per_sm, &wpc)
                   : occupancy<double, false>(f, &per_sm, &wpc);
    else
        rc = exact ? occupancy<float, true>(f, &per_sm, &wpc)
                   : occupancy<float, false>(f, &per_sm, &wpc);
    if (rc) return rc;
    if (per_sm < 1) return HBP_E_UNSUPPORTED;  // e.g. n_hot beyond hbp_hot_capacity
    int64_t wmax = (int64_t)sms * per_sm * wpc;
    int64_t wcap = f->nnz / 1024;
    if (wcap < 1) wcap = 1;
    *workers = wmax < wcap ? wmax : wcap;
    return HBP_OK;
}

int hbp_hot_capacity(int dtype, int mode, int64_t *n_hot_max) {
    if (!n_hot_max || (dtype != HBP_F32 && dtype != HBP_F64) || mode < 0 || mode > 2)
        return HBP_E_ARG;
    const bool warm = mode == 1;
    // f32: 155 KB (hot tier only) / 131 KB (with a warm tier) / 185 KB (packed
    // x: its gathers hit L2, so L1 needs less room -- cfg2 0.990 vs 1.007 ms,
    // while an unpacked launch at 185 KB takes 1.40 ms) of shared memory per
    // SM (sweeps); f64 rings are twice as large, so its staged
    // launch takes a larger carveout
    size_t budget = dtype == HBP_F64 ? 187 * 1024
                    : (warm ? kWarmBudgetDefault : mode == 2 ? kPackedBudgetDefault
                                                              : kHotBudgetDefault);
    if (const char *e = getenv("HBP_HOT_BUDGET_KB")) budget = (size_t)atoi(e) * 1024;
    int dev = 0, optin = 0;
    HBP_CUDA_TRY(cudaGetDevice(&dev));
    HBP_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (budget > (size_t)optin) budget = (size_t)optin;
    size_t ring = 0;
    if (dtype == HBP_F64) hot_ring_bytes<double>(&ring, warm);
    else hot_ring_bytes<float>(&ring, warm);
    const size_t sv = dtype == HBP_F64 ? 8 : 4;
    *n_hot_max = budget > ring ? (int64_t)(((budget - ring) / sv) & ~(size_t)1023) : 0;
    return HBP_OK;
}

int hbp_hot_gather(const void *x, int dtype, const uint32_t *hot_cols, int64_t n_hot,
                   void *x_hot, hbp_stream_t stream) {
    if (n_hot < 0 || (n_hot > 0 && (!x || !hot_cols || !x_hot))) return HBP_E_ARG;
    if (dtype == HBP_F64) return hot_gather<double>(x, hot_cols, n_hot, x_hot, as_stream(stream));
    if (dtype == HBP_F32) return hot_gather<float>(x, hot_cols, n_hot, x_hot, as_stream(stream));
    return HBP_E_ARG;
}

int hbp_stream_set_variant(int v) {
    if (v < 0 || v >= kVariants) return HBP_E_ARG;
    g_variant = v;
    return HBP_OK;
}

int hbp_stream_slices(const hbp_format_t *f, const hbp_balanced_t *b, hbp_stream_t stream) {
    if (!f || !b || b->workers < 1 || !b->slice_lo || !b->slice_g) return HBP_E_ARG;
    if (f->warp_size != 32 || f->row_height % 32) return HBP_E_UNSUPPORTED;
    const int64_t ngroups = f->nzb * (f->row_height / 32);
    const bool exact = f->exact != 0 || f->dtype == HBP_F64;
    const int64_t n = b->pieces > b->workers ? b->pieces : b->workers;
    if (b->pieces > b->workers && (b->fixed_elems < 0 ||
                                   (!b->cost_prefix && b->fixed_elems > f->nnz)))
        return HBP_E_ARG;
    k_stream_slices<<<(unsigned)((n + 127) / 128), 128, 0, as_stream(stream)>>>(
        f->group_start, ngroups, f->nnz, b->workers, exact, exact ? b->hub_min : 0, b->slice_lo,
        b->slice_g, b->pieces, b->fixed_elems, b->cost_prefix);
    return (int)cudaGetLastError();
}

int hbp_group_costs(const hbp_format_t *f, int64_t w_group, int64_t w_short, int64_t w_step,
                    int64_t w_modular, int64_t w_hot, int64_t *cost, hbp_stream_t stream) {
    if (!f || !cost || w_group < 0 || w_short < 0 || w_step < 0 || w_modular < 0 || w_hot < 0 ||
        w_hot > 64)
        return HBP_E_ARG;
    if (f->warp_size != 32 || f->row_height % 32) return HBP_E_UNSUPPORTED;
    if (!f->phases || !f->phase_ptr) return HBP_E_ARG;
    const int64_t ngroups = f->nzb * (f->row_height / 32);
    if (ngroups == 0) return HBP_OK;
    k_group_costs<<<grid_for(ngroups * 32, 256), 256, 0, as_stream(stream)>>>(
        f->group_start, f->phase_ptr, (const uint2 *)f->phases, f->n_hot > 0 ? f->scol : nullptr,
        ngroups, w_group, w_short, w_step, w_modular, w_hot, cost);
    return (int)cudaGetLastError();
}

int hbp_spmv_stream(const hbp_format_t *f, const hbp_balanced_t *b, const void *x, void *y,
                    double *partial, hbp_stream_t stream) {
    if (!f || !b || b->workers < 1) return HBP_E_ARG;
    if (f->warp_size != 32 || f->row_height % 32) return HBP_E_UNSUPPORTED;
    if (!f->phases || !f->phase_ptr) return HBP_E_ARG;  // hbp_phase_emit first
    if (!partial && (!y || f->ncb != 1)) return HBP_E_ARG;
    if (b->rb_done && (!partial || !y || !f->rb_ptr || !f->rb_blk)) return HBP_E_ARG;
    if ((f->reserved & HBP_FLAG_DIRECT_SINGLE) && partial && (!y || !f->rb_ptr)) return HBP_E_ARG;
    if (f->nzb == 0) return HBP_OK;
    if (f->nzb * (f->row_height / 32) >= ((int64_t)1 << 31) - 2) return HBP_E_UNSUPPORTED;
    // slices are addressed with 32-bit offsets
    if ((f->nnz + b->workers - 1) / b->workers > (int64_t)1 << 30) return HBP_E_UNSUPPORTED;
    const bool exact = f->exact != 0 || f->dtype == HBP_F64;
    if ((!exact || b->hub_min > 0) && (!b->part_head || !b->part_tail || !b->counters))
        return HBP_E_ARG;
    if (b->hub_min < 0) return HBP_E_ARG;
    if (b->piece_base != 0) return HBP_E_ARG;  // set by the library only
    if (b->pieces > b->workers) {  // competitive or tail pieces
        if (!b->slice_lo || !b->slice_g || (!b->tail && !b->ticket) || b->rb_done)
            return HBP_E_ARG;
        if (!b->tail && b->hub_min > 0) return HBP_E_ARG;
        if ((f->nnz + b->pieces - 1) / b->pieces > (int64_t)1 << 30) return HBP_E_UNSUPPORTED;
    }
    if (staged(f)) {
        int64_t cap = 0;
        const int rc = hbp_hot_capacity(f->dtype, packed(f) ? 2 : warm(f) ? 1 : 0, &cap);
        if (rc) return rc;
        if (f->n_hot > cap || (f->n_hot & 3) || !b->x_hot) return HBP_E_ARG;
        if (f->n_warm < 0 || (warm(f) && f->cols > (int64_t)1 << 30)) return HBP_E_ARG;
        if (packed(f) && (f->n_warm >= (int64_t)1 << 31 || f->n_warm > f->cols)) return HBP_E_ARG;
        if (f->cols >= (int64_t)1 << 31) return HBP_E_ARG;  // bit 31 flags hot columns
    }
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
