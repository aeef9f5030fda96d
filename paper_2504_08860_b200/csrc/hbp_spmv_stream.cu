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
//      on per-slot mbarriers), NB-3 chunks ahead of the walk;
//   3. the x gathers of chunk c+1 are issued (registers) before the walk of
//      chunk c needs them; when the walk reaches chunk c+1 the products are
//      written over its values (f32 data: f32 products; exact f64 data:
//      __dmul_rn products), so products of the chunks the walk can touch are
//      always resident;
//   4. each group's phases come precomputed from the phase stream (live mask
//      and element offset per phase, hbp_phase_emit); the walk runs
//        - a step-uniform loop while >= KT lanes are live (exact mode: all
//          steps): every live lane adds its element of the step -- each row
//          is summed in step order, bitwise identical to _kernels.py:41-46
//          for f64;
//        - (fast mode) the remaining few-lane phases: short ones lane by
//          lane, long ones with S = 32/k sub-streams per live lane and a
//          shuffle tree;
//   5. a group cut by a slice boundary (fast mode only) leaves per-lane
//      partials; the warp whose piece completes the group's element count
//      (atomic) adds the pieces in slice order -- deterministic.
//
// Precision (fast mode): f32 products (relative error <= 2^-24 each) summed
// in f64, one rounding to f32: componentwise error <= ~1.2e-7 |A||x|.
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

template <typename V, int CH, int NB>
struct __align__(16) WarpSmem {
    uint32_t col[NB * CH];
    V val[NB * CH];  // values, then products in place
    uint32_t ph_mask[33];
    int32_t ph_off[33];
    uint64_t mbar[NB];
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
// k*S <= 32, and ceil(2^16/k) (exact lane / k for lane < 32)
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

template <typename V, bool EXACT>
__device__ __forceinline__ V product(V v, V xv) {
    if (EXACT) return (V)__dmul_rn((double)v, (double)xv);
    return v * xv;
}

// Streams one warp's slice through the shared-memory ring.  All positions
// are 32-bit offsets relative to `base` (slice start rounded down to 16 B).
template <typename V, bool EXACT, int CH, int NB, bool XNA>
struct Ring {
    static constexpr int RMASK = NB * CH - 1;
    static constexpr int EPL = CH / 32;  // elements per lane per chunk
    const hbp_format_t &f;
    WarpSmem<V, CH, NB> &S;
    const V *__restrict__ x;
    int64_t base;
    int32_t len32;        // c_hi - base
    int32_t nchunks;
    int32_t ready = -1;   // chunks <= ready hold products
    int32_t pending = -1; // chunk whose x gathers are in flight
    int32_t issued = 0;   // bulk copies issued (lane 0)
    int32_t res32 = 0;    // products resident for offsets < res32
    int lane;
    uint64_t pe, pl;
    V xr[EPL];            // gathered x of the pending chunk

    __device__ void issue_upto(int32_t last) {  // lane 0
        for (; issued <= last && issued < nchunks; ++issued) {
            const int32_t ca = issued * CH;
            const int32_t n = (ca + CH < len32 ? ca + CH : len32) - ca;
            const int slot = issued % NB;
            const uint32_t bc = (uint32_t)((n * 4 + 15) & ~15);
            const uint32_t bv = (uint32_t)((n * (int)sizeof(V) + 15) & ~15);
            mbar_expect_tx(&S.mbar[slot], bc + bv);
            bulk_g2s(&S.col[slot * CH], f.col + base + ca, bc, &S.mbar[slot], pe);
            bulk_g2s(&S.val[slot * CH], (const V *)f.data + base + ca, bv, &S.mbar[slot], pe);
        }
    }

    // chunk c: wait for its bytes, issue its x gathers into xr
    __device__ __forceinline__ void start(int32_t c) {
        const int slot = c % NB;
        mbar_wait(&S.mbar[slot], (uint32_t)((c / NB) & 1));
        const int32_t n = (c * CH + CH < len32 ? c * CH + CH : len32) - c * CH;
        uint32_t cc[EPL];
        if constexpr (EPL == 4) {
            const uint4 t = *reinterpret_cast<const uint4 *>(&S.col[slot * CH + 4 * lane]);
            cc[0] = t.x, cc[1] = t.y, cc[2] = t.z, cc[3] = t.w;
        } else if constexpr (EPL == 2) {
            const uint2 t = *reinterpret_cast<const uint2 *>(&S.col[slot * CH + 2 * lane]);
            cc[0] = t.x, cc[1] = t.y;
        } else {
#pragma unroll
            for (int e = 0; e < EPL; e += 4) {
                const uint4 t =
                    *reinterpret_cast<const uint4 *>(&S.col[slot * CH + EPL * lane + e]);
                cc[e] = t.x, cc[e + 1] = t.y, cc[e + 2] = t.z, cc[e + 3] = t.w;
            }
        }
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
            if (EPL * lane + e >= n) cc[e] = 0u;  // never gather past the slice
            xr[e] = XNA ? ld_x_na(x + cc[e], pl) : ld_x(x + cc[e], pl);
        }
        pending = c;
    }

    // pending chunk: values -> products (in place)
    __device__ __forceinline__ void finish() {
        const int c = pending;
        const int slot = c % NB;
        V *v = &S.val[slot * CH + EPL * lane];
#pragma unroll
        for (int e = 0; e < EPL; ++e) v[e] = product<V, EXACT>(v[e], xr[e]);
        ready = c;
        res32 = (c * CH + CH < len32 ? c * CH + CH : len32);
        pending = -1;
    }

    // make offsets < need resident (warp-uniform); refills the ring
    __device__ __forceinline__ void advance(int32_t need) {
        while (need > res32) {
            if (pending < 0) {
                if (ready + 1 >= nchunks) return;
                start(ready + 1);
            }
            __syncwarp();  // the walk's reads of the oldest slot are done
            finish();
            fence_proxy_async();  // generic ring accesses precede later bulk writes
            __syncwarp();
            if (ready + 1 < nchunks) start(ready + 1);
            // slots of chunks <= ready - 2 are free (the walk may still read
            // ready - 1 for a step straddling the boundary)
            if (lane == 0) issue_upto(ready + NB - 2);
        }
    }

    __device__ __forceinline__ double at(int32_t o) const { return (double)S.val[o & RMASK]; }
};

template <typename V, bool EXACT, int CH, int NB, int MINB, bool XNA>
__global__ void __launch_bounds__(kThreads, MINB)
    k_spmv_stream(const hbp_format_t f, const hbp_balanced_t b, const V *__restrict__ x,
                  V *__restrict__ y, double *__restrict__ partial) {
    constexpr int KT = 8;  // fast mode: fewer live lanes -> per-phase processing
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WarpSmem<V, CH, NB> &S = reinterpret_cast<WarpSmem<V, CH, NB> *>(smem_raw)[wib];
    const int64_t w = (int64_t)blockIdx.x * kWarps + wib;
    const int64_t Nw = b.workers;
    if (w >= Nw) return;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t R = f.row_height, gpb = R / 32;
    const int64_t ngroups = f.nzb * gpb;
    const int64_t E = f.nnz;
    const int64_t *__restrict__ gs = f.group_start;
    const int64_t *__restrict__ pptr = f.phase_ptr;
    const uint2 *__restrict__ phs = (const uint2 *)f.phases;
    const uint32_t *__restrict__ permp = (const uint32_t *)f.perm;

    Ring<V, EXACT, CH, NB, XNA> ring{f, S, x};
    ring.lane = lane;
    ring.pe = policy_evict_first();
    ring.pl = policy_evict_last();

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
    const int64_t base = c_lo & ~(int64_t)3;
    ring.base = base;
    ring.len32 = (int32_t)(c_hi - base);
    ring.nchunks = c_hi > c_lo ? (ring.len32 + CH - 1) / CH : 0;

    if (lane == 0) {
        for (int i = 0; i < NB; ++i) mbar_init(&S.mbar[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (lane == 0) ring.issue_upto(NB - 3);

    int64_t g = upper_group(gs, ngroups, c_lo);
    if (!(g < ngroups && gs[g] < c_lo)) g = lower_group(gs, ngroups, c_lo);
    const bool last_warp = (w == Nw - 1);

    // prefetched metadata of group g: element range, output rows, phases
    int64_t gs0 = g < ngroups ? gs[g] : E;
    int64_t gs1 = g < ngroups ? gs[g + 1] : E;
    uint32_t perm_n = g < ngroups ? permp[g * 32 + lane] : 0u;
    int64_t pp0 = g < ngroups ? pptr[g] : 0;
    int64_t pp1 = g < ngroups ? pptr[g + 1] : 0;
    uint2 ph_n = make_uint2(0u, 0u);
    if (g < ngroups && lane < pp1 - pp0) ph_n = phs[pp0 + lane];

    for (; g < ngroups && (gs0 < c_hi || last_warp); ++g) {
        const uint32_t row_local = perm_n;
        const int64_t g0 = gs0, g1 = gs1;
        const int np = (int)(pp1 - pp0);
        const uint2 ph = ph_n;
        if (g + 1 < ngroups) {  // prefetch the next group's metadata
            gs0 = g1;
            gs1 = gs[g + 2];
            perm_n = permp[(g + 1) * 32 + lane];
            pp0 = pp1;
            pp1 = pptr[g + 2];
            ph_n = lane < pp1 - pp0 ? phs[pp0 + lane] : make_uint2(0u, 0u);
        }
        const int64_t lo = g0 > c_lo ? g0 : c_lo;
        const int64_t hi = g1 < c_hi ? g1 : c_hi;
        const bool piece = (lo > g0) || (hi < g1);

        double acc = 0.0;
        if (lo < hi) {
            __syncwarp();  // previous group's table reads are done
            if (lane < np) {
                S.ph_mask[lane] = ph.x;
                S.ph_off[lane] = (int32_t)ph.y;
            }
            if (lane == 0) S.ph_off[np] = (int32_t)(g1 - g0);
            __syncwarp();
            const int32_t gb = (int32_t)(g0 - base);  // group start, ring offset (may be < 0)
            const int32_t lo_r = (int32_t)(lo - base), hi_r = (int32_t)(hi - base);
            // start: phase j and step t containing lo
            const int32_t o_lo = lo_r - gb;
            int j = 0;
            while (j + 1 < np && S.ph_off[j + 1] <= o_lo) ++j;
            unsigned pm = S.ph_mask[j];
            int k = __popc(pm);
            int32_t pend_j = gb + S.ph_off[j + 1];  // ring offset where phase j ends
            int32_t pb = gb + S.ph_off[j] + div_small(o_lo - S.ph_off[j], k) * k;
            bool live = (pm >> lane) & 1u;
            int rank = __popc(pm & lt);

            // ---- step-uniform lane walk (exact: all phases; fast: k >= KT)
            while (pb < hi_r && (EXACT || k >= KT)) {
                const int32_t stop = pend_j < hi_r ? pend_j : hi_r;
                if (!piece) {
                    for (; pb < stop; pb += k) {
                        if (pb + k > ring.res32) ring.advance(pb + k);
                        if (live) {
                            const double v = ring.at(pb + rank);
                            acc = EXACT ? __dadd_rn(acc, v) : acc + v;
                        }
                    }
                } else {
                    for (; pb < stop; pb += k) {
                        if (pb + k > ring.res32) ring.advance(pb + k < hi_r ? pb + k : hi_r);
                        const int32_t P = pb + rank;
                        if (live && P >= lo_r && P < hi_r) {
                            const double v = ring.at(P);
                            acc = EXACT ? __dadd_rn(acc, v) : acc + v;
                        }
                    }
                }
                if (pb < pend_j) break;  // reached hi inside the phase
                if (++j == np) break;
                pm = S.ph_mask[j];
                k = __popc(pm);
                pend_j = gb + S.ph_off[j + 1];
                live = (pm >> lane) & 1u;
                rank = __popc(pm & lt);
            }
            // ---- fast mode: phases with few live lanes
            if (!EXACT) {
                while (pb < hi_r && j < np) {
                    const int32_t stop = pend_j < hi_r ? pend_j : hi_r;
                    if (stop - pb > 8 * k && pb >= lo_r) {
                        const int SS = c_streams[k];
                        const int s = (int)(((uint32_t)lane * c_magic16[k]) >> 16);  // lane / k
                        const int r = lane - s * k;
                        const int32_t stride = SS * k;
                        double v = 0.0;
                        for (int32_t q = pb; q < stop; q += stride) {  // SS steps per pass
                            const int32_t need = q + stride < stop ? q + stride : stop;
                            if (need > ring.res32) ring.advance(need);
                            const int32_t P = q + s * k + r;
                            if (s < SS && P < stop) v += ring.at(P);
                        }
                        for (int d = SS >> 1; d >= 1; d >>= 1)
                            v += __shfl_down_sync(FULL, v, d * k);
                        const double tot = __shfl_sync(FULL, v, live ? rank : 0);
                        if (live) acc += tot;
                        pb = stop;
                    } else {
                        // short phase (or a step cut by the slice start): lane by lane
                        const int32_t stop1 = stop - pb > 8 * k ? pb + k : stop;
                        for (; pb < stop1; pb += k) {
                            if (pb + k > ring.res32) ring.advance(pb + k < hi_r ? pb + k : hi_r);
                            const int32_t P = pb + rank;
                            if (live && P >= lo_r && P < hi_r) acc += ring.at(P);
                        }
                        if (pb < pend_j && stop1 != stop) continue;  // rest of this phase
                    }
                    if (pb < pend_j) break;  // reached hi inside the phase
                    if (++j == np) break;
                    pm = S.ph_mask[j];
                    k = __popc(pm);
                    pend_j = gb + S.ph_off[j + 1];
                    live = (pm >> lane) & 1u;
                    rank = __popc(pm & lt);
                }
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

template <typename V, bool EXACT, int CH, int NB, int MINB, bool XNA>
int launch(const hbp_format_t *f, const hbp_balanced_t *b, const void *x, void *y,
           double *partial, cudaStream_t st) {
    const size_t smem = sizeof(WarpSmem<V, CH, NB>) * kWarps;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_spmv_stream<V, EXACT, CH, NB, MINB, XNA>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    unsigned grid = (unsigned)((b->workers + kWarps - 1) / kWarps);
    k_spmv_stream<V, EXACT, CH, NB, MINB, XNA><<<grid, kThreads, smem, st>>>(
        *f, *b, (const V *)x, (V *)y, partial);
    return (int)cudaGetLastError();
}

template <typename V, bool EXACT, int CH, int NB, int MINB, bool XNA>
int occupancy_of(int *per_sm) {
    const size_t smem = sizeof(WarpSmem<V, CH, NB>) * kWarps;
    cudaFuncSetAttribute(k_spmv_stream<V, EXACT, CH, NB, MINB, XNA>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        per_sm, k_spmv_stream<V, EXACT, CH, NB, MINB, XNA>, kThreads, smem);
}

// Tile / occupancy variants (chunk CH, ring slots NB, min CTAs per SM),
// chosen with HBP_STREAM_VARIANT for sweeps; 0 is the default.
constexpr int kVariants = 8;
int variant() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("HBP_STREAM_VARIANT");
        v = e ? atoi(e) : 0;
        if (v < 0 || v >= kVariants) v = 0;
    }
    return v;
}

#define HBP_STREAM_VARIANTS(FN, V, EXACT, ...)                     \
    switch (variant()) {                                            \
        case 1: return FN<V, EXACT, 64, 8, 4, true>(__VA_ARGS__);  \
        case 2: return FN<V, EXACT, 128, 8, 3, true>(__VA_ARGS__); \
        case 3: return FN<V, EXACT, 256, 4, 2, true>(__VA_ARGS__); \
        case 4: return FN<V, EXACT, 128, 8, 2, true>(__VA_ARGS__); \
        case 5: return FN<V, EXACT, 128, 4, 4, true>(__VA_ARGS__); \
        case 6: return FN<V, EXACT, 64, 8, 3, true>(__VA_ARGS__);  \
        case 7: return FN<V, EXACT, 128, 4, 3, false>(__VA_ARGS__); \
        default: return FN<V, EXACT, 128, 4, 3, true>(__VA_ARGS__); \
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
    if (f->dtype == HBP_F64)
        rc = exact ? occupancy<double, true>(&per_sm) : occupancy<double, false>(&per_sm);
    else
        rc = exact ? occupancy<float, true>(&per_sm) : occupancy<float, false>(&per_sm);
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
    if (!f->phases || !f->phase_ptr) return HBP_E_ARG;  // hbp_phase_emit first
    if (!partial && (!y || f->ncb != 1)) return HBP_E_ARG;
    if (f->nzb == 0) return HBP_OK;
    // slices are addressed with 32-bit offsets
    if ((f->nnz + b->workers - 1) / b->workers > (int64_t)1 << 30) return HBP_E_UNSUPPORTED;
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
