// hbp_spmv_stream.cu -- streamed, element-balanced HBP SpMV (W = 32).
//
// Why: in the HBP layout a group's elements are step-major (all live lanes'
// t-th elements, then the (t+1)-th ...).  On skewed matrices a group has ~10
// "phases" (step ranges with a fixed live-lane set) and few live lanes, so a
// lane-per-row walk over global memory pays dependent DRAM round trips (col,
// then x) per phase.  Here memory and the irregular walk are decoupled:
//
//   1. each persistent warp owns an equal slice [c_lo, c_hi) of the element
//      array (exact mode: slice ends rounded up to group boundaries);
//   2. the slice streams through a three-stage register pipeline in chunks
//      of CH elements (CH/32 per lane, 16-byte streaming loads): chunk c+2's
//      col/data loads and chunk c+1's x gathers are in flight while the walk
//      reads chunk c;
//   3. products (f32 data: f32 products; exact f64 data: __dmul_rn) go to a
//      small shared-memory ring of NB = 2 chunks (the walk touches at most
//      the current and the previous chunk); only products live in shared
//      memory, which keeps most of the SM's 256 KB as L1 -- the L1 capacity
//      bounds how many x gathers can be outstanding (measured: kernels with
//      > ~190 KB of shared memory per SM ran 2x slower);
//   4. each group's phases come precomputed from the phase stream (live mask
//      and element offset per phase, hbp_phase_emit); the walk sums
//        - lane by lane in step order (exact mode always): each row in the
//          reference's order, bitwise identical to _kernels.py:41-46 for f64;
//        - (fast mode) long phases with fewer than KT live lanes with
//          S = 32/k sub-streams per live lane and a shuffle tree;
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
    V prod[NB * CH];  // product ring
    uint32_t ph_mask[33];
    int32_t ph_off[33];
};

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

// 16-byte streaming loads (read once: no L1 allocation, L2 evict-first)
__device__ __forceinline__ uint4 ld_stream_v4(const uint32_t *p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void ld_vals4(const float *p, uint64_t pol, float (&o)[4]) {
    uint4 v = ld_stream_v4(reinterpret_cast<const uint32_t *>(p), pol);
    o[0] = __uint_as_float(v.x), o[1] = __uint_as_float(v.y);
    o[2] = __uint_as_float(v.z), o[3] = __uint_as_float(v.w);
}
__device__ __forceinline__ void ld_vals4(const double *p, uint64_t pol, double (&o)[4]) {
    uint4 a = ld_stream_v4(reinterpret_cast<const uint32_t *>(p), pol);
    uint4 b = ld_stream_v4(reinterpret_cast<const uint32_t *>(p + 2), pol);
    o[0] = __hiloint2double(a.y, a.x), o[1] = __hiloint2double(a.w, a.z);
    o[2] = __hiloint2double(b.y, b.x), o[3] = __hiloint2double(b.w, b.z);
}

// Streams one warp's slice through the register pipeline into the product
// ring.  Positions are 32-bit offsets relative to `base` (slice start rounded
// down to 4 elements, 16-byte aligned).  Lane l owns chunk elements
// [4*l + 128*u, +4) for u < CH/128.
template <typename V, bool EXACT, int CH, int NB, bool XNA>
struct Pipe {
    static constexpr int RMASK = NB * CH - 1;
    static constexpr int U = CH / 128;
    const uint32_t *__restrict__ col;
    const V *__restrict__ data;
    const V *__restrict__ x;
    V *prod;              // this warp's ring
    int32_t len32;        // c_hi - base
    int32_t nchunks;
    int32_t ready = -1;   // chunks <= ready have products in the ring
    int32_t res32 = 0;    // products resident for offsets < res32
    int lane;
    uint64_t pe, pl;
    // stage A: col/data of chunk ready+2;  stage B: x gathers of chunk ready+1
    uint32_t a_col[U][4];
    V a_val[U][4];
    V b_x[U][4];
    V b_val[U][4];

    int32_t a_off;  // chunk offset of stage A (its elements past len32 are masked at use)

    // issue chunk c's col/data loads; the registers are not touched until
    // a_to_b() (a consumer here would stall on the loads right away)
    __device__ __forceinline__ void load_a(int32_t c) {
        a_off = c * CH;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t o = c * CH + 128 * u + 4 * lane;
            if (o < len32) {
                const uint4 t = ld_stream_v4(col + o, pe);
                a_col[u][0] = t.x, a_col[u][1] = t.y, a_col[u][2] = t.z, a_col[u][3] = t.w;
                ld_vals4(data + o, pe, a_val[u]);
            }
        }
    }
    __device__ __forceinline__ void a_to_b() {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                // never gather past the slice (tail of the last chunk)
                const bool in = a_off + 128 * u + 4 * lane + e < len32;
                const uint32_t cc = in ? a_col[u][e] : 0u;
                b_x[u][e] = XNA ? ld_x_na(x + cc, pl) : ld_x(x + cc, pl);
                b_val[u][e] = in ? a_val[u][e] : (V)0;
            }
    }
    __device__ __forceinline__ void init(int32_t len, const int64_t base) {
        len32 = len;
        nchunks = (len + CH - 1) / CH;
        load_a(0);
        a_to_b();
        load_a(1);
    }
    // finish chunk ready+1 into the ring, advance the pipeline by one chunk
    __device__ __forceinline__ void step() {
        const int32_t c = ready + 1;
        V *dst = prod + (c * CH) % (NB * CH);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            V p[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) p[e] = product<V, EXACT>(b_val[u][e], b_x[u][e]);
            if (sizeof(V) == 4) {
                *reinterpret_cast<float4 *>(dst + 128 * u + 4 * lane) =
                    make_float4((float)p[0], (float)p[1], (float)p[2], (float)p[3]);
            } else {
                *reinterpret_cast<double2 *>(dst + 128 * u + 4 * lane) =
                    make_double2((double)p[0], (double)p[1]);
                *reinterpret_cast<double2 *>(dst + 128 * u + 4 * lane + 2) =
                    make_double2((double)p[2], (double)p[3]);
            }
        }
        ready = c;
        res32 = (c + 1) * CH < len32 ? (c + 1) * CH : len32;
        a_to_b();
        load_a(c + 2);
        __syncwarp();  // ring writes visible to the walk
    }
    // make offsets < need resident (warp-uniform call)
    __device__ __forceinline__ void advance(int32_t need) {
        while (need > res32 && ready + 1 < nchunks) step();
    }
};

template <typename V, bool EXACT, int CH, int NB, int MINB, bool XNA>
__global__ void __launch_bounds__(kThreads, MINB)
    k_spmv_stream(const hbp_format_t f, const hbp_balanced_t b, const V *__restrict__ x,
                  V *__restrict__ y, double *__restrict__ partial) {
    constexpr int KT = 8;  // fast mode: fewer live lanes -> cooperative long phases
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

    Pipe<V, EXACT, CH, NB, XNA> pipe;
    pipe.col = f.col + base;
    pipe.data = (const V *)f.data + base;
    pipe.x = x;
    pipe.prod = S.prod;
    pipe.lane = lane;
    pipe.pe = policy_evict_first();
    pipe.pl = policy_evict_last();
    pipe.init(c_hi > c_lo ? (int32_t)(c_hi - base) : 0, base);

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

    constexpr int RM = NB * CH - 1;
    const V *rv = S.prod;

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
            // start: phase j and step containing lo
            const int32_t o_lo = lo_r - gb;
            int j = 0;
            while (j + 1 < np && S.ph_off[j + 1] <= o_lo) ++j;
            unsigned pm = S.ph_mask[j];
            int k = __popc(pm);
            int32_t pend_j = gb + S.ph_off[j + 1];  // ring offset where phase j ends
            int32_t pb = gb + S.ph_off[j] + div_small(o_lo - S.ph_off[j], k) * k;
            bool live = (pm >> lane) & 1u;
            int rank = __popc(pm & lt);

            // ---- walk phase by phase.  Steps are summed lane by lane (each
            // lane its own row, in step order); in fast mode long phases with
            // fewer than KT live lanes use S = 32/k sub-streams per lane.
            // Residency checks sit in the outer loops; inner loops only load.
            for (;;) {
                const int32_t stop = pend_j < hi_r ? pend_j : hi_r;
                if (pb < lo_r) {
                    // a step cut by the slice start (fast-mode pieces only)
                    if (pb + k > pipe.res32) pipe.advance(pb + k < hi_r ? pb + k : hi_r);
                    const int32_t P = pb + rank;
                    if (live && P >= lo_r && P < hi_r) acc += (double)rv[P & RM];
                    pb += k;
                    if (pb < stop) continue;  // rest of this phase
                } else if (!EXACT && k < KT && stop - pb > 8 * k) {
                    const int SS = c_streams[k];
                    const int s = (int)(((uint32_t)lane * c_magic16[k]) >> 16);  // lane / k
                    const int32_t stride = SS * k;
                    const bool act = s < SS;
                    double v0 = 0.0, v1 = 0.0;
                    int32_t q = pb;
                    while (q < stop) {
                        const int32_t need = q + stride < stop ? q + stride : stop;
                        if (need > pipe.res32) pipe.advance(need);
                        if (q + stride > stop) {  // last, partial pass
                            const int32_t P = q + lane;
                            if (act && P < stop) v0 += (double)rv[P & RM];
                            q = stop;
                            break;
                        }
                        const int32_t lim = stop < pipe.res32 ? stop : pipe.res32;
                        const int32_t npass = div_small(lim - q - stride, stride) + 1;
                        if (act) {
                            int32_t p = q + lane;
                            int32_t i = 0;
                            for (; i + 2 <= npass; i += 2, p += 2 * stride) {
                                v0 += (double)rv[p & RM];
                                v1 += (double)rv[(p + stride) & RM];
                            }
                            if (i < npass) v0 += (double)rv[p & RM];
                        }
                        q += npass * stride;
                    }
                    double v = v0 + v1;
                    for (int d = SS >> 1; d >= 1; d >>= 1) v += __shfl_down_sync(FULL, v, d * k);
                    const double tot = __shfl_sync(FULL, v, live ? rank : 0);
                    if (live) acc += tot;
                    pb = stop;
                } else {
                    while (pb < stop) {
                        if (pb + k > pipe.res32) pipe.advance(pb + k < hi_r ? pb + k : hi_r);
                        const int32_t lim = stop < pipe.res32 ? stop : pipe.res32;
                        const int32_t nsteps = lim - pb >= k ? div_small(lim - pb, k) : 0;
                        if (nsteps == 0) {  // last step cut by the slice end
                            const int32_t P = pb + rank;
                            if (live && P < hi_r) {
                                const double v = (double)rv[P & RM];
                                acc = EXACT ? __dadd_rn(acc, v) : acc + v;
                            }
                            pb += k;
                            break;
                        }
                        if (live) {
                            int32_t p = pb + rank;
                            for (int32_t i = 0; i < nsteps; ++i, p += k) {
                                const double v = (double)rv[p & RM];
                                acc = EXACT ? __dadd_rn(acc, v) : acc + v;
                            }
                        }
                        pb += nsteps * k;
                    }
                }
                if (pb < pend_j || ++j == np) break;  // reached hi, or the group's end
                pm = S.ph_mask[j];
                k = __popc(pm);
                pend_j = gb + S.ph_off[j + 1];
                live = (pm >> lane) & 1u;
                rank = __popc(pm & lt);
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

// Tile / occupancy variants (chunk CH, ring slots NB, min CTAs per SM, L1
// policy of the x gathers), chosen with HBP_STREAM_VARIANT for sweeps.
constexpr int kVariants = 6;
int variant() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("HBP_STREAM_VARIANT");
        v = e ? atoi(e) : 0;
        if (v < 0 || v >= kVariants) v = 0;
    }
    return v;
}

#define HBP_STREAM_VARIANTS(FN, V, EXACT, ...)                      \
    switch (variant()) {                                             \
        case 1: return FN<V, EXACT, 256, 2, 3, true>(__VA_ARGS__);  \
        case 2: return FN<V, EXACT, 256, 2, 2, true>(__VA_ARGS__);  \
        case 3: return FN<V, EXACT, 128, 2, 4, true>(__VA_ARGS__);  \
        case 4: return FN<V, EXACT, 128, 2, 3, false>(__VA_ARGS__); \
        case 5: return FN<V, EXACT, 128, 2, 4, false>(__VA_ARGS__);  \
        default: return FN<V, EXACT, 128, 2, 3, true>(__VA_ARGS__); \
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
