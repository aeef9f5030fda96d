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
//   3. per chunk the warp gathers x for all CH elements at once and writes
//      the products in place of the values (f32 data: f32 products, exact
//      f64 data: __dmul_rn products), so the ring always holds the products
//      of the two chunks the walk can touch;
//   4. the group's phase table (offset, steps, live mask) is built from the
//      32 slot lengths with ballots; the walk then runs
//        - a step-uniform loop while >= KT lanes are live (exact mode: all
//          steps): every live lane adds its element of the step, phase
//          changes only reload (k, mask, rank) -- each row is summed in
//          step order, bitwise identical to _kernels.py:41-46 for f64;
//        - (fast mode) per remaining phase: short ones lane-serially, long
//          ones with S = 32/k sub-streams per live lane and a shuffle tree;
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
constexpr int NB = 4;  // ring slots (chunks)

template <typename V, int CH>
struct __align__(16) WarpSmem {
    uint32_t col[NB * CH];
    V val[NB * CH];  // values, then products in place
    int32_t ph_off[33];
    int32_t ph_t1[32];
    uint32_t ph_mask[32];
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

__device__ __forceinline__ int64_t div_small(int64_t n, int k) {  // n >= 0, 1 <= k <= 32
    if (n < (1 << 26)) return (int64_t)(((uint64_t)n * c_magic32[k]) >> 32);
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

template <typename V, bool EXACT, int CH, bool XNA>
struct Ring {
    static constexpr int RMASK = NB * CH - 1;
    const hbp_format_t &f;
    WarpSmem<V, CH> &S;
    const V *__restrict__ x;
    int64_t c_lo, c_hi, base, nchunks;
    int64_t ready = -1;   // highest prepared chunk
    int64_t issued = 0;   // chunks whose bulk copy was issued
    int64_t res_hi = 0;   // products resident for positions < res_hi
    int lane;
    uint64_t pe, pl;

    __device__ __forceinline__ int64_t chunk_start(int64_t c) const { return base + c * CH; }

    __device__ void issue_upto(int64_t last) {  // lane 0
        for (; issued <= last && issued < nchunks; ++issued) {
            const int64_t ca = chunk_start(issued);
            const int64_t cb = ca + CH < c_hi ? ca + CH : c_hi;
            const int slot = (int)(issued % NB);
            const uint32_t bc = (uint32_t)(((cb - ca) * 4 + 15) & ~(int64_t)15);
            const uint32_t bv = (uint32_t)(((cb - ca) * (int64_t)sizeof(V) + 15) & ~(int64_t)15);
            mbar_expect_tx(&S.mbar[slot], bc + bv);
            bulk_g2s(&S.col[slot * CH], f.col + ca, bc, &S.mbar[slot], pe);
            bulk_g2s(&S.val[slot * CH], (const V *)f.data + ca, bv, &S.mbar[slot], pe);
        }
    }

    // wait for chunk c's bytes, gather x, overwrite its values with products
    __device__ void prepare(int64_t c) {
        const int slot = (int)(c % NB);
        mbar_wait(&S.mbar[slot], (uint32_t)((c / NB) & 1));
        const int64_t ca = chunk_start(c);
        const int n = (int)((ca + CH < c_hi ? ca + CH : c_hi) - ca);
        constexpr int U = CH / 128;
        uint4 cl[U];
        V vv[U][4];
        V xv[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = 4 * lane + 128 * u;
            cl[u] = *reinterpret_cast<const uint4 *>(&S.col[slot * CH + i]);
            if (i + 3 >= n) {  // never gather past the slice
                if (i >= n) cl[u].x = 0u;
                if (i + 1 >= n) cl[u].y = 0u;
                if (i + 2 >= n) cl[u].z = 0u;
                cl[u].w = 0u;
            }
            if (sizeof(V) == 4) {
                const float4 t = *reinterpret_cast<const float4 *>(&S.val[slot * CH + i]);
                vv[u][0] = t.x, vv[u][1] = t.y, vv[u][2] = t.z, vv[u][3] = t.w;
            } else {
                const double2 t0 = *reinterpret_cast<const double2 *>(&S.val[slot * CH + i]);
                const double2 t1 = *reinterpret_cast<const double2 *>(&S.val[slot * CH + i + 2]);
                vv[u][0] = t0.x, vv[u][1] = t0.y, vv[u][2] = t1.x, vv[u][3] = t1.y;
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
            V p[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) p[e] = product<V, EXACT>(vv[u][e], xv[u][e]);
            if (sizeof(V) == 4) {
                *reinterpret_cast<float4 *>(&S.val[slot * CH + i]) =
                    make_float4((float)p[0], (float)p[1], (float)p[2], (float)p[3]);
            } else {
                *reinterpret_cast<double2 *>(&S.val[slot * CH + i]) =
                    make_double2((double)p[0], (double)p[1]);
                *reinterpret_cast<double2 *>(&S.val[slot * CH + i + 2]) =
                    make_double2((double)p[2], (double)p[3]);
            }
        }
        fence_proxy_async();  // our generic accesses precede later bulk writes of the ring
        __syncwarp();
        ready = c;
        res_hi = ca + n;
        // slots of chunks < c - 1 are free: keep NB - 2 chunks in flight
        if (lane == 0) issue_upto(c + NB - 2);
    }

    // make positions < need resident (warp-uniform call)
    __device__ __forceinline__ void ensure(int64_t need) {
        while (need > res_hi && ready + 1 < nchunks) prepare(ready + 1);
    }

    __device__ __forceinline__ double at(int64_t P) const {
        return (double)S.val[(int)((P - base) & RMASK)];
    }
};

template <typename V, bool EXACT, int CH, int MINB, bool XNA>
__global__ void __launch_bounds__(kThreads, MINB)
    k_spmv_stream(const hbp_format_t f, const hbp_balanced_t b, const V *__restrict__ x,
                  V *__restrict__ y, double *__restrict__ partial) {
    constexpr int KT = 8;  // fast mode: lanes live below which phases go cooperative
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

    Ring<V, EXACT, CH, XNA> ring{f, S, x};
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
    ring.c_lo = c_lo;
    ring.c_hi = c_hi;
    ring.base = c_lo & ~(int64_t)3;
    ring.res_hi = ring.base;
    ring.nchunks = c_hi > c_lo ? (c_hi - ring.base + CH - 1) / CH : 0;

    if (lane == 0) {
        for (int i = 0; i < NB; ++i) mbar_init(&S.mbar[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (lane == 0) ring.issue_upto(NB - 2);

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
            // ---- phase table: ph_off[j] (group offset of phase j), ph_t1[j]
            // (its end step), ph_mask[j] (live lanes)
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
                        S.ph_t1[nph] = (int32_t)t1;
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
            // ---- start: phase j and step t containing group offset lo - g0
            const int32_t o_lo = (int32_t)(lo - g0);
            int j = 0;
            while (j + 1 < nph && S.ph_off[j + 1] <= o_lo) ++j;
            unsigned pm = S.ph_mask[j];
            int k = __popc(pm);
            int32_t t0j = j ? S.ph_t1[j - 1] : 0;
            int32_t t = t0j + (int32_t)div_small(o_lo - S.ph_off[j], k);
            int32_t t1 = S.ph_t1[j];
            int64_t pb = g0 + S.ph_off[j] + (int64_t)(t - t0j) * k;  // first position of step t
            bool live = (pm >> lane) & 1u;
            int rank = __popc(pm & lt);

            // ---- step-uniform lane walk while enough lanes are live
            while (pb < hi && (EXACT || k >= KT)) {
                ring.ensure(pb + k);
                const int64_t P = pb + rank;
                if (live && P >= lo && P < hi) {
                    const double v = ring.at(P);
                    acc = EXACT ? __dadd_rn(acc, v) : acc + v;
                }
                pb += k;
                if (++t == t1) {
                    if (++j == nph) break;
                    pm = S.ph_mask[j];
                    k = __popc(pm);
                    t1 = S.ph_t1[j];
                    live = (pm >> lane) & 1u;
                    rank = __popc(pm & lt);
                }
            }
            // ---- fast mode: remaining phases have few live lanes
            if (!EXACT) {
                while (pb < hi && j < nph) {
                    // steps of this phase inside [.., hi)
                    int32_t steps = t1 - t;
                    const int64_t lim = hi - pb;  // > 0
                    if ((int64_t)steps * k > lim) steps = (int32_t)div_small(lim + k - 1, k);
                    // a step cut by the slice start is handled lane-serially first
                    if (steps > 8 && pb >= lo) {
                        const int SS = c_streams[k];
                        const int s = (int)(((uint32_t)lane * c_magic16[k]) >> 16);  // lane / k
                        const int r = lane - s * k;
                        const int32_t stride = SS * k;
                        const int64_t pend = pb + (int64_t)steps * k;
                        double v = 0.0;
                        for (int64_t q = pb; q < pend; q += stride) {  // one iteration = SS steps
                            ring.ensure(q + stride < pend ? q + stride : pend);
                            const int64_t P = q + s * k + r;
                            if (s < SS && P < pend && P < hi) v += ring.at(P);
                        }
                        for (int d = SS >> 1; d >= 1; d >>= 1)
                            v += __shfl_down_sync(FULL, v, d * k);
                        const double tot = __shfl_sync(FULL, v, live ? rank : 0);
                        if (live) acc += tot;
                        pb = pend;
                        t += steps;
                    } else {
                        const int32_t n1 = steps > 8 ? 1 : steps;
                        for (int32_t i = 0; i < n1; ++i) {
                            ring.ensure(pb + k);
                            const int64_t P = pb + rank;
                            if (live && P >= lo && P < hi) acc += ring.at(P);
                            pb += k;
                        }
                        t += n1;
                    }
                    if (t == t1) {
                        if (++j == nph) break;
                        pm = S.ph_mask[j];
                        k = __popc(pm);
                        t1 = S.ph_t1[j];
                        live = (pm >> lane) & 1u;
                        rank = __popc(pm & lt);
                    }
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
    k_spmv_stream<V, EXACT, CH, MINB, XNA><<<grid, kThreads, smem, st>>>(
        *f, *b, (const V *)x, (V *)y, partial);
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

// Tile / occupancy variants (chunk CH, min CTAs per SM, L1 policy of the x
// gathers), chosen with HBP_STREAM_VARIANT for sweeps; 0 is the default.
constexpr int kVariants = 5;
int variant() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("HBP_STREAM_VARIANT");
        v = e ? atoi(e) : 0;
        if (v < 0 || v >= kVariants) v = 0;
    }
    return v;
}

#define HBP_STREAM_VARIANTS(FN, V, EXACT, ...)                   \
    switch (variant()) {                                          \
        case 1: return FN<V, EXACT, 128, 4, true>(__VA_ARGS__);  \
        case 2: return FN<V, EXACT, 256, 3, true>(__VA_ARGS__);  \
        case 3: return FN<V, EXACT, 128, 3, false>(__VA_ARGS__); \
        case 4: return FN<V, EXACT, 128, 2, true>(__VA_ARGS__);  \
        default: return FN<V, EXACT, 128, 3, true>(__VA_ARGS__); \
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
