// gather_peaks.cu -- measured random-gather ceilings on the B200 (calibration,
// not product code).  Every kernel streams the same u32 index array (16-byte
// coalesced loads), gathers one 4-byte x element per index by one method and
// sums the values (one float per thread is written, so nothing is elided):
//
//   stream_only          indices only (the index stream's own cost)
//   ldg_l1               ld.global.nc            (L1 allocating)
//   ldg_na               ld.global.nc.L1::no_allocate
//   ldg_na_el            ... + L2::evict_last policy
//   ldg_cg               ld.global.cg            (L2 only)
//   lds                  x segment (128 KB) in shared memory, ld.shared
//   dsmem_cN             x segment spread over an N-CTA cluster, ld.shared::cluster
//   tma_g4               cp.async.bulk.tensor.2d ... tile::gather4 (4 rows of 16 B
//                        per op into shared memory, mbarrier completion)
//   stream_val_*         the SpMV access pattern: idx + f32 value streamed,
//                        x gathered (plain / evict hints / persisting L2 window)
//   l2_seq, hbm_seq      sequential read bandwidth (L2-resident / beyond L2)
//
// Build + run:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gp gather_peaks.cu
//               ./gp [log2 n]          -> one JSON line per measurement
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

__device__ unsigned long long g_clk[2];
__device__ unsigned long long g_ns[2];

__device__ __forceinline__ void stamp(int which) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_ns[which] = t;
        g_clk[which] = clock64();
    }
}

__device__ __forceinline__ uint4 ld_idx(const uint4 *p) {
    uint4 v;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}

__global__ void k_fill_idx(uint32_t *idx, int64_t n, uint32_t ncols, uint64_t seed) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        idx[i] = (uint32_t)((z >> 32) % ncols);
    }
}
__global__ void k_fill_f(float *x, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = (float)(i & 1023) * 0.001f;
}

template <int MODE>
__device__ __forceinline__ float gx(const float *x, uint32_t c, uint64_t pol) {
    float v;
    if constexpr (MODE == 0) asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(x + c));
    else if constexpr (MODE == 1)
        asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(x + c));
    else if constexpr (MODE == 2)
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
                     : "=f"(v) : "l"(x + c), "l"(pol));
    else asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(x + c));
    return v;
}

// MODE 0..3: gathers; MODE -1: indices only
template <int MODE, int U>
__global__ void __launch_bounds__(256) k_ldg(const uint32_t *__restrict__ idx, const float *x,
                                             int64_t n4, float *out) {
    stamp(0);
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    float acc = 0.f;
    for (int64_t i = tid; i < n4; i += nth * U) {
        uint4 c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = i + u * nth;
            c[u] = j < n4 ? ld_idx(reinterpret_cast<const uint4 *>(idx) + j) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if constexpr (MODE < 0) {
                acc += (float)(c[u].x ^ c[u].y ^ c[u].z ^ c[u].w);
            } else {
                acc += gx<MODE>(x, c[u].x, pol) + gx<MODE>(x, c[u].y, pol) +
                       gx<MODE>(x, c[u].z, pol) + gx<MODE>(x, c[u].w, pol);
            }
        }
    }
    out[tid] = acc;
    stamp(1);
}

// SpMV access pattern: idx + value streamed (evict-first when HINT), x gathered
template <int HINT, int U>
__global__ void __launch_bounds__(256) k_spmv_pat(const uint32_t *__restrict__ idx,
                                                  const float *__restrict__ val, const float *x,
                                                  int64_t n4, float *out) {
    stamp(0);
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    float acc = 0.f;
    for (int64_t i = tid; i < n4; i += nth * U) {
        uint4 c[U], v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = i + u * nth;
            if (j < n4) {
                if (HINT) {
                    c[u] = ld_idx(reinterpret_cast<const uint4 *>(idx) + j);
                    v[u] = ld_idx(reinterpret_cast<const uint4 *>(val) + j);
                } else {
                    c[u] = __ldg(reinterpret_cast<const uint4 *>(idx) + j);
                    v[u] = __ldg(reinterpret_cast<const uint4 *>(val) + j);
                }
            } else {
                c[u] = v[u] = make_uint4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (HINT) {
                acc += __uint_as_float(v[u].x) * gx<2>(x, c[u].x, pol) +
                       __uint_as_float(v[u].y) * gx<2>(x, c[u].y, pol) +
                       __uint_as_float(v[u].z) * gx<2>(x, c[u].z, pol) +
                       __uint_as_float(v[u].w) * gx<2>(x, c[u].w, pol);
            } else {
                acc += __uint_as_float(v[u].x) * gx<1>(x, c[u].x, pol) +
                       __uint_as_float(v[u].y) * gx<1>(x, c[u].y, pol) +
                       __uint_as_float(v[u].z) * gx<1>(x, c[u].z, pol) +
                       __uint_as_float(v[u].w) * gx<1>(x, c[u].w, pol);
            }
        }
    }
    out[tid] = acc;
    stamp(1);
}

constexpr int SEG = 32768;  // floats per CTA segment (128 KB)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// CL == 0: plain ld.shared on the CTA's own segment; CL >= 1: the segment of
// cluster rank (idx / SEG) % CL through ld.shared::cluster
template <int CL, int U, int ILP = 1>
__global__ void __launch_bounds__(512) k_smem(const uint32_t *__restrict__ idx, const float *x,
                                              int64_t n4, float *out) {
    extern __shared__ __align__(16) float seg[];
    uint32_t rank = 0;
    if (CL >= 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int i = threadIdx.x; i < SEG; i += blockDim.x) seg[i] = x[(int64_t)rank * SEG + i];
    if (CL >= 1) cluster_sync_all();
    else __syncthreads();
    stamp(0);
    const uint32_t base = smem_u32(seg);
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    float accs[ILP * 4] = {};
    for (int64_t i = tid; i < n4; i += nth * U) {
        uint4 c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = i + u * nth;
            c[u] = j < n4 ? ld_idx(reinterpret_cast<const uint4 *>(idx) + j) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float &acc = accs[(u % ILP) * 4 + (ILP > 1 ? 0 : 0)];
            const uint32_t cs[4] = {c[u].x, c[u].y, c[u].z, c[u].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float v;
                const uint32_t a = base + (cs[k] & (SEG - 1)) * 4u;
                if constexpr (CL == 0) {
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
                } else {
                    const uint32_t r = (cs[k] / SEG) % CL;
                    uint32_t ra;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r));
                    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra));
                }
                if constexpr (ILP > 1) accs[(u % ILP) * 4 + k] += v;
                else acc += v;
            }
        }
    }
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < ILP * 4; ++k) acc += accs[k];
    out[tid] = acc;
    stamp(1);
    if (CL >= 1) cluster_sync_all();
}

// TMA gather4: x viewed as [ncols/4][4] f32 (16-byte rows).  Each lane issues
// one gather4 (its 4 indices -> 4 rows = 64 B) per chunk of 128 indices; the
// warp keeps NB chunks in flight in a shared-memory ring.
constexpr int G4_NB = 8;
struct __align__(128) G4Warp {
    float4 rows[G4_NB][32][8];  // 4 rows of 32 B per lane (128 B: TMA destinations are 128 B aligned)
    uint32_t sel[G4_NB][32];
    uint64_t mbar[G4_NB];
};

__global__ void __launch_bounds__(128) k_tma_g4(const __grid_constant__ CUtensorMap tm,
                                                const uint32_t *__restrict__ idx, int64_t nchunks,
                                                float *out) {
    extern __shared__ __align__(128) unsigned char raw[];
    unsigned char *al = raw + ((128u - (smem_u32(raw) & 127u)) & 127u);
    G4Warp &S = reinterpret_cast<G4Warp *>(al)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (lane == 0) {
        for (int s = 0; s < G4_NB; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.mbar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    stamp(0);
    auto issue = [&](int64_t ch, int s) {
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                             smem_u32(&S.mbar[s])),
                         "r"(32 * 128)
                         : "memory");
        __syncwarp();
        const uint4 c = ld_idx(reinterpret_cast<const uint4 *>(idx) + ch * 32 + lane);
        S.sel[s][lane] = (c.x & 7) | ((c.y & 7) << 8) | ((c.z & 7) << 16) | ((c.w & 7) << 24);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(&S.rows[s][lane][0])),
            "l"(&tm), "r"(0), "r"(c.x >> 3), "r"(c.y >> 3), "r"(c.z >> 3), "r"(c.w >> 3),
            "r"(smem_u32(&S.mbar[s]))
            : "memory");
    };
    int64_t it = 0;
    for (int s = 0; s < G4_NB; ++s) {
        const int64_t ch = wg + (int64_t)s * nw;
        if (ch < nchunks) issue(ch, s);
    }
    float acc = 0.f;
    for (int64_t ch = wg; ch < nchunks; ch += nw, ++it) {
        const int s = (int)(it % G4_NB);
        const uint32_t par = (uint32_t)((it / G4_NB) & 1);
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(
                smem_u32(&S.mbar[s])),
            "r"(par)
            : "memory");
        const uint32_t sl = S.sel[s][lane];
        const float *r = reinterpret_cast<const float *>(&S.rows[s][lane][0]);
        acc += r[sl & 7] + r[8 + ((sl >> 8) & 7)] + r[16 + ((sl >> 16) & 7)] + r[24 + ((sl >> 24) & 7)];
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const int64_t nx = ch + (int64_t)G4_NB * nw;
        if (nx < nchunks) issue(nx, s);
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
    stamp(1);
}

__global__ void __launch_bounds__(512) k_seq(const uint4 *__restrict__ a, int64_t n16, int reps,
                                             float *out) {
    stamp(0);
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    for (int r = 0; r < reps; ++r)
        for (int64_t i = tid; i < n16; i += nth * 4) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t j = i + u * nth;
                v[u] = j < n16 ? __ldcg(a + j) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        }
    out[tid] = (float)acc;
    stamp(1);
}

typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static cudaEvent_t e0, e1;
static int g_sms = 148;

template <class F>
static double time_ms(F f, int reps = 7) {
    std::vector<float> t;
    f();
    f();
    CK(cudaDeviceSynchronize());
    for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(e0));
        f();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

static double sm_mhz() {
    unsigned long long c[2], n[2];
    CK(cudaMemcpyFromSymbol(c, g_clk, sizeof c));
    CK(cudaMemcpyFromSymbol(n, g_ns, sizeof n));
    return n[1] > n[0] ? (double)(c[1] - c[0]) * 1e3 / (double)(n[1] - n[0]) : 0.0;
}

static void report(const char *method, double xmb, int64_t n, double ms, const char *extra = "") {
    const double mhz = sm_mhz();
    const double gps = n / (ms * 1e-3) / 1e9;
    const double per_cyc = mhz > 0 ? n / (ms * 1e-3) / (g_sms * mhz * 1e6) : 0.0;
    printf("{\"method\": \"%s\", \"x_mb\": %.1f, \"n\": %lld, \"ms\": %.4f, \"G_per_s\": %.2f, "
           "\"per_sm_cycle\": %.3f, \"sm_mhz\": %.0f, \"ms_per_100M\": %.4f%s}\n",
           method, xmb, (long long)n, ms, gps, per_cyc, mhz, ms * 1e8 / n, extra);
    fflush(stdout);
}

int main(int argc, char **argv) {
    const int lg = argc > 1 ? atoi(argv[1]) : 27;
    const bool only_tma = argc > 2 && strcmp(argv[2], "tma") == 0;
    const int64_t n = (int64_t)1 << lg;
    CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    uint32_t *idx;
    float *x, *out, *val;
    const int64_t xmax = (int64_t)64 << 20;  // 256 MB of f32
    CK(cudaMalloc(&idx, n * 4));
    CK(cudaMalloc(&val, n * 4));
    CK(cudaMalloc(&x, xmax * 4));
    CK(cudaMalloc(&out, (size_t)g_sms * 2048 * 4 * 16));
    k_fill_f<<<1024, 256>>>(x, xmax);
    k_fill_f<<<1024, 256>>>(val, n);
    const int64_t n4 = n / 4;
    const int G = g_sms * 8;  // 8 x 256 threads per SM

    // sequential bandwidths
    if (!only_tma) {
        const int64_t l2b = (int64_t)32 << 20;
        double ms = time_ms([&] { k_seq<<<g_sms * 4, 512>>>((const uint4 *)x, l2b / 16, 16, out); });
        report("l2_seq_read_32MB", 32, l2b * 16 / 4, ms, ", \"GB_per_s\": 0");
        printf("{\"method\": \"l2_seq_read_32MB_GBps\", \"GB_per_s\": %.1f}\n", l2b * 16 / ms / 1e6);
        const int64_t hb = n * 4 * 2;  // idx + val (contiguous allocations, read separately)
        double ms2 = time_ms([&] {
            k_seq<<<g_sms * 4, 512>>>((const uint4 *)idx, n * 4 / 16, 1, out);
            k_seq<<<g_sms * 4, 512>>>((const uint4 *)val, n * 4 / 16, 1, out);
        });
        printf("{\"method\": \"hbm_seq_read\", \"bytes\": %lld, \"ms\": %.4f, \"GB_per_s\": %.1f}\n",
               (long long)hb, ms2, hb / ms2 / 1e6);
    }
    const int64_t xsizes[] = {(int64_t)1 << 20, 6250000, (int64_t)16 << 20, (int64_t)64 << 20};
    const int64_t xsizes_g[] = {(int64_t)16 << 10, (int64_t)1 << 20, 6250000, (int64_t)16 << 20,
                                (int64_t)64 << 20};
    for (int64_t nc : xsizes_g) {
        if (only_tma) break;
        const double xmb = nc * 4.0 / 1e6;
        k_fill_idx<<<2048, 256>>>(idx, n, (uint32_t)nc, 12345);
        CK(cudaDeviceSynchronize());
        report("stream_only", xmb, n, time_ms([&] { k_ldg<-1, 4><<<G, 256>>>(idx, x, n4, out); }));
        report("ldg_l1", xmb, n, time_ms([&] { k_ldg<0, 4><<<G, 256>>>(idx, x, n4, out); }));
        report("ldg_na", xmb, n, time_ms([&] { k_ldg<1, 4><<<G, 256>>>(idx, x, n4, out); }));
        report("ldg_na_el", xmb, n, time_ms([&] { k_ldg<2, 4><<<G, 256>>>(idx, x, n4, out); }));
        report("ldg_cg", xmb, n, time_ms([&] { k_ldg<3, 4><<<G, 256>>>(idx, x, n4, out); }));
        report("ldg_na_u2", xmb, n, time_ms([&] { k_ldg<1, 2><<<G, 256>>>(idx, x, n4, out); }));
        report("spmv_pat_plain", xmb, n,
               time_ms([&] { k_spmv_pat<0, 4><<<G, 256>>>(idx, val, x, n4, out); }));
        report("spmv_pat_hints", xmb, n,
               time_ms([&] { k_spmv_pat<1, 4><<<G, 256>>>(idx, val, x, n4, out); }));
        // persisting L2 window on x (cudaLimitPersistingL2CacheSize at its maximum)
        {
            int maxp = 0;
            CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0));
            CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp));
            cudaStream_t st;
            CK(cudaStreamCreate(&st));
            cudaStreamAttrValue av = {};
            av.accessPolicyWindow.base_ptr = x;
            av.accessPolicyWindow.num_bytes = std::min<size_t>(nc * 4, (size_t)maxp);
            av.accessPolicyWindow.hitRatio = 1.0f;
            av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
            std::vector<float> t;
            for (int r = 0; r < 9; ++r) {
                CK(cudaEventRecord(e0, st));
                k_spmv_pat<0, 4><<<G, 256, 0, st>>>(idx, val, x, n4, out);
                CK(cudaEventRecord(e1, st));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                if (r >= 2) t.push_back(ms);
            }
            std::sort(t.begin(), t.end());
            char ex[96];
            snprintf(ex, sizeof ex, ", \"persist_max_mb\": %.1f", maxp / 1e6);
            report("spmv_pat_persist", xmb, n, t[t.size() / 2], ex);
            av.accessPolicyWindow.num_bytes = 0;
            CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
            CK(cudaCtxResetPersistingL2Cache());
            CK(cudaStreamDestroy(st));
            CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0));
        }
    }
    // shared memory / DSMEM / TMA gather4 (x segment = CL * 128 KB)
    if (!only_tma) {
        k_fill_idx<<<2048, 256>>>(idx, n, (uint32_t)1 << 24, 777);  // any 24-bit value; masked
        CK(cudaDeviceSynchronize());
        const size_t sm = SEG * 4;
        CK(cudaFuncSetAttribute(k_smem<0, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        report("lds_128KB", 0.131, n, time_ms([&] { k_smem<0, 4><<<g_sms, 512, sm>>>(idx, x, n4, out); }));
        // independent accumulators: the shared-memory crossbar's own rate, not
        // the add chain's latency
        CK(cudaFuncSetAttribute(k_smem<0, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        report("lds_128KB_ilp", 0.131, n,
               time_ms([&] { k_smem<0, 4, 4><<<g_sms, 512, sm>>>(idx, x, n4, out); }));
        auto dsm = [&](auto kern, int cl, const char *name) {
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            if (cl > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3((unsigned)(g_sms / cl * cl));
            lc.blockDim = dim3(512);
            lc.dynamicSmemBytes = sm;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            cudaError_t err = cudaSuccess;
            double ms = time_ms([&] { err = cudaLaunchKernelEx(&lc, kern, (const uint32_t *)idx, (const float *)x, n4, out); });
            if (err != cudaSuccess) {
                printf("{\"method\": \"%s\", \"error\": \"%s\"}\n", name, cudaGetErrorString(err));
                cudaGetLastError();
                return;
            }
            report(name, 0.131 * cl, n, ms);
        };
        dsm(k_smem<1, 4>, 1, "dsmem_c1");
        dsm(k_smem<2, 4>, 2, "dsmem_c2");
        dsm(k_smem<4, 4>, 4, "dsmem_c4");
        dsm(k_smem<8, 4>, 8, "dsmem_c8");
        dsm(k_smem<16, 4>, 16, "dsmem_c16");
    }
    {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        EncodeTiled enc = (EncodeTiled)fn;
        for (int64_t nc : xsizes) {
            k_fill_idx<<<2048, 256>>>(idx, n, (uint32_t)nc, 12345);
            CK(cudaDeviceSynchronize());
            CUtensorMap tm;
            cuuint64_t dims[2] = {8, (cuuint64_t)(nc / 8)};
            cuuint64_t strides[1] = {32};
            cuuint32_t box[2] = {8, 1};
            cuuint32_t es[2] = {1, 1};
            CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) {
                printf("{\"method\": \"tma_g4\", \"error\": \"encode %d\"}\n", (int)r);
                break;
            }
            const size_t sm = sizeof(G4Warp) * 4 + 128;
            CK(cudaFuncSetAttribute(k_tma_g4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            for (int cps : {1, 2, 3}) {
                char name[64];
                snprintf(name, sizeof name, "tma_g4_%dcta", cps);
                double ms = time_ms([&] { k_tma_g4<<<g_sms * cps, 128, sm>>>(tm, idx, n / 128, out); });
                cudaError_t err = cudaGetLastError();
                if (err != cudaSuccess) {
                    printf("{\"method\": \"%s\", \"error\": \"%s\"}\n", name, cudaGetErrorString(err));
                    exit(0);
                }
                report(name, nc * 4.0 / 1e6, n, ms);
            }
        }
    }
    CK(cudaDeviceSynchronize());
    return 0;
}
