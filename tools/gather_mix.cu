// gather_mix.cu -- do shared-memory (or cluster DSMEM) gathers and L2 gathers
// share one per-SM rate, or add up?  (calibration, not product code)
//
// Every kernel streams a u32 index array (16-byte loads, evict-first) and
// gathers one f32 per index: a fraction f of the indices (selected by their
// top byte) read a 64 KB x segment in shared memory -- the CTA's own
// (CL = 0, ld.shared) or cluster rank (i >> 14) % CL's (ld.shared::cluster) --
// and the rest read a 16 MB L2-resident x (ld.global.nc.L1::no_allocate,
// evict-last).  Reported: total gathers per SM-cycle.  If the two paths were
// independent, the mixed rate would exceed both pure rates; if they share
// the LSU / MIO path it falls between them (time = n_s / r_s + n_g / r_g).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_mix tools/gather_mix.cu
//   ./tools/gather_mix [log2 n]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

constexpr int SEG = 16384;               // floats per CTA segment (64 KB; 3 CTAs per SM)
constexpr uint32_t XMASK = (1u << 22) - 1;  // 16 MB of f32 in L2

__device__ unsigned long long g_clk[2], g_ns[2];
__device__ __forceinline__ void stamp(int w) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_ns[w] = t;
        g_clk[w] = clock64();
    }
}

__global__ void k_fill_idx(uint32_t *idx, int64_t n, uint64_t seed) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        idx[i] = (uint32_t)(z ^ (z >> 31));
    }
}
__global__ void k_fill_f(float *x, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = (float)(i & 1023) * 0.001f;
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

template <int CL>
__global__ void __launch_bounds__(512) k_mix(const uint32_t *__restrict__ idx, const float *x,
                                             int64_t n4, uint32_t thr, float *out) {
    extern __shared__ __align__(16) float seg[];
    uint32_t rank = 0;
    if (CL >= 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int i = threadIdx.x; i < SEG; i += blockDim.x) seg[i] = x[(int64_t)rank * SEG + i];
    if (CL >= 1)
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
    stamp(0);
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(seg);
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int64_t i = tid; i < n4; i += nth * 4) {
        uint4 c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t j = i + u * nth;
            c[u] = j < n4 ? ld_idx(reinterpret_cast<const uint4 *>(idx) + j) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t cs[4] = {c[u].x, c[u].y, c[u].z, c[u].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float v;
                if ((cs[k] >> 24) < thr) {
                    const uint32_t a = base + (cs[k] & (SEG - 1)) * 4u;
                    if constexpr (CL == 0) {
                        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
                    } else {
                        const uint32_t r = (cs[k] >> 14) % CL;
                        uint32_t ra;
                        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r));
                        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra));
                    }
                } else {
                    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
                                 : "=f"(v)
                                 : "l"(x + (cs[k] & XMASK)), "l"(pol));
                }
                acc[k] += v;
            }
        }
    }
    out[tid] = acc[0] + acc[1] + acc[2] + acc[3];
    stamp(1);
    if (CL >= 1)
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main(int argc, char **argv) {
    const int lg = argc > 1 ? atoi(argv[1]) : 27;
    const int64_t n = (int64_t)1 << lg, n4 = n / 4;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint32_t *idx;
    float *x, *out;
    CK(cudaMalloc(&idx, n * 4));
    CK(cudaMalloc(&x, (size_t)(XMASK + 1) * 4));
    CK(cudaMalloc(&out, (size_t)sms * 3 * 512 * 4));
    k_fill_f<<<1024, 256>>>(x, XMASK + 1);
    k_fill_idx<<<2048, 256>>>(idx, n, 777);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const size_t sm = SEG * 4;
    auto run = [&](auto kern, int cl, const char *name, uint32_t thr) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)(cl > 1 ? 3 * sms / cl * cl : 3 * sms));
        lc.blockDim = dim3(512);
        lc.dynamicSmemBytes = sm;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl > 1 ? cl : 1;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = cl >= 1 ? 1 : 0;
        float best = 1e30f;
        double mhz = 0;
        for (int r = 0; r < 6; ++r) {
            CK(cudaEventRecord(e0));
            CK(cudaLaunchKernelEx(&lc, kern, (const uint32_t *)idx, (const float *)x, n4, thr, out));
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (r > 0 && ms < best) {
                best = ms;
                unsigned long long c[2], t[2];
                CK(cudaMemcpyFromSymbol(c, g_clk, sizeof c));
                CK(cudaMemcpyFromSymbol(t, g_ns, sizeof t));
                mhz = (double)(c[1] - c[0]) / ((double)(t[1] - t[0]) / 1e3);
            }
        }
        const double f = thr / 256.0;
        const double per_cyc = n / (best * 1e-3) / (mhz * 1e6) / sms;
        printf("{\"method\": \"%s\", \"smem_fraction\": %.3f, \"ms\": %.4f, \"G_per_s\": %.2f, "
               "\"per_sm_cycle\": %.3f, \"sm_mhz\": %.0f}\n",
               name, f, best, n / (best * 1e-3) / 1e9, per_cyc, mhz);
        fflush(stdout);
    };
    const uint32_t thrs[] = {0, 64, 128, 192, 256};
    for (uint32_t t : thrs) run(k_mix<0>, 0, "lds_mix", t);
    for (uint32_t t : thrs) run(k_mix<2>, 2, "dsmem_c2_mix", t);
    for (uint32_t t : thrs) run(k_mix<4>, 4, "dsmem_c4_mix", t);
    return 0;
}
