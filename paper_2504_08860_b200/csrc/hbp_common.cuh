// hbp_common.cuh -- shared device helpers for libhbp.so (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "hbp.h"

#define HBP_CUDA_TRY(expr)                          \
    do {                                            \
        cudaError_t _e = (expr);                    \
        if (_e != cudaSuccess) return (int)_e;      \
    } while (0)

#define HBP_LAUNCH_CHECK() HBP_CUDA_TRY(cudaGetLastError())

namespace hbp {

static inline cudaStream_t as_stream(hbp_stream_t s) { return (cudaStream_t)s; }

static inline unsigned grid_for(int64_t n, int threads, int64_t cap = 148LL * 64) {
    int64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

// ---- lane-group ("segment") geometry ---------------------------------------
// A lane group of W <= 32 lanes is the unit that owns one HBP warp group
// (hbp.py:17-19).  A hardware warp holds spw = 32 / W segments; lanes at or
// above spw*W idle.  Segment masks let sub-warp groups use warp intrinsics
// independently (tiled-partition style).
struct Seg {
    int W;            // lanes per group
    int spw;          // segments per warp
    int seg;          // this lane's segment (>= spw: idle lane)
    int q;            // lane within the segment
    unsigned mask;    // member mask of this segment
    int shift;        // bit offset of the segment within the warp
    __device__ __forceinline__ bool idle() const { return seg >= spw; }
};

__device__ __forceinline__ Seg make_seg(int W) {
    Seg s;
    int lane = threadIdx.x & 31;
    s.W = W;
    s.spw = 32 / W;
    s.seg = lane / W;
    s.q = lane - s.seg * W;
    if (s.seg >= s.spw) {
        s.mask = 1u << lane;  // idle lanes form singleton segments
        s.shift = lane;
    } else {
        s.shift = s.seg * W;
        s.mask = (W == 32) ? 0xffffffffu : (((1u << W) - 1u) << s.shift);
    }
    return s;
}

// ballot restricted to the segment, shifted so bit i = lane i of the segment
__device__ __forceinline__ unsigned seg_ballot(const Seg &s, bool p) {
    return __ballot_sync(s.mask, p) >> s.shift;
}

__device__ __forceinline__ uint32_t seg_min_u32(const Seg &s, uint32_t v) {
    return __reduce_min_sync(s.mask, v);
}

__device__ __forceinline__ uint32_t seg_add_u32(const Seg &s, uint32_t v) {
    return __reduce_add_sync(s.mask, v);
}

// 64-bit segment sum for any W (tree toward segment lane 0, then broadcast);
// every shuffle source stays inside the segment.
__device__ __forceinline__ long long seg_add_i64(const Seg &s, long long v) {
    int lane = threadIdx.x & 31;
    for (int off = 1; off < s.W; off <<= 1) {
        bool ok = s.q + off < s.W;
        long long o = __shfl_sync(s.mask, v, ok ? lane + off : lane);
        if (ok) v += o;
    }
    return __shfl_sync(s.mask, v, s.shift);
}

// ---- cache-hinted loads ------------------------------------------------------
// Element arrays (col, data) are streamed once: no L1 allocation, evict-first
// L2 policy.  x is gathered repeatedly: normal L1 allocation, evict-last L2
// policy.  Policies come from createpolicy (one per kernel, kept in a reg).
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t *p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_stream(const float *p, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
                 : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_stream(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_x(const float *p, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_x(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

// x gathers that do not allocate L1 lines (L2 evict-last policy kept)
__device__ __forceinline__ float ld_x_na(const float *p, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
                 : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_x_na(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

// ---- PTX helpers: mbarrier + bulk async copy (sm_90+ / sm_100a) ------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *m, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(m)), "r"(count));
}
__device__ __forceinline__ void mbar_inval(uint64_t *m) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_addr(m)) : "memory");
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

__device__ __forceinline__ int64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (int64_t)t;
}

}  // namespace hbp
