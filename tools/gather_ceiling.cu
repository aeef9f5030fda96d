// gather_ceiling.cu -- calibration microbenchmark (not product code).
// Streams an element array (col u32, val f32) and gathers x[col]: the memory
// traffic of an SpMV with no format bookkeeping at all.  Each warp sums 32
// consecutive products per iteration and writes one float per 1024
// elements, so the loads cannot be elided.  Its time is the floor any SpMV
// over the same column stream can reach on this GPU.
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint4 ldg_stream(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int U>
__global__ void __launch_bounds__(256) k_gather(const uint32_t *__restrict__ col,
                                                const float *__restrict__ val,
                                                const float *__restrict__ x, int64_t n4,
                                                float *__restrict__ out) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    float acc = 0.f;
    for (int64_t i = tid; i < n4; i += nth * U) {
        uint4 c[U];
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = i + u * nth;
            c[u] = j < n4 ? ldg_stream(reinterpret_cast<const uint4 *>(col) + j) : make_uint4(0, 0, 0, 0);
            v[u] = j < n4 ? ldg_stream(reinterpret_cast<const uint4 *>(val) + j) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc += __uint_as_float(v[u].x) * __ldg(x + c[u].x);
            acc += __uint_as_float(v[u].y) * __ldg(x + c[u].y);
            acc += __uint_as_float(v[u].z) * __ldg(x + c[u].z);
            acc += __uint_as_float(v[u].w) * __ldg(x + c[u].w);
        }
    }
    out[tid] = acc;
}

extern "C" int gather_ceiling(const uint32_t *col, const float *val, const float *x, int64_t n,
                              float *out, int blocks, int unroll, void *stream) {
    const int64_t n4 = n / 4;
    cudaStream_t s = (cudaStream_t)stream;
    if (unroll == 1) k_gather<1><<<blocks, 256, 0, s>>>(col, val, x, n4, out);
    else if (unroll == 2) k_gather<2><<<blocks, 256, 0, s>>>(col, val, x, n4, out);
    else k_gather<4><<<blocks, 256, 0, s>>>(col, val, x, n4, out);
    return (int)cudaGetLastError();
}
