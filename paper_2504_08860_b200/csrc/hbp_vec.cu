// hbp_vec.cu -- the vector steps around an iterated SpMV (power iteration,
// config 5: x <- A x / ||A x||_2), so a step is SpMV + two small kernels
// instead of a chain of framework ops.
//
//   hbp_sumsq:  out[0] = sum_i y_i^2 in f64, deterministic (fixed grid, fixed
//               per-block tree, one final block in a fixed order);
//   hbp_scale:  out_i = y_i * (V)(1 / sqrt(sumsq[0]))  (sumsq read on the
//               device after an optional all-reduce: no host round trip).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "hbp.h"
#include "hbp_common.cuh"

using namespace hbp;

namespace {

constexpr int kT = 512;
constexpr int kBlocks = 592;  // 4 x 148 SMs

__device__ __forceinline__ double block_sum(double v, double *sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    v = threadIdx.x < kT / 32 ? sh[threadIdx.x] : 0.0;
    if (wid == 0)
        for (int o = 8; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

template <typename V>
__global__ void __launch_bounds__(kT) k_sumsq_partial(const V *__restrict__ y, int64_t n,
                                                      double *__restrict__ part) {
    __shared__ double sh[kT / 32];
    double s = 0.0;
    const int64_t stride = (int64_t)gridDim.x * kT;
    for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride) {
        const double v = (double)__ldcs(y + i);
        s = fma(v, v, s);
    }
    s = block_sum(s, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kT) k_sumsq_final(const double *__restrict__ part, int n,
                                                    double *__restrict__ out) {
    __shared__ double sh[kT / 32];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += kT) s += part[i];
    s = block_sum(s, sh);
    if (threadIdx.x == 0) out[0] = s;
}

template <typename V>
__global__ void k_scale(const V *__restrict__ y, int64_t n, const double *__restrict__ sumsq,
                        V *__restrict__ out) {
    const V f = (V)(1.0 / sqrt(sumsq[0]));
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = __ldcs(y + i) * f;
}

template <typename V>
__global__ void k_add(V *__restrict__ y, const V *__restrict__ a, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        y[i] = y[i] + __ldcs(a + i);
}

}  // namespace

extern "C" {

int hbp_sumsq(const void *y, int dtype, int64_t n, double *scratch, double *out,
              hbp_stream_t stream) {
    if (n < 0 || !out || !scratch || (n > 0 && !y)) return HBP_E_ARG;
    cudaStream_t st = as_stream(stream);
    if (dtype == HBP_F32)
        k_sumsq_partial<float><<<kBlocks, kT, 0, st>>>((const float *)y, n, scratch);
    else if (dtype == HBP_F64)
        k_sumsq_partial<double><<<kBlocks, kT, 0, st>>>((const double *)y, n, scratch);
    else
        return HBP_E_ARG;
    k_sumsq_final<<<1, kT, 0, st>>>(scratch, kBlocks, out);
    return (int)cudaGetLastError();
}

int hbp_sumsq_scratch(int64_t *doubles) {
    if (!doubles) return HBP_E_ARG;
    *doubles = kBlocks;
    return HBP_OK;
}

int hbp_scale(const void *y, int dtype, int64_t n, const double *sumsq, void *out,
              hbp_stream_t stream) {
    if (n < 0 || !sumsq || (n > 0 && (!y || !out))) return HBP_E_ARG;
    if (n == 0) return HBP_OK;
    cudaStream_t st = as_stream(stream);
    const unsigned grid = grid_for(n, 256, 148LL * 16);
    if (dtype == HBP_F32)
        k_scale<float><<<grid, 256, 0, st>>>((const float *)y, n, sumsq, (float *)out);
    else if (dtype == HBP_F64)
        k_scale<double><<<grid, 256, 0, st>>>((const double *)y, n, sumsq, (double *)out);
    else
        return HBP_E_ARG;
    return (int)cudaGetLastError();
}

int hbp_add(void *y, const void *a, int dtype, int64_t n, hbp_stream_t stream) {
    if (n < 0 || (n > 0 && (!y || !a))) return HBP_E_ARG;
    if (n == 0) return HBP_OK;
    cudaStream_t st = as_stream(stream);
    const unsigned grid = grid_for(n, 256, 148LL * 16);
    if (dtype == HBP_F32) k_add<float><<<grid, 256, 0, st>>>((float *)y, (const float *)a, n);
    else if (dtype == HBP_F64) k_add<double><<<grid, 256, 0, st>>>((double *)y, (const double *)a, n);
    else return HBP_E_ARG;
    return (int)cudaGetLastError();
}

// ---- peer mappings (CUDA IPC) for the fused power iteration
// cuMemGetAddressRange through the runtime's driver entry point (no libcuda
// link dependency: the library still loads on a host without a driver).
typedef int (*hbp_get_range_fn)(unsigned long long *, size_t *, unsigned long long);

int hbp_ipc_export(const void *ptr, void *handle, int64_t *offset) {
    if (!ptr || !handle || !offset) return HBP_E_ARG;
    static_assert(sizeof(cudaIpcMemHandle_t) == HBP_IPC_HANDLE_BYTES, "IPC handle size");
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    HBP_CUDA_TRY(cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &fn, 12000,
                                                  cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) return HBP_E_UNSUPPORTED;
    unsigned long long base = 0;
    size_t size = 0;
    if (((hbp_get_range_fn)fn)(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0)
        return HBP_E_ARG;
    cudaIpcMemHandle_t h;
    HBP_CUDA_TRY(cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base));
    memcpy(handle, &h, sizeof h);
    *offset = (int64_t)((uintptr_t)ptr - (uintptr_t)base);
    return HBP_OK;
}

int hbp_ipc_open(const void *handle, int64_t offset, void **ptr) {
    if (!handle || !ptr || offset < 0) return HBP_E_ARG;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    void *base = nullptr;
    HBP_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *ptr = (char *)base + offset;
    return HBP_OK;
}

int hbp_ipc_close(void *base) {
    if (!base) return HBP_E_ARG;
    HBP_CUDA_TRY(cudaIpcCloseMemHandle(base));
    return HBP_OK;
}

}  // extern "C"
