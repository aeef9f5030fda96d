// hbp_hot.cu -- hot-column staging metadata for hbp_spmv_stream (B200).
//
// A random-column SpMV is bound by the x gathers: every 4-byte gather is its
// own L1 -> L2 sector request (tools/gather_ceiling.cu).  On
// power-law matrices (R-MAT, cfg2/cfg5) a few thousand columns carry a large
// share of the nonzeros, so the stream kernel copies x at the n_hot heaviest
// columns into each SM's shared memory once per SpMV and serves those
// gathers from there.  This file builds the metadata at convert time:
//   deg[c]      column degrees (one pass over the element stream, or over
//               every stride-th element on large matrices: the ranking only
//               steers performance, any hot set gives the same results);
//   hot_cols    the n_hot columns of largest degree (host: stable radix sort);
//   slot_of[c]  hot slot of column c or -1;
//   scol[e]     the element stream's columns with hot ones replaced by
//               HBP_HOT_FLAG | slot (the stream kernel streams scol instead
//               of col; col itself stays the reference's array).
// Products and their order are unchanged, so SpMV results are identical with
// and without staging.
#include <cuda_runtime.h>
#include <stdint.h>

#include "hbp.h"
#include "hbp_common.cuh"

using namespace hbp;

namespace {

// deg[c] += 1 for every element e = i * stride (stride 1: exact degrees)
__global__ void k_col_degree(const uint4 *__restrict__ col4, const uint32_t *__restrict__ col,
                             int64_t nnz, int64_t stride_e, uint32_t *__restrict__ deg) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (stride_e == 1) {
        const int64_t n4 = nnz >> 2;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
            const uint4 c = __ldcs(col4 + i);
            atomicAdd(deg + c.x, 1u);
            atomicAdd(deg + c.y, 1u);
            atomicAdd(deg + c.z, 1u);
            atomicAdd(deg + c.w, 1u);
        }
        for (int64_t i = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
             i += stride)
            atomicAdd(deg + col[i], 1u);
        return;
    }
    const int64_t ns = (nnz + stride_e - 1) / stride_e;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += stride)
        atomicAdd(deg + __ldcs(col + i * stride_e), 1u);
}

__global__ void k_hot_slots(const uint32_t *__restrict__ hot_cols, int64_t n_hot,
                            int32_t *__restrict__ slot_of) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n_hot) slot_of[hot_cols[s]] = (int32_t)s;
}

template <bool PACKED>
__global__ void k_hot_remap(const uint4 *__restrict__ col4, const uint32_t *__restrict__ col,
                            int64_t nnz, const int32_t *__restrict__ slot_of, int32_t n_hot,
                            uint4 *__restrict__ scol4, uint32_t *__restrict__ scol) {
    const int64_t n4 = nnz >> 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    auto map = [&](uint32_t c) -> uint32_t {
        const int32_t s = __ldg(slot_of + c);
        if (s < 0) return PACKED ? 0u : c;  // (packed: every used column has a slot)
        if (s < n_hot) return HBP_HOT_FLAG | (uint32_t)s;
        return PACKED ? (uint32_t)(s - n_hot) : (HBP_WARM_FLAG | (uint32_t)(s - n_hot));
    };
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint4 c = __ldcs(col4 + i);
        __stcs(scol4 + i, make_uint4(map(c.x), map(c.y), map(c.z), map(c.w)));
    }
    for (int64_t i = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
         i += stride)
        scol[i] = map(col[i]);
}

}  // namespace

extern "C" {

int hbp_col_degree(const uint32_t *col, int64_t nnz, int64_t stride, uint32_t *deg,
                   hbp_stream_t stream) {
    if (nnz < 0 || stride < 1 || (nnz > 0 && (!col || !deg))) return HBP_E_ARG;
    if (nnz == 0) return HBP_OK;
    if (((uintptr_t)col & 15) != 0) return HBP_E_ARG;
    k_col_degree<<<grid_for(nnz / (4 * stride) + 1, 256), 256, 0, as_stream(stream)>>>(
        (const uint4 *)col, col, nnz, stride, deg);
    return (int)cudaGetLastError();
}

int hbp_hot_slots(const uint32_t *hot_cols, int64_t n_hot, int32_t *slot_of,
                  hbp_stream_t stream) {
    if (n_hot < 0 || (n_hot > 0 && (!hot_cols || !slot_of))) return HBP_E_ARG;
    if (n_hot == 0) return HBP_OK;
    k_hot_slots<<<(unsigned)((n_hot + 255) / 256), 256, 0, as_stream(stream)>>>(hot_cols, n_hot,
                                                                                 slot_of);
    return (int)cudaGetLastError();
}

int hbp_hot_remap(const uint32_t *col, int64_t nnz, const int32_t *slot_of, int64_t n_hot,
                  uint32_t *scol, hbp_stream_t stream) {
    if (nnz < 0 || n_hot < 0 || n_hot >= (1 << 30) || (nnz > 0 && (!col || !slot_of || !scol)))
        return HBP_E_ARG;
    if (nnz == 0) return HBP_OK;
    if ((((uintptr_t)col | (uintptr_t)scol) & 15) != 0) return HBP_E_ARG;
    k_hot_remap<false><<<grid_for(nnz / 4 + 1, 256), 256, 0, as_stream(stream)>>>(
        (const uint4 *)col, col, nnz, slot_of, (int32_t)n_hot, (uint4 *)scol, scol);
    return (int)cudaGetLastError();
}

int hbp_hot_remap_packed(const uint32_t *col, int64_t nnz, const int32_t *slot_of, int64_t n_hot,
                         uint32_t *scol, hbp_stream_t stream) {
    if (nnz < 0 || n_hot < 0 || n_hot >= (1 << 30) || (nnz > 0 && (!col || !slot_of || !scol)))
        return HBP_E_ARG;
    if (nnz == 0) return HBP_OK;
    if ((((uintptr_t)col | (uintptr_t)scol) & 15) != 0) return HBP_E_ARG;
    k_hot_remap<true><<<grid_for(nnz / 4 + 1, 256), 256, 0, as_stream(stream)>>>(
        (const uint4 *)col, col, nnz, slot_of, (int32_t)n_hot, (uint4 *)scol, scol);
    return (int)cudaGetLastError();
}

}  // extern "C"
