// hbp_baselines.cu -- the paper's comparison kernels on sm_100a.
//
//   CSR (Alg. 1; formats.py:266-273 -> _kernels.py:13-19
//        csr_kernel): one thread per row, left to right in storage order.
//   plain 2D (engine.py:204-225 -> _kernels.py:50-59 block2d_kernel): every
//        nonzero block, each row's run of the block in CSR order (no
//        reordering, no interleaving), into the compact partial; the combine
//        is hbp_combine.  A warp per block, a lane per row.
// Both accumulate unfused in the reference order, so f64 results are
// bitwise identical to the reference; f32 values accumulate in f64.
#include <cuda_runtime.h>
#include <stdint.h>

#include "hbp.h"
#include "hbp_common.cuh"

using namespace hbp;

namespace {

template <typename V>
__device__ __forceinline__ double madd(double s, V v, V xv) {
    return __dadd_rn(s, __dmul_rn((double)v, (double)xv));
}

template <typename V>
__global__ void k_csr(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                      const V *__restrict__ val, int64_t rows, const V *__restrict__ x,
                      V *__restrict__ y) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t j = row_ptr[r], e = row_ptr[r + 1]; j < e; ++j)
            s = madd<V>(s, val[j], __ldg(x + col[j]));
        y[r] = (V)s;
    }
}

template <typename V>
__global__ void k_block2d(const uint32_t *__restrict__ len_local,
                          const int64_t *__restrict__ start_local,
                          const int32_t *__restrict__ blk_br, int64_t nzb, int64_t rows,
                          int64_t R, const int32_t *__restrict__ col, const V *__restrict__ val,
                          const V *__restrict__ x, double *__restrict__ partial) {
    const int lane = threadIdx.x & 31;
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = warp; b < nzb; b += nwarps) {
        int64_t n = rows - (int64_t)blk_br[b] * R;
        if (n > R) n = R;
        for (int64_t r = lane; r < n; r += 32) {
            const int64_t s0 = start_local[b * R + r];
            const uint32_t cnt = len_local[b * R + r];
            double s = 0.0;
            for (uint32_t k = 0; k < cnt; ++k) s = madd<V>(s, val[s0 + k], __ldg(x + col[s0 + k]));
            partial[b * R + r] = s;
        }
    }
}

}  // namespace

extern "C" {

int hbp_csr_spmv(const int64_t *row_ptr, const int32_t *col_idx, const void *values, int dtype,
                 int64_t rows, const void *x, void *y, hbp_stream_t stream) {
    if (rows < 1) return HBP_OK;
    unsigned grid = grid_for(rows, 256);
    cudaStream_t s = as_stream(stream);
    if (dtype == HBP_F64)
        k_csr<double><<<grid, 256, 0, s>>>(row_ptr, col_idx, (const double *)values, rows,
                                           (const double *)x, (double *)y);
    else if (dtype == HBP_F32)
        k_csr<float><<<grid, 256, 0, s>>>(row_ptr, col_idx, (const float *)values, rows,
                                          (const float *)x, (float *)y);
    else
        return HBP_E_ARG;
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_block2d_spmv(const uint32_t *len_local, const int64_t *start_local, const int32_t *blk_br,
                     int64_t nzb, int64_t rows, int64_t row_height, const int32_t *col_idx,
                     const void *values, int dtype, const void *x, double *partial,
                     hbp_stream_t stream) {
    if (nzb <= 0) return HBP_OK;
    unsigned grid = grid_for(nzb * 32, 256);
    cudaStream_t s = as_stream(stream);
    if (dtype == HBP_F64)
        k_block2d<double><<<grid, 256, 0, s>>>(len_local, start_local, blk_br, nzb, rows,
                                               row_height, col_idx, (const double *)values,
                                               (const double *)x, partial);
    else if (dtype == HBP_F32)
        k_block2d<float><<<grid, 256, 0, s>>>(len_local, start_local, blk_br, nzb, rows,
                                              row_height, col_idx, (const float *)values,
                                              (const float *)x, partial);
    else
        return HBP_E_ARG;
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

}  // extern "C"
