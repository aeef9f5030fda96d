// hbp_stats.cu -- per-group lane statistics (the reference's Fig. 6
// load-balance analytics, metrics.py:26-79) on sm_100a.
//
// One thread per (nonzero block, lane group): the group's lane counts are
// the in-block row lengths in slot order (slot -> local row through the
// block's permutation, or the identity), and
//   mean        = sum / n                      (integer sum, exact)
//   std_dev     = sqrt(sum_pw((x - mean)^2) / n)  population std
//   max         = max lane count
//   utilization = sum / (W * max), 1.0 for an all-zero group
// with sum_pw numpy's pairwise float64 summation (sequential below 8 terms,
// 8 interleaved accumulators up to 128), so mean and std_dev are bitwise
// equal to numpy's ndarray.mean() / ndarray.std() on the same lanes.
// Groups of empty blocks are left to the caller's initial values (zeros,
// utilization 1.0).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "hbp.h"
#include "hbp_common.cuh"

using namespace hbp;

namespace {

// numpy pairwise_sum for n <= 128 (here n <= 32)
__device__ double np_pairwise_small(const double *a, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
        return r;
    }
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
}

__global__ void k_group_stats(const int32_t *__restrict__ blk_br,
                              const int32_t *__restrict__ blk_bc, int64_t nzb,
                              const int32_t *__restrict__ len_local,
                              const uint32_t *__restrict__ perm, int64_t rows, int64_t R,
                              int64_t W, int64_t gpc, int32_t *__restrict__ lanes,
                              double *__restrict__ mean, double *__restrict__ stdv,
                              int32_t *__restrict__ maxv, double *__restrict__ util) {
    const int64_t gpb = R / W;
    const int64_t total = nzb * gpb;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / gpb, gi = t - b * gpb;
        const int64_t br = blk_br[b], bc = blk_bc[b];
        const int64_t left = rows - br * R;
        const int64_t n_block = left < R ? left : R;
        if (gi * W >= n_block) continue;
        const int n = (int)((n_block - gi * W) < W ? (n_block - gi * W) : W);
        const int64_t g = bc * gpc + br * gpb + gi;
        double x[32];
        int64_t sum = 0;
        int32_t mx = 0;
        for (int q = 0; q < n; ++q) {
            const int64_t slot = gi * W + q;
            const int64_t row = perm ? (int64_t)perm[b * R + slot] : slot;
            const int32_t c = len_local[b * R + row];
            lanes[g * W + q] = c;
            x[q] = (double)c;
            sum += c;
            mx = c > mx ? c : mx;
        }
        const double m = __ddiv_rn(np_pairwise_small(x, n), (double)n);
        for (int q = 0; q < n; ++q) {
            const double d = __dadd_rn(x[q], -m);
            x[q] = __dmul_rn(d, d);
        }
        mean[g] = m;
        stdv[g] = __dsqrt_rn(__ddiv_rn(np_pairwise_small(x, n), (double)n));
        maxv[g] = mx;
        util[g] = mx > 0 ? __ddiv_rn((double)sum, (double)(W * (int64_t)mx)) : 1.0;
    }
}

}  // namespace

extern "C" int hbp_group_stats(const int32_t *blk_br, const int32_t *blk_bc, int64_t nzb,
                               const int32_t *len_local, const uint32_t *perm, int64_t rows,
                               int64_t row_height, int64_t warp_size, int64_t groups_per_col,
                               int32_t *lanes, double *mean, double *std_dev, int32_t *max_nnz,
                               double *utilization, hbp_stream_t stream) {
    if (nzb < 0 || rows < 0 || row_height < 1 || warp_size < 1 || warp_size > 32 ||
        row_height % warp_size)
        return HBP_E_ARG;
    if (nzb == 0) return HBP_OK;
    if (!blk_br || !blk_bc || !len_local || !lanes || !mean || !std_dev || !max_nnz ||
        !utilization)
        return HBP_E_ARG;
    const int64_t total = nzb * (row_height / warp_size);
    const int threads = 256;
    int64_t blocks = (total + threads - 1) / threads;
    if (blocks > 148 * 64) blocks = 148 * 64;
    k_group_stats<<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(
        blk_br, blk_bc, nzb, len_local, perm, rows, row_height, warp_size, groups_per_col, lanes,
        mean, std_dev, max_nnz, utilization);
    return (int)cudaGetLastError();
}
