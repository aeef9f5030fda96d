// hbp_util.cu -- status strings, device queries, CUB primitives and the
// COO -> CSR tail (formats.py:87-97 canonicalized, formats.py:243-258
// coo_to_csr).
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "hbp.h"
#include "hbp_common.cuh"

using namespace hbp;

namespace {

__global__ void k_coo_finish(const uint64_t *__restrict__ keys, const uint64_t *__restrict__ order,
                             const void *__restrict__ val_in, int64_t nnz, int64_t cols, int f64,
                             int32_t *__restrict__ col_idx, void *__restrict__ val_out,
                             int32_t *__restrict__ dup) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = keys[i];
        col_idx[i] = (int32_t)(k % (uint64_t)cols);
        if (f64) ((double *)val_out)[i] = ((const double *)val_in)[order[i]];
        else ((float *)val_out)[i] = ((const float *)val_in)[order[i]];
        if (i > 0 && keys[i - 1] == k) *dup = 1;
    }
}

// row_ptr[r] = #{keys < r * cols} for r in [0, rows]
__global__ void k_row_ptr(const uint64_t *__restrict__ keys, int64_t nnz, int64_t rows,
                          int64_t cols, int64_t *__restrict__ row_ptr) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        uint64_t v = (uint64_t)r * (uint64_t)cols;
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            int64_t m = (lo + hi) >> 1;
            if (keys[m] < v) lo = m + 1;
            else hi = m;
        }
        row_ptr[r] = lo;
    }
}

__global__ void k_run_heads(const uint64_t *__restrict__ keys, int64_t n, int64_t *__restrict__ h) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        h[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// numpy's pairwise summation (used by np.add.reduceat for each segment
// after the segment's first element): < 8 terms sequential from +0.0; up to
// 128 terms in 8 strided accumulators; above that split at n/2 rounded down
// to a multiple of 8.  Iterative with an explicit stack.
__device__ double np_pairwise(const double *__restrict__ v, const uint64_t *__restrict__ order,
                              int64_t start, int64_t n) {
    struct Frame {
        int64_t s, n;
        int state;
        double left;
    };
    Frame st[48];
    int sp = 0;
    st[0] = {start, n, 0, 0.0};
    double ret = 0.0;
    while (sp >= 0) {
        Frame &fr = st[sp];
        if (fr.n < 8) {
            double r = 0.0;  // numpy starts from 0. here
            for (int64_t i = 0; i < fr.n; ++i) r += v[order[fr.s + i]];
            ret = r;
            --sp;
        } else if (fr.n <= 128) {
            double r[8];
            for (int j = 0; j < 8; ++j) r[j] = v[order[fr.s + j]];
            int64_t i = 8;
            for (; i < fr.n - (fr.n % 8); i += 8)
                for (int j = 0; j < 8; ++j) r[j] += v[order[fr.s + i + j]];
            double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
            for (; i < fr.n; ++i) res += v[order[fr.s + i]];
            ret = res;
            --sp;
        } else {
            int64_t n2 = fr.n / 2;
            n2 -= n2 % 8;
            if (fr.state == 0) {
                fr.state = 1;
                st[++sp] = {fr.s, n2, 0, 0.0};
            } else if (fr.state == 1) {
                fr.left = ret;
                fr.state = 2;
                st[++sp] = {fr.s + n2, fr.n - n2, 0, 0.0};
            } else {
                ret = fr.left + ret;
                --sp;
            }
        }
    }
    return ret;
}

__global__ void k_reduce_runs(const uint64_t *__restrict__ keys, const uint64_t *__restrict__ order,
                              const double *__restrict__ val, const int64_t *__restrict__ incl,
                              int64_t n, int64_t cols, int64_t *__restrict__ row_out,
                              int64_t *__restrict__ col_out, double *__restrict__ val_out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i > 0 && keys[i] == keys[i - 1]) continue;
        int64_t e = i + 1;
        while (e < n && keys[e] == keys[i]) ++e;
        double s = val[order[i]];
        if (e - i > 1) s = s + np_pairwise(val, order, i + 1, e - i - 1);
        int64_t o = incl[i] - 1;
        row_out[o] = (int64_t)(keys[i] / (uint64_t)cols);
        col_out[o] = (int64_t)(keys[i] % (uint64_t)cols);
        val_out[o] = s;
    }
}

}  // namespace

extern "C" {

const char *hbp_status_string(int status) {
    switch (status) {
        case HBP_OK: return "ok";
        case HBP_E_ARG: return "invalid argument";
        case HBP_E_PERM: return "permutation is not a bijection";
        case HBP_E_DUP: return "duplicate (row, col) entries; canonicalize first";
        case HBP_E_UNSUPPORTED: return "geometry not supported by the GPU kernels";
        case HBP_E_FORMAT: return "structurally invalid HBP arrays";
        default: return cudaGetErrorString((cudaError_t)status);
    }
}

int hbp_abi_version(void) { return 3; }

int hbp_struct_sizes(int64_t *sizes) {
    if (!sizes) return HBP_E_ARG;
    sizes[0] = (int64_t)sizeof(hbp_format_t);
    sizes[1] = (int64_t)sizeof(hbp_schedule_t);
    sizes[2] = (int64_t)sizeof(hbp_balanced_t);
    sizes[3] = (int64_t)sizeof(hbp_seg_t);
    return HBP_OK;
}

int hbp_last_error(void) { return (int)cudaGetLastError(); }

int hbp_device_sm_count(int *sms) {
    int dev = 0;
    HBP_CUDA_TRY(cudaGetDevice(&dev));
    HBP_CUDA_TRY(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev));
    return HBP_OK;
}

int hbp_exclusive_sum_i64(const int64_t *in, int64_t *out, int64_t n, void *temp,
                          size_t *temp_bytes, hbp_stream_t stream) {
    HBP_CUDA_TRY(cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, in, out, n, as_stream(stream)));
    return HBP_OK;
}

int hbp_inclusive_sum_i64(const int64_t *in, int64_t *out, int64_t n, void *temp,
                          size_t *temp_bytes, hbp_stream_t stream) {
    HBP_CUDA_TRY(cub::DeviceScan::InclusiveSum(temp, *temp_bytes, in, out, n, as_stream(stream)));
    return HBP_OK;
}

int hbp_sort_pairs_u32(const uint32_t *keys_in, uint32_t *keys_out, const uint32_t *vals_in,
                       uint32_t *vals_out, int64_t n, int end_bit, void *temp,
                       size_t *temp_bytes, hbp_stream_t stream) {
    if (end_bit < 1) end_bit = 1;
    HBP_CUDA_TRY(cub::DeviceRadixSort::SortPairs(temp, *temp_bytes, keys_in, keys_out, vals_in,
                                                 vals_out, n, 0, end_bit, as_stream(stream)));
    return HBP_OK;
}

int hbp_sort_pairs_u64(const uint64_t *keys_in, uint64_t *keys_out, const uint64_t *vals_in,
                       uint64_t *vals_out, int64_t n, int end_bit, void *temp,
                       size_t *temp_bytes, hbp_stream_t stream) {
    if (end_bit < 1) end_bit = 1;
    HBP_CUDA_TRY(cub::DeviceRadixSort::SortPairs(temp, *temp_bytes, keys_in, keys_out, vals_in,
                                                 vals_out, n, 0, end_bit, as_stream(stream)));
    return HBP_OK;
}

int hbp_coo_finish_csr(const uint64_t *sorted_keys, const uint64_t *order, const void *val_in,
                       int64_t nnz, int64_t rows, int64_t cols, int dtype, int64_t *row_ptr,
                       int32_t *col_idx, void *val_out, int32_t *dup_flag, hbp_stream_t stream) {
    if (rows < 0 || cols < 1) return HBP_E_ARG;
    cudaStream_t s = as_stream(stream);
    if (nnz > 0) {
        k_coo_finish<<<grid_for(nnz, 256), 256, 0, s>>>(sorted_keys, order, val_in, nnz, cols,
                                                         dtype == HBP_F64, col_idx, val_out,
                                                         dup_flag);
        HBP_LAUNCH_CHECK();
    }
    k_row_ptr<<<grid_for(rows + 1, 256), 256, 0, s>>>(sorted_keys, nnz, rows, cols, row_ptr);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_coo_run_heads(const uint64_t *sorted_keys, int64_t n, int64_t *head, hbp_stream_t stream) {
    if (n <= 0) return HBP_OK;
    k_run_heads<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(sorted_keys, n, head);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_coo_reduce_runs(const uint64_t *sorted_keys, const uint64_t *order, const double *val_in,
                        const int64_t *head_incl, int64_t n, int64_t cols, int64_t *row_out,
                        int64_t *col_out, double *val_out, hbp_stream_t stream) {
    if (n <= 0) return HBP_OK;
    k_reduce_runs<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(
        sorted_keys, order, val_in, head_incl, n, cols, row_out, col_out, val_out);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

}  // extern "C"

extern "C" {

// Keep `bytes` at `base` (the gathered x vector) resident in L2: set aside
// persisting L2 and attach an access-policy window to `stream`.
int hbp_l2_persist(const void *base, size_t bytes, float hit_ratio, hbp_stream_t stream) {
    int dev = 0, max_persist = 0, max_window = 0;
    HBP_CUDA_TRY(cudaGetDevice(&dev));
    HBP_CUDA_TRY(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
    HBP_CUDA_TRY(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev));
    if (max_persist <= 0 || max_window <= 0) return HBP_E_UNSUPPORTED;
    size_t set_aside = bytes < (size_t)max_persist ? bytes : (size_t)max_persist;
    HBP_CUDA_TRY(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, set_aside));
    cudaStreamAttrValue v = {};
    v.accessPolicyWindow.base_ptr = const_cast<void *>(base);
    v.accessPolicyWindow.num_bytes = bytes < (size_t)max_window ? bytes : (size_t)max_window;
    float hr = (float)set_aside / (float)(v.accessPolicyWindow.num_bytes ? v.accessPolicyWindow.num_bytes : 1);
    v.accessPolicyWindow.hitRatio = hit_ratio < hr ? hit_ratio : hr;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    HBP_CUDA_TRY(cudaStreamSetAttribute(as_stream(stream), cudaStreamAttributeAccessPolicyWindow, &v));
    return HBP_OK;
}

int hbp_l2_persist_reset(hbp_stream_t stream) {
    cudaStreamAttrValue v = {};
    v.accessPolicyWindow.num_bytes = 0;
    HBP_CUDA_TRY(cudaStreamSetAttribute(as_stream(stream), cudaStreamAttributeAccessPolicyWindow, &v));
    HBP_CUDA_TRY(cudaCtxResetPersistingL2Cache());
    return HBP_OK;
}

int hbp_l2_info(int *l2_bytes, int *max_persist, int *max_window) {
    int dev = 0;
    HBP_CUDA_TRY(cudaGetDevice(&dev));
    HBP_CUDA_TRY(cudaDeviceGetAttribute(l2_bytes, cudaDevAttrL2CacheSize, dev));
    HBP_CUDA_TRY(cudaDeviceGetAttribute(max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
    HBP_CUDA_TRY(cudaDeviceGetAttribute(max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev));
    return HBP_OK;
}

}  // extern "C"
