// hbp_reorder.cu -- per-block row orderings on the GPU (sm_100a).
//
//   hash_permutations  reorder.py:174-184 -> _kernels.py:62-92 hash_perm_kernel
//   sort_permutations  reorder.py:187-219 (stable ascending nnz, the sort2D baseline)
//   sort_permutation(counter=...) reorder.py:139-171 (merge-sort comparison count)
//
// The hash is FCFS linear probing: rows claim slots in ascending local-row
// order, each at the first free slot at or after its preliminary slot,
// cyclically (the slot the reference's +1 probe loop reaches); its probe count
// is the cyclic distance (slot - preliminary) mod n.  The claim chain is
// sequential by definition.  Two forms: with few blocks (fewer than a wave of
// warps) one WARP per block keeps the chain short -- the block's occupancy
// bitmap in the warp's registers (word w in lane w, R <= 1024), the
// preliminary slots of 32 rows computed in parallel and broadcast by shuffle,
// each claim one ballot over the lanes' masked free words, claimed slots to
// a per-warp shared table and out as coalesced stores; with many blocks one
// THREAD per block (shared-memory bitmap), 32 chains per warp instruction.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "hbp.h"
#include "hbp_common.cuh"

using namespace hbp;

namespace {

__device__ __forceinline__ int64_t rows_in_block(int64_t rows, int64_t R, int64_t br) {
    int64_t n = rows - br * R;
    return n < R ? n : R;
}

// hash_slot (reorder.py:106-109) reduced modulo the block's row count.
__device__ __forceinline__ uint32_t prelim_slot(uint32_t len, int64_t r, int64_t n, int64_t a,
                                                int64_t b, int64_t c, int64_t d, int64_t bmax,
                                                bool small) {
    int64_t g = a >= 32 ? 0 : (int64_t)(len >> a);
    if (g > bmax) g = bmax;
    if (small) {  // every intermediate below 2^32 (checked on the host)
        uint32_t h = (uint32_t)g * (uint32_t)b + ((uint32_t)r * (uint32_t)c) % (uint32_t)d;
        return h % (uint32_t)n;
    }
    return (uint32_t)((g * b + (r * c) % d) % n);
}

// ------------------------------------- hash: a lane group (L lanes) per block
// L = 8, 16 or 32 lanes own one block (32/L blocks per warp, in lockstep);
// lane l of a group owns bitmap word l (slots 32l .. 32l+31, R <= 32L); words
// past the block's rows are all-taken.  For a row with preliminary slot p
// (word w, bit q):
//   m_l = free bits of lane l at or after p (l == w: bits >= q; l > w: all;
//         l < w: none); the winner is the group's lowest lane with m_l != 0,
//         else (wraparound) its lowest lane with any free bit.
// The winner sets its bit and records slot -> row in shared memory.
template <bool EMPTY, int L>
__global__ void __launch_bounds__(128)
k_hash_perm_warp(const uint32_t *__restrict__ len_local, const int32_t *__restrict__ blk_br,
                 int64_t nzb, int64_t rows, int64_t R, int64_t a, int64_t b, int64_t c, int64_t d,
                 int64_t bmax, int small, uint32_t *__restrict__ perm,
                 unsigned long long *__restrict__ probes) {
    constexpr int S = 32 / L;  // blocks per warp
    constexpr unsigned GMASK = L == 32 ? 0xffffffffu : ((1u << L) - 1u);
    extern __shared__ uint16_t slot_row[];  // [warps * S][R]
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int sub = lane / L, sl = lane - sub * L, shift = sub * L;
    uint16_t *tab = slot_row + ((int64_t)wid * S + sub) * R;
    const int64_t blk = ((int64_t)blockIdx.x * (blockDim.x >> 5) + wid) * S + sub;
    const bool have = blk < nzb;
    unsigned long long my_probes = 0;
    const int64_t n = !have ? 0 : EMPTY ? rows : rows_in_block(rows, R, blk_br[blk]);
    const int nn = (int)n;
    uint32_t word;
    if (sl * 32 >= nn) word = FULL;
    else if (sl * 32 + 32 > nn) word = ~((1u << (nn & 31)) - 1u);
    else word = 0u;
    const uint32_t *lens = (EMPTY || !have) ? nullptr : len_local + blk * R;
    const int nmax = __reduce_max_sync(FULL, (unsigned)nn);
    uint32_t next_len = (!EMPTY && sl < nn) ? __ldg(lens + sl) : 0u;
    for (int base = 0; base < nmax; base += L) {
        const int r = base + sl;
        const uint32_t len = next_len;
        if (!EMPTY && r + L < nn) next_len = __ldg(lens + r + L);
        const uint32_t pre = r < nn ? prelim_slot(len, r, n, a, b, c, d, bmax, small) : 0u;
#pragma unroll 4
        for (int j = 0; j < L; ++j) {
            const bool valid = base + j < nn;
            const uint32_t home = __shfl_sync(FULL, pre, shift + j);
            const int w = (int)(home >> 5);
            const uint32_t fr = ~word;
            uint32_t m = !valid ? 0u : sl == w ? fr & (FULL << (home & 31)) : (sl > w ? fr : 0u);
            uint32_t bal = (__ballot_sync(FULL, m != 0u) >> shift) & GMASK;
            const bool wrap = valid && bal == 0u;  // first free slot from slot 0
            if (__any_sync(FULL, wrap)) {
                const uint32_t b2 = (__ballot_sync(FULL, fr != 0u) >> shift) & GMASK;
                if (wrap) {
                    m = fr;
                    bal = b2;
                }
            }
            if (valid && sl == __ffs(bal) - 1) {
                const int bit = __ffs(m) - 1;
                word |= 1u << bit;
                const uint32_t slot = (uint32_t)(sl * 32 + bit);
                tab[slot] = (uint16_t)(base + j);
                my_probes += slot >= home ? slot - home : slot + (uint32_t)nn - home;
            }
        }
    }
    __syncwarp();
    if (have) {
        uint32_t *out = perm + blk * R;
        for (int s2 = sl; s2 < (int)R; s2 += L) {
            if (s2 < nn) out[s2] = tab[s2];
            else if (!EMPTY) out[s2] = 0u;
        }
    }
    if (probes) {
        for (int o = 16; o; o >>= 1) my_probes += __shfl_xor_sync(FULL, my_probes, o);
        if (lane == 0 && my_probes) atomicAdd(probes, my_probes);
    }
}

// ------------------------------ hash: one thread per block (many blocks, R > 1024)
// The occupancy bitmap of thread t lives in shared memory, word w at
// [w * blockDim + t] (conflict-free); find-next-free scans words.
template <bool EMPTY>
__global__ void k_hash_perm_thread(const uint32_t *__restrict__ len_local,
                                   const int32_t *__restrict__ blk_br, int64_t nzb, int64_t rows,
                                   int64_t R, int64_t a, int64_t b, int64_t c, int64_t d,
                                   int64_t bmax, int small, uint32_t *__restrict__ perm,
                                   unsigned long long *__restrict__ probes) {
    extern __shared__ uint32_t bm[];
    const int T = blockDim.x, t = threadIdx.x;
    int64_t blk = (int64_t)blockIdx.x * T + t;
    unsigned long long my_probes = 0;
    if (blk < nzb) {
        int64_t n = EMPTY ? rows : rows_in_block(rows, R, blk_br[blk]);
        int nw = (int)((n + 31) >> 5);
        for (int w = 0; w < nw; ++w) bm[w * T + t] = 0u;
        if (n & 31) bm[(nw - 1) * T + t] = ~((1u << (n & 31)) - 1u);  // bits >= n: taken
        const uint32_t *lens = len_local + blk * R;
        uint32_t *out = perm + blk * R;
        for (int64_t r = 0; r < n; ++r) {
            uint32_t len = EMPTY ? 0u : lens[r];
            int64_t pos = prelim_slot(len, r, n, a, b, c, d, bmax, small);
            int w = (int)(pos >> 5);
            uint32_t word = bm[w * T + t];
            uint32_t fr = ~word & (0xffffffffu << (pos & 31));
            while (!fr) {
                w = (w + 1 == nw) ? 0 : w + 1;
                word = bm[w * T + t];
                fr = ~word;
            }
            int bit = __ffs(fr) - 1;
            bm[w * T + t] = word | (1u << bit);
            int64_t slot = (int64_t)w * 32 + bit;
            out[slot] = (uint32_t)r;
            my_probes += (unsigned long long)(slot >= pos ? slot - pos : slot + n - pos);
        }
        if (n < R)
            for (int64_t s = n; s < R && !EMPTY; ++s) out[s] = 0u;
    }
    if (probes) {
        for (int o = 16; o; o >>= 1) my_probes += __shfl_xor_sync(0xffffffffu, my_probes, o);
        if ((t & 31) == 0 && my_probes) atomicAdd(probes, my_probes);
    }
}

// ------------------------------------------------- sort2D: block radix sort
// reorder.py:160-171 sort_permutation = np.argsort(nnz, kind="stable"): one
// CTA per nonzero block, keys = slot lengths in blocked (row) order, values =
// local rows; CUB's block radix sort is stable, so ties keep ascending row.
// Rows past the block's height get key max+1 and sort after every real row;
// only the bits up to max+1 are sorted.
constexpr int kSortThreads = 128;

struct MaxOp {
    __device__ __forceinline__ uint32_t operator()(uint32_t x, uint32_t y) const {
        return x > y ? x : y;
    }
};

template <int ITEMS>
__global__ void __launch_bounds__(kSortThreads)
k_sort_perm_radix(const uint32_t *__restrict__ len_local, const int32_t *__restrict__ blk_br,
                  int64_t rows, int64_t R, uint32_t *__restrict__ perm) {
    using Sort = cub::BlockRadixSort<uint32_t, kSortThreads, ITEMS, uint32_t>;
    using Reduce = cub::BlockReduce<uint32_t, kSortThreads>;
    __shared__ union {
        typename Sort::TempStorage sort;
        typename Reduce::TempStorage reduce;
    } tmp;
    __shared__ uint32_t s_top;
    const int64_t blk = blockIdx.x;
    const int n = (int)rows_in_block(rows, R, blk_br[blk]);
    const uint32_t *lens = len_local + blk * R;
    uint32_t key[ITEMS], val[ITEMS], mx = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int r = threadIdx.x * ITEMS + k;
        val[k] = (uint32_t)r;
        key[k] = r < n ? lens[r] : 0u;
        mx = key[k] > mx ? key[k] : mx;
    }
    mx = Reduce(tmp.reduce).Reduce(mx, MaxOp());
    if (threadIdx.x == 0) s_top = mx;
    __syncthreads();
    const uint32_t pad = s_top + 1u;  // lengths are < 2^31 (CSR counts)
#pragma unroll
    for (int k = 0; k < ITEMS; ++k)
        if ((int)(threadIdx.x * ITEMS + k) >= n) key[k] = pad;
    const int end_bit = 32 - __clz(pad);
    Sort(tmp.sort).SortBlockedToStriped(key, val, 0, end_bit);
    uint32_t *out = perm + blk * R;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int i = k * kSortThreads + threadIdx.x;
        if (i < (int)R) out[i] = i < n ? val[k] : 0u;
    }
}

// R > 2048: warp per block, rank(r) = #{r' : len[r'] < len[r]} + #{r' < r : len[r'] == len[r]}.
__global__ void k_sort_perm_rank(const uint32_t *__restrict__ len_local,
                                 const int32_t *__restrict__ blk_br, int64_t nzb, int64_t rows,
                                 int64_t R, uint32_t *__restrict__ perm) {
    int lane = threadIdx.x & 31;
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t blk = warp; blk < nzb; blk += nwarps) {
        int64_t n = rows_in_block(rows, R, blk_br[blk]);
        const uint32_t *lens = len_local + blk * R;
        for (int64_t r = lane; r < n; r += 32) {
            uint32_t lr = lens[r];
            int64_t rank = 0;
            for (int64_t o = 0; o < n; ++o) {
                uint32_t lo = lens[o];
                rank += (lo < lr) || (lo == lr && o < r);
            }
            perm[blk * R + rank] = (uint32_t)r;
        }
        for (int64_t s = n + lane; s < R; s += 32) perm[blk * R + s] = 0u;
    }
}

// ------------------------------------- merge-sort comparison count (one list)
// reorder.py:139-157 _counting_merge_sort splits idx at len//2 and merges
// with `key[left] <= key[right]`, one comparison per emitted element until a
// side runs out.  For a node with sorted halves L, Rt (maxima Lm, Rm): if
// Lm <= Rm the left side runs out first, leaving the right elements with key
// >= Lm unmerged; otherwise the right runs out, leaving left keys > Rm.  So
// comparisons(node) = |L| + |Rt| - leftover, with no sorting needed: node j
// of depth t is found by descending from [0, n) along j's bits.
__global__ void k_merge_comparisons(const int64_t *__restrict__ key, int64_t n,
                                    unsigned long long *__restrict__ out) {
    unsigned long long acc = 0;
    for (int depth = 0; depth < 63 && (1LL << depth) < 2 * n; ++depth) {
        const int64_t nodes = 1LL << depth;
        for (int64_t j = threadIdx.x; j < nodes; j += blockDim.x) {
            int64_t lo = 0, hi = n;
            bool ok = true;
            for (int bit = depth - 1; bit >= 0; --bit) {
                if (hi - lo <= 1) { ok = false; break; }
                const int64_t mid = lo + (hi - lo) / 2;
                if ((j >> bit) & 1) lo = mid;
                else hi = mid;
            }
            if (!ok || hi - lo <= 1) continue;
            const int64_t mid = lo + (hi - lo) / 2;
            int64_t lm = key[lo], rm = key[mid];
            for (int64_t i = lo + 1; i < mid; ++i) lm = key[i] > lm ? key[i] : lm;
            for (int64_t i = mid + 1; i < hi; ++i) rm = key[i] > rm ? key[i] : rm;
            int64_t left_over = 0;
            if (lm <= rm) {
                for (int64_t i = mid; i < hi; ++i) left_over += key[i] >= lm;
            } else {
                for (int64_t i = lo; i < mid; ++i) left_over += key[i] > rm;
            }
            acc += (unsigned long long)(hi - lo - left_over);
        }
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

bool small_hash_math(int64_t R, int64_t b, int64_t c, int64_t d, int64_t bmax) {
    const int64_t lim = 0xffffffffLL;
    return b <= lim && c <= lim && d <= lim && bmax <= lim && (R - 1) * c <= lim &&
           bmax * b + d <= lim;
}

int hash_launch(const uint32_t *len_local, const int32_t *blk_br, int64_t nzb, int64_t rows,
                int64_t R, int64_t a, int64_t b, int64_t c, int64_t d, int64_t bmax,
                uint32_t *perm, unsigned long long *probes, bool empty, cudaStream_t s) {
    const int small = small_hash_math(R, b, c, d, bmax) ? 1 : 0;
    // The claim chain is serial per block either way.  A lane group per block
    // (8-32 lanes, 1-4 blocks per warp) keeps it in registers but leaves most
    // lanes idle on it, so it only wins while the blocks alone cannot fill the
    // GPU (cfg1, 3,068 blocks: 0.105 vs 0.28 ms); beyond that a thread per
    // block runs 32 chains per warp instruction (cfg2 0.36 vs 0.59 ms, cfg3
    // 0.51 vs 1.42 ms; ncu).  A thread-per-block form with its slot table in shared
    // memory and coalesced table stores was slower still (cfg3 1.12 ms: the
    // tables cap it at 6 CTAs of 32 threads per SM).  HBP_HASH_THREAD=0/1
    // forces the warp / thread form (A/B).
    int64_t wave = 148 * 64;
    {
        int dev = 0, sms = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
            wave = (int64_t)sms * 64;
    }
    const char *force = getenv("HBP_HASH_THREAD");
    // lane-group form up to ~3/4 of a wave of its groups (H, 12,208 blocks of
    // R = 512: 0.259 vs 0.308 ms; cfg4, 16,384: 0.320 vs 0.302)
    const int64_t lanes = R <= 256 ? 8 : R <= 512 ? 16 : 32;
    const int form = force ? atoi(force) : (nzb * lanes * 4 <= wave * 32 * 3 ? 0 : 1);
    if (R <= 1024 && form == 0) {
        // lanes per block: the fewest (>= 8) whose bitmap words cover R slots
        const int L = R <= 256 ? 8 : R <= 512 ? 16 : 32;
        const int warps = 4, per_cta = warps * (32 / L);
        const unsigned grid = (unsigned)((nzb + per_cta - 1) / per_cta);
        const size_t smem = (size_t)per_cta * R * sizeof(uint16_t);
#define HBP_HASH_WARP(LL)                                                                     \
    do {                                                                                      \
        if (empty)                                                                            \
            k_hash_perm_warp<true, LL><<<grid, warps * 32, smem, s>>>(                        \
                nullptr, nullptr, nzb, rows, R, a, b, c, d, bmax, small, perm, probes);       \
        else                                                                                  \
            k_hash_perm_warp<false, LL><<<grid, warps * 32, smem, s>>>(                       \
                len_local, blk_br, nzb, rows, R, a, b, c, d, bmax, small, perm, probes);      \
    } while (0)
        if (L == 8) HBP_HASH_WARP(8);
        else if (L == 16) HBP_HASH_WARP(16);
        else HBP_HASH_WARP(32);
#undef HBP_HASH_WARP
        HBP_LAUNCH_CHECK();
        return HBP_OK;
    }
    const int64_t nw = (R + 31) / 32;
    int64_t t = 64;
    while (t > 1 && nw * 4 * t > 48 * 1024) t >>= 1;
    if (nw * 4 * t > 48 * 1024) return HBP_E_UNSUPPORTED;
    const unsigned grid = (unsigned)((nzb + t - 1) / t);
    const size_t smem = (size_t)(nw * 4 * t);
    if (empty)
        k_hash_perm_thread<true><<<grid, (int)t, smem, s>>>(
            nullptr, nullptr, nzb, rows, R, a, b, c, d, bmax, small, perm, probes);
    else
        k_hash_perm_thread<false><<<grid, (int)t, smem, s>>>(
            len_local, blk_br, nzb, rows, R, a, b, c, d, bmax, small, perm, probes);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

}  // namespace

extern "C" {

int hbp_hash_perm(const uint32_t *len_local, const int32_t *blk_br, int64_t nzb, int64_t rows,
                  int64_t row_height, int64_t a, int64_t b, int64_t c, int64_t d,
                  int64_t bucket_max, uint32_t *perm, unsigned long long *probes,
                  hbp_stream_t stream) {
    if (b < 1 || d < 1 || a < 0 || row_height < 1) return HBP_E_ARG;
    if (nzb <= 0) return HBP_OK;
    return hash_launch(len_local, blk_br, nzb, rows, row_height, a, b, c, d, bucket_max, perm,
                       probes, false, as_stream(stream));
}

int hbp_hash_perm_empty(int64_t n, int64_t a, int64_t b, int64_t c, int64_t d,
                        int64_t bucket_max, uint32_t *perm, hbp_stream_t stream) {
    if (n < 1 || b < 1 || d < 1 || a < 0) return HBP_E_ARG;
    // one block; `rows` carries n, R = n
    return hash_launch(nullptr, nullptr, 1, n, n, a, b, c, d, bucket_max, perm, nullptr, true,
                       as_stream(stream));
}

int hbp_sort_perm(const uint32_t *len_local, const int32_t *blk_br, int64_t nzb, int64_t rows,
                  int64_t row_height, uint32_t *perm, hbp_stream_t stream) {
    if (row_height < 1) return HBP_E_ARG;
    if (nzb <= 0) return HBP_OK;
    cudaStream_t s = as_stream(stream);
    const int64_t R = row_height;
    const unsigned grid = (unsigned)nzb;
    if (nzb > 0x7fffffffLL) return HBP_E_UNSUPPORTED;
    if (R <= kSortThreads) k_sort_perm_radix<1><<<grid, kSortThreads, 0, s>>>(len_local, blk_br, rows, R, perm);
    else if (R <= 2 * kSortThreads) k_sort_perm_radix<2><<<grid, kSortThreads, 0, s>>>(len_local, blk_br, rows, R, perm);
    else if (R <= 4 * kSortThreads) k_sort_perm_radix<4><<<grid, kSortThreads, 0, s>>>(len_local, blk_br, rows, R, perm);
    else if (R <= 8 * kSortThreads) k_sort_perm_radix<8><<<grid, kSortThreads, 0, s>>>(len_local, blk_br, rows, R, perm);
    else if (R <= 16 * kSortThreads) k_sort_perm_radix<16><<<grid, kSortThreads, 0, s>>>(len_local, blk_br, rows, R, perm);
    else
        k_sort_perm_rank<<<grid_for(nzb * 32, 256), 256, 0, s>>>(len_local, blk_br, nzb, rows, R,
                                                                 perm);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

int hbp_merge_comparisons(const int64_t *keys, int64_t n, unsigned long long *out,
                          hbp_stream_t stream) {
    if (n < 0) return HBP_E_ARG;
    if (n < 2) return HBP_OK;
    k_merge_comparisons<<<1, 1024, 0, as_stream(stream)>>>(keys, n, out);
    HBP_LAUNCH_CHECK();
    return HBP_OK;
}

}  // extern "C"
