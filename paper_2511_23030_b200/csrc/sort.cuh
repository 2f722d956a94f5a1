// Hand-written stable LSD radix sort and exclusive scan for sm_100a.
//
// Used by K3 (tile binning): a global stable depth order of the visible
// Gaussians on their fp64 camera depth (replaces np.argsort(z, kind="stable"),
// renderloss.py:202) and the per-tile instance sort.  Counts may live in
// device memory (`n_dev`) so the whole render pipeline runs without a host
// round trip; grids are sized for the capacity and idle blocks exit early.
//
// One pass = upsweep (per-block digit histogram) -> per-digit scan over blocks
// -> downsweep (stable in-block ranking with __match_any_sync, then scatter).
#pragma once
#include "common.cuh"

namespace sm {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;   // 2048 keys per block
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kSortWarps = kSortThreads / 32;

__device__ __forceinline__ int64_t load_count(const uint32_t *n_dev, int64_t n_host) {
    return n_dev ? (int64_t)(*n_dev) : n_host;
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads)
radix_upsweep(const K *__restrict__ keys, const uint32_t *n_dev, int64_t n_host, int shift,
              int nbits, uint32_t *__restrict__ hist, int64_t hist_stride) {
    __shared__ uint32_t h[kRadix];
    const int64_t n = load_count(n_dev, n_host);
    const int64_t start = (int64_t)blockIdx.x * kSortTile;
    if (start >= n) return;
    for (int i = threadIdx.x; i < kRadix; i += kSortThreads) h[i] = 0;
    __syncthreads();
    const K mask = (K)((1u << nbits) - 1u);
    const int64_t end = min(n, start + (int64_t)kSortTile);
    for (int64_t i = start + threadIdx.x; i < end; i += kSortThreads) {
        uint32_t d = (uint32_t)((keys[i] >> shift) & mask);
        atomicAdd(&h[d], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += kSortThreads)
        hist[(int64_t)d * hist_stride + blockIdx.x] = h[d];
}

// One CTA per digit: exclusive scan of hist[d][0:nblocks] in place; total out.
__global__ void __launch_bounds__(1024)
radix_scan_digits(uint32_t *__restrict__ hist, int64_t hist_stride, const uint32_t *n_dev,
                  int64_t n_host, uint32_t *__restrict__ digit_total) {
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry;
    const int64_t n = load_count(n_dev, n_host);
    const int64_t nblocks = ceil_div(n, kSortTile);
    uint32_t *row = hist + (int64_t)blockIdx.x * hist_stride;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t base = 0; base < nblocks; base += blockDim.x) {
        int64_t i = base + threadIdx.x;
        uint32_t v = i < nblocks ? row[i] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t s = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;   // inclusive
        }
        __syncthreads();
        uint32_t excl = carry + (warp ? warp_sums[warp - 1] : 0u) + x - v;
        if (i < nblocks) row[i] = excl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) digit_total[blockIdx.x] = carry;
}

// Stable scatter.  Warp w owns the contiguous segment [w*512, w*512+512) of
// the block's tile; lane l's item j is element w*512 + j*32 + l, so the
// (warp, round, lane) order equals the element order.
template <typename K, bool HAS_VAL>
__global__ void __launch_bounds__(kSortThreads)
radix_downsweep(const K *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
                K *__restrict__ keys_out, uint32_t *__restrict__ vals_out,
                const uint32_t *n_dev, int64_t n_host, int shift, int nbits,
                const uint32_t *__restrict__ hist, int64_t hist_stride,
                const uint32_t *__restrict__ digit_total) {
    __shared__ uint32_t wcount[kSortWarps][kRadix];
    __shared__ uint32_t digit_base[kRadix];
    __shared__ uint32_t warp_tot[kSortWarps];
    const int64_t n = load_count(n_dev, n_host);
    const int64_t start = (int64_t)blockIdx.x * kSortTile;
    if (start >= n) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads) (&wcount[0][0])[i] = 0;
    // digit base = exclusive scan of digit totals (256 digits, one per thread)
    {
        uint32_t v = threadIdx.x < kRadix ? digit_total[threadIdx.x] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[warp] = x;
        __syncthreads();
        uint32_t off = 0;
        for (int w = 0; w < warp; w++) off += warp_tot[w];
        if (threadIdx.x < kRadix) digit_base[threadIdx.x] = off + x - v;
    }
    __syncthreads();
    const K mask = (K)((1u << nbits) - 1u);
    K key[kSortItems];
    uint32_t val[kSortItems];
    uint32_t local[kSortItems];
    uint32_t dig[kSortItems];
    const int64_t seg = start + (int64_t)warp * (32 * kSortItems);
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        int64_t i = seg + j * 32 + lane;
        bool ok = i < n;
        key[j] = ok ? keys_in[i] : (K)0;
        if (HAS_VAL) val[j] = ok ? vals_in[i] : 0u;
        dig[j] = ok ? (uint32_t)((key[j] >> shift) & mask) : 0xffffffffu;
    }
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        const uint32_t d = dig[j];
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const unsigned lt = peers & ((1u << lane) - 1u);
        uint32_t cnt = 0;
        if (d != 0xffffffffu) cnt = wcount[warp][d];
        __syncwarp();
        if (d != 0xffffffffu && lt == 0) wcount[warp][d] = cnt + __popc(peers);
        __syncwarp();
        local[j] = cnt + __popc(lt);
    }
    __syncthreads();
    // exclusive prefix across warps per digit
    for (int d = threadIdx.x; d < kRadix; d += kSortThreads) {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; w++) {
            uint32_t c = wcount[w][d];
            wcount[w][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSortItems; j++) {
        const uint32_t d = dig[j];
        if (d == 0xffffffffu) continue;
        const uint32_t pos = digit_base[d] + hist[(int64_t)d * hist_stride + blockIdx.x] +
                             wcount[warp][d] + local[j];
        keys_out[pos] = key[j];
        if (HAS_VAL) vals_out[pos] = val[j];
    }
}

struct SortScratch {
    uint32_t *hist;          // [kRadix][max_blocks]
    uint32_t *digit_total;   // [kRadix]
    int64_t max_blocks;
};

inline int64_t sort_scratch_bytes(int64_t max_n) {
    int64_t mb = ceil_div(max_n > 0 ? max_n : 1, kSortTile);
    return align_up((int64_t)kRadix * mb * 4, 256) + align_up(kRadix * 4, 256);
}

// Sorts keys (and optional u32 values) over bits [begin_bit, end_bit).
// Ping-pongs between (k0,v0) and (k1,v1); returns 0 if the result is in
// buffer 0, 1 if in buffer 1.
template <typename K, bool HAS_VAL>
int radix_sort(K *k0, uint32_t *v0, K *k1, uint32_t *v1, const uint32_t *n_dev, int64_t n_host,
               int64_t max_n, int begin_bit, int end_bit, const SortScratch &s,
               cudaStream_t st) {
    const int64_t grid = ceil_div(max_n > 0 ? max_n : 1, kSortTile);
    int cur = 0;
    for (int shift = begin_bit; shift < end_bit; shift += kRadixBits) {
        const int nbits = min(kRadixBits, end_bit - shift);
        K *ki = cur ? k1 : k0;
        K *ko = cur ? k0 : k1;
        uint32_t *vi = cur ? v1 : v0;
        uint32_t *vo = cur ? v0 : v1;
        radix_upsweep<K><<<(unsigned)grid, kSortThreads, 0, st>>>(ki, n_dev, n_host, shift, nbits,
                                                                  s.hist, s.max_blocks);
        radix_scan_digits<<<kRadix, 1024, 0, st>>>(s.hist, s.max_blocks, n_dev, n_host,
                                                    s.digit_total);
        radix_downsweep<K, HAS_VAL><<<(unsigned)grid, kSortThreads, 0, st>>>(
            ki, vi, ko, vo, n_dev, n_host, shift, nbits, s.hist, s.max_blocks, s.digit_total);
        cur ^= 1;
    }
    return cur;
}

// ------------------------------------------------------------ exclusive scan
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t block_incl_scan(uint32_t x, uint32_t *warp_sums,
                                                    uint32_t *block_total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t s = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_sums[lane] = s;
    }
    __syncthreads();
    uint32_t r = x + (warp ? warp_sums[warp - 1] : 0u);
    if (block_total) *block_total = warp_sums[(blockDim.x >> 5) - 1];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kScanThreads)
scan_reduce(const uint32_t *__restrict__ in, int64_t n, uint32_t *__restrict__ partial) {
    __shared__ uint32_t ws[32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        int64_t i = base + (int64_t)threadIdx.x * kScanItems + j;
        if (i < n) s += in[i];
    }
    uint32_t tot;
    block_incl_scan(s, ws, &tot);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// single CTA: exclusive scan of partial[0:nb], writes total to *total
__global__ void __launch_bounds__(kScanThreads)
scan_partials(uint32_t *__restrict__ partial, int64_t nb, uint32_t *__restrict__ total) {
    __shared__ uint32_t ws[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < nb; base += kScanThreads) {
        int64_t i = base + threadIdx.x;
        uint32_t v = i < nb ? partial[i] : 0u;
        uint32_t bt;
        uint32_t inc = block_incl_scan(v, ws, &bt);
        uint32_t c = carry;
        if (i < nb) partial[i] = c + inc - v;
        __syncthreads();
        if (threadIdx.x == 0) carry = c + bt;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kScanThreads)
scan_downsweep(const uint32_t *__restrict__ in, int64_t n, const uint32_t *__restrict__ partial,
               uint32_t *__restrict__ out) {
    __shared__ uint32_t ws[32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        int64_t i = base + (int64_t)threadIdx.x * kScanItems + j;
        v[j] = i < n ? in[i] : 0u;
        s += v[j];
    }
    uint32_t inc = block_incl_scan(s, ws, nullptr);
    uint32_t run = partial[blockIdx.x] + inc - s;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        int64_t i = base + (int64_t)threadIdx.x * kScanItems + j;
        if (i < n) out[i] = run;
        run += v[j];
    }
}

inline int64_t scan_scratch_bytes(int64_t max_n) {
    return align_up(ceil_div(max_n > 0 ? max_n : 1, kScanTile) * 4, 256);
}

// out = exclusive_scan(in[0:n]); *total = sum.  n is host-known.
inline void exclusive_scan(const uint32_t *in, uint32_t *out, int64_t n, uint32_t *partial,
                           uint32_t *total, cudaStream_t st) {
    const int64_t nb = ceil_div(n > 0 ? n : 1, kScanTile);
    scan_reduce<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, partial);
    scan_partials<<<1, kScanThreads, 0, st>>>(partial, nb, total);
    scan_downsweep<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, partial, out);
}

}  // namespace sm
