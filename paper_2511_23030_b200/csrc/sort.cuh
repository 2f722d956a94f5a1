// Hand-written stable LSD radix sort (onesweep) and exclusive scan, sm_100a.
//
// Used by K3 (tile binning): a global stable depth order of the visible
// Gaussians on their fp64 camera depth (replaces np.argsort(z, kind="stable"),
// renderloss.py:202) and the per-tile instance sort.  Counts may live in
// device memory (`n_dev`) so the render pipeline needs no host round trip and
// can be captured in a CUDA graph; grids are sized for the capacity and idle
// blocks exit immediately.
//
// Onesweep (decoupled look-back): one histogram kernel computes the global
// digit counts of every pass at once; then each pass is ONE kernel.  A block
// takes the next tile id from an atomic counter (so every earlier tile is
// already running), ranks its keys stably in shared memory, publishes its
// per-digit counts, then walks back over its predecessors' published counts
// / inclusive prefixes to get its global offsets, and scatters.
#pragma once
#include "common.cuh"

namespace sm {

constexpr int kSortThreads = 256;
// Keys per thread: 8 (2048-key tiles) for the depth sort's ~0.4M keys --
// enough tiles to fill 148 SMs -- and 16 (4096-key tiles, half the look-back
// chain) for the tile sort's ~2M keys (measured best for each).
constexpr int kSortItems = 8;
constexpr int kSortItemsWide = 16;
constexpr int kSortTile = kSortThreads * kSortItems;   // smallest tile: sizes the scratch
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kMaxPasses = 8;
constexpr uint32_t kFlagAgg = 1u << 30;      // tile aggregate published
constexpr uint32_t kFlagPre = 2u << 30;      // tile inclusive prefix published
constexpr uint32_t kValMask = (1u << 30) - 1;

__device__ __forceinline__ int64_t load_count(const uint32_t *n_dev, int64_t n_host) {
    return n_dev ? (int64_t)(*n_dev) : n_host;
}

// Producer-side histograms: a kernel that writes keys can count their digits
// in shared bins (block_hist_add) and flush them once per block
// (block_hist_flush), which saves onesweep_histogram's extra pass over the
// keys; the sort is then run with hist_ready = true after sort_reset.
__device__ __forceinline__ void block_hist_zero(uint32_t (*h)[256], int npass) {
    for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) (&h[0][0])[i] = 0u;
}

template <typename K>
__device__ __forceinline__ void block_hist_add(uint32_t (*h)[256], K key, int begin_bit, int end_bit) {
    for (int p = 0, shift = begin_bit; shift < end_bit; p++, shift += 8) {
        const int nb = min(8, end_bit - shift);
        atomicAdd(&h[p][(uint32_t)(key >> shift) & ((1u << nb) - 1u)], 1u);
    }
}

__device__ __forceinline__ void block_hist_flush(uint32_t (*h)[256], int npass, uint32_t *hist) {
    for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) {
        const uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

// Global digit histograms of all passes: hist[p][d], p = 0..npasses-1.
template <typename K>
__global__ void __launch_bounds__(kSortThreads)
onesweep_histogram(const K *__restrict__ keys, const uint32_t *n_dev, int64_t n_host, int begin_bit,
                   int end_bit, uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[kMaxPasses][kRadix];
    const int64_t n = load_count(n_dev, n_host);
    const int npass = (end_bit - begin_bit + kRadixBits - 1) / kRadixBits;
    for (int i = threadIdx.x; i < kMaxPasses * kRadix; i += kSortThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * kSortThreads + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kSortThreads) {
        const K k = keys[i];
        for (int p = 0; p < npass; p++) {
            const int shift = begin_bit + p * kRadixBits;
            const int nb = min(kRadixBits, end_bit - shift);
            atomicAdd(&h[p][(uint32_t)(k >> shift) & ((1u << nb) - 1u)], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npass * kRadix; i += kSortThreads) {
        const uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

__device__ __forceinline__ uint32_t ld_status(const uint32_t *p) {
    return *reinterpret_cast<const volatile uint32_t *>(p);
}
__device__ __forceinline__ void st_status(uint32_t *p, uint32_t v) {
    *reinterpret_cast<volatile uint32_t *>(p) = v;
}

// Shared-memory layout of one onesweep pass (dynamic: the 11-bit tile pass
// needs ~96 KB).
template <typename K, bool HAS_VAL, int ITEMS, int RB>
struct PassSmem {
    static constexpr int R = 1 << RB;
    static constexpr size_t o_wcount = 0;                                    // [warps][R]
    static constexpr size_t o_base = o_wcount + (size_t)kSortWarps * R * 4;  // [R]
    static constexpr size_t o_excl = o_base + (size_t)R * 4;                  // [R]
    static constexpr size_t o_wtot = o_excl + (size_t)R * 4;                  // [warps] + s_tile
    static constexpr size_t o_keys = (o_wtot + (kSortWarps + 1) * 4 + 15) / 16 * 16;
    static constexpr size_t o_vals = o_keys + (size_t)kSortThreads * ITEMS * sizeof(K);
    static constexpr size_t bytes = o_vals + (HAS_VAL ? (size_t)kSortThreads * ITEMS * 4 : 0);
};

// Block exclusive scan of one value per thread (256 threads).
__device__ __forceinline__ uint32_t sort_block_excl(uint32_t v, uint32_t *warp_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();   // warp_tot reuse
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    uint32_t off = 0;
    for (int w = 0; w < warp; w++) off += warp_tot[w];
    return off + x - v;
}

// One stable pass over digit bits [shift, shift + nbits), RB-bit digits
// (8: 256 bins, one per thread; 11: 2048 bins, eight per thread -- the tile
// sort of a <= 2048-tile image in a single pass).  ranges_out (nullable,
// RB = 11 tile sort): the block holding tile 0 writes each digit's
// [start, end) of the sorted output (= the per-tile instance ranges), (0, 0)
// for empty digits, for digits < n_ranges.
template <typename K, bool HAS_VAL, int ITEMS, int RB = kRadixBits>
__global__ void __launch_bounds__(kSortThreads)
onesweep_pass(const K *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
              K *__restrict__ keys_out, uint32_t *__restrict__ vals_out, const uint32_t *n_dev,
              int64_t n_host, int shift, int nbits, const uint32_t *__restrict__ hist_p,
              uint32_t *__restrict__ status_p, uint32_t *__restrict__ tile_ctr_p,
              uint32_t *__restrict__ ranges_out = nullptr, int n_ranges = 0) {
    using L = PassSmem<K, HAS_VAL, ITEMS, RB>;
    constexpr int R = L::R;
    constexpr int DPT = R / kSortThreads;   // digits per thread
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t(*wcount)[R] = reinterpret_cast<uint32_t(*)[R]>(smem + L::o_wcount);
    uint32_t *digit_base = reinterpret_cast<uint32_t *>(smem + L::o_base);
    uint32_t *tile_excl = reinterpret_cast<uint32_t *>(smem + L::o_excl);
    uint32_t *warp_tot = reinterpret_cast<uint32_t *>(smem + L::o_wtot);
    uint32_t &s_tile = warp_tot[kSortWarps];
    K *s_keys = reinterpret_cast<K *>(smem + L::o_keys);
    uint32_t *s_vals = reinterpret_cast<uint32_t *>(smem + L::o_vals);
    const int64_t n = load_count(n_dev, n_host);
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr_p, 1u);
    __syncthreads();
    // tiles are handed out in launch order: blocks past the live count (the
    // grid is sized for the capacity) leave before doing any work
    if ((int64_t)s_tile * (kSortThreads * ITEMS) >= n) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kSortWarps * R; i += kSortThreads) (&wcount[0][0])[i] = 0;
    const int d0 = threadIdx.x * DPT;   // this thread's digits d0 .. d0 + DPT - 1
    // global digit base = exclusive scan of this pass's histogram
    {
        uint32_t h[DPT], sum = 0;
#pragma unroll
        for (int j = 0; j < DPT; j++) h[j] = hist_p[d0 + j], sum += h[j];
        uint32_t run = sort_block_excl(sum, warp_tot);
#pragma unroll
        for (int j = 0; j < DPT; j++) {
            digit_base[d0 + j] = run;
            if (ranges_out && s_tile == 0 && d0 + j < n_ranges) {
                ranges_out[2 * (d0 + j)] = h[j] ? run : 0u;
                ranges_out[2 * (d0 + j) + 1] = h[j] ? run + h[j] : 0u;
            }
            run += h[j];
        }
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t start = (int64_t)tile * (kSortThreads * ITEMS);
    const K mask = (K)((1u << nbits) - 1u);
    K key[ITEMS];
    uint32_t val[ITEMS];
    uint32_t local[ITEMS];
    uint32_t dig[ITEMS];
    const int64_t seg = start + (int64_t)warp * (32 * ITEMS);
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
        const int64_t i = seg + j * 32 + lane;
        const bool ok = i < n;
        key[j] = ok ? keys_in[i] : (K)0;
        if (HAS_VAL) val[j] = ok ? vals_in[i] : 0u;
        dig[j] = ok ? (uint32_t)((key[j] >> shift) & mask) : 0xffffffffu;
    }
    // stable in-block ranking: warp w owns the contiguous segment w*32*ITEMS..,
    // item j of lane l is element w*32*ITEMS + j*32 + l, processed in (j, l) order
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
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
    // per digit: exclusive prefix across warps, tile aggregate, publish,
    // decoupled look-back over predecessor tiles, publish prefix
    uint32_t run[DPT];
#pragma unroll
    for (int j = 0; j < DPT; j++) {
        const int d = d0 + j;
        uint32_t r = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; w++) {
            const uint32_t c = wcount[w][d];
            wcount[w][d] = r;
            r += c;
        }
        run[j] = r;
    }
    uint32_t *my = status_p + (int64_t)tile * R + d0;
    if (tile == 0) {
#pragma unroll
        for (int j = 0; j < DPT; j++) st_status(my + j, kFlagPre | run[j]);
    } else {
#pragma unroll
        for (int j = 0; j < DPT; j++) st_status(my + j, kFlagAgg | run[j]);
        uint32_t excl[DPT];
        if (DPT == 1) {   // look back 8 predecessors per round trip (independent loads)
            uint32_t e = 0;
            bool found = false;
            for (int64_t t = (int64_t)tile - 1; t >= 0 && !found; t -= 8) {
                uint32_t sv[8];
#pragma unroll
                for (int k = 0; k < 8; k++) sv[k] = (t - k >= 0) ? ld_status(status_p + (t - k) * R + d0) : kFlagPre;
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    if (found || t - k < 0) continue;
                    uint32_t v = sv[k];
                    while ((v & (kFlagAgg | kFlagPre)) == 0) v = ld_status(status_p + (t - k) * R + d0);
                    e += v & kValMask;
                    found = (v & kFlagPre) != 0;
                }
            }
            excl[0] = e;
        } else {   // DPT digits walk back together, one predecessor per round trip
            unsigned todo = (1u << DPT) - 1u;
#pragma unroll
            for (int j = 0; j < DPT; j++) excl[j] = 0;
            for (int64_t t = (int64_t)tile - 1; t >= 0 && todo; t--) {
                const uint32_t *row = status_p + t * R + d0;
                uint32_t sv[DPT];
#pragma unroll
                for (int j = 0; j < DPT; j++) sv[j] = (todo >> j) & 1u ? ld_status(row + j) : 0u;
#pragma unroll
                for (int j = 0; j < DPT; j++) {
                    if (!((todo >> j) & 1u)) continue;
                    uint32_t v = sv[j];
                    while ((v & (kFlagAgg | kFlagPre)) == 0) v = ld_status(row + j);
                    excl[j] += v & kValMask;
                    if (v & kFlagPre) todo &= ~(1u << j);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < DPT; j++) {
            st_status(my + j, kFlagPre | (excl[j] + run[j]));
            digit_base[d0 + j] += excl[j];
        }
    }
    // tile-local exclusive prefix over digits (block scan of the runs)
    {
        uint32_t sum = 0;
#pragma unroll
        for (int j = 0; j < DPT; j++) sum += run[j];
        uint32_t r = sort_block_excl(sum, warp_tot);
#pragma unroll
        for (int j = 0; j < DPT; j++) {
            tile_excl[d0 + j] = r;
            r += run[j];
        }
    }
    __syncthreads();
    // stage the tile in shared memory in digit order, then write each digit's
    // run to consecutive global addresses (full-sector, coalesced stores)
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
        const uint32_t d = dig[j];
        if (d == 0xffffffffu) continue;
        const uint32_t lp = tile_excl[d] + wcount[warp][d] + local[j];
        s_keys[lp] = key[j];
        if (HAS_VAL) s_vals[lp] = val[j];
    }
    __syncthreads();
    const int cnt = (int)min64((kSortThreads * ITEMS), n - start);
    for (int i = threadIdx.x; i < cnt; i += kSortThreads) {
        const K k = s_keys[i];
        const uint32_t d = (uint32_t)((k >> shift) & mask);
        const uint32_t pos = digit_base[d] + (uint32_t)i - tile_excl[d];
        keys_out[pos] = k;
        if (HAS_VAL) vals_out[pos] = s_vals[i];
    }
}

// Opt-in to > 48 KB of dynamic shared memory, once per instantiation.
template <typename K, bool HAS_VAL, int ITEMS, int RB>
inline size_t pass_smem() {
    static bool done = false;
    const size_t bytes = PassSmem<K, HAS_VAL, ITEMS, RB>::bytes;
    if (!done) {
        cudaFuncSetAttribute(onesweep_pass<K, HAS_VAL, ITEMS, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)bytes);
        done = true;
    }
    return bytes;
}

struct SortScratch {
    uint32_t *hist;      // [kMaxPasses][kRadix]
    uint32_t *status;    // [kMaxPasses][max_tiles][kRadix]
    uint32_t *tile_ctr;  // [kMaxPasses]
    int64_t max_tiles;
};

inline int64_t sort_tiles(int64_t max_n) { return ceil_div(max_n > 0 ? max_n : 1, kSortTile); }

inline int64_t sort_scratch_bytes(int64_t max_n) {
    return align_up((int64_t)kMaxPasses * kRadix * 4, 256) +
           align_up((int64_t)kMaxPasses * sort_tiles(max_n) * kRadix * 4, 256) +
           align_up(kMaxPasses * 4, 256);
}

// Layout: tile counters | histograms | look-back status, contiguous so one
// memset clears what a sort uses.
inline SortScratch sort_scratch(void *base, int64_t max_n) {
    char *b = static_cast<char *>(base);
    SortScratch s;
    s.max_tiles = sort_tiles(max_n);
    s.tile_ctr = reinterpret_cast<uint32_t *>(b);
    b += align_up(kMaxPasses * 4, 256);
    s.hist = reinterpret_cast<uint32_t *>(b);
    b += align_up((int64_t)kMaxPasses * kRadix * 4, 256);
    s.status = reinterpret_cast<uint32_t *>(b);
    return s;
}


// Stable sort of keys (+ optional u32 values) over bits [begin_bit, end_bit).
// Ping-pongs (k0,v0) <-> (k1,v1); returns 0 if the result is in buffer 0.
// `max_n` bounds the count (grids, status rows); the live count is n_dev or n_host.
inline int radix_passes(int begin_bit, int end_bit) {
    return (int)ceil_div(end_bit - begin_bit, kRadixBits);
}

template <int ITEMS = kSortItems>
inline int64_t sort_tile_count(int64_t max_n) {
    return ceil_div(max_n > 0 ? max_n : 1, (int64_t)kSortThreads * ITEMS);
}

// Clears what one sort over bits [begin_bit, end_bit) uses: tile counters,
// histograms, its look-back status rows.
template <int ITEMS = kSortItems>
inline void sort_reset(const SortScratch &s, int64_t max_n, int begin_bit, int end_bit, cudaStream_t st) {
    const int npass = radix_passes(begin_bit, end_bit);
    const int64_t tiles = sort_tile_count<ITEMS>(max_n);
    cudaMemsetAsync(s.tile_ctr, 0,
                    (size_t)(reinterpret_cast<char *>(s.status + (int64_t)npass * tiles * kRadix) -
                             reinterpret_cast<char *>(s.tile_ctr)), st);
}

// hist_ready: the producer already filled the histograms after sort_reset.
template <typename K, bool HAS_VAL, int ITEMS = kSortItems>
int radix_sort(K *k0, uint32_t *v0, K *k1, uint32_t *v1, const uint32_t *n_dev, int64_t n_host,
               int64_t max_n, int begin_bit, int end_bit, const SortScratch &s, cudaStream_t st,
               bool hist_ready = false) {
    const int npass = radix_passes(begin_bit, end_bit);
    const int64_t tiles = sort_tile_count<ITEMS>(max_n);
    if (!hist_ready) {
        sort_reset<ITEMS>(s, max_n, begin_bit, end_bit, st);
        const unsigned hgrid = (unsigned)min64(tiles * 2, 148 * 8);
        onesweep_histogram<K><<<hgrid, kSortThreads, 0, st>>>(k0, n_dev, n_host, begin_bit, end_bit, s.hist);
    }
    int cur = 0;
    for (int p = 0; p < npass; p++) {
        const int shift = begin_bit + p * kRadixBits;
        const int nbits = min(kRadixBits, end_bit - shift);
        K *ki = cur ? k1 : k0;
        K *ko = cur ? k0 : k1;
        uint32_t *vi = cur ? v1 : v0;
        uint32_t *vo = cur ? v0 : v1;
        onesweep_pass<K, HAS_VAL, ITEMS, kRadixBits>
            <<<(unsigned)tiles, kSortThreads, pass_smem<K, HAS_VAL, ITEMS, kRadixBits>(), st>>>(
                ki, vi, ko, vo, n_dev, n_host, shift, nbits, s.hist + p * kRadix,
                s.status + (int64_t)p * tiles * kRadix, s.tile_ctr + p);
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

// single CTA: exclusive scan of partial[0:nb], writes total to *total; with
// cap >= 0 also *over = (total > cap) and *count = over ? 0 : total (the
// render's instance-capacity check, folded in to save a launch)
__global__ void __launch_bounds__(kScanThreads)
scan_partials(uint32_t *__restrict__ partial, int64_t nb, uint32_t *__restrict__ total, int64_t cap,
              uint32_t *__restrict__ over, uint32_t *__restrict__ count) {
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
    if (threadIdx.x == 0) {
        *total = carry;
        if (cap >= 0) {
            const bool of = (int64_t)carry > cap;
            *over = of ? 1u : 0u;
            *count = of ? 0u : carry;
        }
    }
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
                           uint32_t *total, cudaStream_t st, int64_t cap = -1, uint32_t *over = nullptr,
                           uint32_t *count = nullptr) {
    const int64_t nb = ceil_div(n > 0 ? n : 1, kScanTile);
    scan_reduce<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, partial);
    scan_partials<<<1, kScanThreads, 0, st>>>(partial, nb, total, cap, over, count);
    scan_downsweep<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, partial, out);
}

}  // namespace sm
