// K2 projection, K3 depth order + tile binning, K4 front-to-back compositing.
//
// Restates renderloss.render_arrays (renderloss.py:170-218) and the numba
// _composite kernel (renderloss.py:106-152) for sm_100a:
//   * projection in fp64 (it is HBM-bound: 64 B/Gaussian in, 104 B out), so
//     means, conics and the 3-sigma bboxes are the reference's own numbers;
//   * one global stable order of the visible Gaussians by z = np.argsort(z,
//     kind="stable") over the sorted-chunk-id concatenation: a 4-pass radix
//     sort on the fp32-rounded z (z >= near > 0, so the bits order like the
//     values), then runs of equal fp32 keys re-sorted on the fp64 bits;
//   * instances are emitted in depth-rank order and radix-sorted on the tile
//     bits only (stable), giving each 16x16 tile its Gaussians front to back;
//   * compositing in fp32 with the q > 9 decision taken in fp64 whenever the
//     fp32 q lies within a per-Gaussian error band of 9.
#include <cstdio>

#include "prof.cuh"
#include "render.cuh"
#include "sort.cuh"

constexpr bool Exact = true;   // render.cuh DM/DA/DS/DD: explicit rounding in K2

namespace sm {

// ---------------------------------------------------------------- layout
RenderLayout render_layout(const sm_render_dims &d) {
    RenderLayout L;
    const int64_t G = d.max_gaussians > 0 ? d.max_gaussians : 1;
    const int64_t I = d.max_instances > 0 ? d.max_instances : 1;
    L.tiles_x = (int)ceil_div(d.width, kTile);
    L.tiles_y = (int)ceil_div(d.height, kTile);
    L.n_tiles = (int64_t)L.tiles_x * L.tiles_y;
    const int64_t npx = (int64_t)d.width * d.height;
    int rb = 1;
    while ((1ll << rb) < G) rb++;
    int tb = 1;
    while ((1ll << tb) < L.n_tiles) tb++;
    L.rank_bits = rb;
    L.tile_bits = tb;
    L.key_bytes = rb + tb > 32 ? 8 : 4;
    L.depth_passes = ceil_div(32, kRadixBits);   // fp32 key + fp64 tie fixup
    L.tile_passes = (int)ceil_div(tb, kRadixBits);
    L.sort_blocks = ceil_div(G > I ? G : I, kSortTile);
    int64_t off = 0;
    auto take = [&](int64_t bytes) {
        int64_t o = off;
        off += align_up(bytes > 0 ? bytes : 1, 256);
        return o;
    };
    L.o_counters = take(sizeof(sm_render_counters));
    L.o_rec = take(G * (int64_t)sizeof(ProjRec));
    L.o_rec_sorted = take(G * (int64_t)sizeof(ProjRec));
    L.o_p64 = take(G * (int64_t)sizeof(Proj64));
    L.o_dkey0 = take(G * 8);
    L.o_dkey1 = take(G * 8);
    L.o_order0 = take(G * 4);
    L.o_order1 = take(G * 4);
    L.o_tcount = take(G * 4);
    L.o_tcount_r = take(G * 4);
    L.o_tmask = take(G * 4);
    L.o_tmask_r = take(G * 4);
    L.o_toff = take(G * 4);
    L.o_ikey0 = take(I * L.key_bytes);
    L.o_ikey1 = take(I * L.key_bytes);
    L.o_ranges = take(L.n_tiles * 8);
    L.o_pix_cd = take(npx * 16);
    L.o_pix_t = take(npx * 4);
    L.o_pix_tlast = take(npx * 4);
    L.o_pix_last = take(npx * 4);
    L.o_g2d = take(G * (int64_t)sizeof(float) * kG2dStride);
    L.o_sort_hist = take(sort_scratch_bytes(G > I ? G : I));
    L.o_scan = take(scan_scratch_bytes(G));
    L.o_gbuf = take(I * (int64_t)sizeof(float) * kG2dStride);
    L.o_tile_hor = take(L.n_tiles * 4);
    L.o_tile_work = take(L.n_tiles * 4);
    L.o_tile_order = take(L.n_tiles * 4);
    L.total = off;
    return L;
}

// ------------------------------------------------------------- projection
struct CamDev {
    double r[9];
    double t[3];
    double fx, fy, cx, cy, near_plane;
    int width, height, tiles_x, tiles_y;
};

// One Gaussian of K2; returns its 32-bit depth key (for the sort histogram).
__device__ __forceinline__ uint32_t project_one(
    int64_t i, const float4 *__restrict__ params, const int32_t *__restrict__ slots, const CamDev &cam,
    int cull, ProjRec *__restrict__ rec, Proj64 *__restrict__ p64, uint32_t *__restrict__ dkey,
    unsigned long long *__restrict__ zbits, uint32_t *__restrict__ order, uint32_t *__restrict__ tcount,
    uint32_t *__restrict__ tmask) {
    const int64_t slot = slots ? (int64_t)slots[i] : i;
    const float4 A = params[slot * 4 + 0];   // px py pz qw
    const float4 B = params[slot * 4 + 1];   // qx qy qz sx
    const float4 C = params[slot * 4 + 2];   // sy sz op sh0r
    const float4 D = params[slot * 4 + 3];   // sh0g sh0b - -
    order[i] = (uint32_t)i;
    ProjGeom g;
    project_geometry((double)A.x, (double)A.y, (double)A.z, (double)A.w, (double)B.x,
                     (double)B.y, (double)B.z, (double)B.w, (double)C.x, (double)C.y, cam.r,
                     cam.t, cam.fx, cam.fy, cam.cx, cam.cy, g);
    if (!(g.z >= cam.near_plane)) {   // renderloss.py:179 keep = z >= near
        dkey[i] = ~0u;                   // after every kept depth, index order
        tcount[i] = 0;
        return ~0u;
    }
    // depth order key: fp32 z (monotone rounding of z > 0, ordered as uint);
    // ties are resolved on the exact fp64 bits by depth_tie_fixup
    const uint32_t key = __float_as_uint((float)g.z);
    dkey[i] = key;
    zbits[i] = (unsigned long long)__double_as_longlong(g.z);
    // renderloss.py:110-135: conic and clamped 3-sigma bbox (fp64)
    const double a = g.a, b = g.b, c = g.c;
    const double det = DS(DM(a, c), DM(b, b));
    ProjRec r;
    r.op = C.z;
    r.z = (float)g.z;
    const double sh[3] = {(double)C.w, (double)D.x, (double)D.y};
    float col[3];
#pragma unroll
    for (int k = 0; k < 3; k++) {
        const double v = DA(DM(SM_SH_C0, sh[k]), 0.5);
        col[k] = (float)(v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v));
    }
    r.r = col[0];
    r.g = col[1];
    r.b = col[2];
    if (det <= 0.0 || a <= 0.0 || c <= 0.0) {
        tcount[i] = 0;
        r.x0y0 = 0;
        r.x1y1 = (int32_t)0xffffffff;   // empty box
        r.ox = r.oy = r.ia = r.ib = r.ic = r.eps = 0.f;
        r.beta = r.G = 0.f;
        r.K = -1.f;
        rec[i] = r;
        return key;
    }
    const double ia = DD(c, det), ib = DD(-b, det), ic = DD(a, det);
    const double rx = DM(3.0, __dsqrt_rn(a)), ry = DM(3.0, __dsqrt_rn(c));
    double fx0 = ceil(DS(g.u, rx)), fx1 = floor(DA(g.u, rx));
    double fy0 = ceil(DS(g.v, ry)), fy1 = floor(DA(g.v, ry));
    fx0 = fmin(fmax(fx0, 0.0), (double)cam.width);
    fy0 = fmin(fmax(fy0, 0.0), (double)cam.height);
    fx1 = fmax(fmin(fx1, (double)(cam.width - 1)), -1.0);
    fy1 = fmax(fmin(fy1, (double)(cam.height - 1)), -1.0);
    const int x0 = (int)fx0, x1 = (int)fx1, y0 = (int)fy0, y1 = (int)fy1;
    const double dax = DS((double)x0, g.u), day = DS((double)y0, g.v);
    const double sia = DM(kPowScale, ia), sib = DM(kPowScale, ib), sic = DM(kPowScale, ic);
    r.ox = (float)dax;
    r.oy = (float)day;
    r.ia = (float)sia;
    r.ib = (float)sib;
    r.ic = (float)sic;
    {
        // fp32 error band of the corner expansion (stage_anchor +
        // compositing): a few roundings of partial sums bounded by S, the sum
        // of |terms| at the far box corner (<= ~10 ulp of S), plus the
        // direct form's anisotropy bound 36 K for the fp32 anchors of
        // ordinary splats; both with a wide margin
        const double hax = DA(DM(sia, dax), DM(sib, day)), hay = DA(DM(sib, dax), DM(sic, day));
        const double qa = DA(DM(dax, hax), DM(day, hay));
        const double wx = fmax((double)(x1 - x0), 0.0), wy = fmax((double)(y1 - y0), 0.0);
        const double S = fabs(qa) + 2.0 * (fabs(hax) * wx + fabs(hay) * wy) + fabs(sia) * wx * wx +
                         2.0 * fabs(sib) * wx * wy + fabs(sic) * wy * wy;
        const double K = DD(DM(a, c), det);
        r.eps = (float)fmax(1e-5 * S + 1e-6, DM(DM(1e-4, DA(1.0, K)), -kPowScale));
    }
    r.x0y0 = (int32_t)(((uint32_t)y0 << 16) | ((uint32_t)x0 & 0xffffu));
    r.x1y1 = (int32_t)(((uint32_t)(y1 & 0xffff) << 16) | ((uint32_t)x1 & 0xffffu));
    r.beta = (float)DD(b, c);
    r.G = (float)DD(DM(9.0, det), c);
    r.K = cull ? (float)DD(det, DM(c, c)) : -1.f;
    rec[i] = r;
    Proj64 q;
    q.u = g.u;
    q.v = g.v;
    q.ia = ia;
    q.ib = ib;
    q.ic = ic;
    p64[i] = q;
    if (x1 < x0 || y1 < y0) {
        tcount[i] = 0;
        return key;
    }
    // tiles the q <= 9 ellipse reaches (RowSpan); small splats keep them as a mask
    const RowSpan sp(r);
    if (bbox_tiles(r) <= kEmitSmall) {
        const uint32_t m = small_mask(sp);
        tmask[i] = m;
        tcount[i] = (uint32_t)__popc(m);
    } else {
        uint32_t cnt = 0;
        for (int ty = sp.ty0; ty <= sp.ty1; ty++) cnt += (uint32_t)sp.count(ty);
        tcount[i] = cnt;
    }
    return key;
}

// K2 over the visible set; also zeroes the pass's device counters and tile
// ranges and counts the depth keys' digits for the sort (saves two memsets
// and the sort's histogram pass).
#ifndef SM_PROJ_MINB
#define SM_PROJ_MINB 4   // <= 64 registers: 4 x 256 threads per SM, measured best of 1 and 4-6
#endif
__global__ void __launch_bounds__(256, SM_PROJ_MINB)
project_fwd(const float4 *__restrict__ params, const int32_t *__restrict__ slots, int64_t n,
            CamDev cam, int cull, ProjRec *__restrict__ rec, Proj64 *__restrict__ p64,
            uint32_t *__restrict__ dkey, unsigned long long *__restrict__ zbits,
            uint32_t *__restrict__ order,
            uint32_t *__restrict__ tcount, uint32_t *__restrict__ tmask,
            uint32_t *__restrict__ ctr_words, uint32_t *__restrict__ ranges, int64_t n_range_words,
            uint32_t *__restrict__ depth_hist) {
    __shared__ uint32_t h[4][256];
    block_hist_zero(h, 4);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < (int64_t)(sizeof(sm_render_counters) / 4)) ctr_words[i] = 0u;
    if (i < n_range_words) ranges[i] = 0u;
    __syncthreads();
    if (i < n) {
        const uint32_t key = project_one(i, params, slots, cam, cull, rec, p64, dkey, zbits, order, tcount, tmask);
        block_hist_add(h, key, 0, 32);
    }
    __syncthreads();
    block_hist_flush(h, 4, depth_hist);
}

// The 32-bit depth sort is stable, so within a run of equal fp32 keys the
// Gaussians are in index order; np.argsort(z, kind="stable") orders them by
// the fp64 z first.  The run's first thread re-sorts the run (stable
// insertion sort on the fp64 bits) when it holds an inversion -- runs are a
// few elements long (distinct fp64 depths within one fp32 ulp).
__global__ void __launch_bounds__(256)
depth_tie_fixup(const uint32_t *__restrict__ key, uint32_t *__restrict__ order, int64_t n,
                const unsigned long long *__restrict__ zbits) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r + 1 >= n) return;
    const uint32_t k = key[r];
    if (k == ~0u || key[r + 1] != k || (r > 0 && key[r - 1] == k)) return;   // not a run head
    int64_t e = r + 1;
    bool inv = false;
    unsigned long long prev = zbits[order[r]];
    for (; e < n && key[e] == k; e++) {
        const unsigned long long z = zbits[order[e]];
        inv |= z < prev;
        prev = z;
    }
    if (!inv) return;
    for (int64_t a = r + 1; a < e; a++) {   // stable insertion sort of order[r, e) by zbits
        const uint32_t oa = order[a];
        const unsigned long long za = zbits[oa];
        int64_t b = a - 1;
        while (b >= r && zbits[order[b]] > za) {
            order[b + 1] = order[b];
            b--;
        }
        order[b + 1] = oa;
    }
}

__global__ void __launch_bounds__(256)
gather_by_rank(const uint32_t *__restrict__ order, int64_t n, const ProjRec *__restrict__ rec,
               const uint32_t *__restrict__ tcount, const uint32_t *__restrict__ tmask,
               ProjRec *__restrict__ rec_sorted, uint32_t *__restrict__ tcount_r,
               uint32_t *__restrict__ tmask_r) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t i = order[r];
    const uint32_t c = tcount[i];
    tcount_r[r] = c;
    if (c) {
        rec_sorted[r] = rec[i];
        tmask_r[r] = tmask[i];   // meaningful for small splats only
    }
}


// Instance emission.  Splat footprints are heavy-tailed and the biggest
// (nearest) ones sit together at the lowest depth ranks, so emission is split:
// a thread per rank writes splats of <= kEmitSmall tiles directly, larger ones
// are queued and a warp per queued splat writes its tiles in parallel.
// Keys are (tile << rank_bits) | rank at the rank's scanned offset, so the
// array is in rank order whichever thread writes a slot.  KeyT is uint32_t
// while rank_bits + tile_bits <= 32 (up to 2M visible splats at 2048 tiles),
// else 64-bit (the sort then reads twice the bytes).
template <typename KeyT>
__global__ void __launch_bounds__(256)
emit_instances(const ProjRec *__restrict__ rec_sorted, const uint32_t *__restrict__ tcount_r,
               const uint32_t *__restrict__ tmask_r, const uint32_t *__restrict__ toff, int64_t n, sm_render_counters *ctr,
               uint32_t *__restrict__ big, int rank_bits, int tiles_x, KeyT *__restrict__ ikeys) {
    if (ctr->overflow) return;
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t cnt = tcount_r[r];
    if (!cnt) return;
    const ProjRec g = rec_sorted[r];
    if (bbox_tiles(g) > kEmitSmall) {
        big[atomicAdd(&ctr->reserved[1], 1u)] = (uint32_t)r;
        return;
    }
    // kept tiles = set bits of the box mask, row-major
    const int tx0 = rec_x0(g) / kTile, ty0 = rec_y0(g) / kTile, ntx = rec_x1(g) / kTile - tx0 + 1;
    uint32_t o = toff[r];
    for (uint32_t m = tmask_r[r]; m; m &= m - 1) {
        const int bit = __ffs(m) - 1;
        const int t = (ty0 + bit / ntx) * tiles_x + tx0 + bit % ntx;
        ikeys[o++] = ((KeyT)t << rank_bits) | (KeyT)r;
    }
}

template <typename KeyT>
__global__ void __launch_bounds__(256)
emit_big(const ProjRec *__restrict__ rec_sorted, const uint32_t *__restrict__ tcount_r,
         const uint32_t *__restrict__ toff, const sm_render_counters *ctr,
         const uint32_t *__restrict__ big, int rank_bits, int tiles_x, KeyT *__restrict__ ikeys) {
    if (ctr->overflow) return;
    __shared__ BigRowTable tab;
    const uint32_t nbig = ctr->reserved[1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t b = blockIdx.x; b < nbig; b += gridDim.x) {   // a block per big splat
        const uint32_t r = big[b];
        const RowSpan sp(rec_sorted[r]);
        const uint32_t o = toff[r];
        uint32_t base = 0;
        for (int tyb = sp.ty0; tyb <= sp.ty1; tyb += kBigThreads) {
            base = fill_row_table(sp, tyb, base, tab);
            const int nrows = min(kBigThreads, sp.ty1 - tyb + 1);
            for (int i = warp; i < nrows; i += kBigThreads / 32) {
                const int c0 = tab.c0[i], c1 = tab.c1[i], row = (tyb + i) * tiles_x;
                const uint32_t dst = o + tab.off[i] - (uint32_t)c0;
                for (int c = c0 + lane; c <= c1; c += 32)
                    ikeys[dst + (uint32_t)c] = ((KeyT)(row + c) << rank_bits) | (KeyT)r;
            }
        }
    }
}

template <typename KeyT>
__global__ void __launch_bounds__(256)
tile_ranges(const KeyT *__restrict__ ikeys, const sm_render_counters *ctr, int rank_bits,
            uint32_t *__restrict__ ranges) {
    const int64_t n = ctr->reserved[0];
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t t = (uint32_t)(ikeys[p] >> rank_bits);
        if (p == 0 || (ikeys[p - 1] >> rank_bits) != t) ranges[2 * t] = (uint32_t)p;
        if (p == n - 1 || (ikeys[p + 1] >> rank_bits) != t) ranges[2 * t + 1] = (uint32_t)(p + 1);
    }
}

// ------------------------------------------------------------ compositing
// Per-pixel front-to-back state (renderloss.py:136-152 loop body).
struct FwdPix {
    float T, cr, cg, cb, cd, tlast;
    int32_t last;
    bool done;

    // c = {r, g, b, z} of the splat
    __device__ __forceinline__ void add(float op, const float4 &c, float pw, int32_t k) {
        const float alpha = op * ex2_approx(pw);
        const float w = T * alpha;
        cr += w * c.x;
        cg += w * c.y;
        cb += w * c.z;
        cd += w * c.w;
        tlast = T;
        last = k;
        T = T * (1.f - alpha);
        done = T < (float)SM_MIN_T;   // later pairs would be skipped (renderloss.py:143)
    }

    __device__ __forceinline__ void store(int64_t p, float *out_rgb, float *out_depth,
                                          float *out_alpha, float4 *st_cd, float *st_t,
                                          float *st_tlast, int32_t *st_last) const {
        const float A = 1.f - T;   // renderloss.py:216-218 finalize
        out_rgb[3 * p + 0] = fminf(fmaxf(cr, 0.f), 1.f);
        out_rgb[3 * p + 1] = fminf(fmaxf(cg, 0.f), 1.f);
        out_rgb[3 * p + 2] = fminf(fmaxf(cb, 0.f), 1.f);
        out_depth[p] = A > 0.f ? cd / A : 0.f;
        out_alpha[p] = fminf(fmaxf(A, 0.f), 1.f);
        st_cd[p] = make_float4(cr, cg, cb, cd);
        st_t[p] = T;
        st_tlast[p] = tlast;
        st_last[p] = last;
    }
};

// One CTA per 16x16 tile, 256 threads, a pixel each.  The tile's instances
// (depth-rank order) are staged one CTA-width batch at a time in shared
// memory; a warp skips a splat whose 3-sigma box misses its 2 rows
// (warp-uniform), a thread skips it when its column is outside the box, and
// the block stops once every pixel's transmittance is below 1e-10.
#ifndef SM_FWD_MINB
#define SM_FWD_MINB 1
#endif
template <typename KeyT>
__global__ void __launch_bounds__(kTilePx, SM_FWD_MINB)
composite_fwd(const uint32_t *__restrict__ ranges, const KeyT *__restrict__ ikeys,
              KeyT rank_mask, const ProjRec *__restrict__ recs,
              const Proj64 *__restrict__ p64, const uint32_t *__restrict__ order, int width,
              int height, int tiles_x, float *__restrict__ out_rgb, float *__restrict__ out_depth,
              float *__restrict__ out_alpha, float4 *__restrict__ st_cd, float *__restrict__ st_t,
              float *__restrict__ st_tlast, int32_t *__restrict__ st_last, uint32_t *__restrict__ tile_work,
              const uint32_t *__restrict__ launch_order) {
    constexpr int NT = kTilePx;
    // per staged instance, exactly what the pixel loop reads (64 B):
    __shared__ int4 s_box[NT];      // x0, x1 - x0, y0, y1 - y0
    __shared__ float4 s_anch[NT];   // qa, 2 hax, 2 hay, 2 ib (stage_anchor, gradient doubled)
    __shared__ float4 s_cof[NT];    // ia, ic, op, eps
    __shared__ float4 s_col[NT];    // r, g, b, z
    __shared__ uint32_t s_wm[NT];   // bit w: the box reaches warp w's two rows
    __shared__ uint32_t s_rank[NT];
    __shared__ int s_maxlast;
    // longest-first when the caller keeps the previous render's order of this view
    const int tile = launch_order ? (int)launch_order[blockIdx.x] : (int)blockIdx.x;
    const int ty0 = (tile / tiles_x) * kTile;
    const int px = (tile % tiles_x) * kTile + (threadIdx.x & (kTile - 1));
    const int py = ty0 + threadIdx.x / kTile;
    const int wy0 = ty0 + 2 * (threadIdx.x / 32);   // warp's first row
    const uint32_t start = ranges[2 * tile], end = ranges[2 * tile + 1];
    const bool in = px < width && py < height;
    FwdPix s = FwdPix{1.f, 0.f, 0.f, 0.f, 0.f, 1.f, -1, !in};
    bool all_done = s.done;
    for (uint32_t base = start; base < end; base += NT) {
        if (__syncthreads_count(all_done) == NT) break;
        const uint32_t idx = base + threadIdx.x;
        if (idx < end) {
            const uint32_t rk = (uint32_t)(ikeys[idx] & rank_mask);
            s_rank[threadIdx.x] = rk;
            const ProjRec r = recs[rk];
            s_box[threadIdx.x] = make_int4(rec_x0(r), rec_x1(r) - rec_x0(r), rec_y0(r), rec_y1(r) - rec_y0(r));
            const float4 an = stage_anchor(r, p64, order, rk);   // {qa, hax, hay, -}
            s_anch[threadIdx.x] = make_float4(an.x, 2.f * an.y, 2.f * an.z, 2.f * r.ib);
            s_cof[threadIdx.x] = make_float4(r.ia, r.ic, r.op, r.eps);
            s_col[threadIdx.x] = make_float4(r.r, r.g, r.b, r.z);
            const int lo = max(rec_y0(r) - ty0, 0) >> 1, hi = min(rec_y1(r) - ty0, kTile - 1) >> 1;
            s_wm[threadIdx.x] = hi >= lo ? ((2u << hi) - 1u) & ~((1u << lo) - 1u) : 0u;
        }
        __syncthreads();
        const int cnt = (int)min((uint32_t)NT, end - base);
        // the warp walks only the staged splats whose box reaches its two rows,
        // in order: a ballot per 32 of them over the staging-time row masks
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int c = 0; c < cnt; c += 32) {
            if (__all_sync(0xffffffffu, all_done)) break;
            uint32_t m = __ballot_sync(0xffffffffu, c + lane < cnt && ((s_wm[c + lane] >> warp) & 1u));
            if (all_done) continue;
            for (; m; m &= m - 1) {
                const int j = c + __ffs(m) - 1;
                const int4 bx = s_box[j];   // x0, x1 - x0, y0, y1 - y0 (decoded once at staging)
                if ((unsigned)(px - bx.x) > (unsigned)bx.y || (unsigned)(py - bx.z) > (unsigned)bx.w) continue;
                // pw = qa + cx (2 hax + ia cx + 2 ib cy) + cy (2 hay + ic cy)
                const float cx = (float)(px - bx.x), cy = (float)(py - bx.z);
                const float4 an = s_anch[j], cf = s_cof[j];
                const float pw = fmaf(cx, fmaf(cf.x, cx, fmaf(an.w, cy, an.y)), fmaf(cy, fmaf(cf.y, cy, an.z), an.x));
                if (q_within_cutoff(pw, cf.w, p64, order, s_rank[j], px, py)) {
                    s.add(cf.z, s_col[j], pw, (int32_t)(base + j));
                    if (s.done) {
                        all_done = true;
                        break;
                    }
                }
            }
        }
        __syncthreads();
    }
    if (in)
        s.store((int64_t)py * width + px, out_rgb, out_depth, out_alpha, st_cd, st_t, st_tlast, st_last);
    // the backward revisits [start, max last]: its work estimate for scheduling
    if (threadIdx.x == 0) s_maxlast = -1;
    __syncthreads();
    const int wl = __reduce_max_sync(0xffffffffu, s.last);
    if ((threadIdx.x & 31) == 0) atomicMax(&s_maxlast, wl);
    __syncthreads();
    if (threadIdx.x == 0) tile_work[tile] = s_maxlast >= (int)start ? (uint32_t)(s_maxlast - (int)start + 1) : 0u;
}

// Longest-first launch order of the tiles for the backward: a counting sort
// of the tiles into 64 work buckets, heaviest bucket first (one block).  The
// backward's CTAs then start heavy tiles first and light ones fill in behind
// them (LPT), shortening the tail.  Order inside a bucket is arbitrary: tiles
// are independent, so results do not depend on it.  `keep` (nullable) gets
// a copy: the next forward of the same view launches in this order.
constexpr int kWorkBuckets = 64;
__global__ void __launch_bounds__(1024)
order_tiles(const uint32_t *__restrict__ work, int n_tiles, uint32_t *__restrict__ order,
            uint32_t *__restrict__ keep) {
    __shared__ uint32_t hist[kWorkBuckets], base[kWorkBuckets];
    __shared__ uint32_t wmax;
    if (threadIdx.x < kWorkBuckets) hist[threadIdx.x] = 0;
    if (threadIdx.x == 0) wmax = 1;
    __syncthreads();
    for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) atomicMax(&wmax, work[i]);
    __syncthreads();
    const uint32_t div = (wmax + kWorkBuckets - 1) / kWorkBuckets;
    for (int i = threadIdx.x; i < n_tiles; i += blockDim.x)
        atomicAdd(&hist[kWorkBuckets - 1 - min(work[i] / div, (uint32_t)kWorkBuckets - 1)], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int b = 0; b < kWorkBuckets; b++) {
            base[b] = run;
            run += hist[b];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) {
        const uint32_t o = atomicAdd(&base[kWorkBuckets - 1 - min(work[i] / div, (uint32_t)kWorkBuckets - 1)], 1u);
        order[o] = (uint32_t)i;
        if (keep) keep[o] = (uint32_t)i;
    }
}

StreamFork &stream_fork() {
    static thread_local StreamFork forks[64];
    int dev = 0;
    cudaGetDevice(&dev);
    StreamFork &f = forks[dev & 63];
    if (!f.side) {
        cudaStreamCreateWithFlags(&f.side, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&f.join, cudaEventDisableTiming);
    }
    return f;
}

int g_ellipse_cull = 1;   // sm_set_ellipse_cull (tests: culled == unculled, bit for bit)

CamDev make_cam(const sm_camera &c, const RenderLayout &L) {
    CamDev d;
    for (int k = 0; k < 9; k++) d.r[k] = c.r_wc[k];
    for (int k = 0; k < 3; k++) d.t[k] = c.t[k];
    d.fx = c.fx;
    d.fy = c.fy;
    d.cx = c.cx;
    d.cy = c.cy;
    d.near_plane = c.near_plane;
    d.width = c.width;
    d.height = c.height;
    d.tiles_x = L.tiles_x;
    d.tiles_y = L.tiles_y;
    return d;
}

// Emission + tile sort + ranges for one key width.
template <typename KeyT>
static void bin_tiles(const RenderBufs &b, const RenderLayout &L, const sm_render_dims &dims, int64_t n,
                      unsigned gb, const SortScratch &ss, cudaStream_t st) {
    KeyT *k0 = static_cast<KeyT *>(b.ikey0), *k1 = static_cast<KeyT *>(b.ikey1);
    prof_begin(ST_BIN, st);
    gather_by_rank<<<gb, 256, 0, st>>>(b.order0, n, b.rec, b.tcount, b.tmask, b.rec_sorted, b.tcount_r,
                                       b.tmask_r);
    exclusive_scan(b.tcount_r, b.toff, n, b.scan, &b.ctr->n_instances, st, dims.max_instances,
                   &b.ctr->overflow, &b.ctr->reserved[0]);   // + the instance-capacity check
    // b.tcount (per visible index) is dead after gather_by_rank: reuse it as the big-splat queue
    emit_instances<KeyT><<<gb, 256, 0, st>>>(b.rec_sorted, b.tcount_r, b.tmask_r, b.toff, n, b.ctr, b.tcount,
                                             L.rank_bits, L.tiles_x, k0);
    emit_big<KeyT><<<148 * 4, 256, 0, st>>>(b.rec_sorted, b.tcount_r, b.toff, b.ctr, b.tcount, L.rank_bits,
                                            L.tiles_x, k0);
    prof_end(ST_BIN, st);
    prof_begin(ST_TILE_SORT, st);
    // (counting the tile digits inside the emission was measured slower than
    // the sort's own histogram pass: shared-atomic contention on 2 x 256 bins)
    // (a single 11-bit pass with the ranges taken from its digit scan was
    // measured slower: 0.090 vs 0.071 ms at C2 -- 2048 digits per 4096-key
    // block cost more than the second pass)
    const int cur = radix_sort<KeyT, false, kSortItemsWide>(k0, nullptr, k1, nullptr, &b.ctr->reserved[0], 0,
                                            dims.max_instances, L.rank_bits, L.rank_bits + L.tile_bits, ss, st);
    tile_ranges<KeyT><<<148 * 8, 256, 0, st>>>(cur ? k1 : k0, b.ctr, L.rank_bits, b.ranges);
    prof_end(ST_TILE_SORT, st);
}

template <typename KeyT>
static void launch_composite_fwd(const RenderBufs &b, const RenderLayout &L, const sm_render_dims &dims,
                                 float *out_rgb, float *out_depth, float *out_alpha, uint32_t *view_order,
                                 cudaStream_t st) {
    const KeyT rank_mask = (KeyT)((1ull << L.rank_bits) - 1ull);
    const KeyT *ik = static_cast<const KeyT *>(L.tile_passes & 1 ? b.ikey1 : b.ikey0);
    composite_fwd<KeyT><<<(unsigned)L.n_tiles, kTilePx, 0, st>>>(
        b.ranges, ik, rank_mask, b.rec_sorted, b.p64, b.order0, dims.width, dims.height, L.tiles_x,
        out_rgb, out_depth, out_alpha, b.pix_cd, b.pix_t, b.pix_tlast, b.pix_last, b.tile_work, view_order);
    order_tiles<<<1, 1024, 0, st>>>(b.tile_work, (int)L.n_tiles, b.tile_order, view_order);
}

int render_forward(const float *params, const int32_t *slots, int64_t n, const sm_camera &cam,
                   const sm_render_dims &dims, void *ws, int64_t ws_bytes, float *out_rgb,
                   float *out_depth, float *out_alpha, uint32_t *view_order, cudaStream_t st) {
    const RenderLayout L = render_layout(dims);
    if (ws_bytes < L.total) {
        set_error("render workspace too small: %lld < %lld", (long long)ws_bytes, (long long)L.total);
        return SM_ERR_WORKSPACE;
    }
    if (n < 0 || n > dims.max_gaussians) {
        set_error("n=%lld outside [0, max_gaussians=%lld]", (long long)n, (long long)dims.max_gaussians);
        return SM_ERR_INVALID;
    }
    if (cam.width != dims.width || cam.height != dims.height || cam.width < 1 || cam.height < 1) {
        set_error("camera %dx%d does not match workspace %dx%d", cam.width, cam.height, dims.width,
                  dims.height);
        return SM_ERR_DIMENSION;
    }
    if (L.rank_bits + L.tile_bits > 64) {
        set_error("rank bits %d + tile bits %d exceed 64", L.rank_bits, L.tile_bits);
        return SM_ERR_INVALID;
    }
    RenderBufs b = render_bufs(ws, L);
    CamDev cd = make_cam(cam, L);
    if (n == 0) {
        cudaMemsetAsync(b.ctr, 0, sizeof(sm_render_counters), st);
        cudaMemsetAsync(b.ranges, 0, L.n_tiles * 8, st);
    } else {
        const unsigned gb = (unsigned)ceil_div(n, 256);
        const unsigned gp = (unsigned)ceil_div(n > 2 * L.n_tiles + 16 ? n : 2 * L.n_tiles + 16, 256);
        // 32-bit depth keys, ping-pong halves of the dkey0 region; fp64 z bits in dkey1
        uint32_t *dk = reinterpret_cast<uint32_t *>(b.dkey0);
        const SortScratch ss = sort_scratch(b.sort_hist, dims.max_gaussians > dims.max_instances
                                                             ? dims.max_gaussians : dims.max_instances);
        prof_begin(ST_PROJECT, st);
        sort_reset(ss, n, 0, 32, st);   // the projection fills the depth sort's histograms
        project_fwd<<<gp, 256, 0, st>>>(reinterpret_cast<const float4 *>(params), slots, n, cd,
                                        g_ellipse_cull, b.rec, b.p64, dk, b.dkey1, b.order0, b.tcount, b.tmask,
                                        reinterpret_cast<uint32_t *>(b.ctr), b.ranges, 2 * L.n_tiles, ss.hist);
        prof_end(ST_PROJECT, st);
        // global stable depth order: 4 passes over the fp32 key + fp64 tie fixup
        prof_begin(ST_DEPTH_SORT, st);
        const int dcur = radix_sort<uint32_t, true>(dk, b.order0, dk + dims.max_gaussians, b.order1,
                                                    nullptr, n, n, 0, 32, ss, st, /*hist_ready=*/true);
        (void)dcur;   // 4 passes: keys and order end in buffer 0
        depth_tie_fixup<<<gb, 256, 0, st>>>(dk, b.order0, n, b.dkey1);
        prof_end(ST_DEPTH_SORT, st);
        if (L.key_bytes == 8)
            bin_tiles<unsigned long long>(b, L, dims, n, gb, ss, st);
        else
            bin_tiles<uint32_t>(b, L, dims, n, gb, ss, st);
        count_launches(1 + L.depth_passes + 1 + 6 + (1 + L.tile_passes) + 1);
    }
    prof_begin(ST_COMPOSITE_FWD, st);
    if (L.key_bytes == 8)
        launch_composite_fwd<unsigned long long>(b, L, dims, out_rgb, out_depth, out_alpha, view_order, st);
    else
        launch_composite_fwd<uint32_t>(b, L, dims, out_rgb, out_depth, out_alpha, view_order, st);
    prof_end(ST_COMPOSITE_FWD, st);
    count_launches(2);
    SM_CHECK_LAUNCH("render_forward");
    return SM_OK;
}

}  // namespace sm
