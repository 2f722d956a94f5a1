// K5 composite backward + K6 projection backward.
//
// The reference is forward-only (pkg/README.md:125-129); this is the exact
// reverse-mode derivative of the forward in render_fwd.cu (itself the
// restatement of renderloss.py:106-218), with the reference's semantics:
// no alpha cap, T >= 1e-10 checked before a contribution, 3-sigma box,
// q > 9 excluded, colour clip (zero gradient outside [0,1]), final rgb/alpha
// clip, depth = D / alpha.  Oracle: oracle/render_oracle.c or_render_bwd,
// pinned by central differences of the reference forward.
//
// Per pixel the contributors are revisited back to front.  T_k is recovered
// as T_{k+1} / (1 - alpha_k) (the last contributor's T is stored, so
// alpha = 1 never divides by zero), the colour/depth behind k is carried
// normalised (B_k = alpha_{k+1} c_{k+1} + (1 - alpha_{k+1}) B_{k+1}) and
// dA/dalpha_k uses the running product P_k = prod_{j>k} (1 - alpha_j).
// Per-splat sums without floating-point atomics (deterministic): a 10-value
// transposed warp butterfly (14 shuffles), per-warp shared slots added in warp
// order, one gradient slot per (splat, tile) instance, and a fixed-order sum
// over a splat's instances (inline in project_bwd, or a block per big splat).
#include "adam.cuh"
#include "prof.cuh"
#include "render.cuh"

namespace sm {

// Warp sum of 10 per-lane values with 14 shuffles: an 8-wide transposed
// butterfly (offsets 16, 8, 4 halve the value count, 2 and 1 finish) leaves
// the sum of value 4*b4 + 2*b3 + b2 (bits of the lane id) in every lane; a
// 2-wide one leaves value 8 + b4.  Returns (sa, sb).
__device__ __forceinline__ float2 transpose_reduce10(const float (&v)[16], int lane) {
    float a[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const bool hi = lane & 16;
        a[k] = (hi ? v[k + 4] : v[k]) + __shfl_xor_sync(0xffffffffu, hi ? v[k] : v[k + 4], 16);
    }
    float b[2];
#pragma unroll
    for (int k = 0; k < 2; k++) {
        const bool hi = lane & 8;
        b[k] = (hi ? a[k + 2] : a[k]) + __shfl_xor_sync(0xffffffffu, hi ? a[k] : a[k + 2], 8);
    }
    float c;
    {
        const bool hi = lane & 4;
        c = (hi ? b[1] : b[0]) + __shfl_xor_sync(0xffffffffu, hi ? b[0] : b[1], 4);
    }
    c += __shfl_xor_sync(0xffffffffu, c, 2);
    c += __shfl_xor_sync(0xffffffffu, c, 1);
    float d;
    {
        const bool hi = lane & 16;
        d = (hi ? v[9] : v[8]) + __shfl_xor_sync(0xffffffffu, hi ? v[8] : v[9], 16);
    }
    d += __shfl_xor_sync(0xffffffffu, d, 8);
    d += __shfl_xor_sync(0xffffffffu, d, 4);
    d += __shfl_xor_sync(0xffffffffu, d, 2);
    d += __shfl_xor_sync(0xffffffffu, d, 1);
    return make_float2(c, d);
}

// Per-pixel reverse state, initialised from the forward's stored per-pixel
// values.  T holds T_{k+1} while walking back; the stored T before the last
// contributor seeds T_k at k == last (alpha = 1 safe).
struct BwdPix {
    float gCr, gCg, gCb, gD, gA;   // dL/d{C, D, A} of the raw accumulators
    float T, tlast;
    int32_t last;

    __device__ __forceinline__ void init(bool inside, int64_t p, const float *d_rgb,
                                         const float *d_depth, const float *d_alpha,
                                         const float4 *st_cd, const float *st_t,
                                         const float *st_tlast, const int32_t *st_last) {
        gCr = gCg = gCb = gD = gA = 0.f;
        T = tlast = 0.f;
        last = -1;
        if (!inside) return;
        const float4 cd = st_cd[p];
        T = st_t[p];
        tlast = st_tlast[p];
        last = st_last[p];
        const float A = 1.f - T;
        if (d_rgb) {   // rgb = clip(C) (renderloss.py:218): zero gradient outside [0,1]
            gCr = (cd.x >= 0.f && cd.x <= 1.f) ? d_rgb[3 * p + 0] : 0.f;
            gCg = (cd.y >= 0.f && cd.y <= 1.f) ? d_rgb[3 * p + 1] : 0.f;
            gCb = (cd.z >= 0.f && cd.z <= 1.f) ? d_rgb[3 * p + 2] : 0.f;
        }
        if (d_alpha && A >= 0.f && A <= 1.f) gA = d_alpha[p];
        if (d_depth && A > 0.f) {   // depth = D / A (renderloss.py:217)
            const float dd = d_depth[p];
            gD = dd / A;
            gA += -dd * cd.w / (A * A);
        }
    }
};

// A thread's two pixels (same column, rows py and py + 1) walked back
// together in packed fp32x2: .x is row py, .y row py + 1.  A pixel the splat
// does not reach gets G = 0, which makes every contribution exactly zero and
// leaves T, B and P unchanged (1 - 0 = 1), so the step is branch-free.
struct BwdPair {
    float2 gCr, gCg, gCb, gD, gA;
    float2 T, tlast, Br, Bg, Bb, Bz, P;
    int32_t last0, last1;

    __device__ __forceinline__ void init(const BwdPix &a, const BwdPix &b) {
        gCr = make_float2(a.gCr, b.gCr);
        gCg = make_float2(a.gCg, b.gCg);
        gCb = make_float2(a.gCb, b.gCb);
        gD = make_float2(a.gD, b.gD);
        gA = make_float2(a.gA, b.gA);
        T = make_float2(a.T, b.T);
        tlast = make_float2(a.tlast, b.tlast);
        Br = Bg = Bb = Bz = f2s(0.f);
        P = f2s(1.f);
        last0 = a.last;
        last1 = b.last;
    }

    // d{u v ia ib ic op r g b z} of splat g (instance position k) summed over
    // the pair into v[0..9]; then one step back.
    __device__ __forceinline__ void step(const ProjRec &g, float dx, float2 dy, float2 pw, float2 hx,
                                         float2 hy, bool h0, bool h1, int k, float (&v)[16]) {
        const float2 G = make_float2(h0 ? ex2_approx(pw.x) : 0.f, h1 ? ex2_approx(pw.y) : 0.f);
        const float2 alpha = mul2(G, f2s(g.op));
        const float2 oma = sub2(f2s(1.f), alpha);
        // T_k = T_{k+1} / (1 - alpha_k); 1 - alpha >= 2^-24 unless k is the
        // pixel's last contributor (stored T).  Non-hits keep T.
        const float2 Tq = mul2(T, make_float2(rcp_approx(oma.x), rcp_approx(oma.y)));
        float2 Tk;
        Tk.x = !h0 ? T.x : (k == last0 ? tlast.x : Tq.x);
        Tk.y = !h1 ? T.y : (k == last1 ? tlast.y : Tq.y);
        float2 ga = mul2(sub2(f2s(g.r), Br), gCr);
        ga = fma2(sub2(f2s(g.g), Bg), gCg, ga);
        ga = fma2(sub2(f2s(g.b), Bb), gCb, ga);
        ga = fma2(sub2(f2s(g.z), Bz), gD, ga);
        ga = mul2(Tk, fma2(gA, P, ga));
        const float2 wt = mul2(Tk, alpha);
        v[6] = hsum(mul2(wt, gCr));
        v[7] = hsum(mul2(wt, gCg));
        v[8] = hsum(mul2(wt, gCb));
        v[9] = hsum(mul2(wt, gD));
        v[5] = hsum(mul2(ga, G));
        // q = pw / kPowScale; conic grads are w.r.t. the unscaled conic
        const float2 gq = mul2(f2s(-0.5f), mul2(alpha, ga));
        const float2 gqdx = mul2(gq, f2s(dx));
        v[2] = hsum(mul2(gqdx, f2s(dx)));
        v[3] = hsum(mul2(mul2(gqdx, f2s(2.f)), dy));
        v[4] = hsum(mul2(mul2(gq, dy), dy));
        const float2 gqi = mul2(gq, f2s((float)(-2.0 / kPowScale)));
        v[0] = hsum(mul2(gqi, hx));   // C (x - u), from the corner expansion
        v[1] = hsum(mul2(gqi, hy));
        Br = fma2(alpha, f2s(g.r), mul2(oma, Br));
        Bg = fma2(alpha, f2s(g.g), mul2(oma, Bg));
        Bb = fma2(alpha, f2s(g.b), mul2(oma, Bb));
        Bz = fma2(alpha, f2s(g.z), mul2(oma, Bz));
        P = mul2(P, oma);
        T = Tk;
    }
};

// Same tiling as composite_fwd: one CTA per 16x16 tile, 128 threads, each
// owning a pixel pair (BwdPair); warp w covers tile rows 4w .. 4w + 3.
// Instances are revisited from the block's last contributor back to the tile
// start, one CTA-width batch at a time; a warp skips splats missing its rows,
// lying past every one of its pixels' last contributor, or reaching none of
// its pixels.
//
// Determinism: no floating-point atomics.  Each warp's 10 sums for an
// instance land in its own shared slot; after the batch the slots are added
// in warp order and written to the instance's emission slot (toff[rank] + the
// tile's index among the splat's kept tiles); grad_gather then sums a splat's
// instances in a fixed order.  Reruns and CUDA-graph replays are bit-identical
// (the reference's metrics determinism contract, test_acceptance.py crit. 10).
constexpr int kBwdThreads = kTilePx / 2;
#ifndef SM_BWD_MINB
#define SM_BWD_MINB 5   // 5 CTAs x 4 warps per SM: measured best (register cap 102)
#endif

template <typename KeyT>
__global__ void __launch_bounds__(kBwdThreads, SM_BWD_MINB)
composite_bwd(const uint32_t *__restrict__ ranges, const KeyT *__restrict__ ikeys,
              KeyT rank_mask, const ProjRec *__restrict__ recs,
              const Proj64 *__restrict__ p64, const uint32_t *__restrict__ order, int width,
              int height, int tiles_x, const float *__restrict__ d_rgb,
              const float *__restrict__ d_depth, const float *__restrict__ d_alpha,
              const float4 *__restrict__ st_cd, const float *__restrict__ st_t,
              const float *__restrict__ st_tlast, const int32_t *__restrict__ st_last,
              const uint32_t *__restrict__ toff, const uint32_t *__restrict__ tmask_r,
              float *__restrict__ gbuf, int32_t *__restrict__ tile_hor, sm_render_counters *ctr,
              const uint32_t *__restrict__ tile_order) {
    constexpr int NT = kBwdThreads;
    constexpr int NW = NT / 32;
    __shared__ ProjRec s_rec[NT];
    __shared__ uint32_t s_rank[NT];
    __shared__ float4 s_anch[NT];   // {qa, hax, hay, -}: the corner expansion (stage_anchor)
    __shared__ float s_part[NW][NT][10];
    __shared__ int s_maxlast;
    const int warp = threadIdx.x / 32;
    const int tile = (int)tile_order[blockIdx.x];   // heaviest tiles first
    const int lane = threadIdx.x & 31;
    const int ty0 = (tile / tiles_x) * kTile;
    const int px = (tile % tiles_x) * kTile + (threadIdx.x & (kTile - 1));
    const int py = ty0 + 2 * (threadIdx.x / kTile);
    const int wy0 = ty0 + 4 * (threadIdx.x / 32);
    const int start = (int)ranges[2 * tile];
    BwdPair pp;
    {
        BwdPix a, b;
        a.init(px < width && py < height, (int64_t)py * width + px, d_rgb, d_depth, d_alpha, st_cd,
               st_t, st_tlast, st_last);
        b.init(px < width && py + 1 < height, (int64_t)(py + 1) * width + px, d_rgb, d_depth, d_alpha,
               st_cd, st_t, st_tlast, st_last);
        pp.init(a, b);
    }
    int wmax = max(pp.last0, pp.last1);
    if (threadIdx.x == 0) s_maxlast = -1;
    __syncthreads();
#pragma unroll
    for (int o = 16; o; o >>= 1) wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
    if (lane == 0) atomicMax(&s_maxlast, wmax);
    __syncthreads();
    const int maxlast = s_maxlast;
    if (threadIdx.x == 0) {   // rank of the tile's last visited instance (grad_gather's horizon)
        tile_hor[tile] = maxlast >= start ? (int32_t)(uint32_t)(ikeys[maxlast] & rank_mask) : -1;
        if (maxlast >= start) atomicAdd(&ctr->reserved[2], (uint32_t)(maxlast - start + 1));
    }
    const int via = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);   // 0..7
    const int vib = 8 + ((lane >> 4) & 1);                                                // 8..9
    const int tile_x = tile % tiles_x, tile_y = tile / tiles_x;
    for (int bend = maxlast + 1; bend > start; bend -= NT) {
        const int bstart = max(start, bend - NT);
        const int idx = bstart + (int)threadIdx.x;
        if (idx < bend) {
            const uint32_t rk = (uint32_t)(ikeys[idx] & rank_mask);
            s_rank[threadIdx.x] = rk;
            const ProjRec r = recs[rk];
            s_rec[threadIdx.x] = r;
            s_anch[threadIdx.x] = stage_anchor(r, p64, order, rk);
        }
        for (int i = threadIdx.x; i < NW * NT * 10; i += NT) (&s_part[0][0][0])[i] = 0.f;
        __syncthreads();
        const int jtop = min(bend - 1, wmax) - bstart;
        for (int j = jtop; j >= 0; j--) {
            const ProjRec &g = s_rec[j];
            const int y0 = rec_y0(g), y1 = rec_y1(g);
            if (y1 < wy0 || y0 > wy0 + 3) continue;   // warp-uniform row cull
            const int k = bstart + j;
            const int x0 = rec_x0(g);
            // both rows at once; the same q <= 9 decisions as the forward
            // (q_within_cutoff: an fp32 q outside the error band decides alike)
            // pw from the corner expansion, both rows at once; hx, hy = C (x - u)
            const float cx = (float)(px - x0);
            const float2 cy = make_float2((float)(py - y0), (float)(py + 1 - y0));
            const float dx = cx + g.ox;   // offsets from the centre: the conic gradients' factors
            const float2 dy = add2(cy, f2s(g.oy));
            const float4 an = s_anch[j];
            const float2 hx = fma2(f2s(g.ib), cy, f2s(fmaf(g.ia, cx, an.y)));
            const float2 hy = fma2(f2s(g.ic), cy, f2s(fmaf(g.ib, cx, an.z)));
            const float2 pw = fma2(f2s(cx), add2(hx, f2s(an.y)), fma2(cy, add2(hy, f2s(an.z)), f2s(an.x)));
            const float eps = g.eps;
            const float2 d = sub2(pw, f2s(kPowCut));
            const bool col = (unsigned)(px - x0) <= (unsigned)(rec_x1(g) - x0);
            bool h0 = col && (unsigned)(py - y0) <= (unsigned)(y1 - y0) && k <= pp.last0;
            bool h1 = col && (unsigned)(py + 1 - y0) <= (unsigned)(y1 - y0) && k <= pp.last1;
            if ((h0 && fabsf(d.x) <= eps) || (h1 && fabsf(d.y) <= eps)) {   // rare: fp64 band
                h0 = h0 && q_within_cutoff(pw.x, eps, p64, order, s_rank[j], px, py);
                h1 = h1 && q_within_cutoff(pw.y, eps, p64, order, s_rank[j], px, py + 1);
            } else {
                h0 = h0 && d.x >= 0.f;
                h1 = h1 && d.y >= 0.f;
            }
            if (!__any_sync(0xffffffffu, h0 || h1)) continue;
            float v[16];
            pp.step(g, dx, dy, pw, hx, hy, h0, h1, k, v);
            const float2 s = transpose_reduce10(v, lane);
            if (!(lane & 3)) s_part[warp][j][via] = s.x;
            if (!(lane & 15)) s_part[warp][j][vib] = s.y;
        }
        __syncthreads();
        if (idx < bend) {   // warp-ordered sum -> the instance's emission slot
            const ProjRec &g = s_rec[threadIdx.x];
            const uint32_t rk = s_rank[threadIdx.x];
            uint32_t kept;   // the tile's index among the splat's kept tiles
            if (bbox_tiles(g) <= kEmitSmall) {
                const int tx0 = rec_x0(g) / kTile, ty0r = rec_y0(g) / kTile;
                const int bit = (tile_y - ty0r) * (rec_x1(g) / kTile - tx0 + 1) + tile_x - tx0;
                kept = (uint32_t)__popc(tmask_r[rk] & ((1u << bit) - 1u));
            } else {
                kept = RowSpan(g).kept_index(tile_x, tile_y);
            }
            const uint32_t slot = toff[rk] + kept;
            float acc[10];
#pragma unroll
            for (int k = 0; k < 10; k++) {
                float a = 0.f;
#pragma unroll
                for (int w = 0; w < NW; w++) a += s_part[w][threadIdx.x][k];
                acc[k] = a;
            }
            float4 *dst = reinterpret_cast<float4 *>(gbuf + (int64_t)slot * kG2dStride);
            dst[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
            dst[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
            dst[2] = make_float4(acc[8], acc[9], 0.f, 0.f);
        }
        __syncthreads();
    }
}

// Sum of a small splat's visited instance slots (an instance was visited iff
// its rank is <= its tile's horizon rank), walking the kept-tile mask in
// emission order: a culled tile only removes a zero term, so ellipse culling
// stays bit-exact.
__device__ __forceinline__ void sum_slots(const ProjRec &g, uint32_t mask, int64_t r, uint32_t o,
                                          const float *gbuf, const int32_t *tile_hor, int tiles_x,
                                          float (&acc)[10]) {
    const int tx0 = rec_x0(g) / kTile, ty0 = rec_y0(g) / kTile, ntx = rec_x1(g) / kTile - tx0 + 1;
    for (uint32_t m = mask; m; m &= m - 1, o++) {
        const int bit = __ffs(m) - 1;
        if (r > (int64_t)tile_hor[(ty0 + bit / ntx) * tiles_x + tx0 + bit % ntx]) continue;
        const float4 *src = reinterpret_cast<const float4 *>(gbuf + (int64_t)o * kG2dStride);
        const float4 a = src[0], b = src[1], cc = src[2];
        acc[0] += a.x, acc[1] += a.y, acc[2] += a.z, acc[3] += a.w;
        acc[4] += b.x, acc[5] += b.y, acc[6] += b.z, acc[7] += b.w;
        acc[8] += cc.x, acc[9] += cc.y;
    }
}

// Splats with more than kEmitSmall box tiles (queued at emission, rare): one
// block each, fixed-assignment partial sums + fixed-order tree -> g2d[rank].  Smaller splats
// are summed inline by project_bwd.  Both orders are fixed: deterministic.
__global__ void __launch_bounds__(256)
grad_gather_big(const ProjRec *__restrict__ recs, const uint32_t *__restrict__ toff,
                const sm_render_counters *ctr,
                const uint32_t *__restrict__ big, const float *__restrict__ gbuf,
                const int32_t *__restrict__ tile_hor, int tiles_x, float *__restrict__ g2d) {
    __shared__ BigRowTable tab;
    __shared__ float s_part[kBigThreads / 32][10];
    const uint32_t nbig = ctr->overflow ? 0u : ctr->reserved[1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int via = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    const int vib = 8 + ((lane >> 4) & 1);
    for (uint32_t bi = blockIdx.x; bi < nbig; bi += gridDim.x) {   // a block per big splat
        const int64_t r = big[bi];
        const RowSpan sp(recs[r]);
        const uint32_t o = toff[r];
        float v[16];
#pragma unroll
        for (int k = 0; k < 16; k++) v[k] = 0.f;
        uint32_t base = 0;
        // warp w takes box rows ty0 + w (mod 8), lane l the tiles t = l (mod 32):
        // fixed by the box, not by the kept spans (see sum_slots)
        for (int tyb = sp.ty0; tyb <= sp.ty1; tyb += kBigThreads) {
            base = fill_row_table(sp, tyb, base, tab);
            const int nrows = min(kBigThreads, sp.ty1 - tyb + 1);
            for (int i = warp; i < nrows; i += kBigThreads / 32) {
                const int c0 = tab.c0[i], c1 = tab.c1[i], row = (tyb + i) * tiles_x;
                const uint32_t src0 = o + tab.off[i] - (uint32_t)c0;
                for (int c = c0 + (((lane - row - c0) % 32) + 32) % 32; c <= c1; c += 32) {
                    if (r > (int64_t)tile_hor[row + c]) continue;
                    const float4 *src =
                        reinterpret_cast<const float4 *>(gbuf + (int64_t)(src0 + (uint32_t)c) * kG2dStride);
                    const float4 a = src[0], b = src[1], cc = src[2];
                    v[0] += a.x, v[1] += a.y, v[2] += a.z, v[3] += a.w;
                    v[4] += b.x, v[5] += b.y, v[6] += b.z, v[7] += b.w;
                    v[8] += cc.x, v[9] += cc.y;
                }
            }
        }
        const float2 s = transpose_reduce10(v, lane);   // fixed butterfly, then warps in order
        if (!(lane & 3)) s_part[warp][via] = s.x;
        if (!(lane & 15)) s_part[warp][vib] = s.y;
        __syncthreads();
        if (threadIdx.x < 10) {
            float a = 0.f;
#pragma unroll
            for (int w = 0; w < kBigThreads / 32; w++) a += s_part[w][threadIdx.x];
            g2d[r * kG2dStride + threadIdx.x] = a;
        }
        __syncthreads();
    }
}

struct CamBwd {
    double r[9];
    double t[3];
    double fx, fy, cx, cy;
};

// K6: per depth rank, chain the 2D grads through the fp64 projection and
// accumulate the 14 parameter grads into the slot-indexed grad records.
// Two launches on two branches of the stream: small splats (their instance
// slots summed inline) run while grad_gather_big sums the big ones, which a
// second, small launch over the big-splat queue then finishes.  Each splat's
// grads are written by exactly one of them: identical results.
#ifndef SM_PBWD_MINB
#define SM_PBWD_MINB 3   // 3 x 256 threads per SM (<= 85 registers): measured best of 1-3
#endif
template <bool FUSED>
__device__ __forceinline__ void project_bwd_rank(int64_t r, const float (&gk)[10], float4 *params,
                                                 const int32_t *slots, const CamBwd &cam,
                                                 const uint32_t *order, float *grads, const AdamFuse &af);

// Adam of a splat the view does not reach (zero gradient: its moments still
// decay and move it, exactly as the standalone K7 over the active set does).
__device__ __forceinline__ void adam_zero_grad(int64_t slot, float4 *params, const AdamFuse &af) {
    float4 p[4];
#pragma unroll
    for (int q = 0; q < 4; q++) p[q] = params[slot * 4 + q];
    const float g[14] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    adam_record(p, af.m + slot * 4, af.v + slot * 4, g, af.c, adam_pre(af.m + slot * 4, af.c));
#pragma unroll
    for (int q = 0; q < 4; q++) params[slot * 4 + q] = p[q];
}

template <bool FUSED>
__global__ void __launch_bounds__(256, SM_PBWD_MINB)
project_bwd_small(float4 *__restrict__ params, const int32_t *__restrict__ slots, int64_t n,
                  CamBwd cam, const uint32_t *__restrict__ order, const uint32_t *__restrict__ tcount_r,
                  const uint32_t *__restrict__ tmask_r, const ProjRec *__restrict__ recs,
                  const uint32_t *__restrict__ toff, const float *__restrict__ gbuf,
                  const int32_t *__restrict__ tile_hor, int tiles_x, float *__restrict__ grads, AdamFuse af) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    if (FUSED && af.skip && *af.skip) return;   // overflowed forward: no update
    const uint32_t cnt = tcount_r[r];
    if (cnt == 0) {   // culled by the near plane or reaching no tile
        if (FUSED) {
            const uint32_t i = order[r];
            adam_zero_grad(slots ? (int64_t)slots[i] : (int64_t)i, params, af);
        }
        return;
    }
    const ProjRec rec = recs[r];
    if (bbox_tiles(rec) > kEmitSmall) return;   // project_bwd_big
    float gk[10];
#pragma unroll
    for (int k = 0; k < 10; k++) gk[k] = 0.f;
    sum_slots(rec, tmask_r[r], r, toff[r], gbuf, tile_hor, tiles_x, gk);
    project_bwd_rank<FUSED>(r, gk, params, slots, cam, order, grads, af);
}

template <bool FUSED>
__global__ void __launch_bounds__(64)
project_bwd_big(float4 *__restrict__ params, const int32_t *__restrict__ slots, CamBwd cam,
                const uint32_t *__restrict__ order, const sm_render_counters *ctr,
                const uint32_t *__restrict__ big, const float *__restrict__ g2d, float *__restrict__ grads,
                AdamFuse af) {
    const uint32_t nbig = ctr->overflow ? 0u : ctr->reserved[1];
    if (FUSED && af.skip && *af.skip) return;
    for (uint32_t bi = blockIdx.x * blockDim.x + threadIdx.x; bi < nbig; bi += gridDim.x * blockDim.x) {
        const int64_t r = big[bi];
        float gk[10];
#pragma unroll
        for (int k = 0; k < 10; k++) gk[k] = g2d[r * kG2dStride + k];
        project_bwd_rank<FUSED>(r, gk, params, slots, cam, order, grads, af);
    }
}

template <bool FUSED>
__device__ __forceinline__ void project_bwd_rank(int64_t r, const float (&gk)[10], float4 *params,
                                                 const int32_t *slots, const CamBwd &cam,
                                                 const uint32_t *order, float *grads, const AdamFuse &af) {
    const uint32_t i = order[r];
    const int64_t slot = slots ? (int64_t)slots[i] : (int64_t)i;
    AdamPre pre;
    if (FUSED) pre = adam_pre(af.m + slot * 4, af.c);   // before the chain rule's register peak
    const float4 A = params[slot * 4 + 0];
    const float4 B = params[slot * 4 + 1];
    const float4 C = params[slot * 4 + 2];
    const float4 D = params[slot * 4 + 3];
    const double gu = gk[0], gv = gk[1], gia = gk[2], gib = gk[3], gic = gk[4], gop = gk[5];
    const double gcol[3] = {gk[6], gk[7], gk[8]};
    const double gdep = gk[9];
    ProjGeom g;
    const double qw = A.w, qx = B.x, qy = B.y, qz = B.z;
    const double s[3] = {B.w, C.x, C.y};
    project_geometry<false>(A.x, A.y, A.z, qw, qx, qy, qz, s[0], s[1], s[2], cam.r, cam.t, cam.fx, cam.fy,
                     cam.cx, cam.cy, g);
    const double fx = cam.fx, fy = cam.fy;
    const double x = g.x, y = g.y, z = g.z;
    // colour
    const double sh[3] = {C.w, D.x, D.y};
    double gsh[3];
#pragma unroll
    for (int k = 0; k < 3; k++) {
        const double raw = SM_SH_C0 * sh[k] + 0.5;
        gsh[k] = (raw >= 0.0 && raw <= 1.0) ? SM_SH_C0 * gcol[k] : 0.0;
    }
    // conic -> (a, b, c)
    const double a = g.a, b = g.b, c = g.c;
    const double det = a * c - b * b, d2 = det * det;
    const double ga_ = gia * (-c * c / d2) + gib * (b * c / d2) + gic * (-b * b / d2);
    const double gb_ = gia * (2.0 * b * c / d2) + gib * (-1.0 / det - 2.0 * b * b / d2) +
                       gic * (2.0 * a * b / d2);
    const double gc_ = gia * (-b * b / d2) + gib * (a * b / d2) + gic * (-a * a / d2);
    const double G2[4] = {ga_, 0.5 * gb_, 0.5 * gb_, gc_};
    const double J[6] = {fx / z, 0.0, -fx * x / (z * z), 0.0, fy / z, -fy * y / (z * z)};
    const double Sc[9] = {g.Sc[0], g.Sc[1], g.Sc[2], g.Sc[1], g.Sc[3], g.Sc[4], g.Sc[2], g.Sc[4], g.Sc[5]};
    double G2J[6];
#pragma unroll
    for (int i2 = 0; i2 < 2; i2++)
#pragma unroll
        for (int j = 0; j < 3; j++) G2J[i2 * 3 + j] = G2[i2 * 2 + 0] * J[j] + G2[i2 * 2 + 1] * J[3 + j];
    double gSc[9];
#pragma unroll
    for (int rr = 0; rr < 3; rr++)
#pragma unroll
        for (int cc = 0; cc < 3; cc++) gSc[rr * 3 + cc] = J[rr] * G2J[cc] + J[3 + rr] * G2J[3 + cc];
    double gJ[6];
#pragma unroll
    for (int i2 = 0; i2 < 2; i2++)
#pragma unroll
        for (int j = 0; j < 3; j++)
            gJ[i2 * 3 + j] = 2.0 * (G2J[i2 * 3 + 0] * Sc[j] + G2J[i2 * 3 + 1] * Sc[3 + j] +
                                    G2J[i2 * 3 + 2] * Sc[6 + j]);
    double gx = gu * fx / z, gy = gv * fy / z;
    double gz = gu * (-fx * x / (z * z)) + gv * (-fy * y / (z * z)) + gdep;
    gz += gJ[0] * (-fx / (z * z));
    gx += gJ[2] * (-fx / (z * z));
    gz += gJ[2] * (2.0 * fx * x / (z * z * z));
    gz += gJ[4] * (-fy / (z * z));
    gy += gJ[5] * (-fy / (z * z));
    gz += gJ[5] * (2.0 * fy * y / (z * z * z));
    const double *rw = cam.r;
    double gpos[3];
#pragma unroll
    for (int k = 0; k < 3; k++) gpos[k] = rw[k * 3 + 0] * gx + rw[k * 3 + 1] * gy + rw[k * 3 + 2] * gz;
    // gSw = r_wc gSc r_wc^T
    double T1[9], gSw[9];
#pragma unroll
    for (int i2 = 0; i2 < 3; i2++)
#pragma unroll
        for (int j = 0; j < 3; j++)
            T1[i2 * 3 + j] = rw[i2 * 3 + 0] * gSc[0 * 3 + j] + rw[i2 * 3 + 1] * gSc[1 * 3 + j] +
                             rw[i2 * 3 + 2] * gSc[2 * 3 + j];
#pragma unroll
    for (int i2 = 0; i2 < 3; i2++)
#pragma unroll
        for (int j = 0; j < 3; j++)
            gSw[i2 * 3 + j] = T1[i2 * 3 + 0] * rw[j * 3 + 0] + T1[i2 * 3 + 1] * rw[j * 3 + 1] +
                              T1[i2 * 3 + 2] * rw[j * 3 + 2];
    const double *R = g.R;
    double gR[9], gsc[3];
#pragma unroll
    for (int k2 = 0; k2 < 3; k2++) {
        double acc = 0.0;
#pragma unroll
        for (int rr = 0; rr < 3; rr++) {
            double col = gSw[rr * 3 + 0] * R[0 * 3 + k2] + gSw[rr * 3 + 1] * R[1 * 3 + k2] +
                         gSw[rr * 3 + 2] * R[2 * 3 + k2];
            gR[rr * 3 + k2] = 2.0 * col * g.s2[k2];
            acc += R[rr * 3 + k2] * col;
        }
        gsc[k2] = 2.0 * s[k2] * acc;
    }
    const double gw = 2.0 * (-qz * gR[1] + qy * gR[2] + qz * gR[3] - qx * gR[5] - qy * gR[6] + qx * gR[7]);
    const double gqx = 2.0 * (qy * gR[1] + qz * gR[2] + qy * gR[3] - 2.0 * qx * gR[4] - qw * gR[5] +
                              qz * gR[6] + qw * gR[7] - 2.0 * qx * gR[8]);
    const double gqy = 2.0 * (-2.0 * qy * gR[0] + qx * gR[1] + qw * gR[2] + qx * gR[3] + qz * gR[5] -
                              qw * gR[6] + qz * gR[7] - 2.0 * qy * gR[8]);
    const double gqz = 2.0 * (-2.0 * qz * gR[0] - qw * gR[1] + qx * gR[2] + qw * gR[3] -
                              2.0 * qz * gR[4] + qy * gR[5] + qx * gR[6] + qy * gR[7]);
    if (FUSED) {   // fused Adam (single-keyframe step): the gradient never leaves registers
        const float g[14] = {(float)gpos[0], (float)gpos[1], (float)gpos[2], (float)gw, (float)gqx, (float)gqy,
                             (float)gqz, (float)gsc[0], (float)gsc[1], (float)gsc[2], (float)gop,
                             (float)gsh[0], (float)gsh[1], (float)gsh[2]};
        // keep the moment loads below the chain rule (register pressure)
        asm volatile("" ::: "memory");
        float4 p[4] = {params[slot * 4 + 0], params[slot * 4 + 1], params[slot * 4 + 2], params[slot * 4 + 3]};
        adam_record(p, af.m + slot * 4, af.v + slot * 4, g, af.c, pre);
#pragma unroll
        for (int q = 0; q < 4; q++) params[slot * 4 + q] = p[q];
        return;
    }
    float4 *dst = reinterpret_cast<float4 *>(grads) + slot * 4;
    float4 o0 = dst[0], o1 = dst[1], o2 = dst[2], o3 = dst[3];
    o0.x += (float)gpos[0];
    o0.y += (float)gpos[1];
    o0.z += (float)gpos[2];
    o0.w += (float)gw;
    o1.x += (float)gqx;
    o1.y += (float)gqy;
    o1.z += (float)gqz;
    o1.w += (float)gsc[0];
    o2.x += (float)gsc[1];
    o2.y += (float)gsc[2];
    o2.z += (float)gop;
    o2.w += (float)gsh[0];
    o3.x += (float)gsh[1];
    o3.y += (float)gsh[2];
    dst[0] = o0;
    dst[1] = o1;
    dst[2] = o2;
    dst[3] = o3;
}

template <typename KeyT>
static void launch_composite_bwd(const RenderBufs &b, const RenderLayout &L, const sm_render_dims &dims,
                                 const float *d_rgb, const float *d_depth, const float *d_alpha,
                                 cudaStream_t st) {
    const KeyT rank_mask = (KeyT)((1ull << L.rank_bits) - 1ull);
    const KeyT *ik = static_cast<const KeyT *>(L.tile_passes & 1 ? b.ikey1 : b.ikey0);
    composite_bwd<KeyT><<<(unsigned)L.n_tiles, kBwdThreads, 0, st>>>(
        b.ranges, ik, rank_mask, b.rec_sorted, b.p64, b.order0, dims.width, dims.height, L.tiles_x, d_rgb,
        d_depth, d_alpha, b.pix_cd, b.pix_t, b.pix_tlast, b.pix_last, b.toff, b.tmask_r, b.gbuf, b.tile_hor,
        b.ctr, b.tile_order);
}

int render_backward(const float *params, const int32_t *slots, int64_t n, const sm_camera &cam,
                    const sm_render_dims &dims, void *ws, int64_t ws_bytes, const float *d_rgb,
                    const float *d_depth, const float *d_alpha, float *grads, const AdamFuse *fuse,
                    cudaStream_t st) {
    const RenderLayout L = render_layout(dims);
    if (ws_bytes < L.total) {
        set_error("render workspace too small: %lld < %lld", (long long)ws_bytes, (long long)L.total);
        return SM_ERR_WORKSPACE;
    }
    if (n < 0 || n > dims.max_gaussians) {
        set_error("n=%lld outside [0, max_gaussians]", (long long)n);
        return SM_ERR_INVALID;
    }
    if (cam.width != dims.width || cam.height != dims.height) {
        set_error("camera does not match workspace");
        return SM_ERR_DIMENSION;
    }
    if (n == 0) return SM_OK;
    RenderBufs b = render_bufs(ws, L);
    AdamFuse af{};
    if (fuse) af = *fuse;
    float4 *pw = reinterpret_cast<float4 *>(const_cast<float *>(params));   // written only when fused
    prof_begin(ST_COMPOSITE_BWD, st);
    if (L.key_bytes == 8)
        launch_composite_bwd<unsigned long long>(b, L, dims, d_rgb, d_depth, d_alpha, st);
    else
        launch_composite_bwd<uint32_t>(b, L, dims, d_rgb, d_depth, d_alpha, st);
    prof_end(ST_COMPOSITE_BWD, st);
    CamBwd cb;
    for (int k = 0; k < 9; k++) cb.r[k] = cam.r_wc[k];
    for (int k = 0; k < 3; k++) cb.t[k] = cam.t[k];
    cb.fx = cam.fx;
    cb.fy = cam.fy;
    cb.cx = cam.cx;
    cb.cy = cam.cy;
    // big splats on a forked branch (b.tcount holds the big-splat queue)
#ifndef SM_FORK
#define SM_FORK 1   // 0: one branch (A/B timing of the two launches)
#endif
    StreamFork &fk = stream_fork();
    if (SM_FORK) fk.begin(st);
    cudaStream_t side = SM_FORK ? fk.side : st;
    prof_begin(ST_GRAD_GATHER, side);
    grad_gather_big<<<148 * 4, 256, 0, side>>>(b.rec_sorted, b.toff, b.ctr, b.tcount, b.gbuf,
                                                   b.tile_hor, L.tiles_x, b.g2d);
    if (fuse)
        project_bwd_big<true><<<148, 64, 0, side>>>(pw, slots, cb, b.order0, b.ctr, b.tcount, b.g2d, grads, af);
    else
        project_bwd_big<false><<<148, 64, 0, side>>>(pw, slots, cb, b.order0, b.ctr, b.tcount, b.g2d, grads, af);
    prof_end(ST_GRAD_GATHER, side);
    prof_begin(ST_PROJECT_BWD, st);
    if (fuse)
        project_bwd_small<true><<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(
            pw, slots, n, cb, b.order0, b.tcount_r, b.tmask_r, b.rec_sorted, b.toff, b.gbuf, b.tile_hor,
            L.tiles_x, grads, af);
    else
        project_bwd_small<false><<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(
            pw, slots, n, cb, b.order0, b.tcount_r, b.tmask_r, b.rec_sorted, b.toff, b.gbuf, b.tile_hor,
            L.tiles_x, grads, af);
    prof_end(ST_PROJECT_BWD, st);
    if (SM_FORK) fk.end(st);
    count_launches(4);
    SM_CHECK_LAUNCH("render_backward");
    return SM_OK;
}

}  // namespace sm
