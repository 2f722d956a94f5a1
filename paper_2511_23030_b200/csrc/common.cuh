// Shared device helpers for libsplatmap_cuda (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/splatmap_cuda.h"

#define SM_SH_C0 0.28209479177       // core.py:40
#define SM_MIN_T 1e-10               // renderloss.py:26

namespace sm {

void set_error(const char *fmt, ...);
int cuda_status(cudaError_t e, const char *what);

#define SM_CHECK_LAUNCH(what)                                   \
    do {                                                        \
        cudaError_t _e = cudaGetLastError();                    \
        if (_e != cudaSuccess) return ::sm::cuda_status(_e, what); \
    } while (0)

constexpr int kTile = SM_TILE;             // 16x16 pixel tiles
constexpr int kTilePx = kTile * kTile;     // 256 threads per tile CTA

// 64-byte per-Gaussian screen-space record, produced by the projection
// (renderloss.py:176-201) and consumed by compositing (renderloss.py:106-152).
// Compositing evaluates the quadratic form expanded around the box corner
// (x0, y0): qa and (hax, hay) = the form and half its gradient there
// (stage_anchor, when a tile stages the splat) and pw = qa + cx (hx + hax) +
// cy (hy + hay), (cx, cy) = the pixel's integer offset from the corner,
// (hx, hy) = C (x - u).  No fp32 term carries the centre offset: a splat next
// to the near plane has its centre ~1e5 px off screen, and the direct form
// dx (ia dx + 2 ib dy) + ic dy^2 with dx = (px - x0) + ox lost ~1e-3 of q to
// cancellation there (a full-size C4 view's opacity gradients were 1.8e-3
// off; ~3e-7 with the expansion).  ox = x0 - u (fp64-rounded) feeds the
// binning's row spans, the backward's conic gradients (products, no
// cancellation) and the anchors of ordinary splats.
struct __align__(16) ProjRec {
    float ox, oy;          // x0 - u, y0 - v
    float ia, ib, ic;      // conic (c, -b, a)/det pre-scaled by kPowScale (log2 units)
    float op;              // opacity
    float r, g, b;         // clipped SH0 colour
    float z;               // camera depth
    float eps;             // |pw - kPowCut| band that triggers the fp64 decision
    int32_t x0y0;          // (y0 << 16) | x0   clamped 3-sigma bbox
    int32_t x1y1;          // (y1 << 16) | x1
    float beta, G, K;      // ellipse row extent (RowSpan); K <= 0: whole bbox rows
};
static_assert(sizeof(ProjRec) == 64, "ProjRec must be 64 bytes");
constexpr double kAnchorPx = 64.0;

// fp64 side copy for decisions near the q = 9 cutoff (hard part 1)
struct Proj64 {
    double u, v, ia, ib, ic;
};

__device__ __forceinline__ int rec_x0(const ProjRec &r) { return (int)(short)(r.x0y0 & 0xffff); }
__device__ __forceinline__ int rec_y0(const ProjRec &r) { return r.x0y0 >> 16; }
__device__ __forceinline__ int rec_x1(const ProjRec &r) { return (int)(short)(r.x1y1 & 0xffff); }
__device__ __forceinline__ int rec_y1(const ProjRec &r) { return r.x1y1 >> 16; }

// Tile columns [c0, c1] of tile row ty that the splat's q <= 9 ellipse can
// reach (c0 > c1: none).  At row offset dy the ellipse spans
// |dx - beta dy| <= sqrt(G - K dy^2) (beta = b/c, G = 9 det/c, K = det/c^2 of
// the dilated cov2), so over the row band [a0, a1] of pixel-row offsets the
// extreme dx sit at dy = +-beta sqrt(G/K / (K + beta^2)) (= +-3b/sqrt(a), the
// ellipse's side points) clamped into the band.  Widened by 1% of the radius +
// 0.02 px, far above the fp32 evaluation error, so no pixel with q <= 9 is
// ever dropped: the culled tiles are exactly ones the compositor would skip.
// Projection (counts), emission, composite_bwd (slot index) and the gradient
// gather all call this one function, so they agree tile for tile.
struct RowSpan {
    int x0, y0, y1, tx0, tx1, ty0, ty1;
    float beta, G, K, dys, rad, xo, oy;
    bool ell;

    __device__ __forceinline__ explicit RowSpan(const ProjRec &g) {
        x0 = rec_x0(g);
        y0 = rec_y0(g);
        y1 = rec_y1(g);
        tx0 = x0 / SM_TILE;
        tx1 = rec_x1(g) / SM_TILE;
        ty0 = y0 / SM_TILE;
        ty1 = y1 / SM_TILE;
        beta = g.beta;
        G = g.G;
        K = g.K;
        ell = K > 0.f;
        // explicit _rn ops: no FMA contraction, so every kernel inlining this
        // computes the same bits
        dys = ell ? __fmul_rn(beta, __fsqrt_rn(__fdiv_rn(__fdiv_rn(G, K), __fadd_rn(K, __fmul_rn(beta, beta)))))
                  : 0.f;
        rad = __fsqrt_rn(fmaxf(G, 0.f));
        xo = __fsub_rn((float)x0, g.ox);   // pixel column of dx = 0 (the splat's u)
        oy = g.oy;
    }

    __device__ __forceinline__ float half_width(float dy) const {
        return __fsqrt_rn(fmaxf(__fsub_rn(G, __fmul_rn(__fmul_rn(K, dy), dy)), 0.f));
    }

    __device__ __forceinline__ void row(int ty, int &c0, int &c1) const {
        c0 = tx0;
        c1 = tx1;
        if (!ell) return;
        const float a0 = __fadd_rn((float)(max(ty * SM_TILE, y0) - y0), oy);
        const float a1 = __fadd_rn((float)(min(ty * SM_TILE + SM_TILE - 1, y1) - y0), oy);
        const float dr = fminf(fmaxf(dys, a0), a1), dl = fminf(fmaxf(-dys, a0), a1);
        const float xr = __fadd_rn(__fmul_rn(beta, dr), half_width(dr));
        const float xl = __fsub_rn(__fmul_rn(beta, dl), half_width(dl));
        const float m = __fadd_rn(
            __fmul_rn(0.01f, __fadd_rn(rad, __fmul_rn(fabsf(beta), fmaxf(fabsf(a0), fabsf(a1))))), 0.02f);
        const float pl = __fsub_rn(__fadd_rn(xo, xl), m), pr = __fadd_rn(__fadd_rn(xo, xr), m);
        if (!(pl <= pr) || !(pr - pl < 1e7f)) return;   // NaN / inf guard: keep the whole row
        c0 = max(c0, (int)floorf(__fmul_rn(pl, 1.f / SM_TILE)));
        c1 = min(c1, (int)floorf(__fmul_rn(pr, 1.f / SM_TILE)));
    }

    __device__ __forceinline__ int count(int ty) const {
        int c0, c1;
        row(ty, c0, c1);
        return c1 >= c0 ? c1 - c0 + 1 : 0;
    }

    // Index of tile (tx, ty) among the kept tiles (row-major order).
    __device__ __forceinline__ uint32_t kept_index(int tx, int ty) const {
        uint32_t j = 0;
        for (int t = ty0; t < ty; t++) j += (uint32_t)count(t);
        int c0, c1;
        row(ty, c0, c1);
        return j + (uint32_t)(tx - c0);
    }
};

// Exact reference expression (renderloss.py:140) evaluated left to right in
// fp64 with explicit round-to-nearest ops so nvcc cannot contract to FMA.
__device__ __forceinline__ double quad_q64(const Proj64 &p, int px, int py) {
    double dx = __dsub_rn((double)px, p.u);
    double dy = __dsub_rn((double)py, p.v);
    double t1 = __dmul_rn(__dmul_rn(p.ia, dx), dx);
    double t2 = __dmul_rn(__dmul_rn(__dmul_rn(2.0, p.ib), dx), dy);
    double t3 = __dmul_rn(__dmul_rn(p.ic, dy), dy);
    return __dadd_rn(__dadd_rn(t1, t2), t3);
}

// alpha = op * exp(-q/2) = op * 2^(kPowScale * q): the conic is stored
// pre-multiplied by kPowScale so the quadratic form lands directly in the
// exponent of ex2; q > 9 (renderloss.py:141) <=> pw < kPowCut.
constexpr double kPowScale = -0.72134752044448170368;   // -0.5 * log2(e)
constexpr float kPowCut = (float)(9.0 * -0.72134752044448170368);

// The corner expansion's {qa, hax, hay} (see ProjRec).  For a splat whose
// corner lies within kAnchorPx of its centre, fp32 from (ox, oy) is as exact
// as the direct form was; beyond that (huge splats, rare) fp64 from the
// Proj64 side record with explicit roundings.  Both compositing kernels stage
// identical values.
__device__ __forceinline__ float4 anchor_of(const Proj64 &p, int x0, int y0) {
    const double dax = __dsub_rn((double)x0, p.u), day = __dsub_rn((double)y0, p.v);
    const double sia = __dmul_rn(kPowScale, p.ia), sib = __dmul_rn(kPowScale, p.ib);
    const double sic = __dmul_rn(kPowScale, p.ic);
    const double hax = __dadd_rn(__dmul_rn(sia, dax), __dmul_rn(sib, day));
    const double hay = __dadd_rn(__dmul_rn(sib, dax), __dmul_rn(sic, day));
    const double qa = __dadd_rn(__dmul_rn(dax, hax), __dmul_rn(day, hay));
    return make_float4((float)qa, (float)hax, (float)hay, 0.f);
}

__device__ __forceinline__ float4 stage_anchor(const ProjRec &r, const Proj64 *p64, const uint32_t *order,
                                              uint32_t rank) {
    if (fabsf(r.ox) > (float)kAnchorPx || fabsf(r.oy) > (float)kAnchorPx)
        return anchor_of(p64[order[rank]], rec_x0(r), rec_y0(r));
    const float hax = fmaf(r.ia, r.ox, r.ib * r.oy), hay = fmaf(r.ib, r.ox, r.ic * r.oy);
    return make_float4(fmaf(r.ox, hax, r.oy * hay), hax, hay, 0.f);
}

// Packed fp32x2 arithmetic (sm_100 FFMA2 / FMUL2 / FADD2): two pixels' math
// per issue slot in the compositing kernels.
__device__ __forceinline__ float2 f2s(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float hsum(float2 a) { return a.x + a.y; }

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// The q <= 9 decision (renderloss.py:141) both compositing kernels take for
// pixel (px, py) inside a splat's box: pw from the corner expansion in fp32
// (see ProjRec); when |pw - kPowCut| lies within the splat's error band eps
// the exact fp64 quad_q64 decides.  The
// forward and the backward evaluate pw in different (fp32 / packed fp32x2)
// orders; outside the band both equal the exact verdict, inside it both use
// quad_q64, so they always agree.
__device__ __forceinline__ bool q_within_cutoff(float pw, float eps, const Proj64 *p64,
                                                const uint32_t *order, uint32_t rank, int px, int py) {
    const float d = pw - kPowCut;
    return fabsf(d) <= eps ? !(quad_q64(p64[order[rank]], px, py) > 9.0) : d >= 0.f;
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ inline int64_t align_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

}  // namespace sm
