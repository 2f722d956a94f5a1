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
// dx for pixel px is (px - x0) + ox with ox = x0 - u computed in fp64, so
// the fp32 offset keeps ~1e-7 relative precision whatever |u| is.
struct __align__(16) ProjRec {
    float ox, oy;          // x0 - u, y0 - v
    float ia, ib, ic;      // conic (c, -b, a)/det
    float op;              // opacity
    float r, g, b;         // clipped SH0 colour
    float z;               // camera depth
    float eps;             // |q32 - 9| band that triggers the fp64 decision
    int32_t x0y0;          // (y0 << 16) | x0   clamped 3-sigma bbox
    int32_t x1y1;          // (y1 << 16) | x1
    float spare[3];
};
static_assert(sizeof(ProjRec) == 64, "ProjRec must be 64 bytes");

// fp64 side copy for decisions near the q = 9 cutoff (hard part 1)
struct Proj64 {
    double u, v, ia, ib, ic;
};

__device__ __forceinline__ int rec_x0(const ProjRec &r) { return (int)(short)(r.x0y0 & 0xffff); }
__device__ __forceinline__ int rec_y0(const ProjRec &r) { return r.x0y0 >> 16; }
__device__ __forceinline__ int rec_x1(const ProjRec &r) { return (int)(short)(r.x1y1 & 0xffff); }
__device__ __forceinline__ int rec_y1(const ProjRec &r) { return r.x1y1 >> 16; }

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

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t align_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

}  // namespace sm
