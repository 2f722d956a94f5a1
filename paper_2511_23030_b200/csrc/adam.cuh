// K7 Adam arithmetic shared by the standalone kernel (store_kernels.cu) and
// the backward-fused form (render_bwd.cu): per-Gaussian step count, one
// rounding per operation (no FMA contraction), so every path that applies an
// Adam step to a record produces the same bits (the DP packed path, the
// fused single-keyframe path and the standalone kernel are interchangeable).
// Replaces the reference's projected-residual nudge (sim.py:280-317); the
// invariants it restores are the store's (core.py:186-190).
#pragma once
#include "common.cuh"

namespace sm {

struct AdamDev {
    float lr[14];
    float b1, b2, eps, min_scale;
};

inline AdamDev adam_dev(const sm_adam_config &cfg) {
    AdamDev d;
    for (int k = 0; k < 14; k++) d.lr[k] = cfg.lr[k];
    d.b1 = cfg.beta1;
    d.b2 = cfg.beta2;
    d.eps = cfg.eps;
    d.min_scale = cfg.min_scale;
    return d;
}

// Bias corrections of step `step` (IEEE powf / div / sqrt: 1 - 0.999^t
// cancels, keep them exact): 1 / (1 - b1^t) and 1 / sqrt(1 - b2^t).
__device__ __forceinline__ void adam_bias(const AdamDev &c, float step, float &ibc1, float &ibc2s) {
    ibc1 = 1.f / (1.f - powf(c.b1, step));
    ibc2s = 1.f / sqrtf(1.f - powf(c.b2, step));
}

// One scalar: m, v updated in place; returns the new parameter.  Approximate
// sqrt / reciprocal (relative ~3e-7 of the update; oracle tolerance 1e-6).
__device__ __forceinline__ float adam_elem(float p, float &m, float &v, float g, float lr, float ibc1,
                                           float ibc2s, const AdamDev &c) {
    m = __fadd_rn(__fmul_rn(c.b1, m), __fmul_rn(__fsub_rn(1.f, c.b1), g));
    v = __fadd_rn(__fmul_rn(c.b2, v), __fmul_rn(__fmul_rn(__fsub_rn(1.f, c.b2), g), g));
    const float den = __fadd_rn(__fmul_rn(sqrt_approx(v), ibc2s), c.eps);
    return __fsub_rn(p, __fmul_rn(__fmul_rn(__fmul_rn(lr, ibc1), m), rcp_approx(den)));
}

// |q|^2 split as qw^2 + (qx^2 + qy^2 + qz^2) (the quarter kernel holds qw and
// qx..qz in different threads); the inverse norm, 0 for a zero quaternion.
__device__ __forceinline__ float quat_xyz2(float qx, float qy, float qz) {
    return __fadd_rn(__fadd_rn(__fmul_rn(qx, qx), __fmul_rn(qy, qy)), __fmul_rn(qz, qz));
}

// Adam on a whole 16-float record (one thread): p / m / v are the record's
// four float4 quarters; m[3].z carries the per-Gaussian step count.
__device__ __forceinline__ void adam_record(float4 (&p)[4], float4 (&m)[4], float4 (&v)[4], const float (&g)[14],
                                            const AdamDev &c) {
    float pv[16], mv[16], vv[16];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        pv[4 * q] = p[q].x, pv[4 * q + 1] = p[q].y, pv[4 * q + 2] = p[q].z, pv[4 * q + 3] = p[q].w;
        mv[4 * q] = m[q].x, mv[4 * q + 1] = m[q].y, mv[4 * q + 2] = m[q].z, mv[4 * q + 3] = m[q].w;
        vv[4 * q] = v[q].x, vv[4 * q + 1] = v[q].y, vv[4 * q + 2] = v[q].z, vv[4 * q + 3] = v[q].w;
    }
    const float step = mv[14] + 1.f;
    float ibc1, ibc2s;
    adam_bias(c, step, ibc1, ibc2s);
#pragma unroll
    for (int k = 0; k < 14; k++) pv[k] = adam_elem(pv[k], mv[k], vv[k], g[k], c.lr[k], ibc1, ibc2s, c);
    mv[14] = step;
    const float qn = __fsqrt_rn(__fadd_rn(__fmul_rn(pv[3], pv[3]), quat_xyz2(pv[4], pv[5], pv[6])));
    pv[3] = qn > 0.f ? __fmul_rn(pv[3], 1.f / qn) : 1.f;
    const float inv = qn > 0.f ? 1.f / qn : 0.f;
    pv[4] = __fmul_rn(pv[4], inv), pv[5] = __fmul_rn(pv[5], inv), pv[6] = __fmul_rn(pv[6], inv);
    pv[7] = fmaxf(pv[7], c.min_scale), pv[8] = fmaxf(pv[8], c.min_scale), pv[9] = fmaxf(pv[9], c.min_scale);
    pv[10] = fminf(fmaxf(pv[10], 0.f), 1.f);
#pragma unroll
    for (int q = 0; q < 4; q++) {
        p[q] = make_float4(pv[4 * q], pv[4 * q + 1], pv[4 * q + 2], pv[4 * q + 3]);
        m[q] = make_float4(mv[4 * q], mv[4 * q + 1], mv[4 * q + 2], mv[4 * q + 3]);
        v[q] = make_float4(vv[4 * q], vv[4 * q + 1], vv[4 * q + 2], vv[4 * q + 3]);
    }
}

// The backward-fused Adam (single-keyframe mapping step): project_bwd applies
// the step to each splat right after its chain rule, instead of writing the
// gradient record for a separate pass.  m == nullptr: accumulate gradients.
struct AdamFuse {
    float4 *m, *v;
    const uint32_t *skip;   // non-zero: the forward overflowed, no update
    AdamDev c;
};

}  // namespace sm
