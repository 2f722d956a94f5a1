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

// Adam on a whole 16-float record by one thread, streamed quarter by
// quarter (only one m / v quarter live at a time: the fused backward has
// little register room left): p holds the record (updated in place), the
// moments are read and written at m_rec / v_rec; m quarter 3 .z carries the
// per-Gaussian step count.  Same operations, same order as the quarter kernel.
// `m3` = m_rec[3] and the bias corrections of step m3.z + 1, prepared by the
// caller (the fused backward does it before its chain rule, so powf's
// registers are free again at its peak).
struct AdamPre {
    float4 m3;
    float step, ibc1, ibc2s;
};

__device__ __forceinline__ AdamPre adam_pre(const float4 *m_rec, const AdamDev &c) {
    AdamPre a;
    a.m3 = m_rec[3];
    a.step = a.m3.z + 1.f;
    adam_bias(c, a.step, a.ibc1, a.ibc2s);
    return a;
}

__device__ __forceinline__ void adam_record(float4 (&p)[4], float4 *m_rec, float4 *v_rec, const float (&g)[14],
                                            const AdamDev &c, const AdamPre &pre) {
    float4 m3 = pre.m3;
    const float step = pre.step, ibc1 = pre.ibc1, ibc2s = pre.ibc2s;
    float4 m = m_rec[0], v = v_rec[0];
    p[0].x = adam_elem(p[0].x, m.x, v.x, g[0], c.lr[0], ibc1, ibc2s, c);
    p[0].y = adam_elem(p[0].y, m.y, v.y, g[1], c.lr[1], ibc1, ibc2s, c);
    p[0].z = adam_elem(p[0].z, m.z, v.z, g[2], c.lr[2], ibc1, ibc2s, c);
    p[0].w = adam_elem(p[0].w, m.w, v.w, g[3], c.lr[3], ibc1, ibc2s, c);
    m_rec[0] = m, v_rec[0] = v;
    m = m_rec[1], v = v_rec[1];
    p[1].x = adam_elem(p[1].x, m.x, v.x, g[4], c.lr[4], ibc1, ibc2s, c);
    p[1].y = adam_elem(p[1].y, m.y, v.y, g[5], c.lr[5], ibc1, ibc2s, c);
    p[1].z = adam_elem(p[1].z, m.z, v.z, g[6], c.lr[6], ibc1, ibc2s, c);
    p[1].w = adam_elem(p[1].w, m.w, v.w, g[7], c.lr[7], ibc1, ibc2s, c);
    m_rec[1] = m, v_rec[1] = v;
    m = m_rec[2], v = v_rec[2];
    p[2].x = adam_elem(p[2].x, m.x, v.x, g[8], c.lr[8], ibc1, ibc2s, c);
    p[2].y = adam_elem(p[2].y, m.y, v.y, g[9], c.lr[9], ibc1, ibc2s, c);
    p[2].z = adam_elem(p[2].z, m.z, v.z, g[10], c.lr[10], ibc1, ibc2s, c);
    p[2].w = adam_elem(p[2].w, m.w, v.w, g[11], c.lr[11], ibc1, ibc2s, c);
    m_rec[2] = m, v_rec[2] = v;
    v = v_rec[3];
    p[3].x = adam_elem(p[3].x, m3.x, v.x, g[12], c.lr[12], ibc1, ibc2s, c);
    p[3].y = adam_elem(p[3].y, m3.y, v.y, g[13], c.lr[13], ibc1, ibc2s, c);
    m3.z = step;
    m_rec[3] = m3, v_rec[3] = v;
    // quaternion renormalisation, scale floor, opacity clamp (core.py:186-190)
    const float qn = __fsqrt_rn(__fadd_rn(__fmul_rn(p[0].w, p[0].w), quat_xyz2(p[1].x, p[1].y, p[1].z)));
    p[0].w = qn > 0.f ? __fmul_rn(p[0].w, 1.f / qn) : 1.f;
    const float inv = qn > 0.f ? 1.f / qn : 0.f;
    p[1].x = __fmul_rn(p[1].x, inv), p[1].y = __fmul_rn(p[1].y, inv), p[1].z = __fmul_rn(p[1].z, inv);
    p[1].w = fmaxf(p[1].w, c.min_scale), p[2].x = fmaxf(p[2].x, c.min_scale), p[2].y = fmaxf(p[2].y, c.min_scale);
    p[2].z = fminf(fmaxf(p[2].z, 0.f), 1.f);
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
