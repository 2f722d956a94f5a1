// K1 chunk culling + active-set expansion, K7 fused Adam, K8/K9 chunk codec,
// and the bit-exact chunk-id encoder.
#include <cmath>
#include <cstring>

#include "adam.cuh"
#include "common.cuh"
#include "prof.cuh"

namespace sm {

// ------------------------------------------------------------------ K7
// Four threads per Gaussian, one float4 quarter of each record each (so a
// warp streams 8 full 64-byte records per array with 16-byte accesses and a
// thread keeps ~30 registers instead of ~90).  Quarter q holds record scalars
// 4q..4q+3: q0 = px py pz qw, q1 = qx qy qz sx, q2 = sy sz op sh0r,
// q3 = sh0g sh0b - - (m.q3.z = per-Gaussian step count).  The quaternion
// spans q0.w and q1.xyz: its norm is exchanged with one shuffle.  The
// arithmetic is adam.cuh's (bit-identical to the backward-fused form).
__global__ void __launch_bounds__(256)
adam_quarter_kernel(float4 *__restrict__ params, float4 *__restrict__ m, float4 *__restrict__ v,
                    float4 *__restrict__ grads, const int32_t *__restrict__ slots, int64_t n,
                    AdamDev c, const uint32_t *__restrict__ skip, const float4 *__restrict__ packed) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int q = threadIdx.x & 3;
    const int64_t i = t >> 2;
    const bool ok = i < n && !(skip && *skip);
    const int64_t s = ok ? (slots ? (int64_t)slots[i] : i) : 0;
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f), g = p, mm = p, vv = p;
    if (ok) {
        p = params[s * 4 + q];
        g = packed ? packed[i * 4 + q] : grads[s * 4 + q];   // packed: the DP exchange buffer
        mm = m[s * 4 + q];
        vv = v[s * 4 + q];
    }
    // per-Gaussian step count lives in m quarter 3, component z
    const float step = __shfl_sync(0xffffffffu, mm.z, (threadIdx.x & 31) | 3) + 1.f;
    float ibc1, ibc2s;
    adam_bias(c, step, ibc1, ibc2s);
    float pv[4] = {p.x, p.y, p.z, p.w}, gv[4] = {g.x, g.y, g.z, g.w};
    float mv[4] = {mm.x, mm.y, mm.z, mm.w}, vvv[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int idx = 4 * q + k;
        if (idx < 14) pv[k] = adam_elem(pv[k], mv[k], vvv[k], gv[k], c.lr[idx], ibc1, ibc2s, c);
    }
    if (q == 3) mv[2] = step;
    // quaternion renormalisation (core.py:186 unit-norm invariant)
    const float part = q == 0 ? __fmul_rn(pv[3], pv[3]) : (q == 1 ? quat_xyz2(pv[0], pv[1], pv[2]) : 0.f);
    const float other = __shfl_xor_sync(0xffffffffu, part, 1);
    const float qn = __fsqrt_rn(q == 0 ? __fadd_rn(part, other) : __fadd_rn(other, part));
    if (q == 0) pv[3] = qn > 0.f ? __fmul_rn(pv[3], 1.f / qn) : 1.f;
    if (q == 1) {
        const float inv = qn > 0.f ? 1.f / qn : 0.f;
        pv[0] = __fmul_rn(pv[0], inv), pv[1] = __fmul_rn(pv[1], inv), pv[2] = __fmul_rn(pv[2], inv);
        pv[3] = fmaxf(pv[3], c.min_scale);   // sx
    }
    if (q == 2) {
        pv[0] = fmaxf(pv[0], c.min_scale);   // sy
        pv[1] = fmaxf(pv[1], c.min_scale);   // sz
        pv[2] = fminf(fmaxf(pv[2], 0.f), 1.f);   // opacity
    }
    if (!ok) return;
    params[s * 4 + q] = make_float4(pv[0], pv[1], pv[2], pv[3]);
    m[s * 4 + q] = make_float4(mv[0], mv[1], mv[2], mv[3]);
    v[s * 4 + q] = make_float4(vvv[0], vvv[1], vvv[2], vvv[3]);
    if (!packed) grads[s * 4 + q] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// The data-parallel exchange buffer: the active rows' gradient records packed
// in active-set order (packed[i] = grads[slots[i]]), the slab rows zeroed for
// the next accumulation.  One 16-byte quarter per thread.
__global__ void __launch_bounds__(256)
pack_grads_kernel(float4 *__restrict__ grads, const int32_t *__restrict__ slots, int64_t n,
                  float4 *__restrict__ packed) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t i = t >> 2;
    if (i >= n) return;
    const int q = (int)(t & 3);
    const int64_t s = slots ? (int64_t)slots[i] : i;
    packed[t] = grads[s * 4 + q];
    grads[s * 4 + q] = make_float4(0.f, 0.f, 0.f, 0.f);
}

int pack_grads(float *grads, const int32_t *slots, int64_t n, float *packed, cudaStream_t st) {
    if (n < 0) {
        set_error("negative n");
        return SM_ERR_INVALID;
    }
    if (n == 0) return SM_OK;
    count_launches(1);
    pack_grads_kernel<<<(unsigned)ceil_div(n * 4, 256), 256, 0, st>>>(
        reinterpret_cast<float4 *>(grads), slots, n, reinterpret_cast<float4 *>(packed));
    SM_CHECK_LAUNCH("pack_grads");
    return SM_OK;
}

int adam_step(float *params, float *m, float *v, float *grads, const int32_t *slots, int64_t n,
              const sm_adam_config &cfg, const uint32_t *skip, const float *packed, cudaStream_t st) {
    if (n < 0) {
        set_error("negative n");
        return SM_ERR_INVALID;
    }
    if (n == 0) return SM_OK;
    const AdamDev d = adam_dev(cfg);
    prof_begin(ST_ADAM, st);
    count_launches(1);
    adam_quarter_kernel<<<(unsigned)ceil_div(n * 4, 256), 256, 0, st>>>(
        reinterpret_cast<float4 *>(params), reinterpret_cast<float4 *>(m),
        reinterpret_cast<float4 *>(v), reinterpret_cast<float4 *>(grads), slots, n, d, skip,
        reinterpret_cast<const float4 *>(packed));
    prof_end(ST_ADAM, st);
    SM_CHECK_LAUNCH("adam_step");
    return SM_OK;
}

// ------------------------------------------------------ loop closure
// Rigid correction of a chunk's rows in place (loopclose.py:146-150 with
// core.py transform_gaussian + storage_canonical): p' = R p + t and
// q' = normalize(q_t * q) in fp64 from the stored float32 values, rounded
// back to float32; everything else (scale, opacity, SH, Adam state) is kept.
struct RigidDev {
    double r[9];   // R of the transform, row-major
    double t[3];
    double q[4];   // its quaternion (w, x, y, z)
};

__global__ void __launch_bounds__(256)
transform_rows_kernel(float4 *__restrict__ params, int64_t n, RigidDev c) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 A = params[4 * i], B = params[4 * i + 1];   // px py pz qw | qx qy qz sx
    const double p[3] = {A.x, A.y, A.z};
    double w[3];
#pragma unroll
    for (int a = 0; a < 3; a++)
        w[a] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(c.r[3 * a], p[0]), __dmul_rn(c.r[3 * a + 1], p[1])),
                                   __dmul_rn(c.r[3 * a + 2], p[2])),
                         c.t[a]);
    // Hamilton product q_t * q (core.py:76-87), then normalize
    const double aw = c.q[0], ax = c.q[1], ay = c.q[2], az = c.q[3];
    const double bw = A.w, bx = B.x, by = B.y, bz = B.z;
    double q[4];
    q[0] = __dsub_rn(__dsub_rn(__dsub_rn(__dmul_rn(aw, bw), __dmul_rn(ax, bx)), __dmul_rn(ay, by)), __dmul_rn(az, bz));
    q[1] = __dsub_rn(__dadd_rn(__dadd_rn(__dmul_rn(aw, bx), __dmul_rn(ax, bw)), __dmul_rn(ay, bz)), __dmul_rn(az, by));
    q[2] = __dadd_rn(__dadd_rn(__dsub_rn(__dmul_rn(aw, by), __dmul_rn(ax, bz)), __dmul_rn(ay, bw)), __dmul_rn(az, bx));
    q[3] = __dadd_rn(__dsub_rn(__dadd_rn(__dmul_rn(aw, bz), __dmul_rn(ax, by)), __dmul_rn(ay, bx)), __dmul_rn(az, bw));
    const double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(q[0], q[0]), __dmul_rn(q[1], q[1])),
                                                      __dmul_rn(q[2], q[2])),
                                            __dmul_rn(q[3], q[3])));
    A.x = (float)w[0], A.y = (float)w[1], A.z = (float)w[2];
    A.w = (float)__ddiv_rn(q[0], nrm);
    B.x = (float)__ddiv_rn(q[1], nrm), B.y = (float)__ddiv_rn(q[2], nrm), B.z = (float)__ddiv_rn(q[3], nrm);
    params[4 * i] = A;
    params[4 * i + 1] = B;
}

// refine_reset (loopclose.py:228-245): opacity <- value, optimizer state
// fresh (opt_state = b"": zero moments and step count).
__global__ void __launch_bounds__(256)
reset_rows_kernel(float *__restrict__ params, float4 *__restrict__ m, float4 *__restrict__ v, int64_t n,
                  float opacity) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t i = t >> 2;
    if (i >= n) return;
    const int q = (int)(t & 3);
    m[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    v[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (q == 0) params[16 * i + 10] = opacity;
}

int transform_rows(float *params, int64_t n, const double *r, const double *t, const double *q, cudaStream_t st) {
    if (n <= 0) return SM_OK;
    RigidDev c;
    for (int k = 0; k < 9; k++) c.r[k] = r[k];
    for (int k = 0; k < 3; k++) c.t[k] = t[k];
    for (int k = 0; k < 4; k++) c.q[k] = q[k];
    count_launches(1);
    transform_rows_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(reinterpret_cast<float4 *>(params), n, c);
    SM_CHECK_LAUNCH("transform_rows");
    return SM_OK;
}

int reset_rows(float *params, float *m, float *v, int64_t n, float opacity, cudaStream_t st) {
    if (n <= 0) return SM_OK;
    count_launches(1);
    reset_rows_kernel<<<(unsigned)ceil_div(n * 4, 256), 256, 0, st>>>(params, reinterpret_cast<float4 *>(m),
                                                                       reinterpret_cast<float4 *>(v), n, opacity);
    SM_CHECK_LAUNCH("reset_rows");
    return SM_OK;
}

// ------------------------------------------------------ keyframe codec
// .dkf file image (diskformat.py:198-216 pack_keyframe) from a keyframe's
// HBM copy: 140-byte header (host-built) | RGB u8 (H,W,3) | depth f32
// little-endian (H,W).  The keyframe's colours are already its 8-bit values
// (k/255 re-quantises to k), so the file is a byte copy on the device; the
// write-behind then moves it D2H and writes it (no host quantisation).
struct KfHeader {
    uint32_t w[35];   // 140 bytes
};

__global__ void __launch_bounds__(256)
keyframe_pack_kernel(KfHeader h, const uint8_t *__restrict__ rgb, const uint8_t *__restrict__ depth, int64_t npx,
                     uint8_t *__restrict__ out) {
    const int64_t total = 140 + 7 * npx;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        uint8_t b;
        if (i < 140)
            b = (uint8_t)(h.w[i >> 2] >> (8 * (i & 3)));
        else if (i < 140 + 3 * npx)
            b = rgb[i - 140];
        else
            b = depth[i - 140 - 3 * npx];
        out[i] = b;
    }
}

int keyframe_pack(const uint8_t *header, const uint8_t *rgb, const float *depth, int64_t npx, uint8_t *out,
                  cudaStream_t st) {
    KfHeader h;
    memcpy(h.w, header, 140);
    count_launches(1);
    keyframe_pack_kernel<<<148 * 4, 256, 0, st>>>(h, rgb, reinterpret_cast<const uint8_t *>(depth), npx, out);
    SM_CHECK_LAUNCH("keyframe_pack");
    return SM_OK;
}

// ------------------------------------------------------------------ K1
struct CullDev {
    double planes[24];
    double cam[3];
    double maxd, s, half;
};

// culling.py:104-131 in fp64 with every op rounded separately (the reference
// evaluates these with NumPy scalars, one rounding per operation).
__global__ void __launch_bounds__(256)
cull_kernel(const int32_t *__restrict__ coords, int64_t n, CullDev c, uint8_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double mn[3], mx[3];
#pragma unroll
    for (int k = 0; k < 3; k++) {
        const double ctr = __dmul_rn((double)coords[3 * i + k], c.s);   // grid.py:106
        mn[k] = __dsub_rn(ctr, c.half);
        mx[k] = __dadd_rn(ctr, c.half);
    }
    // _nearest_distance: || p - clip(p, min, max) ||
    double d2 = 0.0;
#pragma unroll
    for (int k = 0; k < 3; k++) {
        const double nearest = fmin(fmax(c.cam[k], mn[k]), mx[k]);
        const double d = __dsub_rn(c.cam[k], nearest);
        d2 = __dadd_rn(d2, __dmul_rn(d, d));
    }
    bool vis = !(__dsqrt_rn(d2) > c.maxd);
    // aabb_in_frustum p-vertex OUTSIDE test
#pragma unroll
    for (int pl = 0; pl < 6; pl++) {
        const double nx = c.planes[4 * pl], ny = c.planes[4 * pl + 1], nz = c.planes[4 * pl + 2],
                     d = c.planes[4 * pl + 3];
        const double px = nx >= 0 ? mx[0] : mn[0];
        const double py = ny >= 0 ? mx[1] : mn[1];
        const double pz = nz >= 0 ? mx[2] : mn[2];
        const double val =
            __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(nx, px), __dmul_rn(ny, py)), __dmul_rn(nz, pz)), d);
        if (val < 0.0) vis = false;
    }
    out[i] = vis ? 1 : 0;
}

int cull_chunks(const int32_t *coords, int64_t n, const double *planes, const double *cam,
                double maxd, double s, uint8_t *out, cudaStream_t st) {
    if (n < 0 || s <= 0) {
        set_error("bad cull arguments");
        return SM_ERR_INVALID;
    }
    if (n == 0) return SM_OK;
    CullDev c;
    for (int k = 0; k < 24; k++) c.planes[k] = planes[k];
    for (int k = 0; k < 3; k++) c.cam[k] = cam[k];
    c.maxd = maxd;
    c.s = s;
    c.half = s / 2.0;
    prof_begin(ST_CULL, st);
    count_launches(1);
    cull_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(coords, n, c, out);
    prof_end(ST_CULL, st);
    SM_CHECK_LAUNCH("cull_chunks");
    return SM_OK;
}

// grid.py:110-121 encode_positions: floor((p + s/2) / s) per axis in fp64.
__global__ void __launch_bounds__(256)
encode_kernel(const float *__restrict__ params, int64_t n, double s, double half,
              unsigned long long *__restrict__ ids, unsigned long long *__restrict__ err) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    unsigned long long id = 0;
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 3; k++) {
        const double p = (double)params[i * SM_PARAM_STRIDE + k];
        const double c = floor(__ddiv_rn(__dadd_rn(p, half), s));
        if (!(c >= -1048576.0 && c <= 1048575.0)) bad = true;
        const unsigned long long f = bad ? 0ull : (unsigned long long)(c + 1048576.0);
        id = (id << 21) | f;
    }
    if (bad) atomicMin(err, (unsigned long long)i);
    ids[i] = id;
}

int encode_positions(const float *params, int64_t n, double s, uint64_t *ids, int64_t *err,
                     cudaStream_t st) {
    if (s <= 0 || n < 0) {
        set_error("chunk size must be positive");
        return SM_ERR_INVALID;
    }
    cudaMemsetAsync(err, 0xff, sizeof(int64_t), st);   // -1 as u64 max
    if (n == 0) return SM_OK;
    count_launches(1);
    encode_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(
        params, n, s, s / 2.0, reinterpret_cast<unsigned long long *>(ids),
        reinterpret_cast<unsigned long long *>(err));
    SM_CHECK_LAUNCH("encode_positions");
    return SM_OK;
}

__global__ void __launch_bounds__(256)
expand_kernel(const int64_t *__restrict__ off, const int64_t *__restrict__ cnt,
              const int64_t *__restrict__ prefix, int64_t nseg, int64_t total,
              int32_t *__restrict__ slots) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    int64_t lo = 0, hi = nseg - 1;   // last segment with prefix <= i
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= i) lo = mid;
        else hi = mid - 1;
    }
    slots[i] = (int32_t)(off[lo] + (i - prefix[lo]));
    (void)cnt;
}

int expand_segments(const int64_t *off, const int64_t *cnt, const int64_t *prefix, int64_t nseg,
                    int64_t total, int32_t *slots, cudaStream_t st) {
    if (total <= 0 || nseg <= 0) return SM_OK;
    count_launches(1);
    expand_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, st>>>(off, cnt, prefix, nseg, total, slots);
    SM_CHECK_LAUNCH("expand_segments");
    return SM_OK;
}

// ----------------------------------------------------------------- K8/K9
// .dcg record (diskformat.py:51-66): 59 little-endian f32 + u32 opt_len = 240 B.
// Optional Adam tail (opt_len = 120): "ADM1" | step u32 | m[14] f32 | v[14] f32.
constexpr int kRecWords = 60;
constexpr uint32_t kAdamMagic = 0x314d4441u;   // "ADM1"
constexpr int kAdamTail = 120;

__device__ __forceinline__ int shrest_src(int k) {   // rest index -> sh index
    return k < 15 ? 1 + k : (k < 30 ? 2 + k : 3 + k);
}

// WRITE = false: validation only (the streamer checks a staged chunk on its
// copy stream before the unpack is queued behind the render).
template <bool WRITE>
__global__ void __launch_bounds__(256)
unpack_kernel(const uint8_t *__restrict__ rec, int64_t n, int64_t stride, float *__restrict__ params,
              float *__restrict__ sh_rest, float *__restrict__ m, float *__restrict__ v,
              unsigned long long *__restrict__ err) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t *w = reinterpret_cast<const uint32_t *>(rec + i * stride);
    float f[59];
#pragma unroll
    for (int k = 0; k < 59; k++) f[k] = __uint_as_float(w[k]);
    const uint32_t opt_len = w[59];
    // validate_gaussian_arrays (core.py:208-221)
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 59; k++) ok = ok && isfinite(f[k]);
    ok = ok && f[7] > 0.f && f[8] > 0.f && f[9] > 0.f && f[10] >= 0.f && f[10] <= 1.f;
    const double qn = sqrt((double)f[3] * f[3] + (double)f[4] * f[4] + (double)f[5] * f[5] +
                           (double)f[6] * f[6]);
    ok = ok && fabs(qn - 1.0) <= 1e-6;
    if (stride == 240 + kAdamTail) {
        const uint32_t *t = w + kRecWords;
        ok = ok && opt_len == (uint32_t)kAdamTail && t[0] == kAdamMagic;
    } else {
        ok = ok && opt_len == 0;
    }
    if (!ok) atomicMin(err, (unsigned long long)i);
    if (!WRITE) return;
    float *p = params + i * SM_PARAM_STRIDE;
#pragma unroll
    for (int k = 0; k < 11; k++) p[k] = f[k];
    p[11] = f[11 + 0];
    p[12] = f[11 + 16];
    p[13] = f[11 + 32];
    p[14] = 0.f;
    p[15] = 0.f;
#pragma unroll
    for (int k = 0; k < 45; k++) sh_rest[i * 45 + k] = f[11 + shrest_src(k)];
    float *mm = m + i * SM_PARAM_STRIDE;
    float *vv = v + i * SM_PARAM_STRIDE;
    if (stride == 240 + kAdamTail) {
        const uint32_t *t = w + kRecWords;
#pragma unroll
        for (int k = 0; k < 14; k++) {
            mm[k] = __uint_as_float(t[2 + k]);
            vv[k] = __uint_as_float(t[16 + k]);
        }
        mm[14] = (float)t[1];
        mm[15] = vv[14] = vv[15] = 0.f;
    } else {
#pragma unroll
        for (int k = 0; k < 16; k++) mm[k] = vv[k] = 0.f;
    }
}

__global__ void __launch_bounds__(256)
pack_kernel(const float *__restrict__ params, const float *__restrict__ sh_rest,
            const float *__restrict__ m, const float *__restrict__ v, int64_t n, int64_t stride,
            uint8_t *__restrict__ rec) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t *w = reinterpret_cast<uint32_t *>(rec + i * stride);
    const float *p = params + i * SM_PARAM_STRIDE;
#pragma unroll
    for (int k = 0; k < 11; k++) w[k] = __float_as_uint(p[k]);
    w[11 + 0] = __float_as_uint(p[11]);
    w[11 + 16] = __float_as_uint(p[12]);
    w[11 + 32] = __float_as_uint(p[13]);
#pragma unroll
    for (int k = 0; k < 45; k++) w[11 + shrest_src(k)] = __float_as_uint(sh_rest[i * 45 + k]);
    if (stride == 240 + kAdamTail) {
        w[59] = kAdamTail;
        uint32_t *t = w + kRecWords;
        const float *mm = m + i * SM_PARAM_STRIDE;
        const float *vv = v + i * SM_PARAM_STRIDE;
        t[0] = kAdamMagic;
        t[1] = (uint32_t)mm[14];
#pragma unroll
        for (int k = 0; k < 14; k++) {
            t[2 + k] = __float_as_uint(mm[k]);
            t[16 + k] = __float_as_uint(vv[k]);
        }
    } else {
        w[59] = 0;
    }
}

int chunk_unpack(const uint8_t *rec, int64_t n, int64_t stride, float *params, float *sh_rest,
                 float *m, float *v, int64_t *err, cudaStream_t st) {
    if (stride != 240 && stride != 240 + kAdamTail) {
        set_error("unsupported record stride %lld", (long long)stride);
        return SM_ERR_INVALID;
    }
    cudaMemsetAsync(err, 0xff, sizeof(int64_t), st);
    if (n <= 0) return SM_OK;
    prof_begin(ST_CODEC, st);
    count_launches(1);
    if (params)
        unpack_kernel<true><<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(
            rec, n, stride, params, sh_rest, m, v, reinterpret_cast<unsigned long long *>(err));
    else   // validation only
        unpack_kernel<false><<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(
            rec, n, stride, nullptr, nullptr, nullptr, nullptr, reinterpret_cast<unsigned long long *>(err));
    prof_end(ST_CODEC, st);
    SM_CHECK_LAUNCH("chunk_unpack");
    return SM_OK;
}

int chunk_pack(const float *params, const float *sh_rest, const float *m, const float *v, int64_t n,
               int64_t stride, uint8_t *rec, cudaStream_t st) {
    if (stride != 240 && stride != 240 + kAdamTail) {
        set_error("unsupported record stride %lld", (long long)stride);
        return SM_ERR_INVALID;
    }
    if (n <= 0) return SM_OK;
    prof_begin(ST_CODEC, st);
    count_launches(1);
    pack_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(params, sh_rest, m, v, n, stride, rec);
    prof_end(ST_CODEC, st);
    SM_CHECK_LAUNCH("chunk_pack");
    return SM_OK;
}

}  // namespace sm
