// Ingest path on the device: the edge-driven sampling
// scores and the depth lifting of splatmap sample.py.
//
//   log_norm (sample.py:63-75):  |LoG * luma|, 0-padded, max-normalised
//   sampling_probability (78-84): max(p_input - p_rendered, 0)
//   lift_to_gaussians (104-146):  unproject sampled pixels with depth > 0
//
// All in fp64 like the reference (the probabilities feed the host's
// Generator.choice draw, sample.py:87-101, which stays on the host: NumPy's
// choice without replacement cannot be reproduced on the device).  The luma
// is (0.299 r + 0.587 g) + 0.114 b, the convolution sums the taps row by row;
// the reference's BLAS dot / ndimage.convolve may round in another order,
// so the scores agree to ~1e-15 relative (tests: 1e-12).
#include "common.cuh"
#include "prof.cuh"

namespace sm {

constexpr int kLogMaxR = 3;                    // kernel radius <= 3 (7x7 taps)
constexpr int kLogT = 16;                      // 16x16 output tile
constexpr int kLogS = kLogT + 2 * kLogMaxR;    // staged luma tile

struct LogTaps {
    double k[(2 * kLogMaxR + 1) * (2 * kLogMaxR + 1)];
    int radius;
};

// Colour channel i of an image stored as SM_RGB_U8 (the keyframe's 8-bit
// values: k/255 in float32, core.py:262-267), SM_RGB_F32 or SM_RGB_F64.
__device__ __forceinline__ double rgb_at(const void *rgb, int kind, int64_t i) {
    if (kind == SM_RGB_U8) return (double)((float)static_cast<const uint8_t *>(rgb)[i] / 255.f);
    if (kind == SM_RGB_F32) return (double)static_cast<const float *>(rgb)[i];
    return static_cast<const double *>(rgb)[i];
}

__device__ __forceinline__ double luma_at(const void *rgb, int kind, int W, int H, int x, int y) {
    if (x < 0 || y < 0 || x >= W || y >= H) return 0.0;   // mode="constant", cval=0
    const int64_t p = 3 * ((int64_t)y * W + x);
    const double r = rgb_at(rgb, kind, p), g = rgb_at(rgb, kind, p + 1), b = rgb_at(rgb, kind, p + 2);
    return __dadd_rn(__dadd_rn(__dmul_rn(r, 0.299), __dmul_rn(g, 0.587)), __dmul_rn(b, 0.114));
}

// |LoG response| per pixel and the image's peak (positive doubles order like
// their bit patterns, so the peak is an integer atomicMax).
__global__ void __launch_bounds__(kLogT * kLogT)
log_score_kernel(const void *__restrict__ rgb, int kind, int W, int H, LogTaps taps,
                 double *__restrict__ out, unsigned long long *__restrict__ peak) {
    __shared__ double g[kLogS][kLogS];
    const int r = taps.radius;
    const int x0 = blockIdx.x * kLogT - r, y0 = blockIdx.y * kLogT - r;
    const int S = kLogT + 2 * r;
    for (int i = threadIdx.x; i < S * S; i += blockDim.x) g[i / S][i % S] = luma_at(rgb, kind, W, H, x0 + i % S, y0 + i / S);
    __syncthreads();
    const int tx = threadIdx.x % kLogT, ty = threadIdx.x / kLogT;
    const int x = blockIdx.x * kLogT + tx, y = blockIdx.y * kLogT + ty;
    double v = 0.0;
    if (x < W && y < H) {
        const int n = 2 * r + 1;
        double acc = 0.0;
        for (int i = 0; i < n; i++)
            for (int j = 0; j < n; j++)   // symmetric taps: correlation = convolution
                acc = __dadd_rn(acc, __dmul_rn(taps.k[i * n + j], g[ty + i][tx + j]));
        v = fabs(acc);
        out[(int64_t)y * W + x] = v;
    }
    // block max -> one atomic per warp
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long c = __shfl_xor_sync(0xffffffffu, b, o);
        b = c > b ? c : b;
    }
    if ((threadIdx.x & 31) == 0 && b) atomicMax(peak, b);
}

// ps = max(a / peak_a - b / peak_b, 0) (a peak of 0 leaves its map as is);
// b == nullptr: ps = a / peak_a (log_norm's normalisation alone).
__global__ void __launch_bounds__(256)
sampling_prob_kernel(const double *__restrict__ a, const unsigned long long *__restrict__ pa,
                     const double *__restrict__ b, const unsigned long long *__restrict__ pb, int64_t n,
                     double *__restrict__ ps) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double peak_a = __longlong_as_double((long long)*pa);
    double va = a[i];
    if (peak_a > 0.0) va = __ddiv_rn(va, peak_a);
    if (!b) {
        ps[i] = va;
        return;
    }
    const double peak_b = __longlong_as_double((long long)*pb);
    double vb = b[i];
    if (peak_b > 0.0) vb = __ddiv_rn(vb, peak_b);
    ps[i] = fmax(__dsub_rn(va, vb), 0.0);
}

struct LiftCam {
    double r[9];   // r_wc row-major (world <- camera)
    double t[3];
    double fx, fy, cx, cy;
    double scale_factor;
    float opacity;
};

// One sampled pixel -> one param record (include/splatmap_cuda.h layout),
// float32-canonical like storage_canonical (diskformat.py:69-83); valid[i] =
// depth > 0 (the host keeps the valid ones, in order, like sample.py:122-124).
__global__ void __launch_bounds__(256)
lift_kernel(const int32_t *__restrict__ pix, int64_t k, const float *__restrict__ depth,
            const void *__restrict__ rgb, int kind, int W, int H, LiftCam c,
            float4 *__restrict__ rec, int32_t *__restrict__ valid) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    const int row = pix[2 * i], col = pix[2 * i + 1];
    const int64_t p = (int64_t)row * W + col;
    const double d = (double)depth[p];
    valid[i] = d > 0.0;
    // cam = ((col - cx) / fx * d, (row - cy) / fy * d, d)
    const double cam[3] = {__dmul_rn(__ddiv_rn(__dsub_rn((double)col, c.cx), c.fx), d),
                           __dmul_rn(__ddiv_rn(__dsub_rn((double)row, c.cy), c.fy), d), d};
    double w[3];
#pragma unroll
    for (int a = 0; a < 3; a++)   // world = cam @ r.T + t
        w[a] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(cam[0], c.r[3 * a]), __dmul_rn(cam[1], c.r[3 * a + 1])),
                                   __dmul_rn(cam[2], c.r[3 * a + 2])),
                         c.t[a]);
    double col3[3];
#pragma unroll
    for (int a = 0; a < 3; a++)
        col3[a] = rgb_at(rgb, kind, 3 * p + a);
    const float s = (float)__ddiv_rn(__dmul_rn(c.scale_factor, d), c.fx);
    float sh0[3];
#pragma unroll
    for (int a = 0; a < 3; a++) sh0[a] = (float)__ddiv_rn(__dsub_rn(col3[a], 0.5), SM_SH_C0);
    rec[4 * i + 0] = make_float4((float)w[0], (float)w[1], (float)w[2], 1.f);   // px py pz qw
    rec[4 * i + 1] = make_float4(0.f, 0.f, 0.f, s);                             // qx qy qz sx
    rec[4 * i + 2] = make_float4(s, s, c.opacity, sh0[0]);                      // sy sz op sh0r
    rec[4 * i + 3] = make_float4(sh0[1], sh0[2], 0.f, 0.f);
}

int log_scores(const void *rgb, int kind, int W, int H, const double *taps, int radius, double *out,
               unsigned long long *peak, cudaStream_t st) {
    if (radius < 1 || radius > kLogMaxR || W < 1 || H < 1) {
        set_error("log scores: radius %d (1..%d), image %dx%d", radius, kLogMaxR, W, H);
        return SM_ERR_INVALID;
    }
    LogTaps t;
    const int n = 2 * radius + 1;
    for (int i = 0; i < n * n; i++) t.k[i] = taps[i];
    t.radius = radius;
    cudaMemsetAsync(peak, 0, sizeof(unsigned long long), st);
    dim3 grid((unsigned)ceil_div(W, kLogT), (unsigned)ceil_div(H, kLogT));
    log_score_kernel<<<grid, kLogT * kLogT, 0, st>>>(rgb, kind, W, H, t, out, peak);
    count_launches(1);
    SM_CHECK_LAUNCH("log_scores");
    return SM_OK;
}

int sampling_probability(const double *a, const unsigned long long *pa, const double *b,
                         const unsigned long long *pb, int64_t n, double *ps, cudaStream_t st) {
    if (n <= 0) return SM_OK;
    sampling_prob_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(a, pa, b, pb, n, ps);
    count_launches(1);
    SM_CHECK_LAUNCH("sampling_probability");
    return SM_OK;
}

int lift_pixels(const int32_t *pix, int64_t k, const float *depth, const void *rgb, int kind, int W, int H,
                const double *r_wc, const double *t, double fx, double fy, double cx, double cy,
                double scale_factor, float opacity, float *rec, int32_t *valid, cudaStream_t st) {
    if (k <= 0) return SM_OK;
    LiftCam c;
    for (int i = 0; i < 9; i++) c.r[i] = r_wc[i];
    for (int i = 0; i < 3; i++) c.t[i] = t[i];
    c.fx = fx, c.fy = fy, c.cx = cx, c.cy = cy, c.scale_factor = scale_factor, c.opacity = opacity;
    lift_kernel<<<(unsigned)ceil_div(k, 256), 256, 0, st>>>(pix, k, depth, rgb, kind, W, H, c,
                                                             reinterpret_cast<float4 *>(rec), valid);
    count_launches(1);
    SM_CHECK_LAUNCH("lift_pixels");
    return SM_OK;
}

}  // namespace sm
