// Loss forward + gradient: renderloss.total_loss (renderloss.py:226-274).
//
//   L = (1 - ls) * mean|rgb - gt| + ls * (1 - SSIM) + ld * mean_{gt_d > 0} |d - gt_d|
//
// SSIM follows scikit-image structural_similarity as the reference calls it
// (renderloss.py:237-247): 11x11 Gaussian window (sigma 1.5, truncate 3.5),
// population covariance, C1 = 1e-4, C2 = 9e-4, mean of the S-map over the
// (H-10) x (W-10) valid crop, averaged over the 3 channels.  Every crop
// pixel's window lies inside the image, so the reflect padding never enters
// the value or the gradient.  gt rgb arrives as the keyframe's 8-bit values
// (core.py:262-267 keeps k/255 in float32; u8 / 255.f reproduces it exactly).
//
// Kernel A (per 32x16 tile and channel): separable 11-tap filter of
// x, y, x^2, y^2, xy in shared memory, register-blocked (a thread produces 4
// horizontal or 2 vertical outputs from one window load, ~5x fewer shared
// loads than one output per thread); S and dS/d{mu_x, E[x^2], E[xy]} on the
// crop, L1 / depth partial sums; the last block sums the partials in a fixed
// order (deterministic) and finalises the loss.
// Kernel B: the adjoint filter of those three maps (same blocking) and the
// per-pixel gradients; the depth gradient reads the finished valid count.
#include "common.cuh"
#include "prof.cuh"

namespace sm {

constexpr int kLW = 32, kLH = 16;   // output tile (columns x rows)
constexpr int kHW = kLW + 10, kHH = kLH + 10;   // + 5-px halo each side
__constant__ float c_gw[11];
__constant__ float c_gwp[18];   // c_gwp[j + 3] = c_gw[j] for j in [0, 11), zero elsewhere (j in [-3, 15))

// tap weights of two neighbouring outputs (packed fp32x2 filters): output o
// at input offset k uses c_gw[k - o]
__device__ __forceinline__ float2 wpair(int k, int o) { return make_float2(c_gwp[k - o + 3], c_gwp[k - o + 2]); }

struct LossAcc {
    double l1, ssim, dsum, dcount;
    uint32_t done;   // blocks of kernel A finished (the last one finalises)
};

__device__ __forceinline__ float load_gt(const uint8_t *gt, const float *gtf, int64_t i) {
    return gt ? (float)gt[i] / 255.f : gtf[i];
}

__global__ void __launch_bounds__(256)
loss_fwd_kernel(const float *__restrict__ rgb, const float *__restrict__ depth,
                const uint8_t *__restrict__ gt, const float *__restrict__ gtf,
                const float *__restrict__ gt_depth, int W, int H, int C, float ls, float ld,
                float *__restrict__ dmaps /* [C][3][H*W] */, double *__restrict__ partial,
                LossAcc *acc, float *__restrict__ out, int want_grad) {
    __shared__ float sx[kHH][kHW], sy[kHH][kHW];
    __shared__ float hs[5][kHH][kLW];
    __shared__ float red[4][8];
    __shared__ bool s_last;
    const int ch = blockIdx.z;
    const int tx0 = blockIdx.x * kLW, ty0 = blockIdx.y * kLH;
    const int64_t N = (int64_t)W * H;
    for (int i = threadIdx.x; i < kHH * kHW; i += 256) {
        const int yy = ty0 - 5 + i / kHW, xx = tx0 - 5 + i % kHW;
        float xv = 0.f, yv = 0.f;
        if (yy >= 0 && yy < H && xx >= 0 && xx < W) {
            const int64_t p = (int64_t)yy * W + xx;
            xv = rgb[C * p + ch];
            yv = load_gt(gt, gtf, C * p + ch);
        }
        sx[i / kHW][i % kHW] = xv;
        sy[i / kHW][i % kHW] = yv;
    }
    __syncthreads();
    // horizontal: 26 rows x 32 centres, 4 consecutive centres per thread
    for (int it = threadIdx.x; it < kHH * (kLW / 4); it += 256) {
        const int r = it / (kLW / 4), c0 = 4 * (it % (kLW / 4));
        float2 a[5][2];   // [stat][outputs (0,1) | (2,3)], packed fp32x2
#pragma unroll
        for (int t = 0; t < 5; t++) a[t][0] = a[t][1] = f2s(0.f);
#pragma unroll
        for (int k = 0; k < 14; k++) {
            const float xv = sx[r][c0 + k], yv = sy[r][c0 + k];
            const float v[5] = {xv, yv, xv * xv, yv * yv, xv * yv};
            const float2 w01 = wpair(k, 0), w23 = wpair(k, 2);   // zero taps outside the window
#pragma unroll
            for (int t = 0; t < 5; t++) {
                a[t][0] = fma2(w01, f2s(v[t]), a[t][0]);
                a[t][1] = fma2(w23, f2s(v[t]), a[t][1]);
            }
        }
#pragma unroll
        for (int t = 0; t < 5; t++) {
            hs[t][r][c0 + 0] = a[t][0].x;
            hs[t][r][c0 + 1] = a[t][0].y;
            hs[t][r][c0 + 2] = a[t][1].x;
            hs[t][r][c0 + 3] = a[t][1].y;
        }
    }
    __syncthreads();
    // vertical: 16 x 32 outputs, 2 rows per thread
    const int lx = threadIdx.x % kLW, ly0 = 2 * (threadIdx.x / kLW);
    float2 m2[5];   // (row ly0, row ly0 + 1) per statistic
#pragma unroll
    for (int t = 0; t < 5; t++) m2[t] = f2s(0.f);
#pragma unroll
    for (int k = 0; k < 12; k++) {
        const float2 w = wpair(k, 0);
#pragma unroll
        for (int t = 0; t < 5; t++) m2[t] = fma2(w, f2s(hs[t][ly0 + k][lx]), m2[t]);
    }
    float m[2][5];
#pragma unroll
    for (int t = 0; t < 5; t++) {
        m[0][t] = m2[t].x;
        m[1][t] = m2[t].y;
    }
    float s_val = 0.f, l1 = 0.f, dsum = 0.f, dcnt = 0.f;
#pragma unroll
    for (int o = 0; o < 2; o++) {
        const int x = tx0 + lx, y = ty0 + ly0 + o;
        if (x >= W || y >= H) continue;
        const int64_t p = (int64_t)y * W + x;
        l1 += fabsf(sx[ly0 + o + 5][lx + 5] - sy[ly0 + o + 5][lx + 5]);
        if (ch == 0 && gt_depth && depth && gt_depth[p] > 0.f) {
            dsum += fabsf(depth[p] - gt_depth[p]);
            dcnt += 1.f;
        }
        float dmu = 0.f, dxx = 0.f, dxy = 0.f;
        if (x >= 5 && x < W - 5 && y >= 5 && y < H - 5) {
            const float C1 = 1e-4f, C2 = 9e-4f;
            const float mx = m[o][0], my = m[o][1];
            const float vx = m[o][2] - mx * mx, vy = m[o][3] - my * my, vxy = m[o][4] - mx * my;
            const float A1 = 2.f * mx * my + C1, A2 = 2.f * vxy + C2;
            const float B1 = mx * mx + my * my + C1, B2 = vx + vy + C2;
            const float inv = 1.f / (B1 * B2);
            const float S = A1 * A2 * inv;
            s_val += S;
            dmu = (2.f * my * A2 - 2.f * my * A1) * inv - S * (2.f * mx / B1 - 2.f * mx / B2);
            dxx = -S / B2;
            dxy = 2.f * A1 * inv;
        }
        if (want_grad) {
            dmaps[(int64_t)(ch * 3 + 0) * N + p] = dmu;
            dmaps[(int64_t)(ch * 3 + 1) * N + p] = dxx;
            dmaps[(int64_t)(ch * 3 + 2) * N + p] = dxy;
        }
    }
    // block partials, then the last block sums every block's in a fixed order
    float v[4] = {s_val, l1, dsum, dcnt};
#pragma unroll
    for (int t = 0; t < 4; t++)
#pragma unroll
        for (int o = 16; o; o >>= 1) v[t] += __shfl_xor_sync(0xffffffffu, v[t], o);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int t = 0; t < 4; t++) red[t][threadIdx.x >> 5] = v[t];
    __syncthreads();
    const uint32_t nblk = gridDim.x * gridDim.y * gridDim.z;
    if (threadIdx.x < 4) {
        double sacc = 0;
        for (int w = 0; w < 8; w++) sacc += red[threadIdx.x][w];
        const int64_t blk = ((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        partial[blk * 4 + threadIdx.x] = sacc;
        __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&acc->done, 1u) == nblk - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double *sh = reinterpret_cast<double *>(&hs[0][0][0]);   // [4][256], reused
    double s4[4] = {0, 0, 0, 0};
    for (uint32_t b = threadIdx.x; b < nblk; b += 256)
#pragma unroll
        for (int t = 0; t < 4; t++) s4[t] += __ldcg(&partial[(int64_t)b * 4 + t]);
#pragma unroll
    for (int t = 0; t < 4; t++) sh[t * 256 + threadIdx.x] = s4[t];
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if ((int)threadIdx.x < o)
#pragma unroll
            for (int t = 0; t < 4; t++) sh[t * 256 + threadIdx.x] += sh[t * 256 + threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x) return;
    acc->ssim = sh[0];
    acc->l1 = sh[256];
    acc->dsum = sh[512];
    acc->dcount = sh[768];
    const double Np = (double)W * H;
    const double Nc = (double)(W - 10) * (H - 10);
    const double l1v = sh[256] / ((double)C * Np);
    const double ssim = sh[0] / ((double)C * Nc);
    const double dl = sh[768] > 0 ? sh[512] / sh[768] : 0.0;
    out[0] = (float)((1.0 - ls) * l1v + ls * (1.0 - ssim) + ld * dl);
    out[1] = (float)l1v;
    out[2] = (float)ssim;
    out[3] = (float)dl;
}

__global__ void __launch_bounds__(256)
loss_bwd_kernel(const float *__restrict__ rgb, const float *__restrict__ depth,
                const uint8_t *__restrict__ gt, const float *__restrict__ gtf,
                const float *__restrict__ gt_depth, int W, int H, int C,
                const float *__restrict__ dmaps, const LossAcc *acc, float ls, float ld,
                float *__restrict__ d_rgb, float *__restrict__ d_depth) {
    __shared__ float sm3[3][kHH][kHW];
    __shared__ float ha[3][kHH][kLW];
    const int ch = blockIdx.z;
    const int tx0 = blockIdx.x * kLW, ty0 = blockIdx.y * kLH;
    const int64_t N = (int64_t)W * H;
    for (int i = threadIdx.x; i < kHH * kHW; i += 256) {
        const int yy = ty0 - 5 + i / kHW, xx = tx0 - 5 + i % kHW;
        const bool ok = yy >= 0 && yy < H && xx >= 0 && xx < W;
        const int64_t p = (int64_t)yy * W + xx;
#pragma unroll
        for (int t = 0; t < 3; t++) sm3[t][i / kHW][i % kHW] = ok ? dmaps[(int64_t)(ch * 3 + t) * N + p] : 0.f;
    }
    __syncthreads();
    for (int it = threadIdx.x; it < kHH * (kLW / 4); it += 256) {   // adjoint, horizontal
        const int r = it / (kLW / 4), c0 = 4 * (it % (kLW / 4));
        float2 a[3][2];   // symmetric kernel: adjoint = same taps
#pragma unroll
        for (int t = 0; t < 3; t++) a[t][0] = a[t][1] = f2s(0.f);
#pragma unroll
        for (int k = 0; k < 14; k++) {
            const float2 w01 = wpair(k, 0), w23 = wpair(k, 2);
#pragma unroll
            for (int t = 0; t < 3; t++) {
                const float v = sm3[t][r][c0 + k];
                a[t][0] = fma2(w01, f2s(v), a[t][0]);
                a[t][1] = fma2(w23, f2s(v), a[t][1]);
            }
        }
#pragma unroll
        for (int t = 0; t < 3; t++) {
            ha[t][r][c0 + 0] = a[t][0].x;
            ha[t][r][c0 + 1] = a[t][0].y;
            ha[t][r][c0 + 2] = a[t][1].x;
            ha[t][r][c0 + 3] = a[t][1].y;
        }
    }
    __syncthreads();
    const int lx = threadIdx.x % kLW, ly0 = 2 * (threadIdx.x / kLW);
    float2 a2[3];
#pragma unroll
    for (int t = 0; t < 3; t++) a2[t] = f2s(0.f);
#pragma unroll
    for (int k = 0; k < 12; k++) {
        const float2 w = wpair(k, 0);
#pragma unroll
        for (int t = 0; t < 3; t++) a2[t] = fma2(w, f2s(ha[t][ly0 + k][lx]), a2[t]);
    }
    float a[2][3];
#pragma unroll
    for (int t = 0; t < 3; t++) {
        a[0][t] = a2[t].x;
        a[1][t] = a2[t].y;
    }
    const float Nf = (float)((double)W * H);
    const float Nc = (float)((double)(W - 10) * (H - 10));
    const double nv = acc->dcount;
#pragma unroll
    for (int o = 0; o < 2; o++) {
        const int x = tx0 + lx, y = ty0 + ly0 + o;
        if (x >= W || y >= H) continue;
        const int64_t p = (int64_t)y * W + x;
        const float xv = rgb[C * p + ch];
        const float yv = load_gt(gt, gtf, C * p + ch);
        const float dssim = (a[o][0] + 2.f * xv * a[o][1] + yv * a[o][2]) / Nc;
        const float diff = xv - yv;
        const float sg = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
        d_rgb[C * p + ch] = (1.f - ls) * sg / (float)((double)C * Nf) - ls * dssim / (float)C;
        if (ch == 0 && d_depth) {
            float g = 0.f;
            if (nv > 0 && gt_depth && depth && gt_depth[p] > 0.f) {
                const float dd = depth[p] - gt_depth[p];
                g = ld * (dd > 0.f ? 1.f : (dd < 0.f ? -1.f : 0.f)) / (float)nv;
            }
            d_depth[p] = g;
        }
    }
}

static bool g_weights_set = false;

static int64_t loss_blocks(int W, int H) { return ceil_div(W, kLW) * ceil_div(H, kLH) * 4; }

int64_t loss_workspace_size(int W, int H) {
    return align_up(sizeof(LossAcc), 256) + align_up(loss_blocks(W, H) * 4 * 8, 256) +
           align_up((int64_t)12 * W * H * 4, 256);
}

int loss_forward_backward(const float *rgb, const float *depth, const uint8_t *gt_rgb,
                          const float *gt_rgbf, const float *gt_depth, int W, int H, int C, float ls,
                          float ld, void *ws, int64_t ws_bytes, float *loss_out, float *d_rgb,
                          float *d_depth, cudaStream_t st) {
    if (W < 11 || H < 11) {
        set_error("ssim needs images of at least 11x11, got %dx%d", W, H);
        return SM_ERR_DIMENSION;
    }
    if (C < 1 || C > 4 || (!gt_rgb && !gt_rgbf)) {
        set_error("loss: bad channel count or missing ground truth");
        return SM_ERR_INVALID;
    }
    if (ws_bytes < loss_workspace_size(W, H)) {
        set_error("loss workspace too small");
        return SM_ERR_WORKSPACE;
    }
    if (!g_weights_set) {
        double w[11], s = 0;
        for (int i = -5; i <= 5; i++) {
            w[i + 5] = exp(-0.5 * (double)(i * i) / 2.25);
            s += w[i + 5];
        }
        float wf[11];
        for (int i = 0; i < 11; i++) wf[i] = (float)(w[i] / s);
        cudaError_t e = cudaMemcpyToSymbol(c_gw, wf, sizeof(wf));
        if (e != cudaSuccess) return cuda_status(e, "loss weights");
        float wp[18] = {0};
        for (int i = 0; i < 11; i++) wp[i + 3] = wf[i];
        e = cudaMemcpyToSymbol(c_gwp, wp, sizeof(wp));
        if (e != cudaSuccess) return cuda_status(e, "loss weights");
        g_weights_set = true;
    }
    char *base = static_cast<char *>(ws);
    LossAcc *acc = reinterpret_cast<LossAcc *>(base);
    double *partial = reinterpret_cast<double *>(base + align_up(sizeof(LossAcc), 256));
    float *dmaps = reinterpret_cast<float *>(base + align_up(sizeof(LossAcc), 256) +
                                             align_up(loss_blocks(W, H) * 4 * 8, 256));
    dim3 grid((unsigned)ceil_div(W, kLW), (unsigned)ceil_div(H, kLH), (unsigned)C);
    const int want = d_rgb != nullptr;
    prof_begin(ST_LOSS, st);
    cudaMemsetAsync(&acc->done, 0, sizeof(uint32_t), st);   // block counter (any workspace state)
    loss_fwd_kernel<<<grid, 256, 0, st>>>(rgb, depth, gt_rgb, gt_rgbf, gt_depth, W, H, C, ls, ld, dmaps,
                                          partial, acc, loss_out, want);
    if (want)
        loss_bwd_kernel<<<grid, 256, 0, st>>>(rgb, depth, gt_rgb, gt_rgbf, gt_depth, W, H, C, dmaps,
                                              acc, ls, ld, d_rgb, d_depth);
    prof_end(ST_LOSS, st);
    count_launches(want ? 2 : 1);
    SM_CHECK_LAUNCH("loss_forward_backward");
    return SM_OK;
}

}  // namespace sm
