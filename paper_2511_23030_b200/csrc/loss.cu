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
// Kernel A (per 16x16 tile and channel, separable filter in shared memory):
// S and dS/d{mu_x, E[x^2], E[xy]} on the crop, plus L1 / depth partial sums.
// Kernel B: adjoint filter of those three maps and the final per-pixel grads.
#include "common.cuh"
#include "prof.cuh"

namespace sm {

constexpr int kLT = 16;            // output tile
constexpr int kLH = kLT + 10;      // tile + halo
__constant__ float c_gw[11];

struct LossAcc {
    double l1, ssim, dsum, dcount;
    float out[4];
};

__global__ void __launch_bounds__(256)
loss_fwd_kernel(const float *__restrict__ rgb, const float *__restrict__ depth,
                const uint8_t *__restrict__ gt, const float *__restrict__ gtf,
                const float *__restrict__ gt_depth, int W, int H, int C,
                float *__restrict__ dmaps /* [C][3 maps][H*W] */, double *__restrict__ partial,
                int want_grad) {
    __shared__ float sx[kLH][kLH], sy[kLH][kLH];
    __shared__ float hs[5][kLH][kLT];
    __shared__ float red[4][8];
    const int ch = blockIdx.z;
    const int tx0 = blockIdx.x * kLT, ty0 = blockIdx.y * kLT;
    const int64_t N = (int64_t)W * H;
    for (int i = threadIdx.x; i < kLH * kLH; i += 256) {
        const int yy = ty0 - 5 + i / kLH, xx = tx0 - 5 + i % kLH;
        float xv = 0.f, yv = 0.f;
        if (yy >= 0 && yy < H && xx >= 0 && xx < W) {
            const int64_t p = (int64_t)yy * W + xx;
            xv = rgb[C * p + ch];
            yv = gt ? (float)gt[C * p + ch] / 255.f : gtf[C * p + ch];
        }
        sx[i / kLH][i % kLH] = xv;
        sy[i / kLH][i % kLH] = yv;
    }
    __syncthreads();
    // horizontal pass: rows of the haloed tile, 16 output columns
    for (int i = threadIdx.x; i < kLH * kLT; i += 256) {
        const int r = i / kLT, c = i % kLT;
        float a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
#pragma unroll
        for (int k = 0; k < 11; k++) {
            const float w = c_gw[k], xv = sx[r][c + k], yv = sy[r][c + k];
            a0 += w * xv;
            a1 += w * yv;
            a2 += w * xv * xv;
            a3 += w * yv * yv;
            a4 += w * xv * yv;
        }
        hs[0][r][c] = a0;
        hs[1][r][c] = a1;
        hs[2][r][c] = a2;
        hs[3][r][c] = a3;
        hs[4][r][c] = a4;
    }
    __syncthreads();
    const int lx = threadIdx.x % kLT, ly = threadIdx.x / kLT;
    const int x = tx0 + lx, y = ty0 + ly;
    float s_val = 0.f, l1 = 0.f, dsum = 0.f, dcnt = 0.f;
    if (x < W && y < H) {
        const int64_t p = (int64_t)y * W + x;
        l1 = fabsf(sx[ly + 5][lx + 5] - sy[ly + 5][lx + 5]);
        if (ch == 0 && gt_depth && depth && gt_depth[p] > 0.f) {
            dsum = fabsf(depth[p] - gt_depth[p]);
            dcnt = 1.f;
        }
        float dmu = 0.f, dxx = 0.f, dxy = 0.f;
        if (x >= 5 && x < W - 5 && y >= 5 && y < H - 5) {
            float m[5] = {0, 0, 0, 0, 0};
#pragma unroll
            for (int k = 0; k < 11; k++) {
                const float w = c_gw[k];
#pragma unroll
                for (int t = 0; t < 5; t++) m[t] += w * hs[t][ly + k][lx];
            }
            const float C1 = 1e-4f, C2 = 9e-4f;
            const float mx = m[0], my = m[1];
            const float vx = m[2] - mx * mx, vy = m[3] - my * my, vxy = m[4] - mx * my;
            const float A1 = 2.f * mx * my + C1, A2 = 2.f * vxy + C2;
            const float B1 = mx * mx + my * my + C1, B2 = vx + vy + C2;
            const float inv = 1.f / (B1 * B2);
            const float S = A1 * A2 * inv;
            s_val = S;
            if (want_grad) {
                dmu = (2.f * my * A2 - 2.f * my * A1) * inv - S * (2.f * mx / B1 - 2.f * mx / B2);
                dxx = -S / B2;
                dxy = 2.f * A1 * inv;
            }
        }
        if (want_grad) {
            dmaps[(int64_t)(ch * 3 + 0) * N + p] = dmu;
            dmaps[(int64_t)(ch * 3 + 1) * N + p] = dxx;
            dmaps[(int64_t)(ch * 3 + 2) * N + p] = dxy;
        }
    }
    // block reduction of the four partial sums
    float v[4] = {s_val, l1, dsum, dcnt};
#pragma unroll
    for (int t = 0; t < 4; t++)
#pragma unroll
        for (int o = 16; o; o >>= 1) v[t] += __shfl_xor_sync(0xffffffffu, v[t], o);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int t = 0; t < 4; t++) red[t][threadIdx.x >> 5] = v[t];
    __syncthreads();
    if (threadIdx.x < 4) {   // per-block partials, summed in a fixed order by loss_finalize
        double s = 0;
        for (int w = 0; w < 8; w++) s += red[threadIdx.x][w];
        const int64_t blk = ((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        partial[blk * 4 + threadIdx.x] = s;
    }
}

// Deterministic (fixed-order) reduction of the per-block partials, then the
// loss terms.  One block of 256 threads.
__global__ void __launch_bounds__(256)
loss_finalize(const double *__restrict__ partial, int64_t nblk, LossAcc *acc, int W, int H, int C,
              float ls, float ld, float *out) {
    __shared__ double sh[4][256];
    double s[4] = {0, 0, 0, 0};
    for (int64_t b = threadIdx.x; b < nblk; b += 256)
#pragma unroll
        for (int t = 0; t < 4; t++) s[t] += partial[b * 4 + t];
#pragma unroll
    for (int t = 0; t < 4; t++) sh[t][threadIdx.x] = s[t];
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if ((int)threadIdx.x < o)
#pragma unroll
            for (int t = 0; t < 4; t++) sh[t][threadIdx.x] += sh[t][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x) return;
    acc->ssim = sh[0][0];
    acc->l1 = sh[1][0];
    acc->dsum = sh[2][0];
    acc->dcount = sh[3][0];
    const double N = (double)W * H;
    const double Nc = (double)(W - 10) * (H - 10);
    const double l1 = acc->l1 / ((double)C * N);
    const double ssim = acc->ssim / ((double)C * Nc);
    const double dl = acc->dcount > 0 ? acc->dsum / acc->dcount : 0.0;
    const double total = (1.0 - ls) * l1 + ls * (1.0 - ssim) + ld * dl;
    out[0] = (float)total;
    out[1] = (float)l1;
    out[2] = (float)ssim;
    out[3] = (float)dl;
}

__global__ void __launch_bounds__(256)
loss_bwd_kernel(const float *__restrict__ rgb, const float *__restrict__ depth,
                const uint8_t *__restrict__ gt, const float *__restrict__ gtf,
                const float *__restrict__ gt_depth, int W, int H, int C,
                const float *__restrict__ dmaps, const LossAcc *acc, float ls, float ld,
                float *__restrict__ d_rgb, float *__restrict__ d_depth) {
    __shared__ float sm3[3][kLH][kLH];
    __shared__ float hs[3][kLH][kLT];
    const int ch = blockIdx.z;
    const int tx0 = blockIdx.x * kLT, ty0 = blockIdx.y * kLT;
    const int64_t N = (int64_t)W * H;
    for (int i = threadIdx.x; i < kLH * kLH; i += 256) {
        const int yy = ty0 - 5 + i / kLH, xx = tx0 - 5 + i % kLH;
        const bool ok = yy >= 0 && yy < H && xx >= 0 && xx < W;
        const int64_t p = (int64_t)yy * W + xx;
#pragma unroll
        for (int t = 0; t < 3; t++) sm3[t][i / kLH][i % kLH] = ok ? dmaps[(int64_t)(ch * 3 + t) * N + p] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kLH * kLT; i += 256) {
        const int r = i / kLT, c = i % kLT;
        float a[3] = {0, 0, 0};
#pragma unroll
        for (int k = 0; k < 11; k++) {
            const float w = c_gw[k];   // symmetric kernel: adjoint = same taps
#pragma unroll
            for (int t = 0; t < 3; t++) a[t] += w * sm3[t][r][c + k];
        }
#pragma unroll
        for (int t = 0; t < 3; t++) hs[t][r][c] = a[t];
    }
    __syncthreads();
    const int lx = threadIdx.x % kLT, ly = threadIdx.x / kLT;
    const int x = tx0 + lx, y = ty0 + ly;
    if (x >= W || y >= H) return;
    float a[3] = {0, 0, 0};
#pragma unroll
    for (int k = 0; k < 11; k++) {
        const float w = c_gw[k];
#pragma unroll
        for (int t = 0; t < 3; t++) a[t] += w * hs[t][ly + k][lx];
    }
    const int64_t p = (int64_t)y * W + x;
    const float xv = rgb[C * p + ch];
    const float yv = gt ? (float)gt[C * p + ch] / 255.f : gtf[C * p + ch];
    const float Nc = (float)((double)(W - 10) * (H - 10));
    const float dssim = (a[0] + 2.f * xv * a[1] + yv * a[2]) / Nc;
    const float diff = xv - yv;
    const float sg = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
    d_rgb[C * p + ch] = (1.f - ls) * sg / (float)((double)C * N) - ls * dssim / (float)C;
    if (ch == 0 && d_depth) {
        float g = 0.f;
        const double nv = acc->dcount;
        if (nv > 0 && gt_depth && depth && gt_depth[p] > 0.f) {
            const float dd = depth[p] - gt_depth[p];
            g = ld * (dd > 0.f ? 1.f : (dd < 0.f ? -1.f : 0.f)) / (float)nv;
        }
        d_depth[p] = g;
    }
}

static bool g_weights_set = false;

static int64_t loss_blocks(int W, int H) { return ceil_div(W, kLT) * ceil_div(H, kLT) * 4; }

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
        g_weights_set = true;
    }
    char *base = static_cast<char *>(ws);
    LossAcc *acc = reinterpret_cast<LossAcc *>(base);
    double *partial = reinterpret_cast<double *>(base + align_up(sizeof(LossAcc), 256));
    float *dmaps = reinterpret_cast<float *>(base + align_up(sizeof(LossAcc), 256) +
                                             align_up(loss_blocks(W, H) * 4 * 8, 256));
    dim3 grid((unsigned)ceil_div(W, kLT), (unsigned)ceil_div(H, kLT), (unsigned)C);
    const int64_t nblk = (int64_t)grid.x * grid.y * grid.z;
    const int want = d_rgb != nullptr;
    prof_begin(ST_LOSS, st);
    loss_fwd_kernel<<<grid, 256, 0, st>>>(rgb, depth, gt_rgb, gt_rgbf, gt_depth, W, H, C, dmaps,
                                          partial, want);
    loss_finalize<<<1, 256, 0, st>>>(partial, nblk, acc, W, H, C, ls, ld, loss_out);
    if (want)
        loss_bwd_kernel<<<grid, 256, 0, st>>>(rgb, depth, gt_rgb, gt_rgbf, gt_depth, W, H, C, dmaps,
                                              acc, ls, ld, d_rgb, d_depth);
    prof_end(ST_LOSS, st);
    count_launches(want ? 3 : 2);
    SM_CHECK_LAUNCH("loss_forward_backward");
    return SM_OK;
}

}  // namespace sm
