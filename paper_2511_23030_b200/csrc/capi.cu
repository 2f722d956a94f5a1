// extern "C" entry points of libsplatmap_cuda.so (declared in include/splatmap_cuda.h).
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "adam.cuh"
#include "render.cuh"

namespace sm {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_status(cudaError_t e, const char *what) {
    set_error("%s: CUDA error %d (%s)", what, (int)e, cudaGetErrorString(e));
    return SM_ERR_CUDA;
}

int64_t loss_workspace_size(int W, int H);
extern int g_ellipse_cull;
int loss_forward_backward(const float *, const float *, const uint8_t *, const float *, const float *,
                          int, int, int, float, float, void *, int64_t, float *, float *, float *,
                          cudaStream_t);
int adam_step(float *, float *, float *, float *, const int32_t *, int64_t, const sm_adam_config &,
              const uint32_t *, const float *, cudaStream_t);
int pack_grads(float *, const int32_t *, int64_t, float *, cudaStream_t);
int transform_rows(float *, int64_t, const double *, const double *, const double *, cudaStream_t);
int reset_rows(float *, float *, float *, int64_t, float, cudaStream_t);
int keyframe_pack(const uint8_t *, const uint8_t *, const float *, int64_t, uint8_t *, cudaStream_t);
int log_scores(const void *, int, int, int, const double *, int, double *, unsigned long long *, cudaStream_t);
int sampling_probability(const double *, const unsigned long long *, const double *, const unsigned long long *,
                         int64_t, double *, cudaStream_t);
int lift_pixels(const int32_t *, int64_t, const float *, const void *, int, int, int, const double *,
                const double *, double, double, double, double, double, float, float *, int32_t *, cudaStream_t);
int cull_chunks(const int32_t *, int64_t, const double *, const double *, double, double, uint8_t *,
                cudaStream_t);
int encode_positions(const float *, int64_t, double, uint64_t *, int64_t *, cudaStream_t);
int expand_segments(const int64_t *, const int64_t *, const int64_t *, int64_t, int64_t, int32_t *,
                    cudaStream_t);
int chunk_unpack(const uint8_t *, int64_t, int64_t, float *, float *, float *, float *, int64_t *,
                 cudaStream_t);
int chunk_pack(const float *, const float *, const float *, const float *, int64_t, int64_t,
               uint8_t *, cudaStream_t);

}  // namespace sm

using namespace sm;

#define SM_STREAM(s) reinterpret_cast<cudaStream_t>(s)

extern "C" {

int sm_abi_version(void) { return SM_ABI_VERSION; }

const char *sm_last_error(void) { return g_err; }

int sm_device_sm_count(void) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return n;
}

int64_t sm_render_workspace_size(const sm_render_dims *dims) {
    if (!dims) return -1;
    return render_layout(*dims).total;
}

int sm_render_forward(const float *params, const int32_t *slots, int64_t n, const sm_camera *cam,
                      const sm_render_dims *dims, void *workspace, int64_t workspace_bytes,
                      float *out_rgb, float *out_depth, float *out_alpha, void *stream) {
    if (!cam || !dims || !workspace || !out_rgb || !out_depth || !out_alpha || (n > 0 && !params)) {
        set_error("sm_render_forward: null argument");
        return SM_ERR_INVALID;
    }
    return render_forward(params, slots, n, *cam, *dims, workspace, workspace_bytes, out_rgb,
                          out_depth, out_alpha, nullptr, SM_STREAM(stream));
}

int sm_render_forward_ordered(const float *params, const int32_t *slots, int64_t n, const sm_camera *cam,
                              const sm_render_dims *dims, void *workspace, int64_t workspace_bytes,
                              uint32_t *tile_order, float *out_rgb, float *out_depth, float *out_alpha,
                              void *stream) {
    if (!cam || !dims || !workspace || !tile_order || !out_rgb || !out_depth || !out_alpha ||
        (n > 0 && !params)) {
        set_error("sm_render_forward_ordered: null argument");
        return SM_ERR_INVALID;
    }
    return render_forward(params, slots, n, *cam, *dims, workspace, workspace_bytes, out_rgb,
                          out_depth, out_alpha, tile_order, SM_STREAM(stream));
}

int sm_render_backward(const float *params, const int32_t *slots, int64_t n, const sm_camera *cam,
                       const sm_render_dims *dims, void *workspace, int64_t workspace_bytes,
                       const float *d_rgb, const float *d_depth, const float *d_alpha, float *grads,
                       void *stream) {
    if (!cam || !dims || !workspace || (n > 0 && (!params || !grads))) {
        set_error("sm_render_backward: null argument");
        return SM_ERR_INVALID;
    }
    return render_backward(params, slots, n, *cam, *dims, workspace, workspace_bytes, d_rgb, d_depth,
                           d_alpha, grads, nullptr, SM_STREAM(stream));
}

int sm_render_backward_adam(float *params, const int32_t *slots, int64_t n, const sm_camera *cam,
                            const sm_render_dims *dims, void *workspace, int64_t workspace_bytes,
                            const float *d_rgb, const float *d_depth, const float *d_alpha, float *adam_m,
                            float *adam_v, const sm_adam_config *cfg, const uint32_t *skip_flag, void *stream) {
    if (!cam || !dims || !workspace || !cfg || (n > 0 && (!params || !adam_m || !adam_v))) {
        set_error("sm_render_backward_adam: null argument");
        return SM_ERR_INVALID;
    }
    AdamFuse af;
    af.m = reinterpret_cast<float4 *>(adam_m);
    af.v = reinterpret_cast<float4 *>(adam_v);
    af.skip = skip_flag;
    af.c = adam_dev(*cfg);
    return render_backward(params, slots, n, *cam, *dims, workspace, workspace_bytes, d_rgb, d_depth,
                           d_alpha, nullptr, &af, SM_STREAM(stream));
}

void sm_set_ellipse_cull(int on) { g_ellipse_cull = on ? 1 : 0; }

int64_t sm_render_ws_offset(const sm_render_dims *dims, int which) {
    if (!dims) return -1;
    const RenderLayout L = render_layout(*dims);
    switch (which) {
        case SM_WS_TILE_RANGES: return L.o_ranges;
        case SM_WS_PIX_LAST: return L.o_pix_last;
        case SM_WS_DEPTH_ORDER: return L.o_order0;
        case SM_WS_RANK_TILES: return L.o_tcount_r;
        case SM_WS_TILE_KEYS: return L.tile_passes & 1 ? L.o_ikey1 : L.o_ikey0;
        default: return -1;
    }
}

int sm_render_key_layout(const sm_render_dims *dims, int32_t *rank_bits, int32_t *key_bytes) {
    if (!dims || !rank_bits || !key_bytes) {
        set_error("sm_render_key_layout: null argument");
        return SM_ERR_INVALID;
    }
    const RenderLayout L = render_layout(*dims);
    *rank_bits = L.rank_bits;
    *key_bytes = L.key_bytes;
    return SM_OK;
}

int64_t sm_loss_workspace_size(int32_t width, int32_t height) { return loss_workspace_size(width, height); }

int sm_loss_forward_backward(const float *rgb, const float *depth, const uint8_t *gt_rgb_u8,
                             const float *gt_rgb_f32, const float *gt_depth, int32_t width,
                             int32_t height, int32_t channels, float lambda_s, float lambda_depth,
                             void *workspace, int64_t workspace_bytes, float *loss_out, float *d_rgb,
                             float *d_depth, void *stream) {
    if (!rgb || !workspace || !loss_out) {
        set_error("sm_loss_forward_backward: null argument");
        return SM_ERR_INVALID;
    }
    return loss_forward_backward(rgb, depth, gt_rgb_u8, gt_rgb_f32, gt_depth, width, height, channels,
                                 lambda_s, lambda_depth, workspace, workspace_bytes, loss_out, d_rgb,
                                 d_depth, SM_STREAM(stream));
}

int sm_adam_step(float *params, float *m, float *v, float *grads, const int32_t *slots, int64_t n,
                 const sm_adam_config *cfg, const uint32_t *skip_flag, void *stream) {
    if (!cfg || (n > 0 && (!params || !m || !v || !grads))) {
        set_error("sm_adam_step: null argument");
        return SM_ERR_INVALID;
    }
    return adam_step(params, m, v, grads, slots, n, *cfg, skip_flag, nullptr, SM_STREAM(stream));
}

int sm_pack_grads(float *grads, const int32_t *slots, int64_t n, float *packed, void *stream) {
    if (n > 0 && (!grads || !packed)) {
        set_error("sm_pack_grads: null argument");
        return SM_ERR_INVALID;
    }
    return pack_grads(grads, slots, n, packed, SM_STREAM(stream));
}

int sm_adam_step_packed(float *params, float *m, float *v, const float *packed_grads, const int32_t *slots,
                        int64_t n, const sm_adam_config *cfg, const uint32_t *skip_flag, void *stream) {
    if (!cfg || (n > 0 && (!params || !m || !v || !packed_grads))) {
        set_error("sm_adam_step_packed: null argument");
        return SM_ERR_INVALID;
    }
    return adam_step(params, m, v, nullptr, slots, n, *cfg, skip_flag, packed_grads, SM_STREAM(stream));
}

int sm_cull_chunks(const int32_t *coords, int64_t n, const double *planes, const double *cam_center,
                   double max_distance, double chunk_size, uint8_t *visible_out, void *stream) {
    if (!planes || !cam_center || (n > 0 && (!coords || !visible_out))) {
        set_error("sm_cull_chunks: null argument");
        return SM_ERR_INVALID;
    }
    return cull_chunks(coords, n, planes, cam_center, max_distance, chunk_size, visible_out,
                       SM_STREAM(stream));
}

int sm_encode_positions(const float *params, int64_t n, double chunk_size, uint64_t *ids_out,
                        int64_t *err_out, void *stream) {
    if (!err_out || (n > 0 && (!params || !ids_out))) {
        set_error("sm_encode_positions: null argument");
        return SM_ERR_INVALID;
    }
    return encode_positions(params, n, chunk_size, ids_out, err_out, SM_STREAM(stream));
}

int sm_expand_segments(const int64_t *seg_offset, const int64_t *seg_count, const int64_t *seg_prefix,
                       int64_t n_segments, int64_t total, int32_t *slots_out, void *stream) {
    return expand_segments(seg_offset, seg_count, seg_prefix, n_segments, total, slots_out,
                           SM_STREAM(stream));
}

int sm_chunk_unpack(const uint8_t *records, int64_t n, int64_t stride, float *params, float *sh_rest,
                    float *adam_m, float *adam_v, int64_t *err_out, void *stream) {
    const bool validate_only = !params && !sh_rest && !adam_m && !adam_v;
    if (!err_out || (n > 0 && (!records || (!validate_only && (!params || !sh_rest || !adam_m || !adam_v))))) {
        set_error("sm_chunk_unpack: null argument");
        return SM_ERR_INVALID;
    }
    return chunk_unpack(records, n, stride, params, sh_rest, adam_m, adam_v, err_out,
                        SM_STREAM(stream));
}

int sm_chunk_pack(const float *params, const float *sh_rest, const float *adam_m, const float *adam_v,
                  int64_t n, int64_t stride, uint8_t *records, void *stream) {
    if (n > 0 && (!params || !sh_rest || !adam_m || !adam_v || !records)) {
        set_error("sm_chunk_pack: null argument");
        return SM_ERR_INVALID;
    }
    return chunk_pack(params, sh_rest, adam_m, adam_v, n, stride, records, SM_STREAM(stream));
}


int sm_log_scores(const void *rgb, int32_t rgb_kind, int32_t width, int32_t height, const double *taps,
                  int32_t radius, double *scores_out, uint64_t *peak_out, void *stream) {
    if (!rgb || !taps || !scores_out || !peak_out || rgb_kind < SM_RGB_U8 || rgb_kind > SM_RGB_F64) {
        set_error("sm_log_scores: null argument or bad rgb_kind");
        return SM_ERR_INVALID;
    }
    return log_scores(rgb, rgb_kind, width, height, taps, radius, scores_out,
                      reinterpret_cast<unsigned long long *>(peak_out), SM_STREAM(stream));
}

int sm_sampling_probability(const double *scores_input, const uint64_t *peak_input,
                            const double *scores_rendered, const uint64_t *peak_rendered, int64_t n,
                            double *ps_out, void *stream) {
    if (n > 0 && (!scores_input || !peak_input || !ps_out || (!scores_rendered != !peak_rendered))) {
        set_error("sm_sampling_probability: null argument");
        return SM_ERR_INVALID;
    }
    return sampling_probability(scores_input, reinterpret_cast<const unsigned long long *>(peak_input),
                                scores_rendered, reinterpret_cast<const unsigned long long *>(peak_rendered), n,
                                ps_out, SM_STREAM(stream));
}

int sm_lift_pixels(const int32_t *pixels, int64_t k, const float *depth, const void *rgb, int32_t rgb_kind,
                   int32_t width, int32_t height, const double *r_wc, const double *t, double fx, double fy,
                   double cx, double cy, double scale_factor, float opacity, float *params_out,
                   int32_t *valid_out, void *stream) {
    if (k > 0 && (!pixels || !depth || !rgb || !r_wc || !t || !params_out || !valid_out || rgb_kind < SM_RGB_U8 ||
                  rgb_kind > SM_RGB_F64)) {
        set_error("sm_lift_pixels: null argument or bad rgb_kind");
        return SM_ERR_INVALID;
    }
    return lift_pixels(pixels, k, depth, rgb, rgb_kind, width, height, r_wc, t, fx, fy, cx, cy, scale_factor,
                       opacity, params_out, valid_out, SM_STREAM(stream));
}

int sm_transform_rows(float *params, int64_t n, const double *rotation, const double *translation,
                      const double *quaternion, void *stream) {
    if (n > 0 && (!params || !rotation || !translation || !quaternion)) {
        set_error("sm_transform_rows: null argument");
        return SM_ERR_INVALID;
    }
    return transform_rows(params, n, rotation, translation, quaternion, SM_STREAM(stream));
}

int sm_reset_rows(float *params, float *adam_m, float *adam_v, int64_t n, float opacity, void *stream) {
    if (n > 0 && (!params || !adam_m || !adam_v)) {
        set_error("sm_reset_rows: null argument");
        return SM_ERR_INVALID;
    }
    return reset_rows(params, adam_m, adam_v, n, opacity, SM_STREAM(stream));
}

int sm_keyframe_pack(const uint8_t *header, const uint8_t *rgb_u8, const float *depth, int32_t width,
                     int32_t height, uint8_t *out, void *stream) {
    if (!header || !rgb_u8 || !depth || !out || width < 1 || height < 1) {
        set_error("sm_keyframe_pack: null argument or empty image");
        return SM_ERR_INVALID;
    }
    return keyframe_pack(header, rgb_u8, depth, (int64_t)width * height, out, SM_STREAM(stream));
}

}  // extern "C"
