/*
 * splatmap_cuda.h -- C ABI of libsplatmap_cuda.so, the B200 (sm_100a) data
 * plane of the chunked-3DGS mapping hot path.
 *
 * The reference (splatmap, pure Python + numba) has no FFI; the entry points
 * below are what its Python API would bind for the hot path.  Each cites the
 * reference function whose work it replaces (paths relative to
 * /root/reference/pkg/src/splatmap/).  See INTEGRATION.md for the ctypes
 * binding a maintainer would add to the reference.
 *
 * Conventions
 *  - Every pointer argument is a DEVICE pointer unless documented as host.
 *  - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *  - Calls are asynchronous on `stream`; they never allocate: scratch comes
 *    from a caller-owned workspace sized by the matching *_workspace_size().
 *  - Return value: SM_OK (0) or an SM_ERR_* code; sm_last_error() gives the
 *    thread-local message.  Codes map to splatmap's SplatmapError subclasses
 *    (errors.py) in the Python layer.
 *  - Gaussian parameters live in "param records": 16 floats per Gaussian,
 *    [px py pz | qw qx qy qz | sx sy sz | opacity | sh0_r sh0_g sh0_b | pad pad]
 *    (the 14 trainable scalars of core.py:165-190, SH degree-0 at sh[0,16,32]).
 *  - Not re-entrant per workspace (one render in flight per workspace).
 */
#ifndef SPLATMAP_CUDA_H
#define SPLATMAP_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SM_ABI_VERSION 1
#define SM_PARAM_STRIDE 16
#define SM_TILE 16

enum {
    SM_OK = 0,
    SM_ERR_INVALID = 1,    /* bad argument                       -> ValueError       */
    SM_ERR_CUDA = 2,       /* CUDA runtime failure               -> DeviceFailure    */
    SM_ERR_WORKSPACE = 3,  /* workspace too small                -> ValueError       */
    SM_ERR_RANGE = 4,      /* chunk coordinate out of +-2^20     -> OutOfRange       */
    SM_ERR_CORRUPT = 5,    /* malformed chunk record             -> CorruptChunk     */
    SM_ERR_DIMENSION = 6   /* image size mismatch / too small    -> DimensionMismatch*/
};

/* Pinhole camera of one view.  r_wc = quat_to_matrix(pose.rotation) (core.py:88),
 * row-major, world<-camera; t = camera centre (core.py:111-127);
 * intrinsics as core.py:145-162. */
typedef struct sm_camera {
    double r_wc[9];
    double t[3];
    double fx, fy, cx, cy, near_plane, far_plane;
    int32_t width, height;
} sm_camera;

/* Static capacities a render workspace is carved for. */
typedef struct sm_render_dims {
    int64_t max_gaussians;   /* >= n of every render using this workspace   */
    int64_t max_instances;   /* tile-instance capacity (overflow is flagged) */
    int32_t width, height;
} sm_render_dims;

/* Device-side counters at the head of every render workspace (readable with
 * one 64-byte D2H copy after the stream is synchronised). */
typedef struct sm_render_counters {
    uint32_t n_instances;    /* tile instances emitted by the last forward   */
    uint32_t overflow;       /* 1 if n_instances > max_instances (no image)  */
    uint32_t n_visible;      /* Gaussians with >= 1 tile                     */
    uint32_t n_fallback;     /* not maintained (reserved)                    */
    uint32_t reserved[12];   /* [0] sort count, [1] big-splat queue length,
                              * [2] instances the last backward revisited    */
} sm_render_counters;

typedef struct sm_adam_config {
    float lr[14];            /* per trainable scalar (record order)           */
    float beta1, beta2, eps;
    float min_scale;         /* scales are clamped to >= min_scale            */
} sm_adam_config;

int sm_abi_version(void);
const char *sm_last_error(void);
int sm_device_sm_count(void);

/* ---------------------------------------------------------------- render
 * Replaces renderloss.render_arrays (renderloss.py:170-218) incl. the numba
 * _composite kernel (renderloss.py:106-152): EWA projection + SH0 colour (K2),
 * global stable depth order + tile binning + radix sort + tile ranges (K3),
 * front-to-back compositing (K4).  Output images are fp32, row-major:
 * rgb (H,W,3), depth (H,W), alpha (H,W) -- RenderedFrame (renderloss.py:29-33).
 * `slots` (nullable) maps visible index i -> param record; NULL = identity. */
int64_t sm_render_workspace_size(const sm_render_dims *dims);
int sm_render_forward(const float *params, const int32_t *slots, int64_t n,
                      const sm_camera *cam /* host */, const sm_render_dims *dims /* host */,
                      void *workspace, int64_t workspace_bytes,
                      float *out_rgb, float *out_depth, float *out_alpha, void *stream);

/* sm_render_forward with a caller-kept tile schedule for one view (no
 * reference counterpart; renderloss.py:170 render_arrays is the computation).
 * tile_order: device uint32 [tiles_x * tiles_y], a permutation of the tile
 * indices (identity for a view's first render).  The compositing CTAs take
 * their tiles in this order, and on return it holds this render's
 * longest-first order (tiles ranked by the instances the backward revisits),
 * so re-rendering the same view (a mapping keyframe) starts its heaviest
 * tiles first.  Outputs are identical to sm_render_forward for any
 * permutation: tiles are independent. */
int sm_render_forward_ordered(const float *params, const int32_t *slots, int64_t n,
                              const sm_camera *cam, const sm_render_dims *dims,
                              void *workspace, int64_t workspace_bytes, uint32_t *tile_order,
                              float *out_rgb, float *out_depth, float *out_alpha, void *stream);

/* Reverse-order backward of the last sm_render_forward on this workspace
 * (no reference counterpart: the reference is forward-only, README.md:125).
 * Upstream grads d_* are (H,W,3)/(H,W)/(H,W) fp32, each nullable (= zero).
 * grads: param-record-shaped [slot][16] buffer, ACCUMULATED (+=). */
int sm_render_backward(const float *params, const int32_t *slots, int64_t n,
                       const sm_camera *cam, const sm_render_dims *dims,
                       void *workspace, int64_t workspace_bytes,
                       const float *d_rgb, const float *d_depth, const float *d_alpha,
                       float *grads, void *stream);

/* sm_render_backward + the K7 Adam step fused into its last stage (the
 * single-keyframe mapping step, sim.py:319-370 with the nudge replaced by
 * training): each active splat's gradient goes straight from the chain rule
 * into its Adam update (params / adam_m / adam_v updated in place, the
 * same arithmetic as sm_adam_step, bit for bit), splats the view does not
 * reach get their zero-gradient step; no gradient buffer.  skip_flag as in
 * sm_adam_step. */
int sm_render_backward_adam(float *params, const int32_t *slots, int64_t n,
                            const sm_camera *cam, const sm_render_dims *dims,
                            void *workspace, int64_t workspace_bytes,
                            const float *d_rgb, const float *d_depth, const float *d_alpha,
                            float *adam_m, float *adam_v, const sm_adam_config *cfg /* host */,
                            const uint32_t *skip_flag, void *stream);

/* Tile binning keeps only the tiles a splat's q <= 9 ellipse reaches (on, the
 * default) or every tile of its 3-sigma box (off).  Images and gradients are
 * bit-identical either way (the dropped tiles are ones the compositor skips
 * anyway); the switch exists so tests can prove that.  Process-global; takes
 * effect at the next sm_render_forward (CUDA graphs keep their captured value). */
void sm_set_ellipse_cull(int on);

/* Diagnostics: byte offset inside a render workspace of an internal buffer
 * (SM_WS_TILE_RANGES: uint32 [n_tiles][2] instance range per tile;
 * SM_WS_PIX_LAST: int32 [H*W] position of each pixel's last contributor in its
 * tile's instance list; SM_WS_DEPTH_ORDER: the stable depth order, kept
 * Gaussians first = np.argsort(z, kind="stable"), renderloss.py:202), or -1.
 * Valid after sm_render_forward. */
#define SM_WS_TILE_RANGES 0
#define SM_WS_PIX_LAST 1
#define SM_WS_DEPTH_ORDER 2   /* uint32 [n]: depth rank -> visible index */
#define SM_WS_RANK_TILES 3    /* uint32 [n]: kept tiles per depth rank   */
#define SM_WS_TILE_KEYS 4     /* [counters.n_instances] sorted instance keys
                               * (tile << rank_bits) | depth rank, uint32 or
                               * uint64 (sm_render_key_layout)            */
int64_t sm_render_ws_offset(const sm_render_dims *dims, int which);
/* Bit layout of the SM_WS_TILE_KEYS keys of a workspace (host-only). */
int sm_render_key_layout(const sm_render_dims *dims, int32_t *rank_bits, int32_t *key_bytes);

/* ------------------------------------------------------------------ loss
 * renderloss.total_loss / image_loss / ssim / depth_loss (renderloss.py:226-274):
 * (1-ls)*L1 + ls*(1-SSIM 11x11 sigma 1.5, 5-px crop, channel mean)
 * + ld*mean_{gt_depth>0}|D-Dgt|, and its gradient w.r.t. rgb/depth.
 * Images are (H,W,C) fp32 row-major, C = channels (1..4).  Ground truth is
 * either the keyframe's 8-bit RGB (gt_rgb_u8, core.py:262-267 keeps k/255)
 * or fp32 (gt_rgb_f32); exactly one non-NULL.  depth/gt_depth nullable
 * (no depth term).  loss_out: device float[4] = {total, l1, ssim, depth_l1}.
 * d_rgb/d_depth nullable (forward only). */
int64_t sm_loss_workspace_size(int32_t width, int32_t height);
int sm_loss_forward_backward(const float *rgb, const float *depth, const uint8_t *gt_rgb_u8,
                             const float *gt_rgb_f32, const float *gt_depth, int32_t width,
                             int32_t height, int32_t channels, float lambda_s, float lambda_depth,
                             void *workspace, int64_t workspace_bytes, float *loss_out,
                             float *d_rgb, float *d_depth, void *stream);

/* ------------------------------------------------------------------ adam
 * Fused Adam on the active set (replaces the _nudge_visible stand-in,
 * sim.py:280-317).  For each slot in `slots[0:n]`: Adam on the 14 scalars
 * (per-Gaussian step count in m[slot*16+14]), then quaternion
 * renormalisation, scale >= min_scale, opacity clamp to [0,1] (core.py
 * invariants 186-190), and grads[slot] is zeroed.  skip_flag (nullable,
 * device uint32) suppresses the update when non-zero (render overflow). */
int sm_adam_step(float *params, float *m, float *v, float *grads, const int32_t *slots,
                 int64_t n, const sm_adam_config *cfg /* host */, const uint32_t *skip_flag,
                 void *stream);

/* Data-parallel exchange (no reference counterpart -- the
 * reference is single-process).  sm_pack_grads gathers the gradient records
 * of the active set into packed[i] = grads[slots[i]] ([n][16] floats, the
 * buffer the ranks sum with one NCCL all-reduce) and zeroes those slab rows;
 * sm_adam_step_packed is sm_adam_step reading gradient i from packed[i]
 * (bit-identical to sm_adam_step on the same sums). */
int sm_pack_grads(float *grads, const int32_t *slots, int64_t n, float *packed, void *stream);
int sm_adam_step_packed(float *params, float *m, float *v, const float *packed_grads,
                        const int32_t *slots, int64_t n, const sm_adam_config *cfg /* host */,
                        const uint32_t *skip_flag, void *stream);

/* --------------------------------------------------------------- culling
 * Per-chunk frustum + distance test, brute force over a chunk table; equal
 * to culling.visible_chunks (culling.py:134-182) / _chunk_passes (126-131):
 * p-vertex OUTSIDE test against 6 planes (host-extracted with
 * extract_frustum, culling.py:80-101) and nearest-point distance, fp64
 * without contraction.  coords int32 [n][3]; planes host double[6][4];
 * visible_out uint8 [n]. */
int sm_cull_chunks(const int32_t *coords, int64_t n, const double *planes /* host */,
                   const double *cam_center /* host */, double max_distance, double chunk_size,
                   uint8_t *visible_out, void *stream);

/* grid.encode_positions (grid.py:110-121) on float32-canonical positions:
 * floor((p + s/2)/s) in fp64 then 21-bit packing.  err_out (device int64)
 * receives the first offending index or -1. */
int sm_encode_positions(const float *params /* records */, int64_t n, double chunk_size,
                        uint64_t *ids_out, int64_t *err_out, void *stream);

/* Active-set expansion: segments (offset, count) in visible-chunk order
 * (sorted chunk ids, sim.py:236-253) -> slots[0:total]. */
int sm_expand_segments(const int64_t *seg_offset, const int64_t *seg_count,
                       const int64_t *seg_prefix, int64_t n_segments, int64_t total,
                       int32_t *slots_out, void *stream);

/* ----------------------------------------------------------------- codec
 * .dcg record codec (diskformat.py:51-66 layout, pack_chunk 86-109,
 * unpack_chunk 137-186) between AoS records and device SoA: param records
 * [16], SH rest [45] (sh indices 1..15, 17..31, 33..47) and Adam moments.
 * stride 240: opt_len = 0 (fresh Adam state, the b"" contract of
 * loopclose.py:241); stride 360: a 120-byte opt_state tail
 * "ADM1" | step u32 | m[14] f32 | v[14] f32.  Unpack validates the record
 * invariants (diskformat.py:153 -> core.py:208-221) and the tail; err_out
 * (device int64) receives the first bad record index or -1.  With params,
 * sh_rest, adam_m and adam_v all NULL it only validates (the streamer checks
 * a staged chunk on its copy stream, then queues the unpack behind the
 * render).  Foreign opt_state payloads take the host path. */
int sm_chunk_unpack(const uint8_t *records, int64_t n, int64_t stride, float *params,
                    float *sh_rest, float *adam_m, float *adam_v, int64_t *err_out, void *stream);
int sm_chunk_pack(const float *params, const float *sh_rest, const float *adam_m,
                  const float *adam_v, int64_t n, int64_t stride, uint8_t *records, void *stream);

/* ---------------------------------------------------------------- ingest
 * splatmap sample.py on the device (fp64, like the reference).
 * sm_log_scores: |LoG * luma| of an (H,W,3) image (sample.py:63-75 log_norm
 * before its max-normalisation; luma 0.299 r + 0.587 g + 0.114 b, zero
 * padding, taps = host log_kernel(sigma, radius) (2r+1)^2 doubles, radius
 * <= 3), written to scores_out [H*W] fp64, and the image's peak to *peak_out
 * (device uint64, the fp64 bit pattern).  rgb_kind: SM_RGB_U8 (the
 * keyframe's 8-bit colours, k/255 in float32 as core.py:262-267),
 * SM_RGB_F32 or SM_RGB_F64.
 * sm_sampling_probability: max(a / peak_a - b / peak_b, 0) (sample.py:78-84
 * with log_norm's normalisation; a peak of 0 leaves its map unscaled);
 * scores_rendered / peak_rendered NULL: the normalised input scores.
 * sm_lift_pixels: sample.py:104-146 lift_to_gaussians for k (row, col)
 * int32 pairs: float32-canonical param records [k][16] and valid_out[k] =
 * depth > 0 (the caller keeps the valid ones in order).  r_wc / t host. */
#define SM_RGB_U8 0
#define SM_RGB_F32 1
#define SM_RGB_F64 2
int sm_log_scores(const void *rgb, int32_t rgb_kind, int32_t width, int32_t height,
                  const double *taps /* host */, int32_t radius, double *scores_out, uint64_t *peak_out,
                  void *stream);
int sm_sampling_probability(const double *scores_input, const uint64_t *peak_input,
                            const double *scores_rendered, const uint64_t *peak_rendered, int64_t n,
                            double *ps_out, void *stream);
int sm_lift_pixels(const int32_t *pixels, int64_t k, const float *depth, const void *rgb,
                   int32_t rgb_kind, int32_t width, int32_t height, const double *r_wc /* host */,
                   const double *t /* host */, double fx, double fy, double cx, double cy,
                   double scale_factor, float opacity, float *params_out, int32_t *valid_out,
                   void *stream);

/* ---------------------------------------------------------- loop closure
 * loopclose.py on the device.
 * sm_transform_rows: _transform_chunk (loopclose.py:146-150) on n param
 * records in place -- p' = R p + t, q' = normalize(q_t * q) (core.py:76-87,
 * 141-142, 309-314) in fp64 from the float32 values, stored float32
 * (storage_canonical); scale, opacity, SH and Adam state untouched.
 * rotation (row-major 3x3), translation, quaternion (w,x,y,z) are host.
 * sm_reset_rows: refine_reset (loopclose.py:228-245) on n rows: opacity <-
 * `opacity`, Adam moments and step count zeroed (opt_state = b""). */
int sm_transform_rows(float *params, int64_t n, const double *rotation /* host */,
                      const double *translation /* host */, const double *quaternion /* host */,
                      void *stream);
int sm_reset_rows(float *params, float *adam_m, float *adam_v, int64_t n, float opacity, void *stream);

/* .dkf keyframe file (diskformat.py:198-216 pack_keyframe) assembled on the
 * device from the keyframe tier's HBM copy: header (host, 140 bytes, the
 * <4sIQ7d6dIIdI layout) | rgb_u8 (H,W,3) | depth f32 (H,W); out receives
 * 140 + 7 W H bytes (device memory, or pinned host memory: the write-behind
 * has the kernel fill its pinned staging buffer directly).  Byte-identical
 * to pack_keyframe. */
int sm_keyframe_pack(const uint8_t *header /* host */, const uint8_t *rgb_u8, const float *depth,
                     int32_t width, int32_t height, uint8_t *out, void *stream);

/* ------------------------------------------------------------ profiling
 * No reference counterpart (the reference bills a deterministic cost model,
 * sim.py:53-57).  When enabled, each stage (project_fwd, depth_sort,
 * bin_emit, tile_sort, composite_fwd, loss, composite_bwd, project_bwd,
 * adam, cull, codec) records a CUDA event pair on its launch stream;
 * collect() blocks on them and returns per-stage summed ms and call counts
 * (then resets).  sm_launch_count() = kernels launched by this library. */
void sm_profile_enable(int on);
long long sm_launch_count(void);
int sm_profile_stage_count(void);
const char *sm_profile_stage_name(int stage);
int sm_profile_collect(double *ms_out, long long *calls_out);
/* CUDA-graph capture of the step: stage events and kernel counts recorded
 * while capturing are filed under the returned graph id; after each replay
 * completes, sm_profile_graph_replayed(gid) accounts them again. */
int sm_profile_capture_begin(void);
void sm_profile_capture_end(void);
void sm_profile_graph_replayed(int gid);
void sm_profile_graph_free(int gid);
long long sm_profile_graph_timing_errors(void);

#ifdef __cplusplus
}
#endif
#endif /* SPLATMAP_CUDA_H */
