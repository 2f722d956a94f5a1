// Render pipeline shared declarations: workspace layout + fp64 projection.
#pragma once
#include "common.cuh"

namespace sm {

constexpr int kG2dStride = 12;   // per-rank 2D grads: u v ia ib ic op r g b z - -
constexpr uint32_t kEmitSmall = 32;   // splats with more box tiles are emitted / gathered per warp

// Tiles of the 3-sigma box.  The small / big split is taken on this count, not
// on the kept (ellipse) count, so a splat's gradient is summed by the same
// path, in the same order, whether or not tiles were culled.
__device__ __forceinline__ uint32_t bbox_tiles(const ProjRec &g) {
    return (uint32_t)((rec_x1(g) / kTile - rec_x0(g) / kTile + 1) * (rec_y1(g) / kTile - rec_y0(g) / kTile + 1));
}

// Small splats (<= kEmitSmall box tiles) carry their kept tiles as a bit mask
// over the box in row-major order (bit (ty - ty0) * ntx + tx - tx0), computed
// once by the projection: emission walks the set bits, the kept index of a
// tile is the popcount below its bit.
__device__ __forceinline__ uint32_t small_mask(const RowSpan &sp) {
    const int ntx = sp.tx1 - sp.tx0 + 1;
    uint32_t m = 0;
    for (int ty = sp.ty0, bit = 0; ty <= sp.ty1; ty++, bit += ntx) {
        int c0, c1;
        sp.row(ty, c0, c1);
        if (c1 >= c0) m |= (0xffffffffu >> (31 - (c1 - c0))) << (bit + c0 - sp.tx0);
    }
    return m;
}

// Big splats are handled by a 256-thread block: thread i evaluates tile row
// tyb + i (RowSpan), a block scan turns the row counts into kept-index
// offsets, then warp w walks rows w, w + 8, ... with its lanes across columns.
constexpr int kBigThreads = 256;
struct BigRowTable {
    int c0[kBigThreads], c1[kBigThreads];
    uint32_t off[kBigThreads];
    uint32_t wsum[kBigThreads / 32];
};

// Fills rows tyb .. tyb + 255 (clipped to the box); returns base + their count.
__device__ __forceinline__ uint32_t fill_row_table(const RowSpan &sp, int tyb, uint32_t base,
                                                   BigRowTable &t) {
    __syncthreads();   // the previous user of the table is done
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ty = tyb + (int)threadIdx.x;
    int c0 = 0, c1 = -1;
    if (ty <= sp.ty1) sp.row(ty, c0, c1);
    const uint32_t cnt = c1 >= c0 ? (uint32_t)(c1 - c0 + 1) : 0u;
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) t.wsum[warp] = x;
    __syncthreads();
    uint32_t pre = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kBigThreads / 32; w++) {
        const uint32_t s = t.wsum[w];
        pre += w < warp ? s : 0u;
        total += s;
    }
    t.c0[threadIdx.x] = c0;
    t.c1[threadIdx.x] = c1;
    t.off[threadIdx.x] = base + pre + x - cnt;
    __syncthreads();
    return base + total;
}

struct RenderLayout {
    int tiles_x, tiles_y;
    int64_t n_tiles;
    int rank_bits, tile_bits;
    int key_bytes;   // tile-instance keys: 4 while rank_bits + tile_bits <= 32, else 8
    int depth_passes, tile_passes;
    int64_t sort_blocks;
    int64_t o_counters, o_rec, o_rec_sorted, o_p64, o_dkey0, o_dkey1, o_order0, o_order1;
    int64_t o_tcount, o_tcount_r, o_tmask, o_tmask_r, o_toff, o_ikey0, o_ikey1, o_ranges;
    int64_t o_pix_cd, o_pix_t, o_pix_tlast, o_pix_last, o_g2d, o_sort_hist, o_scan;
    int64_t o_gbuf, o_tile_hor, o_tile_work, o_tile_order;
    int64_t total;
};

RenderLayout render_layout(const sm_render_dims &d);

struct RenderBufs {
    sm_render_counters *ctr;
    ProjRec *rec, *rec_sorted;
    Proj64 *p64;
    unsigned long long *dkey0, *dkey1;
    uint32_t *order0, *order1, *tcount, *tcount_r, *tmask, *tmask_r, *toff, *ranges;
    void *ikey0, *ikey1;   // uint32_t or unsigned long long (key_bytes)
    float4 *pix_cd;
    float *pix_t, *pix_tlast;
    int32_t *pix_last;
    float *g2d;
    uint32_t *sort_hist, *scan;
    float *gbuf;         // per-instance gradient slots [max_instances][12] (backward)
    int32_t *tile_hor;   // per-tile horizon rank (backward)
    uint32_t *tile_work;    // per-tile instances the forward composited (backward's work)
    uint32_t *tile_order;   // tiles by descending work: the backward's launch order
};

inline RenderBufs render_bufs(void *ws, const RenderLayout &L) {
    char *b = static_cast<char *>(ws);
    RenderBufs r;
    r.ctr = reinterpret_cast<sm_render_counters *>(b + L.o_counters);
    r.rec = reinterpret_cast<ProjRec *>(b + L.o_rec);
    r.rec_sorted = reinterpret_cast<ProjRec *>(b + L.o_rec_sorted);
    r.p64 = reinterpret_cast<Proj64 *>(b + L.o_p64);
    r.dkey0 = reinterpret_cast<unsigned long long *>(b + L.o_dkey0);
    r.dkey1 = reinterpret_cast<unsigned long long *>(b + L.o_dkey1);
    r.order0 = reinterpret_cast<uint32_t *>(b + L.o_order0);
    r.order1 = reinterpret_cast<uint32_t *>(b + L.o_order1);
    r.tcount = reinterpret_cast<uint32_t *>(b + L.o_tcount);
    r.tcount_r = reinterpret_cast<uint32_t *>(b + L.o_tcount_r);
    r.tmask = reinterpret_cast<uint32_t *>(b + L.o_tmask);
    r.tmask_r = reinterpret_cast<uint32_t *>(b + L.o_tmask_r);
    r.toff = reinterpret_cast<uint32_t *>(b + L.o_toff);
    r.ikey0 = b + L.o_ikey0;
    r.ikey1 = b + L.o_ikey1;
    r.ranges = reinterpret_cast<uint32_t *>(b + L.o_ranges);
    r.pix_cd = reinterpret_cast<float4 *>(b + L.o_pix_cd);
    r.pix_t = reinterpret_cast<float *>(b + L.o_pix_t);
    r.pix_tlast = reinterpret_cast<float *>(b + L.o_pix_tlast);
    r.pix_last = reinterpret_cast<int32_t *>(b + L.o_pix_last);
    r.g2d = reinterpret_cast<float *>(b + L.o_g2d);
    r.sort_hist = reinterpret_cast<uint32_t *>(b + L.o_sort_hist);
    r.scan = reinterpret_cast<uint32_t *>(b + L.o_scan);
    r.gbuf = reinterpret_cast<float *>(b + L.o_gbuf);
    r.tile_hor = reinterpret_cast<int32_t *>(b + L.o_tile_hor);
    r.tile_work = reinterpret_cast<uint32_t *>(b + L.o_tile_work);
    r.tile_order = reinterpret_cast<uint32_t *>(b + L.o_tile_order);
    return r;
}

// fp64 projection of one Gaussian (renderloss.py:176-199).  Keeps the
// intermediates the backward needs.  Every operation is an explicit
// round-to-nearest op (no FMA contraction) in a fixed order, so the host
// restatement (oracle/bin_oracle.c, gcc -ffp-contract=off) reproduces the
// projected records -- and through them the tile keys and ranges -- bit for
// bit; on an HBM-bound kernel the unfused fp64 ops cost nothing measurable.
// Exact = true: every operation an explicit round-to-nearest op (the
// forward, whose records must match oracle/bin_oracle.c bit for bit);
// false: the compiler may contract to FMA (the backward's chain rule, which
// is only held to the gradient tolerance and is register-bound).
#define DM(a, b) (Exact ? __dmul_rn((a), (b)) : (a) * (b))
#define DA(a, b) (Exact ? __dadd_rn((a), (b)) : (a) + (b))
#define DS(a, b) (Exact ? __dsub_rn((a), (b)) : (a) - (b))
#define DD(a, b) (Exact ? __ddiv_rn((a), (b)) : (a) / (b))
struct ProjGeom {
    double x, y, z;        // camera-frame centre
    double u, v;           // pixel mean
    double a, b, c;        // cov2 (+0.3 on the diagonal)
    double R[9];           // Gaussian rotation (unnormalised-quaternion formula)
    double s2[3];
    double Sc[6];          // camera covariance, symmetric: xx xy xz yy yz zz
};

template <bool Exact = true>
__device__ __forceinline__ void project_geometry(double px, double py, double pz, double qw,
                                                 double qx, double qy, double qz, double sx,
                                                 double sy, double sz, const double *rwc,
                                                 const double *t, double fx, double fy,
                                                 double cx, double cy, ProjGeom &g) {
    const double d0 = DS(px, t[0]), d1 = DS(py, t[1]), d2 = DS(pz, t[2]);
    // cam = (p - t) @ r_wc, each component (d0 r0j + d1 r1j) + d2 r2j
    g.x = DA(DA(DM(d0, rwc[0]), DM(d1, rwc[3])), DM(d2, rwc[6]));
    g.y = DA(DA(DM(d0, rwc[1]), DM(d1, rwc[4])), DM(d2, rwc[7]));
    g.z = DA(DA(DM(d0, rwc[2]), DM(d1, rwc[5])), DM(d2, rwc[8]));   // the depth-order key
    const double x = g.x, y = g.y, z = g.z;
    g.u = DA(DD(DM(fx, x), z), cx);
    g.v = DA(DD(DM(fy, y), z), cy);
    // renderloss.py:155-167
    double *R = g.R;
    R[0] = DS(1.0, DM(2.0, DA(DM(qy, qy), DM(qz, qz))));
    R[1] = DM(2.0, DS(DM(qx, qy), DM(qw, qz)));
    R[2] = DM(2.0, DA(DM(qx, qz), DM(qw, qy)));
    R[3] = DM(2.0, DA(DM(qx, qy), DM(qw, qz)));
    R[4] = DS(1.0, DM(2.0, DA(DM(qx, qx), DM(qz, qz))));
    R[5] = DM(2.0, DS(DM(qy, qz), DM(qw, qx)));
    R[6] = DM(2.0, DS(DM(qx, qz), DM(qw, qy)));
    R[7] = DM(2.0, DA(DM(qy, qz), DM(qw, qx)));
    R[8] = DS(1.0, DM(2.0, DA(DM(qx, qx), DM(qy, qy))));
    g.s2[0] = DM(sx, sx);
    g.s2[1] = DM(sy, sy);
    g.s2[2] = DM(sz, sz);
    // M = W R where W = r_wc^T  (W_ij = rwc[j*3+i]);  Sc = M diag(s2) M^T
    double M[9];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int k = 0; k < 3; k++)
            M[i * 3 + k] = DA(DA(DM(rwc[0 * 3 + i], R[0 * 3 + k]), DM(rwc[1 * 3 + i], R[1 * 3 + k])),
                              DM(rwc[2 * 3 + i], R[2 * 3 + k]));
    double S[3][3];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = i; j < 3; j++) {
            const double s = DA(DA(DM(DM(M[i * 3 + 0], g.s2[0]), M[j * 3 + 0]),
                                   DM(DM(M[i * 3 + 1], g.s2[1]), M[j * 3 + 1])),
                                DM(DM(M[i * 3 + 2], g.s2[2]), M[j * 3 + 2]));
            S[i][j] = s;
            S[j][i] = s;
        }
    g.Sc[0] = S[0][0];
    g.Sc[1] = S[0][1];
    g.Sc[2] = S[0][2];
    g.Sc[3] = S[1][1];
    g.Sc[4] = S[1][2];
    g.Sc[5] = S[2][2];
    // J = [[fx/z, 0, -fx x/z^2], [0, fy/z, -fy y/z^2]]
    const double zz = DM(z, z);
    const double j00 = DD(fx, z), j02 = -DD(DM(fx, x), zz);
    const double j11 = DD(fy, z), j12 = -DD(DM(fy, y), zz);
    // cov2 = J Sc J^T
    const double a00 = DA(DM(j00, S[0][0]), DM(j02, S[2][0]));
    const double a01 = DA(DM(j00, S[0][1]), DM(j02, S[2][1]));
    const double a02 = DA(DM(j00, S[0][2]), DM(j02, S[2][2]));
    const double b11 = DA(DM(j11, S[1][1]), DM(j12, S[2][1]));
    const double b12 = DA(DM(j11, S[1][2]), DM(j12, S[2][2]));
    g.a = DA(DA(DM(a00, j00), DM(a02, j02)), 0.3);
    g.b = DA(DM(a01, j11), DM(a02, j12));
    g.c = DA(DA(DM(b11, j11), DM(b12, j12)), 0.3);
}

// A second branch of the caller's stream (one per host thread and device)
// for launches that can overlap the main chain: begin() forks it off the
// caller's stream, end() joins it back, so every entry point keeps the
// caller-stream semantics and CUDA-graph capture records the two branches.
struct StreamFork {
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    void begin(cudaStream_t st) {
        cudaEventRecord(fork, st);
        cudaStreamWaitEvent(side, fork, 0);
    }
    void end(cudaStream_t st) {
        cudaEventRecord(join, side);
        cudaStreamWaitEvent(st, join, 0);
    }
};
StreamFork &stream_fork();

int render_forward(const float *params, const int32_t *slots, int64_t n, const sm_camera &cam,
                   const sm_render_dims &dims, void *ws, int64_t ws_bytes, float *out_rgb,
                   float *out_depth, float *out_alpha, uint32_t *view_order, cudaStream_t st);
struct AdamFuse;
int render_backward(const float *params, const int32_t *slots, int64_t n, const sm_camera &cam,
                    const sm_render_dims &dims, void *ws, int64_t ws_bytes, const float *d_rgb,
                    const float *d_depth, const float *d_alpha, float *grads, const AdamFuse *fuse,
                    cudaStream_t st);

}  // namespace sm
