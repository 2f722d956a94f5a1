/*
 * bin_oracle.c -- CPU restatement of K2 (projection records) and K3 (global
 * depth order, tile binning, tile-sorted instance keys, tile ranges).
 *
 * TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py CPU
 * legs); nothing in the product package loads it.
 *
 * The reference has no tile binning: renderloss.py composites every pixel
 * of each Gaussian's clamped 3-sigma box (renderloss.py:122-135) in the
 * global order np.argsort(z, kind="stable") (renderloss.py:202).  The device
 * splits that loop into 16x16 tiles.  This file restates, in plain C with
 * -ffp-contract=off, exactly the arithmetic the device performs, so tests
 * can require the device's sorted (tile, rank) keys and per-tile instance
 * ranges to be BIT-EXACT:
 *
 *  - projection (renderloss.py:176-199): cam = (p - t) @ r_wc,
 *    u = fx x / z + cx, R(q) (renderloss.py:155-167), Sc = M diag(s^2) M^T,
 *    cov2 = J Sc J^T + 0.3 I -- fp64, left-to-right, one rounding per op
 *    (csrc/render.cuh project_geometry uses __dmul_rn/__dadd_rn in the same
 *    order);
 *  - near test z >= near (renderloss.py:179), conic det > 0, a > 0, c > 0;
 *  - 3-sigma box x0 = ceil(u - 3 sqrt a), x1 = floor(u + 3 sqrt a) clamped
 *    to the image (renderloss.py:122-135);
 *  - depth order: stable sort of the kept Gaussians by fp32(z), ties by the
 *    fp64 z bits (= np.argsort(z, kind="stable") on the kept set, because
 *    rounding to fp32 is monotone), culled Gaussians after, in index order;
 *  - tiles: every 16x16 tile the box touches (ellipse cull off), or the
 *    tiles of each tile row whose column span the q <= 9 ellipse can reach
 *    (ellipse cull on: csrc/common.cuh RowSpan, fp32 with explicit ops);
 *  - keys (tile << rank_bits) | depth rank, sorted ascending (= the device's
 *    stable tile sort of rank-ordered emissions); ranges [start, end) per
 *    tile, (0, 0) for tiles with no instance.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TILE 16
static const double kPowScale = -0.72134752044448170368; /* -0.5 log2 e */

typedef struct {
    float ox, oy, beta, G, K;
    int x0, y0, x1, y1;
    int valid; /* kept by near + conic + non-empty box */
} rec_t;

static void project(const float *p, const double *rwc, const double *t, double fx, double fy,
                    double cx, double cy, double near, int W, int H, int cull, rec_t *r,
                    double *z_out, int *kept) {
    const double px = p[0], py = p[1], pz = p[2], qw = p[3], qx = p[4], qy = p[5], qz = p[6];
    const double sx = p[7], sy = p[8], sz = p[9];
    const double d0 = px - t[0], d1 = py - t[1], d2 = pz - t[2];
    const double x = (d0 * rwc[0] + d1 * rwc[3]) + d2 * rwc[6];
    const double y = (d0 * rwc[1] + d1 * rwc[4]) + d2 * rwc[7];
    const double z = (d0 * rwc[2] + d1 * rwc[5]) + d2 * rwc[8];
    *z_out = z;
    r->valid = 0;
    *kept = z >= near;
    if (!*kept) return;
    const double u = fx * x / z + cx, v = fy * y / z + cy;
    double R[9];
    R[0] = 1.0 - 2.0 * (qy * qy + qz * qz);
    R[1] = 2.0 * (qx * qy - qw * qz);
    R[2] = 2.0 * (qx * qz + qw * qy);
    R[3] = 2.0 * (qx * qy + qw * qz);
    R[4] = 1.0 - 2.0 * (qx * qx + qz * qz);
    R[5] = 2.0 * (qy * qz - qw * qx);
    R[6] = 2.0 * (qx * qz - qw * qy);
    R[7] = 2.0 * (qy * qz + qw * qx);
    R[8] = 1.0 - 2.0 * (qx * qx + qy * qy);
    const double s2[3] = {sx * sx, sy * sy, sz * sz};
    double M[9], S[3][3];
    for (int i = 0; i < 3; i++)
        for (int k = 0; k < 3; k++)
            M[i * 3 + k] = (rwc[0 * 3 + i] * R[0 * 3 + k] + rwc[1 * 3 + i] * R[1 * 3 + k]) +
                           rwc[2 * 3 + i] * R[2 * 3 + k];
    for (int i = 0; i < 3; i++)
        for (int j = i; j < 3; j++) {
            const double s = ((M[i * 3 + 0] * s2[0]) * M[j * 3 + 0] + (M[i * 3 + 1] * s2[1]) * M[j * 3 + 1]) +
                             (M[i * 3 + 2] * s2[2]) * M[j * 3 + 2];
            S[i][j] = s;
            S[j][i] = s;
        }
    const double zz = z * z;
    const double j00 = fx / z, j02 = -((fx * x) / zz);
    const double j11 = fy / z, j12 = -((fy * y) / zz);
    const double a00 = j00 * S[0][0] + j02 * S[2][0];
    const double a01 = j00 * S[0][1] + j02 * S[2][1];
    const double a02 = j00 * S[0][2] + j02 * S[2][2];
    const double b11 = j11 * S[1][1] + j12 * S[2][1];
    const double b12 = j11 * S[1][2] + j12 * S[2][2];
    const double a = (a00 * j00 + a02 * j02) + 0.3;
    const double b = a01 * j11 + a02 * j12;
    const double c = (b11 * j11 + b12 * j12) + 0.3;
    const double det = a * c - b * b;
    if (det <= 0.0 || a <= 0.0 || c <= 0.0) return;
    const double rx = 3.0 * sqrt(a), ry = 3.0 * sqrt(c);
    double fx0 = ceil(u - rx), fx1 = floor(u + rx);
    double fy0 = ceil(v - ry), fy1 = floor(v + ry);
    fx0 = fmin(fmax(fx0, 0.0), (double)W);
    fy0 = fmin(fmax(fy0, 0.0), (double)H);
    fx1 = fmax(fmin(fx1, (double)(W - 1)), -1.0);
    fy1 = fmax(fmin(fy1, (double)(H - 1)), -1.0);
    r->x0 = (int)fx0;
    r->x1 = (int)fx1;
    r->y0 = (int)fy0;
    r->y1 = (int)fy1;
    r->ox = (float)((double)r->x0 - u);
    r->oy = (float)((double)r->y0 - v);
    r->beta = (float)(b / c);
    r->G = (float)((9.0 * det) / c);
    r->K = cull ? (float)(det / (c * c)) : -1.f;
    (void)kPowScale;
    r->valid = !(r->x1 < r->x0 || r->y1 < r->y0);
}

/* csrc/common.cuh RowSpan::row: kept tile columns [c0, c1] of tile row ty. */
typedef struct {
    int x0, y0, y1, tx0, tx1, ty0, ty1, ell;
    float beta, G, K, dys, rad, xo, oy;
} span_t;

static void span_init(const rec_t *g, span_t *s) {
    s->x0 = g->x0;
    s->y0 = g->y0;
    s->y1 = g->y1;
    s->tx0 = g->x0 / TILE;
    s->tx1 = g->x1 / TILE;
    s->ty0 = g->y0 / TILE;
    s->ty1 = g->y1 / TILE;
    s->beta = g->beta;
    s->G = g->G;
    s->K = g->K;
    s->ell = g->K > 0.f;
    s->dys = s->ell ? s->beta * sqrtf((s->G / s->K) / (s->K + s->beta * s->beta)) : 0.f;
    s->rad = sqrtf(fmaxf(s->G, 0.f));
    s->xo = (float)g->x0 - g->ox;
    s->oy = g->oy;
}

static float half_width(const span_t *s, float dy) { return sqrtf(fmaxf(s->G - (s->K * dy) * dy, 0.f)); }

static void span_row(const span_t *s, int ty, int *c0, int *c1) {
    *c0 = s->tx0;
    *c1 = s->tx1;
    if (!s->ell) return;
    const int lo = ty * TILE > s->y0 ? ty * TILE : s->y0;
    const int hi = ty * TILE + TILE - 1 < s->y1 ? ty * TILE + TILE - 1 : s->y1;
    const float a0 = (float)(lo - s->y0) + s->oy;
    const float a1 = (float)(hi - s->y0) + s->oy;
    const float dr = fminf(fmaxf(s->dys, a0), a1), dl = fminf(fmaxf(-s->dys, a0), a1);
    const float xr = s->beta * dr + half_width(s, dr);
    const float xl = s->beta * dl - half_width(s, dl);
    const float m = 0.01f * (s->rad + fabsf(s->beta) * fmaxf(fabsf(a0), fabsf(a1))) + 0.02f;
    const float pl = (s->xo + xl) - m, pr = (s->xo + xr) + m;
    if (!(pl <= pr) || !(pr - pl < 1e7f)) return;
    const int l = (int)floorf(pl * (1.f / TILE)), h = (int)floorf(pr * (1.f / TILE));
    if (l > *c0) *c0 = l;
    if (h < *c1) *c1 = h;
}

typedef struct {
    uint32_t key;
    uint64_t zbits;
    int64_t idx;
} dk_t;

static int cmp_depth(const void *pa, const void *pb) {
    const dk_t *a = (const dk_t *)pa, *b = (const dk_t *)pb;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    if (a->zbits != b->zbits) return a->zbits < b->zbits ? -1 : 1;
    return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

static int cmp_u64(const void *pa, const void *pb) {
    const uint64_t a = *(const uint64_t *)pa, b = *(const uint64_t *)pb;
    return a < b ? -1 : (a > b);
}

/*
 * params: n x 16 float32 records (include/splatmap_cuda.h layout).
 * order_out [n]: depth rank -> index.  keys_out: capacity max_keys, sorted
 * (tile << rank_bits) | rank.  ranges_out [tiles][2].  Returns the number of
 * instances (> max_keys: nothing written to keys_out beyond capacity), or -1
 * on allocation failure.
 */
int64_t ob_bin_tiles(int64_t n, const float *params, const double *rwc, const double *t, double fx, double fy,
                     double cx, double cy, double near, int W, int H, int cull, int rank_bits,
                     int64_t *order_out, uint64_t *keys_out, int64_t max_keys, uint32_t *ranges_out) {
    rec_t *rec = (rec_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(rec_t));
    dk_t *dk = (dk_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(dk_t));
    if (!rec || !dk) {
        free(rec);
        free(dk);
        return -1;
    }
    for (int64_t i = 0; i < n; i++) {
        double z;
        int kept;
        project(params + 16 * i, rwc, t, fx, fy, cx, cy, near, W, H, cull, &rec[i], &z, &kept);
        float zf = (float)z;
        uint32_t kb;
        memcpy(&kb, &zf, 4);
        uint64_t zb;
        memcpy(&zb, &z, 8);
        dk[i].key = kept ? kb : 0xffffffffu;
        dk[i].zbits = kept ? zb : 0;
        dk[i].idx = i;
    }
    qsort(dk, (size_t)n, sizeof(dk_t), cmp_depth);
    const int tiles_x = (W + TILE - 1) / TILE, tiles_y = (H + TILE - 1) / TILE;
    int64_t count = 0;
    for (int64_t r = 0; r < n; r++) {
        order_out[r] = dk[r].idx;
        const rec_t *g = &rec[dk[r].idx];
        if (!g->valid) continue;
        span_t s;
        span_init(g, &s);
        for (int ty = s.ty0; ty <= s.ty1; ty++) {
            int c0, c1;
            span_row(&s, ty, &c0, &c1);
            for (int tx = c0; tx <= c1; tx++) {
                if (count < max_keys) keys_out[count] = ((uint64_t)(ty * tiles_x + tx) << rank_bits) | (uint64_t)r;
                count++;
            }
        }
    }
    if (count <= max_keys) {
        qsort(keys_out, (size_t)count, sizeof(uint64_t), cmp_u64);
        memset(ranges_out, 0, sizeof(uint32_t) * 2 * (size_t)tiles_x * tiles_y);
        for (int64_t p = 0; p < count; p++) {
            const uint64_t tile = keys_out[p] >> rank_bits;
            if (p == 0 || (keys_out[p - 1] >> rank_bits) != tile) ranges_out[2 * tile] = (uint32_t)p;
            if (p == count - 1 || (keys_out[p + 1] >> rank_bits) != tile) ranges_out[2 * tile + 1] = (uint32_t)(p + 1);
        }
    }
    free(rec);
    free(dk);
    return count;
}
