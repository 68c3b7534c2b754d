/*
 * TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT PATH.
 *
 * CPU restatement (float64, scalar C) of the reference rasterizer hot path of
 * `convexsplat` 0.1.0 (/root/reference/pkg/src/convexsplat).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm
 * may load this library, and only as the checker or the timed CPU baseline.
 *
 * Every function cites the reference lines it restates.  Arithmetic order is
 * pinned where it feeds a discrete decision (hull, bbox, depth order):
 *   - projection  x_cam = fma(p2,R2, fma(p1,R1, p0*R0)) + t   (OpenBLAS dgemm
 *     order of `points @ R.T`, projection.py:30)
 *   - every other reduction is a plain left-to-right sum, no contraction
 *     (compile with -ffp-contract=off).
 * The oracle is pinned against vectors produced by the reference itself
 * (tests/golden/make_golden.py writes the .npz fixtures; tests/test_oracle_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_ALPHA_MAX (1.0 - 1e-6)   /* rasterize.py:30 */
#define OR_MASK_GATE 0.01           /* rasterize.py:26 */
#define OR_CROSS_TOL 1e-9           /* projection.py:19 */
#define OR_SH_COEFFS 16             /* model.py:15 */
#define OR_MAXPTS 64                /* graham_scan scratch bound */

enum { OR_VISIBLE = 0, OR_MASKED = 1, OR_NEAR = 2, OR_DEGENERATE = 3, OR_EMPTY_BBOX = 4 };
enum { OR_MODE_NONE = 0, OR_MODE_SQRT = 1, OR_MODE_DEPTH = 2, OR_MODE_DEPTH2 = 3 };

typedef struct {
    double fx, fy, cx, cy;
    double R[9];
    double t[3];
    double z_near;
    int32_t width, height, ortho, pad_;
} or_camera;

typedef struct {
    double cutoff, floor;
    double background[3];
    int32_t tile, sh_degree, mode, n_threads;
} or_settings;

typedef struct {
    int32_t n, k;
    const double *points;      /* [n,k,3] */
    const double *raw_delta, *raw_sigma, *raw_opacity, *raw_mask;  /* [n] */
    const double *sh;          /* [n,16,3] */
} or_params;

typedef struct {
    int32_t *status;    /* [n] */
    int32_t *hull_n;    /* [n] */
    int32_t *hull;      /* [n,k]  (-1 padded) */
    int32_t *bbox;      /* [n,4]  x0,x1,y0,y1 */
    int32_t *order;     /* [n]    first n_visible valid */
    double *pixels;     /* [n,k,2] */
    double *normals;    /* [n,k,2] */
    double *offsets;    /* [n,k] */
    double *depth, *scale, *delta_s, *sigma_s, *opacity;  /* [n] */
    double *color;      /* [n,3] */
    double *view_dir;   /* [n,3] */
    double *view_dist;  /* [n] */
    int32_t n_visible;
    int32_t k;          /* row stride of hull/normals/offsets/pixels */
} or_view;

/* ------------------------------------------------------------------ */
/* activations, model.py:21-54; scipy expit(x) == 1/(1+exp(-x))        */
static double expit(double x) { return 1.0 / (1.0 + exp(-x)); }

/* field.py:26-35 */
static double depth_scale(int mode, double d) {
    switch (mode) {
    case OR_MODE_NONE: return 1.0;
    case OR_MODE_SQRT: return sqrt(d);
    case OR_MODE_DEPTH: return d;
    default: return d * d;
    }
}
/* field.py:38-48 */
static double depth_scale_grad(int mode, double d) {
    switch (mode) {
    case OR_MODE_NONE: return 0.0;
    case OR_MODE_SQRT: return 0.5 / sqrt(d);
    case OR_MODE_DEPTH: return 1.0;
    default: return 2.0 * d;
    }
}

/* ------------------------------------------------------------------ */
/* spherical harmonics, harmonics.py:7-24 constants                     */
static const double C0 = 0.28209479177387814;
static const double C1 = 0.4886025119029199;
static const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                             -1.0925484305920792, 0.5462742152960396};
static const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                             0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                             -0.5900435899266435};

/* harmonics.py:33-59 */
static int sh_basis(const double *d, int deg, double *out) {
    double x = d[0], y = d[1], z = d[2];
    out[0] = C0;
    if (deg >= 1) { out[1] = -C1 * y; out[2] = C1 * z; out[3] = -C1 * x; }
    if (deg >= 2) {
        double xx = x * x, yy = y * y, zz = z * z;
        out[4] = C2[0] * x * y;
        out[5] = C2[1] * y * z;
        out[6] = C2[2] * (2.0 * zz - xx - yy);
        out[7] = C2[3] * x * z;
        out[8] = C2[4] * (xx - yy);
    }
    if (deg >= 3) {
        double xx = x * x, yy = y * y, zz = z * z;
        out[9] = C3[0] * y * (3.0 * xx - yy);
        out[10] = C3[1] * x * y * z;
        out[11] = C3[2] * y * (4.0 * zz - xx - yy);
        out[12] = C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
        out[13] = C3[4] * x * (4.0 * zz - xx - yy);
        out[14] = C3[5] * z * (xx - yy);
        out[15] = C3[6] * x * (xx - 3.0 * yy);
    }
    return (deg + 1) * (deg + 1);
}

/* harmonics.py:62-98, rows (n,3) */
static void sh_basis_grad(const double *d, int deg, double g[16][3]) {
    double x = d[0], y = d[1], z = d[2];
    memset(g, 0, sizeof(double) * 48);
    if (deg >= 1) { g[1][1] = -C1; g[2][2] = C1; g[3][0] = -C1; }
    if (deg >= 2) {
        g[4][0] = C2[0] * y; g[4][1] = C2[0] * x;
        g[5][1] = C2[1] * z; g[5][2] = C2[1] * y;
        g[6][0] = -2.0 * C2[2] * x; g[6][1] = -2.0 * C2[2] * y; g[6][2] = 4.0 * C2[2] * z;
        g[7][0] = C2[3] * z; g[7][2] = C2[3] * x;
        g[8][0] = 2.0 * C2[4] * x; g[8][1] = -2.0 * C2[4] * y;
    }
    if (deg >= 3) {
        double xx = x * x, yy = y * y, zz = z * z;
        g[9][0] = C3[0] * 6.0 * x * y; g[9][1] = C3[0] * 3.0 * (xx - yy);
        g[10][0] = C3[1] * y * z; g[10][1] = C3[1] * x * z; g[10][2] = C3[1] * x * y;
        g[11][0] = -2.0 * C3[2] * x * y; g[11][1] = C3[2] * (4.0 * zz - xx - 3.0 * yy);
        g[11][2] = 8.0 * C3[2] * y * z;
        g[12][0] = -6.0 * C3[3] * x * z; g[12][1] = -6.0 * C3[3] * y * z;
        g[12][2] = C3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy);
        g[13][0] = C3[4] * (4.0 * zz - 3.0 * xx - yy); g[13][1] = -2.0 * C3[4] * x * y;
        g[13][2] = 8.0 * C3[4] * x * z;
        g[14][0] = 2.0 * C3[5] * x * z; g[14][1] = -2.0 * C3[5] * y * z; g[14][2] = C3[5] * (xx - yy);
        g[15][0] = C3[6] * 3.0 * (xx - yy); g[15][1] = -6.0 * C3[6] * x * y;
    }
}

/* ------------------------------------------------------------------ */
/* projection.py:43-44 (Python floats: no FMA)                          */
static double cross3(const double *o, const double *a, const double *b) {
    return (a[0] - o[0]) * (b[1] - o[1]) - (a[1] - o[1]) * (b[0] - o[0]);
}

/* comparator of projection.py:73-85, returns -1/0/1 */
static int hull_cmp(const double *pts, int ref, int a, int b, double tol) {
    double c = cross3(pts + 2 * ref, pts + 2 * a, pts + 2 * b);
    if (c > tol) return -1;
    if (c < -tol) return 1;
    double ax = pts[2 * a] - pts[2 * ref], ay = pts[2 * a + 1] - pts[2 * ref + 1];
    double bx = pts[2 * b] - pts[2 * ref], by = pts[2 * b + 1] - pts[2 * ref + 1];
    double da = ax * ax + ay * ay;
    double db = bx * bx + by * by;
    if (da < db) return -1;
    if (da > db) return 1;
    return 0;
}

/* CPython (<=3.12) list.sort for n < 64 elements with a cmp_to_key key:
 * count_run (strictly descending prefix reversed) then binary insertion
 * sort; "less" is cmp(x, y) < 0.  Restates Objects/listobject.c, which the
 * reference invokes via rest.sort(key=cmp_to_key(compare)) at
 * projection.py:87. */
static void py_list_sort(int *v, int m, const double *pts, int ref, double tol) {
    if (m < 2) return;
#define LT(x, y) (hull_cmp(pts, ref, (x), (y), tol) < 0)
    int run = 2;
    if (LT(v[1], v[0])) {
        while (run < m && LT(v[run], v[run - 1])) run++;
        for (int i = 0, j = run - 1; i < j; i++, j--) { int t = v[i]; v[i] = v[j]; v[j] = t; }
    } else {
        while (run < m && !LT(v[run], v[run - 1])) run++;
    }
    for (int start = run; start < m; start++) {
        int pivot = v[start];
        int l = 0, r = start;
        do {
            int p = l + ((r - l) >> 1);
            if (LT(pivot, v[p])) r = p; else l = p + 1;
        } while (l < r);
        for (int p = start; p > l; p--) v[p] = v[p - 1];
        v[l] = pivot;
    }
#undef LT
}

/* projection.py:47-113.  Returns hull size (0 == None). */
int or_graham_scan(int n, const double *pts, int32_t *out) {
    if (n < 3 || n > OR_MAXPTS) return 0;
    int unique[OR_MAXPTS], nu = 0;
    for (int i = 0; i < n; i++) {
        int dup = 0;
        for (int j = 0; j < nu; j++) {
            int u = unique[j];
            if (pts[2 * u] == pts[2 * i] && pts[2 * u + 1] == pts[2 * i + 1]) { dup = 1; break; }
        }
        if (!dup) unique[nu++] = i;
    }
    if (nu < 3) return 0;
    int ref = unique[0];
    for (int j = 1; j < nu; j++) {
        int u = unique[j];
        double uy = pts[2 * u + 1], ux = pts[2 * u];
        double ry = pts[2 * ref + 1], rx = pts[2 * ref];
        if (uy < ry || (uy == ry && ux < rx)) ref = u;
    }
    int rest[OR_MAXPTS], m = 0;
    for (int j = 0; j < nu; j++) if (unique[j] != ref) rest[m++] = unique[j];
    py_list_sort(rest, m, pts, ref, OR_CROSS_TOL);

    int st[OR_MAXPTS], sn = 0;
    st[sn++] = ref;
    for (int j = 0; j < m; j++) {
        int c = rest[j];
        while (sn >= 2 && cross3(pts + 2 * st[sn - 2], pts + 2 * st[sn - 1], pts + 2 * c) <= OR_CROSS_TOL) sn--;
        st[sn++] = c;
    }
    int changed = 1;
    while (changed && sn >= 3) {
        changed = 0;
        for (int kk = 0; kk < sn; kk++) {
            int a = st[(kk - 1 + sn) % sn], b = st[kk], c = st[(kk + 1) % sn];
            if (cross3(pts + 2 * a, pts + 2 * b, pts + 2 * c) <= OR_CROSS_TOL) {
                for (int q = kk; q < sn - 1; q++) st[q] = st[q + 1];
                sn--;
                changed = 1;
                break;
            }
        }
    }
    if (sn < 3) return 0;
    int start = 0;
    for (int q = 0; q < sn; q++) if (st[q] == ref) { start = q; break; }
    for (int q = 0; q < sn; q++) out[q] = st[(start + q) % sn];
    return sn;
}

/* ------------------------------------------------------------------ */
/* Camera.center, model.py:164-166: (-R^T) t                             */
static void cam_center(const or_camera *cam, double *c) {
    for (int j = 0; j < 3; j++) {
        double s = 0.0;
        for (int i = 0; i < 3; i++) s += (-cam->R[3 * i + j]) * cam->t[i];
        c[j] = s;
    }
}

/* prepare one convex: rasterize.py:88-120; returns status */
static int prepare_one(const or_camera *cam, const or_settings *st, const or_params *P, int i,
                       const double *cc, or_view *V) {
    const int k = P->k;
    const double *pts = P->points + (size_t)i * k * 3;
    int32_t *hull = V->hull + (size_t)i * k;
    for (int j = 0; j < k; j++) hull[j] = -1;
    V->hull_n[i] = 0;
    /* rasterize.py:89 mask gate */
    double mask = expit(P->raw_mask[i]);
    if (mask <= OR_MASK_GATE) return OR_MASKED;
    /* projection.py:22-40 */
    double *px = V->pixels + (size_t)i * k * 2;
    double z[OR_MAXPTS];
    for (int j = 0; j < k; j++) {
        const double *p = pts + 3 * j;
        double xc[3];
        for (int c = 0; c < 3; c++)
            xc[c] = fma(p[2], cam->R[3 * c + 2], fma(p[1], cam->R[3 * c + 1], p[0] * cam->R[3 * c])) + cam->t[c];
        z[j] = xc[2];
        if (cam->ortho) {
            px[2 * j] = cam->fx * xc[0] + cam->cx;
            px[2 * j + 1] = cam->fy * xc[1] + cam->cy;
        } else {
            px[2 * j] = (cam->fx * xc[0]) / xc[2] + cam->cx;
            px[2 * j + 1] = (cam->fy * xc[1]) / xc[2] + cam->cy;
        }
    }
    for (int j = 0; j < k; j++) if (z[j] <= cam->z_near) return OR_NEAR;
    /* projection.py:47-113 */
    int h = or_graham_scan(k, px, hull);
    if (h == 0) { for (int j = 0; j < k; j++) hull[j] = -1; return OR_DEGENERATE; }
    V->hull_n[i] = h;
    /* projection.py:116-128 */
    double *nrm = V->normals + (size_t)i * k * 2, *off = V->offsets + (size_t)i * k;
    for (int j = 0; j < h; j++) {
        const double *v0 = px + 2 * hull[j], *v1 = px + 2 * hull[(j + 1) % h];
        double ex = v1[0] - v0[0], ey = v1[1] - v0[1];
        double nx = ey, ny = -ex;
        double len = sqrt(nx * nx + ny * ny);
        nx = nx / len; ny = ny / len;
        nrm[2 * j] = nx; nrm[2 * j + 1] = ny;
        off[j] = -(nx * v0[0] + ny * v0[1]);
    }
    /* rasterize.py:99-103 */
    double zs = 0.0;
    for (int j = 0; j < k; j++) zs += z[j];
    double depth = zs / k;
    double s = depth_scale(st->mode, cam->ortho ? 1.0 : depth);
    double delta_s = s * exp(P->raw_delta[i]);
    double sigma_s = s * exp(P->raw_sigma[i]);
    double o = expit(P->raw_opacity[i]);
    V->depth[i] = depth; V->scale[i] = s; V->delta_s[i] = delta_s; V->sigma_s[i] = sigma_s;
    V->opacity[i] = o;
    /* projection.py:136-177 */
    int32_t *bb = V->bbox + 4 * i;
    double cut = st->cutoff;
    if (o <= cut) return OR_EMPTY_BBOX;
    if (cut <= 0.0) {
        bb[0] = 0; bb[1] = cam->width; bb[2] = 0; bb[3] = cam->height;
    } else {
        double eps = cut / o;
        if (0.5 < eps) eps = 0.5;
        double margin = log((1.0 - eps) / eps) / (sigma_s * delta_s);
        double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
        for (int j = 0; j < h; j++) {
            const double *pv = nrm + 2 * ((j - 1 + h) % h), *nv = nrm + 2 * j;
            double den = 1.0 + (pv[0] * nv[0] + pv[1] * nv[1]);
            if (!(den >= 1e-12)) den = 1e-12;
            const double *v = px + 2 * hull[j];
            double ix = v[0] + (margin * (pv[0] + nv[0])) / den;
            double iy = v[1] + (margin * (pv[1] + nv[1])) / den;
            if (ix < xmin) xmin = ix;
            if (ix > xmax) xmax = ix;
            if (iy < ymin) ymin = iy;
            if (iy > ymax) ymax = iy;
        }
        double x0 = ceil(xmin - 0.5), x1 = floor(xmax - 0.5) + 1.0;
        double y0 = ceil(ymin - 0.5), y1 = floor(ymax - 0.5) + 1.0;
        if (x0 < 0.0) x0 = 0.0;
        if (y0 < 0.0) y0 = 0.0;
        if (x1 > cam->width) x1 = cam->width;
        if (y1 > cam->height) y1 = cam->height;
        if (!(x0 < x1) || !(y0 < y1)) return OR_EMPTY_BBOX;
        bb[0] = (int32_t)x0; bb[1] = (int32_t)x1; bb[2] = (int32_t)y0; bb[3] = (int32_t)y1;
    }
    /* rasterize.py:110-114, model.py:109-111 */
    double ctr[3] = {0.0, 0.0, 0.0};
    for (int j = 0; j < k; j++) for (int c = 0; c < 3; c++) ctr[c] += pts[3 * j + c];
    double vd[3];
    for (int c = 0; c < 3; c++) vd[c] = ctr[c] / k - cc[c];
    double dist = sqrt(vd[0] * vd[0] + vd[1] * vd[1] + vd[2] * vd[2]);
    double *dir = V->view_dir + 3 * i;
    if (dist > 0) { dir[0] = vd[0] / dist; dir[1] = vd[1] / dist; dir[2] = vd[2] / dist; }
    else { dir[0] = 0.0; dir[1] = 0.0; dir[2] = 1.0; }
    V->view_dist[i] = dist;
    /* harmonics.py:101-109 */
    double basis[16];
    int nb = sh_basis(dir, st->sh_degree, basis);
    const double *sh = P->sh + (size_t)i * OR_SH_COEFFS * 3;
    for (int c = 0; c < 3; c++) {
        double acc = 0.0;
        for (int b = 0; b < nb; b++) acc += basis[b] * sh[3 * b + c];
        double raw = 0.5 + acc;
        V->color[3 * i + c] = raw > 0.0 ? raw : 0.0;
    }
    return OR_VISIBLE;
}

static const double *g_sort_depth;
static int depth_index_cmp(const void *a, const void *b) {
    int ia = *(const int32_t *)a, ib = *(const int32_t *)b;
    double da = g_sort_depth[ia], db = g_sort_depth[ib];
    if (da < db) return -1;
    if (da > db) return 1;
    return (ia > ib) - (ia < ib);
}

/* rasterize.py:77-122 */
int or_prepare_view(const or_camera *cam, const or_settings *st, const or_params *P, or_view *V) {
    double cc[3];
    cam_center(cam, cc);
    int n = P->n;
    V->k = P->k;
#ifdef _OPENMP
    int nt = st->n_threads > 0 ? st->n_threads : 1;
#pragma omp parallel for schedule(dynamic, 1024) num_threads(nt)
#endif
    for (int i = 0; i < n; i++) V->status[i] = prepare_one(cam, st, P, i, cc, V);
    int nv = 0;
    for (int i = 0; i < n; i++) if (V->status[i] == OR_VISIBLE) V->order[nv++] = i;
    g_sort_depth = V->depth;
    qsort(V->order, nv, sizeof(int32_t), depth_index_cmp);
    V->n_visible = nv;
    return nv;
}

/* rasterize.py:134-144: CSR of per-tile candidate lists (values = position
 * in the prepared order).  Returns P; writes items only when items != NULL. */
int64_t or_bin_tiles(const or_view *V, int width, int height, int ts, int64_t *tile_off, int32_t *items) {
    int tx_n = (width + ts - 1) / ts, ty_n = (height + ts - 1) / ts;
    int64_t T = (int64_t)tx_n * ty_n;
    int64_t *cnt = calloc((size_t)T + 1, sizeof(int64_t));
    for (int kk = 0; kk < V->n_visible; kk++) {
        const int32_t *bb = V->bbox + 4 * V->order[kk];
        for (int ty = bb[2] / ts; ty <= (bb[3] - 1) / ts; ty++)
            for (int tx = bb[0] / ts; tx <= (bb[1] - 1) / ts; tx++) cnt[(int64_t)ty * tx_n + tx]++;
    }
    tile_off[0] = 0;
    for (int64_t t = 0; t < T; t++) tile_off[t + 1] = tile_off[t] + cnt[t];
    int64_t P = tile_off[T];
    if (items) {
        for (int64_t t = 0; t < T; t++) cnt[t] = tile_off[t];
        for (int kk = 0; kk < V->n_visible; kk++) {
            const int32_t *bb = V->bbox + 4 * V->order[kk];
            for (int ty = bb[2] / ts; ty <= (bb[3] - 1) / ts; ty++)
                for (int tx = bb[0] / ts; tx <= (bb[1] - 1) / ts; tx++) items[cnt[(int64_t)ty * tx_n + tx]++] = kk;
        }
    }
    free(cnt);
    return P;
}


/* ------------------------------------------------------------------ */
/* Per-pixel field: projection.py:131-133 distances, field.py:51-59 LSE,
 * field.py:70-72 indicator. */
static inline void field_at(const double *nrm, const double *off, int h, double delta_s, double sigma_s,
                            double qx, double qy, double *dist, double *phi, double *ind) {
    double m = -INFINITY;
    for (int j = 0; j < h; j++) {
        dist[j] = qx * nrm[2 * j] + qy * nrm[2 * j + 1] + off[j];
        double zj = delta_s * dist[j];
        if (zj > m) m = zj;
    }
    double s = 0.0;
    for (int j = 0; j < h; j++) s += exp(delta_s * dist[j] - m);
    *phi = m + log(s);
    *ind = expit(-sigma_s * *phi);
}

typedef struct {
    double *image;       /* [H,W,3] */
    double *trans;       /* [H,W]   final transmittance */
    int32_t *count;      /* [H,W] */
    double *wsum;        /* [H,W] */
    double *depth;       /* [H,W]   new output: sum_n T*alpha*depth_n */
    uint8_t *visible;    /* [n] */
    int64_t n_eval;      /* (pixel, candidate) pairs evaluated while alive */
    int64_t n_blend;     /* pairs blended */
} or_frame;

/* Decisions of another implementation to follow instead of re-deciding
 * them (the decision-forced check): pixel p blended the pair indices
 * pos[off[p] .. off[p+1]) in that order, and channel c of its C + T*bg lay
 * in [0,1] iff bit c of clamp[p].  NULL = decide as the reference does. */
typedef struct {
    const int64_t *off;     /* [H*W+1] */
    const int32_t *pos;     /* [off[H*W]] pair indices into items */
    const uint8_t *clamp;   /* [H*W] or NULL */
} or_forced;

/* rasterize.py:178-204 for one tile (with `fd`: the blend decisions of fd
 * instead of the predicates of rasterize.py:194-195). */
static void render_tile(const or_camera *cam, const or_settings *st, const or_view *V,
                        const int64_t *tile_off, const int32_t *items, int64_t t, or_frame *F,
                        int64_t *ne, int64_t *nb, const or_forced *fd, int64_t *cur) {
    const int W = cam->width, H = cam->height, ts = st->tile, k = V->k;
    const int tx_n = (W + ts - 1) / ts;
    const double cut = st->cutoff, flo = st->floor;
    int ty = (int)(t / tx_n), tx = (int)(t % tx_n);
    int ty0 = ty * ts, ty1 = ty0 + ts < H ? ty0 + ts : H;
    int tx0 = tx * ts, tx1 = tx0 + ts < W ? tx0 + ts : W;
    double dist[OR_MAXPTS];
    for (int64_t e = tile_off[t]; e < tile_off[t + 1]; e++) {
        int kk = items[e], i = V->order[kk];
        const int32_t *bb = V->bbox + 4 * i;
        int y0 = bb[2] > ty0 ? bb[2] : ty0, y1 = bb[3] < ty1 ? bb[3] : ty1;
        int x0 = bb[0] > tx0 ? bb[0] : tx0, x1 = bb[1] < tx1 ? bb[1] : tx1;
        if (y0 >= y1 || x0 >= x1) continue;
        const int h = V->hull_n[i];
        const double *nrm = V->normals + (size_t)i * k * 2, *off = V->offsets + (size_t)i * k;
        const double ds = V->delta_s[i], ss = V->sigma_s[i], o = V->opacity[i];
        const double *col = V->color + 3 * i;
        int any = 0;
        for (int y = y0; y < y1; y++) {
            for (int x = x0; x < x1; x++) {
                size_t p = (size_t)y * W + x;
                double T = F->trans[p];
                if (fd) {
                    if (!(cur[p] < fd->off[p + 1] && fd->pos[cur[p]] == e)) continue;
                    cur[p]++;
                } else if (flo > 0.0 && !(T >= flo)) {
                    continue;   /* dead pixel: blend predicate false */
                }
                double phi, ind;
                field_at(nrm, off, h, ds, ss, x + 0.5, y + 0.5, dist, &phi, &ind);
                (*ne)++;
                double a = o * ind;
                if (a > OR_ALPHA_MAX) a = OR_ALPHA_MAX;
                if (!fd && !(a >= cut)) continue;
                double w = T * a;
                F->image[3 * p] += w * col[0];
                F->image[3 * p + 1] += w * col[1];
                F->image[3 * p + 2] += w * col[2];
                F->wsum[p] += w;
                F->depth[p] += w * V->depth[i];
                F->trans[p] = T * (1.0 - a);
                F->count[p] += 1;
                any = 1;
                (*nb)++;
            }
        }
        if (any) F->visible[i] = 1;
    }
}

/* rasterize.py:156-209.  The frame buffers must be zeroed by the caller;
 * trans is initialised here.  tiles [t_begin, t_end) only (bounded CPU
 * samples); the background composite/clip runs over those tiles' pixels. */
int or_render_forced(const or_camera *cam, const or_settings *st, const or_view *V, const int64_t *tile_off,
                     const int32_t *items, int64_t t_begin, int64_t t_end, const int64_t *tile_list,
                     const or_forced *fd, or_frame *F);

int or_render(const or_camera *cam, const or_settings *st, const or_view *V, const int64_t *tile_off,
              const int32_t *items, int64_t t_begin, int64_t t_end, const int64_t *tile_list, or_frame *F) {
    return or_render_forced(cam, st, V, tile_off, items, t_begin, t_end, tile_list, NULL, F);
}

/* or_render with the blend decisions of `fd` (NULL: the reference's own). */
int or_render_forced(const or_camera *cam, const or_settings *st, const or_view *V, const int64_t *tile_off,
                     const int32_t *items, int64_t t_begin, int64_t t_end, const int64_t *tile_list,
                     const or_forced *fd, or_frame *F) {
    const int W = cam->width, H = cam->height, ts = st->tile;
    const int tx_n = (W + ts - 1) / ts;
    int64_t *cur = NULL;
    if (fd) {
        cur = malloc(sizeof(int64_t) * (size_t)W * H);
        if (!cur) return 1;
        memcpy(cur, fd->off, sizeof(int64_t) * (size_t)W * H);
    }
    for (size_t p = 0; p < (size_t)W * H; p++) F->trans[p] = 1.0;
    int64_t ne = 0, nb = 0;
#ifdef _OPENMP
    int nt = st->n_threads > 0 ? st->n_threads : 1;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : ne, nb) num_threads(nt)
#endif
    for (int64_t q = t_begin; q < t_end; q++)
        render_tile(cam, st, V, tile_off, items, tile_list ? tile_list[q] : q, F, &ne, &nb, fd, cur);
    F->n_eval = ne;
    F->n_blend = nb;
    /* rasterize.py:206-209 */
    for (int64_t q = t_begin; q < t_end; q++) {
        int64_t t = tile_list ? tile_list[q] : q;
        int ty = (int)(t / tx_n), tx = (int)(t % tx_n);
        for (int y = ty * ts; y < ty * ts + ts && y < H; y++)
            for (int x = tx * ts; x < tx * ts + ts && x < W; x++) {
                size_t p = (size_t)y * W + x;
                for (int c = 0; c < 3; c++) {
                    double v = F->image[3 * p + c] + F->trans[p] * st->background[c];
                    F->image[3 * p + c] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
                }
            }
    }
    free(cur);
    return 0;
}

/* ------------------------------------------------------------------ */
typedef struct {
    double *d_points;       /* [n,k,3] */
    double *d_raw_delta, *d_raw_sigma, *d_raw_opacity, *d_raw_mask;  /* [n] */
    double *d_sh;           /* [n,16,3] */
    uint8_t *visible;       /* [n] */
    int64_t n_eval;         /* reverse-walk evaluations (pixel in bbox, position <= last) */
} or_grads;

/* screen-space accumulators per prepared primitive (backward.py:102-108) */
typedef struct {
    double *d_color;    /* [V,3] */
    double *d_oeff, *d_sig, *d_del;  /* [V] */
    double *gn;         /* [V,k,2] */
    double *gs;         /* [V,k] */
} or_screen;

#ifdef _OPENMP
#define OR_ACC(dst, v) do { double v_ = (v); _Pragma("omp atomic") dst += v_; } while (0)
#else
#define OR_ACC(dst, v) ((dst) += (v))
#endif

/* backward.py:110-205 for one tile.  With `fd`, the blend predicate of
 * rasterize.py:194-195 / backward.py:146-150 and the clip test of
 * backward.py:154-158 are replaced by fd's recorded decisions; everything
 * else (field, transmittance, gradients) is recomputed in float64. */
static void backward_tile(const or_camera *cam, const or_settings *st, const or_view *V,
                          const int64_t *tile_off, const int32_t *items, int64_t t, const double *d_image,
                          or_screen *S, uint8_t *visible, int64_t *ne, const or_forced *fd) {
    const int W = cam->width, H = cam->height, ts = st->tile, k = V->k;
    const int tx_n = (W + ts - 1) / ts;
    const double cut = st->cutoff, flo = st->floor;
    int ty = (int)(t / tx_n), tx = (int)(t % tx_n);
    int ty0 = ty * ts, ty1 = ty0 + ts < H ? ty0 + ts : H;
    int tx0 = tx * ts, tx1 = tx0 + ts < W ? tx0 + ts : W;
    int th = ty1 - ty0, tw = tx1 - tx0;
    double T[256 * 4], cpre[256 * 4 * 3], S3[256 * 4 * 3], g[256 * 4 * 3];
    int last[256 * 4];
    int64_t cur[256 * 4];   /* forced: next recorded decision of the pixel */
    if (th * tw > 256 * 4) return;  /* tile sizes above 32x32 unsupported by the oracle */
    for (int p = 0; p < th * tw; p++) {
        T[p] = 1.0; last[p] = -1;
        cpre[3 * p] = cpre[3 * p + 1] = cpre[3 * p + 2] = 0.0;
        if (fd) cur[p] = fd->off[(size_t)(ty0 + p / tw) * W + tx0 + p % tw];
    }
    double dist[OR_MAXPTS], wts[OR_MAXPTS];
    int64_t e0 = tile_off[t], e1 = tile_off[t + 1];
    /* forward re-walk, backward.py:135-152 */
    for (int64_t e = e0; e < e1; e++) {
        int kk = items[e], i = V->order[kk];
        const int32_t *bb = V->bbox + 4 * i;
        int y0 = bb[2] > ty0 ? bb[2] : ty0, y1 = bb[3] < ty1 ? bb[3] : ty1;
        int x0 = bb[0] > tx0 ? bb[0] : tx0, x1 = bb[1] < tx1 ? bb[1] : tx1;
        if (y0 >= y1 || x0 >= x1) continue;
        const int h = V->hull_n[i];
        const double *nrm = V->normals + (size_t)i * k * 2, *off = V->offsets + (size_t)i * k;
        const double ds = V->delta_s[i], ss = V->sigma_s[i], o = V->opacity[i];
        const double *col = V->color + 3 * i;
        int any = 0;
        for (int y = y0; y < y1; y++) for (int x = x0; x < x1; x++) {
            int p = (y - ty0) * tw + (x - tx0);
            double phi, ind;
            field_at(nrm, off, h, ds, ss, x + 0.5, y + 0.5, dist, &phi, &ind);
            double a = o * ind;
            if (a > OR_ALPHA_MAX) a = OR_ALPHA_MAX;
            int blend;
            if (fd) {
                const size_t pix = (size_t)y * W + x;
                blend = cur[p] < fd->off[pix + 1] && fd->pos[cur[p]] == e;
                if (blend) cur[p]++;
            } else {
                blend = (flo > 0.0) ? (T[p] >= flo && a >= cut) : (a >= cut);
            }
            if (!blend) continue;
            double w = T[p] * a;
            for (int c = 0; c < 3; c++) cpre[3 * p + c] += w * col[c];
            T[p] *= 1.0 - a;
            last[p] = kk;
            any = 1;
        }
        if (any) visible[i] = 1;
    }
    /* backward.py:154-162 */
    for (int p = 0; p < th * tw; p++) {
        int y = ty0 + p / tw, x = tx0 + p % tw;
        if (fd) cur[p] = fd->off[(size_t)y * W + x + 1] - 1;   /* reverse cursor */
        for (int c = 0; c < 3; c++) {
            double v = cpre[3 * p + c] + T[p] * st->background[c];
            int inside = (v >= 0.0) && (v <= 1.0);
            if (fd && fd->clamp) inside = (fd->clamp[(size_t)y * W + x] >> c) & 1;
            g[3 * p + c] = inside ? d_image[((size_t)y * W + x) * 3 + c] : 0.0;
            S3[3 * p + c] = T[p] * st->background[c];
        }
    }
    /* back to front, backward.py:163-205 */
    for (int64_t e = e1 - 1; e >= e0; e--) {
        int kk = items[e], i = V->order[kk];
        const int32_t *bb = V->bbox + 4 * i;
        int y0 = bb[2] > ty0 ? bb[2] : ty0, y1 = bb[3] < ty1 ? bb[3] : ty1;
        int x0 = bb[0] > tx0 ? bb[0] : tx0, x1 = bb[1] < tx1 ? bb[1] : tx1;
        if (y0 >= y1 || x0 >= x1) continue;
        const int h = V->hull_n[i];
        const double *nrm = V->normals + (size_t)i * k * 2, *off = V->offsets + (size_t)i * k;
        const double ds = V->delta_s[i], ss = V->sigma_s[i], o = V->opacity[i];
        const double *col = V->color + 3 * i;
        double acc_col[3] = {0, 0, 0}, acc_o = 0, acc_sig = 0, acc_del = 0;
        double acc_gn[OR_MAXPTS][2], acc_gs[OR_MAXPTS];
        for (int j = 0; j < h; j++) { acc_gn[j][0] = acc_gn[j][1] = 0.0; acc_gs[j] = 0.0; }
        int touched = 0;
        for (int y = y0; y < y1; y++) for (int x = x0; x < x1; x++) {
            int p = (y - ty0) * tw + (x - tx0);
            if (!(kk <= last[p])) continue;
            double qx = x + 0.5, qy = y + 0.5, phi, ind;
            field_at(nrm, off, h, ds, ss, qx, qy, dist, &phi, &ind);
            (*ne)++;
            double a_raw = o * ind;
            double a = a_raw < OR_ALPHA_MAX ? a_raw : OR_ALPHA_MAX;
            if (fd) {
                const size_t pix = (size_t)y * W + x;
                if (!(cur[p] >= fd->off[pix] && fd->pos[cur[p]] == e)) continue;
                cur[p]--;
            } else if (!(a >= cut)) {
                continue;
            }
            touched = 1;
            double om = 1.0 - a;
            double tp = T[p] / om;
            double w = tp * a;
            double *gg = g + 3 * p, *sb = S3 + 3 * p;
            for (int c = 0; c < 3; c++) acc_col[c] += gg[c] * w;
            double dA = 0.0;
            for (int c = 0; c < 3; c++) dA += gg[c] * (tp * col[c] - sb[c] / om);
            if (!(a_raw < OR_ALPHA_MAX)) dA = 0.0;
            double dI = dA * o;
            acc_o += dA * ind;
            double slope = ind * (1.0 - ind);
            double dphi = dI * (-ss) * slope;
            acc_sig += dI * (-phi) * slope;
            /* field.py:62-67 softmax_over_lines */
            double m = -INFINITY;
            for (int j = 0; j < h; j++) { double zj = ds * dist[j]; if (zj > m) m = zj; }
            double den = 0.0;
            for (int j = 0; j < h; j++) { wts[j] = exp(ds * dist[j] - m); den += wts[j]; }
            double wl = 0.0;
            for (int j = 0; j < h; j++) { wts[j] /= den; wl += wts[j] * dist[j]; }
            acc_del += dphi * wl;
            for (int j = 0; j < h; j++) {
                double dl = dphi * ds * wts[j];
                acc_gn[j][0] += dl * qx;
                acc_gn[j][1] += dl * qy;
                acc_gs[j] += dl;
            }
            for (int c = 0; c < 3; c++) sb[c] += w * col[c];
            T[p] = tp;
        }
        if (!touched) continue;
        for (int c = 0; c < 3; c++) OR_ACC(S->d_color[3 * kk + c], acc_col[c]);
        OR_ACC(S->d_oeff[kk], acc_o);
        OR_ACC(S->d_sig[kk], acc_sig);
        OR_ACC(S->d_del[kk], acc_del);
        for (int j = 0; j < h; j++) {
            OR_ACC(S->gn[((size_t)kk * k + j) * 2], acc_gn[j][0]);
            OR_ACC(S->gn[((size_t)kk * k + j) * 2 + 1], acc_gn[j][1]);
            OR_ACC(S->gs[(size_t)kk * k + j], acc_gs[j]);
        }
    }
}

/* backward.py:215-282, one prepared primitive */
static void chain_one(const or_camera *cam, const or_settings *st, const or_params *P, const or_view *V,
                      const or_screen *S, int kk, or_grads *G) {
    const int k = V->k, i = V->order[kk], h = V->hull_n[i];
    const int32_t *hull = V->hull + (size_t)i * k;
    const double *px = V->pixels + (size_t)i * k * 2;
    const double *nrm = V->normals + (size_t)i * k * 2;
    const double *gn0 = S->gn + (size_t)kk * k * 2, *gs = S->gs + (size_t)kk * k;
    double dpix[OR_MAXPTS][2];
    for (int j = 0; j < k; j++) dpix[j][0] = dpix[j][1] = 0.0;
    double de[OR_MAXPTS][2];
    for (int j = 0; j < h; j++) {
        const double *v0 = px + 2 * hull[j], *v1 = px + 2 * hull[(j + 1) % h];
        double ex = v1[0] - v0[0], ey = v1[1] - v0[1];
        double raw_len = hypot(ey, ex);
        double gx = gn0[2 * j] - gs[j] * v0[0], gy = gn0[2 * j + 1] - gs[j] * v0[1];
        double nd = nrm[2 * j] * gx + nrm[2 * j + 1] * gy;
        double rx = (gx - nrm[2 * j] * nd) / raw_len, ry = (gy - nrm[2 * j + 1] * nd) / raw_len;
        de[j][0] = -ry;
        de[j][1] = rx;
    }
    for (int j = 0; j < h; j++) {   /* np.add.at(d_pix, idx_b, d_edge) */
        int b = hull[(j + 1) % h];
        dpix[b][0] += de[j][0];
        dpix[b][1] += de[j][1];
    }
    for (int j = 0; j < h; j++) {   /* np.add.at(d_pix, idx_a, -d_edge - n*gs) */
        int a = hull[j];
        dpix[a][0] += -de[j][0] - nrm[2 * j] * gs[j];
        dpix[a][1] += -de[j][1] - nrm[2 * j + 1] * gs[j];
    }
    const double *pts = P->points + (size_t)i * k * 3;
    double *dp = G->d_points + (size_t)i * k * 3;
    const double *R = cam->R;
    for (int j = 0; j < k; j++) {
        const double *p = pts + 3 * j;
        double xc[3];
        for (int c = 0; c < 3; c++)
            xc[c] = fma(p[2], R[3 * c + 2], fma(p[1], R[3 * c + 1], p[0] * R[3 * c])) + cam->t[c];
        double gx = dpix[j][0], gy = dpix[j][1], dc[3];
        if (cam->ortho) {
            dc[0] = cam->fx * gx; dc[1] = cam->fy * gy; dc[2] = 0.0;
        } else {
            double z = xc[2];
            dc[0] = cam->fx / z * gx;
            dc[1] = cam->fy / z * gy;
            dc[2] = -(cam->fx * xc[0] / (z * z)) * gx - (cam->fy * xc[1] / (z * z)) * gy;
        }
        for (int c = 0; c < 3; c++) dp[3 * j + c] += dc[0] * R[c] + dc[1] * R[3 + c] + dc[2] * R[6 + c];
    }
    const double delta = exp(P->raw_delta[i]), sigma = exp(P->raw_sigma[i]), s = V->scale[i];
    const double dd = S->d_del[kk], dsg = S->d_sig[kk];
    G->d_raw_delta[i] += dd * s * delta;
    G->d_raw_sigma[i] += dsg * s * sigma;
    if (!cam->ortho) {
        double d_depth = (dd * delta + dsg * sigma) * depth_scale_grad(st->mode, V->depth[i]);
        for (int j = 0; j < k; j++)
            for (int c = 0; c < 3; c++) dp[3 * j + c] += d_depth * R[6 + c] / k;
    }
    const double o = expit(P->raw_opacity[i]), m = expit(P->raw_mask[i]), doe = S->d_oeff[kk];
    G->d_raw_opacity[i] += doe * o * (1.0 - o);
    G->d_raw_mask[i] += doe * o * m * (1.0 - m);
    /* harmonics.py:112-128 */
    const double *dir = V->view_dir + 3 * i;
    const double *sh = P->sh + (size_t)i * OR_SH_COEFFS * 3;
    double basis[16], bg[16][3];
    int nb = sh_basis(dir, st->sh_degree, basis);
    double deff[3];
    for (int c = 0; c < 3; c++) {
        double raw = 0.0;
        for (int b = 0; b < nb; b++) raw += basis[b] * sh[3 * b + c];
        raw = 0.5 + raw;
        deff[c] = raw > 0.0 ? S->d_color[3 * kk + c] : 0.0;
    }
    double *dsh = G->d_sh + (size_t)i * OR_SH_COEFFS * 3;
    for (int b = 0; b < nb; b++) for (int c = 0; c < 3; c++) dsh[3 * b + c] += basis[b] * deff[c];
    sh_basis_grad(dir, st->sh_degree, bg);
    double ddir[3] = {0, 0, 0};
    for (int b = 0; b < nb; b++) {
        double vb = sh[3 * b] * deff[0] + sh[3 * b + 1] * deff[1] + sh[3 * b + 2] * deff[2];
        for (int a = 0; a < 3; a++) ddir[a] += bg[b][a] * vb;
    }
    double dot = dir[0] * ddir[0] + dir[1] * ddir[1] + dir[2] * ddir[2];
    double dist = V->view_dist[i];
    for (int c = 0; c < 3; c++) {
        double dcen = (ddir[c] - dir[c] * dot) / dist;
        for (int j = 0; j < k; j++) dp[3 * j + c] += dcen / k;
    }
}

/* backward.py:76-212.  Gradient buffers must be zeroed by the caller
 * (accumulation semantics of GradientBuffer.add, backward.py:65-73). */
int or_backward_forced(const or_camera *cam, const or_settings *st, const or_params *P, const or_view *V,
                       const int64_t *tile_off, const int32_t *items, const double *d_image,
                       const int64_t *tile_list, int64_t n_list, const or_forced *fd, or_grads *G);

int or_backward(const or_camera *cam, const or_settings *st, const or_params *P, const or_view *V,
                const int64_t *tile_off, const int32_t *items, const double *d_image, const int64_t *tile_list,
                int64_t n_list, or_grads *G) {
    return or_backward_forced(cam, st, P, V, tile_off, items, d_image, tile_list, n_list, NULL, G);
}

/* or_backward with the blend / clip decisions of `fd` (NULL: the reference's own). */
int or_backward_forced(const or_camera *cam, const or_settings *st, const or_params *P, const or_view *V,
                       const int64_t *tile_off, const int32_t *items, const double *d_image,
                       const int64_t *tile_list, int64_t n_list, const or_forced *fd, or_grads *G) {
    const int W = cam->width, H = cam->height, ts = st->tile, k = V->k;
    const int64_t T = (int64_t)((W + ts - 1) / ts) * ((H + ts - 1) / ts);
    const int nv = V->n_visible;
    if (ts * ts > 1024) return 1;
    or_screen S;
    S.d_color = calloc((size_t)nv * 3 + 1, sizeof(double));
    S.d_oeff = calloc((size_t)nv + 1, sizeof(double));
    S.d_sig = calloc((size_t)nv + 1, sizeof(double));
    S.d_del = calloc((size_t)nv + 1, sizeof(double));
    S.gn = calloc((size_t)nv * k * 2 + 1, sizeof(double));
    S.gs = calloc((size_t)nv * k + 1, sizeof(double));
    int64_t ne = 0;
    const int64_t nt_list = tile_list ? n_list : T;
#ifdef _OPENMP
    int nt = st->n_threads > 0 ? st->n_threads : 1;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : ne) num_threads(nt)
#endif
    for (int64_t q = 0; q < nt_list; q++)
        backward_tile(cam, st, V, tile_off, items, tile_list ? tile_list[q] : q, d_image, &S, G->visible, &ne, fd);
    G->n_eval = ne;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 256) num_threads(nt)
#endif
    for (int kk = 0; kk < nv; kk++) chain_one(cam, st, P, V, &S, kk, G);
    free(S.d_color); free(S.d_oeff); free(S.d_sig); free(S.d_del); free(S.gn); free(S.gs);
    return 0;
}

int or_max_points(void) { return OR_MAXPTS; }

/* The reference's own blend decisions (rasterize.py:178-204), in the format
 * of or_forced: with pos == NULL, writes counts[p] (blends of pixel p); with
 * pos, writes pixel p's blended pair indices at pos[off[p] ...] in blend
 * order (off = exclusive scan of the counts). */
int or_blend_decisions(const or_camera *cam, const or_settings *st, const or_view *V, const int64_t *tile_off,
                       const int32_t *items, int64_t *counts_or_off, int32_t *pos) {
    const int W = cam->width, H = cam->height, ts = st->tile, k = V->k;
    const int tx_n = (W + ts - 1) / ts, ty_n = (H + ts - 1) / ts;
    double dist[OR_MAXPTS];
    double *T = malloc(sizeof(double) * (size_t)W * H);
    int64_t *cur = malloc(sizeof(int64_t) * (size_t)W * H);
    if (!T || !cur) { free(T); free(cur); return 1; }
    for (size_t p = 0; p < (size_t)W * H; p++) {
        T[p] = 1.0;
        cur[p] = pos ? counts_or_off[p] : 0;
    }
    for (int64_t t = 0; t < (int64_t)tx_n * ty_n; t++) {
        int ty = (int)(t / tx_n), tx = (int)(t % tx_n);
        int ty0 = ty * ts, ty1 = ty0 + ts < H ? ty0 + ts : H;
        int tx0 = tx * ts, tx1 = tx0 + ts < W ? tx0 + ts : W;
        for (int64_t e = tile_off[t]; e < tile_off[t + 1]; e++) {
            int i = V->order[items[e]];
            const int32_t *bb = V->bbox + 4 * i;
            int y0 = bb[2] > ty0 ? bb[2] : ty0, y1 = bb[3] < ty1 ? bb[3] : ty1;
            int x0 = bb[0] > tx0 ? bb[0] : tx0, x1 = bb[1] < tx1 ? bb[1] : tx1;
            const double *nrm = V->normals + (size_t)i * k * 2, *off = V->offsets + (size_t)i * k;
            for (int y = y0; y < y1; y++)
                for (int x = x0; x < x1; x++) {
                    size_t p = (size_t)y * W + x;
                    if (st->floor > 0.0 && !(T[p] >= st->floor)) continue;
                    double phi, ind;
                    field_at(nrm, off, V->hull_n[i], V->delta_s[i], V->sigma_s[i], x + 0.5, y + 0.5, dist, &phi,
                             &ind);
                    double a = V->opacity[i] * ind;
                    if (a > OR_ALPHA_MAX) a = OR_ALPHA_MAX;
                    if (!(a >= st->cutoff)) continue;
                    T[p] *= 1.0 - a;
                    if (pos) pos[cur[p]] = (int32_t)e;
                    cur[p]++;
                }
        }
    }
    if (!pos)
        for (size_t p = 0; p < (size_t)W * H; p++) counts_or_off[p] = cur[p];
    free(T);
    free(cur);
    return 0;
}

/* Analysis helper (test only): the pixels whose reference walk
 * (rasterize.py:178-204, as or_blend_decisions) meets a decision within
 * relative eps of its threshold -- alpha against the cutoff, or T against the
 * floor.  A float32 renderer may decide those either way; near_tie[p] = 1. */
int or_near_ties(const or_camera *cam, const or_settings *st, const or_view *V, const int64_t *tile_off,
                 const int32_t *items, double eps, uint8_t *near_tie) {
    const int W = cam->width, H = cam->height, ts = st->tile, k = V->k;
    const int tx_n = (W + ts - 1) / ts, ty_n = (H + ts - 1) / ts;
    double dist[OR_MAXPTS];
    double *T = malloc(sizeof(double) * (size_t)W * H);
    if (!T) return 1;
    for (size_t p = 0; p < (size_t)W * H; p++) { T[p] = 1.0; near_tie[p] = 0; }
    for (int64_t t = 0; t < (int64_t)tx_n * ty_n; t++) {
        int ty = (int)(t / tx_n), tx = (int)(t % tx_n);
        int ty0 = ty * ts, ty1 = ty0 + ts < H ? ty0 + ts : H;
        int tx0 = tx * ts, tx1 = tx0 + ts < W ? tx0 + ts : W;
        for (int64_t e = tile_off[t]; e < tile_off[t + 1]; e++) {
            int i = V->order[items[e]];
            const int32_t *bb = V->bbox + 4 * i;
            int y0 = bb[2] > ty0 ? bb[2] : ty0, y1 = bb[3] < ty1 ? bb[3] : ty1;
            int x0 = bb[0] > tx0 ? bb[0] : tx0, x1 = bb[1] < tx1 ? bb[1] : tx1;
            const double *nrm = V->normals + (size_t)i * k * 2, *off = V->offsets + (size_t)i * k;
            for (int y = y0; y < y1; y++)
                for (int x = x0; x < x1; x++) {
                    size_t p = (size_t)y * W + x;
                    if (st->floor > 0.0) {
                        if (fabs(T[p] - st->floor) <= eps * st->floor) near_tie[p] = 1;
                        if (!(T[p] >= st->floor)) continue;
                    }
                    double phi, ind;
                    field_at(nrm, off, V->hull_n[i], V->delta_s[i], V->sigma_s[i], x + 0.5, y + 0.5, dist, &phi,
                             &ind);
                    double a = V->opacity[i] * ind;
                    if (a > OR_ALPHA_MAX) a = OR_ALPHA_MAX;
                    if (fabs(a - st->cutoff) <= eps * st->cutoff) near_tie[p] = 1;
                    if (!(a >= st->cutoff)) continue;
                    T[p] *= 1.0 - a;
                }
        }
    }
    free(T);
    return 0;
}

/* Analysis helper (test/tooling only): for each listed tile, the 256-bit
 * mask (bit = ly*16+lx) of pixels that EVALUATE each candidate of the tile
 * list in the reference walk (bbox holds the pixel and T >= floor when the
 * candidate is reached), in list order.  masks: [sum of list lengths][8]. */
int64_t or_eval_masks(const or_camera *cam, const or_settings *st, const or_view *V, const int64_t *tile_off,
                      const int32_t *items, const int64_t *tile_list, int64_t n_list, uint32_t *masks) {
    const int W = cam->width, H = cam->height, ts = st->tile, k = V->k;
    const int tx_n = (W + ts - 1) / ts;
    double dist[OR_MAXPTS];
    int64_t w = 0;
    if (ts != 16) return -1;
    for (int64_t q = 0; q < n_list; q++) {
        int64_t t = tile_list[q];
        int ty = (int)(t / tx_n), tx = (int)(t % tx_n);
        int ty0 = ty * ts, tx0 = tx * ts;
        double T[256];
        for (int p = 0; p < 256; p++) T[p] = 1.0;
        for (int64_t e = tile_off[t]; e < tile_off[t + 1]; e++, w++) {
            uint32_t *m = masks + 8 * w;
            for (int b = 0; b < 8; b++) m[b] = 0;
            int i = V->order[items[e]];
            const int32_t *bb = V->bbox + 4 * i;
            const int h = V->hull_n[i];
            const double *nrm = V->normals + (size_t)i * k * 2, *off = V->offsets + (size_t)i * k;
            for (int ly = 0; ly < 16; ly++) for (int lx = 0; lx < 16; lx++) {
                int x = tx0 + lx, y = ty0 + ly, p = ly * 16 + lx;
                if (x >= W || y >= H || x < bb[0] || x >= bb[1] || y < bb[2] || y >= bb[3]) continue;
                if (st->floor > 0.0 && !(T[p] >= st->floor)) continue;
                m[p >> 5] |= 1u << (p & 31);
                double phi, ind;
                field_at(nrm, off, h, V->delta_s[i], V->sigma_s[i], x + 0.5, y + 0.5, dist, &phi, &ind);
                double a = V->opacity[i] * ind;
                if (a > OR_ALPHA_MAX) a = OR_ALPHA_MAX;
                if (a >= st->cutoff) T[p] *= 1.0 - a;
            }
        }
    }
    return w;
}
