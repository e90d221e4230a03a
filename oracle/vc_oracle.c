/*
 * vc_oracle.c -- CPU restatement of the voxelcast per-pixel raycaster.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle for the
 * B200 kernels in paper_1609_01317_b200/csrc.  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl
 * reference leg may load it.  The product path never links it.
 *
 * It restates, function by function, the float64 arithmetic of the
 * reference kernel layer /root/reference/pkg/src/voxelcast/_kernels.py
 * (numba, fastmath off, no FMA contraction -- compile with
 * -ffp-contract=off).  Every function cites the reference lines it
 * follows.  By default the oracle is the brute-force renderer
 * (render_frame(..., use_octree=False)), which the reference guarantees is
 * pixel-identical to the octree path (pkg/tests/test_render.py:125-139);
 * with use_octree set it marches the reference's merged octree segments
 * (collect_segments, _kernels.py:267-342), which changes the sample count
 * and, under use_adaptive, which samples exist.  The adaptive stride
 * (use_adaptive, _kernels.py:437-463) and the segments are restated over the
 * reference's flat octree arrays (built by oracle.build_octree_flat).
 *
 * Parity is pinned against golden fixtures produced by running the
 * reference itself (tests/golden/make_golden.py).
 *
 * Voxel storage: dtype 0 = uint8, 1 = uint16, 2 = float32; flat with x
 * fastest (volume.py:51-52, _kernels.py:41-42).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define VCO_MAX_LUT 64

/* _kernels.py:14-30 */
enum { INTERP_NEAREST = 0, INTERP_LINEAR = 1, INTERP_TRILINEAR = 2 };
enum { OP_CENTRAL = 0, OP_SOBEL3D = 1, OP_ZUCKER_HUMMEL = 2 };
enum { MODE_SURFACE = 0, MODE_COMPOSITED = 1 };
static const double GRAD_EPS = 1e-8;
#define OPAQUE_ALPHA (1.0 - 1e-6)
static const double MIN_REMAINING = 0.01;
static const int GRAD_SAMPLES[3] = {6, 26, 26};

typedef struct {
    const void *data;
    int dtype;
    int nx, ny, nz;
} vco_vol;

/* Scalars of _kernels.render_tile (_kernels.py:583-627) minus the octree. */
typedef struct {
    double spacing[3];
    double eye[3], right[3], up[3], fwd[3];
    double half_w, half_h;
    int32_t width, height;
    double clip_lo[3], clip_hi[3];
    double light_pos[3], light_col[3];
    double t_low, t_high;
    int32_t lut_n;
    double lut_hu[VCO_MAX_LUT];
    double lut_rgba[VCO_MAX_LUT * 4];
    double mu_water;
    int32_t op, interp, mode;
    double coarse, fine;
    int32_t refine_iters;
    double bg[4];
    /* adaptive stride (use_adaptive, _kernels.py:437-463) over the
     * reference's flat octree arrays (octree.py:111-136) */
    int32_t use_adaptive, adapt_jump;
    double detail_eps;
    const int32_t *nbounds;   /* N x 6 (lo xyz, hi xyz) */
    const double *sminmax;    /* N x 2 padded range */
    const int32_t *nchildren; /* N x 8, -1 padded */
    /* use_octree (raycast.py:187): march only the merged t-segments of
     * octree leaves whose padded range overlaps the window
     * (collect_segments, _kernels.py:267-342) */
    int32_t use_octree;
} vco_params;

/* _kernels.py:35-37 */
static inline double lerp(double f0, double f1, double t) { return f0 + (f1 - f0) * t; }

/* _kernels.py:40-42 */
static inline double fetch(const vco_vol *v, int i, int j, int k) {
    int64_t idx = ((int64_t)k * v->ny + j) * (int64_t)v->nx + i;
    switch (v->dtype) {
    case 0: return (double)((const uint8_t *)v->data)[idx];
    case 1: return (double)((const uint16_t *)v->data)[idx];
    default: return (double)((const float *)v->data)[idx];
    }
}

/* _kernels.py:45-49 */
static inline double round_half_away(double x) {
    if (x >= 0.0) return floor(x + 0.5);
    return ceil(x - 0.5);
}

/* _kernels.py:52-64 */
static inline void cell(double v, int n, int *i0, int *i1, double *f) {
    int a = (int)floor(v);
    if (a > n - 2) a = n - 2;
    if (a < 0) a = 0;
    int b = a + 1;
    if (b > n - 1) b = n - 1;
    *i0 = a;
    *i1 = b;
    *f = v - (double)a;
}

/* _kernels.py:67-72 */
static double sample_nearest(const vco_vol *v, double x, double y, double z) {
    return fetch(v, (int)round_half_away(x), (int)round_half_away(y), (int)round_half_away(z));
}

/* _kernels.py:75-101 */
static double sample_linear(const vco_vol *v, double x, double y, double z) {
    double fx = fabs(x - round_half_away(x));
    double fy = fabs(y - round_half_away(y));
    double fz = fabs(z - round_half_away(z));
    int axis;
    if (fy > fx && fy >= fz) axis = 1;
    else if (fz > fx && fz > fy) axis = 2;
    else axis = 0;
    int a0, a1;
    double f;
    if (axis == 0) {
        int j = (int)round_half_away(y), k = (int)round_half_away(z);
        cell(x, v->nx, &a0, &a1, &f);
        return lerp(fetch(v, a0, j, k), fetch(v, a1, j, k), f);
    }
    if (axis == 1) {
        int i = (int)round_half_away(x), k = (int)round_half_away(z);
        cell(y, v->ny, &a0, &a1, &f);
        return lerp(fetch(v, i, a0, k), fetch(v, i, a1, k), f);
    }
    int i = (int)round_half_away(x), j = (int)round_half_away(y);
    cell(z, v->nz, &a0, &a1, &f);
    return lerp(fetch(v, i, j, a0), fetch(v, i, j, a1), f);
}

/* _kernels.py:104-115 */
static double sample_trilinear(const vco_vol *v, double x, double y, double z) {
    int i0, i1, j0, j1, k0, k1;
    double fx, fy, fz;
    cell(x, v->nx, &i0, &i1, &fx);
    cell(y, v->ny, &j0, &j1, &fy);
    cell(z, v->nz, &k0, &k1, &fz);
    double x00 = lerp(fetch(v, i0, j0, k0), fetch(v, i1, j0, k0), fx);
    double x10 = lerp(fetch(v, i0, j1, k0), fetch(v, i1, j1, k0), fx);
    double x01 = lerp(fetch(v, i0, j0, k1), fetch(v, i1, j0, k1), fx);
    double x11 = lerp(fetch(v, i0, j1, k1), fetch(v, i1, j1, k1), fx);
    double y0 = lerp(x00, x10, fy);
    double y1 = lerp(x01, x11, fy);
    return lerp(y0, y1, fz);
}

/* _kernels.py:118-127 */
static double sample_any(const vco_vol *v, double x, double y, double z, int interp) {
    if (x < 0.0 || x > (double)(v->nx - 1) || y < 0.0 || y > (double)(v->ny - 1) || z < 0.0 ||
        z > (double)(v->nz - 1))
        return 0.0;
    if (interp == INTERP_TRILINEAR) return sample_trilinear(v, x, y, z);
    if (interp == INTERP_LINEAR) return sample_linear(v, x, y, z);
    return sample_nearest(v, x, y, z);
}

/* _kernels.py:130-137 */
static inline double smooth_weight(int u, int w) {
    if (u == 0 && w == 0) return 6.0;
    if (u == 0 || w == 0) return 3.0;
    return 1.0;
}

/* _kernels.py:140-177; taps are always trilinear (interp code 2). */
static void grad_raw(const vco_vol *v, double x, double y, double z, int op, double g[3]) {
    double gx = 0.0, gy = 0.0, gz = 0.0;
    if (op == OP_CENTRAL) {
        gx = sample_any(v, x + 1.0, y, z, 2) - sample_any(v, x - 1.0, y, z, 2);
        gy = sample_any(v, x, y + 1.0, z, 2) - sample_any(v, x, y - 1.0, z, 2);
        gz = sample_any(v, x, y, z + 1.0, 2) - sample_any(v, x, y, z - 1.0, 2);
    } else if (op == OP_SOBEL3D) {
        for (int i = -1; i < 2; i++)
            for (int j = -1; j < 2; j++)
                for (int k = -1; k < 2; k++) {
                    if (i == 0 && j == 0 && k == 0) continue;
                    double s = sample_any(v, x + (double)i, y + (double)j, z + (double)k, 2);
                    gx += ((double)i * smooth_weight(j, k)) * s;
                    gy += ((double)j * smooth_weight(i, k)) * s;
                    gz += ((double)k * smooth_weight(i, j)) * s;
                }
    } else {
        for (int i = -1; i < 2; i++)
            for (int j = -1; j < 2; j++)
                for (int k = -1; k < 2; k++) {
                    if (i == 0 && j == 0 && k == 0) continue;
                    double s = sample_any(v, x + (double)i, y + (double)j, z + (double)k, 2);
                    double inv = 1.0 / sqrt((double)(i * i + j * j + k * k));
                    gx += ((double)i * inv) * s;
                    gy += ((double)j * inv) * s;
                    gz += ((double)k * inv) * s;
                }
    }
    g[0] = gx;
    g[1] = gy;
    g[2] = gz;
}

/* _kernels.py:180-185 */
static void normalize3(const double g[3], double eps, double u[3]) {
    double n = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    if (n <= eps) {
        u[0] = u[1] = u[2] = 0.0;
        return;
    }
    u[0] = g[0] / n;
    u[1] = g[1] / n;
    u[2] = g[2] / n;
}

/* _kernels.py:188-212 */
static int slab_interval(const double org[3], const double dirv[3], const double lo[3],
                         const double hi[3], double *t0, double *t1) {
    double tmin = -1e300, tmax = 1e300;
    for (int a = 0; a < 3; a++) {
        double o = org[a], d = dirv[a];
        if (d == 0.0) {
            if (o < lo[a] || o > hi[a]) return 0;
        } else {
            double inv = 1.0 / d;
            double ta = (lo[a] - o) * inv;
            double tb = (hi[a] - o) * inv;
            if (ta > tb) {
                double s = ta;
                ta = tb;
                tb = s;
            }
            if (ta > tmin) tmin = ta;
            if (tb < tmax) tmax = tb;
        }
    }
    if (tmin > tmax) return 0;
    *t0 = tmin;
    *t1 = tmax;
    return 1;
}

/* _kernels.py:215-224 */
int vco_box_interval(const double org[3], const double dirv[3], const double lo[3],
                     const double hi[3], double out[2]) {
    double t0 = 0.0, t1 = 0.0;
    int hit = slab_interval(org, dirv, lo, hi, &t0, &t1);
    if (!hit || t1 < 0.0) {
        out[0] = out[1] = 0.0;
        return 0;
    }
    if (t0 < 0.0) t0 = 0.0;
    out[0] = t0;
    out[1] = t1;
    return 1;
}

static inline void voxel_pos(const double org[3], const double dirv[3], const double sp[3],
                             double t, double p[3]) {
    /* _kernels.py:414-416 */
    p[0] = (org[0] + t * dirv[0]) / sp[0] - 0.5;
    p[1] = (org[1] + t * dirv[1]) / sp[1] - 0.5;
    p[2] = (org[2] + t * dirv[2]) / sp[2] - 0.5;
}

/* _kernels.py:345-364 */
static int leaf_for_point(const vco_params *P, int ix, int iy, int iz) {
    int idx = 0;
    while (P->nchildren[idx * 8] >= 0) {
        int nxt = idx;
        for (int c = 0; c < 8; c++) {
            int ci = P->nchildren[idx * 8 + c];
            if (ci < 0) break;
            const int32_t *b = P->nbounds + ci * 6;
            if (b[0] <= ix && ix < b[3] && b[1] <= iy && iy < b[4] && b[2] <= iz && iz < b[5]) {
                nxt = ci;
                break;
            }
        }
        if (nxt == idx) break;
        idx = nxt;
    }
    return idx;
}

/* _kernels.py:227-264 */
static int node_interval(const vco_params *P, int idx, const double sp[3], const double org[3],
                         const double dirv[3], double *t0, double *t1) {
    const int32_t *b = P->nbounds + idx * 6;
    double tmin = -1e300, tmax = 1e300;
    for (int a = 0; a < 3; a++) {
        double lo = (double)b[a] * sp[a], hi = (double)b[3 + a] * sp[a];
        double o = org[a], d = dirv[a];
        if (d == 0.0) {
            if (o < lo || o > hi) return 0;
        } else {
            double inv = 1.0 / d;
            double ta = (lo - o) * inv, tb = (hi - o) * inv;
            if (ta > tb) {
                double s = ta;
                ta = tb;
                tb = s;
            }
            if (ta > tmin) tmin = ta;
            if (tb < tmax) tmax = tb;
        }
    }
    if (tmin > tmax) return 0;
    *t0 = tmin;
    *t1 = tmax;
    return 1;
}

/* _kernels.py:437-463: lattice steps after an out-of-window sample at p */
static int64_t adaptive_stride(const vco_vol *v, const vco_params *P, const double sp[3],
                               const double org[3], const double dirv[3], const double p[3],
                               int64_t k, double t_enter, double coarse) {
    int64_t step_k = 1;
    int ix = (int)floor(p[0]), iy = (int)floor(p[1]), iz = (int)floor(p[2]);
    if (ix < 0) ix = 0;
    if (iy < 0) iy = 0;
    if (iz < 0) iz = 0;
    if (ix > v->nx - 1) ix = v->nx - 1;
    if (iy > v->ny - 1) iy = v->ny - 1;
    if (iz > v->nz - 1) iz = v->nz - 1;
    int leaf = leaf_for_point(P, ix, iy, iz);
    if (P->sminmax[leaf * 2 + 1] - P->sminmax[leaf * 2] < P->detail_eps) {
        double la, lb;
        if (node_interval(P, leaf, sp, org, dirv, &la, &lb)) {
            step_k = P->adapt_jump;
            int64_t kex = (int64_t)floor((lb - t_enter) / coarse) + 1;
            if (kex - k < step_k) step_k = kex - k;
            if (step_k < 1) step_k = 1;
        }
    }
    return step_k;
}

#define VCO_SEG_CAP 4096   /* seg0 / seg1 of raycast.py:499 */
#define VCO_STACK_CAP 512  /* stack of raycast.py:499 */

/* _kernels.py:267-342: depth-first near-to-far walk emitting the merged
 * t-intervals of leaves whose padded range overlaps [t_low, t_high]. */
static int collect_segments(const vco_params *P, const double sp[3], const double org[3],
                            const double dirv[3], double tray0, double tray1, double t_low,
                            double t_high, int32_t *stack, double *seg0, double *seg1) {
    int nseg = 0, top = 0;
    stack[top++] = 0;
    double child_t[8];
    int32_t child_i[8];
    while (top > 0) {
        int32_t idx = stack[--top];
        double a0, b0;
        if (!node_interval(P, idx, sp, org, dirv, &a0, &b0)) continue;
        if (a0 < tray0) a0 = tray0;
        if (b0 > tray1) b0 = tray1;
        if (b0 < a0) continue;
        if (P->nchildren[idx * 8] < 0) {
            if (P->sminmax[idx * 2] <= t_high && P->sminmax[idx * 2 + 1] >= t_low) {
                if (nseg > 0 && a0 <= seg1[nseg - 1] + 1e-9) {
                    if (b0 > seg1[nseg - 1]) seg1[nseg - 1] = b0;
                } else if (nseg < VCO_SEG_CAP) {
                    seg0[nseg] = a0;
                    seg1[nseg] = b0;
                    nseg++;
                } else {
                    seg1[nseg - 1] = b0;
                }
            }
        } else {
            int cnt = 0;
            for (int c = 0; c < 8; c++) {
                int32_t ci = P->nchildren[idx * 8 + c];
                if (ci < 0) break;
                double ca, cb;
                if (!node_interval(P, ci, sp, org, dirv, &ca, &cb) || cb < tray0 || ca > tray1) continue;
                child_t[cnt] = ca;
                child_i[cnt] = ci;
                cnt++;
            }
            /* insertion sort, farthest entry first so nearest pops first */
            for (int a = 1; a < cnt; a++) {
                double tv = child_t[a];
                int32_t iv = child_i[a];
                int b = a - 1;
                while (b >= 0 && child_t[b] < tv) {
                    child_t[b + 1] = child_t[b];
                    child_i[b + 1] = child_i[b];
                    b--;
                }
                child_t[b + 1] = tv;
                child_i[b + 1] = iv;
            }
            for (int a = 0; a < cnt && top < VCO_STACK_CAP; a++) stack[top++] = child_i[a];
        }
    }
    return nseg;
}

/* _kernels.py:367-465 over segments [seg0[i], seg1[i]] (one segment
 * [t_enter, t_exit] when the octree is off); adaptive stride when P
 * (non-NULL) asks for it. */
static int first_hit_seg(const vco_vol *v, const vco_params *P, const double sp[3], const double org[3],
                         const double dirv[3], double t_enter, double t_exit, const double *seg0,
                         const double *seg1, int nseg, double coarse, double fine, double t_low,
                         double t_high, int interp, int64_t *counter, double *t_hit, double *t_before,
                         int *bracket) {
    int64_t k = 0;
    for (int si = 0; si < nseg; si++) {
    double s0 = seg0[si], s1 = seg1[si];
    if (s1 > t_exit) s1 = t_exit;
    int64_t kk = (int64_t)floor((s0 - t_enter) / coarse);
    if (kk > k) k = kk;
    for (;;) {
        double t = t_enter + (double)k * coarse;
        if (t > s1 + 1e-12 || t > t_exit + 1e-12) break;
        double p[3];
        voxel_pos(org, dirv, sp, t, p);
        *counter += 1;
        double val = sample_any(v, p[0], p[1], p[2], interp);
        if (t_low <= val && val <= t_high) {
            int64_t j = 1;
            for (;;) {
                double tb = t - (double)j * fine;
                if (tb < t_enter - 1e-12) {
                    double th = t - (double)(j - 1) * fine;
                    *t_hit = th;
                    *t_before = th;
                    *bracket = 0;
                    return 1;
                }
                double b[3];
                voxel_pos(org, dirv, sp, tb, b);
                *counter += 1;
                double vb = sample_any(v, b[0], b[1], b[2], interp);
                if (vb < t_low || vb > t_high) {
                    *t_hit = t - (double)(j - 1) * fine;
                    *t_before = tb;
                    *bracket = 1;
                    return 1;
                }
                j += 1;
            }
        }
        if (P && P->use_adaptive) k += adaptive_stride(v, P, sp, org, dirv, p, k, t_enter, coarse);
        else k += 1;
    }
    }
    *t_hit = *t_before = 0.0;
    *bracket = 0;
    return 0;
}

static int first_hit_p(const vco_vol *v, const vco_params *P, const double sp[3], const double org[3],
                       const double dirv[3], double t_enter, double t_exit, double coarse,
                       double fine, double t_low, double t_high, int interp, int64_t *counter,
                       double *t_hit, double *t_before, int *bracket) {
    const double s0 = t_enter, s1 = t_exit;
    return first_hit_seg(v, P, sp, org, dirv, t_enter, t_exit, &s0, &s1, 1, coarse, fine, t_low, t_high,
                         interp, counter, t_hit, t_before, bracket);
}

static int first_hit(const vco_vol *v, const double sp[3], const double org[3],
                     const double dirv[3], double t_enter, double t_exit, double coarse,
                     double fine, double t_low, double t_high, int interp, int64_t *counter,
                     double *t_hit, double *t_before, int *bracket) {
    return first_hit_p(v, NULL, sp, org, dirv, t_enter, t_exit, coarse, fine, t_low, t_high, interp,
                       counter, t_hit, t_before, bracket);
}

/* _kernels.py:468-487 */
static double bisect_window(const vco_vol *v, const double sp[3], const double org[3],
                            const double dirv[3], double t_before, double t_after, double t_low,
                            double t_high, int iters, int interp, int64_t *counter) {
    double tb = t_before, ta = t_after;
    for (int it = 0; it < iters; it++) {
        double tm = 0.5 * (tb + ta);
        double p[3];
        voxel_pos(org, dirv, sp, tm, p);
        *counter += 1;
        double val = sample_any(v, p[0], p[1], p[2], interp);
        if (t_low <= val && val <= t_high) ta = tm;
        else tb = tm;
    }
    return ta;
}

/* _kernels.py:490-511 */
static void lut_eval(const vco_params *P, double hu, double out[4]) {
    int n = P->lut_n;
    const double *H = P->lut_hu, *C = P->lut_rgba;
    if (hu <= H[0]) {
        memcpy(out, C, 4 * sizeof(double));
        return;
    }
    if (hu >= H[n - 1]) {
        memcpy(out, C + 4 * (n - 1), 4 * sizeof(double));
        return;
    }
    int i = 0;
    while (i + 1 < n - 1 && H[i + 1] <= hu) i += 1;
    double t = (hu - H[i]) / (H[i + 1] - H[i]);
    for (int c = 0; c < 4; c++) out[c] = lerp(C[4 * i + c], C[4 * (i + 1) + c], t);
}

/* _kernels.py:514-525 */
static inline double clamp01(double v) {
    if (v < 0.0) return 0.0;
    if (v > 1.0) return 1.0;
    return v;
}
static inline uint8_t quant(double v) { return (uint8_t)(int)(clamp01(v) * 255.0 + 0.5); }

/* _kernels.py:528-579 */
static void shade_sample(const vco_vol *v, const vco_params *P, const double org[3],
                         const double dirv[3], double t, int64_t *counter, double out[4]) {
    const double *sp = P->spacing;
    double wx = org[0] + t * dirv[0];
    double wy = org[1] + t * dirv[1];
    double wz = org[2] + t * dirv[2];
    double px = wx / sp[0] - 0.5;
    double py = wy / sp[1] - 0.5;
    double pz = wz / sp[2] - 0.5;
    *counter += 1;
    double val = sample_any(v, px, py, pz, P->interp);
    double g[3], u[3];
    grad_raw(v, px, py, pz, P->op, g);
    *counter += GRAD_SAMPLES[P->op];
    normalize3(g, GRAD_EPS, u);
    double snx = -u[0], sny = -u[1], snz = -u[2];
    double lx = P->light_pos[0] - wx;
    double ly = P->light_pos[1] - wy;
    double lz = P->light_pos[2] - wz;
    double ln = sqrt(lx * lx + ly * ly + lz * lz);
    double illum = 0.0;
    if (ln > 0.0) illum = (lx * snx + ly * sny + lz * snz) / ln;
    illum = clamp01(illum);
    double hu = (val - P->mu_water) / P->mu_water * 1000.0;
    double m[4];
    lut_eval(P, hu, m);
    out[0] = clamp01(illum * P->light_col[0] * m[0]);
    out[1] = clamp01(illum * P->light_col[1] * m[1]);
    out[2] = clamp01(illum * P->light_col[2] * m[2]);
    out[3] = m[3];
}

/* _kernels.py:582-797 for rows [y0, y1). */
static void render_rows(const vco_vol *v, const vco_params *P, int y0, int y1, uint8_t *out,
                        int64_t *counter) {
    int32_t *stack = NULL;
    double *seg0 = NULL, *seg1 = NULL;
    if (P->use_octree) {  /* per-band scratch, like raycast.py:499 */
        stack = (int32_t *)malloc(VCO_STACK_CAP * sizeof(int32_t));
        seg0 = (double *)malloc(VCO_SEG_CAP * sizeof(double));
        seg1 = (double *)malloc(VCO_SEG_CAP * sizeof(double));
    }
    uint8_t bgr = quant(P->bg[0]), bgg = quant(P->bg[1]), bgb = quant(P->bg[2]),
            bga = quant(P->bg[3]);
    const double *org = P->eye;
    double dirv[3];
    const int W = P->width, H = P->height;
    for (int py = y0; py < y1; py++) {
        double v_ndc = 1.0 - 2.0 * ((double)py + 0.5) / (double)H;
        for (int px = 0; px < W; px++) {
            uint8_t *o = out + ((int64_t)py * W + px) * 4;
            double u_ndc = 2.0 * ((double)px + 0.5) / (double)W - 1.0;
            double dx = P->fwd[0] + u_ndc * P->half_w * P->right[0] + v_ndc * P->half_h * P->up[0];
            double dy = P->fwd[1] + u_ndc * P->half_w * P->right[1] + v_ndc * P->half_h * P->up[1];
            double dz = P->fwd[2] + u_ndc * P->half_w * P->right[2] + v_ndc * P->half_h * P->up[2];
            double dn = sqrt(dx * dx + dy * dy + dz * dz);
            dirv[0] = dx / dn;
            dirv[1] = dy / dn;
            dirv[2] = dz / dn;
            double iv[2];
            if (!vco_box_interval(org, dirv, P->clip_lo, P->clip_hi, iv)) {
                o[0] = bgr; o[1] = bgg; o[2] = bgb; o[3] = bga;
                continue;
            }
            double t_enter = iv[0], t_exit = iv[1];
            double t_in, t_before;
            int bracket;
            int found;
            if (P->use_octree) {
                int nseg = collect_segments(P, P->spacing, org, dirv, t_enter, t_exit, P->t_low, P->t_high,
                                            stack, seg0, seg1);
                found = first_hit_seg(v, P, P->spacing, org, dirv, t_enter, t_exit, seg0, seg1, nseg,
                                      P->coarse, P->fine, P->t_low, P->t_high, P->interp, counter, &t_in,
                                      &t_before, &bracket);
            } else {
                found = first_hit_p(v, P, P->spacing, org, dirv, t_enter, t_exit, P->coarse, P->fine,
                                    P->t_low, P->t_high, P->interp, counter, &t_in, &t_before,
                                    &bracket);
            }
            if (!found) {
                o[0] = bgr; o[1] = bgg; o[2] = bgb; o[3] = bga;
                continue;
            }
            double t_star = t_in;
            if (bracket && P->refine_iters > 0)
                t_star = bisect_window(v, P->spacing, org, dirv, t_before, t_in, P->t_low,
                                       P->t_high, P->refine_iters, P->interp, counter);
            double c[4];
            shade_sample(v, P, org, dirv, t_star, counter, c);
            if (P->mode == MODE_SURFACE) {
                o[0] = quant(c[0]); o[1] = quant(c[1]); o[2] = quant(c[2]); o[3] = 255;
                continue;
            }
            double acc_r = c[3] * c[0], acc_g = c[3] * c[1], acc_b = c[3] * c[2];
            double remain = 1.0 - c[3];
            if (c[3] < OPAQUE_ALPHA && remain >= MIN_REMAINING) {
                int64_t m = 1;
                for (;;) {
                    double t = t_star + (double)m * P->coarse;
                    if (t > t_exit + 1e-12) break;
                    double p[3];
                    voxel_pos(org, dirv, P->spacing, t, p);
                    *counter += 1;
                    double val = sample_any(v, p[0], p[1], p[2], P->interp);
                    if (P->t_low <= val && val <= P->t_high) {
                        double s[4];
                        shade_sample(v, P, org, dirv, t, counter, s);
                        acc_r += remain * s[3] * s[0];
                        acc_g += remain * s[3] * s[1];
                        acc_b += remain * s[3] * s[2];
                        remain *= 1.0 - s[3];
                        if (s[3] >= OPAQUE_ALPHA || remain < MIN_REMAINING) break;
                    }
                    m += 1;
                }
            }
            acc_r += remain * P->bg[0];
            acc_g += remain * P->bg[1];
            acc_b += remain * P->bg[2];
            o[0] = quant(acc_r); o[1] = quant(acc_g); o[2] = quant(acc_b); o[3] = 255;
        }
    }
    free(stack);
    free(seg0);
    free(seg1);
}

/* ---- exported entry points (ctypes) ---------------------------------- */

double vco_sample(const void *data, int dtype, int nx, int ny, int nz, double x, double y,
                  double z, int interp) {
    vco_vol v = {data, dtype, nx, ny, nz};
    return sample_any(&v, x, y, z, interp);
}

void vco_sample_many(const void *data, int dtype, int nx, int ny, int nz, const double *pts,
                     int64_t n, int interp, double *out) {
    vco_vol v = {data, dtype, nx, ny, nz};
    for (int64_t i = 0; i < n; i++) out[i] = sample_any(&v, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], interp);
}

void vco_grad_raw_many(const void *data, int dtype, int nx, int ny, int nz, const double *pts,
                       int64_t n, int op, double *out) {
    vco_vol v = {data, dtype, nx, ny, nz};
    for (int64_t i = 0; i < n; i++) grad_raw(&v, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], op, out + 3 * i);
}

void vco_normalize3(const double *g, double *u) { normalize3(g, GRAD_EPS, u); }

/* first_hit + bisect for one ray (march_surface / refine_hitpoint). */
int vco_first_hit(const void *data, int dtype, int nx, int ny, int nz, const double sp[3],
                  const double org[3], const double dirv[3], double t_enter, double t_exit,
                  double coarse, double fine, double t_low, double t_high, int interp,
                  double out[3], int64_t *counter) {
    vco_vol v = {data, dtype, nx, ny, nz};
    int bracket = 0;
    int found = first_hit(&v, sp, org, dirv, t_enter, t_exit, coarse, fine, t_low, t_high,
                          interp, counter, &out[0], &out[1], &bracket);
    out[2] = bracket;
    return found;
}

double vco_bisect(const void *data, int dtype, int nx, int ny, int nz, const double sp[3],
                  const double org[3], const double dirv[3], double t_before, double t_after,
                  double t_low, double t_high, int iters, int interp, int64_t *counter) {
    vco_vol v = {data, dtype, nx, ny, nz};
    return bisect_window(&v, sp, org, dirv, t_before, t_after, t_low, t_high, iters, interp,
                         counter);
}

void vco_lut_eval(const vco_params *P, double hu, double out[4]) { lut_eval(P, hu, out); }

/* Lattice gradient volume: grad_raw at every integer point, the reference
 * arithmetic driven over the grid.  out is (nz, ny, nx, 4) float32 with
 * (gx, gy, gz, value).  Rows split across threads. */
typedef struct {
    const vco_vol *v;
    int op;
    float *out;
    int z0, z1;
} grad_job;

static void *grad_worker(void *arg) {
    grad_job *J = (grad_job *)arg;
    const vco_vol *v = J->v;
    for (int k = J->z0; k < J->z1; k++)
        for (int j = 0; j < v->ny; j++)
            for (int i = 0; i < v->nx; i++) {
                double g[3];
                grad_raw(v, (double)i, (double)j, (double)k, J->op, g);
                float *o = J->out + (((int64_t)k * v->ny + j) * v->nx + i) * 4;
                o[0] = (float)g[0];
                o[1] = (float)g[1];
                o[2] = (float)g[2];
                o[3] = (float)fetch(v, i, j, k);
            }
    return NULL;
}

void vco_grad_volume(const void *data, int dtype, int nx, int ny, int nz, int op, float *out,
                     int threads) {
    vco_vol v = {data, dtype, nx, ny, nz};
    if (threads < 1) threads = 1;
    if (threads > nz) threads = nz;
    pthread_t th[256];
    grad_job jobs[256];
    if (threads > 256) threads = 256;
    for (int t = 0; t < threads; t++) {
        jobs[t].v = &v;
        jobs[t].op = op;
        jobs[t].out = out;
        jobs[t].z0 = (int)((int64_t)nz * t / threads);
        jobs[t].z1 = (int)((int64_t)nz * (t + 1) / threads);
        pthread_create(&th[t], NULL, grad_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
}

/* Whole frame (or rows [y0, y1)), work split in bands of `band` rows
 * (raycast.py:476-505 hands 16-row bands to a thread pool); here each
 * worker pulls the next band from a shared counter, so every host thread
 * stays busy down to single-row bands and small row samples.
 * Output rows outside [y0, y1) are untouched. */
typedef struct {
    const vco_vol *v;
    const vco_params *P;
    uint8_t *out;
    int y0, y1, band;
    int *next;
    int64_t counter;
} render_job;

static void *render_worker(void *arg) {
    render_job *J = (render_job *)arg;
    for (;;) {
        int b = __atomic_fetch_add(J->next, J->band, __ATOMIC_RELAXED);
        if (b >= J->y1) break;
        int e = b + J->band;
        if (e > J->y1) e = J->y1;
        render_rows(J->v, J->P, b, e, J->out, &J->counter);
    }
    return NULL;
}

int64_t vco_render(const void *data, int dtype, int nx, int ny, int nz, const vco_params *P,
                   int y0, int y1, uint8_t *out, int threads) {
    vco_vol v = {data, dtype, nx, ny, nz};
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    /* bands of up to 4 rows, at least two per thread when the range allows */
    int band = (y1 - y0) / (2 * threads);
    if (band > 4) band = 4;
    if (band < 1) band = 1;
    if (threads > y1 - y0) threads = y1 - y0 > 0 ? y1 - y0 : 1;
    int next = y0;
    pthread_t th[256];
    render_job jobs[256];
    for (int t = 0; t < threads; t++) {
        jobs[t] = (render_job){&v, P, out, y0, y1, band, &next, 0};
        pthread_create(&th[t], NULL, render_worker, &jobs[t]);
    }
    int64_t total = 0;
    for (int t = 0; t < threads; t++) {
        pthread_join(th[t], NULL);
        total += jobs[t].counter;
    }
    return total;
}

int vco_params_size(void) { return (int)sizeof(vco_params); }
