/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the tilefusion hot path.
 * See tf_oracle.h for the contract and the arithmetic rules.  Each function
 * cites the reference lines it restates (paths relative to
 * /root/reference/pkg/src/tilefusion/).  Compiled with -ffp-contract=off.
 */
#include "tf_oracle.h"

#include <math.h>
#include <stddef.h>
#include <pthread.h>
#include <string.h>

#define IDX3(n, z, y, x) ((((int64_t)(z)) * (n) + (y)) * (n) + (x))

/* Minimal pthread parallel-for over independent rows: worker w takes rows
 * w, w + nthreads, ...  Each row's work is independent of the others in every
 * caller, so the results do not depend on nthreads. */
typedef int64_t (*row_fn)(void *ctx, int64_t row);
typedef struct {
    row_fn fn;
    void *ctx;
    int64_t rows, first, step, sum;
} par_job;

static void *par_worker(void *arg) {
    par_job *j = (par_job *)arg;
    int64_t s = 0;
    for (int64_t r = j->first; r < j->rows; r += j->step) s += j->fn(j->ctx, r);
    j->sum = s;
    return NULL;
}

static int64_t par_rows(row_fn fn, void *ctx, int64_t rows, int nthreads) {
    if (nthreads > 256) nthreads = 256;
    if (nthreads <= 1 || rows < 2) {
        int64_t s = 0;
        for (int64_t r = 0; r < rows; ++r) s += fn(ctx, r);
        return s;
    }
    pthread_t tid[256];
    par_job jobs[256];
    int started = 0;
    for (int w = 0; w < nthreads; ++w) {
        jobs[w] = (par_job){fn, ctx, rows, w, nthreads, 0};
        if (pthread_create(&tid[w], NULL, par_worker, &jobs[w]) != 0) break;
        started++;
    }
    int64_t total = 0;
    for (int w = 0; w < started; ++w) {
        pthread_join(tid[w], NULL);
        total += jobs[w].sum;
    }
    /* rows of workers that failed to start run here */
    for (int w = started; w < nthreads; ++w) {
        par_worker(&jobs[w]);
        total += jobs[w].sum;
    }
    return total;
}

/* ------------------------------------------------------------------------ */
/* integration: _kernels.py:71-133                                           */
/* ------------------------------------------------------------------------ */

/* One voxel of the projective update; returns 1 when the voxel was written. */
static int integrate_voxel(float *tsdf, float *weight, int64_t lin, double gx,
                           double gy, double gz, const double *depth,
                           int64_t height, int64_t width, const double *r,
                           const double *t, const double *c, double fx,
                           double fy, double cx, double cy, double tau,
                           double max_w, double sw) {
    /* :104-106, evaluated left to right, no contraction */
    double pcx = r[0] * gx + r[1] * gy + r[2] * gz + t[0];
    double pcy = r[3] * gx + r[4] * gy + r[5] * gz + t[1];
    double pcz = r[6] * gx + r[7] * gy + r[8] * gz + t[2];
    if (pcz <= 0.0) return 0;                                   /* :107 */
    double u = fx * pcx / pcz + cx;                             /* :109 */
    double v = fy * pcy / pcz + cy;                             /* :110 */
    double uf = floor(u + 0.5), vf = floor(v + 0.5);            /* :111-112 */
    /* :113 — compared as doubles so huge values never hit int conversion */
    if (!(uf >= 0.0 && uf < (double)width && vf >= 0.0 && vf < (double)height))
        return 0;
    int64_t ui = (int64_t)uf, vi = (int64_t)vf;
    double d = depth[vi * width + ui];                          /* :115 */
    if (d <= 0.0) return 0;                                     /* :116 */
    double rx = ((double)ui - cx) / fx;                         /* :118 */
    double ry = ((double)vi - cy) / fy;                         /* :119 */
    double ray_scale = sqrt(rx * rx + ry * ry + 1.0);           /* :120 */
    double ddx = gx - c[0], ddy = gy - c[1], ddz = gz - c[2];   /* :121-123 */
    double dist = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);      /* :124 */
    double sdf = d - dist / ray_scale;                          /* :125 */
    if (sdf < -tau) return 0;                                   /* :126 */
    double clamped = sdf < tau ? sdf : tau;                     /* :128 */
    /* numba types float(f32) as float32 (:129-130), so w_old * v_old is a
     * float32 product; the sum and the division are float64 (:131-132). */
    float w_old = weight[lin];
    float v_old = tsdf[lin];
    float wv = w_old * v_old;
    double w_sum = (double)w_old + sw;                          /* :131 */
    tsdf[lin] = (float)(((double)wv + sw * clamped) / w_sum);   /* :132 */
    weight[lin] = (float)(max_w < w_sum ? max_w : w_sum);         /* :133 */
    return 1;
}

typedef struct {
    float *tsdf, *weight;
    int64_t n;
    const int64_t *ht;
    double vs;
    const double *depth;
    int64_t height, width;
    const double *r, *t, *c;
    double fx, fy, cx, cy, tau, max_w, sw;
} integ_args;

/* one z slice, loops in the reference order iz -> iy -> ix (:98-103) */
static int64_t integrate_slice(void *ctx, int64_t iz) {
    const integ_args *a = (const integ_args *)ctx;
    int64_t n = a->n, updated = 0;
    double gz = (double)(iz + a->ht[2]) * a->vs;                    /* :99 */
    for (int64_t iy = 0; iy < n; ++iy) {
        double gy = (double)(iy + a->ht[1]) * a->vs;                /* :101 */
        for (int64_t ix = 0; ix < n; ++ix) {
            double gx = (double)(ix + a->ht[0]) * a->vs;            /* :103 */
            updated += integrate_voxel(a->tsdf, a->weight, IDX3(n, iz, iy, ix), gx,
                                       gy, gz, a->depth, a->height, a->width, a->r,
                                       a->t, a->c, a->fx, a->fy, a->cx, a->cy,
                                       a->tau, a->max_w, a->sw);
        }
    }
    return updated;
}

int64_t tfo_integrate(float *tsdf, float *weight, int64_t n, const int64_t ht[3],
                      double vs, const double *depth, int64_t height,
                      int64_t width, const double r_cw[9], const double t_cw[3],
                      const double cam[3], double fx, double fy, double cx,
                      double cy, double tau, double max_w, double sw,
                      int nthreads) {
    integ_args a = {tsdf, weight, n, ht, vs, depth, height, width, r_cw, t_cw,
                    cam, fx, fy, cx, cy, tau, max_w, sw};
    return par_rows(integrate_slice, &a, n, nthreads);
}

/* ------------------------------------------------------------------------ */
/* trilinear sample: _kernels.py:28-68                                       */
/* ------------------------------------------------------------------------ */

int tfo_sample(const float *tsdf, const float *weight, int64_t n, double qx,
               double qy, double qz, double *value) {
    double fxl = floor(qx), fyl = floor(qy), fzl = floor(qz);
    /* :38 bounds, compared as doubles */
    if (!(fxl >= 0.0 && fyl >= 0.0 && fzl >= 0.0 && fxl <= (double)(n - 2) &&
          fyl <= (double)(n - 2) && fzl <= (double)(n - 2)))
        return 0;
    int64_t ix = (int64_t)fxl, iy = (int64_t)fyl, iz = (int64_t)fzl;
    int64_t b = IDX3(n, iz, iy, ix);
    int64_t sy = n, sz = n * n;
    /* corner order c[z][y][x] */
    const int64_t off[8] = {0, 1, sy, sy + 1, sz, sz + 1, sz + sy, sz + sy + 1};
    for (int k = 0; k < 8; ++k)                                  /* :40-50 */
        if (weight[b + off[k]] <= 0.0f) return 0;
    double fx = qx - (double)ix, fy = qy - (double)iy, fz = qz - (double)iz;
    double c000 = tsdf[b + off[0]], c100 = tsdf[b + off[1]];
    double c010 = tsdf[b + off[2]], c110 = tsdf[b + off[3]];
    double c001 = tsdf[b + off[4]], c101 = tsdf[b + off[5]];
    double c011 = tsdf[b + off[6]], c111 = tsdf[b + off[7]];
    double c00 = c000 * (1.0 - fx) + c100 * fx;                  /* :62-65 */
    double c10 = c010 * (1.0 - fx) + c110 * fx;
    double c01 = c001 * (1.0 - fx) + c101 * fx;
    double c11 = c011 * (1.0 - fx) + c111 * fx;
    double c0 = c00 * (1.0 - fy) + c10 * fy;                     /* :66-67 */
    double c1 = c01 * (1.0 - fy) + c11 * fy;
    *value = c0 * (1.0 - fz) + c1 * fz;                          /* :68 */
    return 1;
}

/* ------------------------------------------------------------------------ */
/* raycast: _kernels.py:136-451                                              */
/* ------------------------------------------------------------------------ */

typedef struct {
    const float *tsdf, *weight;
    int64_t n;
    double htx, hty, htz; /* origin voxel as doubles (exact for |ht| < 2^53) */
    double vs;
    double ox, oy, oz, dx, dy, dz;
    int64_t samples;
} ray_ctx;

/* local lattice coordinate of fine point k: _kernels.py:164-167, :357-359 */
static int ray_sample_at(ray_ctx *r, int64_t k, double *value) {
    double tk = (double)k * r->vs;
    double kx = (r->ox + tk * r->dx) / r->vs - r->htx;
    double ky = (r->oy + tk * r->dy) / r->vs - r->hty;
    double kz = (r->oz + tk * r->dz) / r->vs - r->htz;
    r->samples++;
    return tfo_sample(r->tsdf, r->weight, r->n, kx, ky, kz, value);
}

typedef struct {
    double t, hx, hy, hz, nx, ny, nz;
} ray_hit;

/* _scan_crossing: _kernels.py:136-243 */
static int scan_crossing(ray_ctx *r, int64_t scan_from, int64_t scan_end,
                         int sp_valid, double sp_v, ray_hit *hit) {
    const int64_t n = r->n;
    const double delta = r->vs;
    for (int64_t k = scan_from; k <= scan_end; ++k) {
        double s = 0.0;
        int sv = ray_sample_at(r, k, &s);
        if (sp_valid && sp_v > 0.0 && sv && s <= 0.0) {           /* :169 */
            double ta = (double)(k - 1) * delta;
            double tstar = ta + delta * (sp_v / (sp_v - s));        /* :171 */
            if (tstar >= 0.0) {
                double hx = r->ox + tstar * r->dx;
                double hy = r->oy + tstar * r->dy;
                double hz = r->oz + tstar * r->dz;
                double qx = hx / r->vs - r->htx;
                double qy = hy / r->vs - r->hty;
                double qz = hz / r->vs - r->htz;
                double fcx = floor(qx), fcy = floor(qy), fcz = floor(qz);
                int inside = fcx >= 0.0 && fcy >= 0.0 && fcz >= 0.0 &&
                             fcx <= (double)(n - 2) && fcy <= (double)(n - 2) &&
                             fcz <= (double)(n - 2);
                if (inside) {
                    int64_t cix = (int64_t)fcx, ciy = (int64_t)fcy, ciz = (int64_t)fcz;
                    int64_t b = IDX3(n, ciz, ciy, cix), sy = n, sz = n * n;
                    const int64_t off[8] = {0, 1, sy, sy + 1, sz, sz + 1, sz + sy,
                                            sz + sy + 1};
                    int observed = 1;
                    for (int q = 0; q < 8; ++q)                     /* :189-196 */
                        if (!(r->weight[b + off[q]] > 0.0f)) observed = 0;
                    if (observed) {
                        double gfx = qx - (double)cix;
                        double gfy = qy - (double)ciy;
                        double gfz = qz - (double)ciz;
                        const float *T = r->tsdf;
                        /* corners stay float32 (numba float(f32) -> f32), so
                         * the edge differences are float32 ops (:201-226) */
                        float c000 = T[b + off[0]], c100 = T[b + off[1]];
                        float c010 = T[b + off[2]], c110 = T[b + off[3]];
                        float c001 = T[b + off[4]], c101 = T[b + off[5]];
                        float c011 = T[b + off[6]], c111 = T[b + off[7]];
                        /* analytic trilinear gradient, :209-226 */
                        double gx = (double)(c100 - c000) * (1.0 - gfy) * (1.0 - gfz) +
                                    (double)(c110 - c010) * gfy * (1.0 - gfz) +
                                    (double)(c101 - c001) * (1.0 - gfy) * gfz +
                                    (double)(c111 - c011) * gfy * gfz;
                        double gy = (double)(c010 - c000) * (1.0 - gfx) * (1.0 - gfz) +
                                    (double)(c110 - c100) * gfx * (1.0 - gfz) +
                                    (double)(c011 - c001) * (1.0 - gfx) * gfz +
                                    (double)(c111 - c101) * gfx * gfz;
                        double gz = (double)(c001 - c000) * (1.0 - gfx) * (1.0 - gfy) +
                                    (double)(c011 - c010) * (1.0 - gfx) * gfy +
                                    (double)(c101 - c100) * gfx * (1.0 - gfy) +
                                    (double)(c111 - c110) * gfx * gfy;
                        double gnorm = sqrt(gx * gx + gy * gy + gz * gz);
                        if (gnorm > 0.0) {
                            if (gx * r->dx + gy * r->dy + gz * r->dz > 0.0) {
                                gx = -gx;
                                gy = -gy;
                                gz = -gz;
                            }
                            hit->t = tstar;
                            hit->hx = hx;
                            hit->hy = hy;
                            hit->hz = hz;
                            hit->nx = gx / gnorm;
                            hit->ny = gy / gnorm;
                            hit->nz = gz / gnorm;
                            return 1;
                        }
                    }
                }
            }
        }
        sp_valid = sv;                                              /* :241-242 */
        sp_v = s;
    }
    return 0;
}

/* _hit_wins: _kernels.py:246-263 */
static int hit_wins(const ray_hit *h, double cur, double cnx, double cny,
                    double cnz) {
    if (h->t < cur) return 1;
    if (h->t > cur) return 0;
    if (h->nx != cnx) return h->nx > cnx;
    if (h->ny != cny) return h->ny > cny;
    return h->nz > cnz;
}

static void merge_hit(const ray_hit *h, double *dist, double *vert,
                      double *norm) {
    if (hit_wins(h, dist[0], norm[0], norm[1], norm[2])) {
        dist[0] = h->t;
        vert[0] = h->hx;
        vert[1] = h->hy;
        vert[2] = h->hz;
        norm[0] = h->nx;
        norm[1] = h->ny;
        norm[2] = h->nz;
    }
}

/* the scan start value: reuse the last march sample when it is the point
 * just before scan_from, else sample it (:373-382, :423-432) */
static void scan_seed(ray_ctx *r, int64_t k0, int prev_has, int64_t prev_j,
                      double prev_v, int *sp_valid, double *sp_v) {
    if (prev_has && k0 == prev_j) {
        *sp_valid = 1;
        *sp_v = prev_v;
    } else {
        *sp_v = 0.0;
        *sp_valid = ray_sample_at(r, k0, sp_v);
    }
}

typedef struct {
    const float *tsdf, *weight;
    int64_t n;
    const int64_t *ht;
    double vs, tau;
    int64_t coarse;
    const double *R, *cam;
    double fx, fy, cx, cy;
    int64_t height, width;
    double *out_dist, *out_vert, *out_norm;
    double bmin[3], bmax[3];
} rc_args;

/* one image row of the per-pixel march (:305-451) */
static int64_t raycast_row(void *ctx, int64_t py) {
    const rc_args *A = (const rc_args *)ctx;
    const float *tsdf = A->tsdf, *weight = A->weight;
    const int64_t n = A->n, coarse = A->coarse, width = A->width;
    const int64_t *ht = A->ht;
    const double vs = A->vs, delta = A->vs;
    const double near_thresh = 0.99 * A->tau;                       /* :25, :298 */
    const double *R = A->R, *cam = A->cam;
    const double fx = A->fx, fy = A->fy, cx = A->cx, cy = A->cy;
    const double *bmin = A->bmin, *bmax = A->bmax;
    double *out_dist = A->out_dist, *out_vert = A->out_vert, *out_norm = A->out_norm;
    int64_t total = 0;
    for (int64_t px = 0; px < width; ++px) {
            ray_ctx r;
            r.tsdf = tsdf;
            r.weight = weight;
            r.n = n;
            r.htx = (double)ht[0];
            r.hty = (double)ht[1];
            r.htz = (double)ht[2];
            r.vs = vs;
            r.samples = 0;
            double rx = ((double)px - cx) / fx;                     /* :307-308 */
            double ry = ((double)py - cy) / fy;
            double dx = R[0] * rx + R[1] * ry + R[2];               /* :309-311 */
            double dy = R[3] * rx + R[4] * ry + R[5];
            double dz = R[6] * rx + R[7] * ry + R[8];
            double dn = sqrt(dx * dx + dy * dy + dz * dz);
            r.dx = dx / dn;
            r.dy = dy / dn;
            r.dz = dz / dn;
            r.ox = cam[0];
            r.oy = cam[1];
            r.oz = cam[2];
            /* slab test, :320-344 */
            double t_lo = 0.0, t_hi = 1.0e30;
            int miss = 0;
            const double o_a[3] = {r.ox, r.oy, r.oz};
            const double d_a[3] = {r.dx, r.dy, r.dz};
            for (int a = 0; a < 3; ++a) {
                if (fabs(d_a[a]) < 1.0e-15) {
                    if (o_a[a] < bmin[a] || o_a[a] > bmax[a]) {
                        miss = 1;
                        break;
                    }
                } else {
                    double t1 = (bmin[a] - o_a[a]) / d_a[a];
                    double t2 = (bmax[a] - o_a[a]) / d_a[a];
                    if (t1 > t2) {
                        double tmp = t1;
                        t1 = t2;
                        t2 = tmp;
                    }
                    if (t1 > t_lo) t_lo = t1;
                    if (t2 < t_hi) t_hi = t2;
                }
            }
            if (miss || t_lo > t_hi) goto next_pixel;
            int64_t j = (int64_t)ceil(t_lo / delta);                 /* :345-348 */
            if (j < 0) j = 0;
            int64_t j_end = (int64_t)floor(t_hi / delta);
            int prev_has = 0;
            double prev_v = 0.0;
            int64_t prev_j = -1, last_j = j - 1, swept_j = j - 1;
            int finished = 0;
            double *pd = out_dist + py * width + px;
            double *pv = out_vert + (py * width + px) * 3;
            double *pn = out_norm + (py * width + px) * 3;
            while (j <= j_end) {                                     /* :355 */
                double value = 0.0;
                int valid = ray_sample_at(&r, j, &value);
                int do_scan = 0;
                if (!valid || value <= 0.0) {                         /* :362-369 */
                    if (prev_has && prev_v > 0.0)
                        do_scan = 1;
                    else if (swept_j < j - 1 && (valid || coarse > 2))
                        do_scan = 1;
                }
                if (do_scan) {
                    int64_t scan_from = (prev_j > swept_j ? prev_j : swept_j) + 1;
                    int sp_valid;
                    double sp_v;
                    scan_seed(&r, scan_from - 1, prev_has, prev_j, prev_v, &sp_valid,
                              &sp_v);
                    ray_hit h;
                    int found = scan_crossing(&r, scan_from, j, sp_valid, sp_v, &h);
                    swept_j = j;
                    if (found) {
                        merge_hit(&h, pd, pv, pn);
                        finished = 1;
                        break;
                    }
                }
                last_j = j;                                           /* :406 */
                if (valid) {
                    prev_has = 1;
                    prev_v = value;
                    prev_j = j;
                    if (fabs(value) < near_thresh)
                        j += 1;
                    else
                        j = (j / coarse + 1) * coarse;
                } else {
                    j = (j / coarse + 1) * coarse;
                }
            }
            if (!finished) {                                          /* :417-451 */
                int64_t scan_from = (last_j > swept_j ? last_j : swept_j) + 1;
                if (scan_from <= j_end) {
                    int sp_valid;
                    double sp_v;
                    scan_seed(&r, scan_from - 1, prev_has, prev_j, prev_v, &sp_valid,
                              &sp_v);
                    ray_hit h;
                    if (scan_crossing(&r, scan_from, j_end, sp_valid, sp_v, &h))
                        merge_hit(&h, pd, pv, pn);
                }
            }
            total += r.samples;
        next_pixel:;
    }
    return total;
}

int64_t tfo_raycast(const float *tsdf, const float *weight, int64_t n,
                    const int64_t ht[3], double vs, double tau, int64_t coarse,
                    const double R[9], const double cam[3], double fx, double fy,
                    double cx, double cy, int64_t height, int64_t width,
                    double *out_dist, double *out_vert, double *out_norm,
                    int nthreads) {
    rc_args a = {tsdf, weight, n, ht, vs, tau, coarse, R, cam, fx, fy, cx, cy,
                 height, width, out_dist, out_vert, out_norm, {0}, {0}};
    for (int k = 0; k < 3; ++k) {                                   /* :299-304 */
        a.bmin[k] = (double)ht[k] * vs;
        a.bmax[k] = (double)(ht[k] + n - 1) * vs;
    }
    return par_rows(raycast_row, &a, height, nthreads);
}

/* ------------------------------------------------------------------------ */
/* extraction: _kernels.py:454-578                                           */
/* ------------------------------------------------------------------------ */

/* sign change against an observed +x/+y/+z neighbour (:462-475) */
int64_t tfo_extract_bound(const float *tsdf, const float *weight, int64_t n) {
    int64_t count = 0;
    for (int64_t iz = 0; iz < n; ++iz)
        for (int64_t iy = 0; iy < n; ++iy)
            for (int64_t ix = 0; ix < n; ++ix) {
                int64_t i = IDX3(n, iz, iy, ix);
                if (weight[i] <= 0.0f) continue;
                int pos0 = tsdf[i] > 0.0f;
                int found = 0;
                if (ix + 1 < n && weight[i + 1] > 0.0f && ((tsdf[i + 1] > 0.0f) != pos0))
                    found = 1;
                if (!found && iy + 1 < n && weight[i + n] > 0.0f &&
                    ((tsdf[i + n] > 0.0f) != pos0))
                    found = 1;
                if (!found && iz + 1 < n && weight[i + n * n] > 0.0f &&
                    ((tsdf[i + n * n] > 0.0f) != pos0))
                    found = 1;
                count += found;
            }
    return count;
}

int64_t tfo_extract(const float *tsdf, const float *weight, int64_t n,
                    const int64_t ht[3], double vs, double *out_verts,
                    double *out_norms) {
    int64_t count = 0;
    const int64_t stride[3] = {1, n, n * n};
    for (int64_t iz = 0; iz < n; ++iz)
        for (int64_t iy = 0; iy < n; ++iy)
            for (int64_t ix = 0; ix < n; ++ix) {
                int64_t i = IDX3(n, iz, iy, ix);
                if (weight[i] <= 0.0f) continue;
                const int64_t pos[3] = {ix, iy, iz};
                float v0 = tsdf[i];                                  /* float32 in numba */
                int pos0 = v0 > 0.0f;
                double best_alpha = 2.0;
                int best_axis = -1;
                for (int a = 0; a < 3; ++a) {                        /* :502-522 */
                    if (pos[a] + 1 < n && weight[i + stride[a]] > 0.0f) {
                        float v1 = tsdf[i + stride[a]];
                        if ((v1 > 0.0f) != pos0) {
                            /* float32 subtraction and division, widened */
                            double alpha = (double)(v0 / (v0 - v1));
                            if (alpha < best_alpha) {
                                best_alpha = alpha;
                                best_axis = a;
                            }
                        }
                    }
                }
                if (best_axis < 0) continue;
                double g[3];
                for (int a = 0; a < 3; ++a) {                        /* :526-558 */
                    int im = pos[a] - 1 >= 0 && weight[i - stride[a]] > 0.0f;
                    int ip = pos[a] + 1 < n && weight[i + stride[a]] > 0.0f;
                    double vm = im ? (double)tsdf[i - stride[a]] : 0.0;
                    double vp = ip ? (double)tsdf[i + stride[a]] : 0.0;
                    if (im && ip)
                        g[a] = (vp - vm) * 0.5;
                    else if (ip)
                        g[a] = vp - (double)v0;
                    else if (im)
                        g[a] = (double)v0 - vm;
                    else
                        g[a] = 0.0;
                }
                double gnorm = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
                if (gnorm == 0.0) continue;
                double vtx[3];
                for (int a = 0; a < 3; ++a) vtx[a] = (double)(pos[a] + ht[a]) * vs;
                vtx[best_axis] += best_alpha * vs;                   /* :565-570 */
                for (int a = 0; a < 3; ++a) {
                    out_verts[count * 3 + a] = vtx[a];
                    out_norms[count * 3 + a] = g[a] / gnorm;
                }
                count++;
            }
    return count;
}

/* ------------------------------------------------------------------------ */
/* vertex / normal maps: geometry.py:59-68, :261-302                         */
/* ------------------------------------------------------------------------ */

void tfo_vertex_normal_map(const double *depth, int64_t h, int64_t w, double fx,
                           double fy, double cx, double cy, double *verts,
                           double *norms, uint8_t *valid) {
    for (int64_t y = 0; y < h; ++y)
        for (int64_t x = 0; x < w; ++x) {
            double d = depth[y * w + x];
            double *v = verts + (y * w + x) * 3;
            if (d > 0.0) {                                           /* :269-271 */
                v[0] = (((double)x - cx) / fx) * d;
                v[1] = (((double)y - cy) / fy) * d;
                v[2] = 1.0 * d;
            } else {
                v[0] = v[1] = v[2] = 0.0;
            }
        }
    for (int64_t y = 0; y < h; ++y)
        for (int64_t x = 0; x < w; ++x) {
            int64_t p = y * w + x;
            double *nr = norms + p * 3;
            nr[0] = nr[1] = nr[2] = 0.0;
            valid[p] = 0;
            if (y + 1 >= h || x + 1 >= w) continue;                  /* last row / col */
            if (!(depth[p] > 0.0 && depth[p + 1] > 0.0 && depth[p + w] > 0.0))
                continue;                                            /* :289-292 */
            const double *v0 = verts + p * 3;
            const double *vx = verts + (p + 1) * 3;
            const double *vy = verts + (p + w) * 3;
            double a[3] = {vx[0] - v0[0], vx[1] - v0[1], vx[2] - v0[2]};
            double b[3] = {vy[0] - v0[0], vy[1] - v0[1], vy[2] - v0[2]};
            double c0 = a[1] * b[2] - a[2] * b[1];                   /* np.cross */
            double c1 = a[2] * b[0] - a[0] * b[2];
            double c2 = a[0] * b[1] - a[1] * b[0];
            double nn = sqrt(c0 * c0 + c1 * c1 + c2 * c2);           /* np.linalg.norm */
            if (!(nn > 0.0)) continue;                               /* :293 */
            double u0 = c0 / nn, u1 = c1 / nn, u2 = c2 / nn;
            double toward = (u0 * v0[0] + u2 * v0[2]) + u1 * v0[1]; /* einsum :298 */
            if (toward > 0.0) {
                u0 = -u0;
                u1 = -u1;
                u2 = -u2;
            }
            nr[0] = u0;
            nr[1] = u1;
            nr[2] = u2;
            valid[p] = 1;
        }
}

/* ------------------------------------------------------------------------ */
/* ICP per-pixel terms: tracking.py:62-120                                   */
/* ------------------------------------------------------------------------ */

/* (N,3) @ R.T as OpenBLAS computes it: FMA chain over k */
static void rot_apply(const double *R, const double *s, double *o) {
    for (int i = 0; i < 3; ++i) {
        double acc = s[0] * R[i * 3 + 0];
        acc = fma(s[1], R[i * 3 + 1], acc);
        acc = fma(s[2], R[i * 3 + 2], acc);
        o[i] = acc;
    }
}

/* 3-term einsum "...i,...i->..." as numpy evaluates it: (p0 + p2) + p1 */
static double dot_np(const double *a, const double *b) {
    return (a[0] * b[0] + a[2] * b[2]) + a[1] * b[1];
}

void tfo_icp_reduce(const double *src_v, const double *src_n,
                    const uint8_t *src_valid, int64_t sh, int64_t sw,
                    const double *mdl_v, const double *mdl_n,
                    const uint8_t *mdl_valid, int64_t mh, int64_t mw,
                    const double r_est[9], const double t_est[3],
                    const double r_ref[9], const double t_ref[3], double fx,
                    double fy, double cx, double cy, int64_t img_w,
                    int64_t img_h, double max_d2, double cos_min, double *out) {
    memset(out, 0, 29 * sizeof(double));
    for (int64_t p = 0; p < sh * sw; ++p) {
        if (!src_valid[p]) continue;
        double pw[3], nw[3], pr[3];
        rot_apply(r_est, src_v + p * 3, pw);                          /* :76 */
        for (int i = 0; i < 3; ++i) pw[i] = pw[i] + t_est[i];
        rot_apply(r_est, src_n + p * 3, nw);                          /* :77 */
        rot_apply(r_ref, pw, pr);                                     /* :80 */
        for (int i = 0; i < 3; ++i) pr[i] = pr[i] + t_ref[i];
        double z = pr[2];
        if (!(z > 1.0e-9)) continue;                                  /* :82 */
        double u = fx * pr[0] / z + cx;                               /* :84 */
        double v = fy * pr[1] / z + cy;                               /* :85 */
        double uf = floor(u + 0.5), vf = floor(v + 0.5);
        if (!(uf >= 0.0 && uf < (double)img_w && vf >= 0.0 && vf < (double)img_h))
            continue;                                                 /* :88 */
        int64_t ui = (int64_t)uf, vi = (int64_t)vf;
        if (vi >= mh || ui >= mw) continue;
        int64_t m = vi * mw + ui;
        if (!mdl_valid[m]) continue;                                  /* :91 */
        const double *q = mdl_v + m * 3;
        const double *nm = mdl_n + m * 3;
        double diff[3] = {pw[0] - q[0], pw[1] - q[1], pw[2] - q[2]};
        if (!(dot_np(diff, diff) <= max_d2)) continue;                /* :96 */
        if (!(dot_np(nm, nw) >= cos_min)) continue;                   /* :97-98 */
        double e[3] = {q[0] - pw[0], q[1] - pw[1], q[2] - pw[2]};
        double r = dot_np(nm, e);                                     /* :105 */
        double a[6];
        a[0] = pw[1] * nm[2] - pw[2] * nm[1];                         /* :106 */
        a[1] = pw[2] * nm[0] - pw[0] * nm[2];
        a[2] = pw[0] * nm[1] - pw[1] * nm[0];
        a[3] = nm[0];
        a[4] = nm[1];
        a[5] = nm[2];
        int k = 0;
        for (int i = 0; i < 6; ++i)
            for (int jj = i; jj < 6; ++jj) out[k++] += a[i] * a[jj];  /* :107 */
        for (int i = 0; i < 6; ++i) out[21 + i] += a[i] * r;          /* :108 */
        out[27] += r * r;
        out[28] += 1.0;
    }
}

/* ------------------------------------------------------------------------ */
/* endpoint cells: volumes.py:318-327                                        */
/* ------------------------------------------------------------------------ */

int64_t tfo_endpoint_cells(const double *depth, int64_t h, int64_t w, double fx,
                           double fy, double cx, double cy, const double R[9],
                           const double T[3], double block_side,
                           int64_t *cells) {
    int64_t count = 0;
    for (int64_t y = 0; y < h; ++y)
        for (int64_t x = 0; x < w; ++x) {
            double d = depth[y * w + x];
            if (!(d > 0.0)) continue;
            double ray[3] = {((double)x - cx) / fx, ((double)y - cy) / fy, 1.0};
            double rr[3];
            rot_apply(R, ray, rr);                                    /* :318 */
            double nn = sqrt(rr[0] * rr[0] + rr[1] * rr[1] + rr[2] * rr[2]);
            for (int a = 0; a < 3; ++a) {
                double unit = rr[a] / nn;                             /* :319 */
                double pt = T[a] + d * unit;                          /* :324 */
                cells[count * 3 + a] = (int64_t)floor(pt / block_side); /* :326 */
            }
            count++;
        }
    return count;
}
