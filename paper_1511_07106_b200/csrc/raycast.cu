// Multi-volume truncated-SDF raycast with nearest-surface merge (sm_100a).
//
// Replaces _kernels.raycast_kernel + _sample + _scan_crossing + _hit_wins
// (reference _kernels.py:28-68, :136-451).  One thread per pixel marches the
// camera-anchored lattice through every volume of the launch, keeps the best
// hit under the _hit_wins total order in registers, and writes the pixel once.
//
// Because _hit_wins is a strict total order, the merged result does not
// depend on the order volumes are visited (the reference's own invariant,
// test_acceptance.py:349-361).  The kernel therefore visits a ray's volumes
// nearest-entry first and skips a volume outright when no hit inside it can
// beat the current best: every hit of a volume whose first lattice index is
// j0 has tstar >= (j0 - 1) * delta (_kernels.py:170-171), so a volume with
// (j0 - 1) * delta > best is provably irrelevant.  Everything else — the
// sample positions, the coarse/fine stepping, both re-walk rules, the
// crossing interpolation and the analytic normal — is the reference's
// arithmetic in the reference's order.
#include <climits>
#include <math.h>
#include <stdlib.h>

#include "tf_common.cuh"

#include <mutex>

namespace tf {

struct RayGeom {
    Mat3 r_wc;
    Vec3 cam;
    double fx, fy, cx, cy;
    int64_t width, height;
    double near_thresh;  // NEAR_SURFACE_FRACTION * tau (_kernels.py:25, :298)
    int64_t coarse;
    int exact_only;      // TF_DEBUG_EXACT_ONLY: plain reference march for every ray
    int lane0_only;      // TF_DEBUG_LANE0_ONLY: only lane 0 of each warp traces (timing studies)
    float good_t;        // brick-summary threshold for this tau
    int uniform_vs;      // every volume of the launch has the same voxel size
    double inv_vs;       // 1 / that voxel size (uniform_vs only)
    int row_mod, row_rem;  // trace only the block rows ty with ty % row_mod == row_rem
    int fresh;           // the map starts empty: not read, every traced pixel written
};

struct Hit {
    double t, hx, hy, hz, nx, ny, nz;
};

// _hit_wins (_kernels.py:246-263)
__device__ __forceinline__ bool hit_wins(const Hit &h, const Hit &cur) {
    return record_wins(h.t, h.nx, h.ny, h.nz, cur.t, cur.nx, cur.ny, cur.nz);
}

// 8 corners of the cell with minimum corner (ix, iy, iz): c[z][y][x] order
struct Cell {
    float2 c[8];
};

__device__ __forceinline__ void load_cell(const float2 *__restrict__ vox, int64_t n, int64_t ix,
                                          int64_t iy, int64_t iz, Cell &cell) {
    const float2 *b = vox + vox_index(n, iz, iy, ix);
    const int64_t sy = n, sz = n * n;
    if (!TF_IN_BOUNDS(ix >= 0 && iy >= 0 && iz >= 0 && ix + 1 < n && iy + 1 < n && iz + 1 < n)) {
        for (int c = 0; c < 8; ++c) cell.c[c] = make_float2(0.f, 0.f);
        return;
    }
    cell.c[0] = __ldg(b);
    cell.c[1] = __ldg(b + 1);
    cell.c[2] = __ldg(b + sy);
    cell.c[3] = __ldg(b + sy + 1);
    cell.c[4] = __ldg(b + sz);
    cell.c[5] = __ldg(b + sz + 1);
    cell.c[6] = __ldg(b + sz + sy);
    cell.c[7] = __ldg(b + sz + sy + 1);
}

__device__ __forceinline__ bool cell_observed(const Cell &cell) {
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 8; ++k) ok &= !(cell.c[k].y <= 0.0f);  // :40-50
    return ok;
}

// _sample (_kernels.py:28-68)
__device__ __forceinline__ bool sample(const float2 *__restrict__ vox, int64_t n, double qx,
                                       double qy, double qz, double &value) {
    const double flx = floor(qx), fly = floor(qy), flz = floor(qz);
    const double hi = (double)(n - 2);
    if (!(flx >= 0.0 && fly >= 0.0 && flz >= 0.0 && flx <= hi && fly <= hi && flz <= hi))
        return false;
    const int64_t ix = (int64_t)flx, iy = (int64_t)fly, iz = (int64_t)flz;
    Cell cell;
    load_cell(vox, n, ix, iy, iz, cell);
    if (!cell_observed(cell)) return false;
    const double fx = dsub(qx, flx), fy = dsub(qy, fly), fz = dsub(qz, flz);
    const double gx = dsub(1.0, fx), gy = dsub(1.0, fy), gz = dsub(1.0, fz);
    const double c00 = dadd(dmul((double)cell.c[0].x, gx), dmul((double)cell.c[1].x, fx));
    const double c10 = dadd(dmul((double)cell.c[2].x, gx), dmul((double)cell.c[3].x, fx));
    const double c01 = dadd(dmul((double)cell.c[4].x, gx), dmul((double)cell.c[5].x, fx));
    const double c11 = dadd(dmul((double)cell.c[6].x, gx), dmul((double)cell.c[7].x, fx));
    const double c0 = dadd(dmul(c00, gy), dmul(c10, fy));
    const double c1 = dadd(dmul(c01, gy), dmul(c11, fy));
    value = dadd(dmul(c0, gz), dmul(c1, fz));
    return true;
}

struct Ray {
    const float2 *vox;
    int64_t n;
    double htx, hty, htz, vs;
    double ox, oy, oz, dx, dy, dz;
    unsigned long long samples;
    double ivs;  // an approximation of 1 / vs for div_vs (0: always the IEEE division)
};

// RN(x / b), the IEEE quotient, from an approximate reciprocal: a
// Newton-corrected q1 is returned only when it is PROVED to be the correctly
// rounded quotient — its remainder x - q1 b (one FMA; exact whenever q1 is
// within one ulp, i.e. whenever the test can pass) is below half an ulp of q1
// times |b|, and q1 is not a power of two (where the spacing below halves).
// Anything else — ties, huge / tiny magnitudes, a poor reciprocal — takes
// the IEEE division.  So the result is ddiv(x, b) bit for bit, always.
__device__ __forceinline__ double div_vs(double x, double b, double inv) {
    const double ax = fabs(x);
    if (ax >= 0x1p-900 && ax <= 0x1p900) {
        const double q0 = dmul(x, inv);
        const double q1 = __fma_rn(__fma_rn(-q0, b, x), inv, q0);
        const double r1 = __fma_rn(-q1, b, x);
        const long long bits = __double_as_longlong(q1);
        const double half_ulp = __longlong_as_double(bits & 0x7FF0000000000000ll) * 0x1p-53;
        if ((bits & 0x000FFFFFFFFFFFFFll) != 0 && fabs(r1) < half_ulp * fabs(b)) return q1;
    }
    return ddiv(x, b);
}

// fine lattice point k in local voxel coordinates (:164-167, :357-359)
__device__ __noinline__ bool sample_at(Ray &r, int64_t k, double &value) {
    const double tk = dmul((double)k, r.vs);
    const double kx = dsub(div_vs(dadd(r.ox, dmul(tk, r.dx)), r.vs, r.ivs), r.htx);
    const double ky = dsub(div_vs(dadd(r.oy, dmul(tk, r.dy)), r.vs, r.ivs), r.hty);
    const double kz = dsub(div_vs(dadd(r.oz, dmul(tk, r.dz)), r.vs, r.ivs), r.htz);
    r.samples++;
    return sample(r.vox, r.n, kx, ky, kz, value);
}

// (edge * a) * b with the edge a float32 difference (numba types the corners
// float32, _kernels.py:201-226)
__device__ __forceinline__ double gterm(float hi, float lo, double a, double b) {
    return dmul(dmul((double)fsubr(hi, lo), a), b);
}

// Crossing acceptance of _scan_crossing (_kernels.py:170-240) for the
// consecutive samples (k-1, k) with exact values sp_v > 0 >= s.
__device__ __noinline__ bool accept_crossing(const Ray &r, int64_t k, double sp_v, double s, Hit &hit) {
    const double delta = r.vs;
    const double hi = (double)(r.n - 2);
    const double ta = dmul((double)(k - 1), delta);
    const double tstar = dadd(ta, dmul(delta, ddiv(sp_v, dsub(sp_v, s))));  // :171
    if (!(tstar >= 0.0)) return false;
    const double hx = dadd(r.ox, dmul(tstar, r.dx));
    const double hy = dadd(r.oy, dmul(tstar, r.dy));
    const double hz = dadd(r.oz, dmul(tstar, r.dz));
    const double qx = dsub(div_vs(hx, r.vs, r.ivs), r.htx);
    const double qy = dsub(div_vs(hy, r.vs, r.ivs), r.hty);
    const double qz = dsub(div_vs(hz, r.vs, r.ivs), r.htz);
    const double fcx = floor(qx), fcy = floor(qy), fcz = floor(qz);
    if (!(fcx >= 0.0 && fcy >= 0.0 && fcz >= 0.0 && fcx <= hi && fcy <= hi && fcz <= hi)) return false;
    Cell cell;
    load_cell(r.vox, r.n, (int64_t)fcx, (int64_t)fcy, (int64_t)fcz, cell);
    bool observed = true;
#pragma unroll
    for (int q = 0; q < 8; ++q) observed &= cell.c[q].y > 0.0f;  // :189-196
    if (!observed) return false;
    const double gfx = dsub(qx, fcx), gfy = dsub(qy, fcy), gfz = dsub(qz, fcz);
    const double ofx = dsub(1.0, gfx), ofy = dsub(1.0, gfy), ofz = dsub(1.0, gfz);
    const float c000 = cell.c[0].x, c100 = cell.c[1].x, c010 = cell.c[2].x, c110 = cell.c[3].x,
                c001 = cell.c[4].x, c101 = cell.c[5].x, c011 = cell.c[6].x, c111 = cell.c[7].x;
    double gx = dadd(dadd(dadd(gterm(c100, c000, ofy, ofz), gterm(c110, c010, gfy, ofz)),
                          gterm(c101, c001, ofy, gfz)),
                     gterm(c111, c011, gfy, gfz));                          // :209-214
    double gy = dadd(dadd(dadd(gterm(c010, c000, ofx, ofz), gterm(c110, c100, gfx, ofz)),
                          gterm(c011, c001, ofx, gfz)),
                     gterm(c111, c101, gfx, gfz));                          // :215-220
    double gz = dadd(dadd(dadd(gterm(c001, c000, ofx, ofy), gterm(c011, c010, ofx, gfy)),
                          gterm(c101, c100, gfx, ofy)),
                     gterm(c111, c110, gfx, gfy));                          // :221-226
    const double gnorm = dsqrt(dadd(dadd(dmul(gx, gx), dmul(gy, gy)), dmul(gz, gz)));
    if (!(gnorm > 0.0)) return false;
    if (dadd(dadd(dmul(gx, r.dx), dmul(gy, r.dy)), dmul(gz, r.dz)) > 0.0) {
        gx = -gx;
        gy = -gy;
        gz = -gz;
    }
    hit.t = tstar;
    hit.hx = hx;
    hit.hy = hy;
    hit.hz = hz;
    hit.nx = ddiv(gx, gnorm);
    hit.ny = ddiv(gy, gnorm);
    hit.nz = ddiv(gz, gnorm);
    return true;
}

// _scan_crossing (_kernels.py:136-243)
__device__ bool scan_crossing(Ray &r, int64_t scan_from, int64_t scan_end, bool sp_valid,
                              double sp_v, Hit &hit) {
    for (int64_t k = scan_from; k <= scan_end; ++k) {
        double s = 0.0;
        const bool sv = sample_at(r, k, s);
        if (sp_valid && sp_v > 0.0 && sv && s <= 0.0 && accept_crossing(r, k, sp_v, s, hit))
            return true;                                               // :169-240
        sp_valid = sv;
        sp_v = s;
    }
    return false;
}

// Entry lattice interval of the ray in one volume's sampleable box
// (_kernels.py:299-348); false on a miss.
__device__ __forceinline__ bool ray_interval(const TfVolume &vol, const double o[3],
                                             const double d[3], int64_t &j0, int64_t &j_end) {
    double t_lo = 0.0, t_hi = 1.0e30;
    const double vs = vol.voxel_size;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double mn = dmul((double)vol.origin[a], vs);
        const double mx = dmul((double)(vol.origin[a] + vol.n - 1), vs);
        if (fabs(d[a]) < 1.0e-15) {
            if (o[a] < mn || o[a] > mx) return false;
        } else {
            double t1 = ddiv(dsub(mn, o[a]), d[a]);
            double t2 = ddiv(dsub(mx, o[a]), d[a]);
            if (t1 > t2) {
                const double tmp = t1;
                t1 = t2;
                t2 = tmp;
            }
            if (t1 > t_lo) t_lo = t1;
            if (t2 < t_hi) t_hi = t2;
        }
    }
    if (t_lo > t_hi) return false;
    j0 = (int64_t)ceil(ddiv(t_lo, vs));
    if (j0 < 0) j0 = 0;
    j_end = (int64_t)floor(ddiv(t_hi, vs));
    return true;
}

// ray_interval with its eight divisions replaced by products with 1/d (per
// ray) and 1/vs: every candidate t is then within 2^-50 |t| of the reference's
// quotient, so t_lo / t_hi are within E = 2^-46 max|t| of the reference's (max
// and min are 1-Lipschitz), and j0 / j_end = ceil / floor of t / vs within
// (E + 2^-52 |t|) / vs.  When the hit-or-miss test or a ceil / floor is closer
// than that to flipping, the exact ray_interval decides.  Same (j0, j_end) and
// result as ray_interval, bit for bit.
__device__ __forceinline__ bool ray_interval_fast(const TfVolume &vol, const double o[3], const double d[3],
                                                  const double inv_d[3], const double inv_vs, int64_t &j0,
                                                  int64_t &j_end) {
    double t_lo = 0.0, t_hi = 1.0e30, tmax = 0.0;
    const double vs = vol.voxel_size;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double mn = dmul((double)vol.origin[a], vs);
        const double mx = dmul((double)(vol.origin[a] + vol.n - 1), vs);
        if (fabs(d[a]) < 1.0e-15) {
            if (o[a] < mn || o[a] > mx) return false;
        } else {
            double t1 = dmul(dsub(mn, o[a]), inv_d[a]);
            double t2 = dmul(dsub(mx, o[a]), inv_d[a]);
            if (t1 > t2) {
                const double tmp = t1;
                t1 = t2;
                t2 = tmp;
            }
            tmax = fmax(tmax, fmax(fabs(t1), fabs(t2)));
            if (t1 > t_lo) t_lo = t1;
            if (t2 < t_hi) t_hi = t2;
        }
    }
    const double e = 0x1p-46 * tmax;
    if (t_lo - t_hi > 2.0 * e) return false;                   // certainly a miss
    bool sure = t_hi - t_lo > 2.0 * e;                         // certainly not a miss
    const double xl = dmul(t_lo, inv_vs), xh = dmul(t_hi, inv_vs);
    const double ml = (e + 0x1p-52 * fabs(t_lo)) * inv_vs * 2.0, mh = (e + 0x1p-52 * fabs(t_hi)) * inv_vs * 2.0;
    const double cl = ceil(xl), fh = floor(xh);
    // t_lo == 0 exactly iff the reference's is (the candidates' signs are exact)
    sure = sure && (t_lo == 0.0 || (cl - xl > ml && xl - (cl - 1.0) > ml)) && xh - fh > mh && fh + 1.0 - xh > mh;
    if (!sure) return ray_interval(vol, o, d, j0, j_end);
    j0 = (int64_t)cl;
    if (j0 < 0) j0 = 0;
    j_end = (int64_t)fh;
    return true;
}

// The per-volume march of raycast_kernel (_kernels.py:349-451), merging into
// `best`.  Returns whether `best` changed.
__device__ __noinline__ bool march_volume(Ray &r, int64_t j, int64_t j_end, int64_t coarse,
                             double near_thresh, Hit &best) {
    bool prev_has = false;
    double prev_v = 0.0;
    int64_t prev_j = -1, last_j = j - 1, swept_j = j - 1;
    while (j <= j_end) {
        double value = 0.0;
        const bool valid = sample_at(r, j, value);
        bool do_scan = false;
        if (!valid || value <= 0.0) {                                   // :362-369
            if (prev_has && prev_v > 0.0)
                do_scan = true;
            else if (swept_j < j - 1 && (valid || coarse > 2))
                do_scan = true;
        }
        if (do_scan) {
            const int64_t scan_from = (prev_j > swept_j ? prev_j : swept_j) + 1;
            const int64_t k0 = scan_from - 1;
            bool sp_valid;
            double sp_v = 0.0;
            if (prev_has && k0 == prev_j) {
                sp_valid = true;
                sp_v = prev_v;
            } else {
                sp_valid = sample_at(r, k0, sp_v);
            }
            Hit h;
            const bool found = scan_crossing(r, scan_from, j, sp_valid, sp_v, h);
            swept_j = j;
            if (found) {
                if (hit_wins(h, best)) {
                    best = h;
                    return true;
                }
                return false;                                           // finished
            }
        }
        last_j = j;
        if (valid) {
            prev_has = true;
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
    // exit re-walk (:417-451)
    const int64_t scan_from = (last_j > swept_j ? last_j : swept_j) + 1;
    if (scan_from <= j_end) {
        const int64_t k0 = scan_from - 1;
        bool sp_valid;
        double sp_v = 0.0;
        if (prev_has && k0 == prev_j) {
            sp_valid = true;
            sp_v = prev_v;
        } else {
            sp_valid = sample_at(r, k0, sp_v);
        }
        Hit h;
        if (scan_crossing(r, scan_from, j_end, sp_valid, sp_v, h) && hit_wins(h, best)) {
            best = h;
            return true;
        }
    }
    return false;
}


// ---- certified fast march -------------------------------------------------
//
// The reference samples the lattice point k at q = (o + (k vs) d) / vs - ht,
// i.e. q ~= q0 + k d with q0 = o / vs - ht; the difference between the
// reference's rounded q and fma(k, d, q0) is < 1e-9 voxel here (|q|, k,
// |o / vs|, |ht| < 1e6).  fast_sample() takes floor(q) from a 20-bit fixed
// point of q and evaluates the trilinear value in float32, then CERTIFIES
// every decision the march takes from the sample: the cell index (q farther
// than 4 * 2^-20 from an integer), validity (exact weights), the sign
// (|value| > 2e-5 max|corner|, > 5x the float32 + fixed-point error) and the
// near-surface test (| |value| - 0.99 tau | above the same bound).  An
// uncertain sample makes the caller redo the whole ray-volume march with the
// exact reference arithmetic; a crossing is recomputed from the two exact
// samples (k-1, k) and accepted with the reference's exact arithmetic.  So
// every output bit is the reference's, at ~6 float64 ops per sample instead
// of 3 divisions and 11 conversions.

// The march only ever consumes three facts about a sample: valid, value > 0
// and |value| < 0.99 tau.  fast_sample() returns them certified, or kUnsure
// when any of them is too close to call; an unsure sample is then evaluated
// with the exact reference arithmetic (sample_at), so every decision is the
// reference's.
enum : unsigned { kValidBit = 1u, kPosBit = 2u, kNearBit = 4u, kUnsure = 8u, kSummaryBit = 16u };

struct FastRay {
    const float2 *vox;
    int n;
    double q0x, q0y, q0z, dx, dy, dz;
    float near, near_tol;
    const unsigned *bad;  // brick summary (NULL: not usable for this tau)
    unsigned nb;
    float idfx, idfy, idfz;  // 1 / d (approximate; only used with margins)
    const unsigned char *flags;  // per-brick flags (bit0 never observed, bit1 free)
};

// What the rare exact paths need beyond the FastRay, by reference into the
// kernel's parameter space (two pointers instead of a dozen live doubles).
struct RayRef {
    const TfVolume *vol;
    const RayGeom *g;
};

// the exact reference view of the ray (sample_at / accept_crossing)
__device__ __forceinline__ Ray make_ray(const FastRay &fr, const RayRef &rr) {
    Ray r;
    r.vox = fr.vox;
    r.n = rr.vol->n;
    r.htx = (double)rr.vol->origin[0];
    r.hty = (double)rr.vol->origin[1];
    r.htz = (double)rr.vol->origin[2];
    r.vs = rr.vol->voxel_size;
    r.ivs = rr.g->uniform_vs ? rr.g->inv_vs : 0.0;
    r.ox = rr.g->cam.v[0];
    r.oy = rr.g->cam.v[1];
    r.oz = rr.g->cam.v[2];
    r.dx = fr.dx;
    r.dy = fr.dy;
    r.dz = fr.dz;
    r.samples = 0;
    return r;
}

// floor(q) from a 20-bit fixed point: bits = round(q 2^20) mod 2^32 (q in
// (-2^11, 4096)), cell = bits >> 20 (floor(q) mod 2^12), fraction field
// fq = bits & (2^20 - 1).  The reference's q differs from fma(k, d, q0) by
// < 1e-9, so the floor is certain unless q is within 1.5 * 2^-20 of an
// integer, i.e. unless fq is 0, 1 or 2^20 - 1.
__device__ __forceinline__ unsigned fixed_bits(double q) {
    return (unsigned)__double2loint(dadd(q, 6442450944.0));  // + 1.5 * 2^32: ulp = 2^-20
}
__device__ __forceinline__ bool fixed_unsure(unsigned bits) { return ((bits + 1u) & 0xFFFFFu) < 3u; }
// fq * 2^-20 exactly (fq < 2^20 fits the float mantissa shifted by 3)
__device__ __forceinline__ float fixed_frac(unsigned bits) {
    return __int_as_float(0x3F800000 | ((bits & 0xFFFFFu) << 3)) - 1.0f;
}

__device__ __forceinline__ float lerpf(float a, float b, float t) { return fmaf(t, b - a, a); }

__device__ __forceinline__ unsigned fast_sample(const FastRay &r, int k, bool use_summary) {
    const double kd = (double)k;
    const unsigned bx_ = fixed_bits(dfma(kd, r.dx, r.q0x));
    const unsigned by_ = fixed_bits(dfma(kd, r.dy, r.q0y));
    const unsigned bz_ = fixed_bits(dfma(kd, r.dz, r.q0z));
    if (fixed_unsure(bx_) || fixed_unsure(by_) || fixed_unsure(bz_)) return kUnsure;
    const unsigned ix = bx_ >> 20, iy = by_ >> 20, iz = bz_ >> 20;
    const unsigned top = (unsigned)(r.n - 2);
    if (ix > top || iy > top || iz > top) return 0u;                  // invalid (:38)
    if (!TF_IN_BOUNDS(ix + 1 < (unsigned)r.n && iy + 1 < (unsigned)r.n && iz + 1 < (unsigned)r.n)) return 0u;
    if (use_summary) {
        // min corner in a never-observed brick: certainly invalid (:40-50);
        // every corner in bricks whose voxels are all observed and >= T:
        // certainly valid, positive and not near the surface
        const unsigned bx = ix >> 3, by = iy >> 3, bz = iz >> 3;
        const unsigned st = __ldg(&r.bad[(bz * r.nb + by) * r.nb + bx]);
        if ((st >> 16) == 0u) return kSummaryBit;
        if ((st & 0xFFFFu) == 0u) {
            const unsigned ex = ((ix & 7u) == 7u), ey = ((iy & 7u) == 7u), ez = ((iz & 7u) == 7u);
            bool good = true;
#pragma unroll
            for (unsigned c = 1; c < 8; ++c) {
                if (((c & 1u) && !ex) || ((c & 2u) && !ey) || ((c & 4u) && !ez)) continue;
                const unsigned nbx = bx + (c & 1u), nby = by + ((c >> 1) & 1u), nbz = bz + (c >> 2);
                good = good && TF_IN_BOUNDS(nbx < r.nb && nby < r.nb && nbz < r.nb) &&
                       (__ldg(&r.bad[(nbz * r.nb + nby) * r.nb + nbx]) & 0xFFFFu) == 0u;
            }
            if (good) return kValidBit | kPosBit | kSummaryBit;
        }
    }
    const unsigned n = (unsigned)r.n;
    const float2 *b = r.vox + ((size_t)(iz * n + iy) * n + ix);
    const float2 c000 = __ldg(b), c100 = __ldg(b + 1), c010 = __ldg(b + n), c110 = __ldg(b + n + 1);
    const float fx = fixed_frac(bx_), fy = fixed_frac(by_), fz = fixed_frac(bz_);
    const float2 c001 = __ldg(b + n * n), c101 = __ldg(b + n * n + 1);
    const float2 c011 = __ldg(b + n * n + n), c111 = __ldg(b + n * n + n + 1);
    const float wmin = fminf(fminf(fminf(c000.y, c100.y), fminf(c010.y, c110.y)),
                             fminf(fminf(c001.y, c101.y), fminf(c011.y, c111.y)));
    if (wmin <= 0.0f) return 0u;                                      // invalid (:40-50)
    const float v = lerpf(lerpf(lerpf(c000.x, c100.x, fx), lerpf(c010.x, c110.x, fx), fy),
                          lerpf(lerpf(c001.x, c101.x, fx), lerpf(c011.x, c111.x, fx), fy), fz);
    const float cmax = fmaxf(fmaxf(fmaxf(fabsf(c000.x), fabsf(c100.x)), fabsf(c010.x)),
                             fmaxf(fmaxf(fabsf(c110.x), fabsf(c001.x)),
                                   fmaxf(fmaxf(fabsf(c101.x), fabsf(c011.x)), fabsf(c111.x))));
    const float ev = 2e-5f * cmax + 1e-30f;
    const float av = fabsf(v);
    if (av <= ev || fabsf(av - r.near) <= ev + r.near_tol) return kUnsure;
    return kValidBit | (v > 0.f ? kPosBit : 0u) | (av < r.near ? kNearBit : 0u);
}

// Region of lattice point j for the brick DDA: when the cell of j certainly
// has its min corner in a never-observed or free-space superbrick (64^3) or
// brick (8^3), returns its flags (bit0 never observed, bit1 free space) and
// sets `exit` to a k >= j - 1 such that for j <= k <= exit the min corner
// certainly stays in that box — for free space also at most n - 2, so the
// cell stays in the volume.  Returns 0 for an ordinary brick (exit = its box)
// and -1 if undecided.  The exit is computed in float from the position
// inside the box (truncated to 2^-17 voxel) against box faces pulled in by
// 1e-4 voxel, and the step count shrunk by 1e-6 relative: both bound the
// float rounding, and the < 1e-9 error of q against the reference.
__device__ __forceinline__ int region_at(const FastRay &r, int j, int &exit) {
    const double kd = (double)j;
    const unsigned bits[3] = {fixed_bits(dfma(kd, r.dx, r.q0x)), fixed_bits(dfma(kd, r.dy, r.q0y)),
                              fixed_bits(dfma(kd, r.dz, r.q0z))};
    if (fixed_unsure(bits[0]) || fixed_unsure(bits[1]) || fixed_unsure(bits[2])) return -1;
    const unsigned lo[3] = {bits[0] >> 20, bits[1] >> 20, bits[2] >> 20};
    const unsigned top = (unsigned)(r.n - 2);
    if (lo[0] > top || lo[1] > top || lo[2] > top) return -1;
    const unsigned ns = (r.nb + 7u) >> 3;
    const unsigned char *sflags = r.flags + (size_t)r.nb * r.nb * r.nb;
    // both levels loaded up front: one memory round trip, not two
    const int sfl = __ldg(&sflags[((lo[2] >> 6) * ns + (lo[1] >> 6)) * ns + (lo[0] >> 6)]) & 3;
    const int bfl = __ldg(&r.flags[((lo[2] >> 3) * r.nb + (lo[1] >> 3)) * r.nb + (lo[0] >> 3)]) & 3;
    const int fl = sfl ? sfl : bfl;
    const unsigned shift = sfl ? 6u : 3u;
    const unsigned mask = (1u << shift) - 1u;
    const float idf[3] = {r.idfx, r.idfy, r.idfz};
    float steps = 1.0e8f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        // position inside the box, truncated to 2^-17 (23 bits)
        const unsigned x = ((lo[a] & mask) << 17) | ((bits[a] & 0xFFFFFu) >> 3);
        const float local = (__int_as_float(0x4B000000 | x) - 8388608.0f) * 7.62939453125e-06f;  // 2^-17
        float face;
        if (idf[a] >= 0.0f) {
            face = (float)(1u << shift);
            if (fl & 2) face = fminf(face, (float)(top + 1u - (lo[a] & ~mask)));  // cap at n - 1
            face -= 1e-4f;
        } else {
            face = 1e-4f;
        }
        steps = fminf(steps, (face - local) * idf[a]);  // 0 * inf = NaN is ignored by fminf
    }
    exit = steps < 0.0f ? j - 1 : j + (int)(steps * 0.999999f);
    return fl;
}

// certified decisions of lattice point k (exact fallback when unsure)
__device__ __forceinline__ unsigned cert_sample(const FastRay &fr, const RayRef &er, int k,
                                                unsigned long long &samples,
                                                unsigned long long &exact_samples,
                                                bool use_summary = true) {
    ++samples;
    const unsigned s = fast_sample(fr, k, use_summary && fr.bad != nullptr);
    if (s & kSummaryBit) exact_samples += 1ull << 44;  // summary-certified (counter in the high bits)
    if (!(s & kUnsure)) return s & ~kSummaryBit;
    ++exact_samples;
    Ray r = make_ray(fr, er);
    double v = 0.0;
    if (!sample_at(r, k, v)) return 0u;
    return kValidBit | (v > 0.0 ? kPosBit : 0u) | (fabs(v) < er.g->near_thresh ? kNearBit : 0u);
}

// _scan_crossing on certified decisions; the crossing itself is exact.
// Returns whether a crossing was accepted (into `hit`).
// `end_s` = the decisions of point `end` when the march just sampled it
// (kNoDecision otherwise): the reference samples it again; the result is the same.
constexpr unsigned kNoDecision = 0x80000000u;
__device__ __forceinline__ bool scan_fast(const FastRay &fr, const RayRef &er, int from, int end,
                                          unsigned sp, Hit &hit, unsigned long long &samples,
                                          unsigned long long &exact_samples, unsigned end_s = kNoDecision) {
    for (int k = from; k <= end; ++k) {
        unsigned s;
        if (k == end && end_s != kNoDecision) {
            ++samples;
            s = end_s;
        } else if (k == end - 1 && end_s != kNoDecision &&
                   (sp & (kValidBit | kPosBit)) != (kValidBit | kPosBit) &&
                   (end_s & (kValidBit | kPosBit)) != kValidBit) {
            // no crossing can involve point end - 1: one at end - 1 needs a
            // valid positive seed, one at end a valid non-positive end point
            ++samples;
            s = 0u;
        } else {
            s = cert_sample(fr, er, k, samples, exact_samples);
        }
        // sp_valid and sp_v > 0 and sv and s <= 0 (:169)
        if ((sp & (kValidBit | kPosBit)) == (kValidBit | kPosBit) && (s & (kValidBit | kPosBit)) == kValidBit) {
            Ray r = make_ray(fr, er);
            double e0 = 0.0, e1 = 0.0;
            const bool v0 = sample_at(r, k - 1, e0), v1 = sample_at(r, k, e1);
            exact_samples += 2;
            if (!v0 || !v1 || !(e0 > 0.0) || !(e1 <= 0.0)) {
                // a certified decision disagreed with the exact arithmetic: never
                // expected; counted (TF_STAT_CERT_FAILURES) so tests catch it
                exact_samples += 1ull << 40;
            } else if (accept_crossing(r, k, e0, e1, hit)) {
                return true;
            }
        }
        sp = s;
    }
    return false;
}

// march_volume on certified decisions (_kernels.py:349-451); same control flow.
// Returns whether `best` changed.
#ifdef TF_RAY_DIAG
// diagnostics build (TFB200_NVCC_EXTRA=-DTF_RAY_DIAG): cycles / calls per
// phase of march_fast into the debug ray buffer slots 4..11 of the pixel
#define DIAG_T0 const long long _t0 = clock64();
#define DIAG_ACC(i) diag[i] += clock64() - _t0; diag[(i) + 4] += 1;
#define DIAG_PARAM , int64_t *diag
#define DIAG_ARG , diag
#else
#define DIAG_T0
#define DIAG_ACC(i)
#define DIAG_PARAM
#define DIAG_ARG
#endif
__device__ bool march_fast(const FastRay &fr, const RayRef &er, int j, const int j_end, const int coarse,
                           Hit &best, unsigned long long &samples, unsigned long long &exact_samples,
                           const long long deadline, bool &aborted DIAG_PARAM) {
    unsigned prev = 0u;  // decisions of the last valid march sample
    bool prev_has = false;
    int prev_j = -1, last_j = j - 1, swept_j = j - 1;
    int phase = j % coarse;  // j mod coarse, tracked so no division runs per step
    // current brick region (DDA over 8^3 bricks): fine points j <= region_end
    // have their min corner in one brick of kind region_kind (bit0 never
    // observed, bit1 free space, 0 = ordinary)
    int region_end = -1, region_kind = 0, region_start = 0;
    unsigned last_s = kNoDecision;  // decisions of march point last_j
    unsigned tick = 0;
    while (j <= j_end) {
        // the warp ran past its budget: hand the ray to the cooperative pass
        // (the clock is read every 8th step: the budget is a heuristic)
        if ((++tick & 7u) == 0u && clock64() > deadline) {
            aborted = true;
            return false;
        }
        if (fr.flags && j > region_end) {
            int ex = j - 1;
            DIAG_T0
            const int fl = region_at(fr, j, ex);
            DIAG_ACC(0)
            region_start = j;
            if (fl < 0 || ex < j) {
                region_end = j;  // undecided: this point normally, retry at the next
                region_kind = 0;
            } else {
                region_end = ex >= j_end ? j_end : ex;
                region_kind = fl & 3;
            }
        }
        if (region_kind & 2) {
            // free space: every march point in [j, region_end] is valid, positive
            // and not near -> coarse steps, no scans (:362-416)
            const int m = coarse == 2 ? (region_end & ~1) : region_end - region_end % coarse;
            const int p_last = m > j ? m : j;
            const int first = j + (coarse - phase);
            const int cnt = 1 + (m > j ? (coarse == 2 ? (m - first) >> 1 : (m - first) / coarse) + 1 : 0);
            samples += cnt;
            exact_samples += (unsigned long long)cnt << 44;
            prev_has = true;
            prev = kValidBit | kPosBit;
            prev_j = last_j = p_last;
            last_s = kValidBit | kPosBit;
            if (p_last != j) phase = 0;
            j = p_last + (coarse - phase);
            phase = 0;
            continue;
        }
        if ((region_kind & 1) && j > region_start) {
            // never observed: the march points in [j, region_end] are invalid and any
            // scan covers (max(prev_j, swept_j), p] inside the region: nothing found
            // (:362-405); j is a multiple of coarse here (invalid -> coarse step)
            const int cnt = (coarse == 2 ? (region_end - j) >> 1 : (region_end - j) / coarse) + 1;
            const int p_last = j + (cnt - 1) * coarse;
            const bool A = prev_has && (prev & kPosBit);
            if (A || (coarse > 2 && (cnt >= 2 || swept_j < j - 1))) swept_j = p_last;
            last_j = p_last;
            last_s = 0u;  // invalid
            samples += cnt;
            exact_samples += (unsigned long long)cnt << 44;
            j = p_last + coarse;
            phase = 0;
            continue;
        }
        // inside a known ordinary brick region the per-sample summary cannot help
        DIAG_T0
        const bool use_sum = region_end < j || region_kind != 0;
        const unsigned s = cert_sample(fr, er, j, samples, exact_samples, use_sum);
        DIAG_ACC(1)
        const bool valid = s & kValidBit;
        bool do_scan = false;
        if (!valid || !(s & kPosBit)) {                                 // :362-369
            if (prev_has && (prev & kPosBit))
                do_scan = true;
            else if (swept_j < j - 1 && (valid || coarse > 2))
                do_scan = true;
        }
        if (do_scan) {
            DIAG_T0
            const int scan_from = (prev_j > swept_j ? prev_j : swept_j) + 1;
            const int k0 = scan_from - 1;
            unsigned sp;
            if (prev_has && k0 == prev_j) {
                sp = prev;
            } else if (k0 == last_j && last_s != kNoDecision) {
                ++samples;  // the reference samples the seed again (:371-382)
                sp = last_s;
            } else {
                sp = cert_sample(fr, er, k0, samples, exact_samples);
            }
            Hit h;
            const bool found = scan_fast(fr, er, scan_from, j, sp, h, samples, exact_samples, s);
            DIAG_ACC(2)
            swept_j = j;
            if (found) {
                if (hit_wins(h, best)) {
                    best = h;
                    return true;
                }
                return false;
            }
        }
        last_j = j;
        last_s = s;
        if (valid) {
            prev_has = true;
            prev = s;
            prev_j = j;
        }
        if (valid && (s & kNearBit)) {  // fine step
            ++j;
            phase = phase + 1 == coarse ? 0 : phase + 1;
        } else {                         // next multiple of coarse
            j += coarse - phase;
            phase = 0;
        }
    }
    const int scan_from = (last_j > swept_j ? last_j : swept_j) + 1;  // :417-451
    if (scan_from <= j_end) {
        const int k0 = scan_from - 1;
        unsigned sp;
        if (prev_has && k0 == prev_j) {
            sp = prev;
        } else if (k0 == last_j && last_s != kNoDecision) {
            ++samples;
            sp = last_s;
        } else {
            sp = cert_sample(fr, er, k0, samples, exact_samples);
        }
        Hit h;
        if (scan_fast(fr, er, scan_from, j_end, sp, h, samples, exact_samples) && hit_wins(h, best)) {
            best = h;
            return true;
        }
    }
    return false;
}

// unit ray direction of pixel (px, py) (_kernels.py:307-315)
__device__ __forceinline__ void ray_direction(const RayGeom &g, int64_t px, int64_t py, double d[3]) {
    const double *R = g.r_wc.m;
    const double rx = ddiv(dsub((double)px, g.cx), g.fx);
    const double ry = ddiv(dsub((double)py, g.cy), g.fy);
#pragma unroll
    for (int a = 0; a < 3; ++a) d[a] = dadd(dadd(dmul(R[3 * a], rx), dmul(R[3 * a + 1], ry)), R[3 * a + 2]);
    const double dn = dsqrt(dadd(dadd(dmul(d[0], d[0]), dmul(d[1], d[1])), dmul(d[2], d[2])));
    d[0] = ddiv(d[0], dn);
    d[1] = ddiv(d[1], dn);
    d[2] = ddiv(d[2], dn);
}

// the exact (Ray) and certified (FastRay) views of a ray in one volume;
// false when the certified march cannot be used (forced exact, or
// coordinates too large to certify)
__device__ __forceinline__ bool setup_volume(const RayGeom &g, const TfVolume &vol, const double o[3],
                                             const double d[3], int64_t j_end, Ray &r, FastRay &fr) {
    r.vox = (const float2 *)vol.voxels_dev;
    r.n = vol.n;
    r.htx = (double)vol.origin[0];
    r.hty = (double)vol.origin[1];
    r.htz = (double)vol.origin[2];
    r.vs = vol.voxel_size;
    r.ivs = g.uniform_vs ? g.inv_vs : 0.0;
    r.ox = o[0];
    r.oy = o[1];
    r.oz = o[2];
    r.dx = d[0];
    r.dy = d[1];
    r.dz = d[2];
    r.samples = 0;
    const double q0x = dsub(ddiv(o[0], r.vs), r.htx);
    const double q0y = dsub(ddiv(o[1], r.vs), r.hty);
    const double q0z = dsub(ddiv(o[2], r.vs), r.htz);
    const double mag = fabs(q0x) + fabs(q0y) + fabs(q0z) + fabs(r.htx) + fabs(r.hty) + fabs(r.htz) +
                       (double)j_end;
    const bool summ = vol.brick_state_dev != nullptr && vol.summary_threshold == g.good_t;
    fr = FastRay{r.vox, (int)vol.n, q0x, q0y, q0z, d[0], d[1], d[2],
                 (float)g.near_thresh, (float)g.near_thresh * 2.4e-7f,
                 summ ? vol.brick_state_dev : nullptr, (unsigned)((vol.n + 7) / 8),
                 1.0f / (float)d[0], 1.0f / (float)d[1], 1.0f / (float)d[2],
                 summ ? vol.brick_flags_dev : nullptr};
    return !g.exact_only && vol.n <= 4000 && mag < 1e6 && j_end < (1 << 30) && g.coarse < (1 << 20);
}

// a warp traces 8x4 pixels; a block of kBX x kBY pixels (kBX/8 x kBY/4 warps)

template <int kBX, int kBY, int kMinBlocks>
__global__ void __launch_bounds__(kBX * kBY, kMinBlocks) raycast_kernel(
    const __grid_constant__ VolumeTable vt, const __grid_constant__ RayGeom g,
    double *__restrict__ out_dist, double *__restrict__ out_vert, double *__restrict__ out_norm,
    unsigned long long *__restrict__ stats, int64_t *__restrict__ clocks, unsigned *__restrict__ rescue,
    unsigned *__restrict__ rescue_count, long long budget) {
    constexpr int kList = 4;
    __shared__ int2 s_list[kList][kBX * kBY];
    const long long t_start = clock64();
    const long long deadline = budget > 0 ? t_start + budget : LLONG_MAX;
    long long t_start_ns = 0;
    if (clocks) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start_ns));
    // warps tile the block's pixels in 8x4 units, row-major
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t px = (int64_t)blockIdx.x * kBX + (w % (kBX / 8)) * 8 + (lane & 7);
    // tile rows are dispatched centre-out: rays near the image centre row run
    // longest in typical scenes, so they start first and the tail is short
    // block rows are dispatched centre-out over this launch's subset of rows
    // (every row_mod-th from row_rem; all rows by default)
    const int by = (int)blockIdx.y, mid = (int)(gridDim.y >> 1);
    const int ty = g.row_rem + g.row_mod * ((by & 1) ? mid - ((by + 1) >> 1) : mid + (by >> 1));
    const int64_t py = (int64_t)ty * kBY + (w / (kBX / 8)) * 4 + (lane >> 3);
    unsigned long long samples = 0, hits = 0, exact_samples = 0;
    if (px < g.width && py < g.height && !(g.lane0_only && lane != 0)) {
        const int64_t p = py * g.width + px;
        Hit best{INFINITY, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // RayMap.empty's record
        if (!g.fresh) {
            best.t = out_dist[p];
            best.hx = out_vert[3 * p + 0];
            best.hy = out_vert[3 * p + 1];
            best.hz = out_vert[3 * p + 2];
            best.nx = out_norm[3 * p + 0];
            best.ny = out_norm[3 * p + 1];
            best.nz = out_norm[3 * p + 2];
        }
        double d[3];
        ray_direction(g, px, py, d);
        const double o[3] = {g.cam.v[0], g.cam.v[1], g.cam.v[2]};

        // Volumes are visited nearest entry first (the skip test below then
        // prunes whatever lies behind a hit; any order gives the same map, the
        // merge is order-free).  The order comes in batches of kList entries
        // (lattice entry index, exit index | volume << 26) kept sorted in
        // shared memory, one column per thread: no per-thread local arrays.
        // A ray crossing more than kList volumes rebuilds the next batch from
        // the ones after the last entry marched.  Launches mixing voxel sizes,
        // or lattice indices beyond 2^26, take the volumes in index order.
        bool changed = false, aborted = false;
        // n entries in the current batch, bi the next one to march; flags:
        // bit 0 = more volumes after the batch, bit 1 = index order (the
        // cursor of a rebuild is the batch's last entry, read back from smem)
        int n = 0, bi = 0, flags = g.uniform_vs ? 1 : 3;
        while (!aborted) {
            int v;
            int64_t lo, hi;
            if (!(flags & 2) && bi == n) {
                if (!(flags & 1)) break;
                int cur_lo = -1, cur_v = -1;
                if (n > 0) {
                    const int2 c = s_list[n - 1][threadIdx.x];
                    cur_lo = c.x;
                    cur_v = (int)((unsigned)c.y >> 26);
                }
                n = bi = 0;
                flags = 0;
                double inv_d[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) inv_d[c] = fabs(d[c]) < 1.0e-15 ? 0.0 : ddiv(1.0, d[c]);
                for (int u = 0; u < vt.count; ++u) {
                    int64_t a, b;
                    if (!ray_interval_fast(vt.vol[u], o, d, inv_d, g.inv_vs, a, b)) continue;
                    if (b >= (1ll << 26) || a >= (1ll << 30)) {  // decided on the first build
                        flags = 2;
                        break;
                    }
                    const int ia = (int)a;
                    if (ia < cur_lo || (ia == cur_lo && u <= cur_v)) continue;  // an earlier batch
                    int pos = n;
                    while (pos > 0 && s_list[pos - 1][threadIdx.x].x > ia) {
                        if (pos < kList) s_list[pos][threadIdx.x] = s_list[pos - 1][threadIdx.x];
                        --pos;
                    }
                    if (pos < kList) s_list[pos][threadIdx.x] = make_int2(ia, (int)b | (u << 26));
                    if (n < kList) ++n;
                    else flags = 1;
                }
                if (!(flags & 2) && n == 0) break;
            }
            if (!(flags & 2)) {
                const int2 e = s_list[bi++][threadIdx.x];
                v = (int)((unsigned)e.y >> 26);
                lo = e.x;
                hi = e.y & ((1 << 26) - 1);
            } else {  // index order; bi walks the volumes
                while (bi < vt.count && !ray_interval(vt.vol[bi], o, d, lo, hi)) ++bi;
                if (bi == vt.count) break;
                v = bi++;
            }
            const TfVolume &vol = vt.vol[v];
            // no hit of this volume can have tstar below (j0 - 1) * delta
            if (dmul((double)(lo - 1), vol.voxel_size) > best.t) continue;
            Ray r;
            FastRay fr;
            if (setup_volume(g, vol, o, d, hi, r, fr)) {
#ifdef TF_RAY_DIAG
                int64_t *diag = clocks ? clocks + 12 * p + 4 : nullptr;
                if (!diag) __trap();
#endif
                DIAG_T0
                changed |= march_fast(fr, RayRef{&vol, &g}, (int)lo, (int)hi, (int)g.coarse, best,
                                      samples, exact_samples, deadline, aborted DIAG_ARG);
                DIAG_ACC(3)
            } else {  // forced, or coordinates too large to certify: the exact reference march
                changed |= march_volume(r, lo, hi, g.coarse, g.near_thresh, best);
                samples += r.samples;
                exact_samples += r.samples;
            }
        }
        if (aborted) {
            // finished by raycast_coop_kernel (one warp per ray); nothing of
            // this partial march is kept (a fresh map gets the empty record,
            // which the cooperative pass merges into)
            samples = exact_samples = 0;
            rescue[atomicAdd(rescue_count, 1u)] = (unsigned)p;
            changed = false;
            if (g.fresh) best = Hit{INFINITY, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        }
        if ((changed || g.fresh) && TF_IN_BOUNDS(p < g.width * g.height)) {
            hits = changed ? 1 : 0;
            out_dist[p] = best.t;
            out_vert[3 * p + 0] = best.hx;
            out_vert[3 * p + 1] = best.hy;
            out_vert[3 * p + 2] = best.hz;
            out_norm[3 * p + 0] = best.nx;
            out_norm[3 * p + 1] = best.ny;
            out_norm[3 * p + 2] = best.nz;
        }
    }
    if (clocks && px < g.width && py < g.height) {
        const int64_t q = 12 * (py * g.width + px);
#ifndef TF_RAY_DIAG
        // timeline: the pixel's start / end on the global nanosecond timer
        clocks[q + 4] = t_start_ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(clocks[q + 5]));
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        clocks[q + 6] = smid;
#endif
        clocks[q] = clock64() - t_start;
        clocks[q + 1] = (int64_t)samples;
        clocks[q + 2] = (int64_t)(exact_samples & ((1ull << 40) - 1));
        clocks[q + 3] = (int64_t)(exact_samples >> 44);
    }
    if (stats) {
        unsigned long long *const dst[5] = {&stats[TF_STAT_RAY_SAMPLES], &stats[TF_STAT_RAY_HITS],
                                            &stats[TF_STAT_EXACT_SAMPLES], &stats[TF_STAT_CERT_FAILURES],
                                            &stats[TF_STAT_SUMMARY_SAMPLES]};
        block_count_add<5>(dst, {samples, hits, exact_samples & ((1ull << 40) - 1),
                                 (exact_samples >> 40) & 15ull, exact_samples >> 44});
    }
}

// ---- cooperative march: one warp per ray ---------------------------------
//
// Rays that graze partially observed space evaluate hundreds of samples and
// keep a whole warp busy long after the rest of the frame is done (their
// lanes diverge on every step).  raycast_kernel hands such rays over when
// its warp exceeds a cycle budget; here the 32 lanes of a warp decide 32
// consecutive fine lattice points of ONE ray at once (certified decisions,
// as in the per-lane march) and then replay the reference's march over those
// decisions warp-uniformly: the same march points, scans, seeds, crossings
// and exit re-walk as march_volume (_kernels.py:349-451), so the result is
// the same bits.

// decisions of 64 consecutive fine points [base, base + 63] of one ray
struct CoopWindow {
    int base;
    unsigned long long v, pos, nr;  // valid / value > 0 / |value| < 0.99 tau
};

// decisions of 32 consecutive points: bit i = point a + i
struct Dec32 {
    unsigned v, pos, nr;
};

// the 32 lanes decide points [b, b + 31] (only those in [lo, hi]; others read as invalid)
__device__ __forceinline__ Dec32 coop_half(const FastRay &fr, const RayRef &er, int b, int lo, int hi,
                                           unsigned long long &exact_samples) {
    const int lane = threadIdx.x & 31, k = b + lane;
    unsigned s = 0u;
    if (k >= lo && k <= hi) {
        unsigned long long uncounted = 0;
        s = cert_sample(fr, er, k, uncounted, exact_samples);
    }
    return Dec32{__ballot_sync(0xffffffffu, s & kValidBit), __ballot_sync(0xffffffffu, s & kPosBit),
                 __ballot_sync(0xffffffffu, s & kNearBit)};
}

// decisions of [a, a + 31] (warp-uniform); slides the window forward as the
// march advances, decides look-backs below it directly
__device__ Dec32 coop_range(const FastRay &fr, const RayRef &er, CoopWindow &w, int a, int lo, int hi,
                            unsigned long long &exact_samples) {
    if (a < w.base) return coop_half(fr, er, a, lo, hi, exact_samples);
    if (a + 31 > w.base + 63) {
        if (a + 31 <= w.base + 95) {  // slide by 32
            w.base += 32;
            const Dec32 h = coop_half(fr, er, w.base + 32, lo, hi, exact_samples);
            w.v = (w.v >> 32) | ((unsigned long long)h.v << 32);
            w.pos = (w.pos >> 32) | ((unsigned long long)h.pos << 32);
            w.nr = (w.nr >> 32) | ((unsigned long long)h.nr << 32);
        } else {  // jump, keeping 16 points of look-back below a
            w.base = a - 16;
            const Dec32 l = coop_half(fr, er, w.base, lo, hi, exact_samples);
            const Dec32 h = coop_half(fr, er, w.base + 32, lo, hi, exact_samples);
            w.v = l.v | ((unsigned long long)h.v << 32);
            w.pos = l.pos | ((unsigned long long)h.pos << 32);
            w.nr = l.nr | ((unsigned long long)h.nr << 32);
        }
    }
    const int i = a - w.base;
    return Dec32{(unsigned)(w.v >> i), (unsigned)(w.pos >> i), (unsigned)(w.nr >> i)};
}

__device__ __forceinline__ unsigned dec_bits(const Dec32 &d, int i) {
    return ((d.v >> i) & 1u) * kValidBit | ((d.pos >> i) & 1u) * kPosBit | ((d.nr >> i) & 1u) * kNearBit;
}

// _scan_crossing over [from, end] with seed decisions sp (warp-uniform):
// crossing candidates (previous valid > 0, this valid <= 0, :169) come from
// the decision masks 32 points at a time; each is checked exactly in order
__device__ bool coop_scan(const FastRay &fr, const RayRef &er, CoopWindow &w, int lo, int hi, int from, int end,
                          unsigned sp, Hit &hit, unsigned long long &samples,
                          unsigned long long &exact_samples) {
    samples += (unsigned long long)(end - from + 1);
    for (int a = from; a <= end; a += 32) {
        const Dec32 d = coop_range(fr, er, w, a, lo, hi, exact_samples);
        const unsigned vp = d.v & d.pos;
        const unsigned vp_prev = (vp << 1) | ((sp & (kValidBit | kPosBit)) == (kValidBit | kPosBit) ? 1u : 0u);
        unsigned cand = vp_prev & d.v & ~d.pos;
        const int len = end - a + 1;
        if (len < 32) cand &= (1u << len) - 1u;
        while (cand) {
            const int k = a + __ffs(cand) - 1;
            cand &= cand - 1;
            Ray r = make_ray(fr, er);
            double e0 = 0.0, e1 = 0.0;
            const bool v0 = sample_at(r, k - 1, e0), v1 = sample_at(r, k, e1);
            exact_samples += 2;
            if (!v0 || !v1 || !(e0 > 0.0) || !(e1 <= 0.0)) {
                exact_samples += 1ull << 40;  // certified decision disagreed: counted, never expected
            } else if (accept_crossing(r, k, e0, e1, hit)) {
                return true;
            }
        }
        sp = ((vp >> 31) & 1u) ? (kValidBit | kPosBit) : 0u;  // only "valid and > 0" matters here
    }
    return false;
}

// march_volume (_kernels.py:349-451) replayed warp-uniformly over decision
// masks.  With coarse == 2, runs of march points that change nothing but
// counters are consumed in one step: invalid march points (each followed by
// a scan when the last valid sample was positive: the scans tile one range,
// searched once) and valid, positive, not-near march points (no scan).
__device__ bool march_coop(const FastRay &fr, const RayRef &er, int j, const int j_end, const int coarse,
                           Hit &best, unsigned long long &samples, unsigned long long &exact_samples) {
    const int lo = j - 1, hi = j_end;  // the only points the reference can sample
    CoopWindow w;
    w.base = INT_MIN / 2;
    w.v = w.pos = w.nr = 0ull;
    unsigned prev = 0u;
    bool prev_has = false;
    int prev_j = -1, last_j = j - 1, swept_j = j - 1;
    while (j <= j_end) {
        const Dec32 d = coop_range(fr, er, w, j, lo, hi, exact_samples);
        const unsigned s = dec_bits(d, 0);
        const bool valid = s & kValidBit;
        if (coarse == 2 && !(j & 1)) {
            // even march points j, j + 2, ... of this 32-point block (<= j_end)
            const int span = min(j_end - j, 31);
            const unsigned inblk = span >= 31 ? 0xffffffffu : ((2u << span) - 1u);
            const unsigned even = 0x55555555u & inblk;
            if (!valid) {
                // run of invalid march points
                const unsigned stop = d.v & even;
                const int f = stop ? __ffs(stop) - 1 : (span >= 31 ? 32 : span + 1);
                const int m = (f + 1) >> 1;  // march points j, ..., j + 2(m-1)
                const int jl = j + 2 * (m - 1);
                samples += m;
                if (prev_has && (prev & kPosBit)) {  // every one of them scans (:362-369)
                    const int scan_from = (prev_j > swept_j ? prev_j : swept_j) + 1;
                    const int k0 = scan_from - 1;
                    unsigned sp;
                    if (k0 == prev_j) {
                        sp = prev;
                    } else {
                        sp = dec_bits(coop_range(fr, er, w, k0, lo, hi, exact_samples), 0);
                        ++samples;
                    }
                    samples += m - 1;  // the later scans' seeds
                    Hit h;
                    if (coop_scan(fr, er, w, lo, hi, scan_from, jl, sp, h, samples, exact_samples)) {
                        if (hit_wins(h, best)) {
                            best = h;
                            return true;
                        }
                        return false;
                    }
                    swept_j = jl;
                }
                last_j = jl;
                j = jl + 2;
                continue;
            }
            if ((s & (kPosBit | kNearBit)) == kPosBit) {
                // run of valid, positive, not-near march points: no scans
                const unsigned stop = ~(d.v & d.pos & ~d.nr) & even;
                const int f = stop ? __ffs(stop) - 1 : (span >= 31 ? 32 : span + 1);
                const int m = (f + 1) >> 1;
                const int jl = j + 2 * (m - 1);
                samples += m;
                prev_has = true;
                prev = kValidBit | kPosBit;
                prev_j = last_j = jl;
                j = jl + 2;
                continue;
            }
        }
        // one march point (:356-416)
        ++samples;
        bool do_scan = false;
        if (!valid || !(s & kPosBit)) {
            if (prev_has && (prev & kPosBit))
                do_scan = true;
            else if (swept_j < j - 1 && (valid || coarse > 2))
                do_scan = true;
        }
        if (do_scan) {
            const int scan_from = (prev_j > swept_j ? prev_j : swept_j) + 1;
            const int k0 = scan_from - 1;
            unsigned sp;
            if (prev_has && k0 == prev_j) {
                sp = prev;
            } else {
                sp = dec_bits(coop_range(fr, er, w, k0, lo, hi, exact_samples), 0);
                ++samples;
            }
            Hit h;
            const bool found = coop_scan(fr, er, w, lo, hi, scan_from, j, sp, h, samples, exact_samples);
            swept_j = j;
            if (found) {
                if (hit_wins(h, best)) {
                    best = h;
                    return true;
                }
                return false;
            }
        }
        last_j = j;
        if (valid) {
            prev_has = true;
            prev = s;
            prev_j = j;
        }
        if (valid && (s & kNearBit))
            j += 1;
        else
            j = (j / coarse + 1) * coarse;
    }
    const int scan_from = (last_j > swept_j ? last_j : swept_j) + 1;  // :417-451
    if (scan_from <= j_end) {
        const int k0 = scan_from - 1;
        unsigned sp;
        if (prev_has && k0 == prev_j) {
            sp = prev;
        } else {
            sp = dec_bits(coop_range(fr, er, w, k0, lo, hi, exact_samples), 0);
            ++samples;
        }
        Hit h;
        if (coop_scan(fr, er, w, lo, hi, scan_from, j_end, sp, h, samples, exact_samples) && hit_wins(h, best)) {
            best = h;
            return true;
        }
    }
    return false;
}

// the rays raycast_kernel handed over: one warp per ray, every lane holds the
// same ray state; lane 0 writes
__device__ void coop_whole_rays(const VolumeTable &vt, const RayGeom &g, double *__restrict__ out_dist,
                                double *__restrict__ out_vert, double *__restrict__ out_norm,
                                const unsigned *__restrict__ rescue, const unsigned count, const unsigned first,
                                const unsigned warp, const unsigned nwarps, unsigned long long &samples,
                                unsigned long long &hits, unsigned long long &exact_samples) {
    const int lane = threadIdx.x & 31;
    for (unsigned i = first + warp; i < count; i += nwarps) {
        const int64_t p = rescue[i];
        const int64_t py = p / g.width, px = p - py * g.width;
        Hit best;
        best.t = out_dist[p];
        best.hx = out_vert[3 * p + 0];
        best.hy = out_vert[3 * p + 1];
        best.hz = out_vert[3 * p + 2];
        best.nx = out_norm[3 * p + 0];
        best.ny = out_norm[3 * p + 1];
        best.nz = out_norm[3 * p + 2];
        double d[3];
        ray_direction(g, px, py, d);
        const double o[3] = {g.cam.v[0], g.cam.v[1], g.cam.v[2]};
        // volumes nearest entry first, each pick re-scanning the intervals (a
        // rare path: rays beyond the split capacity; no per-lane arrays)
        bool changed = false;
        int64_t cur_lo = -1;
        int cur_v = -1;
        while (true) {
            int pick = -1;
            int64_t lo = 0, hi = 0;
            for (int u = 0; u < vt.count; ++u) {
                int64_t a, b;
                if (!ray_interval(vt.vol[u], o, d, a, b)) continue;
                if (a < cur_lo || (a == cur_lo && u <= cur_v)) continue;
                if (pick < 0 || a < lo) {
                    pick = u;
                    lo = a;
                    hi = b;
                }
            }
            if (pick < 0) break;
            cur_lo = lo;
            cur_v = pick;
            const TfVolume &vol = vt.vol[pick];
            if (dmul((double)(lo - 1), vol.voxel_size) > best.t) continue;
            Ray r;
            FastRay fr;
            if (setup_volume(g, vol, o, d, hi, r, fr)) {
                changed |= march_coop(fr, RayRef{&vol, &g}, (int)lo, (int)hi, (int)g.coarse, best,
                                      samples, exact_samples);
            } else {
                changed |= march_volume(r, lo, hi, g.coarse, g.near_thresh, best);
                samples += r.samples;
                exact_samples += r.samples;
            }
        }
        if (changed && lane == 0) {
            ++hits;
            out_dist[p] = best.t;
            out_vert[3 * p + 0] = best.hx;
            out_vert[3 * p + 1] = best.hy;
            out_vert[3 * p + 2] = best.hz;
            out_norm[3 * p + 0] = best.nx;
            out_norm[3 * p + 1] = best.ny;
            out_norm[3 * p + 2] = best.nz;
        }
    }
}

// The first `cap` handed-over rays, split into (ray, volume) items, one warp
// each: a ray's marches through different volumes are independent (each
// returns its first accepted crossing whatever the running best is; the
// nearest-entry order only lets the per-lane pass skip volumes), so they run
// in parallel and raycast_coop_merge_kernel folds the per-volume hits with
// _hit_wins — the same result, with the pass bounded by the slowest
// ray-volume march instead of the slowest ray.  slots: 8 doubles per item
// (t, hit xyz, normal xyz; t = +inf: no hit).
__global__ void __launch_bounds__(128, 4) raycast_coop_items_kernel(
    const __grid_constant__ VolumeTable vt, const __grid_constant__ RayGeom g,
    unsigned long long *__restrict__ stats, const unsigned *__restrict__ rescue,
    const unsigned *__restrict__ rescue_count, const unsigned cap, double *__restrict__ slots,
    double *__restrict__ out_dist, double *__restrict__ out_vert, double *__restrict__ out_norm) {
    const int lane = threadIdx.x & 31;
    const unsigned all = *rescue_count;
    const unsigned count = min(all, cap);
    const unsigned nitems = count * (unsigned)vt.count;
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
    unsigned long long samples = 0, exact_samples = 0;
    for (unsigned i = warp; i < nitems; i += nwarps) {
        const unsigned ray = i / (unsigned)vt.count;
        const int v = (int)(i - ray * (unsigned)vt.count);
        const int64_t p = rescue[ray];
        const int64_t py = p / g.width, px = p - py * g.width;
        double d[3];
        ray_direction(g, px, py, d);
        const double o[3] = {g.cam.v[0], g.cam.v[1], g.cam.v[2]};
        Hit best{INFINITY, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        bool found = false;
        int64_t jlo = 0, jhi = 0;
        const TfVolume &vol = vt.vol[v];
        if (ray_interval(vol, o, d, jlo, jhi)) {
            Ray r;
            FastRay fr;
            if (setup_volume(g, vol, o, d, jhi, r, fr)) {
                found = march_coop(fr, RayRef{&vol, &g}, (int)jlo, (int)jhi, (int)g.coarse, best, samples,
                                   exact_samples);
            } else {
                found = march_volume(r, jlo, jhi, g.coarse, g.near_thresh, best);
                samples += r.samples;
                exact_samples += r.samples;
            }
        }
        if (lane == 0) {
            double *sl = slots + 8 * (size_t)i;
            sl[0] = found ? best.t : INFINITY;
            sl[1] = best.hx;
            sl[2] = best.hy;
            sl[3] = best.hz;
            sl[4] = best.nx;
            sl[5] = best.ny;
            sl[6] = best.nz;
        }
    }
    // rays beyond the split capacity (usually none): one warp per whole ray,
    // written directly (they have no slots)
    unsigned long long hits = 0;
    coop_whole_rays(vt, g, out_dist, out_vert, out_norm, rescue, all, cap, warp, nwarps, samples, hits,
                    exact_samples);
    if (stats && threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(&stats[TF_STAT_COOP_RAYS], (unsigned long long)all);
    if (stats && lane == 0) {  // every lane counted the same item: lane 0 reports
        atomicAdd(&stats[TF_STAT_RAY_SAMPLES], samples);
        atomicAdd(&stats[TF_STAT_RAY_HITS], hits);
        atomicAdd(&stats[TF_STAT_EXACT_SAMPLES], exact_samples & ((1ull << 40) - 1));
        atomicAdd(&stats[TF_STAT_CERT_FAILURES], (exact_samples >> 40) & 15ull);
    }
}

// one thread per split ray: fold its volumes' hits into the map (_hit_wins)
__global__ void raycast_coop_merge_kernel(const int nvol, const unsigned *__restrict__ rescue,
                                          const unsigned *__restrict__ rescue_count, const unsigned cap,
                                          const double *__restrict__ slots, double *__restrict__ out_dist,
                                          double *__restrict__ out_vert, double *__restrict__ out_norm,
                                          unsigned long long *__restrict__ stats) {
    const unsigned j = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned count = min(*rescue_count, cap);
    unsigned long long hits = 0;
    if (j < count) {
        const int64_t p = rescue[j];
        Hit best{out_dist[p], out_vert[3 * p], out_vert[3 * p + 1], out_vert[3 * p + 2],
                 out_norm[3 * p], out_norm[3 * p + 1], out_norm[3 * p + 2]};
        bool changed = false;
        for (int v = 0; v < nvol; ++v) {
            const double *sl = slots + 8 * ((size_t)j * nvol + v);
            if (!(sl[0] < INFINITY)) continue;
            const Hit h{sl[0], sl[1], sl[2], sl[3], sl[4], sl[5], sl[6]};
            if (hit_wins(h, best)) {
                best = h;
                changed = true;
            }
        }
        if (changed) {
            hits = 1;
            out_dist[p] = best.t;
            out_vert[3 * p + 0] = best.hx;
            out_vert[3 * p + 1] = best.hy;
            out_vert[3 * p + 2] = best.hz;
            out_norm[3 * p + 0] = best.nx;
            out_norm[3 * p + 1] = best.ny;
            out_norm[3 * p + 2] = best.nz;
        }
    }
    if (stats) warp_count_add(&stats[TF_STAT_RAY_HITS], hits);
}

__global__ void raymap_merge_kernel(double *__restrict__ dd, double *__restrict__ dv,
                                    double *__restrict__ dn, const double *__restrict__ sd,
                                    const double *__restrict__ sv, const double *__restrict__ sn,
                                    int64_t npix) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npix) return;
    Hit h{sd[p], 0, 0, 0, sn[3 * p], sn[3 * p + 1], sn[3 * p + 2]};
    Hit cur{dd[p], 0, 0, 0, dn[3 * p], dn[3 * p + 1], dn[3 * p + 2]};
    if (hit_wins(h, cur)) {
        dd[p] = sd[p];
        for (int a = 0; a < 3; ++a) {
            dv[3 * p + a] = sv[3 * p + a];
            dn[3 * p + a] = sn[3 * p + a];
        }
    }
}

__global__ void trilinear_sample_kernel(const TfVolume vol, const double *__restrict__ pts,
                                        int64_t npts, double *__restrict__ values,
                                        uint8_t *__restrict__ valid) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npts) return;
    // q = point / voxel_size - origin_voxel (tsdf.py:149)
    const double qx = dsub(ddiv(pts[3 * i + 0], vol.voxel_size), (double)vol.origin[0]);
    const double qy = dsub(ddiv(pts[3 * i + 1], vol.voxel_size), (double)vol.origin[1]);
    const double qz = dsub(ddiv(pts[3 * i + 2], vol.voxel_size), (double)vol.origin[2]);
    double v = 0.0;
    const bool ok = sample((const float2 *)vol.voxels_dev, vol.n, qx, qy, qz, v);
    values[i] = ok ? v : 0.0;
    valid[i] = ok ? 1 : 0;
}

// _hit_wins over packed (t, nx, ny, nz) records: the cross-GPU row-block
// reduction exchanges only these (vertices follow from t, tf_raymap_vertices)
__global__ void raymap_merge_packed_kernel(double4 *__restrict__ dst, const double4 *__restrict__ src,
                                           int64_t npix) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npix) return;
    const double4 a = src[p], b = dst[p];
    const Hit h{a.x, 0, 0, 0, a.y, a.z, a.w};
    const Hit cur{b.x, 0, 0, 0, b.y, b.z, b.w};
    if (hit_wins(h, cur)) dst[p] = a;
}

// hit vertex = o + t d with the raycast's own arithmetic (accept_crossing:
// dadd(o, dmul(tstar, d)), d from ray_direction), so a vertex rebuilt from t
// is the one the raycast wrote; 0 where there is no hit (RayMap.empty)
__global__ void raymap_vertices_kernel(const __grid_constant__ RayGeom g, const double *__restrict__ dist,
                                       int64_t dist_stride, double *__restrict__ vert, int64_t row0,
                                       int64_t nrows) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrows * g.width) return;
    const int64_t py = row0 + i / g.width, px = i % g.width;
    const double t = dist[i * dist_stride];
    double v[3] = {0.0, 0.0, 0.0};
    if (t < INFINITY) {
        double d[3];
        ray_direction(g, px, py, d);
#pragma unroll
        for (int a = 0; a < 3; ++a) v[a] = dadd(g.cam.v[a], dmul(t, d[a]));
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) vert[3 * i + a] = v[a];
}

// colour at a rendered hit (tf_raycast_colors): the hit point from t with the
// raycast's arithmetic, then the first volume whose cell around it has all
// 8 corner colours observed, trilinear in float32
__global__ void raycast_colors_kernel(const __grid_constant__ VolumeTable vt, const __grid_constant__ RayGeom g,
                                      const double *__restrict__ dist, float *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.width * g.height) return;
    const int64_t py = i / g.width, px = i - py * g.width;
    const double t = dist[i];
    float rgb[3] = {0.f, 0.f, 0.f};
    if (t < INFINITY) {
        double d[3];
        ray_direction(g, px, py, d);
        const double h[3] = {dadd(g.cam.v[0], dmul(t, d[0])), dadd(g.cam.v[1], dmul(t, d[1])),
                             dadd(g.cam.v[2], dmul(t, d[2]))};
        for (int v = 0; v < vt.count; ++v) {
            const TfVolume &vol = vt.vol[v];
            if (!vol.color_dev) continue;
            double q[3], fl[3];
            bool inside = true;
            for (int a = 0; a < 3; ++a) {
                q[a] = dsub(ddiv(h[a], vol.voxel_size), (double)vol.origin[a]);
                fl[a] = floor(q[a]);
                inside = inside && fl[a] >= 0.0 && fl[a] <= (double)(vol.n - 2);
            }
            if (!inside) continue;
            const int64_t n = vol.n, x = (int64_t)fl[0], y = (int64_t)fl[1], z = (int64_t)fl[2];
            const uchar4 *c = reinterpret_cast<const uchar4 *>(vol.color_dev) + (z * n + y) * n + x;
            const uchar4 k[8] = {c[0], c[1], c[n], c[n + 1], c[n * n], c[n * n + 1], c[n * n + n],
                                 c[n * n + n + 1]};
            bool seen = true;
            for (int j = 0; j < 8; ++j) seen = seen && k[j].w > 0;
            if (!seen) continue;
            const float fx = (float)(q[0] - fl[0]), fy = (float)(q[1] - fl[1]), fz = (float)(q[2] - fl[2]);
            const float w8[8] = {(1 - fx) * (1 - fy) * (1 - fz), fx * (1 - fy) * (1 - fz),
                                 (1 - fx) * fy * (1 - fz),       fx * fy * (1 - fz),
                                 (1 - fx) * (1 - fy) * fz,       fx * (1 - fy) * fz,
                                 (1 - fx) * fy * fz,             fx * fy * fz};
            for (int j = 0; j < 8; ++j) {
                rgb[0] += w8[j] * (float)k[j].x;
                rgb[1] += w8[j] * (float)k[j].y;
                rgb[2] += w8[j] * (float)k[j].z;
            }
            break;
        }
    }
    out[3 * i + 0] = rgb[0];
    out[3 * i + 1] = rgb[1];
    out[3 * i + 2] = rgb[2];
}

}  // namespace tf

using namespace tf;

TF_BOUNDS_READER(raycast)

// Rescue list + per-(ray, volume) hit slots of the cooperative pass.  They
// come from the caller's workspace (tf_raycast_ws, sized by
// tf_raycast_workspace_size); tf_raycast without a workspace keeps a small
// per-(device, stream) table of buffers, least recently used evicted.
namespace {
constexpr unsigned kCoopSplitRays = 16384;

int64_t rescue_slot_offset(int64_t npix) { return (npix + 1 + 63) / 64 * 64; }  // words, 256-B aligned

int64_t rescue_words(int64_t npix, int nvol_launch) {
    return rescue_slot_offset(npix) + (int64_t)kCoopSplitRays * nvol_launch * 16;
}
}  // namespace

static unsigned *rescue_buffer(cudaStream_t stream, int64_t words) {
    struct Buf {
        int dev;
        cudaStream_t stream;
        unsigned *ptr;
        int64_t words;
        unsigned long long used;
    };
    constexpr int kBufs = 16;
    static std::mutex mu;
    static Buf bufs[kBufs];
    static int nbufs = 0;
    static unsigned long long tick = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    Buf *b = nullptr;
    for (int i = 0; i < nbufs; ++i)
        if (bufs[i].dev == dev && bufs[i].stream == stream) b = &bufs[i];
    if (!b) {
        if (nbufs < kBufs) {
            b = &bufs[nbufs++];
        } else {  // evict the least recently used entry (its stream may still use it)
            b = &bufs[0];
            for (int i = 1; i < kBufs; ++i)
                if (bufs[i].used < b->used) b = &bufs[i];
            if (b->ptr) {
                int cur = dev;
                cudaSetDevice(b->dev);
                cudaStreamSynchronize(b->stream);
                cudaFree(b->ptr);
                cudaSetDevice(cur);
            }
        }
        *b = Buf{dev, stream, nullptr, 0, 0};
    }
    b->used = ++tick;
    if (b->words < words) {
        if (b->ptr) {
            cudaStreamSynchronize(stream);  // the old buffer may still be in use on this stream
            cudaFree(b->ptr);
            b->ptr = nullptr;
            b->words = 0;
        }
        if (cudaMalloc((void **)&b->ptr, (size_t)words * sizeof(unsigned)) != cudaSuccess) return nullptr;
        b->words = words;
    }
    return b->ptr;
}

namespace tf {
// test hook: random and adversarial (volume, ray) pairs through
// ray_interval_fast vs ray_interval; counts result / (j0, j_end) mismatches
// and how often the fast path fell back (out[0], out[1])
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 33;
    return x;
}
__device__ __forceinline__ double unif(unsigned long long &st) {  // [0, 1)
    st = mix64(st + 0x9E3779B97F4A7C15ull);
    return (double)(st >> 11) * 0x1p-53;
}
__global__ void ray_interval_check_kernel(int64_t n, unsigned long long seed, unsigned long long *out) {
    const double vss[5] = {0.004, 0.001, 0.0029296875, 0.1, 0.0117647058823529};
    unsigned long long bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long st = seed ^ (0xD1B54A32D192ED03ull * (unsigned long long)(i + 1));
        TfVolume vol{};
        vol.voxel_size = vss[(int)(unif(st) * 5.0)];
        vol.n = 2 + (int64_t)(unif(st) * 600.0);
        for (int a = 0; a < 3; ++a) vol.origin[a] = (int64_t)(unif(st) * 1200.0) - 600;
        double d[3], o[3];
        double nn = 0.0;
        for (int a = 0; a < 3; ++a) {
            d[a] = unif(st) * 2.0 - 1.0;
            const double r = unif(st);
            if (r < 0.1) d[a] = 0.0;
            else if (r < 0.13) d[a] = 1e-16;
            nn += d[a] * d[a];
        }
        if (nn == 0.0) d[0] = nn = 1.0;
        nn = sqrt(nn);
        for (int a = 0; a < 3; ++a) d[a] /= nn;
        const double vs = vol.voxel_size, lo0 = (double)vol.origin[0] * vs;
        for (int a = 0; a < 3; ++a)
            o[a] = ((double)vol.origin[a] + (unif(st) * 1.6 - 0.3) * (double)vol.n) * vs;
        const double r = unif(st);
        if (r < 0.2) {  // on a face of the box
            const int a = (int)(unif(st) * 3.0);
            o[a] = dmul((double)(vol.origin[a] + (unif(st) < 0.5 ? 0 : vol.n - 1)), vs);
        } else if (r < 0.4 && fabs(d[0]) > 0.1) {  // the x-entry t an integer multiple of vs
            const double k = floor(unif(st) * 400.0) + 1.0;
            o[0] = dsub(lo0, dmul(dmul(k, vs), d[0]));
        }
        int64_t a0 = -7, a1 = -7, b0 = -7, b1 = -7;
        double inv_d[3];
        for (int c = 0; c < 3; ++c) inv_d[c] = fabs(d[c]) < 1.0e-15 ? 0.0 : ddiv(1.0, d[c]);
        const bool h0 = ray_interval(vol, o, d, a0, a1);
        const bool h1 = ray_interval_fast(vol, o, d, inv_d, 1.0 / vs, b0, b1);
        bad += h0 != h1 || (h0 && (a0 != b0 || a1 != b1));
    }
    if (bad) atomicAdd(&out[0], bad);
}
// test hook: div_vs against the IEEE division on random and adversarial
// (x, b) pairs, with the exact reciprocal and with perturbed ones
__global__ void div_check_kernel(int64_t n, unsigned long long seed, unsigned long long *out) {
    const double vss[6] = {0.004, 0.001, 0.0029296875, 0.1, 0.0117647058823529, 3.0};
    unsigned long long bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long st = seed ^ (0xA0761D6478BD642Full * (unsigned long long)(i + 1));
        const double r = unif(st);
        double b = r < 0.5 ? vss[(int)(unif(st) * 6.0)] : ldexp(1.0 + unif(st), (int)(unif(st) * 40.0) - 20);
        double x;
        const double c = unif(st);
        if (c < 0.3) {  // near-multiples of b: quotients at or next to integers and halves
            x = dmul((double)((int64_t)(unif(st) * 4096.0) - 2048) * 0.5, b);
            if (unif(st) < 0.5)  // a neighbouring double (one ulp up or down in magnitude)
                x = __longlong_as_double(__double_as_longlong(x) + (unif(st) < 0.5 ? 1 : -1));
        } else {
            x = ldexp(1.0 + unif(st), (int)(unif(st) * 60.0) - 40);
            if (unif(st) < 0.5) x = -x;
        }
        const double exact_inv = 1.0 / b;
        const double p = unif(st);
        const double inv = p < 0.6 ? exact_inv
                                   : (p < 0.8 ? __longlong_as_double(__double_as_longlong(exact_inv) + 1)
                                              : exact_inv * (1.0 + 1e-9));
        bad += __double_as_longlong(div_vs(x, b, inv)) != __double_as_longlong(__ddiv_rn(x, b));
    }
    if (bad) atomicAdd(out, bad);
}
}  // namespace tf

extern "C" int64_t tf_debug_div_check(int64_t n, uint64_t seed) {
    unsigned long long *d = nullptr, h = 0;
    if (n <= 0) return 0;
    if (cudaMalloc(&d, sizeof(h)) != cudaSuccess) return -1;
    cudaMemset(d, 0, sizeof(h));
    tf::div_check_kernel<<<1184, 256>>>(n, seed, d);
    const bool ok = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaFree(d);
    return ok ? (int64_t)h : -1;
}

extern "C" int64_t tf_debug_ray_interval_check(int64_t n, uint64_t seed) {
    unsigned long long *d = nullptr, h = 0;
    if (n <= 0) return 0;
    if (cudaMalloc(&d, sizeof(h)) != cudaSuccess) return -1;
    cudaMemset(d, 0, sizeof(h));
    tf::ray_interval_check_kernel<<<1184, 256>>>(n, seed, d);
    const bool ok = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaFree(d);
    return ok ? (int64_t)h : -1;
}

extern "C" size_t tf_raycast_workspace_size(int nvol, const TfCamera *cam) {
    if (!cam || nvol <= 0 || cam->width <= 0 || cam->height <= 0) return 0;
    const int per = nvol < TFB200_MAX_VOLUMES_PER_LAUNCH ? nvol : TFB200_MAX_VOLUMES_PER_LAUNCH;
    return (size_t)rescue_words(cam->width * cam->height, per) * sizeof(unsigned);
}

__global__ void raymap_reset_kernel(double *__restrict__ dist, double *__restrict__ vert,
                                    double *__restrict__ norm, int64_t npix);

static int raycast_impl(const TfVolume *vols, int nvol, const TfCamera *cam, double tau,
                        int64_t coarse_step, const double r_wc[9], const double cam_center[3],
                        double *dist, double *vert, double *norm, void *workspace,
                        size_t workspace_bytes, uint64_t *stats, void *stream_, int row_mod, int row_rem,
                        int flags = 0);

extern "C" int tf_raycast_ws(const TfVolume *vols, int nvol, const TfCamera *cam, double tau,
                             int64_t coarse_step, const double r_wc[9], const double cam_center[3],
                             double *dist, double *vert, double *norm, void *workspace,
                             size_t workspace_bytes, uint64_t *stats, void *stream_) {
    if (!workspace && nvol > 0) return tf_set_error(TF_EINVAL, "tf_raycast_ws: null workspace");
    return raycast_impl(vols, nvol, cam, tau, coarse_step, r_wc, cam_center, dist, vert, norm,
                        workspace, workspace_bytes, stats, stream_, 1, 0);
}

extern "C" int tf_raycast_rows(const TfVolume *vols, int nvol, const TfCamera *cam, double tau,
                               int64_t coarse_step, const double r_wc[9], const double cam_center[3],
                               double *dist, double *vert, double *norm, void *workspace,
                               size_t workspace_bytes, int row_mod, int row_rem, uint64_t *stats,
                               void *stream_) {
    if (!workspace && nvol > 0) return tf_set_error(TF_EINVAL, "tf_raycast_rows: null workspace");
    if (row_mod < 1 || row_rem < 0 || row_rem >= row_mod)
        return tf_set_error(TF_EINVAL, "tf_raycast_rows: bad row subset");
    return raycast_impl(vols, nvol, cam, tau, coarse_step, r_wc, cam_center, dist, vert, norm,
                        workspace, workspace_bytes, stats, stream_, row_mod, row_rem);
}

extern "C" int tf_raycast_ex(const TfVolume *vols, int nvol, const TfCamera *cam, double tau,
                             int64_t coarse_step, const double r_wc[9], const double cam_center[3],
                             double *dist, double *vert, double *norm, void *workspace,
                             size_t workspace_bytes, int row_mod, int row_rem, int flags, uint64_t *stats,
                             void *stream_) {
    if (!workspace && nvol > 0) return tf_set_error(TF_EINVAL, "tf_raycast_ex: null workspace");
    if (row_mod < 1 || row_rem < 0 || row_rem >= row_mod)
        return tf_set_error(TF_EINVAL, "tf_raycast_ex: bad row subset");
    if ((flags & TF_RAYCAST_FRESH) && row_mod != 1)
        return tf_set_error(TF_EINVAL, "tf_raycast_ex: TF_RAYCAST_FRESH traces every row");
    return raycast_impl(vols, nvol, cam, tau, coarse_step, r_wc, cam_center, dist, vert, norm, workspace,
                        workspace_bytes, stats, stream_, row_mod, row_rem, flags);
}

extern "C" int tf_raycast(const TfVolume *vols, int nvol, const TfCamera *cam, double tau,
                          int64_t coarse_step, const double r_wc[9], const double cam_center[3],
                          double *dist, double *vert, double *norm, uint64_t *stats,
                          void *stream_) {
    return raycast_impl(vols, nvol, cam, tau, coarse_step, r_wc, cam_center, dist, vert, norm,
                        nullptr, 0, stats, stream_, 1, 0);
}

static int raycast_impl(const TfVolume *vols, int nvol, const TfCamera *cam, double tau,
                        int64_t coarse_step, const double r_wc[9], const double cam_center[3],
                        double *dist, double *vert, double *norm, void *workspace,
                        size_t workspace_bytes, uint64_t *stats, void *stream_, int row_mod, int row_rem,
                        int flags) {
    cudaStream_t stream = (cudaStream_t)stream_;
    if (nvol == 0) return TF_OK;
    if (!vols || nvol < 0 || !cam || !r_wc || !cam_center || !dist || !vert || !norm)
        return tf_set_error(TF_EINVAL, "tf_raycast: null argument");
    if (cam->width <= 0 || cam->height <= 0 || coarse_step < 1)
        return tf_set_error(TF_EINVAL, "tf_raycast: bad image size or coarse step");
    RayGeom g{};
    for (int i = 0; i < 9; ++i) g.r_wc.m[i] = r_wc[i];
    for (int i = 0; i < 3; ++i) g.cam.v[i] = cam_center[i];
    g.fx = cam->fx;
    g.fy = cam->fy;
    g.cx = cam->cx;
    g.cy = cam->cy;
    g.width = cam->width;
    g.height = cam->height;
    g.near_thresh = 0.99 * tau;
    g.coarse = coarse_step;
    g.exact_only = (tf_debug_flags() & TF_DEBUG_EXACT_ONLY) ? 1 : 0;
    g.lane0_only = (tf_debug_flags() & TF_DEBUG_LANE0_ONLY) ? 1 : 0;
    g.good_t = good_threshold(tau);
    g.row_mod = row_mod;
    g.row_rem = row_rem;
    g.uniform_vs = 1;
    g.inv_vs = 1.0 / vols[0].voxel_size;
    for (int v = 1; v < nvol; ++v)
        if (vols[v].voxel_size != vols[0].voxel_size) g.uniform_vs = 0;
    for (int first = 0; first < nvol; first += TFB200_MAX_VOLUMES_PER_LAUNCH) {
        VolumeTable vt{};
        vt.count = nvol - first < TFB200_MAX_VOLUMES_PER_LAUNCH ? nvol - first
                                                                : TFB200_MAX_VOLUMES_PER_LAUNCH;
        for (int v = 0; v < vt.count; ++v) {
            vt.vol[v] = vols[first + v];
            if (!vt.vol[v].voxels_dev || vt.vol[v].n < 2 || !(vt.vol[v].voxel_size > 0.0))
                return tf_set_error(TF_EINVAL, "tf_raycast: bad volume %d", first + v);
        }
        // TF_RAYCAST_FRESH: the first launch writes every pixel (the map's
        // previous contents are never read); later chunks merge into it
        g.fresh = (flags & TF_RAYCAST_FRESH) && first == 0 ? 1 : 0;
        if (g.fresh && g.lane0_only) {  // (a debug mode that traces a subset of the pixels)
            const int64_t npix = cam->width * cam->height;
            raymap_reset_kernel<<<(unsigned)((3 * npix + 255) / 256), 256, 0, stream>>>(dist, vert, norm, npix);
            g.fresh = 0;
        }
        void *prof = tf_profile_begin(TF_PROF_RAYCAST, stream);
        static const int shape = [] {
            const char *e = getenv("TFB200_RAY_SHAPE");  // tuning knob: block shape variant
            return e ? atoi(e) : 0;
        }();
        static const long long base_budget = [] {
            // cycles a warp of the per-lane march may run before its unfinished
            // rays move to the cooperative pass (0: never), for up to 8 volumes
            const char *e = getenv("TFB200_RAY_BUDGET");
            return e ? atoll(e) : 1400000ll;
        }();
        // the bulk of the per-lane work grows with the volumes a ray crosses:
        // the budget scales with the square root of the launch's volumes beyond
        // 8 (config 3, 8 volumes: 1.4 M cycles optimal, 2.0 M 30 % slower;
        // config 4, 16 volumes: 1.4 M -> 1.90 ms, 2.0 M -> 1.45, 2.5 M -> 1.49,
        // 2.8 M -> 1.54, 4 M -> 1.70 ms)
        static const double row_exp = [] {
            const char *e = getenv("TFB200_RAY_ROW_EXP");  // tuning knob (A/B): budget ~ row_mod^-exp
            return e ? atof(e) : 0.5;
        }();
        // a launch over 1/row_mod of the rows ends sooner: its budget shrinks
        // with it, or its slowest warps (not the rows' work) set its length
        // (projected replicated-mode rates at 2 / 4 / 8 ranks, exponent 1.0:
        // 836 / 326 / 242 frames/s — the cooperative pass drowns; 0.7: 948 /
        // 783 / 653; 0.5: 896 / 954 / 929; 0: 782 / 788 / 790)
        const long long budget = (long long)(
            (vt.count > 8 ? (double)base_budget * sqrt(vt.count / 8.0) : (double)base_budget) /
            pow((double)g.row_mod, row_exp));
        const bool coop_all = (tf_debug_flags() & TF_DEBUG_COOP_ALL) != 0;
        unsigned long long *st = (unsigned long long *)stats;
        int64_t *clk = tf_ray_clock_buffer();
        const int64_t npix = cam->width * cam->height;
        // [0] = count, then pixel indices; then the per-(ray, volume) hit slots
        // of the first kCoopSplitRays handed-over rays (8 doubles each)
        const int64_t slot_off = rescue_slot_offset(npix);
        const int64_t words = rescue_words(npix, vt.count);
        unsigned *rescue = nullptr;
        if (workspace) {
            if (workspace_bytes < (size_t)words * sizeof(unsigned) || ((uintptr_t)workspace & 255u))
                return tf_set_error(TF_EINVAL, "tf_raycast_ws: workspace too small or not 256-byte aligned");
            rescue = (unsigned *)workspace;
        } else {
            rescue = rescue_buffer(stream, words);
        }
        if (!rescue || cudaMemsetAsync(rescue, 0, sizeof(unsigned), stream) != cudaSuccess)
            return tf_set_error(TF_ECUDA, "tf_raycast: cannot allocate the rescue list");
        auto launch = [&](auto kern, int bx, int by) {
            const int rows = (int)((cam->height + by - 1) / by);  // block rows of the image
            dim3 grid((unsigned)((cam->width + bx - 1) / bx),
                      (unsigned)((rows - g.row_rem + g.row_mod - 1) / g.row_mod));
            kern<<<grid, bx * by, 0, stream>>>(vt, g, dist, vert, norm, st, clk, rescue + 1, rescue,
                                               coop_all ? 1ll : budget);
        };
        // 16x8-pixel blocks of 4 warps, 5 blocks per SM (96 registers): a
        // block whose slowest warp runs to its budget holds a fifth of an SM,
        // not all of it, while neighbouring warps still share L1 lines; 20
        // warps per SM hide more latency than the spills cost (32x16 blocks of
        // 16 warps at 128 registers: 0.938 ms; 16x8 x4: 0.859; 16x8 x5: 0.839)
        switch (shape) {
        case 1: launch(raycast_kernel<32, 16, 1>, 32, 16); break;
        case 2: launch(raycast_kernel<16, 8, 4>, 16, 8); break;
        case 3: launch(raycast_kernel<32, 8, 2>, 32, 8); break;
        case 4: launch(raycast_kernel<8, 16, 5>, 8, 16); break;
        default: launch(raycast_kernel<16, 8, 5>, 16, 8); break;
        }
        int rc = tf_check_launch("raycast_kernel");
        if (rc) return rc;
        if (budget > 0 || coop_all) {
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            void *pc = tf_profile_begin(TF_PROF_RAYCAST_COOP, stream);
            double *slots = (double *)(rescue + slot_off);
            raycast_coop_items_kernel<<<(unsigned)sms * 8, 128, 0, stream>>>(vt, g, st, rescue + 1, rescue,
                                                                           kCoopSplitRays, slots, dist, vert,
                                                                           norm);
            if ((rc = tf_check_launch("raycast_coop_items_kernel"))) return rc;
            raycast_coop_merge_kernel<<<kCoopSplitRays / 128, 128, 0, stream>>>(
                vt.count, rescue + 1, rescue, kCoopSplitRays, slots, dist, vert, norm, st);
            if ((rc = tf_check_launch("raycast_coop_merge_kernel"))) return rc;
            tf_profile_end(pc, stream);
        }
        tf_profile_end(prof, stream);
    }
    return TF_OK;
}

// RayMap.empty in place: +inf distances, zero vertices and normals (one
// launch instead of three)
__global__ void raymap_reset_kernel(double *__restrict__ dist, double *__restrict__ vert,
                                    double *__restrict__ norm, int64_t npix) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * npix;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < npix) dist[i] = INFINITY;
        vert[i] = 0.0;
        norm[i] = 0.0;
    }
}

extern "C" int tf_raymap_reset(double *dist_dev, double *vert_dev, double *norm_dev, int64_t npix,
                               void *stream_) {
    if (npix <= 0) return TF_OK;
    if (!dist_dev || !vert_dev || !norm_dev) return tf_set_error(TF_EINVAL, "tf_raymap_reset: null argument");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    raymap_reset_kernel<<<(unsigned)sms * 4, 256, 0, (cudaStream_t)stream_>>>(dist_dev, vert_dev, norm_dev, npix);
    return tf_check_launch("raymap_reset_kernel");
}

extern "C" int tf_raymap_merge_packed(double *dst_dev, const double *src_dev, int64_t npix, void *stream_) {
    if (npix <= 0) return TF_OK;
    if (!dst_dev || !src_dev) return tf_set_error(TF_EINVAL, "tf_raymap_merge_packed: null argument");
    if (((uintptr_t)dst_dev | (uintptr_t)src_dev) & 31u)
        return tf_set_error(TF_EINVAL, "tf_raymap_merge_packed: records must be 32-byte aligned");
    raymap_merge_packed_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, (cudaStream_t)stream_>>>(
        (double4 *)dst_dev, (const double4 *)src_dev, npix);
    return tf_check_launch("raymap_merge_packed_kernel");
}

extern "C" int tf_raymap_vertices(const double *dist_dev, int64_t dist_stride, double *vert_dev,
                                  const TfCamera *cam, const double r_wc[9], const double cam_center[3],
                                  int64_t row0, int64_t nrows, void *stream_) {
    if (nrows <= 0) return TF_OK;
    if (!dist_dev || !vert_dev || !cam || !r_wc || !cam_center || dist_stride < 1 || row0 < 0 ||
        row0 + nrows > cam->height)
        return tf_set_error(TF_EINVAL, "tf_raymap_vertices: bad argument");
    RayGeom g{};
    for (int i = 0; i < 9; ++i) g.r_wc.m[i] = r_wc[i];
    for (int i = 0; i < 3; ++i) g.cam.v[i] = cam_center[i];
    g.fx = cam->fx;
    g.fy = cam->fy;
    g.cx = cam->cx;
    g.cy = cam->cy;
    g.width = cam->width;
    g.height = cam->height;
    const int64_t n = nrows * cam->width;
    raymap_vertices_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream_>>>(
        g, dist_dev, dist_stride, vert_dev, row0, nrows);
    return tf_check_launch("raymap_vertices_kernel");
}

extern "C" int tf_raymap_merge(double *dd, double *dv, double *dn, const double *sd,
                               const double *sv, const double *sn, int64_t npix, void *stream_) {
    if (npix <= 0) return TF_OK;
    if (!dd || !dv || !dn || !sd || !sv || !sn)
        return tf_set_error(TF_EINVAL, "tf_raymap_merge: null argument");
    raymap_merge_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, (cudaStream_t)stream_>>>(
        dd, dv, dn, sd, sv, sn, npix);
    return tf_check_launch("raymap_merge_kernel");
}

extern "C" int tf_trilinear_sample(const TfVolume *vol, const double *pts, int64_t npts,
                                   double *values, uint8_t *valid, void *stream_) {
    if (npts <= 0) return TF_OK;
    if (!vol || !pts || !values || !valid || !vol->voxels_dev)
        return tf_set_error(TF_EINVAL, "tf_trilinear_sample: null argument");
    trilinear_sample_kernel<<<(unsigned)((npts + 127) / 128), 128, 0, (cudaStream_t)stream_>>>(
        *vol, pts, npts, values, valid);
    return tf_check_launch("trilinear_sample_kernel");
}

extern "C" int tf_raycast_colors(const TfVolume *vols, int nvol, const TfCamera *cam, const double r_wc[9],
                                 const double cam_center[3], const double *dist, float *colors, void *stream_) {
    if (!cam || !r_wc || !cam_center || !dist || !colors || nvol < 0 || (nvol > 0 && !vols))
        return tf_set_error(TF_EINVAL, "tf_raycast_colors: bad argument");
    RayGeom g{};
    for (int i = 0; i < 9; ++i) g.r_wc.m[i] = r_wc[i];
    for (int i = 0; i < 3; ++i) g.cam.v[i] = cam_center[i];
    g.fx = cam->fx;
    g.fy = cam->fy;
    g.cx = cam->cx;
    g.cy = cam->cy;
    g.width = cam->width;
    g.height = cam->height;
    const int64_t npix = cam->width * cam->height;
    if (npix <= 0) return TF_OK;
    // the first volume in order with a coloured cell wins: all volumes go in one launch
    if (nvol > TFB200_MAX_VOLUMES_PER_LAUNCH)
        return tf_set_error(TF_EINVAL, "tf_raycast_colors: more than %d volumes", TFB200_MAX_VOLUMES_PER_LAUNCH);
    VolumeTable vt{};
    vt.count = nvol;
    for (int v = 0; v < nvol; ++v) vt.vol[v] = vols[v];
    raycast_colors_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, (cudaStream_t)stream_>>>(vt, g, dist, colors);
    return tf_check_launch("raycast_colors_kernel");
}
