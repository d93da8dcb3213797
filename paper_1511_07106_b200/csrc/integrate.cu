// Projective TSDF integration, fused over many volumes (sm_100a).
//
// Replaces _kernels.integrate_kernel (reference _kernels.py:71-133).  Three
// launches per frame, all on the caller's stream:
//
//   1. frame_prep   — per pixel {depth, ray_scale} tables (ray_scale is a pure
//                     function of the rounded pixel, :118-120, so it is
//                     computed once per pixel instead of once per voxel): an
//                     exact float64 table and a float32 copy for screening,
//                     plus a max-depth mip over 16x16-pixel tiles for culling;
//   2. brick_cull   — one thread per 8^3 brick of every volume; a brick is
//                     dropped only when NO voxel in it can pass the
//                     reference's gates (behind the camera, projecting outside
//                     the image, no valid depth, or more than tau behind every
//                     depth it can see), with explicit rounding margins;
//   3. brick_update — persistent warps walk the surviving bricks.  Each voxel
//                     is first SCREENED in float32 with rigorous error bounds:
//                     its pixel is decided when u+0.5 / v+0.5 are not within
//                     the bound of an integer, and its class (skip / free
//                     space, i.e. sdf >= tau so the clamped value is exactly
//                     tau / near the surface) when the float32 sdf is not within
//                     the bound of +-tau.  Free-space voxels (the large
//                     majority) then need only the exact running-mean update;
//                     every undecided voxel runs the reference's full float64
//                     arithmetic (same op order, round-to-nearest intrinsics,
//                     float32 where numba types it float32).  Results are
//                     bit-identical to the exact path for every voxel
//                     (tests: TF_DEBUG_EXACT_ONLY and TF_DEBUG_NO_CULL runs).
//                     Voxel pairs move as 16-byte loads / stores and each
//                     thread keeps 8 voxels in flight to cover HBM latency.
//
// Work therefore scales with voxels near the camera frustum, not with n^3,
// and the only HBM traffic per voxel update is its 8-byte read + 8-byte write.
#include <math.h>

#include <cmath>

#include "tf_common.cuh"

#include <mutex>
#include <cuda.h>  // CUtensorMap (the encoder is fetched through cudaGetDriverEntryPoint)

namespace tf {

constexpr int kBrick = 8;         // brick edge in voxels
constexpr int kTile = 16;         // frame_prep block edge in pixels
constexpr int kCellShift = 2;     // finest depth-mip cell: 4x4 pixels (level l: 4 << l)
constexpr int kMaxMipLevels = 12;

struct MipDesc {
    int levels;
    int64_t tiles_x[kMaxMipLevels], tiles_y[kMaxMipLevels], offset[kMaxMipLevels];
    int64_t total;
};

struct BrickTable {
    int count;
    int64_t nb[TFB200_MAX_VOLUMES_PER_LAUNCH];            // bricks per axis
    int64_t offset[TFB200_MAX_VOLUMES_PER_LAUNCH + 1];    // prefix of nb^3
};

struct FrameGeom {
    Mat3 r_cw;
    Vec3 t_cw;
    Vec3 cam;
    double fx, fy, cx, cy;
    int64_t width, height;
    double tau, max_w, sw;
    double sw_tau;  // RN(sample_weight * tau): the free-space numerator term (:132)
    int unit_sw;    // sample_weight == 1 and max_weight finite: float32 weight path
    float max_w32;  // RN32(max_weight)
    // float32 copies for the conservative screen
    float r32[9];
    float fx32, fy32, cx32, cy32, tau32, w32, h32;
    float good_t;  // free-space summary threshold for this tau
    const uint8_t *rgb;  // colour frame (tf_integrate_rgb) or null
};

// brick summary maintained by this call for volume `vol`?
__device__ __forceinline__ bool keeps_summary(const TfVolume &vol, const FrameGeom &f) {
    return vol.brick_state_dev != nullptr && vol.summary_threshold == f.good_t;
}

// Bricks whose packed state changed this call: each listed once (dirty
// bitmap), so the flag pass visits only them and their lower neighbours.
struct ChangedList {
    uint32_t *list;
    unsigned *count;
    unsigned *dirty;
};

__device__ __forceinline__ void mark_changed(const ChangedList &c, unsigned g) {
    if (!c.list) return;
    const unsigned bit = 1u << (g & 31u);
    if (!(atomicOr(&c.dirty[g >> 5], bit) & bit)) c.list[atomicAdd(c.count, 1u)] = g;
}

__device__ __forceinline__ void summary_add(const TfVolume &vol, int64_t lin, unsigned delta) {
    const int64_t n = vol.n, nb = (n + 7) / 8;
    const int64_t x = lin % n, y = (lin / n) % n, z = lin / (n * n);
    atomicAdd(&vol.brick_state_dev[((z >> 3) * nb + (y >> 3)) * nb + (x >> 3)], delta);
}

static MipDesc make_mip(int64_t width, int64_t height) {
    MipDesc m{};
    int64_t off = 0;
    int l = 0;
    for (; l < kMaxMipLevels; ++l) {
        int64_t cell = (int64_t)1 << (kCellShift + l);
        m.tiles_x[l] = (width + cell - 1) / cell;
        m.tiles_y[l] = (height + cell - 1) / cell;
        m.offset[l] = off;
        off += m.tiles_x[l] * m.tiles_y[l];
        if (m.tiles_x[l] == 1 && m.tiles_y[l] == 1) {
            ++l;
            break;
        }
    }
    m.levels = l;
    m.total = off;
    return m;
}

// ---------------------------------------------------------------------------
// 1. pixel table + max-depth mip
// ---------------------------------------------------------------------------

// One 16x16 block per finest tile.  Depths are >= 0, so their IEEE bit
// patterns order like the values and the coarser levels use atomicMax on the
// bits (exact; order-independent).
// order-preserving float <-> uint32 keys (for atomicMin over signed floats)
__device__ __forceinline__ unsigned fkey(float f) {
    const unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float fkey_dec(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

__global__ void __launch_bounds__(256) frame_prep_kernel(
    const double *__restrict__ depth, double2 *__restrict__ table, float2 *__restrict__ table32,
    unsigned long long *__restrict__ mip, unsigned *__restrict__ qmip, const double tau,
    const MipDesc m, const double fx,
    const double fy, const double cx, const double cy, const int64_t width,
    const int64_t height, unsigned *__restrict__ zero_a, const int zero_a_words,
    unsigned *__restrict__ zero_b, const int64_t zero_b_words) {
    // the first chunk's brick / queue counters and dirty bitmap start at zero
    // (instead of two memsets before the culling)
    {
        const int64_t tid = ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * (kTile * kTile) +
                            threadIdx.y * kTile + threadIdx.x;
        const int64_t nthreads = (int64_t)gridDim.x * gridDim.y * (kTile * kTile);
        if (tid < zero_a_words) zero_a[tid] = 0u;
        for (int64_t i = tid; i < zero_b_words; i += nthreads) zero_b[i] = 0u;
    }
    const int64_t ui = (int64_t)blockIdx.x * kTile + threadIdx.x;
    const int64_t vi = (int64_t)blockIdx.y * kTile + threadIdx.y;
    double d = 0.0;
    // free-space key: q = (d - tau) * ray_scale rounded down, -inf without depth;
    // a voxel at distance dist seen through this pixel has sdf >= tau iff dist <= q
    unsigned qk = 0xffffffffu;
    if (ui < width && vi < height) {
        d = depth[vi * width + ui];
        // _kernels.py:118-120
        const double rx = ddiv(dsub((double)ui, cx), fx);
        const double ry = ddiv(dsub((double)vi, cy), fy);
        const double rs = dsqrt(dadd(dadd(dmul(rx, rx), dmul(ry, ry)), 1.0));
        table[vi * width + ui] = make_double2(d, rs);
        // screening copy: d32 > 0 exactly when d > 0 (tiny depths clamp up)
        const float d32 = d > 0.0 ? fmaxf(__double2float_rn(d), 1.17549435e-38f) : 0.0f;
        table32[vi * width + ui] = make_float2(d32, __double2float_rn(rs));
        qk = fkey(d > 0.0 ? __double2float_rd((d - tau) * rs) : -INFINITY);
    }
    // max-depth (IEEE bits of non-negative doubles order like the values) and
    // min free-space key mips: the cells of sizes 4, 8 and 16 px lie inside
    // this block and are written directly; coarser ones take atomics
    __shared__ unsigned long long sd[kTile * kTile];
    __shared__ unsigned sq[kTile * kTile];
    __shared__ unsigned long long cd[21];  // 16 + 4 + 1 in-block cells
    __shared__ unsigned cq[21];
    const int t = threadIdx.y * kTile + threadIdx.x;
    sd[t] = (unsigned long long)__double_as_longlong(d > 0.0 ? d : 0.0);
    sq[t] = qk;
    __syncthreads();
    if (t < 16) {  // 4x4-pixel cells
        const int ix = t & 3, iy = t >> 2;
        unsigned long long b = 0;
        unsigned q = 0xffffffffu;
        for (int yy = 0; yy < 4; ++yy)
            for (int xx = 0; xx < 4; ++xx) {
                const int s2 = (iy * 4 + yy) * kTile + ix * 4 + xx;
                b = sd[s2] > b ? sd[s2] : b;
                q = min(q, sq[s2]);
            }
        cd[t] = b;
        cq[t] = q;
    }
    __syncthreads();
    if (t < 4) {  // 8x8
        const int ix = t & 1, iy = t >> 1;
        unsigned long long b = 0;
        unsigned q = 0xffffffffu;
        for (int k = 0; k < 4; ++k) {
            const int c = (iy * 2 + (k >> 1)) * 4 + ix * 2 + (k & 1);
            b = cd[c] > b ? cd[c] : b;
            q = min(q, cq[c]);
        }
        cd[16 + t] = b;
        cq[16 + t] = q;
    }
    __syncthreads();
    if (t == 0) {  // 16x16
        unsigned long long b = 0;
        unsigned q = 0xffffffffu;
        for (int k = 0; k < 4; ++k) {
            b = cd[16 + k] > b ? cd[16 + k] : b;
            q = min(q, cq[16 + k]);
        }
        cd[20] = b;
        cq[20] = q;
    }
    __syncthreads();
    if (t < 21) {
        const int l = t < 16 ? 0 : (t < 20 ? 1 : 2);
        const int per = 4 >> l, k = t - (l == 0 ? 0 : (l == 1 ? 16 : 20));
        const int64_t gx = (int64_t)blockIdx.x * per + (k % per), gy = (int64_t)blockIdx.y * per + (k / per);
        if (l < m.levels && gx < m.tiles_x[l] && gy < m.tiles_y[l]) {
            mip[m.offset[l] + gy * m.tiles_x[l] + gx] = cd[t];
            qmip[m.offset[l] + gy * m.tiles_x[l] + gx] = cq[t];
        }
    }
    if (t == 0) {
        for (int l = 3; l < m.levels; ++l) {
            const int64_t tx = (int64_t)blockIdx.x >> (l - 2), ty = (int64_t)blockIdx.y >> (l - 2);
            if (tx >= m.tiles_x[l] || ty >= m.tiles_y[l]) break;
            atomicMax(&mip[m.offset[l] + ty * m.tiles_x[l] + tx], cd[20]);
            atomicMin(&qmip[m.offset[l] + ty * m.tiles_x[l] + tx], cq[20]);
        }
    }
}

// Max depth over the pixel rectangle [u0,u1]x[v0,v1] (inclusive), read from
// the coarsest-enough mip level so at most 4x4 cells are visited.  Conservative
// (cells cover a superset of the rectangle).
__device__ double rect_max_depth(const unsigned long long *__restrict__ mip, const MipDesc &m,
                                 int64_t u0, int64_t u1, int64_t v0, int64_t v1) {
    int l = 0;
    while (l + 1 < m.levels &&
           (((u1 >> (kCellShift + l)) - (u0 >> (kCellShift + l)) + 1) > 4 ||
            ((v1 >> (kCellShift + l)) - (v0 >> (kCellShift + l)) + 1) > 4))
        ++l;
    unsigned long long best = 0;
    const int64_t tx0 = u0 >> (kCellShift + l), tx1 = u1 >> (kCellShift + l);
    const int64_t ty0 = v0 >> (kCellShift + l), ty1 = v1 >> (kCellShift + l);
    for (int64_t ty = ty0; ty <= ty1; ++ty)
        for (int64_t tx = tx0; tx <= tx1; ++tx) {
            const unsigned long long b = __ldg(&mip[m.offset[l] + ty * m.tiles_x[l] + tx]);
            best = b > best ? b : best;
        }
    return __longlong_as_double((long long)best);
}

// Min of the free-space key over the pixel rectangle (same level choice as
// rect_max_depth; cells cover a superset, so the min is a lower bound).
__device__ float rect_min_q(const unsigned *__restrict__ qmip, const MipDesc &m, int64_t u0,
                            int64_t u1, int64_t v0, int64_t v1) {
    int l = 0;
    while (l + 1 < m.levels &&
           (((u1 >> (kCellShift + l)) - (u0 >> (kCellShift + l)) + 1) > 4 ||
            ((v1 >> (kCellShift + l)) - (v0 >> (kCellShift + l)) + 1) > 4))
        ++l;
    unsigned best = 0xffffffffu;
    for (int64_t ty = v0 >> (kCellShift + l); ty <= (v1 >> (kCellShift + l)); ++ty)
        for (int64_t tx = u0 >> (kCellShift + l); tx <= (u1 >> (kCellShift + l)); ++tx)
            best = min(best, __ldg(&qmip[m.offset[l] + ty * m.tiles_x[l] + tx]));
    return fkey_dec(best);
}

// ---------------------------------------------------------------------------
// 2. conservative brick culling
// ---------------------------------------------------------------------------

__device__ __forceinline__ int find_volume(const BrickTable &bt, int64_t g) {
    int v = 0;
    while (v + 1 < bt.count && g >= bt.offset[v + 1]) ++v;
    return v;
}

// Returns true when some voxel of the brick may pass every gate of
// _kernels.py:107-127.  Evaluated in float32 around a float64 brick origin;
// every comparison carries an explicit bound on the float32 error plus a wide
// safety factor, so a brick is dropped only if no voxel can be updated.
// Returns 0 (no voxel can update), 1 (some may) or 2 (every voxel certainly is
// a free-space update: in front of the camera, projecting inside the image
// onto pixels with depth, and closer than (d - tau) * ray_scale for every pixel
// its projection box covers -> sdf >= tau, clamped value exactly tau).
__device__ int box_may_update(const TfVolume &vol, const int64_t i0[3], const int64_t len[3],
                              const FrameGeom &f, const unsigned long long *__restrict__ mip,
                              const unsigned *__restrict__ qmip, const MipDesc &m, bool allow_free) {
    // the voxel box i0 .. i0 + len - 1 (clipped to the volume)
    const int64_t n = vol.n;
    double g0[3];
    float ext[3], gmin[3], gmax[3];
    float gabs = 0.f;
    for (int a = 0; a < 3; ++a) {
        const int64_t i1 = min(i0[a] + len[a] - 1, n - 1);
        // the reference's voxel centres (i + ht) * vs are monotone in i
        g0[a] = (double)(i0[a] + vol.origin[a]) * vol.voxel_size;
        const double g1 = (double)(i1 + vol.origin[a]) * vol.voxel_size;
        ext[a] = (float)(g1 - g0[a]);
        gmin[a] = (float)g0[a];
        gmax[a] = (float)g1;
        gabs += fmaxf(fabsf(gmin[a]), fabsf(gmax[a]));
    }
    const double *R = f.r_cw.m;
    float pc0[3];
    float pabs = 0.f;
    for (int r = 0; r < 3; ++r) {
        pc0[r] = (float)(R[3 * r] * g0[0] + R[3 * r + 1] * g0[1] + R[3 * r + 2] * g0[2] + f.t_cw.v[r]);
        pabs += fabsf(pc0[r]);
    }
    // float32 error of corner camera coordinates (origin rounding, column
    // products, three adds) — 2^-19 of the magnitudes is > 8x the true bound
    const float err = 1.9073486e-6f * (pabs + ext[0] + ext[1] + ext[2]) + 1e-30f;
    float zmin = 3e38f, zmax = -3e38f, xabs = 0.f, yabs = 0.f;
    float pcs[8][3];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const float e0 = (c & 1) ? ext[0] : 0.f, e1 = (c & 2) ? ext[1] : 0.f, e2 = (c & 4) ? ext[2] : 0.f;
#pragma unroll
        for (int r = 0; r < 3; ++r)
            pcs[c][r] = pc0[r] + f.r32[3 * r] * e0 + f.r32[3 * r + 1] * e1 + f.r32[3 * r + 2] * e2;
        zmin = fminf(zmin, pcs[c][2]);
        zmax = fmaxf(zmax, pcs[c][2]);
        xabs = fmaxf(xabs, fabsf(pcs[c][0]));
        yabs = fmaxf(yabs, fabsf(pcs[c][1]));
    }
    if (zmax < -2.f * err) return 0;  // every voxel has pcz <= 0 (:107)

    int64_t u0 = 0, u1 = f.width - 1, v0 = 0, v1 = f.height - 1;
    bool box_inside = false;  // projection box certainly inside the image
    if (zmin > 0.01f + 2.f * err) {
        // in front of the camera: all voxel projections lie inside the
        // projected corners' bounding box (convexity), up to rounding
        float umin = 3e38f, umax = -3e38f, vmin = 3e38f, vmax = -3e38f;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const float rz = 1.0f / pcs[c][2];
            const float u = f.fx32 * (pcs[c][0] * rz) + f.cx32;
            const float v = f.fy32 * (pcs[c][1] * rz) + f.cy32;
            umin = fminf(umin, u);
            umax = fmaxf(umax, u);
            vmin = fminf(vmin, v);
            vmax = fmaxf(vmax, v);
        }
        const float zl = zmin - 2.f * err;
        const float mu = f.fx32 * (2.f * err / zl) * (1.f + xabs / zl) * 1.5f +
                         3.8e-6f * (fabsf(umin) + fabsf(umax) + fabsf(f.cx32)) + 1e-3f;
        const float mv = f.fy32 * (2.f * err / zl) * (1.f + yabs / zl) * 1.5f +
                         3.8e-6f * (fabsf(vmin) + fabsf(vmax) + fabsf(f.cy32)) + 1e-3f;
        const float fu0 = floorf(umin - mu + 0.5f), fu1 = floorf(umax + mu + 0.5f);
        const float fv0 = floorf(vmin - mv + 0.5f), fv1 = floorf(vmax + mv + 0.5f);
        if (fu1 < 0.f || fv1 < 0.f || fu0 > f.w32 - 1.f || fv0 > f.h32 - 1.f)
            return 0;  // outside the image (:113)
        box_inside = fu0 >= 0.f && fv0 >= 0.f && fu1 <= f.w32 - 1.f && fv1 <= f.h32 - 1.f;
        u0 = fu0 < 0.f ? 0 : (int64_t)fu0;
        v0 = fv0 < 0.f ? 0 : (int64_t)fv0;
        u1 = fu1 > f.w32 - 1.f ? f.width - 1 : (int64_t)fu1;
        v1 = fv1 > f.h32 - 1.f ? f.height - 1 : (int64_t)fv1;
    }
    const float dmax = __double2float_ru(rect_max_depth(mip, m, u0, u1, v0, v1));
    if (!(dmax > 0.f)) return 0;  // no valid depth reachable (:116)

    // sdf = d - dist / ray_scale < -tau for every voxel (:125-127)?
    float dd2 = 0.f, cabs = 0.f;
    for (int a = 0; a < 3; ++a) {
        const float c = (float)f.cam.v[a];
        const float s = fmaxf(fmaxf(gmin[a] - c, c - gmax[a]), 0.f);
        dd2 += s * s;
        cabs += fabsf(c);
    }
    const float dist_lb = sqrtf(dd2) * (1.f - 1e-5f) - 1.9073486e-6f * (gabs + cabs);
    const float ax = fmaxf(fabsf((float)u0 - f.cx32), fabsf((float)u1 - f.cx32)) / f.fx32;
    const float ay = fmaxf(fabsf((float)v0 - f.cy32), fabsf((float)v1 - f.cy32)) / f.fy32;
    const float rs_ub = sqrtf(ax * ax + ay * ay + 1.f) * (1.f + 1e-5f);
    const float q_lb = dist_lb / rs_ub;
    const float margin = 1e-5f * (dmax + fabsf(q_lb) + f.tau32) + 1e-6f;
    if (dmax - q_lb < -f.tau32 - margin) return 0;
    if (allow_free && box_inside) {
        // farthest voxel (distance is convex: a corner) vs the smallest
        // (d - tau) * ray_scale over the box, with float32 margins
        float dd2max = 0.f;
        for (int c = 0; c < 8; ++c) {
            float q2 = 0.f;
            for (int a = 0; a < 3; ++a) {
                const float e = (((c >> a) & 1) ? gmax[a] : gmin[a]) - (float)f.cam.v[a];
                q2 += e * e;
            }
            dd2max = fmaxf(dd2max, q2);
        }
        const float dist_ub = sqrtf(dd2max) * 1.00002f + 3.8e-6f * (gabs + cabs) + 1e-6f;
        const float qmin = rect_min_q(qmip, m, u0, u1, v0, v1);
        if (qmin > 0.f && dist_ub <= qmin * 0.99998f) return 2;
    }
    return 1;
}

// box of span^3 bricks starting at brick (bx, by, bz)
__device__ __forceinline__ int brick_may_update(const TfVolume &vol, int64_t bx, int64_t by, int64_t bz,
                                                const FrameGeom &f, const unsigned long long *__restrict__ mip,
                                                const unsigned *__restrict__ qmip, const MipDesc &m,
                                                bool allow_free, int span = 1) {
    const int64_t i0[3] = {bx * kBrick, by * kBrick, bz * kBrick};
    const int64_t len[3] = {(int64_t)kBrick * span, (int64_t)kBrick * span, (int64_t)kBrick * span};
    return box_may_update(vol, i0, len, f, mip, qmip, m, allow_free);
}

// Stage 3: classes of every general brick's four 8x4x4 parts (part p = hy +
// 2 zh: y rows 4 hy .. 4 hy + 3, z layers 4 zh .. 4 zh + 3 — the general
// kernel's lane layout), one thread per part: part_class[4 k + p] =
// box_may_update of the part (0 no voxel can update, 1 maybe, 2 every voxel a
// free-space update).  The general kernel skips class-0 parts and streams
// class-2 parts without screening.
__global__ void __launch_bounds__(256) part_cull_kernel(
    const __grid_constant__ VolumeTable vt, const __grid_constant__ BrickTable bt,
    const __grid_constant__ FrameGeom f, const __grid_constant__ MipDesc m,
    const unsigned long long *__restrict__ mip, const unsigned *__restrict__ qmip,
    const uint32_t *__restrict__ active, const unsigned int *__restrict__ active_count,
    uint8_t *__restrict__ part_class, const int allow_free) {
    const unsigned total = *active_count * 4u;
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const unsigned g = active[t >> 2];
        const int p = (int)(t & 3u);
        const int v = find_volume(bt, g);
        const TfVolume &vol = vt.vol[v];
        const int64_t nb = bt.nb[v], local = (int64_t)g - bt.offset[v];
        const int64_t bx = local % nb, by = (local / nb) % nb, bz = local / (nb * nb);
        const int64_t i0[3] = {bx * kBrick, by * kBrick + 4 * (p & 1), bz * kBrick + 4 * (p >> 1)};
        const int64_t len[3] = {kBrick, 4, 4};
        int c = 0;
        if (i0[1] < vol.n && i0[2] < vol.n) c = box_may_update(vol, i0, len, f, mip, qmip, m, allow_free != 0);
        part_class[t] = (uint8_t)c;
    }
}

constexpr int kMacro = 4;  // macro cull box: 4^3 bricks = 32^3 voxels

// Stage 1: one thread per 32^3 macro box of every volume.  Culled macros
// drop their 64 bricks; certified free-space macros put all their bricks on
// the free list; the rest go to stage 2.
__global__ void __launch_bounds__(256) macro_cull_kernel(
    const __grid_constant__ VolumeTable vt, const __grid_constant__ BrickTable bt,
    const __grid_constant__ FrameGeom f, const __grid_constant__ MipDesc m,
    const unsigned long long *__restrict__ mip, const unsigned *__restrict__ qmip,
    uint32_t *__restrict__ macros, unsigned int *__restrict__ macro_count,
    uint32_t *__restrict__ active_free, unsigned int *__restrict__ free_count, const int no_cull,
    const int allow_free) {
    // macro index space: volume v owns nm(v)^3 macros after mfirst(v)
    int64_t mfirst[TFB200_MAX_VOLUMES_PER_LAUNCH + 1];
    mfirst[0] = 0;
    for (int v = 0; v < bt.count; ++v) {
        const int64_t nm = (bt.nb[v] + kMacro - 1) / kMacro;
        mfirst[v + 1] = mfirst[v] + nm * nm * nm;
    }
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int kind = 0;
    int v = 0;
    int64_t mx = 0, my = 0, mz = 0, nm = 1;
    if (g < mfirst[bt.count]) {
        while (g >= mfirst[v + 1]) ++v;
        nm = (bt.nb[v] + kMacro - 1) / kMacro;
        const int64_t local = g - mfirst[v];
        mx = local % nm;
        my = (local / nm) % nm;
        mz = local / (nm * nm);
        kind = brick_may_update(vt.vol[v], mx * kMacro, my * kMacro, mz * kMacro, f, mip, qmip, m,
                                allow_free != 0, kMacro);
        if (no_cull && kind == 0) kind = 1;
    }
    if (kind == 2) {  // every brick of the macro is certified free space
        const int64_t nb = bt.nb[v];
        unsigned cnt = 0;
        uint32_t ids[kMacro * kMacro * kMacro];
        for (int k = 0; k < kMacro * kMacro * kMacro; ++k) {
            const int64_t bx = mx * kMacro + (k & 3), by = my * kMacro + ((k >> 2) & 3),
                          bz = mz * kMacro + (k >> 4);
            if (bx < nb && by < nb && bz < nb) ids[cnt++] = (uint32_t)(bt.offset[v] + (bz * nb + by) * nb + bx);
        }
        const unsigned base = atomicAdd(free_count, cnt);
        for (unsigned k = 0; k < cnt; ++k) active_free[base + k] = ids[k];
        if (vt.vol[v].counters_dev) atomicAdd((unsigned long long *)&vt.vol[v].counters_dev[1], (unsigned long long)cnt);
    }
    const int lane = threadIdx.x & 31;
    const unsigned mg = __ballot_sync(0xffffffffu, kind == 1);
    if (mg) {
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(macro_count, (unsigned)__popc(mg));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (kind == 1) macros[base + __popc(mg & ((1u << lane) - 1u))] = (uint32_t)g;
    }
}

// Stage 2: one thread per brick of every surviving macro (grid-stride).
__global__ void __launch_bounds__(256) brick_cull_kernel(
    const __grid_constant__ VolumeTable vt, const __grid_constant__ BrickTable bt,
    const __grid_constant__ FrameGeom f, const __grid_constant__ MipDesc m,
    const unsigned long long *__restrict__ mip, const unsigned *__restrict__ qmip,
    const uint32_t *__restrict__ macros, const unsigned int *__restrict__ macro_count,
    uint32_t *__restrict__ active, unsigned int *__restrict__ active_count,
    uint32_t *__restrict__ active_free, unsigned int *__restrict__ free_count, const int no_cull,
    const int allow_free) {
    int64_t mfirst[TFB200_MAX_VOLUMES_PER_LAUNCH + 1];
    mfirst[0] = 0;
    for (int v = 0; v < bt.count; ++v) {
        const int64_t nm = (bt.nb[v] + kMacro - 1) / kMacro;
        mfirst[v + 1] = mfirst[v] + nm * nm * nm;
    }
    const unsigned total = *macro_count * (kMacro * kMacro * kMacro);
    const int lane = threadIdx.x & 31;
    for (unsigned t0 = blockIdx.x * blockDim.x; t0 < total; t0 += gridDim.x * blockDim.x) {
        const unsigned t = t0 + threadIdx.x;
        int kind = 0, vol_of = 0;
        uint32_t gb = 0;
        if (t < total) {
            const int64_t gm = macros[t >> 6];
            const int sub = t & 63;
            int v = 0;
            while (gm >= mfirst[v + 1]) ++v;
            vol_of = v;
            const int64_t nb = bt.nb[v], nm = (nb + kMacro - 1) / kMacro, local = gm - mfirst[v];
            const int64_t bx = (local % nm) * kMacro + (sub & 3), by = ((local / nm) % nm) * kMacro + ((sub >> 2) & 3),
                          bz = (local / (nm * nm)) * kMacro + (sub >> 4);
            if (bx < nb && by < nb && bz < nb) {
                gb = (uint32_t)(bt.offset[v] + (bz * nb + by) * nb + bx);
                kind = brick_may_update(vt.vol[v], bx, by, bz, f, mip, qmip, m, allow_free != 0);
                if (no_cull && kind == 0) kind = 1;
            }
        }
        // per-volume work counters (ownership balance): one atomic per volume
        // present in the warp
        {
            const unsigned peers = __match_any_sync(0xffffffffu, kind ? vol_of : -1);
            if (kind && vt.vol[vol_of].counters_dev) {
                const unsigned g1 = __ballot_sync(peers, kind == 1) & peers, g2 = peers & ~g1;
                if (lane == __ffs(peers) - 1) {
                    if (g1) atomicAdd((unsigned long long *)&vt.vol[vol_of].counters_dev[0], (unsigned long long)__popc(g1));
                    if (g2) atomicAdd((unsigned long long *)&vt.vol[vol_of].counters_dev[1], (unsigned long long)__popc(g2));
                }
            }
        }
        // warp-aggregated appends (list order is irrelevant: voxels are independent)
        const unsigned mg = __ballot_sync(0xffffffffu, kind == 1), mf = __ballot_sync(0xffffffffu, kind == 2);
        if (mg) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(active_count, (unsigned)__popc(mg));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (kind == 1) active[base + __popc(mg & ((1u << lane) - 1u))] = gb;
        }
        if (mf) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(free_count, (unsigned)__popc(mf));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (kind == 2) active_free[base + __popc(mf & ((1u << lane) - 1u))] = gb;
        }
    }
}

__device__ __forceinline__ float2 free_update(float2 old, const FrameGeom &f, const double2 *rcp);
__device__ __forceinline__ void fill_rcp(double2 *rcp);
__device__ __forceinline__ unsigned free_state_delta(float2 old, float2 nv, float t);

// Certified free-space bricks: every voxel gets the clamped-to-tau running
// mean (_kernels.py:128-133 with clamped == tau).  Pure streaming: 16-byte
// voxel pairs, four lanes per 64-byte row, eight rows per warp instruction,
// four rows' loads in flight per lane.
// One certified free-space brick (global brick id g) by one warp.
__device__ __forceinline__ void free_brick(const VolumeTable &vt, const BrickTable &bt, const FrameGeom &f,
                                           const unsigned g, const int lane, const int fixed_point,
                                           const double2 *rcp, const ChangedList &changed,
                                           unsigned &updates, unsigned &nop) {
    const float2 fixed = make_float2(f.tau32, (float)f.max_w);
    const int vi = find_volume(bt, g);
    const TfVolume &vol = vt.vol[vi];
    const unsigned n = (unsigned)vol.n, nb = (unsigned)bt.nb[vi];
    const unsigned local = g - (unsigned)bt.offset[vi];
    const unsigned x = (local % nb) * kBrick + 2 * (lane & 3);
    const unsigned y0 = ((local / nb) % nb) * kBrick, z0 = (local / (nb * nb)) * kBrick;
    float2 *vox = (float2 *)vol.voxels_dev;
    const bool keep = keeps_summary(vol, f);
    unsigned dbad = 0;
    if ((n & 1u) == 0u && n - z0 >= (unsigned)kBrick && n - y0 >= (unsigned)kBrick &&
        n - (x - 2 * (lane & 3)) >= (unsigned)kBrick) {
        // interior brick, even n: 16-byte pairs, never split
#pragma unroll 1
        for (int h = 0; h < 8; h += 4) {
            float4 o[4];
            size_t lin[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const unsigned r = (unsigned)(lane >> 2) + 8u * (h + k);  // row = y + 8 z
                lin[k] = ((size_t)(z0 + (r >> 3)) * n + (y0 + (r & 7u))) * n + x;
                if (!TF_IN_BOUNDS(lin[k] + 1 < (size_t)n * n * n)) lin[k] = 0;
                o[k] = *reinterpret_cast<const float4 *>(vox + lin[k]);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 a = make_float2(o[k].x, o[k].y), b = make_float2(o[k].z, o[k].w);
                const bool na = fixed_point && a.x == fixed.x && a.y == fixed.y;
                const bool nbq = fixed_point && b.x == fixed.x && b.y == fixed.y;
                updates += 2;
                nop += (na ? 1u : 0u) + (nbq ? 1u : 0u);
                if (na && nbq) continue;  // provably unchanged (host-verified fixed point)
                const float2 ua = na ? a : free_update(a, f, rcp);
                const float2 ub = nbq ? b : free_update(b, f, rcp);
                if (keep) dbad += free_state_delta(a, ua, f.good_t) + free_state_delta(b, ub, f.good_t);
                *reinterpret_cast<float4 *>(vox + lin[k]) = make_float4(ua.x, ua.y, ub.x, ub.y);
            }
        }
    } else {
        // edge brick or odd n: per voxel
#pragma unroll 1
        for (int it = 0; it < 8; ++it) {
            const unsigned r = (unsigned)(lane >> 2) + 8u * it;
            const unsigned y = y0 + (r & 7u), z = z0 + (r >> 3);
            if (y >= n || z >= n) continue;
            for (unsigned xx = x; xx < x + 2 && xx < n; ++xx) {
                const size_t lin = ((size_t)z * n + y) * n + xx;
                if (!TF_IN_BOUNDS(lin < (size_t)n * n * n)) continue;
                const float2 a = vox[lin];
                ++updates;
                if (fixed_point && a.x == fixed.x && a.y == fixed.y) {
                    ++nop;
                    continue;
                }
                const float2 ua = free_update(a, f, rcp);
                if (keep) dbad += free_state_delta(a, ua, f.good_t);
                vox[lin] = ua;
            }
        }
    }
    if (keep) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dbad += __shfl_xor_sync(0xffffffffu, dbad, o);
        if (lane == 0 && dbad) {
            atomicAdd(&vol.brick_state_dev[local], dbad);
            mark_changed(changed, g);
        }
    }
}

// Certified free-space bricks: every voxel gets the clamped-to-tau running
// mean (_kernels.py:128-133 with clamped == tau).  Pure streaming: 16-byte
// voxel pairs, four lanes per 64-byte row, eight rows per warp instruction,
// four rows' loads in flight per lane.
__global__ void __launch_bounds__(256, 4) brick_free_kernel(
    const __grid_constant__ VolumeTable vt, const __grid_constant__ BrickTable bt,
    const __grid_constant__ FrameGeom f, const uint32_t *__restrict__ list,
    const unsigned int *__restrict__ list_count, const int fixed_point,
    unsigned long long *__restrict__ stats, const ChangedList changed) {
    __shared__ double2 rcp[257];
    fill_rcp(rcp);
    const unsigned count = *list_count;
    const int lane = threadIdx.x & 31;
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
    unsigned updates = 0, nop = 0;
    unsigned g_next = warp < count ? list[warp] : 0u;  // next brick id, loaded one brick ahead
    for (unsigned i = warp; i < count; i += nwarps) {
        const unsigned g = g_next;
        if (i + nwarps < count) g_next = list[i + nwarps];
        free_brick(vt, bt, f, g, lane, fixed_point, rcp, changed, updates, nop);
    }
    if (stats) {
        warp_count_add(&stats[TF_STAT_VOXEL_UPDATES], updates);
        warp_count_add(&stats[TF_STAT_FREE_KERNEL_UPDATES], updates);
        warp_count_add(&stats[TF_STAT_SWEPT_VOXELS], updates);
        warp_count_add(&stats[TF_STAT_NOOP_UPDATES], nop);
    }
}

// ---- the same, staged through shared memory by TMA (TFB200_FREE_TMA=1) ----
//
// Each warp double-buffers its bricks: while it updates brick i from shared
// memory, the tensor-memory accelerator already brings brick i + nwarps
// (one 8x8x8 box of 8-byte voxels, 4 KB, cp.async.bulk.tensor.3d against a
// per-volume tensor map; completion counted on an mbarrier) — 4 KB in flight
// per warp without a register per byte.  Edge bricks and odd n take
// free_brick().  Measured (config 3, A/B): update bracket 0.167 vs 0.160 ms
// for the register-staged kernel above, and 0.201 ms with 64 row-sized 1-D
// bulk copies per brick instead of the box — so it is not the default.

__device__ __forceinline__ unsigned smem_addr(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)), "r"(parity)
        : "memory");
}

struct FreeBrickPos {
    int vi;
    unsigned n, local, x0, y0, z0;
};

__device__ __forceinline__ FreeBrickPos free_brick_pos(const BrickTable &bt, const VolumeTable &vt, unsigned g) {
    FreeBrickPos b;
    b.vi = find_volume(bt, g);
    b.n = (unsigned)vt.vol[b.vi].n;
    const unsigned nb = (unsigned)bt.nb[b.vi];
    b.local = g - (unsigned)bt.offset[b.vi];
    b.x0 = (b.local % nb) * kBrick;
    b.y0 = ((b.local / nb) % nb) * kBrick;
    b.z0 = (b.local / (nb * nb)) * kBrick;
    return b;
}

__device__ __forceinline__ bool free_brick_stageable(const FreeBrickPos &b) {
    return (b.n & 1u) == 0u && b.n - b.z0 >= (unsigned)kBrick && b.n - b.y0 >= (unsigned)kBrick &&
           b.n - b.x0 >= (unsigned)kBrick;
}

// one tensor map per volume of the launch: the voxels as an n^3 box of
// 8-byte elements, loaded in 8^3 boxes (one brick, 4 KB, x fastest)
struct alignas(64) BrickMaps {
    CUtensorMap m[TFB200_MAX_VOLUMES_PER_LAUNCH];
};

// the brick's 64 rows (y + 8 z) of 64 bytes into buf: one TMA box load,
// issued and armed by lane 0
__device__ __forceinline__ void free_brick_issue(const BrickMaps &maps, const FreeBrickPos &b, int lane,
                                                 unsigned char *buf, uint64_t *bar) {
    if (lane != 0) return;
    mbar_expect_tx(bar, 64u * 64u);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(buf)),
        "l"(reinterpret_cast<uint64_t>(&maps.m[b.vi])), "r"((int)b.x0), "r"((int)b.y0), "r"((int)b.z0),
        "r"(smem_addr(bar))
        : "memory");
}

// free_brick's interior path with the old values read from the staged rows
__device__ __forceinline__ void free_brick_staged(const VolumeTable &vt, const FrameGeom &f, const FreeBrickPos &b,
                                                  unsigned g, int lane, int fixed_point, const double2 *rcp,
                                                  const ChangedList &changed, const unsigned char *buf,
                                                  unsigned &updates, unsigned &nop) {
    const float2 fixed = make_float2(f.tau32, (float)f.max_w);
    const TfVolume &vol = vt.vol[b.vi];
    float2 *vox = (float2 *)vol.voxels_dev;
    const bool keep = keeps_summary(vol, f);
    const unsigned x = b.x0 + 2 * (lane & 3);
    unsigned dbad = 0;
#pragma unroll 2
    for (int k = 0; k < 8; ++k) {
        const unsigned r = (unsigned)(lane >> 2) + 8u * k;  // row = y + 8 z
        const float4 o = *reinterpret_cast<const float4 *>(buf + 64u * r + 16u * (lane & 3));
        const size_t lin = ((size_t)(b.z0 + (r >> 3)) * b.n + (b.y0 + (r & 7u))) * b.n + x;
        const float2 a = make_float2(o.x, o.y), c = make_float2(o.z, o.w);
        const bool na = fixed_point && a.x == fixed.x && a.y == fixed.y;
        const bool nc = fixed_point && c.x == fixed.x && c.y == fixed.y;
        updates += 2;
        nop += (na ? 1u : 0u) + (nc ? 1u : 0u);
        if (na && nc) continue;  // provably unchanged (host-verified fixed point)
        const float2 ua = na ? a : free_update(a, f, rcp);
        const float2 uc = nc ? c : free_update(c, f, rcp);
        if (keep) dbad += free_state_delta(a, ua, f.good_t) + free_state_delta(c, uc, f.good_t);
        if (TF_IN_BOUNDS(lin + 1 < (size_t)b.n * b.n * b.n))
            *reinterpret_cast<float4 *>(vox + lin) = make_float4(ua.x, ua.y, uc.x, uc.y);
    }
    if (keep) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dbad += __shfl_xor_sync(0xffffffffu, dbad, o);
        if (lane == 0 && dbad) {
            atomicAdd(&vol.brick_state_dev[b.local], dbad);
            mark_changed(changed, g);
        }
    }
}

constexpr int kFreeTmaWarps = 8;

__global__ void __launch_bounds__(256, 3) brick_free_tma_kernel(
    const __grid_constant__ VolumeTable vt, const __grid_constant__ BrickTable bt,
    const __grid_constant__ FrameGeom f, const __grid_constant__ BrickMaps maps, const uint32_t *__restrict__ list,
    const unsigned int *__restrict__ list_count, const int fixed_point,
    unsigned long long *__restrict__ stats, const ChangedList changed) {
    extern __shared__ __align__(128) unsigned char stage_mem[];  // [warp][2][4096]
    __shared__ __align__(8) uint64_t bars[kFreeTmaWarps][2];
    __shared__ double2 rcp[257];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        mbar_init(&bars[w][0], 1);
        mbar_init(&bars[w][1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fill_rcp(rcp);  // (its __syncthreads also publishes the barriers)
    unsigned char *buf[2] = {stage_mem + (size_t)w * 8192u, stage_mem + (size_t)w * 8192u + 4096u};
    const unsigned count = *list_count;
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
    unsigned updates = 0, nop = 0;
    unsigned phase[2] = {0u, 0u};
    int stage = 0;
    FreeBrickPos cur{};
    unsigned gcur = 0;
    bool cur_staged = false;
    if (warp < count) {
        gcur = list[warp];
        cur = free_brick_pos(bt, vt, gcur);
        cur_staged = free_brick_stageable(cur);
        if (cur_staged) free_brick_issue(maps, cur, lane, buf[0], &bars[w][0]);
    }
    for (unsigned i = warp; i < count; i += nwarps) {
        // prefetch the warp's next brick into the other stage (its previous
        // contents were consumed in the last iteration: every lane's reads
        // are ordered before the copy by the warp barrier + proxy fence)
        FreeBrickPos nxt{};
        unsigned gnext = 0;
        bool next_staged = false;
        if (i + nwarps < count) {
            gnext = list[i + nwarps];
            nxt = free_brick_pos(bt, vt, gnext);
            next_staged = free_brick_stageable(nxt);
            if (next_staged) {
                __syncwarp();
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                free_brick_issue(maps, nxt, lane, buf[stage ^ 1], &bars[w][stage ^ 1]);
            }
        }
        if (cur_staged) {
            mbar_wait(&bars[w][stage], phase[stage]);
            phase[stage] ^= 1u;
            free_brick_staged(vt, f, cur, gcur, lane, fixed_point, rcp, changed, buf[stage], updates, nop);
        } else {
            free_brick(vt, bt, f, gcur, lane, fixed_point, rcp, changed, updates, nop);
        }
        cur = nxt;
        gcur = gnext;
        cur_staged = next_staged;
        stage ^= 1;
    }
    if (stats) {
        warp_count_add(&stats[TF_STAT_VOXEL_UPDATES], updates);
        warp_count_add(&stats[TF_STAT_FREE_KERNEL_UPDATES], updates);
        warp_count_add(&stats[TF_STAT_SWEPT_VOXELS], updates);
        warp_count_add(&stats[TF_STAT_NOOP_UPDATES], nop);
    }
}

// ---------------------------------------------------------------------------
// 3. exact per-voxel update over the surviving bricks
// ---------------------------------------------------------------------------

// _kernels.py:99-133 for one voxel; returns 1 when the voxel was written.
__device__ __forceinline__ int update_voxel(float2 *__restrict__ vox, int64_t lin, double gx,
                                            double gy, double gz,
                                            const double2 *__restrict__ table,
                                            const FrameGeom &f, unsigned *dbad = nullptr,
                                            uint8_t *color = nullptr, const float2 *old_in = nullptr) {
    const double *R = f.r_cw.m;
    const double pcx = dot3_plus(R[0], gx, R[1], gy, R[2], gz, f.t_cw.v[0]);  // :104
    const double pcy = dot3_plus(R[3], gx, R[4], gy, R[5], gz, f.t_cw.v[1]);  // :105
    const double pcz = dot3_plus(R[6], gx, R[7], gy, R[8], gz, f.t_cw.v[2]);  // :106
    if (!(pcz > 0.0)) return 0;                                                 // :107
    const double u = dadd(ddiv(dmul(f.fx, pcx), pcz), f.cx);                     // :109
    const double v = dadd(ddiv(dmul(f.fy, pcy), pcz), f.cy);                     // :110
    const double uf = floor(dadd(u, 0.5)), vf = floor(dadd(v, 0.5));            // :111-112
    if (!(uf >= 0.0 && uf < (double)f.width && vf >= 0.0 && vf < (double)f.height))
        return 0;                                                               // :113
    if (!TF_IN_BOUNDS((int64_t)vf * f.width + (int64_t)uf < f.width * f.height)) return 0;
    const double2 px = __ldg(&table[(int64_t)vf * f.width + (int64_t)uf]);
    const double d = px.x;                                                      // :115
    if (!(d > 0.0)) return 0;                                                   // :116
    const double ddx = dsub(gx, f.cam.v[0]), ddy = dsub(gy, f.cam.v[1]),
                 ddz = dsub(gz, f.cam.v[2]);                                    // :121-123
    const double dist = dsqrt(dadd(dadd(dmul(ddx, ddx), dmul(ddy, ddy)), dmul(ddz, ddz)));
    const double sdf = dsub(d, ddiv(dist, px.y));                               // :125
    if (sdf < -f.tau) return 0;                                                 // :126
    const double clamped = sdf < f.tau ? sdf : f.tau;                           // :128
    const float2 old = old_in ? *old_in : vox[lin];
    // numba types float(f32) as float32: the product is a float32 op (:129-132)
    const float wv = fmulr(old.y, old.x);
    const double w_sum = dadd((double)old.y, f.sw);                             // :131
    const double t_new = ddiv(dadd((double)wv, dmul(f.sw, clamped)), w_sum);    // :132
    const double w_new = f.max_w < w_sum ? f.max_w : w_sum;                     // :133
    const float2 nv = make_float2(__double2float_rn(t_new), __double2float_rn(w_new));
    vox[lin] = nv;
    if (dbad) *dbad = voxel_state(nv, f.good_t) - voxel_state(old, f.good_t);
    if (color && f.rgb && sdf < f.tau) {
        // colour running mean while in the truncation band (tfb200.h, tf_integrate_rgb)
        uchar4 *cp = reinterpret_cast<uchar4 *>(color) + lin;
        const uchar4 c = *cp;
        const uint8_t *o = f.rgb + 3 * ((int64_t)vf * f.width + (int64_t)uf);
        const float w = (float)c.w, w1 = w + 1.0f;
        uchar4 nc;
        nc.x = (unsigned char)rintf(__fdiv_rn(__fadd_rn(__fmul_rn(w, (float)c.x), (float)o[0]), w1));
        nc.y = (unsigned char)rintf(__fdiv_rn(__fadd_rn(__fmul_rn(w, (float)c.y), (float)o[1]), w1));
        nc.z = (unsigned char)rintf(__fdiv_rn(__fadd_rn(__fmul_rn(w, (float)c.z), (float)o[2]), w1));
        nc.w = c.w == 255 ? 255 : (unsigned char)(c.w + 1);
        *cp = nc;
    }
    return 1;
}

// Reference-order exact update of every voxel of every surviving brick
// (TF_DEBUG_EXACT_ONLY; the fast kernel below must match it bit for bit).
__global__ void __launch_bounds__(256) brick_update_exact_kernel(
    const __grid_constant__ VolumeTable vt, const __grid_constant__ BrickTable bt,
    const __grid_constant__ FrameGeom f, const double2 *__restrict__ table,
    const uint32_t *__restrict__ active, const unsigned int *__restrict__ active_count,
    unsigned long long *__restrict__ stats) {
    const unsigned count = *active_count;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long updates = 0, swept = 0;
    // lane -> (x, y) inside an 8x4 slab of the brick; the warp covers x-rows of
    // 8 consecutive voxels (64 contiguous bytes each)
    const int lx = lane & 7, ly = lane >> 3;
    for (int64_t i = warp; i < count; i += nwarps) {
        const int64_t g = active[i];
        const int vi = find_volume(bt, g);
        const TfVolume vol = vt.vol[vi];
        const int64_t n = vol.n, nb = bt.nb[vi], local = g - bt.offset[vi];
        const int64_t x = (local % nb) * kBrick + lx;
        const int64_t y0 = ((local / nb) % nb) * kBrick + ly;
        const int64_t z0 = (local / (nb * nb)) * kBrick;
        float2 *vox = (float2 *)vol.voxels_dev;
        const double vs = vol.voxel_size;
        const double gx = dmul((double)(x + vol.origin[0]), vs);                // :103
        for (int hy = 0; hy < 2; ++hy) {
            const int64_t y = y0 + 4 * hy;
            const double gy = dmul((double)(y + vol.origin[1]), vs);            // :101
            for (int iz = 0; iz < kBrick; ++iz) {
                const int64_t z = z0 + iz;
                if (x < n && y < n && z < n) {
                    const double gz = dmul((double)(z + vol.origin[2]), vs);    // :99
                    swept += 1;
                    unsigned db = 0;
                    const int64_t lin = vox_index(n, z, y, x);
                    updates += update_voxel(vox, lin, gx, gy, gz, table, f, &db, vol.color_dev);
                    if (db && keeps_summary(vol, f)) summary_add(vol, lin, db);
                }
            }
        }
    }
    if (stats) {
        warp_count_add(&stats[TF_STAT_VOXEL_UPDATES], updates);
        warp_count_add(&stats[TF_STAT_SWEPT_VOXELS], swept);
    }
    (void)lane;
}


// out-of-line copy for the rare queue-overflow path of the fast kernel
__device__ __noinline__ int update_voxel_slow(float2 *__restrict__ vox, int64_t lin, double gx,
                                              double gy, double gz,
                                              const double2 *__restrict__ table,
                                              const FrameGeom &f, unsigned *dbad, uint8_t *color) {
    return update_voxel(vox, lin, gx, gy, gz, table, f, dbad, color);
}

// ---- float32 screening ------------------------------------------------------
//
// For each voxel the screen either decides exactly what the reference's float64
// arithmetic decides, or defers the voxel to the exact kernel.  Bounds:
//  * camera coordinates pc are float32 around a float64 column base, with
//    |error| <= epc (2^-20 of the magnitudes: > 8x the real bound);
//  * u + 0.5 = fx * pcx * rcp(pcz) + (cx + 0.5) with rcp.approx (rel. error
//    <= 2^-22), |error| <= du, a per-batch bound computed from the batch's
//    smallest pcz and largest |pcx|; a voxel whose u + 0.5 lies within du of an
//    integer is deferred (~0.1% of voxels), otherwise floor() is exact;
//  * sdf = d - dist / rs is compared against +-tau through squared distances
//    with 1e-5 relative and explicit absolute margins; only voxels in the
//    +-tau band (near the surface) are deferred.

enum : int { kSkip = 0, kFree = 1, kExact = 2 };

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

struct ScreenConst {
    float tau_ea;     // tau + float32 rounding allowance of d and tau
    float fxh, fyh;   // fx, fy
    float cxh, cyh;   // cx + 0.5, cy + 0.5
};

// packed-state change of a free-space update old -> nv (nv.y > 0 always)
__device__ __forceinline__ unsigned free_state_delta(float2 old, float2 nv, float t) {
    const unsigned was_obs = old.y > 0.0f ? 1u : 0u;
    const unsigned old_bad = (was_obs && old.x >= t) ? 0u : 1u;
    const unsigned new_bad = nv.x >= t ? 0u : 1u;
    return (new_bad - old_bad) + ((1u - was_obs) << 16);
}

// a / b correctly rounded for the running-mean denominator b = w + sw.  When
// b is an integer in [1, 256] (integral weights, the reference default), one
// multiplication by RN(1/b) from a per-block table and one fused correction:
// q = RN(a r), e = a - q b (exact with FMA), RN(q + e r) — Markstein's
// theorem (r within 1/2 ulp of 1/b, q within 1 ulp of a/b) makes the result
// RN(a / b), the IEEE quotient, as long as nothing underflows (|a| >= 2^-900
// guards that).  Any other b takes the IEEE division.  Checked against
// __ddiv_rn by tf_debug_weight_division_check (GPU test).
__device__ __forceinline__ double div_weight(double a, double b, const double2 *__restrict__ rcp) {
    const int bi = __double2int_rz(b);
    if (bi >= 1 && bi <= 256 && (double)bi == b && fabs(a) >= 0x1p-900) {
        const double r = rcp[bi].x;
        const double q = dmul(a, r);
        const double e = __fma_rn(-q, b, a);
        return __fma_rn(e, r, q);
    }
    return ddiv(a, b);
}

// RN(1/b) for b = 1..256, evaluated at compile time (IEEE division, correctly
// rounded; entry 0 unused).  Computing it per block with __drcp_rn cost ~10 %
// of the update kernel's stall samples (block start-up behind a barrier).
struct RcpTable {
    double v[257];
    constexpr RcpTable() : v{} {
        for (int b = 1; b <= 256; ++b) v[b] = 1.0 / (double)b;
    }
};
__device__ const RcpTable g_rcp_table = RcpTable();

// {RN(1/b), b} into shared memory; every thread of the block must call it
__device__ __forceinline__ void fill_rcp(double2 *rcp) {
    for (int b = threadIdx.x; b <= 256; b += blockDim.x) rcp[b] = make_double2(g_rcp_table.v[b], (double)b);
    __syncthreads();
}

// running weighted mean with clamped == tau (_kernels.py:129-133)
__device__ __forceinline__ float2 free_update(float2 old, const FrameGeom &f, const double2 *rcp) {
    const float wv = fmulr(old.y, old.x);
    if (f.unit_sw) {
        // sample_weight 1 and an integral weight w in [0, 255]: w + 1 is exact
        // in float32, so the float64 weight sum, its integer test and
        // RN32(min(max_w, w + 1)) = min(RN32(max_w), w + 1) need no float64
        // conversions; the quotient is div_weight's (same operations).
        // m = 2^23 + w for integral 0 <= w < 2^23: its low bits index the table.
        const float m = __fadd_rn(old.y, 8388608.0f);
        if (old.y >= 0.0f && old.y <= 255.0f && __fsub_rn(m, 8388608.0f) == old.y) {
            const double2 rb = rcp[__float_as_uint(m) - 0x4AFFFFFFu];  // {RN(1/(w+1)), w+1}
            const double a = dadd((double)wv, f.sw_tau);
            if (fabs(a) >= 0x1p-900) {
                const double q = dmul(a, rb.x);
                const double t = __fma_rn(__fma_rn(-q, rb.y, a), rb.x, q);
                return make_float2(__double2float_rn(t), fminf(__fadd_rn(old.y, 1.0f), f.max_w32));
            }
        }
    }
    const double w_sum = dadd((double)old.y, f.sw);
    const double t_new = div_weight(dadd((double)wv, f.sw_tau), w_sum, rcp);
    const double w_new = f.max_w < w_sum ? f.max_w : w_sum;
    return make_float2(__double2float_rn(t_new), __double2float_rn(w_new));
}

// test hook: random (a, b) pairs through div_weight vs __ddiv_rn
__global__ void weight_division_check_kernel(int64_t n, unsigned long long seed, unsigned long long *mismatches) {
    __shared__ double2 rcp[257];
    fill_rcp(rcp);
    unsigned long long bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long x = seed ^ (0x9E3779B97F4A7C15ull * (unsigned long long)(i + 1));
        x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 33;
        const double b = (double)(1 + (x & 255u));
        // a: random 52-bit mantissa, exponent in [-40, 12), random sign
        const int ex = (int)((x >> 8) % 52u) - 40;
        const unsigned long long m = (x >> 14) | 0x10000000000000ull;
        double a = ldexp((double)(m & 0x1FFFFFFFFFFFFFull), ex - 52);
        if (x & (1ull << 63)) a = -a;
        const double got = div_weight(a, b, rcp), want = __ddiv_rn(a, b);
        bad += __double_as_longlong(got) != __double_as_longlong(want);
    }
    if (bad) atomicAdd(mismatches, bad);
}

constexpr int kZBatch = 4;  // voxels in flight per thread

// Lane layout per warp and brick: x = lane & 7, y = lane >> 3 (+4 for the
// second half); each lane walks its (x, y) column's 8 z voxels in two
// batches, so a warp instruction touches four 64-byte rows.  Column-level
// work (float64 base, error bounds, whole-column rejection) is amortised over
// the column; per voxel the screen is ~25 float32 instructions.
//
// kClassify: the screen alone.  No voxel is read or written: the decisions
// depend only on the frame (depth tables) and the geometry, so this runs in
// tf_integrate_prepare, next to the previous frame's raycast.  Each lane
// stores one word per brick (masks[32 i + lane]): bit hy*8 + z = a
// free-space update of voxel (x, y_base + 4 hy, z0 + z); bit 16 + hy*8 + z
// = an undecided voxel the full queue could not take (exact, in place, by
// brick_apply_kernel); undecided voxels go to the exact queue as here.
template <bool kClassify>
__global__ void __launch_bounds__(256, 3) brick_update_kernel(
    const __grid_constant__ VolumeTable vt, const __grid_constant__ BrickTable bt,
    const __grid_constant__ FrameGeom f, const double2 *__restrict__ table,
    const float2 *__restrict__ table32, const uint32_t *__restrict__ active,
    const unsigned int *__restrict__ active_count, unsigned long long *__restrict__ queue,
    unsigned long long *__restrict__ queue_count, const unsigned long long queue_cap,
    const int fixed_point, unsigned long long *__restrict__ stats, const ChangedList changed,
    const uint8_t *__restrict__ part_class, uint32_t *__restrict__ masks) {
    __shared__ double2 rcp[257];
    fill_rcp(rcp);
    const unsigned count = *active_count;
    const int lane = threadIdx.x & 31;
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
    const int lx = lane & 7, ly = lane >> 3;
    const float tau_ea = f.tau32 + 2.4e-7f * (f.tau32 + 16.f);  // d < 16 m rounding allowance
    const float2 fixed = make_float2(f.tau32, (float)f.max_w);
    const float hw = 0.5f * f.w32, hh = 0.5f * f.h32;
    const float k3u = 9.6e-7f * f.fx32, k3v = 9.6e-7f * f.fy32;
    const float k2u = 9.6e-7f * (fabsf(f.cx32) + 2.f), k2v = 9.6e-7f * (fabsf(f.cy32) + 2.f);
    unsigned updates = 0, swept = 0, nop = 0, col_skipped = 0, depth_skipped = 0, all_free = 0;
    unsigned part_free = 0, part_skip = 0;
    unsigned g_next = warp < count ? active[warp] : 0u;  // next brick id, loaded one brick ahead
    auto classes = [&](unsigned k) -> unsigned {
        const uchar4 c = reinterpret_cast<const uchar4 *>(part_class)[k];
        return (unsigned)c.x | ((unsigned)c.y << 2) | ((unsigned)c.z << 4) | ((unsigned)c.w << 6);
    };
    unsigned pc_next = part_class && warp < count ? classes(warp) : 0x55u;
    for (unsigned i = warp; i < count; i += nwarps) {
        const unsigned g = g_next;
        // classes of the brick's four 8x4x4 parts (2 bits each, part = hy + 2 zh:
        // 0 no voxel can update, 1 screen voxel by voxel, 2 every voxel a
        // free-space update), certified by the culling stage
        const unsigned pcls = pc_next;
        if (i + nwarps < count) {
            g_next = active[i + nwarps];
            if (part_class) pc_next = classes(i + nwarps);
        }
        const int vi = find_volume(bt, g);
        const TfVolume &vol = vt.vol[vi];
        const unsigned n = (unsigned)vol.n, nb = (unsigned)bt.nb[vi];
        const unsigned local = g - (unsigned)bt.offset[vi];
        const unsigned bxy = local % (nb * nb);
        const unsigned x = (bxy % nb) * kBrick + lx;
        const unsigned z0 = (local / (nb * nb)) * kBrick;
        const unsigned y_base = (bxy / nb) * kBrick + ly;
        const unsigned nz = min(n - z0, (unsigned)kBrick);
        float2 *vox = (float2 *)vol.voxels_dev;
        const double vs = vol.voxel_size;
        const float vs32 = (float)vs;
        const double *R = f.r_cw.m;
        const double gx = dmul((double)((int64_t)x + vol.origin[0]), vs);
        const double gz0 = dmul((double)((int64_t)z0 + vol.origin[2]), vs);
        const float szx = f.r32[2] * vs32, szy = f.r32[5] * vs32, szz = f.r32[8] * vs32;
        const float zspan = (float)(nz - 1);
        const bool keep = keeps_summary(vol, f);
        unsigned dbad = 0;  // change of this brick's packed state (summary)
        unsigned brick_free = 0, brick_vox = 0;  // free-space class / voxels of this brick (lane)
        uint32_t fmask = 0;  // kClassify: this lane's word
#pragma unroll 1
        for (int hy = 0; hy < 2; ++hy) {
            const unsigned y = y_base + 4 * hy;
            const bool row_in = x < n && y < n;
            // classes of this half's two parts (z layers 0-3, 4-7); warp-uniform
            const unsigned pc_lo = (pcls >> (2 * hy)) & 3u, pc_hi = (pcls >> (2 * hy + 4)) & 3u;
            if (pc_lo == 0u && pc_hi == 0u) {  // no voxel of the half-brick can update
                part_skip += kBrick / kZBatch;
                continue;
            }
            const double gy = dmul((double)((int64_t)y + vol.origin[1]), vs);
            // float32 column bases at z0 (plain float64, then rounded)
            const float pbx = (float)(R[0] * gx + R[1] * gy + R[2] * gz0 + f.t_cw.v[0]);
            const float pby = (float)(R[3] * gx + R[4] * gy + R[5] * gz0 + f.t_cw.v[1]);
            const float pbz = (float)(R[6] * gx + R[7] * gy + R[8] * gz0 + f.t_cw.v[2]);
            const float dbx = (float)(gx - f.cam.v[0]);
            const float dby = (float)(gy - f.cam.v[1]);
            const float dbz = (float)(gz0 - f.cam.v[2]);
            const float walk = 14.f * vs32;
            const float epc = 9.5367432e-7f * (fabsf(pbx) + fabsf(pby) + fabsf(pbz) + walk) + 1e-30f;
            const float epd = 9.5367432e-7f * (fabsf(dbx) + fabsf(dby) + fabsf(dbz) + walk) + 1e-30f;
            const float mabs = 8.f * epd * (fabsf(dbx) + fabsf(dby) + fabsf(dbz) + 8.f * vs32 + epd);
            const float k1u = f.fx32 * epc * 1.05f, k1v = f.fy32 * epc * 1.05f;
            // column bound: all voxels in front by > 64 epc -> one (du, dv) for the
            // column from its smallest pcz and largest |pcx|, |pcy| (linear in z)
            const float pz1 = fmaf(zspan, szz, pbz);
            const float zlo = fminf(pbz, pz1) - epc;
            const bool front = zlo > 64.f * epc;
            float du = 0.f, dv = 0.f;
            bool col_live = row_in;
            if (front) {
                const float rzm = 1.0f / zlo;
                const float px1 = fmaf(zspan, szx, pbx), py1 = fmaf(zspan, szy, pby);
                const float xnm = (fmaxf(fabsf(pbx), fabsf(px1)) + epc) * rzm;
                const float ynm = (fmaxf(fabsf(pby), fabsf(py1)) + epc) * rzm;
                du = fmaf(k1u, rzm * (1.f + xnm), fmaf(k3u, xnm, k2u));
                dv = fmaf(k1v, rzm * (1.f + ynm), fmaf(k3v, ynm, k2v));
                // the column's projections lie between its end projections
                const float a0 = fmaf(f.fx32, pbx / pbz, f.cx32 + 0.5f), a1 = fmaf(f.fx32, px1 / pz1, f.cx32 + 0.5f);
                const float b0 = fmaf(f.fy32, pby / pbz, f.cy32 + 0.5f), b1 = fmaf(f.fy32, py1 / pz1, f.cy32 + 0.5f);
                if (fmaxf(a0, a1) + du < 0.f || fminf(a0, a1) - du >= f.w32 ||
                    fmaxf(b0, b1) + dv < 0.f || fminf(b0, b1) - dv >= f.h32)
                    col_live = false;  // whole column clearly outside the image (:113)
            } else if (fmaxf(pbz, pz1) + epc < 0.f) {
                col_live = false;      // whole column behind the camera (:107)
            }
            if (row_in) {
                swept += nz;
                brick_vox += nz;
            }
            if (row_in && !col_live) col_skipped += nz;
            // every column of the warp outside the image / behind the camera:
            // nothing of this half-brick can update (its parts are all-skip)
            if (!__any_sync(0xffffffffu, col_live)) {
                part_skip += kBrick / kZBatch;
                continue;
            }
            const float hu = 0.5f - du, hv = 0.5f - dv;
            const bool fast = front && hu > 0.f && hv > 0.f;
            unsigned exact_mask = 0;
#pragma unroll 1
            for (int zb = 0; zb < kBrick; zb += kZBatch) {
                const unsigned pc = zb < kZBatch ? pc_lo : pc_hi;
                const unsigned nzb = (unsigned)zb < nz ? min(nz - (unsigned)zb, (unsigned)kZBatch) : 0u;
                if (pc == 0u) {  // certified: no voxel of the part can update
                    if (row_in) swept -= nzb;
                    ++part_skip;
                    continue;
                }
                if (pc == 2u) {  // certified: every voxel of the part is a free-space update
                    if (kClassify) {
                        if (row_in) {
                            fmask |= ((1u << nzb) - 1u) << (8 * hy + zb);
                            brick_free += nzb;
                        }
                        ++part_free;
                        continue;
                    }
                    const size_t row = ((size_t)(z0 + zb) * n + y) * n + x;
                    if (!TF_IN_BOUNDS(!row_in || nzb == 0u || row + (size_t)(nzb - 1) * n * n < (size_t)n * n * n))
                        continue;
                    float2 old[kZBatch];
#pragma unroll
                    for (int j = 0; j < kZBatch; ++j)
                        old[j] = row_in && (unsigned)j < nzb ? vox[(size_t)row + (size_t)j * n * n]
                                                            : make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = 0; j < kZBatch; ++j) {
                        if (!(row_in && (unsigned)j < nzb)) continue;
                        ++updates;
                        ++brick_free;
                        if (fixed_point && old[j].x == fixed.x && old[j].y == fixed.y) {
                            ++nop;
                        } else {
                            const float2 nv = free_update(old[j], f, rcp);
                            vox[(size_t)row + (size_t)j * n * n] = nv;
                            if (keep) dbad += free_state_delta(old[j], nv, f.good_t);
                        }
                    }
                    ++part_free;
                    continue;
                }
                int cls[kZBatch];
                unsigned pix[kZBatch];
                // A: pixel of every voxel of the batch
#pragma unroll
                for (int j = 0; j < kZBatch; ++j) {
                    const float kz = (float)(zb + j);
                    const float pcx = fmaf(kz, szx, pbx), pcy = fmaf(kz, szy, pby), pcz = fmaf(kz, szz, pbz);
                    int c = kSkip;
                    pix[j] = 0;
                    if (col_live && (unsigned)(zb + j) < nz) {
                        float ddu = du, ddv = dv;
                        bool ok = fast;
                        if (!fast) {  // rare: per-voxel bound (near the camera plane)
                            ok = pcz > 64.f * epc;
                            if (ok) {
                                const float rz = rcp_approx(pcz);
                                const float xn = fabsf(pcx * rz), yn = fabsf(pcy * rz);
                                ddu = fmaf(k1u, rz * (1.f + xn), fmaf(k3u, xn, k2u));
                                ddv = fmaf(k1v, rz * (1.f + yn), fmaf(k3v, yn, k2v));
                            } else {
                                c = (pcz + epc < 0.f) ? kSkip : kExact;  // behind (:107) / on the plane
                            }
                        }
                        if (ok) {
                            const float rz = rcp_approx(pcz);
                            const float a = fmaf(f.fx32, pcx * rz, f.cx32 + 0.5f);
                            const float b = fmaf(f.fy32, pcy * rz, f.cy32 + 0.5f);
                            const float fa = floorf(a), fb = floorf(b);
                            if (fabsf(a - hw) >= hw + ddu || fabsf(b - hh) >= hh + ddv) {
                                c = kSkip;  // clearly outside the image (:113)
                            } else if (fabsf(a - fa - 0.5f) >= 0.5f - ddu || fabsf(b - fb - 0.5f) >= 0.5f - ddv) {
                                c = kExact;  // within the bound of a rounding edge
                            } else {
                                const int ui = (int)fa, vi2 = (int)fb;  // saturating conversion
                                if ((unsigned)ui < (unsigned)f.width && (unsigned)vi2 < (unsigned)f.height) {
                                    c = kFree;
                                    pix[j] = (unsigned)vi2 * (unsigned)f.width + (unsigned)ui;
                                }
                            }
                        }
                    }
                    cls[j] = c;
                }
                // B: screening depth / ray scale of the decided pixels
                float2 px[kZBatch];
#pragma unroll
                for (int j = 0; j < kZBatch; ++j)
                    px[j] = cls[j] == kFree && TF_IN_BOUNDS(pix[j] < (unsigned)(f.width * f.height))
                                ? __ldg(&table32[pix[j]]) : make_float2(0.f, 0.f);
                // C: sdf class (dist <= (d - tau) rs  => free;  dist > (d + tau) rs  => skip)
#pragma unroll
                for (int j = 0; j < kZBatch; ++j) {
                    if (cls[j] != kFree) continue;
                    const float d = px[j].x, rs = px[j].y;
                    const float ddz = fmaf((float)(zb + j), vs32, dbz);
                    const float dist2 = fmaf(dbx, dbx, fmaf(dby, dby, ddz * ddz));
                    const float A = (d - tau_ea) * rs, B = (d + tau_ea) * rs;
                    int c = kExact;
                    if (!(d > 0.f)) c = kSkip;  // d32 > 0 exactly when d > 0
                    else if (A > 0.f && fmaf(dist2, 1.00001f, mabs) <= A * A * 0.99999f) c = kFree;
                    else if (fmaf(dist2, 0.99999f, -mabs) > B * B * 1.00001f) c = kSkip;
                    depth_skipped += c == kSkip;
                    cls[j] = c;
                }
                if (kClassify) {
#pragma unroll
                    for (int j = 0; j < kZBatch; ++j) {
                        if (cls[j] == kFree) {
                            fmask |= 1u << (8 * hy + zb + j);
                            ++brick_free;
                        }
                        if (cls[j] == kExact) exact_mask |= 1u << (zb + j);
                    }
                } else {
                // D: load the voxels with a free-space update
                const size_t row = ((size_t)(z0 + zb) * n + y) * n + x;
                float2 old[kZBatch];
#pragma unroll
                for (int j = 0; j < kZBatch; ++j) {
                    if (cls[j] == kFree && !TF_IN_BOUNDS(row + (size_t)j * n * n < (size_t)n * n * n)) cls[j] = kSkip;
                    old[j] = cls[j] == kFree ? vox[(size_t)row + (size_t)j * n * n] : make_float2(0.f, 0.f);
                }
                // E: free-space updates
#pragma unroll
                for (int j = 0; j < kZBatch; ++j) {
                    if (cls[j] == kFree) {
                        ++updates;
                        ++brick_free;
                        if (fixed_point && old[j].x == fixed.x && old[j].y == fixed.y) {
                            ++nop;  // (tau32, max_w) is a host-verified fixed point
                        } else {
                            const float2 nv = free_update(old[j], f, rcp);
                            vox[(size_t)row + (size_t)j * n * n] = nv;
                            if (keep) dbad += free_state_delta(old[j], nv, f.good_t);
                        }
                    }
                    if (cls[j] == kExact) exact_mask |= 1u << (zb + j);
                }
                }
                if (stats) {  // the batch is one 8x4x4 part of the brick
                    bool lf = true, ls = true;
#pragma unroll
                    for (int j = 0; j < kZBatch; ++j) {
                        lf = lf && cls[j] == kFree;
                        ls = ls && cls[j] == kSkip;
                    }
                    lf = __all_sync(0xffffffffu, lf);
                    ls = __all_sync(0xffffffffu, ls);
                    part_free += lf;
                    part_skip += ls;
                }
            }
            // undecided voxels of the column go to the exact kernel; one queue
            // reservation per warp (a lane-order scan of the counts): per-lane
            // atomics on the one counter serialise when many columns are
            // undecided (axis-aligned views put whole voxel planes on pixel
            // edges: 1.1 ms instead of 0.3 for the general kernel)
            if (__any_sync(0xffffffffu, exact_mask != 0u)) {
                const unsigned c = __popc(exact_mask);
                unsigned incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += t;
                }
                unsigned long long wbase = 0;
                if (lane == 31) wbase = atomicAdd(queue_count, (unsigned long long)incl);
                wbase = __shfl_sync(0xffffffffu, wbase, 31);
                const unsigned long long base = wbase + (incl - c);
                unsigned k = 0;
                for (unsigned m = exact_mask; m; m &= m - 1, ++k) {
                    const unsigned zz = __ffs(m) - 1;
                    const unsigned long long lin = (unsigned long long)(z0 + zz) * n * n + (unsigned long long)y * n + x;
                    if (base + k < queue_cap) {
                        // (volume, z, y, x) packed 6 / 16 / 16 / 16 bits (n <= 65535)
                        queue[base + k] = ((unsigned long long)vi << 48) | ((unsigned long long)(z0 + zz) << 32) |
                                          ((unsigned long long)y << 16) | x;
                    } else if (kClassify) {  // queue full: brick_apply_kernel updates it in place
                        fmask |= 1u << (16 + 8 * hy + zz);
                    } else {  // queue full: exact update in place (still exact)
                        const double gz = dmul((double)((int64_t)(z0 + zz) + vol.origin[2]), vs);
                        unsigned db = 0;
                        updates += update_voxel_slow(vox, (int64_t)lin, gx, gy, gz, table, f, &db,
                                                     vol.color_dev);
                        dbad += db;
                    }
                }
            }
        }
        if (kClassify) masks[(size_t)i * 32 + lane] = fmask;
        if (keep && !kClassify) {  // one atomic per brick and warp
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dbad += __shfl_xor_sync(0xffffffffu, dbad, o);
            if (lane == 0 && dbad) {
                atomicAdd(&vol.brick_state_dev[local], dbad);
                mark_changed(changed, g);
            }
        }
        if (stats && __reduce_add_sync(0xffffffffu, brick_free) == __reduce_add_sync(0xffffffffu, brick_vox))
            ++all_free;  // (counted on every lane; lane 0's count is reported)
    }
    if (stats) {
        warp_count_add(&stats[TF_STAT_VOXEL_UPDATES], updates);
        warp_count_add(&stats[TF_STAT_SWEPT_VOXELS], swept);
        warp_count_add(&stats[TF_STAT_NOOP_UPDATES], nop);
        warp_count_add(&stats[TF_STAT_COL_SKIPPED], col_skipped);
        warp_count_add(&stats[TF_STAT_DEPTH_SKIPPED], depth_skipped);
        if (lane == 0 && all_free) atomicAdd(&stats[TF_STAT_GENERAL_ALL_FREE], (unsigned long long)all_free);
        if (lane == 0 && part_free) atomicAdd(&stats[TF_STAT_PART_ALL_FREE], (unsigned long long)part_free);
        if (lane == 0 && part_skip) atomicAdd(&stats[TF_STAT_PART_ALL_SKIP], (unsigned long long)part_skip);
    }
}

// The voxel updates of the general bricks classified by
// brick_update_kernel<true> in the prepare phase: the masked free-space
// updates (and, only when the exact queue overflowed, the exact updates of
// the voxels it could not take).  Streaming like brick_free_kernel: the
// lane's 16 voxels' loads are issued before any update.
__global__ void __launch_bounds__(256, 4) brick_apply_kernel(
    const __grid_constant__ VolumeTable vt, const __grid_constant__ BrickTable bt,
    const __grid_constant__ FrameGeom f, const double2 *__restrict__ table,
    const uint32_t *__restrict__ active, const unsigned int *__restrict__ active_count,
    const uint32_t *__restrict__ masks, const int fixed_point, unsigned long long *__restrict__ stats,
    const ChangedList changed, const uint32_t *__restrict__ free_list,
    const unsigned int *__restrict__ free_count) {
    __shared__ double2 rcp[257];
    fill_rcp(rcp);
    // optionally the certified free-space bricks first (free_list: one
    // streaming kernel for both kinds, TFB200_FUSED_STREAM)
    const unsigned fc = free_list ? *free_count : 0u;
    const unsigned count = *active_count;
    const int lane = threadIdx.x & 31;
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
    const float2 fixed = make_float2(f.tau32, (float)f.max_w);
    unsigned updates = 0, nop = 0, free_updates = 0;
    for (unsigned ii = warp; ii < fc + count; ii += nwarps) {
        if (ii < fc) {
            unsigned fu = 0;
            free_brick(vt, bt, f, free_list[ii], lane, fixed_point, rcp, changed, fu, nop);
            free_updates += fu;
            continue;
        }
        const unsigned i = ii - fc;
        const uint32_t w = masks[(size_t)i * 32 + lane];
        if (!__any_sync(0xffffffffu, w != 0u)) continue;
        const unsigned g = active[i];
        const int vi = find_volume(bt, g);
        const TfVolume &vol = vt.vol[vi];
        const unsigned n = (unsigned)vol.n, nb = (unsigned)bt.nb[vi];
        const unsigned local = g - (unsigned)bt.offset[vi];
        const unsigned bxy = local % (nb * nb);
        const unsigned x = (bxy % nb) * kBrick + (lane & 7);
        const unsigned z0 = (local / (nb * nb)) * kBrick;
        const unsigned y_base = (bxy / nb) * kBrick + (lane >> 3);
        float2 *vox = (float2 *)vol.voxels_dev;
        const bool keep = keeps_summary(vol, f);
        unsigned dbad = 0;
#pragma unroll 1
        for (int hy = 0; hy < 2; ++hy) {
            const unsigned fm = (w >> (8 * hy)) & 0xffu;
            if (!__any_sync(0xffffffffu, fm != 0u)) continue;
            const size_t row = ((size_t)z0 * n + (y_base + 4 * hy)) * n + x;
            float2 old[kBrick];
#pragma unroll
            for (int z = 0; z < kBrick; ++z) {
                const bool on = (fm >> z) & 1u;
                const size_t lin = row + (size_t)z * n * n;
                old[z] = on && TF_IN_BOUNDS(lin < (size_t)n * n * n) ? vox[lin] : make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int z = 0; z < kBrick; ++z) {
                if (!((fm >> z) & 1u)) continue;
                const size_t lin = row + (size_t)z * n * n;
                if (!TF_IN_BOUNDS(lin < (size_t)n * n * n)) continue;
                ++updates;
                if (fixed_point && old[z].x == fixed.x && old[z].y == fixed.y) {
                    ++nop;  // (tau32, max_w) is a host-verified fixed point
                } else {
                    const float2 nv = free_update(old[z], f, rcp);
                    vox[lin] = nv;
                    if (keep) dbad += free_state_delta(old[z], nv, f.good_t);
                }
            }
        }
        if (w >> 16) {  // the exact queue was full (rare): exact updates in place
            const double vs = vol.voxel_size;
            const double gx = dmul((double)((int64_t)x + vol.origin[0]), vs);
            for (uint32_t m = w >> 16; m; m &= m - 1) {
                const unsigned b = __ffs(m) - 1, hy = b >> 3, z = z0 + (b & 7u), y = y_base + 4 * hy;
                const int64_t lin = ((int64_t)z * n + y) * n + x;
                unsigned db = 0;
                updates += update_voxel_slow(vox, lin, gx, dmul((double)((int64_t)y + vol.origin[1]), vs),
                                             dmul((double)((int64_t)z + vol.origin[2]), vs), table, f, &db,
                                             vol.color_dev);
                dbad += db;
            }
        }
        if (keep) {  // one atomic per brick and warp
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dbad += __shfl_xor_sync(0xffffffffu, dbad, o);
            if (lane == 0 && dbad) {
                atomicAdd(&vol.brick_state_dev[local], dbad);
                mark_changed(changed, g);
            }
        }
    }
    if (stats) {
        warp_count_add(&stats[TF_STAT_VOXEL_UPDATES], updates + free_updates);
        warp_count_add(&stats[TF_STAT_NOOP_UPDATES], nop);
        if (free_list) {
            warp_count_add(&stats[TF_STAT_FREE_KERNEL_UPDATES], free_updates);
            warp_count_add(&stats[TF_STAT_SWEPT_VOXELS], free_updates);
        }
    }
}

// The exact reference arithmetic for every queued (undecided) voxel; one
// thread per voxel, so the float64 path runs without divergence.
__global__ void __launch_bounds__(256) exact_queue_kernel(
    const __grid_constant__ VolumeTable vt, const __grid_constant__ BrickTable bt,
    const __grid_constant__ FrameGeom f,
    const double2 *__restrict__ table, const unsigned long long *__restrict__ queue,
    const unsigned long long *__restrict__ queue_count, const unsigned long long queue_cap,
    unsigned long long *__restrict__ stats, const ChangedList changed,
    const unsigned *__restrict__ active_count, const unsigned *__restrict__ free_count,
    const unsigned long long total_bricks, const unsigned long long *__restrict__ prep_stats) {
    const unsigned long long total = min(*queue_count, queue_cap);
    unsigned long long updates = 0;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long e = queue[i];
        const int v = (int)(e >> 48);
        const int64_t z = (int64_t)((e >> 32) & 0xFFFFu), y = (int64_t)((e >> 16) & 0xFFFFu),
                      x = (int64_t)(e & 0xFFFFu);
        const TfVolume &vol = vt.vol[v];
        const int64_t n = vol.n;
        const int64_t lin = (z * n + y) * n + x;
        if (!TF_IN_BOUNDS(v < vt.count && x < n && y < n && z < n)) continue;
        // the voxel's old value is loaded before the float64 projection, so its
        // HBM round trip overlaps the arithmetic instead of following it
        const float2 old = ((const float2 *)vol.voxels_dev)[lin];
        const double vs = vol.voxel_size;
        unsigned db = 0;
        updates += update_voxel((float2 *)vol.voxels_dev, lin, dmul((double)(x + vol.origin[0]), vs),
                                dmul((double)(y + vol.origin[1]), vs),
                                dmul((double)(z + vol.origin[2]), vs), table, f, &db, vol.color_dev, &old);
        if (db && keeps_summary(vol, f)) {
            summary_add(vol, lin, db);
            const int64_t nb = bt.nb[v];
            mark_changed(changed, (unsigned)(bt.offset[v] + ((z >> 3) * nb + (y >> 3)) * nb + (x >> 3)));
        }
    }
    if (stats) {
        warp_count_add(&stats[TF_STAT_VOXEL_UPDATES], updates);
        warp_count_add(&stats[TF_STAT_EXACT_UPDATES], updates);
        if (blockIdx.x == 0 && threadIdx.x == 0) {  // this call's brick counters (brick_stats_kernel)
            stats[TF_STAT_EXACT_VOXELS] += *queue_count;
            stats[TF_STAT_ACTIVE_BRICKS] += *active_count + *free_count;
            stats[TF_STAT_FREE_BRICKS] += *free_count;
            stats[TF_STAT_TOTAL_BRICKS] += total_bricks;
            if (prep_stats)  // the screen's counters, counted in the prepare phase (atomics:
                             // other blocks are adding to the same counters)
                for (int k = 0; k < TF_STAT_COUNT; ++k)
                    if (prep_stats[k]) atomicAdd(&stats[k], prep_stats[k]);
        }
    }
}

__global__ void brick_stats_kernel(const unsigned int *__restrict__ active_count,
                                   const unsigned int *__restrict__ free_count,
                                   unsigned long long total, unsigned long long *stats) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        stats[TF_STAT_ACTIVE_BRICKS] += *active_count + *free_count;
        stats[TF_STAT_FREE_BRICKS] += *free_count;
        stats[TF_STAT_TOTAL_BRICKS] += total;
    }
}

// Flag byte of brick (bx, by, bz) from the packed states: bit0 = never
// observed, bit1 = it and its existing +1 neighbours contain only good voxels
// (every cell whose min corner lies in it has only good corners).
__device__ __forceinline__ unsigned char brick_flag(const unsigned *st, int64_t nb, int64_t bx,
                                                    int64_t by, int64_t bz) {
    const unsigned s0 = st[(bz * nb + by) * nb + bx];
    unsigned char fl = (s0 >> 16) == 0u ? 1 : 0;
    bool good = (s0 & 0xFFFFu) == 0u;
    for (int c = 1; c < 8 && good; ++c) {
        const int64_t x = bx + (c & 1), y = by + ((c >> 1) & 1), z = bz + (c >> 2);
        if (x < nb && y < nb && z < nb) good = (st[(z * nb + y) * nb + x] & 0xFFFFu) == 0u;
    }
    return fl | (good ? 2 : 0);
}

// flags of every brick (after a full summary build)
__global__ void __launch_bounds__(256) brick_flags_all_kernel(const TfVolume vol) {
    const int64_t nb = (vol.n + 7) / 8, total = nb * nb * nb;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < total;
         b += (int64_t)gridDim.x * blockDim.x)
        vol.brick_flags_dev[b] = brick_flag(vol.brick_state_dev, nb, b % nb, (b / nb) % nb, b / (nb * nb));
}

// flags of the bricks whose 9^3 region contains an active brick (the only
// ones whose flags can have changed this frame); duplicate writes agree
__global__ void __launch_bounds__(256) brick_flags_active_kernel(
    const __grid_constant__ VolumeTable vt, const __grid_constant__ BrickTable bt,
    const __grid_constant__ FrameGeom f, const uint32_t *__restrict__ active,
    const unsigned int *__restrict__ active_count) {
    const unsigned count = *active_count;
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < count * 8u; t += gridDim.x * blockDim.x) {
        const unsigned g = active[t >> 3];
        const int vi = find_volume(bt, g);
        const TfVolume &vol = vt.vol[vi];
        if (!keeps_summary(vol, f) || !vol.brick_flags_dev) continue;
        const int64_t nb = bt.nb[vi], local = g - bt.offset[vi];
        const int c = t & 7;
        const int64_t bx = local % nb - (c & 1), by = (local / nb) % nb - ((c >> 1) & 1),
                      bz = local / (nb * nb) - (c >> 2);
        if (bx < 0 || by < 0 || bz < 0) continue;
        vol.brick_flags_dev[(bz * nb + by) * nb + bx] = brick_flag(vol.brick_state_dev, nb, bx, by, bz);
    }
}

// superbrick (8^3 bricks) flags: AND of the member bricks' flags.  One warp
// per (volume, superbrick) over all volumes of the launch; each lane ANDs 16
// flag bytes read as 4 x uint32 words of 4 consecutive x bricks.
__global__ void __launch_bounds__(256) super_flags_kernel(const __grid_constant__ VolumeTable vt,
                                                          const __grid_constant__ FrameGeom f,
                                                          int check_threshold) {
    const int lane = threadIdx.x & 31;
    int64_t first[TFB200_MAX_VOLUMES_PER_LAUNCH + 1];
    first[0] = 0;
    for (int v = 0; v < vt.count; ++v) {
        const int64_t nb = (vt.vol[v].n + 7) / 8, ns = (nb + 7) / 8;
        first[v + 1] = first[v] + ns * ns * ns;
    }
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < first[vt.count];
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int v = 0;
        while (w >= first[v + 1]) ++v;
        const TfVolume &vol = vt.vol[v];
        if (!vol.brick_flags_dev || (check_threshold && !keeps_summary(vol, f))) continue;
        const int64_t nb = (vol.n + 7) / 8, ns = (nb + 7) / 8, sb = w - first[v];
        const int64_t sx = sb % ns, sy = (sb / ns) % ns, sz = sb / (ns * ns);
        const unsigned char *bf = vol.brick_flags_dev;
        unsigned acc = 3u;
        // 64 (y, z) rows of 8 x bricks; lane handles rows lane and lane + 32
        const int64_t bx0 = sx * 8;
        const bool whole = (nb & 7) == 0 && ((uintptr_t)bf & 7) == 0;  // full aligned rows: one load each
#pragma unroll
        for (int r = lane; r < 64; r += 32) {
            const int64_t by = sy * 8 + (r & 7), bz = sz * 8 + (r >> 3);
            if (by >= nb || bz >= nb) continue;
            const int64_t row = (bz * nb + by) * nb + bx0;
            if (whole) {
                const unsigned long long q = *reinterpret_cast<const unsigned long long *>(bf + row);
                const unsigned lo = (unsigned)q & (unsigned)(q >> 32);
                acc &= lo & (lo >> 8) & (lo >> 16) & (lo >> 24);
            } else {
                for (int k = 0; k < 8 && bx0 + k < nb; ++k) acc &= bf[row + k];
            }
        }
        acc = __reduce_and_sync(0xffffffffu, acc);
        if (lane == 0) vol.brick_flags_dev[nb * nb * nb + sb] = (unsigned char)acc;
    }
}

// bad-voxel count of every brick from scratch (one warp per brick)
__global__ void __launch_bounds__(256) brick_summary_kernel(const TfVolume vol) {
    const int64_t n = vol.n, nb = (n + 7) / 8, total = nb * nb * nb;
    const int lane = threadIdx.x & 31;
    const float2 *vox = (const float2 *)vol.voxels_dev;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < total;
         b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t x = (b % nb) * 8 + (lane & 7), y0 = ((b / nb) % nb) * 8 + (lane >> 3);
        const int64_t z0 = (b / (nb * nb)) * 8;
        unsigned bad = 0;
        for (int hy = 0; hy < 2; ++hy)
            for (int k = 0; k < 8; ++k) {
                const int64_t y = y0 + 4 * hy, z = z0 + k;
                if (x < n && y < n && z < n) bad += voxel_state(vox[vox_index(n, z, y, x)], vol.summary_threshold);
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
        if (lane == 0) vol.brick_state_dev[b] = bad;
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

TF_BOUNDS_READER(integrate)

struct IntegrateLayout {
    size_t table_off, table32_off, mip_off, qmip_off, count_off, active_off, free_off, macro_off, queue_off,
        changed_off, dirty_off, dirty_bytes, part_off, mask_off, mask_bytes, total;
    unsigned long long queue_cap;
};

// counters area (count_off): brick / free / macro / changed counts at 0, 8,
// 16, 24, the queue count at 64; the prepare phase's screen counters
// (TF_STAT_COUNT words) at kPrepStatsOff; zeroed by frame_prep_kernel
constexpr size_t kPrepStatsOff = 256, kCountBytes = 512;

// the screen's per-brick masks (128 bytes per general brick) are kept for
// launches of up to 8 M bricks (1 GB); larger launches screen and update in
// one kernel in the finish phase
constexpr int64_t kMaskMaxBricks = 8ll << 20;

// capacity of the exact-voxel queue; overflow is handled inline (still exact)
constexpr unsigned long long kQueueCap = 8ull << 20;

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

static IntegrateLayout layout_for(int64_t total_bricks_max, const TfCamera *cam) {
    const MipDesc m = make_mip(cam->width, cam->height);
    IntegrateLayout L{};
    size_t off = 0;
    L.table_off = off;
    off = align_up(off + (size_t)(cam->width * cam->height) * sizeof(double2), 256);
    L.table32_off = off;
    off = align_up(off + (size_t)(cam->width * cam->height) * sizeof(float2), 256);
    L.mip_off = off;
    off = align_up(off + (size_t)m.total * sizeof(unsigned long long), 256);
    L.qmip_off = off;
    off = align_up(off + (size_t)m.total * sizeof(unsigned), 256);
    L.count_off = off;
    off = align_up(off + kCountBytes, 256);
    L.active_off = off;
    off = align_up(off + (size_t)total_bricks_max * sizeof(uint32_t), 256);
    L.free_off = off;
    off = align_up(off + (size_t)total_bricks_max * sizeof(uint32_t), 256);
    L.macro_off = off;
    off = align_up(off + (size_t)total_bricks_max * sizeof(uint32_t), 256);
    L.queue_off = off;
    L.queue_cap = kQueueCap;
    off = align_up(off + (size_t)L.queue_cap * sizeof(unsigned long long), 256);
    L.changed_off = off;
    off = align_up(off + (size_t)total_bricks_max * sizeof(uint32_t), 256);
    L.dirty_off = off;
    L.dirty_bytes = (size_t)((total_bricks_max + 31) / 32) * sizeof(uint32_t);
    off = align_up(off + L.dirty_bytes, 256);
    L.part_off = off;  // part classes of the general bricks, 4 bytes per active entry
    off = align_up(off + (size_t)total_bricks_max * 4, 256);
    L.mask_off = off;  // screen masks of the general bricks, 32 words per active entry
    L.mask_bytes = total_bricks_max <= kMaskMaxBricks ? (size_t)total_bricks_max * 128 : 0;
    off = align_up(off + L.mask_bytes, 256);
    L.total = off;
    return L;
}

static int64_t bricks_of(const TfVolume *vols, int nvol, int64_t *max_chunk) {
    int64_t total = 0, chunk = 0, best = 0;
    for (int v = 0; v < nvol; ++v) {
        const int64_t nb = (vols[v].n + kBrick - 1) / kBrick;
        total += nb * nb * nb;
        chunk += nb * nb * nb;
        if ((v + 1) % TFB200_MAX_VOLUMES_PER_LAUNCH == 0 || v + 1 == nvol) {
            best = chunk > best ? chunk : best;
            chunk = 0;
        }
    }
    if (max_chunk) *max_chunk = best;
    return total;
}

}  // namespace tf

using namespace tf;

extern "C" size_t tf_integrate_workspace_size(const TfVolume *vols, int nvol, const TfCamera *cam) {
    if (!vols || nvol < 0 || !cam || cam->width <= 0 || cam->height <= 0) return 0;
    int64_t chunk = 0;
    bricks_of(vols, nvol, &chunk);
    return layout_for(chunk, cam).total;
}

// Per-device side stream (and fork / join events) for kernels that run next
// to the caller's stream inside one call; joined back before the call returns.
struct SideStream {
    std::mutex mu;
    cudaStream_t stream = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};

static SideStream *side_stream() {
    constexpr int kMaxDev = 64;
    static SideStream sides[kMaxDev];
    static std::mutex init_mu;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
    std::lock_guard<std::mutex> lock(init_mu);
    SideStream &s = sides[dev];
    if (!s.stream) {
        if (cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming) != cudaSuccess)
            return nullptr;
    }
    return &s;
}

// phases: 1 = prepare (pixel tables, mips, culling into the workspace),
// 2 = finish (the voxel updates and summary upkeep), 3 = both.  More volumes
// than one launch holds reuse the workspace per chunk, so there prepare does
// nothing and finish runs both phases.
static int integrate_impl(const TfVolume *vols, int nvol, const double *depth, const uint8_t *rgb,
                          const TfCamera *cam, const double r_cw[9], const double t_cw[3],
                          const double cam_center[3], double tau, double max_weight,
                          double sample_weight, void *workspace, size_t workspace_bytes,
                          uint64_t *stats, void *stream_, int phases) {
    cudaStream_t stream = (cudaStream_t)stream_;
    if (nvol == 0) return TF_OK;
    if (!vols || nvol < 0 || !depth || !cam || !r_cw || !t_cw || !cam_center || !workspace)
        return tf_set_error(TF_EINVAL, "tf_integrate: null argument");
    if (cam->width <= 0 || cam->height <= 0)
        return tf_set_error(TF_EINVAL, "tf_integrate: bad image size");
    for (int v = 0; v < nvol; ++v) {
        if (!vols[v].voxels_dev || vols[v].n < 2 || !(vols[v].voxel_size > 0.0))
            return tf_set_error(TF_EINVAL, "tf_integrate: bad volume %d", v);
        if (vols[v].n > 65535)  // 16-bit voxel coordinates in the exact queue
            return tf_set_error(TF_EINVAL, "tf_integrate: volume %d: n = %lld > 65535", v, (long long)vols[v].n);
    }
    int64_t chunk = 0;
    bricks_of(vols, nvol, &chunk);
    if (chunk > (int64_t)0xffffffffLL)
        return tf_set_error(TF_EINVAL, "tf_integrate: too many bricks in one launch");
    const IntegrateLayout L = layout_for(chunk, cam);
    if (workspace_bytes < L.total)
        return tf_set_error(TF_EINVAL, "tf_integrate: workspace %zu < %zu bytes", workspace_bytes,
                            L.total);
    char *ws = (char *)workspace;
    double2 *table = (double2 *)(ws + L.table_off);
    float2 *table32 = (float2 *)(ws + L.table32_off);
    unsigned long long *mip = (unsigned long long *)(ws + L.mip_off);
    unsigned *qmip = (unsigned *)(ws + L.qmip_off);
    unsigned int *fcount = (unsigned int *)(ws + L.count_off + 8);
    uint32_t *active_free = (uint32_t *)(ws + L.free_off);
    uint32_t *macros = (uint32_t *)(ws + L.macro_off);
    unsigned int *mcount = (unsigned int *)(ws + L.count_off + 16);
    unsigned int *count = (unsigned int *)(ws + L.count_off);
    unsigned long long *qcount = (unsigned long long *)(ws + L.count_off + 64);
    unsigned long long *queue = (unsigned long long *)(ws + L.queue_off);
    uint32_t *active = (uint32_t *)(ws + L.active_off);
    uint8_t *part_class = (uint8_t *)(ws + L.part_off);
    uint32_t *masks = (uint32_t *)(ws + L.mask_off);
    unsigned long long *prep_stats = (unsigned long long *)(ws + L.count_off + kPrepStatsOff);
    static const int use_split = [] {
        // tuning knob (A/B): the screen of the general bricks in the prepare
        // phase (brick_update_kernel<true> + brick_apply_kernel) instead of
        // one kernel in the finish phase
        const char *e = getenv("TFB200_SPLIT_SCREEN");
        return e ? atoi(e) : 1;
    }();
    static const unsigned long long queue_cap_env = [] {
        // test knob: a smaller exact queue, so the overflow paths (exact
        // updates in place) run (tests/test_gpu_parity.py)
        const char *e = getenv("TFB200_QUEUE_CAP");
        return e ? strtoull(e, nullptr, 10) : ~0ull;
    }();
    const unsigned long long queue_cap = L.queue_cap < queue_cap_env ? L.queue_cap : queue_cap_env;
    static const int use_parts = [] {
        const char *e = getenv("TFB200_PARTS");  // tuning knob (A/B): part classes from the cull stage
        return e ? atoi(e) : 1;
    }();
    const MipDesc m = make_mip(cam->width, cam->height);
    bool do_prep = (phases & 1) != 0;
    const bool do_fin = (phases & 2) != 0;
    if (nvol > TFB200_MAX_VOLUMES_PER_LAUNCH) {
        if (!do_fin) return TF_OK;
        do_prep = true;
    }

    void *prof_all = do_fin ? tf_profile_begin(TF_PROF_INTEGRATE_ALL, stream) : nullptr;
    int rc = TF_OK;
    if (do_prep) {
        if (cudaMemsetAsync(mip, 0, (size_t)m.total * sizeof(unsigned long long), stream) != cudaSuccess ||
            cudaMemsetAsync(qmip, 0xff, (size_t)m.total * sizeof(unsigned), stream) != cudaSuccess)
            return tf_set_error(TF_ECUDA, "tf_integrate: memset failed");
        dim3 pblock(kTile, kTile);
        dim3 pgrid((unsigned)((cam->width + kTile - 1) / kTile), (unsigned)((cam->height + kTile - 1) / kTile));
        frame_prep_kernel<<<pgrid, pblock, 0, stream>>>(depth, table, table32, mip, qmip, tau, m, cam->fx,
                                                        cam->fy, cam->cx, cam->cy, cam->width,
                                                        cam->height, count, (int)(kCountBytes / 4),
                                                        (unsigned *)(ws + L.dirty_off),
                                                        (int64_t)(L.dirty_bytes / sizeof(unsigned)));
        rc = tf_check_launch("frame_prep_kernel");
        if (rc) return rc;
    }

    FrameGeom f{};
    for (int i = 0; i < 9; ++i) f.r_cw.m[i] = r_cw[i];
    for (int i = 0; i < 3; ++i) {
        f.t_cw.v[i] = t_cw[i];
        f.cam.v[i] = cam_center[i];
    }
    f.fx = cam->fx;
    f.fy = cam->fy;
    f.cx = cam->cx;
    f.cy = cam->cy;
    f.width = cam->width;
    f.height = cam->height;
    f.tau = tau;
    f.max_w = max_weight;
    f.sw = sample_weight;
    f.sw_tau = sample_weight * tau;  // IEEE double product, as the reference's sw * clamped
    f.unit_sw = sample_weight == 1.0 && std::isfinite(max_weight);
    f.max_w32 = (float)max_weight;
    f.rgb = rgb;
    for (int i = 0; i < 9; ++i) f.r32[i] = (float)r_cw[i];
    f.fx32 = (float)cam->fx;
    f.fy32 = (float)cam->fy;
    f.cx32 = (float)cam->cx;
    f.cy32 = (float)cam->cy;
    f.tau32 = (float)tau;
    f.w32 = (float)cam->width;
    f.h32 = (float)cam->height;
    f.good_t = good_threshold(tau);

    // Is the saturated free-space state (tau32, max_w) a fixed point of the
    // free-space update?  Evaluated here with the kernel's exact IEEE
    // operations (host code is built with -ffp-contract=off); when it is,
    // such voxels are provably unchanged and their store is skipped.
    int fixed_point = 0;
    if (!(tf_debug_flags() & TF_DEBUG_NO_FIXEDPOINT)) {
        const volatile float t32 = (float)tau, w32 = (float)max_weight;
        const volatile float wv = t32 * w32;
        const volatile double w_sum = (double)w32 + sample_weight;
        const volatile double num = (double)wv + f.sw_tau;
        const volatile double t_new = num / w_sum;
        const double w_new = max_weight < w_sum ? max_weight : w_sum;
        fixed_point = ((float)t_new == t32) && ((float)w_new == w32);
    }

    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);

    for (int first = 0; first < nvol; first += TFB200_MAX_VOLUMES_PER_LAUNCH) {
        const int cnt = nvol - first < TFB200_MAX_VOLUMES_PER_LAUNCH ? nvol - first
                                                                     : TFB200_MAX_VOLUMES_PER_LAUNCH;
        VolumeTable vt{};
        BrickTable bt{};
        vt.count = cnt;
        bt.count = cnt;
        int64_t off = 0;
        for (int v = 0; v < cnt; ++v) {
            vt.vol[v] = vols[first + v];
            const int64_t nb = (vols[first + v].n + kBrick - 1) / kBrick;
            bt.nb[v] = nb;
            bt.offset[v] = off;
            off += nb * nb * nb;
        }
        bt.offset[cnt] = off;
        const ChangedList changed{(uint32_t *)(ws + L.changed_off), (unsigned *)(ws + L.count_off + 24),
                                  (unsigned *)(ws + L.dirty_off)};
        const int exact_only = (tf_debug_flags() & TF_DEBUG_EXACT_ONLY) ? 1 : 0;
        const int no_cull = (tf_debug_flags() & TF_DEBUG_NO_CULL) ? 1 : 0;
        const bool split = use_split && L.mask_bytes > 0 && !exact_only;
        static const int gen_grid = [] {
            const char *e = getenv("TFB200_GEN_GRID");  // tuning knob (A/B): blocks per SM
            return e ? atoi(e) : 9;
        }();
        if (do_prep) {
            if (first > 0 &&  // chunk 0's were zeroed by frame_prep_kernel
                (cudaMemsetAsync(count, 0, kCountBytes, stream) != cudaSuccess ||  // counters
                 cudaMemsetAsync(ws + L.dirty_off, 0, L.dirty_bytes, stream) != cudaSuccess))
                return tf_set_error(TF_ECUDA, "tf_integrate: memset failed");
            int64_t macros_total = 0;
            for (int v = 0; v < cnt; ++v) {
                const int64_t nm = (bt.nb[v] + kMacro - 1) / kMacro;
                macros_total += nm * nm * nm;
            }
            macro_cull_kernel<<<(unsigned)((macros_total + 255) / 256), 256, 0, stream>>>(
                vt, bt, f, m, mip, qmip, macros, mcount, active_free, fcount, no_cull, exact_only ? 0 : 1);
            if ((rc = tf_check_launch("macro_cull_kernel"))) return rc;
            brick_cull_kernel<<<(unsigned)sms * 8, 256, 0, stream>>>(
                vt, bt, f, m, mip, qmip, macros, mcount, active, count, active_free, fcount, no_cull,
                exact_only ? 0 : 1);
            if ((rc = tf_check_launch("brick_cull_kernel"))) return rc;
            if (use_parts && !no_cull) {
                part_cull_kernel<<<(unsigned)sms * 8, 256, 0, stream>>>(vt, bt, f, m, mip, qmip, active, count,
                                                                       part_class, exact_only ? 0 : 1);
                if ((rc = tf_check_launch("part_cull_kernel"))) return rc;
            }
            if (split) {  // the screen: masks + exact queue, no voxel touched
                void *ps = tf_profile_begin(TF_PROF_INTEGRATE_SCREEN, stream);
                brick_update_kernel<true><<<(unsigned)(sms * gen_grid), 256, 0, stream>>>(
                    vt, bt, f, table, table32, active, count, queue, qcount, queue_cap, fixed_point, prep_stats,
                    changed, use_parts && !no_cull ? part_class : nullptr, masks);
                tf_profile_end(ps, stream);
                if ((rc = tf_check_launch("brick_update_kernel<screen>"))) return rc;
            }
        }
        if (!do_fin) continue;
        void *prof = tf_profile_begin(TF_PROF_INTEGRATE_UPDATE, stream);
        if (tf_debug_flags() & TF_DEBUG_EXACT_ONLY) {
            brick_update_exact_kernel<<<(unsigned)sms * 8, 256, 0, stream>>>(
                vt, bt, f, table, active, count, (unsigned long long *)stats);
        } else {
            // the certified free-space bricks (bandwidth-bound) run on a side
            // stream next to the general bricks (issue-bound): disjoint bricks
            static const int free_serial = [] {
                // tuning knob (A/B): the free-brick kernel in stream order
                // instead of on a side stream next to the general kernel (0.423
                // vs 0.371 ms update bracket, config 3); interleaving free bricks
                // into the general kernel's work items measured 0.471 ms (the
                // streaming loses its memory parallelism at 3 blocks / SM)
                const char *e = getenv("TFB200_FREE_SERIAL");
                return e ? atoi(e) : 0;
            }();
            SideStream *side = free_serial ? nullptr : side_stream();
            if (!free_serial && !side) return tf_set_error(TF_ECUDA, "tf_integrate: cannot create the side stream");
            std::unique_lock<std::mutex> side_lock;
            if (side) side_lock = std::unique_lock<std::mutex>(side->mu);
            const cudaStream_t fs = side ? side->stream : stream;
            if (side) {
                cudaEventRecord(side->fork, stream);
                cudaStreamWaitEvent(side->stream, side->fork, 0);
            }
            static const int free_grid = [] {  // tuning knob (A/B): blocks per SM
                const char *e = getenv("TFB200_FREE_GRID");
                return e ? atoi(e) : 4;
            }();
            static const int apply_grid = [] {  // tuning knob (A/B): blocks per SM
                const char *e = getenv("TFB200_APPLY_GRID");
                return e ? atoi(e) : 4;
            }();
            static const int exact_first = [] {  // tuning knob (A/B): exact queue before the masked updates
                const char *e = getenv("TFB200_EXACT_FIRST");
                return e ? atoi(e) : 0;
            }();
            auto launch_exact = [&]() -> int {
                void *pe = tf_profile_begin(TF_PROF_INTEGRATE_EXACT, stream);
                exact_queue_kernel<<<(unsigned)sms * 8, 256, 0, stream>>>(vt, bt, f, table, queue, qcount,
                                                                         queue_cap,
                                                                         (unsigned long long *)stats, changed,
                                                                         count, fcount, (unsigned long long)off,
                                                                         split ? prep_stats : nullptr);
                tf_profile_end(pe, stream);
                return tf_check_launch("exact_queue_kernel");
            };
            static const int fused_stream = [] {
                // tuning knob (A/B): 2 (default) = the free-space bricks and the
                // masked updates in one streaming kernel with the exact band
                // beside it on the side stream (bracket 0.161 -> 0.156 ms);
                // 1 = the same with the exact band after it (0.187); 0 = free
                // kernel on the side stream beside the masked updates, then the
                // exact band
                const char *e = getenv("TFB200_FUSED_STREAM");
                return e ? atoi(e) : 2;
            }();
            if (split && fused_stream) {
                if (fused_stream == 2 && side) {  // the exact band beside the stream, on the side stream
                    exact_queue_kernel<<<(unsigned)sms * 8, 256, 0, fs>>>(
                        vt, bt, f, table, queue, qcount, queue_cap, (unsigned long long *)stats, changed, count,
                        fcount, (unsigned long long)off, prep_stats);
                    if ((rc = tf_check_launch("exact_queue_kernel"))) return rc;
                    cudaEventRecord(side->join, fs);
                }
                void *pg2 = tf_profile_begin(TF_PROF_INTEGRATE_GENERAL, stream);
                brick_apply_kernel<<<(unsigned)(sms * apply_grid), 256, 0, stream>>>(
                    vt, bt, f, table, active, count, masks, fixed_point, (unsigned long long *)stats, changed,
                    active_free, fcount);
                tf_profile_end(pg2, stream);
                if ((rc = tf_check_launch("brick_apply_kernel<fused>"))) return rc;
                if (fused_stream == 2 && side) cudaStreamWaitEvent(stream, side->join, 0);
                else if ((rc = launch_exact())) return rc;
            } else {
            if (split && exact_first && (rc = launch_exact())) return rc;
            static const int free_tma = [] {  // tuning knob (A/B): free bricks staged by bulk copies
                const char *e = getenv("TFB200_FREE_TMA");
                return e ? atoi(e) : 0;
            }();
            void *pf = tf_profile_begin(TF_PROF_INTEGRATE_FREE, fs);
            BrickMaps maps;  // the kernel parameter (copied at launch)
            bool maps_ok = free_tma != 0;
            if (maps_ok) {
                using Encode = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                            const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                            const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
                static Encode encode = [] {
                    void *fn = nullptr;
                    cudaDriverEntryPointQueryResult q{};
                    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
                        q != cudaDriverEntryPointSuccess)
                        return (Encode) nullptr;
                    return (Encode)fn;
                }();
                for (int v = 0; v < cnt && maps_ok; ++v) {
                    const cuuint64_t n = (cuuint64_t)vt.vol[v].n;
                    if (!encode || (n & 1u)) {  // odd n: rows are not 16-byte strided
                        maps_ok = false;
                        break;
                    }
                    const cuuint64_t dims[3] = {n, n, n}, strides[2] = {n * 8, n * n * 8};
                    const cuuint32_t box[3] = {8, 8, 8}, estr[3] = {1, 1, 1};
                    maps_ok = encode(&maps.m[v], CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, vt.vol[v].voxels_dev, dims,
                                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
                }
            }
            if (maps_ok) {
                constexpr int smem = kFreeTmaWarps * 2 * 4096;
                // (per device: set on every call)
                if (cudaFuncSetAttribute(brick_free_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
                    cudaSuccess)
                    return tf_set_error(TF_ECUDA, "tf_integrate: shared memory attribute");
                brick_free_tma_kernel<<<(unsigned)(sms * 3), 256, smem, fs>>>(
                    vt, bt, f, maps, active_free, fcount, fixed_point, (unsigned long long *)stats, changed);
            } else
            brick_free_kernel<<<(unsigned)(sms * free_grid), 256, 0, fs>>>(vt, bt, f, active_free, fcount, fixed_point,
                                                                (unsigned long long *)stats, changed);
            tf_profile_end(pf, fs);
            if ((rc = tf_check_launch("brick_free_kernel"))) return rc;
            if (side) cudaEventRecord(side->join, fs);
            void *pg = tf_profile_begin(TF_PROF_INTEGRATE_GENERAL, stream);
            if (split) {
                brick_apply_kernel<<<(unsigned)(sms * apply_grid), 256, 0, stream>>>(
                    vt, bt, f, table, active, count, masks, fixed_point, (unsigned long long *)stats, changed,
                    nullptr, nullptr);
                tf_profile_end(pg, stream);
                if ((rc = tf_check_launch("brick_apply_kernel"))) return rc;
            } else {
                brick_update_kernel<false><<<(unsigned)(sms * gen_grid), 256, 0, stream>>>(
                    vt, bt, f, table, table32, active, count, queue, qcount, queue_cap, fixed_point,
                    (unsigned long long *)stats, changed, use_parts && !no_cull ? part_class : nullptr, nullptr);
                tf_profile_end(pg, stream);
                if ((rc = tf_check_launch("brick_update_kernel"))) return rc;
            }
            if (!(split && exact_first) && (rc = launch_exact())) return rc;
            if (side) cudaStreamWaitEvent(stream, side->join, 0);
            }
        }
        tf_profile_end(prof, stream);
        if ((rc = tf_check_launch("brick_update_kernel"))) return rc;
        bool any_summary = false;
        for (int v = 0; v < cnt; ++v)
            any_summary |= vt.vol[v].brick_flags_dev && vt.vol[v].brick_state_dev &&
                           vt.vol[v].summary_threshold == f.good_t;
        if (any_summary && exact_only) {  // the reference-order kernel does not list changes
            brick_flags_active_kernel<<<(unsigned)sms * 4, 256, 0, stream>>>(vt, bt, f, active, count);
            if ((rc = tf_check_launch("brick_flags_active_kernel"))) return rc;
            brick_flags_active_kernel<<<(unsigned)sms * 4, 256, 0, stream>>>(vt, bt, f, active_free, fcount);
            if ((rc = tf_check_launch("brick_flags_active_kernel"))) return rc;
        } else if (any_summary) {
            // flags depend on a brick's own and its +1 neighbours' states: the
            // bricks whose state changed and their lower neighbours
            brick_flags_active_kernel<<<(unsigned)sms * 4, 256, 0, stream>>>(vt, bt, f, changed.list,
                                                                          changed.count);
            if ((rc = tf_check_launch("brick_flags_active_kernel"))) return rc;
        }
        if (any_summary) {
            super_flags_kernel<<<(unsigned)sms * 4, 256, 0, stream>>>(vt, f, 1);
            if ((rc = tf_check_launch("super_flags_kernel"))) return rc;
        }
        if (stats && exact_only) {  // otherwise exact_queue_kernel counted them
            brick_stats_kernel<<<1, 32, 0, stream>>>(count, fcount, (unsigned long long)off,
                                                     (unsigned long long *)stats);
            if ((rc = tf_check_launch("brick_stats_kernel"))) return rc;
        }
    }
    if (prof_all) tf_profile_end(prof_all, stream);
    return TF_OK;
}

extern "C" int tf_integrate_rgb(const TfVolume *vols, int nvol, const double *depth, const uint8_t *rgb,
                                const TfCamera *cam, const double r_cw[9], const double t_cw[3],
                                const double cam_center[3], double tau, double max_weight,
                                double sample_weight, void *workspace, size_t workspace_bytes,
                                uint64_t *stats, void *stream) {
    return integrate_impl(vols, nvol, depth, rgb, cam, r_cw, t_cw, cam_center, tau, max_weight, sample_weight,
                          workspace, workspace_bytes, stats, stream, 3);
}

extern "C" int tf_integrate(const TfVolume *vols, int nvol, const double *depth,
                            const TfCamera *cam, const double r_cw[9], const double t_cw[3],
                            const double cam_center[3], double tau, double max_weight,
                            double sample_weight, void *workspace, size_t workspace_bytes,
                            uint64_t *stats, void *stream) {
    return integrate_impl(vols, nvol, depth, nullptr, cam, r_cw, t_cw, cam_center, tau, max_weight,
                          sample_weight, workspace, workspace_bytes, stats, stream, 3);
}

extern "C" int tf_integrate_prepare(const TfVolume *vols, int nvol, const double *depth, const TfCamera *cam,
                                    const double r_cw[9], const double t_cw[3], const double cam_center[3],
                                    double tau, double max_weight, double sample_weight, void *workspace,
                                    size_t workspace_bytes, void *stream) {
    return integrate_impl(vols, nvol, depth, nullptr, cam, r_cw, t_cw, cam_center, tau, max_weight,
                          sample_weight, workspace, workspace_bytes, nullptr, stream, 1);
}

extern "C" int tf_integrate_finish(const TfVolume *vols, int nvol, const double *depth, const uint8_t *rgb,
                                   const TfCamera *cam, const double r_cw[9], const double t_cw[3],
                                   const double cam_center[3], double tau, double max_weight,
                                   double sample_weight, void *workspace, size_t workspace_bytes,
                                   uint64_t *stats, void *stream) {
    return integrate_impl(vols, nvol, depth, rgb, cam, r_cw, t_cw, cam_center, tau, max_weight, sample_weight,
                          workspace, workspace_bytes, stats, stream, 2);
}

extern "C" float tf_good_threshold(double tau) { return good_threshold(tau); }

extern "C" int tf_brick_summary(const TfVolume *vol, void *stream_) {
    if (!vol || !vol->voxels_dev || !vol->brick_state_dev || vol->n < 2)
        return tf_set_error(TF_EINVAL, "tf_brick_summary: bad argument");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    brick_summary_kernel<<<(unsigned)sms * 8, 256, 0, (cudaStream_t)stream_>>>(*vol);
    int rc = tf_check_launch("brick_summary_kernel");
    if (rc || !vol->brick_flags_dev) return rc;
    brick_flags_all_kernel<<<(unsigned)sms * 8, 256, 0, (cudaStream_t)stream_>>>(*vol);
    if ((rc = tf_check_launch("brick_flags_all_kernel"))) return rc;
    VolumeTable vt{};
    vt.count = 1;
    vt.vol[0] = *vol;
    FrameGeom f{};
    super_flags_kernel<<<(unsigned)sms * 2, 256, 0, (cudaStream_t)stream_>>>(vt, f, 0);
    return tf_check_launch("super_flags_kernel");
}

extern "C" int64_t tf_debug_weight_division_check(int64_t n, uint64_t seed) {
    unsigned long long *d = nullptr, h = 0;
    if (n <= 0) return 0;
    if (cudaMalloc(&d, sizeof(h)) != cudaSuccess) return -1;
    cudaMemset(d, 0, sizeof(h));
    weight_division_check_kernel<<<1184, 256>>>(n, seed, d);
    const bool ok = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaFree(d);
    return ok ? (int64_t)h : -1;
}
