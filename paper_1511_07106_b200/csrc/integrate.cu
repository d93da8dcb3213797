// Projective TSDF integration, fused over many volumes (sm_100a).
//
// Replaces _kernels.integrate_kernel (reference _kernels.py:71-133).  Three
// launches per frame, all on the caller's stream:
//
//   1. frame_prep   — per pixel {depth, ray_scale} table (ray_scale is a pure
//                     function of the rounded pixel, :118-120, so it is
//                     computed once per pixel instead of once per voxel) and a
//                     max-depth mip over 16x16-pixel tiles for culling;
//   2. brick_cull   — one thread per 8^3 brick of every volume; a brick is
//                     dropped only when NO voxel in it can pass the
//                     reference's gates (behind the camera, projecting outside
//                     the image, no valid depth, or more than tau behind every
//                     depth it can see), with explicit rounding margins;
//   3. brick_update — persistent warps walk the surviving bricks and run the
//                     reference's per-voxel arithmetic exactly (same op order,
//                     round-to-nearest intrinsics, f32 where numba types it
//                     f32), reading/writing each voxel's float2 once.
//
// Work therefore scales with voxels near the camera frustum, not with n^3,
// and the only HBM traffic per voxel update is its 8-byte read + 8-byte write.
#include <math.h>

#include "tf_common.cuh"

namespace tf {

constexpr int kBrick = 8;         // brick edge in voxels
constexpr int kTile = 16;         // finest depth-mip tile in pixels
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
};

static MipDesc make_mip(int64_t width, int64_t height) {
    MipDesc m{};
    int64_t off = 0;
    int l = 0;
    for (; l < kMaxMipLevels; ++l) {
        int64_t cell = (int64_t)kTile << l;
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
__global__ void __launch_bounds__(256) frame_prep_kernel(
    const double *__restrict__ depth, double2 *__restrict__ table,
    unsigned long long *__restrict__ mip, const MipDesc m, const double fx,
    const double fy, const double cx, const double cy, const int64_t width,
    const int64_t height) {
    const int64_t ui = (int64_t)blockIdx.x * kTile + threadIdx.x;
    const int64_t vi = (int64_t)blockIdx.y * kTile + threadIdx.y;
    double d = 0.0;
    if (ui < width && vi < height) {
        d = depth[vi * width + ui];
        // _kernels.py:118-120
        const double rx = ddiv(dsub((double)ui, cx), fx);
        const double ry = ddiv(dsub((double)vi, cy), fy);
        const double rs = dsqrt(dadd(dadd(dmul(rx, rx), dmul(ry, ry)), 1.0));
        table[vi * width + ui] = make_double2(d, rs);
    }
    // block max of the (non-negative) depths
    double v = d > 0.0 ? d : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __shared__ double wmax[8];
    const int t = threadIdx.y * kTile + threadIdx.x;
    if ((t & 31) == 0) wmax[t >> 5] = v;
    __syncthreads();
    if (t == 0) {
        double b = wmax[0];
        for (int i = 1; i < 8; ++i) b = fmax(b, wmax[i]);
        const unsigned long long bits = (unsigned long long)__double_as_longlong(b);
        mip[m.offset[0] + (int64_t)blockIdx.y * m.tiles_x[0] + blockIdx.x] = bits;
        for (int l = 1; l < m.levels; ++l) {
            const int64_t tx = (int64_t)blockIdx.x >> l, ty = (int64_t)blockIdx.y >> l;
            atomicMax(&mip[m.offset[l] + ty * m.tiles_x[l] + tx], bits);
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
           (((u1 >> (4 + l)) - (u0 >> (4 + l)) + 1) > 4 || ((v1 >> (4 + l)) - (v0 >> (4 + l)) + 1) > 4))
        ++l;
    unsigned long long best = 0;
    const int64_t tx0 = u0 >> (4 + l), tx1 = u1 >> (4 + l);
    const int64_t ty0 = v0 >> (4 + l), ty1 = v1 >> (4 + l);
    for (int64_t ty = ty0; ty <= ty1; ++ty)
        for (int64_t tx = tx0; tx <= tx1; ++tx) {
            const unsigned long long b = __ldg(&mip[m.offset[l] + ty * m.tiles_x[l] + tx]);
            best = b > best ? b : best;
        }
    return __longlong_as_double((long long)best);
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
// _kernels.py:107-127.  All margins are orders of magnitude above the FP64
// rounding of the reference's per-voxel arithmetic (relative ~1e-15).
__device__ bool brick_may_update(const TfVolume &vol, int64_t bx, int64_t by, int64_t bz,
                                 const FrameGeom &f, const unsigned long long *__restrict__ mip,
                                 const MipDesc &m) {
    const int64_t n = vol.n;
    const int64_t i0[3] = {bx * kBrick, by * kBrick, bz * kBrick};
    double gmin[3], gmax[3], gabs = 0.0;
    for (int a = 0; a < 3; ++a) {
        const int64_t i1 = min(i0[a] + kBrick - 1, n - 1);
        // the reference's voxel centres (i + ht) * vs are monotone in i
        gmin[a] = (double)(i0[a] + vol.origin[a]) * vol.voxel_size;
        gmax[a] = (double)(i1 + vol.origin[a]) * vol.voxel_size;
        gabs += fmax(fabs(gmin[a]), fabs(gmax[a]));
    }
    const double *R = f.r_cw.m, *T = f.t_cw.v;
    const double tabs = fabs(T[0]) + fabs(T[1]) + fabs(T[2]);
    const double err = 1e-12 * (gabs + tabs + 1.0);  // bound on pc rounding, meters
    double zmin = 1e300, zmax = -1e300, xabs = 0.0, yabs = 0.0;
    double pcs[8][3];
    for (int c = 0; c < 8; ++c) {
        const double g[3] = {(c & 1) ? gmax[0] : gmin[0], (c & 2) ? gmax[1] : gmin[1],
                             (c & 4) ? gmax[2] : gmin[2]};
        for (int r = 0; r < 3; ++r)
            pcs[c][r] = R[r * 3 + 0] * g[0] + R[r * 3 + 1] * g[1] + R[r * 3 + 2] * g[2] + T[r];
        zmin = fmin(zmin, pcs[c][2]);
        zmax = fmax(zmax, pcs[c][2]);
        xabs = fmax(xabs, fabs(pcs[c][0]));
        yabs = fmax(yabs, fabs(pcs[c][1]));
    }
    if (zmax <= -2.0 * err) return false;  // every voxel has pcz <= 0 (:107)

    int64_t u0 = 0, u1 = f.width - 1, v0 = 0, v1 = f.height - 1;
    if (zmin > 0.01 + 2.0 * err) {
        // in front of the camera: the projections of all voxels lie inside the
        // projected corners' bounding box (convexity), up to rounding
        double umin = 1e300, umax = -1e300, vmin = 1e300, vmax = -1e300;
        for (int c = 0; c < 8; ++c) {
            const double u = f.fx * pcs[c][0] / pcs[c][2] + f.cx;
            const double v = f.fy * pcs[c][1] / pcs[c][2] + f.cy;
            umin = fmin(umin, u);
            umax = fmax(umax, u);
            vmin = fmin(vmin, v);
            vmax = fmax(vmax, v);
        }
        const double zl = zmin - 2.0 * err;
        const double mu = f.fx * (2.0 * err / zl + xabs * 2.0 * err / (zl * zl)) +
                          1e-9 * (fabs(umin) + fabs(umax) + fabs(f.cx)) + 1e-6;
        const double mv = f.fy * (2.0 * err / zl + yabs * 2.0 * err / (zl * zl)) +
                          1e-9 * (fabs(vmin) + fabs(vmax) + fabs(f.cy)) + 1e-6;
        const double fu0 = floor(umin - mu + 0.5), fu1 = floor(umax + mu + 0.5);
        const double fv0 = floor(vmin - mv + 0.5), fv1 = floor(vmax + mv + 0.5);
        if (fu1 < 0.0 || fv1 < 0.0 || fu0 > (double)(f.width - 1) || fv0 > (double)(f.height - 1))
            return false;  // outside the image (:113)
        u0 = fu0 < 0.0 ? 0 : (int64_t)fu0;
        v0 = fv0 < 0.0 ? 0 : (int64_t)fv0;
        u1 = fu1 > (double)(f.width - 1) ? f.width - 1 : (int64_t)fu1;
        v1 = fv1 > (double)(f.height - 1) ? f.height - 1 : (int64_t)fv1;
    }
    const double dmax = rect_max_depth(mip, m, u0, u1, v0, v1);
    if (!(dmax > 0.0)) return false;  // no valid depth reachable (:116)

    // sdf = d - dist / ray_scale < -tau for every voxel (:125-127)?
    double dd2 = 0.0;
    for (int a = 0; a < 3; ++a) {
        const double lo = gmin[a] - f.cam.v[a], hi = f.cam.v[a] - gmax[a];
        const double s = fmax(fmax(lo, hi), 0.0);
        dd2 += s * s;
    }
    const double dist_lb = sqrt(dd2) * (1.0 - 1e-12);
    const double ax = fmax(fabs((double)u0 - f.cx), fabs((double)u1 - f.cx)) / f.fx;
    const double ay = fmax(fabs((double)v0 - f.cy), fabs((double)v1 - f.cy)) / f.fy;
    const double rs_ub = sqrt(ax * ax + ay * ay + 1.0) * (1.0 + 1e-12);
    const double q_lb = dist_lb / rs_ub;
    const double margin = 1e-9 * (dmax + q_lb + f.tau) + 1e-12;
    if (dmax - q_lb < -f.tau - margin) return false;
    return true;
}

__global__ void __launch_bounds__(256) brick_cull_kernel(
    const __grid_constant__ VolumeTable vt, const __grid_constant__ BrickTable bt,
    const __grid_constant__ FrameGeom f, const __grid_constant__ MipDesc m,
    const unsigned long long *__restrict__ mip, uint32_t *__restrict__ active,
    unsigned int *__restrict__ active_count, const int no_cull) {
    const int64_t total = bt.offset[bt.count];
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool keep = false;
    if (g < total) {
        const int v = find_volume(bt, g);
        const int64_t local = g - bt.offset[v], nb = bt.nb[v];
        keep = no_cull || brick_may_update(vt.vol[v], local % nb, (local / nb) % nb,
                                           local / (nb * nb), f, mip, m);
    }
    // warp-aggregated append (list order is irrelevant: voxels are independent)
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (mask) {
        const int lane = threadIdx.x & 31;
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(active_count, (unsigned)__popc(mask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) active[base + __popc(mask & ((1u << lane) - 1u))] = (uint32_t)g;
    }
}

// ---------------------------------------------------------------------------
// 3. exact per-voxel update over the surviving bricks
// ---------------------------------------------------------------------------

// _kernels.py:99-133 for one voxel; returns 1 when the voxel was written.
__device__ __forceinline__ int update_voxel(float2 *__restrict__ vox, int64_t lin, double gx,
                                            double gy, double gz,
                                            const double2 *__restrict__ table,
                                            const FrameGeom &f) {
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
    const double2 px = __ldg(&table[(int64_t)vf * f.width + (int64_t)uf]);
    const double d = px.x;                                                      // :115
    if (!(d > 0.0)) return 0;                                                   // :116
    const double ddx = dsub(gx, f.cam.v[0]), ddy = dsub(gy, f.cam.v[1]),
                 ddz = dsub(gz, f.cam.v[2]);                                    // :121-123
    const double dist = dsqrt(dadd(dadd(dmul(ddx, ddx), dmul(ddy, ddy)), dmul(ddz, ddz)));
    const double sdf = dsub(d, ddiv(dist, px.y));                               // :125
    if (sdf < -f.tau) return 0;                                                 // :126
    const double clamped = sdf < f.tau ? sdf : f.tau;                           // :128
    const float2 old = vox[lin];
    // numba types float(f32) as float32: the product is a float32 op (:129-132)
    const float wv = fmulr(old.y, old.x);
    const double w_sum = dadd((double)old.y, f.sw);                             // :131
    const double t_new = ddiv(dadd((double)wv, dmul(f.sw, clamped)), w_sum);    // :132
    const double w_new = f.max_w < w_sum ? f.max_w : w_sum;                     // :133
    vox[lin] = make_float2(__double2float_rn(t_new), __double2float_rn(w_new));
    return 1;
}

__global__ void __launch_bounds__(256) brick_update_kernel(
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
                    updates += update_voxel(vox, vox_index(n, z, y, x), gx, gy, gz, table, f);
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

__global__ void brick_stats_kernel(const unsigned int *__restrict__ active_count,
                                   unsigned long long total, unsigned long long *stats) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        stats[TF_STAT_ACTIVE_BRICKS] += *active_count;
        stats[TF_STAT_TOTAL_BRICKS] += total;
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

struct IntegrateLayout {
    size_t table_off, mip_off, count_off, active_off, total;
};

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

static IntegrateLayout layout_for(int64_t total_bricks_max, const TfCamera *cam) {
    const MipDesc m = make_mip(cam->width, cam->height);
    IntegrateLayout L{};
    size_t off = 0;
    L.table_off = off;
    off = align_up(off + (size_t)(cam->width * cam->height) * sizeof(double2), 256);
    L.mip_off = off;
    off = align_up(off + (size_t)m.total * sizeof(unsigned long long), 256);
    L.count_off = off;
    off = align_up(off + 256, 256);
    L.active_off = off;
    off = align_up(off + (size_t)total_bricks_max * sizeof(uint32_t), 256);
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

extern "C" int tf_integrate(const TfVolume *vols, int nvol, const double *depth,
                            const TfCamera *cam, const double r_cw[9], const double t_cw[3],
                            const double cam_center[3], double tau, double max_weight,
                            double sample_weight, void *workspace, size_t workspace_bytes,
                            uint64_t *stats, void *stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    if (nvol == 0) return TF_OK;
    if (!vols || nvol < 0 || !depth || !cam || !r_cw || !t_cw || !cam_center || !workspace)
        return tf_set_error(TF_EINVAL, "tf_integrate: null argument");
    if (cam->width <= 0 || cam->height <= 0)
        return tf_set_error(TF_EINVAL, "tf_integrate: bad image size");
    for (int v = 0; v < nvol; ++v)
        if (!vols[v].voxels_dev || vols[v].n < 2 || !(vols[v].voxel_size > 0.0))
            return tf_set_error(TF_EINVAL, "tf_integrate: bad volume %d", v);
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
    unsigned long long *mip = (unsigned long long *)(ws + L.mip_off);
    unsigned int *count = (unsigned int *)(ws + L.count_off);
    uint32_t *active = (uint32_t *)(ws + L.active_off);
    const MipDesc m = make_mip(cam->width, cam->height);

    void *prof_all = tf_profile_begin(TF_PROF_INTEGRATE_ALL, stream);
    if (cudaMemsetAsync(mip, 0, (size_t)m.total * sizeof(unsigned long long), stream) != cudaSuccess)
        return tf_set_error(TF_ECUDA, "tf_integrate: memset failed");
    dim3 pblock(kTile, kTile);
    dim3 pgrid((unsigned)m.tiles_x[0], (unsigned)m.tiles_y[0]);
    frame_prep_kernel<<<pgrid, pblock, 0, stream>>>(depth, table, mip, m, cam->fx, cam->fy,
                                                    cam->cx, cam->cy, cam->width, cam->height);
    int rc = tf_check_launch("frame_prep_kernel");
    if (rc) return rc;

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
        if (cudaMemsetAsync(count, 0, sizeof(unsigned int), stream) != cudaSuccess)
            return tf_set_error(TF_ECUDA, "tf_integrate: memset failed");
        const unsigned cull_blocks = (unsigned)((off + 255) / 256);
        brick_cull_kernel<<<cull_blocks, 256, 0, stream>>>(vt, bt, f, m, mip, active, count,
                                                           (tf_debug_flags() & TF_DEBUG_NO_CULL) ? 1 : 0);
        if ((rc = tf_check_launch("brick_cull_kernel"))) return rc;
        void *prof = tf_profile_begin(TF_PROF_INTEGRATE_UPDATE, stream);
        brick_update_kernel<<<(unsigned)sms * 8, 256, 0, stream>>>(
            vt, bt, f, table, active, count, (unsigned long long *)stats);
        tf_profile_end(prof, stream);
        if ((rc = tf_check_launch("brick_update_kernel"))) return rc;
        if (stats) {
            brick_stats_kernel<<<1, 32, 0, stream>>>(count, (unsigned long long)off,
                                                     (unsigned long long *)stats);
            if ((rc = tf_check_launch("brick_stats_kernel"))) return rc;
        }
    }
    tf_profile_end(prof_all, stream);
    return TF_OK;
}
