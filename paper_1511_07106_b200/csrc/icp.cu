// Projective point-to-plane ICP kernels (sm_100a).
//
//   vertex_normal_kernel — geometry.depth_to_vertices + compute_normals
//                          (reference geometry.py:261-302) for one pyramid
//                          level, reading the full-resolution depth at stride
//                          2^level (DepthFrame.downsampled, :256-258);
//   icp_terms_kernel     — the per-pixel part of tracking._solve_step
//                          (tracking.py:76-108): transform, project, gate,
//                          and accumulate A^T A (21), A^T r (6), sum r^2 and the
//                          inlier count with a fixed-shape FP64 shuffle tree;
//   icp_finish_kernel    — fixed-order sum of the per-block partials.
//
// Per-pixel arithmetic reproduces what numpy does on the reference host:
// (N,3)@(3,3) goes through OpenBLAS dgemm, an FMA chain over k; a 3-term
// einsum dot is (p0 + p2) + p1; np.cross / np.linalg.norm are plain.  The
// inlier decisions therefore match the reference bit for bit; only the
// summation order of the 29 sums (BLAS a.T @ a) differs.
#include <math.h>

#include "tf_common.cuh"

namespace tf {

constexpr int kIcpThreads = 256;
constexpr int kIcpTerms = 29;

// numpy (N,3) @ R.T via OpenBLAS: acc = s0*R0; acc = fma(s1,R1,acc); acc = fma(s2,R2,acc)
__device__ __forceinline__ void rot_apply(const double *R, const double s[3], double o[3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i) o[i] = dfma(s[2], R[3 * i + 2], dfma(s[1], R[3 * i + 1], dmul(s[0], R[3 * i])));
}

// np.einsum("...i,...i->...") over 3 terms: (p0 + p2) + p1
__device__ __forceinline__ double dot_np(const double a[3], const double b[3]) {
    return dadd(dadd(dmul(a[0], b[0]), dmul(a[2], b[2])), dmul(a[1], b[1]));
}

struct LevelCam {
    double fx, fy, cx, cy;
    int64_t width, height;
};

__device__ __forceinline__ void vertex_at(const double *__restrict__ depth, int64_t full_w,
                                          int stride, const LevelCam &c, int64_t x, int64_t y,
                                          double v[3], bool &ok) {
    const double d = depth[(y * stride) * full_w + x * stride];
    ok = d > 0.0;
    if (ok) {
        // pixel_rays (geometry.py:65-67) times depth (:269)
        v[0] = dmul(ddiv(dsub((double)x, c.cx), c.fx), d);
        v[1] = dmul(ddiv(dsub((double)y, c.cy), c.fy), d);
        v[2] = dmul(1.0, d);
    } else {
        v[0] = v[1] = v[2] = 0.0;  // :271
    }
}

__global__ void __launch_bounds__(256) vertex_normal_kernel(
    const double *__restrict__ depth, int64_t full_w, int stride, const LevelCam c,
    double *__restrict__ verts, double *__restrict__ norms, uint8_t *__restrict__ valid) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t y = blockIdx.y;
    if (x >= c.width || y >= c.height) return;
    const int64_t p = y * c.width + x;
    double v0[3];
    bool ok0;
    vertex_at(depth, full_w, stride, c, x, y, v0, ok0);
    verts[3 * p + 0] = v0[0];
    verts[3 * p + 1] = v0[1];
    verts[3 * p + 2] = v0[2];
    double nr[3] = {0.0, 0.0, 0.0};
    bool good = false;
    if (ok0 && x + 1 < c.width && y + 1 < c.height) {
        double vx[3], vy[3];
        bool okx, oky;
        vertex_at(depth, full_w, stride, c, x + 1, y, vx, okx);
        vertex_at(depth, full_w, stride, c, x, y + 1, vy, oky);
        if (okx && oky) {                                             // :289-292
            const double a[3] = {dsub(vx[0], v0[0]), dsub(vx[1], v0[1]), dsub(vx[2], v0[2])};
            const double b[3] = {dsub(vy[0], v0[0]), dsub(vy[1], v0[1]), dsub(vy[2], v0[2])};
            const double c0 = dsub(dmul(a[1], b[2]), dmul(a[2], b[1]));  // np.cross
            const double c1 = dsub(dmul(a[2], b[0]), dmul(a[0], b[2]));
            const double c2 = dsub(dmul(a[0], b[1]), dmul(a[1], b[0]));
            const double nn = dsqrt(dadd(dadd(dmul(c0, c0), dmul(c1, c1)), dmul(c2, c2)));
            if (nn > 0.0) {                                           // :293
                double u[3] = {ddiv(c0, nn), ddiv(c1, nn), ddiv(c2, nn)};
                if (dot_np(u, v0) > 0.0) {                            // :298-299
                    u[0] = -u[0];
                    u[1] = -u[1];
                    u[2] = -u[2];
                }
                nr[0] = u[0];
                nr[1] = u[1];
                nr[2] = u[2];
                good = true;
            }
        }
    }
    norms[3 * p + 0] = nr[0];
    norms[3 * p + 1] = nr[1];
    norms[3 * p + 2] = nr[2];
    valid[p] = good ? 1 : 0;
}

struct IcpParams {
    Mat3 r_est, r_ref;
    Vec3 t_est, t_ref;
    LevelCam cam;
    int64_t src_w, src_h, mdl_w, mdl_h;
    int stride;
    double max_d2, cos_min;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dadd(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

__global__ void __launch_bounds__(kIcpThreads) icp_terms_kernel(
    const double *__restrict__ sv, const double *__restrict__ sn, const uint8_t *__restrict__ sok,
    const double *__restrict__ md, const double *__restrict__ mv, const double *__restrict__ mn,
    const __grid_constant__ IcpParams P, double *__restrict__ partials) {
    const int64_t npix = P.src_w * P.src_h;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double a[6] = {0, 0, 0, 0, 0, 0}, r = 0.0, cnt = 0.0;
    if (p < npix && sok[p]) {
        const double s[3] = {sv[3 * p], sv[3 * p + 1], sv[3 * p + 2]};
        const double snr[3] = {sn[3 * p], sn[3 * p + 1], sn[3 * p + 2]};
        double pw[3], nw[3], pr[3];
        rot_apply(P.r_est.m, s, pw);                                  // :76
        for (int i = 0; i < 3; ++i) pw[i] = dadd(pw[i], P.t_est.v[i]);
        rot_apply(P.r_est.m, snr, nw);                                // :77
        rot_apply(P.r_ref.m, pw, pr);                                 // :80
        for (int i = 0; i < 3; ++i) pr[i] = dadd(pr[i], P.t_ref.v[i]);
        const double z = pr[2];
        bool ok = z > 1.0e-9;                                         // :82
        double uf = 0.0, vf = 0.0;
        if (ok) {
            const double u = dadd(ddiv(dmul(P.cam.fx, pr[0]), z), P.cam.cx);  // :84
            const double v = dadd(ddiv(dmul(P.cam.fy, pr[1]), z), P.cam.cy);  // :85
            uf = floor(dadd(u, 0.5));
            vf = floor(dadd(v, 0.5));
            ok = uf >= 0.0 && uf < (double)P.cam.width && vf >= 0.0 && vf < (double)P.cam.height;
        }
        if (ok) {
            const int64_t mx = (int64_t)uf * P.stride, my = (int64_t)vf * P.stride;
            ok = mx < P.mdl_w && my < P.mdl_h;
            if (ok) {
                const int64_t m = my * P.mdl_w + mx;
                ok = isfinite(md[m]);                                 // RayMap.valid (tsdf.py:178-180)
                if (ok) {
                    const double q[3] = {mv[3 * m], mv[3 * m + 1], mv[3 * m + 2]};
                    const double nm[3] = {mn[3 * m], mn[3 * m + 1], mn[3 * m + 2]};
                    const double diff[3] = {dsub(pw[0], q[0]), dsub(pw[1], q[1]), dsub(pw[2], q[2])};
                    ok = dot_np(diff, diff) <= P.max_d2 && dot_np(nm, nw) >= P.cos_min;  // :96-98
                    if (ok) {
                        const double e[3] = {dsub(q[0], pw[0]), dsub(q[1], pw[1]), dsub(q[2], pw[2])};
                        r = dot_np(nm, e);                            // :105
                        a[0] = dsub(dmul(pw[1], nm[2]), dmul(pw[2], nm[1]));  // :106
                        a[1] = dsub(dmul(pw[2], nm[0]), dmul(pw[0], nm[2]));
                        a[2] = dsub(dmul(pw[0], nm[1]), dmul(pw[1], nm[0]));
                        a[3] = nm[0];
                        a[4] = nm[1];
                        a[5] = nm[2];
                        cnt = 1.0;
                    }
                }
            }
        }
    }
    // 29 terms: A^T A upper triangle, A^T r, r^2, count
    double t[kIcpTerms];
    int k = 0;
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = i; j < 6; ++j) t[k++] = dmul(a[i], a[j]);
#pragma unroll
    for (int i = 0; i < 6; ++i) t[21 + i] = dmul(a[i], r);
    t[27] = dmul(r, r);
    t[28] = cnt;
    __shared__ double wsum[kIcpThreads / 32][kIcpTerms];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < kIcpTerms; ++i) {
        const double s = warp_sum(t[i]);
        if (lane == 0) wsum[w][i] = s;
    }
    __syncthreads();
    if (threadIdx.x < kIcpTerms) {
        double s = 0.0;
        for (int i = 0; i < kIcpThreads / 32; ++i) s = dadd(s, wsum[i][threadIdx.x]);
        partials[(int64_t)blockIdx.x * kIcpTerms + threadIdx.x] = s;
    }
}

// warp k sums term k over all block partials in a fixed order
__global__ void icp_finish_kernel(const double *__restrict__ partials, int64_t nblocks,
                                  double *__restrict__ out) {
    const int lane = threadIdx.x & 31, k = threadIdx.x >> 5;
    if (k >= kIcpTerms) return;
    double s = 0.0;
    for (int64_t b = lane; b < nblocks; b += 32) s = dadd(s, partials[b * kIcpTerms + k]);
    s = warp_sum(s);
    if (lane == 0) out[k] = s;
}

}  // namespace tf

using namespace tf;

extern "C" int tf_vertex_normal_map(const double *depth, int64_t full_w, int64_t full_h, int level,
                                    const TfCamera *cam, double *verts, double *norms,
                                    uint8_t *valid, void *stream_) {
    if (!depth || !cam || !verts || !norms || !valid || level < 0 || level > 20)
        return tf_set_error(TF_EINVAL, "tf_vertex_normal_map: bad argument");
    const int stride = 1 << level;
    const int64_t lw = (full_w + stride - 1) / stride, lh = (full_h + stride - 1) / stride;
    if (cam->width != lw || cam->height != lh)
        return tf_set_error(TF_EINVAL,
                            "tf_vertex_normal_map: depth shape (%lld, %lld) does not match "
                            "intrinsics %lldx%lld",
                            (long long)lh, (long long)lw, (long long)cam->height,
                            (long long)cam->width);
    LevelCam c{cam->fx, cam->fy, cam->cx, cam->cy, cam->width, cam->height};
    dim3 grid((unsigned)((lw + 255) / 256), (unsigned)lh);
    vertex_normal_kernel<<<grid, 256, 0, (cudaStream_t)stream_>>>(depth, full_w, stride, c, verts,
                                                                  norms, valid);
    return tf_check_launch("vertex_normal_kernel");
}

extern "C" size_t tf_icp_workspace_size(int64_t src_pixels) {
    const int64_t blocks = (src_pixels + kIcpThreads - 1) / kIcpThreads;
    return (size_t)(blocks > 0 ? blocks : 1) * kIcpTerms * sizeof(double);
}

extern "C" int tf_icp_reduce(const double *sv, const double *sn, const uint8_t *sok, int64_t sw,
                             int64_t sh, const double *md, const double *mv, const double *mn,
                             int64_t mw, int64_t mh, int level, const TfCamera *cam,
                             const double r_est[9], const double t_est[3], const double r_ref[9],
                             const double t_ref[3], double max_d2, double cos_min,
                             void *workspace, size_t workspace_bytes, double *out29,
                             void *stream_) {
    if (!sv || !sn || !sok || !md || !mv || !mn || !cam || !r_est || !t_est || !r_ref || !t_ref ||
        !workspace || !out29 || level < 0 || level > 20 || sw <= 0 || sh <= 0)
        return tf_set_error(TF_EINVAL, "tf_icp_reduce: bad argument");
    if (workspace_bytes < tf_icp_workspace_size(sw * sh))
        return tf_set_error(TF_EINVAL, "tf_icp_reduce: workspace too small");
    IcpParams P{};
    for (int i = 0; i < 9; ++i) {
        P.r_est.m[i] = r_est[i];
        P.r_ref.m[i] = r_ref[i];
    }
    for (int i = 0; i < 3; ++i) {
        P.t_est.v[i] = t_est[i];
        P.t_ref.v[i] = t_ref[i];
    }
    P.cam = LevelCam{cam->fx, cam->fy, cam->cx, cam->cy, cam->width, cam->height};
    P.src_w = sw;
    P.src_h = sh;
    P.mdl_w = mw;
    P.mdl_h = mh;
    P.stride = 1 << level;
    P.max_d2 = max_d2;
    P.cos_min = cos_min;
    const int64_t blocks = (sw * sh + kIcpThreads - 1) / kIcpThreads;
    double *partials = (double *)workspace;
    cudaStream_t stream = (cudaStream_t)stream_;
    icp_terms_kernel<<<(unsigned)blocks, kIcpThreads, 0, stream>>>(sv, sn, sok, md, mv, mn, P,
                                                                   partials);
    int rc = tf_check_launch("icp_terms_kernel");
    if (rc) return rc;
    icp_finish_kernel<<<1, 32 * kIcpTerms, 0, stream>>>(partials, blocks, out29);
    return tf_check_launch("icp_finish_kernel");
}
