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
    const double *state;  // device-resident tracking: estimate + flags (kSt*), else null
};

// device tracking state (doubles): estimate R (row-major) and t, flags, last
// successful step's count and rms
enum : int { kStR = 0, kStT = 9, kStLost = 12, kStCount = 13, kStRms = 14, kStLevelDone = 15,
             kStSize = 16 };

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dadd(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

constexpr int kFoldThreads = 256;

// The 29 sums over the block partials ([nblocks][29] doubles) by one block of
// kFoldThreads threads, in a fixed order: thread t folds blocks t, t + 256,
// ... (all 29 terms at once: independent loads, many in flight), then the
// shuffle tree per warp, then the warps in order.  Deterministic; the same
// function serves tf_icp_reduce and tf_icp_track.
__device__ void fold_partials(const double *__restrict__ partials, int64_t nblocks, double *sums) {
    __shared__ double wpart[kFoldThreads / 32][kIcpTerms];
    double acc[kIcpTerms];
#pragma unroll
    for (int k = 0; k < kIcpTerms; ++k) acc[k] = 0.0;
    for (int64_t b = threadIdx.x; b < nblocks; b += kFoldThreads) {
        const double *p = partials + b * kIcpTerms;
#pragma unroll
        for (int k = 0; k < kIcpTerms; ++k) acc[k] = dadd(acc[k], p[k]);
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < kIcpTerms; ++k) {
        const double s = warp_sum(acc[k]);
        if (lane == 0) wpart[w][k] = s;
    }
    __syncthreads();
    if (threadIdx.x < kIcpTerms) {
        double s = 0.0;
        for (int i = 0; i < kFoldThreads / 32; ++i) s = dadd(s, wpart[i][threadIdx.x]);
        sums[threadIdx.x] = s;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kIcpThreads) icp_terms_kernel(
    const double *__restrict__ sv, const double *__restrict__ sn, const uint8_t *__restrict__ sok,
    const double *__restrict__ md, const double *__restrict__ mv, const double *__restrict__ mn,
    const __grid_constant__ IcpParams P, double *__restrict__ partials) {
    const int64_t npix = P.src_w * P.src_h;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double a[6] = {0, 0, 0, 0, 0, 0}, r = 0.0, cnt = 0.0;
    double Re[9], te[3];
    bool live = true;
    if (P.state) {  // device-resident tracking: nothing to do once lost or converged
        live = P.state[kStLost] == 0.0 && P.state[kStLevelDone] == 0.0;
        for (int i = 0; i < 9; ++i) Re[i] = P.state[kStR + i];
        for (int i = 0; i < 3; ++i) te[i] = P.state[kStT + i];
    } else {
        for (int i = 0; i < 9; ++i) Re[i] = P.r_est.m[i];
        for (int i = 0; i < 3; ++i) te[i] = P.t_est.v[i];
    }
    if (!live) return;
    if (p < npix && sok[p]) {
        const double s[3] = {sv[3 * p], sv[3 * p + 1], sv[3 * p + 2]};
        const double snr[3] = {sn[3 * p], sn[3 * p + 1], sn[3 * p + 2]};
        double pw[3], nw[3], pr[3];
        rot_apply(Re, s, pw);                                         // :76
        for (int i = 0; i < 3; ++i) pw[i] = dadd(pw[i], te[i]);
        rot_apply(Re, snr, nw);                                       // :77
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
            ok = mx < P.mdl_w && my < P.mdl_h && TF_IN_BOUNDS(mx >= 0 && my >= 0);
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

// the 29 sums of tf_icp_reduce (fold_partials' order)
__global__ void __launch_bounds__(kFoldThreads) icp_finish_kernel(const double *__restrict__ partials,
                                                                  int64_t nblocks, double *__restrict__ out) {
    __shared__ double sums[kIcpTerms];
    fold_partials(partials, nblocks, sums);
    if (threadIdx.x < kIcpTerms) out[threadIdx.x] = sums[threadIdx.x];
}


// ---- device-resident tracking (track(), tracking.py:123-196) --------------
//
// One single-warp kernel per ICP iteration folds the block partials (same
// fixed order as icp_finish_kernel) and does the host part of _solve_step
// (tracking.py:100-120) and the pose update (:178-183) in FP64 on the device:
// pair minimum, cond(A^T A) > 1e12 gate, LU solve with partial pivoting (as
// LAPACK gesv), finiteness, Rodrigues, re-orthonormalisation to the polar
// factor (the U V^T of the reference's SVD), convergence test.  No host round
// trip per iteration: the whole pyramid is queued at once and later kernels
// return immediately once the state says lost / level converged.  Deltas
// agree with numpy to rounding (the parity bar for ICP is 1e-5 m / 1e-6 rad;
// counts are exact).

// 6x6 symmetric Jacobi eigenvalues (rare path: only when the cheap bound
// cannot decide the conditioning gate)
__device__ void sym6_eigenvalues(const double A[36], double ev[6]) {
    double a[36];
    for (int i = 0; i < 36; ++i) a[i] = A[i];
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0;
        for (int pp = 0; pp < 6; ++pp)
            for (int q = pp + 1; q < 6; ++q) off += a[pp * 6 + q] * a[pp * 6 + q];
        if (off == 0.0) break;
        for (int pp = 0; pp < 6; ++pp)
            for (int q = pp + 1; q < 6; ++q) {
                const double apq = a[pp * 6 + q];
                if (apq == 0.0) continue;
                const double theta = (a[q * 6 + q] - a[pp * 6 + pp]) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
                for (int k = 0; k < 6; ++k) {  // columns p, q
                    const double akp = a[k * 6 + pp], akq = a[k * 6 + q];
                    a[k * 6 + pp] = c * akp - sn * akq;
                    a[k * 6 + q] = sn * akp + c * akq;
                }
                for (int k = 0; k < 6; ++k) {  // rows p, q
                    const double apk = a[pp * 6 + k], aqk = a[q * 6 + k];
                    a[pp * 6 + k] = c * apk - sn * aqk;
                    a[q * 6 + k] = sn * apk + c * aqk;
                }
            }
    }
    for (int i = 0; i < 6; ++i) ev[i] = a[i * 6 + i];
}

// LU with partial pivoting of A (in place) -> false if singular
__device__ bool lu6(double A[36], int piv[6]) {
    for (int k = 0; k < 6; ++k) {
        int m = k;
        for (int i = k + 1; i < 6; ++i)
            if (fabs(A[i * 6 + k]) > fabs(A[m * 6 + k])) m = i;
        piv[k] = m;
        if (A[m * 6 + k] == 0.0) return false;
        if (m != k)
            for (int j = 0; j < 6; ++j) {
                const double t = A[k * 6 + j];
                A[k * 6 + j] = A[m * 6 + j];
                A[m * 6 + j] = t;
            }
        const double inv = 1.0 / A[k * 6 + k];
        for (int i = k + 1; i < 6; ++i) {
            const double l = A[i * 6 + k] * inv;
            A[i * 6 + k] = l;
            for (int j = k + 1; j < 6; ++j) A[i * 6 + j] -= l * A[k * 6 + j];
        }
    }
    return true;
}

__device__ void lu6_solve(const double LU[36], const int piv[6], double b[6]) {
    for (int k = 0; k < 6; ++k)
        if (piv[k] != k) {
            const double t = b[k];
            b[k] = b[piv[k]];
            b[piv[k]] = t;
        }
    for (int i = 1; i < 6; ++i)
        for (int j = 0; j < i; ++j) b[i] -= LU[i * 6 + j] * b[j];
    for (int i = 5; i >= 0; --i) {
        for (int j = i + 1; j < 6; ++j) b[i] -= LU[i * 6 + j] * b[j];
        b[i] /= LU[i * 6 + i];
    }
}

// np.linalg.cond(A) > 1e12 for symmetric positive semi-definite A; LU of A
// given.  ||A||_F ||A^-1||_F >= cond_2 >= it / 6 decides almost every case;
// the rest (and any doubt) takes the Jacobi eigenvalues.
__device__ bool ill_conditioned(const double A[36], const double LU[36], const int piv[6]) {
    double fa = 0.0, fi = 0.0;
    for (int i = 0; i < 36; ++i) fa += A[i] * A[i];
    for (int c = 0; c < 6; ++c) {
        double e[6] = {0, 0, 0, 0, 0, 0};
        e[c] = 1.0;
        lu6_solve(LU, piv, e);
        for (int i = 0; i < 6; ++i) fi += e[i] * e[i];
    }
    const double upper = sqrt(fa) * sqrt(fi);
    if (isfinite(upper) && upper <= 1.0e12 * (1.0 - 1e-9)) return false;
    if (isfinite(upper) && upper / 6.0 > 1.0e12 * (1.0 + 1e-9)) return true;
    double ev[6];
    sym6_eigenvalues(A, ev);
    double lo = fabs(ev[0]), hi = fabs(ev[0]);
    for (int i = 1; i < 6; ++i) {
        lo = fmin(lo, fabs(ev[i]));
        hi = fmax(hi, fabs(ev[i]));
    }
    return !(hi / lo <= 1.0e12);  // lo == 0 -> inf -> ill-conditioned
}

// 3x3 helpers (row-major)
__device__ __forceinline__ void mat3_mul(const double A[9], const double B[9], double C[9]) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            C[i * 3 + j] = A[i * 3] * B[j] + A[i * 3 + 1] * B[3 + j] + A[i * 3 + 2] * B[6 + j];
}

// orthogonal polar factor of a near-rotation (= U V^T of its SVD): Newton
// X <- (X + X^-T) / 2, quadratic from the first step
__device__ void polar3(double X[9]) {
    for (int it = 0; it < 8; ++it) {
        const double c00 = X[4] * X[8] - X[5] * X[7], c01 = X[5] * X[6] - X[3] * X[8],
                     c02 = X[3] * X[7] - X[4] * X[6];
        const double c10 = X[2] * X[7] - X[1] * X[8], c11 = X[0] * X[8] - X[2] * X[6],
                     c12 = X[1] * X[6] - X[0] * X[7];
        const double c20 = X[1] * X[5] - X[2] * X[4], c21 = X[2] * X[3] - X[0] * X[5],
                     c22 = X[0] * X[4] - X[1] * X[3];
        const double det = X[0] * c00 + X[1] * c01 + X[2] * c02;
        const double inv = 1.0 / det;  // X^-T = cofactor / det
        const double cof[9] = {c00, c01, c02, c10, c11, c12, c20, c21, c22};
        double change = 0.0;
        for (int i = 0; i < 9; ++i) {
            const double nx = 0.5 * (X[i] + cof[i] * inv);
            change = fmax(change, fabs(nx - X[i]));
            X[i] = nx;
        }
        if (change < 1e-17) break;
    }
}

__device__ void icp_apply_delta(const double b[6], double step_eps, double *__restrict__ st);

// the host part of _solve_step and the pose update for one thread (the
// reference order, operation for operation)
__device__ void icp_step_serial(const double *sums, int min_pairs, double step_eps,
                                             double *__restrict__ st) {
    const int count = (int)llrint(sums[28]);
    if (count < min_pairs) {  // :101-102
        st[kStLost] = 1.0;
        return;
    }
    double A[36], LU[36], b[6];
    int kk = 0;
    for (int i = 0; i < 6; ++i)
        for (int j = i; j < 6; ++j) {
            A[i * 6 + j] = A[j * 6 + i] = sums[kk];
            ++kk;
        }
    for (int i = 0; i < 36; ++i) LU[i] = A[i];
    for (int i = 0; i < 6; ++i) b[i] = sums[21 + i];
    int piv[6];
    if (!lu6(LU, piv) || ill_conditioned(A, LU, piv)) {  // :111-112, LinAlgError
        st[kStLost] = 1.0;
        return;
    }
    lu6_solve(LU, piv, b);  // :114
    bool finite = true;
    for (int i = 0; i < 6; ++i) finite &= isfinite(b[i]);
    if (!finite) {  // :117
        st[kStLost] = 1.0;
        return;
    }
    st[kStCount] = (double)count;
    st[kStRms] = sqrt(sums[27] / (double)count);  // :119
    icp_apply_delta(b, step_eps, st);
}


// Pose update shared by both step variants: Rodrigues on delta[:3]
// (geometry.py:211-219) left-multiplied, re-orthonormalised (:178-181), the
// convergence test (:182-183).
__device__ void icp_apply_delta(const double b[6], double step_eps, double *__restrict__ st) {
    const double ang = sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
    double rot[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    if (ang != 0.0) {
        const double x = b[0] / ang, y = b[1] / ang, z = b[2] / ang;
        const double K[9] = {0.0, -z, y, z, 0.0, -x, -y, x, 0.0};
        double K2[9];
        mat3_mul(K, K, K2);
        const double sa = sin(ang), ca = 1.0 - cos(ang);
        for (int i = 0; i < 9; ++i) rot[i] += sa * K[i] + ca * K2[i];
    }
    double R[9], Rn[9], t[3];
    for (int i = 0; i < 9; ++i) R[i] = st[kStR + i];
    mat3_mul(rot, R, Rn);
    for (int i = 0; i < 3; ++i)
        t[i] = rot[i * 3] * st[kStT] + rot[i * 3 + 1] * st[kStT + 1] + rot[i * 3 + 2] * st[kStT + 2] + b[3 + i];
    polar3(Rn);
    for (int i = 0; i < 9; ++i) st[kStR + i] = Rn[i];
    for (int i = 0; i < 3; ++i) st[kStT + i] = t[i];
    double dn = 0.0;
    for (int i = 0; i < 6; ++i) dn += b[i] * b[i];
    if (sqrt(dn) < step_eps) st[kStLevelDone] = 1.0;
}

// One ICP iteration's host part on the device (tracking.py:100-120,
// :178-183): the 29 sums folded from the block partials (fold_partials), then
// one thread does the 6x6 work and the pose update (icp_step_serial).  A
// warp-parallel LU with the matrix in registers measured no faster: the step
// is a chain of dependent latencies either way (~18 us per launch).
__global__ void __launch_bounds__(kFoldThreads, 1) icp_step_kernel(const double *__restrict__ partials, int64_t nblocks, int min_pairs,
                                double step_eps, double *__restrict__ st) {
    if (st[kStLost] != 0.0 || st[kStLevelDone] != 0.0) return;
    __shared__ double sums[kIcpTerms];
    fold_partials(partials, nblocks, sums);
    if (threadIdx.x == 0) icp_step_serial(sums, min_pairs, step_eps, st);
}

__global__ void icp_level_start_kernel(double *st) { st[kStLevelDone] = 0.0; }

}  // namespace tf

using namespace tf;

TF_BOUNDS_READER(icp)

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
    icp_finish_kernel<<<1, kFoldThreads, 0, stream>>>(partials, blocks, out29);
    return tf_check_launch("icp_finish_kernel");
}

extern "C" size_t tf_icp_track_state_size(void) { return kStSize * sizeof(double); }

extern "C" int tf_icp_track(int nlevels, const double *const *src_verts, const double *const *src_norms,
                            const uint8_t *const *src_valid, const TfCamera *level_cams,
                            const int *iterations, const int *min_pairs, const double *md,
                            const double *mv, const double *mn, int64_t mw, int64_t mh,
                            const double r_ref[9], const double t_ref[3], const double r_init[9],
                            const double t_init[3], double max_d2, double cos_min, double step_eps,
                            void *workspace, size_t workspace_bytes, double *state, void *stream_) {
    if (nlevels < 1 || nlevels > 20 || !src_verts || !src_norms || !src_valid || !level_cams ||
        !iterations || !min_pairs || !md || !mv || !mn || !r_ref || !t_ref || !r_init || !t_init ||
        !workspace || !state)
        return tf_set_error(TF_EINVAL, "tf_icp_track: bad argument");
    if (workspace_bytes < tf_icp_workspace_size(level_cams[0].width * level_cams[0].height))
        return tf_set_error(TF_EINVAL, "tf_icp_track: workspace too small");
    cudaStream_t stream = (cudaStream_t)stream_;
    double init[kStSize] = {};
    for (int i = 0; i < 9; ++i) init[kStR + i] = r_init[i];
    for (int i = 0; i < 3; ++i) init[kStT + i] = t_init[i];
    // pageable source: the call returns once the bytes are staged, so the
    // stack array may go out of scope
    if (cudaMemcpyAsync(state, init, sizeof(init), cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return tf_set_error(TF_ECUDA, "tf_icp_track: state upload failed");
    double *partials = (double *)workspace;
    int rc = TF_OK;
    for (int level = nlevels - 1; level >= 0; --level) {  // coarsest first (:154)
        const TfCamera &cam = level_cams[level];
        IcpParams P{};
        for (int i = 0; i < 9; ++i) P.r_ref.m[i] = r_ref[i];
        for (int i = 0; i < 3; ++i) P.t_ref.v[i] = t_ref[i];
        P.cam = LevelCam{cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height};
        P.src_w = cam.width;
        P.src_h = cam.height;
        P.mdl_w = mw;
        P.mdl_h = mh;
        P.stride = 1 << level;
        P.max_d2 = max_d2;
        P.cos_min = cos_min;
        P.state = state;
        const int64_t blocks = (cam.width * cam.height + kIcpThreads - 1) / kIcpThreads;
        icp_level_start_kernel<<<1, 1, 0, stream>>>(state);
        if ((rc = tf_check_launch("icp_level_start_kernel"))) return rc;
        for (int it = 0; it < iterations[level]; ++it) {
            icp_terms_kernel<<<(unsigned)blocks, kIcpThreads, 0, stream>>>(
                src_verts[level], src_norms[level], src_valid[level], md, mv, mn, P, partials);
            if ((rc = tf_check_launch("icp_terms_kernel"))) return rc;
            icp_step_kernel<<<1, kFoldThreads, 0, stream>>>(partials, blocks, min_pairs[level], step_eps,
                                                            state);
            if ((rc = tf_check_launch("icp_step_kernel"))) return rc;
        }
    }
    return TF_OK;
}
