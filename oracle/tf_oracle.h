/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the tilefusion hot path.
 *
 * A plain-C restatement of the reference algorithms (tilefusion, numba/numpy),
 * used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs as the checker and the CPU baseline.  Nothing in the
 * product package links or calls this library.
 *
 * Parity pinning: validated against the live reference package and against
 * golden fixtures generated from it (tests/golden/make_golden.py,
 * tests/test_oracle_golden.py).
 *
 * Arithmetic rules:
 *   - compiled with -ffp-contract=off: every a*b+c is two rounded ops, exactly
 *     like the numba kernels (0 vfmadd in their JIT asm);
 *   - where the reference goes through numpy/OpenBLAS, the restatement uses
 *     the order those libraries were measured to use here: (N,3)@(3,3) is an
 *     FMA chain over k (OpenBLAS Haswell dgemm), a 3-term einsum dot is
 *     (p0 + p2) + p1, np.cross and np.linalg.norm are plain.
 */
#ifndef TF_ORACLE_H
#define TF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* _kernels.integrate_kernel (_kernels.py:71-133).  Separate [z][y][x] f32
 * tsdf / weight arrays like TsdfSubvolume (tsdf.py:72-78).  Returns the number
 * of voxel updates (voxels passing every gate). */
int64_t tfo_integrate(float *tsdf, float *weight, int64_t n, const int64_t ht[3],
                      double voxel_size, const double *depth, int64_t height,
                      int64_t width, const double r_cw[9], const double t_cw[3],
                      const double cam_center[3], double fx, double fy, double cx,
                      double cy, double tau, double max_weight,
                      double sample_weight, int nthreads);

/* _kernels._sample (_kernels.py:28-68).  Returns 1 and writes *value when the
 * 2x2x2 neighbourhood is inside and observed, else returns 0. */
int tfo_sample(const float *tsdf, const float *weight, int64_t n, double qx,
               double qy, double qz, double *value);

/* _kernels.raycast_kernel (_kernels.py:266-451), merging into the maps in
 * place with _hit_wins (:246-263).  Returns the number of _sample calls. */
int64_t tfo_raycast(const float *tsdf, const float *weight, int64_t n,
                    const int64_t ht[3], double voxel_size, double tau,
                    int64_t coarse_step, const double r_wc[9],
                    const double cam_center[3], double fx, double fy, double cx,
                    double cy, int64_t height, int64_t width, double *out_dist,
                    double *out_vert, double *out_norm, int nthreads);

/* _kernels.extract_bound / extract_kernel (_kernels.py:454-578). */
int64_t tfo_extract_bound(const float *tsdf, const float *weight, int64_t n);
int64_t tfo_extract(const float *tsdf, const float *weight, int64_t n,
                    const int64_t ht[3], double voxel_size, double *out_verts,
                    double *out_norms);

/* geometry.depth_to_vertices + compute_normals (geometry.py:261-302) for one
 * pyramid level.  valid = vertex_ok & normal_ok (geometry.py:313-317). */
void tfo_vertex_normal_map(const double *depth, int64_t height, int64_t width,
                           double fx, double fy, double cx, double cy,
                           double *verts, double *norms, uint8_t *valid);

/* Per-pixel part of tracking._solve_step (tracking.py:76-108), summed in
 * pixel order.  out[0..20] = upper triangle of A^T A (row major),
 * out[21..26] = A^T r, out[27] = sum r^2, out[28] = count. */
void tfo_icp_reduce(const double *src_v, const double *src_n,
                    const uint8_t *src_valid, int64_t src_h, int64_t src_w,
                    const double *mdl_v, const double *mdl_n,
                    const uint8_t *mdl_valid, int64_t mdl_h, int64_t mdl_w,
                    const double r_est[9], const double t_est[3],
                    const double r_ref[9], const double t_ref[3], double fx,
                    double fy, double cx, double cy, int64_t img_w,
                    int64_t img_h, double max_d2, double cos_min, double *out);

/* volumes.bin_endpoints (volumes.py:305-331): per-pixel endpoint cell (i,j,k)
 * in block units, written for valid pixels in row-major pixel order.
 * Returns the number of valid pixels. */
int64_t tfo_endpoint_cells(const double *depth, int64_t height, int64_t width,
                           double fx, double fy, double cx, double cy,
                           const double r_wc[9], const double t_wc[3],
                           double block_side, int64_t *cells);

#ifdef __cplusplus
}
#endif
#endif
