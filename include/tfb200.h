/*
 * tfb200 — C ABI of the B200-native tilefusion hot path (libtfb200.so).
 *
 * Each entry point replaces one operator of the reference package
 * (/root/reference/pkg/src/tilefusion, cited file:line) and is what a
 * ctypes / cffi binding of that operator binds (INTEGRATION.md shows the
 * stubs).  Conventions:
 *
 *   - every pointer named *_dev is caller-owned device memory on the current
 *     device (PyTorch tensors' data_ptr()); small matrices / vectors
 *     (r_*[9], t_*[3]) and descriptors are HOST memory read during the call;
 *   - calls are asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and never synchronise the device, allocate, or copy
 *     device->host; scratch comes from a caller workspace sized by the
 *     matching *_workspace_size() call;
 *   - the return value is 0 on success, a negative TF_E* code otherwise, with
 *     a message available from tf_last_error() (thread-local).  No C++
 *     exception crosses the ABI;
 *   - voxels are AoS float2 (tsdf, weight) [n][n][n] with x fastest — the
 *     interleaved body of the reference spill format (volumes.py:43-66), so a
 *     spill is one raw copy;
 *   - results are bit-identical to the reference kernels: the exact paths use
 *     IEEE round-to-nearest FP64 ops in the reference's evaluation order with
 *     no contraction, and float32 where numba types the reference's
 *     arithmetic as float32.
 */
#ifndef TFB200_H
#define TFB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TFB200_ABI_VERSION 2
#define TFB200_MAX_VOLUMES_PER_LAUNCH 64

enum {
    TF_OK = 0,
    TF_EINVAL = -1,  /* bad argument (sizes, null pointers, workspace too small) */
    TF_ECUDA = -2,   /* CUDA launch / runtime error */
};

/* One TSDF subvolume resident on the device (tsdf.py:41-107).
 *
 * brick_state_dev (optional, may be NULL): uint32 per 8^3 brick (x fastest,
 * ceil(n/8)^3 entries): low 16 bits = voxels that are NOT "observed and
 * >= summary_threshold", high 16 bits = observed voxels (weight > 0), and a
 * derived flag byte per brick (brick_flags_dev, same indexing).  Built
 * by tf_brick_summary for a truncation tau (summary_threshold =
 * tf_good_threshold(tau)) and kept exact by tf_integrate; tf_raycast uses it
 * to certify free-space and never-observed samples without gathering voxels.
 * Ignored (not used, not maintained) when NULL or when summary_threshold
 * does not match the call's tau. */
typedef struct TfVolume {
    void *voxels_dev;    /* float2[n][n][n]: (tsdf, weight), x fastest */
    int64_t n;           /* voxels_per_side */
    int64_t origin[3];   /* origin_voxel: global voxel of local (0,0,0) */
    double voxel_size;   /* side_length / voxels_per_side (tsdf.py:80-82) */
    uint32_t *brick_state_dev;
    uint8_t *brick_flags_dev;  /* per brick: bit0 never observed, bit1 the brick
                                  and its +1 neighbours are all-good (cells with
                                  a min corner in it are free space); followed
                                  by ceil(nb/8)^3 superbrick (64^3) bytes, the
                                  AND of their bricks' flags */
    float summary_threshold;
    int32_t reserved;
    uint8_t *color_dev;  /* optional (NULL = none): uchar4[n][n][n] = (r, g, b, w),
                            the running mean of the RGB observations of the
                            voxel while it lay in the truncation band, w their
                            count (saturating at 255).  Not in the reference
                            (SPEC.md:8): the rule is this library's own. */
    uint64_t *counters_dev; /* optional (NULL = none): uint64[2] accumulated by
                               tf_integrate's culling stage: [0] general bricks
                               (8^3, swept voxel by voxel), [1] certified
                               free-space bricks — the per-volume work measure
                               the multi-GPU ownership balances on */
} TfVolume;

/* Pinhole intrinsics of one pyramid level (geometry.py:27-57). */
typedef struct TfCamera {
    double fx, fy, cx, cy;
    int64_t width, height;
} TfCamera;

/* Per-call counters written (accumulated) to a device uint64[16]. */
enum {
    TF_STAT_VOXEL_UPDATES = 0, /* voxels passing every integration gate */
    TF_STAT_SWEPT_VOXELS = 1,  /* voxels evaluated after brick culling */
    TF_STAT_ACTIVE_BRICKS = 2,
    TF_STAT_TOTAL_BRICKS = 3,
    TF_STAT_RAY_SAMPLES = 4,   /* trilinear _sample calls (_kernels.py:28) */
    TF_STAT_RAY_HITS = 5,      /* hits merged by this raycast call */
    TF_STAT_EXACT_VOXELS = 6,  /* voxels the float32 screen deferred to the exact path */
    TF_STAT_NOOP_UPDATES = 7,  /* updates proven to leave the voxel unchanged (store skipped) */
    TF_STAT_COL_SKIPPED = 8,   /* swept voxels rejected as whole columns */
    TF_STAT_DEPTH_SKIPPED = 9, /* swept voxels rejected by the depth test (d <= 0 / sdf < -tau) */
    TF_STAT_FREE_BRICKS = 10,  /* active bricks certified all free space (streaming kernel) */
    TF_STAT_EXACT_SAMPLES = 11, /* ray samples evaluated with the exact arithmetic */
    TF_STAT_CERT_FAILURES = 12, /* certified decisions contradicted by exact ones (must be 0) */
    TF_STAT_SUMMARY_SAMPLES = 13, /* ray samples certified by the brick summary alone */
    TF_STAT_GENERAL_ALL_FREE = 14, /* general-path bricks whose voxels all turned out free space */
    TF_STAT_COOP_RAYS = 15,   /* rays finished by the warp-cooperative raycast pass */
    TF_STAT_FREE_KERNEL_UPDATES = 16, /* voxel updates by the certified free-space brick kernel */
    TF_STAT_EXACT_UPDATES = 17,       /* voxel updates by the exact (reference arithmetic) queue */
    TF_STAT_PART_ALL_FREE = 18,  /* 8x4x4 parts of general bricks whose voxels all were free-space updates */
    TF_STAT_PART_ALL_SKIP = 19,  /* 8x4x4 parts of general bricks whose voxels all were rejected */
    TF_STAT_COUNT = 24
};

int tf_abi_version(void);
const char *tf_last_error(void);

/* Measurement hooks.  tf_launch_count: kernels launched by this library so
 * far.  With tf_profile_enable(1), each tf_integrate / tf_raycast brackets its
 * kernels with CUDA events on the caller's stream; tf_profile_read waits for
 * them and returns summed milliseconds and launch counts per kind:
 * 0 = integration voxel-update kernel, 1 = whole tf_integrate, 2 = raycast. */
enum { TF_PROF_INTEGRATE_UPDATE = 0, TF_PROF_INTEGRATE_ALL = 1, TF_PROF_RAYCAST = 2,
       TF_PROF_INTEGRATE_FREE = 3, TF_PROF_INTEGRATE_GENERAL = 4, TF_PROF_INTEGRATE_EXACT = 5,
       TF_PROF_RAYCAST_COOP = 6, TF_PROF_INTEGRATE_SCREEN = 7, TF_PROF_KINDS = 8 };
uint64_t tf_launch_count(void);
/* Debug: index violations counted by a bounds-checked build of the library
 * (compiled with -DTF_BOUNDS_CHECK: guarded loads / stores are skipped and
 * counted instead of faulting — the stand-in for compute-sanitizer memcheck,
 * which is closed on the GPU pool); UINT64_MAX from a plain build. */
uint64_t tf_debug_bounds_violations(void);

/* Debug: when set (device int64[12*H*W] per raycast call), tf_raycast writes per
 * pixel {SM clock cycles, samples, exact samples, summary-certified samples,
 * region evaluations at brick level by kind 0..3, at superbrick level 0..3};
 * NULL disables. */
void tf_debug_ray_clock_buffer(int64_t *buffer_dev);

/* Test hook (synchronous): n random (a, b) pairs, b an integer in [1, 256],
 * through the table-driven correctly rounded division of the running-mean
 * update vs. IEEE division; returns the number of mismatches (-1 on error). */
int64_t tf_debug_weight_division_check(int64_t n, uint64_t seed);
/* Test hook (synchronous): n random and adversarial (volume, ray) pairs
 * through the raycast's division-free ray/box interval vs. the reference's
 * (_kernels.py:299-348); returns the number of mismatches (-1 on error). */
int64_t tf_debug_ray_interval_check(int64_t n, uint64_t seed);
/* Test hook (synchronous): the raycast's certified quotient by the voxel size
 * (reciprocal + correction, proved or else IEEE) vs. IEEE division on n random
 * and adversarial pairs; returns the number of mismatches (-1 on error). */
int64_t tf_debug_div_check(int64_t n, uint64_t seed);
void tf_profile_enable(int on);
int tf_profile_read(double *ms_by_kind, int64_t *launches_by_kind, int nkinds);

/* Test hooks (bitwise-equality proofs at full size): TF_DEBUG_NO_CULL makes
 * tf_integrate sweep every brick (culling never drops an update);
 * TF_DEBUG_EXACT_ONLY runs the plain reference-order float64 arithmetic for
 * every voxel / ray instead of the float32-screened / certified fast paths; TF_DEBUG_NO_FIXEDPOINT
 * stores every free-space update even when it provably leaves the voxel
 * unchanged. */
enum { TF_DEBUG_NO_CULL = 1u, TF_DEBUG_EXACT_ONLY = 2u, TF_DEBUG_NO_FIXEDPOINT = 4u,
       TF_DEBUG_LANE0_ONLY = 8u /* tf_raycast traces only lane 0 of each warp (timing) */,
       TF_DEBUG_COOP_ALL = 16u /* tf_raycast traces every ray with the warp-cooperative march */ };
void tf_set_debug_flags(uint32_t flags);
uint32_t tf_debug_flags(void);

/* ---- integration: replaces _kernels.integrate_kernel (_kernels.py:71-133),
 * called by tsdf.integrate (tsdf.py:110-144), fused over `nvol` volumes.
 * r_cw / t_cw: Pose.invert() of the camera pose, cam_center its translation
 * (tsdf.py:126-135). `depth_dev`: f64 [height][width] z-depth, 0 = invalid.
 * stats_dev may be NULL. */
size_t tf_integrate_workspace_size(const TfVolume *vols, int nvol, const TfCamera *cam);
int tf_integrate(const TfVolume *vols, int nvol, const double *depth_dev,
                 const TfCamera *cam, const double r_cw[9], const double t_cw[3],
                 const double cam_center[3], double tau, double max_weight,
                 double sample_weight, void *workspace_dev, size_t workspace_bytes,
                 uint64_t *stats_dev, void *stream);

/* tf_integrate with colour: rgb_dev (uint8 [H][W][3], NULL = none) is fused
 * into the color_dev of every volume that has one.  A voxel's colour takes the
 * observation of the pixel its TSDF update used, only when that update lies
 * in the truncation band (sdf < tau, i.e. not clamped): c <- rint((w c + o) /
 * (w + 1)) per channel in float32, w <- min(w + 1, 255).  TSDF and weights are
 * exactly those of tf_integrate. */
int tf_integrate_rgb(const TfVolume *vols, int nvol, const double *depth_dev,
                     const uint8_t *rgb_dev, const TfCamera *cam, const double r_cw[9],
                     const double t_cw[3], const double cam_center[3], double tau,
                     double max_weight, double sample_weight, void *workspace_dev,
                     size_t workspace_bytes, uint64_t *stats_dev, void *stream);

/* tf_integrate_rgb in two halves, so the first can run on another stream
 * while the previous frame's raycast still occupies the GPU:
 * tf_integrate_prepare builds the per-frame pixel tables, depth mips, the
 * culled brick lists and the float32 screen of the general bricks' voxels
 * (free-space masks and the exact-voxel queue) in the workspace (it reads the
 * depth frame and the volumes' geometry, never their voxels or summaries);
 * tf_integrate_finish then runs the voxel updates and the summary upkeep.  finish must follow a
 * prepare with the same arguments on the same workspace (the caller orders
 * the two streams), and no other integrate call may use that workspace in
 * between.  With more volumes than one launch holds, prepare does nothing
 * and finish does both. */
int tf_integrate_prepare(const TfVolume *vols, int nvol, const double *depth_dev,
                         const TfCamera *cam, const double r_cw[9], const double t_cw[3],
                         const double cam_center[3], double tau, double max_weight,
                         double sample_weight, void *workspace_dev, size_t workspace_bytes,
                         void *stream);
int tf_integrate_finish(const TfVolume *vols, int nvol, const double *depth_dev,
                        const uint8_t *rgb_dev, const TfCamera *cam, const double r_cw[9],
                        const double t_cw[3], const double cam_center[3], double tau,
                        double max_weight, double sample_weight, void *workspace_dev,
                        size_t workspace_bytes, uint64_t *stats_dev, void *stream);

/* ---- raycast: replaces _kernels.raycast_kernel (_kernels.py:266-451) with
 * its helpers _sample / _scan_crossing / _hit_wins, called by tsdf.raycast
 * (tsdf.py:193-225), fused over `nvol` volumes sharing one voxel size.
 * Merges into existing maps with the _hit_wins total order, exactly like
 * calling the reference once per volume in any order.
 * dist_dev f64 [H][W] (+inf = none), vert_dev / norm_dev f64 [H][W][3]. */
int tf_raycast(const TfVolume *vols, int nvol, const TfCamera *cam, double tau,
               int64_t coarse_step, const double r_wc[9], const double cam_center[3],
               double *dist_dev, double *vert_dev, double *norm_dev,
               uint64_t *stats_dev, void *stream);
/* tf_raycast with the cooperative pass's scratch (rescue list and per-(ray,
 * volume) hit slots) taken from a caller workspace of at least
 * tf_raycast_workspace_size(nvol, cam) bytes, 256-byte aligned, used by one
 * stream at a time.  tf_raycast keeps an internal per-(device, stream)
 * buffer instead (least recently used of 16 evicted). */
size_t tf_raycast_workspace_size(int nvol, const TfCamera *cam);
int tf_raycast_ws(const TfVolume *vols, int nvol, const TfCamera *cam, double tau,
                  int64_t coarse_step, const double r_wc[9], const double cam_center[3],
                  double *dist_dev, double *vert_dev, double *norm_dev, void *workspace_dev,
                  size_t workspace_bytes, uint64_t *stats_dev, void *stream);
/* tf_raycast_ws over a subset of the image: only the rows of the 8-pixel
 * block rows ty with ty % row_mod == row_rem are traced (the others are left
 * as they are) — the image-partitioned raycast of the replicated multi-GPU
 * mode, where every rank holds every volume and traces 1/row_mod of the
 * rows; the ranks' maps merge into the full-image result bit for bit. */
int tf_raycast_rows(const TfVolume *vols, int nvol, const TfCamera *cam, double tau,
                    int64_t coarse_step, const double r_wc[9], const double cam_center[3],
                    double *dist_dev, double *vert_dev, double *norm_dev, void *workspace_dev,
                    size_t workspace_bytes, int row_mod, int row_rem, uint64_t *stats_dev,
                    void *stream);
/* tf_raycast_rows with flags.  TF_RAYCAST_FRESH: the map is taken as empty
 * (RayMap.empty / tf_raymap_reset) without reading it — every pixel is
 * written, so no reset launch is needed first; requires row_mod == 1. */
#define TF_RAYCAST_FRESH 1
int tf_raycast_ex(const TfVolume *vols, int nvol, const TfCamera *cam, double tau,
                  int64_t coarse_step, const double r_wc[9], const double cam_center[3],
                  double *dist_dev, double *vert_dev, double *norm_dev, void *workspace_dev,
                  size_t workspace_bytes, int row_mod, int row_rem, int flags, uint64_t *stats_dev,
                  void *stream);

/* ---- trilinear_sample (tsdf.py:147-153 / _kernels._sample :28-68) for
 * `npoints` world points (f64 [N][3]); writes value and validity per point. */
int tf_trilinear_sample(const TfVolume *vol, const double *points_dev, int64_t npoints,
                        double *values_dev, uint8_t *valid_dev, void *stream);

/* ---- free-space brick summaries (see TfVolume.brick_bad_dev). */
float tf_good_threshold(double tau);
int tf_brick_summary(const TfVolume *vol, void *stream);

/* Colours of a rendered ray map: for every pixel with a finite distance the
 * hit point o + t d (the raycast's own arithmetic) is looked up in the first
 * volume (in `vols` order) whose cell around it has all 8 corner colours
 * observed (w > 0): trilinear RGB in float32 into colors_dev (float32
 * [H][W][3]); 0 elsewhere.  Not in the reference. */
int tf_raycast_colors(const TfVolume *vols, int nvol, const TfCamera *cam, const double r_wc[9],
                      const double cam_center[3], const double *dist_dev, float *colors_dev,
                      void *stream);

/* ---- raymap merge: _hit_wins (_kernels.py:246-263) of a partial map into
 * `dst` (the cross-GPU reduction of DESIGN.md "Multi-GPU"). */
int tf_raymap_merge(double *dst_dist_dev, double *dst_vert_dev, double *dst_norm_dev,
                    const double *src_dist_dev, const double *src_vert_dev,
                    const double *src_norm_dev, int64_t npixels, void *stream);

/* Packed form for the cross-GPU row-block exchange: records of 4 doubles
 * (t, nx, ny, nz), 32-byte aligned; dst[p] = src[p] where _hit_wins(src, dst). */
int tf_raymap_merge_packed(double *dst_dev, const double *src_dev, int64_t npixels, void *stream);

/* RayMap.empty in place (tsdf.py:156-190): +inf distances, zero vertices and
 * normals, in one launch. */
int tf_raymap_reset(double *dist_dev, double *vert_dev, double *norm_dev, int64_t npixels, void *stream);

/* Vertices of rows [row0, row0 + nrows) rebuilt from their hit distances
 * (dist_dev[i * dist_stride], row-major from row0): o + t d with the
 * raycast's own arithmetic (bit-identical to what tf_raycast writes), 0 where
 * t = +inf.  vert_dev: nrows * width * 3 doubles. */
int tf_raymap_vertices(const double *dist_dev, int64_t dist_stride, double *vert_dev,
                       const TfCamera *cam, const double r_wc[9], const double cam_center[3],
                       int64_t row0, int64_t nrows, void *stream);

/* ---- ICP source maps: geometry.depth_to_vertices + compute_normals
 * (geometry.py:261-302) of pyramid level `level` (stride 2^level subsampling of
 * the full-resolution depth, geometry.py:256-258), with that level's camera.
 * Outputs are dense level-sized arrays; valid = vertex_ok & normal_ok. */
int tf_vertex_normal_map(const double *depth_dev, int64_t full_width, int64_t full_height,
                         int level, const TfCamera *level_cam, double *verts_dev,
                         double *norms_dev, uint8_t *valid_dev, void *stream);

/* ---- ICP normal equations: the per-pixel part of tracking._solve_step
 * (tracking.py:76-108) with a deterministic FP64 tree reduction.  The model
 * maps are the full-resolution RayMap viewed at stride 2^level
 * (RayMap.downsampled, tsdf.py:185-190).  out29_dev (device, 29 doubles):
 * upper triangle of A^T A (21, row major), A^T r (6), sum r^2, count. */
size_t tf_icp_workspace_size(int64_t src_pixels);
int tf_icp_reduce(const double *src_verts_dev, const double *src_norms_dev,
                  const uint8_t *src_valid_dev, int64_t src_width, int64_t src_height,
                  const double *mdl_dist_dev, const double *mdl_vert_dev,
                  const double *mdl_norm_dev, int64_t mdl_full_width,
                  int64_t mdl_full_height, int level, const TfCamera *level_cam,
                  const double r_est[9], const double t_est[3], const double r_ref[9],
                  const double t_ref[3], double max_dist_sq, double cos_min,
                  void *workspace_dev, size_t workspace_bytes, double *out29_dev,
                  void *stream);

/* Device-resident track() (tracking.py:123-196): the whole pyramid, coarsest
 * level first, iterations[l] steps per level, queued without host round trips.
 * Per step: icp_terms (as tf_icp_reduce) and one single-warp kernel doing the
 * host part of _solve_step (:100-120: pair minimum min_pairs[l], cond > 1e12
 * gate, LU solve, finiteness) and the pose update (:178-183: Rodrigues,
 * re-orthonormalisation, |delta| < step_eps ends the level).  state_dev
 * (tf_icp_track_state_size() bytes) receives doubles {R[9] row-major, t[3],
 * lost, count, rms, scratch}: the refined estimate, or lost = 1 (the caller
 * then keeps its seed, :187-193); count / rms of the last successful step.
 * Level l's source maps are src_*[l] (tf_vertex_normal_map at level l). */
size_t tf_icp_track_state_size(void);
int tf_icp_track(int nlevels, const double *const *src_verts_dev, const double *const *src_norms_dev,
                 const uint8_t *const *src_valid_dev, const TfCamera *level_cams,
                 const int *iterations, const int *min_pairs, const double *mdl_dist_dev,
                 const double *mdl_vert_dev, const double *mdl_norm_dev, int64_t mdl_full_width,
                 int64_t mdl_full_height, const double r_ref[9], const double t_ref[3],
                 const double r_init[9], const double t_init[3], double max_dist_sq, double cos_min,
                 double step_eps, void *workspace_dev, size_t workspace_bytes, double *state_dev,
                 void *stream);

/* ---- extraction: _kernels.extract_bound / extract_kernel
 * (_kernels.py:454-578), called by tsdf.extract_points (tsdf.py:261-280).
 * Two calls: tf_extract_count writes the vertex count (device int64) after an
 * order-preserving scan kept in the workspace; tf_extract_emit then writes
 * the vertices in the reference's (z, y, x) voxel order. */
size_t tf_extract_workspace_size(int64_t n);
int tf_extract_count(const TfVolume *vol, void *workspace_dev, size_t workspace_bytes,
                     int64_t *count_dev, void *stream);
int tf_extract_emit(const TfVolume *vol, const void *workspace_dev, size_t workspace_bytes,
                    double *verts_dev, double *norms_dev, void *stream);

/* ---- endpoint cells: volumes.bin_endpoints (volumes.py:305-331): per valid
 * pixel the tile-lattice cell of its endpoint, as int64 [H*W][3] with
 * cells of invalid pixels set to INT64_MIN. */
int tf_endpoint_cells(const double *depth_dev, const TfCamera *cam, const double r_wc[9],
                      const double t_wc[3], double block_side, int64_t *cells_dev,
                      void *stream);

/* ---- the whole of volumes.bin_endpoints' arithmetic (volumes.py:305-331)
 * on the device: the endpoint cell of every valid pixel (tf_endpoint_cells'
 * arithmetic) counted in a hash table in the workspace (np.unique(...,
 * return_counts=True), :327), compacted into out_dev = int64 [2 + 4 *
 * capacity]: out[0] = distinct cells n, out[1] = overflow (1: a cell beyond
 * +-2^20 blocks, or more than `capacity` cells — bin on the host instead),
 * then n records (cx, cy, cz, count) in no particular order.  Stream-ordered,
 * no host synchronisation: one small D2H of out_dev per frame.  The
 * workspace (tf_bin_endpoints_workspace_size(capacity) bytes, 256-byte
 * aligned) must be zero before the first call; each call leaves it zero. */
size_t tf_bin_endpoints_workspace_size(int64_t capacity);
int tf_bin_endpoints(const double *depth_dev, const TfCamera *cam, const double r_wc[9],
                     const double t_wc[3], double block_side, int64_t capacity, void *workspace_dev,
                     size_t workspace_bytes, int64_t *out_dev, void *stream);

/* ---- packed spill images: the opt-in capacity mode of the pinned-host spill
 * tier (spill_tier="host_packed"; not the parity format, SURVEY.md §7 hard
 * part 5).  (tsdf, weight) f32 pairs -> tsdf IEEE half (round to nearest,
 * |error| <= 2^-11 |tsdf| <= 4.9e-4 tau) + weight uint8 (round to nearest,
 * saturating at 255: exact for integral weights <= 255) in two planes of
 * `count` entries: 3 B per voxel crosses the host link instead of 8. */
int tf_pack_voxels(const void *voxels_dev, int64_t count, void *tsdf_half_dev, uint8_t *weight_dev,
                   void *stream);
int tf_unpack_voxels(const void *tsdf_half_dev, const uint8_t *weight_dev, int64_t count,
                     void *voxels_dev, void *stream);

/* ---- multi-GPU ray-map reduction over peer memory (the
 * survey's tf_comm_init / tf_exchange_* rows).  One process per GPU.  Each
 * rank owns a "region" in its own HBM holding its partial ray map (what its
 * tf_raycast over its own volumes writes) and its copy of the merged model;
 * the regions are mapped into every peer with CUDA IPC (NVLink / NVSwitch).
 * tf_comm_reduce_raymap is ONE kernel per rank: it signals "partial ready"
 * to every peer, waits for theirs, folds the peers' (t, normal) records of
 * its row block with the _hit_wins total order in rank order
 * (_kernels.py:246-263; equal to the single-GPU raycast over all volumes,
 * bit for bit), takes the winner's vertex, stores the merged rows straight
 * into every rank's model (all-gather by stores), and its last block
 * signals "done"; a one-warp kernel then waits for every peer's "done", after
 * which the local model is complete and every peer has finished reading the
 * local partial.  Replaces the NCCL all-to-all + merge + all-gather of the
 * row-block exchange (distributed.rowblock_exchange).  Waits time out after
 * TF_COMM_TIMEOUT_NS (error flag, tf_comm_error) instead of hanging.
 *
 * Region layout (offsets in bytes, TF_COMM_* indices): flags, partial
 * distance [H][W] f64, partial vertices [H][W][3], partial normals
 * [H][W][3], model distance, model vertices, model normals. */
#define TF_COMM_HANDLE_BYTES 64
#define TF_COMM_MAX_RANKS 64
#define TF_COMM_TIMEOUT_NS 20000000000ull
enum { TF_COMM_FLAGS = 0, TF_COMM_PART_DIST, TF_COMM_PART_VERT, TF_COMM_PART_NORM,
       TF_COMM_MODEL_DIST, TF_COMM_MODEL_VERT, TF_COMM_MODEL_NORM, TF_COMM_NSECTIONS };
enum { TF_COMM_NOWAIT = 1u /* no flags, no waits: emulated ranks on one device (tests) */ };
typedef struct TfComm TfComm;

/* Allocates (cudaMalloc on the current device) and initialises this rank's
 * region: no-hit partial and model (+inf distance, zero vectors), zero flags. */
int tf_comm_create(int rank, int world, int64_t width, int64_t height, TfComm **out);
/* Region base and section offsets (TF_COMM_NSECTIONS entries). */
int tf_comm_layout(const TfComm *comm, void **base, int64_t *offsets);
/* IPC handle of this rank's region (TF_COMM_HANDLE_BYTES bytes). */
int tf_comm_export(const TfComm *comm, void *handle);
/* Maps every peer's region (handles: world x TF_COMM_HANDLE_BYTES, rank
 * order; this rank's own entry is ignored). */
int tf_comm_import(TfComm *comm, const void *handles);
/* Test hook: the comms of `world` emulated ranks living in this process on
 * one device see each other's regions directly (no IPC). */
int tf_comm_link_local(TfComm *const *comms, int world);
/* The reduction described above, asynchronous on `stream`. */
int tf_comm_reduce_raymap(TfComm *comm, unsigned flags, void *stream);
/* Synchronous read of the region's error flag (1 = a wait timed out). */
int tf_comm_error(const TfComm *comm, int *error);
/* Non-blocking read of the error flag as of the last reduction that has
 * completed on its stream (each tf_comm_reduce_raymap queues a copy of the
 * flag into pinned host memory): the per-frame check of ShardedFusion. */
int tf_comm_error_poll(const TfComm *comm, int *error);
int tf_comm_destroy(TfComm *comm);

#ifdef __cplusplus
}
#endif
#endif /* TFB200_H */
