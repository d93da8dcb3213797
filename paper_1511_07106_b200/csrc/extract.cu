// Surface point extraction and endpoint binning (sm_100a).
//
//   extract_*  — _kernels.extract_bound / extract_kernel (reference
//                _kernels.py:454-578) as an order-preserving stream
//                compaction: a per-block count, an exclusive scan of the block
//                counts, then each block re-derives its vertices and writes them
//                at its scanned offset, so the output order is the reference's
//                (z, y, x) voxel order (the bitwise-repeat gate,
//                test_acceptance.py:363-386, depends on it).
//   endpoint_* — the per-pixel part of volumes.bin_endpoints (volumes.py:318-326).
#include <math.h>

#include <algorithm>

#include "tf_common.cuh"

namespace tf {

constexpr int kExtractThreads = 256;

struct Emit {
    double v[3], n[3];
};

// extract_kernel body for one voxel (_kernels.py:496-577); false = no vertex
__device__ __forceinline__ bool extract_voxel(const float2 *__restrict__ vox, int64_t n,
                                              const int64_t origin[3], double vs, int64_t lin,
                                              Emit *e) {
    const float2 c = vox[lin];
    if (c.y <= 0.0f) return false;                                   // :496
    const int64_t ix = lin % n, iy = (lin / n) % n, iz = lin / (n * n);
    const int64_t pos[3] = {ix, iy, iz};
    const int64_t stride[3] = {1, n, n * n};
    const float v0 = c.x;  // numba float(f32) stays float32
    const bool pos0 = v0 > 0.0f;
    double best_alpha = 2.0;
    int best_axis = -1;
    float2 nb_p[3], nb_m[3];
    bool has_p[3], has_m[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        has_p[a] = pos[a] + 1 < n;
        has_m[a] = pos[a] - 1 >= 0;
        nb_p[a] = has_p[a] ? vox[lin + stride[a]] : make_float2(0.f, 0.f);
        nb_m[a] = has_m[a] ? vox[lin - stride[a]] : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {                                    // :502-522
        if (has_p[a] && nb_p[a].y > 0.0f) {
            const float v1 = nb_p[a].x;
            if ((v1 > 0.0f) != pos0) {
                const double alpha = (double)fdivr(v0, fsubr(v0, v1));  // float32 ops
                if (alpha < best_alpha) {
                    best_alpha = alpha;
                    best_axis = a;
                }
            }
        }
    }
    if (best_axis < 0) return false;
    double g[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {                                    // :526-558
        const bool im = has_m[a] && nb_m[a].y > 0.0f;
        const bool ip = has_p[a] && nb_p[a].y > 0.0f;
        const double vm = im ? (double)nb_m[a].x : 0.0;
        const double vp = ip ? (double)nb_p[a].x : 0.0;
        if (im && ip)
            g[a] = dmul(dsub(vp, vm), 0.5);
        else if (ip)
            g[a] = dsub(vp, (double)v0);
        else if (im)
            g[a] = dsub((double)v0, vm);
        else
            g[a] = 0.0;
    }
    const double gnorm = dsqrt(dadd(dadd(dmul(g[0], g[0]), dmul(g[1], g[1])), dmul(g[2], g[2])));
    if (gnorm == 0.0) return false;                                  // :560
    if (e) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            e->v[a] = dmul((double)(pos[a] + origin[a]), vs);        // :562-564
            e->n[a] = ddiv(g[a], gnorm);
        }
        e->v[best_axis] = dadd(e->v[best_axis], dmul(best_alpha, vs));  // :565-570
    }
    return true;
}

struct ExtractVol {
    const float2 *vox;
    int64_t n;
    int64_t origin[3];
    double vs;
};

__global__ void __launch_bounds__(kExtractThreads) extract_count_kernel(const ExtractVol ev,
                                                                        int64_t *__restrict__ counts) {
    const int64_t total = ev.n * ev.n * ev.n;
    const int64_t lin = (int64_t)blockIdx.x * kExtractThreads + threadIdx.x;
    const bool hit = lin < total && extract_voxel(ev.vox, ev.n, ev.origin, ev.vs, lin, nullptr);
    const int c = __syncthreads_count(hit);
    if (threadIdx.x == 0) counts[blockIdx.x] = c;
}

// exclusive scan of `nb` block counts in place; single block, fixed order
__global__ void __launch_bounds__(1024) scan_kernel(int64_t *__restrict__ counts, int64_t nb,
                                                    int64_t *__restrict__ total_out) {
    __shared__ int64_t part[1024];
    const int t = threadIdx.x;
    const int64_t per = (nb + 1023) / 1024;
    const int64_t b0 = t * per, b1 = min(nb, b0 + per);
    int64_t s = 0;
    for (int64_t b = b0; b < b1; ++b) s += counts[b];
    part[t] = s;
    __syncthreads();
    if (t == 0) {
        int64_t run = 0;
        for (int i = 0; i < 1024; ++i) {
            const int64_t x = part[i];
            part[i] = run;
            run += x;
        }
        *total_out = run;
    }
    __syncthreads();
    int64_t run = part[t];
    for (int64_t b = b0; b < b1; ++b) {
        const int64_t x = counts[b];
        counts[b] = run;
        run += x;
    }
}

__global__ void __launch_bounds__(kExtractThreads) extract_emit_kernel(
    const ExtractVol ev, const int64_t *__restrict__ offsets, double *__restrict__ verts,
    double *__restrict__ norms) {
    const int64_t total = ev.n * ev.n * ev.n;
    const int64_t lin = (int64_t)blockIdx.x * kExtractThreads + threadIdx.x;
    Emit e;
    const bool hit = lin < total && extract_voxel(ev.vox, ev.n, ev.origin, ev.vs, lin, &e);
    __shared__ int wcount[kExtractThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned mask = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) wcount[w] = __popc(mask);
    __syncthreads();
    int before = 0;
    for (int i = 0; i < w; ++i) before += wcount[i];
    if (hit) {
        const int64_t o = offsets[blockIdx.x] + before + __popc(mask & ((1u << lane) - 1u));
        for (int a = 0; a < 3; ++a) {
            verts[3 * o + a] = e.v[a];
            norms[3 * o + a] = e.n[a];
        }
    }
}

// ---- endpoint cells (volumes.py:318-326) -----------------------------------
struct EndpointGeom {
    Mat3 r;
    Vec3 t;
    double fx, fy, cx, cy, block_side;
    int64_t width, height;
};

// the endpoint cell of pixel p (valid depth): volumes.py:318-326
__device__ __forceinline__ void endpoint_cell(const double *__restrict__ depth, const EndpointGeom &g,
                                              int64_t p, double d, int64_t c[3]) {
    const int64_t x = p % g.width, y = p / g.width;
    const double ray[3] = {ddiv(dsub((double)x, g.cx), g.fx), ddiv(dsub((double)y, g.cy), g.fy), 1.0};
    double rr[3];
    // pixel_rays() @ R.T through OpenBLAS: FMA chain over k
#pragma unroll
    for (int i = 0; i < 3; ++i)
        rr[i] = dfma(ray[2], g.r.m[3 * i + 2], dfma(ray[1], g.r.m[3 * i + 1], dmul(ray[0], g.r.m[3 * i])));
    const double nn = dsqrt(dadd(dadd(dmul(rr[0], rr[0]), dmul(rr[1], rr[1])), dmul(rr[2], rr[2])));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double pt = dadd(g.t.v[a], dmul(d, ddiv(rr[a], nn)));  // :319, :324
        const double q = floor(ddiv(pt, g.block_side));            // :326
        // int64 conversion of the reference; saturate far outside any key range
        c[a] = q >= 9.0e18 ? INT64_MAX : (q <= -9.0e18 ? INT64_MIN + 1 : (int64_t)q);
    }
}

// ---- endpoint histogram: np.unique(cells, axis=0, return_counts=True)
// (volumes.py:327) as a hash table in the workspace.  Keys pack the cell's
// three coordinates in 21 bits each (|c| < 2^20: 1 km at 1 mm blocks), top
// bit set so an empty slot (0) never matches; a cell out of that range or a
// full table raises the overflow flag (the caller then bins on the host).
constexpr int kCellBits = 21;
constexpr long long kCellLim = 1ll << (kCellBits - 1);

struct HistHeader {
    unsigned long long n;         // distinct cells compacted
    unsigned long long overflow;  // 1: a cell out of range or the table / output full
};

__device__ __forceinline__ unsigned long long pack_cell(const int64_t c[3], bool &ok) {
    ok = c[0] >= -kCellLim && c[0] < kCellLim && c[1] >= -kCellLim && c[1] < kCellLim &&
         c[2] >= -kCellLim && c[2] < kCellLim;
    const unsigned long long m = (1ull << kCellBits) - 1ull;
    return (1ull << 63) | (((unsigned long long)c[0] & m) << (2 * kCellBits)) |
           (((unsigned long long)c[1] & m) << kCellBits) | ((unsigned long long)c[2] & m);
}

__device__ __forceinline__ int64_t unpack_coord(unsigned long long key, int shift) {
    const long long v = (long long)((key >> shift) & ((1ull << kCellBits) - 1ull));
    return v >= kCellLim ? v - 2 * kCellLim : v;
}

__global__ void __launch_bounds__(256) endpoint_hist_kernel(const double *__restrict__ depth,
                                                            const EndpointGeom g,
                                                            unsigned long long *__restrict__ keys,
                                                            unsigned long long *__restrict__ counts,
                                                            const unsigned long long tmask,
                                                            HistHeader *__restrict__ hdr) {
    const int64_t npix = g.width * g.height;
    for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x; p0 < npix; p0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = p0 + threadIdx.x;
        const double d = p < npix ? depth[p] : 0.0;
        const bool valid = d > 0.0;  // volumes.py:322
        unsigned long long key = 0;
        if (valid) {
            int64_t c[3];
            endpoint_cell(depth, g, p, d, c);
            bool ok;
            key = pack_cell(c, ok);
            if (!ok) {
                atomicExch(&hdr->overflow, 1ull);
                key = 0;
            }
        }
        // lanes with the same cell add once (neighbouring pixels share cells)
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        if (key && (threadIdx.x & 31) == __ffs(peers) - 1) {
            const unsigned long long cnt = __popc(peers);
            unsigned long long h = (key * 0x9E3779B97F4A7C15ull) >> 20;
            for (unsigned long long probe = 0;; ++probe) {
                if (probe > tmask) {
                    atomicExch(&hdr->overflow, 1ull);
                    break;
                }
                const unsigned long long slot = (h + probe) & tmask;
                if (!TF_IN_BOUNDS(slot <= tmask)) break;
                const unsigned long long prev = atomicCAS(&keys[slot], 0ull, key);
                if (prev == 0ull || prev == key) {
                    atomicAdd(&counts[slot], cnt);
                    break;
                }
            }
        }
    }
}

// occupied slots -> out records (cx, cy, cz, count); the table is left empty
__global__ void __launch_bounds__(256) endpoint_compact_kernel(unsigned long long *__restrict__ keys,
                                                               unsigned long long *__restrict__ counts,
                                                               const unsigned long long tsize,
                                                               HistHeader *__restrict__ hdr,
                                                               int64_t *__restrict__ out,
                                                               const int64_t cap) {
    for (unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; s < tsize;
         s += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long key = keys[s];
        if (!key) continue;
        const unsigned long long i = atomicAdd(&hdr->n, 1ull);
        if ((int64_t)i < cap) {
            int64_t *r = out + 2 + 4 * i;
            r[0] = unpack_coord(key, 2 * kCellBits);
            r[1] = unpack_coord(key, kCellBits);
            r[2] = unpack_coord(key, 0);
            r[3] = (int64_t)counts[s];
        } else {
            atomicExch(&hdr->overflow, 1ull);
        }
        keys[s] = 0ull;
        counts[s] = 0ull;
    }
}

__global__ void endpoint_header_kernel(HistHeader *__restrict__ hdr, int64_t *__restrict__ out) {
    out[0] = (int64_t)hdr->n;
    out[1] = (int64_t)hdr->overflow;
    hdr->n = 0ull;
    hdr->overflow = 0ull;
}

__global__ void endpoint_cells_kernel(const double *__restrict__ depth, const EndpointGeom g,
                                      int64_t *__restrict__ cells) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.width * g.height) return;
    const double d = depth[p];
    if (!(d > 0.0)) {
        cells[3 * p] = cells[3 * p + 1] = cells[3 * p + 2] = INT64_MIN;
        return;
    }
    const int64_t x = p % g.width, y = p / g.width;
    const double ray[3] = {ddiv(dsub((double)x, g.cx), g.fx), ddiv(dsub((double)y, g.cy), g.fy), 1.0};
    double rr[3];
    // pixel_rays() @ R.T through OpenBLAS: FMA chain over k
#pragma unroll
    for (int i = 0; i < 3; ++i)
        rr[i] = dfma(ray[2], g.r.m[3 * i + 2], dfma(ray[1], g.r.m[3 * i + 1], dmul(ray[0], g.r.m[3 * i])));
    const double nn = dsqrt(dadd(dadd(dmul(rr[0], rr[0]), dmul(rr[1], rr[1])), dmul(rr[2], rr[2])));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double pt = dadd(g.t.v[a], dmul(d, ddiv(rr[a], nn)));  // :319, :324
        cells[3 * p + a] = (int64_t)floor(ddiv(pt, g.block_side));  // :326
    }
}

static size_t extract_blocks(int64_t n) {
    const int64_t total = n * n * n;
    return (size_t)((total + kExtractThreads - 1) / kExtractThreads);
}

}  // namespace tf

using namespace tf;

TF_BOUNDS_READER(extract)

extern "C" size_t tf_extract_workspace_size(int64_t n) {
    if (n < 2) return 0;
    return (extract_blocks(n) + 1) * sizeof(int64_t);
}

static ExtractVol to_ev(const TfVolume *vol) {
    ExtractVol ev;
    ev.vox = (const float2 *)vol->voxels_dev;
    ev.n = vol->n;
    for (int a = 0; a < 3; ++a) ev.origin[a] = vol->origin[a];
    ev.vs = vol->voxel_size;
    return ev;
}

extern "C" int tf_extract_count(const TfVolume *vol, void *workspace, size_t workspace_bytes,
                                int64_t *count_dev, void *stream_) {
    if (!vol || !vol->voxels_dev || vol->n < 2 || !workspace || !count_dev)
        return tf_set_error(TF_EINVAL, "tf_extract_count: bad argument");
    if (workspace_bytes < tf_extract_workspace_size(vol->n))
        return tf_set_error(TF_EINVAL, "tf_extract_count: workspace too small");
    const size_t nb = extract_blocks(vol->n);
    if (nb > 0x7fffffffu) return tf_set_error(TF_EINVAL, "tf_extract_count: volume too large");
    cudaStream_t stream = (cudaStream_t)stream_;
    int64_t *counts = (int64_t *)workspace;
    extract_count_kernel<<<(unsigned)nb, kExtractThreads, 0, stream>>>(to_ev(vol), counts);
    int rc = tf_check_launch("extract_count_kernel");
    if (rc) return rc;
    scan_kernel<<<1, 1024, 0, stream>>>(counts, (int64_t)nb, count_dev);
    return tf_check_launch("scan_kernel");
}

extern "C" int tf_extract_emit(const TfVolume *vol, const void *workspace, size_t workspace_bytes,
                               double *verts, double *norms, void *stream_) {
    if (!vol || !vol->voxels_dev || vol->n < 2 || !workspace || !verts || !norms)
        return tf_set_error(TF_EINVAL, "tf_extract_emit: bad argument");
    if (workspace_bytes < tf_extract_workspace_size(vol->n))
        return tf_set_error(TF_EINVAL, "tf_extract_emit: workspace too small");
    const size_t nb = extract_blocks(vol->n);
    extract_emit_kernel<<<(unsigned)nb, kExtractThreads, 0, (cudaStream_t)stream_>>>(
        to_ev(vol), (const int64_t *)workspace, verts, norms);
    return tf_check_launch("extract_emit_kernel");
}

extern "C" int tf_endpoint_cells(const double *depth, const TfCamera *cam, const double r_wc[9],
                                 const double t_wc[3], double block_side, int64_t *cells,
                                 void *stream_) {
    if (!depth || !cam || !r_wc || !t_wc || !cells || !(block_side > 0.0))
        return tf_set_error(TF_EINVAL, "tf_endpoint_cells: bad argument");
    EndpointGeom g{};
    for (int i = 0; i < 9; ++i) g.r.m[i] = r_wc[i];
    for (int i = 0; i < 3; ++i) g.t.v[i] = t_wc[i];
    g.fx = cam->fx;
    g.fy = cam->fy;
    g.cx = cam->cx;
    g.cy = cam->cy;
    g.block_side = block_side;
    g.width = cam->width;
    g.height = cam->height;
    const int64_t npix = cam->width * cam->height;
    if (npix <= 0) return TF_OK;
    endpoint_cells_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, (cudaStream_t)stream_>>>(depth, g,
                                                                                             cells);
    return tf_check_launch("endpoint_cells_kernel");
}

// table slots: the power of two >= 2 x capacity (load factor <= 1/2)
static unsigned long long hist_slots(int64_t capacity) {
    unsigned long long t = 64;
    while (t < 2ull * (unsigned long long)capacity) t <<= 1;
    return t;
}

extern "C" size_t tf_bin_endpoints_workspace_size(int64_t capacity) {
    if (capacity < 1) return 0;
    return 256 + (size_t)hist_slots(capacity) * 16;
}

extern "C" int tf_bin_endpoints(const double *depth, const TfCamera *cam, const double r_wc[9],
                                const double t_wc[3], double block_side, int64_t capacity,
                                void *workspace, size_t workspace_bytes, int64_t *out, void *stream_) {
    if (!depth || !cam || !r_wc || !t_wc || !out || !workspace || !(block_side > 0.0) || capacity < 1)
        return tf_set_error(TF_EINVAL, "tf_bin_endpoints: bad argument");
    if (workspace_bytes < tf_bin_endpoints_workspace_size(capacity) || ((uintptr_t)workspace & 255u))
        return tf_set_error(TF_EINVAL, "tf_bin_endpoints: workspace too small or not 256-byte aligned");
    EndpointGeom g{};
    for (int i = 0; i < 9; ++i) g.r.m[i] = r_wc[i];
    for (int i = 0; i < 3; ++i) g.t.v[i] = t_wc[i];
    g.fx = cam->fx;
    g.fy = cam->fy;
    g.cx = cam->cx;
    g.cy = cam->cy;
    g.block_side = block_side;
    g.width = cam->width;
    g.height = cam->height;
    const unsigned long long tsize = hist_slots(capacity);
    HistHeader *hdr = (HistHeader *)workspace;
    unsigned long long *keys = (unsigned long long *)((char *)workspace + 256);
    unsigned long long *counts = keys + tsize;
    cudaStream_t stream = (cudaStream_t)stream_;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t npix = cam->width * cam->height;
    if (npix > 0) {
        const unsigned blocks = (unsigned)std::min<int64_t>((npix + 255) / 256, (int64_t)sms * 8);
        endpoint_hist_kernel<<<blocks, 256, 0, stream>>>(depth, g, keys, counts, tsize - 1, hdr);
        int rc = tf_check_launch("endpoint_hist_kernel");
        if (rc) return rc;
    }
    endpoint_compact_kernel<<<(unsigned)std::min<unsigned long long>((tsize + 255) / 256, 1024ull), 256, 0,
                              stream>>>(keys, counts, tsize, hdr, out, capacity);
    int rc = tf_check_launch("endpoint_compact_kernel");
    if (rc) return rc;
    endpoint_header_kernel<<<1, 1, 0, stream>>>(hdr, out);
    return tf_check_launch("endpoint_header_kernel");
}

// ---- packed spill images (opt-in capacity mode, not the parity format) -----
// tsdf as IEEE half (round to nearest: |error| <= 2^-11 |tsdf| <= 4.9e-4 tau),
// weight as uint8 (round to nearest, saturating at 255: exact for the
// reference's integral weights up to 255; max_weight defaults to 128) — 3 B
// per voxel instead of 8 in two planes.  SURVEY.md §7 hard part 5: the
// parity format stays f32 / f32; this only shrinks what crosses the host link.
#include <cuda_fp16.h>

namespace tf {
__global__ void pack_voxels_kernel(const float2 *__restrict__ vox, int64_t count, __half *__restrict__ t,
                                   uint8_t *__restrict__ w) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float2 v = vox[i];
        t[i] = __float2half_rn(v.x);
        w[i] = (uint8_t)fminf(fmaxf(rintf(v.y), 0.0f), 255.0f);
    }
}

__global__ void unpack_voxels_kernel(const __half *__restrict__ t, const uint8_t *__restrict__ w,
                                     int64_t count, float2 *__restrict__ vox) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        vox[i] = make_float2(__half2float(t[i]), (float)w[i]);
}
}  // namespace tf

static unsigned pack_grid(int64_t count) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (count + 255) / 256;
    return (unsigned)(want < (int64_t)sms * 8 ? (want > 0 ? want : 1) : (int64_t)sms * 8);
}

extern "C" int tf_pack_voxels(const void *voxels_dev, int64_t count, void *tsdf_half_dev, uint8_t *weight_dev,
                              void *stream) {
    if (count <= 0) return TF_OK;
    if (!voxels_dev || !tsdf_half_dev || !weight_dev) return tf_set_error(TF_EINVAL, "tf_pack_voxels: null argument");
    tf::pack_voxels_kernel<<<pack_grid(count), 256, 0, (cudaStream_t)stream>>>(
        (const float2 *)voxels_dev, count, (__half *)tsdf_half_dev, weight_dev);
    return tf_check_launch("pack_voxels_kernel");
}

extern "C" int tf_unpack_voxels(const void *tsdf_half_dev, const uint8_t *weight_dev, int64_t count,
                                void *voxels_dev, void *stream) {
    if (count <= 0) return TF_OK;
    if (!voxels_dev || !tsdf_half_dev || !weight_dev) return tf_set_error(TF_EINVAL, "tf_unpack_voxels: null argument");
    tf::unpack_voxels_kernel<<<pack_grid(count), 256, 0, (cudaStream_t)stream>>>(
        (const __half *)tsdf_half_dev, weight_dev, count, (float2 *)voxels_dev);
    return tf_check_launch("unpack_voxels_kernel");
}
