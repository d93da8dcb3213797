// Shared device helpers for libtfb200 (sm_100a).
//
// Exactness: the reference kernels are numba-compiled scalar FP64 with no
// FMA contraction.  Every arithmetic step on an exact path
// goes through the round-to-nearest intrinsics below, which the compiler
// never fuses or reorders, so results do not depend on -fmad.  The library
// is additionally built with --fmad=false.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tfb200.h"

namespace tf {

// ---- exact IEEE round-to-nearest building blocks -------------------------
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fmulr(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fsubr(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fdivr(float a, float b) { return __fdiv_rn(a, b); }

// Python's left-to-right a*b + c*d + e*f + g without contraction.
__device__ __forceinline__ double dot3_plus(double a0, double b0, double a1, double b1,
                                            double a2, double b2, double c) {
    return dadd(dadd(dadd(dmul(a0, b0), dmul(a1, b1)), dmul(a2, b2)), c);
}

// ---- small POD parameter blocks passed by value ---------------------------
struct Mat3 {
    double m[9];
};
struct Vec3 {
    double v[3];
};

struct VolumeTable {
    int count;
    TfVolume vol[TFB200_MAX_VOLUMES_PER_LAUNCH];
};

__device__ __forceinline__ int64_t vox_index(int64_t n, int64_t z, int64_t y, int64_t x) {
    return (z * n + y) * n + x;
}

// Free-space summary threshold: a voxel is "good" when observed and its tsdf
// >= T, T = 0.99 tau (1 + 4e-6) rounded up to float32.  Any trilinear value of
// good corners is then > 0.99 tau (the reference's near-surface threshold,
// _kernels.py:25, :298) with margin far above float64 rounding.
__host__ __device__ inline float good_threshold(double tau) {
    const double near = 0.99 * tau;
    const double want = near * (1.0 + 4e-6);
    float t = (float)want;
    if ((double)t < want) t = nextafterf(t, 3.0e38f);
    return t;
}

__device__ __forceinline__ int voxel_bad(float2 v, float t) { return !(v.y > 0.0f && v.x >= t); }

// packed brick-state contribution of one voxel: not-good (low 16 bits) and
// observed (high 16 bits); deltas of packed values add up exactly mod 2^32
__device__ __forceinline__ unsigned voxel_state(float2 v, float t) {
    return (unsigned)voxel_bad(v, t) | ((v.y > 0.0f ? 1u : 0u) << 16);
}

// _hit_wins (_kernels.py:246-263) on (t, normal) records: the smaller t wins;
// on an exact tie the larger nx, then ny, then nz.  A strict total order, so
// folds over partial ray maps are order-free.
__device__ __forceinline__ bool record_wins(double t, double nx, double ny, double nz, double ct,
                                            double cnx, double cny, double cnz) {
    if (t < ct) return true;
    if (t > ct) return false;
    if (nx != cnx) return nx > cnx;
    if (ny != cny) return ny > cny;
    return nz > cnz;
}

// ---- bounds-checked debug build (-DTF_BOUNDS_CHECK) ------------------------
// compute-sanitizer is closed on the GPU pool; this build stands in for its
// memcheck: every guarded index is checked, a violation is counted (per
// translation unit) and the access is skipped instead of faulting.
// tf_debug_bounds_violations() (api.cu) sums the counters; the plain build
// compiles the guards away (TF_IN_BOUNDS(c) == true).
#ifdef TF_BOUNDS_CHECK
static __device__ unsigned long long tf_bounds_hits;
#define TF_IN_BOUNDS(cond) ((cond) || (atomicAdd(&::tf::tf_bounds_hits, 1ull), false))
#define TF_BOUNDS_READER(name)                                                              \
    extern "C" unsigned long long tf_bounds_read_##name(void) {                           \
        unsigned long long v = 0;                                                           \
        cudaMemcpyFromSymbol(&v, ::tf::tf_bounds_hits, sizeof(v));                         \
        return v;                                                                           \
    }
#else
#define TF_IN_BOUNDS(cond) true
#define TF_BOUNDS_READER(name)
#endif

// Warp-aggregated 64-bit counter add (integer: order-independent, exact).
__device__ __forceinline__ void warp_count_add(unsigned long long *dst, unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// Block-aggregated counter adds for the end of a persistent kernel: every
// warp of the grid finishes at about the same time, and per-warp atomics on a
// handful of addresses then queue up behind each other; here the warps' sums
// meet in shared memory and one thread per block adds each counter.  Every
// thread of the block must call it.
template <int N>
__device__ __forceinline__ void block_count_add(unsigned long long *const (&dst)[N],
                                                const unsigned long long (&v)[N]) {
    __shared__ unsigned long long part[N];
    if (threadIdx.x < N) part[threadIdx.x] = 0ull;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < N; ++i) {
        unsigned long long s = v[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((threadIdx.x & 31) == 0 && s) atomicAdd_block(&part[i], s);
    }
    __syncthreads();
    if (threadIdx.x < N && part[threadIdx.x]) atomicAdd(dst[threadIdx.x], part[threadIdx.x]);
}

}  // namespace tf

// ---- host-side error plumbing (api.cu) --------------------------------------
int tf_set_error(int code, const char *fmt, ...);
int tf_check_launch(const char *what);
void tf_count_launch(unsigned n);
int64_t *tf_ray_clock_buffer();
void *tf_profile_begin(int kind, cudaStream_t stream);
void tf_profile_end(void *token, cudaStream_t stream);
