// Multi-GPU ray-map reduction over peer memory (sm_100a, NVLink / NVSwitch).
//
// every rank raycasts only the volumes it owns into a partial
// ray map; the partials are reduced with the _hit_wins total order
// (_kernels.py:246-263) and every rank needs the merged model (ICP runs
// replicated on it).  Instead of NCCL collectives (all-to-all of packed
// records, a merge launch per peer, an all-gather and copies), each rank runs
// ONE kernel that reads its row block of every peer's partial straight out of
// the peers' HBM (CUDA IPC mappings), folds the records in rank order, and
// stores the merged rows straight into every rank's model — the exchange and
// the merge are the same loads and stores.  Synchronisation is two flag
// waves through the same mappings (release / acquire at system scope):
//
//   ready  every block of the reduce kernel tells every peer "my partial
//          is final" (the raycast precedes it on the stream; the first
//          resident block raises it); every block waits for all ranks'
//          ready before reading;
//   done   the reduce kernel's last block (grid-wide counter) tells every
//          peer "my rows are in your model and I have stopped reading your
//          partial"; comm_wait_done_kernel (one warp) waits for all ranks'
//          done, so the local model is complete for the next kernel on the
//          stream, and the next frame's raycast may overwrite the partial.
//
// A peer can only write into this rank's model after this rank's ready for
// the same frame, which the stream orders after every read of the previous
// model (ICP), so the model is never overwritten while in use.  Waits give up
// after TF_COMM_TIMEOUT_NS with the region's error flag raised (no hang).
//
// Exactness: the winner is chosen by the strict total order, and its vertex
// is the one its raycast wrote (not recomputed), so every rank's model equals
// the single-GPU raycast over all volumes bit for bit (the reference's
// order-free merge, test_acceptance.py:349-361).  On one device the data path
// is tested with emulated ranks (TF_COMM_NOWAIT: one kernel per rank, no
// waits — ranks that wait on one another never share a GPU).
#include <stddef.h>
#include <string.h>

#include <new>

#include "tf_common.cuh"

struct TfComm {
    int rank = 0, world = 1, dev = 0, grid = 1;
    int64_t width = 0, height = 0;
    char *base = nullptr;
    size_t bytes = 0;
    int64_t off[TF_COMM_NSECTIONS] = {};
    char *peer[TF_COMM_MAX_RANKS] = {};
    bool ipc_opened[TF_COMM_MAX_RANKS] = {};
    unsigned long long epoch = 0;
    unsigned *err_host = nullptr;  // pinned copy of the error flag, refreshed after every reduction
};

namespace tf {
namespace {

constexpr int64_t kFlagsBytes = 4096;

struct CommFlags {
    unsigned long long ready[TF_COMM_MAX_RANKS];  // [r] = last frame rank r's partial was final
    unsigned long long done[TF_COMM_MAX_RANKS];   // [r] = last frame rank r finished its rows
    unsigned long long counter;                   // finished blocks of this rank's reduce kernels
    unsigned error;                               // 1: a wait timed out
};
static_assert(sizeof(CommFlags) <= (size_t)kFlagsBytes, "flags section too small");

struct PeerTable {
    char *base[TF_COMM_MAX_RANKS];
    int64_t off[TF_COMM_NSECTIONS];
    int rank, world, wait;
    int64_t width, row0, nrows;
    unsigned long long epoch;
};

template <typename T>
__device__ __forceinline__ T *section(const PeerTable &pt, int r, int s) {
    return reinterpret_cast<T *>(pt.base[r] + pt.off[s]);
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// spin until *flag >= epoch; after the timeout raise the error flag and go
// on.  Once the flag is raised every later wait returns at once, so a broken
// exchange costs one timeout, not one per frame (the host reports the error).
__device__ void wait_flag(const unsigned long long *flag, unsigned long long epoch, unsigned *error) {
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(flag) < epoch) {
        if (*(volatile unsigned *)error || globaltimer_ns() - t0 > TF_COMM_TIMEOUT_NS) {
            atomicOr(error, 1u);
            return;
        }
        __nanosleep(100);
    }
}

__global__ void __launch_bounds__(256) raymap_reduce_kernel(const __grid_constant__ PeerTable pt) {
    CommFlags *mine = section<CommFlags>(pt, pt.rank, TF_COMM_FLAGS);
    if (pt.wait) {
        // my partial is final (the raycast precedes this kernel on the stream)
        // -> every rank.  Every block raises it (the same value, idempotent),
        // so the flag goes up as soon as ANY block of the grid is resident —
        // no rank waits on a block of another rank that is still queued behind
        // whatever else that GPU runs
        if (threadIdx.x < pt.world) {
            __threadfence_system();
            st_release_sys(&section<CommFlags>(pt, threadIdx.x, TF_COMM_FLAGS)->ready[pt.rank], pt.epoch);
        }
        if (threadIdx.x < pt.world) wait_flag(&mine->ready[threadIdx.x], pt.epoch, &mine->error);
        __syncthreads();
    }
    const int64_t npix = pt.nrows * pt.width, p0 = pt.row0 * pt.width;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npix;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = p0 + i;
        if (!TF_IN_BOUNDS(p < pt.width * (pt.row0 + pt.nrows))) break;
        // rank 0's record, then the others folded in rank order (merge_blocks)
        const double *n0 = section<const double>(pt, 0, TF_COMM_PART_NORM) + 3 * p;
        double t = __ldcv(section<const double>(pt, 0, TF_COMM_PART_DIST) + p);
        double nx = __ldcv(n0), ny = __ldcv(n0 + 1), nz = __ldcv(n0 + 2);
        int win = 0;
        for (int r = 1; r < pt.world; ++r) {
            const double *nr = section<const double>(pt, r, TF_COMM_PART_NORM) + 3 * p;
            const double rt = __ldcv(section<const double>(pt, r, TF_COMM_PART_DIST) + p);
            const double rx = __ldcv(nr), ry = __ldcv(nr + 1), rz = __ldcv(nr + 2);
            if (record_wins(rt, rx, ry, rz, t, nx, ny, nz)) {
                win = r;
                t = rt;
                nx = rx;
                ny = ry;
                nz = rz;
            }
        }
        // the winner's vertex as its raycast wrote it (0 when no rank hit)
        const double *wv = section<const double>(pt, win, TF_COMM_PART_VERT) + 3 * p;
        const double vx = __ldcv(wv), vy = __ldcv(wv + 1), vz = __ldcv(wv + 2);
        for (int r = 0; r < pt.world; ++r) {  // all-gather by stores
            section<double>(pt, r, TF_COMM_MODEL_DIST)[p] = t;
            double *mv = section<double>(pt, r, TF_COMM_MODEL_VERT) + 3 * p;
            double *mn = section<double>(pt, r, TF_COMM_MODEL_NORM) + 3 * p;
            mv[0] = vx;
            mv[1] = vy;
            mv[2] = vz;
            mn[0] = nx;
            mn[1] = ny;
            mn[2] = nz;
        }
    }
    if (pt.wait) {
        __shared__ int last;
        __threadfence_system();  // this thread's peer stores are performed system-wide
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long old = atomicAdd(&mine->counter, 1ull);
            __threadfence_system();
            last = old + 1ull == pt.epoch * (unsigned long long)gridDim.x;
        }
        __syncthreads();
        if (last && threadIdx.x < pt.world) {  // every block's rows are out -> every rank
            __threadfence_system();
            st_release_sys(&section<CommFlags>(pt, threadIdx.x, TF_COMM_FLAGS)->done[pt.rank], pt.epoch);
        }
    }
}

__global__ void comm_wait_done_kernel(const __grid_constant__ PeerTable pt) {
    CommFlags *mine = section<CommFlags>(pt, pt.rank, TF_COMM_FLAGS);
    if (threadIdx.x < pt.world) wait_flag(&mine->done[threadIdx.x], pt.epoch, &mine->error);
}

__global__ void fill_f64_kernel(double *p, int64_t n, double v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

int cuda_fail(cudaError_t e, const char *what) {
    return tf_set_error(TF_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

}  // namespace
}  // namespace tf

using tf::cuda_fail;

TF_BOUNDS_READER(comm)

extern "C" int tf_comm_create(int rank, int world, int64_t width, int64_t height, TfComm **out) {
    if (!out || world < 1 || world > TF_COMM_MAX_RANKS || rank < 0 || rank >= world || width < 1 ||
        height < 1)
        return tf_set_error(TF_EINVAL, "tf_comm_create: bad argument");
    *out = nullptr;
    TfComm *c = new (std::nothrow) TfComm();
    if (!c) return tf_set_error(TF_EINVAL, "tf_comm_create: out of host memory");
    c->rank = rank;
    c->world = world;
    c->width = width;
    c->height = height;
    cudaGetDevice(&c->dev);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->dev);
    c->grid = sms;  // one block per SM: every block of the reduce kernel is resident
    const int64_t px = width * height;
    const int64_t sizes[TF_COMM_NSECTIONS] = {tf::kFlagsBytes, 8 * px, 24 * px, 24 * px,
                                              8 * px,           24 * px, 24 * px};
    int64_t off = 0;
    for (int s = 0; s < TF_COMM_NSECTIONS; ++s) {
        c->off[s] = off;
        off += (sizes[s] + 255) / 256 * 256;
    }
    c->bytes = (size_t)off;
    cudaError_t e = cudaMalloc((void **)&c->base, c->bytes);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "tf_comm_create: cudaMalloc");
    }
    // zero flags and vectors, +inf distances (RayMap.empty)
    e = cudaMemset(c->base, 0, c->bytes);
    if (e == cudaSuccess) {
        tf::fill_f64_kernel<<<256, 256>>>((double *)(c->base + c->off[TF_COMM_PART_DIST]), px, INFINITY);
        tf::fill_f64_kernel<<<256, 256>>>((double *)(c->base + c->off[TF_COMM_MODEL_DIST]), px, INFINITY);
        tf_count_launch(2);
        e = cudaDeviceSynchronize();
    }
    if (e != cudaSuccess) {
        cudaFree(c->base);
        delete c;
        return cuda_fail(e, "tf_comm_create: init");
    }
    e = cudaHostAlloc((void **)&c->err_host, sizeof(unsigned), cudaHostAllocDefault);
    if (e != cudaSuccess) {
        cudaFree(c->base);
        delete c;
        return cuda_fail(e, "tf_comm_create: cudaHostAlloc");
    }
    *c->err_host = 0u;
    c->peer[rank] = c->base;
    *out = c;
    return TF_OK;
}

extern "C" int tf_comm_layout(const TfComm *c, void **base, int64_t *offsets) {
    if (!c || !base || !offsets) return tf_set_error(TF_EINVAL, "tf_comm_layout: null argument");
    *base = c->base;
    for (int s = 0; s < TF_COMM_NSECTIONS; ++s) offsets[s] = c->off[s];
    return TF_OK;
}

extern "C" int tf_comm_export(const TfComm *c, void *handle) {
    if (!c || !handle) return tf_set_error(TF_EINVAL, "tf_comm_export: null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == TF_COMM_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, c->base);
    if (e != cudaSuccess) return cuda_fail(e, "tf_comm_export: cudaIpcGetMemHandle");
    memcpy(handle, &h, sizeof(h));
    return TF_OK;
}

extern "C" int tf_comm_import(TfComm *c, const void *handles) {
    if (!c || !handles) return tf_set_error(TF_EINVAL, "tf_comm_import: null argument");
    for (int r = 0; r < c->world; ++r) {
        if (r == c->rank || c->ipc_opened[r]) continue;
        cudaIpcMemHandle_t h;
        memcpy(&h, (const char *)handles + (size_t)r * TF_COMM_HANDLE_BYTES, sizeof(h));
        void *p = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return cuda_fail(e, "tf_comm_import: cudaIpcOpenMemHandle");
        c->peer[r] = (char *)p;
        c->ipc_opened[r] = true;
    }
    return TF_OK;
}

extern "C" int tf_comm_link_local(TfComm *const *comms, int world) {
    if (!comms || world < 1 || world > TF_COMM_MAX_RANKS)
        return tf_set_error(TF_EINVAL, "tf_comm_link_local: bad argument");
    for (int i = 0; i < world; ++i)
        if (!comms[i] || comms[i]->rank != i || comms[i]->world != world ||
            comms[i]->width != comms[0]->width || comms[i]->height != comms[0]->height)
            return tf_set_error(TF_EINVAL, "tf_comm_link_local: comms must be ranks 0..world-1 of one shape");
    for (int i = 0; i < world; ++i)
        for (int r = 0; r < world; ++r) comms[i]->peer[r] = comms[r]->base;
    return TF_OK;
}

extern "C" int tf_comm_reduce_raymap(TfComm *c, unsigned flags, void *stream_) {
    if (!c) return tf_set_error(TF_EINVAL, "tf_comm_reduce_raymap: null argument");
    for (int r = 0; r < c->world; ++r)
        if (!c->peer[r]) return tf_set_error(TF_EINVAL, "tf_comm_reduce_raymap: rank %d not mapped", r);
    const cudaStream_t stream = (cudaStream_t)stream_;
    const bool wait = !(flags & TF_COMM_NOWAIT);
    tf::PeerTable pt{};
    for (int r = 0; r < c->world; ++r) pt.base[r] = c->peer[r];
    for (int s = 0; s < TF_COMM_NSECTIONS; ++s) pt.off[s] = c->off[s];
    pt.rank = c->rank;
    pt.world = c->world;
    pt.wait = wait ? 1 : 0;
    pt.width = c->width;
    const int64_t rows = (c->height + c->world - 1) / c->world;  // distributed.row_block
    pt.row0 = (int64_t)c->rank * rows < c->height ? (int64_t)c->rank * rows : c->height;
    pt.nrows = pt.row0 + rows < c->height ? rows : c->height - pt.row0;
    if (wait) pt.epoch = ++c->epoch;
    tf::raymap_reduce_kernel<<<c->grid, 256, 0, stream>>>(pt);
    int rc = tf_check_launch("raymap_reduce_kernel");
    if (rc || !wait) return rc;
    tf::comm_wait_done_kernel<<<1, 64, 0, stream>>>(pt);
    rc = tf_check_launch("comm_wait_done_kernel");
    if (rc) return rc;
    // stream-ordered copy of the (sticky) error flag into pinned memory, so
    // the host can poll it every frame without a synchronisation
    const cudaError_t e = cudaMemcpyAsync(c->err_host, c->base + c->off[TF_COMM_FLAGS] + offsetof(tf::CommFlags, error),
                                          sizeof(unsigned), cudaMemcpyDeviceToHost, stream);
    return e == cudaSuccess ? TF_OK : cuda_fail(e, "tf_comm_reduce_raymap: error flag copy");
}

extern "C" int tf_comm_error_poll(const TfComm *c, int *error) {
    if (!c || !error) return tf_set_error(TF_EINVAL, "tf_comm_error_poll: null argument");
    *error = (int)*(volatile unsigned *)c->err_host;
    return TF_OK;
}

extern "C" int tf_comm_error(const TfComm *c, int *error) {
    if (!c || !error) return tf_set_error(TF_EINVAL, "tf_comm_error: null argument");
    unsigned v = 0;
    const cudaError_t e = cudaMemcpy(&v, c->base + c->off[TF_COMM_FLAGS] + offsetof(tf::CommFlags, error),
                                     sizeof(v), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "tf_comm_error");
    *error = (int)v;
    return TF_OK;
}

extern "C" int tf_comm_destroy(TfComm *c) {
    if (!c) return TF_OK;
    for (int r = 0; r < c->world; ++r)
        if (c->ipc_opened[r]) cudaIpcCloseMemHandle(c->peer[r]);
    cudaFree(c->base);
    if (c->err_host) cudaFreeHost(c->err_host);
    delete c;
    return TF_OK;
}
