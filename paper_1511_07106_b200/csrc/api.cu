// C ABI plumbing of libtfb200: version and thread-local error reporting.
#include <stdarg.h>
#include <stdio.h>

#include <atomic>

#include "tf_common.cuh"

static thread_local char g_last_error[512] = "";
static uint32_t g_debug_flags = 0;

extern "C" void tf_set_debug_flags(uint32_t flags) { g_debug_flags = flags; }
extern "C" uint32_t tf_debug_flags(void) { return g_debug_flags; }

int tf_set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
    return code;
}

// Reports (and clears) a launch-configuration error of the last launch.
// Asynchronous faults surface at the caller's next synchronisation.
void tf_count_launch(unsigned n);

int tf_check_launch(const char *what) {
    tf_count_launch(1);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return tf_set_error(TF_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e),
                            cudaGetErrorString(e));
    return TF_OK;
}

extern "C" int tf_abi_version(void) { return TFB200_ABI_VERSION; }

// Bounds violations counted by a -DTF_BOUNDS_CHECK build (tf_common.cuh,
// TF_IN_BOUNDS); UINT64_MAX from a plain build.
#ifdef TF_BOUNDS_CHECK
extern "C" unsigned long long tf_bounds_read_integrate(void);
extern "C" unsigned long long tf_bounds_read_raycast(void);
extern "C" unsigned long long tf_bounds_read_extract(void);
extern "C" unsigned long long tf_bounds_read_icp(void);
extern "C" unsigned long long tf_bounds_read_comm(void);
extern "C" uint64_t tf_debug_bounds_violations(void) {
    return tf_bounds_read_integrate() + tf_bounds_read_raycast() + tf_bounds_read_extract() +
           tf_bounds_read_icp() + tf_bounds_read_comm();
}
#else
extern "C" uint64_t tf_debug_bounds_violations(void) { return ~0ull; }
#endif

// ---- launch counting and kernel timing -------------------------------------
// Every kernel launch of the library bumps g_launches.  When profiling is on,
// the main kernel of each tf_integrate / tf_raycast call is bracketed by a
// pair of CUDA events on the caller's stream; tf_profile_read() waits for
// them and returns the summed device time per kind.
#include <mutex>
#include <vector>

static std::atomic<unsigned long long> g_launches{0};
static int g_profile_on = 0;
struct ProfPair {
    int kind;
    cudaEvent_t start, stop;
};
static std::mutex g_prof_mu;
static std::vector<ProfPair> g_prof_live;
static std::vector<ProfPair> g_prof_free;

void tf_count_launch(unsigned n) { g_launches += n; }

extern "C" uint64_t tf_launch_count(void) { return g_launches.load(); }

static int64_t *g_ray_clock = nullptr;
extern "C" void tf_debug_ray_clock_buffer(int64_t *buf) { g_ray_clock = buf; }
int64_t *tf_ray_clock_buffer() { return g_ray_clock; }

extern "C" void tf_profile_enable(int on) { g_profile_on = on; }

void *tf_profile_begin(int kind, cudaStream_t stream) {
    if (!g_profile_on) return nullptr;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    ProfPair p;
    if (!g_prof_free.empty()) {
        p = g_prof_free.back();
        g_prof_free.pop_back();
    } else {
        cudaEventCreate(&p.start);
        cudaEventCreate(&p.stop);
    }
    p.kind = kind;
    cudaEventRecord(p.start, stream);
    g_prof_live.push_back(p);
    return (void *)(uintptr_t)g_prof_live.size();
}

void tf_profile_end(void *token, cudaStream_t stream) {
    if (!token) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    const size_t i = (size_t)(uintptr_t)token - 1;
    if (i < g_prof_live.size()) cudaEventRecord(g_prof_live[i].stop, stream);
}

extern "C" int tf_profile_read(double *ms_by_kind, int64_t *launches_by_kind, int nkinds) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (int k = 0; k < nkinds; ++k) {
        ms_by_kind[k] = 0.0;
        launches_by_kind[k] = 0;
    }
    int rc = TF_OK;
    for (ProfPair &p : g_prof_live) {
        float ms = 0.f;
        if (cudaEventSynchronize(p.stop) != cudaSuccess ||
            cudaEventElapsedTime(&ms, p.start, p.stop) != cudaSuccess)
            rc = tf_set_error(TF_ECUDA, "tf_profile_read: event timing failed");
        if (p.kind >= 0 && p.kind < nkinds) {
            ms_by_kind[p.kind] += ms;
            launches_by_kind[p.kind] += 1;
        }
        g_prof_free.push_back(p);
    }
    g_prof_live.clear();
    return rc;
}

extern "C" const char *tf_last_error(void) { return g_last_error; }
