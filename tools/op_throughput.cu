// Microbenchmark: per-SM throughput of the instruction classes the exact
// kernels lean on (FP64 arithmetic, double<->float/int conversions, floor,
// division, square root).  Many independent chains per thread, full grid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/opt tools/op_throughput.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

#define KERNEL(name, T, init, body)                                              \
    __global__ void name(T *out, T seed) {                                       \
        T v[CH];                                                                 \
        _Pragma("unroll") for (int c = 0; c < CH; ++c) v[c] = init;              \
        for (int i = 0; i < ITERS; ++i) {                                        \
            _Pragma("unroll") for (int c = 0; c < CH; ++c) { T x = v[c]; body; v[c] = x; } \
        }                                                                        \
        T s = 0;                                                                 \
        _Pragma("unroll") for (int c = 0; c < CH; ++c) s += v[c];                \
        if (s == (T)-12345.678) out[threadIdx.x] = s;                            \
    }

KERNEL(k_dfma, double, seed + c, x = __fma_rn(x, 1.0000001, 1e-9))
KERNEL(k_ffma, float, seed + c, x = __fmaf_rn(x, 1.0000001f, 1e-9f))
KERNEL(k_dadd, double, seed + c, x = __dadd_rn(x, 1e-9))
KERNEL(k_f2f_up, double, seed + c, x = (double)(float)x + 1e-9)        // F2F.F32.F64 + F2F.F64.F32
KERNEL(k_d2i, double, seed + c, x = (double)__double2int_rd(x) + 0.25) // F2I.F64 + I2F.F64
KERNEL(k_floor, double, seed + c, x = floor(x) + 0.25)                 // FRND.F64
KERNEL(k_ddiv, double, seed + c, x = __ddiv_rn(1.0000001, x) + 1.0)
KERNEL(k_dsqrt, double, seed + c + 2.0, x = __dsqrt_rn(x) + 1.0)
KERNEL(k_rcp64h, double, seed + c + 2.0, x = __drcp_rn(x) + 1.0)
KERNEL(k_frcp, float, seed + c + 2.0f, x = __frcp_rn(x) + 1.0f)
KERNEL(k_f2i32, float, seed + c, x = (float)__float2int_rd(x) + 0.25f)  // F2I + I2F fp32

template <typename K, typename T>
void run(const char *name, K k, T seed, int ops_per_body) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    T *out;
    cudaMalloc(&out, 1024 * sizeof(T));
    dim3 grid(sms * 8), block(256);
    k<<<grid, block>>>(out, seed);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<<<grid, block>>>(out, seed);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double thread_ops = 5.0 * grid.x * block.x * (double)ITERS * CH * ops_per_body;
    const double per_s = thread_ops / (ms * 1e-3);
    // lanes / clk / SM at the max clock (clocks may be lower under load)
    printf("%-10s %8.3f ms  %9.1f Gop/s  %6.1f lane-ops/clk/SM (at %d MHz)\n", name, ms, per_s / 1e9,
           per_s / (sms * (clk * 1e3)), clk / 1000);
    cudaFree(out);
}

int main() {
    run("DFMA", k_dfma, 1.0, 1);
    run("FFMA", k_ffma, 1.0f, 1);
    run("DADD", k_dadd, 1.0, 1);
    run("F2F x2", k_f2f_up, 1.0, 2);
    run("F2I+I2F64", k_d2i, 1.5, 2);
    run("floor64", k_floor, 1.5, 1);
    run("DDIV", k_ddiv, 1.5, 1);
    run("DSQRT", k_dsqrt, 1.5, 1);
    run("DRCP_rn", k_rcp64h, 1.5, 1);
    run("FRCP_rn", k_frcp, 1.5f, 1);
    run("F2I+I2F32", k_f2i32, 1.5f, 2);
    return 0;
}
