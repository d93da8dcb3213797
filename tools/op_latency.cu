// Dependent-chain latency of the ops on the raycast's per-sample critical
// path, one warp alone on the GPU (cycles per op, clock64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/op_latency tools/op_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CHAIN 4096
__global__ void lat(long long *out, double seed, const unsigned *chase_small, const unsigned *chase_big) {
    long long t0, t1;
    double d = seed;
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < CHAIN; ++i) d = __fma_rn(d, 0.999999, 1e-7);
    t1 = clock64();
    out[0] = (t1 - t0);
    double e = d;
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < CHAIN; ++i) e = __dadd_rn(e, 1e-9);
    t1 = clock64();
    out[1] = (t1 - t0);
    int k = (int)e;
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < CHAIN; ++i) k = __double2loint(__dadd_rn((double)k, 6442450944.0)) & 1023;
    t1 = clock64();
    out[2] = (t1 - t0);
    unsigned u = (unsigned)k;
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < CHAIN; ++i) u = u * 1664525u + 1013904223u;
    t1 = clock64();
    out[3] = (t1 - t0);
    float f = (float)u;
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < CHAIN; ++i) f = fmaf(f, 0.9999f, 1e-4f);
    t1 = clock64();
    out[4] = (t1 - t0);
    unsigned p = (unsigned)f & 255u;
    t0 = clock64();
    for (int i = 0; i < CHAIN; ++i) p = __ldg(&chase_small[p]);
    t1 = clock64();
    out[5] = (t1 - t0);
    t0 = clock64();
    for (int i = 0; i < CHAIN; ++i) p = __ldg(&chase_big[p]);
    t1 = clock64();
    out[6] = (t1 - t0);
    double g = (double)p;
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < CHAIN; ++i) g = (double)((int)g + 1);
    t1 = clock64();
    out[7] = (t1 - t0);
    out[8] = (long long)(d + e + f + g);
}

int main() {
    const int small = 256, big = 1 << 24;  // 1 KB (L1) and 64 MB (L2/HBM) pointer chases
    unsigned *hs = new unsigned[small], *hb = new unsigned[big];
    for (int i = 0; i < small; ++i) hs[i] = (i * 97 + 13) % small;
    unsigned long long x = 88172645463325252ull;
    for (int i = 0; i < big; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        hb[i] = (unsigned)(x % big);
    }
    unsigned *ds, *db;
    long long *dout, hout[9];
    cudaMalloc(&ds, small * 4); cudaMalloc(&db, (size_t)big * 4); cudaMalloc(&dout, 9 * 8);
    cudaMemcpy(ds, hs, small * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, hb, (size_t)big * 4, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) lat<<<1, 32>>>(dout, 1.0, ds, db);
    cudaMemcpy(hout, dout, 9 * 8, cudaMemcpyDeviceToHost);
    const char *names[] = {"DFMA", "DADD", "DADD+lo32+LOP (fixed_bits)", "IMAD", "FFMA",
                           "LDG L1-hit chase", "LDG 64MB chase (L2/HBM)", "F2I+I2F.F64"};
    for (int i = 0; i < 8; ++i) printf("%-28s %7.1f cycles\n", names[i], (double)hout[i] / CHAIN);
    return 0;
}
