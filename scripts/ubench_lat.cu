// Single-warp dependent-chain latency probe (cycles per op) for the ops on
// the k-means++ walk's critical path.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, long long* cyc, int iters, double seed) {
    double d = seed + threadIdx.x * 1e-9;
    long long li = threadIdx.x + 3;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (MODE == 0) d = __dadd_rn(d, 1.0000001);
            if (MODE == 1) d = __dmul_rn(d, 0.9999999);
            if (MODE == 2) d = fma(d, 0.9999999, 1e-9);
            if (MODE == 3) li = li + ((li & 1) ? 7 : 3);
            if (MODE == 4) d = __shfl_sync(0xffffffffu, d, (threadIdx.x + 1) & 31);
            if (MODE == 5) { d = floor(d * 1.5); }
            if (MODE == 6) { li = __double2ll_rn((double)li * 1.0000001); }
        }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = d + (double)li;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
    const char* names[] = {"DADD", "DMUL", "DFMA", "IADD64+SEL parity", "SHFL.f64", "DMUL+FRND", "I2F+DMUL+F2I"};
    for (int m = 0; m < 7; ++m) {
        long long h = 0;
        for (int rep = 0; rep < 2; ++rep) {
            if (m == 0) k<0><<<1, 32>>>(o, c, 1000, 1.0);
            if (m == 1) k<1><<<1, 32>>>(o, c, 1000, 1.0);
            if (m == 2) k<2><<<1, 32>>>(o, c, 1000, 1.0);
            if (m == 3) k<3><<<1, 32>>>(o, c, 1000, 1.0);
            if (m == 4) k<4><<<1, 32>>>(o, c, 1000, 1.0);
            if (m == 5) k<5><<<1, 32>>>(o, c, 1000, 1.0);
            if (m == 6) k<6><<<1, 32>>>(o, c, 1000, 1.0);
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        }
        printf("%-20s %6.1f cycles/op\n", names[m], h / 16000.0);
    }
    return 0;
}
