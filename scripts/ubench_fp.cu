// Throughput probe: DFMA, F2F.F64.F32 (+DFMA), FFMA per SM per clock.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters, float seed) {
    float f[8]; double d[8];
    for (int j = 0; j < 8; ++j) { f[j] = seed + threadIdx.x + j; d[j] = f[j]; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (MODE == 0) d[j] = fma(d[j], 0.999, 1e-3);
            if (MODE == 1) { d[j] = fma((double)f[j], 0.999, d[j]); f[j] += 1.0f; }
            if (MODE == 2) f[j] = fmaf(f[j], 0.999f, 1e-3f);
        }
    }
    double s = 0; for (int j = 0; j < 8; ++j) s += d[j] + f[j];
    if (s == 12345.0) out[0] = s;
}
int main() {
    float* o; cudaMalloc(&o, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096, blocks = sms * 4, threads = 512;
    const char* names[3] = {"DFMA", "F2F.F64.F32+DFMA", "FFMA(+FADD)"};
    for (int m = 0; m < 3; ++m) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (m == 0) k<0><<<blocks, threads>>>(o, iters, 1.f);
            if (m == 1) k<1><<<blocks, threads>>>(o, iters, 1.f);
            if (m == 2) k<2><<<blocks, threads>>>(o, iters, 1.f);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = (double)blocks * threads * iters * 8;
            if (rep) printf("%-20s %8.3f ms  %8.1f Gop/s  %6.1f op/clk/SM (clk %d MHz)\n", names[m], ms, ops / ms / 1e6,
                            ops / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000);
        }
    }
    return 0;
}
