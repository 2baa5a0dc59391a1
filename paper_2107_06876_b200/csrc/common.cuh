// Shared device helpers for the LCN-Sinkhorn hot path (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cmath>
#include <mutex>
#include <set>
#include <utility>
#include <stdexcept>
#include <string>

namespace lcnb {

// ---- status / errors --------------------------------------------------------
// Host-side exception carrying an lcn_status; converted at the C-ABI edge.
struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Status(100, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CUDA_OK(x) ::lcnb::cuda_check((x), #x)
#define LAUNCH_OK(what) ::lcnb::cuda_check(cudaGetLastError(), what)

// Kernels whose dynamic shared memory varies between calls get the device's
// opt-in maximum once per (kernel, device). A per-call cudaFuncSetAttribute
// races with launches from other host threads (the build runs its k-means
// jobs on parallel threads): one thread could lower the limit just before
// another thread's larger launch.
template <class K>
void allow_max_dyn_smem(K* kernel) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> g(mu);
    if (!done.insert({reinterpret_cast<const void*>(kernel), dev}).second) return;
    int optin = 0;
    cuda_check(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev),
               "cudaDeviceGetAttribute(MaxSharedMemoryPerBlockOptin)");
    cudaFuncAttributes fa{};
    cuda_check(cudaFuncGetAttributes(&fa, kernel), "cudaFuncGetAttributes");
    cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    optin - static_cast<int>(fa.sharedSizeBytes)),
               "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
}

// ---- exact fp64 arithmetic -------------------------------------------------
// The reference computes in plain fp64 with no FMA contraction (built without
// -march). Every op that must reproduce its bits uses the
// explicitly rounded intrinsics so nvcc cannot contract a*b+c into an FMA.
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }

// kmeans.cpp:12-19 sqdist: s = 0; for k: diff = x_k - y_k; s += diff*diff.
template <typename TX, typename TY>
__device__ __forceinline__ double sqdist_exact(const TX* x, const TY* y, int d) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
        double diff = xsub(static_cast<double>(x[k]), static_cast<double>(y[k]));
        s = xadd(s, xmul(diff, diff));
    }
    return s;
}

// geometry.cpp:45-76 cost_value (+ the documented squared-L2 kind 3),
// same operation order, no contraction.
template <typename TX, typename TY>
__device__ __forceinline__ double cost_exact(int kind, const TX* x, const TY* y, int d) {
    if (kind == 0 || kind == 3) {
        double s = sqdist_exact(x, y, d);
        return kind == 0 ? __dsqrt_rn(s) : s;
    }
    if (kind == 1) {
        double s = 0.0;
        for (int k = 0; k < d; ++k) s = xadd(s, xmul(static_cast<double>(x[k]), static_cast<double>(y[k])));
        return -s;
    }
    double dot = 0.0, nx = 0.0, ny = 0.0;
    for (int k = 0; k < d; ++k) {
        double a = static_cast<double>(x[k]), b = static_cast<double>(y[k]);
        dot = xadd(dot, xmul(a, b));
        nx = xadd(nx, xmul(a, a));
        ny = xadd(ny, xmul(b, b));
    }
    if (nx == 0.0 || ny == 0.0) return __longlong_as_double(0x7ff8000000000001ll);  // flagged by caller
    double c = __ddiv_rn(dot, __dsqrt_rn(xmul(nx, ny)));
    c = c > 1.0 ? 1.0 : c;
    c = c < -1.0 ? -1.0 : c;
    return __dsqrt_rn(xsub(1.0, c));
}

// ---- warp / block reductions ------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

constexpr double kNegInf = -__builtin_huge_val();
constexpr double kPosInf = __builtin_huge_val();

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// ---- programmatic dependent launch (sm_90+) ---------------------------------
// A chain of short dependent kernels (the k-means++ step) pays a kernel
// boundary per launch. Launched with programmatic stream serialisation, the
// next kernel is set up while this one runs: its CTAs start once every CTA
// of this grid has executed pdl_launch_dependents() (or exited) and block in
// pdl_wait() until this grid has completed and its writes are visible. Both
// are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    CUDA_OK(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(std::forward<Args>(args))...));
}

}  // namespace lcnb
