// Dense anchor with the kernel recomputed every half-iteration (configs[2]:
// "exp(-C/lambda) is recomputed on the fly per iteration as a tensor-core GEMM
// fused with log-sum-exp"): no n x m storage. The reference streams a stored
// log K (operator.cpp:125-140 rows, :178-192 columns; build_cost / build_kernel
// geometry.cpp:113-144); here each half-iteration is
//   out_i = LSE_j( -c(x_i, y_j) / lambda + log v_j )
// with x.y from tcgen05 3xTF32 MMAs (tc_block.cuh operands and pipeline),
// c(x, y) from the dot and exact fp64 norms, and the log-sum-exp fused into
// the epilogue: per (row, 128-column tile) a partial (max, sum), merged per
// row in tile order by a second kernel (deterministic).
//
// CTA (persistent, one per SM): warp 0 bulk-copies the row tile's and the
// column tile's k-blocks into a 2-stage ring, warp 1 issues
// tcgen05.mma.kind::tf32 (hi.hi + hi.lo + lo.hi) into one of two TMEM
// accumulators, 8 epilogue warps tcgen05.ld the 128 x 128 dots to a shared
// staging tile and reduce each row with its lanes along the columns.
#include "op.cuh"
#include "tc_block.cuh"

namespace lcnb {

namespace {

using namespace tcb;

// The cost from the FP32-accurate dot and the fp64 norms (cost_value,
// geometry.cpp:45-76), in fp32: the dot already carries ~1e-7 relative error,
// and fp32 keeps the epilogue off the fp64 pipe (sqrt in fp64 is a
// multi-instruction sequence per entry).
__device__ __forceinline__ float dense_cost(int kind, float dot, float nx, float ny) {
    if (kind == 1) return -dot;
    if (kind == 2) {
        float c = dot * rsqrtf(nx * ny);
        c = fminf(fmaxf(c, -1.0f), 1.0f);
        return sqrtf(1.0f - c);
    }
    const float sq = fmaxf(nx + ny - 2.0f * dot, 0.0f);
    return kind == 0 ? sqrtf(sq) : sq;
}

// items: it -> (row tile it / ntb, column tile it % ntb)
__global__ void __launch_bounds__(kThreads, 1) dense_lse_tc_kernel(const unsigned char* __restrict__ A,
                                                                   const unsigned char* __restrict__ B, int KB,
                                                                   int nta, int ntb, long long rows, long long cols,
                                                                   const double* __restrict__ na,
                                                                   const double* __restrict__ nb, int kind, double inv,
                                                                   const double* __restrict__ lv,
                                                                   const int* __restrict__ done,
                                                                   double* __restrict__ PM, double* __restrict__ PS) {
    if (done && *done) return;
    extern __shared__ __align__(1024) unsigned char dyn_raw[];
    const uint32_t raw = smem_u32(dyn_raw);
    unsigned char* ring = dyn_raw + ((1024u - (raw & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + kStages * kStage);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* tfull = bars + 2 * kStages;
    uint64_t* tempty = tfull + kAcc;
    uint32_t& tmem_slot = *reinterpret_cast<uint32_t*>(tempty + kAcc);
    float* stage = reinterpret_cast<float*>(ring + kStages * kStage + 128);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nitems = nta * ntb;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                     "n"(kAcc * kM)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < kAcc; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 32 * kEpiWarps);
        }
        fence_mbar_init();
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_slot;
    const size_t tile_bytes = static_cast<size_t>(KB) * kKBlock;

    if (warp == 0) {
        if (lane == 0) {
            uint32_t g = 0;
            for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
                const unsigned char* a = A + static_cast<size_t>(it / ntb) * tile_bytes;
                const unsigned char* b = B + static_cast<size_t>(it % ntb) * tile_bytes;
                for (int kb = 0; kb < KB; ++kb, ++g) {
                    const uint32_t s = g % kStages;
                    if (g >= kStages) mbar_wait_spin(&empty[s], ((g / kStages) - 1) & 1);
                    mbar_arrive_expect_tx(&full[s], kStage);
                    bulk_g2s(ring + s * kStage, a + static_cast<size_t>(kb) * kKBlock, kKBlock, &full[s]);
                    bulk_g2s(ring + s * kStage + kKBlock, b + static_cast<size_t>(kb) * kKBlock, kKBlock, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
        uint32_t g = 0, j = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++j) {
            const uint32_t buf = j % kAcc;
            if (j >= kAcc) mbar_wait_spin(&tempty[buf], ((j / kAcc) - 1) & 1);
            fence_after();
            const uint32_t dt = tmem + buf * kM;
            for (int kb = 0; kb < KB; ++kb, ++g) {
                const uint32_t s = g % kStages;
                mbar_wait_spin(&full[s], (g / kStages) & 1);
                fence_after();
                const uint32_t base = smem_u32(ring + s * kStage);
                const uint64_t ah = desc_sw128(base), al = desc_sw128(base + kHalf);
                const uint64_t bh = desc_sw128(base + kKBlock), bl = desc_sw128(base + kKBlock + kHalf);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint64_t off = static_cast<uint64_t>(ks * 32) >> 4;
                    mma_ss_elect(dt, ah + off, bh + off, (kb | ks) ? 1u : 0u);
                    mma_ss_elect(dt, ah + off, bl + off, 1u);
                    mma_ss_elect(dt, al + off, bh + off, 1u);
                }
                commit_elect(&empty[s]);
            }
            commit_elect(&tfull[buf]);
        }
        __syncwarp();
    } else {
        const int q = warp & 3;
        const int row = 32 * q + lane;
        const int c0 = ((warp - 2) >> 2) * kEpiCols;
        const int ew = warp - 2;
        uint32_t j = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++j) {
            const uint32_t buf = j % kAcc;
            const int at = it / ntb, ct = it % ntb;
            // this lane's columns of the tile: lane + 32 k
            double cl[4];
            float cn[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const long long c = static_cast<long long>(ct) * kM + lane + 32 * k;
                cl[k] = c < cols ? lv[c] : kNegInf;
                cn[k] = c < cols ? static_cast<float>(nb[c]) : 0.0f;
            }
            const float finv = static_cast<float>(inv);
            mbar_wait_spin(&tfull[buf], (j / kAcc) & 1);
            fence_after();
            uint32_t v[kEpiCols];
            const uint32_t ta = tmem + (static_cast<uint32_t>(32 * q) << 16) + buf * kM + c0;
            ld32(ta, v);
            ld32(ta + 32, v + 32);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            fence_before();
            mbar_arrive(&tempty[buf]);
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
#pragma unroll
            for (int c = 0; c < kEpiCols; ++c) stage[row * kStageLd + c0 + c] = __uint_as_float(v[c]);
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
            constexpr int kRows = kM / kEpiWarps;  // 16 rows per warp
#pragma unroll 2
            for (int i = 0; i < kRows; ++i) {
                const int r = ew * kRows + i;
                const long long gr = static_cast<long long>(at) * kM + r;
                if (gr >= rows) break;  // uniform across the warp
                const float nx = static_cast<float>(na[gr]);
                double x[4], mx = kNegInf;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float c = dense_cost(kind, stage[r * kStageLd + lane + 32 * k], nx, cn[k]);
                    x[k] = cl[k] == kNegInf ? kNegInf : cl[k] - static_cast<double>(c * finv);
                    mx = fmax(mx, x[k]);
                }
                mx = warp_max(mx);
                float s = 0.0f;
                if (mx != kNegInf) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) s += __expf(static_cast<float>(x[k] - mx));
                }
                s = warp_sum(s);
                if (lane == 0) {
                    PM[gr * ntb + ct] = mx;
                    PS[gr * ntb + ct] = static_cast<double>(s);
                }
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kAcc * kM) : "memory");
    }
}

// per row: (max, sum) of its column-tile partials, in tile order
__global__ void lse_merge_kernel(const double* __restrict__ PM, const double* __restrict__ PS, long long rows, int nt,
                                 const int* __restrict__ done, double* __restrict__ M, double* __restrict__ S) {
    if (done && *done) return;
    const long long r = blockIdx.x * 256LL + threadIdx.x;
    if (r >= rows) return;
    const double* pm = PM + r * nt;
    const double* ps = PS + r * nt;
    double mx = kNegInf;
    for (int t = 0; t < nt; ++t) mx = fmax(mx, pm[t]);
    double s = 0.0;
    if (mx != kNegInf)
        for (int t = 0; t < nt; ++t)
            if (pm[t] != kNegInf) s += ps[t] * exp(pm[t] - mx);
    M[r] = mx;
    S[r] = s;
}

__global__ void sqnorm_kernel(const double* __restrict__ X, long long N, int d, double* __restrict__ out) {
    const long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < N) {
        double s = 0.0;
        for (int k = 0; k < d; ++k) s = xadd(s, xmul(X[i * d + k], X[i * d + k]));
        out[i] = s;
    }
}

}  // namespace

// Operands of the recomputed dense kernel: the union's points packed into
// 128-row tf32 hi/lo tiles (sources, then targets) and their fp64 |x|^2.
void dense_tc_prepare(Op& op) {
    Ctx& ctx = *op.ctx;
    cudaStream_t s = ctx.stream;
    const long long n = static_cast<long long>(op.n), m = static_cast<long long>(op.m);
    const int d = static_cast<int>(op.d), KB = static_cast<int>(ceil_div(d, 32));
    if (op.cost == 2) throw Status(2, "dense recompute: the cosine-derived cost keeps the stored operator");
    op.dtc_nta = static_cast<int>(ceil_div(n, kM));
    op.dtc_ntb = static_cast<int>(ceil_div(m, kM));
    std::vector<PackTile> tiles;
    for (long long r0 = 0; r0 < n; r0 += kM)
        tiles.push_back({static_cast<uint32_t>(r0), static_cast<uint32_t>(std::min<long long>(kM, n - r0)), ~0u});
    for (long long r0 = 0; r0 < m; r0 += kM)
        tiles.push_back({static_cast<uint32_t>(n + r0), static_cast<uint32_t>(std::min<long long>(kM, m - r0)), ~0u});
    op.dtc_tiles.resize(tiles.size() * KB * kKBlock);
    DevBuf<PackTile> dt;
    dt.upload(tiles.data(), tiles.size(), s);
    tcb_pack_kernel<double><<<dim3(static_cast<unsigned>(tiles.size()), KB), 256, 0, s>>>(
        op.X.get(), d, d, nullptr, dt.get(), KB, nullptr, op.dtc_tiles.get());
    op.dtc_norm.resize(static_cast<size_t>(n + m));
    sqnorm_kernel<<<ceil_div(n + m, 256), 256, 0, s>>>(op.X.get(), n + m, d, op.dtc_norm.get());
    op.dtc_pm.resize(static_cast<size_t>(std::max(n * op.dtc_ntb, m * op.dtc_nta)));
    op.dtc_ps.resize(op.dtc_pm.size());
    LAUNCH_OK("dense recompute operands");
    ctx.sync();
    op.dense_tc = true;
    op.nnz = static_cast<unsigned long long>(n * m);
}

// One half-iteration's (max, sum) per output: rows (transposed = false:
// M[i], S[i] over targets j with log v = log t) or columns (transposed: over
// sources with log v = log s).
void dense_tc_lse(Op& op, bool transposed, const double* lv, const int* done, double* M, double* S) {
    Ctx& ctx = *op.ctx;
    static std::atomic<bool> attr[64];
    if (ctx.device >= 64 || !attr[ctx.device]) {
        CUDA_OK(cudaFuncSetAttribute(dense_lse_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        if (ctx.device < 64) attr[ctx.device] = true;
    }
    const int KB = static_cast<int>(ceil_div(op.d, 32));
    const size_t tb = static_cast<size_t>(KB) * kKBlock;
    const unsigned char* P = op.dtc_tiles.get();
    const unsigned char* Q = P + static_cast<size_t>(op.dtc_nta) * tb;
    const long long n = static_cast<long long>(op.n), m = static_cast<long long>(op.m);
    const int nta = transposed ? op.dtc_ntb : op.dtc_nta, ntb = transposed ? op.dtc_nta : op.dtc_ntb;
    const long long rows = transposed ? m : n, cols = transposed ? n : m;
    const double* na = op.dtc_norm.get() + (transposed ? n : 0);
    const double* nb = op.dtc_norm.get() + (transposed ? 0 : n);
    const int grid = std::min(nta * ntb, ctx.num_sms);
    dense_lse_tc_kernel<<<grid, kThreads, kSmem, ctx.stream>>>(transposed ? Q : P, transposed ? P : Q, KB, nta, ntb,
                                                               rows, cols, na, nb, op.cost, 1.0 / op.lambda, lv, done,
                                                               op.dtc_pm.get(), op.dtc_ps.get());
    lse_merge_kernel<<<ceil_div(rows, 256), 256, 0, ctx.stream>>>(op.dtc_pm.get(), op.dtc_ps.get(), rows, ntb, done, M,
                                                                  S);
}

}  // namespace lcnb
