// Dense anchor with the kernel recomputed every half-iteration (configs[2]:
// "exp(-C/lambda) is recomputed on the fly per iteration as a tensor-core GEMM
// fused with log-sum-exp"): no n x m storage. The reference streams a stored
// log K (operator.cpp:125-140 rows, :178-192 columns; build_cost / build_kernel
// geometry.cpp:113-144); here each half-iteration is
//   out_i = LSE_j( -c(x_i, y_j) / lambda + log v_j )
// with x.y from tcgen05 3xTF32 MMAs (tc_block.cuh operands and pipeline),
// c(x, y) from the dot and exact fp64 norms, and the log-sum-exp fused into
// the epilogue: per (row, 64-column half tile) a partial (max, sum), merged
// per row in order by a second kernel (deterministic).
//
// CTA (persistent, one per SM): warp 0 bulk-copies the row tile's and the
// column tile's k-blocks into a 3-stage ring, warp 1 issues
// tcgen05.mma.kind::tf32 (hi.hi + hi.lo + lo.hi) into one of two TMEM
// accumulators, 8 epilogue warps tcgen05.ld their row's 64 dots and reduce
// them in registers.
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

// Items are (row tile, pair of column tiles): one UMMA of M = 128, N = 256
// per k-step, so a stage of 96 KB (the row tile's hi / lo k-block and both
// column tiles') carries 2 x 128 x 256 x 32 x 3 flop -- 64 flop per byte
// against 48 for 128-wide tiles; the operand feed, not the tensor pipe, bounds
// this kernel (profiles/dense_tc_r02.json). The epilogue reads the
// accumulators straight from TMEM (no staging tile).
constexpr int kN2 = 2 * kM;                         // UMMA N
constexpr int kDStage = kKBlock + 2 * kKBlock;      // A k-block + two B k-blocks: 96 KB
constexpr int kDS = 2;
constexpr int kDSmem = kDS * kDStage + 2 * (kN2 * 8 + kN2 * 4) + 1024 + 128;
constexpr uint32_t kIdesc2 = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(kN2 >> 3) << 17) |
                             (static_cast<uint32_t>(kM >> 4) << 24);

__device__ __forceinline__ void mma2_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(kIdesc2), "r"(acc)
        : "memory");
}

// Epilogue thread = (accumulator row = TMEM lane, half h of the 256 columns,
// i.e. column tile 2 cp + h): its 128 dots from four tcgen05.ld's, the
// per-column log v and |y|^2 from a shared table; online (max, sum) written
// as that column tile's partial.
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
    double* col_lv = reinterpret_cast<double*>(ring + kDS * kDStage);  // [2][kN2]
    float* col_nb = reinterpret_cast<float*>(col_lv + 2 * kN2);        // [2][kN2]
    uint64_t* bars = reinterpret_cast<uint64_t*>(col_nb + 2 * kN2);
    uint64_t* full = bars;
    uint64_t* empty = bars + kDS;
    uint64_t* tfull = bars + 2 * kDS;
    uint64_t* tempty = tfull + kAcc;
    uint32_t& tmem_slot = *reinterpret_cast<uint32_t*>(tempty + kAcc);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ntp = (ntb + 1) / 2;  // column tile pairs
    const int nitems = nta * ntp;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                     "n"(kAcc * kN2)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int s = 0; s < kDS; ++s) {
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
                const int cp = it % ntp;
                const unsigned char* a = A + static_cast<size_t>(it / ntp) * tile_bytes;
                const unsigned char* b0 = B + static_cast<size_t>(2 * cp) * tile_bytes;
                // an odd last pair reads tile 0 as its second tile (masked in the epilogue)
                const unsigned char* b1 = 2 * cp + 1 < ntb ? b0 + tile_bytes : B;
                for (int kb = 0; kb < KB; ++kb, ++g) {
                    const uint32_t s = g % kDS;
                    if (g >= kDS) mbar_wait_spin(&empty[s], ((g / kDS) - 1) & 1);
                    unsigned char* st = ring + s * kDStage;
                    const size_t ko = static_cast<size_t>(kb) * kKBlock;
                    mbar_arrive_expect_tx(&full[s], kDStage);
                    bulk_g2s(st, a + ko, kKBlock, &full[s]);                          // A hi | A lo
                    bulk_g2s(st + kKBlock, b0 + ko, kHalf, &full[s]);                 // B0 hi
                    bulk_g2s(st + kKBlock + kHalf, b1 + ko, kHalf, &full[s]);         // B1 hi
                    bulk_g2s(st + 2 * kKBlock, b0 + ko + kHalf, kHalf, &full[s]);     // B0 lo
                    bulk_g2s(st + 2 * kKBlock + kHalf, b1 + ko + kHalf, kHalf, &full[s]);  // B1 lo
                }
            }
        }
    } else if (warp == 1) {
        uint32_t g = 0, j = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++j) {
            const uint32_t buf = j % kAcc;
            if (j >= kAcc) mbar_wait_spin(&tempty[buf], ((j / kAcc) - 1) & 1);
            fence_after();
            const uint32_t dt = tmem + buf * kN2;
            for (int kb = 0; kb < KB; ++kb, ++g) {
                const uint32_t s = g % kDS;
                mbar_wait_spin(&full[s], (g / kDS) & 1);
                fence_after();
                const uint32_t base = smem_u32(ring + s * kDStage);
                const uint64_t ah = desc_sw128(base), al = desc_sw128(base + kHalf);
                const uint64_t bh = desc_sw128(base + kKBlock), bl = desc_sw128(base + 2 * kKBlock);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint64_t off = static_cast<uint64_t>(ks * 32) >> 4;
                    mma2_elect(dt, ah + off, bh + off, (kb | ks) ? 1u : 0u);
                    mma2_elect(dt, ah + off, bl + off, 1u);
                    mma2_elect(dt, al + off, bh + off, 1u);
                }
                commit_elect(&empty[s]);
            }
            commit_elect(&tfull[buf]);
        }
        __syncwarp();
    } else {
        const int q = warp & 3;
        const int row = 32 * q + lane;
        const int h = (warp - 2) >> 2;  // column tile of the pair
        const int et = tid - 64;        // 0..255
        const float finv = static_cast<float>(inv);
        uint32_t j = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++j) {
            const uint32_t buf = j % kAcc;
            const int at = it / ntp, cp = it % ntp;
            const int cb = j & 1;  // column-table buffer (the previous item may still read the other)
            {
                const long long c = static_cast<long long>(cp) * kN2 + et;
                col_lv[cb * kN2 + et] = c < cols ? lv[c] : kNegInf;
                col_nb[cb * kN2 + et] = c < cols ? static_cast<float>(nb[c]) : 0.0f;
            }
            const long long gr = static_cast<long long>(at) * kM + row;
            const float nx = gr < rows ? static_cast<float>(na[gr]) : 0.0f;
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");  // column table visible
            mbar_wait_spin(&tfull[buf], (j / kAcc) & 1);
            fence_after();
            const uint32_t ta = tmem + (static_cast<uint32_t>(32 * q) << 16) + buf * kN2 + h * kM;
            const double* tl = col_lv + cb * kN2 + h * kM;
            const float* tn = col_nb + cb * kN2 + h * kM;
            double mx = kNegInf;
            float sum = 0.0f;
#pragma unroll
            for (int part = 0; part < 4; ++part) {
                uint32_t v[32];
                ld32(ta + 32 * part, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (part == 3) {
                    fence_before();
                    mbar_arrive(&tempty[buf]);
                }
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const double l = tl[32 * part + c];
                    if (l == kNegInf) continue;
                    const double x =
                        l - static_cast<double>(dense_cost(kind, __uint_as_float(v[c]), nx, tn[32 * part + c]) * finv);
                    if (x > mx) {
                        sum = sum * __expf(static_cast<float>(mx - x)) + 1.0f;
                        mx = x;
                    } else {
                        sum += __expf(static_cast<float>(x - mx));
                    }
                }
            }
            const int ct = 2 * cp + h;
            if (gr < rows && ct < ntb) {
                PM[gr * ntb + ct] = mx;
                PS[gr * ntb + ct] = static_cast<double>(sum);
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kAcc * kN2) : "memory");
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
        CUDA_OK(cudaFuncSetAttribute(dense_lse_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDSmem));
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
    const int grid = std::min(nta * ((ntb + 1) / 2), ctx.num_sms);
    dense_lse_tc_kernel<<<grid, kThreads, kDSmem, ctx.stream>>>(transposed ? Q : P, transposed ? P : Q, KB, nta, ntb,
                                                               rows, cols, na, nb, op.cost, 1.0 / op.lambda, lv, done,
                                                               op.dtc_pm.get(), op.dtc_ps.get());
    lse_merge_kernel<<<ceil_div(rows, 256), 256, 0, ctx.stream>>>(op.dtc_pm.get(), op.dtc_ps.get(), rows, ntb, done,
                                                                  M, S);
}

}  // namespace lcnb
