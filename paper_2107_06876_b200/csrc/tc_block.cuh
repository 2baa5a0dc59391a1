// Tensor-core (tcgen05) block contractions of the operator build:
// dot products of 128-row tiles of a "row" operand against 128-row tiles of a
// "column" operand, in the FP32-accurate 3xTF32 split
//   x.y ~ x_hi.y_hi + x_hi.y_lo + x_lo.y_hi   (hi = fp32 with the low 13
//   mantissa bits cleared, lo = the fp32 remainder, read as tf32)
// accumulated in fp32 in tensor memory, each 128 x 128 result handed to an
// epilogue functor (the cost transform + exp / log K / delta of the caller).
// Used for the within-bucket distance blocks of K^sp (sparse_kernel.cpp:51-80),
// the point x landmark blocks U and V (nystrom.cpp:53-64) and the delta SDDMM
// U_b W_b (sparse_kernel.cpp:82-117 via NystromFactors::entry,
// nystrom.cpp:127-132).
//
// Operands are packed once into the UMMA K-major 128-byte-swizzle layout by
// tcb_pack_kernel: tile t, k-block kb (32 tf32 columns) = [hi 16 KB][lo 16 KB],
// 128 rows of 128 bytes with 16-byte chunks XOR-swizzled by (row & 7).
//
// CTA (320 threads, persistent, 1 per SM):
//   warp 0  producer: per item and k-block one 1-D bulk copy (TMA engine) of
//           the row tile's k-block and one of the column tile's into a
//           3-stage ring (64 KB per stage), completion on an mbarrier
//   warp 1  TMEM owner + MMA issuer: one elected lane issues
//           tcgen05.mma.cta_group::1.kind::tf32 (A and B from shared memory
//           by UMMA descriptors, M = N = 128, K = 8) into one of two 128-column
//           fp32 accumulators and tcgen05.commit's the stage / accumulator
//   warps 2-9 epilogue: thread = (accumulator row = TMEM lane, half of the
//           128 columns); tcgen05.ld of its 64 dot products into a shared
//           staging tile (the accumulator is released at once), then each
//           warp takes 16 rows with its lanes along the columns, so every
//           per-column load and every output store of the functor is one
//           coalesced 128-byte access per warp.
#pragma once
#include <cstdint>

#include "async.cuh"
#include "common.cuh"
#include "ctx.cuh"

namespace lcnb {
namespace tcb {

constexpr int kM = 128;               // rows per tile (both operands), UMMA M and N
constexpr int kHalf = kM * 128;       // one k-block half (hi or lo): 128 rows x 32 tf32 = 16 KB
constexpr int kKBlock = 2 * kHalf;    // hi + lo
constexpr int kStage = 2 * kKBlock;   // row-tile k-block + column-tile k-block: 64 KB
constexpr int kStages = 2;
constexpr int kAcc = 2;               // accumulator buffers (128 TMEM columns each)
constexpr int kEpiWarps = 8;           // two per TMEM lane quadrant, 64 columns each
constexpr int kEpiCols = kM / 2;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kStageLd = kM + 1;      // fp32 staging row stride (conflict-free both ways)
constexpr int kStageBytes = kM * kStageLd * 4;
constexpr int kSmem = kStages * kStage + kStageBytes + 1024 + 128;
// instruction descriptor: D f32 (bits 4-5 = 1), A tf32 (7-9 = 2), B tf32
// (10-12 = 2), both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(kM >> 3) << 17) |
                            (static_cast<uint32_t>(kM >> 4) << 24);

// byte offset of element (r, k) (k < 32) inside one k-block half
__host__ __device__ __forceinline__ uint32_t half_offset(int r, int k) {
    return static_cast<uint32_t>(r * 128 + ((((k >> 2) ^ (r & 7))) << 4) + (k & 3) * 4);
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups
// 1024 B apart (SBO), descriptor version 1 (sm_100)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t desc = 0;
    desc |= static_cast<uint64_t>((saddr >> 4) & 0x3fffu);
    desc |= static_cast<uint64_t>(1u) << 16;
    desc |= static_cast<uint64_t>(1024u >> 4) << 32;
    desc |= static_cast<uint64_t>(1u) << 46;
    desc |= static_cast<uint64_t>(2u) << 61;
    return desc;
}

// converged-warp issue: one elected lane executes the MMA (A and B in smem)
__device__ __forceinline__ void mma_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(kIdesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
}

// One packed tile: rows idx[off + r] (r < count; idx == nullptr: rows off + r)
// of a row-major matrix; rows past count are zero. center != ~0u subtracts
// row `center` of the caller's center matrix (fp64) from every row first.
struct PackTile {
    uint32_t off, count, center;
};

// grid (tiles, k-blocks), 256 threads: one k-block of one tile, hi and lo.
// Thread e -> (row e / 32, column e % 32): a warp reads 32 consecutive
// features of a row and writes them into one swizzled 128-byte row.
template <typename T>
__global__ void __launch_bounds__(256) tcb_pack_kernel(const T* __restrict__ X, long long ld, int d,
                                                        const uint32_t* __restrict__ idx,
                                                        const PackTile* __restrict__ tiles, int KB,
                                                        const double* __restrict__ centers,
                                                        unsigned char* __restrict__ out) {
    const PackTile tl = tiles[blockIdx.x];
    const int kb = blockIdx.y;
    unsigned char* hi = out + (static_cast<size_t>(blockIdx.x) * KB + kb) * kKBlock;
    unsigned char* lo = hi + kHalf;
    for (int e = threadIdx.x; e < kM * 32; e += 256) {
        const int r = e >> 5, k = e & 31, kk = kb * 32 + k;
        float h = 0.0f, l = 0.0f;
        if (static_cast<uint32_t>(r) < tl.count && kk < d) {
            const long long row = idx ? static_cast<long long>(idx[tl.off + r]) : static_cast<long long>(tl.off) + r;
            double v = static_cast<double>(X[row * ld + kk]);
            if (tl.center != ~0u) v -= centers[static_cast<long long>(tl.center) * d + kk];
            h = tf32_hi(static_cast<float>(v));
            l = static_cast<float>(v - static_cast<double>(h));
        }
        const uint32_t o = half_offset(r, k);
        *reinterpret_cast<float*>(hi + o) = h;
        *reinterpret_cast<float*>(lo + o) = l;
    }
}

// items: int4 {row tile, column tile, tag, tag2}. The functor provides
//   Item item(int4)                   per-item context (bucket offsets, ...)
//   Row row(Item, r)                  per-row context (r = tile row 0..127)
//   Pre pre(Item, Row, c)             the entry's loads (c = tile column)
//   void apply(Item, Row, Pre, c, d)  compute and store one entry (d = dot)
//   void finish()                     after the last item (all threads)
template <class Epi>
__global__ void __launch_bounds__(kThreads, 1) tcb_kernel(const unsigned char* __restrict__ A,
                                                          const unsigned char* __restrict__ B, int KB,
                                                          const int4* __restrict__ items, int nitems, Epi epi,
                                                          unsigned long long* __restrict__ trace) {
    extern __shared__ __align__(1024) unsigned char dyn_raw[];
    const uint32_t raw = smem_u32(dyn_raw);
    unsigned char* ring = dyn_raw + ((1024u - (raw & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + kStages * kStage);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* tfull = bars + 2 * kStages;
    uint64_t* tempty = tfull + kAcc;
    uint32_t& tmem_slot = *reinterpret_cast<uint32_t*>(tempty + kAcc);
    float* stage = reinterpret_cast<float*>(ring + kStages * kStage + 128);  // kM x kStageLd dots
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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
                const int4 item = items[it];
                const unsigned char* a = A + static_cast<size_t>(item.x) * tile_bytes;
                const unsigned char* b = B + static_cast<size_t>(item.y) * tile_bytes;
                for (int kb = 0; kb < KB; ++kb, ++g) {
                    const uint32_t s = g % kStages;
                    if (g >= kStages) mbar_wait_spin(&empty[s], ((g / kStages) - 1) & 1);
                    if (trace && blockIdx.x == 0 && kb == 0 && it < 16 * gridDim.x) trace[(it / gridDim.x) * 8 + 0] = gtimer();
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
            if (trace && lane == 0 && blockIdx.x == 0 && it < 16 * gridDim.x) trace[(it / gridDim.x) * 8 + 5] = gtimer();
            const uint32_t dt = tmem + buf * kM;
            for (int kb = 0; kb < KB; ++kb, ++g) {
                const uint32_t s = g % kStages;
                mbar_wait_spin(&full[s], (g / kStages) & 1);
                fence_after();
                if (trace && lane == 0 && blockIdx.x == 0 && it < 16 * gridDim.x)
                    trace[(it / gridDim.x) * 8 + (kb == 0 ? 1 : 2)] = gtimer();
                const uint32_t base = smem_u32(ring + s * kStage);
                const uint64_t ah = desc_sw128(base), al = desc_sw128(base + kHalf);
                const uint64_t bh = desc_sw128(base + kKBlock), bl = desc_sw128(base + kKBlock + kHalf);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint64_t off = static_cast<uint64_t>(ks * 32) >> 4;  // 32 bytes = 8 tf32 along K
                    mma_ss_elect(dt, ah + off, bh + off, (kb | ks) ? 1u : 0u);  // hi . hi
                    mma_ss_elect(dt, ah + off, bl + off, 1u);                   // hi . lo
                    mma_ss_elect(dt, al + off, bh + off, 1u);                   // lo . hi
                }
                commit_elect(&empty[s]);
            }
            commit_elect(&tfull[buf]);
        }
        __syncwarp();
    } else {
        const int q = warp & 3;  // TMEM lane quadrant this warp may access
        const int row = 32 * q + lane;
        const int c0 = ((warp - 2) >> 2) * kEpiCols;  // this warp's half of the columns
        uint32_t j = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++j) {
            const uint32_t buf = j % kAcc;
            const int4 item = items[it];
            mbar_wait_spin(&tfull[buf], (j / kAcc) & 1);
            fence_after();
            if (trace && tid == 64 && blockIdx.x == 0 && it < 16 * gridDim.x) trace[(it / gridDim.x) * 8 + 3] = gtimer();
            uint32_t v[kEpiCols];
            const uint32_t ta = tmem + (static_cast<uint32_t>(32 * q) << 16) + buf * kM + c0;
            ld32(ta, v);
            ld32(ta + 32, v + 32);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            fence_before();
            mbar_arrive(&tempty[buf]);
            // named barrier 1 (epilogue warps): the previous item's rows are
            // processed before the staging tile is overwritten
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
#pragma unroll
            for (int c = 0; c < kEpiCols; ++c) stage[row * kStageLd + c0 + c] = __uint_as_float(v[c]);
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
            // rows in batches of kRB, loads of a whole batch issued before any
            // use (the per-row and per-entry inputs are HBM-latency loads)
            const int ew = warp - 2;
            const auto I = epi.item(item);
            constexpr int kRB = Epi::kRB, kCK = kM / 32;
#pragma unroll 1
            for (int rb = 0; rb < kM / kEpiWarps; rb += kRB) {
                typename Epi::Row R[kRB];
                typename Epi::Pre P[kRB][kCK];
#pragma unroll
                for (int i = 0; i < kRB; ++i) R[i] = epi.row(I, ew * (kM / kEpiWarps) + rb + i);
#pragma unroll
                for (int i = 0; i < kRB; ++i)
#pragma unroll
                    for (int k = 0; k < kCK; ++k) P[i][k] = epi.pre(I, R[i], lane + 32 * k);
#pragma unroll
                for (int i = 0; i < kRB; ++i) {
                    const int r = ew * (kM / kEpiWarps) + rb + i;
#pragma unroll
                    for (int k = 0; k < kCK; ++k)
                        epi.apply(I, R[i], P[i][k], lane + 32 * k, stage[r * kStageLd + lane + 32 * k]);
                }
            }
            if (trace && tid == 64 && blockIdx.x == 0 && it < 16 * gridDim.x) trace[(it / gridDim.x) * 8 + 4] = gtimer();
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kAcc * kM) : "memory");
    }
    epi.finish();
}

}  // namespace tcb
}  // namespace lcnb
