// Tensor-core (tcgen05) assignment filter for the k-means of the LSH / landmark
// build: the fp32 filter of kmeans.cu on the 5th-generation tensor cores.
//
// Scores v(c) = |c_f|^2 - 2 x.c_f for 128 points (one CTA) against every
// centroid, 64 centroids per tile, with the dot products in 3xTF32:
//   x.c ~ x_hi.c_hi + x_hi.c_lo + x_lo.c_hi   (hi = fp32 with the low 13
//   mantissa bits cleared, lo = fp32 remainder)
// accumulated in fp32 in tensor memory. Per point the best and second-best
// score are kept; a point whose gap exceeds twice the rigorous error bound
// (tf32 truncation of the lo parts, the dropped lo.lo term, fp32 accumulation,
// fp32 rounding of c and |c_f|^2, and the fp64 fold of the reference) gets the
// best centroid; every other point goes to the exact fp64 scan, so the result
// is bit-identical to kmeans.cpp:67-85.
//
// CTA (320 threads, 1 per SM), clusters of 2 CTAs (LCN_TC_CLUSTER; 4 measured
// 9 % slower: the stage ring advances at the pace of the cluster's slowest CTA):
//   warp 0  producer: 1-D bulk copies (TMA) of pre-swizzled centroid tiles
//           (128 centroids; a stage holds 32 features of their hi + lo
//           halves, 32 KB, six stages); each CTA of the cluster loads its
//           share of every stage and multicasts it to the cluster, so L2
//           serves each stage once per cluster
//   warp 1  owns the TMEM allocation; the converged warp runs the issue loop
//           and one elected lane issues tcgen05.mma.kind::tf32 (A = points
//           from TMEM, B = centroids from shared memory via UMMA descriptors
//           = base descriptor + compile-time offsets, D = fp32 accumulators
//           in TMEM, four buffers) and tcgen05.commit: to the local
//           accumulator barrier, and multicast to every CTA's stage barrier
//   warps 2-9 epilogue: two warps per TMEM lane quadrant, thread = (point,
//           half of the 64 columns of a tile); tcgen05.ld of 32 accumulators,
//           four interleaved branch-free top-2 trackers, merged per row at
//           the end
// Measured (2M points x 4096 centroids, d = 128): 7.96 ms, tensor pipe 73 %
// active (64-centroid tiles with clusters of 4: 10.7 ms / 53 %).
// TMEM columns: [0,128) x_hi, [128,256) x_lo, [256,512) two 128-column D buffers.
#include <cstdint>

#include "async.cuh"
#include "common.cuh"
#include "ctx.cuh"
#include "kmeans_tc.cuh"

namespace lcnb {
namespace {

constexpr int kTM = 128;        // points per CTA (UMMA_M, TMEM lanes)
constexpr int kTN = 128;        // centroids per tile (UMMA_N)
constexpr int kTD = 128;        // padded feature count (tf32 columns)
#ifndef LCN_TC_KSTAGE
#define LCN_TC_KSTAGE 32
#endif
constexpr int kTK = LCN_TC_KSTAGE;  // features per ring stage (a tile is kTD / kTK stages)
constexpr int kTKS = kTD / kTK;
constexpr int kTHalf = kTN * kTK * 4;   // bytes of one stage half (hi or lo): 32 KB
constexpr int kTStage = 2 * kTHalf;     // hi + lo
constexpr int kTStages = (3 * 64) / kTK;  // 192 KB of ring
#ifndef LCN_TC_CLUSTER
#define LCN_TC_CLUSTER 2
#endif
constexpr int kTCluster = LCN_TC_CLUSTER;  // CTAs sharing each centroid stage (multicast)
constexpr int kTAcc = 2;                // accumulator buffers in TMEM (columns 256..511)
constexpr int kTSlice = kTStage / kTCluster;
constexpr int kTEpi = 8;              // epilogue warps: two per TMEM lane quadrant
constexpr int kTThreads = 64 + 32 * kTEpi;

// element (r, k) of a swizzled stage half (k < kTK): K-major, 128-byte
// swizzle atoms of 8 rows x 32 tf32; K blocks of 32 features stacked (kTN
// rows each)
__host__ __device__ __forceinline__ uint32_t tile_offset(int r, int k) {
    const int kb = k >> 5, j = k & 31, chunk = j >> 2, w = j & 3;
    return static_cast<uint32_t>(kb * (kTN * 128) + r * 128 + ((chunk ^ (r & 7)) << 4) + w * 4);
}

__device__ __forceinline__ float tf32_hi(float x) {
    return __uint_as_float(__float_as_uint(x) & 0xffffe000u);
}

// Centroid tiles: hi and lo halves in the swizzled layout, |c_f|^2 (fp32,
// +inf for padding), and max_c max(|c|^2, |c_f|^2).
__global__ void __launch_bounds__(128) tc_prep_kernel(const double* __restrict__ C, int k, int d, int ntile,
                                                       unsigned char* __restrict__ tiles, float* __restrict__ ncf,
                                                       unsigned long long* __restrict__ cmax,
                                                       const uint32_t* __restrict__ perm) {
    __shared__ double r1[4], r2[4];
    const int c = blockIdx.x;  // centroid slot (padded to ntile * kTN); perm: slot -> centroid
    const int t = c / kTN, r = c % kTN;
    double s1 = 0.0, s2 = 0.0;
    for (int kk = threadIdx.x; kk < kTD; kk += 128) {
        // stage t * kTKS + kk / kTK holds features [kh kTK, (kh + 1) kTK) of tile t
        unsigned char* hi = tiles + (static_cast<size_t>(t) * kTKS + kk / kTK) * kTStage;
        unsigned char* lo = hi + kTHalf;
        const long long cc = perm && c < k ? static_cast<long long>(perm[c]) : c;
        const double v = (c < k && kk < d) ? C[cc * d + kk] : 0.0;
        const float f = static_cast<float>(v);
        const float h = tf32_hi(f);
        *reinterpret_cast<float*>(hi + tile_offset(r, kk % kTK)) = h;
        *reinterpret_cast<float*>(lo + tile_offset(r, kk % kTK)) = f - h;  // exact
        s1 += static_cast<double>(f) * static_cast<double>(f);
        s2 += v * v;
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if ((threadIdx.x & 31) == 0) { r1[threadIdx.x >> 5] = s1; r2[threadIdx.x >> 5] = s2; }
    __syncthreads();
    if (threadIdx.x == 0) {
        s1 = r1[0] + r1[1] + r1[2] + r1[3];
        s2 = r2[0] + r2[1] + r2[2] + r2[3];
        ncf[c] = c < k ? static_cast<float>(s1) : kPosInf;
        if (c < k) atomicMax(cmax, static_cast<unsigned long long>(__double_as_longlong(fmax(s1, s2))));
    }
}

// ---- tcgen05 / TMEM primitives (inline PTX, sm_100a) -----------------------
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B
// apart (SBO), version 1 (sm_100), base offset 0 (atoms 1024-byte aligned)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    uint64_t desc = 0;
    desc |= static_cast<uint64_t>((saddr >> 4) & 0x3fffu);          // start address
    desc |= static_cast<uint64_t>(1u) << 16;                         // LBO (unused for K-major swizzle)
    desc |= static_cast<uint64_t>(1024u >> 4) << 32;                 // SBO
    desc |= static_cast<uint64_t>(1u) << 46;                         // descriptor version (sm_100)
    desc |= static_cast<uint64_t>(2u) << 61;                         // SWIZZLE_128B
    return desc;
}

// instruction descriptor: D f32, A/B tf32, both K-major, N = kTN, M = kTM
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(kTN >> 3) << 17) |
                            (static_cast<uint32_t>(kTM >> 4) << 24);

__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(kIdesc), "r"(acc)
        : "memory");
}

// whole-warp (converged) issue: one elected lane executes the tcgen05 op, so
// ptxas needs no per-instruction election loop
__device__ __forceinline__ void tc_mma_tf32_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(kIdesc), "r"(acc)
        : "memory");
}
// the three 3xTF32 products of one K step under one election:
// x_hi.c_hi (accumulate unless first), x_hi.c_lo, x_lo.c_hi
__device__ __forceinline__ void tc_mma3_tf32_elect(uint32_t d_tmem, uint32_t a_hi, uint32_t a_lo, uint64_t b_hi,
                                                   uint64_t b_lo, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, q, e;\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "setp.eq.b32 q, %5, %5;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %6, q;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %6, q;\n\t}" ::"r"(d_tmem),
        "r"(a_hi), "r"(a_lo), "l"(b_hi), "l"(b_lo), "r"(acc), "r"(kIdesc)
        : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_commit_multicast_elect(uint64_t* bar, uint16_t cta_mask) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            smem_u32(bar)),
        "h"(cta_mask)
        : "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// arrive (once) on the barrier at this offset in every CTA of cta_mask when
// this thread's prior tcgen05 operations complete
__device__ __forceinline__ void tc_commit_multicast(uint64_t* bar, uint16_t cta_mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(cta_mask)
        : "memory");
}

__device__ __forceinline__ void tc_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
}

__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(taddr) : "memory");
}

__device__ __forceinline__ void tc_ld64(uint32_t taddr, uint32_t (&r)[64]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63]) : "r"(taddr) : "memory");
}

}  // namespace

// Work counter (bench.py's distance roofline): point x tile products this
// filter evaluated, summed over launches (tile skipping and the bound-failing
// row lists make it data dependent). One atomic per CTA.
__device__ unsigned long long g_tc_point_tiles = 0;

__global__ void __cluster_dims__(kTCluster, 1, 1) __launch_bounds__(kTThreads, 1) assign_filter_tc_kernel(
    const float* __restrict__ X, long long N, int d, const unsigned char* __restrict__ tiles,
    const float* __restrict__ ncf, int ntile, const unsigned long long* __restrict__ cmax,
    uint32_t* __restrict__ out, uint32_t* __restrict__ amb, unsigned* __restrict__ namb,
    float* __restrict__ dbg, int hh_only, const uint32_t* __restrict__ rows, float* __restrict__ ub,
    float* __restrict__ lb, const int* __restrict__ tl_off, const int* __restrict__ tl, float* __restrict__ lbt,
    const uint32_t* __restrict__ perm) {
    // all shared memory is dynamic (no static __shared__): the stage ring must
    // sit on 1024-byte swizzle-atom boundaries of the shared window
    extern __shared__ __align__(1024) unsigned char dyn_raw[];
    const uint32_t raw = smem_u32(dyn_raw);
    unsigned char* ring = dyn_raw + ((1024u - (raw & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + kTStages * kTStage);
    uint64_t* full = bars;
    uint64_t* empty = bars + kTStages;
    uint64_t* tfull = bars + 2 * kTStages;
    uint64_t* tempty = tfull + kTAcc;
    uint32_t& tmem_slot = *reinterpret_cast<uint32_t*>(tempty + kTAcc);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long p0 = static_cast<long long>(blockIdx.x) * kTM;

    if (warp == 1) {  // TMEM: all 512 columns (one CTA per SM)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    const uint32_t crank = cluster_ctarank();
    const uint16_t cmask = static_cast<uint16_t>((1u << kTCluster) - 1u);
    if (tid == 0) {
        for (int s = 0; s < kTStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTCluster);  // every CTA of the cluster releases the stage
        }
        for (int b = 0; b < kTAcc; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 32 * kTEpi);
        }
        fence_mbar_init();
    }
    // epilogue threads: own point row -> TMEM lane (hi, lo), |x|^2; the two
    // warps of a lane quadrant split the features (prologue) and each tile's
    // 64 accumulator columns (epilogue)
    double xn = 0.0;
    const int eq = warp - 2;                // epilogue warp 0..kTEpi-1
    const int lane_base = 32 * (warp & 3);  // TMEM lanes this warp may access
    const int half = eq >= 0 ? eq / 4 : 0;  // which half of the columns
    const int row = lane_base + lane;       // point within the CTA tile
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // every CTA's barriers exist before any multicast lands
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    // tile list (Lloyd's tile skipping): this cluster evaluates the centroid
    // tiles tl[tl_off[c] .. tl_off[c + 1]) in order, both CTAs the same ones
    // (their stages are multicast); else every tile
    int nt = ntile;
    const int* tlist = nullptr;
    if (tl_off) {
        const int cl = static_cast<int>(blockIdx.x) / kTCluster;
        tlist = tl + tl_off[cl];
        nt = tl_off[cl + 1] - tl_off[cl];
    }
    if (tid == 0 && p0 < N)
        atomicAdd(&g_tc_point_tiles, static_cast<unsigned long long>(min(static_cast<long long>(kTM), N - p0)) *
                                         static_cast<unsigned long long>(nt));
    if (eq >= 0) {
        const long long p = p0 + row;
        // rows: the points of this call are rows[0 .. N) (lloyd's bound-failing list)
        const float* xr = X + (rows && p < N ? static_cast<long long>(rows[p]) : p) * d;
        for (int c0 = half * (kTD / 2); c0 < (half + 1) * (kTD / 2); c0 += 32) {
            uint32_t vh[32], vl[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int kk = c0 + j;
                const float x = (p < N && kk < d) ? xr[kk] : 0.0f;
                const float h = tf32_hi(x);
                vh[j] = __float_as_uint(h);
                vl[j] = __float_as_uint(x - h);
                xn += static_cast<double>(x) * static_cast<double>(x);
            }
            tc_st32(tmem + (static_cast<uint32_t>(lane_base) << 16) + c0, vh);
            tc_st32(tmem + (static_cast<uint32_t>(lane_base) << 16) + kTD + c0, vl);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        // the two halves' |x|^2 -> both (the per-tile bounds need it early)
        double* xnx = reinterpret_cast<double*>(reinterpret_cast<float*>(tempty + kTAcc + 2) + 3 * kTM + 2) + kTM;
        xnx[half * kTM + row] = xn;
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kTEpi) : "memory");
        xn += xnx[(1 - half) * kTM + row];
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp == 0) {
        // ---------------- producer ----------------
        // this CTA loads slice crank of each stage and multicasts it to the
        // cluster; its own barrier expects the whole stage (all slices)
        if (lane == 0) {
            for (int g = 0; g < nt * kTKS; ++g) {  // stage g: listed tile g / kTKS, features (g % kTKS) kTK ..
                const int s = g % kTStages;
                const int tile = tlist ? tlist[g / kTKS] : g / kTKS;
                if (g >= kTStages) mbar_wait(&empty[s], ((g / kTStages) - 1) & 1);
                mbar_arrive_expect_tx(&full[s], kTStage);
                bulk_g2s_multicast(ring + s * kTStage + crank * kTSlice,
                                   tiles + (static_cast<size_t>(tile) * kTKS + g % kTKS) * kTStage + crank * kTSlice,
                                   kTSlice, &full[s], cmask);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        // The whole warp runs the issue loop (converged); one elected lane
        // issues each tcgen05 op. The descriptors of a stage are its base
        // descriptor plus compile-time 16-byte-unit offsets (the start
        // address field sits in the low bits and never carries inside the
        // ring).
        int g = 0;  // ring stage counter
        for (int t = 0; t < nt; ++t) {
            const int b = t % kTAcc;
            if (t >= kTAcc) mbar_wait(&tempty[b], ((t / kTAcc) - 1) & 1);
            const uint32_t dt = tmem + 256 + b * kTN;
            for (int kh = 0; kh < kTKS; ++kh, ++g) {
                const int s = g % kTStages;
                mbar_wait(&full[s], (g / kTStages) & 1);
                tc_fence_after();
                const uint64_t dh0 = umma_desc_sw128(smem_u32(ring + s * kTStage));
                const uint64_t dl0 = dh0 + (kTHalf >> 4);
                const uint32_t ah = tmem + kh * kTK, al = tmem + kTD + kh * kTK;
                if (hh_only == 1) {
#pragma unroll
                    for (int ks = 0; ks < kTK / 8; ++ks) {
                        const uint64_t off = ((ks >> 2) * (kTN * 128) + (ks & 3) * 32) >> 4;
                        tc_mma_tf32_elect(dt, ah + ks * 8, dh0 + off, (kh | ks) ? 1u : 0u);
                    }
                } else {
#pragma unroll
                    for (int ks = 0; ks < kTK / 8; ++ks) {
                        const uint64_t off = ((ks >> 2) * (kTN * 128) + (ks & 3) * 32) >> 4;
                        // x_hi . c_hi, x_hi . c_lo, x_lo . c_hi
                        tc_mma3_tf32_elect(dt, ah + ks * 8, al + ks * 8, dh0 + off, dl0 + off, (kh | ks) ? 1u : 0u);
                    }
                }
                tc_commit_multicast_elect(&empty[s], cmask);  // stage consumed (in every CTA's view)
            }
            tc_commit_elect(&tfull[b]);  // accumulator ready
        }
        __syncwarp();
    } else {
        // ---------------- epilogue: thread = (point, column half) --------
        // Four independent running top-2 trackers per thread (columns j = u
        // mod 4 of its half of each tile) keep the dependency chains short:
        //   v2 = min(v2, max(v1, v)), v1 = min(v1, v), index on v < v1
        // (the sequential update for finite scores). They merge into the best
        // score (first index on ties) and the second-smallest score of the
        // whole multiset, then the two halves of a row merge the same way.
        constexpr int kCh = 4, kHC = kTN / 2;  // columns per thread and tile
        float v1[kCh], v2[kCh];
        int i1[kCh];
#pragma unroll
        for (int c = 0; c < kCh; ++c) v1[c] = v2[c] = kPosInf, i1[c] = 0;
        // per-tile bound terms: |x|^2 and the filter's error E (as below)
        const double u24 = 5.9604644775390625e-08;  // 2^-24
        const double Cb = sqrt(__longlong_as_double(*cmax)) * (1.0 + 1e-12);
        const double xb2 = sqrt(xn) * (1.0 + 1e-12);
        const double dot_rel2 = 2.0 * (3.0 * 9.5367431640625e-07 + 56.0 * 1.1920928955078125e-07);
        const double Eb = 1.05 * ((dot_rel2 + 4.0 * u24) * xb2 * Cb + 4.0 * u24 * Cb * Cb + u24 * u24 * Cb * Cb) +
                          1e-12 * (xb2 + Cb) * (xb2 + Cb);
        const long long pq = p0 + row;
        const long long qq = rows && pq < N ? static_cast<long long>(rows[pq]) : pq;
        for (int t = 0; t < nt; ++t) {
            const int b = t % kTAcc;
            const int tile = tlist ? tlist[t] : t;
            float tmin = kPosInf;  // this half's minimum score in the tile
            const uint32_t tcol = tmem + (static_cast<uint32_t>(lane_base) << 16) + 256 + b * kTN + half * kHC;
#pragma unroll 1
            for (int ch = 0; ch < kHC / 32; ++ch) {
                // |c|^2 of these 32 columns while the accumulator is in flight
                float4 nc[8];
                const float4* nc4 = reinterpret_cast<const float4*>(ncf + tile * kTN + half * kHC + ch * 32);
#pragma unroll
                for (int j4 = 0; j4 < 8; ++j4) nc[j4] = __ldg(nc4 + j4);
                if (ch == 0) {
                    mbar_wait(&tfull[b], (t / kTAcc) & 1);
                    tc_fence_after();
                }
                uint32_t r[32];
                tc_ld32(tcol + ch * 32, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (ch == kHC / 32 - 1) {
                    tc_fence_before();
                    mbar_arrive(&tempty[b]);
                }
                if (dbg && blockIdx.x == 0 && t == 0)  // test hook: raw accumulators of centroids 0..63
                    for (int j = 0; j < 32; ++j) {
                        const int col = half * kHC + ch * 32 + j;
                        if (col < 64) dbg[row * 64 + col] = __uint_as_float(r[j]);
                    }
                const int base = tile * kTN + half * kHC + ch * 32;
#pragma unroll
                for (int j4 = 0; j4 < 8; ++j4) {
                    const float ncj[4] = {nc[j4].x, nc[j4].y, nc[j4].z, nc[j4].w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int j = 4 * j4 + u;
                        const float v = fmaf(-2.0f, __uint_as_float(r[j]), ncj[u]);
                        const bool lt1 = v < v1[u];
                        v2[u] = fminf(v2[u], fmaxf(v1[u], v));
                        i1[u] = lt1 ? base + j : i1[u];
                        v1[u] = fminf(v1[u], v);
                        tmin = fminf(tmin, v);
                    }
                }
            }
            if (lbt && pq < N) {
                // a lower bound on the true distance to every centroid of the
                // tile (this half): D >= |x|^2 + v - E, folds within 1e-12
                const double lo = (xn + static_cast<double>(tmin) - Eb) * (1.0 - 1e-12);
                lbt[(qq * ntile + tile) * 2 + half] = __double2float_rd(__dsqrt_rd(fmax(lo, 0.0)));
            }
        }
        // merge the trackers: best value, lowest index among equal bests,
        // second smallest of the multiset
        float bv = v1[0], sv = v2[0];
        int bi = i1[0];
#pragma unroll
        for (int c = 1; c < kCh; ++c) {
            sv = fminf(fminf(sv, v2[c]), fmaxf(bv, v1[c]));
            if (v1[c] < bv || (v1[c] == bv && i1[c] < bi)) bi = i1[c];
            bv = fminf(bv, v1[c]);
        }
        // merge the two halves of each row through shared memory (named
        // barrier 1: the epilogue warps only)
        float* xb = reinterpret_cast<float*>(tempty + kTAcc + 2);  // 128 x {bv, sv, bi} + xn
        if (half == 1) {
            xb[3 * row] = bv;
            xb[3 * row + 1] = sv;
            xb[3 * row + 2] = __int_as_float(bi);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kTEpi) : "memory");
        if (half == 0) {
        {
            const float ov = xb[3 * row], os = xb[3 * row + 1];
            const int oi = __float_as_int(xb[3 * row + 2]);
            sv = fminf(fminf(sv, os), fmaxf(bv, ov));
            if (ov < bv || (ov == bv && oi < bi)) bi = oi;
            bv = fminf(bv, ov);
        }
        const float v1m = bv, v2m = sv;
        const int i1m = bi;
        const long long p = p0 + row;
        if (p < N) {
            const double u = 5.9604644775390625e-08;  // 2^-24
            const double C = sqrt(__longlong_as_double(*cmax)) * (1.0 + 1e-12);
            const double x = sqrt(xn) * (1.0 + 1e-12);
            // 2 x.c term: 3xTF32 (lo truncation 2 x 2^-20, dropped lo.lo 2^-20) and
            // fp32 tensor-core accumulation (<= 56 roundings of 2^-23), doubled
            const double dot_rel = 2.0 * (3.0 * 9.5367431640625e-07 + 56.0 * 1.1920928955078125e-07);
            const double E = 1.05 * ((dot_rel + 4.0 * u) * x * C + 4.0 * u * C * C + u * u * C * C) +
                             1e-12 * (x + C) * (x + C);
            const double gap = static_cast<double>(v2m) - static_cast<double>(v1m);
            const long long q = rows ? static_cast<long long>(rows[p]) : p;
            if (gap > 2.0 * E) {
                out[q] = perm ? perm[i1m] : static_cast<uint32_t>(i1m);  // slot -> centroid
                if (ub) {
                    // Lloyd's bounds on true distances (lloyd_device): every
                    // fold D(x, c) lies within E of |x|^2 + v(c), the fold
                    // within 1e-12 (relative) of the true square
                    const double hi = (xn + static_cast<double>(v1m) + E) * (1.0 + 1e-12);
                    const double lo = (xn + static_cast<double>(v2m) - E) * (1.0 - 1e-12);
                    ub[q] = __double2float_ru(__dsqrt_ru(fmax(hi, 0.0)));
                    lb[q] = __double2float_rd(__dsqrt_rd(fmax(lo, 0.0)));
                }
            } else {
                amb[atomicAdd(namb, 1u)] = static_cast<uint32_t>(q);
            }
        }
        }  // half 0
    }
    tc_fence_before();
    __syncthreads();
    // no CTA leaves while a peer may still multicast into it or arrive on its
    // barriers
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// Host side: prepare the centroid tiles and launch. Returns false when the
// shape is not handled (d > kTD).
bool assign_filter_tc(Ctx& ctx, const float* X, long long N, int d, const double* C, int k, uint32_t* out,
                      uint32_t* amb, unsigned* namb, float* dbg_acc, int hh_only, const uint32_t* rows, float* ub,
                      float* lb, const int* tl_off, const int* tl, float* lbt, const uint32_t* perm) {
    if (d > kTD || d < 1) return false;
    cudaStream_t s = ctx.stream;
    const int ntile = static_cast<int>(ceil_div(k, kTN));
    DevBuf<unsigned char> tiles(static_cast<size_t>(ntile) * kTKS * kTStage);
    DevBuf<float> ncf(static_cast<size_t>(ntile) * kTN);
    DevBuf<unsigned long long> cmax(1);
    cmax.zero(s);
    tc_prep_kernel<<<ntile * kTN, 128, 0, s>>>(C, k, d, ntile, tiles.get(), ncf.get(), cmax.get(), perm);
    // ring + barriers (2 kTStages + 2 kTAcc) + TMEM slot + row-merge buffer
    const int smem = kTStages * kTStage + 1024 + (2 * kTStages + 2 * kTAcc + 2) * 8 + (3 * kTM + 2) * 4 + 3 * kTM * 8 + 64;
    static std::atomic<bool> attr[64];  // set once per device; concurrent build jobs may race here (benign, idempotent)
    if (ctx.device >= 64 || !attr[ctx.device]) {
        CUDA_OK(cudaFuncSetAttribute(assign_filter_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        if (ctx.device < 64) attr[ctx.device] = true;
    }
    // grid: whole clusters (CTAs past N only help stream the centroid stages)
    const long long grid = ceil_div(ceil_div(N, kTM), kTCluster) * kTCluster;
    assign_filter_tc_kernel<<<static_cast<unsigned>(grid), kTThreads, smem, s>>>(
        X, N, d, tiles.get(), ncf.get(), ntile, cmax.get(), out, amb, namb, dbg_acc, hh_only, rows, ub, lb, tl_off, tl,
        lbt, perm);
    LAUNCH_OK("assign_filter_tc_kernel");
    return true;
}

unsigned long long tc_point_tiles(bool reset) {
    unsigned long long v = 0;
    CUDA_OK(cudaMemcpyFromSymbol(&v, g_tc_point_tiles, sizeof(v)));
    if (reset) {
        const unsigned long long z = 0;
        CUDA_OK(cudaMemcpyToSymbol(g_tc_point_tiles, &z, sizeof(z)));
    }
    return v;
}

int assign_tc_tile_count(int k) { return static_cast<int>(ceil_div(k, kTN)); }
constexpr int kTcClusterPoints = kTM * kTCluster;
static_assert(kTcClusterPoints == 256, "lloyd's tile lists assume 256 points per cluster");

}  // namespace lcnb
