// Context, device buffers and the internal operator/result structures.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "comm.cuh"
#include "common.cuh"

namespace lcnb {

// Stream of the API call in progress on this thread (set by the C-ABI guard;
// 0 = legacy default stream outside any call).
inline cudaStream_t& alloc_stream() {
    thread_local cudaStream_t s = nullptr;
    return s;
}

// Owning device allocation, stream-ordered: cudaMallocAsync / cudaFreeAsync
// on the calling API's stream from the device's default pool (kept resident,
// see lcn_ctx_create). A synchronous cudaFree stalls the device at every
// temporary; the pool hands memory back without synchronising. Destroy entry
// points synchronise the device before freeing (objects may be released from
// any thread / stream).
template <typename T>
class DevBuf {
  public:
    DevBuf() = default;
    explicit DevBuf(size_t n) { resize(n); }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p_ = o.p_; n_ = o.n_; o.p_ = nullptr; o.n_ = 0; }
        return *this;
    }
    void resize(size_t n) {
        if (n == n_) return;
        release();
        if (n) CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), alloc_stream()));
        n_ = n;
    }
    void release() {
        if (p_) cudaFreeAsync(p_, alloc_stream());
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    size_t bytes() const { return n_ * sizeof(T); }
    void upload(const T* h, size_t n, cudaStream_t s) {
        resize(n);
        if (n) CUDA_OK(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void download(T* h, size_t n, cudaStream_t s) const {
        if (n) CUDA_OK(cudaMemcpyAsync(h, p_, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    void zero(cudaStream_t s) {
        if (n_) CUDA_OK(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
    }

  private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

// Row stride of a bucket block: m_b padded to a multiple of 4 entries.
__host__ __device__ __forceinline__ unsigned long long row_stride(unsigned long long mb) { return (mb + 3ull) & ~3ull; }

struct Ctx {
    int device = 0;
    int store_fp64 = 0;
    int exact_build = 0;  // LCN_EXACT_BUILD: fp64 CUDA-core build tiles even in fp32 storage
    int dense_recompute = 0;  // LCN_DENSE_RECOMPUTE: dense operators recompute exp(-C/lambda) per iteration
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    int profile = 0;
    std::string last_error;
    // k-means assignment filter statistics (points filtered / sent to the exact scan)
    long long filter_points = 0, filter_ambiguous = 0;
    // sharded solve: the communicator over the ranks that
    // share one problem (comm.cuh; null = single-GPU solve). LCN operators
    // built on a context with a communicator are bucket-sharded (op.cuh
    // ShardState).
    std::shared_ptr<Comm> comm;
    // cuBLAS handle (lazy; plain library GEMMs: W = V A^-T and its residual)
    void* cublas = nullptr;
    int rank() const { return comm ? comm->rank : 0; }
    int world() const { return comm ? comm->world : 1; }
    void activate() const { CUDA_OK(cudaSetDevice(device)); }
    void sync() const { CUDA_OK(cudaStreamSynchronize(stream)); }
};

// Points of one side, device-resident. Values are fp64 (exact promotion of
// the caller's fp64, or of fp32 for the device entry points).
struct DevPoints {
    DevBuf<double> x;  // n x d row-major
    size_t n = 0, d = 0;
};

// One LSH band in bucket-blocked form: sources and targets
// sorted stably by bucket; bucket b owns the dense n_b x m_b block at
// blk_off[b]. Rows/cols of a block are in increasing point index.
struct Band {
    size_t nb = 0;                 // bucket count (range)
    DevBuf<uint32_t> src_order;    // n: source indices grouped by bucket
    DevBuf<uint32_t> tgt_order;    // m
    DevBuf<uint32_t> src_start;    // nb+1
    DevBuf<uint32_t> tgt_start;    // nb+1
    DevBuf<unsigned long long> blk_off;  // nb+1 (entries): block b, n_b rows x row_stride(m_b)
    DevBuf<unsigned long long> blkT_off; // nb+1: transposed block b, m_b rows x row_stride(n_b) (lcn)
    DevBuf<uint32_t> src_bucket;   // n
    DevBuf<uint32_t> tgt_bucket;   // m
    DevBuf<uint32_t> src_local;    // n: position inside its bucket
    DevBuf<uint32_t> tgt_local;    // m
    DevBuf<uint32_t> src_pos;      // n (+16): position of each source in src_order
    DevBuf<uint32_t> tgt_pos;      // m (+16)
    DevBuf<uint32_t> work;         // list of buckets with a nonempty block
    size_t n_work = 0;
    unsigned long long entries = 0;       // padded block entries held in HBM
    unsigned long long entriesT = 0;      // padded transposed-block entries
    unsigned long long real_entries = 0;  // sum n_b * m_b
    std::vector<uint32_t> h_src_start, h_tgt_start;
    std::vector<unsigned long long> h_blk_off, h_blkT_off;
};

}  // namespace lcnb
