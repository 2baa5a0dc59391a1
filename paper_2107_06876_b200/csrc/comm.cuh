// Collective transport of the sharded solve. The sharded LCN iteration needs
// exactly one collective per half-iteration -- an all-gather of each rank's
// packed [low-rank partial | shift | error | flags | exported scalings]
// (sinkhorn.cu, lcn_iteration_shard) -- plus one all-gather of the owned
// result slices at the end, so the transport is just all-gather.
//   NcclComm      one process (or thread) per GPU, NCCL over NVLink / NVSwitch
//   LoopbackComm  ranks as host threads of one process sharing a device: the
//                 all-gather is host barrier + device copies. Kernels never
//                 wait on one another (every rank synchronises its own stream
//                 before the barrier), so several ranks can share one GPU for
//                 testing the multi-rank CUDA path (B200_PROFILING.md: no
//                 inter-rank spinning kernels on one device).
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <memory>
#include <mutex>
#include <vector>

namespace lcnb {

struct Comm {
    int rank = 0, world = 1;
    virtual ~Comm() = default;
    // recv holds world * bytes: rank r's send at offset r * bytes
    virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
    virtual const char* kind() const = 0;
};

std::shared_ptr<Comm> make_nccl_comm(int world, int rank, const unsigned char* id128);

struct LoopbackGroup {
    explicit LoopbackGroup(int w) : world(w), sends(w, nullptr) {}
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long generation = 0;
    bool aborted = false;
    std::vector<const void*> sends;
    void barrier();  // throws after abort()
    void abort();
};

std::shared_ptr<Comm> make_loopback_comm(std::shared_ptr<LoopbackGroup> g, int rank);

}  // namespace lcnb
