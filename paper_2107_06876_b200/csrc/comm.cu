// Collective transports of the sharded solve (comm.cuh).
#include <nccl.h>

#include <string>

#include "comm.cuh"
#include "common.cuh"

namespace lcnb {

namespace {

struct NcclComm final : Comm {
    ncclComm_t c = nullptr;
    ~NcclComm() override {
        if (c) ncclCommDestroy(c);
    }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        const ncclResult_t r = ncclAllGather(send, recv, bytes, ncclUint8, c, s);
        if (r != ncclSuccess) throw Status(100, std::string("ncclAllGather: ") + ncclGetErrorString(r));
    }
    const char* kind() const override { return "nccl"; }
};

struct LoopbackComm final : Comm {
    std::shared_ptr<LoopbackGroup> g;
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        CUDA_OK(cudaStreamSynchronize(s));  // own send data complete
        g->sends[rank] = send;
        g->barrier();                       // every rank's send data complete
        for (int r = 0; r < world; ++r)
            CUDA_OK(cudaMemcpyAsync(static_cast<char*>(recv) + static_cast<size_t>(r) * bytes, g->sends[r], bytes,
                                    cudaMemcpyDefault, s));
        CUDA_OK(cudaStreamSynchronize(s));
        g->barrier();                       // nobody reuses a send buffer before all copies are done
    }
    const char* kind() const override { return "loopback"; }
};

}  // namespace

void LoopbackGroup::barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw Status(6, "loopback communicator: another rank failed");
    const unsigned long long gen = generation;
    if (++arrived == world) {
        arrived = 0;
        ++generation;
        cv.notify_all();
        return;
    }
    cv.wait(lk, [&] { return generation != gen || aborted; });
    if (generation == gen) throw Status(6, "loopback communicator: another rank failed");
}

void LoopbackGroup::abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
}

std::shared_ptr<Comm> make_nccl_comm(int world, int rank, const unsigned char* id128) {
    auto c = std::make_shared<NcclComm>();
    ncclUniqueId id;
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    memcpy(&id, id128, 128);
    const ncclResult_t r = ncclCommInitRank(&c->c, world, id, rank);
    if (r != ncclSuccess) throw Status(100, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    c->rank = rank;
    c->world = world;
    return c;
}

std::shared_ptr<Comm> make_loopback_comm(std::shared_ptr<LoopbackGroup> g, int rank) {
    auto c = std::make_shared<LoopbackComm>();
    c->g = std::move(g);
    c->rank = rank;
    c->world = c->g->world;
    return c;
}

}  // namespace lcnb
