// comm.cuh -- transports of the multi-GPU path: the collectives the
// distributed step needs, enqueued on a CUDA stream.
//   NcclTransport   one rank per process (or per thread), a library-owned NCCL communicator built
//                   from a 128-byte ncclUniqueId; libnccl is dlopen'ed at fmm_create_dist (the
//                   copy the process already loaded -- torch's -- if any), so libfmm has no link-time
//                   NCCL dependency.  Point-to-point messages are grouped ncclSend/ncclRecv over
//                   NVLink/NVSwitch; failures map to FMM_ERR_NCCL.
//   LocalTransport  K ranks inside ONE process, one host thread per rank (fmm_group): the host
//                   threads meet at barriers to swap device pointers and events, every copy is a
//                   cudaMemcpyAsync ordered by cudaStreamWaitEvent on the peer's event -- nothing on
//                   the device ever waits for another rank's kernel, so the ranks may share a GPU
//                   (single-GPU parity tests) or sit on several GPUs of one process.
#pragma once
#include <condition_variable>
#include <mutex>
#include <vector>

#include "common.cuh"

struct CommMsg {
    int peer;
    void* ptr;
    size_t bytes;
};

struct Transport {
    int nranks = 1, rank = 0;
    std::string err;
    virtual ~Transport() {}
    // in place, element-wise over all ranks: op 0 sum, 1 min, 2 max (device fp64 [count])
    virtual fmm_status allreduce_f64(double* buf, size_t count, int op, cudaStream_t s) = 0;
    // recv (device [nranks][bytes]) <- every rank's send (device [bytes])
    virtual fmm_status allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
    // one group of point-to-point messages; the k-th send to peer p matches p's k-th receive from
    // this rank (sizes must agree); zero-byte messages are skipped
    virtual fmm_status sendrecv(const std::vector<CommMsg>& sends, const std::vector<CommMsg>& recvs,
                                cudaStream_t s) = 0;
    // abort: every rank blocked in (or later entering) a collective returns an error
    virtual void abort() {}
};

// K ranks of one process (include/fmm.h fmm_group)
struct LocalGroup {
    int nranks = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    bool aborted = false;
    int nctx = 0;   // contexts attached
    // per-rank slots of the collective in progress
    struct Slot {
        const void* send = nullptr;
        void* recv = nullptr;
        double* red = nullptr;
        std::vector<CommMsg> sends;
        cudaEvent_t ready = nullptr, copied = nullptr;
        int device = 0;
    };
    std::vector<Slot> slots;
    // host barrier; false if the group was aborted
    bool barrier();
};

fmm_status transport_nccl(int nranks, int rank, const void* unique_id, int device, Transport** out, std::string& err);
fmm_status transport_local(LocalGroup* g, int rank, int device, Transport** out, std::string& err);
fmm_status nccl_unique_id(void* out128, std::string& err);
