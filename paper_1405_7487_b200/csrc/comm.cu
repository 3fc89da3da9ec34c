// comm.cu -- NCCL and in-process transports of the multi-GPU path (comm.cuh).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "comm.cuh"

// ------------------------------------------------------------------------------- NCCL (dlopen)
namespace {

struct NcclApi {
    void* handle = nullptr;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclCommAbort) CommAbort = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    std::string load_error;
};

NcclApi& nccl_state() {
    static NcclApi api;
    return api;
}

const NcclApi* nccl_api() {
    NcclApi& api = nccl_state();
    static std::once_flag once;
    std::call_once(once, [&api] {
        // the copy the process already has (torch's bundled libnccl), else the system one
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            api.handle = dlopen(nm, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
            if (api.handle) break;
        }
        if (!api.handle)
            for (const char* nm : names) {
                api.handle = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
                if (api.handle) break;
            }
        if (!api.handle) {
            const char* e = dlerror();
            api.load_error = std::string("dlopen libnccl.so.2 failed: ") + (e ? e : "?");
            return;
        }
#define FMM_NCCL_SYM(field, name)                                                  \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(api.handle, name));    \
    if (!api.field) {                                                              \
        api.load_error = std::string("libnccl lacks ") + name;                     \
        api.handle = nullptr;                                                      \
        return;                                                                    \
    }
        FMM_NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
        FMM_NCCL_SYM(CommInitRank, "ncclCommInitRank");
        FMM_NCCL_SYM(CommDestroy, "ncclCommDestroy");
        FMM_NCCL_SYM(CommAbort, "ncclCommAbort");
        FMM_NCCL_SYM(AllReduce, "ncclAllReduce");
        FMM_NCCL_SYM(AllGather, "ncclAllGather");
        FMM_NCCL_SYM(Send, "ncclSend");
        FMM_NCCL_SYM(Recv, "ncclRecv");
        FMM_NCCL_SYM(GroupStart, "ncclGroupStart");
        FMM_NCCL_SYM(GroupEnd, "ncclGroupEnd");
        FMM_NCCL_SYM(GetErrorString, "ncclGetErrorString");
#undef FMM_NCCL_SYM
    });
    return api.handle ? &api : nullptr;
}

std::string nccl_load_error() {
    nccl_api();
    const std::string& e = nccl_state().load_error;
    return e.empty() ? std::string("libnccl unavailable") : e;
}

#define FMM_NCCL_TRY(expr)                                                                   \
    do {                                                                                     \
        ncclResult_t _r = (expr);                                                            \
        if (_r != ncclSuccess) {                                                             \
            err = std::string(#expr) + ": " + api->GetErrorString(_r);                       \
            return FMM_ERR_NCCL;                                                             \
        }                                                                                    \
    } while (0)

#define FMM_CU_TRY(expr)                                                                     \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess) {                                                             \
            err = std::string(#expr) + ": " + cudaGetErrorString(_e);                        \
            return FMM_ERR_CUDA;                                                             \
        }                                                                                    \
    } while (0)

struct NcclTransport : Transport {
    const NcclApi* api = nullptr;
    ncclComm_t comm = nullptr;
    ~NcclTransport() override {
        if (comm) api->CommDestroy(comm);
    }
    void abort() override {
        if (comm) {
            api->CommAbort(comm);
            comm = nullptr;
        }
    }
    fmm_status allreduce_f64(double* buf, size_t count, int op, cudaStream_t s) override {
        const ncclRedOp_t o = op == 0 ? ncclSum : op == 1 ? ncclMin : ncclMax;
        if (count) FMM_NCCL_TRY(api->AllReduce(buf, buf, count, ncclFloat64, o, comm, s));
        return FMM_OK;
    }
    fmm_status allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        if (bytes) FMM_NCCL_TRY(api->AllGather(send, recv, bytes, ncclUint8, comm, s));
        return FMM_OK;
    }
    fmm_status sendrecv(const std::vector<CommMsg>& sends, const std::vector<CommMsg>& recvs, cudaStream_t s) override {
        // messages to self are device copies (k-th send to self -> k-th receive from self)
        std::vector<const CommMsg*> self_s, self_r;
        for (const CommMsg& m : sends)
            if (m.peer == rank && m.bytes) self_s.push_back(&m);
        for (const CommMsg& m : recvs)
            if (m.peer == rank && m.bytes) self_r.push_back(&m);
        if (self_s.size() != self_r.size()) {
            err = "sendrecv: unmatched message to self";
            return FMM_ERR_ARG;
        }
        for (size_t k = 0; k < self_s.size(); ++k) {
            if (self_s[k]->bytes != self_r[k]->bytes) {
                err = "sendrecv: size mismatch (self)";
                return FMM_ERR_ARG;
            }
            FMM_CU_TRY(cudaMemcpyAsync(self_r[k]->ptr, self_s[k]->ptr, self_s[k]->bytes, cudaMemcpyDeviceToDevice, s));
        }
        FMM_NCCL_TRY(api->GroupStart());
        for (const CommMsg& m : sends)
            if (m.peer != rank && m.bytes) FMM_NCCL_TRY(api->Send(m.ptr, m.bytes, ncclUint8, m.peer, comm, s));
        for (const CommMsg& m : recvs)
            if (m.peer != rank && m.bytes) FMM_NCCL_TRY(api->Recv(m.ptr, m.bytes, ncclUint8, m.peer, comm, s));
        FMM_NCCL_TRY(api->GroupEnd());
        return FMM_OK;
    }
};

// ------------------------------------------------------------------------------- in-process
__global__ void k_reduce_ranks(const double* __restrict__ tmp, int nranks, size_t count, int op,
                               double* __restrict__ out) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        double v = tmp[i];
        for (int r = 1; r < nranks; ++r) {   // rank order: deterministic sums
            const double x = tmp[(size_t)r * count + i];
            v = op == 0 ? v + x : op == 1 ? fmin(v, x) : fmax(v, x);
        }
        out[i] = v;
    }
}

struct LocalTransport : Transport {
    LocalGroup* g = nullptr;
    int device = 0;
    cudaEvent_t ready = nullptr, copied = nullptr;
    double* tmp = nullptr;
    size_t tmp_bytes = 0;
    ~LocalTransport() override {
        if (ready) cudaEventDestroy(ready);
        if (copied) cudaEventDestroy(copied);
        if (tmp) cudaFree(tmp);
        std::lock_guard<std::mutex> lk(g->mu);
        --g->nctx;
    }
    void abort() override {
        std::lock_guard<std::mutex> lk(g->mu);
        g->aborted = true;
        g->cv.notify_all();
    }
    fmm_status sync(const char* what) {
        if (!g->barrier()) {
            err = std::string(what) + ": group aborted by another rank";
            return FMM_ERR_STATE;
        }
        return FMM_OK;
    }
    // wait for every rank's `copied` record of this collective, then the closing barrier (no rank
    // re-records its events before all waits on them are enqueued)
    fmm_status finish(cudaStream_t s, const char* what) {
        FMM_TRY(sync(what));
        for (int j = 0; j < nranks; ++j) FMM_CU_TRY(cudaStreamWaitEvent(s, g->slots[j].copied, 0));
        return sync(what);
    }
    fmm_status allreduce_f64(double* buf, size_t count, int op, cudaStream_t s) override {
        LocalGroup::Slot& me = g->slots[rank];
        FMM_CU_TRY(cudaEventRecord(ready, s));
        me.red = buf;
        me.ready = ready;
        me.copied = copied;
        FMM_TRY(sync("allreduce"));
        const size_t need = (size_t)nranks * count * 8;
        if (need > tmp_bytes) {
            if (tmp) cudaFree(tmp);
            tmp = nullptr;
            FMM_CU_TRY(cudaMalloc(&tmp, need));
            tmp_bytes = need;
        }
        for (int j = 0; j < nranks; ++j) {
            FMM_CU_TRY(cudaStreamWaitEvent(s, g->slots[j].ready, 0));
            if (count)
                FMM_CU_TRY(cudaMemcpyAsync(tmp + (size_t)j * count, g->slots[j].red, count * 8, cudaMemcpyDefault, s));
        }
        FMM_CU_TRY(cudaEventRecord(copied, s));
        FMM_TRY(finish(s, "allreduce"));
        if (count) {
            k_reduce_ranks<<<(unsigned)std::min<size_t>((count + 255) / 256, 1024), 256, 0, s>>>(tmp, nranks, count, op,
                                                                                                buf);
            FMM_CU_TRY(cudaGetLastError());
        }
        return FMM_OK;
    }
    fmm_status allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        LocalGroup::Slot& me = g->slots[rank];
        FMM_CU_TRY(cudaEventRecord(ready, s));
        me.send = send;
        me.ready = ready;
        me.copied = copied;
        FMM_TRY(sync("allgather"));
        for (int j = 0; j < nranks; ++j) {
            FMM_CU_TRY(cudaStreamWaitEvent(s, g->slots[j].ready, 0));
            if (bytes)
                FMM_CU_TRY(cudaMemcpyAsync((char*)recv + (size_t)j * bytes, g->slots[j].send, bytes, cudaMemcpyDefault, s));
        }
        FMM_CU_TRY(cudaEventRecord(copied, s));
        return finish(s, "allgather");
    }
    fmm_status sendrecv(const std::vector<CommMsg>& sends, const std::vector<CommMsg>& recvs, cudaStream_t s) override {
        LocalGroup::Slot& me = g->slots[rank];
        FMM_CU_TRY(cudaEventRecord(ready, s));
        me.sends = sends;
        me.ready = ready;
        me.copied = copied;
        FMM_TRY(sync("sendrecv"));
        std::vector<size_t> next(nranks, 0);   // per sender: messages to this rank consumed
        std::vector<bool> waited(nranks, false);
        fmm_status st = FMM_OK;
        for (const CommMsg& r : recvs) {
            if (!r.bytes) continue;
            if (r.peer < 0 || r.peer >= nranks) {
                err = "sendrecv: bad peer";
                st = FMM_ERR_ARG;
                break;
            }
            const std::vector<CommMsg>& ps = g->slots[r.peer].sends;
            size_t& k = next[r.peer];
            while (k < ps.size() && (ps[k].peer != rank || ps[k].bytes == 0)) ++k;
            if (k == ps.size() || ps[k].bytes != r.bytes) {
                err = "sendrecv: no matching send of the same size from rank " + std::to_string(r.peer);
                st = FMM_ERR_ARG;
                break;
            }
            if (!waited[r.peer]) {
                FMM_CU_TRY(cudaStreamWaitEvent(s, g->slots[r.peer].ready, 0));
                waited[r.peer] = true;
            }
            FMM_CU_TRY(cudaMemcpyAsync(r.ptr, ps[k].ptr, r.bytes, cudaMemcpyDefault, s));
            ++k;
        }
        FMM_CU_TRY(cudaEventRecord(copied, s));
        const fmm_status st2 = finish(s, "sendrecv");
        return st != FMM_OK ? st : st2;
    }
};

}  // namespace

bool LocalGroup::barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) return false;
    const uint64_t gen = generation;
    if (++arrived == nranks) {
        arrived = 0;
        ++generation;
        cv.notify_all();
        return true;
    }
    cv.wait(lk, [&] { return generation != gen || aborted; });
    return !aborted;
}

fmm_status nccl_unique_id(void* out128, std::string& err) {
    const NcclApi* api = nccl_api();
    if (!api) {
        err = nccl_load_error();
        return FMM_ERR_NCCL;
    }
    ncclUniqueId id;
    FMM_NCCL_TRY(api->GetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
    return FMM_OK;
}

fmm_status transport_nccl(int nranks, int rank, const void* unique_id, int device, Transport** out, std::string& err) {
    const NcclApi* api = nccl_api();
    if (!api) {
        err = nccl_load_error();
        return FMM_ERR_NCCL;
    }
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    DeviceGuard g(device);
    auto* t = new NcclTransport();
    t->api = api;
    t->nranks = nranks;
    t->rank = rank;
    const ncclResult_t r = api->CommInitRank(&t->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        err = std::string("ncclCommInitRank: ") + api->GetErrorString(r);
        t->comm = nullptr;
        delete t;
        return FMM_ERR_NCCL;
    }
    *out = t;
    return FMM_OK;
}

fmm_status transport_local(LocalGroup* grp, int rank, int device, Transport** out, std::string& err) {
    {
        std::lock_guard<std::mutex> lk(grp->mu);
        if (rank < 0 || rank >= grp->nranks) {
            err = "fmm_create_dist: rank outside the group";
            return FMM_ERR_ARG;
        }
        ++grp->nctx;
    }
    DeviceGuard g(device);
    auto* t = new LocalTransport();
    t->g = grp;
    t->nranks = grp->nranks;
    t->rank = rank;
    t->device = device;
    if (cudaEventCreateWithFlags(&t->ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&t->copied, cudaEventDisableTiming) != cudaSuccess) {
        err = "cudaEventCreate failed";
        delete t;
        return FMM_ERR_CUDA;
    }
    *out = t;
    return FMM_OK;
}
