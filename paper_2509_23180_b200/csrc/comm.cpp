// Rank-to-rank transport of the subdomain-sharded solve (the
// interface lines of every operator application, <= 32 KB per arm, and the
// command words).  Two implementations behind one interface:
//   * NCCL point-to-point (ncclSend / ncclRecv on the caller's stream) over
//     NVLink / NVSwitch between one process per GPU; libnccl.so.2 is opened
//     with dlopen when a communicator is created (the copy torch already
//     loaded when there is one), so the library itself has no NCCL link
//     dependency;
//   * an in-process loopback for testing the multi-rank protocol on one GPU:
//     ranks are host threads of one process, a send stages the bytes in a
//     device buffer and a recv copies them out on the receiver's stream.  No
//     kernel ever waits on another rank's kernel (the hand-off is host-side),
//     so it is safe to run every rank on the same device.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string.h>

#include "fd_internal.h"

namespace fd {

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

static NcclApi &nccl() {
    static std::mutex mu;
    static NcclApi api;
    static bool tried = false;
    std::lock_guard<std::mutex> g(mu);
    if (!tried) {
        tried = true;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the copy already in the process
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
            api.init_rank = (decltype(api.init_rank))dlsym(h, "ncclCommInitRank");
            api.destroy = (decltype(api.destroy))dlsym(h, "ncclCommDestroy");
            api.send = (decltype(api.send))dlsym(h, "ncclSend");
            api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
            api.group_start = (decltype(api.group_start))dlsym(h, "ncclGroupStart");
            api.group_end = (decltype(api.group_end))dlsym(h, "ncclGroupEnd");
            api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
        }
    }
    if (!api.send || !api.recv || !api.init_rank)
        FD_FAIL(FD_ERR_UNSUPPORTED, "NCCL (libnccl.so.2) is not available in this process");
    return api;
}

static void nccl_check(ncclResult_t r, const char *what) {
    if (r != ncclSuccess) {
        std::string m = std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "NCCL error");
        FD_FAIL(FD_ERR_CUDA, m);
    }
}

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    ~NcclTransport() override {
        if (comm) nccl().destroy(comm);
    }
    void send(const void *buf, size_t bytes, int peer, cudaStream_t s) override {
        nccl_check(nccl().send(buf, bytes, ncclInt8, peer, comm, s), "ncclSend");
    }
    void recv(void *buf, size_t bytes, int peer, cudaStream_t s) override {
        nccl_check(nccl().recv(buf, bytes, ncclInt8, peer, comm, s), "ncclRecv");
    }
    void group_start() override { nccl_check(nccl().group_start(), "ncclGroupStart"); }
    void group_end() override { nccl_check(nccl().group_end(), "ncclGroupEnd"); }
};

// in-process ranks: one message queue per (src, dst)
struct LoopHub {
    struct Msg {
        void *dev;
        size_t bytes;
        cudaEvent_t ready;
    };
    std::mutex mu;
    std::condition_variable cv;
    std::map<std::pair<int, int>, std::deque<Msg>> q;
};

struct LoopTransport : Transport {
    std::shared_ptr<LoopHub> hub;
    void send(const void *buf, size_t bytes, int peer, cudaStream_t s) override {
        LoopHub::Msg m{};
        m.bytes = bytes;
        FD_CUDA(cudaMallocAsync(&m.dev, std::max<size_t>(bytes, 8), s));
        FD_CUDA(cudaMemcpyAsync(m.dev, buf, bytes, cudaMemcpyDeviceToDevice, s));
        FD_CUDA(cudaEventCreateWithFlags(&m.ready, cudaEventDisableTiming));
        FD_CUDA(cudaEventRecord(m.ready, s));
        std::lock_guard<std::mutex> g(hub->mu);
        hub->q[{rank, peer}].push_back(m);
        hub->cv.notify_all();
    }
    void recv(void *buf, size_t bytes, int peer, cudaStream_t s) override {
        LoopHub::Msg m{};
        {
            std::unique_lock<std::mutex> g(hub->mu);
            auto &dq = hub->q[{peer, rank}];
            hub->cv.wait(g, [&] { return !dq.empty(); });
            m = dq.front();
            dq.pop_front();
        }
        if (m.bytes != bytes) FD_FAIL(FD_ERR_VALIDATION, "loopback: message size mismatch");
        FD_CUDA(cudaStreamWaitEvent(s, m.ready, 0));
        FD_CUDA(cudaMemcpyAsync(buf, m.dev, bytes, cudaMemcpyDeviceToDevice, s));
        FD_CUDA(cudaFreeAsync(m.dev, s));
        FD_CUDA(cudaEventDestroy(m.ready));
    }
};

}  // namespace fd

using namespace fd;

extern "C" {

int fd_comm_unique_id(char *id) {
    try {
        if (!id) FD_FAIL(FD_ERR_VALIDATION, "null id buffer");
        ncclUniqueId u;
        nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
        memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    } catch (const Error &e) {
        set_error(e.msg);
        return e.code;
    }
    return FD_OK;
}

int fd_comm_init(fd_comm *out, int nranks, int rank, const char *id, int device) {
    try {
        if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) FD_FAIL(FD_ERR_VALIDATION, "bad communicator arguments");
        *out = nullptr;
        FD_CUDA(cudaSetDevice(device));
        auto t = std::make_unique<NcclTransport>();
        ncclUniqueId u;
        memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
        nccl_check(nccl().init_rank(&t->comm, nranks, u, rank), "ncclCommInitRank");
        t->nranks = nranks;
        t->rank = rank;
        *out = new fd_comm_s{std::move(t), device};
    } catch (const Error &e) {
        set_error(e.msg);
        return e.code;
    }
    return FD_OK;
}

int fd_comm_init_loopback(fd_comm *outs, int nranks, int device) {
    try {
        if (!outs || nranks < 1) FD_FAIL(FD_ERR_VALIDATION, "bad loopback arguments");
        auto hub = std::make_shared<LoopHub>();
        for (int r = 0; r < nranks; ++r) {
            auto t = std::make_unique<LoopTransport>();
            t->hub = hub;
            t->nranks = nranks;
            t->rank = r;
            outs[r] = new fd_comm_s{std::move(t), device};
        }
    } catch (const Error &e) {
        set_error(e.msg);
        return e.code;
    }
    return FD_OK;
}

int fd_comm_rank(fd_comm c, int *rank, int *nranks) {
    if (!c) return FD_ERR_VALIDATION;
    if (rank) *rank = c->t->rank;
    if (nranks) *nranks = c->t->nranks;
    return FD_OK;
}

int fd_comm_destroy(fd_comm c) {
    delete c;
    return FD_OK;
}

}  // extern "C"
