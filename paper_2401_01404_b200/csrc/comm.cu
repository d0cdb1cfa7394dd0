// comm.cu — NCCL (dlopen'ed libnccl.so.2) and in-process loopback collectives.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "comm.cuh"
#include "common.cuh"

namespace nrg {

// ---------------------------------------------------------------- NCCL
namespace {
struct NcclApi {
    void* h = nullptr;
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclGetErrorString) errStr = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (!api.h) {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (!api.h) fail(100, std::string("cannot load NCCL: ") + dlerror());
#define NRG_SYM(field, sym)                                                         \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(api.h, #sym));          \
    if (!api.field) fail(100, "NCCL symbol missing: " #sym);
        NRG_SYM(getUniqueId, ncclGetUniqueId)
        NRG_SYM(commInitRank, ncclCommInitRank)
        NRG_SYM(commDestroy, ncclCommDestroy)
        NRG_SYM(allGather, ncclAllGather)
        NRG_SYM(allReduce, ncclAllReduce)
        NRG_SYM(broadcast, ncclBroadcast)
        NRG_SYM(send, ncclSend)
        NRG_SYM(recv, ncclRecv)
        NRG_SYM(groupStart, ncclGroupStart)
        NRG_SYM(groupEnd, ncclGroupEnd)
        NRG_SYM(errStr, ncclGetErrorString)
#undef NRG_SYM
    }
    return api;
}

void nccheck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(100, std::string("NCCL ") + what + ": " + nccl().errStr(r));
}

struct NcclComm final : Comm {
    ncclComm_t comm = nullptr;
    uint64_t* dscratch = nullptr;
    size_t dscratch_n = 0;
    // device staging for the host-scalar collectives, grown on demand (the routing
    // matrix of exchange_and_score is world^2 counts)
    uint64_t* scratch(size_t n) {
        if (n > dscratch_n) {
            if (dscratch) NRG_CUDA(cudaFree(dscratch));
            dscratch = nullptr;
            dscratch_n = std::max<size_t>(n, 64);
            NRG_CUDA(cudaMalloc(&dscratch, dscratch_n * 8));
        }
        return dscratch;
    }
    ~NcclComm() override {
        if (comm) nccl().commDestroy(comm);
        if (dscratch) cudaFree(dscratch);
    }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        nccheck(nccl().allGather(send, recv, bytes, ncclUint8, comm, s), "allgather");
        NRG_CUDA(cudaStreamSynchronize(s));
    }
    void allgatherv(const void* send, void* recv, const std::vector<size_t>& bytes, cudaStream_t s) override {
        std::vector<size_t> off(world, 0);
        for (int r = 1; r < world; ++r) off[r] = off[r - 1] + bytes[r - 1];
        nccheck(nccl().groupStart(), "group");
        for (int r = 0; r < world; ++r) {
            if (r == rank) continue;
            if (bytes[rank]) nccheck(nccl().send(send, bytes[rank], ncclUint8, r, comm, s), "send");
            if (bytes[r]) nccheck(nccl().recv(static_cast<char*>(recv) + off[r], bytes[r], ncclUint8, r, comm, s), "recv");
        }
        nccheck(nccl().groupEnd(), "group");
        if (bytes[rank] && static_cast<const char*>(send) != static_cast<char*>(recv) + off[rank])
            NRG_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + off[rank], send, bytes[rank], cudaMemcpyDeviceToDevice, s));
        NRG_CUDA(cudaStreamSynchronize(s));
    }
    void alltoallv(const void* send, const std::vector<size_t>& sb, const std::vector<size_t>& so, void* recv,
                   const std::vector<size_t>& rb, const std::vector<size_t>& ro, cudaStream_t s) override {
        nccheck(nccl().groupStart(), "group");
        for (int r = 0; r < world; ++r) {
            if (r == rank) continue;
            if (sb[r]) nccheck(nccl().send(static_cast<const char*>(send) + so[r], sb[r], ncclUint8, r, comm, s), "send");
            if (rb[r]) nccheck(nccl().recv(static_cast<char*>(recv) + ro[r], rb[r], ncclUint8, r, comm, s), "recv");
        }
        nccheck(nccl().groupEnd(), "group");
        if (sb[rank])
            NRG_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + ro[rank], static_cast<const char*>(send) + so[rank],
                                     sb[rank], cudaMemcpyDeviceToDevice, s));
        NRG_CUDA(cudaStreamSynchronize(s));
    }
    void allreduce_u64(uint64_t* v, int n, bool mx, cudaStream_t s) override {
        uint64_t* d = scratch((size_t)n);
        NRG_CUDA(cudaMemcpyAsync(d, v, (size_t)n * 8, cudaMemcpyHostToDevice, s));
        nccheck(nccl().allReduce(d, d, n, ncclUint64, mx ? ncclMax : ncclSum, comm, s), "allreduce");
        NRG_CUDA(cudaMemcpyAsync(v, d, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
        NRG_CUDA(cudaStreamSynchronize(s));
    }
    void bcast_f64(double* v, int n, cudaStream_t s) override {
        uint64_t* d = scratch((size_t)n);
        NRG_CUDA(cudaMemcpyAsync(d, v, (size_t)n * 8, cudaMemcpyHostToDevice, s));
        nccheck(nccl().broadcast(d, d, n, ncclFloat64, 0, comm, s), "broadcast");
        NRG_CUDA(cudaMemcpyAsync(v, d, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
        NRG_CUDA(cudaStreamSynchronize(s));
    }
};
}  // namespace

int nccl_unique_id(uint8_t id[128]) {
    ncclUniqueId u;
    nccheck(nccl().getUniqueId(&u), "unique id");
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, 128);
    return 0;
}

Comm* make_nccl_comm(const uint8_t id[128], int rank, int world, int device) {
    NRG_CUDA(cudaSetDevice(device));
    auto* c = new NcclComm();
    c->rank = rank;
    c->world = world;
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    try {
        nccheck(nccl().commInitRank(&c->comm, world, u, rank), "comm init");
        c->scratch((size_t)world * world);
    } catch (...) {
        delete c;
        throw;
    }
    return c;
}

// ---------------------------------------------------------------- host transport
namespace {
// collectives through caller-supplied callbacks on host buffers: device data staged
// through pinned memory (grown on demand) around each call
struct HostComm final : Comm {
    nrg_host_transport t{};
    void* pin_send = nullptr;
    void* pin_recv = nullptr;
    size_t cap_send = 0, cap_recv = 0;
    ~HostComm() override {
        if (pin_send) cudaFreeHost(pin_send);
        if (pin_recv) cudaFreeHost(pin_recv);
    }
    static void* grow(void*& p, size_t& cap, size_t n) {
        if (n > cap) {
            if (p) NRG_CUDA(cudaFreeHost(p));
            p = nullptr;
            cap = std::max<size_t>(n, 1 << 16);
            NRG_CUDA(cudaMallocHost(&p, cap));
        }
        return p;
    }
    static void ok(int rc, const char* what) {
        if (rc) fail(100, std::string("host transport: ") + what + " failed (" + std::to_string(rc) + ")");
    }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        allgatherv(send, recv, std::vector<size_t>(world, bytes), s);
    }
    void allgatherv(const void* send, void* recv, const std::vector<size_t>& bytes, cudaStream_t s) override {
        size_t tot = 0;
        for (size_t b : bytes) tot += b;
        void* hs = grow(pin_send, cap_send, bytes[rank]);
        void* hr = grow(pin_recv, cap_recv, tot);
        if (bytes[rank]) NRG_CUDA(cudaMemcpyAsync(hs, send, bytes[rank], cudaMemcpyDeviceToHost, s));
        NRG_CUDA(cudaStreamSynchronize(s));
        std::vector<uint64_t> rb(bytes.begin(), bytes.end());
        ok(t.allgatherv(t.user, hs, bytes[rank], hr, rb.data()), "allgatherv");
        if (tot) NRG_CUDA(cudaMemcpyAsync(recv, hr, tot, cudaMemcpyHostToDevice, s));
        NRG_CUDA(cudaStreamSynchronize(s));
    }
    void alltoallv(const void* send, const std::vector<size_t>& sb, const std::vector<size_t>& so, void* recv,
                   const std::vector<size_t>& rb, const std::vector<size_t>& ro, cudaStream_t s) override {
        size_t st = 0, rt = 0;
        for (int r = 0; r < world; ++r) {
            st = std::max(st, so[r] + sb[r]);
            rt = std::max(rt, ro[r] + rb[r]);
        }
        void* hs = grow(pin_send, cap_send, st);
        void* hr = grow(pin_recv, cap_recv, rt);
        if (st) NRG_CUDA(cudaMemcpyAsync(hs, send, st, cudaMemcpyDeviceToHost, s));
        NRG_CUDA(cudaStreamSynchronize(s));
        std::vector<uint64_t> a(sb.begin(), sb.end()), b(so.begin(), so.end()), c(rb.begin(), rb.end()),
            d(ro.begin(), ro.end());
        ok(t.alltoallv(t.user, hs, a.data(), b.data(), hr, c.data(), d.data()), "alltoallv");
        if (rt) NRG_CUDA(cudaMemcpyAsync(recv, hr, rt, cudaMemcpyHostToDevice, s));
        NRG_CUDA(cudaStreamSynchronize(s));
    }
    void allreduce_u64(uint64_t* v, int n, bool mx, cudaStream_t) override {
        ok(t.allreduce_u64(t.user, v, n, mx ? 1 : 0), "allreduce_u64");
    }
    void bcast_f64(double* v, int n, cudaStream_t) override { ok(t.bcast_f64(t.user, v, n), "bcast_f64"); }
};
}  // namespace

Comm* make_host_comm(const nrg_host_transport& t, int rank, int world) {
    if (!t.allgatherv || !t.alltoallv || !t.allreduce_u64 || !t.bcast_f64) fail(22, "host transport: missing callback");
    auto* c = new HostComm();
    c->t = t;
    c->rank = rank;
    c->world = world;
    return c;
}

uint64_t route_plan(int world, int rank, const uint64_t* mat, std::vector<size_t>& sb, std::vector<size_t>& so,
                    std::vector<size_t>& rb, std::vector<size_t>& ro) {
    sb.assign(world, 0);
    so.assign(world, 0);
    rb.assign(world, 0);
    ro.assign(world, 0);
    size_t off = 0, roff = 0;
    uint64_t q = 0;
    for (int r = 0; r < world; ++r) {
        sb[r] = (size_t)mat[(size_t)rank * world + r] * 8;  // my requests to owner r
        so[r] = off;
        off += sb[r];
        rb[r] = (size_t)mat[(size_t)r * world + rank] * 8;  // requester r's keys I own
        ro[r] = roff;
        roff += rb[r];
        q += mat[(size_t)r * world + rank];
    }
    return q;
}

// ---------------------------------------------------------------- loopback
struct LoopbackGroup {
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t phase = 0;
    std::vector<const void*> ptr;
    std::vector<std::vector<size_t>> sizes, offs;
    std::vector<std::vector<uint64_t>> u64;
    std::vector<double> f64;
    explicit LoopbackGroup(int w) : world(w), ptr(w), sizes(w), offs(w), u64(w) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t my = phase;
        if (++arrived == world) {
            arrived = 0;
            ++phase;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return phase != my; });
        }
    }
};

LoopbackGroup* loopback_group_create(int world) { return new LoopbackGroup(world); }
void loopback_group_destroy(LoopbackGroup* g) { delete g; }

namespace {
struct LoopbackComm final : Comm {
    LoopbackGroup* g;
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        std::vector<size_t> b(world, bytes);
        allgatherv(send, recv, b, s);
    }
    void allgatherv(const void* send, void* recv, const std::vector<size_t>& bytes, cudaStream_t s) override {
        NRG_CUDA(cudaStreamSynchronize(s));
        g->ptr[rank] = send;
        g->barrier();
        size_t off = 0;
        for (int r = 0; r < world; ++r) {
            if (bytes[r]) NRG_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + off, g->ptr[r], bytes[r], cudaMemcpyDeviceToDevice, s));
            off += bytes[r];
        }
        NRG_CUDA(cudaStreamSynchronize(s));
        g->barrier();
    }
    void alltoallv(const void* send, const std::vector<size_t>& sb, const std::vector<size_t>& so, void* recv,
                   const std::vector<size_t>& rb, const std::vector<size_t>& ro, cudaStream_t s) override {
        NRG_CUDA(cudaStreamSynchronize(s));
        g->ptr[rank] = send;
        g->sizes[rank] = sb;
        g->offs[rank] = so;
        g->barrier();
        for (int r = 0; r < world; ++r) {
            const size_t n = g->sizes[r][rank];
            if (n != rb[r]) fail(100, "loopback alltoallv: size mismatch");
            if (n)
                NRG_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + ro[r], static_cast<const char*>(g->ptr[r]) + g->offs[r][rank],
                                         n, cudaMemcpyDeviceToDevice, s));
        }
        NRG_CUDA(cudaStreamSynchronize(s));
        g->barrier();
    }
    void allreduce_u64(uint64_t* v, int n, bool mx, cudaStream_t) override {
        g->u64[rank].assign(v, v + n);
        g->barrier();
        for (int t = 0; t < n; ++t) {
            uint64_t acc = mx ? 0 : 0;
            for (int r = 0; r < world; ++r) acc = mx ? std::max(acc, g->u64[r][t]) : acc + g->u64[r][t];
            v[t] = acc;
        }
        g->barrier();
    }
    void bcast_f64(double* v, int n, cudaStream_t) override {
        if (rank == 0) g->f64.assign(v, v + n);
        g->barrier();
        std::memcpy(v, g->f64.data(), n * 8);
        g->barrier();
    }
};
}  // namespace

Comm* make_loopback_comm(LoopbackGroup* g, int rank) {
    auto* c = new LoopbackComm();
    c->g = g;
    c->rank = rank;
    c->world = g->world;
    return c;
}

}  // namespace nrg
