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

// ---------------------------------------------------------------- self-test
// Every collective of the interface on seeded patterns, checked on every rank (all ranks
// call it together): the same code validates the NCCL, host-transport and loopback
// backends, at any world size (world = 1 runs the NCCL calls against the rank itself).
namespace {
inline uint8_t pat(int from, int to, size_t i) { return (uint8_t)(mix64(((uint64_t)from << 40) ^ ((uint64_t)to << 20) ^ i) >> 56); }
}  // namespace

void comm_selftest(Comm& cm, cudaStream_t s) {
    const int W = cm.world, R = cm.rank;
    auto upload = [&](const std::vector<uint8_t>& h) {
        uint8_t* d = nullptr;
        NRG_CUDA(cudaMalloc(&d, std::max<size_t>(h.size(), 16)));
        if (!h.empty()) NRG_CUDA(cudaMemcpyAsync(d, h.data(), h.size(), cudaMemcpyHostToDevice, s));
        return d;
    };
    auto download = [&](const uint8_t* d, size_t n) {
        std::vector<uint8_t> h(n);
        if (n) NRG_CUDA(cudaMemcpyAsync(h.data(), d, n, cudaMemcpyDeviceToHost, s));
        NRG_CUDA(cudaStreamSynchronize(s));
        return h;
    };
    // allgather: 1000 bytes per rank
    {
        const size_t nb = 1000;
        std::vector<uint8_t> h(nb);
        for (size_t i = 0; i < nb; ++i) h[i] = pat(R, W, i);
        uint8_t* ds = upload(h);
        uint8_t* dr = upload(std::vector<uint8_t>(nb * W, 0xEE));
        cm.allgather(ds, dr, nb, s);
        const auto got = download(dr, nb * W);
        for (int r = 0; r < W; ++r)
            for (size_t i = 0; i < nb; ++i)
                if (got[r * nb + i] != pat(r, W, i)) fail(100, "comm selftest: allgather mismatch");
        cudaFree(ds), cudaFree(dr);
    }
    // allgatherv: ragged sizes, every third rank contributes nothing
    {
        std::vector<size_t> nb(W), off(W, 0);
        for (int r = 0; r < W; ++r) nb[r] = r % 3 == 2 ? 0 : 100 * (size_t)(r + 1) + 7;
        for (int r = 1; r < W; ++r) off[r] = off[r - 1] + nb[r - 1];
        const size_t tot = off[W - 1] + nb[W - 1];
        std::vector<uint8_t> h(nb[R]);
        for (size_t i = 0; i < nb[R]; ++i) h[i] = pat(R, W + 1, i);
        uint8_t* ds = upload(h);
        uint8_t* dr = upload(std::vector<uint8_t>(tot, 0xEE));
        cm.allgatherv(ds, dr, nb, s);
        const auto got = download(dr, tot);
        for (int r = 0; r < W; ++r)
            for (size_t i = 0; i < nb[r]; ++i)
                if (got[off[r] + i] != pat(r, W + 1, i)) fail(100, "comm selftest: allgatherv mismatch");
        cudaFree(ds), cudaFree(dr);
    }
    // alltoallv: rank r sends sz(r, q) bytes to q (some pairs empty)
    {
        auto sz = [](int from, int to) { return (size_t)((from * 7 + to * 3) % 5) * 64 + ((from + to) % 4 == 3 ? 0 : 8); };
        std::vector<size_t> sb(W), so(W, 0), rb(W), ro(W, 0);
        for (int q = 0; q < W; ++q) sb[q] = sz(R, q), rb[q] = sz(q, R);
        for (int q = 1; q < W; ++q) so[q] = so[q - 1] + sb[q - 1], ro[q] = ro[q - 1] + rb[q - 1];
        std::vector<uint8_t> h(so[W - 1] + sb[W - 1]);
        for (int q = 0; q < W; ++q)
            for (size_t i = 0; i < sb[q]; ++i) h[so[q] + i] = pat(R, q, i);
        const size_t tot = ro[W - 1] + rb[W - 1];
        uint8_t* ds = upload(h);
        uint8_t* dr = upload(std::vector<uint8_t>(tot, 0xEE));
        cm.alltoallv(ds, sb, so, dr, rb, ro, s);
        const auto got = download(dr, tot);
        for (int q = 0; q < W; ++q)
            for (size_t i = 0; i < rb[q]; ++i)
                if (got[ro[q] + i] != pat(q, R, i)) fail(100, "comm selftest: alltoallv mismatch");
        cudaFree(ds), cudaFree(dr);
    }
    // host-scalar collectives; the long vector is a world x world routing matrix and more
    for (const int n : {3, W * W + 70}) {
        std::vector<uint64_t> v(n), mx(n);
        for (int t = 0; t < n; ++t) v[t] = (uint64_t)(R + 1) * (t + 1), mx[t] = mix64((uint64_t)R * 1000003 + t) >> 8;
        cm.allreduce_u64(v.data(), n, false, s);
        cm.allreduce_u64(mx.data(), n, true, s);
        for (int t = 0; t < n; ++t) {
            uint64_t want = 0;
            for (int r = 0; r < W; ++r) want = std::max(want, mix64((uint64_t)r * 1000003 + t) >> 8);
            if (v[t] != (uint64_t)W * (W + 1) / 2 * (t + 1) || mx[t] != want) fail(100, "comm selftest: allreduce mismatch");
        }
    }
    {
        double v[5];
        for (int t = 0; t < 5; ++t) v[t] = R == 0 ? 0.1 * (t + 1) : -1.0;
        cm.bcast_f64(v, 5, s);
        for (int t = 0; t < 5; ++t)
            if (v[t] != 0.1 * (t + 1)) fail(100, "comm selftest: broadcast mismatch");
    }
}

}  // namespace nrg
