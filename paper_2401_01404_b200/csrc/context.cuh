// context.cuh — device-resident state of one GCD problem on one B200.
//
// Layout in HBM, node-major like the reference's SampleMatrix
// (inc/sample_matrix.hpp:12-13):
//   Xb   u32  [N][Mw]   bit-packed +/-1 spins (Ising), bit m%32 of word m/32, 1 = +1
//   Xd   f64  [N][Mp]   samples (Gaussian)
//   H    f64  [N][Mp]   neighbour sums m_i = sum_j W_ij X_j  (inc/sparse_weights.hpp:164)
//   theta f64 [N]
//   W    open-addressing hash pair_key -> w  (inc/sparse_weights.hpp:162)
//   per-generation snapshot (frozen W, inc/model.hpp:32-35):
//     Ising:    T64 f64 [N][Mp] = tanh(H+theta), T32 copy, int8 T8 + bit planes P8 + per-node
//               {step, error, sum} Q8 for the screen, Tsq = sum T64^2
//     Gaussian: U   f64 [N][Mp] = X + theta^2 H,  xx f64 [N] = sum x^2
//   DistanceCache: open-addressing hash pair_key -> dist (inc/model.hpp:36-97)
// Mp = M rounded up to 256 (one 16-byte fp16 load per lane per 256 samples); padding is zero.
#pragma once
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <unordered_map>
#include <mutex>

#include <cuda_fp16.h>

#include "common.cuh"

namespace nrg {

enum Kind { ISING = 0, GAUSSIAN = 1 };
enum Mode { EXACT = 0, GRADIENT = 1, TABLE = 2, LINE = 3 };

// Stream the calling API entry works on; device buffers are allocated and freed in
// that stream's order from the device's memory pool (release threshold pinned, so
// scratch buffers are recycled without cudaMalloc/cudaFree synchronisation).
inline thread_local cudaStream_t tl_stream = nullptr;
inline bool sync_alloc() {  // NRG_SYNC_ALLOC=1: plain cudaMalloc/cudaFree (A/B testing)
    static const bool v = getenv("NRG_SYNC_ALLOC") != nullptr;
    return v;
}
struct StreamScope {
    cudaStream_t prev;
    explicit StreamScope(cudaStream_t s) : prev(tl_stream) { tl_stream = s; }
    ~StreamScope() { tl_stream = prev; }
};

// Freed blocks of a stream, by size class, kept on the host for that stream's next
// allocation of the same class: a sweep allocates and frees ~600 scratch buffers, and the
// pool calls (~1 us each) were host time the device spent starved between small kernels.
// Stream-ordered like the pool: a block freed on stream s is reused only on s.  Dropped
// (returned to the pool) when the stream's context goes (StreamOwner).
struct BlockCache {
    std::mutex mu;
    std::unordered_map<cudaStream_t, std::unordered_map<size_t, std::vector<void*>>> free;
    static BlockCache& get() {
        static BlockCache* bc = new BlockCache();  // process lifetime (no static-destruction order issue)
        return *bc;
    }
    void* take(cudaStream_t s, size_t bytes) {
        std::lock_guard<std::mutex> lk(mu);
        auto it = free.find(s);
        if (it == free.end()) return nullptr;
        auto jt = it->second.find(bytes);
        if (jt == it->second.end() || jt->second.empty()) return nullptr;
        void* p = jt->second.back();
        jt->second.pop_back();
        return p;
    }
    void put(cudaStream_t s, size_t bytes, void* p) {
        std::lock_guard<std::mutex> lk(mu);
        free[s][bytes].push_back(p);
    }
    void drop(cudaStream_t s) {
        std::unordered_map<size_t, std::vector<void*>> blocks;
        {
            std::lock_guard<std::mutex> lk(mu);
            auto it = free.find(s);
            if (it == free.end()) return;
            blocks.swap(it->second);
            free.erase(it);
        }
        for (auto& kv : blocks)
            for (void* p : kv.second) cudaFreeAsync(p, s);
    }
};
inline bool block_cache_on() {
    static const bool v = getenv("NRG_NO_BLOCK_CACHE") == nullptr;
    return v;
}
// Only small blocks are kept: a multi-GB buffer (the distance memo, config 5's candidate
// arrays) goes straight back to the pool, where any later request can use its memory --
// hoarded by exact size class it ran config 5 out of memory and left freed 2-4 GB memo
// blocks idle while new ones were mapped.
constexpr size_t kBlockCacheMax = (size_t)32 << 20;

// grow-only device buffer (RAII, move-only, stream-ordered)
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), s(o.s) {
        o.p = nullptr;
        o.bytes = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            bytes = o.bytes;
            s = o.s;
            o.p = nullptr;
            o.bytes = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void* ensure(size_t b) {
        if (b > bytes) {
            release();
            // size classes (4 per octave): requests of similar size land on the same
            // block size, so the stream-ordered pool reuses freed blocks exactly instead
            // of mapping new memory for each slightly different size
            size_t nb = b + b / 4 + 256;
            if (nb > (1u << 20)) {
                int lg = 63 - __builtin_clzll((unsigned long long)nb);
                const size_t q = (size_t)1 << (lg - 2);
                nb = (nb + q - 1) / q * q;
            }
            s = tl_stream;
            static const bool dbg = getenv("NRG_DEBUG_ALLOC") != nullptr;
            const auto t0 = dbg ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point();
            if (sync_alloc()) {
                NRG_CUDA(cudaMalloc(&p, nb));
            } else if (!(block_cache_on() && s && nb <= kBlockCacheMax && (p = BlockCache::get().take(s, nb)))) {
                cudaError_t e = cudaMallocAsync(&p, nb, s);
                if (e == cudaErrorMemoryAllocation) {
                    // return every cached block to the pool, let queued frees land, retry once
                    cudaGetLastError();
                    BlockCache::get().drop(s);
                    cudaStreamSynchronize(s);
                    e = cudaMallocAsync(&p, nb, s);
                }
                NRG_CUDA(e);
            }
            if (dbg) {
                const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                if (ms > 1.0) fprintf(stderr, "alloc %.3f GB took %.1f ms\n", nb / 1e9, ms);
            }
            bytes = nb;
        }
        return p;
    }
    template <class T>
    T* as(size_t count) {
        return static_cast<T*>(ensure(count * sizeof(T) + 16));
    }
    void release() {
        if (p) {
            if (sync_alloc())
                cudaFree(p);
            else if (block_cache_on() && s && bytes <= kBlockCacheMax)
                BlockCache::get().put(s, bytes, p);
            else
                cudaFreeAsync(p, s);
        }
        p = nullptr;
        bytes = 0;
    }
};

struct HashView {
    uint64_t* keys;
    double* vals;
    uint64_t mask;  // capacity - 1 (power of two)
};

// A dense level's distances, sparse: bit t of `bits` is set for the screen's survivors
// (and existing couplings) among the triangle's pairs; their values sit in `vals` at
// rank(t) = rank[t / 32] + popcount of the lower bits of word t / 32 (NaN-boxed worklist
// entries until the lazy K2 resolves them); every other pair is pruned: -base exactly.
struct DenseView {
    const uint32_t* bits;
    const uint32_t* rank;
    double* vals;
    double pruned;
};
// The distance memo's values: a pair the screen pruned is never written (its distance is
// -base exactly: bit clear in the survivor bitmap, the L2-resident test every read makes);
// the rest (K2 results) are written with their bit set.  Saves the K1 screen a scattered
// 8-byte store into the multi-GB value array for every pruned pair.
struct MemoView {
    const uint32_t* bits;
    const double* vals;
    double pruned;
};
__device__ __forceinline__ double memo_value(const MemoView& C, uint64_t s) {
    if (!C.bits) return C.vals[s];
    return (__ldg(&C.bits[s >> 5]) >> (s & 31)) & 1u ? C.vals[s] : C.pruned;
}

__device__ __forceinline__ uint32_t dense_rank(const DenseView& D, uint64_t t) {
    const uint32_t w = D.bits[t >> 5];
    return D.rank[t >> 5] + __popc(w & ((1u << (t & 31)) - 1u));
}
__device__ __forceinline__ double dense_value(const DenseView& D, uint64_t t) {
    const uint32_t w = __ldg(&D.bits[t >> 5]);
    const uint32_t bit = 1u << (t & 31);
    if (!(w & bit)) return D.pruned;
    return D.vals[__ldg(&D.rank[t >> 5]) + __popc(w & (bit - 1u))];
}

__device__ __forceinline__ double hash_get(const HashView h, uint64_t key, double dflt) {
    uint64_t s = slot_of(key, h.mask);
    for (;;) {
        const uint64_t k = h.keys[s];
        if (k == key) return h.vals[s];
        if (k == kEmptyKey) return dflt;
        s = (s + 1) & h.mask;
    }
}

// Bloom bit of node v in a partner mask: a clear bit proves (u, v) holds no coupling
__host__ __device__ __forceinline__ unsigned long long bloom_bit(int v) {
    return 1ull << (((uint32_t)v * 0x9E3779B1u) >> 26);
}

struct IsingSnap {
    const uint32_t* Xb;
    const float* T32;    // fp32 copy for the Newton iterations ahead of the final fp64 pass
    const double* T64;
    const int8_t* T8;    // int8 field T8 = round(T / d) for the screen (partner side)
    const uint32_t* P8;  // T8's 8 bit planes per 32-sample word (screen, register side)
    const float4* Q8;    // per node {d, E = sum |T - d T8| rounded up, sum T8 (int bits), 0}
    const unsigned long long* BL;  // per node 64-bit Bloom mask of its coupling partners
    const double* Tsq;   // sum T64^2 per node (L''(0) = -(2M - Tsq_a - Tsq_b) for w_cur = 0)
    int M, Mp, Mw;
    const uint32_t* P4;  // 4 bit planes of T4 = round(T / d4) per 32-sample word (first-pass screen)
    const float4* Q4;    // per node {d4, E4 = sum |T - d4 T4| rounded up, sum T4, 0}
};

struct GaussSnap {
    const double* X;
    const double* U;
    const double* xx;
    const double* theta;
    int M, Mp;
    const float* U32;  // screen copies (fp32) and ||U|| per node
    const float* X32;
    const double* nu;
    const unsigned long long* BL;
};

// outputs of a scoring pass: either scattered into the distance cache (slot-indexed)
// or written per entry
struct ScoreOut {
    double* cache_vals = nullptr;
    const uint32_t* slot = nullptr;
    // cache_bits (the distance memo's survivor bitmap): pruned pairs are not written,
    // refined ones are written and their bit set (MemoView)
    uint32_t* cache_bits = nullptr;
    double* dist = nullptr;
    double* w = nullptr;
    double* gain = nullptr;
    uint8_t* warn = nullptr;
};

enum Counter { C_MISSES = 0, C_HITS = 1, C_EVALS = 2, C_WARN = 3, C_N = 4 };
enum Phase { P_SCORE = 0, P_KNN = 1, P_SELECT = 2, P_UPDATE = 3, P_THETA = 4, P_LOGPOST = 5, P_SNAP = 6, P_N = 7 };
// per-kernel timing tags beyond the phases (K1 screen, K2 refine)
enum { T_K1 = P_N, T_K2 = P_N + 1 };

struct StreamOwner {  // declared first in Context: destroyed after every DevBuf member
    cudaStream_t s = nullptr;
    ~StreamOwner() {
        if (s) {
            BlockCache::get().drop(s);  // the stream's cached blocks back to the pool, in its order
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

struct Context {
    StreamOwner stream_owner;
    int n = 0, M = 0, kind = 0, device = 0;
    int Mp = 0, Mw = 0;
    double lambda = 0.0;
    cudaStream_t stream = nullptr;
    bool have_samples = false;

    // samples
    DevBuf Xb, Xd;
    // state
    DevBuf H, theta;
    DevBuf Wkeys, Wvals;
    uint64_t Wcap = 0;
    DevBuf Wcount;  // u64[2]: live, used (occupied incl. tombstones)
    uint64_t state_version = 1;
    // Per-node staleness flags (u8[n]): bit 0 theta_i not yet re-optimised for the current
    // row H_i, bit 1 the snapshot row, bit 2 the node's log-posterior term.  Set by the
    // kernels that change H_i (the update kernel) or theta_i (the theta pass), cleared by
    // the consumer that refreshes the row, so a sweep recomputes only the rows it touched
    // (a third of the nodes early in a config-4 reconstruction, a tenth near convergence).
    // flags_version is the state version the flags describe: a mutation that does not
    // maintain them bumps state_version only, and the next consumer marks every row.
    DevBuf row_flags, lp_node;
    uint64_t flags_version = 0;
    uint8_t* dflags() { return static_cast<uint8_t*>(row_flags.p); }
    void sync_flags() {
        static const bool off = getenv("NRG_NO_ROW_FLAGS") != nullptr;  // every row, every time
        if (!off && flags_version == state_version && row_flags.p) return;
        uint8_t* f = row_flags.as<uint8_t>((size_t)n);
        NRG_CUDA(cudaMemsetAsync(f, 7, (size_t)n, stream));
        flags_version = state_version;
    }
    // a state change whose kernels kept the flags exact
    void bump_flagged() {
        const bool ok = flags_version == state_version;
        ++state_version;
        if (ok) flags_version = state_version;
    }

    // snapshot
    DevBuf T32, T64, T8, P8, Q8, BL, Tsq, U, xx;
    DevBuf P4, Q4;  // 4-bit field planes and {d4, E4, sum T4} for the first-pass screen
    DevBuf U32, X32, nu;  // Gaussian screen: fp32 copies of U and X, ||U_i|| (fp64, rounded up)
    uint64_t snap_version = 0;
    uint64_t lp_version = 0;  // log_posterior memo (state version it was computed at)
    double lp_value = 0.0;
    bool base_valid = false;
    double base = 0.0;

    // distance cache
    DevBuf Ckeys, Cvals, Ccount;  // Ccount: u64 live
    DevBuf Csurv;                 // survivor bitmap over the memo's slots (MemoView)
    uint64_t Ccap = 0;
    uint64_t cache_live_host = 0;
    uint64_t cache_live_bound = 0;  // host upper bound on the live count (claims <= reserved)

    // dense FindBest level (find_best.cu): the exact distances of every pair of a deep
    // level's node set S_D (row-major upper triangle over positions in S_D), computed once
    // by the tensor-core screen and held SPARSE (DenseView: a survivor bitmap over the
    // triangle, per-word ranks, and the survivors' values; every other pair is pruned,
    // dist = -base exactly) -- L2-sized instead of 8 bytes per pair; S_D and every deeper
    // level (subsets of S_D) look their
    // distances up here instead of claiming and scoring them one by one.  `dloc` maps a
    // global id to its position in S_D (-1 outside), `dbits` marks the pairs probed so
    // far (the generation's cache-miss count stays the reference's).
    bool dense_active = false;
    uint64_t dense_n = 0;
    DevBuf dsurv, drank, dval, dloc, dbits;
    uint64_t dval_n = 0;
    DevBuf kx_cid, kx_csl, kx_ws, kx_wp, kx_wsl, kx_wd;  // find_knn candidate / worklist scratch
    // Lazy K2 at the dense root: the screen's survivors (the pairs K2 must refine) sit in
    // the triangle as NaN-boxed indices into this worklist and are refined only when a
    // dense level first probes them (dense_resolve_*, exhaustive_tc.cu).
    DevBuf dwl_es, dwl_ep, dwl_slot, dwl_sg, dwl_sf;
    uint64_t dwl_n = 0;
    DevBuf dres_idx, dres_g, dres_f, dres_cnt;
    DevBuf dmark;  // one bit per triangle slot: still marked (L2-resident; the test a probe makes)
    // tensor-core screen scratch (score_all_pairs_tc), grow-only
    DevBuf tc_zx, tc_zt, tc_q, tc_si, tc_sj, tc_sg, tc_sf, tc_ns, tc_es, tc_ep, tc_slot, tc_idx, tc_loc, tc_cnt,
        tc_tmp;

    // test metrics
    DevBuf table, line;
    uint64_t table_n = 0, line_n = 0;

    // counters
    DevBuf counters;  // u64[C_N]
    double phase_ms[P_N] = {0};
    // per-kernel stats: K1 screen ms / launches / pairs, K2 refine ms / launches / survivors
    double k1_ms = 0, k1_launches = 0, k1_pairs = 0, k2_ms = 0, k2_launches = 0, k2_pairs = 0;
    double tail_rounds = 0;  // apply_updates: parallel rounds spent on tie tails
    double tc_launches = 0, tc_pairs = 0;  // tensor-core exhaustive screen
    double cache_flushes = 0;              // distance-cache flushes (generation exceeded 2^31 slots)
    double flushes_at_gen = 0;             // cache_flushes when the current generation began
    // K2 launch shape: the largest survivor count of a K2 launch (device, reset per
    // generation) and whether this generation may need the warp kernel (see refine_survivors)
    DevBuf k2max;
    bool k2_wide = true;
    uint64_t launches0 = 0;

    // Deferred device timing: tic/toc record events on the stream and queue a span;
    // spans are resolved (event elapsed times added to the phase / kernel totals) by
    // flush_timing() at API boundaries, so the timers never stall the stream.  Pair
    // counts known only on the device are copied (asynchronously) into pinned slots.
    struct Span {
        int tag;
        cudaEvent_t a, b;
        double pairs;
        int pin;  // pinned count slot (-1: `pairs` is the count)
    };
    std::vector<cudaEvent_t> ev_free, ev_used, ev_hold;
    std::vector<Span> spans;
    cudaEvent_t ev_open = nullptr;
    uint64_t* pin_counts = nullptr;  // pinned host copy of the count log
    DevBuf count_log;
    int pin_next = 0;
    static constexpr int kPinSlots = 1 << 14;

    // scratch
    DevBuf s_a, s_b, s_c, s_d, s_e, s_f, s_g, s_h, s_i, s_j, s_k, s_l, s_m, s_n, s_o;
    DevBuf red;  // reduction scratch
    // scorer-private scratch (score_entries only)
    DevBuf sc_surv, sc_g, sc_flag, sc_w32, sc_n, sc_rchk, sc_rn;
    std::vector<char> host_scratch;
    // truth of the last device generator call (edges i < j, couplings / precision
    // off-diagonals, fields / precision diagonal), for evaluation against the truth
    std::vector<int32_t> truth_i, truth_j;
    std::vector<double> truth_w, truth_node;

    // multi-GPU: node-sharded NNDescent + key-sharded distance cache (comm.cuh)
    void* comm = nullptr;  // nrg::Comm*
    int rank = 0, world = 1;

    ~Context();

    uint32_t* dXb() { return static_cast<uint32_t*>(Xb.p); }
    double* dXd() { return static_cast<double*>(Xd.p); }
    double* dH() { return static_cast<double*>(H.p); }
    double* dtheta() { return static_cast<double*>(theta.p); }
    uint64_t* dcounters() { return static_cast<uint64_t*>(counters.p); }
    HashView Wview() {
        return {static_cast<uint64_t*>(Wkeys.p), static_cast<double*>(Wvals.p), Wcap - 1};
    }
    HashView Cview() {
        return {static_cast<uint64_t*>(Ckeys.p), static_cast<double*>(Cvals.p), Ccap - 1};
    }
    MemoView mview() {
        return {static_cast<const uint32_t*>(Csurv.p), static_cast<const double*>(Cvals.p), -(base + 0.0)};
    }
    uint32_t* dsurvbits() { return static_cast<uint32_t*>(Csurv.p); }
    DenseView dview() {
        return {static_cast<const uint32_t*>(dsurv.p), static_cast<const uint32_t*>(drank.p),
                static_cast<double*>(dval.p), -(base + 0.0)};
    }
    IsingSnap isnap() {
        return {dXb(), static_cast<float*>(T32.p), static_cast<double*>(T64.p), static_cast<int8_t*>(T8.p),
                static_cast<uint32_t*>(P8.p), static_cast<float4*>(Q8.p),
                static_cast<unsigned long long*>(BL.p), static_cast<double*>(Tsq.p), M, Mp, Mw,
                static_cast<uint32_t*>(P4.p), static_cast<float4*>(Q4.p)};
    }
    GaussSnap gsnap() {
        return {dXd(), static_cast<double*>(U.p), static_cast<double*>(xx.p), dtheta(), M, Mp,
                static_cast<float*>(U32.p), static_cast<float*>(X32.p), static_cast<double*>(nu.p),
                static_cast<unsigned long long*>(BL.p)};
    }
    void sync() { NRG_CUDA(cudaStreamSynchronize(stream)); }

    // pinned host staging (grow-only) for the host-side planning steps' copies
    struct PinBuf {
        void* p = nullptr;
        size_t bytes = 0;
        ~PinBuf() {
            if (p) cudaFreeHost(p);
        }
        template <class T>
        T* as(size_t count) {
            const size_t b = count * sizeof(T) + 16;
            if (b > bytes) {
                if (p) cudaFreeHost(p);
                p = nullptr;
                NRG_CUDA(cudaMallocHost(&p, b + b / 4));
                bytes = b + b / 4;
            }
            return static_cast<T*>(p);
        }
    };
    PinBuf hp_dep, hp_ord, hp_i, hp_j, hp_ch, hp_pairs, hp_small, hp_apply, hp_tail;
    // device tie-tail walk (update.cu): per-node modification stamps, applied list, counts
    DevBuf tail_mod, tail_apply, tail_cnt;
    uint32_t tail_stamp = 0;

    // one device scalar read back through pinned memory (a DMA straight into the
    // host buffer; a pageable destination is staged by the driver)
    template <class T>
    T read_scalar(const T* d) {
        T* h = hp_small.as<T>(1);
        NRG_CUDA(cudaMemcpyAsync(h, d, sizeof(T), cudaMemcpyDeviceToHost, stream));
        sync();
        return *h;
    }

    // side stream for work whose result is needed only later (the dense root's miss
    // recount): fork() orders it after everything queued so far; join_side() makes the
    // main stream wait for it (before the distance cache is cleared, resized or its
    // counters read)
    cudaStream_t side = nullptr;
    cudaEvent_t side_fork = nullptr, side_done = nullptr;
    bool side_pending = false;
    cudaStream_t fork() {
        if (!side) {
            NRG_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
            NRG_CUDA(cudaEventCreateWithFlags(&side_fork, cudaEventDisableTiming));
            NRG_CUDA(cudaEventCreateWithFlags(&side_done, cudaEventDisableTiming));
        }
        NRG_CUDA(cudaEventRecord(side_fork, stream));
        NRG_CUDA(cudaStreamWaitEvent(side, side_fork, 0));
        return side;
    }
    void fork_done() {
        NRG_CUDA(cudaEventRecord(side_done, side));
        side_pending = true;
    }
    void join_side() {
        if (!side_pending) return;
        NRG_CUDA(cudaStreamWaitEvent(stream, side_done, 0));
        side_pending = false;
    }

    // phase timing (device events around a region on this stream, resolved lazily)
    cudaEvent_t take_event() {
        cudaEvent_t e;
        if (ev_free.empty()) {
            NRG_CUDA(cudaEventCreate(&e));
        } else {
            e = ev_free.back();
            ev_free.pop_back();
        }
        ev_used.push_back(e);
        return e;
    }
    void tic() {
        ev_open = take_event();
        NRG_CUDA(cudaEventRecord(ev_open, stream));
    }
    void toc(int tag) {
        if (!ev_open) return;
        cudaEvent_t b = take_event();
        NRG_CUDA(cudaEventRecord(b, stream));
        spans.push_back({tag, ev_open, b, 0.0, -1});
        if (spans.size() >= 4096 || pin_next >= kPinSlots - 64) flush_timing();
    }
    // a kernel-level span: mark() before the launch, span() after (independent of tic/toc)
    cudaEvent_t mark() {
        cudaEvent_t a = take_event();
        ev_hold.push_back(a);
        NRG_CUDA(cudaEventRecord(a, stream));
        return a;
    }
    void span(int tag, cudaEvent_t a, double pairs, int pin = -1) {
        cudaEvent_t b = take_event();
        NRG_CUDA(cudaEventRecord(b, stream));
        for (size_t t = 0; t < ev_hold.size(); ++t)
            if (ev_hold[t] == a) {
                ev_hold[t] = ev_hold.back();
                ev_hold.pop_back();
                break;
            }
        spans.push_back({tag, a, b, pairs, pin});
    }
    // a slot of the device count log: the kernel that knows a count writes it there
    // (no copy in the stream); flush_timing reads the log back once
    unsigned long long* log_slot(int* slot) {
        if (!pin_counts) NRG_CUDA(cudaMallocHost(&pin_counts, kPinSlots * 8));
        if (pin_next >= kPinSlots) flush_timing();
        *slot = pin_next++;
        return static_cast<unsigned long long*>(count_log.ensure(kPinSlots * 8)) + *slot;
    }
    void flush_timing();
};

// ---- state.cu
void ctx_init(Context& c, int n, int m, int kind, double lambda, int device);
void upload_samples_f64(Context& c, const double* X);
void upload_spins_i8(Context& c, const int8_t* X);
void upload_spins_packed(Context& c, const uint8_t* bits, uint64_t row_bytes);
void set_theta(Context& c, const double* th);
void reset_state_empty(Context& c);
// ---- io.cu (binary sample / state files)
void write_samples_file(const char* path, uint64_t n, uint64_t m, int kind, const double* X);
void read_samples_info(const char* path, uint64_t* n, uint64_t* m, int* kind);
void read_samples_file(const char* path, double* X);
void load_samples_file(Context& c, const char* path);
void save_samples_file(Context& c, const char* path);
void write_state_file(const char* path, uint64_t n, const double* theta, uint64_t ne, const int32_t* ei,
                      const int32_t* ej, const double* w);
void read_state_info(const char* path, uint64_t* n, uint64_t* ne);
void read_state_file(const char* path, double* theta, int32_t* ei, int32_t* ej, double* w);
void w_reserve(Context& c, uint64_t extra);
void get_state(Context& c, double* theta, uint64_t cap, int32_t* ei, int32_t* ej, double* w,
               uint64_t* n_edges);
void get_sums(Context& c, double* out);
void ensure_snapshot(Context& c);
void snapshot_rows(Context& c, const int32_t* rows, uint64_t nr);  // only these rows are stale
double log_posterior(Context& c);
double generation_base(Context& c);
void begin_generation(Context& c);
void cache_reserve(Context& c, uint64_t extra);
void counters_add_host(Context& c, int which, uint64_t v);
void set_table(Context& c, uint64_t n, const double* t);
void set_line(Context& c, uint64_t n, const double* pos);

// ---- score.cu
// score a worklist of pairs (s[e], p[e]) against the frozen snapshot
// n_dev (optional): the worklist length lives on the device, n is then its capacity
void score_entries(Context& c, int mode, const int32_t* s, const int32_t* p, uint64_t n,
                   const ScoreOut& out, const unsigned long long* n_dev = nullptr);
// all pairs of `nodes` (device, n entries): dist[e] for e in the row-major upper triangle
void score_all_pairs(Context& c, int mode, const int32_t* nodes, uint64_t n, double* dist);
// tensor-core all-pairs screen (exhaustive_tc.cu); false = not applicable, nothing written
// use_cache: pairs already in this generation's distance cache take the cached value
// lazy (dense root): survivors are left as markers for dense_resolve_* (worklist kept
// in the Context) instead of being refined here
bool score_all_pairs_tc(Context& c, const int32_t* nodes, uint64_t n, double* dist, bool use_cache = false,
                        bool lazy = false);
// Lazy K2 resolution: kernels that meet a triangle slot call dense_resolve_slot (claims a
// marked pair for refinement); dense_resolve_end refines what was claimed.  Distances of
// those slots are valid after dense_resolve_end.
struct DenseResolve {
    DenseView D{nullptr, nullptr, nullptr, 0.0};  // D.bits null: nothing marked (no lazy worklist)
    const float* sg = nullptr;
    const uint8_t* sf = nullptr;
    uint64_t* idx = nullptr;
    float* g = nullptr;
    uint8_t* f = nullptr;
    unsigned long long* cnt = nullptr;
    uint32_t* mark = nullptr;
};
constexpr unsigned long long kMarkTag = 0x7ff4ull << 48;
__device__ __forceinline__ void dense_resolve_slot(const DenseResolve& R, uint32_t s) {
    if (!R.D.bits) return;
    // the marked-slot bitmap (L2) answers for the unmarked majority; clearing the bit
    // claims the pair, and only then is its triangle slot (the NaN-boxed index) read
    const uint32_t bit = 1u << (s & 31);
    if (!(__ldcg(&R.mark[s >> 5]) & bit)) return;
    if (!(atomicAnd(&R.mark[s >> 5], ~bit) & bit)) return;
    const unsigned long long v = __ldcg(reinterpret_cast<const unsigned long long*>(R.D.vals) + dense_rank(R.D, s));
    if ((v & (0xffffull << 48)) != kMarkTag) return;
    const uint64_t t = v & 0xffffffffffffull;
    const unsigned long long at = atomicAdd(R.cnt, 1ull);
    R.idx[at] = t;
    R.g[at] = R.sg[t];
    R.f[at] = R.sf[t];
}
DenseResolve dense_resolve_begin(Context& c);
void dense_resolve_end(Context& c);
// the marked pairs among: a flat slot list / NNDescent candidate rows / every pair of a
// subset of the root (the FindBest base case below a dense root)
void dense_resolve_slots(Context& c, const uint32_t* slots, uint64_t n);
void dense_resolve_rows(Context& c, const uint32_t* cand_slot, const int32_t* cand_cnt, uint64_t lo, uint64_t own,
                        uint64_t capn);
void dense_resolve_subtri(Context& c, const int32_t* nodes, uint64_t n);
void refine_survivors(Context& c, const int32_t* s, const int32_t* p, const uint64_t* surv, const float* surv_g,
                      const uint8_t* surv_flag, uint64_t ns, double base, const ScoreOut& out,
                      const unsigned long long* ns_dev = nullptr);
// cached distance lookups for a batch (probe/claim/score/gather), device arrays
void distance_batch(Context& c, int mode, const int32_t* i, const int32_t* j, uint64_t n,
                    double* dist);
// optimize_edge against the current (live) state
void optimize_edge_live(Context& c, const int32_t* i, const int32_t* j, uint64_t n, double* w,
                        double* gain, uint8_t* warn);
void edge_gradient_live(Context& c, const int32_t* i, const int32_t* j, uint64_t n, double* g);
uint64_t sample_scored_pairs(Context& c, uint64_t cap, uint64_t seed, int32_t* oi, int32_t* oj);

// ---- update.cu
// candidates (device arrays, canonical i<j) in order; assign==nullptr -> optimize_edge;
// dist (optional, device): the candidates' distances, used only to find a tie tail;
// fb_sorted: the list is a FindBest result (sorted by distance), which takes list-order
// tickets; any other list takes dependency-level order.  Results never depend on either.
double apply_updates(Context& c, const int32_t* ci, const int32_t* cj, uint64_t n,
                     const double* assign, const double* dist = nullptr, bool fb_sorted = false);
void theta_pass(Context& c, double* out_only);
// set_edges into an empty coupling table with distinct pairs (false: not applicable)
bool set_edges_bulk(Context& c, const int32_t* ci, const int32_t* cj, uint64_t n, const double* w);
// reconstruct_cd's candidate list: all pairs i < j row-major, constant tie distance
void all_pairs_list(Context& c, int32_t* ci, int32_t* cj, double* tie);

// ---- knn.cu
struct KnnParamsD {
    double eps = 1e-3;
    uint64_t seed = 0;
    int max_sweeps = 100, scan_floor = 8, width_floor = 4;
    bool reverse = false;
};
struct KnnResultD {
    int k = 0;
    int sweeps = 0;
    std::vector<double> churn;
    // device arrays, n*k: global ids and dists, rows sorted by (dist, id)
    int32_t* ids = nullptr;
    double* dists = nullptr;
};
// sorted_valid: d_nodes is known strictly ascending and in range (skips sort + validation)
void find_knn(Context& c, int mode, int k, const int32_t* d_nodes, uint64_t n,
              const KnnParamsD& p, bool exhaustive, KnnResultD& out, DevBuf& ids_buf,
              DevBuf& dist_buf, bool sorted_valid = false);

// ---- find_best.cu
struct TraceLevelD {
    int level, k, exhaustive, knn_sweeps;
    uint64_t nodes, dedup_size;
};
struct BestPairsD {
    // device arrays of the result (sorted by (dist,i,j))
    uint64_t count = 0;
    bool short_count = false;
    std::vector<TraceLevelD> trace;
};
void find_best(Context& c, int mode, uint64_t m, const int32_t* d_nodes, uint64_t n, double knn_eps,
               uint64_t seed, bool reverse, bool exhaustive, BestPairsD& res, DevBuf& out_i,
               DevBuf& out_j, DevBuf& out_d);

// ---- gen.cu
void generate_ising(Context& c, double mean_deg, double w_sigma, double th_sigma, int burn_in,
                    int thin, uint64_t seed);
void generate_ising_powerlaw(Context& c, double gamma, int dmin, double w_sigma, double th_sigma, int burn_in,
                             int thin, uint64_t seed);
void generate_ising_graph(Context& c, uint64_t ne, const int32_t* ei, const int32_t* ej, const double* w,
                          const double* theta, int burn_in, int thin, uint64_t seed);
void generate_gaussian(Context& c, int degree, double amp, int burn_in, int thin, uint64_t seed);
void generate_gaussian_graph(Context& c, uint64_t ne, const int32_t* ei, const int32_t* ej, const double* kij,
                             const double* kdiag, int burn_in, int thin, uint64_t seed);

}  // namespace nrg
