// state.cu — context lifecycle, samples, SparseWeights on device, the per-generation
// snapshot (K0) and log_posterior.
//
// Reference: inc/sparse_weights.hpp (SparseWeights), inc/model.hpp:133-162
// (log_posterior), :404-416 (make_empty_state), :36-97 (DistanceCache).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "comm.cuh"
#include "context.cuh"

namespace nrg {

Context::~Context() {
    if (device >= 0) cudaSetDevice(device);
    // DevBuf members release themselves; the device must be current for cudaFree
    if (side) {
        cudaStreamSynchronize(side);
        cudaStreamDestroy(side);
        cudaEventDestroy(side_fork);
        cudaEventDestroy(side_done);
    }
    if (stream) cudaStreamSynchronize(stream);
    for (cudaEvent_t e : ev_free) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_used) cudaEventDestroy(e);
    if (pin_counts) cudaFreeHost(pin_counts);
    tl_stream = stream;  // members free in stream order; StreamOwner destroys the stream last
    delete static_cast<Comm*>(comm);
}

void Context::flush_timing() {
    join_side();
    if (pin_next)
        NRG_CUDA(cudaMemcpyAsync(pin_counts, count_log.p, (size_t)pin_next * 8, cudaMemcpyDeviceToHost, stream));
    if (!spans.empty() || pin_next) NRG_CUDA(cudaStreamSynchronize(stream));
    for (const Span& sp : spans) {
        float ms = 0.f;
        NRG_CUDA(cudaEventElapsedTime(&ms, sp.a, sp.b));
        const double cnt = sp.pin >= 0 ? (double)pin_counts[sp.pin] : sp.pairs;
        if (sp.tag < P_N) {
            phase_ms[sp.tag] += ms;
        } else if (sp.tag == T_K1) {
            k1_ms += ms;
            k1_launches += 1;
            k1_pairs += cnt;
        } else if (sp.tag == T_K2) {
            k2_ms += ms;
            k2_launches += 1;
            k2_pairs += cnt;
        }
    }
    spans.clear();
    pin_next = 0;
    // every event but the open one (a tic still waiting for its toc) is free again
    std::vector<cudaEvent_t> keep(ev_hold);
    if (ev_open) keep.push_back(ev_open);
    for (cudaEvent_t e : ev_used)
        if (std::find(keep.begin(), keep.end(), e) == keep.end()) ev_free.push_back(e);
    ev_used = keep;
}

static uint64_t next_pow2(uint64_t v) {
    uint64_t c = 1;
    while (c < v) c <<= 1;
    return c;
}

void ctx_init(Context& c, int n, int m, int kind, double lambda, int device) {
    if (n < 1 || m < 0) fail(22, "SampleMatrix: bad dimensions");
    if (!(lambda >= 0.0)) fail(22, "lambda must be >= 0");
    if (kind != ISING && kind != GAUSSIAN) fail(22, "unknown model kind");
    c.n = n;
    c.M = m;
    c.kind = kind;
    c.lambda = lambda;
    c.device = device;
    NRG_CUDA(cudaSetDevice(device));
    NRG_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    c.stream_owner.s = c.stream;
    tl_stream = c.stream;
    {
        cudaMemPool_t pool;
        NRG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        NRG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        // Back the pool with physical memory once per device and process: a first large
        // allocation, freed, stays in the pool (threshold above), so the sweeps' scratch
        // is carved from mapped memory -- mapping fresh pool memory mid-sweep measured
        // anywhere from 3 to 300 ms per few hundred MB.  40 GB: config 4 peaks near 20 GB while
        // the distance memo is re-sized (with 16 GB, sweeps of 50-80 ms instead of 33 ms
        // showed up every few generations).  NRG_POOL_RESERVE_GB overrides (0 disables); at
        // most a quarter of the free memory.
        static bool reserved[64] = {};
        if (device >= 0 && device < 64 && !reserved[device]) {
            reserved[device] = true;
            const char* e = getenv("NRG_POOL_RESERVE_GB");
            size_t want = (size_t)((e ? atof(e) : 40.0) * (1ull << 30));
            size_t fr = 0, tot = 0;
            NRG_CUDA(cudaMemGetInfo(&fr, &tot));
            want = std::min(want, fr / 4);
            if (want >= (64ull << 20)) {
                void* p = nullptr;
                if (cudaMallocAsync(&p, want, c.stream) == cudaSuccess) {
                    NRG_CUDA(cudaFreeAsync(p, c.stream));
                    NRG_CUDA(cudaStreamSynchronize(c.stream));
                } else {
                    cudaGetLastError();
                }
            }
        }
    }
    // Mp = 256 * HQ: one 16-byte fp16 load per lane per 256 samples in the Ising screen
    // (score.cu instantiates HQ = 1..8, i.e. M <= 2048; larger M uses the fp64 path)
    c.Mp = 256 * (int)std::max<int64_t>(1, ceil_div(m, 256));
    c.Mw = c.Mp / 32;
    const size_t nm = (size_t)n * c.Mp;
    c.H.ensure(nm * sizeof(double));
    NRG_CUDA(cudaMemsetAsync(c.H.p, 0, nm * sizeof(double), c.stream));
    c.theta.ensure(n * sizeof(double));
    NRG_CUDA(cudaMemsetAsync(c.theta.p, 0, n * sizeof(double), c.stream));
    c.counters.ensure(C_N * sizeof(uint64_t));
    NRG_CUDA(cudaMemsetAsync(c.counters.p, 0, C_N * sizeof(uint64_t), c.stream));
    c.Wcap = 1u << 16;
    c.Wkeys.ensure(c.Wcap * 8);
    c.Wvals.ensure(c.Wcap * 8);
    c.Wcount.ensure(16);
    NRG_CUDA(cudaMemsetAsync(c.Wkeys.p, 0xff, c.Wcap * 8, c.stream));
    NRG_CUDA(cudaMemsetAsync(c.Wcount.p, 0, 16, c.stream));
    c.Ccount.ensure(8);
    c.sync();
}

// ---------------------------------------------------------------- samples
__global__ void pack_spins_f64_kernel(const double* __restrict__ X, int rows, int M, int Mw,
                                      uint32_t* __restrict__ Xb, int* __restrict__ bad) {
    // one warp per (row, 32-sample word)
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t total = (int64_t)rows * Mw;
    if (wid >= total) return;
    const int r = (int)(wid / Mw), w = (int)(wid % Mw);
    const int m = w * 32 + lane;
    bool bit = false;
    if (m < M) {
        const double v = X[(size_t)r * M + m];
        if (v != 1.0 && v != -1.0) atomicExch(bad, 1);
        bit = v > 0.0;
    }
    const uint32_t word = __ballot_sync(0xffffffffu, bit);
    if (lane == 0) Xb[(size_t)r * Mw + w] = word;
}

__global__ void pack_spins_i8_kernel(const int8_t* __restrict__ X, int rows, int M, int Mw,
                                     uint32_t* __restrict__ Xb, int* __restrict__ bad) {
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t total = (int64_t)rows * Mw;
    if (wid >= total) return;
    const int r = (int)(wid / Mw), w = (int)(wid % Mw);
    const int m = w * 32 + lane;
    bool bit = false;
    if (m < M) {
        const int v = X[(size_t)r * M + m];
        if (v != 1 && v != -1) atomicExch(bad, 1);
        bit = v > 0;
    }
    const uint32_t word = __ballot_sync(0xffffffffu, bit);
    if (lane == 0) Xb[(size_t)r * Mw + w] = word;
}

// rows of LSB-first bit-packed spins (the sample-file layout: bit t of a row = spin t is
// +1) into the device words: word w of row r = bytes 4w..4w+3 of the row, bits past M
// cleared
__global__ void repack_bits_kernel(const uint8_t* __restrict__ src, int rows, uint64_t row_bytes, int M, int Mw,
                                   uint32_t* __restrict__ Xb) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)rows * Mw) return;
    const int r = (int)(t / Mw), w = (int)(t % Mw);
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint64_t b = (uint64_t)4 * w + k;
        if (b < row_bytes && (int)(8 * b) < M) v |= (uint32_t)src[(size_t)r * row_bytes + b] << (8 * k);
    }
    const int lo = 32 * w;
    if (M - lo < 32) v &= (M - lo <= 0) ? 0u : ((1u << (M - lo)) - 1u);
    Xb[(size_t)r * Mw + w] = v;
}

static void reset_state(Context& c);
void upload_spins_packed(Context& c, const uint8_t* bits, uint64_t row_bytes) {
    if (c.kind != ISING) fail(22, "packed spins are only valid for the ising model");
    if (row_bytes * 8 < (uint64_t)c.M) fail(22, "packed spin rows shorter than M bits");
    c.Xb.ensure((size_t)c.n * c.Mw * 4);
    const int rows_per = std::max<int>(1, (int)std::min<int64_t>(c.n, (256ll << 20) / std::max<uint64_t>(1, row_bytes)));
    uint8_t* d = c.s_a.as<uint8_t>((size_t)rows_per * row_bytes);
    for (int r0 = 0; r0 < c.n; r0 += rows_per) {
        const int rows = std::min(rows_per, c.n - r0);
        NRG_CUDA(cudaMemcpyAsync(d, bits + (size_t)r0 * row_bytes, (size_t)rows * row_bytes, cudaMemcpyHostToDevice,
                                 c.stream));
        const int64_t words = (int64_t)rows * c.Mw;
        repack_bits_kernel<<<(unsigned)ceil_div(words, 256), 256, 0, c.stream>>>(d, rows, row_bytes, c.M, c.Mw,
                                                                              c.dXb() + (size_t)r0 * c.Mw);
        NRG_LAUNCH_CHECK();
    }
    reset_state(c);
    c.sync();
    c.have_samples = true;
}

__global__ void gauss_theta_rms_kernel(const double* __restrict__ X, int M, int Mp,
                                       double* __restrict__ theta, int* __restrict__ bad) {
    // make_empty_state (inc/model.hpp:404-416): theta = max(rms, 1e-8); block per row
    const int r = blockIdx.x;
    double a = 0.0;
    for (int m = threadIdx.x; m < M; m += blockDim.x) {
        const double v = X[(size_t)r * Mp + m];
        if (!isfinite(v)) atomicExch(bad, 1);
        a += v * v;
    }
    __shared__ double sh[32];
    a = warp_sum(a);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
        v = warp_sum(v);
        if (threadIdx.x == 0) {
            const double rms = M > 0 ? sqrt(v / M) : 1.0;
            theta[r] = fmax(rms, 1e-8);
        }
    }
}

static void reset_state(Context& c) {
    const size_t nm = (size_t)c.n * c.Mp;
    NRG_CUDA(cudaMemsetAsync(c.H.p, 0, nm * sizeof(double), c.stream));
    NRG_CUDA(cudaMemsetAsync(c.theta.p, 0, c.n * sizeof(double), c.stream));
    NRG_CUDA(cudaMemsetAsync(c.Wkeys.p, 0xff, c.Wcap * 8, c.stream));
    NRG_CUDA(cudaMemsetAsync(c.Wcount.p, 0, 16, c.stream));
    c.state_version++;
    c.base_valid = false;
}

void upload_samples_f64(Context& c, const double* X) {
    DevBuf& tmp = c.s_a;
    int* bad = c.s_b.as<int>(1);
    NRG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c.stream));
    if (c.kind == ISING) {
        c.Xb.ensure((size_t)c.n * c.Mw * 4);
        // chunked upload: rows per chunk bounded to ~256 MB of doubles
        const int rows_per = std::max<int>(1, (int)std::min<int64_t>(c.n, (256ll << 20) / (8ll * std::max(1, c.M))));
        double* d = tmp.as<double>((size_t)rows_per * std::max(1, c.M));
        for (int r0 = 0; r0 < c.n; r0 += rows_per) {
            const int rows = std::min(rows_per, c.n - r0);
            NRG_CUDA(cudaMemcpyAsync(d, X + (size_t)r0 * c.M, (size_t)rows * c.M * 8,
                                     cudaMemcpyHostToDevice, c.stream));
            const int64_t warps = (int64_t)rows * c.Mw;
            pack_spins_f64_kernel<<<(unsigned)ceil_div(warps * 32, 256), 256, 0, c.stream>>>(
                d, rows, c.M, c.Mw, c.dXb() + (size_t)r0 * c.Mw, bad);
            NRG_LAUNCH_CHECK();
        }
    } else {
        c.Xd.ensure((size_t)c.n * c.Mp * 8);
        NRG_CUDA(cudaMemsetAsync(c.Xd.p, 0, (size_t)c.n * c.Mp * 8, c.stream));
        if (c.M > 0)
            NRG_CUDA(cudaMemcpy2DAsync(c.Xd.p, (size_t)c.Mp * 8, X, (size_t)c.M * 8, (size_t)c.M * 8,
                                       c.n, cudaMemcpyHostToDevice, c.stream));
    }
    reset_state(c);
    if (c.kind == GAUSSIAN) {
        gauss_theta_rms_kernel<<<c.n, 256, 0, c.stream>>>(c.dXd(), c.M, c.Mp, c.dtheta(), bad);
        NRG_LAUNCH_CHECK();
    }
    int hbad = 0;
    hbad = c.read_scalar(bad);
    if (hbad) {
        c.have_samples = false;
        fail(22, c.kind == ISING ? "ising model requires +/-1 data" : "gaussian samples must be finite");
    }
    c.have_samples = true;
}

void upload_spins_i8(Context& c, const int8_t* X) {
    if (c.kind != ISING) fail(22, "int8 spins are only valid for the ising model");
    int* bad = c.s_b.as<int>(1);
    NRG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c.stream));
    c.Xb.ensure((size_t)c.n * c.Mw * 4);
    const int rows_per = std::max<int>(1, (int)std::min<int64_t>(c.n, (256ll << 20) / std::max(1, c.M)));
    int8_t* d = c.s_a.as<int8_t>((size_t)rows_per * std::max(1, c.M));
    for (int r0 = 0; r0 < c.n; r0 += rows_per) {
        const int rows = std::min(rows_per, c.n - r0);
        NRG_CUDA(cudaMemcpyAsync(d, X + (size_t)r0 * c.M, (size_t)rows * c.M, cudaMemcpyHostToDevice,
                                 c.stream));
        const int64_t warps = (int64_t)rows * c.Mw;
        pack_spins_i8_kernel<<<(unsigned)ceil_div(warps * 32, 256), 256, 0, c.stream>>>(
            d, rows, c.M, c.Mw, c.dXb() + (size_t)r0 * c.Mw, bad);
        NRG_LAUNCH_CHECK();
    }
    reset_state(c);
    int hbad = 0;
    hbad = c.read_scalar(bad);
    if (hbad) {
        c.have_samples = false;
        fail(22, "ising model requires +/-1 data");
    }
    c.have_samples = true;
}

void reset_state_empty(Context& c) {
    if (!c.have_samples) fail(22, "no samples uploaded");
    reset_state(c);
    if (c.kind == GAUSSIAN) {
        int* bad = c.s_b.as<int>(1);
        gauss_theta_rms_kernel<<<c.n, 256, 0, c.stream>>>(c.dXd(), c.M, c.Mp, c.dtheta(), bad);
        NRG_LAUNCH_CHECK();
    }
    begin_generation(c);
    c.sync();
}

void set_theta(Context& c, const double* th) {
    if (c.kind == GAUSSIAN)
        for (int i = 0; i < c.n; ++i)
            if (!(th[i] > 0.0)) fail(22, "gaussian model requires theta > 0");
    NRG_CUDA(cudaMemcpyAsync(c.theta.p, th, c.n * 8, cudaMemcpyHostToDevice, c.stream));
    c.sync();
    c.state_version++;
}

// ---------------------------------------------------------------- W hash
__global__ void w_rehash_kernel(const uint64_t* __restrict__ ok, const double* __restrict__ ov,
                                uint64_t ocap, HashView nw, unsigned long long* used) {
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ocap) return;
    const uint64_t k = ok[s];
    if (k >= kTombKey) return;
    uint64_t t = slot_of(k, nw.mask);
    for (;;) {
        const unsigned long long prev =
            atomicCAS((unsigned long long*)&nw.keys[t], (unsigned long long)kEmptyKey, (unsigned long long)k);
        if (prev == kEmptyKey) {
            nw.vals[t] = ov[s];
            atomicAdd(used, 1ull);
            return;
        }
        t = (t + 1) & nw.mask;
    }
}

// make room for `extra` new inserts (load factor <= 1/2, counting tombstones)
void w_reserve(Context& c, uint64_t extra) {
    uint64_t cnt[2];
    NRG_CUDA(cudaMemcpyAsync(cnt, c.Wcount.p, 16, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    const uint64_t live = cnt[0], used = cnt[1];
    if ((used + extra) * 2 <= c.Wcap) return;
    const uint64_t ncap = std::max<uint64_t>(1u << 16, next_pow2(4 * (live + extra)));
    DevBuf nk, nv;
    nk.ensure(ncap * 8);
    nv.ensure(ncap * 8);
    NRG_CUDA(cudaMemsetAsync(nk.p, 0xff, ncap * 8, c.stream));
    uint64_t* dcnt = static_cast<uint64_t*>(c.Wcount.p);
    NRG_CUDA(cudaMemsetAsync(dcnt + 1, 0, 8, c.stream));
    HashView nw{static_cast<uint64_t*>(nk.p), static_cast<double*>(nv.p), ncap - 1};
    w_rehash_kernel<<<(unsigned)ceil_div(c.Wcap, 256), 256, 0, c.stream>>>(
        static_cast<uint64_t*>(c.Wkeys.p), static_cast<double*>(c.Wvals.p), c.Wcap, nw,
        (unsigned long long*)(dcnt + 1));
    NRG_LAUNCH_CHECK();
    c.sync();
    c.Wkeys = std::move(nk);
    c.Wvals = std::move(nv);
    c.Wcap = ncap;
}

// live couplings, compacted on the device with packed keys (i << ib) | j (ib = bits of N - 1)
__global__ void w_live_kernel(const uint64_t* __restrict__ keys, const double* __restrict__ vals, uint64_t cap,
                              int ib, uint64_t* __restrict__ okey, double* __restrict__ oval,
                              unsigned long long* __restrict__ cnt) {
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t k = s < cap ? keys[s] : kEmptyKey;
    const bool live = k < kTombKey;
    const unsigned b = __ballot_sync(0xffffffffu, live);
    const int lane = threadIdx.x & 31;
    unsigned long long at = 0;
    if (lane == 0 && b) at = atomicAdd(cnt, (unsigned long long)__popc(b));
    at = __shfl_sync(0xffffffffu, at, 0);
    if (live) {
        const uint64_t t = at + __popc(b & ((1u << lane) - 1u));
        okey[t] = ((k >> 32) << ib) | (k & 0xffffffffu);
        oval[t] = vals[s];
    }
}

__global__ void split_keys_kernel(const uint64_t* __restrict__ k, uint64_t n, int ib, int32_t* __restrict__ oi,
                                  int32_t* __restrict__ oj) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    oi[t] = (int32_t)(k[t] >> ib);
    oj[t] = (int32_t)(k[t] & ((1ull << ib) - 1));
}

void get_state(Context& c, double* theta, uint64_t cap, int32_t* ei, int32_t* ej, double* w,
               uint64_t* n_edges) {
    if (theta) NRG_CUDA(cudaMemcpyAsync(theta, c.theta.p, c.n * 8, cudaMemcpyDeviceToHost, c.stream));
    if (cap == 0) {  // count only: the table's live counter (no scan)
        *n_edges = c.read_scalar(static_cast<const uint64_t*>(c.Wcount.p));
        return;
    }
    int ib = 1;
    while (ib < 31 && (1ll << ib) < (long long)c.n) ++ib;
    DevBuf kb, vb, cb, tb;
    uint64_t* k0 = kb.as<uint64_t>(2 * c.Wcap);
    double* v0 = vb.as<double>(2 * c.Wcap);
    unsigned long long* cnt = cb.as<unsigned long long>(1);
    NRG_CUDA(cudaMemsetAsync(cnt, 0, 8, c.stream));
    w_live_kernel<<<(unsigned)ceil_div(c.Wcap, 256), 256, 0, c.stream>>>(
        static_cast<const uint64_t*>(c.Wkeys.p), static_cast<const double*>(c.Wvals.p), c.Wcap, ib, k0, v0, cnt);
    NRG_LAUNCH_CHECK();
    unsigned long long ne = 0;
    ne = c.read_scalar(cnt);
    *n_edges = ne;
    const uint64_t take = std::min<uint64_t>(ne, cap);
    if (!take || !(ei || ej || w)) return;
    // (i, j) order == pair_key order (inc/sparse_weights.hpp rows are read back sorted)
    uint64_t* k1 = k0 + c.Wcap;
    double* v1 = v0 + c.Wcap;
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, k0, k1, v0, v1, (int64_t)ne, 0, 2 * ib, c.stream);
    void* tmp = tb.ensure(bytes);
    cub::DeviceRadixSort::SortPairs(tmp, bytes, k0, k1, v0, v1, (int64_t)ne, 0, 2 * ib, c.stream);
    NRG_LAUNCH_CHECK();
    // (i, j) split on the device (k0 is free again: it holds the int32 pairs now)
    int32_t* di = reinterpret_cast<int32_t*>(k0);
    int32_t* dj = di + take;
    split_keys_kernel<<<(unsigned)ceil_div(take, 256), 256, 0, c.stream>>>(k1, take, ib, di, dj);
    NRG_LAUNCH_CHECK();
    if (ei) NRG_CUDA(cudaMemcpyAsync(ei, di, take * 4, cudaMemcpyDeviceToHost, c.stream));
    if (ej) NRG_CUDA(cudaMemcpyAsync(ej, dj, take * 4, cudaMemcpyDeviceToHost, c.stream));
    if (w) NRG_CUDA(cudaMemcpyAsync(w, v1, take * 8, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
}

void get_sums(Context& c, double* out) {
    if (c.M > 0)
        NRG_CUDA(cudaMemcpy2DAsync(out, (size_t)c.M * 8, c.H.p, (size_t)c.Mp * 8, (size_t)c.M * 8, c.n,
                                   cudaMemcpyDeviceToHost, c.stream));
    c.sync();
}

// ---------------------------------------------------------------- snapshot (K0)
// Ising: T = tanh(H + theta) per node-sample: fp64 master, fp32 copy for the Newton
// iterations, sum T^2 per node, and the int8 copy for the screen: T8 = round(T / d)
// with the per-node step d = max|T| / 127 (rounded up), its 8 two's-complement bit
// planes per 32-sample word (the screen's register-side operand), and per node
// {d, E = sum |T - d T8| (rounded up: the screen's rigorous error), sum T8}.
__global__ void __launch_bounds__(256) snapshot_ising_kernel(const double* __restrict__ H,
                                                             const double* __restrict__ theta, int M, int Mp,
                                                             double* __restrict__ T64, float* __restrict__ T32,
                                                             int8_t* __restrict__ T8, uint32_t* __restrict__ P8,
                                                             float4* __restrict__ Q, double* __restrict__ Tsq,
                                                             const int32_t* __restrict__ rows, uint32_t* __restrict__ P4,
                                                             float4* __restrict__ Q4, const uint32_t* __restrict__ Xb,
                                                             uint8_t* __restrict__ flags) {
    const int r = rows ? rows[blockIdx.x] : (int)blockIdx.x;
    // only the rows whose H_i or theta_i changed since their last snapshot (flag bit 1)
    if (flags) {
        if (!(flags[r] & 2)) return;
        __syncthreads();
        if (threadIdx.x == 0) flags[r] &= (uint8_t)~2;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double th = theta[r];
    __shared__ double sh[8], sq[8], sh4[8];
    __shared__ int si[8], si4[8];
    __shared__ float s_d, s_d4;
    double mx = 0.0, q = 0.0;
    // rows of up to 2048 samples stay in registers between the two phases (thread
    // threadIdx.x owns samples threadIdx.x + 256 k in both), their H loads issued together
    constexpr int KMAX = 8;
    const bool in_regs = Mp <= 256 * KMAX && blockDim.x == 256;
    double tv[KMAX];
    if (in_regs) {
        double hv[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int m = threadIdx.x + 256 * k;
            hv[k] = m < M ? H[(size_t)r * Mp + m] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int m = threadIdx.x + 256 * k;
            tv[k] = 0.0;
            if (m < Mp) {
                const double t = m < M ? tanh(hv[k] + th) : 0.0;
                tv[k] = t;
                T64[(size_t)r * Mp + m] = t;
                T32[(size_t)r * Mp + m] = (float)t;
                mx = fmax(mx, fabs(t));
                q += t * t;
            }
        }
    } else {
        for (int m = threadIdx.x; m < Mp; m += blockDim.x) {
            double t = 0.0;
            if (m < M) t = tanh(H[(size_t)r * Mp + m] + th);
            T64[(size_t)r * Mp + m] = t;
            T32[(size_t)r * Mp + m] = (float)t;
            mx = fmax(mx, fabs(t));
            q += t * t;
        }
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    q = warp_sum(q);
    if (lane == 0) {
        sh[wid] = mx;
        sq[wid] = q;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < 8; ++w) {
            a = fmax(a, sh[w]);
            b += sq[w];
        }
        Tsq[r] = b;
        s_d = a > 0.0 ? __double2float_ru(a / 127.0) : 1.0f;
        s_d4 = a > 0.0 ? __double2float_ru(a / 7.0) : 1.0f;
    }
    __syncthreads();
    const double d = (double)s_d, d4 = (double)s_d4;
    // quantisation by the reciprocal (two fp64 divisions per sample were the kernel's
    // longest dependency); the error sums below use the levels actually chosen, so the
    // screen's bounds stay rigorous whichever way a boundary case rounds
    const double rd = 1.0 / d, rd4 = 1.0 / d4;
    const int Mw = Mp >> 5;
    double e = 0.0, e4 = 0.0;
    int sum = 0, sum4 = 0, npl = 0;  // npl: samples with x = +1 (the 4-bit screen's offset term)
    auto quant = [&](int w, double t) {
        if (lane == 0 && Xb) npl += __popc(Xb[(size_t)r * Mw + w]);
        const int m = 32 * w + lane;
        int v = (int)rint(t * rd);
        v = max(-127, min(127, v));
        e += fabs(t - d * (double)v);
        sum += v;
        T8[(size_t)r * Mp + m] = (int8_t)v;
        uint32_t mine = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t pl = __ballot_sync(0xffffffffu, ((uint32_t)v >> k) & 1u);
            if (lane == k) mine = pl;
        }
        if (lane < 8) P8[((size_t)r * Mw + w) * 8 + lane] = mine;
        if (P4) {
            // the 4-bit field of the first-pass screen: T4 = round(T / d4), |T4| <= 7
            int v4 = (int)rint(t * rd4);
            v4 = max(-7, min(7, v4));
            e4 += fabs(t - d4 * (double)v4);
            sum4 += v4;
            uint32_t mine4 = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t pl = __ballot_sync(0xffffffffu, ((uint32_t)v4 >> k) & 1u);
                if (lane == k) mine4 = pl;
            }
            if (lane < 4) P4[((size_t)r * Mw + w) * 4 + lane] = mine4;
        }
    };
    if (in_regs) {
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int w = wid + 8 * k;  // sample 32 w + lane = threadIdx.x + 256 k
            if (w < Mw) quant(w, tv[k]);
        }
    } else {
        for (int w = wid; w < Mw; w += 8) quant(w, T64[(size_t)r * Mp + 32 * w + lane]);  // 0 on padding
    }
    e = warp_sum(e);
    e4 = warp_sum(e4);
    for (int o = 16; o; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        sum4 += __shfl_xor_sync(0xffffffffu, sum4, o);
    }
    __shared__ int snpl[8];
    __syncthreads();
    if (lane == 0) {
        sh[wid] = e;
        si[wid] = sum;
        sh4[wid] = e4;
        si4[wid] = sum4;
        snpl[wid] = npl;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, a4 = 0.0;
        int b = 0, b4 = 0, np = 0;
        for (int w = 0; w < 8; ++w) {
            a += sh[w];
            b += si[w];
            a4 += sh4[w];
            b4 += si4[w];
            np += snpl[w];
        }
        Q[r] = make_float4(s_d, __double2float_ru(a * (1.0 + 1e-12)), __int_as_float(b), 0.f);
        if (Q4) Q4[r] = make_float4(s_d4, __double2float_ru(a4 * (1.0 + 1e-12)), __int_as_float(b4), __int_as_float(np));
    }
}

// Gaussian: U = X + theta^2 H (the current residual), xx = sum x^2
// Gaussian snapshot: U = X + theta^2 H (fp64) and xx = sum x^2, plus the screen's fp32
// copies of U and X and ||U|| (fp64 sum, the screen's error bound scales with it)
__global__ void snapshot_gauss_kernel(const double* __restrict__ X, const double* __restrict__ H,
                                      const double* __restrict__ theta, int M, int Mp,
                                      double* __restrict__ U, double* __restrict__ xx,
                                      const int32_t* __restrict__ rows, float* __restrict__ U32,
                                      float* __restrict__ X32, double* __restrict__ nu,
                                      uint8_t* __restrict__ flags) {
    const int r = rows ? rows[blockIdx.x] : (int)blockIdx.x;
    if (flags) {
        if (!(flags[r] & 2)) return;
        __syncthreads();
        if (threadIdx.x == 0) flags[r] &= (uint8_t)~2;
    }
    const double t2 = theta[r] * theta[r];
    double a = 0.0, b = 0.0;
    for (int m = threadIdx.x; m < Mp; m += blockDim.x) {
        const double x = X[(size_t)r * Mp + m];
        const double u = m < M ? x + t2 * H[(size_t)r * Mp + m] : 0.0;
        U[(size_t)r * Mp + m] = u;
        if (U32) {
            U32[(size_t)r * Mp + m] = (float)u;
            X32[(size_t)r * Mp + m] = (float)x;
        }
        a += x * x;
        b += u * u;
    }
    __shared__ double sh[32], sh2[32];
    a = warp_sum(a);
    b = warp_sum(b);
    if ((threadIdx.x & 31) == 0) {
        sh[threadIdx.x >> 5] = a;
        sh2[threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
        double w = threadIdx.x < (blockDim.x >> 5) ? sh2[threadIdx.x] : 0.0;
        v = warp_sum(v);
        w = warp_sum(w);
        if (threadIdx.x == 0) {
            xx[r] = v;
            if (nu) nu[r] = sqrt(w) * (1.0 + 1e-12);
        }
    }
}

// partner Bloom masks from W (the screen skips the coupling probe on a clear bit)
__global__ void bloom_kernel(const uint64_t* __restrict__ keys, uint64_t cap, unsigned long long* __restrict__ bl) {
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= cap) return;
    const uint64_t k = keys[s];
    if (k >= kTombKey) return;
    const int u = (int)(k >> 32), v = (int)(k & 0xffffffffu);
    atomicOr(&bl[u], bloom_bit(v));
    atomicOr(&bl[v], bloom_bit(u));
}
static void build_bloom(Context& c) {
    c.BL.ensure((size_t)c.n * 8);
    NRG_CUDA(cudaMemsetAsync(c.BL.p, 0, (size_t)c.n * 8, c.stream));
    if (c.Wcap) {
        bloom_kernel<<<(unsigned)ceil_div(c.Wcap, 256), 256, 0, c.stream>>>(
            static_cast<uint64_t*>(c.Wkeys.p), c.Wcap, static_cast<unsigned long long*>(c.BL.p));
        NRG_LAUNCH_CHECK();
    }
}

void ensure_snapshot(Context& c) {
    if (!c.have_samples) fail(22, "no samples uploaded");
    if (c.snap_version == c.state_version) return;
    c.tic();
    c.sync_flags();
    uint8_t* flags = c.dflags();
    const size_t nm = (size_t)c.n * c.Mp;
    if (c.kind == ISING) {
        if (!c.T64.p || !c.Q8.p || (c.Mw == 32 && !c.P4.p)) {  // first snapshot: every row
            NRG_CUDA(cudaMemsetAsync(flags, 7, (size_t)c.n, c.stream));
        }
        c.T64.ensure(nm * 8);
        c.T32.ensure(nm * 4);
        c.T8.ensure(nm);
        c.P8.ensure(nm);
        c.Q8.ensure((size_t)c.n * 16);
        c.Tsq.ensure((size_t)c.n * 8);
        // the 4-bit first pass runs on the pipelined K1 only (M in (992, 1024])
        if (c.Mw == 32) {
            c.P4.ensure(nm / 2);
            c.Q4.ensure((size_t)c.n * 16);
        }
        snapshot_ising_kernel<<<c.n, 256, 0, c.stream>>>(c.dH(), c.dtheta(), c.M, c.Mp,
                                                         static_cast<double*>(c.T64.p),
                                                         static_cast<float*>(c.T32.p),
                                                         static_cast<int8_t*>(c.T8.p),
                                                         static_cast<uint32_t*>(c.P8.p),
                                                         static_cast<float4*>(c.Q8.p),
                                                         static_cast<double*>(c.Tsq.p), nullptr,
                                                         static_cast<uint32_t*>(c.P4.p),
                                                         static_cast<float4*>(c.Q4.p), c.dXb(), flags);
        build_bloom(c);
    } else {
        if (!c.U.p || !c.nu.p) NRG_CUDA(cudaMemsetAsync(flags, 7, (size_t)c.n, c.stream));
        c.U.ensure(nm * 8);
        c.xx.ensure((size_t)c.n * 8);
        c.U32.ensure(nm * 4);
        c.X32.ensure(nm * 4);
        c.nu.ensure((size_t)c.n * 8);
        snapshot_gauss_kernel<<<c.n, 256, 0, c.stream>>>(c.dXd(), c.dH(), c.dtheta(), c.M, c.Mp,
                                                         static_cast<double*>(c.U.p),
                                                         static_cast<double*>(c.xx.p), nullptr,
                                                         static_cast<float*>(c.U32.p), static_cast<float*>(c.X32.p),
                                                         static_cast<double*>(c.nu.p), flags);
        build_bloom(c);
    }
    NRG_LAUNCH_CHECK();
    c.toc(P_SNAP);
    c.snap_version = c.state_version;
}

// Refresh the snapshot rows of `rows` (device list, nr entries, every stale row among them:
// the endpoints a tie-tail round just changed); the rest of the snapshot must be current.
void snapshot_rows(Context& c, const int32_t* rows, uint64_t nr) {
    if (c.snap_version == c.state_version) return;
    if (nr == 0) {
        c.snap_version = c.state_version;
        return;
    }
    c.tic();
    c.sync_flags();
    if (c.kind == ISING)
        snapshot_ising_kernel<<<(unsigned)nr, 256, 0, c.stream>>>(
            c.dH(), c.dtheta(), c.M, c.Mp, static_cast<double*>(c.T64.p), static_cast<float*>(c.T32.p),
            static_cast<int8_t*>(c.T8.p), static_cast<uint32_t*>(c.P8.p), static_cast<float4*>(c.Q8.p),
            static_cast<double*>(c.Tsq.p), rows, static_cast<uint32_t*>(c.P4.p), static_cast<float4*>(c.Q4.p),
            c.dXb(), c.dflags());
    else
        snapshot_gauss_kernel<<<(unsigned)nr, 256, 0, c.stream>>>(
            c.dXd(), c.dH(), c.dtheta(), c.M, c.Mp, static_cast<double*>(c.U.p), static_cast<double*>(c.xx.p), rows,
            static_cast<float*>(c.U32.p), static_cast<float*>(c.X32.p), static_cast<double*>(c.nu.p), c.dflags());
    build_bloom(c);  // the rows' couplings changed too
    NRG_LAUNCH_CHECK();
    c.toc(P_SNAP);
    c.snap_version = c.state_version;
}

// ---------------------------------------------------------------- log_posterior
__device__ __forceinline__ double log_2cosh(double z) {  // inc/common.hpp:40-43
    const double a = fabs(z);
    return a + log1p(exp(-2.0 * a));
}

template <int BLOCK>
__device__ double block_sum(double v, double* sh) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < 32) {
        r = threadIdx.x < BLOCK / 32 ? sh[threadIdx.x] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;  // valid in thread 0
}

__global__ void __launch_bounds__(256) logpost_node_kernel(int kind, const uint32_t* __restrict__ Xb,
                                                           const double* __restrict__ Xd,
                                                           const double* __restrict__ H,
                                                           const double* __restrict__ theta, int M,
                                                           int Mp, int Mw, double* __restrict__ out, int r0 = 0,
                                                           uint8_t* __restrict__ flags = nullptr) {
    __shared__ double sh[32];
    const int r = r0 + blockIdx.x;
    // out[] persists between calls: a node whose row and theta did not change keeps its term
    if (flags) {
        if (!(flags[r] & 4)) return;
        __syncthreads();
        if (threadIdx.x == 0) flags[r] &= (uint8_t)~4;
    }
    const double th = theta[r];
    double a = 0.0;
    if (kind == ISING) {
        for (int m = threadIdx.x; m < M; m += 256) {
            const double z = H[(size_t)r * Mp + m] + th;
            const double x = (Xb[(size_t)r * Mw + (m >> 5)] >> (m & 31)) & 1u ? 1.0 : -1.0;
            a += x * z - log_2cosh(z);
        }
        a = block_sum<256>(a, sh);
        if (threadIdx.x == 0) out[r] = a;
    } else {
        const double t2 = th * th;
        for (int m = threadIdx.x; m < M; m += 256) {
            const double rr = Xd[(size_t)r * Mp + m] + t2 * H[(size_t)r * Mp + m];
            a += rr * rr;
        }
        a = block_sum<256>(a, sh);
        if (threadIdx.x == 0) out[r] = -a / (2.0 * t2) - M * log(th);
    }
}

__global__ void __launch_bounds__(1024) reduce_fixed_kernel(const double* __restrict__ v, uint64_t n,
                                                            double* __restrict__ out) {
    __shared__ double sh[32];
    double a = 0.0;
    for (uint64_t t = threadIdx.x; t < n; t += 1024) a += v[t];
    a = block_sum<1024>(a, sh);
    if (threadIdx.x == 0) *out = a;
}

__global__ void __launch_bounds__(256) w_abs_partial_kernel(const uint64_t* __restrict__ keys,
                                                            const double* __restrict__ vals,
                                                            uint64_t cap, double* __restrict__ part) {
    __shared__ double sh[32];
    double a = 0.0;
    for (uint64_t s = (uint64_t)blockIdx.x * 256 + threadIdx.x; s < cap; s += (uint64_t)gridDim.x * 256)
        if (keys[s] < kTombKey) a += fabs(vals[s]);
    a = block_sum<256>(a, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = a;
}

__global__ void clear_flag_outside_kernel(uint8_t* __restrict__ flags, int n, int lo, int hi, uint8_t bit) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && (i < lo || i >= hi)) flags[i] &= (uint8_t)~bit;
}

double log_posterior(Context& c) {
    if (!c.have_samples) fail(22, "no samples uploaded");
    // memo per state version: the GCD loop's objective after a sweep is the next
    // generation's base (inc/reconstruct.hpp:174-176, inc/model.hpp:73-81), same state
    if (c.lp_version == c.state_version) return c.lp_value;
    c.tic();
    // per-node terms (persistent: only the nodes flagged stale are recomputed; a sharded job
    // computes its node range and all-gathers the per-node values, so the fixed-order
    // reduction below is bitwise the single-GPU one)
    c.sync_flags();
    uint8_t* flags = c.dflags();
    if (!c.lp_node.p) NRG_CUDA(cudaMemsetAsync(flags, 7, (size_t)c.n, c.stream));  // first call: every node
    double* part = c.lp_node.as<double>((size_t)c.n);
    double* wpart = c.red.as<double>(1024 + 8);
    double* res = wpart + 1024;
    uint64_t lo = 0, hi = (uint64_t)c.n;
    if (c.world > 1) shard_range((uint64_t)c.n, c.rank, c.world, lo, hi);
    if (hi > lo)
        logpost_node_kernel<<<(unsigned)(hi - lo), 256, 0, c.stream>>>(c.kind, c.dXb(), c.dXd(), c.dH(), c.dtheta(),
                                                                     c.M, c.Mp, c.Mw, part, (int)lo, flags);
    NRG_LAUNCH_CHECK();
    if (c.world > 1) {
        std::vector<size_t> bytes(c.world);
        for (int r = 0; r < c.world; ++r) {
            uint64_t l, h;
            shard_range((uint64_t)c.n, r, c.world, l, h);
            bytes[r] = (h - l) * 8;
        }
        static_cast<Comm*>(c.comm)->allgatherv(part + lo, part, bytes, c.stream);
        clear_flag_outside_kernel<<<(unsigned)ceil_div(c.n, 256), 256, 0, c.stream>>>(flags, c.n, (int)lo, (int)hi, 4);
        NRG_LAUNCH_CHECK();
    }
    reduce_fixed_kernel<<<1, 1024, 0, c.stream>>>(part, c.n, res);
    NRG_LAUNCH_CHECK();
    const int nb = 592;
    w_abs_partial_kernel<<<nb, 256, 0, c.stream>>>(static_cast<uint64_t*>(c.Wkeys.p),
                                                   static_cast<double*>(c.Wvals.p), c.Wcap, wpart);
    reduce_fixed_kernel<<<1, 1024, 0, c.stream>>>(wpart, nb, res + 1);
    NRG_LAUNCH_CHECK_N(2);
    double h[2];
    NRG_CUDA(cudaMemcpyAsync(h, res, 16, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    c.toc(P_LOGPOST);
    const double acc = h[0] - c.lambda * h[1];
    if (!std::isfinite(acc)) fail(75, "log_posterior is not finite");
    c.lp_version = c.state_version;
    c.lp_value = acc;
    return acc;
}

// DistanceCache::base (inc/model.hpp:73-81): once per generation
double generation_base(Context& c) {
    if (!c.base_valid) {
        c.base = log_posterior(c);
        // one base for the whole job: pruned pairs tie at exactly -base on every rank
        if (c.world > 1) static_cast<Comm*>(c.comm)->bcast_f64(&c.base, 1, c.stream);
        c.base_valid = true;
    }
    return c.base;
}

// ---------------------------------------------------------------- distance cache
__global__ void cache_rehash_kernel(const uint64_t* __restrict__ ok, const double* __restrict__ ov,
                                    const uint32_t* __restrict__ obits, uint64_t ocap, HashView nw,
                                    uint32_t* __restrict__ nbits) {
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ocap) return;
    const uint64_t k = ok[s];
    if (k == kEmptyKey) return;
    const bool surv = (obits[s >> 5] >> (s & 31)) & 1u;  // pruned entries carry no value
    uint64_t t = slot_of(k, nw.mask);
    for (;;) {
        const unsigned long long prev =
            atomicCAS((unsigned long long*)&nw.keys[t], (unsigned long long)kEmptyKey, (unsigned long long)k);
        if (prev == kEmptyKey) {
            if (surv) {
                nw.vals[t] = ov[s];
                atomicOr(&nbits[t >> 5], 1u << (t & 31));
            }
            return;
        }
        t = (t + 1) & nw.mask;
    }
}

void cache_reserve(Context& c, uint64_t extra) {
    c.join_side();
    const uint64_t kMax = 1ull << 31;
    // claims never exceed what was reserved: while the host bound fits, no readback
    if (c.Ccap) {
        const uint64_t b = c.cache_live_bound + extra;
        if (b * 10 <= c.Ccap * 6 || (c.Ccap == kMax && b * 100 <= kMax * 85)) {
            c.cache_live_bound = b;
            c.cache_live_host = c.cache_live_bound - extra;
            return;
        }
    }
    uint64_t live = 0;
    if (c.Ccap) {
        live = c.read_scalar(static_cast<const uint64_t*>(c.Ccount.p));
    }
    c.cache_live_host = live;
    // load factor <= 0.6; slot indices are 31-bit (bit 31 flags remote slots), so at the
    // 2^31-slot ceiling the table runs up to 0.85 full (longer probes, still exact)
    uint64_t need = live + extra;
    c.cache_live_bound = need;
    if (c.Ccap && (need * 10 <= c.Ccap * 6 || (c.Ccap == kMax && need * 100 <= kMax * 85))) return;
    if (need * 100 > kMax * 85 && c.Ccap && live) {
        // the generation's pairs no longer fit 31-bit slots: flush the memo.  Callers
        // reserve between sweeps, when no cache slot is referenced (rows, candidate
        // lists and FindBest keys carry distances); within a generation distances are
        // deterministic, so a flushed pair is re-scored to the same value.
        NRG_CUDA(cudaMemsetAsync(c.Ckeys.p, 0xff, c.Ccap * 8, c.stream));
        NRG_CUDA(cudaMemsetAsync(c.Csurv.p, 0, c.Ccap / 8, c.stream));
        NRG_CUDA(cudaMemsetAsync(c.Ccount.p, 0, 8, c.stream));
        c.sync();
        c.cache_flushes += 1;
        c.cache_live_host = live = 0;
        need = extra;
        c.cache_live_bound = need;
        if (need * 10 <= c.Ccap * 6 || (c.Ccap == kMax && need * 100 <= kMax * 85)) return;
    }
    const uint64_t ncap = std::max<uint64_t>(1u << 20, std::min<uint64_t>(next_pow2(2 * need), kMax));
    if (need * 100 > ncap * 85) fail(100, "distance cache: one sweep needs more than 2^31 slots");
    if (ncap == c.Ccap) return;
    DevBuf nk, nv, nb;
    nk.ensure(ncap * 8);
    nv.ensure(ncap * 8);
    nb.ensure(ncap / 8);
    NRG_CUDA(cudaMemsetAsync(nk.p, 0xff, ncap * 8, c.stream));
    NRG_CUDA(cudaMemsetAsync(nb.p, 0, ncap / 8, c.stream));
    HashView nw{static_cast<uint64_t*>(nk.p), static_cast<double*>(nv.p), ncap - 1};
    if (c.Ccap && live) {
        cache_rehash_kernel<<<(unsigned)ceil_div(c.Ccap, 256), 256, 0, c.stream>>>(
            static_cast<uint64_t*>(c.Ckeys.p), static_cast<double*>(c.Cvals.p), static_cast<uint32_t*>(c.Csurv.p),
            c.Ccap, nw, static_cast<uint32_t*>(nb.p));
        NRG_LAUNCH_CHECK();
    }
    if (!c.Ccap) NRG_CUDA(cudaMemsetAsync(c.Ccount.p, 0, 8, c.stream));
    c.sync();
    c.Ckeys = std::move(nk);
    c.Cvals = std::move(nv);
    c.Csurv = std::move(nb);
    c.Ccap = ncap;
}

void begin_generation(Context& c) {
    c.join_side();
    if (c.Ccap) {
        // size the (now empty) memo for the previous generation's pairs + 30%: growing
        // here costs an allocation, growing mid-generation a rehash of every entry
        uint64_t live = 0, k2max = ~0ull;
        live = c.read_scalar(static_cast<const uint64_t*>(c.Ccount.p));
        if (c.k2max.p) k2max = c.read_scalar(static_cast<const uint64_t*>(c.k2max.p));
        // the next generation launches the warp kernel too only if this one needed it
        // (3 x 148 x 32 x 4: CTA-mode capacity with room; a wrong guess costs time only)
        c.k2_wide = k2max > 3ull * 148 * 32 * 4 / 2;
        if (c.k2max.p) NRG_CUDA(cudaMemsetAsync(c.k2max.p, 0, 8, c.stream));
        // (shrinks too: clearing and scanning an oversized memo costs HBM time every sweep)
        const uint64_t want = std::min<uint64_t>(live + live / 10 * 3, (1ull << 31) * 6 / 10);
        // target load 0.75 at the previous count + 30% (power-of-two capacities: the real load
        // is between half of that and that).  A table twice the size probes a little faster
        // but costs more to clear and to scan (the dense root's recount): config 4 measured
        // 31.7 ms per sweep at 2^29 slots, 31.4 at 2^28
        static const uint64_t load_pct = getenv("NRG_MEMO_LOAD_PCT") ? strtoull(getenv("NRG_MEMO_LOAD_PCT"), nullptr, 10) : 75;
        const uint64_t ncap =
            std::max<uint64_t>(1u << 20, std::min<uint64_t>(next_pow2(want * 100 / load_pct + 1), 1ull << 31));
        // a generation that flushed the memo counted only the pairs since its last flush:
        // keep the size (config 5 would otherwise free and re-map tens of GB every sweep)
        const bool flushed = c.cache_flushes != c.flushes_at_gen;
        // shrink only when the need plus another 30% fits half the table: a count that
        // hovers at a power-of-two boundary (config 4: 161M * 10/6 vs 2^28) otherwise frees
        // and re-maps 2 x 4 GB every few generations, a 20-80 ms stall each time
        const bool shrink = ncap < c.Ccap && (want * 100 / load_pct) / 10 * 13 < c.Ccap / 2;
        if ((ncap > c.Ccap || shrink) && !(flushed && ncap < c.Ccap)) {
            c.Ckeys = DevBuf();
            c.Cvals = DevBuf();
            c.Csurv = DevBuf();
            c.Ckeys.ensure(ncap * 8);
            c.Cvals.ensure(ncap * 8);
            c.Csurv.ensure(ncap / 8);
            c.Ccap = ncap;
        }
        NRG_CUDA(cudaMemsetAsync(c.Ckeys.p, 0xff, c.Ccap * 8, c.stream));
        NRG_CUDA(cudaMemsetAsync(c.Csurv.p, 0, c.Ccap / 8, c.stream));
        NRG_CUDA(cudaMemsetAsync(c.Ccount.p, 0, 8, c.stream));
    }
    c.cache_live_host = 0;
    c.cache_live_bound = 0;
    c.base_valid = false;
    c.flushes_at_gen = c.cache_flushes;
}

__global__ void add_u64_kernel(unsigned long long* p, unsigned long long v) { *p += v; }

void counters_add_host(Context& c, int which, uint64_t v) {
    add_u64_kernel<<<1, 1, 0, c.stream>>>((unsigned long long*)(c.dcounters() + which), (unsigned long long)v);
    NRG_LAUNCH_CHECK();
}

void set_table(Context& c, uint64_t n, const double* t) {
    if (n > (uint64_t)c.n) fail(22, "table larger than the node count");
    c.table.ensure(n * n * 8);
    NRG_CUDA(cudaMemcpyAsync(c.table.p, t, n * n * 8, cudaMemcpyHostToDevice, c.stream));
    c.sync();
    c.table_n = n;
}

void set_line(Context& c, uint64_t n, const double* pos) {
    c.line.ensure(n * 8);
    NRG_CUDA(cudaMemcpyAsync(c.line.p, pos, n * 8, cudaMemcpyHostToDevice, c.stream));
    c.sync();
    c.line_n = n;
}

}  // namespace nrg
