// gen.cu — synthetic Ising data on the device ("device data
// pipeline").  Truth: Erdos-Renyi by the geometric skip over the upper-triangle
// index (the scheme of inc/synth.hpp:260-292), w ~ N(0, w_sigma^2),
// theta ~ N(0, th_sigma^2), drawn from SplitRng(mix64(seed,0)) exactly like the
// checker's generator.  Samples: Gibbs sweeps with P(x_i=+1|rest) =
// sigmoid(2(m_i+theta_i)) (inc/synth.hpp:133-158), parallelised by a greedy graph
// colouring (nodes of one colour are conditionally independent), burn-in then one
// recorded sample every `thin` sweeps.  The chain differs from the reference's
// sequential sweep order; it targets the same stationary distribution.
#include <algorithm>
#include <cmath>
#include <vector>

#include "context.cuh"

namespace nrg {

static double h_uniform(SplitRng& r) { return r.uniform(); }
static double h_normal(SplitRng& r) {  // inc/random.hpp:55-60
    double u1 = h_uniform(r), u2 = h_uniform(r);
    while (u1 <= 0.0) u1 = h_uniform(r);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586477 * u2);
}

// software grid barrier for the cooperative (co-resident) launch below
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

// The whole chain in one launch: colour classes updated in order with a grid barrier
// between them; samples recorded after burn-in every `thin` sweeps.
__global__ void gibbs_persistent_kernel(const int32_t* __restrict__ members, const int* __restrict__ cstart, int ncol,
                                        const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                                        const double* __restrict__ nw, const double* __restrict__ theta,
                                        int8_t* spin, uint64_t key, int64_t sweeps, int burn_in, int thin, int M,
                                        int Mw, int n, uint32_t* __restrict__ Xb, unsigned* bar) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nth = gridDim.x * blockDim.x;
    int rec = 0;
    for (int64_t s = 0; s < sweeps; ++s) {
        for (int k = 0; k < ncol; ++k) {
            for (int t = cstart[k] + tid; t < cstart[k + 1]; t += nth) {
                const int i = members[t];
                double field = theta[i];
                for (int64_t q = off[i]; q < off[i + 1]; ++q) field += nw[q] * (double)__ldcg(&spin[nbr[q]]);
                const uint64_t r = mix64(key ^ mix64((uint64_t)s * 0x9e3779b97f4a7c15ULL + (uint64_t)i));
                const double u = (double)(r >> 11) * 0x1.0p-53;
                const double z = 2.0 * field;
                const double p = z >= 0.0 ? 1.0 / (1.0 + exp(-z)) : exp(z) / (1.0 + exp(z));
                __stcg(&spin[i], (int8_t)(u < p ? 1 : -1));
            }
            grid_sync(bar, gridDim.x);
        }
        if (s >= burn_in && (s - burn_in + 1) % thin == 0 && rec < M) {
            for (int i = tid; i < n; i += nth) {
                uint32_t* w = &Xb[(size_t)i * Mw + (rec >> 5)];
                const uint32_t bit = 1u << (rec & 31);
                *w = __ldcg(&spin[i]) > 0 ? (*w | bit) : (*w & ~bit);
            }
            ++rec;
            grid_sync(bar, gridDim.x);
        }
    }
}

// The coloured Gibbs chain on a given truth (edges ea-eb with couplings ew, fields th):
// greedy colouring in id order, one cooperative launch for all sweeps, samples into Xb,
// fresh empty state afterwards.
// Gaussian chain for precision K (off-diagonals on the graph, diagonal kd):
// x_i | rest ~ N(-sum_j K_ij x_j / K_ii, 1 / K_ii), colour classes in order with a grid
// barrier in between; samples after burn-in every `thin` sweeps into Xd [N][Mp].
__global__ void gauss_gibbs_kernel(const int32_t* __restrict__ members, const int* __restrict__ cstart, int ncol,
                                   const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                                   const double* __restrict__ nw, const double* __restrict__ kd, double* xs,
                                   uint64_t key, int64_t sweeps, int burn_in, int thin, int M, int Mp, int n,
                                   double* __restrict__ Xd, unsigned* bar) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nth = gridDim.x * blockDim.x;
    int rec = 0;
    for (int64_t s = 0; s < sweeps; ++s) {
        for (int k = 0; k < ncol; ++k) {
            for (int t = cstart[k] + tid; t < cstart[k + 1]; t += nth) {
                const int i = members[t];
                double acc = 0.0;
                for (int64_t q = off[i]; q < off[i + 1]; ++q) acc += nw[q] * __ldcg(&xs[nbr[q]]);
                const uint64_t r = mix64(key ^ mix64((uint64_t)s * 0x9e3779b97f4a7c15ULL + (uint64_t)i));
                const uint64_t r2 = mix64(r ^ 0xd1b54a32d192ed03ULL);
                const double u1 = ((double)(r >> 11) + 0.5) * 0x1.0p-53, u2 = (double)(r2 >> 11) * 0x1.0p-53;
                const double z = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
                __stcg(&xs[i], -acc / kd[i] + z * rsqrt(kd[i]));
            }
            grid_sync(bar, gridDim.x);
        }
        if (s >= burn_in && (s - burn_in + 1) % thin == 0 && rec < M) {
            for (int i = tid; i < n; i += nth) Xd[(size_t)i * Mp + rec] = __ldcg(&xs[i]);
            ++rec;
            grid_sync(bar, gridDim.x);
        }
    }
}

// Truth graph in CSR with a greedy colouring in id order: nodes of one colour are
// conditionally independent and are updated together.
struct ColoredGraph {
    std::vector<int64_t> off;
    std::vector<int32_t> nbr, members;
    std::vector<double> nwt;
    std::vector<int> cstart;
    int ncol = 0;
};

static ColoredGraph build_colored(int n, const std::vector<int32_t>& ea, const std::vector<int32_t>& eb,
                                  const std::vector<double>& ew) {
    ColoredGraph G;
    const size_t ne = ea.size();
    G.off.assign(n + 1, 0);
    for (size_t e = 0; e < ne; ++e) {
        ++G.off[ea[e] + 1];
        ++G.off[eb[e] + 1];
    }
    for (int i = 0; i < n; ++i) G.off[i + 1] += G.off[i];
    std::vector<int64_t> fill(G.off.begin(), G.off.end() - 1);
    G.nbr.assign(2 * ne + 1, 0);
    G.nwt.assign(2 * ne + 1, 0.0);
    for (size_t e = 0; e < ne; ++e) {
        G.nbr[fill[ea[e]]] = eb[e];
        G.nwt[fill[ea[e]]++] = ew[e];
        G.nbr[fill[eb[e]]] = ea[e];
        G.nwt[fill[eb[e]]++] = ew[e];
    }
    std::vector<int> color(n, -1);
    {
        std::vector<int> mark;
        for (int i = 0; i < n; ++i) {
            mark.assign(G.ncol + 2, 0);
            for (int64_t q = G.off[i]; q < G.off[i + 1]; ++q)
                if (color[G.nbr[q]] >= 0) mark[color[G.nbr[q]]] = 1;
            int col = 0;
            while (mark[col]) ++col;
            color[i] = col;
            G.ncol = std::max(G.ncol, col + 1);
        }
    }
    G.cstart.assign(G.ncol + 1, 0);
    for (int i = 0; i < n; ++i) ++G.cstart[color[i] + 1];
    for (int k = 0; k < G.ncol; ++k) G.cstart[k + 1] += G.cstart[k];
    G.members.resize(n);
    std::vector<int> f(G.cstart.begin(), G.cstart.end() - 1);
    for (int i = 0; i < n; ++i) G.members[f[color[i]]++] = i;
    return G;
}

// Device copy of a coloured graph (+ per-node vector `th`).
struct DevGraph {
    DevBuf off, nbr, nw, th, mem, cs;
    int64_t* d_off;
    int32_t* d_nbr;
    double* d_nw;
    double* d_th;
    int32_t* d_mem;
    int* d_cstart;
    DevGraph(Context& c, const ColoredGraph& G, const std::vector<double>& th) {
        const int n = (int)G.members.size();
        const size_t m = G.nbr.size();
        d_off = off.as<int64_t>(n + 1);
        d_nbr = nbr.as<int32_t>(m);
        d_nw = nw.as<double>(m);
        d_th = this->th.as<double>(n);
        d_mem = mem.as<int32_t>(n);
        d_cstart = cs.as<int>(G.ncol + 1);
        NRG_CUDA(cudaMemcpyAsync(d_off, G.off.data(), (n + 1) * 8, cudaMemcpyHostToDevice, c.stream));
        NRG_CUDA(cudaMemcpyAsync(d_nbr, G.nbr.data(), m * 4, cudaMemcpyHostToDevice, c.stream));
        NRG_CUDA(cudaMemcpyAsync(d_nw, G.nwt.data(), m * 8, cudaMemcpyHostToDevice, c.stream));
        NRG_CUDA(cudaMemcpyAsync(d_th, th.data(), n * 8, cudaMemcpyHostToDevice, c.stream));
        NRG_CUDA(cudaMemcpyAsync(d_mem, G.members.data(), n * 4, cudaMemcpyHostToDevice, c.stream));
        NRG_CUDA(cudaMemcpyAsync(d_cstart, G.cstart.data(), (G.ncol + 1) * 4, cudaMemcpyHostToDevice, c.stream));
        c.sync();
    }
};

// The coloured Gibbs chain on a given truth (edges ea-eb with couplings ew, fields th):
// one cooperative launch for all sweeps, samples into Xb, fresh empty state afterwards.
static void gibbs_ising(Context& c, const std::vector<int32_t>& ea, const std::vector<int32_t>& eb,
                        const std::vector<double>& ew, const std::vector<double>& th, int burn_in, int thin,
                        uint64_t seed) {
    const int n = c.n;
    c.truth_i = ea;
    c.truth_j = eb;
    c.truth_w = ew;
    c.truth_node = th;
    const ColoredGraph G = build_colored(n, ea, eb, ew);
    DevGraph D(c, G, th);
    int ncol = G.ncol;
    DevBuf dspin;
    int8_t* d_spin = dspin.as<int8_t>(n);
    int64_t* d_off = D.d_off;
    int32_t* d_nbr = D.d_nbr;
    double* d_nw = D.d_nw;
    double* d_th = D.d_th;
    int32_t* d_mem = D.d_mem;
    int* d_cstart_g = D.d_cstart;
    // ---- device chain
    {
        SplitRng rd(mix64(seed, 1));
        std::vector<int8_t> s0(n);
        for (int i = 0; i < n; ++i) s0[i] = h_uniform(rd) < 0.5 ? -1 : 1;
        NRG_CUDA(cudaMemcpyAsync(d_spin, s0.data(), n, cudaMemcpyHostToDevice, c.stream));
        c.sync();
    }
    c.Xb.ensure((size_t)n * c.Mw * 4);
    NRG_CUDA(cudaMemsetAsync(c.Xb.p, 0, (size_t)n * c.Mw * 4, c.stream));
    const uint64_t key = mix64(seed, 2);
    const int64_t sweeps = (int64_t)burn_in + (int64_t)c.M * thin;
    {
        DevBuf dbar;
        int* d_cstart = d_cstart_g;
        unsigned* bar = dbar.as<unsigned>(2);
        NRG_CUDA(cudaMemsetAsync(bar, 0, 8, c.stream));
        int per = 0, sms = 0;
        NRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gibbs_persistent_kernel, 256, 0));
        NRG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
        int grid = std::max(1, std::min(per * sms, (n + 255) / 256));
        uint32_t* xb = c.dXb();
        int M = c.M, Mw = c.Mw;
        int64_t sw = sweeps;
        void* args[] = {&d_mem, &d_cstart, &ncol, &d_off, &d_nbr, &d_nw, &d_th, &d_spin, (void*)&key, &sw,
                        &burn_in, &thin, &M, &Mw, (void*)&n, &xb, &bar};
        NRG_CUDA(cudaLaunchCooperativeKernel((void*)gibbs_persistent_kernel, grid, 256, args, 0, c.stream));
        NRG_LAUNCH_CHECK();
        c.sync();
    }
    // fresh state: make_empty_state for Ising (theta = 0, W empty, sums 0)
    const size_t nm = (size_t)n * c.Mp;
    NRG_CUDA(cudaMemsetAsync(c.H.p, 0, nm * 8, c.stream));
    NRG_CUDA(cudaMemsetAsync(c.theta.p, 0, n * 8, c.stream));
    NRG_CUDA(cudaMemsetAsync(c.Wkeys.p, 0xff, c.Wcap * 8, c.stream));
    NRG_CUDA(cudaMemsetAsync(c.Wcount.p, 0, 16, c.stream));
    c.sync();
    c.state_version++;
    c.base_valid = false;
    c.have_samples = true;
}


void generate_ising(Context& c, double mean_deg, double w_sigma, double th_sigma, int burn_in, int thin,
                    uint64_t seed) {
    if (c.kind != ISING) fail(22, "generate_ising needs an ising context");
    const int n = c.n;
    if (n < 2 || !(mean_deg >= 0.0) || mean_deg >= n - 1) fail(22, "generate_ising: bad spec");
    if (burn_in < 0 || thin < 1) fail(22, "generate_ising: bad Gibbs params");
    // ---- truth (host, O(E))
    SplitRng rt(mix64(seed, 0));
    const double p = mean_deg / (double)(n - 1);
    std::vector<int32_t> ea, eb;
    std::vector<double> ew;
    if (p > 0.0) {
        const double log1mp = std::log1p(-p);
        const uint64_t total = (uint64_t)n * (uint64_t)(n - 1) / 2;
        uint64_t idx = 0;
        bool first = true;
        auto row_start = [&](int64_t q) { return (uint64_t)q * (uint64_t)(2 * (int64_t)n - q - 1) / 2; };
        for (;;) {
            double u = h_uniform(rt);
            while (u >= 1.0) u = h_uniform(rt);
            const double skip = std::floor(std::log1p(-u) / log1mp);
            idx += first ? (uint64_t)skip : (uint64_t)skip + 1;
            first = false;
            if (idx >= total) break;
            int64_t i = n - 2 - (int64_t)std::floor((std::sqrt(8.0 * (double)(total - 1 - idx) + 1.0) - 1.0) / 2.0);
            while (i > 0 && row_start(i) > idx) --i;
            while (row_start(i + 1) <= idx) ++i;
            const int64_t j = i + 1 + (int64_t)(idx - row_start(i));
            ea.push_back((int32_t)i);
            eb.push_back((int32_t)j);
            ew.push_back(w_sigma * h_normal(rt));
        }
    }
    std::vector<double> th(n);
    for (int i = 0; i < n; ++i) th[i] = th_sigma * h_normal(rt);
    gibbs_ising(c, ea, eb, ew, th, burn_in, thin, seed);
}


// Erased configuration model with a discrete power-law degree sequence
// P(d) ~ d^-gamma, d >= dmin (config 5: gamma 2.5, dmin 2, mean about 4), capped at
// sqrt(n) so the pairing stays simple-graph friendly; self-loops and multi-edges are
// erased.  w ~ N(0, w_sigma^2), theta ~ N(0, th_sigma^2).
void generate_ising_powerlaw(Context& c, double gamma, int dmin, double w_sigma, double th_sigma, int burn_in,
                             int thin, uint64_t seed) {
    if (c.kind != ISING) fail(22, "generate_ising_powerlaw needs an ising context");
    const int n = c.n;
    if (n < 2 || !(gamma > 1.0) || dmin < 1 || burn_in < 0 || thin < 1) fail(22, "generate_ising_powerlaw: bad spec");
    SplitRng rt(mix64(seed, 0));
    const int dmax = std::max(dmin, (int)std::sqrt((double)n));
    std::vector<double> cdf(dmax - dmin + 1);
    double acc = 0.0;
    for (int d = dmin; d <= dmax; ++d) cdf[d - dmin] = (acc += std::pow((double)d, -gamma));
    for (double& v : cdf) v /= acc;
    std::vector<int32_t> stubs;
    for (int i = 0; i < n; ++i) {
        const double u = h_uniform(rt);
        const int d = dmin + (int)(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
        for (int t = 0; t < d; ++t) stubs.push_back(i);
    }
    if (stubs.size() & 1) stubs.push_back((int32_t)(h_uniform(rt) * n) % n);
    for (size_t t = stubs.size() - 1; t > 0; --t) std::swap(stubs[t], stubs[(size_t)(h_uniform(rt) * (t + 1)) % (t + 1)]);
    std::vector<uint64_t> keys;
    keys.reserve(stubs.size() / 2);
    for (size_t t = 0; t + 1 < stubs.size(); t += 2) {
        const int a = stubs[t], b = stubs[t + 1];
        if (a != b) keys.push_back(((uint64_t)std::min(a, b) << 32) | (uint32_t)std::max(a, b));
    }
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    std::vector<int32_t> ea, eb;
    std::vector<double> ew;
    for (uint64_t k : keys) {
        ea.push_back((int32_t)(k >> 32));
        eb.push_back((int32_t)(k & 0xffffffffu));
        ew.push_back(w_sigma * h_normal(rt));
    }
    std::vector<double> th(n);
    for (int i = 0; i < n; ++i) th[i] = th_sigma * h_normal(rt);
    gibbs_ising(c, ea, eb, ew, th, burn_in, thin, seed);
}

// Coloured Gibbs samples of a caller-supplied Ising truth (edges must be distinct,
// i != j; theta per node).
void generate_ising_graph(Context& c, uint64_t ne, const int32_t* ei, const int32_t* ej, const double* w,
                          const double* theta, int burn_in, int thin, uint64_t seed) {
    if (c.kind != ISING) fail(22, "generate_ising_graph needs an ising context");
    if (burn_in < 0 || thin < 1) fail(22, "generate_ising_graph: bad Gibbs params");
    std::vector<int32_t> ea(ne), eb(ne);
    std::vector<double> ew(w, w + ne), th(theta, theta + c.n);
    for (uint64_t e = 0; e < ne; ++e) {
        if (ei[e] < 0 || ej[e] < 0 || ei[e] >= c.n || ej[e] >= c.n) fail(34, "generate_ising_graph: node id out of range");
        if (ei[e] == ej[e]) fail(22, "generate_ising_graph: self-loop");
        ea[e] = std::min(ei[e], ej[e]);
        eb[e] = std::max(ei[e], ej[e]);
    }
    gibbs_ising(c, ea, eb, ew, th, burn_in, thin, seed);
}

// The coloured Gaussian chain on precision K (off-diagonals ew on edges ea-eb,
// diagonal kd); samples into Xd, then the empty Gaussian state (theta = row RMS).
static void gauss_chain(Context& c, const std::vector<int32_t>& ea, const std::vector<int32_t>& eb,
                        const std::vector<double>& ew, const std::vector<double>& kd, int burn_in, int thin,
                        uint64_t seed) {
    const int n = c.n;
    c.truth_i = ea;
    c.truth_j = eb;
    c.truth_w = ew;
    c.truth_node = kd;
    const ColoredGraph G = build_colored(n, ea, eb, ew);
    DevGraph D(c, G, kd);
    DevBuf dxs, dbar;
    double* xs = dxs.as<double>(n);
    NRG_CUDA(cudaMemsetAsync(xs, 0, (size_t)n * 8, c.stream));
    c.Xd.ensure((size_t)n * c.Mp * 8);
    NRG_CUDA(cudaMemsetAsync(c.Xd.p, 0, (size_t)n * c.Mp * 8, c.stream));
    unsigned* bar = dbar.as<unsigned>(2);
    NRG_CUDA(cudaMemsetAsync(bar, 0, 8, c.stream));
    int per = 0, sms = 0;
    NRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gauss_gibbs_kernel, 256, 0));
    NRG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
    int grid = std::max(1, std::min(per * sms, (n + 255) / 256));
    uint64_t key = mix64(seed, 2);
    int64_t sweeps = (int64_t)burn_in + (int64_t)c.M * thin;
    int ncol = G.ncol, M = c.M, Mp = c.Mp, nn = n;
    double* xd = c.dXd();
    void* args[] = {&D.d_mem, &D.d_cstart, &ncol, &D.d_off, &D.d_nbr, &D.d_nw, &D.d_th, &xs, &key, &sweeps,
                    &burn_in, &thin, &M, &Mp, &nn, &xd, &bar};
    NRG_CUDA(cudaLaunchCooperativeKernel((void*)gauss_gibbs_kernel, grid, 256, args, 0, c.stream));
    NRG_LAUNCH_CHECK();
    c.sync();
    c.have_samples = true;
    reset_state_empty(c);  // make_empty_state: theta = row RMS, W empty, sums 0
}

// Gaussian samples for a caller-supplied precision matrix (distinct off-diagonal edges,
// positive diagonal) — SURVEY §8f row 2; sample_gaussian (inc/synth.hpp:95-124) draws
// the same law by sparse Cholesky.
void generate_gaussian_graph(Context& c, uint64_t ne, const int32_t* ei, const int32_t* ej, const double* kij,
                             const double* kdiag, int burn_in, int thin, uint64_t seed) {
    if (c.kind != GAUSSIAN) fail(22, "generate_gaussian_graph needs a gaussian context");
    if (burn_in < 0 || thin < 1) fail(22, "generate_gaussian_graph: bad Gibbs params");
    std::vector<int32_t> ea(ne), eb(ne);
    std::vector<double> ew(kij, kij + ne), kd(kdiag, kdiag + c.n);
    for (uint64_t e = 0; e < ne; ++e) {
        if (ei[e] < 0 || ej[e] < 0 || ei[e] >= c.n || ej[e] >= c.n) fail(34, "generate_gaussian_graph: node id out of range");
        if (ei[e] == ej[e]) fail(22, "generate_gaussian_graph: diagonal entries go in kdiag");
        ea[e] = std::min(ei[e], ej[e]);
        eb[e] = std::max(ei[e], ej[e]);
    }
    for (int i = 0; i < c.n; ++i)
        if (!(kd[i] > 0.0)) fail(22, "generate_gaussian_graph: the diagonal must be positive");
    gauss_chain(c, ea, eb, ew, kd, burn_in, thin, seed);
}

// Config 3: random d-regular graph (pairing model, resampled until simple), precision
// off-diagonals K_ij ~ U(-amp, amp), diagonal K_ii = sum_j |K_ij| + 0.5 (diagonally
// dominant), samples by the coloured Gibbs chain (the stationary law of the spec's sparse
// Cholesky draw); the context gets the empty Gaussian state (theta = row RMS).
void generate_gaussian(Context& c, int degree, double amp, int burn_in, int thin, uint64_t seed) {
    if (c.kind != GAUSSIAN) fail(22, "generate_gaussian needs a gaussian context");
    const int n = c.n;
    if (degree < 1 || degree >= n || ((int64_t)n * degree) % 2 || !(amp >= 0.0) || burn_in < 0 || thin < 1)
        fail(22, "generate_gaussian: bad spec");
    SplitRng rt(mix64(seed, 0));
    std::vector<int32_t> stubs((size_t)n * degree), ea, eb;
    std::vector<uint64_t> keys;
    bool ok = false;
    for (int attempt = 0; attempt < 10000 && !ok; ++attempt) {
        for (int i = 0; i < n; ++i)
            for (int t = 0; t < degree; ++t) stubs[(size_t)i * degree + t] = i;
        for (size_t t = stubs.size() - 1; t > 0; --t)
            std::swap(stubs[t], stubs[(size_t)(h_uniform(rt) * (t + 1)) % (t + 1)]);
        keys.clear();
        ok = true;
        for (size_t t = 0; t + 1 < stubs.size() && ok; t += 2) {
            const int a = stubs[t], b = stubs[t + 1];
            if (a == b) ok = false;
            keys.push_back(((uint64_t)std::min(a, b) << 32) | (uint32_t)std::max(a, b));
        }
        if (ok) {
            std::sort(keys.begin(), keys.end());
            ok = std::adjacent_find(keys.begin(), keys.end()) == keys.end();
        }
    }
    if (!ok) fail(100, "generate_gaussian: no simple regular graph found");
    std::vector<double> ew, kd(n, 0.5);
    for (uint64_t k : keys) {
        ea.push_back((int32_t)(k >> 32));
        eb.push_back((int32_t)(k & 0xffffffffu));
        const double v = amp * (2.0 * h_uniform(rt) - 1.0);
        ew.push_back(v);
        kd[ea.back()] += std::fabs(v);
        kd[eb.back()] += std::fabs(v);
    }
    gauss_chain(c, ea, eb, ew, kd, burn_in, thin, seed);
}

}  // namespace nrg
