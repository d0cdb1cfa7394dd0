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
    const size_t ne = ea.size();
    std::vector<int64_t> off(n + 1, 0);
    for (size_t e = 0; e < ne; ++e) {
        ++off[ea[e] + 1];
        ++off[eb[e] + 1];
    }
    for (int i = 0; i < n; ++i) off[i + 1] += off[i];
    std::vector<int64_t> fill(off.begin(), off.end() - 1);
    std::vector<int32_t> nbr(2 * ne + 1);
    std::vector<double> nwt(2 * ne + 1);
    for (size_t e = 0; e < ne; ++e) {
        nbr[fill[ea[e]]] = eb[e];
        nwt[fill[ea[e]]++] = ew[e];
        nbr[fill[eb[e]]] = ea[e];
        nwt[fill[eb[e]]++] = ew[e];
    }
    // greedy colouring in id order
    std::vector<int> color(n, -1);
    int ncol = 0;
    {
        std::vector<int> mark;
        for (int i = 0; i < n; ++i) {
            mark.assign(ncol + 2, 0);
            for (int64_t q = off[i]; q < off[i + 1]; ++q)
                if (color[nbr[q]] >= 0) mark[color[nbr[q]]] = 1;
            int col = 0;
            while (mark[col]) ++col;
            color[i] = col;
            ncol = std::max(ncol, col + 1);
        }
    }
    std::vector<int32_t> members;
    std::vector<int> cstart(ncol + 1, 0);
    for (int i = 0; i < n; ++i) ++cstart[color[i] + 1];
    for (int k = 0; k < ncol; ++k) cstart[k + 1] += cstart[k];
    members.resize(n);
    {
        std::vector<int> f(cstart.begin(), cstart.end() - 1);
        for (int i = 0; i < n; ++i) members[f[color[i]]++] = i;
    }
    // ---- device chain
    DevBuf doff, dnbr, dnw, dth, dmem, dspin;
    int64_t* d_off = doff.as<int64_t>(n + 1);
    int32_t* d_nbr = dnbr.as<int32_t>(2 * ne + 1);
    double* d_nw = dnw.as<double>(2 * ne + 1);
    double* d_th = dth.as<double>(n);
    int32_t* d_mem = dmem.as<int32_t>(n);
    int8_t* d_spin = dspin.as<int8_t>(n);
    NRG_CUDA(cudaMemcpyAsync(d_off, off.data(), (n + 1) * 8, cudaMemcpyHostToDevice, c.stream));
    NRG_CUDA(cudaMemcpyAsync(d_nbr, nbr.data(), (2 * ne + 1) * 4, cudaMemcpyHostToDevice, c.stream));
    NRG_CUDA(cudaMemcpyAsync(d_nw, nwt.data(), (2 * ne + 1) * 8, cudaMemcpyHostToDevice, c.stream));
    NRG_CUDA(cudaMemcpyAsync(d_th, th.data(), n * 8, cudaMemcpyHostToDevice, c.stream));
    NRG_CUDA(cudaMemcpyAsync(d_mem, members.data(), n * 4, cudaMemcpyHostToDevice, c.stream));
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
        DevBuf dcs, dbar;
        int* d_cstart = dcs.as<int>(ncol + 1);
        unsigned* bar = dbar.as<unsigned>(2);
        NRG_CUDA(cudaMemcpyAsync(d_cstart, cstart.data(), (ncol + 1) * 4, cudaMemcpyHostToDevice, c.stream));
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

}  // namespace nrg
