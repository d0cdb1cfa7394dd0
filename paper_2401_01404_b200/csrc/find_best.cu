// find_best.cu — FindBest (Alg. 3) on the device: find_best / find_best_exhaustive
// (inc/find_best.hpp:88-208).
//
// Per level: k = ceil(4m/|S|) NNDescent digraph; D+ = the 2m smallest directed
// entries under (dist, src, dst); D = unique undirected pairs of D+; S' = nodes whose
// every out-entry lies in D+, i.e. whose worst entry is <= the 2m-th key (a local
// test once the threshold is known); recurse on S' (order preserved); merge D with
// the recursive result and keep the (dist,i,j)-smallest want.  Base case |S|^2 <= 4m:
// exhaustive all-pairs scan.  All selection is done with CUB radix sorts over
// composite (dist, i, j) keys, which are total orders, so results are identical to
// the reference's nth_element + sort.
#include <cub/cub.cuh>
#include <cuda/std/tuple>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "context.cuh"

namespace nrg {

struct TriKey {
    uint64_t d;
    uint32_t a, b;
};
struct TriKeyDecomposer {
    __host__ __device__ cuda::std::tuple<uint64_t&, uint32_t&, uint32_t&> operator()(TriKey& k) const {
        return {k.d, k.a, k.b};
    }
};
__device__ __forceinline__ bool trikey_le(const TriKey& x, const TriKey& y) {
    if (x.d != y.d) return x.d < y.d;
    if (x.a != y.a) return x.a < y.a;
    return x.b <= y.b;
}

static void sort_trikeys(Context& c, TriKey* in, TriKey* out, uint64_t n, DevBuf& tmpb) {
    if (!n) return;
    size_t bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, bytes, in, out, (int64_t)n, TriKeyDecomposer{}, c.stream);
    void* tmp = tmpb.ensure(bytes);
    cub::DeviceRadixSort::SortKeys(tmp, bytes, in, out, (int64_t)n, TriKeyDecomposer{}, c.stream);
    NRG_LAUNCH_CHECK();
}

__global__ void tri_from_pairs_kernel(const int32_t* __restrict__ nodes, uint64_t n, const double* __restrict__ dist,
                                      TriKey* __restrict__ out) {
    // row-major upper triangle: candidate (min, max, dist) (inc/common.hpp:27-30)
    const uint64_t a = blockIdx.x;
    if (a >= n) return;
    const uint64_t base = a * (2 * n - a - 1) / 2;
    for (uint64_t c = a + 1 + threadIdx.x; c < n; c += blockDim.x) {
        const uint64_t e = base + (c - a - 1);
        const int32_t x = nodes[a], y = nodes[c];
        TriKey k;
        k.d = dkey(dist[e]);
        k.a = (uint32_t)min(x, y);
        k.b = (uint32_t)max(x, y);
        out[e] = k;
    }
}

__global__ void directed_keys_kernel(const int32_t* __restrict__ nodes, const int32_t* __restrict__ ids,
                                     const double* __restrict__ dists, uint64_t n, int k, TriKey* __restrict__ out) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * (uint64_t)k) return;
    TriKey t;
    t.d = dkey(dists[e]);
    t.a = (uint32_t)nodes[e / k];
    t.b = (uint32_t)ids[e];
    out[e] = t;
}

// canonical pair keys of D+ with an index back into the sorted directed list
__global__ void dplus_pairkeys_kernel(const TriKey* __restrict__ dir, uint64_t m2, uint64_t* __restrict__ pk,
                                      uint32_t* __restrict__ idx) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m2) return;
    pk[e] = pair_key((int32_t)dir[e].a, (int32_t)dir[e].b);
    idx[e] = (uint32_t)e;
}

__global__ void unique_flags_kernel(const uint64_t* __restrict__ keys, uint64_t n, uint8_t* __restrict__ flag) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) flag[e] = (e == 0 || keys[e] != keys[e - 1]) ? 1 : 0;
}

__global__ void d_pairs_kernel(const TriKey* __restrict__ dir, const uint32_t* __restrict__ idx_sorted,
                               const uint8_t* __restrict__ flag, uint64_t n, TriKey* __restrict__ out,
                               unsigned long long* __restrict__ cnt) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n || !flag[e]) return;
    const TriKey& t = dir[idx_sorted[e]];
    TriKey o;
    o.d = t.d;
    o.a = min(t.a, t.b);
    o.b = max(t.a, t.b);
    out[atomicAdd(cnt, 1ull)] = o;
}

// S': worst entry of node li (last of its (dist,id)-sorted row) <= threshold key
__global__ void saturated_kernel(const int32_t* __restrict__ nodes, const int32_t* __restrict__ ids,
                                 const double* __restrict__ dists, uint64_t n, int k, TriKey thr,
                                 uint8_t* __restrict__ flag) {
    const uint64_t li = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= n) return;
    bool all = true;
    for (int t = 0; t < k && all; ++t) {
        TriKey x;
        x.d = dkey(dists[li * k + t]);
        x.a = (uint32_t)nodes[li];
        x.b = (uint32_t)ids[li * k + t];
        all = trikey_le(x, thr);
    }
    flag[li] = all ? 1 : 0;
}

__global__ void trikey_pk_kernel(const TriKey* __restrict__ in, uint64_t n, uint64_t* __restrict__ pk,
                                 uint32_t* __restrict__ idx) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    pk[e] = ((uint64_t)in[e].a << 32) | in[e].b;
    idx[e] = (uint32_t)e;
}
__global__ void gather_trikey_kernel(const TriKey* __restrict__ in, const uint32_t* __restrict__ idx,
                                     const uint8_t* __restrict__ flag, uint64_t n, TriKey* __restrict__ out,
                                     unsigned long long* __restrict__ cnt) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n || !flag[e]) return;
    out[atomicAdd(cnt, 1ull)] = in[idx[e]];
}
__global__ void unpack_trikey_kernel(const TriKey* __restrict__ in, uint64_t n, int32_t* __restrict__ oi,
                                     int32_t* __restrict__ oj, double* __restrict__ od) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    oi[e] = (int32_t)in[e].a;
    oj[e] = (int32_t)in[e].b;
    od[e] = dkey_inv(in[e].d);
}

static inline unsigned g256(uint64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, 256)); }

// union of two candidate lists without duplicate pairs, then the (dist,i,j)-smallest
// `want` (inc/find_best.hpp:171-174 + :62-70)
static uint64_t merge_select(Context& c, TriKey* buf, uint64_t n, uint64_t want, DevBuf& outb) {
    DevBuf pkb, idxb, pk2b, idx2b, flagb, tmpb, ub, cntb, sb;
    uint64_t* pk = pkb.as<uint64_t>(n);
    uint32_t* idx = idxb.as<uint32_t>(n);
    uint64_t* pk2 = pk2b.as<uint64_t>(n);
    uint32_t* idx2 = idx2b.as<uint32_t>(n);
    uint8_t* flag = flagb.as<uint8_t>(n);
    TriKey* uniq = ub.as<TriKey>(n);
    unsigned long long* cnt = cntb.as<unsigned long long>(1);
    if (n) {
        trikey_pk_kernel<<<g256(n), 256, 0, c.stream>>>(buf, n, pk, idx);
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, pk, pk2, idx, idx2, (int64_t)n, 0, 64, c.stream);
        void* tmp = tmpb.ensure(bytes);
        cub::DeviceRadixSort::SortPairs(tmp, bytes, pk, pk2, idx, idx2, (int64_t)n, 0, 64, c.stream);
        unique_flags_kernel<<<g256(n), 256, 0, c.stream>>>(pk2, n, flag);
        NRG_CUDA(cudaMemsetAsync(cnt, 0, 8, c.stream));
        gather_trikey_kernel<<<g256(n), 256, 0, c.stream>>>(buf, idx2, flag, n, uniq, cnt);
        NRG_LAUNCH_CHECK();
    }
    unsigned long long nu = 0;
    if (n) {
        NRG_CUDA(cudaMemcpyAsync(&nu, cnt, 8, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    }
    TriKey* sorted = outb.as<TriKey>(std::max<uint64_t>(nu, 1));
    sort_trikeys(c, uniq, sorted, nu, tmpb);
    c.sync();
    return std::min<uint64_t>(nu, want);
}

// result of a level: TriKey list (a<b canonical) sorted by (dist, a, b)
static uint64_t find_best_impl(Context& c, int mode, uint64_t m, const int32_t* S, uint64_t n, double knn_eps,
                               uint64_t seed, bool reverse, int level, std::vector<TraceLevelD>& trace,
                               DevBuf& result) {
    if (n < 2) return 0;
    const uint64_t total = n * (n - 1) / 2;
    const uint64_t want = std::min(m, total);
    if (n * n <= 4 * m) {
        // base case: exhaustive scan (inc/find_best.hpp:98-104)
        DevBuf distb, keysb, tmpb;
        double* dist = distb.as<double>(total);
        score_all_pairs(c, mode, S, n, dist);
        c.tic();
        TriKey* keys = keysb.as<TriKey>(total);
        tri_from_pairs_kernel<<<(unsigned)n, 256, 0, c.stream>>>(S, n, dist, keys);
        NRG_LAUNCH_CHECK();
        TriKey* out = result.as<TriKey>(total);
        sort_trikeys(c, keys, out, total, tmpb);
        c.sync();
        c.toc(P_SELECT);
        trace.push_back({level, 0, 1, 0, n, 0});
        return want;
    }
    const int k = (int)((4 * m + n - 1) / n);
    KnnParamsD kp;
    kp.eps = knn_eps;
    kp.seed = mix64(seed, (uint64_t)level);
    kp.reverse = reverse;
    KnnResultD knn;
    DevBuf kid, kdist;
    const bool dbg = getenv("NRG_DEBUG_LEVELS") != nullptr;
    uint64_t m0 = 0;
    double t0 = 0.0, s0 = 0.0, k20 = 0.0;
    if (dbg) {
        NRG_CUDA(cudaMemcpyAsync(&m0, c.dcounters() + C_MISSES, 8, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        t0 = c.phase_ms[P_KNN];
        s0 = c.phase_ms[P_SCORE];
        k20 = c.k2_pairs;
    }
    find_knn(c, mode, k, S, n, kp, false, knn, kid, kdist);
    if (dbg) {
        uint64_t m1 = 0;
        NRG_CUDA(cudaMemcpyAsync(&m1, c.dcounters() + C_MISSES, 8, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        fprintf(stderr, "level %d: n=%llu k=%d sweeps=%d knn_ms=%.2f score_ms=%.2f unique_pairs=%llu survivors=%.0f\n",
                level, (unsigned long long)n, k, knn.sweeps, c.phase_ms[P_KNN] - t0, c.phase_ms[P_SCORE] - s0,
                (unsigned long long)(m1 - m0), c.k2_pairs - k20);
    }
    c.tic();
    const uint64_t nd = n * (uint64_t)knn.k;
    DevBuf dirb, dir2b, tmpb;
    TriKey* dir = dirb.as<TriKey>(nd);
    TriKey* dirs = dir2b.as<TriKey>(nd);
    directed_keys_kernel<<<g256(nd), 256, 0, c.stream>>>(S, knn.ids, knn.dists, n, knn.k, dir);
    NRG_LAUNCH_CHECK();
    sort_trikeys(c, dir, dirs, nd, tmpb);
    const uint64_t dplus = std::min<uint64_t>(2 * m, nd);
    // D: unique undirected pairs of D+
    DevBuf pkb, idxb, pk2b, idx2b, flagb, cntb;
    uint64_t* pk = pkb.as<uint64_t>(dplus);
    uint32_t* idx = idxb.as<uint32_t>(dplus);
    uint64_t* pk2 = pk2b.as<uint64_t>(dplus);
    uint32_t* idx2 = idx2b.as<uint32_t>(dplus);
    uint8_t* flag = flagb.as<uint8_t>(std::max<uint64_t>(dplus, n));
    unsigned long long* cnt = cntb.as<unsigned long long>(2);
    dplus_pairkeys_kernel<<<g256(dplus), 256, 0, c.stream>>>(dirs, dplus, pk, idx);
    {
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, pk, pk2, idx, idx2, (int64_t)dplus, 0, 64, c.stream);
        void* tmp = tmpb.ensure(bytes);
        cub::DeviceRadixSort::SortPairs(tmp, bytes, pk, pk2, idx, idx2, (int64_t)dplus, 0, 64, c.stream);
    }
    unique_flags_kernel<<<g256(dplus), 256, 0, c.stream>>>(pk2, dplus, flag);
    DevBuf dpairsb;
    TriKey* dpairs = dpairsb.as<TriKey>(dplus);
    NRG_CUDA(cudaMemsetAsync(cnt, 0, 16, c.stream));
    d_pairs_kernel<<<g256(dplus), 256, 0, c.stream>>>(dirs, idx2, flag, dplus, dpairs, cnt);
    NRG_LAUNCH_CHECK();
    // threshold key = the dplus-th smallest directed entry
    TriKey thr;
    NRG_CUDA(cudaMemcpyAsync(&thr, dirs + (dplus - 1), sizeof(TriKey), cudaMemcpyDeviceToHost, c.stream));
    unsigned long long nD = 0;
    NRG_CUDA(cudaMemcpyAsync(&nD, cnt, 8, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    // S'
    saturated_kernel<<<g256(n), 256, 0, c.stream>>>(S, knn.ids, knn.dists, n, knn.k, thr, flag);
    NRG_LAUNCH_CHECK();
    DevBuf satb, nsatb;
    int32_t* sat = satb.as<int32_t>(n);
    int* nsat = nsatb.as<int>(1);
    {
        size_t bytes = 0;
        cub::DeviceSelect::Flagged(nullptr, bytes, S, flag, sat, nsat, (int64_t)n, c.stream);
        void* tmp = tmpb.ensure(bytes);
        cub::DeviceSelect::Flagged(tmp, bytes, S, flag, sat, nsat, (int64_t)n, c.stream);
    }
    int hsat = 0;
    NRG_CUDA(cudaMemcpyAsync(&hsat, nsat, 4, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    c.toc(P_SELECT);
    trace.push_back({level, k, 0, knn.sweeps, n, (uint64_t)nD});
    kid.release();
    kdist.release();
    dirb.release();

    DevBuf rec;
    const uint64_t nrec = find_best_impl(c, mode, m, sat, (uint64_t)hsat, knn_eps, seed, reverse, level + 1, trace, rec);
    c.tic();
    // merge D with the recursive result (dropping duplicates) and select
    DevBuf allb;
    TriKey* all = allb.as<TriKey>(nD + nrec + 1);
    if (nD) NRG_CUDA(cudaMemcpyAsync(all, dpairs, nD * sizeof(TriKey), cudaMemcpyDeviceToDevice, c.stream));
    if (nrec)
        NRG_CUDA(cudaMemcpyAsync(all + nD, rec.p, nrec * sizeof(TriKey), cudaMemcpyDeviceToDevice, c.stream));
    const uint64_t cntres = merge_select(c, all, nD + nrec, want, result);
    c.toc(P_SELECT);
    return cntres;
}

void find_best(Context& c, int mode, uint64_t m, const int32_t* d_nodes, uint64_t n, double knn_eps,
               uint64_t seed, bool reverse, bool exhaustive, BestPairsD& res, DevBuf& out_i, DevBuf& out_j,
               DevBuf& out_d) {
    if (m < 1) fail(22, exhaustive ? "find_best_exhaustive: m must be >= 1" : "find_best: m must be >= 1");
    if (n < 2) fail(22, exhaustive ? "find_best_exhaustive: need two nodes" : "find_best: need at least two nodes");
    if (mode == TABLE && !c.table_n) fail(22, "no distance table set");
    if (mode == LINE && !c.line_n) fail(22, "no line metric set");
    const uint64_t total = n * (n - 1) / 2;
    res.short_count = m > total;
    res.trace.clear();
    DevBuf result;
    uint64_t cnt;
    if (exhaustive) {
        DevBuf distb, keysb, tmpb;
        double* dist = distb.as<double>(total);
        score_all_pairs(c, mode, d_nodes, n, dist);
        TriKey* keys = keysb.as<TriKey>(total);
        tri_from_pairs_kernel<<<(unsigned)n, 256, 0, c.stream>>>(d_nodes, n, dist, keys);
        NRG_LAUNCH_CHECK();
        distb.release();
        TriKey* out = result.as<TriKey>(total);
        sort_trikeys(c, keys, out, total, tmpb);
        cnt = std::min(m, total);
        res.trace.push_back({0, 0, 1, 0, n, 0});
    } else {
        cnt = find_best_impl(c, mode, m, d_nodes, n, knn_eps, seed, reverse, 0, res.trace, result);
    }
    res.count = cnt;
    int32_t* oi = out_i.as<int32_t>(std::max<uint64_t>(cnt, 1));
    int32_t* oj = out_j.as<int32_t>(std::max<uint64_t>(cnt, 1));
    double* od = out_d.as<double>(std::max<uint64_t>(cnt, 1));
    if (cnt) {
        unpack_trikey_kernel<<<g256(cnt), 256, 0, c.stream>>>(static_cast<TriKey*>(result.p), cnt, oi, oj, od);
        NRG_LAUNCH_CHECK();
    }
    c.sync();
}

}  // namespace nrg
