// update.cu — coordinate updates on the device.
//
// apply_updates: detail::apply_edge_updates with the sequential semantics
// (inc/reconstruct.hpp:74-82): candidates in list order, each re-optimised against
// the CURRENT sums, then set_edge (inc/sparse_weights.hpp:54-85).  Pair p only
// depends on the latest earlier pair sharing an endpoint, so a persistent kernel
// takes pairs in list order (atomic ticket), waits for those two predecessors and
// runs node-disjoint pairs concurrently — the wavefront schedule without per-level
// launches.  The result equals the sequential loop pair by pair.
//
// theta_pass: detail::theta_pass (inc/reconstruct.hpp:129-138) with optimize_theta
// (inc/model.hpp:222-268): Ising by safeguarded Newton on the concave per-node
// objective over [-20, 20] (boundary optima returned exactly, as golden_max's
// best-evaluated-point rule does); Gaussian in closed form with the reference's
// 1e-8 clamp and warnings.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "comm.cuh"
#include "pairscore.cuh"

namespace nrg {

__global__ void dep_keys_kernel(const int32_t* __restrict__ ci, const int32_t* __restrict__ cj, uint64_t n,
                                uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    keys[2 * p] = ((uint64_t)(uint32_t)ci[p] << 32) | (uint32_t)p;
    keys[2 * p + 1] = ((uint64_t)(uint32_t)cj[p] << 32) | (uint32_t)p;
    vals[2 * p] = (uint32_t)(2 * p);
    vals[2 * p + 1] = (uint32_t)(2 * p + 1);
}
__global__ void dep_link_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t m,
                                int32_t* __restrict__ dep) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    int32_t prev = -1;
    if (t > 0 && (keys[t] >> 32) == (keys[t - 1] >> 32)) prev = (int32_t)(keys[t - 1] & 0xffffffffu);
    dep[vals[t]] = prev;  // dep[2p + side] = previous pair index on that endpoint
}

// coherent (L2) hash lookup for the update kernel
__device__ __forceinline__ double hash_get_cg(const HashView h, uint64_t key) {
    uint64_t s = slot_of(key, h.mask);
    for (;;) {
        const uint64_t k = __ldcg(&h.keys[s]);
        if (k == key) return __ldcg(&h.vals[s]);
        if (k == kEmptyKey) return 0.0;
        s = (s + 1) & h.mask;
    }
}
// set W[key] = w: update in place, tombstone on zero, insert into the first empty
// slot otherwise (tombstones are never reused while the table is shared)
__device__ __forceinline__ void hash_set(HashView h, uint64_t key, double w, unsigned long long* cnt) {
    uint64_t s = slot_of(key, h.mask);
    for (;;) {
        const uint64_t k = __ldcg(&h.keys[s]);
        if (k == key) {
            if (w == 0.0) {
                __stcg(&h.keys[s], kTombKey);
                atomicAdd(&cnt[0], (unsigned long long)-1ll);
            } else {
                __stcg(&h.vals[s], w);
            }
            return;
        }
        if (k == kEmptyKey) {
            if (w == 0.0) return;  // absent and zero: nothing stored
            // claim the slot first, then store the value: writing the value before the CAS
            // lets a losing inserter of another key overwrite the winner's value.  Only
            // this pair's successors read vals[s], and they are ordered after us by the
            // done flags; concurrent probes for other keys compare keys only.
            const unsigned long long prev =
                atomicCAS((unsigned long long*)&h.keys[s], (unsigned long long)kEmptyKey, (unsigned long long)key);
            if (prev == kEmptyKey) {
                __stcg(&h.vals[s], w);
                atomicAdd(&cnt[0], 1ull);
                atomicAdd(&cnt[1], 1ull);
                return;
            }
            continue;  // lost the slot to another key: re-examine it
        }
        s = (s + 1) & h.mask;
    }
}

struct UpdateArgs {
    int kind;
    const uint32_t* Xb;
    const double* Xd;
    double* H;
    const double* theta;
    int M, Mp, Mw;
    HashView W;
    unsigned long long* Wcnt;
    const int32_t* ci;
    const int32_t* cj;
    const double* assign;
    const int32_t* dep;
    const uint32_t* order;  // ticket -> pair (dependency-level order) or nullptr (list order)
    uint64_t n;
    double lambda;
    int* done;
    unsigned long long* ticket;
    double* absdelta;
    uint64_t* counters;
    int stage;  // stage tanh(H + theta) of both rows in shared memory once per pair
    uint8_t* flags;  // per-node staleness flags (context.cuh): both endpoints of a changed coupling
};

// One CTA per update: the chain of dependent updates is the critical path (thousands
// of levels at config 4), so per-update latency, not throughput, bounds the phase;
// NT threads share each pass over the samples with block reductions.
template <int NT>
__global__ void __launch_bounds__(NT, 768 / NT) update_kernel(UpdateArgs A) {
    extern __shared__ double stage_smem[];
    __shared__ double red[4 * (NT / 32) + 4];
    __shared__ unsigned long long s_p;
    __shared__ double s_w;
    const int tid = threadIdx.x;
    const BlockScope<NT> sc{red};
    double* ta = stage_smem;
    double* tb = ta + A.Mp;
    uint64_t evals = 0, warns = 0;
    for (;;) {
        if (tid == 0) {
            unsigned long long p = atomicAdd(A.ticket, 1ull);
            if (p < A.n && A.order) p = (unsigned long long)A.order[p];  // level-ordered tickets
            if (p < A.n) {
                // wait for the predecessors on both endpoints
                const int d0 = A.dep[2 * p], d1 = A.dep[2 * p + 1];
                if (d0 >= 0)
                    while (atomicAdd(&A.done[d0], 0) == 0) __nanosleep(32);
                if (d1 >= 0)
                    while (atomicAdd(&A.done[d1], 0) == 0) __nanosleep(32);
                __threadfence();
            }
            s_p = p;
        }
        __syncthreads();
        const unsigned long long p = s_p;
        if (p >= A.n) break;
        __threadfence();
        const int i0 = A.ci[p], j0 = A.cj[p];
        const int a = min(i0, j0), b = max(i0, j0);
        const uint64_t key = pair_key(a, b);
        // one thread reads W and broadcasts (threads are not in lockstep)
        if (tid == 0) s_w = hash_get_cg(A.W, key);
        __syncthreads();
        const double wcur = s_w;
        double w;
        if (A.assign) {
            w = A.assign[p];
        } else if (A.kind == ISING) {
            EdgeOptD r;
            if (A.stage) {
                const double tha = __ldcg(&A.theta[a]), thb = __ldcg(&A.theta[b]);
                // four samples per row per thread in flight before their tanh
                for (int m0 = tid; m0 < A.M; m0 += 4 * NT) {
                    double ha[4], hb[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int m = m0 + u * NT;
                        ha[u] = m < A.M ? __ldcg(&A.H[(size_t)a * A.Mp + m]) : 0.0;
                        hb[u] = m < A.M ? __ldcg(&A.H[(size_t)b * A.Mp + m]) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int m = m0 + u * NT;
                        if (m < A.M) {
                            ta[m] = tanh(ha[u] + tha);
                            tb[m] = tanh(hb[u] + thb);
                        }
                    }
                }
                __syncthreads();
                r = ising_optimize_edge64<TStaged, BlockScope<NT>>(TStaged{ta, tb, a}, A.Xb, A.Mw, A.M, a, b, wcur,
                                                                   A.lambda, sc);
            } else {
                r = ising_optimize_edge64<TLive, BlockScope<NT>>(TLive{A.H, A.theta, A.Mp}, A.Xb, A.Mw, A.M, a, b,
                                                                 wcur, A.lambda, sc);
            }
            w = r.w;
            evals += r.passes;
            warns += r.warn;
        } else {
            const ULive Uf{A.Xd, A.H, A.theta, A.Mp};
            double xxa = 0.0, xxb = 0.0, z0 = 0.0, z1 = 0.0;
            for (int m = tid; m < A.M; m += NT) {
                const double va = A.Xd[(size_t)a * A.Mp + m], vb = A.Xd[(size_t)b * A.Mp + m];
                xxa += va * va;
                xxb += vb * vb;
            }
            sc.sum4(xxa, xxb, z0, z1);
            const double tha = __ldcg(&A.theta[a]), thb = __ldcg(&A.theta[b]);
            const GaussCoef cf = gauss_coef<ULive, BlockScope<NT>>(Uf, A.Xd, A.Mp, A.M, a, b, tha * tha, thb * thb,
                                                                  xxa, xxb, sc);
            const EdgeOptD r = gauss_optimize(cf, wcur, A.lambda);
            w = r.w;
            evals += r.passes;
        }
        // Delta accumulation and set_edge (inc/reconstruct.hpp:78-79)
        const double delta = w - wcur;
        if (delta != 0.0) {
            double* Ha = A.H + (size_t)a * A.Mp;
            double* Hb = A.H + (size_t)b * A.Mp;
            if (A.kind == ISING) {
                for (int m0 = tid; m0 < A.M; m0 += 4 * NT) {  // four samples per row in flight
                    double va[4], vb[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int m = m0 + u * NT;
                        va[u] = m < A.M ? __ldcg(&Ha[m]) : 0.0;
                        vb[u] = m < A.M ? __ldcg(&Hb[m]) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int m = m0 + u * NT;
                        if (m < A.M) {
                            const uint32_t wa = A.Xb[(size_t)a * A.Mw + (m >> 5)], wb = A.Xb[(size_t)b * A.Mw + (m >> 5)];
                            const double xa = xsign(wa, m & 31), xb = xsign(wb, m & 31);
                            __stcg(&Ha[m], va[u] + delta * xb);
                            __stcg(&Hb[m], vb[u] + delta * xa);
                        }
                    }
                }
            } else {
                for (int m = tid; m < A.M; m += NT) {
                    const double xa = A.Xd[(size_t)a * A.Mp + m], xb = A.Xd[(size_t)b * A.Mp + m];
                    __stcg(&Ha[m], __dadd_rn(__ldcg(&Ha[m]), __dmul_rn(delta, xb)));
                    __stcg(&Hb[m], __dadd_rn(__ldcg(&Hb[m]), __dmul_rn(delta, xa)));
                }
            }
        }
        __threadfence();
        __syncthreads();  // every thread has read W / H and written H before W and the flag publish
        if (tid == 0) {
            if (delta != 0.0 && A.flags) A.flags[a] = A.flags[b] = 7;
            A.absdelta[p] = fabs(w - wcur);
            if (delta != 0.0 || w == 0.0) hash_set(A.W, key, w, A.Wcnt);
            __threadfence();
            atomicExch(&A.done[p], 1);
        }
    }
    if (tid == 0) {
        if (evals) atomicAdd((unsigned long long*)&A.counters[C_EVALS], (unsigned long long)evals);
        if (warns) atomicAdd((unsigned long long*)&A.counters[C_WARN], (unsigned long long)warns);
    }
}

// ---------------------------------------------------------------- bulk set_edges
// set_edges on an empty coupling table with distinct pairs (e.g. a state loaded into a
// fresh context): the result of the reference's sequential set_edge calls
// (inc/sparse_weights.hpp:54-85) is, per node i, H_i = sum over its incident pairs in list
// order of w x_other — each H_i[m] sees exactly the sequential additions, in order — so
// one pass per node over its incidence list reproduces it bitwise, without the
// dependency-ordered kernel.
__global__ void inc_keys_kernel(const int32_t* __restrict__ ci, const int32_t* __restrict__ cj, uint64_t n, int ib,
                                uint64_t* __restrict__ keys, uint64_t* __restrict__ canon) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const uint64_t a = (uint64_t)ci[e], b = (uint64_t)cj[e];
    keys[2 * e] = (a << 32) | e;
    keys[2 * e + 1] = (b << 32) | e;
    canon[e] = a < b ? (a << ib) | b : (b << ib) | a;
}
__global__ void dup_flag_kernel(const uint64_t* __restrict__ sorted, uint64_t n, int* __restrict__ dup) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e > 0 && e < n && sorted[e] == sorted[e - 1]) *dup = 1;
}
__global__ void inc_start_kernel(const uint64_t* __restrict__ sorted, uint64_t ne, uint64_t* __restrict__ start,
                                 int nnodes) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ne) return;
    const uint64_t node = sorted[t] >> 32;
    const uint64_t prev = t ? (sorted[t - 1] >> 32) : (uint64_t)-1;
    if (node != prev) start[node] = t;
    if (t == ne - 1) start[nnodes] = ne;  // sentinel read only through the next-start search
}
__global__ void bulk_sums_kernel(int kind, const uint32_t* __restrict__ Xb, const double* __restrict__ Xd, int M,
                                 int Mp, int Mw, const uint64_t* __restrict__ sorted, uint64_t ne,
                                 const uint64_t* __restrict__ start, const int32_t* __restrict__ ci,
                                 const int32_t* __restrict__ cj, const double* __restrict__ w,
                                 double* __restrict__ H) {
    const int i = blockIdx.x;
    const uint64_t s0 = start[i];
    if (s0 == ~0ull) return;  // no incident pair
    double* Hi = H + (size_t)i * Mp;
    for (int m = threadIdx.x; m < M; m += blockDim.x) {
        double acc = Hi[m];
        for (uint64_t t = s0; t < ne && (sorted[t] >> 32) == (uint64_t)i; ++t) {
            const uint64_t e = sorted[t] & 0xffffffffu;
            const int o = ci[e] == i ? cj[e] : ci[e];
            const double x = kind == ISING ? xsign(Xb[(size_t)o * Mw + (m >> 5)], m & 31) : Xd[(size_t)o * Mp + m];
            acc = kind == ISING ? acc + w[e] * x : __dadd_rn(acc, __dmul_rn(w[e], x));
        }
        Hi[m] = acc;
    }
}
__global__ void bulk_insert_kernel(HashView W, const int32_t* __restrict__ ci, const int32_t* __restrict__ cj,
                                   const double* __restrict__ w, uint64_t n, unsigned long long* __restrict__ cnt) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n || w[e] == 0.0) return;  // absent and zero: nothing stored
    const uint64_t key = pair_key(ci[e], cj[e]);
    uint64_t s = slot_of(key, W.mask);
    for (;;) {
        const unsigned long long prev =
            atomicCAS((unsigned long long*)&W.keys[s], (unsigned long long)kEmptyKey, (unsigned long long)key);
        if (prev == kEmptyKey) {
            W.vals[s] = w[e];
            atomicAdd(&cnt[0], 1ull);
            atomicAdd(&cnt[1], 1ull);
            return;
        }
        s = (s + 1) & W.mask;
    }
}

bool set_edges_bulk(Context& c, const int32_t* ci, const int32_t* cj, uint64_t n, const double* w) {
    if (n == 0 || n >= (1ull << 31)) return false;
    uint64_t cnt[2];
    NRG_CUDA(cudaMemcpyAsync(cnt, c.Wcount.p, 16, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (cnt[1] != 0) return false;  // the table holds (or held) couplings: sequential path
    int ib = 1;
    while (ib < 31 && (1ll << ib) < (long long)c.n) ++ib;
    DevBuf kb, k2b, cb, c2b, sb, db, tb;
    const uint64_t ne = 2 * n;
    uint64_t* keys = kb.as<uint64_t>(ne);
    uint64_t* keys2 = k2b.as<uint64_t>(ne);
    uint64_t* canon = cb.as<uint64_t>(n);
    uint64_t* canon2 = c2b.as<uint64_t>(n);
    int* dup = db.as<int>(1);
    NRG_CUDA(cudaMemsetAsync(dup, 0, 4, c.stream));
    inc_keys_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(ci, cj, n, ib, keys, canon);
    size_t b1 = 0, b2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b1, canon, canon2, (int64_t)n, 0, 2 * ib, c.stream);
    cub::DeviceRadixSort::SortKeys(nullptr, b2, keys, keys2, (int64_t)ne, 0, 32 + ib, c.stream);
    void* tmp = tb.ensure(std::max(b1, b2));
    cub::DeviceRadixSort::SortKeys(tmp, b1, canon, canon2, (int64_t)n, 0, 2 * ib, c.stream);
    dup_flag_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(canon2, n, dup);
    NRG_LAUNCH_CHECK();
    int hdup = 0;
    hdup = c.read_scalar(dup);
    if (hdup) return false;  // a pair listed twice: its second Delta depends on the first
    c.tic();
    w_reserve(c, n);
    cub::DeviceRadixSort::SortKeys(tmp, b2, keys, keys2, (int64_t)ne, 0, 32 + ib, c.stream);
    uint64_t* start = sb.as<uint64_t>((uint64_t)c.n + 1);
    NRG_CUDA(cudaMemsetAsync(start, 0xff, ((uint64_t)c.n + 1) * 8, c.stream));
    inc_start_kernel<<<(unsigned)ceil_div(ne, 256), 256, 0, c.stream>>>(keys2, ne, start, c.n);
    bulk_sums_kernel<<<(unsigned)c.n, 256, 0, c.stream>>>(c.kind, c.dXb(), c.dXd(), c.M, c.Mp, c.Mw, keys2, ne, start,
                                                         ci, cj, w, c.dH());
    bulk_insert_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(
        c.Wview(), ci, cj, w, n, static_cast<unsigned long long*>(c.Wcount.p));
    NRG_LAUNCH_CHECK();
    c.state_version++;
    c.toc(P_UPDATE);
    return true;
}

__global__ void __launch_bounds__(1024) sum_fixed_kernel(const double* __restrict__ v, uint64_t n,
                                                         double* __restrict__ out) {
    __shared__ double sh[32];
    double a = 0.0;
    // contiguous slices per thread, then a fixed tree: deterministic
    const uint64_t per = (n + 1023) / 1024;
    const uint64_t lo = threadIdx.x * per, hi = min(n, lo + per);
    for (uint64_t t = lo; t < hi; ++t) a += v[t];
    a = warp_sum(a);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x < 32) {
        double r = sh[threadIdx.x];
        r = warp_sum(r);
        if (threadIdx.x == 0) *out = r;
    }
}

template <int kUpdNT>
static int update_grid(Context& c, size_t smem) {
    int sms = 0, per = 0;
    NRG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
    if (smem > 48 * 1024)
        NRG_CUDA(cudaFuncSetAttribute(update_kernel<kUpdNT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    NRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, update_kernel<kUpdNT>, kUpdNT, smem));
    if (per < 1) fail(100, "update kernel does not fit on an SM");
    return sms * per;  // persistent grid: every CTA resident (the dependency waits need it)
}

// The dependency-ordered kernel over candidates [0, n) of (ci, cj): |w - w_cur| per
// pair into absdelta.
// disjoint: the caller guarantees the pairs share no node (a tie-tail round's applied
// set), so no pair waits on another: every dependency is empty without the sort
static void ordered_run(Context& c, const int32_t* ci, const int32_t* cj, uint64_t n, const double* assign,
                        double* absdelta, bool level_order = true, bool disjoint = false) {
    if (n == 0) return;
    DevBuf kb, vb, k2b, v2b, depb, doneb, tb, tmpb;
    int32_t* dep = depb.as<int32_t>(2 * n);
    int* done = doneb.as<int>(n);
    unsigned long long* ticket = tb.as<unsigned long long>(1);
    if (disjoint) {
        NRG_CUDA(cudaMemsetAsync(dep, 0xff, 8 * n, c.stream));  // -1: no predecessor
    } else {
        uint64_t* keys = kb.as<uint64_t>(2 * n);
        uint32_t* vals = vb.as<uint32_t>(2 * n);
        uint64_t* keys2 = k2b.as<uint64_t>(2 * n);
        uint32_t* vals2 = v2b.as<uint32_t>(2 * n);
        dep_keys_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(ci, cj, n, keys, vals);
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, keys2, vals, vals2, (int64_t)(2 * n), 0, 64, c.stream);
        void* tmp = tmpb.ensure(bytes);
        cub::DeviceRadixSort::SortPairs(tmp, bytes, keys, keys2, vals, vals2, (int64_t)(2 * n), 0, 64, c.stream);
        dep_link_kernel<<<(unsigned)ceil_div(2 * n, 256), 256, 0, c.stream>>>(keys2, vals2, 2 * n, dep);
    }
    NRG_CUDA(cudaMemsetAsync(done, 0, n * 4, c.stream));
    NRG_CUDA(cudaMemsetAsync(ticket, 0, 8, c.stream));
    NRG_LAUNCH_CHECK();
    // Tickets in dependency-level order (longest predecessor chain, then list index):
    // a pair's predecessors sit at strictly lower levels, so they hold earlier tickets
    // (no deadlock) and a whole wavefront is in flight at once.  In list order the
    // resident CTAs only ever see a window of consecutive pairs, which for lists like
    // reconstruct_cd's row-major all-pairs share one node and run one at a time.
    DevBuf ordb;
    uint32_t* order = nullptr;
    size_t nlevels = 0;
    if (n >= 4096 && level_order && !disjoint && !NRG_ENV_ON("NRG_LIST_ORDER_TICKETS")) {
        int32_t* hdep = c.hp_dep.as<int32_t>(2 * n);
        NRG_CUDA(cudaMemcpyAsync(hdep, dep, 8 * n, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        std::vector<uint32_t> lev(n), cnt(1, 0);
        for (uint64_t p = 0; p < n; ++p) {
            uint32_t l = 0;
            if (hdep[2 * p] >= 0) l = std::max(l, lev[hdep[2 * p]] + 1);
            if (hdep[2 * p + 1] >= 0) l = std::max(l, lev[hdep[2 * p + 1]] + 1);
            lev[p] = l;
            if (l >= cnt.size()) cnt.resize(l + 1, 0);
            ++cnt[l];
        }
        nlevels = cnt.size();
        std::vector<uint32_t> start(cnt.size(), 0);
        uint32_t* hord = c.hp_ord.as<uint32_t>(n);
        for (size_t l = 1; l < cnt.size(); ++l) start[l] = start[l - 1] + cnt[l - 1];
        for (uint64_t p = 0; p < n; ++p) hord[start[lev[p]]++] = (uint32_t)p;
        if (NRG_ENV_ON("NRG_DEBUG_UPD")) {
            uint32_t mx = 0;
            for (uint32_t v : cnt) mx = std::max(mx, v);
            fprintf(stderr, "ordered_run: n=%llu levels=%zu widest=%u\n", (unsigned long long)n, cnt.size(), mx);
        }
        order = ordb.as<uint32_t>(n);
        // pinned and stream-ordered: the next planning step syncs before hord is rewritten
        NRG_CUDA(cudaMemcpyAsync(order, hord, 4 * n, cudaMemcpyHostToDevice, c.stream));
    }
    UpdateArgs A;
    A.kind = c.kind;
    A.Xb = c.dXb();
    A.Xd = c.dXd();
    A.H = c.dH();
    A.theta = c.dtheta();
    A.M = c.M;
    A.Mp = c.Mp;
    A.Mw = c.Mw;
    A.W = c.Wview();
    A.Wcnt = static_cast<unsigned long long*>(c.Wcount.p);
    A.ci = ci;
    A.cj = cj;
    A.assign = assign;
    A.dep = dep;
    A.order = order;
    A.n = n;
    A.lambda = c.lambda;
    A.done = done;
    A.ticket = ticket;
    A.absdelta = absdelta;
    A.counters = c.dcounters();
    c.sync_flags();
    A.flags = c.dflags();
    const size_t smem = (size_t)2 * c.Mp * sizeof(double);
    A.stage = (c.kind == ISING && smem <= 160 * 1024) ? 1 : 0;
    const size_t smem_use = A.stage ? smem : 0;
    // wide, shallow dependency structures (the steady-state lists: ~50k updates in ~60
    // levels) are bound by how many updates are in flight: 128-thread CTAs (twice as
    // many); deep chains (first sweeps, reconstruct_cd) by per-update latency: 256
    static const int nt_env = getenv("NRG_UPD_NT") ? atoi(getenv("NRG_UPD_NT")) : 0;
    const int nt = nt_env ? nt_env
                          : ((nlevels > 0 && n >= 256 * nlevels) || (!level_order && n >= 4096) ? 128 : 256);
    int grid = (int)std::min<uint64_t>(nt == 128 ? update_grid<128>(c, smem_use) : update_grid<256>(c, smem_use), n);
    const bool dbg = NRG_ENV_ON("NRG_DEBUG_UPDATES");
    if (dbg && NRG_ENV_ON("NRG_DEBUG_SERIAL")) grid = 1;
    if (nt == 128)
        update_kernel<128><<<grid, 128, smem_use, c.stream>>>(A);
    else
        update_kernel<256><<<grid, 256, smem_use, c.stream>>>(A);
    NRG_LAUNCH_CHECK();
    if (dbg) {
        std::vector<int32_t> hd(2 * n), hi(n), hj(n);
        std::vector<int> hdone(n);
        NRG_CUDA(cudaMemcpyAsync(hd.data(), dep, 8 * n, cudaMemcpyDeviceToHost, c.stream));
        NRG_CUDA(cudaMemcpyAsync(hi.data(), ci, 4 * n, cudaMemcpyDeviceToHost, c.stream));
        NRG_CUDA(cudaMemcpyAsync(hj.data(), cj, 4 * n, cudaMemcpyDeviceToHost, c.stream));
        NRG_CUDA(cudaMemcpyAsync(hdone.data(), done, 4 * n, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        std::vector<int32_t> last(c.n, -1);
        int bad = 0, ndone = 0;
        for (uint64_t p = 0; p < n; ++p) {
            const int e0 = last[hi[p]], e1 = last[hj[p]];
            if (hd[2 * p] != e0 || hd[2 * p + 1] != e1) {
                if (bad < 10)
                    fprintf(stderr, "dep mismatch p=%llu (%d,%d): got %d %d want %d %d\n", (unsigned long long)p, hi[p],
                            hj[p], hd[2 * p], hd[2 * p + 1], e0, e1);
                ++bad;
            }
            last[hi[p]] = last[hj[p]] = (int32_t)p;
            ndone += hdone[p];
        }
        fprintf(stderr, "apply_updates debug: n=%llu grid=%d dep mismatches=%d done=%d\n", (unsigned long long)n, grid,
                bad, ndone);
    }
}

__global__ void tail_start_kernel(const double* __restrict__ dist, uint64_t n, unsigned long long* k) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p + 1 < n && dist[p] != dist[n - 1]) atomicMax(k, (unsigned long long)(p + 1));
}

// changed[p - lo] = 1 when the re-evaluated coupling of pair p differs from the current one
// tail[0] += changed entries, tail[1] = min(first changed, relative to lo) (set to the
// tail length by the caller)
__global__ void change_flags_kernel(const int32_t* __restrict__ ci, const int32_t* __restrict__ cj, uint64_t lo,
                                    uint64_t n, const double* __restrict__ w, HashView W,
                                    uint8_t* __restrict__ changed, unsigned long long* __restrict__ tail) {
    const uint64_t p = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool ch = false;
    if (p < n) {
        const int i = ci[p], j = cj[p];
        const double wcur = hash_get(W, pair_key(min(i, j), max(i, j)), 0.0);
        ch = w[p - lo] != wcur;
        changed[p - lo] = ch ? 1 : 0;
    }
    if (!tail) return;
    const unsigned b = __ballot_sync(0xffffffffu, ch);
    if ((threadIdx.x & 31) == 0 && b) {
        atomicAdd(&tail[0], (unsigned long long)__popc(b));
        atomicMin(&tail[1], (unsigned long long)(p - lo + (__ffs(b) - 1)));
    }
}

__global__ void tail_init_kernel(unsigned long long* tail, uint64_t m) {
    tail[0] = 0;
    tail[1] = m;
    tail[2] = 0;
    tail[3] = 0;
}

// One tie-tail round's walk (the sequential semantics of apply_updates, on the device):
// from the first changing entry, every changing entry is applied until the first entry
// (changing or not) that touches a node an applied entry modified; that entry starts the
// next round.  One CTA, 1024 entries per step: conflicts with earlier steps through a
// per-node stamp, within the step against the step's changing entries (at most the
// round's change budget, kTailRounds).  tail[2] = applied count, tail[3] = stop (absolute).
__global__ void __launch_bounds__(1024) tail_walk_kernel(const int32_t* __restrict__ ci,
                                                          const int32_t* __restrict__ cj, uint64_t lo, uint64_t n,
                                                          const uint8_t* __restrict__ changed,
                                                          uint32_t* __restrict__ mod, uint32_t stamp,
                                                          uint32_t* __restrict__ apply,
                                                          unsigned long long* __restrict__ tail, uint64_t budget) {
    __shared__ int s_a[1024], s_b[1024], s_pos[1024];
    __shared__ int s_nch, s_stop;
    const int tid = threadIdx.x;
    uint64_t na = 0;
    if (tail[0] > budget) return;  // more changes than rounds left: the host orders the rest
    const uint64_t first = tail[1];
    for (uint64_t base = lo + first; base < n; base += 1024) {
        const uint64_t p = base + tid;
        const bool valid = p < n;
        const int a = valid ? ci[p] : -1, b = valid ? cj[p] : -1;
        const bool ch = valid && changed[p - lo];
        bool conf = valid && (mod[a] == stamp || mod[b] == stamp);
        if (tid == 0) {
            s_nch = 0;
            s_stop = 1024;
        }
        __syncthreads();
        if (ch) {
            const int q = atomicAdd(&s_nch, 1);
            s_a[q] = a;
            s_b[q] = b;
            s_pos[q] = tid;
        }
        __syncthreads();
        const int nch = s_nch;
        for (int q = 0; q < nch; ++q)
            if (s_pos[q] < tid && (a == s_a[q] || a == s_b[q] || b == s_a[q] || b == s_b[q])) conf = true;
        if (conf) atomicMin(&s_stop, tid);
        __syncthreads();
        const int stop = s_stop;
        // applied: the changing entries before the stop, in list order
        int before = 0;
        for (int q = 0; q < nch; ++q) before += s_pos[q] < stop && s_pos[q] < tid ? 1 : 0;
        if (ch && tid < stop) {
            apply[na + before] = (uint32_t)p;
            mod[a] = stamp;
            mod[b] = stamp;
        }
        for (int q = 0; q < nch; ++q) na += s_pos[q] < stop ? 1 : 0;
        __syncthreads();  // stamps visible to the next step
        if (stop < 1024) {
            if (tid == 0) {
                tail[2] = na;
                tail[3] = base + (uint64_t)stop;
            }
            return;
        }
    }
    if (tid == 0) {
        tail[2] = na;
        tail[3] = n;
    }
}

__global__ void gather_pairs_kernel(const int32_t* __restrict__ ci, const int32_t* __restrict__ cj,
                                    const uint32_t* __restrict__ idx, uint32_t m, int32_t* __restrict__ oi,
                                    int32_t* __restrict__ oj) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    oi[t] = ci[idx[t]];
    oj[t] = cj[idx[t]];
}

__global__ void scatter_delta_kernel(const double* __restrict__ d, const uint32_t* __restrict__ idx, uint32_t m,
                                     double* __restrict__ absdelta) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m) absdelta[idx[t]] = d[t];
}

constexpr uint64_t kTailMin = 256;  // shorter tie tails go through the ordered kernel
constexpr int kTailRounds = 64;     // rounds before the rest of a tail is ordered instead

// detail::apply_edge_updates, sequential semantics.  A FindBest list sorted by
// distance ends in a block of exact ties -- at a converging state mostly the
// zero-gain (kink) pairs, listed by (i, j), so a few low-id nodes sit in tens of
// thousands of them and the dependency chain through those nodes is as long as the
// block.  Such a tail is resolved in rounds instead: every remaining pair is
// re-evaluated in parallel against the current state, then walked in list order
// keeping the set of nodes the round modifies.  A pair touching none of them sees
// exactly the state the sequential loop would give it, so its evaluation stands:
// no-ops are done, changing pairs are applied (node-disjoint, so one ordered launch
// applies them all exactly).  The first pair touching a modified node ends the round
// and starts the next.  The prefix before the tail, and a tail with more changes
// than rounds left, go through the dependency-ordered kernel.  `dist` (device,
// optional) only locates the tail; results never depend on it.
// Precision note: a round decides "changes / does not change" with score_entries
// (warp-scope reductions), while the applied pairs are re-optimised by update_kernel
// (block-scope reductions).  Kink decisions (w_cur = 0 staying 0) are exact on both
// paths (integer screen + error band), but for an existing coupling the two
// reductions may disagree in the last ulp of w*, so the tail matches the sequential
// loop to rounding (|dw| ~ 1e-15), not bitwise; tests/test_gpu_updates.py checks it
// against the ordered path at 1e-9.
double apply_updates(Context& c, const int32_t* ci, const int32_t* cj, uint64_t n, const double* assign,
                     const double* dist, bool fb_sorted) {
    if (n == 0) return 0.0;
    if (n >= (1ull << 31)) fail(22, "apply_updates: too many candidates");
    c.tic();
    w_reserve(c, n);
    DevBuf adb, sb, kb, wb, fb, ib, pib, pjb, ddb;
    double* absdelta = adb.as<double>(n);
    NRG_CUDA(cudaMemsetAsync(absdelta, 0, n * 8, c.stream));
    uint64_t k = n;
    if (!assign && dist && n >= kTailMin && !getenv("NRG_ORDERED_ONLY")) {
        unsigned long long* dk = kb.as<unsigned long long>(1);
        NRG_CUDA(cudaMemsetAsync(dk, 0, 8, c.stream));
        tail_start_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(dist, n, dk);
        NRG_LAUNCH_CHECK();
        unsigned long long hk = 0;
        hk = c.read_scalar(dk);
        if (n - hk >= kTailMin) k = hk;
    }
    // a FindBest list (sorted by distance, flagged by gcd_iteration) is already a
    // spread-out order: consecutive candidates rarely share a node, so list-order tickets
    // keep the wavefront busy and the host-side level ordering (a round trip) costs more
    // than it gains; every other list (reconstruct_cd's row-major all-pairs, lists passed
    // to nrg_apply_updates / edited by a candidate hook, set_edges) takes level order
    static const bool fb_level = NRG_ENV_ON("NRG_FB_LEVEL_ORDER");
    ordered_run(c, ci, cj, k, assign, absdelta, !fb_sorted || fb_level);
    uint64_t start = k;
    if (start < n) {
        // the round's walk runs on the device (tail_walk_kernel: one readback per round);
        // NRG_HOST_TAIL_WALK=1 walks the change flags on the host instead (A/B, same result)
        static const bool host_walk = NRG_ENV_ON("NRG_HOST_TAIL_WALK");
        const uint64_t nt = n - start;
        int32_t* hi = host_walk ? c.hp_i.as<int32_t>(nt) : nullptr;
        int32_t* hj = host_walk ? c.hp_j.as<int32_t>(nt) : nullptr;
        uint8_t* hch = host_walk ? c.hp_ch.as<uint8_t>(nt) : nullptr;
        if (host_walk) {
            NRG_CUDA(cudaMemcpyAsync(hi, ci + start, nt * 4, cudaMemcpyDeviceToHost, c.stream));
            NRG_CUDA(cudaMemcpyAsync(hj, cj + start, nt * 4, cudaMemcpyDeviceToHost, c.stream));
        }
        unsigned long long* tail = c.tail_cnt.as<unsigned long long>(4);
        unsigned long long* htail = c.hp_tail.as<unsigned long long>(4);
        uint32_t* mod_dev = nullptr;
        if (!host_walk) {
            if (!c.tail_mod.p) {
                mod_dev = c.tail_mod.as<uint32_t>((uint64_t)c.n);
                NRG_CUDA(cudaMemsetAsync(mod_dev, 0, (size_t)c.n * 4, c.stream));
                c.tail_stamp = 0;
            }
            mod_dev = static_cast<uint32_t*>(c.tail_mod.p);
        }
        uint32_t* apply_dev = host_walk ? nullptr : c.tail_apply.as<uint32_t>(nt);
        std::vector<uint8_t> mod(c.n, 0);
        std::vector<int32_t> touched;
        std::vector<uint32_t> apply;
        DevBuf rowsb;
        int32_t* rows_dev = nullptr;
        uint64_t n_rows = 0;
        for (int round = 0; start < n; ++round) {
            if (round == kTailRounds) {
                ordered_run(c, ci + start, cj + start, n - start, nullptr, absdelta + start);
                break;
            }
            c.bump_flagged();  // the evaluation snapshot must include every update so far
            c.toc(P_UPDATE);   // snapshot refreshes time themselves (P_SNAP)
            // the rows the updates so far changed (their staleness flags): after a round, the
            // endpoints of the pairs it applied; before the first, whatever the ordered part hit
            if (round > 0 && c.flags_version == c.state_version)
                snapshot_rows(c, rows_dev, n_rows);
            else
                ensure_snapshot(c);
            const uint64_t m = n - start;
            double* w = wb.as<double>(m);
            ScoreOut out;
            out.w = w;
            score_entries(c, EXACT, ci + start, cj + start, m, out);  // times itself as P_SCORE
            c.tic();
            uint8_t* ch = fb.as<uint8_t>(m);
            if (!host_walk) {
                tail_init_kernel<<<1, 1, 0, c.stream>>>(tail, m);
                change_flags_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, c.stream>>>(ci, cj, start, n, w, c.Wview(),
                                                                                      ch, tail);
                tail_walk_kernel<<<1, 1024, 0, c.stream>>>(ci, cj, start, n, ch, mod_dev, ++c.tail_stamp, apply_dev,
                                                           tail, (uint64_t)(kTailRounds - round));
                NRG_LAUNCH_CHECK_N(3);
                NRG_CUDA(cudaMemcpyAsync(htail, tail, 32, cudaMemcpyDeviceToHost, c.stream));
                c.sync();
                c.tail_rounds++;
                const uint64_t nch = htail[0], na = htail[2], stop = htail[3];
                if (NRG_ENV_ON("NRG_DEBUG_TAIL"))
                    fprintf(stderr, "tail round %d: start=%llu m=%llu changed=%llu applied=%llu stop=%llu\n", round,
                            (unsigned long long)start, (unsigned long long)m, (unsigned long long)nch,
                            (unsigned long long)na, (unsigned long long)stop);
                if (nch > (uint64_t)(kTailRounds - round)) {
                    ordered_run(c, ci + start, cj + start, m, nullptr, absdelta + start);
                    break;
                }
                if (na) {
                    int32_t* pi = pib.as<int32_t>(na);
                    int32_t* pj = pjb.as<int32_t>(na);
                    double* dd = ddb.as<double>(na);
                    gather_pairs_kernel<<<ceil_div(na, 256), 256, 0, c.stream>>>(ci, cj, apply_dev, (uint32_t)na, pi,
                                                                                pj);
                    NRG_LAUNCH_CHECK();
                    ordered_run(c, pi, pj, na, nullptr, dd, true, /*disjoint=*/true);
                    scatter_delta_kernel<<<ceil_div(na, 256), 256, 0, c.stream>>>(dd, apply_dev, (uint32_t)na,
                                                                                 absdelta);
                    NRG_LAUNCH_CHECK();
                    rows_dev = rowsb.as<int32_t>(2 * (size_t)na);
                    NRG_CUDA(cudaMemcpyAsync(rows_dev, pi, na * 4, cudaMemcpyDeviceToDevice, c.stream));
                    NRG_CUDA(cudaMemcpyAsync(rows_dev + na, pj, na * 4, cudaMemcpyDeviceToDevice, c.stream));
                    n_rows = 2 * na;
                } else {
                    n_rows = 0;
                }
                start = stop;
                continue;
            }
            change_flags_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, c.stream>>>(ci, cj, start, n, w, c.Wview(), ch,
                                                                                  nullptr);
            NRG_LAUNCH_CHECK();
            NRG_CUDA(cudaMemcpyAsync(hch, ch, m, cudaMemcpyDeviceToHost, c.stream));
            c.sync();
            c.tail_rounds++;
            uint64_t nch = 0, first = m;
            for (uint64_t q = 0; q < m; ++q)
                if (hch[q]) {
                    if (!nch) first = q;
                    ++nch;
                }
            if (nch > (uint64_t)(kTailRounds - round)) {
                // more changes than rounds left (a tail still far from converged, e.g. the
                // first sweep): the ordered kernel is the faster exact path
                ordered_run(c, ci + start, cj + start, m, nullptr, absdelta + start);
                break;
            }
            apply.clear();
            // nothing is modified before the first changing pair: the scan starts there
            // (no change at all: every remaining result stands, the tail is done)
            uint64_t p = start + first;
            for (; p < n; ++p) {
                const uint64_t q = p - k;
                const int a = hi[q], b = hj[q];
                if (mod[a] || mod[b]) break;
                if (hch[p - start]) {
                    apply.push_back((uint32_t)p);
                    mod[a] = mod[b] = 1;
                    touched.push_back(a);
                    touched.push_back(b);
                }
            }
            if (NRG_ENV_ON("NRG_DEBUG_TAIL")) {
                fprintf(stderr, "tail round %d: start=%llu m=%llu changed=%llu applied=%zu stop=%llu\n", round,
                        (unsigned long long)start, (unsigned long long)m, (unsigned long long)nch, apply.size(),
                        (unsigned long long)p);
            }
            for (int32_t v : touched) mod[v] = 0;
            touched.clear();
            if (!apply.empty()) {
                const uint32_t na = (uint32_t)apply.size();
                uint32_t* di = ib.as<uint32_t>(na);
                int32_t* pi = pib.as<int32_t>(na);
                int32_t* pj = pjb.as<int32_t>(na);
                double* dd = ddb.as<double>(na);
                uint32_t* hap = c.hp_apply.as<uint32_t>(na);  // pinned: the copy is a DMA, not a staged one
                std::copy(apply.begin(), apply.end(), hap);
                NRG_CUDA(cudaMemcpyAsync(di, hap, na * 4, cudaMemcpyHostToDevice, c.stream));
                gather_pairs_kernel<<<ceil_div(na, 256), 256, 0, c.stream>>>(ci, cj, di, na, pi, pj);
                NRG_LAUNCH_CHECK();
                ordered_run(c, pi, pj, na, nullptr, dd);
                scatter_delta_kernel<<<ceil_div(na, 256), 256, 0, c.stream>>>(dd, di, na, absdelta);
                NRG_LAUNCH_CHECK();
                rows_dev = rowsb.as<int32_t>(2 * (size_t)na);
                NRG_CUDA(cudaMemcpyAsync(rows_dev, pi, na * 4, cudaMemcpyDeviceToDevice, c.stream));
                NRG_CUDA(cudaMemcpyAsync(rows_dev + na, pj, na * 4, cudaMemcpyDeviceToDevice, c.stream));
                n_rows = 2 * (uint64_t)na;
                c.sync();  // `apply` is reused next round
            } else {
                n_rows = 0;
            }
            start = p;
        }
    }
    double* sum = sb.as<double>(1);
    sum_fixed_kernel<<<1, 1024, 0, c.stream>>>(absdelta, n, sum);
    NRG_LAUNCH_CHECK();
    double h = 0.0;
    h = c.read_scalar(sum);
    c.toc(P_UPDATE);
    c.bump_flagged();
    return h;
}

// all pairs i < j of 0..n-1 in row-major order (reconstruct_cd's list,
// inc/reconstruct.hpp:190-192), with a constant tie distance
__global__ void all_pairs_kernel(uint64_t n, int32_t* __restrict__ ci, int32_t* __restrict__ cj,
                                 double* __restrict__ tie) {
    const uint64_t i = blockIdx.x;
    if (i >= n) return;
    const uint64_t off = i * (2 * n - i - 1) / 2;
    for (uint64_t j = i + 1 + threadIdx.x; j < n; j += blockDim.x) {
        ci[off + j - i - 1] = (int32_t)i;
        cj[off + j - i - 1] = (int32_t)j;
        tie[off + j - i - 1] = 0.0;
    }
}
void all_pairs_list(Context& c, int32_t* ci, int32_t* cj, double* tie) {
    all_pairs_kernel<<<(unsigned)c.n, 256, 0, c.stream>>>((uint64_t)c.n, ci, cj, tie);
    NRG_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- theta pass
__global__ void __launch_bounds__(256) theta_kernel(int kind, const uint32_t* __restrict__ Xb,
                                                    const double* __restrict__ Xd, const double* __restrict__ H,
                                                    const double* __restrict__ theta_in, int n, int M, int Mp,
                                                    int Mw, double* __restrict__ theta_out, uint64_t* counters,
                                                    int i0 = 0, uint8_t* __restrict__ flags = nullptr) {
    const int lane = threadIdx.x & 31;
    const int i = i0 + (int)(((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (i >= n) return;  // n: the end of this launch's node range
    if (flags) {
        // theta_i maximises a function of row H_i only: a row no update touched since its
        // theta was optimised keeps it (the reference re-runs its search from the optimum)
        if (!(flags[i] & 1)) {
            if (lane == 0) theta_out[i] = theta_in[i];
            return;
        }
        __syncwarp();
        if (lane == 0) flags[i] = 6;  // theta current; snapshot row and objective term stale
    }
    if (M == 0) {
        if (lane == 0) theta_out[i] = theta_in[i];
        return;
    }
    const double* h = H + (size_t)i * Mp;
    if (kind == ISING) {
        // f'(th) = sum x - tanh(s + th), f'' = -sum sech^2(s + th) < 0
        double sx = 0.0;
        for (int k = 0; k * 32 < M; ++k) {
            const int m = lane + 32 * k;
            if (m < M) sx += xsign(Xb[(size_t)i * Mw + k], lane);
        }
        sx = warp_sum(sx);
        auto deriv = [&](double th, double& d2) {
            double g = 0.0, gg = 0.0;
            for (int m0 = lane; m0 < M; m0 += 128) {  // four loads in flight, same sum order
                double hv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) hv[u] = m0 + 32 * u < M ? h[m0 + 32 * u] : 0.0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (m0 + 32 * u < M) {
                        const double t = tanh(hv[u] + th);
                        g += t;
                        gg += 1.0 - t * t;
                    }
                }
            }
            g = warp_sum(g);
            gg = warp_sum(gg);
            d2 = -gg;
            return sx - g;
        };
        // Safeguarded Newton on the concave objective over [-20, 20] (the reference's
        // golden_max bracket, inc/model.hpp:222-241), warm-started from the current theta:
        // between sweeps theta moves little, so two or three passes reach the root.
        // Near the bracket ends fp64 tanh saturates (f' can be exactly 0 on a flat
        // stretch), so there the from-scratch procedure decides: boundary optima (f' of
        // one sign over the whole bracket) are returned exactly, as golden_max does.
        double d2;
        int passes = 0;
        double res = 0.0;
        {
            double lo = -20.0, hi = 20.0;
            double th = fmin(19.0, fmax(-19.0, theta_in[i]));
            if (!isfinite(th)) th = 0.0;
            for (int it = 0; it < 100; ++it) {
                const double g = deriv(th, d2);
                ++passes;
                if (g > 0.0) lo = th; else if (g < 0.0) hi = th; else { res = th; break; }
                double tn = th - g / d2;
                if (!(tn > lo && tn < hi) || !isfinite(tn)) tn = 0.5 * (lo + hi);
                const bool done = fabs(tn - th) <= 1e-13 * fmax(1.0, fabs(tn)) || hi - lo <= 1e-14;
                th = tn;
                res = th;
                if (done || fabs(th) > 15.0) break;
            }
        }
        if (fabs(res) > 15.0) {
            const double ghi = deriv(20.0, d2);
            passes += 2;
            if (ghi >= 0.0) {
                res = 20.0;
            } else {
                const double glo = deriv(-20.0, d2);
                if (glo <= 0.0) {
                    res = -20.0;
                } else {
                    double lo = -20.0, hi = 20.0, th = 0.0;
                    double g = deriv(th, d2);
                    for (int it = 0; it < 100; ++it) {
                        ++passes;
                        if (g > 0.0) lo = th; else hi = th;
                        double tn = th - g / d2;
                        if (!(tn > lo && tn < hi) || !isfinite(tn)) tn = 0.5 * (lo + hi);
                        const bool done = fabs(tn - th) <= 1e-13 * fmax(1.0, fabs(tn)) || hi - lo <= 1e-14;
                        th = tn;
                        if (done) break;
                        g = deriv(th, d2);
                    }
                    res = th;
                }
            }
        }
        if (lane == 0) {
            theta_out[i] = res;
            atomicAdd((unsigned long long*)&counters[C_EVALS], (unsigned long long)passes);
        }
    } else {
        // -A/(2 th^2) - B th^2/2 - M log th: th^2 = 2A / (M + sqrt(M^2 + 4AB))
        double A = 0.0, B = 0.0;
        for (int m = lane; m < M; m += 32) {
            const double x = Xd[(size_t)i * Mp + m];
            A += x * x;
            B += h[m] * h[m];
        }
        A = warp_sum(A);
        B = warp_sum(B);
        if (lane == 0) {
            double th;
            bool warn = false;
            if (A == 0.0) {
                th = 1e-8;
                warn = true;
            } else {
                const double t2 = 2.0 * A / ((double)M + sqrt((double)M * (double)M + 4.0 * A * B));
                th = sqrt(t2);
                if (th <= 1e-8 * (1.0 + 1e-6)) {
                    th = 1e-8;
                    warn = true;
                }
            }
            theta_out[i] = th;
            atomicAdd((unsigned long long*)&counters[C_EVALS], 1ull);
            if (warn) atomicAdd((unsigned long long*)&counters[C_WARN], 1ull);
        }
    }
}

// theta pass (inc/reconstruct.hpp:129-138).  In a sharded job every rank optimises the
// fields of its node range and the ranges are all-gathered: each theta_i
// is a function of node i's row only, so the result is bitwise the single-GPU pass.
__global__ void flags_outside_kernel(uint8_t* __restrict__ flags, int n, int lo, int hi, uint8_t test, uint8_t set_to,
                                     uint8_t clear) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || (i >= lo && i < hi)) return;
    const uint8_t f = flags[i];
    if (f & test) flags[i] = set_to ? set_to : (uint8_t)(f & ~clear);
}

void theta_pass(Context& c, double* out_only) {
    c.tic();
    double* out = out_only ? out_only : c.s_n.as<double>(c.n);
    uint64_t lo = 0, hi = (uint64_t)c.n;
    if (c.world > 1) shard_range((uint64_t)c.n, c.rank, c.world, lo, hi);
    uint8_t* flags = nullptr;
    if (!out_only) {
        c.sync_flags();
        flags = c.dflags();
    }
    if (hi > lo)
        theta_kernel<<<(unsigned)ceil_div((int64_t)(hi - lo) * 32, 256), 256, 0, c.stream>>>(
            c.kind, c.dXb(), c.dXd(), c.dH(), c.dtheta(), (int)hi, c.M, c.Mp, c.Mw, out, c.dcounters(), (int)lo, flags);
    NRG_LAUNCH_CHECK();
    if (c.world > 1) {
        std::vector<size_t> bytes(c.world);
        for (int r = 0; r < c.world; ++r) {
            uint64_t l, h;
            shard_range((uint64_t)c.n, r, c.world, l, h);
            bytes[r] = (h - l) * 8;
        }
        static_cast<Comm*>(c.comm)->allgatherv(out + lo, out, bytes, c.stream);
        if (flags) {  // the other ranks' rows: the same flag transition their owners made
            flags_outside_kernel<<<(unsigned)ceil_div(c.n, 256), 256, 0, c.stream>>>(flags, c.n, (int)lo, (int)hi, 1, 6, 0);
            NRG_LAUNCH_CHECK();
        }
    }
    if (!out_only) {
        NRG_CUDA(cudaMemcpyAsync(c.theta.p, out, (size_t)c.n * 8, cudaMemcpyDeviceToDevice, c.stream));
        if (flags)
            c.bump_flagged();
        else
            c.state_version++;
    }
    c.toc(P_THETA);
}

}  // namespace nrg
