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
#include <chrono>
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

// Sorting (dist, a, b) keys takes 16 radix passes over 128 bits.  Node ids need only
// ib = bits(N - 1) bits and a level's distances span few of the 64 dkey bits, so the
// keys are packed as ((dkey - dmin) << 2 ib) | (a << ib) | b — the same total order —
// into 64 or 128 bits and sorted over just the occupied bits (about 10 passes).
struct Key128 {
    uint64_t hi, lo;
};
struct Key128Decomposer {
    __host__ __device__ cuda::std::tuple<uint64_t&, uint64_t&> operator()(Key128& k) const { return {k.hi, k.lo}; }
};
static int id_bits(const Context& c) {
    int b = 1;
    while (b < 32 && (1ull << b) < (uint64_t)c.n) ++b;
    return b;
}
__global__ void dkey_range_kernel(const TriKey* __restrict__ in, uint64_t n, unsigned long long* __restrict__ mm) {
    unsigned long long lo = ~0ull, hi = 0ull;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long d = in[e].d;
        lo = d < lo ? d : lo;
        hi = d > hi ? d : hi;
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&mm[0], lo);
        atomicMax(&mm[1], hi);
    }
}
template <class K>
__global__ void pack_trikey_kernel(const TriKey* __restrict__ in, uint64_t n, uint64_t dmin, int ib,
                                   K* __restrict__ out) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const TriKey t = in[e];
    const uint64_t dd = t.d - dmin;
    const uint64_t ids = ((uint64_t)t.a << ib) | t.b;
    if constexpr (sizeof(K) == 8) {
        out[e] = (K)((dd << (2 * ib)) | ids);
    } else {
        Key128 k;
        k.lo = (dd << (2 * ib)) | ids;
        k.hi = dd >> (64 - 2 * ib);
        out[e] = k;
    }
}
template <class K>
__global__ void unpack_trikey_kernel2(const K* __restrict__ in, uint64_t n, uint64_t dmin, int ib,
                                      TriKey* __restrict__ out) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    uint64_t lo, hi;
    if constexpr (sizeof(K) == 8) {
        lo = (uint64_t)in[e];
        hi = 0;
    } else {
        lo = in[e].lo;
        hi = in[e].hi;
    }
    const uint64_t m = (1ull << ib) - 1;
    TriKey t;
    t.b = (uint32_t)(lo & m);
    t.a = (uint32_t)((lo >> ib) & m);
    t.d = dmin + ((lo >> (2 * ib)) | (2 * ib ? hi << (64 - 2 * ib) : 0));
    out[e] = t;
}

static void sort_trikeys(Context& c, TriKey* in, TriKey* out, uint64_t n, DevBuf& tmpb) {
    if (!n) return;
    if (NRG_ENV_ON("NRG_SORT_FULL")) {
        size_t bytes = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, bytes, in, out, (int64_t)n, TriKeyDecomposer{}, c.stream);
        void* tmp = tmpb.ensure(bytes);
        cub::DeviceRadixSort::SortKeys(tmp, bytes, in, out, (int64_t)n, TriKeyDecomposer{}, c.stream);
        NRG_LAUNCH_CHECK();
        return;
    }
    DevBuf mmb, kb;
    unsigned long long* mm = mmb.as<unsigned long long>(2);
    const unsigned long long init[2] = {~0ull, 0ull};
    NRG_CUDA(cudaMemcpyAsync(mm, init, 16, cudaMemcpyHostToDevice, c.stream));
    dkey_range_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 148 * 4), 256, 0, c.stream>>>(in, n, mm);
    NRG_LAUNCH_CHECK();
    unsigned long long h[2];
    NRG_CUDA(cudaMemcpyAsync(h, mm, 16, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    const int ib = id_bits(c);
    const uint64_t span = h[1] - h[0];
    int db = 0;
    while (db < 64 && (span >> db)) ++db;
    const int total = db + 2 * ib;
    const unsigned g = (unsigned)ceil_div(n, 256);
    if (total <= 64) {
        uint64_t* k0 = kb.as<uint64_t>(2 * n);
        uint64_t* k1 = k0 + n;
        pack_trikey_kernel<uint64_t><<<g, 256, 0, c.stream>>>(in, n, h[0], ib, k0);
        size_t bytes = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, bytes, k0, k1, (int64_t)n, 0, total, c.stream);
        void* tmp = tmpb.ensure(bytes);
        cub::DeviceRadixSort::SortKeys(tmp, bytes, k0, k1, (int64_t)n, 0, total, c.stream);
        unpack_trikey_kernel2<uint64_t><<<g, 256, 0, c.stream>>>(k1, n, h[0], ib, out);
    } else {
        Key128* k0 = kb.as<Key128>(2 * n);
        Key128* k1 = k0 + n;
        pack_trikey_kernel<Key128><<<g, 256, 0, c.stream>>>(in, n, h[0], ib, k0);
        size_t bytes = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, bytes, k0, k1, (int64_t)n, Key128Decomposer{}, 0, total, c.stream);
        void* tmp = tmpb.ensure(bytes);
        cub::DeviceRadixSort::SortKeys(tmp, bytes, k0, k1, (int64_t)n, Key128Decomposer{}, 0, total, c.stream);
        unpack_trikey_kernel2<Key128><<<g, 256, 0, c.stream>>>(k1, n, h[0], ib, out);
    }
    NRG_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- radix select
// The K smallest of n distinct (dist, a, b) keys, unsorted, and a threshold T such that
// an input key is among the K smallest iff it is <= T (the reference's nth_element,
// inc/find_best.hpp:114-131: D+ and the S' test need the set and its largest key, not
// an order).  MSD radix select in ONE cooperative launch, without a host round trip:
// a first pass finds the range of the distance keys, so the select runs over the packed
// key ((dkey - dmin) << 2 ib | a << ib | b -- the same order over only the occupied bits,
// ~70 instead of 98 at config 4) in 12-bit digits: per pass every CTA histograms the
// digit of the keys still matching the prefix (a warp whose keys share a digit -- the
// tie block at -base -- adds once), one grid barrier, then every CTA scans the same 4096
// counts and extends the prefix identically.  Once the remaining rank equals the size of
// the prefix group, the whole group is in and the passes stop (T = prefix with the
// unresolved bits set: no input key lies between the group's largest key and T).
__device__ __forceinline__ void sel_grid_sync(unsigned* bar, unsigned nblocks) {
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
            while (*gen == g) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}
constexpr int kSelThreads = 1024;
constexpr int kSelBits = 12, kSelBins = 1 << kSelBits;
constexpr int kSelMaxPass = (64 + 62 + kSelBits - 1) / kSelBits;
// bits [shift, shift + width) of the 128-bit value (hi, lo), width <= 32
__device__ __forceinline__ unsigned sel_digit(uint64_t hi, uint64_t lo, int shift, int width) {
    uint64_t v;
    if (shift >= 64)
        v = hi >> (shift - 64);
    else if (shift == 0)
        v = lo;
    else
        v = (lo >> shift) | (hi << (64 - shift));
    return (unsigned)v & ((1u << width) - 1u);
}
__global__ void __launch_bounds__(kSelThreads) trikey_select_kernel(const TriKey* __restrict__ in, uint64_t n,
                                                                    uint64_t K, int ib, unsigned* __restrict__ hist,
                                                                    unsigned long long* __restrict__ mm,
                                                                    unsigned* bar, TriKey* __restrict__ out,
                                                                    unsigned long long* __restrict__ cnt,
                                                                    TriKey* __restrict__ thr) {
    __shared__ unsigned sh[kSelBins];
    __shared__ unsigned wsum[kSelThreads / 32];
    __shared__ unsigned long long s_mm[2][kSelThreads / 32];
    __shared__ uint64_t s_p[2], s_m[2];  // prefix and mask over the packed key (hi, lo)
    __shared__ unsigned long long s_krem;
    __shared__ int s_done;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int lob = 2 * ib;  // <= 62
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + tid, st = (uint64_t)gridDim.x * blockDim.x;
    // range of the distance keys (mm[0] = max of ~d, mm[1] = max of d; zero-initialised)
    {
        unsigned long long a = 0ull, b = 0ull;
        for (uint64_t e = t0; e < n; e += st) {
            const unsigned long long d = in[e].d;
            a = max(a, ~d);
            b = max(b, d);
        }
        for (int o = 16; o; o >>= 1) {
            a = max(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if (lane == 0) {
            s_mm[0][wid] = a;
            s_mm[1][wid] = b;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < kSelThreads / 32; ++w) {
                a = max(a, s_mm[0][w]);
                b = max(b, s_mm[1][w]);
            }
            atomicMax(&mm[0], a);
            atomicMax(&mm[1], b);
            s_p[0] = s_p[1] = s_m[0] = s_m[1] = 0;
            s_krem = K;
            s_done = 0;
        }
        sel_grid_sync(bar, gridDim.x);
    }
    const uint64_t dmin = ~__ldcg(&mm[0]), dmax = __ldcg(&mm[1]);
    const uint64_t span = dmax - dmin;
    const int db = 64 - __clzll((long long)span);  // bits of d - dmin (0 when every d is equal)
    const int T = db + lob;
    const int npass = (T + kSelBits - 1) / kSelBits;
    // packed key of an entry: lo = (dd << lob) | ids, hi = the bits of dd past lo
    auto pack = [&](const TriKey& k, uint64_t& hi, uint64_t& lo) {
        const uint64_t dd = k.d - dmin;
        lo = (dd << lob) | ((uint64_t)k.a << ib) | k.b;
        hi = dd >> (64 - lob);
    };
    for (int pass = 0; pass < npass && !s_done; ++pass) {
        const int top = T - kSelBits * pass;          // this pass resolves bits [shift, top)
        const int shift = max(0, top - kSelBits), width = top - shift;
        const uint64_t ph = s_p[0], pl = s_p[1], mh = s_m[0], ml = s_m[1];
        for (int b = tid; b < kSelBins; b += kSelThreads) sh[b] = 0u;
        __syncthreads();
        for (uint64_t e0 = (uint64_t)blockIdx.x * blockDim.x; e0 < n; e0 += st) {
            const uint64_t e = e0 + tid;
            bool hit = false;
            unsigned dg = 0;
            if (e < n) {
                uint64_t hi, lo;
                pack(in[e], hi, lo);
                hit = (hi & mh) == ph && (lo & ml) == pl;
                dg = sel_digit(hi, lo, shift, width);
            }
            const unsigned act = __ballot_sync(0xffffffffu, hit);
            if (act) {
                const int lead = __ffs(act) - 1;
                const unsigned ldg = __shfl_sync(0xffffffffu, dg, lead);
                const unsigned same = __ballot_sync(0xffffffffu, hit && dg == ldg);
                if (lane == lead) atomicAdd(&sh[ldg], (unsigned)__popc(same));
                if (hit && dg != ldg) atomicAdd(&sh[dg], 1u);
            }
        }
        __syncthreads();
        for (int b = tid; b < kSelBins; b += kSelThreads)
            if (sh[b]) atomicAdd(&hist[pass * kSelBins + b], sh[b]);
        sel_grid_sync(bar, gridDim.x);
        // every CTA: the bin holding the krem-th key of the group (block scan of the counts;
        // thread t owns bins [per t, per (t + 1)))
        constexpr int per = kSelBins / kSelThreads;
        unsigned c[per], mine = 0;
#pragma unroll
        for (int q = 0; q < per; ++q) {
            c[q] = __ldcg(&hist[pass * kSelBins + tid * per + q]);
            mine += c[q];
        }
        unsigned incl = mine;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) wsum[wid] = incl;
        __syncthreads();
        unsigned long long excl = incl - mine;
        for (int w = 0; w < wid; ++w) excl += wsum[w];
        const unsigned long long krem = s_krem;
        __syncthreads();  // every thread has read s_krem
        if (excl < krem && krem <= excl + mine) {
            unsigned long long below = excl;
            int q = 0;
            for (; q < per - 1; ++q) {
                if (below + c[q] >= krem) break;
                below += c[q];
            }
            const unsigned bin = (unsigned)(tid * per + q);
            // prefix and mask gain the bits [shift, shift + width) of the 128-bit key
            const uint64_t wm = (width >= 64 ? ~0ull : (1ull << width) - 1);
            if (shift >= 64) {
                s_p[0] |= (uint64_t)bin << (shift - 64);
                s_m[0] |= wm << (shift - 64);
            } else {
                s_p[1] |= (uint64_t)bin << shift;
                s_m[1] |= wm << shift;
                if (shift + width > 64) {
                    s_p[0] |= (uint64_t)bin >> (64 - shift);
                    s_m[0] |= wm >> (64 - shift);
                }
            }
            s_krem = krem - below;
            if (krem - below == c[q]) s_done = 1;  // the whole prefix group is in
        }
        __syncthreads();
    }
    // threshold in packed form: the prefix with every unresolved bit of the T-bit key set
    const uint64_t full_lo = T >= 64 ? ~0ull : (1ull << T) - 1;
    const uint64_t full_hi = T > 64 ? (1ull << (T - 64)) - 1 : 0ull;
    const uint64_t th = s_p[0] | (~s_m[0] & full_hi), tl = s_p[1] | (~s_m[1] & full_lo);
    for (uint64_t e0 = (uint64_t)blockIdx.x * blockDim.x; e0 < n; e0 += st) {
        const uint64_t e = e0 + tid;
        bool keep = false;
        TriKey k;
        if (e < n) {
            k = in[e];
            uint64_t hi, lo;
            pack(k, hi, lo);
            keep = hi < th || (hi == th && lo <= tl);
        }
        // one reservation per CTA and step (a returning atomic per warp on one address
        // serialises in L2: 50k of them at level 0)
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) wsum[wid] = (unsigned)__popc(bal);
        __syncthreads();
        if (tid == 0) {
            unsigned tot = 0;
            for (int w = 0; w < kSelThreads / 32; ++w) tot += wsum[w];
            s_krem = tot ? atomicAdd(cnt, (unsigned long long)tot) : 0ull;
        }
        __syncthreads();
        unsigned long long at = s_krem;
        for (int w = 0; w < wid; ++w) at += wsum[w];
        if (keep) out[at + __popc(bal & ((1u << lane) - 1u))] = k;
        __syncthreads();  // wsum / s_krem are rewritten next step
    }
    if (blockIdx.x == 0 && tid == 0) {
        // back to (dist, a, b): dd = threshold >> lob; past the keys' span (unresolved
        // distance bits) every key is in: T = (dmax, largest ids)
        const uint64_t ddt = (tl >> lob) | (th << (64 - lob));
        const bool over = (th >> lob) != 0 || ddt > span;
        const uint64_t idm = (1ull << ib) - 1;
        TriKey t;
        t.d = over ? dmax : dmin + ddt;
        t.a = over ? (uint32_t)idm : (uint32_t)((tl >> ib) & idm);
        t.b = over ? (uint32_t)idm : (uint32_t)(tl & idm);
        *thr = t;
    }
}

// out (K entries, any order) and *thr on the device; no host round trip
static void select_trikeys(Context& c, const TriKey* in, uint64_t n, uint64_t K, TriKey* out, TriKey* thr,
                           DevBuf& scratch) {
    static int grid = 0;
    if (!grid) {
        int per = 0;
        NRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, trikey_select_kernel, kSelThreads, 0));
        int sms = 0;
        NRG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
        grid = std::max(1, std::min(per, 1)) * sms;  // one CTA per SM: 4096 histogram adds per CTA and pass
    }
    const int ib = id_bits(c);
    if (2 * ib > 62) fail(100, "select: node ids wider than 31 bits");
    const size_t words = (size_t)kSelMaxPass * kSelBins + 4 + 2 + 2;  // hist, range (2 u64), barrier, count (u64)
    unsigned* hist = scratch.as<unsigned>(words);
    unsigned long long* mm = reinterpret_cast<unsigned long long*>(hist + (size_t)kSelMaxPass * kSelBins);
    unsigned* bar = reinterpret_cast<unsigned*>(mm + 2);
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(bar + 2);
    NRG_CUDA(cudaMemsetAsync(hist, 0, words * 4, c.stream));
    const unsigned g = (unsigned)std::min<uint64_t>((uint64_t)grid, std::max<uint64_t>(1, ceil_div(n, kSelThreads)));
    void* args[] = {(void*)&in, (void*)&n, (void*)&K, (void*)&ib, (void*)&hist, (void*)&mm, (void*)&bar, (void*)&out,
                    (void*)&cnt, (void*)&thr};
    NRG_CUDA(cudaLaunchCooperativeKernel((void*)trikey_select_kernel, g, kSelThreads, args, 0, c.stream));
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
// canonical pair (min << ib) | max: equal exactly for equal pairs, sorted over 2 ib bits
__global__ void dplus_pairkeys_kernel(const TriKey* __restrict__ dir, uint64_t m2, int ib, uint64_t* __restrict__ pk,
                                      uint32_t* __restrict__ idx) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m2) return;
    const uint64_t a = dir[e].a, b = dir[e].b;
    pk[e] = a < b ? (a << ib) | b : (b << ib) | a;
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

// S': every out-entry of node li lies in D+ (inc/find_best.hpp:150-163).  Rows are sorted
// by (dist, id) and (dist, li, id) orders them the same way, so the last entry decides.
__global__ void saturated_kernel(const int32_t* __restrict__ nodes, const int32_t* __restrict__ ids,
                                 const double* __restrict__ dists, uint64_t n, int k, const TriKey* __restrict__ thrp,
                                 uint8_t* __restrict__ flag) {
    const uint64_t li = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= n) return;
    const TriKey thr = *thrp;
    TriKey x;
    x.d = dkey(dists[li * k + (k - 1)]);
    x.a = (uint32_t)nodes[li];
    x.b = (uint32_t)ids[li * k + (k - 1)];
    flag[li] = trikey_le(x, thr) ? 1 : 0;
}

__global__ void trikey_pk_kernel(const TriKey* __restrict__ in, uint64_t n, int ib, uint64_t* __restrict__ pk,
                                 uint32_t* __restrict__ idx) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    pk[e] = ((uint64_t)in[e].a << ib) | in[e].b;
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

// ---------------------------------------------------------------- dense levels
// A deep level whose per-node candidate sets approach the level itself (cap^2 ~ |S|) probes
// a large share of its |S|^2/2 pairs, each through a claim in the DRAM-resident distance
// cache and a K1 screen.  There the exhaustive tensor-core screen of S (score_all_pairs_tc,
// ~1e11 pairs/s) is cheaper than the probes: the level and every deeper one (subsets of S)
// then look distances up in that triangle.  The NNDescent/FindBest semantics, the values
// (the same deterministic scores) and the miss counting are unchanged.
__global__ void dense_loc_kernel(const int32_t* __restrict__ nodes, uint64_t n, int32_t* __restrict__ loc) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) loc[nodes[t]] = (int32_t)t;
}
// base case below a dense root: the level's own triangle gathered from the root's
__global__ void dense_subtri_kernel(const int32_t* __restrict__ nodes, uint64_t n, const int32_t* __restrict__ loc,
                                    DenseView D, uint64_t dn, TriKey* __restrict__ out) {
    const uint64_t a = blockIdx.x;
    if (a >= n) return;
    const uint64_t base = a * (2 * n - a - 1) / 2;
    const int32_t x = nodes[a];
    const uint64_t ra = (uint64_t)loc[x];
    for (uint64_t c = a + 1 + threadIdx.x; c < n; c += blockDim.x) {
        const int32_t y = nodes[c];
        const uint64_t rb = (uint64_t)loc[y];
        const uint64_t lo = ra < rb ? ra : rb, hi = ra < rb ? rb : ra;
        TriKey k;
        k.d = dkey(dense_value(D, lo * (2 * dn - lo - 1) / 2 + (hi - lo - 1)));
        k.a = (uint32_t)min(x, y);
        k.b = (uint32_t)max(x, y);
        out[base + (c - a - 1)] = k;
    }
}

// Settles the dense root's probe counts (see dense_probe, knn.cu): every probe there was
// counted as a hit; of the U distinct pairs probed (bits set), the ones no shallower level
// had scored (absent from the distance cache: U - F) are the generation's misses.
// count_bits: the probed pairs (bits) count as misses on one rank only; every rank
// moves the probed pairs its shard of the key-sharded cache already held back to hits
__global__ void dense_recount_kernel(HashView h, const int32_t* __restrict__ loc, const uint32_t* __restrict__ sq,
                                     uint64_t dn, uint64_t* __restrict__ counters, int count_bits) {
    long long d = 0;
    const uint64_t Wd = (dn + 31) >> 5;
    const int lane = threadIdx.x & 31;
    if (count_bits) {
        // distinct probed pairs: the square mark matrix OR its transpose, above the diagonal;
        // one warp per 32 x 32 bit block (I <= J), lane r = row r of the block
        const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
        for (uint64_t blk = warp0; blk < Wd * Wd; blk += nwarps) {
            const uint64_t I = blk / Wd, J = blk % Wd;
            if (J < I) continue;
            const uint64_t ra = 32 * I + lane, rb = 32 * J + lane;
            const uint32_t A = ra < dn ? sq[ra * Wd + J] : 0u;
            const uint32_t B = rb < dn ? sq[rb * Wd + I] : 0u;
            // transpose of B (bit c of lane r = bit r of B's lane c): five block-swap steps
            uint32_t T = B;
#pragma unroll
            for (int j = 16; j; j >>= 1) {
                const uint32_t hi = j == 16 ? 0xffff0000u : j == 8 ? 0xff00ff00u : j == 4 ? 0xf0f0f0f0u
                                  : j == 2 ? 0xccccccccu : 0xaaaaaaaau;  // columns with bit j set
                const uint32_t y = __shfl_xor_sync(0xffffffffu, T, j);
                T = (lane & j) ? ((T & hi) | ((y >> j) & ~hi)) : ((T & ~hi) | ((y << j) & hi));
            }
            uint32_t X = A | T;
            if (I == J) X &= lane == 31 ? 0u : (~0u << (lane + 1));  // columns past the diagonal
            d += __popc(X);
        }
    }
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, st = (uint64_t)gridDim.x * blockDim.x;
    if (h.keys) {
        for (uint64_t s = t0; s <= h.mask; s += st) {
            const uint64_t key = __ldcs(&h.keys[s]);
            if (key >= kTombKey) continue;
            const int32_t la = loc[(uint32_t)(key >> 32)], lb = loc[(uint32_t)(key & 0xffffffffu)];
            if (la < 0 || lb < 0) continue;
            const uint64_t a = (uint64_t)la, b = (uint64_t)lb;
            d -= ((sq[a * Wd + (b >> 5)] >> (b & 31)) | (sq[b * Wd + (a >> 5)] >> (a & 31))) & 1u;
        }
    }
    for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (lane == 0 && d) {
        atomicAdd((unsigned long long*)&counters[C_MISSES], (unsigned long long)d);
        atomicAdd((unsigned long long*)&counters[C_HITS], (unsigned long long)(-d));
    }
}

// The level that set up the dense root tears it down (also on throw).  In a sharded job
// (world > 1) a dense level is replicated: every rank screens the whole level with the
// tensor cores and runs its NNDescent/FindBest as a single-rank job (world 1 inside the
// region, no collectives -- every rank holds the same triangle and computes the same
// lists), which keeps the fast dense path of the single-GPU run instead of switching to
// the claim path.  The miss/hit counters count the region once job-wide: ranks other than
// 0 restore their pre-region counters and contribute only their cache shard's overlap.
struct DenseGuard {
    Context& c;
    bool owner = false;
    int real_rank = 0, real_world = 1;
    uint64_t saved[2] = {0, 0};
    explicit DenseGuard(Context& cc) : c(cc) {}
    void replicate() {
        real_rank = c.rank;
        real_world = c.world;
        if (real_rank != 0) {
            NRG_CUDA(cudaMemcpyAsync(saved, c.dcounters(), 16, cudaMemcpyDeviceToHost, c.stream));
            c.sync();
        }
        c.rank = 0;
        c.world = 1;
    }
    ~DenseGuard() {
        if (owner) {
            const uint64_t pairs = c.dense_n * (c.dense_n - 1) / 2;
            const HashView h = (c.Ckeys.p && c.Ccap) ? c.Cview() : HashView{nullptr, nullptr, 0};
            if (real_world > 1) {
                c.rank = real_rank;
                c.world = real_world;
                if (real_rank != 0)
                    cudaMemcpyAsync(c.dcounters(), saved, 16, cudaMemcpyHostToDevice, c.stream);
            }
            // off the critical path: only the counters need it (and the cache must not
            // change under it: join_side() before any clear, resize or counter read)
            cudaStream_t ss = c.fork();
            dense_recount_kernel<<<148 * 8, 256, 0, ss>>>(h, static_cast<const int32_t*>(c.dloc.p),
                                                          static_cast<const uint32_t*>(c.dbits.p), c.dense_n,
                                                          c.dcounters(), real_rank == 0 ? 1 : 0);
            c.fork_done();
            c.dense_active = false;
            c.dense_n = 0;  // the buffers stay (grow-only): the next generation reuses them
            c.dwl_n = 0;
        }
    }
};

static uint64_t dense_max_n() {
    const char* e = getenv("NRG_DENSE_N");
    return e ? (uint64_t)strtoull(e, nullptr, 10) : 65535;  // the tensor-core screen's limit
}
// a level goes dense when its candidate sets (up to cap^2 per node) cover at least
// 1/ratio of the level
static uint64_t dense_ratio() {
    const char* e = getenv("NRG_DENSE_RATIO");
    return e ? (uint64_t)strtoull(e, nullptr, 10) : 32;
}

__global__ void ascending_check_kernel(const int32_t* __restrict__ v, uint64_t n, int n_total, int* __restrict__ bad) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    if (v[t] < 0 || v[t] >= n_total || (t > 0 && v[t] <= v[t - 1])) *bad = 1;
}

// Unique undirected pairs of a TriKey list by hashing canonical pair keys into an
// L2-resident table: duplicates of a pair carry the same distance (one value per pair and
// generation), so any representative gives the same canonical (dist, min, max) entry and
// the result is order-independent -- no sort needed.
__global__ void pair_dedup_kernel(const TriKey* __restrict__ in, uint64_t n, int ib, uint64_t* __restrict__ table,
                                  uint64_t mask, TriKey* __restrict__ out, unsigned long long* __restrict__ cnt) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool keep = false;
    TriKey o;
    if (e < n) {
        const TriKey t = in[e];
        o.d = t.d;
        o.a = min(t.a, t.b);
        o.b = max(t.a, t.b);
        const uint64_t key = ((uint64_t)o.a << ib) | o.b;
        uint64_t s = slot_of(key, mask);
        for (;;) {
            const unsigned long long prev =
                atomicCAS((unsigned long long*)&table[s], (unsigned long long)kEmptyKey, (unsigned long long)key);
            if (prev == kEmptyKey) {
                keep = true;
                break;
            }
            if (prev == key) break;
            s = (s + 1) & mask;
        }
    }
    // one reservation per CTA (a returning atomic per warp on one address serialises in L2)
    __shared__ unsigned s_w[8];
    __shared__ unsigned long long s_base;
    const unsigned b = __ballot_sync(0xffffffffu, keep);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) s_w[wid] = (unsigned)__popc(b);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned tot = 0;
        for (int w = 0; w < 8; ++w) tot += s_w[w];
        s_base = tot ? atomicAdd(cnt, (unsigned long long)tot) : 0ull;
    }
    __syncthreads();
    unsigned long long at = s_base;
    for (int w = 0; w < wid; ++w) at += s_w[w];
    if (keep) out[at + __popc(b & ((1u << lane) - 1u))] = o;
}
static void pair_dedup(Context& c, const TriKey* in, uint64_t n, TriKey* out, unsigned long long* cnt, DevBuf& tabb) {
    uint64_t cap = 1024;
    while (cap < 2 * n) cap <<= 1;
    uint64_t* table = tabb.as<uint64_t>(cap);
    NRG_CUDA(cudaMemsetAsync(table, 0xff, cap * 8, c.stream));
    NRG_CUDA(cudaMemsetAsync(cnt, 0, 8, c.stream));
    if (n) {
        pair_dedup_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(in, n, id_bits(c), table, cap - 1, out,
                                                                          cnt);
        NRG_LAUNCH_CHECK();
    }
}

static inline unsigned g256(uint64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, 256)); }

// union of two candidate lists without duplicate pairs, then the (dist,i,j)-smallest
// `want` (inc/find_best.hpp:171-174 + :62-70)
// sorted == false (inner levels): the whole unique set is returned, unsorted.  The parent
// keeps the top `want` of (its D U this set), and an entry outside this level's top `want`
// has `want` better entries here, so it can never enter the parent's top `want`: the
// result is the same as with the truncated list, and only the root level sorts.
static uint64_t merge_select(Context& c, TriKey* buf, uint64_t n, uint64_t want, DevBuf& outb, bool sorted) {
    DevBuf tmpb, ub, cntb, tabb;
    TriKey* uniq = ub.as<TriKey>(std::max<uint64_t>(n, 1));
    unsigned long long* cnt = cntb.as<unsigned long long>(1);
    unsigned long long nu = 0;
    if (NRG_ENV_ON("NRG_SORT_DEDUP")) {
        DevBuf pkb, idxb, pk2b, idx2b, flagb;
        uint64_t* pk = pkb.as<uint64_t>(n);
        uint32_t* idx = idxb.as<uint32_t>(n);
        uint64_t* pk2 = pk2b.as<uint64_t>(n);
        uint32_t* idx2 = idx2b.as<uint32_t>(n);
        uint8_t* flag = flagb.as<uint8_t>(n);
        if (n) {
            const int ib = id_bits(c);
            trikey_pk_kernel<<<g256(n), 256, 0, c.stream>>>(buf, n, ib, pk, idx);
            size_t bytes = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, bytes, pk, pk2, idx, idx2, (int64_t)n, 0, 2 * ib, c.stream);
            void* tmp = tmpb.ensure(bytes);
            cub::DeviceRadixSort::SortPairs(tmp, bytes, pk, pk2, idx, idx2, (int64_t)n, 0, 2 * ib, c.stream);
            unique_flags_kernel<<<g256(n), 256, 0, c.stream>>>(pk2, n, flag);
            NRG_CUDA(cudaMemsetAsync(cnt, 0, 8, c.stream));
            gather_trikey_kernel<<<g256(n), 256, 0, c.stream>>>(buf, idx2, flag, n, uniq, cnt);
            NRG_LAUNCH_CHECK();
        }
    } else {
        pair_dedup(c, buf, n, uniq, cnt, tabb);
    }
    if (n) {
        nu = c.read_scalar(cnt);
    }
    if (!sorted) {
        outb = std::move(ub);
        return nu;
    }
    // the root: select the `want` smallest (device radix select), then sort only those
    uint64_t ns = nu;
    const TriKey* src = uniq;
    DevBuf selb, thrb, sscr;
    if (nu > want && !NRG_ENV_ON("NRG_SORT_DPLUS")) {
        TriKey* picked = selb.as<TriKey>(want);
        select_trikeys(c, uniq, nu, want, picked, thrb.as<TriKey>(1), sscr);
        src = picked;
        ns = want;
    }
    TriKey* out = outb.as<TriKey>(std::max<uint64_t>(nu, 1));
    sort_trikeys(c, const_cast<TriKey*>(src), out, ns, tmpb);
    return std::min<uint64_t>(nu, want);
}

// result of a level: TriKey list (a<b canonical) sorted by (dist, a, b)
static uint64_t find_best_impl(Context& c, int mode, uint64_t m, const int32_t* S, uint64_t n, double knn_eps,
                               uint64_t seed, bool reverse, int level, std::vector<TraceLevelD>& trace,
                               DevBuf& result, bool sorted, bool root) {
    if (n < 2) return 0;
    const uint64_t total = n * (n - 1) / 2;
    const uint64_t want = std::min(m, total);
    if (n * n <= 4 * m) {
        // base case: exhaustive scan (inc/find_best.hpp:98-104)
        DevBuf distb, keysb, tmpb;
        TriKey* keys = keysb.as<TriKey>(total);
        if (mode == EXACT && c.dense_active && c.world == 1) {
            dense_resolve_subtri(c, S, n);
            c.tic();
            dense_subtri_kernel<<<(unsigned)n, 256, 0, c.stream>>>(S, n, static_cast<const int32_t*>(c.dloc.p),
                                                                  c.dview(), c.dense_n, keys);
            NRG_LAUNCH_CHECK();
            // counted as score_all_pairs counts the base case: every pair a probe
            counters_add_host(c, C_MISSES, total);
        } else {
            double* dist = distb.as<double>(total);
            score_all_pairs(c, mode, S, n, dist);
            c.tic();
            tri_from_pairs_kernel<<<(unsigned)n, 256, 0, c.stream>>>(S, n, dist, keys);
            NRG_LAUNCH_CHECK();
        }
        uint64_t ret = want;
        if (root) {
            TriKey* out = result.as<TriKey>(total);
            sort_trikeys(c, keys, out, total, tmpb);
        } else {
            result = std::move(keysb);  // all pairs, unsorted (see merge_select)
            ret = total;
        }
        c.toc(P_SELECT);
        trace.push_back({level, 0, 1, 0, n, 0});
        return ret;
    }
    const int k = (int)((4 * m + n - 1) / n);
    DenseGuard dg(c);
    {
        const uint64_t kw = (uint64_t)std::max(k, 4);
        const uint64_t cap = reverse ? std::max<uint64_t>(2 * kw, 8) : std::max<uint64_t>(kw, 8);
        if (!c.dense_active && mode == EXACT && c.kind == ISING && n <= dense_max_n() &&
            dense_ratio() * cap * cap >= n) {
            c.join_side();  // a previous root's recount still reads dloc / dbits

            if (NRG_ENV_ON("NRG_DEBUG_LEVELS")) c.flush_timing();
            const double ph0 = c.phase_ms[P_SCORE];
            const auto w0 = std::chrono::steady_clock::now();
            // the level's distances, sparse (Context::dview): survivors only
            const bool ok = score_all_pairs_tc(c, S, n, nullptr, true, !NRG_ENV_ON("NRG_DENSE_EAGER"));
            if (NRG_ENV_ON("NRG_DEBUG_LEVELS")) {
                c.flush_timing();
                fprintf(stderr, "dense root level %d: n=%llu setup wall_ms=%.2f score_phase_ms=%.2f ok=%d\n", level,
                        (unsigned long long)n,
                        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count(),
                        c.phase_ms[P_SCORE] - ph0, (int)ok);
            }
            if (ok) {
                int32_t* loc = c.dloc.as<int32_t>(c.n);
                NRG_CUDA(cudaMemsetAsync(loc, 0xff, (size_t)c.n * 4, c.stream));
                dense_loc_kernel<<<g256(n), 256, 0, c.stream>>>(S, n, loc);
                NRG_LAUNCH_CHECK();
                // probe marks: square bit matrix over the root's positions (row = probing node)
                const uint64_t mwords = n * ((n + 31) / 32);
                uint32_t* bits = c.dbits.as<uint32_t>(mwords);
                NRG_CUDA(cudaMemsetAsync(bits, 0, mwords * 4, c.stream));
                c.dense_active = true;
                c.dense_n = n;
                dg.owner = true;
                if (c.world > 1) dg.replicate();
            }
        }
    }
    KnnParamsD kp;
    kp.eps = knn_eps;
    kp.seed = mix64(seed, (uint64_t)level);
    kp.reverse = reverse;
    KnnResultD knn;
    DevBuf kid, kdist;
    const bool dbg = NRG_ENV_ON("NRG_DEBUG_LEVELS");
    uint64_t m0 = 0;
    double t0 = 0.0, s0 = 0.0, k20 = 0.0;
    if (dbg) {
        c.flush_timing();
        m0 = c.read_scalar(c.dcounters() + C_MISSES);
        t0 = c.phase_ms[P_KNN];
        s0 = c.phase_ms[P_SCORE];
        k20 = c.k2_pairs;
    }
    find_knn(c, mode, k, S, n, kp, false, knn, kid, kdist, sorted);
    if (dbg) {
        uint64_t m1 = 0;
        c.flush_timing();
        m1 = c.read_scalar(c.dcounters() + C_MISSES);
        fprintf(stderr, "level %d: n=%llu k=%d sweeps=%d knn_ms=%.2f score_ms=%.2f unique_pairs=%llu survivors=%.0f\n",
                level, (unsigned long long)n, k, knn.sweeps, c.phase_ms[P_KNN] - t0, c.phase_ms[P_SCORE] - s0,
                (unsigned long long)(m1 - m0), c.k2_pairs - k20);
    }
    c.tic();
    const uint64_t nd = n * (uint64_t)knn.k;
    DevBuf dirb, dir2b, tmpb, thrb, selb;
    TriKey* dir = dirb.as<TriKey>(nd);
    TriKey* dirs = dir2b.as<TriKey>(nd);
    directed_keys_kernel<<<g256(nd), 256, 0, c.stream>>>(S, knn.ids, knn.dists, n, knn.k, dir);
    NRG_LAUNCH_CHECK();
    const uint64_t dplus = std::min<uint64_t>(2 * m, nd);
    // D+ (the dplus smallest directed entries, any order) and its largest key: a device
    // radix select (NRG_SORT_DPLUS=1: the full sort, D+ its sorted prefix)
    TriKey* thr = thrb.as<TriKey>(1);
    if (NRG_ENV_ON("NRG_SORT_DPLUS")) {
        sort_trikeys(c, dir, dirs, nd, tmpb);
        NRG_CUDA(cudaMemcpyAsync(thr, dirs + (dplus - 1), sizeof(TriKey), cudaMemcpyDeviceToDevice, c.stream));
    } else {
        select_trikeys(c, dir, nd, dplus, dirs, thr, selb);
    }
    // D: unique undirected pairs of D+
    DevBuf pkb, idxb, pk2b, idx2b, flagb, cntb;
    uint64_t* pk = pkb.as<uint64_t>(dplus);
    uint32_t* idx = idxb.as<uint32_t>(dplus);
    uint64_t* pk2 = pk2b.as<uint64_t>(dplus);
    uint32_t* idx2 = idx2b.as<uint32_t>(dplus);
    uint8_t* flag = flagb.as<uint8_t>(std::max<uint64_t>(dplus, n));
    unsigned long long* cnt = cntb.as<unsigned long long>(2);  // |D|, |S'|
    DevBuf dpairsb, dtabb;
    TriKey* dpairs = dpairsb.as<TriKey>(dplus);
    NRG_CUDA(cudaMemsetAsync(cnt, 0, 16, c.stream));
    if (NRG_ENV_ON("NRG_SORT_DEDUP")) {
        const int ib = id_bits(c);
        dplus_pairkeys_kernel<<<g256(dplus), 256, 0, c.stream>>>(dirs, dplus, ib, pk, idx);
        {
            size_t bytes = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, bytes, pk, pk2, idx, idx2, (int64_t)dplus, 0, 2 * ib, c.stream);
            void* tmp = tmpb.ensure(bytes);
            cub::DeviceRadixSort::SortPairs(tmp, bytes, pk, pk2, idx, idx2, (int64_t)dplus, 0, 2 * ib, c.stream);
        }
        unique_flags_kernel<<<g256(dplus), 256, 0, c.stream>>>(pk2, dplus, flag);
        d_pairs_kernel<<<g256(dplus), 256, 0, c.stream>>>(dirs, idx2, flag, dplus, dpairs, cnt);
        NRG_LAUNCH_CHECK();
    } else {
        // D: unique undirected pairs of D+ (inc/find_best.hpp:133-145)
        pair_dedup(c, dirs, dplus, dpairs, cnt, dtabb);
    }
    // S': the threshold key (the dplus-th smallest directed entry) stays on the device;
    // |D| and |S'| come back in one round trip
    saturated_kernel<<<g256(n), 256, 0, c.stream>>>(S, knn.ids, knn.dists, n, knn.k, thr, flag);
    NRG_LAUNCH_CHECK();
    DevBuf satb;
    int32_t* sat = satb.as<int32_t>(n);
    {
        size_t bytes = 0;
        cub::DeviceSelect::Flagged(nullptr, bytes, S, flag, sat, cnt + 1, (int64_t)n, c.stream);
        void* tmp = tmpb.ensure(bytes);
        cub::DeviceSelect::Flagged(tmp, bytes, S, flag, sat, cnt + 1, (int64_t)n, c.stream);
    }
    // |D| and |S'| in one round trip
    unsigned long long* hc = c.hp_small.as<unsigned long long>(2);
    NRG_CUDA(cudaMemcpyAsync(hc, cnt, 16, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    const unsigned long long nD = hc[0];
    const int hsat = (int)hc[1];
    c.toc(P_SELECT);
    trace.push_back({level, k, 0, knn.sweeps, n, (uint64_t)nD});
    kid.release();
    kdist.release();
    dirb.release();

    DevBuf rec;
    // S' keeps S's order (DeviceSelect), so a sorted S gives a sorted S'
    const uint64_t nrec =
        find_best_impl(c, mode, m, sat, (uint64_t)hsat, knn_eps, seed, reverse, level + 1, trace, rec, sorted, false);
    c.tic();
    // merge D with the recursive result (dropping duplicates) and select
    DevBuf allb;
    TriKey* all = allb.as<TriKey>(nD + nrec + 1);
    if (nD) NRG_CUDA(cudaMemcpyAsync(all, dpairs, nD * sizeof(TriKey), cudaMemcpyDeviceToDevice, c.stream));
    if (nrec)
        NRG_CUDA(cudaMemcpyAsync(all + nD, rec.p, nrec * sizeof(TriKey), cudaMemcpyDeviceToDevice, c.stream));
    const uint64_t cntres = merge_select(c, all, nD + nrec, want, result, root);
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
        // a strictly ascending, in-range node list (the GCD loop's 0..N-1) needs no per-level
        // sort or validation; anything else takes find_knn's checked path
        DevBuf okb;
        int* ok = okb.as<int>(1);
        NRG_CUDA(cudaMemsetAsync(ok, 0, 4, c.stream));
        ascending_check_kernel<<<g256(n), 256, 0, c.stream>>>(d_nodes, n, c.n, ok);
        NRG_LAUNCH_CHECK();
        int hbad = 0;
        hbad = c.read_scalar(ok);
        cnt = find_best_impl(c, mode, m, d_nodes, n, knn_eps, seed, reverse, 0, res.trace, result, hbad == 0, true);
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
