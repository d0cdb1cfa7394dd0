// knn.cu — NNDescent (Alg. 4) on the device: find_knn / find_knn_exhaustive
// (inc/knn.hpp:150-314).
//
// Reference-exact semantics, re-expressed as sets so each phase is data-parallel:
//   * initial graph: per node SplitRng(seed).split(id+1), Floyd sampling of kw
//     distinct ranks over the id-sorted node set, self skipped (:171-200);
//   * per sweep the snapshot S, the capped undirected view U (out-lists by (dist,id),
//     then in-lists by (dist, src) while rows have room; cap = max(kw, scan_floor))
//     (:202-247);
//   * the scan replaces a node's worst entry with any strictly better 2-hop candidate
//     not already listed (:249-270).  With a fixed per-generation distance, the final
//     list is exactly the (dist,id)-top-kw of (snapshot list U candidates) — the
//     visit-order independence the reference tests (test_knn.cpp:154-194) — so a
//     sweep is: gather+dedup 2-hop candidates (one CTA per node, smem hash set or
//     bitmap; paths whose two hops were both already in U last sweep are skipped, see
//     u_new_kernel), claim them in the distance cache (one score per pair per
//     generation, inc/model.hpp:54-70), score the claimed worklist, then merge top-kw
//     per node;
//   * churn = entries that entered from the candidate set (:273-290);
//   * trim to k (:292-305); exhaustive fallbacks (:156-164).
#include <cub/cub.cuh>

#include <algorithm>
#include <numeric>
#include <vector>

#include "comm.cuh"
#include "context.cuh"

namespace nrg {

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ bool entry_less(double da, int ia, double db, int ib) {
    // entry_better (inc/knn.hpp:25-28)
    return da < db || (da == db && ia < ib);
}

__global__ void iota_kernel(int32_t* v, uint64_t n) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) v[t] = (int32_t)t;
}
__global__ void scatter_loc_kernel(const int32_t* __restrict__ nodes, uint64_t n, int32_t* __restrict__ loc,
                                   int n_total, int* __restrict__ bad) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int g = nodes[t];
    if (g < 0 || g >= n_total) {
        if (bad) atomicExch(bad, 1);
        return;
    }
    if (atomicExch(&loc[g], (int32_t)t) != -1 && bad) atomicExch(bad, 2);  // duplicate node
}
__global__ void rank_kernel(const int32_t* __restrict__ perm, uint64_t n, int32_t* __restrict__ rank) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) rank[perm[t]] = (int32_t)t;
}

// initial out-neighbours: Floyd sampling (inc/knn.hpp:177-199).  One warp per node.  The
// stream is counter-based (draw i = mix64 of key and i + 1, one draw per pick), so the
// draws of a round of 32 picks are computed by the lanes in parallel; only the membership
// rule (a draw already picked is replaced by t) runs in pick order, on registers.
// (nodes, rank, gid, qi, qj point at this rank's first own row; `own` rows, n = level size)
__device__ __forceinline__ uint64_t floyd_draw(const SplitRng& r, uint64_t i, uint64_t t) {
    return __umul64hi(mix64(r.key + 0x9e3779b97f4a7c15ULL * (i + 1)), t + 1);  // SplitRng::below, draw i
}
__global__ void knn_init_kernel(const int32_t* __restrict__ nodes, const int32_t* __restrict__ sorted_ids,
                                const int32_t* __restrict__ rank, const int32_t* __restrict__ loc, uint64_t own,
                                uint64_t n, int kw, uint64_t seed, int32_t* __restrict__ gid,
                                int32_t* __restrict__ qi, int32_t* __restrict__ qj) {
    const uint64_t li = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (li >= own) return;
    const SplitRng root(seed);
    const SplitRng r = root.split((uint64_t)nodes[li] + 1);
    const uint64_t self = (uint64_t)rank[li];
    int32_t* picks = gid + li * kw;  // ranks first, local ids after
    const uint64_t tbase = n - 1 - (uint64_t)kw;
    for (int base = 0; base < kw; base += 32) {
        const int i = base + lane;
        const uint64_t t = tbase + (uint64_t)i;
        const uint64_t v = i < kw ? floyd_draw(r, (uint64_t)i, t) : 0;
        // against the picks of earlier rounds
        bool hit = false;
        for (int q = 0; q < base; ++q) hit |= ((uint64_t)picks[q] == v);
        // within the round, in pick order
        uint64_t mine = 0;
        const int cnt = min(32, kw - base);
        for (int s = 0; s < cnt; ++s) {
            const uint64_t vs = __shfl_sync(0xffffffffu, v, s);
            const bool hs = __shfl_sync(0xffffffffu, (int)hit, s) != 0;
            const bool dup = __any_sync(0xffffffffu, lane < s && mine == vs);
            if (lane == s) mine = (hs || dup) ? t : v;
        }
        if (i < kw) picks[i] = (int32_t)mine;
        __syncwarp();
    }
    for (int t = lane; t < kw; t += 32) {
        uint64_t rk = (uint64_t)picks[t];
        if (rk >= self) ++rk;
        const int32_t g = sorted_ids[rk];
        picks[t] = loc[g];  // local index
        qi[li * kw + t] = nodes[li];
        qj[li * kw + t] = g;
    }
}

// the same draws with the membership test on a per-warp bitmap of the picked ranks (small
// levels with wide rows: O(kw) per node instead of O(kw^2 / 32))
__global__ void knn_init_bits_kernel(const int32_t* __restrict__ nodes, const int32_t* __restrict__ sorted_ids,
                                     const int32_t* __restrict__ rank, const int32_t* __restrict__ loc, uint64_t own,
                                     uint64_t n, int kw, uint64_t seed, int32_t* __restrict__ gid,
                                     int32_t* __restrict__ qi, int32_t* __restrict__ qj) {
    extern __shared__ uint32_t init_bits[];
    const int words = (int)((n + 31) / 32);
    uint32_t* bm = init_bits + (size_t)(threadIdx.x >> 5) * words;
    const uint64_t li = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (li >= own) return;
    for (int w = lane; w < words; w += 32) bm[w] = 0u;
    __syncwarp();
    int32_t* picks = gid + li * kw;
    const SplitRng root(seed);
    const SplitRng r = root.split((uint64_t)nodes[li] + 1);
    const uint64_t tbase = n - 1 - (uint64_t)kw;
    for (int base = 0; base < kw; base += 32) {
        const int i = base + lane;
        const uint64_t t = tbase + (uint64_t)i;
        const uint32_t v = i < kw ? (uint32_t)floyd_draw(r, (uint64_t)i, t) : 0u;
        uint32_t mine = 0;
        const int cnt = min(32, kw - base);
        for (int s = 0; s < cnt; ++s) {
            const uint32_t vs = __shfl_sync(0xffffffffu, v, s);
            const bool dup = (bm[vs >> 5] >> (vs & 31)) & 1u;  // every lane reads the same word
            const uint32_t pick = dup ? (uint32_t)(tbase + (uint64_t)(base + s)) : vs;
            __syncwarp();
            if (lane == s) {
                mine = pick;
                bm[pick >> 5] |= 1u << (pick & 31);
            }
            __syncwarp();
        }
        if (i < kw) picks[i] = (int32_t)mine;
    }
    __syncwarp();
    const uint64_t self = (uint64_t)rank[li];
    for (int t = lane; t < kw; t += 32) {
        uint64_t rk = (uint64_t)picks[t];
        if (rk >= self) ++rk;
        const int32_t g = sorted_ids[rk];
        picks[t] = loc[g];
        qi[li * kw + t] = nodes[li];
        qj[li * kw + t] = g;
    }
}

// sort each row (kw entries) by (dist, id): one CTA per row, bitonic in shared memory
template <int NT>
__global__ void __launch_bounds__(NT) row_sort_kernel(int32_t* __restrict__ gid, double* __restrict__ gd,
                                                      const int32_t* __restrict__ nodes, uint64_t n, int kw, int P) {
    extern __shared__ unsigned char rs_smem[];
    double* bd = reinterpret_cast<double*>(rs_smem);
    int32_t* bi = reinterpret_cast<int32_t*>(bd + P);
    int32_t* bg = bi + P;
    const uint64_t li = blockIdx.x;
    const int tid = threadIdx.x;
    for (int t = tid; t < P; t += NT) {
        if (t < kw) {
            bd[t] = gd[li * kw + t];
            bi[t] = gid[li * kw + t];
            bg[t] = nodes[bi[t]];
        } else {
            bd[t] = INFINITY;
            bi[t] = -1;
            bg[t] = 0x7fffffff;
        }
    }
    __syncthreads();
    for (int k2 = 2; k2 <= P; k2 <<= 1) {
        for (int j = k2 >> 1; j > 0; j >>= 1) {
            for (int t = tid; t < P; t += NT) {
                const int ixj = t ^ j;
                if (ixj > t) {
                    const bool up = (t & k2) == 0;
                    const bool gt = bd[ixj] < bd[t] || (bd[ixj] == bd[t] && bg[ixj] < bg[t]);
                    if (gt == up) {
                        const double td = bd[t]; bd[t] = bd[ixj]; bd[ixj] = td;
                        const int ti = bi[t]; bi[t] = bi[ixj]; bi[ixj] = ti;
                        const int tg = bg[t]; bg[t] = bg[ixj]; bg[ixj] = tg;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int t = tid; t < kw; t += NT) {
        gd[li * kw + t] = bd[t];
        gid[li * kw + t] = bi[t];
    }
}

// rows of up to 32 entries: one warp per row, an entry per lane; entries are distinct in
// (dist, global id), so an entry's place is the number of entries ahead of it (kw rounds
// of shuffles, no shared memory, no barriers)
__global__ void __launch_bounds__(256) row_sort_warp_kernel(int32_t* __restrict__ gid, double* __restrict__ gd,
                                                            const int32_t* __restrict__ nodes, uint64_t n, int kw) {
    const uint64_t li = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (li >= n) return;
    const bool have = lane < kw;
    const double d = have ? gd[li * kw + lane] : 0.0;
    const int32_t id = have ? gid[li * kw + lane] : 0;
    const int32_t g = have ? nodes[id] : 0;
    int ahead = 0;
    for (int s = 0; s < kw; ++s) {
        const double ds = __shfl_sync(0xffffffffu, d, s);
        const int32_t gs = __shfl_sync(0xffffffffu, g, s);
        ahead += (ds < d || (ds == d && gs < g)) ? 1 : 0;
    }
    if (have) {
        gd[li * kw + ahead] = d;
        gid[li * kw + ahead] = id;
    }
}

// ---------------------------------------------------------------- cache claim
__device__ __forceinline__ uint64_t cache_claim_k(HashView h, uint64_t key, bool& mine) {
    uint64_t s = slot_of(key, h.mask);
    for (;;) {
        const uint64_t k = __ldcg(&h.keys[s]);
        if (k == key) {
            mine = false;
            return s;
        }
        if (k == kEmptyKey) {
            const unsigned long long prev = atomicCAS((unsigned long long*)&h.keys[s],
                                                      (unsigned long long)kEmptyKey, (unsigned long long)key);
            if (prev == kEmptyKey) {
                mine = true;
                return s;
            }
            if (prev == key) {
                mine = false;
                return s;
            }
        }
        s = (s + 1) & h.mask;
    }
}

constexpr uint32_t kRemote = 0x80000000u;  // cand slot flag: value comes from a remote owner


struct ClaimSink {
    int32_t* ws;
    int32_t* wp;
    uint32_t* wslot;
    unsigned long long* wcount;
    uint64_t* counters;
    uint64_t* live;
    // remote routing (world > 1): keys owned by other ranks
    int rank = 0, world = 1;
    uint64_t* rkeys = nullptr;
    int32_t* rdest = nullptr;
    unsigned long long* rcount = nullptr;
    // dense level (Context::dense_active): slots index the level's exhaustive distance
    // triangle; nothing is claimed or scored, probes are only counted
    const int32_t* dloc = nullptr;
    uint32_t* dbits = nullptr;
    uint64_t dn = 0;
    // fold: misses and the memo's live count are added once per claim phase from wcount
    // (fold_claims_kernel) and hits once per warp at kernel end, instead of three hot
    // global atomics per warp and chunk
    bool fold = false;
    // wl_slots (single rank): a candidate this node claims gets slot kRemote | worklist
    // index, so the merge reads its distance from the worklist-ordered array the screen
    // writes alongside the memo (mostly contiguous), not from a random memo slot
    bool wl_slots = false;
};

__global__ void fold_claims_kernel(const unsigned long long* __restrict__ wcount, uint64_t* __restrict__ counters,
                                   uint64_t* __restrict__ live) {
    counters[C_MISSES] += *wcount;
    *live += *wcount;
}
__device__ __forceinline__ void flush_hits(const ClaimSink& sink, unsigned long long hits) {
    hits = __reduce_add_sync(0xffffffffu, (unsigned)hits);
    if ((threadIdx.x & 31) == 0 && hits) atomicAdd((unsigned long long*)&sink.counters[C_HITS], hits);
}

// row-major upper-triangle index of positions a < b among n (inc/find_best.hpp:78-79)
__device__ __forceinline__ uint64_t tri_index(uint64_t a, uint64_t b, uint64_t n) {
    return a * (2 * n - a - 1) / 2 + (b - a - 1);
}

// Probe of pair (ra, rb) (positions in the dense root) at a dense level: its slot in the
// triangle; the pair's bit is marked (fire-and-forget RED) and the probe counted as a hit.
// dense_recount (find_best.cu) settles the counts once the root is done: of the U marked
// pairs, those F the generation had not scored at a shallower level (absent from the
// distance cache) move from the hits to the misses — the reference's DistanceCache
// misses/hits (inc/model.hpp:54-70) without a round trip per probe.
__device__ __forceinline__ uint32_t dense_probe(uint32_t* __restrict__ dbits, uint64_t dn, uint64_t ra, uint64_t rb) {
    const uint64_t t = ra < rb ? tri_index(ra, rb, dn) : tri_index(rb, ra, dn);
    // marks: a square bit matrix over root positions, row = the probing node (a node's marks
    // of one sweep fall in one row: whole words of its candidate bitset at the root level);
    // dense_recount symmetrises it
    atomicOr(&dbits[ra * ((dn + 31) >> 5) + (rb >> 5)], 1u << (rb & 31));
    return (uint32_t)t;
}

// warp-cooperative claim of one candidate per lane (active lanes given by `valid`).
// Uncached metrics (h.keys == nullptr) claim every candidate into its flat slot.
__device__ __forceinline__ uint32_t claim_warp(HashView h, const ClaimSink& sink, bool valid, int32_t gs,
                                               int32_t gp, uint64_t flat = 0, unsigned* hit_acc = nullptr) {
    bool mine = false, remote = false;
    uint64_t sl = 0;
    int dest = 0;
    const uint64_t key = pair_key(gs, gp);
    if (sink.dloc) {
        if (valid) sl = dense_probe(sink.dbits, sink.dn, (uint64_t)sink.dloc[gs], (uint64_t)sink.dloc[gp]);
        const unsigned hb = __ballot_sync(0xffffffffu, valid);
        if ((threadIdx.x & 31) == 0 && hb)
            atomicAdd((unsigned long long*)&sink.counters[C_HITS], (unsigned long long)__popc(hb));
        return (uint32_t)sl;
    }
    if (valid) {
        if (!h.keys) {
            sl = flat;
            mine = true;
        } else if (sink.world > 1 && (dest = key_owner(key, sink.world)) != sink.rank) {
            remote = true;
        } else {
            sl = cache_claim_k(h, key, mine);
        }
    }
    const int lane = threadIdx.x & 31;
    {
        const unsigned rb = __ballot_sync(0xffffffffu, remote);
        unsigned long long r0 = 0;
        if (lane == 0 && rb) r0 = atomicAdd(sink.rcount, (unsigned long long)__popc(rb));
        r0 = __shfl_sync(0xffffffffu, r0, 0);
        if (remote) {
            const uint64_t at = r0 + __popc(rb & ((1u << lane) - 1));
            sink.rkeys[at] = key;
            sink.rdest[at] = dest;
            sl = kRemote | (uint32_t)at;
        }
    }
    const unsigned ball = __ballot_sync(0xffffffffu, mine);
    const unsigned hits = __ballot_sync(0xffffffffu, valid && !mine && !remote);
    unsigned long long b0 = 0;
    if (lane == 0 && ball) b0 = atomicAdd(sink.wcount, (unsigned long long)__popc(ball));
    b0 = __shfl_sync(0xffffffffu, b0, 0);
    if (mine) {
        const uint64_t at = b0 + __popc(ball & ((1u << lane) - 1));
        sink.ws[at] = gs;
        sink.wp[at] = gp;
        sink.wslot[at] = (uint32_t)sl;
        if (sink.wl_slots) sl = kRemote | (uint32_t)at;
    }
    if (lane == 0 && h.keys) {
        if (ball && !sink.fold) {
            atomicAdd((unsigned long long*)&sink.counters[C_MISSES], (unsigned long long)__popc(ball));
            atomicAdd((unsigned long long*)sink.live, (unsigned long long)__popc(ball));
        }
        if (hits) {
            if (sink.fold && hit_acc)
                *hit_acc += __popc(hits);
            else
                atomicAdd((unsigned long long*)&sink.counters[C_HITS], (unsigned long long)__popc(hits));
        }
    }
    return (uint32_t)sl;
}

// batch claim for a flat query list (init distances)
__global__ void claim_list_kernel(HashView h, ClaimSink sink, const int32_t* __restrict__ qi,
                                  const int32_t* __restrict__ qj, uint64_t n, uint32_t* __restrict__ slot) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = e < n;
    unsigned hit_acc = 0;
    const uint32_t sl = claim_warp(h, sink, valid, valid ? qi[e] : 0, valid ? qj[e] : 0, 0, &hit_acc);
    if (valid) slot[e] = sl;
    if (sink.fold) flush_hits(sink, hit_acc);
}
// the distance behind a candidate slot: a dense level's sparse triangle (D.bits set), a
// worklist / remote answer (kRemote), or the distance memo
__device__ __forceinline__ double slot_value(const DenseView& D, const MemoView& V, const double* __restrict__ rvals,
                                             uint32_t sl) {
    if (D.bits) return dense_value(D, sl);
    return (sl & kRemote) ? rvals[sl & ~kRemote] : memo_value(V, sl);
}
__global__ void gather_vals_kernel(DenseView D, MemoView V, const double* __restrict__ rvals,
                                   const uint32_t* __restrict__ slot, uint64_t n, double* __restrict__ out) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) out[e] = slot_value(D, V, rvals, slot[e]);
}

// ---------------------------------------------------------------- key-sharded cache exchange
__global__ void dest_hist_kernel(const int32_t* __restrict__ dest, uint64_t n, unsigned long long* __restrict__ cnt) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) atomicAdd(&cnt[dest[t]], 1ull);
}
__global__ void gather_u64_kernel(const uint64_t* __restrict__ in, const int32_t* __restrict__ perm, uint64_t n,
                                  uint64_t* __restrict__ out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) out[t] = in[perm[t]];
}
__global__ void scatter_f64_kernel(const double* __restrict__ in, const int32_t* __restrict__ perm, uint64_t n,
                                   double* __restrict__ out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) out[perm[t]] = in[t];
}
// owner side: claim incoming keys (sorted, so worklist runs share their first node)
__global__ void claim_keys_kernel(HashView h, ClaimSink sink, const uint64_t* __restrict__ keys,
                                  const int32_t* __restrict__ idx, uint64_t n, uint32_t* __restrict__ slot_of) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = e < n;
    const uint64_t k = valid ? keys[e] : 0;
    ClaimSink local = sink;
    local.world = 1;  // owner: claim here
    const uint32_t sl = claim_warp(h, local, valid, (int32_t)(k >> 32), (int32_t)(k & 0xffffffffu));
    if (valid) slot_of[idx[e]] = sl;
}
__global__ void answer_kernel(MemoView vals, const uint32_t* __restrict__ slot_of, uint64_t n,
                              double* __restrict__ out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) out[t] = memo_value(vals, slot_of[t]);
}

// ---------------------------------------------------------------- U (capped undirected view)
// out-part: rows of the (sorted) snapshot; in-part appended while rows have room
__global__ void u_out_kernel(const int32_t* __restrict__ gid, uint64_t n, int kw, int cap,
                             int32_t* __restrict__ adj, int32_t* __restrict__ alen) {
    // one thread per entry (coalesced over the rows)
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * (uint64_t)kw) return;
    const uint64_t li = e / kw;
    const int t = (int)(e - li * kw);
    adj[li * cap + t] = gid[e];
    if (t == 0) alen[li] = kw;
}
__global__ void in_keys_kernel(const int32_t* __restrict__ gid, const double* __restrict__ gd,
                               const int32_t* __restrict__ nodes, uint64_t n, int kw,
                               uint32_t* __restrict__ k_tgt, uint64_t* __restrict__ k_d,
                               uint32_t* __restrict__ k_src, int32_t* __restrict__ v_src) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * kw) return;
    const uint64_t li = e / kw;
    k_tgt[e] = (uint32_t)gid[e];
    k_d[e] = dkey(gd[e]);
    k_src[e] = (uint32_t)nodes[li];
    v_src[e] = (int32_t)li;
}
// one thread per target: walk its in-edges in (dist, src) order
__global__ void u_in_kernel(const uint32_t* __restrict__ tgt_sorted, const int32_t* __restrict__ src_sorted,
                            uint64_t ne, uint64_t n, int cap, int32_t* __restrict__ adj,
                            int32_t* __restrict__ alen, const uint64_t* __restrict__ seg_start) {
    const uint64_t lt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (lt >= n) return;
    int32_t* row = adj + lt * cap;
    int len = alen[lt];
    for (uint64_t e = seg_start[lt]; e < ne && tgt_sorted[e] == lt && len < cap; ++e) {
        const int32_t s = src_sorted[e];
        bool dup = false;
        for (int t = 0; t < len; ++t)
            if (row[t] == s) {
                dup = true;
                break;
            }
        if (!dup) row[len++] = s;
    }
    alen[lt] = len;
}
__global__ void seg_start_kernel(const uint32_t* __restrict__ tgt_sorted, uint64_t ne, uint64_t n,
                                 uint64_t* __restrict__ seg_start) {
    const uint64_t lt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (lt >= n) return;
    // lower_bound of lt in tgt_sorted
    uint64_t lo = 0, hi = ne;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (tgt_sorted[mid] < lt) lo = mid + 1; else hi = mid;
    }
    seg_start[lt] = lo;
}

// reverse-list variant (nrg_knn_params.reverse): every in-edge is admitted into a
// separate reverse row (capped), so U = out ∪ in regardless of kw >= scan_floor.
__global__ void u_rev_kernel(const uint32_t* __restrict__ tgt_sorted, const int32_t* __restrict__ src_sorted,
                             uint64_t ne, uint64_t n, int kw, int cap, int32_t* __restrict__ adj,
                             int32_t* __restrict__ alen, const uint64_t* __restrict__ seg_start) {
    const uint64_t lt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (lt >= n) return;
    int32_t* row = adj + lt * cap;
    int len = alen[lt];
    for (uint64_t e = seg_start[lt]; e < ne && tgt_sorted[e] == lt && len < cap; ++e) {
        const int32_t s = src_sorted[e];
        bool dup = false;
        for (int t = 0; t < kw; ++t)
            if (row[t] == s) {
                dup = true;
                break;
            }
        if (!dup) row[len++] = s;
    }
    alen[lt] = len;
}

// Incremental local join (exact under the set semantics): newf[i][a] = 1 when entry a
// of U(i) was not in U(i) in the previous sweep.  A 2-hop path i -> u -> v with both
// hops old was already a candidate of i in the previous sweep of this generation,
// where it lost to i's row; rows only improve and distances are fixed within a
// generation, so it cannot enter now and the gather skips it.  One warp per node.
__global__ void u_new_kernel(const int32_t* __restrict__ adj, const int32_t* __restrict__ alen,
                             const int32_t* __restrict__ adjp, const int32_t* __restrict__ alenp, uint64_t n,
                             int cap, int first, uint8_t* __restrict__ newf) {
    const uint64_t li = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (li >= n) return;
    const int len = alen[li], lenp = first ? 0 : alenp[li];
    const int32_t* row = adj + li * cap;
    const int32_t* prow = adjp + li * cap;
    for (int a = lane; a < len; a += 32) {
        const int32_t v = row[a];
        bool seen = false;
        for (int t = 0; t < lenp && !seen; ++t) seen = prow[t] == v;
        newf[li * cap + a] = seen ? 0 : 1;
    }
}

// ---------------------------------------------------------------- gather + claim
// One CTA per node.  Dedup set in shared memory: open-addressing int hash (tsize
// slots) or a bitmap over the level's n local ids (bitmap == true).
template <int NT>
__global__ void __launch_bounds__(NT) knn_gather_kernel(const int32_t* __restrict__ nodes, uint64_t n,
                                                        const int32_t* __restrict__ adj,
                                                        const int32_t* __restrict__ alen, int cap,
                                                        const int32_t* __restrict__ gid, int kw, bool bitmap,
                                                        int tsize, HashView h, ClaimSink sink,
                                                        uint64_t capn, int32_t* __restrict__ cand_id,
                                                        uint32_t* __restrict__ cand_slot,
                                                        int32_t* __restrict__ cand_cnt, uint64_t lo, int lw,
                                                        const uint8_t* __restrict__ newf, bool do_claim) {
    extern __shared__ int32_t tab[];
    __shared__ int ncand;
    const uint64_t li = lo + blockIdx.x;
    const int tid = threadIdx.x;
    const int words = bitmap ? (int)((n + 31) / 32) : tsize;
    for (int t = tid; t < words; t += NT) tab[t] = bitmap ? 0 : -1;
    if (tid == 0) ncand = 0;
    __syncthreads();
    auto insert = [&](int32_t v) -> bool {
        if (bitmap) {
            const uint32_t bit = 1u << (v & 31);
            return !(atomicOr((uint32_t*)&tab[v >> 5], bit) & bit);
        }
        const uint32_t mask = (uint32_t)tsize - 1;
        uint32_t s = ((uint32_t)v * 2654435761u) & mask;
        for (;;) {
            const int32_t prev = atomicCAS(&tab[s], -1, v);
            if (prev == -1) return true;
            if (prev == v) return false;
            s = (s + 1) & mask;
        }
    };
    // seed with self and the sweep-start list (the `contains` / self checks, :262-264)
    if (tid == 0) insert((int32_t)li);
    for (int t = tid; t < kw; t += NT) insert(gid[li * kw + t]);
    __syncthreads();
    const int32_t* row_i = adj + li * cap;
    const int len_i = alen[li];
    int32_t* my_ids = cand_id + li * capn;
    // 2-hop rows side by side: a group of 2^lw >= cap threads per row
    // (rows wider than a warp: one warp per row, lanes striding it, so the CTA keeps
    // NT/32 rows' dependent loads in flight instead of walking rows one at a time)
    const int gl = lw < 5 ? lw : 5;
    const int gw = 1 << gl;
    const int rows = NT / gw;
    const int r = tid >> gl, b0 = tid & (gw - 1);
    for (int a0 = 0; a0 < len_i; a0 += rows) {
        const int a = a0 + r;
        if (a < len_i) {
            const int32_t lj = row_i[a];
            const int len_j = alen[lj];
            const int32_t* row_j = adj + (uint64_t)lj * cap;
            const bool old_a = !newf[li * cap + a];
            for (int b = b0; b < len_j; b += gw) {
                if (old_a && !newf[(uint64_t)lj * cap + b]) continue;  // old-old: lost last sweep
                const int32_t v = row_j[b];
                if (insert(v)) {
                    const int at = atomicAdd(&ncand, 1);
                    my_ids[at] = v;
                }
            }
        }
    }
    __syncthreads();
    const int cnt = ncand;
    if (!do_claim) {  // cached metrics claim in claim_cands_kernel after the exact reservation
        if (tid == 0) cand_cnt[li] = cnt;
        return;
    }
    // claim (pair_key(nodes[li], nodes[v])) in the per-generation distance cache
    const int32_t gs = nodes[li];
    unsigned hit_acc = 0;
    for (int t0 = 0; t0 < cnt; t0 += NT) {
        const int t = t0 + tid;
        const bool valid = t < cnt;
        const int32_t v = valid ? my_ids[t] : 0;
        const uint32_t sl = claim_warp(h, sink, valid, gs, valid ? nodes[v] : 0, li * capn + t, &hit_acc);
        if (valid) cand_slot[li * capn + t] = sl;
    }
    if (sink.fold) flush_hits(sink, hit_acc);
    if (tid == 0) cand_cnt[li] = cnt;
}

// knn_gather_kernel for narrow levels: one warp per node, WPB nodes per CTA (a
// 32-thread CTA per node caps residency at 32 warps per SM; the claims are bound by the
// latency of DRAM-resident probes, so more warps in flight is what pays)
template <int WPB>
__global__ void __launch_bounds__(32 * WPB) knn_gather_warp_kernel(
    const int32_t* __restrict__ nodes, uint64_t n, const int32_t* __restrict__ adj, const int32_t* __restrict__ alen,
    int cap, const int32_t* __restrict__ gid, int kw, bool bitmap, int tsize, HashView h, ClaimSink sink,
    uint64_t capn, int32_t* __restrict__ cand_id, uint32_t* __restrict__ cand_slot, int32_t* __restrict__ cand_cnt,
    uint64_t lo, uint64_t own, int lw, const uint8_t* __restrict__ newf, bool do_claim) {
    extern __shared__ int32_t tab_all[];
    __shared__ int ncand_s[WPB];
    const int wid = threadIdx.x >> 5, tid = threadIdx.x & 31;
    const uint64_t node = (uint64_t)blockIdx.x * WPB + wid;
    if (node >= own) return;  // whole warp: no block-wide barriers below
    const uint64_t li = lo + node;
    const int words = bitmap ? (int)((n + 31) / 32) : tsize;
    int32_t* tab = tab_all + (size_t)wid * words;
    int& ncand = ncand_s[wid];
    for (int t = tid; t < words; t += 32) tab[t] = bitmap ? 0 : -1;
    if (tid == 0) ncand = 0;
    __syncwarp();
    auto insert = [&](int32_t v) -> bool {
        if (bitmap) {
            const uint32_t bit = 1u << (v & 31);
            return !(atomicOr((uint32_t*)&tab[v >> 5], bit) & bit);
        }
        const uint32_t mask = (uint32_t)tsize - 1;
        uint32_t s = ((uint32_t)v * 2654435761u) & mask;
        for (;;) {
            const int32_t prev = atomicCAS(&tab[s], -1, v);
            if (prev == -1) return true;
            if (prev == v) return false;
            s = (s + 1) & mask;
        }
    };
    if (tid == 0) insert((int32_t)li);
    for (int t = tid; t < kw; t += 32) insert(gid[li * kw + t]);
    __syncwarp();
    const int32_t* row_i = adj + li * cap;
    const int len_i = alen[li];
    int32_t* my_ids = cand_id + li * capn;
    const int gl = lw < 5 ? lw : 5;
    const int gw = 1 << gl;
    const int rows = 32 / gw;
    const int r = tid >> gl, b0 = tid & (gw - 1);
    for (int a0 = 0; a0 < len_i; a0 += rows) {
        const int a = a0 + r;
        if (a < len_i) {
            const int32_t lj = row_i[a];
            const int len_j = alen[lj];
            const int32_t* row_j = adj + (uint64_t)lj * cap;
            const bool old_a = !newf[li * cap + a];
            for (int b = b0; b < len_j; b += gw) {
                if (old_a && !newf[(uint64_t)lj * cap + b]) continue;  // old-old: lost last sweep
                const int32_t v = row_j[b];
                if (insert(v)) {
                    const int at = atomicAdd(&ncand, 1);
                    my_ids[at] = v;
                }
            }
        }
    }
    __syncwarp();
    const int cnt = ncand;
    if (!do_claim) {
        if (tid == 0) cand_cnt[li] = cnt;
        return;
    }
    const int32_t gs = nodes[li];
    unsigned hit_acc = 0;
    for (int t0 = 0; t0 < cnt; t0 += 32) {
        const int t = t0 + tid;
        const bool valid = t < cnt;
        const int32_t v = valid ? my_ids[t] : 0;
        const uint32_t sl = claim_warp(h, sink, valid, gs, valid ? nodes[v] : 0, li * capn + t, &hit_acc);
        if (valid) cand_slot[li * capn + t] = sl;
    }
    if (sink.fold) flush_hits(sink, hit_acc);
    if (tid == 0) cand_cnt[li] = cnt;
}

// claims of the gathered candidates, one warp per node (after cache_reserve sized the
// table for exactly this sweep's candidates)
__global__ void claim_cands_kernel(const int32_t* __restrict__ nodes, HashView h, ClaimSink sink, uint64_t own,
                                   uint64_t lo, uint64_t capn, const int32_t* __restrict__ cand_id,
                                   uint32_t* __restrict__ cand_slot, const int32_t* __restrict__ cand_cnt) {
    const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= own) return;
    const uint64_t li = lo + w;
    const int cnt = cand_cnt[li];
    const int32_t gs = nodes[li];
    for (int t0 = 0; t0 < cnt; t0 += 32) {
        const int t = t0 + lane;
        const bool valid = t < cnt;
        const int32_t v = valid ? cand_id[li * capn + t] : 0;
        const uint32_t sl = claim_warp(h, sink, valid, gs, valid ? nodes[v] : 0, li * capn + t);
        if (valid) cand_slot[li * capn + t] = sl;
    }
}

// the same claims with every candidate in flight at once: blockIdx.y strides a node's
// candidate row in blocks of 256 (wide rows at deep levels: a warp per node walks
// thousands of dependent cache probes one chunk at a time)
__global__ void claim_cands_flat_kernel(const int32_t* __restrict__ nodes, HashView h, ClaimSink sink, uint64_t own,
                                        uint64_t lo, uint64_t capn, const int32_t* __restrict__ cand_id,
                                        uint32_t* __restrict__ cand_slot, const int32_t* __restrict__ cand_cnt) {
    const uint64_t li = lo + blockIdx.x;
    const int cnt = cand_cnt[li];
    const int t = (int)blockIdx.y * blockDim.x + threadIdx.x;
    if ((int)blockIdx.y * (int)blockDim.x >= cnt) return;  // whole block past the row
    const bool valid = t < cnt;
    const int32_t gs = nodes[li];
    const int32_t v = valid ? cand_id[li * capn + t] : 0;
    const uint32_t sl = claim_warp(h, sink, valid, gs, valid ? nodes[v] : 0, li * capn + t);
    if (valid) cand_slot[li * capn + t] = sl;
}

__global__ void sum_counts_kernel(const int32_t* __restrict__ cnt, uint64_t n, unsigned long long* __restrict__ out) {
    unsigned long long a = 0;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x)
        a += (unsigned long long)cnt[t];
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0 && a) atomicAdd(out, a);
}

// ---------------------------------------------------------------- gather, deep levels
// For small levels with wide rows (n <= kBitsMaxN ids, cap >= 32) the 2-hop candidate set
// is an OR of row bitsets: U(j) as a bitset over the level's ids, and new(U(j)) (the
// entries that were not in U(j) last sweep).  cand(i) = OR over a in U(i) of
// (a new in U(i) ? U(a) : new(U(a))) minus i's current row and i itself: the same set
// the incremental join inserts one by one, without contended shared atomics.
// bit-set levels: U(i) as a bitset, then the new flags against last sweep's bitset (the
// set semantics of u_new_kernel, O(1) per entry) and the bitset of new entries
__global__ void u_set_kernel(const int32_t* __restrict__ adj, const int32_t* __restrict__ alen, uint64_t n, int cap,
                             int W, uint32_t* __restrict__ ub) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * (uint64_t)cap) return;
    const uint64_t i = t / cap;
    if ((int)(t - i * cap) >= alen[i]) return;
    const int32_t j = adj[t];
    atomicOr(&ub[i * W + (j >> 5)], 1u << (j & 31));
}
__global__ void u_new_bits_kernel(const int32_t* __restrict__ adj, const int32_t* __restrict__ alen, uint64_t n,
                                  int cap, int W, const uint32_t* __restrict__ ubp, int first,
                                  uint8_t* __restrict__ newf, uint32_t* __restrict__ nb,
                                  uint8_t* __restrict__ hasnew) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * (uint64_t)cap) return;
    const uint64_t i = t / cap;
    if ((int)(t - i * cap) >= alen[i]) return;
    const int32_t j = adj[t];
    const bool fresh = first || !((ubp[i * W + (j >> 5)] >> (j & 31)) & 1u);
    newf[t] = fresh ? 1 : 0;
    if (fresh) {
        atomicOr(&nb[i * W + (j >> 5)], 1u << (j & 31));
        hasnew[i] = 1;
    }
}
// u_set_kernel and u_new_bits_kernel in one pass over the U entries
__global__ void u_bits_kernel(const int32_t* __restrict__ adj, const int32_t* __restrict__ alen, uint64_t n, int cap,
                              int W, uint32_t* __restrict__ ub, const uint32_t* __restrict__ ubp, int first,
                              uint8_t* __restrict__ newf, uint32_t* __restrict__ nb, uint8_t* __restrict__ hasnew) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * (uint64_t)cap) return;
    const uint64_t i = t / cap;
    if ((int)(t - i * cap) >= alen[i]) return;
    const int32_t j = adj[t];
    const uint32_t bit = 1u << (j & 31);
    atomicOr(&ub[i * W + (j >> 5)], bit);
    const bool fresh = first || !(ubp[i * W + (j >> 5)] & bit);
    newf[t] = fresh ? 1 : 0;
    if (fresh) {
        atomicOr(&nb[i * W + (j >> 5)], bit);
        hasnew[i] = 1;
    }
}
constexpr int kBitsMaxN = 32768;
template <int NT>
__global__ void __launch_bounds__(NT) knn_gather_bits_kernel(const int32_t* __restrict__ nodes, uint64_t n,
                                                             const int32_t* __restrict__ adj,
                                                             const int32_t* __restrict__ alen, int cap,
                                                             const int32_t* __restrict__ gid, int kw, int W,
                                                             const uint32_t* __restrict__ ub,
                                                             const uint32_t* __restrict__ nb,
                                                             const uint8_t* __restrict__ newf, HashView h,
                                                             ClaimSink sink, uint64_t capn,
                                                             int32_t* __restrict__ cand_id,
                                                             uint32_t* __restrict__ cand_slot,
                                                             int32_t* __restrict__ cand_cnt, uint64_t lo, bool do_claim,
                                                             const int32_t* __restrict__ rootpos,
                                                             const uint8_t* __restrict__ hasnew,
                                                             bool count_only = false,
                                                             const unsigned long long* __restrict__ sv_off = nullptr,
                                                             const int32_t* __restrict__ sv_id = nullptr,
                                                             int32_t* __restrict__ full_cnt = nullptr,
                                                             int cov_full = 0,
                                                             unsigned long long* __restrict__ cov_short = nullptr) {
    extern __shared__ uint32_t bits_smem[];
    uint32_t* acc = bits_smem;     // OR of the 2-hop rows
    uint32_t* excl = acc + W;      // i's current row and i itself
    int32_t* srcs = reinterpret_cast<int32_t*>(excl + W);  // rows to OR: 2 lj + (row is new in U(i))
    __shared__ int s_nsrc;
    typedef cub::BlockScan<int, NT> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int s_total;
    const uint64_t li = lo + blockIdx.x;
    const int tid = threadIdx.x;
    for (int w = tid; w < W; w += NT) acc[w] = excl[w] = 0u;
    if (tid == 0) s_nsrc = 0;
    __syncthreads();
    if (tid == 0) atomicOr(&excl[li >> 5], 1u << (li & 31));
    for (int t = tid; t < kw; t += NT) {
        const int32_t v = gid[li * kw + t];
        atomicOr(&excl[v >> 5], 1u << (v & 31));
    }
    const int32_t* row_i = adj + li * cap;
    const int len_i = alen[li];
    // the rows that contribute: U(a) for a new in U(i), new(U(a)) for an old a that has new
    // entries (an old a without any contributes nothing: its new-bitset is empty)
    for (int a = tid; a < len_i; a += NT) {
        const int32_t lj = row_i[a];
        const bool nw = newf[li * cap + a] != 0;
        if (nw || hasnew[lj]) srcs[atomicAdd(&s_nsrc, 1)] = 2 * lj + (nw ? 1 : 0);
    }
    __syncthreads();
    const int nsrc = s_nsrc;
    if (2 * cap < W) {
        // rows shorter than the bitsets: walk the source rows' entries (a warp per row,
        // lanes over entries) into the shared bitmap instead of reading W words per row
        const int lane = tid & 31, wid = tid >> 5;
        for (int q = wid; q < nsrc; q += NT / 32) {
            const int32_t e = srcs[q];
            const uint64_t lj = (uint64_t)(e >> 1);
            const int len_j = alen[lj];
            const int32_t* row_j = adj + lj * cap;
            const uint8_t* nf_j = newf + lj * cap;
            for (int b = lane; b < len_j; b += 32) {
                if (!(e & 1) && !nf_j[b]) continue;  // old hop: only its new entries
                const int32_t v = row_j[b];
                atomicOr(&acc[v >> 5], 1u << (v & 31));
            }
        }
    } else if (W <= NT) {
        // G threads per word, each ORs every G-th row into a register
        const int G = NT / W;
        const int w = tid % W, g = tid / W;
        if (g < G) {
            uint32_t r = 0u;
            for (int q = g; q < nsrc; q += G) {
                const int32_t e = srcs[q];
                r |= ((e & 1) ? ub : nb)[(uint64_t)(e >> 1) * W + w];
            }
            if (r) atomicOr(&acc[w], r);
        }
    } else {
        for (int w = tid; w < W; w += NT) {
            uint32_t r = 0u;
            for (int q = 0; q < nsrc; ++q) {
                const int32_t e = srcs[q];
                r |= ((e & 1) ? ub : nb)[(uint64_t)(e >> 1) * W + w];
            }
            acc[w] = r;
        }
    }
    __syncthreads();
    // candidate ids in increasing order: popcounts of the thread's words, block scan
    constexpr int kMaxWpt = kBitsMaxN / 32 / NT + 1;
    int cnt = 0;
    uint32_t cw[kMaxWpt];
#pragma unroll
    for (int q = 0; q < kMaxWpt; ++q) {
        const int w = tid * kMaxWpt + q;
        cw[q] = w < W ? (acc[w] & ~excl[w]) : 0u;
        cnt += __popc(cw[q]);
    }
    int off = 0, total = 0;
    Scan(scan_tmp).ExclusiveSum(cnt, off, total);
    if (count_only) {  // the size of the candidate set only (the coverage test of a dense level)
        if (tid == 0) cand_cnt[li] = total;
        return;
    }
    int32_t* my_ids = cand_id + li * capn;
    constexpr int kSvMax = 256, kEarlyMax = 512;
    if (rootpos && sv_off && (int)(sv_off[li + 1] - sv_off[li]) <= kSvMax &&
        (uint64_t)(sv_off[li + 1] - sv_off[li]) + (uint64_t)kw <= min((uint64_t)kEarlyMax, capn)) {
        // Dense level, short list.  Every pair outside the screen's survivor list ties at
        // -base, and among tied candidates only the kw smallest ids can enter a row; so the
        // merge needs the node's survivors that are candidates plus the first kw other
        // candidates -- a list of kw + a few entries instead of thousands (same merged row,
        // same churn; the resolve and merge kernels read it unchanged).  Every candidate is
        // still probed (marked and counted).
        __shared__ int32_t s_sv[kSvMax];
        __shared__ int32_t s_early[kEarlyMax];  // the first kw + sdeg candidates, in id order
        __shared__ int s_n;
        uint32_t* my_slot = cand_slot + li * capn;
        const uint64_t ra = (uint64_t)rootpos[li];
        const unsigned long long s0 = sv_off[li];
        const int sdeg = (int)(sv_off[li + 1] - s0);
        const int need = kw + sdeg;
        if (tid == 0) s_n = 0;
        __syncthreads();
        // the node's survivors that are candidates (the others do not take part)
        for (int e = tid; e < sdeg; e += NT) {
            const int32_t v = sv_id[s0 + e];
            const bool isc = (acc[v >> 5] & ~excl[v >> 5]) >> (v & 31) & 1u;
            s_sv[e] = isc ? v : -1;
            if (isc) {
                const int at = atomicAdd(&s_n, 1);
                my_ids[at] = v;
                const uint64_t rb = (uint64_t)rootpos[v];
                my_slot[at] = (uint32_t)(ra < rb ? tri_index(ra, rb, sink.dn) : tri_index(rb, ra, sink.dn));
            }
        }
        // marks go into row ra of the square matrix: at the dense root itself (local id = root
        // position) a candidate word is a word of that row; deeper, consecutive candidates
        // that share a word go out together
        const bool ident = sink.dn == n;
        uint32_t* mrow = sink.dbits + ra * ((sink.dn + 31) >> 5);
        uint64_t pw = ~0ull;
        uint32_t pbits = 0u;
#pragma unroll
        for (int q = 0; q < kMaxWpt; ++q) {
            const int w = tid * kMaxWpt + q;
            const uint32_t m = cw[q];
            if (!m) continue;
            if (off < need) {
                int o = off;
                for (uint32_t mm = m; mm && o < need; mm &= mm - 1, ++o) s_early[o] = 32 * w + __ffs(mm) - 1;
            }
            off += __popc(m);
            if (ident) {
                atomicOr(&mrow[w], m);
            } else {
                for (uint32_t mm = m; mm; mm &= mm - 1) {
                    const uint64_t rb = (uint64_t)rootpos[32 * w + __ffs(mm) - 1];
                    if ((rb >> 5) != pw) {
                        if (pbits) atomicOr(&mrow[pw], pbits);
                        pw = rb >> 5;
                        pbits = 0u;
                    }
                    pbits |= 1u << (rb & 31);
                }
            }
        }
        if (pbits) atomicOr(&mrow[pw], pbits);
        if (tid == 0 && total) atomicAdd((unsigned long long*)&sink.counters[C_HITS], (unsigned long long)total);
        __syncthreads();
        // rank of an early candidate among the candidates outside the survivor list
        const int nearly = min(total, need);
        for (int e = tid; e < nearly; e += NT) {
            const int32_t v = s_early[e];
            int below = 0;
            bool is_sv = false;
            for (int u = 0; u < sdeg; ++u) {
                const int32_t x = s_sv[u];
                is_sv |= x == v;
                below += (x >= 0 && x < v) ? 1 : 0;
            }
            if (!is_sv && e - below < kw) {
                const int at = atomicAdd(&s_n, 1);
                my_ids[at] = v;
                const uint64_t rb = (uint64_t)rootpos[v];
                my_slot[at] = (uint32_t)(ra < rb ? tri_index(ra, rb, sink.dn) : tri_index(rb, ra, sink.dn));
            }
        }
        __syncthreads();
        if (tid == 0) {
            cand_cnt[li] = s_n;
            full_cnt[li] = total;
            if (cov_short && total < cov_full) atomicAdd(cov_short, 1ull);  // a node short of full coverage
        }
        return;
    }
    if (rootpos) {
        // dense level: slots in the root's distance triangle, probes marked and counted here
        uint32_t* my_slot = cand_slot + li * capn;
        const uint64_t ra = (uint64_t)rootpos[li];
#pragma unroll
        for (int q = 0; q < kMaxWpt; ++q) {
            const int w = tid * kMaxWpt + q;
            for (uint32_t m = cw[q]; m; m &= m - 1) {
                const int v = 32 * w + __ffs(m) - 1;
                my_ids[off] = v;
                my_slot[off++] = dense_probe(sink.dbits, sink.dn, ra, (uint64_t)rootpos[v]);
            }
        }
        const int probes = warp_sum(cnt);
        if ((tid & 31) == 0 && probes)
            atomicAdd((unsigned long long*)&sink.counters[C_HITS], (unsigned long long)probes);
        if (tid == 0) {
            cand_cnt[li] = total;
            if (full_cnt) full_cnt[li] = total;
            if (cov_short && total < cov_full) atomicAdd(cov_short, 1ull);
        }
        return;
    }
#pragma unroll
    for (int q = 0; q < kMaxWpt; ++q) {
        const int w = tid * kMaxWpt + q;
        for (uint32_t m = cw[q]; m; m &= m - 1) my_ids[off++] = 32 * w + __ffs(m) - 1;
    }
    if (tid == 0) s_total = total;
    __syncthreads();
    const int ncand = s_total;
    if (tid == 0 && cov_short && ncand < cov_full) atomicAdd(cov_short, 1ull);
    if (!do_claim) {
        if (tid == 0) cand_cnt[li] = ncand;
        return;
    }
    const int32_t gs = nodes[li];
    for (int t0 = 0; t0 < ncand; t0 += NT) {
        const int t = t0 + tid;
        const bool valid = t < ncand;
        const int32_t v = valid ? my_ids[t] : 0;
        const uint32_t sl = claim_warp(h, sink, valid, gs, valid ? nodes[v] : 0, li * capn + t);
        if (valid) cand_slot[li * capn + t] = sl;
    }
    if (tid == 0) cand_cnt[li] = ncand;
}

// ---------------------------------------------------------------- merge top-kw
// One CTA per node: keep the (dist,id)-smallest kw of (current row U candidates).
// Candidates are consumed in blocks of (buf_cap - kw); those beating the current
// worst are appended after the row, and the new row is selected by rank: entries are
// distinct in (dist, global id), so an entry's rank is the number of entries ahead of
// it and the ranks < kw are the new row, in order (one barrier; blocks of more than 96
// entries are bitonic-sorted instead).
// Counts entries that came from the candidate set (churn).
template <int NT>
__global__ void __launch_bounds__(NT) knn_merge_kernel(const int32_t* __restrict__ nodes, uint64_t n,
                                                       int32_t* __restrict__ gid, double* __restrict__ gd, int kw,
                                                       const int32_t* __restrict__ cand_id,
                                                       const uint32_t* __restrict__ cand_slot,
                                                       const int32_t* __restrict__ cand_cnt, uint64_t capn,
                                                       DenseView D, MemoView cvals,
                                                       const double* __restrict__ rvals, int buf_cap,
                                                       unsigned long long* __restrict__ churn, uint64_t lo) {
    extern __shared__ unsigned char smem_raw[];
    double* bd = reinterpret_cast<double*>(smem_raw);
    double* od = bd + buf_cap;                               // selected row (kw)
    int32_t* bi = reinterpret_cast<int32_t*>(od + kw);       // local id
    int32_t* bg = bi + buf_cap;                               // global id (tie order)
    int32_t* bo = bg + buf_cap;                               // origin: 1 = candidate
    int32_t* oi = bo + buf_cap;
    int32_t* og = oi + kw;
    int32_t* oo = og + kw;
    __shared__ int nb;
    const uint64_t li = lo + blockIdx.x;
    const int tid = threadIdx.x;
    const int cnt = cand_cnt[li];
    if (cnt == 0) return;
    int32_t* row_id = gid + li * kw;
    double* row_d = gd + li * kw;
    for (int t = tid; t < kw; t += NT) {
        bd[t] = row_d[t];
        bi[t] = row_id[t];
        bg[t] = nodes[row_id[t]];
        bo[t] = 0;
    }
    __syncthreads();
    const int B = buf_cap - kw;
    bool changed_any = false;
    for (int blk = 0; blk < cnt; blk += B) {
        if (tid == 0) nb = kw;
        __syncthreads();
        const double wd = bd[kw - 1];
        const int wg = bg[kw - 1];
        const int end = min(cnt, blk + B);
        for (int t = blk + tid; t < end; t += NT) {
            const int32_t v = cand_id[li * capn + t];
            const uint32_t sl = cand_slot[li * capn + t];
            const double d = slot_value(D, cvals, rvals, sl);
            const int g = nodes[v];
            if (entry_less(d, g, wd, wg)) {
                const int at = atomicAdd(&nb, 1);
                bd[at] = d;
                bi[at] = v;
                bg[at] = g;
                bo[at] = 1;
            }
        }
        __syncthreads();
        const int m = nb;
        if (m == kw) continue;  // nothing beats the worst
        changed_any = true;
        if (m > 96) {  // large blocks (first sweeps, wide rows): bitonic sort of the buffer
            int P = 1;
            while (P < m) P <<= 1;
            for (int t = m + tid; t < P; t += NT) {
                bd[t] = INFINITY;
                bg[t] = 0x7fffffff;
                bi[t] = -1;
                bo[t] = 0;
            }
            __syncthreads();
            for (int k2 = 2; k2 <= P; k2 <<= 1) {
                for (int j = k2 >> 1; j > 0; j >>= 1) {
                    for (int t = tid; t < P; t += NT) {
                        const int ixj = t ^ j;
                        if (ixj > t) {
                            const bool up = (t & k2) == 0;
                            const bool gt = entry_less(bd[ixj], bg[ixj], bd[t], bg[t]);
                            if (gt == up) {
                                const double td = bd[t]; bd[t] = bd[ixj]; bd[ixj] = td;
                                const int ti = bi[t]; bi[t] = bi[ixj]; bi[ixj] = ti;
                                const int tg = bg[t]; bg[t] = bg[ixj]; bg[ixj] = tg;
                                const int to = bo[t]; bo[t] = bo[ixj]; bo[ixj] = to;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            continue;
        }
        for (int t = tid; t < m; t += NT) {
            const double d = bd[t];
            const int g = bg[t];
            int r = 0;
            for (int j = 0; j < m; ++j) r += entry_less(bd[j], bg[j], d, g) ? 1 : 0;
            if (r < kw) {
                od[r] = d;
                oi[r] = bi[t];
                og[r] = g;
                oo[r] = bo[t];
            }
        }
        __syncthreads();
        for (int t = tid; t < kw; t += NT) {
            bd[t] = od[t];
            bi[t] = oi[t];
            bg[t] = og[t];
            bo[t] = oo[t];
        }
        __syncthreads();
    }
    if (!changed_any) return;
    int ch = 0;
    for (int t = tid; t < kw; t += NT) {
        row_d[t] = bd[t];
        row_id[t] = bi[t];
        ch += bo[t];
    }
    ch = warp_sum(ch);
    if ((tid & 31) == 0 && ch) atomicAdd(churn, (unsigned long long)ch);
}

// Narrow rows (kw <= 64): one warp per node, 8 nodes per CTA, so many more merges are in
// flight than with a 32-thread CTA per node (the resident-CTA limit).  Candidates are
// consumed 64 at a time; those beating the current worst are ballot-compacted after the
// row and the new row is selected by rank (as knn_merge_kernel).
constexpr int kMergeWarps = 8;
constexpr int kMergeBlk = 64;
__global__ void __launch_bounds__(32 * kMergeWarps) knn_merge_warp_kernel(
    const int32_t* __restrict__ nodes, uint64_t n, int32_t* __restrict__ gid, double* __restrict__ gd, int kw,
    const int32_t* __restrict__ cand_id, const uint32_t* __restrict__ cand_slot,
    const int32_t* __restrict__ cand_cnt, uint64_t capn, DenseView D, MemoView cvals,
    const double* __restrict__ rvals, unsigned long long* __restrict__ churn, uint64_t lo, uint64_t own) {
    extern __shared__ unsigned char merge_warp_smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t node = (uint64_t)blockIdx.x * kMergeWarps + wib;
    if (node >= own) return;
    const uint64_t li = lo + node;
    const int cnt = cand_cnt[li];
    if (cnt == 0) return;
    const int cap = kw + kMergeBlk;
    unsigned char* base = merge_warp_smem + (size_t)wib * ((size_t)cap + kw) * 20;
    double* bd = reinterpret_cast<double*>(base);
    double* od = bd + cap;
    int32_t* bi = reinterpret_cast<int32_t*>(od + kw);
    int32_t* bg = bi + cap;
    int32_t* bo = bg + cap;
    int32_t* oi = bo + cap;
    int32_t* og = oi + kw;
    int32_t* oo = og + kw;
    int32_t* row_id = gid + li * kw;
    double* row_d = gd + li * kw;
    for (int t = lane; t < kw; t += 32) {
        bd[t] = row_d[t];
        bi[t] = row_id[t];
        bg[t] = nodes[row_id[t]];
        bo[t] = 0;
    }
    __syncwarp();
    bool changed_any = false;
    for (int blk = 0; blk < cnt; blk += kMergeBlk) {
        const double wd = bd[kw - 1];
        const int wg = bg[kw - 1];
        int m = kw;
        // the block's candidates (kMergeBlk / 32 per lane) are all loaded before any is
        // compared: their dependent loads (slot -> cached distance, id -> global id) are
        // in flight together instead of one 32-wide step at a time
        constexpr int kPer = kMergeBlk / 32;
        double dv[kPer];
        int32_t vv[kPer], gv[kPer];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int t = blk + 32 * q + lane;
            dv[q] = 0.0;
            vv[q] = gv[q] = 0;
            if (t < cnt) {
                vv[q] = cand_id[li * capn + t];
                const uint32_t sl = cand_slot[li * capn + t];
                dv[q] = slot_value(D, cvals, rvals, sl);
                gv[q] = nodes[vv[q]];
            }
        }
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int t = blk + 32 * q + lane;
            const bool better = t < cnt && entry_less(dv[q], gv[q], wd, wg);
            const unsigned bal = __ballot_sync(0xffffffffu, better);
            if (better) {
                const int at = m + __popc(bal & ((1u << lane) - 1u));
                bd[at] = dv[q];
                bi[at] = vv[q];
                bg[at] = gv[q];
                bo[at] = 1;
            }
            m += __popc(bal);
        }
        __syncwarp();
        if (m == kw) continue;  // nothing beats the worst
        changed_any = true;
        for (int t = lane; t < m; t += 32) {
            const double d = bd[t];
            const int g = bg[t];
            int r = 0;
            for (int j = 0; j < m; ++j) r += entry_less(bd[j], bg[j], d, g) ? 1 : 0;
            if (r < kw) {
                od[r] = d;
                oi[r] = bi[t];
                og[r] = g;
                oo[r] = bo[t];
            }
        }
        __syncwarp();
        for (int t = lane; t < kw; t += 32) {
            bd[t] = od[t];
            bi[t] = oi[t];
            bg[t] = og[t];
            bo[t] = oo[t];
        }
        __syncwarp();
    }
    if (!changed_any) return;
    int ch = 0;
    for (int t = lane; t < kw; t += 32) {
        row_d[t] = bd[t];
        row_id[t] = bi[t];
        ch += bo[t];
    }
    ch = warp_sum(ch);
    if (lane == 0 && ch) atomicAdd(churn, (unsigned long long)ch);
}

// ---------------------------------------------------------------- exhaustive
// rows of (id-sorted) candidates with distances from the triangular array
__global__ void exh_fill2_kernel(const int32_t* __restrict__ sorted_loc, const int32_t* __restrict__ rank,
                                 uint64_t n, const double* __restrict__ tri, uint64_t* __restrict__ keys,
                                 int32_t* __restrict__ vals) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * (n - 1)) return;
    const uint64_t li = e / (n - 1), t = e % (n - 1);
    const uint64_t self = (uint64_t)rank[li];
    const uint64_t pos = t < self ? t : t + 1;
    const uint64_t lj = (uint64_t)sorted_loc[pos];
    const uint64_t a = li < lj ? li : lj, b = li < lj ? lj : li;
    // row-major upper triangle offset of (a, b)
    const uint64_t off = a * (2 * n - a - 1) / 2 + (b - a - 1);
    keys[e] = dkey(tri[off]);
    vals[e] = (int32_t)lj;
}
__global__ void exh_take_kernel(const uint64_t* __restrict__ keys, const int32_t* __restrict__ vals,
                                uint64_t n, int k, const int32_t* __restrict__ nodes,
                                int32_t* __restrict__ out_id, double* __restrict__ out_d) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * (uint64_t)k) return;
    const uint64_t li = e / k, t = e % k;
    out_id[e] = nodes[vals[li * (n - 1) + t]];
    out_d[e] = dkey_inv(keys[li * (n - 1) + t]);
}
__global__ void seg_offsets_kernel(int* __restrict__ off, uint64_t nseg, uint64_t len) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t <= nseg) off[t] = (int)(t * len);
}

static void knn_exhaustive(Context& c, int mode, int k, const int32_t* d_nodes, uint64_t n,
                           const int32_t* sorted_loc, const int32_t* rank, KnnResultD& out, DevBuf& ids_buf,
                           DevBuf& dist_buf) {
    const uint64_t np = n * (n - 1) / 2;
    double* tri = c.s_h.as<double>(np);
    score_all_pairs(c, mode, d_nodes, n, tri);
    const uint64_t ne = n * (n - 1);
    if (ne > (uint64_t)INT32_MAX) fail(100, "exhaustive kNN too large for one segmented sort");
    uint64_t* keys = c.s_i.as<uint64_t>(ne);
    int32_t* vals = c.s_j.as<int32_t>(ne);
    uint64_t* keys2 = c.s_f.as<uint64_t>(ne);
    int32_t* vals2 = c.s_g.as<int32_t>(ne);
    exh_fill2_kernel<<<(unsigned)ceil_div(ne, 256), 256, 0, c.stream>>>(sorted_loc, rank, n, tri, keys, vals);
    int* off = c.s_e.as<int>(n + 1);
    seg_offsets_kernel<<<(unsigned)ceil_div(n + 1, 256), 256, 0, c.stream>>>(off, n, n - 1);
    NRG_LAUNCH_CHECK();
    size_t tmp = 0;
    cub::DeviceSegmentedSort::StableSortPairs(nullptr, tmp, keys, keys2, vals, vals2, (int)ne, (int)n, off,
                                              off + 1, c.stream);
    void* dtmp = c.s_k.ensure(tmp);
    cub::DeviceSegmentedSort::StableSortPairs(dtmp, tmp, keys, keys2, vals, vals2, (int)ne, (int)n, off, off + 1,
                                              c.stream);
    out.k = k;
    out.sweeps = 0;
    out.churn.clear();
    out.ids = ids_buf.as<int32_t>(n * k);
    out.dists = dist_buf.as<double>(n * k);
    exh_take_kernel<<<(unsigned)ceil_div(n * k, 256), 256, 0, c.stream>>>(keys2, vals2, n, k, d_nodes, out.ids,
                                                                        out.dists);
    NRG_LAUNCH_CHECK();
    c.sync();
}


// ---------------------------------------------------------------- in-edge order
template <class T>
__global__ void gather_kernel(const T* __restrict__ in, const int32_t* __restrict__ perm, uint64_t n,
                              T* __restrict__ out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) out[t] = in[perm[t]];
}

// in-edges ordered by (target, dist, source id) — the per-target (dist, src) order of
// inc/knn.hpp:234-246 — by three stable LSD radix passes over a permutation
static void in_edge_sort(Context& c, uint64_t ne, const uint32_t* tgt, const uint64_t* dk, const uint32_t* src,
                         const int32_t* srcloc, uint32_t* tgt_sorted, int32_t* src_sorted, DevBuf& pa,
                         DevBuf& pb, DevBuf& k64, DevBuf& k32, DevBuf& tmpb) {
    int32_t* p0 = pa.as<int32_t>(ne);
    int32_t* p1 = pb.as<int32_t>(ne);
    uint64_t* kbuf = k64.as<uint64_t>(2 * ne);
    uint32_t* kb32 = k32.as<uint32_t>(2 * ne);
    const unsigned g = (unsigned)ceil_div(ne, 256);
    iota_kernel<<<g, 256, 0, c.stream>>>(p0, ne);
    size_t t1 = 0, t2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, kb32, kb32 + ne, p0, p1, (int)ne, 0, 32, c.stream);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, kbuf, kbuf + ne, p0, p1, (int)ne, 0, 64, c.stream);
    void* tmp = tmpb.ensure(std::max(t1, t2));
    // pass 1: source id
    cub::DeviceRadixSort::SortPairs(tmp, t1, src, kb32 + ne, p0, p1, (int)ne, 0, 32, c.stream);
    // pass 2: dist (stable)
    gather_kernel<uint64_t><<<g, 256, 0, c.stream>>>(dk, p1, ne, kbuf);
    cub::DeviceRadixSort::SortPairs(tmp, t2, kbuf, kbuf + ne, p1, p0, (int)ne, 0, 64, c.stream);
    // pass 3: target (stable)
    gather_kernel<uint32_t><<<g, 256, 0, c.stream>>>(tgt, p0, ne, kb32);
    cub::DeviceRadixSort::SortPairs(tmp, t1, kb32, tgt_sorted, p0, p1, (int)ne, 0, 32, c.stream);
    gather_kernel<int32_t><<<g, 256, 0, c.stream>>>(srcloc, p1, ne, src_sorted);
    NRG_LAUNCH_CHECK();
}


// ---------------------------------------------------------------- key-sharded exchange (host)
struct ExchangeBufs {
    DevBuf rkeys, rdest, rcount, perm, perm2, dsorted, skeys, hist, recv_keys, ridx, sorted_keys, sorted_idx, slot_of,
        ans, resp, rvals, ws2, wp2, wsl2, tmp;
};

static void score_claimed(Context& c, int mode, int32_t* ws, int32_t* wp, uint32_t* wslot, uint64_t nw);

// Route the remote requests of the last claim phase to their owner ranks, claim them
// there, score every pair this rank claimed (local + remote), answer the requests.
// On return X.rvals holds the distance of request r (slot kRemote | r) of this rank.
static void exchange_and_score(Context& c, int mode, const ClaimSink& sink, uint64_t nw_local, ExchangeBufs& X,
                               uint64_t reserve_hint) {
    Comm* comm = static_cast<Comm*>(c.comm);
    const int W = c.world, me = c.rank;
    unsigned long long R = 0;
    if (W > 1) {
        R = c.read_scalar(sink.rcount);
    }
    (void)reserve_hint;
    if (W == 1) {
        score_claimed(c, mode, sink.ws, sink.wp, sink.wslot, nw_local);
        return;
    }
    // 1. requests grouped by owner rank
    int32_t* perm = X.perm.as<int32_t>(R + 1);
    int32_t* perm2 = X.perm2.as<int32_t>(R + 1);
    int32_t* dsorted = X.dsorted.as<int32_t>(R + 1);
    uint64_t* skeys = X.skeys.as<uint64_t>(R + 1);
    unsigned long long* hist = X.hist.as<unsigned long long>(W);
    NRG_CUDA(cudaMemsetAsync(hist, 0, 8 * W, c.stream));
    if (R) {
        iota_kernel<<<(unsigned)ceil_div(R, 256), 256, 0, c.stream>>>(perm, R);
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, sink.rdest, dsorted, perm, perm2, (int64_t)R, 0, 16, c.stream);
        void* tmp = X.tmp.ensure(tb);
        cub::DeviceRadixSort::SortPairs(tmp, tb, sink.rdest, dsorted, perm, perm2, (int64_t)R, 0, 16, c.stream);
        dest_hist_kernel<<<(unsigned)ceil_div(R, 256), 256, 0, c.stream>>>(sink.rdest, R, hist);
        gather_u64_kernel<<<(unsigned)ceil_div(R, 256), 256, 0, c.stream>>>(sink.rkeys, perm2, R, skeys);
        NRG_LAUNCH_CHECK_N(3);
    }
    std::vector<uint64_t> cnt(W), mat((size_t)W * W, 0);
    NRG_CUDA(cudaMemcpyAsync(cnt.data(), hist, 8 * W, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    for (int d = 0; d < W; ++d) mat[(size_t)me * W + d] = cnt[d];
    comm->allreduce_u64(mat.data(), W * W, false, c.stream);
    std::vector<size_t> sb, so, rb, ro;
    const uint64_t Q = route_plan(W, me, mat.data(), sb, so, rb, ro);
    uint64_t* recv_keys = X.recv_keys.as<uint64_t>(Q + 1);
    comm->alltoallv(skeys, sb, so, recv_keys, rb, ro, c.stream);
    // 2. owner side: claim (key-sorted for K1 locality), score local + remote claims
    uint32_t* slot_of = X.slot_of.as<uint32_t>(Q + 1);
    int32_t* ws2 = X.ws2.as<int32_t>(Q + 1);
    int32_t* wp2 = X.wp2.as<int32_t>(Q + 1);
    uint32_t* wsl2 = X.wsl2.as<uint32_t>(Q + 1);
    unsigned long long nw2 = 0;
    if (Q) {
        int32_t* ridx = X.ridx.as<int32_t>(Q);
        uint64_t* sk = X.sorted_keys.as<uint64_t>(Q);
        int32_t* si = X.sorted_idx.as<int32_t>(Q);
        iota_kernel<<<(unsigned)ceil_div(Q, 256), 256, 0, c.stream>>>(ridx, Q);
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, recv_keys, sk, ridx, si, (int64_t)Q, 0, 64, c.stream);
        void* tmp = X.tmp.ensure(tb);
        cub::DeviceRadixSort::SortPairs(tmp, tb, recv_keys, sk, ridx, si, (int64_t)Q, 0, 64, c.stream);
        ClaimSink s2 = sink;
        s2.ws = ws2;
        s2.wp = wp2;
        s2.wslot = wsl2;
        s2.wcount = sink.wcount + 1;
        NRG_CUDA(cudaMemsetAsync(s2.wcount, 0, 8, c.stream));
        claim_keys_kernel<<<(unsigned)ceil_div(Q, 256), 256, 0, c.stream>>>(c.Cview(), s2, sk, si, Q, slot_of);
        NRG_LAUNCH_CHECK_N(2);
        nw2 = c.read_scalar(s2.wcount);
    }
    score_claimed(c, mode, sink.ws, sink.wp, sink.wslot, nw_local);
    score_claimed(c, mode, ws2, wp2, wsl2, nw2);
    // 3. answers back to the requesters, scattered into request order
    double* ans = X.ans.as<double>(Q + 1);
    double* resp = X.resp.as<double>(R + 1);
    double* rvals = X.rvals.as<double>(R + 1);
    if (Q) {
        answer_kernel<<<(unsigned)ceil_div(Q, 256), 256, 0, c.stream>>>(c.mview(), slot_of, Q, ans);
        NRG_LAUNCH_CHECK();
    }
    comm->alltoallv(ans, rb, ro, resp, sb, so, c.stream);
    if (R) {
        scatter_f64_kernel<<<(unsigned)ceil_div(R, 256), 256, 0, c.stream>>>(resp, perm2, R, rvals);
        NRG_LAUNCH_CHECK();
    }
}

// nodes whose candidate count falls short of every other node outside the row
__global__ void coverage_kernel(const int32_t* __restrict__ cand_cnt, uint64_t own, int full,
                                unsigned long long* __restrict__ short_nodes) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool sh = t < own && cand_cnt[t] < full;
    const unsigned b = __ballot_sync(0xffffffffu, sh);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(short_nodes, (unsigned long long)__popc(b));
}

// ---------------------------------------------------------------- covered dense levels
// A dense FindBest level (distances from the level's exhaustive triangle) whose FIRST sweep
// gives every node the whole level as candidates (deep levels: cap^2 >= n) ends with each row
// the exact top-kw of the level, the next sweep settled (churn 0), every pair of the level
// probed once from each side, and every survivor among the level's pairs refined.  All of
// that follows from the coverage alone, so when the candidate-set SIZES (the OR of the
// U-row bitsets, no candidate lists) show full coverage the level is finished directly:
// probe marks by rows of the triangle, the survivors' refinement from the screen's
// worklist, and the rows from each node's few survivors plus the smallest ids (every other
// pair ties at -base).  Same rows, sweeps, churn, marks, hit and eval counts as the sweeps
// (tests/test_gpu_search.py::test_dense_levels_equal_claim_path).
__global__ void cover_members_kernel(const int32_t* __restrict__ rootpos, uint64_t n, uint32_t* __restrict__ M) {
    const uint64_t a = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a < n) atomicOr(&M[rootpos[a] >> 5], 1u << (rootpos[a] & 31));
}
// every pair of the level probed from both sides: row ra of the square mark matrix takes the
// level's member mask (without ra itself)
__global__ void cover_mark_kernel(const int32_t* __restrict__ rootpos, uint64_t n, uint64_t dn,
                                  const uint32_t* __restrict__ M, uint32_t* __restrict__ dbits) {
    const uint64_t a = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (a >= n) return;
    const uint64_t ra = (uint64_t)rootpos[a], Wd = (dn + 31) >> 5;
    for (uint64_t w = lane; w < Wd; w += 32) {
        uint32_t val = M[w];
        if (w == (ra >> 5)) val &= ~(1u << (ra & 31));
        if (val) atomicOr(&dbits[ra * Wd + w], val);
    }
}
// the screen's worklist entries with both endpoints in the level: claim the pair for the
// lazy K2, and count / fill the two endpoints' survivor lists (a pair listed twice -- a
// survivor that is also an existing coupling -- is taken once: `seen` over triangle slots)
__global__ void cover_worklist_kernel(DenseResolve R, const int32_t* __restrict__ es, const int32_t* __restrict__ ep,
                                      const uint32_t* __restrict__ wrank, uint64_t nw,
                                      const int32_t* __restrict__ loc, const int32_t* __restrict__ dloc, uint64_t dn,
                                      uint32_t* __restrict__ seen, uint8_t* __restrict__ keep,
                                      unsigned long long* __restrict__ deg, const unsigned long long* __restrict__ off,
                                      int32_t* __restrict__ adj_id, uint32_t* __restrict__ adj_rank, int pass,
                                      bool claim) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nw) return;
    const int32_t u = es[e], v = ep[e];
    const int32_t a = loc[u], b = loc[v];
    if (pass == 0) {
        keep[e] = 0;
        if (a < 0 || b < 0) return;
        const uint64_t ra = (uint64_t)dloc[u], rb = (uint64_t)dloc[v];
        const uint64_t t = ra < rb ? tri_index(ra, rb, dn) : tri_index(rb, ra, dn);
        const uint32_t bit = 1u << (t & 31);
        if (atomicOr(&seen[t >> 5], bit) & bit) return;
        keep[e] = 1;
        if (claim) dense_resolve_slot(R, (uint32_t)t);
        atomicAdd(&deg[a], 1ull);
        atomicAdd(&deg[b], 1ull);
    } else if (keep[e]) {
        unsigned long long at = off[a] + atomicAdd(&deg[a], 1ull);
        adj_id[at] = b;
        adj_rank[at] = wrank[e];
        at = off[b] + atomicAdd(&deg[b], 1ull);
        adj_id[at] = a;
        adj_rank[at] = wrank[e];
    }
}
// one CTA per node: the survivors that beat the tie value, by (dist, global id), then the
// smallest ids (local order = global order: the level's node list is ascending); churn =
// entries that were not in the sweep-start (initial) row
__global__ void __launch_bounds__(128) cover_rows_kernel(const int32_t* __restrict__ nodes, uint64_t n, int kw,
                                                         const unsigned long long* __restrict__ off,
                                                         const int32_t* __restrict__ adj_id,
                                                         const uint32_t* __restrict__ adj_rank,
                                                         const double* __restrict__ vals, double pruned,
                                                         int32_t* __restrict__ gid, double* __restrict__ gd,
                                                         unsigned long long* __restrict__ churn) {
    extern __shared__ unsigned char cover_smem[];
    double* od = reinterpret_cast<double*>(cover_smem);
    int32_t* oi = reinterpret_cast<int32_t*>(od + kw);
    int32_t* init = oi + kw;
    int32_t* flag = init + kw;  // kw + 1 entries
    __shared__ int s_nb, s_ch;
    const uint64_t i = blockIdx.x;
    const int tid = threadIdx.x;
    const unsigned long long a0 = off[i];
    const int s = (int)(off[i + 1] - a0);
    for (int t = tid; t < kw; t += 128) init[t] = gid[i * kw + t];
    if (tid == 0) s_nb = s_ch = 0;
    __syncthreads();
    int mine = 0;
    for (int t = tid; t < s; t += 128) {
        const double d = vals[adj_rank[a0 + t]];
        if (!(d < pruned)) continue;
        ++mine;
        const int32_t v = adj_id[a0 + t];
        const int g = nodes[v];
        int r = 0;
        for (int u = 0; u < s; ++u) {
            const double du = vals[adj_rank[a0 + u]];
            if (du < pruned) r += entry_less(du, nodes[adj_id[a0 + u]], d, g) ? 1 : 0;
        }
        if (r < kw) {
            od[r] = d;
            oi[r] = v;
        }
    }
    if (mine) atomicAdd(&s_nb, mine);
    __syncthreads();
    const int sp = min(s_nb, kw);
    // the first kw + 1 ids hold at least kw - sp nodes outside {i} and the sp chosen
    for (int v = tid; v <= kw; v += 128) {
        bool ok = (uint64_t)v != i && (uint64_t)v < n;
        for (int u = 0; ok && u < sp; ++u) ok = oi[u] != v;
        flag[v] = ok ? 1 : 0;
    }
    __syncthreads();
    if (tid == 0) {
        int pos = sp;
        for (int v = 0; v <= kw && pos < kw; ++v)
            if (flag[v]) {
                od[pos] = pruned;
                oi[pos++] = v;
            }
    }
    __syncthreads();
    int ch = 0;
    for (int t = tid; t < kw; t += 128) {
        const int32_t v = oi[t];
        bool in = false;
        for (int u = 0; !in && u < kw; ++u) in = init[u] == v;
        ch += in ? 0 : 1;
        gid[i * kw + t] = v;
        gd[i * kw + t] = od[t];
    }
    if (ch) atomicAdd(&s_ch, ch);
    __syncthreads();
    if (tid == 0 && s_ch) atomicAdd(churn, (unsigned long long)s_ch);
}

// ---------------------------------------------------------------- driver
__global__ void to_global_kernel(const int32_t* __restrict__ gid, const double* __restrict__ gd,
                                 const int32_t* __restrict__ nodes, uint64_t n, int kw, int k,
                                 int32_t* __restrict__ out_id, double* __restrict__ out_d) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * (uint64_t)k) return;
    const uint64_t li = e / k, t = e % k;
    out_id[e] = nodes[gid[li * kw + t]];
    out_d[e] = gd[li * kw + t];
}

static void score_claimed(Context& c, int mode, int32_t* ws, int32_t* wp, uint32_t* wslot, uint64_t nw) {
    if (!nw) return;
    ScoreOut so;
    so.cache_vals = c.Cview().vals;
    so.cache_bits = c.dsurvbits();
    so.slot = wslot;
    score_entries(c, mode, ws, wp, nw, so);
}

// Per-node lists of the level's pairs on the dense root's survivor worklist (local ids),
// for the short candidate lists of knn_gather_bits_kernel.  off: n + 1 offsets.
struct LevelSurvivors {
    DevBuf seenb, keepb, degb, offb, idb, rkb, tmpb;
    const unsigned long long* off = nullptr;
    const int32_t* id = nullptr;
};
static void level_survivors(Context& c, const int32_t* loc, uint64_t n, LevelSurvivors& L) {
    const uint64_t nw = c.dwl_n, dn = c.dense_n;
    unsigned long long* deg = L.degb.as<unsigned long long>(n + 1);
    unsigned long long* off = L.offb.as<unsigned long long>(n + 1);
    int32_t* adj_id = L.idb.as<int32_t>(2 * nw + 1);
    uint32_t* adj_rank = L.rkb.as<uint32_t>(2 * nw + 1);
    NRG_CUDA(cudaMemsetAsync(deg, 0, (n + 1) * 8, c.stream));
    NRG_CUDA(cudaMemsetAsync(off, 0, (n + 1) * 8, c.stream));
    if (nw) {
        const uint64_t swords = dn * (dn - 1) / 2 / 32 + 1;
        uint32_t* seen = L.seenb.as<uint32_t>(swords);
        uint8_t* keep = L.keepb.as<uint8_t>(nw);
        NRG_CUDA(cudaMemsetAsync(seen, 0, swords * 4, c.stream));
        const DenseResolve R{};  // no claims here
        const int32_t* es = static_cast<const int32_t*>(c.dwl_es.p);
        const int32_t* ep = static_cast<const int32_t*>(c.dwl_ep.p);
        const uint32_t* wr = static_cast<const uint32_t*>(c.dwl_slot.p);
        const int32_t* dloc = static_cast<const int32_t*>(c.dloc.p);
        cover_worklist_kernel<<<(unsigned)ceil_div(nw, 256), 256, 0, c.stream>>>(R, es, ep, wr, nw, loc, dloc, dn, seen,
                                                                                keep, deg, off, adj_id, adj_rank, 0,
                                                                                false);
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, deg, off, (int64_t)(n + 1), c.stream);
        void* tmp = L.tmpb.ensure(tb);
        cub::DeviceScan::ExclusiveSum(tmp, tb, deg, off, (int64_t)(n + 1), c.stream);
        NRG_CUDA(cudaMemsetAsync(deg, 0, (n + 1) * 8, c.stream));
        cover_worklist_kernel<<<(unsigned)ceil_div(nw, 256), 256, 0, c.stream>>>(R, es, ep, wr, nw, loc, dloc, dn, seen,
                                                                                keep, deg, off, adj_id, adj_rank, 1,
                                                                                false);
        NRG_LAUNCH_CHECK_N(2);
    }
    L.off = off;
    L.id = adj_id;
}

// Finish a dense level whose first sweep covers every node (see "covered dense levels").
// gid holds the initial rows (local ids, unsorted).  Returns false (nothing changed) when
// some node's candidate set falls short; the sweeps then run as usual.
static bool cover_level(Context& c, const int32_t* d_nodes, uint64_t n, int kw, int cap, const int32_t* loc,
                        const int32_t* rootpos, int32_t* gid, double* gd, const KnnParamsD& p, KnnResultD& out) {
    const int Wb = (int)((n + 31) / 32);
    const uint64_t full = n - 1 - (uint64_t)kw;
    DevBuf adjb, alenb, ubb, newfb, hnb, cntb, chb;
    int32_t* adj = adjb.as<int32_t>(n * cap);
    int32_t* alen = alenb.as<int32_t>(n);
    uint32_t* ub = ubb.as<uint32_t>(n * (uint64_t)Wb);
    uint8_t* newf = newfb.as<uint8_t>(n * cap);
    uint8_t* hasnew = hnb.as<uint8_t>(n);
    int32_t* cand_cnt = cntb.as<int32_t>(n);
    unsigned long long* ch = chb.as<unsigned long long>(2);  // churn, nodes short of full coverage
    c.tic();
    u_out_kernel<<<(unsigned)ceil_div(n * (uint64_t)kw, 256), 256, 0, c.stream>>>(gid, n, kw, cap, adj, alen);
    NRG_CUDA(cudaMemsetAsync(ub, 0, n * (uint64_t)Wb * 4, c.stream));
    NRG_CUDA(cudaMemsetAsync(newf, 1, n * cap, c.stream));  // first sweep: every entry is new
    NRG_CUDA(cudaMemsetAsync(hasnew, 1, n, c.stream));
    NRG_CUDA(cudaMemsetAsync(ch, 0, 16, c.stream));
    u_set_kernel<<<(unsigned)ceil_div(n * (uint64_t)cap, 256), 256, 0, c.stream>>>(adj, alen, n, cap, Wb, ub);
    ClaimSink sk{};
    knn_gather_bits_kernel<256><<<(unsigned)n, 256, 2 * Wb * 4 + 4 * cap, c.stream>>>(
        d_nodes, n, adj, alen, cap, gid, kw, Wb, ub, ub, newf, HashView{nullptr, nullptr, 0}, sk, 0, nullptr, nullptr,
        cand_cnt, 0, false, rootpos, hasnew, /*count_only=*/true);
    coverage_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(cand_cnt, n, (int)full, ch + 1);
    NRG_LAUNCH_CHECK_N(4);
    unsigned long long* hc = c.hp_small.as<unsigned long long>(2);
    NRG_CUDA(cudaMemcpyAsync(hc, ch, 16, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (hc[1] != 0) {
        c.toc(P_KNN);
        return false;
    }
    // probes: the initial rows (n kw) and the sweep's candidates (n (n - 1 - kw)), all hits
    // until the dense root's recount; marks: every pair of the level
    counters_add_host(c, C_HITS, n * (n - 1));
    const uint64_t dn = c.dense_n;
    DevBuf mb, seenb, keepb, degb, offb, aidb, arkb, tmpb;
    const uint64_t mwords = dn / 32 + 2;
    uint32_t* M = mb.as<uint32_t>(mwords);
    NRG_CUDA(cudaMemsetAsync(M, 0, mwords * 4, c.stream));
    cover_members_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(rootpos, n, M);
    cover_mark_kernel<<<(unsigned)ceil_div(n * 32, 256), 256, 0, c.stream>>>(rootpos, n, dn, M,
                                                                           static_cast<uint32_t*>(c.dbits.p));
    NRG_LAUNCH_CHECK_N(2);
    // survivors of the level: claimed for K2, listed per node
    const uint64_t nw = c.dwl_n;
    unsigned long long* deg = degb.as<unsigned long long>(n + 1);
    unsigned long long* off = offb.as<unsigned long long>(n + 1);
    NRG_CUDA(cudaMemsetAsync(deg, 0, (n + 1) * 8, c.stream));
    int32_t* adj_id = aidb.as<int32_t>(2 * nw + 1);
    uint32_t* adj_rank = arkb.as<uint32_t>(2 * nw + 1);
    if (nw) {
        const uint64_t swords = dn * (dn - 1) / 2 / 32 + 1;
        uint32_t* seen = seenb.as<uint32_t>(swords);
        uint8_t* keep = keepb.as<uint8_t>(nw);
        NRG_CUDA(cudaMemsetAsync(seen, 0, swords * 4, c.stream));
        const DenseResolve R = dense_resolve_begin(c);
        const int32_t* es = static_cast<const int32_t*>(c.dwl_es.p);
        const int32_t* ep = static_cast<const int32_t*>(c.dwl_ep.p);
        const uint32_t* wr = static_cast<const uint32_t*>(c.dwl_slot.p);
        const int32_t* dloc = static_cast<const int32_t*>(c.dloc.p);
        cover_worklist_kernel<<<(unsigned)ceil_div(nw, 256), 256, 0, c.stream>>>(R, es, ep, wr, nw, loc, dloc, dn, seen,
                                                                                keep, deg, off, adj_id, adj_rank, 0, true);
        NRG_LAUNCH_CHECK();
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, deg, off, (int64_t)(n + 1), c.stream);
        void* tmp = tmpb.ensure(tb);
        cub::DeviceScan::ExclusiveSum(tmp, tb, deg, off, (int64_t)(n + 1), c.stream);
        NRG_CUDA(cudaMemsetAsync(deg, 0, (n + 1) * 8, c.stream));
        cover_worklist_kernel<<<(unsigned)ceil_div(nw, 256), 256, 0, c.stream>>>(R, es, ep, wr, nw, loc, dloc, dn, seen,
                                                                                keep, deg, off, adj_id, adj_rank, 1, true);
        NRG_LAUNCH_CHECK();
        c.toc(P_KNN);
        dense_resolve_end(c);  // K2 on the claimed pairs (times itself)
        c.tic();
    } else {
        NRG_CUDA(cudaMemsetAsync(off, 0, (n + 1) * 8, c.stream));
    }
    const DenseView D = c.dview();
    cover_rows_kernel<<<(unsigned)n, 128, (size_t)kw * 16 + (size_t)(kw + 1) * 4 + 16, c.stream>>>(
        d_nodes, n, kw, off, adj_id, adj_rank, D.vals, D.pruned, gid, gd, ch);
    NRG_LAUNCH_CHECK();
    NRG_CUDA(cudaMemcpyAsync(hc, ch, 16, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    c.toc(P_KNN);
    out.sweeps = 1;
    out.churn.clear();
    const double ratio = (double)hc[0] / ((double)kw * (double)n);
    out.churn.push_back(ratio);
    if (!(ratio < p.eps) && p.max_sweeps > 1) {
        ++out.sweeps;  // the next sweep, settled in advance: churn 0 < eps
        out.churn.push_back(0.0);
    }
    return true;
}

void find_knn(Context& c, int mode, int k, const int32_t* d_nodes, uint64_t n, const KnnParamsD& p,
              bool exhaustive, KnnResultD& out, DevBuf& ids_buf, DevBuf& dist_buf, bool sorted_valid) {
    if (n < 2) fail(22, exhaustive ? "find_knn_exhaustive: need two nodes" : "find_knn: need at least two nodes");
    if (!exhaustive) {
        if (k < 1) fail(22, "find_knn: k must be >= 1");
        if (!(p.eps > 0.0)) fail(22, "find_knn: eps must be > 0");
    }
    if (n > (uint64_t)INT32_MAX) fail(22, "find_knn: too many nodes");
    if (mode == TABLE && !c.table_n) fail(22, "no distance table set");
    if (mode == LINE && !c.line_n) fail(22, "no line metric set");
    if (mode == EXACT || mode == GRADIENT) ensure_snapshot(c);
    // collective in multi-rank jobs: every rank resolves the generation's base here
    if (mode == EXACT) generation_base(c);

    // local index map, id-sorted node set and ranks.  A node list already strictly
    // ascending and in range (FindBest's levels: subsets of a sorted list, in order) is
    // its own sorted order: no sort, no validation round trip.
    int32_t* loc = c.s_a.as<int32_t>(c.n);
    NRG_CUDA(cudaMemsetAsync(loc, 0xff, (size_t)c.n * 4, c.stream));
    DevBuf sbuf_ids, sbuf_loc, sbuf_rank, stmp;
    const int32_t* sorted_ids = d_nodes;
    int32_t* sorted_loc;
    int32_t* rank;
    if (sorted_valid) {
        scatter_loc_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(d_nodes, n, loc, c.n, nullptr);
        sorted_loc = sbuf_loc.as<int32_t>(n);
        iota_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(sorted_loc, n);
        rank = sorted_loc;  // identity
        NRG_LAUNCH_CHECK();
    } else {
        int* bad = c.s_b.as<int>(1);
        NRG_CUDA(cudaMemsetAsync(bad, 0, 4, c.stream));
        scatter_loc_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(d_nodes, n, loc, c.n, bad);
        NRG_LAUNCH_CHECK();
        int32_t* sids = sbuf_ids.as<int32_t>(n);
        sorted_loc = sbuf_loc.as<int32_t>(n);
        rank = sbuf_rank.as<int32_t>(n);
        {
            int32_t* iota = rank;  // temporarily
            iota_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(iota, n);
            size_t tmp = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tmp, d_nodes, sids, iota, sorted_loc, (int)n, 0, 32,
                                            c.stream);
            void* dt = stmp.ensure(tmp);
            cub::DeviceRadixSort::SortPairs(dt, tmp, d_nodes, sids, iota, sorted_loc, (int)n, 0, 32, c.stream);
            rank_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(sorted_loc, n, rank);
            NRG_LAUNCH_CHECK();
        }
        sorted_ids = sids;
        int hbad = 0;
        hbad = c.read_scalar(bad);
        if (hbad == 1) fail(34, "node id out of range");
        if (hbad == 2) fail(22, "find_knn: duplicate node ids");
    }

    if (exhaustive || (uint64_t)k + 1 >= n) {
        knn_exhaustive(c, mode, (int)std::min<uint64_t>((uint64_t)k, n - 1), d_nodes, n, sorted_loc, rank, out,
                       ids_buf, dist_buf);
        return;
    }
    const int kw = std::max(k, p.width_floor);
    if ((uint64_t)kw + 1 >= n) {
        knn_exhaustive(c, mode, k, d_nodes, n, sorted_loc, rank, out, ids_buf, dist_buf);
        return;
    }
    const int cap = p.reverse ? std::max(2 * kw, p.scan_floor) : std::max(kw, p.scan_floor);

    // working graph (local ids, sorted rows)
    DevBuf gid_buf, gd_buf;
    int32_t* gid = gid_buf.as<int32_t>(n * kw);
    double* gd = gd_buf.as<double>(n * kw);
    // wcount[2] (claims) and churn[2] side by side: one clear and one readback per sweep
    unsigned long long* wcount = c.s_c.as<unsigned long long>(4);
    const bool cached = (mode == EXACT || mode == GRADIENT);
    // dense level: distances come from the level's exhaustive triangle (find_best.cu)
    const bool dense = mode == EXACT && c.dense_active && c.world == 1;
    const DenseView dview = dense ? c.dview() : DenseView{nullptr, nullptr, nullptr, 0.0};
    DevBuf rootposb;
    int32_t* rootpos = nullptr;
    if (dense) {
        rootpos = rootposb.as<int32_t>(n);
        gather_kernel<int32_t><<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(
            static_cast<const int32_t*>(c.dloc.p), d_nodes, n, rootpos);
        NRG_LAUNCH_CHECK();
    }
    // node shard of this rank; the distance cache is sharded by key
    const int W = cached ? c.world : 1;
    uint64_t lo = 0, hi = n;
    if (c.world > 1) shard_range(n, c.rank, c.world, lo, hi);
    const uint64_t own = hi - lo;
    ExchangeBufs X;
    auto sink_for = [&](int32_t* ws, int32_t* wp, uint32_t* wslot, uint64_t rcap) {
        ClaimSink s;
        s.ws = ws;
        s.wp = wp;
        s.wslot = wslot;
        s.wcount = wcount;
        s.counters = c.dcounters();
        s.live = static_cast<uint64_t*>(c.Ccount.p);
        s.rank = c.rank;
        s.world = W;
        s.fold = W == 1 && cached && !dense && !NRG_ENV_ON("NRG_NO_FOLD");
        if (dense) {
            s.dloc = static_cast<const int32_t*>(c.dloc.p);
            s.dbits = static_cast<uint32_t*>(c.dbits.p);
            s.dn = c.dense_n;
        }
        if (W > 1) {
            s.rkeys = X.rkeys.as<uint64_t>(rcap);
            s.rdest = X.rdest.as<int32_t>(rcap);
            s.rcount = X.rcount.as<unsigned long long>(1);
            NRG_CUDA(cudaMemsetAsync(s.rcount, 0, 8, c.stream));
        }
        return s;
    };
    // rows [lo, hi) of the graph are this rank's; make every rank's copy whole
    auto allgather_rows = [&](int32_t* gid_, double* gd_, int kwid) {
        if (c.world == 1) return;
        Comm* comm = static_cast<Comm*>(c.comm);
        std::vector<size_t> bi(c.world), bd(c.world);
        for (int r = 0; r < c.world; ++r) {
            uint64_t l, h;
            shard_range(n, r, c.world, l, h);
            bi[r] = (h - l) * kwid * 4;
            bd[r] = (h - l) * kwid * 8;
        }
        comm->allgatherv(gid_ + lo * kwid, gid_, bi, c.stream);
        comm->allgatherv(gd_ + lo * kwid, gd_, bd, c.stream);
    };

    // ---- initial graph
    c.tic();
    {
        const uint64_t nq = own * kw;
        DevBuf qib, qjb, slb;
        int32_t* qi = qib.as<int32_t>(nq + 1);
        int32_t* qj = qjb.as<int32_t>(nq + 1);
        if (n <= 16384 && kw >= 64)
            knn_init_bits_kernel<<<(unsigned)ceil_div(own * 32, 128), 128, 4 * ((n + 31) / 32) * 4, c.stream>>>(
                d_nodes + lo, sorted_ids, rank + lo, loc, own, n, kw, p.seed, gid + lo * kw, qi, qj);
        else
            knn_init_kernel<<<(unsigned)ceil_div(own * 32, 128), 128, 0, c.stream>>>(
                d_nodes + lo, sorted_ids, rank + lo, loc, own, n, kw, p.seed, gid + lo * kw, qi, qj);
        NRG_LAUNCH_CHECK();
        c.toc(P_KNN);
        // a dense level the first sweep covers entirely is finished from the coverage alone
        if (dense && sorted_valid && cap == kw && n <= (uint64_t)kBitsMaxN && cap >= 32 && p.max_sweeps >= 1 &&
            // (worth the size pass only where full coverage is likely: random initial rows give a
            // node ~cap^2 two-hop paths; at cap^2 ~ 4 n some node still misses a few others)
            (uint64_t)cap * cap >= 6 * (n - 1 - (uint64_t)kw) && !NRG_ENV_ON("NRG_NO_COVER_LEVEL") &&
            !NRG_ENV_ON("NRG_DENSE_EAGER") &&  // (the survivor lists come from the lazy root's worklist)
            !NRG_ENV_ON("NRG_NO_COVERAGE_SKIP") && !NRG_ENV_ON("NRG_KNN_HASH_GATHER") && !getenv("NRG_KNN_FULL_JOIN") &&
            cover_level(c, d_nodes, n, kw, cap, loc, rootpos, gid, gd, p, out)) {
            out.k = k;
            out.ids = ids_buf.as<int32_t>(n * k);
            out.dists = dist_buf.as<double>(n * k);
            to_global_kernel<<<(unsigned)ceil_div(n * k, 256), 256, 0, c.stream>>>(gid, gd, d_nodes, n, kw, k, out.ids,
                                                                                 out.dists);
            NRG_LAUNCH_CHECK();
            return;
        }
        if (cached) {
            if (!dense) cache_reserve(c, n * (uint64_t)kw);
            uint32_t* slot = slb.as<uint32_t>(nq + 1);
            DevBuf wsb, wpb, wslb;
            int32_t* ws = wsb.as<int32_t>(nq + 1);
            int32_t* wp = wpb.as<int32_t>(nq + 1);
            uint32_t* wsl = wslb.as<uint32_t>(nq + 1);
            NRG_CUDA(cudaMemsetAsync(wcount, 0, 16, c.stream));
            const ClaimSink sk = sink_for(ws, wp, wsl, nq + 1);
            if (nq) {
                claim_list_kernel<<<(unsigned)ceil_div(nq, 256), 256, 0, c.stream>>>(c.Cview(), sk, qi, qj, nq, slot);
                if (sk.fold)
                    fold_claims_kernel<<<1, 1, 0, c.stream>>>(wcount, c.dcounters(), sk.live);
                NRG_LAUNCH_CHECK();
            }
            if (dense) {
            } else if (c.world == 1) {
                // claimed count stays on the device: the screen strides over it
                ScoreOut so;
                so.cache_vals = c.Cview().vals;
                so.cache_bits = c.dsurvbits();
                so.slot = wsl;
                score_entries(c, mode, ws, wp, nq + 1, so, wcount);
            } else {
                unsigned long long nw = 0;
                nw = c.read_scalar(wcount);
                exchange_and_score(c, mode, sk, nw, X, 0);
            }
            if (dense) dense_resolve_slots(c, slot, nq);  // refine the marked pairs first
            if (nq) {
                gather_vals_kernel<<<(unsigned)ceil_div(nq, 256), 256, 0, c.stream>>>(
                    dview, c.mview(), static_cast<double*>(X.rvals.p), slot, nq, gd + lo * kw);
                NRG_LAUNCH_CHECK();
            }
        } else {
            ScoreOut so;
            so.dist = gd + lo * kw;
            score_entries(c, mode, qi, qj, nq, so);
        }
        c.tic();
        int P = 1;
        while (P < kw) P <<= 1;
        const size_t rs_smem = (size_t)P * 16;
        if (rs_smem > 200 * 1024) fail(100, "find_knn: kw too large for the row sort");
        if (rs_smem > 48 * 1024)
            NRG_CUDA(cudaFuncSetAttribute(row_sort_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)rs_smem));
        if (own) {
            if (kw <= 32)
                row_sort_warp_kernel<<<(unsigned)ceil_div(own * 32, 256), 256, 0, c.stream>>>(gid + lo * kw, gd + lo * kw,
                                                                                           d_nodes, own, kw);
            else if (P <= 64)
                row_sort_kernel<32><<<(unsigned)own, 32, rs_smem, c.stream>>>(gid + lo * kw, gd + lo * kw, d_nodes, own,
                                                                             kw, P);
            else
                row_sort_kernel<128><<<(unsigned)own, 128, rs_smem, c.stream>>>(gid + lo * kw, gd + lo * kw, d_nodes,
                                                                               own, kw, P);
            NRG_LAUNCH_CHECK();
        }
        allgather_rows(gid, gd, kw);
        c.toc(P_KNN);
    }

    // ---- sweeps
    const uint64_t capn = std::min<uint64_t>((uint64_t)cap * cap, n - 1);
    DevBuf adjb, alenb, adjpb, alenpb, newfb, ccntb, churnb, churnb2, ubitsb, ubitsb2, nbitsb, hasnewb;
    // the n x cap^2 candidate and worklist arrays (GBs at deep config-5 levels) persist in
    // the context: re-mapping them per level and generation cost ~6 ms per GB
    DevBuf &cidb = c.kx_cid, &cslb = c.kx_csl, &wsb = c.kx_ws, &wpb = c.kx_wp, &wslb = c.kx_wsl;
    int32_t* adj = adjb.as<int32_t>(n * cap);
    int32_t* alen = alenb.as<int32_t>(n);
    int32_t* adjp = adjpb.as<int32_t>(n * cap);  // U of the previous sweep
    int32_t* alenp = alenpb.as<int32_t>(n);
    uint8_t* newf = newfb.as<uint8_t>(n * cap);
    const bool incremental = !getenv("NRG_KNN_FULL_JOIN");
    int32_t* cand_id = cidb.as<int32_t>(n * capn);
    uint32_t* cand_slot = cslb.as<uint32_t>(n * capn);
    int32_t* cand_cnt = ccntb.as<int32_t>(n);
    // churn[0]: entries this sweep changed; churn[1]: nodes whose candidate set missed
    // some node (bit-set gathers of one rank; read back together)
    unsigned long long* churn = wcount + 2;
    const uint64_t wmax = n * capn;
    int32_t* ws = wsb.as<int32_t>(wmax);
    int32_t* wp = wpb.as<int32_t>(wmax);
    uint32_t* wsl = wslb.as<uint32_t>(wmax);
    // uncached metrics (TABLE / LINE): per-candidate distances in a flat array
    DevBuf flatb;
    double* flat_d = cached ? nullptr : flatb.as<double>(wmax);
    if (!cached && wmax >= (1ull << 32)) fail(100, "find_knn: candidate buffer exceeds 2^32");
    // dedup structure: hash of 2x(cap^2 + kw + 1) slots vs bitmap of n bits
    const uint64_t hash_slots = [&] {
        uint64_t s = 64;
        while (s < 2 * (capn + kw + 1)) s <<= 1;
        return s;
    }();
    const uint64_t bitmap_words = (n + 31) / 32;
    const bool use_bitmap = bitmap_words < hash_slots;
    const uint64_t tab_bytes = 4 * (use_bitmap ? bitmap_words : hash_slots);
    if (tab_bytes > 200 * 1024) fail(100, "find_knn: dedup table exceeds shared memory");
    const int big = capn > 256 ? 1 : 0;
    if (tab_bytes > 48 * 1024) {
        NRG_CUDA(cudaFuncSetAttribute(knn_gather_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)tab_bytes));
        NRG_CUDA(cudaFuncSetAttribute(knn_gather_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)tab_bytes));
    }
    // merge buffer
    // merge buffer: a power of two >= kw + 64 (bitonic width), at least 256
    // merge buffer: a power of two >= kw + 64; wide rows take big candidate blocks (fewer
    // block sorts when a first sweep's candidates mostly beat the row)
    static const int merge_buf_min = getenv("NRG_MERGE_BUF") ? atoi(getenv("NRG_MERGE_BUF")) : 256;
    const int buf_cap = [&] {
        int b = kw > 64 ? merge_buf_min : 256;
        while (b < kw + 64) b <<= 1;
        return b;
    }();
    if ((size_t)buf_cap * 20 > 200 * 1024) fail(100, "find_knn: kw too large for the merge buffer");
    const size_t merge_smem = (size_t)(buf_cap + kw) * (8 + 4 + 4 + 4);
    if (merge_smem > 48 * 1024)
        NRG_CUDA(cudaFuncSetAttribute(knn_merge_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)merge_smem));
    if (merge_smem > 48 * 1024)
        NRG_CUDA(cudaFuncSetAttribute(knn_merge_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)merge_smem));

    out.sweeps = 0;
    out.churn.clear();
    DevBuf ktgt, kd, ksrc, vsrc, ktgt2, kd2, ksrc2, vsrc2, segb, sorttmp, permb, perm2b;
    // dense bit-set levels: per-node survivor lists for the gathers' short candidate lists
    LevelSurvivors LS;
    DevBuf fullb;
    int32_t* full_cnt = nullptr;
    if (dense && n <= (uint64_t)kBitsMaxN && cap >= 32 && !NRG_ENV_ON("NRG_KNN_HASH_GATHER") &&
        !NRG_ENV_ON("NRG_NO_SHORT_LISTS") && !NRG_ENV_ON("NRG_DENSE_EAGER")) {
        c.tic();
        level_survivors(c, loc, n, LS);
        full_cnt = fullb.as<int32_t>(n);
        c.toc(P_KNN);
    }
    for (int sweep = 0; sweep < p.max_sweeps; ++sweep) {
        c.tic();
        // U
        u_out_kernel<<<(unsigned)ceil_div(n * (uint64_t)kw, 256), 256, 0, c.stream>>>(gid, n, kw, cap, adj, alen);
        NRG_LAUNCH_CHECK();
        if (cap > kw) {
            const uint64_t ne = n * kw;
            uint32_t* a_t = ktgt.as<uint32_t>(ne);
            uint64_t* a_d = kd.as<uint64_t>(ne);
            uint32_t* a_s = ksrc.as<uint32_t>(ne);
            int32_t* a_v = vsrc.as<int32_t>(ne);
            in_keys_kernel<<<(unsigned)ceil_div(ne, 256), 256, 0, c.stream>>>(gid, gd, d_nodes, n, kw, a_t, a_d, a_s,
                                                                           a_v);
            NRG_LAUNCH_CHECK();
            uint32_t* tgt_sorted = ktgt2.as<uint32_t>(ne);
            int32_t* src_sorted = vsrc2.as<int32_t>(ne);
            in_edge_sort(c, ne, a_t, a_d, a_s, a_v, tgt_sorted, src_sorted, permb, perm2b, kd2, ksrc2, sorttmp);
            uint64_t* seg = segb.as<uint64_t>(n);
            seg_start_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(tgt_sorted, ne, n, seg);
            if (p.reverse)
                u_rev_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, c.stream>>>(tgt_sorted, src_sorted, ne, n, kw, cap,
                                                                            adj, alen, seg);
            else
                u_in_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, c.stream>>>(tgt_sorted, src_sorted, ne, n, cap, adj,
                                                                           alen, seg);
            NRG_LAUNCH_CHECK();
        }
        const int Wb = (int)((n + 31) / 32);
        static const uint64_t bits_max_n =
            getenv("NRG_BITS_MAXN") ? strtoull(getenv("NRG_BITS_MAXN"), nullptr, 10) : (uint64_t)kBitsMaxN;
        const bool bitsmode = n <= std::min<uint64_t>(bits_max_n, kBitsMaxN) && cap >= 32 &&
                              !NRG_ENV_ON("NRG_KNN_HASH_GATHER");
        if (bitsmode) {
            // U bitsets ping-pong between sweeps: last sweep's set answers the new flags
            uint32_t* ubc = (sweep & 1 ? ubitsb2 : ubitsb).as<uint32_t>(n * (uint64_t)Wb);
            uint32_t* ubp = (sweep & 1 ? ubitsb : ubitsb2).as<uint32_t>(n * (uint64_t)Wb);
            // new-entry bitsets and the has-new flags share one buffer (one clear)
            uint32_t* nbits = nbitsb.as<uint32_t>(n * (uint64_t)Wb + (n + 3) / 4);
            uint8_t* hasnew = reinterpret_cast<uint8_t*>(nbits + n * (uint64_t)Wb);
            NRG_CUDA(cudaMemsetAsync(ubc, 0, n * (uint64_t)Wb * 4, c.stream));
            NRG_CUDA(cudaMemsetAsync(nbits, 0, n * (uint64_t)Wb * 4 + n, c.stream));
            const unsigned g = (unsigned)ceil_div(n * (uint64_t)cap, 256);
            u_bits_kernel<<<g, 256, 0, c.stream>>>(adj, alen, n, cap, Wb, ubc, ubp,
                                                  (sweep == 0 || !incremental) ? 1 : 0, newf, nbits, hasnew);
        } else {
            u_new_kernel<<<(unsigned)ceil_div(n * 32, 256), 256, 0, c.stream>>>(adj, alen, adjp, alenp, n, cap,
                                                                             (sweep == 0 || !incremental) ? 1 : 0,
                                                                             newf);
        }
        NRG_LAUNCH_CHECK();
        c.toc(P_KNN);
        // gather (own nodes), then — for the cached metric — reserve the distance cache
        // for exactly this sweep's candidates (job-wide: remote keys land on their owner)
        // and claim them; uncached metrics claim flat slots inside the gather
        // the worst case (every node gathers capn new pairs) normally fits the cache
        // with room to spare: reserve it and claim inside the gather; otherwise gather,
        // count, reserve exactly and claim in a second pass
        const bool fused = !cached || dense || (c.cache_live_host + wmax) * 10 <= (1ull << 31) * 6;
        if (cached && fused && !dense) cache_reserve(c, wmax);
        c.tic();
        NRG_CUDA(cudaMemsetAsync(wcount, 0, 32, c.stream));  // and churn
        ClaimSink sk = sink_for(ws, wp, wsl, own * capn + 1);
        // own claims resolve through the worklist-ordered distances (single rank, a memo
        // and worklist small enough for 31-bit indices)
        const bool wl = W == 1 && cached && !dense && wmax < (uint64_t)kRemote && !NRG_ENV_ON("NRG_NO_WL_SLOTS");
        double* wdist = wl ? c.kx_wd.as<double>(wmax) : nullptr;
        sk.wl_slots = wl;
        if (own) {
            int lw = 0;
            while ((1 << lw) < cap) ++lw;
            const HashView hv0 = fused && cached ? c.Cview() : HashView{nullptr, nullptr, 0};
            const int W = Wb;
            if (bitsmode) {
                uint32_t* ub = static_cast<uint32_t*>((sweep & 1 ? ubitsb2 : ubitsb).p);
                uint32_t* nbits = static_cast<uint32_t*>(nbitsb.p);
                knn_gather_bits_kernel<256><<<(unsigned)own, 256, 2 * W * 4 + 4 * cap, c.stream>>>(
                    d_nodes, n, adj, alen, cap, gid, kw, W, ub, nbits, newf, hv0, sk, capn, cand_id, cand_slot, cand_cnt,
                    lo, fused, rootpos,
                    reinterpret_cast<const uint8_t*>(static_cast<const uint32_t*>(nbitsb.p) + n * (uint64_t)Wb), false,
                    LS.off, LS.id, full_cnt, (int)(n - 1 - (uint64_t)kw),
                    (c.world == 1 && !NRG_ENV_ON("NRG_NO_COVERAGE_SKIP")) ? churn + 1 : nullptr);
            } else if (big)
                knn_gather_kernel<256><<<(unsigned)own, 256, tab_bytes, c.stream>>>(
                    d_nodes, n, adj, alen, cap, gid, kw, use_bitmap, (int)hash_slots, hv0, sk, capn, cand_id,
                    cand_slot, cand_cnt, lo, lw, newf, fused);
            else if (!NRG_ENV_ON("NRG_GATHER_CTA") && tab_bytes * 4 <= 48 * 1024)
                knn_gather_warp_kernel<4><<<(unsigned)ceil_div(own, 4), 128, 4 * tab_bytes, c.stream>>>(
                    d_nodes, n, adj, alen, cap, gid, kw, use_bitmap, (int)hash_slots, hv0, sk, capn, cand_id,
                    cand_slot, cand_cnt, lo, own, lw, newf, fused);
            else
                knn_gather_kernel<32><<<(unsigned)own, 32, tab_bytes, c.stream>>>(
                    d_nodes, n, adj, alen, cap, gid, kw, use_bitmap, (int)hash_slots, hv0, sk, capn, cand_id,
                    cand_slot, cand_cnt, lo, lw, newf, fused);
            NRG_LAUNCH_CHECK();
        }
        if (cached && !fused) {
            unsigned long long* tot = churnb2.as<unsigned long long>(1);
            NRG_CUDA(cudaMemsetAsync(tot, 0, 8, c.stream));
            if (own) {
                sum_counts_kernel<<<(unsigned)std::min<uint64_t>(ceil_div(own, 256), 1184), 256, 0, c.stream>>>(
                    cand_cnt + lo, own, tot);
                NRG_LAUNCH_CHECK();
            }
            uint64_t total = 0;
            total = c.read_scalar(tot);
            if (c.world > 1) static_cast<Comm*>(c.comm)->allreduce_u64(&total, 1, false, c.stream);
            c.toc(P_KNN);
            cache_reserve(c, total);
            c.tic();
            if (own) {
                if (capn > 256)
                    claim_cands_flat_kernel<<<dim3((unsigned)own, (unsigned)ceil_div(capn, 256)), 256, 0, c.stream>>>(
                        d_nodes, c.Cview(), sk, own, lo, capn, cand_id, cand_slot, cand_cnt);
                else
                    claim_cands_kernel<<<(unsigned)ceil_div(own * 32, 256), 256, 0, c.stream>>>(
                        d_nodes, c.Cview(), sk, own, lo, capn, cand_id, cand_slot, cand_cnt);
                NRG_LAUNCH_CHECK();
            }
        }
        if (sk.fold) {  // this sweep's claims into the miss count and the memo's live count
            fold_claims_kernel<<<1, 1, 0, c.stream>>>(wcount, c.dcounters(), sk.live);
            NRG_LAUNCH_CHECK();
        }
        c.toc(P_KNN);
        unsigned long long nw = 0;
        if (cached && !dense && c.world == 1) {
            // claimed count stays on the device: the screen strides over it
            ScoreOut so;
            so.cache_vals = c.Cview().vals;
            so.cache_bits = c.dsurvbits();
            so.slot = wsl;
            so.dist = wdist;  // the worklist-ordered copy the merge reads (wl slots)
            score_entries(c, mode, ws, wp, own * capn + 1, so, wcount);
        } else if (!dense) {
            nw = c.read_scalar(wcount);
        }
        if (cached && !dense && c.world > 1) {
            exchange_and_score(c, mode, sk, nw, X, 0);
        } else if (nw && !dense && !cached) {
            ScoreOut so;
            so.cache_vals = flat_d;
            so.slot = wsl;
            score_entries(c, mode, ws, wp, nw, so);
        }
        if (dense) dense_resolve_rows(c, cand_slot, cand_cnt, lo, own, capn);  // refine the marked pairs first
        // distances behind the candidate slots: the memo (pruned pairs implicit), or the
        // flat per-candidate array of an uncached metric
        const MemoView dvals = cached ? c.mview() : MemoView{nullptr, flat_d, 0.0};
        const double* rvals = wl ? wdist : static_cast<double*>(X.rvals.p);
        c.tic();
        if (own) {
            if (kw > 64)
                knn_merge_kernel<128><<<(unsigned)own, 128, merge_smem, c.stream>>>(
                    d_nodes, n, gid, gd, kw, cand_id, cand_slot, cand_cnt, capn, dview, dvals, rvals, buf_cap, churn, lo);
            else if (!NRG_ENV_ON("NRG_MERGE_CTA"))
                knn_merge_warp_kernel<<<(unsigned)ceil_div(own, kMergeWarps), 32 * kMergeWarps,
                                        (size_t)kMergeWarps * (2 * kw + kMergeBlk) * 20, c.stream>>>(
                    d_nodes, n, gid, gd, kw, cand_id, cand_slot, cand_cnt, capn, dview, dvals, rvals, churn, lo, own);
            else
                knn_merge_kernel<32><<<(unsigned)own, 32, merge_smem, c.stream>>>(
                    d_nodes, n, gid, gd, kw, cand_id, cand_slot, cand_cnt, capn, dview, dvals, rvals, buf_cap, churn, lo);
            NRG_LAUNCH_CHECK();
        }
        // Full coverage: when every node's candidate set (bit-set gathers: the 2-hop set minus
        // the row and the node) was all the other nodes, each merged row is the exact top-kw
        // of the level, so the next sweep cannot change an entry: its churn is 0 and the loop
        // ends there.  That sweep is recorded (sweeps, churn trace) without being run -- it
        // would only re-probe pairs this sweep already probed (hits, no misses).
        const bool cov_check = bitsmode && c.world == 1 && !NRG_ENV_ON("NRG_NO_COVERAGE_SKIP");
        // (the bit-set gather counts the nodes short of full coverage into churn[1] itself)
        unsigned long long* hc = c.hp_small.as<unsigned long long>(4);
        NRG_CUDA(cudaMemcpyAsync(hc, wcount, 32, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        unsigned long long changed = hc[2];
        const bool covered = cov_check && hc[3] == 0;
        // the sweep's actual claims tighten the memo's host-side occupancy bound (reserved
        // for the worst case, n x cap^2): fewer reserves fall back to reading the live count
        if (sk.fold && fused) c.cache_live_bound = c.cache_live_host + hc[0];
        allgather_rows(gid, gd, kw);
        if (c.world > 1) {
            uint64_t ch = changed;
            static_cast<Comm*>(c.comm)->allreduce_u64(&ch, 1, false, c.stream);
            changed = ch;
        }
        c.toc(P_KNN);
        std::swap(adj, adjp);  // this sweep's U is the next sweep's "previous"
        std::swap(alen, alenp);
        ++out.sweeps;
        const double ratio = (double)changed / ((double)kw * (double)n);
        out.churn.push_back(ratio);
        if (ratio < p.eps) break;
        if (covered && sweep + 1 < p.max_sweeps) {
            ++out.sweeps;  // the next sweep, settled in advance: churn 0 < eps
            out.churn.push_back(0.0);
            break;
        }
    }
    // trim to k / convert to global ids
    out.k = k;
    out.ids = ids_buf.as<int32_t>(n * k);
    out.dists = dist_buf.as<double>(n * k);
    to_global_kernel<<<(unsigned)ceil_div(n * k, 256), 256, 0, c.stream>>>(gid, gd, d_nodes, n, kw, k, out.ids,
                                                                         out.dists);
    NRG_LAUNCH_CHECK();  // stream-ordered: callers read the lists on this stream
}

}  // namespace nrg
