// score.cu — the pair-scoring kernels: distance() (inc/model.hpp:377-386) for
// worklists of candidate pairs.
//
// Ising exact mode (M <= 2048) runs two kernels:
//   K1 (every pair, bandwidth-bound): g0 = 2<x_a,x_b> - <x_b,T_a> - <x_a,T_b> in exact
//      integer arithmetic on the snapshot's int8 field (per-node step d, rigorous
//      quantisation error E per node): popcount over bit planes and dp4a.
//      |g0| <= lambda - err  =>  pruned: w* = 0, gain = 0 exactly, dist = -base (the
//      reference's tie value, inc/model.hpp:205-209).  Streams M + M/8 bytes per pair.
//   K2 (survivors, a few per mille at a converging state): Newton in fp32 on the fp32
//      field, then ONE fp64 pass over T64 that evaluates L', L'' and the slice gain at
//      the fp32 root and applies the second-order Newton correction.  Existing edges
//      (w_cur != 0) and kink decisions inside the error band take the full fp64 routine
//      (pairscore.cuh).
// The stationary node's operands (first entry of a worklist run) stay in registers
// across consecutive entries, so each pair streams only its partner.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pairscore.cuh"

#ifndef NRG_K2_MINB
#define NRG_K2_MINB 6  // CTAs per SM of the CTA-per-survivor K2 (85 registers, no spills; 4 at 128 registers)
#endif
#ifndef NRG_K1S_MINB
#define NRG_K1S_MINB 3
#endif

namespace nrg {

// Register side of the screen for one node: for each 32-sample word w = lane + 32 q
// (q < HW) the 8 bit planes of T8 (sum_{m: b_m = 1} T8_m = sum_k 2^k popc(P_k & b) with
// the sign plane weighted -2^7), the spins as +-1 bytes for dp4a, and the spin word.
template <int HW>
struct Src8 {
    uint32_t P[HW][8];
    uint32_t X[HW][8];
    uint32_t b[HW];
};

// 4 spin bits -> 4 bytes of +1 (bit 1) / -1 (bit 0)
__device__ __forceinline__ uint32_t pm1_bytes(uint32_t nib) {
    const uint32_t m = ((nib & 0xfu) * 0x00204081u) & 0x01010101u;  // bit i -> byte i bit 0
    return ((m * 0xffu) ^ 0xfefefefeu) | 0x01010101u;               // 1 -> 0x01, 0 -> 0xff
}

template <int HW>
__device__ __forceinline__ void load_src8(Src8<HW>& c, const IsingSnap& S, int row, int lane) {
#pragma unroll
    for (int q = 0; q < HW; ++q) {
        const int w = lane + 32 * q;
        if (w < S.Mw) {
            const uint4* pp = reinterpret_cast<const uint4*>(S.P8 + ((size_t)row * S.Mw + w) * 8);
            const uint4 p0 = __ldg(pp), p1 = __ldg(pp + 1);
            c.P[q][0] = p0.x, c.P[q][1] = p0.y, c.P[q][2] = p0.z, c.P[q][3] = p0.w;
            c.P[q][4] = p1.x, c.P[q][5] = p1.y, c.P[q][6] = p1.z, c.P[q][7] = p1.w;
            c.b[q] = __ldg(&S.Xb[(size_t)row * S.Mw + w]);
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) c.P[q][k] = 0u;
            c.b[q] = 0u;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) c.X[q][j] = pm1_bytes(c.b[q] >> (4 * j));
    }
}

// a refined distance into the memo (and its survivor bit) or a plain slot array
__device__ __forceinline__ void memo_store(const ScoreOut& out, uint64_t e, double v) {
    const uint32_t s = out.slot[e];
    out.cache_vals[s] = v;
    if (out.cache_bits) atomicOr(&out.cache_bits[s >> 5], 1u << (s & 31));
}

// K1: the bandwidth-bound screen on the int8 field.  Per pair (s stationary, p streamed)
//   g0 = 2<x_s,x_p> - sum_m x_p T_s - sum_m x_s T_p
//      ~ 2 (M - 2 popc(b_s ^ b_p)) - d_s (2 sum_{b_p=1} T8_s - sum T8_s) - d_p sum x_s T8_p
// in exact integer arithmetic (popc over the source's bit planes, dp4a of the partner's
// int8 field against the source's +-1 bytes), |g0 - g| <= E_s + E_p (+ fp32 rounding).
// Pruned pairs are finished here; the rest (survivors, existing edges, kink decisions
// inside the error band) are appended to a compacted list for K2.  Streams M + M/8 bytes
// per pair.
template <int HW>
__global__ void __launch_bounds__(256, HW == 1 ? 4 : 3) ising_screen_kernel(IsingSnap S, HashView W,
                                                              const int32_t* __restrict__ es,
                                                              const int32_t* __restrict__ ep, uint64_t n,
                                                              int chunk, double lambda, double base,
                                                              ScoreOut out, uint64_t* __restrict__ surv,
                                                              float* __restrict__ surv_g,
                                                              uint8_t* __restrict__ surv_flag,
                                                              unsigned long long* __restrict__ nsurv,
                                                              uint64_t* counters,
                                                              const unsigned long long* __restrict__ n_dev,
                                                              unsigned long long* __restrict__ cnt_log) {
    if (n_dev) n = min(n, (uint64_t)*n_dev);
    if (cnt_log && blockIdx.x == 0 && threadIdx.x == 0) *cnt_log = n;
    const int lane = threadIdx.x & 31;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    Src8<HW> cs;
    int cur = -1;
    float4 qs = make_float4(0.f, 0.f, 0.f, 0.f);
    unsigned long long bl_s = 0;
    uint64_t evals = 0;
    const float err0 = 4.f * (float)S.M * 5.9604645e-08f;  // fp32 rounding of the combination
    const float lam = (float)lambda;
    const double pruned_dist = -(base + 0.0);
    for (uint64_t c0 = warp0 * chunk; c0 < n; c0 += nwarps * chunk) {
        const uint64_t c1 = min(c0 + (uint64_t)chunk, n);
        for (uint64_t e = c0; e < c1; ++e) {
            const int s = es[e], p = ep[e];
            if (s != cur) {
                load_src8<HW>(cs, S, s, lane);
                qs = __ldg(&S.Q8[s]);
                bl_s = __ldg(&S.BL[s]);
                cur = s;
            }
            // partner loads first (the W lookup and the per-node constants overlap them)
            uint4 t0[HW], t1[HW];
            uint32_t bp[HW];
#pragma unroll
            for (int q = 0; q < HW; ++q) {
                const int w = lane + 32 * q;
                if (w < S.Mw) {
                    const uint4* tp = reinterpret_cast<const uint4*>(S.T8 + (size_t)p * S.Mp + 32 * w);
                    t0[q] = __ldg(tp);
                    t1[q] = __ldg(tp + 1);
                    bp[q] = __ldg(&S.Xb[(size_t)p * S.Mw + w]);
                } else {
                    t0[q] = t1[q] = make_uint4(0u, 0u, 0u, 0u);
                    bp[q] = 0u;
                }
            }
            const float4 qp = __ldg(&S.Q8[p]);
            const double wcur = (bl_s & bloom_bit(p)) ? hash_get(W, pair_key(s, p), 0.0) : 0.0;
            bool pruned = false;
            float gk = 0.f;
            uint8_t flag = 2;  // 2: existing edge (full fp64), 1: kink inside the error band, 0: survivor
            if (wcur == 0.0) {
                int a1 = 0, a2 = 0, diff = 0;
#pragma unroll
                for (int q = 0; q < HW; ++q) {
                    const uint32_t b = bp[q];
                    int lo = 0;
#pragma unroll
                    for (int k = 0; k < 7; ++k) lo += __popc(cs.P[q][k] & b) << k;
                    a1 += lo - (__popc(cs.P[q][7] & b) << 7);
                    const uint32_t tw[8] = {t0[q].x, t0[q].y, t0[q].z, t0[q].w, t1[q].x, t1[q].y, t1[q].z, t1[q].w};
#pragma unroll
                    for (int j = 0; j < 8; ++j) a2 = __dp4a((int)tw[j], (int)cs.X[q][j], a2);
                    diff += __popc(cs.b[q] ^ b);
                }
                // one packed reduction for (a1, diff): |a1| <= 127 M < 2^19, diff <= M < 2^12
                // (REDUX: one instruction per warp sum)
                const int v = __reduce_add_sync(0xffffffffu, (a1 << 12) + diff);
                a2 = __reduce_add_sync(0xffffffffu, a2);
                const int dsum = v & 4095;
                const int asum = (v - dsum) >> 12;
                const float A = qs.x * (float)(2 * asum - __float_as_int(qs.z));
                const float B = qp.x * (float)a2;
                const float g = (float)(2 * (S.M - 2 * dsum)) - (A + B);
                const float err = (qs.y + qp.y) * 1.0001f + err0;
                pruned = fabsf(g) <= lam - err;
                flag = fabsf(g) < lam + err ? 1 : 0;
                gk = g;
                ++evals;
            }
            if (pruned) {
                // L1 kink: w* = 0 and gain = 0 exactly (inc/model.hpp:205-209)
                if (lane == 0) {
                    if (out.cache_vals && !out.cache_bits) out.cache_vals[out.slot[e]] = pruned_dist;
                    if (out.dist) out.dist[e] = pruned_dist;
                    if (out.w) out.w[e] = 0.0;
                    if (out.gain) out.gain[e] = 0.0;
                    if (out.warn) out.warn[e] = 0;
                }
            } else if (lane == 0) {
                const unsigned long long at = atomicAdd(nsurv, 1ull);
                surv[at] = e;
                surv_g[at] = gk;
                surv_flag[at] = flag;
            }
        }
    }
    if (lane == 0 && counters) atomicAdd((unsigned long long*)&counters[C_EVALS], (unsigned long long)evals);
}

// K1 with several pairs per warp: 32/G pairs at a time, a group of G lanes per pair with
// WPL 32-sample words per lane (word r + G q), segmented butterfly sums inside each
// group; otherwise the arithmetic, bound and outputs of ising_screen_kernel.  Short rows
// (Mw <= 16) need it to keep every lane busy; longer rows use it to share the per-pair
// overhead (indices, coupling probe, decision, outputs) between pairs.  Each warp takes
// 32 consecutive entries per chunk (indices loaded lane-parallel).
// FULL: Mw == G * WPL (every lane's words exist; sizes and offsets compile-time)
template <int G, int WPL, bool FULL>
__global__ void __launch_bounds__(256, WPL == 1 ? 4 : NRG_K1S_MINB) ising_screen_small_kernel(IsingSnap S, HashView W,
                                                                    const int32_t* __restrict__ es,
                                                                    const int32_t* __restrict__ ep, uint64_t n,
                                                                    double lambda, double base, ScoreOut out,
                                                                    uint64_t* __restrict__ surv,
                                                                    float* __restrict__ surv_g,
                                                                    uint8_t* __restrict__ surv_flag,
                                                                    unsigned long long* __restrict__ nsurv,
                                                                    uint64_t* counters,
                                                                    const unsigned long long* __restrict__ n_dev,
                                                                    unsigned long long* __restrict__ cnt_log) {
    if (n_dev) n = min(n, (uint64_t)*n_dev);
    if (cnt_log && blockIdx.x == 0 && threadIdx.x == 0) *cnt_log = n;
    constexpr int P = 32 / G;  // pairs per step
    const uint32_t Mw = FULL ? (uint32_t)(G * WPL) : (uint32_t)S.Mw;
    const uint32_t Mp = FULL ? (uint32_t)(32 * G * WPL) : (uint32_t)S.Mp;
    const int lane = threadIdx.x & 31, grp = lane / G, r = lane % G;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t Ps[WPL][8], Xs[WPL][8], bs[WPL];
    int cur = -1;
    uint64_t evals = 0;
    const float err0 = 4.f * (float)S.M * 5.9604645e-08f;
    const float lam = (float)lambda;
    const double pruned_dist = -(base + 0.0);
    for (uint64_t c0 = warp0 * 32; c0 < n; c0 += nwarps * 32) {
        const int len = (int)min((uint64_t)32, n - c0);
        const int li = lane < len ? lane : 0;
        const int my_s = es[c0 + li], my_p = ep[c0 + li];
        // per-entry operands of the decision, loaded ahead of the step loop
        const float4 qs = __ldg(&S.Q8[my_s]), qp = __ldg(&S.Q8[my_p]);
        const unsigned long long bl_s = __ldg(&S.BL[my_s]);
        int my_v = 0, my_a2 = 0;
        for (int k0 = 0; k0 < len; k0 += P) {
            const int t = k0 + grp;  // this group's entry (offset in the chunk)
            const bool live = t < len;
            const int s = __shfl_sync(0xffffffffu, my_s, live ? t : 0);
            const int p = __shfl_sync(0xffffffffu, my_p, live ? t : 0);
            if (s != cur) {
#pragma unroll
                for (int q = 0; q < WPL; ++q) {
                    const uint32_t w = r + G * q;  // word of this lane
                    if (FULL || w < Mw) {
                        const uint64_t sw = (uint64_t)(uint32_t)s * Mw + w;
                        const uint4* pp = reinterpret_cast<const uint4*>(S.P8 + sw * 8);
                        const uint4 p0 = __ldg(pp), p1 = __ldg(pp + 1);
                        Ps[q][0] = p0.x, Ps[q][1] = p0.y, Ps[q][2] = p0.z, Ps[q][3] = p0.w;
                        Ps[q][4] = p1.x, Ps[q][5] = p1.y, Ps[q][6] = p1.z, Ps[q][7] = p1.w;
                        bs[q] = __ldg(&S.Xb[sw]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 8; ++j) Ps[q][j] = 0u;
                        bs[q] = 0u;
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) Xs[q][j] = pm1_bytes(bs[q] >> (4 * j));
                }
                cur = s;
            }
            uint4 t0[WPL], t1[WPL];
            uint32_t bp[WPL];
#pragma unroll
            for (int q = 0; q < WPL; ++q) {
                const uint32_t w = r + G * q;
                t0[q] = t1[q] = make_uint4(0u, 0u, 0u, 0u);
                bp[q] = 0u;
                if (FULL || w < Mw) {
                    const uint4* tp = reinterpret_cast<const uint4*>(S.T8 + (uint64_t)(uint32_t)p * Mp + 32 * w);
                    t0[q] = __ldg(tp);
                    t1[q] = __ldg(tp + 1);
                    bp[q] = __ldg(&S.Xb[(uint64_t)(uint32_t)p * Mw + w]);
                }
            }
            int a1 = 0, a2 = 0, diff = 0;
#pragma unroll
            for (int q = 0; q < WPL; ++q) {
                int l7 = 0;
#pragma unroll
                for (int j = 0; j < 7; ++j) l7 += __popc(Ps[q][j] & bp[q]) << j;
                a1 += l7 - (__popc(Ps[q][7] & bp[q]) << 7);
                const uint32_t tw[8] = {t0[q].x, t0[q].y, t0[q].z, t0[q].w, t1[q].x, t1[q].y, t1[q].z, t1[q].w};
#pragma unroll
                for (int j = 0; j < 8; ++j) a2 = __dp4a((int)tw[j], (int)Xs[q][j], a2);
                diff += __popc(bs[q] ^ bp[q]);
            }
            int v = (a1 << 12) + diff;
#pragma unroll
            for (int o = G / 2; o; o >>= 1) {
                v += __shfl_xor_sync(0xffffffffu, v, o);
                a2 += __shfl_xor_sync(0xffffffffu, a2, o);
            }
            // hand each group's sums to the lane that owns the entry
            const int src = ((lane - k0) & (P - 1)) * G;
            const int vv = __shfl_sync(0xffffffffu, v, src);
            const int aa = __shfl_sync(0xffffffffu, a2, src);
            if (lane >= k0 && lane < k0 + P) {
                my_v = vv;
                my_a2 = aa;
            }
        }
        // the decision, one entry per lane: couplings (Bloom-filtered probe), the bound
        int my_code = 3;
        float my_g = 0.f;
        const double wcur = (lane < len && (bl_s & bloom_bit(my_p))) ? hash_get(W, pair_key(my_s, my_p), 0.0) : 0.0;
        if (wcur == 0.0) {
            const int dsum = my_v & 4095;
            const int asum = (my_v - dsum) >> 12;
            const float A = qs.x * (float)(2 * asum - __float_as_int(qs.z));
            const float B = qp.x * (float)my_a2;
            my_g = (float)(2 * (S.M - 2 * dsum)) - (A + B);
            const float err = (qs.y + qp.y) * 1.0001f + err0;
            my_code = fabsf(my_g) <= lam - err ? 0 : (fabsf(my_g) < lam + err ? 2 : 1);
            if (lane < len) ++evals;
        }
        const uint64_t e = c0 + lane;
        if (lane < len && my_code == 0) {
            if (out.cache_vals && !out.cache_bits) out.cache_vals[out.slot[e]] = pruned_dist;
            if (out.dist) out.dist[e] = pruned_dist;
            if (out.w) out.w[e] = 0.0;
            if (out.gain) out.gain[e] = 0.0;
            if (out.warn) out.warn[e] = 0;
        }
        const unsigned sv = __ballot_sync(0xffffffffu, lane < len && my_code != 0);
        if (sv) {
            unsigned long long at = 0;
            if (lane == 0) at = atomicAdd(nsurv, (unsigned long long)__popc(sv));
            at = __shfl_sync(0xffffffffu, at, 0);
            if ((sv >> lane) & 1u) {
                const unsigned long long i = at + __popc(sv & ((1u << lane) - 1u));
                surv[i] = e;
                surv_g[i] = my_g;
                surv_flag[i] = (uint8_t)(my_code == 1 ? 0 : (my_code == 2 ? 1 : 2));
            }
        }
    }
    evals = warp_sum((int)evals);
    if (lane == 0 && counters && evals) atomicAdd((unsigned long long*)&counters[C_EVALS], (unsigned long long)evals);
}

// K1, software-pipelined (FULL rows only): the partner rows of the next step are copied
// into shared memory with cp.async while the current step computes, so each warp keeps
// two steps of partner loads in flight without holding them in registers (the small
// kernel is bound by the latency of its partner loads at the occupancy its registers
// allow).  Arithmetic, bound and outputs are those of ising_screen_small_kernel.
// smem: a shared-window address (computed once per thread: converting a generic
// pointer inside the loop costs an S2R of the CTA's shared window per conversion)
__device__ __forceinline__ void cp_async16(uint32_t sa, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// FOUR: the first pass on the stationary node's 4-bit field (4 bit planes instead of 8,
// error E4): pairs it proves pruned are finished; every other pair (and every existing
// coupling) goes to the recheck list `surv`, which the 8-bit pass (FOUR = false, sel =
// that list) screens exactly as before, so K2 sees the same survivors and inputs.
template <int G, int WPL, int NS, bool FOUR>
__global__ void __launch_bounds__(256, NRG_K1S_MINB) ising_screen_pipe_kernel(IsingSnap S, HashView W,
                                                                    const int32_t* __restrict__ es,
                                                                    const int32_t* __restrict__ ep, uint64_t n,
                                                                    double lambda, double base, ScoreOut out,
                                                                    uint64_t* __restrict__ surv,
                                                                    float* __restrict__ surv_g,
                                                                    uint8_t* __restrict__ surv_flag,
                                                                    unsigned long long* __restrict__ nsurv,
                                                                    uint64_t* counters,
                                                                    const unsigned long long* __restrict__ n_dev,
                                                                    unsigned long long* __restrict__ cnt_log,
                                                                    const uint64_t* __restrict__ sel) {
    if (n_dev) n = min(n, (uint64_t)*n_dev);
    if (cnt_log && blockIdx.x == 0 && threadIdx.x == 0) *cnt_log = n;
    constexpr int P = 32 / G;                      // pairs per step
    constexpr uint32_t Mw = G * WPL, Mp = 32 * Mw;  // words / bytes of a row
    // staged partner row: int8 field (4-bit planes in the FOUR pass) + spin words
    constexpr int FB = FOUR ? Mp / 2 : Mp;
    constexpr int RB = FB + 4 * Mw;
    constexpr int CH = RB / 16;                     // 16-byte chunks per staged row
    extern __shared__ __align__(16) unsigned char k1p_smem[];
    const int lane = threadIdx.x & 31, grp = lane / G, r = lane % G;
    unsigned char* wbuf = k1p_smem + (size_t)(threadIdx.x >> 5) * NS * P * RB;  // [stage][pair][row]
    const uint32_t wbuf_sa = (uint32_t)__cvta_generic_to_shared(wbuf);
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    constexpr int NP = FOUR ? 4 : 8;  // bit planes of the stationary field
    uint32_t Ps[WPL][NP], Xs[WPL][8], bs[WPL];
    int cur = -1;
    uint64_t evals = 0;
    const float err0 = 4.f * (float)S.M * 5.9604645e-08f;
    const float lam = (float)lambda;
    const double pruned_dist = -(base + 0.0);
    // stage the partner row of this group's entry into ring buffer `st` (one commit group
    // per step, empty past the chunk's end, so wait_group counts stay uniform).  Lane r of
    // the group copies the 16-byte chunks r, r + G, ... of the field, then of the spin
    // words: per-lane base addresses, the chunk offsets are immediates.
    static_assert((FB / 16) % G == 0, "field chunks must split evenly over the group");
    constexpr int KF = FB / 16 / G;               // field chunks per lane
    constexpr int XC = 4 * Mw / 16;               // spin-word chunks of a row
    constexpr int KX = (XC + G - 1) / G;
    const uint32_t dst_lane = wbuf_sa + (uint32_t)(grp * RB + 16 * r);
    const unsigned char* field = FOUR ? reinterpret_cast<const unsigned char*>(S.P4)
                                      : reinterpret_cast<const unsigned char*>(S.T8);
    const unsigned char* spins = reinterpret_cast<const unsigned char*>(S.Xb);
    auto stage = [&](int st, int p, bool any) {
        if (any) {
            const uint32_t dst = dst_lane + (uint32_t)(st * P * RB);
            const unsigned char* t8 = field + (uint64_t)(uint32_t)p * FB + 16 * r;
            const unsigned char* xb = spins + (uint64_t)(uint32_t)p * (Mw * 4) + 16 * r;
#pragma unroll
            for (int k = 0; k < KF; ++k) cp_async16(dst + 16 * G * k, t8 + 16 * G * k);
#pragma unroll
            for (int k = 0; k < KX; ++k)
                if (XC % G == 0 || r + G * k < XC) cp_async16(dst + FB + 16 * G * k, xb + 16 * G * k);
        }
        cp_async_commit();
    };
    // entries per warp chunk: 32, except on a recheck list (a device-side count that is
    // usually a few hundred entries): spread over the resident warps, so no warp walks 16
    // dependent steps while the others idle
    int chunk = 32;
    if (sel) {
        const uint64_t per = (n + nwarps - 1) / nwarps;
        chunk = (int)min((uint64_t)32, max((uint64_t)P, (per + P - 1) / P * P));
    }
    for (uint64_t c0 = warp0 * chunk; c0 < n; c0 += nwarps * chunk) {
        const int len = (int)min((uint64_t)chunk, n - c0);
        const int li = lane < len ? lane : 0;
        const uint64_t my_e = sel ? sel[c0 + li] : c0 + li;
        const int my_s = es[my_e], my_p = ep[my_e];
        const float4 qs = __ldg(FOUR ? &S.Q4[my_s] : &S.Q8[my_s]), qp = __ldg(FOUR ? &S.Q4[my_p] : &S.Q8[my_p]);
        const unsigned long long bl_s = __ldg(&S.BL[my_s]);
        int my_v = 0, my_a2 = 0;
#pragma unroll
        for (int j = 0; j < NS - 1; ++j) {
            const int tj = j * P + grp;
            const int pj = __shfl_sync(0xffffffffu, my_p, tj < len ? tj : 0);
            stage(j, pj, j * P < len);
        }
        for (int k0 = 0, st = 0; k0 < len; k0 += P, st = st + 1 == NS ? 0 : st + 1) {
            const int t = k0 + grp;
            const bool live = t < len;
            const int s = __shfl_sync(0xffffffffu, my_s, live ? t : 0);
            // the rows NS-1 steps ahead go in flight while this step computes
            const int ka = k0 + (NS - 1) * P;
            const int ta = ka + grp;
            const int pa = __shfl_sync(0xffffffffu, my_p, ta < len ? ta : 0);
            stage(st == 0 ? NS - 1 : st - 1, pa, ka < len);
            if (s != cur) {
#pragma unroll
                for (int q = 0; q < WPL; ++q) {
                    const uint32_t w = r + G * q;
                    const uint64_t sw = (uint64_t)(uint32_t)s * Mw + w;
                    if constexpr (FOUR) {
                        const uint4 p0 = __ldg(reinterpret_cast<const uint4*>(S.P4 + sw * 4));
                        Ps[q][0] = p0.x, Ps[q][1] = p0.y, Ps[q][2] = p0.z, Ps[q][3] = p0.w;
                    } else {
                        const uint4* pp = reinterpret_cast<const uint4*>(S.P8 + sw * 8);
                        const uint4 p0 = __ldg(pp), p1 = __ldg(pp + 1);
                        Ps[q][0] = p0.x, Ps[q][1] = p0.y, Ps[q][2] = p0.z, Ps[q][3] = p0.w;
                        Ps[q][4] = p1.x, Ps[q][5] = p1.y, Ps[q][6] = p1.z, Ps[q][7] = p1.w;
                    }
                    bs[q] = __ldg(&S.Xb[sw]);
                    if constexpr (!FOUR) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) Xs[q][j] = pm1_bytes(bs[q] >> (4 * j));
                    }
                }
                cur = s;
            }
            cp_async_wait<NS - 1>();
            __syncwarp();
            const unsigned char* row = wbuf + (size_t)(st * P + grp) * RB;
            int a1 = 0, a2 = 0, diff = 0;
            if constexpr (FOUR && WPL % 2 == 0) {
                // carry-save form: offset-binary planes (T4 + 8: the sign plane inverted) of the
                // lane's two words summed bit-sliced per weight (w1 half adder, w2/w4/w8 full
                // adders), 5 popcounts per side instead of 8; the offset 8 npl comes off below
                auto csa = [](uint32_t x0, uint32_t x1, uint32_t y0, uint32_t y1, uint32_t z0, uint32_t z1, uint32_t u0,
                              uint32_t u1) {
                    uint32_t s1 = x0 ^ x1, c = x0 & x1;
                    const uint32_t s2 = y0 ^ y1 ^ c;
                    c = (y0 & y1) | (c & (y0 ^ y1));
                    const uint32_t s4 = z0 ^ z1 ^ c;
                    c = (z0 & z1) | (c & (z0 ^ z1));
                    const uint32_t s8 = u0 ^ u1 ^ c;
                    c = (u0 & u1) | (c & (u0 ^ u1));
                    return __popc(s1) + (__popc(s2) << 1) + (__popc(s4) << 2) + (__popc(s8) << 3) + (__popc(c) << 4);
                };
#pragma unroll
                for (int q = 0; q < WPL; q += 2) {
                    const uint32_t w0 = r + G * q, w1 = r + G * (q + 1);
                    const uint32_t bp0 = *reinterpret_cast<const uint32_t*>(row + FB + 4 * w0);
                    const uint32_t bp1 = *reinterpret_cast<const uint32_t*>(row + FB + 4 * w1);
                    const uint4 q0 = *reinterpret_cast<const uint4*>(row + 16 * w0);
                    const uint4 q1 = *reinterpret_cast<const uint4*>(row + 16 * w1);
                    a1 += csa(Ps[q][0] & bp0, Ps[q + 1][0] & bp1, Ps[q][1] & bp0, Ps[q + 1][1] & bp1, Ps[q][2] & bp0,
                              Ps[q + 1][2] & bp1, ~Ps[q][3] & bp0, ~Ps[q + 1][3] & bp1);
                    a2 += csa(q0.x & bs[q], q1.x & bs[q + 1], q0.y & bs[q], q1.y & bs[q + 1], q0.z & bs[q],
                              q1.z & bs[q + 1], ~q0.w & bs[q], ~q1.w & bs[q + 1]);
                    diff += __popc(bs[q] ^ bp0) + __popc(bs[q + 1] ^ bp1);
                }
            } else
#pragma unroll
            for (int q = 0; q < WPL; ++q) {
                const uint32_t w = r + G * q;
                const uint32_t bp = *reinterpret_cast<const uint32_t*>(row + FB + 4 * w);
                int l7 = 0;
#pragma unroll
                for (int j = 0; j < NP - 1; ++j) l7 += __popc(Ps[q][j] & bp) << j;
                a1 += l7 - (__popc(Ps[q][NP - 1] & bp) << (NP - 1));
                if constexpr (FOUR) {
                    // partner's 4-bit planes against the stationary spins: sum of T4_p over
                    // the samples with x_s = +1 (B = d_p (2 a2 - sum4_p) below)
                    const uint4 pp = *reinterpret_cast<const uint4*>(row + 16 * w);
                    a2 += __popc(pp.x & bs[q]) + (__popc(pp.y & bs[q]) << 1) + (__popc(pp.z & bs[q]) << 2) -
                          (__popc(pp.w & bs[q]) << 3);
                } else {
                    const uint4 t0 = *reinterpret_cast<const uint4*>(row + 32 * w);
                    const uint4 t1 = *reinterpret_cast<const uint4*>(row + 32 * w + 16);
                    const uint32_t tw[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
#pragma unroll
                    for (int j = 0; j < 8; ++j) a2 = __dp4a((int)tw[j], (int)Xs[q][j], a2);
                }
                diff += __popc(bs[q] ^ bp);
            }
            __syncwarp();  // the buffer is re-staged NS - 1 steps from now
            int v = (a1 << 12) + diff;
#pragma unroll
            for (int o = G / 2; o; o >>= 1) {
                v += __shfl_xor_sync(0xffffffffu, v, o);
                a2 += __shfl_xor_sync(0xffffffffu, a2, o);
            }
            const int src = ((lane - k0) & (P - 1)) * G;
            const int vv = __shfl_sync(0xffffffffu, v, src);
            const int aa = __shfl_sync(0xffffffffu, a2, src);
            if (lane >= k0 && lane < k0 + P) {
                my_v = vv;
                my_a2 = aa;
            }
        }
        int my_code = 3;
        float my_g = 0.f;
        const double wcur = (lane < len && (bl_s & bloom_bit(my_p))) ? hash_get(W, pair_key(my_s, my_p), 0.0) : 0.0;
        if (wcur == 0.0) {
            const int dsum = my_v & 4095;
            int asum = (my_v - dsum) >> 12;
            int bsum = my_a2;
            if (FOUR && WPL % 2 == 0) {  // offset-binary sums: remove 8 per +1 sample
                asum -= 8 * __float_as_int(qp.w);
                bsum -= 8 * __float_as_int(qs.w);
            }
            const float A = qs.x * (float)(2 * asum - __float_as_int(qs.z));
            const float B = FOUR ? qp.x * (float)(2 * bsum - __float_as_int(qp.z)) : qp.x * (float)my_a2;
            my_g = (float)(2 * (S.M - 2 * dsum)) - (A + B);
            const float err = (qs.y + qp.y) * 1.0001f + err0;
            my_code = fabsf(my_g) <= lam - err ? 0 : (fabsf(my_g) < lam + err ? 2 : 1);
            if (lane < len && (!FOUR || my_code == 0)) ++evals;  // rechecked pairs count in the 8-bit pass
        }
        const uint64_t e = my_e;
        if (lane < len && my_code == 0) {
            if (out.cache_vals && !out.cache_bits) out.cache_vals[out.slot[e]] = pruned_dist;
            if (out.dist) out.dist[e] = pruned_dist;
            if (out.w) out.w[e] = 0.0;
            if (out.gain) out.gain[e] = 0.0;
            if (out.warn) out.warn[e] = 0;
        }
        const unsigned sv = __ballot_sync(0xffffffffu, lane < len && my_code != 0);
        if (sv) {
            unsigned long long at = 0;
            if (lane == 0) at = atomicAdd(nsurv, (unsigned long long)__popc(sv));
            at = __shfl_sync(0xffffffffu, at, 0);
            if ((sv >> lane) & 1u) {
                const unsigned long long i = at + __popc(sv & ((1u << lane) - 1u));
                surv[i] = e;
                if (!FOUR) {
                    surv_g[i] = my_g;
                    surv_flag[i] = (uint8_t)(my_code == 1 ? 0 : (my_code == 2 ? 1 : 2));
                }
            }
        }
    }
    evals = warp_sum((int)evals);
    if (lane == 0 && counters && evals) atomicAdd((unsigned long long*)&counters[C_EVALS], (unsigned long long)evals);
}

// K2: survivors.  Certain survivors (w_cur = 0, |g0| > lambda + err) start Newton
// from K1's fp32 g0 and the per-node sums Tsq = sum T^2 (second derivative at 0 is
// -(2M - Tsq_a - Tsq_b)), so no pass is spent at w = 0; Newton then runs in fp32 on
// the fp32 field copy (8 bytes per sample pair per pass) to fp32 convergence, and one
// fp64 pass on T64 evaluates the objective, the exact derivative and the second-order
// correction (the gain is exact to O(du^3), du ~ 1e-7 / M).  Existing edges and kink
// decisions inside the error band take the full fp64 routine.  (A third-derivative
// start computed in K1 was tried: it cost K1 35% for no K2 gain.)
__global__ void __launch_bounds__(128) ising_refine_kernel(IsingSnap S, HashView W, const int32_t* __restrict__ es,
                                                            const int32_t* __restrict__ ep,
                                                            const uint64_t* __restrict__ surv,
                                                            const float* __restrict__ surv_g,
                                                            const uint8_t* __restrict__ surv_flag, uint64_t ns,
                                                            double lambda, double base, ScoreOut out,
                                                            uint64_t* counters,
                                                            const unsigned long long* __restrict__ ns_dev,
                                                            unsigned long long* __restrict__ cnt_log,
                                                            uint64_t min_ns = 0) {
    if (ns_dev) ns = min(ns, (uint64_t)*ns_dev);
    if (ns <= min_ns) return;  // few survivors: the CTA kernel launched before this one took them
    if (cnt_log && blockIdx.x == 0 && threadIdx.x == 0) *cnt_log = ns;
    const int lane = threadIdx.x & 31;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ns; t += nwarps) {
    const uint64_t e = surv[t];
    const int s = es[e], p = ep[e];
    const int a = s < p ? s : p, b = s < p ? p : s;
    const TSnap T64{S.T64, S.Mp};
    EdgeOptD r;
    // a certain survivor was screened assuming w_cur = 0 (K1 checks W; the tensor-core
    // exhaustive screen does not): existing edges take the full routine
    const double wcur = hash_get(W, pair_key(a, b), 0.0);
    if (surv_flag[t] == 0 && wcur == 0.0) {
        const float g = surv_g[t];
        const double dir = g > 0.f ? 1.0 : -1.0;
        const double phi0 = fabs((double)g) - lambda;
        const double phi1 = -(2.0 * S.M - S.Tsq[a] - S.Tsq[b]);
        const int dot = spin_dot(S.Xb, S.Mw, S.M, a, b);
        const double u0 = phi0 / fmax(-phi1, 1e-300);
        int passes = 0;
        bool conv = false;
        const double u = ising_newton32(S, a, b, lambda, dir, u0, dot, &passes, &conv);
        r = ising_newton64_at(T64, S.Xb, S.Mw, S.M, a, b, 0.0, lambda, dir, u, conv ? 0.0 : u, passes, dot);
    } else {
        r = ising_optimize_edge64(T64, S.Xb, S.Mw, S.M, a, b, wcur, lambda);
    }
    if (lane == 0) {
        const double dist = -(base + r.gain);
        if (out.cache_vals) memo_store(out, e, dist);
        if (out.dist) out.dist[e] = dist;
        if (out.w) out.w[e] = r.w;
        if (out.gain) out.gain[e] = r.gain;
        if (out.warn) out.warn[e] = (uint8_t)r.warn;
        if (counters) {
            atomicAdd((unsigned long long*)&counters[C_EVALS], (unsigned long long)r.passes);
            if (r.warn) atomicAdd((unsigned long long*)&counters[C_WARN], 1ull);
        }
    }
    }
}

// K2 with one CTA per survivor: the per-sample loops of a pass cover M in one or two
// steps of NT * KU independent samples, so a pass costs about one memory latency plus a
// block reduction instead of M / 128 dependent warp steps; a launch holds a few thousand
// survivors at most, so per-survivor latency, not throughput, bounds K2.
template <int NT, int KU>
__global__ void __launch_bounds__(NT, NRG_K2_MINB) ising_refine_cta_kernel(IsingSnap S, HashView W, const int32_t* __restrict__ es,
                                                               const int32_t* __restrict__ ep,
                                                               const uint64_t* __restrict__ surv,
                                                               const float* __restrict__ surv_g,
                                                               const uint8_t* __restrict__ surv_flag, uint64_t ns,
                                                               double lambda, double base, ScoreOut out,
                                                               uint64_t* counters,
                                                               const unsigned long long* __restrict__ ns_dev,
                                                               unsigned long long* __restrict__ cnt_log,
                                                               uint64_t max_ns, unsigned long long* k2max) {
    __shared__ double red[4 * (NT / 32) + 4];
    extern __shared__ double k2_rows[];  // T64 rows a, b (Mp each), then T32 rows a, b
    const BlockScope<NT, KU> sc{red};
    if (ns_dev) ns = min(ns, (uint64_t)*ns_dev);
    if (cnt_log && blockIdx.x == 0 && threadIdx.x == 0) *cnt_log = ns;
    if (blockIdx.x == 0 && threadIdx.x == 0 && k2max) atomicMax(k2max, (unsigned long long)ns);
    if (ns > max_ns) return;  // many survivors: the warp kernel launched after this one takes them
    const int Mp = S.Mp;
    double* ta = k2_rows;
    double* tb = k2_rows + Mp;
    float* fa = reinterpret_cast<float*>(k2_rows + 2 * Mp);
    float* fb = fa + Mp;
    for (uint64_t t = blockIdx.x; t < ns; t += gridDim.x) {
        const uint64_t e = surv[t];
        const int s = es[e], p = ep[e];
        const int a = s < p ? s : p, b = s < p ? p : s;
        const double wcur = hash_get(W, pair_key(a, b), 0.0);
        const bool certain = surv_flag[t] == 0 && wcur == 0.0;
        // stage the rows once: every pass of this survivor reads them from shared memory
        {
            const double2* ga = reinterpret_cast<const double2*>(S.T64 + (size_t)a * Mp);
            const double2* gb = reinterpret_cast<const double2*>(S.T64 + (size_t)b * Mp);
            for (int k = threadIdx.x; k < Mp / 2; k += NT) {
                reinterpret_cast<double2*>(ta)[k] = __ldg(&ga[k]);
                reinterpret_cast<double2*>(tb)[k] = __ldg(&gb[k]);
            }
            if (certain) {
                const float4* ha = reinterpret_cast<const float4*>(S.T32 + (size_t)a * Mp);
                const float4* hb = reinterpret_cast<const float4*>(S.T32 + (size_t)b * Mp);
                for (int k = threadIdx.x; k < Mp / 4; k += NT) {
                    reinterpret_cast<float4*>(fa)[k] = __ldg(&ha[k]);
                    reinterpret_cast<float4*>(fb)[k] = __ldg(&hb[k]);
                }
            }
            __syncthreads();
        }
        const TStaged T64{ta, tb, a};
        EdgeOptD r;
        if (certain) {
            const float g = surv_g[t];
            const double dir = g > 0.f ? 1.0 : -1.0;
            const double phi0 = fabs((double)g) - lambda;
            const double phi1 = -(2.0 * S.M - S.Tsq[a] - S.Tsq[b]);
            const int dot = spin_dot<BlockScope<NT, KU>>(S.Xb, S.Mw, S.M, a, b, sc);
            const double u0 = phi0 / fmax(-phi1, 1e-300);
            int passes = 0;
            bool conv = false;
            const double u = ising_newton32<BlockScope<NT, KU>, true>(S, a, b, lambda, dir, u0, dot, &passes, &conv,
                                                                       sc, fa, fb);
            r = ising_newton64_at<TStaged, BlockScope<NT, KU>>(T64, S.Xb, S.Mw, S.M, a, b, 0.0, lambda, dir, u,
                                                                conv ? 0.0 : u, passes, dot, sc);
        } else {
            r = ising_optimize_edge64<TStaged, BlockScope<NT, KU>>(T64, S.Xb, S.Mw, S.M, a, b, wcur, lambda, sc);
        }
        __syncthreads();  // rows restaged for the next survivor
        if (threadIdx.x == 0) {
            const double dist = -(base + r.gain);
            if (out.cache_vals) memo_store(out, e, dist);
            if (out.dist) out.dist[e] = dist;
            if (out.w) out.w[e] = r.w;
            if (out.gain) out.gain[e] = r.gain;
            if (out.warn) out.warn[e] = (uint8_t)r.warn;
            if (counters) {
                atomicAdd((unsigned long long*)&counters[C_EVALS], (unsigned long long)r.passes);
                if (r.warn) atomicAdd((unsigned long long*)&counters[C_WARN], 1ull);
            }
        }
    }
}

// Gaussian screen (exact mode): for w_cur = 0 the slice maximum is at the kink (w* = 0,
// gain exactly 0, dist = -base) iff |P| <= lambda, P = <u_a, x_b> + <u_b, x_a>
// (gauss_optimize).  P is formed in fp32 from fp32 copies of U and X with a rigorous
// bound, |P32 - P64| <= (2 (M/32 + 8) 2^-24 + 1e-12)(||u_a|| ||x_b|| + ||u_b|| ||x_a||)
// (input rounding, per-lane fp32 accumulation of M/16 products, a 5-level warp tree, and
// the fp64 path's own rounding; Cauchy-Schwarz for sum |u x|); pairs it cannot settle,
// and existing couplings, go to the fp64 kernel.  The stationary node's rows stay in
// registers across a worklist run.  NF: float4 per lane per row (Mp = 128 NF).
template <int NF>
__global__ void __launch_bounds__(256) gauss_screen_kernel(GaussSnap G, HashView W, const int32_t* __restrict__ es,
                                                           const int32_t* __restrict__ ep, uint64_t n,
                                                           const unsigned long long* __restrict__ n_dev,
                                                           double lambda, double base, ScoreOut out,
                                                           uint64_t* __restrict__ surv,
                                                           unsigned long long* __restrict__ nsurv,
                                                           uint64_t* counters,
                                                           unsigned long long* __restrict__ cnt_log = nullptr) {
    if (n_dev) n = min(n, (uint64_t)*n_dev);
    if (cnt_log && blockIdx.x == 0 && threadIdx.x == 0) *cnt_log = n;
    const int lane = threadIdx.x & 31;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const int Mp = 128 * NF;
    float4 us[NF], xs[NF];
    int cur = -1;
    const double relerr = 2.0 * ((double)G.M / 32.0 + 8.0) * 5.9604644775390625e-08 + 1e-12;
    const double pruned_dist = -(base + 0.0);
    uint64_t evals = 0;
    for (uint64_t c0 = warp0 * 32; c0 < n; c0 += nwarps * 32) {
        const int len = (int)min((uint64_t)32, n - c0);
        const int li = lane < len ? lane : 0;
        const int my_s = es[c0 + li], my_p = ep[c0 + li];
        float my_P = 0.f;
        for (int k = 0; k < len; ++k) {
            const int s = __shfl_sync(0xffffffffu, my_s, k);
            const int p = __shfl_sync(0xffffffffu, my_p, k);
            if (s != cur) {
                const float4* u4 = reinterpret_cast<const float4*>(G.U32 + (size_t)s * Mp);
                const float4* x4 = reinterpret_cast<const float4*>(G.X32 + (size_t)s * Mp);
#pragma unroll
                for (int q = 0; q < NF; ++q) {
                    us[q] = __ldg(&u4[lane + 32 * q]);
                    xs[q] = __ldg(&x4[lane + 32 * q]);
                }
                cur = s;
            }
            const float4* up = reinterpret_cast<const float4*>(G.U32 + (size_t)p * Mp);
            const float4* xp = reinterpret_cast<const float4*>(G.X32 + (size_t)p * Mp);
            float acc = 0.f;
#pragma unroll
            for (int q = 0; q < NF; ++q) {
                const float4 a = __ldg(&xp[lane + 32 * q]), b = __ldg(&up[lane + 32 * q]);
                acc = fmaf(us[q].x, a.x, acc);
                acc = fmaf(us[q].y, a.y, acc);
                acc = fmaf(us[q].z, a.z, acc);
                acc = fmaf(us[q].w, a.w, acc);
                acc = fmaf(b.x, xs[q].x, acc);
                acc = fmaf(b.y, xs[q].y, acc);
                acc = fmaf(b.z, xs[q].z, acc);
                acc = fmaf(b.w, xs[q].w, acc);
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == k) my_P = acc;
        }
        const uint64_t e = c0 + lane;
        bool settled = false;
        if (lane < len) {
            const int a = min(my_s, my_p), b = max(my_s, my_p);
            const bool maybe_edge = (G.BL[a] & bloom_bit(b)) != 0ull;
            const double wcur = maybe_edge ? hash_get(W, pair_key(a, b), 0.0) : 0.0;
            if (wcur == 0.0) {
                const double bound = relerr * (G.nu[a] * sqrt(G.xx[b]) + G.nu[b] * sqrt(G.xx[a])) * 1.01;
                settled = fabs((double)my_P) <= lambda - bound;
                ++evals;
            }
            if (settled) {
                if (out.cache_vals && !out.cache_bits) out.cache_vals[out.slot[e]] = pruned_dist;
                if (out.dist) out.dist[e] = pruned_dist;
                if (out.w) out.w[e] = 0.0;
                if (out.gain) out.gain[e] = 0.0;
                if (out.warn) out.warn[e] = 0;
            }
        }
        const unsigned sv = __ballot_sync(0xffffffffu, lane < len && !settled);
        if (sv) {
            unsigned long long at = 0;
            if (lane == 0) at = atomicAdd(nsurv, (unsigned long long)__popc(sv));
            at = __shfl_sync(0xffffffffu, at, 0);
            if ((sv >> lane) & 1u) surv[at + __popc(sv & ((1u << lane) - 1u))] = e;
        }
    }
    evals = warp_sum((int)evals);
    if (lane == 0 && counters && evals) atomicAdd((unsigned long long*)&counters[C_EVALS], (unsigned long long)evals);
}

// fp64 kernels for the remaining modes: Ising exact (M > 2048), Ising gradient,
// Gaussian exact / gradient.  One warp per entry.
__global__ void __launch_bounds__(256) generic_score_kernel(int kind, int mode, IsingSnap S, GaussSnap G,
                                                            HashView W, const int32_t* __restrict__ es,
                                                            const int32_t* __restrict__ ep, uint64_t n,
                                                            double lambda, double base, ScoreOut out,
                                                            uint64_t* counters,
                                                            const uint64_t* __restrict__ sel = nullptr,
                                                            const unsigned long long* __restrict__ n_dev = nullptr) {
    if (n_dev) n = min(n, (uint64_t)*n_dev);
    const int lane = threadIdx.x & 31;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t evals = 0, warns = 0;
    for (uint64_t t = warp0; t < n; t += nwarps) {
        const uint64_t e = sel ? sel[t] : t;
        const int s = es[e], p = ep[e];
        const int a = s < p ? s : p, b = s < p ? p : s;
        const double wcur = hash_get(W, pair_key(a, b), 0.0);
        double dist;
        EdgeOptD r;
        r.w = 0.0;
        r.gain = 0.0;
        r.warn = 0;
        r.passes = 1;
        if (kind == ISING) {
            const TSnap T{S.T64, S.Mp};
            if (mode == EXACT) {
                r = ising_optimize_edge64(T, S.Xb, S.Mw, S.M, a, b, wcur, lambda);
                dist = -(base + r.gain);
            } else {
                const double g = ising_gradient64(T, S.Xb, S.Mw, S.M, a, b);
                const double sg = wcur > 0.0 ? 1.0 : (wcur < 0.0 ? -1.0 : 0.0);
                dist = -fabs(g - lambda * sg);
            }
        } else {
            const USnap Uf{G.U, G.Mp};
            const double ta = G.theta[a], tb = G.theta[b];
            const GaussCoef cf = gauss_coef(Uf, G.X, G.Mp, G.M, a, b, ta * ta, tb * tb, G.xx[a], G.xx[b]);
            if (mode == EXACT) {
                r = gauss_optimize(cf, wcur, lambda);
                dist = -(base + r.gain);
            } else {
                const double sg = wcur > 0.0 ? 1.0 : (wcur < 0.0 ? -1.0 : 0.0);
                dist = -fabs(-cf.P - lambda * sg);
            }
        }
        evals += r.passes;
        warns += r.warn;
        if (lane == 0) {
            if (out.cache_vals) memo_store(out, e, dist);
            if (out.dist) out.dist[e] = dist;
            if (out.w) out.w[e] = r.w;
            if (out.gain) out.gain[e] = r.gain;
            if (out.warn) out.warn[e] = (uint8_t)r.warn;
        }
    }
    if (lane == 0 && counters) {
        atomicAdd((unsigned long long*)&counters[C_EVALS], (unsigned long long)evals);
        if (warns) atomicAdd((unsigned long long*)&counters[C_WARN], (unsigned long long)warns);
    }
}

// test metrics (TableMetric / LineMetric)
__global__ void metric_score_kernel(int mode, const double* __restrict__ table, uint64_t tn,
                                    const double* __restrict__ pos, const int32_t* __restrict__ es,
                                    const int32_t* __restrict__ ep, uint64_t n, ScoreOut out) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const int s = es[e], p = ep[e];
    const int a = s < p ? s : p, b = s < p ? p : s;
    const double d = mode == TABLE ? table[(uint64_t)a * tn + b] : fabs(pos[s] - pos[p]);
    if (out.cache_vals) memo_store(out, e, d);
    if (out.dist) out.dist[e] = d;
}

static int num_sms(Context& c) {
    static int sms = 0;
    if (!sms) NRG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
    return sms;
}

// K2 over a survivor list (entries surv[t] of the worklist (s, p)), timed into k2_*.
// ns_dev: the survivor count lives on the device (ns is then the list's capacity); the
// grid strides over it, so no host round trip sits between K1 and K2.
void refine_survivors(Context& c, const int32_t* s, const int32_t* p, const uint64_t* surv, const float* surv_g,
                      const uint8_t* surv_flag, uint64_t ns, double base, const ScoreOut& out,
                      const unsigned long long* ns_dev) {
    if (!ns) return;
    const cudaEvent_t a = c.mark();
    const uint64_t rb = std::min<uint64_t>(ceil_div((int64_t)ns * 32, 128), (uint64_t)num_sms(c) * 16);
    int slot = -1;
    unsigned long long* lg = ns_dev ? c.log_slot(&slot) : nullptr;
    // CTA-per-survivor K2 (NT 128, 4 samples per thread per step); NRG_K2_WARP=1 keeps
    // the warp-per-survivor kernel (A/B: profiles/r01_k2_cta/)
    if (!NRG_ENV_ON("NRG_K2_WARP")) {
        const uint64_t cb = std::min<uint64_t>(ns, (uint64_t)num_sms(c) * 32);
        const size_t smem = (size_t)c.Mp * 24;
        static size_t smem_set = 0;
        if (smem > smem_set) {
            NRG_CUDA(cudaFuncSetAttribute(ising_refine_cta_kernel<128, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
            smem_set = smem;
        }
        // The survivor count is on the device.  Up to 4 survivors per CTA the CTA kernel
        // (latency-bound launches), beyond that the warp kernel (first sweeps: millions,
        // throughput-bound); each exits at once when the count is the other's.  When the
        // last generation's launches all fit CTA mode (the steady state) only the CTA
        // kernel is launched and takes any count.
        const uint64_t max_ns = c.k2_wide ? 4 * cb : ~0ull;
        if (!c.k2max.p) NRG_CUDA(cudaMemsetAsync(c.k2max.as<unsigned long long>(1), 0, 8, c.stream));
        unsigned long long* k2max = static_cast<unsigned long long*>(c.k2max.p);
        ising_refine_cta_kernel<128, 4><<<(unsigned)cb, 128, smem, c.stream>>>(
            c.isnap(), c.Wview(), s, p, surv, surv_g, surv_flag, ns, c.lambda, base, out, c.dcounters(), ns_dev, lg,
            max_ns, k2max);
        if (c.k2_wide && ns > max_ns)
            ising_refine_kernel<<<(unsigned)rb, 128, 0, c.stream>>>(c.isnap(), c.Wview(), s, p, surv, surv_g,
                                                                    surv_flag, ns, c.lambda, base, out, c.dcounters(),
                                                                    ns_dev, lg, max_ns);

    } else {
        ising_refine_kernel<<<(unsigned)rb, 128, 0, c.stream>>>(c.isnap(), c.Wview(), s, p, surv, surv_g, surv_flag,
                                                                ns, c.lambda, base, out, c.dcounters(), ns_dev, lg);
    }
    NRG_LAUNCH_CHECK();
    c.span(T_K2, a, (double)ns, slot);
}

void score_entries(Context& c, int mode, const int32_t* s, const int32_t* p, uint64_t n,
                   const ScoreOut& out, const unsigned long long* n_dev) {
    if (n == 0) return;
    if (n_dev && !(mode == EXACT && ((c.kind == ISING && (c.Mp + 1023) / 1024 <= 2) ||
                                     (c.kind == GAUSSIAN && c.Mp <= 1024 && !NRG_ENV_ON("NRG_NO_GAUSS_SCREEN"))))) {
        // only the screen takes a device-side count: settle it here for the other paths
        unsigned long long h = 0;
        h = c.read_scalar(n_dev);
        n = std::min<uint64_t>(n, h);
        n_dev = nullptr;
        if (n == 0) return;
    }
    c.tic();
    if (mode == TABLE || mode == LINE) {
        if (mode == TABLE && !c.table_n) fail(22, "no distance table set");
        if (mode == LINE && !c.line_n) fail(22, "no line metric set");
        metric_score_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(
            mode, static_cast<double*>(c.table.p), c.table_n, static_cast<double*>(c.line.p), s, p, n,
            out);
        NRG_LAUNCH_CHECK();
        c.toc(P_SCORE);
        return;
    }
    ensure_snapshot(c);
    // the generation base only enters distances (update rounds ask for w alone)
    const double base = (mode == EXACT && (out.dist || out.cache_vals)) ? generation_base(c) : 0.0;
    c.tic();
    const int sms = num_sms(c);
    const int HW = (c.Mp + 1023) / 1024;  // 32-sample words per lane
    if (c.kind == ISING && mode == EXACT && HW <= 2) {
        const int chunk = 8;
        const uint64_t chunks = (n + chunk - 1) / chunk;
        const uint64_t blocks = std::min<uint64_t>((chunks + 7) / 8, (uint64_t)sms * 12);
        const IsingSnap S = c.isnap();
        const HashView W = c.Wview();
        uint64_t* surv = c.sc_surv.as<uint64_t>(n);
        float* surv_g = c.sc_g.as<float>(n);
        uint8_t* surv_flag = c.sc_flag.as<uint8_t>(n);
        unsigned long long* nsurv = c.sc_n.as<unsigned long long>(1);
        NRG_CUDA(cudaMemsetAsync(nsurv, 0, 8, c.stream));
        const cudaEvent_t k1a = c.mark();
        int k1slot = -1;
        unsigned long long* k1log = n_dev ? c.log_slot(&k1slot) : nullptr;
#define NRG_LAUNCH_MQ(Q)                                                                              \
    ising_screen_kernel<Q><<<(unsigned)blocks, 256, 0, c.stream>>>(S, W, s, p, n, chunk, c.lambda, base, \
                                                                    out, surv, surv_g, surv_flag, nsurv,   \
                                                                    c.dcounters(), n_dev, k1log)
        const int G = c.Mw <= 4 ? 4 : (c.Mw <= 8 ? 8 : 16);
        const int WPL = (c.Mw + G - 1) / G;  // 1, 2 (M <= 1024) or up to 4 (M <= 2048)
        if (!NRG_ENV_ON("NRG_K1_WIDE") && (WPL == 1 || (WPL == 2 && !NRG_ENV_ON("NRG_K1_ONE_PAIR")))) {
            const uint64_t sblocks = std::min<uint64_t>(ceil_div(n, 8 * 32), (uint64_t)sms * 16);
#define NRG_LAUNCH_SMALL(GG, WW, FF)                                                                          \
    ising_screen_small_kernel<GG, WW, FF><<<(unsigned)sblocks, 256, 0, c.stream>>>(S, W, s, p, n, c.lambda,   \
                                                                                 base, out, surv, surv_g,      \
                                                                                 surv_flag, nsurv,             \
                                                                                 c.dcounters(), n_dev, k1log)
            const bool full = c.Mw == G * WPL && !NRG_ENV_ON("NRG_K1_NOFULL");
            if (WPL == 2 && full && !NRG_ENV_ON("NRG_K1_NOPIPE")) {
                static const int ns = getenv("NRG_K1_STAGES") ? atoi(getenv("NRG_K1_STAGES")) : 2;
                const bool four = S.P4 && !NRG_ENV_ON("NRG_K1_NO4");
                // first pass (4-bit): prunes what it can, lists the rest for the exact 8-bit pass
                uint64_t* rl = four ? c.sc_rchk.as<uint64_t>(n) : nullptr;
                unsigned long long* rn = four ? c.sc_rn.as<unsigned long long>(1) : nullptr;
                if (four) NRG_CUDA(cudaMemsetAsync(rn, 0, 8, c.stream));
                static const int g4 = getenv("NRG_K1_G4") ? atoi(getenv("NRG_K1_G4")) : 8;  // lanes per pair (4-bit pass)
                // the recheck pass strides over a device-side count that is a fraction of a percent of
                // n in the steady state: one resident wave of CTAs (3 per SM) instead of a grid sized
                // for n, whose empty CTAs cost ~20 us per launch
                static const int rwaves = getenv("NRG_K1R_CTAS") ? atoi(getenv("NRG_K1R_CTAS")) : 3;
                const uint64_t rblocks = std::min<uint64_t>(sblocks, (uint64_t)sms * rwaves);
#define NRG_LAUNCH_PIPE(NSV)                                                                                       \
    {                                                                                                              \
        constexpr size_t smem = (size_t)8 * (NSV) * 2 * (1024 + 128);                                             \
        constexpr size_t smem4 = (size_t)8 * (NSV) * 2 * (512 + 128);                                             \
        static bool attr = false;                                                                                  \
        if (!attr) {                                                                                               \
            NRG_CUDA(cudaFuncSetAttribute(ising_screen_pipe_kernel<16, 2, NSV, false>,                             \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));                \
            NRG_CUDA(cudaFuncSetAttribute(ising_screen_pipe_kernel<16, 2, NSV, true>,                              \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));                \
            attr = true;                                                                                           \
        }                                                                                                          \
        if (four) {                                                                                                \
            if (g4 == 8) {                                                                                         \
                constexpr size_t sm8 = (size_t)8 * (NSV) * 4 * (512 + 128);                                        \
                static bool attr8 = false;                                                                         \
                if (!attr8) {                                                                                      \
                    NRG_CUDA(cudaFuncSetAttribute(ising_screen_pipe_kernel<8, 4, NSV, true>,                       \
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm8));         \
                    attr8 = true;                                                                                  \
                }                                                                                                  \
                ising_screen_pipe_kernel<8, 4, NSV, true><<<(unsigned)sblocks, 256, sm8, c.stream>>>(              \
                    S, W, s, p, n, c.lambda, base, out, rl, nullptr, nullptr, rn, c.dcounters(), n_dev, k1log,      \
                    nullptr);                                                                                      \
            } else if (g4 == 4) {                                                                                  \
                constexpr size_t sm4 = (size_t)8 * (NSV) * 8 * (512 + 128);                                        \
                static bool attr4 = false;                                                                         \
                if (!attr4) {                                                                                      \
                    NRG_CUDA(cudaFuncSetAttribute(ising_screen_pipe_kernel<4, 8, NSV, true>,                       \
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4));         \
                    attr4 = true;                                                                                  \
                }                                                                                                  \
                ising_screen_pipe_kernel<4, 8, NSV, true><<<(unsigned)sblocks, 256, sm4, c.stream>>>(              \
                    S, W, s, p, n, c.lambda, base, out, rl, nullptr, nullptr, rn, c.dcounters(), n_dev, k1log,      \
                    nullptr);                                                                                      \
            } else                                                                                                 \
                ising_screen_pipe_kernel<16, 2, NSV, true><<<(unsigned)sblocks, 256, smem4, c.stream>>>(           \
                    S, W, s, p, n, c.lambda, base, out, rl, nullptr, nullptr, rn, c.dcounters(), n_dev, k1log,      \
                    nullptr);                                                                                      \
            ising_screen_pipe_kernel<16, 2, NSV, false><<<(unsigned)rblocks, 256, smem, c.stream>>>(               \
                S, W, s, p, n, c.lambda, base, out, surv, surv_g, surv_flag, nsurv, c.dcounters(), rn, nullptr,    \
                rl);                                                                                               \
        } else {                                                                                                   \
            ising_screen_pipe_kernel<16, 2, NSV, false><<<(unsigned)sblocks, 256, smem, c.stream>>>(               \
                S, W, s, p, n, c.lambda, base, out, surv, surv_g, surv_flag, nsurv, c.dcounters(), n_dev, k1log,   \
                nullptr);                                                                                          \
        }                                                                                                          \
    }
                switch (ns) {
                    case 2: NRG_LAUNCH_PIPE(2); break;
                    case 3: NRG_LAUNCH_PIPE(3); break;
                    default: NRG_LAUNCH_PIPE(4); break;
                }
#undef NRG_LAUNCH_PIPE
            } else if (WPL == 2) {
                if (full) NRG_LAUNCH_SMALL(16, 2, true); else NRG_LAUNCH_SMALL(16, 2, false);
            } else {
                switch (G) {
                    case 4: if (full) NRG_LAUNCH_SMALL(4, 1, true); else NRG_LAUNCH_SMALL(4, 1, false); break;
                    case 8: if (full) NRG_LAUNCH_SMALL(8, 1, true); else NRG_LAUNCH_SMALL(8, 1, false); break;
                    default: if (full) NRG_LAUNCH_SMALL(16, 1, true); else NRG_LAUNCH_SMALL(16, 1, false); break;
                }
            }
#undef NRG_LAUNCH_SMALL
        } else {
            switch (HW) {
                case 1: NRG_LAUNCH_MQ(1); break;
                case 2: NRG_LAUNCH_MQ(2); break;
                default: fail(100, "unsupported padded sample count");
            }
        }
#undef NRG_LAUNCH_MQ
        NRG_LAUNCH_CHECK();
        c.span(T_K1, k1a, (double)n, k1slot);
        // K2 strides over the device-side survivor count (no host round trip)
        refine_survivors(c, s, p, surv, surv_g, surv_flag, n, base, out, nsurv);
    } else if (c.kind == GAUSSIAN && mode == EXACT && c.Mp <= 1024 && !NRG_ENV_ON("NRG_NO_GAUSS_SCREEN")) {
        // screen in fp32, the pairs it cannot settle (and existing couplings) in fp64
        uint64_t* surv = c.sc_surv.as<uint64_t>(n);
        unsigned long long* nsurv = c.sc_n.as<unsigned long long>(1);
        NRG_CUDA(cudaMemsetAsync(nsurv, 0, 8, c.stream));
        const uint64_t sblocks = std::min<uint64_t>(ceil_div(n, 8 * 32), (uint64_t)sms * 16);
        const GaussSnap G = c.gsnap();
        // timed like K1 (the screen every pair takes): kernel_stats' k1_* describe it
        const cudaEvent_t k1a = c.mark();
        int k1slot = -1;
        unsigned long long* k1log = c.log_slot(&k1slot);
        switch (c.Mp / 128) {
            case 2: gauss_screen_kernel<2><<<(unsigned)sblocks, 256, 0, c.stream>>>(G, c.Wview(), s, p, n, n_dev, c.lambda, base, out, surv, nsurv, c.dcounters(), k1log); break;
            case 4: gauss_screen_kernel<4><<<(unsigned)sblocks, 256, 0, c.stream>>>(G, c.Wview(), s, p, n, n_dev, c.lambda, base, out, surv, nsurv, c.dcounters(), k1log); break;
            case 6: gauss_screen_kernel<6><<<(unsigned)sblocks, 256, 0, c.stream>>>(G, c.Wview(), s, p, n, n_dev, c.lambda, base, out, surv, nsurv, c.dcounters(), k1log); break;
            default: gauss_screen_kernel<8><<<(unsigned)sblocks, 256, 0, c.stream>>>(G, c.Wview(), s, p, n, n_dev, c.lambda, base, out, surv, nsurv, c.dcounters(), k1log); break;
        }
        NRG_LAUNCH_CHECK();
        c.span(T_K1, k1a, (double)n, k1slot);
        const uint64_t blocks = std::min<uint64_t>((n + 7) / 8, (uint64_t)sms * 16);
        generic_score_kernel<<<(unsigned)blocks, 256, 0, c.stream>>>(
            c.kind, mode, c.isnap(), G, c.Wview(), s, p, n, c.lambda, base, out, c.dcounters(), surv, nsurv);
        NRG_LAUNCH_CHECK();
    } else {
        const uint64_t blocks = std::min<uint64_t>((n + 7) / 8, (uint64_t)sms * 16);
        generic_score_kernel<<<(unsigned)blocks, 256, 0, c.stream>>>(
            c.kind, mode, c.isnap(), c.gsnap(), c.Wview(), s, p, n, c.lambda, base, out, c.dcounters());
        NRG_LAUNCH_CHECK();
    }
    c.toc(P_SCORE);
}

// ---------------------------------------------------------------- all pairs
__global__ void fill_rows_kernel(const int32_t* __restrict__ nodes, uint64_t n, uint64_t r0, uint64_t r1,
                                 const uint64_t* __restrict__ off, int32_t* __restrict__ es,
                                 int32_t* __restrict__ ep) {
    // one block per row a in [r0, r1): pairs (nodes[a], nodes[c]) for c > a
    const uint64_t a = r0 + blockIdx.x;
    if (a >= r1) return;
    const uint64_t base = off[a] - off[r0];
    for (uint64_t c = a + 1 + threadIdx.x; c < n; c += blockDim.x) {
        es[base + (c - a - 1)] = nodes[a];
        ep[base + (c - a - 1)] = nodes[c];
    }
}

void score_all_pairs(Context& c, int mode, const int32_t* nodes, uint64_t n, double* dist) {
    // row-major upper triangle (inc/find_best.hpp:72-86), chunked by rows
    if (n < 2) return;
    if (mode == EXACT && score_all_pairs_tc(c, nodes, n, dist)) {
        if (c.rank == 0) counters_add_host(c, C_MISSES, n * (n - 1) / 2);
        return;
    }
    std::vector<uint64_t> off(n + 1, 0);
    for (uint64_t a = 0; a < n; ++a) off[a + 1] = off[a] + (n - a - 1);
    uint64_t* doff = c.s_o.as<uint64_t>(n + 1);
    NRG_CUDA(cudaMemcpyAsync(doff, off.data(), (n + 1) * 8, cudaMemcpyHostToDevice, c.stream));
    const uint64_t maxp = 1ull << 25;
    uint64_t r0 = 0;
    while (r0 < n - 1) {
        uint64_t r1 = r0 + 1;
        while (r1 < n && off[r1 + 1] - off[r0] <= maxp) ++r1;
        const uint64_t cnt = off[r1] - off[r0];
        int32_t* es = c.s_m.as<int32_t>(cnt);
        int32_t* ep = c.s_n.as<int32_t>(cnt);
        fill_rows_kernel<<<(unsigned)(r1 - r0), 256, 0, c.stream>>>(nodes, n, r0, r1, doff, es, ep);
        NRG_LAUNCH_CHECK();
        ScoreOut out;
        out.dist = dist + off[r0];
        score_entries(c, mode, es, ep, cnt, out);
        r0 = r1;
    }
    // probes count as misses (no cache on this path); replicated on every rank, counted once
    if (c.rank == 0) counters_add_host(c, C_MISSES, n * (n - 1) / 2);
}

// ---------------------------------------------------------------- cached batch lookups
__device__ __forceinline__ uint64_t cache_claim(HashView h, uint64_t key, bool& mine) {
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

__global__ void probe_claim_kernel(HashView h, const int32_t* __restrict__ qi, const int32_t* __restrict__ qj,
                                   uint64_t n, uint32_t* __restrict__ slot, int32_t* __restrict__ ws,
                                   int32_t* __restrict__ wp, uint32_t* __restrict__ wslot,
                                   unsigned long long* __restrict__ wcount, uint64_t* counters,
                                   uint64_t* live) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool mine = false;
    uint64_t sl = 0;
    if (e < n) {
        sl = cache_claim(h, pair_key(qi[e], qj[e]), mine);
        slot[e] = (uint32_t)sl;
    }
    const unsigned ball = __ballot_sync(0xffffffffu, mine);
    const int lane = threadIdx.x & 31;
    unsigned long long basei = 0;
    if (lane == 0 && ball) basei = atomicAdd(wcount, (unsigned long long)__popc(ball));
    basei = __shfl_sync(0xffffffffu, basei, 0);
    if (mine) {
        const uint64_t at = basei + __popc(ball & ((1u << lane) - 1));
        ws[at] = qi[e];
        wp[at] = qj[e];
        wslot[at] = (uint32_t)sl;
    }
    const unsigned hitb = __ballot_sync(0xffffffffu, e < n && !mine);
    if (lane == 0) {
        if (ball) {
            atomicAdd((unsigned long long*)&counters[C_MISSES], (unsigned long long)__popc(ball));
            atomicAdd((unsigned long long*)live, (unsigned long long)__popc(ball));
        }
        if (hitb) atomicAdd((unsigned long long*)&counters[C_HITS], (unsigned long long)__popc(hitb));
    }
}

__global__ void gather_cache_kernel(MemoView C, const uint32_t* __restrict__ slot, uint64_t n,
                                    double* __restrict__ out) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) out[e] = memo_value(C, slot[e]);
}

void distance_batch(Context& c, int mode, const int32_t* qi, const int32_t* qj, uint64_t n, double* dist) {
    if (n == 0) return;
    if (mode == TABLE || mode == LINE) {
        ScoreOut out;
        out.dist = dist;
        score_entries(c, mode, qi, qj, n, out);
        return;
    }
    cache_reserve(c, n);
    uint32_t* slot = c.s_c.as<uint32_t>(n);
    int32_t* ws = c.s_d.as<int32_t>(n);
    int32_t* wp = c.s_e.as<int32_t>(n);
    uint32_t* wslot = c.s_f.as<uint32_t>(n);
    unsigned long long* wcount = c.s_g.as<unsigned long long>(1);
    NRG_CUDA(cudaMemsetAsync(wcount, 0, 8, c.stream));
    probe_claim_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(
        c.Cview(), qi, qj, n, slot, ws, wp, wslot, wcount, c.dcounters(), static_cast<uint64_t*>(c.Ccount.p));
    NRG_LAUNCH_CHECK();
    unsigned long long nw = 0;
    nw = c.read_scalar(wcount);
    ScoreOut out;
    out.cache_vals = c.Cview().vals;
    out.cache_bits = c.dsurvbits();
    out.slot = wslot;
    score_entries(c, mode, ws, wp, nw, out);
    gather_cache_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(c.mview(), slot, n, dist);
    NRG_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- scored-pair sample
__global__ void sample_keys_kernel(const uint64_t* __restrict__ keys, uint64_t cap, uint64_t stride,
                                   uint64_t seed, uint64_t limit, int32_t* __restrict__ oi,
                                   int32_t* __restrict__ oj, unsigned long long* __restrict__ cnt) {
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= cap) return;
    const uint64_t k = keys[s];
    if (k == kEmptyKey) return;
    if (mix64(k ^ seed) % stride != 0) return;
    const unsigned long long at = atomicAdd(cnt, 1ull);
    if (at < limit) {
        oi[at] = (int32_t)(k >> 32);
        oj[at] = (int32_t)(k & 0xffffffffu);
    }
}

uint64_t sample_scored_pairs(Context& c, uint64_t cap, uint64_t seed, int32_t* oi, int32_t* oj) {
    if (!c.Ccap || !cap) return 0;
    uint64_t live = 0;
    live = c.read_scalar(static_cast<const uint64_t*>(c.Ccount.p));
    const uint64_t stride = std::max<uint64_t>(1, live / cap);
    unsigned long long* cnt = c.s_g.as<unsigned long long>(1);
    NRG_CUDA(cudaMemsetAsync(cnt, 0, 8, c.stream));
    sample_keys_kernel<<<(unsigned)ceil_div(c.Ccap, 256), 256, 0, c.stream>>>(
        static_cast<uint64_t*>(c.Ckeys.p), c.Ccap, stride, seed, cap, oi, oj, cnt);
    NRG_LAUNCH_CHECK();
    unsigned long long h = 0;
    h = c.read_scalar(cnt);
    return std::min<uint64_t>(h, cap);
}

// ---------------------------------------------------------------- live optimize_edge / gradient
__global__ void __launch_bounds__(256) live_opt_kernel(int kind, const uint32_t* __restrict__ Xb,
                                                       const double* __restrict__ Xd,
                                                       const double* __restrict__ H,
                                                       const double* __restrict__ theta, int M, int Mp,
                                                       int Mw, HashView W, const int32_t* __restrict__ qi,
                                                       const int32_t* __restrict__ qj, uint64_t n,
                                                       double lambda, int want_grad, double* __restrict__ w,
                                                       double* __restrict__ gain, uint8_t* __restrict__ warn,
                                                       uint64_t* counters) {
    const int lane = threadIdx.x & 31;
    const uint64_t e = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (e >= n) return;
    const int a = min(qi[e], qj[e]), b = max(qi[e], qj[e]);
    const double wcur = hash_get(W, pair_key(a, b), 0.0);
    const double sg = wcur > 0.0 ? 1.0 : (wcur < 0.0 ? -1.0 : 0.0);
    EdgeOptD r;
    if (kind == ISING) {
        const TLive T{H, theta, Mp};
        if (want_grad) {
            const double g = ising_gradient64(T, Xb, Mw, M, a, b);
            if (lane == 0) w[e] = g - lambda * sg;
            return;
        }
        r = ising_optimize_edge64(T, Xb, Mw, M, a, b, wcur, lambda);
    } else {
        const ULive Uf{Xd, H, theta, Mp};
        double xxa = 0.0, xxb = 0.0;
        for (int m = lane; m < M; m += 32) {
            const double va = Xd[(size_t)a * Mp + m], vb = Xd[(size_t)b * Mp + m];
            xxa += va * va;
            xxb += vb * vb;
        }
        xxa = warp_sum(xxa);
        xxb = warp_sum(xxb);
        const double ta = theta[a], tb = theta[b];
        const GaussCoef cf = gauss_coef(Uf, Xd, Mp, M, a, b, ta * ta, tb * tb, xxa, xxb);
        if (want_grad) {
            if (lane == 0) w[e] = -cf.P - lambda * sg;
            return;
        }
        r = gauss_optimize(cf, wcur, lambda);
    }
    if (lane == 0) {
        if (w) w[e] = r.w;
        if (gain) gain[e] = r.gain;
        if (warn) warn[e] = (uint8_t)r.warn;
        atomicAdd((unsigned long long*)&counters[C_EVALS], (unsigned long long)r.passes);
        if (r.warn) atomicAdd((unsigned long long*)&counters[C_WARN], 1ull);
    }
}

void optimize_edge_live(Context& c, const int32_t* i, const int32_t* j, uint64_t n, double* w,
                        double* gain, uint8_t* warn) {
    if (!n) return;
    live_opt_kernel<<<(unsigned)ceil_div(n * 32, 256), 256, 0, c.stream>>>(
        c.kind, c.dXb(), c.dXd(), c.dH(), c.dtheta(), c.M, c.Mp, c.Mw, c.Wview(), i, j, n, c.lambda, 0, w,
        gain, warn, c.dcounters());
    NRG_LAUNCH_CHECK();
}

void edge_gradient_live(Context& c, const int32_t* i, const int32_t* j, uint64_t n, double* g) {
    if (!n) return;
    live_opt_kernel<<<(unsigned)ceil_div(n * 32, 256), 256, 0, c.stream>>>(
        c.kind, c.dXb(), c.dXd(), c.dH(), c.dtheta(), c.M, c.Mp, c.Mw, c.Wview(), i, j, n, c.lambda, 1, g,
        nullptr, nullptr, c.dcounters());
    NRG_LAUNCH_CHECK();
}

}  // namespace nrg
