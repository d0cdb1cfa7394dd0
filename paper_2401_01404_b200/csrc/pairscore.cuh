// pairscore.cuh — device routines for the pair score (inc/model.hpp:201-217) and the
// edge gradient (:175-195), shared by the scoring kernels and the update kernel.
//
// Ising, any pair (a, b) with current coupling w_cur:
//   y_a = x_b tanh(z_a(w_cur)),  y_b = x_a tanh(z_b(w_cur)),  s = x_a x_b,  D = w - w_cur
//   x_b tanh z_a(w)         = (y_a + tanh D) / (1 + y_a tanh D)                      (q_a)
//   l_a(w) - l_a(w_cur)     = s D - ln(cosh D + y_a sinh D)
//   ln(cosh D + y sinh D)   = |D| + log1p(-(1 - sgn(D) y)/2 * (1 - e^{-2|D|}))      (stable)
//   L'(w)  = sum 2s - q_a - q_b,     L''(w) = -sum (1-q_a^2) + (1-q_b^2)
// so the whole 1-D problem depends only on x_a, x_b, T_a, T_b and w_cur.  The
// reference's golden search (inc/line_search.hpp) returns the best evaluated point
// within ~1e-8 of the maximiser of this concave slice; we solve L'(w) = sign(g0)
// lambda by safeguarded Newton instead and report the same (w*, gain) to within
// the parity tolerances.  Every order-dependent accumulation runs with canonical
// roles a = min(i,j), b = max(i,j) so a pair's score is bitwise independent of which
// node asked for it.
#pragma once
#include "context.cuh"

namespace nrg {

__device__ __forceinline__ double xsign(uint32_t word, int bit) {
    return ((word >> bit) & 1u) ? 1.0 : -1.0;
}

// Reduction scope of the per-sample loops: one warp (scoring kernels) or one CTA
// (update kernel, where a dependency chain of updates makes per-update latency the
// bound).  Element m of a row is owned by thread m % NT of the scope.
struct WarpScope {
    static constexpr int NT = 32;
    static constexpr int KU = 4;  // independent accumulator sets per thread (fp64 passes)
    __device__ __forceinline__ int tid() const { return threadIdx.x & 31; }
    __device__ __forceinline__ void sum4(double& a, double& b, double& c, double& d) const {
        a = warp_sum(a);
        b = warp_sum(b);
        c = warp_sum(c);
        d = warp_sum(d);
    }
    __device__ __forceinline__ double sum(double a) const { return warp_sum(a); }
};
template <int NT_, int KU_ = 1>
struct BlockScope {
    static constexpr int NT = NT_;
    static constexpr int KU = KU_;
    double* red;  // shared scratch: 4 * (NT/32) + 4 doubles
    __device__ __forceinline__ int tid() const { return threadIdx.x; }
    __device__ __forceinline__ void sum4(double& a, double& b, double& c, double& d) const {
        constexpr int W = NT / 32;
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        a = warp_sum(a);
        b = warp_sum(b);
        c = warp_sum(c);
        d = warp_sum(d);
        if (lane == 0) {
            red[4 * w + 0] = a;
            red[4 * w + 1] = b;
            red[4 * w + 2] = c;
            red[4 * w + 3] = d;
        }
        __syncthreads();
        if (w == 0) {
            double x0 = lane < W ? red[4 * lane + 0] : 0.0, x1 = lane < W ? red[4 * lane + 1] : 0.0;
            double x2 = lane < W ? red[4 * lane + 2] : 0.0, x3 = lane < W ? red[4 * lane + 3] : 0.0;
            x0 = warp_sum(x0);
            x1 = warp_sum(x1);
            x2 = warp_sum(x2);
            x3 = warp_sum(x3);
            if (lane == 0) {
                red[4 * W + 0] = x0;
                red[4 * W + 1] = x1;
                red[4 * W + 2] = x2;
                red[4 * W + 3] = x3;
            }
        }
        __syncthreads();
        a = red[4 * W + 0];
        b = red[4 * W + 1];
        c = red[4 * W + 2];
        d = red[4 * W + 3];
        __syncthreads();  // scratch reusable
    }
    __device__ __forceinline__ double sum(double a) const {
        double b = 0.0, c = 0.0, d = 0.0;
        sum4(a, b, c, d);
        return a;
    }
};

// Result of one fp64 pass over the samples at coupling w (D = w - w_cur).
struct Pass64 {
    double Lp;    // L'(w)
    double Lpp;   // L''(w)
    double Lppp;  // L'''(w)
    double Flik;  // likelihood part of F(w) - F(w_cur)
};

// T provider: snapshot rows (T64) or live rows tanh(H + theta)
struct TSnap {
    const double* T64;
    int Mp;
    __device__ __forceinline__ double operator()(int row, int m) const {
        return T64[(size_t)row * Mp + m];
    }
};
struct TLive {
    const double* H;
    const double* theta;
    int Mp;
    __device__ __forceinline__ double operator()(int row, int m) const {
        return tanh(__ldcg(&H[(size_t)row * Mp + m]) + __ldcg(&theta[row]));
    }
};

// 1/x for x = (1 + y_a tanh D)(1 + y_b tanh D) in (0, 4): the MUFU.RCP64H seed
// (rcp.approx.ftz.f64, ~2^-22) refined by two fp64 Newton steps (~2^-88 before
// rounding); a third of the cost of an IEEE divide and no fp32 round trip.
__device__ __forceinline__ double rcp64(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = r * fma(-x, r, 2.0);
    r = r * fma(-x, r, 2.0);
    return r;
}

// <x_a, x_b> = M - 2 popc(x_a ^ x_b) (padding bits are zero in both rows)
template <class SC = WarpScope>
__device__ __forceinline__ int spin_dot(const uint32_t* __restrict__ Xb, int Mw, int M, int a, int b,
                                        const SC& sc = SC()) {
    double d = 0.0;
    for (int k = sc.tid(); k < Mw; k += SC::NT) d += (double)__popc(__ldg(&Xb[(size_t)a * Mw + k]) ^ __ldg(&Xb[(size_t)b * Mw + k]));
    return M - 2 * (int)sc.sum(d);
}

// One fp64 pass over the samples by the whole scope (result valid in every thread).
// With t = tanh D, A = 1 + y_a t, B = 1 + y_b t:
//   q_a = (y_a + t) B / (A B),  q_b = (y_b + t) A / (A B)        (one reciprocal)
//   L'  = 2 <x_a,x_b> - sum (q_a + q_b),   L'' = -sum (1-q_a^2) + (1-q_b^2)
//   F   = 2 D <x_a,x_b> - 2 M ln cosh D - sum log1p((y_a + y_b) t + y_a y_b t^2)
// (ln(cosh D + y sinh D) = ln cosh D + ln(1 + y t), and 1 + (y_a + y_b) t + y_a y_b t^2
// = A B).  kNeedF adds the objective, kL3 the third derivative (kink pass only).
template <class TP, bool kNeedF, class SC = WarpScope, bool kL3 = false>
__device__ __forceinline__ Pass64 ising_pass64(const TP& T, const uint32_t* __restrict__ Xb, int Mw,
                                               int M, int a, int b, double D, int dot, const SC& sc = SC()) {
    // kU independent accumulator sets per thread for a warp scope: the fp64 add chains,
    // not the math, bound a single-set loop at the occupancy the scoring kernels run at
    // (a CTA scope has enough warps and only a few samples per thread)
    constexpr int kU = SC::KU;
    const int tid = sc.tid();
    const double t = tanh(D);
    const double omt2 = 1.0 - t * t;
    const double t2 = t * t;
    // objective: sum ln(A B) as one log per kU samples of the product (A B >= 1/4 for
    // |t| <= 1/2, so a product of kU factors stays far from under/overflow); per-sample
    // log1p beyond that
    const bool prodlog = fabs(t) <= 0.5;
    double Sq[kU], Lq[kU], L3q[kU], Slq[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) Sq[u] = Lq[u] = L3q[u] = Slq[u] = 0.0;
    double P = 1.0;
    int nP = 0;
    for (int m0 = tid; m0 < M; m0 += SC::NT * kU) {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int m = m0 + u * SC::NT;
            if (m < M) {
                const uint32_t wa = __ldg(&Xb[(size_t)a * Mw + (m >> 5)]);
                const uint32_t wb = __ldg(&Xb[(size_t)b * Mw + (m >> 5)]);
                const double xa = xsign(wa, m & 31), xb = xsign(wb, m & 31);
                const double ya = xb * T(a, m);
                const double yb = xa * T(b, m);
                const double A = fma(ya, t, 1.0), B = fma(yb, t, 1.0);
                const double AB = A * B;
                const double r = rcp64(AB);
                const double da = B * r, db = A * r;
                const double qa = (ya + t) * da, qb = (yb + t) * db;
                Sq[u] += qa + qb;
                const double d1a = (1.0 - ya * ya) * omt2 * da * da, d1b = (1.0 - yb * yb) * omt2 * db * db;
                Lq[u] -= d1a + d1b;
                if (kL3) L3q[u] += 2.0 * (qa * d1a + qb * d1b);
                if (kNeedF) {
                    if (prodlog) P *= AB;
                    else Slq[u] += log1p(fma((ya + yb), t, ya * yb * t2));
                }
            }
        }
        if (kNeedF && prodlog && (nP += kU) >= 4) {
            Slq[0] += log(P);
            P = 1.0;
            nP = 0;
        }
    }
    if (kNeedF && prodlog && nP) Slq[0] += log(P);
    double Sqs = Sq[0], Lpp = Lq[0], L3 = L3q[0], Sl = Slq[0];
#pragma unroll
    for (int u = 1; u < kU; ++u) {
        Sqs += Sq[u];
        Lpp += Lq[u];
        L3 += L3q[u];
        Sl += Slq[u];
    }
    sc.sum4(Sqs, Lpp, L3, Sl);
    Pass64 r;
    r.Lp = 2.0 * dot - Sqs;
    r.Lpp = Lpp;
    r.Lppp = L3;
    if (kNeedF) {
        const double ad = fabs(D);
        const double lncosh = ad + log1p(exp(-2.0 * ad)) - 0.69314718055994530942;
        r.Flik = (2.0 * D * dot - 2.0 * M * lncosh) - Sl;
    } else {
        r.Flik = 0.0;
    }
    return r;
}

// fp32 pass over the fp32 field copy (warp scope): L'(w) and L''(w) at w = dir u for
// w_cur = 0, for the Newton iterations ahead of the final fp64 pass.  Lane l owns
// samples 4 l + 128 j .. +3 (one 16-byte load per row and step).
struct Pass32 {
    float Lp, Lpp;
};
__device__ __forceinline__ float rcp32(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// kStaged: the two fp32 rows sit in shared memory at sa / sb (T32 unused)
template <class SC = WarpScope, bool kStaged = false>
__device__ __forceinline__ Pass32 ising_pass32(const float* __restrict__ T32, int Mp, const uint32_t* __restrict__ Xb,
                                               int Mw, int M, int a, int b, float t, int dot, const SC& sc = SC(),
                                               const float* sa = nullptr, const float* sb = nullptr) {
    const int lane = sc.tid();
    const float4* Ta = reinterpret_cast<const float4*>(kStaged ? sa : T32 + (size_t)a * Mp);
    const float4* Tb = reinterpret_cast<const float4*>(kStaged ? sb : T32 + (size_t)b * Mp);
    float Sq = 0.f, Lq = 0.f;
    for (int m0 = 4 * lane; m0 < M; m0 += 4 * SC::NT) {
        float4 va, vb;
        if constexpr (kStaged) {
            va = Ta[m0 >> 2];
            vb = Tb[m0 >> 2];
        } else {
            va = __ldg(&Ta[m0 >> 2]);
            vb = __ldg(&Tb[m0 >> 2]);
        }
        const uint32_t wa = __ldg(&Xb[(size_t)a * Mw + (m0 >> 5)]) >> (m0 & 31);
        const uint32_t wb = __ldg(&Xb[(size_t)b * Mw + (m0 >> 5)]) >> (m0 & 31);
        const float ta[4] = {va.x, va.y, va.z, va.w}, tb[4] = {vb.x, vb.y, vb.z, vb.w};
        float s = 0.f, l = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (m0 + c < M) {
                const float ya = ((wb >> c) & 1u) ? ta[c] : -ta[c];
                const float yb = ((wa >> c) & 1u) ? tb[c] : -tb[c];
                const float A = fmaf(ya, t, 1.f), B = fmaf(yb, t, 1.f);
                const float r = rcp32(A * B);
                const float da = B * r, db = A * r;
                s += (ya + t) * da + (yb + t) * db;
                l += fmaf(-ya, ya, 1.f) * da * da + fmaf(-yb, yb, 1.f) * db * db;
            }
        }
        Sq += s;
        Lq += l;
    }
    if constexpr (SC::NT == 32) {
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            Sq += __shfl_xor_sync(0xffffffffu, Sq, o);
            Lq += __shfl_xor_sync(0xffffffffu, Lq, o);
        }
    } else {
        double x = Sq, y = Lq, z = 0.0, w = 0.0;
        sc.sum4(x, y, z, w);
        Sq = (float)x;
        Lq = (float)y;
    }
    return {(float)(2 * dot) - Sq, -(1.f - t * t) * Lq};
}

struct EdgeOptD {
    double w, gain;
    int warn;
    int passes;
};

// Safeguarded Newton for phi(u) = dir L'(w) - lambda = 0 on u > 0 (w = dir u,
// D = w - w_cur), from the iterate u.  Passes without the objective until the last
// step predicts convergence (|du_last| small: the first pass when the caller already
// converged u, e.g. in fp32); that pass evaluates the slice gain and applies the
// second-order Newton correction, so the gain is exact to O(du^3).
template <class TP, class SC = WarpScope>
__device__ EdgeOptD ising_newton64_at(const TP& T, const uint32_t* __restrict__ Xb, int Mw, int M, int a, int b,
                                      double w_cur, double lambda, double dir, double u, double du_last,
                                      int passes, int dot, const SC& sc = SC()) {
    EdgeOptD r;
    r.warn = 0;
    r.passes = passes;
    double lo = 0.0, hi = INFINITY, prevF = -INFINITY;
    for (int it = 0; it < 100; ++it) {
        const double scale = fmax(u, 1e-3);
        const bool final_try = fabs(du_last) <= 0.03 * scale;
        const double D = dir * u - w_cur;
        const Pass64 p = final_try ? ising_pass64<TP, true, SC>(T, Xb, Mw, M, a, b, D, dot, sc)
                                   : ising_pass64<TP, false, SC>(T, Xb, Mw, M, a, b, D, dot, sc);
        ++r.passes;
        const double phi = dir * p.Lp - lambda, dphi = p.Lpp;
        const double du = (dphi < 0.0) ? -phi / dphi : NAN;
        if (final_try && isfinite(du) && fabs(du) <= 1e-3 * scale) {
            const double gain = (p.Flik - lambda * u) + lambda * fabs(w_cur) + 0.5 * phi * du;
            if (gain < 0.0) {  // inc/model.hpp:215
                r.w = w_cur;
                r.gain = 0.0;
            } else {
                r.w = dir * (u + du);
                r.gain = gain;
            }
            return r;
        }
        if (phi > 0.0) lo = u; else hi = u;
        double un = u + du;
        if (!(un > lo && un < hi) || !isfinite(un)) un = isinf(hi) ? fmax(2.0 * u, 1.0) : 0.5 * (lo + hi);
        if (un > 0x1.0p64) {  // bracket failure (inc/line_search.hpp:64-84 cap)
            r.warn = 1;
            break;
        }
        if (isinf(hi) && un > 64.0) {
            // separable columns: the slice saturates numerically; stop once the
            // objective no longer increases (the reference's doubling stops there too)
            const Pass64 pf = ising_pass64<TP, true, SC>(T, Xb, Mw, M, a, b, dir * un - w_cur, dot, sc);
            ++r.passes;
            const double F = pf.Flik - lambda * un;
            if (!(F > prevF)) break;
            prevF = F;
        }
        du_last = un - u;
        u = un;
        if (hi - lo <= 1e-15 * fmax(1.0, u)) du_last = 0.0;
    }
    // plateau / bracket failure: objective at the last iterate
    const Pass64 pf = ising_pass64<TP, true, SC>(T, Xb, Mw, M, a, b, dir * u - w_cur, dot, sc);
    ++r.passes;
    const double gain = (pf.Flik - lambda * u) + lambda * fabs(w_cur);
    if (gain < 0.0) {
        r.w = w_cur;
        r.gain = 0.0;
    } else {
        r.w = dir * u;
        r.gain = gain;
    }
    return r;
}

// Newton from the quadratic model phi0 + phi1 u + phi2 u^2 / 2 of phi at u = 0.
template <class TP, class SC = WarpScope>
__device__ EdgeOptD ising_newton64(const TP& T, const uint32_t* __restrict__ Xb, int Mw, int M, int a, int b,
                                   double w_cur, double lambda, double dir, double phi0, double phi1,
                                   double phi2, int passes, int dot, const SC& sc = SC()) {
    const double disc = phi1 * phi1 - 2.0 * phi2 * phi0;
    double u = (disc >= 0.0 && phi1 < 0.0) ? 2.0 * phi0 / (-phi1 + sqrt(disc)) : phi0 / fmax(-phi1, 1e-300);
    if (!(u > 0.0) || !isfinite(u)) u = 1.0;
    return ising_newton64_at<TP, SC>(T, Xb, Mw, M, a, b, w_cur, lambda, dir, u, u, passes, dot, sc);
}

// Newton iterations in fp32 for a certain survivor (w_cur = 0, |g0| > lambda) from the
// quadratic-model start u; returns the fp32-converged iterate (|error| ~ 1e-7 / M) for
// the single fp64 objective pass, or the start when fp32 cannot be trusted (|u| large,
// no descent).  Adds the passes spent to *passes.
template <class SC = WarpScope, bool kStaged = false>
__device__ __forceinline__ double ising_newton32(const IsingSnap& S, int a, int b, double lambda, double dir,
                                                 double u0, int dot, int* passes, bool* conv, const SC& sc = SC(),
                                                 const float* sa = nullptr, const float* sb = nullptr) {
    *conv = false;
    float u = (float)u0;
    const float lam = (float)lambda, fd = (float)dir;
    for (int it = 0; it < 12; ++it) {
        if (!(u > 0.f && u < 2.f)) return u0;
        const Pass32 p = ising_pass32<SC, kStaged>(S.T32, S.Mp, S.Xb, S.Mw, S.M, a, b, tanhf(fd * u), dot, sc, sa, sb);
        ++*passes;
        const float phi = fd * p.Lp - lam;
        if (!(p.Lpp < 0.f)) return u0;
        const float du = -phi / p.Lpp;
        float un = u + du;
        if (!(un > 0.f)) un = 0.5f * u;
        u = un;
        if (fabsf(du) <= 1e-4f * fmaxf(u, 1e-3f)) {
            *conv = true;
            return (double)u;
        }
    }
    return (double)u;
}

// Full fp64 optimize_edge for the Ising slice (a < b canonical): the kink pass at
// w = 0 (inc/model.hpp:204-209), then ising_newton64.  Used for existing edges,
// uncertain kink decisions and the update kernel.
template <class TP, class SC = WarpScope>
__device__ EdgeOptD ising_optimize_edge64(const TP& T, const uint32_t* __restrict__ Xb, int Mw, int M,
                                          int a, int b, double w_cur, double lambda, const SC& sc = SC()) {
    const int dot = spin_dot<SC>(Xb, Mw, M, a, b, sc);
    const Pass64 p0 = w_cur != 0.0 ? ising_pass64<TP, true, SC, true>(T, Xb, Mw, M, a, b, -w_cur, dot, sc)
                                   : ising_pass64<TP, false, SC, true>(T, Xb, Mw, M, a, b, 0.0, dot, sc);
    const double g0 = p0.Lp;
    if (fabs(g0) <= lambda) {
        EdgeOptD r;
        r.warn = 0;
        r.passes = 1;
        double gain = p0.Flik + lambda * fabs(w_cur);  // F(0) - F(w_cur)
        if (w_cur == 0.0) gain = 0.0;
        r.w = 0.0;
        r.gain = gain < 0.0 ? 0.0 : gain;
        return r;
    }
    const double dir = g0 > 0.0 ? 1.0 : -1.0;
    return ising_newton64<TP, SC>(T, Xb, Mw, M, a, b, w_cur, lambda, dir, fabs(g0) - lambda, p0.Lpp,
                                  dir * p0.Lppp, 1, dot, sc);
}

// T rows staged in shared memory (update kernel: tanh computed once per pair)
struct TStaged {
    const double* ta;
    const double* tb;
    int a;
    __device__ __forceinline__ double operator()(int row, int m) const { return row == a ? ta[m] : tb[m]; }
};

// fp64 likelihood derivative at the current coupling with the L1 subgradient:
// edge_gradient (inc/model.hpp:175-195).  g = sum 2 x_a x_b - x_b T_a - x_a T_b.
template <class TP>
__device__ __forceinline__ double ising_gradient64(const TP& T, const uint32_t* __restrict__ Xb, int Mw,
                                                   int M, int a, int b) {
    const int lane = threadIdx.x & 31;
    double g = 0.0;
    for (int k = 0; k * 32 < M; ++k) {
        const int m = lane + 32 * k;
        const uint32_t wa = __ldg(&Xb[(size_t)a * Mw + k]);
        const uint32_t wb = __ldg(&Xb[(size_t)b * Mw + k]);
        if (m < M) {
            const double xa = xsign(wa, lane), xb = xsign(wb, lane);
            g += (2.0 * xa * xb - xb * T(a, m)) - xa * T(b, m);
        }
    }
    return warp_sum(g);
}

// Gaussian closed form: with u = x + theta^2 s (current
// residual), P = <u_a,x_b> + <u_b,x_a>, Hc = theta_a^2 |x_b|^2 + theta_b^2 |x_a|^2,
//   F(w) - F(w_cur) = -D P - D^2 Hc / 2 - lambda(|w| - |w_cur|),   D = w - w_cur
//   g0 = L'(0) = -P + Hc w_cur,   w* = sign(g0)(|g0| - lambda)/Hc
struct GaussCoef {
    double P, Hc;
};
template <class UP, class SC = WarpScope>
__device__ __forceinline__ GaussCoef gauss_coef(const UP& Uf, const double* __restrict__ X, int Mp, int M,
                                                int a, int b, double ta2, double tb2, double xxa,
                                                double xxb, const SC& sc = SC()) {
    double P = 0.0;
    for (int m = sc.tid(); m < M; m += SC::NT) {
        const double xa = X[(size_t)a * Mp + m], xb = X[(size_t)b * Mp + m];
        P += Uf(a, m) * xb + Uf(b, m) * xa;
    }
    GaussCoef c;
    c.P = sc.sum(P);
    c.Hc = ta2 * xxb + tb2 * xxa;
    return c;
}
__device__ __forceinline__ EdgeOptD gauss_optimize(const GaussCoef& c, double w_cur, double lambda) {
    EdgeOptD r;
    r.warn = 0;
    r.passes = 1;
    const double g0 = -c.P + c.Hc * w_cur;
    double w;
    if (fabs(g0) <= lambda || !(c.Hc > 0.0)) {
        w = 0.0;
    } else {
        w = (g0 > 0.0 ? 1.0 : -1.0) * (fabs(g0) - lambda) / c.Hc;
    }
    const double D = w - w_cur;
    double gain = -D * c.P - 0.5 * D * D * c.Hc - lambda * (fabs(w) - fabs(w_cur));
    if (w == 0.0 && w_cur == 0.0) gain = 0.0;
    if (gain < 0.0) {
        if (w == 0.0) {
            r.w = 0.0;  // kink branch clamps the gain only (inc/model.hpp:206-208)
        } else {
            r.w = w_cur;
        }
        r.gain = 0.0;
    } else {
        r.w = w;
        r.gain = gain;
    }
    return r;
}

struct USnap {
    const double* U;
    int Mp;
    __device__ __forceinline__ double operator()(int row, int m) const { return U[(size_t)row * Mp + m]; }
};
struct ULive {
    const double* X;
    const double* H;
    const double* theta;
    int Mp;
    __device__ __forceinline__ double operator()(int row, int m) const {
        const double t = __ldcg(&theta[row]);
        return X[(size_t)row * Mp + m] + t * t * __ldcg(&H[(size_t)row * Mp + m]);
    }
};

}  // namespace nrg
