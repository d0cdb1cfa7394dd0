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
    __device__ __forceinline__ int tid() const { return threadIdx.x & 31; }
    __device__ __forceinline__ void sum4(double& a, double& b, double& c, double& d) const {
        a = warp_sum(a);
        b = warp_sum(b);
        c = warp_sum(c);
        d = warp_sum(d);
    }
    __device__ __forceinline__ double sum(double a) const { return warp_sum(a); }
};
template <int NT_>
struct BlockScope {
    static constexpr int NT = NT_;
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

// 1/x for x = (1 + y_a tanh D)(1 + y_b tanh D) in (0, 4): fp32 reciprocal refined by two fp64 Newton
// steps (relative error ~2^-96 before rounding), a third of the cost of an IEEE divide
__device__ __forceinline__ double rcp64(double x) {
    double r = (double)__frcp_rn((float)x);
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
// (ln(cosh D + y sinh D) = ln cosh D + ln(1 + y t); one log1p per sample for both
// sides).  kNeedF adds the objective, kL3 the third derivative (kink pass only).
template <class TP, bool kNeedF, class SC = WarpScope, bool kL3 = false>
__device__ __forceinline__ Pass64 ising_pass64(const TP& T, const uint32_t* __restrict__ Xb, int Mw,
                                               int M, int a, int b, double D, int dot, const SC& sc = SC()) {
    const int tid = sc.tid();
    const double t = tanh(D);
    const double omt2 = 1.0 - t * t;
    const double t2 = t * t;
    double Sq = 0.0, Lpp = 0.0, L3 = 0.0, Sl = 0.0;
    for (int m = tid; m < M; m += SC::NT) {
        const uint32_t wa = __ldg(&Xb[(size_t)a * Mw + (m >> 5)]);
        const uint32_t wb = __ldg(&Xb[(size_t)b * Mw + (m >> 5)]);
        const double xa = xsign(wa, m & 31), xb = xsign(wb, m & 31);
        const double ya = xb * T(a, m);
        const double yb = xa * T(b, m);
        const double A = fma(ya, t, 1.0), B = fma(yb, t, 1.0);
        const double r = rcp64(A * B);
        const double da = B * r, db = A * r;
        const double qa = (ya + t) * da, qb = (yb + t) * db;
        Sq += qa + qb;
        const double d1a = (1.0 - ya * ya) * omt2 * da * da, d1b = (1.0 - yb * yb) * omt2 * db * db;
        Lpp -= d1a + d1b;
        if (kL3) L3 += 2.0 * (qa * d1a + qb * d1b);
        if (kNeedF) Sl += log1p(fma((ya + yb), t, ya * yb * t2));
    }
    sc.sum4(Sq, Lpp, L3, Sl);
    Pass64 r;
    r.Lp = 2.0 * dot - Sq;
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

struct EdgeOptD {
    double w, gain;
    int warn;
    int passes;
};

// Safeguarded Newton for phi(u) = dir L'(dir u) - lambda = 0 on u > 0 (D = dir u - w_cur),
// started from the root of the quadratic model phi0 + phi1 u + phi2 u^2/2 (phi1 < 0).
// Passes without the log1p objective until the step predicts convergence; the last
// pass evaluates the slice gain and applies the second-order Newton correction.
template <class TP, class SC = WarpScope>
__device__ EdgeOptD ising_newton64(const TP& T, const uint32_t* __restrict__ Xb, int Mw, int M, int a, int b,
                                   double w_cur, double lambda, double dir, double phi0, double phi1,
                                   double phi2, int passes, int dot, const SC& sc = SC()) {
    EdgeOptD r;
    r.warn = 0;
    r.passes = passes;
    double u;
    {
        const double disc = phi1 * phi1 - 2.0 * phi2 * phi0;
        u = (disc >= 0.0 && phi1 < 0.0) ? 2.0 * phi0 / (-phi1 + sqrt(disc)) : phi0 / fmax(-phi1, 1e-300);
        if (!(u > 0.0) || !isfinite(u)) u = 1.0;
    }
    double lo = 0.0, hi = INFINITY, du_last = u, prevF = -INFINITY;
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
