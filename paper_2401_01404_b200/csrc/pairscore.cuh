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

// Result of one fp64 pass over the samples at coupling w (D = w - w_cur).
struct Pass64 {
    double Lp;    // L'(w)
    double Lpp;   // L''(w)
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

// One warp-wide fp64 pass (all lanes participate; result valid in all lanes).
template <class TP, bool kNeedF>
__device__ __forceinline__ Pass64 ising_pass64(const TP& T, const uint32_t* __restrict__ Xb, int Mw,
                                               int M, int a, int b, double D) {
    const int lane = threadIdx.x & 31;
    const double t = tanh(D);
    const double omt2 = 1.0 - t * t;
    const double A = fabs(D);
    const double sg = D > 0.0 ? 1.0 : (D < 0.0 ? -1.0 : 0.0);
    const double E = -expm1(-2.0 * A);  // 1 - e^{-2|D|}
    double Lp = 0.0, Lpp = 0.0, F = 0.0;
    for (int k = 0; k * 32 < M; ++k) {
        const int m = lane + 32 * k;
        const uint32_t wa = __ldg(&Xb[(size_t)a * Mw + k]);
        const uint32_t wb = __ldg(&Xb[(size_t)b * Mw + k]);
        if (m < M) {
            const double xa = xsign(wa, lane), xb = xsign(wb, lane);
            const double ya = xb * T(a, m);
            const double yb = xa * T(b, m);
            const double s = xa * xb;
            const double da = 1.0 / (1.0 + ya * t);
            const double db = 1.0 / (1.0 + yb * t);
            const double qa = (ya + t) * da, qb = (yb + t) * db;
            Lp += (2.0 * s - qa) - qb;
            Lpp -= (1.0 - ya * ya) * omt2 * da * da + (1.0 - yb * yb) * omt2 * db * db;
            if (kNeedF) {
                const double la = A + log1p(-0.5 * (1.0 - sg * ya) * E);
                const double lb = A + log1p(-0.5 * (1.0 - sg * yb) * E);
                F += (2.0 * s * D - la) - lb;
            }
        }
    }
    Pass64 r;
    r.Lp = warp_sum(Lp);
    r.Lpp = warp_sum(Lpp);
    r.Flik = kNeedF ? warp_sum(F) : 0.0;
    return r;
}

struct EdgeOptD {
    double w, gain;
    int warn;
    int passes;
};

// Full fp64 optimize_edge for the Ising slice (a < b canonical).  Used for existing
// edges, uncertain kink decisions, fp32 fallbacks and the update kernel.
template <class TP>
__device__ EdgeOptD ising_optimize_edge64(const TP& T, const uint32_t* __restrict__ Xb, int Mw, int M,
                                          int a, int b, double w_cur, double lambda) {
    EdgeOptD r;
    r.warn = 0;
    r.passes = 1;
    // kink test at w = 0 (inc/model.hpp:204-209)
    const Pass64 p0 = ising_pass64<TP, true>(T, Xb, Mw, M, a, b, -w_cur);
    const double g0 = p0.Lp;
    if (fabs(g0) <= lambda) {
        double gain = p0.Flik + lambda * fabs(w_cur);  // F(0) - F(w_cur)
        if (w_cur == 0.0) gain = 0.0;
        r.w = 0.0;
        r.gain = gain < 0.0 ? 0.0 : gain;
        return r;
    }
    const double dir = g0 > 0.0 ? 1.0 : -1.0;
    // phi(u) = dir L'(dir u) - lambda, decreasing in u >= 0; phi(0) > 0
    double lo = 0.0, hi = INFINITY, u = 0.0;
    double phi = fabs(g0) - lambda, dphi = p0.Lpp;
    double Fpen = p0.Flik;  // F_lik(0) - F_lik(w_cur) - lambda*0
    double best_u = 0.0, best_F = Fpen, best_phi = phi, best_dphi = dphi;
    for (int it = 0; it < 80; ++it) {
        if (phi > 0.0) lo = u; else hi = u;
        double un = u - phi / dphi;
        if (!(un > lo && un < hi) || !isfinite(un)) un = isinf(hi) ? fmax(2.0 * u, 1.0) : 0.5 * (lo + hi);
        if (un > 0x1.0p64) {  // bracket failure (inc/line_search.hpp:64-84 cap)
            r.warn = 1;
            break;
        }
        const bool done = fabs(un - u) <= 1e-13 * fmax(1.0, un);
        u = un;
        const Pass64 p = ising_pass64<TP, true>(T, Xb, Mw, M, a, b, dir * u - w_cur);
        ++r.passes;
        phi = dir * p.Lp - lambda;
        dphi = p.Lpp;
        const double F = p.Flik - lambda * u;
        if (F >= best_F || done) {
            // plateau guard: the slice saturates numerically for separable columns
            if (!(F > best_F) && isinf(hi) && u > 64.0) {
                break;
            }
            best_u = u;
            best_F = F;
            best_phi = phi;
            best_dphi = dphi;
        }
        if (done) break;
    }
    // second-order correction to the last Newton iterate
    double gain = best_F + lambda * fabs(w_cur);
    double wstar = dir * best_u;
    if (best_dphi < 0.0 && isfinite(best_phi)) {
        const double du = -best_phi / best_dphi;
        if (fabs(du) <= 1e-6 * fmax(1.0, best_u)) {
            gain += 0.5 * best_phi * du;
            wstar = dir * (best_u + du);
        }
    }
    if (gain < 0.0) {  // inc/model.hpp:215
        r.w = w_cur;
        r.gain = 0.0;
    } else {
        r.w = wstar;
        r.gain = gain;
    }
    return r;
}

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
template <class UP>
__device__ __forceinline__ GaussCoef gauss_coef(const UP& Uf, const double* __restrict__ X, int Mp, int M,
                                                int a, int b, double ta2, double tb2, double xxa,
                                                double xxb) {
    const int lane = threadIdx.x & 31;
    double P = 0.0;
    for (int m = lane; m < M; m += 32) {
        const double xa = X[(size_t)a * Mp + m], xb = X[(size_t)b * Mp + m];
        P += Uf(a, m) * xb + Uf(b, m) * xa;
    }
    GaussCoef c;
    c.P = warp_sum(P);
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
