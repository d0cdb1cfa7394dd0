// api.cu — the extern "C" boundary (include/netrec_b200.h) and the GCD loop body.
//
// Errors: nrg::Error codes map to the reference's exception types
// (22 invalid_argument, 34 out_of_range, 75 overflow_error, 5/100 runtime_error).
#include <chrono>
#include <cmath>
#include <thread>
#include <cstring>
#include <new>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/netrec_b200.h"
#include <memory>

#include "comm.cuh"
#include "context.cuh"

struct nrg_ctx {
    nrg::Context c;
    cudaEvent_t t0 = nullptr, t1 = nullptr, cand_ev = nullptr;
    ~nrg_ctx() {
        if (t0) cudaEventDestroy(t0);
        if (t1) cudaEventDestroy(t1);
        if (cand_ev) cudaEventDestroy(cand_ev);
    }
    // result buffers
    nrg::DevBuf out_i, out_j, out_d, q_i, q_j, q_d, q_e, q_f, q_u8, knn_ids, knn_d;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const nrg::Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_err = "out of host memory";
        return NRG_EIO;
    } catch (const std::exception& e) {
        g_err = e.what();
        return NRG_EIO;
    }
}

template <class F>
int guardx(nrg_ctx* x, F&& f) {
    if (!x) {
        g_err = "null context";
        return NRG_EINVAL;
    }
    return guard([&] {
        NRG_CUDA(cudaSetDevice(x->c.device));
        nrg::StreamScope ss(x->c.stream);
        f();
    });
}

void check_pairs(const nrg_ctx* x, uint64_t n, const int32_t* i, const int32_t* j) {
    for (uint64_t t = 0; t < n; ++t) {
        if (i[t] == j[t]) nrg::fail(22, "pair operations need i != j");
        if (i[t] < 0 || j[t] < 0 || i[t] >= x->c.n || j[t] >= x->c.n) nrg::fail(34, "node id out of range");
    }
}

template <class T>
T* to_dev(nrg_ctx* x, nrg::DevBuf& b, const T* h, uint64_t n) {
    T* d = b.as<T>(std::max<uint64_t>(n, 1));
    if (n) NRG_CUDA(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, x->c.stream));
    return d;
}
template <class T>
void to_host(nrg_ctx* x, T* h, const T* d, uint64_t n) {
    if (h && n) NRG_CUDA(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, x->c.stream));
}
void need_samples(nrg_ctx* x) {
    if (!x->c.have_samples) nrg::fail(22, "no samples uploaded");
}

__global__ void iota_kernel(int32_t* __restrict__ v, uint64_t n) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) v[t] = (int32_t)t;
}

__global__ void pack_pairs_kernel(const int32_t* __restrict__ i, const int32_t* __restrict__ j,
                                  const double* __restrict__ d, uint64_t k, nrg_pair* __restrict__ out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < k) out[t] = {i[t], j[t], d[t]};
}

void gcd_iteration(nrg_ctx* x, const nrg_gcd_cfg* cfg, int iter, nrg_iter_record* rec, nrg_pair* cands, uint64_t cap,
                   uint64_t* n_cands) {
    nrg::Context& c = x->c;
    need_samples(x);
    if (!(cfg->kappa > 0.0)) nrg::fail(22, "reconstruct_gcd: kappa must be > 0");
    const int n = c.n;
    const double mm = std::nearbyint(cfg->kappa * (double)n);  // round-half-even, inc/reconstruct.hpp:154-155
    const uint64_t m = (uint64_t)std::max(1.0, mm);
    const auto t0 = std::chrono::steady_clock::now();
    nrg::begin_generation(c);
    int32_t* dall = x->q_i.as<int32_t>((uint64_t)n);  // every node, 0..n-1
    iota_kernel<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(dall, (uint64_t)n);
    NRG_LAUNCH_CHECK();
    nrg::BestPairsD best;
    nrg::find_best(c, cfg->mode, m, dall, (uint64_t)n, cfg->knn_eps, nrg::mix64(cfg->seed, (uint64_t)iter),
                   cfg->reverse != 0, false, best, x->out_i, x->out_j, x->out_d);
    // the candidates, packed on the device into the caller's record layout, go down through
    // pinned memory while the updates run; the host copy into `cands` waits until then
    const uint64_t kc = (cands && cap) ? std::min(cap, best.count) : 0;
    nrg::DevBuf packed;
    nrg_pair* hp = nullptr;
    if (kc) {
        nrg_pair* dp = packed.as<nrg_pair>(kc);
        pack_pairs_kernel<<<(unsigned)((kc + 255) / 256), 256, 0, c.stream>>>(
            static_cast<int32_t*>(x->out_i.p), static_cast<int32_t*>(x->out_j.p),
            static_cast<double*>(x->out_d.p), kc, dp);
        NRG_LAUNCH_CHECK();
        hp = c.hp_pairs.as<nrg_pair>(kc);
        NRG_CUDA(cudaMemcpyAsync(hp, dp, kc * sizeof(nrg_pair), cudaMemcpyDeviceToHost, c.stream));
        if (!x->cand_ev) NRG_CUDA(cudaEventCreateWithFlags(&x->cand_ev, cudaEventDisableTiming));
        NRG_CUDA(cudaEventRecord(x->cand_ev, c.stream));
    }
    // the host copy into the caller's buffer (first-touch pages: ~1.5 ms at config 4) runs
    // on a helper thread while the updates run on the device
    std::thread copier;
    if (kc) {
        const cudaEvent_t ev = x->cand_ev;
        copier = std::thread([ev, cands, hp, kc] {
            if (cudaEventSynchronize(ev) == cudaSuccess) std::memcpy(cands, hp, kc * sizeof(nrg_pair));
        });
    }
    struct Join {
        std::thread& t;
        ~Join() {
            if (t.joinable()) t.join();
        }
    } join{copier};
    if (n_cands) *n_cands = best.count;
    const double delta = nrg::apply_updates(c, static_cast<int32_t*>(x->out_i.p), static_cast<int32_t*>(x->out_j.p),
                                            best.count, nullptr, static_cast<double*>(x->out_d.p),
                                            /*fb_sorted=*/true);
    nrg::theta_pass(c, nullptr);
    c.sync();  // IterationRecord.seconds covers FindBest + updates + theta pass (inc/reconstruct.hpp:163-173)
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const double obj = nrg::log_posterior(c);
    if (rec) *rec = {iter, 0, delta, secs, best.count, obj};
}
}  // namespace

extern "C" {

const char* nrg_last_error(void) { return g_err.c_str(); }
int nrg_version(void) { return 1; }

int nrg_create(nrg_ctx** out, int32_t n, int32_t m, int32_t kind, double lambda, int32_t device) {
    return guard([&] {
        nrg::StreamScope ss(nullptr);
        auto* x = new nrg_ctx();
        try {
            nrg::ctx_init(x->c, n, m, kind, lambda, device);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}

int nrg_destroy(nrg_ctx* x) {
    return guardx(x, [&] { delete x; });
}

int nrg_upload_samples(nrg_ctx* x, const double* X) {
    return guardx(x, [&] { nrg::upload_samples_f64(x->c, X); });
}
int nrg_upload_spins_i8(nrg_ctx* x, const int8_t* X) {
    return guardx(x, [&] { nrg::upload_spins_i8(x->c, X); });
}
int nrg_upload_spins_packed(nrg_ctx* x, const uint8_t* bits, uint64_t row_bytes) {
    return guardx(x, [&] { nrg::upload_spins_packed(x->c, bits, row_bytes); });
}

int nrg_reset_state(nrg_ctx* x) {
    return guardx(x, [&] { nrg::reset_state_empty(x->c); });
}

int nrg_set_theta(nrg_ctx* x, const double* theta) {
    return guardx(x, [&] {
        need_samples(x);
        if (theta) nrg::set_theta(x->c, theta);
    });
}

int nrg_set_edges(nrg_ctx* x, uint64_t n, const int32_t* ei, const int32_t* ej, const double* w) {
    return guardx(x, [&] {
        need_samples(x);
        for (uint64_t t = 0; t < n; ++t) {
            if (ei[t] < 0 || ej[t] < 0 || ei[t] >= x->c.n || ej[t] >= x->c.n) nrg::fail(34, "node id out of range");
            if (ei[t] == ej[t]) nrg::fail(22, "set_edge: diagonal entries live in theta");
        }
        int32_t* di = to_dev(x, x->q_i, ei, n);
        int32_t* dj = to_dev(x, x->q_j, ej, n);
        double* dw = to_dev(x, x->q_d, w, n);
        if (getenv("NRG_NO_BULK_SET") || !nrg::set_edges_bulk(x->c, di, dj, n, dw))
            nrg::apply_updates(x->c, di, dj, n, dw);
    });
}

int nrg_get_state(nrg_ctx* x, double* theta, uint64_t cap, int32_t* ei, int32_t* ej, double* w, uint64_t* n_edges) {
    return guardx(x, [&] { nrg::get_state(x->c, theta, cap, ei, ej, w, n_edges); });
}

int nrg_get_sums(nrg_ctx* x, double* out) {
    return guardx(x, [&] { nrg::get_sums(x->c, out); });
}

int nrg_begin_generation(nrg_ctx* x) {
    return guardx(x, [&] { nrg::begin_generation(x->c); });
}

int nrg_log_posterior(nrg_ctx* x, double* out) {
    return guardx(x, [&] { *out = nrg::log_posterior(x->c); });
}

int nrg_distance(nrg_ctx* x, int32_t mode, uint64_t n, const int32_t* i, const int32_t* j, double* dist) {
    return guardx(x, [&] {
        if (mode != NRG_TABLE && mode != NRG_LINE) need_samples(x);
        check_pairs(x, n, i, j);
        int32_t* di = to_dev(x, x->q_i, i, n);
        int32_t* dj = to_dev(x, x->q_j, j, n);
        double* dd = x->q_d.as<double>(std::max<uint64_t>(n, 1));
        nrg::distance_batch(x->c, mode, di, dj, n, dd);
        to_host(x, dist, dd, n);
        x->c.sync();
    });
}

int nrg_optimize_edge(nrg_ctx* x, uint64_t n, const int32_t* i, const int32_t* j, double* w, double* gain,
                      uint8_t* warn) {
    return guardx(x, [&] {
        need_samples(x);
        check_pairs(x, n, i, j);
        int32_t* di = to_dev(x, x->q_i, i, n);
        int32_t* dj = to_dev(x, x->q_j, j, n);
        double* dw = x->q_d.as<double>(std::max<uint64_t>(n, 1));
        double* dg = x->q_e.as<double>(std::max<uint64_t>(n, 1));
        uint8_t* du = x->q_u8.as<uint8_t>(std::max<uint64_t>(n, 1));
        nrg::optimize_edge_live(x->c, di, dj, n, dw, dg, du);
        to_host(x, w, dw, n);
        to_host(x, gain, dg, n);
        to_host(x, warn, du, n);
        x->c.sync();
    });
}

int nrg_edge_gradient(nrg_ctx* x, uint64_t n, const int32_t* i, const int32_t* j, double* g) {
    return guardx(x, [&] {
        need_samples(x);
        check_pairs(x, n, i, j);
        int32_t* di = to_dev(x, x->q_i, i, n);
        int32_t* dj = to_dev(x, x->q_j, j, n);
        double* dg = x->q_d.as<double>(std::max<uint64_t>(n, 1));
        nrg::edge_gradient_live(x->c, di, dj, n, dg);
        to_host(x, g, dg, n);
        x->c.sync();
    });
}

int nrg_optimize_theta(nrg_ctx* x, double* out) {
    return guardx(x, [&] {
        need_samples(x);
        double* d = x->q_d.as<double>(x->c.n);
        nrg::theta_pass(x->c, d);
        to_host(x, out, d, (uint64_t)x->c.n);
        x->c.sync();
    });
}

int nrg_set_table(nrg_ctx* x, uint64_t n, const double* table) {
    return guardx(x, [&] { nrg::set_table(x->c, n, table); });
}
int nrg_set_line(nrg_ctx* x, uint64_t n, const double* pos) {
    return guardx(x, [&] { nrg::set_line(x->c, n, pos); });
}

int nrg_find_knn(nrg_ctx* x, int32_t mode, int32_t k, const int32_t* nodes, uint64_t n, const nrg_knn_params* p,
                 int32_t exhaustive, int32_t* ids, double* dists, int32_t* k_out, int32_t* sweeps, double* churn,
                 int32_t churn_cap, int32_t* n_churn) {
    return guardx(x, [&] {
        if (mode != NRG_TABLE && mode != NRG_LINE) need_samples(x);
        nrg::KnnParamsD kp;
        if (p) {
            kp.eps = p->eps;
            kp.seed = p->seed;
            kp.max_sweeps = p->max_sweeps;
            kp.scan_floor = p->scan_floor;
            kp.width_floor = p->width_floor;
            kp.reverse = p->reverse != 0;
        }
        int32_t* dn = to_dev(x, x->q_j, nodes, n);
        nrg::KnnResultD r;
        nrg::find_knn(x->c, mode, k, dn, n, kp, exhaustive != 0, r, x->knn_ids, x->knn_d);
        *k_out = r.k;
        if (sweeps) *sweeps = r.sweeps;
        to_host(x, ids, r.ids, n * (uint64_t)r.k);
        to_host(x, dists, r.dists, n * (uint64_t)r.k);
        x->c.sync();
        if (n_churn) *n_churn = (int32_t)r.churn.size();
        for (int t = 0; t < (int)r.churn.size() && t < churn_cap; ++t) churn[t] = r.churn[t];
    });
}

int nrg_find_best(nrg_ctx* x, int32_t mode, uint64_t m, const int32_t* nodes, uint64_t n, const nrg_fb_params* p,
                  int32_t exhaustive, nrg_pair* out, uint64_t cap, uint64_t* n_out, nrg_trace_level* trace,
                  int32_t trace_cap, int32_t* n_levels, int32_t* short_count) {
    return guardx(x, [&] {
        if (mode != NRG_TABLE && mode != NRG_LINE) need_samples(x);
        int32_t* dn = to_dev(x, x->q_j, nodes, n);
        nrg::BestPairsD best;
        nrg::find_best(x->c, mode, m, dn, n, p ? p->knn_eps : 1e-3, p ? p->seed : 0, p ? p->reverse != 0 : false,
                       exhaustive != 0, best, x->out_i, x->out_j, x->out_d);
        const uint64_t k = std::min(cap, best.count);
        std::vector<int32_t> hi(k), hj(k);
        std::vector<double> hd(k);
        to_host(x, hi.data(), static_cast<int32_t*>(x->out_i.p), k);
        to_host(x, hj.data(), static_cast<int32_t*>(x->out_j.p), k);
        to_host(x, hd.data(), static_cast<double*>(x->out_d.p), k);
        x->c.sync();
        for (uint64_t t = 0; t < k; ++t) out[t] = {hi[t], hj[t], hd[t]};
        *n_out = best.count;
        if (n_levels) *n_levels = (int32_t)best.trace.size();
        for (int t = 0; t < (int)best.trace.size() && t < trace_cap; ++t) {
            const auto& l = best.trace[t];
            trace[t] = {l.level, l.k, l.exhaustive, l.knn_sweeps, l.nodes, l.dedup_size};
        }
        if (short_count) *short_count = best.short_count ? 1 : 0;
    });
}

int nrg_apply_updates(nrg_ctx* x, const nrg_pair* cands, uint64_t n, double* delta) {
    return guardx(x, [&] {
        need_samples(x);
        std::vector<int32_t> hi(n), hj(n);
        std::vector<double> hd(n);
        for (uint64_t t = 0; t < n; ++t) {
            hi[t] = cands[t].i;
            hj[t] = cands[t].j;
            hd[t] = cands[t].dist;
        }
        check_pairs(x, n, hi.data(), hj.data());
        int32_t* di = to_dev(x, x->q_i, hi.data(), n);
        int32_t* dj = to_dev(x, x->q_j, hj.data(), n);
        double* dd = to_dev(x, x->q_d, hd.data(), n);
        const double d = nrg::apply_updates(x->c, di, dj, n, nullptr, dd);
        if (delta) *delta = d;
    });
}

int nrg_theta_pass(nrg_ctx* x) {
    return guardx(x, [&] {
        need_samples(x);
        nrg::theta_pass(x->c, nullptr);
    });
}

int nrg_gcd_iteration(nrg_ctx* x, const nrg_gcd_cfg* cfg, int32_t iter, nrg_iter_record* rec, nrg_pair* cands,
                      uint64_t cap, uint64_t* n_cands) {
    return guardx(x, [&] { gcd_iteration(x, cfg, iter, rec, cands, cap, n_cands); });
}

int nrg_reconstruct_gcd(nrg_ctx* x, const nrg_gcd_cfg* cfg, nrg_iter_record* recs, int32_t rec_cap, int32_t* n_iters,
                        int32_t* converged) {
    return guardx(x, [&] {
        need_samples(x);
        if (!(cfg->kappa > 0.0)) nrg::fail(22, "reconstruct_gcd: kappa must be > 0");
        const double eps = cfg->eps > 0.0 ? cfg->eps : 1e-6 * x->c.n;
        *converged = 0;
        *n_iters = 0;
        for (int iter = 1; iter <= cfg->max_iters; ++iter) {
            nrg_iter_record r;
            gcd_iteration(x, cfg, iter, &r, nullptr, 0, nullptr);
            if (*n_iters < rec_cap) recs[*n_iters] = r;
            ++*n_iters;
            if (r.delta < eps) {
                *converged = 1;
                break;
            }
        }
    });
}

int nrg_reconstruct_cd(nrg_ctx* x, double eps, int32_t max_iters, int32_t threads, nrg_iter_record* recs,
                       int32_t rec_cap, int32_t* n_iters, int32_t* converged) {
    (void)threads;
    return guardx(x, [&] {
        need_samples(x);
        nrg::Context& c = x->c;
        const uint64_t n = (uint64_t)c.n;
        const uint64_t np = n * (n - 1) / 2;
        if (np >= (1ull << 31)) nrg::fail(22, "reconstruct_cd: too many pairs (n > 65535)");
        const double eps_eff = eps > 0.0 ? eps : 1e-6 * (double)n;
        nrg::DevBuf bi, bj, bd;
        int32_t* ci = bi.as<int32_t>(np);
        int32_t* cj = bj.as<int32_t>(np);
        double* tie = bd.as<double>(np);
        nrg::all_pairs_list(c, ci, cj, tie);
        *converged = 0;
        *n_iters = 0;
        for (int iter = 1; iter <= max_iters; ++iter) {
            const auto t0 = std::chrono::steady_clock::now();
            // every pair of the row-major list ties: apply_updates resolves the list in
            // parallel rounds once few couplings still move, in dependency order otherwise
            const double delta = nrg::apply_updates(c, ci, cj, np, nullptr, tie);
            nrg::theta_pass(c, nullptr);
            const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            const double obj = nrg::log_posterior(c);
            if (*n_iters < rec_cap) recs[*n_iters] = {iter, 0, delta, secs, np, obj};
            ++*n_iters;
            if (delta < eps_eff) {
                *converged = 1;
                break;
            }
        }
    });
}

int nrg_counters(nrg_ctx* x, uint64_t* misses, uint64_t* hits, uint64_t* evals, uint64_t* warnings) {
    return guardx(x, [&] {
        uint64_t h[nrg::C_N];
        x->c.join_side();
        NRG_CUDA(cudaMemcpyAsync(h, x->c.counters.p, sizeof(h), cudaMemcpyDeviceToHost, x->c.stream));
        x->c.sync();
        if (misses) *misses = h[nrg::C_MISSES];
        if (hits) *hits = h[nrg::C_HITS];
        if (evals) *evals = h[nrg::C_EVALS];
        if (warnings) *warnings = h[nrg::C_WARN];
    });
}

int nrg_reset_counters(nrg_ctx* x) {
    return guardx(x, [&] {
        x->c.flush_timing();
        NRG_CUDA(cudaMemsetAsync(x->c.counters.p, 0, nrg::C_N * 8, x->c.stream));
        for (double& v : x->c.phase_ms) v = 0.0;
        x->c.k1_ms = x->c.k1_launches = x->c.k1_pairs = x->c.k2_ms = x->c.k2_launches = x->c.k2_pairs = 0;
        x->c.tail_rounds = 0;
        x->c.tc_launches = x->c.tc_pairs = x->c.cache_flushes = 0;
        x->c.launches0 = nrg::g_launches.load();
        x->c.sync();
    });
}

int nrg_phase_times(nrg_ctx* x, double* ms, int32_t cap) {
    return guardx(x, [&] {
        x->c.flush_timing();
        for (int t = 0; t < nrg::P_N && t < cap; ++t) ms[t] = x->c.phase_ms[t];
    });
}

int nrg_timer(nrg_ctx* x, int32_t op, double* ms) {
    return guardx(x, [&] {
        if (!x->t0) {
            NRG_CUDA(cudaEventCreate(&x->t0));
            NRG_CUDA(cudaEventCreate(&x->t1));
        }
        if (op == 0) {
            NRG_CUDA(cudaEventRecord(x->t0, x->c.stream));
        } else {
            NRG_CUDA(cudaEventRecord(x->t1, x->c.stream));
            NRG_CUDA(cudaEventSynchronize(x->t1));
            float f = 0.f;
            NRG_CUDA(cudaEventElapsedTime(&f, x->t0, x->t1));
            if (ms) *ms = f;
        }
    });
}

int nrg_kernel_stats(nrg_ctx* x, double* out, int32_t cap) {
    return guardx(x, [&] {
        x->c.flush_timing();
        const nrg::Context& c = x->c;
        const double v[11] = {c.k1_ms, c.k1_launches, c.k1_pairs, c.k2_ms, c.k2_launches, c.k2_pairs,
                              (double)(nrg::g_launches.load() - c.launches0), c.tail_rounds, c.tc_launches,
                              c.tc_pairs, c.cache_flushes};
        for (int t = 0; t < 11 && t < cap; ++t) out[t] = v[t];
    });
}

int nrg_sample_scored_pairs(nrg_ctx* x, uint64_t cap, uint64_t seed, int32_t* i, int32_t* j, uint64_t* n_out) {
    return guardx(x, [&] {
        int32_t* di = x->q_i.as<int32_t>(std::max<uint64_t>(cap, 1));
        int32_t* dj = x->q_j.as<int32_t>(std::max<uint64_t>(cap, 1));
        const uint64_t k = nrg::sample_scored_pairs(x->c, cap, seed, di, dj);
        to_host(x, i, di, k);
        to_host(x, j, dj, k);
        x->c.sync();
        *n_out = k;
    });
}

int nrg_recall_curve(uint64_t m, const nrg_pair* exact, const nrg_pair* approx, double* out) {
    // recall_curve (inc/find_best.hpp:211-231), host-side bookkeeping
    return guard([&] {
        std::unordered_map<uint64_t, char> se, sa;
        se.reserve(m * 2);
        sa.reserve(m * 2);
        uint64_t common = 0;
        for (uint64_t r = 0; r < m; ++r) {
            const uint64_t ke = nrg::pair_key(exact[r].i, exact[r].j);
            const uint64_t ka = nrg::pair_key(approx[r].i, approx[r].j);
            if (sa.count(ke)) ++common;
            se.emplace(ke, 1);
            if (se.count(ka)) ++common;
            sa.emplace(ka, 1);
            out[r] = (double)common / (double)(r + 1);
        }
    });
}

int nrg_generate_gaussian_graph(nrg_ctx* x, uint64_t n_edges, const int32_t* ei, const int32_t* ej, const double* kij,
                                const double* kdiag, int32_t burn_in, int32_t thin, uint64_t seed, double* X_out) {
    return guardx(x, [&] {
        nrg::generate_gaussian_graph(x->c, n_edges, ei, ej, kij, kdiag, burn_in, thin, seed);
        if (X_out) {
            nrg::Context& c = x->c;
            NRG_CUDA(cudaMemcpy2DAsync(X_out, (size_t)c.M * 8, c.Xd.p, (size_t)c.Mp * 8, (size_t)c.M * 8, c.n,
                                       cudaMemcpyDeviceToHost, c.stream));
            c.sync();
        }
    });
}

namespace {
// the bit-packed samples as int8 on the host
void unpack_spins(nrg_ctx* x, int8_t* X_out) {
    if (!X_out) return;
    nrg::Context& c = x->c;
    std::vector<uint32_t> bits((size_t)c.n * c.Mw);
    NRG_CUDA(cudaMemcpyAsync(bits.data(), c.Xb.p, bits.size() * 4, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    for (int i = 0; i < c.n; ++i)
        for (int m = 0; m < c.M; ++m)
            X_out[(size_t)i * c.M + m] = ((bits[(size_t)i * c.Mw + (m >> 5)] >> (m & 31)) & 1u) ? 1 : -1;
}
}  // namespace

int nrg_generate_ising(nrg_ctx* x, double mean_deg, double w_sigma, double th_sigma, int32_t burn_in, int32_t thin,
                       uint64_t seed, int8_t* X_out) {
    return guardx(x, [&] {
        nrg::generate_ising(x->c, mean_deg, w_sigma, th_sigma, burn_in, thin, seed);
        unpack_spins(x, X_out);
    });
}

int nrg_generated_truth(nrg_ctx* x, uint64_t cap, int32_t* ei, int32_t* ej, double* w, double* node_out,
                        uint64_t* n_edges) {
    return guardx(x, [&] {
        const nrg::Context& c = x->c;
        if (c.truth_node.empty()) nrg::fail(NRG_EINVAL, "no generated data in this context");
        const uint64_t ne = c.truth_i.size();
        if (n_edges) *n_edges = ne;
        for (uint64_t e = 0; e < std::min(cap, ne); ++e) {
            ei[e] = c.truth_i[e];
            ej[e] = c.truth_j[e];
            w[e] = c.truth_w[e];
        }
        if (node_out) std::copy(c.truth_node.begin(), c.truth_node.end(), node_out);
    });
}

int nrg_generate_ising_powerlaw(nrg_ctx* x, double gamma, int32_t dmin, double w_sigma, double th_sigma,
                                int32_t burn_in, int32_t thin, uint64_t seed, int8_t* X_out) {
    return guardx(x, [&] {
        nrg::generate_ising_powerlaw(x->c, gamma, dmin, w_sigma, th_sigma, burn_in, thin, seed);
        unpack_spins(x, X_out);
    });
}

int nrg_generate_ising_graph(nrg_ctx* x, uint64_t n_edges, const int32_t* ei, const int32_t* ej, const double* w,
                             const double* theta, int32_t burn_in, int32_t thin, uint64_t seed, int8_t* X_out) {
    return guardx(x, [&] {
        nrg::generate_ising_graph(x->c, n_edges, ei, ej, w, theta, burn_in, thin, seed);
        unpack_spins(x, X_out);
    });
}

int nrg_generate_gaussian(nrg_ctx* x, int32_t degree, double amp, int32_t burn_in, int32_t thin, uint64_t seed,
                          double* X_out) {
    return guardx(x, [&] {
        nrg::generate_gaussian(x->c, degree, amp, burn_in, thin, seed);
        if (X_out) {
            nrg::Context& c = x->c;
            NRG_CUDA(cudaMemcpy2DAsync(X_out, (size_t)c.M * 8, c.Xd.p, (size_t)c.Mp * 8, (size_t)c.M * 8, c.n,
                                       cudaMemcpyDeviceToHost, c.stream));
            c.sync();
        }
    });
}

int nrg_write_samples_file(const char* path, int32_t n, int32_t m, int32_t kind, const double* X) {
    return guard([&] {
        if (n < 1 || m < 0) nrg::fail(22, "bad shape");
        nrg::write_samples_file(path, (uint64_t)n, (uint64_t)m, kind, X);
    });
}
int nrg_read_samples_info(const char* path, int32_t* n, int32_t* m, int32_t* kind) {
    return guard([&] {
        uint64_t nn = 0, mm = 0;
        int k = 0;
        nrg::read_samples_info(path, &nn, &mm, &k);
        *n = (int32_t)nn;
        *m = (int32_t)mm;
        *kind = k;
    });
}
int nrg_read_samples_file(const char* path, double* X) {
    return guard([&] { nrg::read_samples_file(path, X); });
}
int nrg_load_samples_file(nrg_ctx* x, const char* path) {
    return guardx(x, [&] { nrg::load_samples_file(x->c, path); });
}
int nrg_save_samples_file(nrg_ctx* x, const char* path) {
    return guardx(x, [&] { nrg::save_samples_file(x->c, path); });
}
int nrg_write_state_file(const char* path, int32_t n, const double* theta, uint64_t n_edges, const int32_t* ei,
                         const int32_t* ej, const double* w) {
    return guard([&] {
        if (n < 1) nrg::fail(22, "bad shape");
        nrg::write_state_file(path, (uint64_t)n, theta, n_edges, ei, ej, w);
    });
}
int nrg_read_state_info(const char* path, int32_t* n, uint64_t* n_edges) {
    return guard([&] {
        uint64_t nn = 0;
        nrg::read_state_info(path, &nn, n_edges);
        *n = (int32_t)nn;
    });
}
int nrg_read_state_file(const char* path, double* theta, int32_t* ei, int32_t* ej, double* w) {
    return guard([&] { nrg::read_state_file(path, theta, ei, ej, w); });
}
int nrg_load_state_file(nrg_ctx* x, const char* path) {
    return guardx(x, [&] {
        need_samples(x);
        uint64_t n = 0, ne = 0;
        nrg::read_state_info(path, &n, &ne);
        if (n != (uint64_t)x->c.n) nrg::fail(22, "state file size does not match the context");
        std::vector<double> th(n), w(ne);
        std::vector<int32_t> ei(ne), ej(ne);
        nrg::read_state_file(path, th.data(), ei.data(), ej.data(), w.data());
        check_pairs(x, ne, ei.data(), ej.data());
        // everything validated before the current state is touched
        for (uint64_t i = 0; i < n; ++i)
            if (!std::isfinite(th[i]) || (x->c.kind == nrg::GAUSSIAN && !(th[i] > 0.0)))
                nrg::fail(22, x->c.kind == nrg::GAUSSIAN ? "gaussian model requires theta > 0" : "non-finite theta");
        for (uint64_t e = 0; e < ne; ++e)
            if (!std::isfinite(w[e])) nrg::fail(22, "non-finite coupling in state file");
        nrg::reset_state_empty(x->c);
        nrg::set_theta(x->c, th.data());
        if (ne) {
            int32_t* di = to_dev(x, x->q_i, ei.data(), ne);
            int32_t* dj = to_dev(x, x->q_j, ej.data(), ne);
            double* dw = to_dev(x, x->q_d, w.data(), ne);
            nrg::apply_updates(x->c, di, dj, ne, dw);
        }
    });
}
int nrg_save_state_file(nrg_ctx* x, const char* path) {
    return guardx(x, [&] {
        nrg::Context& c = x->c;
        std::vector<double> th(c.n);
        uint64_t ne = 0;
        nrg::get_state(c, th.data(), 0, nullptr, nullptr, nullptr, &ne);
        std::vector<int32_t> ei(ne + 1), ej(ne + 1);
        std::vector<double> w(ne + 1);
        nrg::get_state(c, th.data(), ne, ei.data(), ej.data(), w.data(), &ne);
        nrg::write_state_file(path, (uint64_t)c.n, th.data(), ne, ei.data(), ej.data(), w.data());
    });
}

int nrg_comm_unique_id(uint8_t id[128]) {
    return guard([&] { nrg::nccl_unique_id(id); });
}

int nrg_comm_init(nrg_ctx* x, const uint8_t id[128], int32_t rank, int32_t world) {
    return guardx(x, [&] {
        if (world < 1 || rank < 0 || rank >= world) nrg::fail(NRG_EINVAL, "bad rank/world");
        delete static_cast<nrg::Comm*>(x->c.comm);
        x->c.comm = nullptr;
        x->c.rank = 0;
        x->c.world = 1;
        if (world == 1) return;
        x->c.comm = nrg::make_nccl_comm(id, rank, world, x->c.device);
        x->c.rank = rank;
        x->c.world = world;
    });
}

int nrg_loopback_create(int32_t world, void** group) {
    return guard([&] {
        if (world < 1) nrg::fail(NRG_EINVAL, "bad world");
        *group = nrg::loopback_group_create(world);
    });
}

int nrg_loopback_destroy(void* group) {
    return guard([&] { nrg::loopback_group_destroy(static_cast<nrg::LoopbackGroup*>(group)); });
}

int nrg_comm_init_loopback(nrg_ctx* x, void* group, int32_t rank) {
    return guardx(x, [&] {
        auto* g = static_cast<nrg::LoopbackGroup*>(group);
        delete static_cast<nrg::Comm*>(x->c.comm);
        nrg::Comm* cm = nrg::make_loopback_comm(g, rank);
        x->c.comm = cm;
        x->c.rank = rank;
        x->c.world = cm->world;
    });
}

int nrg_comm_init_host(nrg_ctx* x, const nrg_host_transport* t, int32_t rank, int32_t world) {
    return guardx(x, [&] {
        if (!t) nrg::fail(NRG_EINVAL, "null transport");
        if (world < 1 || rank < 0 || rank >= world) nrg::fail(NRG_EINVAL, "bad rank/world");
        delete static_cast<nrg::Comm*>(x->c.comm);
        x->c.comm = nullptr;
        x->c.rank = 0;
        x->c.world = 1;
        if (world == 1) return;
        x->c.comm = nrg::make_host_comm(*t, rank, world);
        x->c.rank = rank;
        x->c.world = world;
    });
}

int nrg_comm_selftest(nrg_ctx* x) {
    return guardx(x, [&] {
        if (x->c.comm) {
            nrg::comm_selftest(*static_cast<nrg::Comm*>(x->c.comm), x->c.stream);
            return;
        }
        uint8_t id[128];
        nrg::nccl_unique_id(id);
        std::unique_ptr<nrg::Comm> one(nrg::make_nccl_comm(id, 0, 1, x->c.device));
        nrg::comm_selftest(*one, x->c.stream);
    });
}

int nrg_route_plan(int32_t world, int32_t rank, const uint64_t* counts, uint64_t* send_bytes, uint64_t* send_off,
                   uint64_t* recv_bytes, uint64_t* recv_off, uint64_t* n_recv) {
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world || !counts) nrg::fail(NRG_EINVAL, "bad rank/world");
        std::vector<size_t> sb, so, rb, ro;
        const uint64_t q = nrg::route_plan(world, rank, counts, sb, so, rb, ro);
        for (int r = 0; r < world; ++r) {
            send_bytes[r] = sb[r];
            send_off[r] = so[r];
            recv_bytes[r] = rb[r];
            recv_off[r] = ro[r];
        }
        if (n_recv) *n_recv = q;
    });
}

int nrg_shard_range(uint64_t n, int32_t rank, int32_t world, uint64_t* lo, uint64_t* hi) {
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world) nrg::fail(NRG_EINVAL, "bad rank/world");
        nrg::shard_range(n, rank, world, *lo, *hi);
    });
}

int32_t nrg_key_owner(uint64_t key, int32_t world) { return world > 1 ? nrg::key_owner(key, world) : 0; }

}  // extern "C"
