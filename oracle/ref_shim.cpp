// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// Compiles the UNMODIFIED reference headers (netrec, /root/reference/proj/include)
// into oracle/_ref/libnetrec_ref.so behind a flat extern "C" surface that mirrors
// include/netrec_b200.h, so tests can run the reference and the device library on
// identical inputs, and bench.py's reference arm / cpu_baseline can time the
// reference's own CPU path.  Only tests/, __graft_entry__.smoke() and bench.py's
// reference/cpu_baseline legs may load this library.
//
// Every entry point forwards to the reference symbol cited beside it; no
// algorithm is restated here.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <numeric>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "netrec/find_best.hpp"
#include "netrec/knn.hpp"
#include "netrec/model.hpp"
#include "netrec/reconstruct.hpp"

using namespace netrec;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

#define GUARD(...)                                                    \
    try {                                                             \
        __VA_ARGS__;                                                       \
        return 0;                                                     \
    } catch (const std::invalid_argument& e) {                        \
        return fail(e, 22);                                           \
    } catch (const std::out_of_range& e) {                            \
        return fail(e, 34);                                           \
    } catch (const std::overflow_error& e) {                          \
        return fail(e, 75);                                           \
    } catch (const std::exception& e) {                               \
        return fail(e, 5);                                            \
    }

struct Handle {
    ModelKind kind;
    double lambda;
    SampleMatrix X;
    SparseWeights state;
    std::unique_ptr<PseudoLikelihood> model;
    DistanceCache cache;
    // TableMetric-style distance (test_findbest.cpp:20-37): d[min*n+max]
    std::vector<double> table;
    std::size_t table_n = 0;
    std::uint64_t table_probes = 0;

    Handle(int n, int m, ModelKind k, double lam)
        : kind(k), lambda(lam), X(n, m), state(n, m) {}
};

struct TableDist {
    Handle* h;
    double operator()(NodeId i, NodeId j) const {
        const std::size_t a = static_cast<std::size_t>(std::min(i, j));
        const std::size_t b = static_cast<std::size_t>(std::max(i, j));
        return h->table[a * h->table_n + b];
    }
};

// mode 0 = exact, 1 = gradient (inc/model.hpp:20-21); mode 2 = table metric
template <class Fn>
void with_dist(Handle* h, int mode, Fn&& fn) {
    if (mode == 2) {
        if (h->table.empty()) throw std::invalid_argument("no distance table set");
        fn(TableDist{h});
        return;
    }
    const ModelDistance d(*h->model, h->cache,
                          mode == 0 ? DistanceMode::exact : DistanceMode::gradient);
    fn(d);
}

struct RefPair {  // == nrg_pair / CandidateEdge layout
    std::int32_t i, j;
    double dist;
};
static_assert(sizeof(RefPair) == 16);

struct RefTraceLevel {  // == nrg_trace_level
    std::int32_t level;
    std::int32_t k;
    std::int32_t exhaustive;
    std::int32_t knn_sweeps;
    std::uint64_t nodes;
    std::uint64_t dedup_size;
};

struct RefIterRecord {  // == nrg_iter_record
    std::int32_t iter;
    std::int32_t pad;
    double delta;
    double seconds;
    std::uint64_t candidates;
    double objective;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// kind: 0 ising, 1 gaussian. X row-major N*M. theta == nullptr -> make_empty_state
// (inc/model.hpp:404-416); PseudoLikelihood validation (inc/model.hpp:113-124).
int ref_create(void** out, int n, int m, int kind, double lambda, const double* X,
               const double* theta) {
    GUARD({
        auto h = std::make_unique<Handle>(n, m, kind == 0 ? ModelKind::ising : ModelKind::gaussian,
                                          lambda);
        for (int i = 0; i < n; ++i)
            for (int t = 0; t < m; ++t) h->X.set(i, t, X[static_cast<std::size_t>(i) * m + t]);
        h->state = make_empty_state(h->kind, h->X);
        if (theta)
            for (int i = 0; i < n; ++i) h->state.set_theta(i, theta[i]);
        h->model = std::make_unique<PseudoLikelihood>(h->kind, lambda, h->X, h->state);
        *out = h.release();
    })
}

void ref_destroy(void* p) { delete static_cast<Handle*>(p); }

// SparseWeights::set_edge (inc/sparse_weights.hpp:54-85), in order
int ref_set_edges(void* p, std::uint64_t n, const std::int32_t* ei, const std::int32_t* ej,
                  const double* w) {
    auto* h = static_cast<Handle*>(p);
    GUARD(for (std::uint64_t t = 0; t < n; ++t) h->state.set_edge(ei[t], ej[t], w[t], h->X));
}

int ref_set_theta(void* p, const double* theta) {
    auto* h = static_cast<Handle*>(p);
    GUARD(for (NodeId i = 0; i < h->state.num_nodes(); ++i) h->state.set_theta(i, theta[i]));
}

// sorted_edges (inc/sparse_weights.hpp:107-117) + theta
int ref_get_state(void* p, double* theta, std::uint64_t cap, std::int32_t* ei, std::int32_t* ej,
                  double* w, std::uint64_t* n_edges) {
    auto* h = static_cast<Handle*>(p);
    GUARD({
        for (NodeId i = 0; i < h->state.num_nodes(); ++i) theta[i] = h->state.theta(i);
        const auto e = h->state.sorted_edges();
        *n_edges = e.size();
        for (std::size_t t = 0; t < e.size() && t < cap; ++t) {
            ei[t] = e[t].i;
            ej[t] = e[t].j;
            w[t] = e[t].dist;
        }
    })
}

int ref_get_sums(void* p, double* out) {
    auto* h = static_cast<Handle*>(p);
    GUARD({
        const int M = h->state.num_samples();
        for (NodeId i = 0; i < h->state.num_nodes(); ++i) {
            const auto r = h->state.sums_row(i);
            std::memcpy(out + static_cast<std::size_t>(i) * M, r.data(), sizeof(double) * M);
        }
    })
}

int ref_log_posterior(void* p, double* out) {  // inc/model.hpp:133-162
    auto* h = static_cast<Handle*>(p);
    GUARD(*out = h->model->log_posterior());
}

void ref_begin_generation(void* p) { static_cast<Handle*>(p)->cache.begin_generation(); }

int ref_set_table(void* p, std::uint64_t n, const double* table) {
    auto* h = static_cast<Handle*>(p);
    GUARD({
        h->table.assign(table, table + n * n);
        h->table_n = n;
    })
}

// distance() through ModelDistance + the handle's cache (inc/model.hpp:377-400)
int ref_distance(void* p, int mode, std::uint64_t n, const std::int32_t* i, const std::int32_t* j,
                 double* dist) {
    auto* h = static_cast<Handle*>(p);
    GUARD(with_dist(h, mode, [&](auto&& d) {
        for (std::uint64_t t = 0; t < n; ++t) dist[t] = d(i[t], j[t]);
    }));
}

// distance() for a pair list under parallel_for (the CPU pair-score baseline,
// BASELINE.md §3 item 1)
int ref_distance_parallel(void* p, int mode, std::uint64_t n, const std::int32_t* i,
                          const std::int32_t* j, double* dist, int threads) {
    auto* h = static_cast<Handle*>(p);
    GUARD(with_dist(h, mode, [&](auto&& d) {
        parallel_for(n, threads, [&](std::size_t b, std::size_t e) {
            for (std::size_t t = b; t < e; ++t) dist[t] = d(i[t], j[t]);
        });
    }));
}

int ref_optimize_edge(void* p, std::uint64_t n, const std::int32_t* i, const std::int32_t* j,
                      double* w, double* gain, std::uint8_t* warn) {  // inc/model.hpp:201-217
    auto* h = static_cast<Handle*>(p);
    GUARD(for (std::uint64_t t = 0; t < n; ++t) {
        const EdgeOpt r = h->model->optimize_edge(i[t], j[t]);
        w[t] = r.w;
        gain[t] = r.gain;
        if (warn) warn[t] = r.warning ? 1 : 0;
    });
}

// optimize_edge over a pair list under parallel_for (make_slice keeps its scratch
// thread_local, inc/model.hpp:301) -- bench.py's config-4 parity block
int ref_optimize_edge_parallel(void* p, std::uint64_t n, const std::int32_t* i, const std::int32_t* j,
                               double* w, double* gain, std::uint8_t* warn, int threads) {
    auto* h = static_cast<Handle*>(p);
    GUARD(parallel_for(n, threads, [&](std::size_t b, std::size_t e) {
        for (std::size_t t = b; t < e; ++t) {
            const EdgeOpt r = h->model->optimize_edge(i[t], j[t]);
            w[t] = r.w;
            gain[t] = r.gain;
            if (warn) warn[t] = r.warning ? 1 : 0;
        }
    }));
}

int ref_edge_gradient(void* p, std::uint64_t n, const std::int32_t* i, const std::int32_t* j,
                      double* g) {  // inc/model.hpp:175-195
    auto* h = static_cast<Handle*>(p);
    GUARD(for (std::uint64_t t = 0; t < n; ++t) g[t] = h->model->edge_gradient(i[t], j[t]));
}

int ref_edge_objective(void* p, std::int32_t i, std::int32_t j, double w, double* out) {
    auto* h = static_cast<Handle*>(p);
    GUARD(*out = h->model->edge_objective(i, j, w));
}

int ref_optimize_theta(void* p, double* out) {  // inc/model.hpp:222-268
    auto* h = static_cast<Handle*>(p);
    GUARD(for (NodeId i = 0; i < h->state.num_nodes(); ++i) out[i] = h->model->optimize_theta(i));
}

// find_knn / find_knn_exhaustive (inc/knn.hpp:150-314). ids/dists: n*k in heap order.
int ref_find_knn(void* p, int mode, int k, const std::int32_t* nodes, std::uint64_t n, double eps,
                 std::uint64_t seed, int max_sweeps, int scan_floor, int width_floor, int threads,
                 int exhaustive, std::int32_t* ids, double* dists, int* k_out, int* sweeps,
                 double* churn, int churn_cap, int* n_churn) {
    auto* h = static_cast<Handle*>(p);
    GUARD(with_dist(h, mode, [&](auto&& d) {
        KnnParams kp;
        kp.eps = eps;
        kp.seed = seed;
        kp.max_sweeps = max_sweeps;
        kp.scan_floor = scan_floor;
        kp.width_floor = width_floor;
        kp.threads = threads;
        const std::span<const NodeId> s(nodes, n);
        const KnnResult r = exhaustive ? find_knn_exhaustive(k, s, d, threads)
                                       : find_knn(k, s, d, kp);
        const int kk = r.graph.k();
        *k_out = kk;
        *sweeps = r.sweeps;
        const auto all = r.graph.all_entries();
        for (std::size_t t = 0; t < all.size(); ++t) {
            ids[t] = all[t].id;
            dists[t] = all[t].dist;
        }
        *n_churn = static_cast<int>(r.sweep_churn.size());
        for (int t = 0; t < *n_churn && t < churn_cap; ++t) churn[t] = r.sweep_churn[t];
    }));
}

// find_best / find_best_exhaustive (inc/find_best.hpp:186-208)
int ref_find_best(void* p, int mode, std::uint64_t m, const std::int32_t* nodes, std::uint64_t n,
                  double knn_eps, std::uint64_t seed, int threads, int exhaustive, RefPair* out,
                  std::uint64_t cap, std::uint64_t* n_out, RefTraceLevel* tr, int tr_cap,
                  int* n_levels, int* short_count) {
    auto* h = static_cast<Handle*>(p);
    GUARD(with_dist(h, mode, [&](auto&& d) {
        FindBestParams fp;
        fp.knn_eps = knn_eps;
        fp.seed = seed;
        fp.threads = threads;
        const std::span<const NodeId> s(nodes, n);
        const BestPairsResult r =
            exhaustive ? find_best_exhaustive(m, s, d, threads) : find_best(m, s, d, fp);
        *n_out = r.pairs.size();
        for (std::size_t t = 0; t < r.pairs.size() && t < cap; ++t)
            out[t] = {r.pairs[t].i, r.pairs[t].j, r.pairs[t].dist};
        *n_levels = static_cast<int>(r.trace.levels.size());
        for (int t = 0; t < *n_levels && t < tr_cap; ++t) {
            const auto& lv = r.trace.levels[static_cast<std::size_t>(t)];
            tr[t] = {lv.level, lv.k, lv.exhaustive ? 1 : 0, lv.knn_sweeps, lv.nodes, lv.dedup_size};
        }
        *short_count = r.short_count ? 1 : 0;
    }));
}

// detail::apply_edge_updates (inc/reconstruct.hpp:70-127)
int ref_apply_updates(void* p, std::uint64_t n, const RefPair* cands, int threads, double* delta) {
    auto* h = static_cast<Handle*>(p);
    GUARD({
        std::vector<CandidateEdge> c(n);
        for (std::uint64_t t = 0; t < n; ++t) c[t] = {cands[t].i, cands[t].j, cands[t].dist};
        *delta = detail::apply_edge_updates(*h->model, c, threads);
    })
}

int ref_theta_pass(void* p, int threads) {  // inc/reconstruct.hpp:129-138
    auto* h = static_cast<Handle*>(p);
    GUARD(detail::theta_pass(*h->model, threads));
}

// reconstruct_gcd (inc/reconstruct.hpp:148-181). cand_out (optional) receives the
// candidate list of every iteration back to back (cand_cap entries in total).
int ref_reconstruct_gcd(void* p, double kappa, double eps, int max_iters, int mode, double knn_eps,
                        std::uint64_t seed, int threads, RefIterRecord* recs, int rec_cap,
                        int* n_iters, int* converged, RefPair* cand_out, std::uint64_t cand_cap,
                        std::uint64_t* n_cand) {
    auto* h = static_cast<Handle*>(p);
    GUARD({
        ReconstructionConfig cfg;
        cfg.kappa = kappa;
        cfg.eps = eps;
        cfg.max_iters = max_iters;
        cfg.mode = mode == 0 ? DistanceMode::exact : DistanceMode::gradient;
        cfg.knn_eps = knn_eps;
        cfg.seed = seed;
        cfg.threads = threads;
        std::uint64_t filled = 0;
        if (cand_out)
            cfg.candidate_hook = [&](int, std::vector<CandidateEdge>& v) {
                for (const auto& e : v)
                    if (filled < cand_cap) cand_out[filled++] = {e.i, e.j, e.dist};
            };
        const ReconstructionResult r = reconstruct_gcd(*h->model, cfg);
        if (n_cand) *n_cand = filled;
        *converged = r.converged ? 1 : 0;
        *n_iters = static_cast<int>(r.trace.iterations.size());
        for (int t = 0; t < *n_iters && t < rec_cap; ++t) {
            const auto& it = r.trace.iterations[static_cast<std::size_t>(t)];
            recs[t] = {it.iter, 0, it.delta, it.seconds, it.candidates, it.objective};
        }
    })
}

// reconstruct_cd (inc/reconstruct.hpp:185-207), the reference itself
int ref_reconstruct_cd(void* p, double eps, int max_iters, int threads, RefIterRecord* recs, int rec_cap,
                       int* n_iters, int* converged) {
    auto* h = static_cast<Handle*>(p);
    GUARD({
        const ReconstructionResult r = reconstruct_cd(*h->model, eps, max_iters, threads);
        *converged = r.converged ? 1 : 0;
        *n_iters = static_cast<int>(r.trace.iterations.size());
        for (int t = 0; t < *n_iters && t < rec_cap; ++t) {
            const auto& it = r.trace.iterations[static_cast<std::size_t>(t)];
            recs[t] = {it.iter, 0, it.delta, it.seconds, it.candidates, it.objective};
        }
    })
}

int ref_counters(void* p, std::uint64_t* misses, std::uint64_t* hits, std::uint64_t* evals,
                 std::uint64_t* warnings) {
    auto* h = static_cast<Handle*>(p);
    GUARD({
        *misses = h->cache.misses();
        *hits = h->cache.hits();
        *evals = h->model->likelihood_evals();
        *warnings = h->model->warning_count();
    })
}

// recall_curve (inc/find_best.hpp:211-231)
int ref_recall_curve(std::uint64_t m, const RefPair* exact, const RefPair* approx, double* out) {
    GUARD({
        BestPairsResult a, b;
        for (std::uint64_t t = 0; t < m; ++t) {
            a.pairs.push_back({exact[t].i, exact[t].j, exact[t].dist});
            b.pairs.push_back({approx[t].i, approx[t].j, approx[t].dist});
        }
        const auto c = recall_curve(a, b);
        std::copy(c.begin(), c.end(), out);
    })
}

// SplitRng (inc/random.hpp:25-65), for pinning the device/oracle RNG ports
std::uint64_t ref_mix64(std::uint64_t a, std::uint64_t b) { return mix64(a, b); }
void ref_rng_stream(std::uint64_t seed, std::uint64_t split, int n, std::uint64_t bound,
                    std::uint64_t* out) {
    SplitRng r = SplitRng(seed);
    if (split) r = r.split(split);
    for (int t = 0; t < n; ++t) out[t] = bound ? r.below(bound) : r();
}

}  // extern "C"
