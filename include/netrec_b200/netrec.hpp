// include/netrec_b200/netrec.hpp — drop-in C++ API of the reference's GCD hot path,
// backed by libnetrec_b200.so (include/netrec_b200.h).
//
// Mirrors the declarations a caller of the reference uses (namespace netrec;
// /root/reference/proj/include/netrec/ = inc/):
//   SampleMatrix (inc/sample_matrix.hpp), SparseWeights (inc/sparse_weights.hpp),
//   PseudoLikelihood / DistanceCache / ModelDistance / distance / make_empty_state
//   (inc/model.hpp), find_knn / find_knn_exhaustive (inc/knn.hpp), find_best /
//   find_best_exhaustive / recall_curve (inc/find_best.hpp), reconstruct_gcd and
//   detail::apply_edge_updates / detail::theta_pass (inc/reconstruct.hpp).
// Same names, argument meanings and exception types.  The search templates dispatch
// on the distance type: ModelDistance and DeviceTableDistance run on the GPU; any
// other callable is rejected at compile time (there is no CPU fallback).
//
// State ownership: the caller owns SampleMatrix and SparseWeights exactly as in the
// reference; PseudoLikelihood mirrors them into one device context, re-uploads the
// state when the host copy changed, and writes device-side updates back into the
// caller's SparseWeights after every mutating call.
#ifndef NETREC_B200_NETREC_HPP
#define NETREC_B200_NETREC_HPP

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <numeric>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <utility>
#include <vector>

#include "../netrec_b200.h"

// This header defines the reference's hot-path types and functions itself; mark the
// reference headers that define them as already included, so reference headers that
// only *use* them (inc/io.hpp, the CLI's text formats, the experiment harness
// inc/bench.hpp with netrec_b200/synth.hpp) compile unchanged against these definitions.
#define NETREC_COMMON_HPP
#define NETREC_RANDOM_HPP
#define NETREC_SAMPLE_MATRIX_HPP
#define NETREC_SPARSE_WEIGHTS_HPP
#define NETREC_LINE_SEARCH_HPP
#define NETREC_MODEL_HPP
#define NETREC_KNN_HPP
#define NETREC_FIND_BEST_HPP
#define NETREC_RECONSTRUCT_HPP

namespace netrec {

using NodeId = std::int32_t;

// ---------------------------------------------------------------- errors
namespace detail {
inline void check(int rc) {
    if (rc == NRG_OK) return;
    const std::string msg = nrg_last_error();
    switch (rc) {
        case NRG_EINVAL: throw std::invalid_argument(msg);
        case NRG_ERANGE: throw std::out_of_range(msg);
        case NRG_EOVERFLOW: throw std::overflow_error(msg);
        default: throw std::runtime_error(msg);
    }
}
}  // namespace detail

// ---------------------------------------------------------------- common (inc/common.hpp)
struct CandidateEdge {
    NodeId i;
    NodeId j;
    double dist;
};
static_assert(sizeof(CandidateEdge) == sizeof(nrg_pair));
inline bool candidate_less(const CandidateEdge& a, const CandidateEdge& b) {
    if (a.dist != b.dist) return a.dist < b.dist;
    if (a.i != b.i) return a.i < b.i;
    return a.j < b.j;
}
inline CandidateEdge make_candidate(NodeId a, NodeId b, double dist) {
    if (a > b) std::swap(a, b);
    return CandidateEdge{a, b, dist};
}
// SplitMix64 finalizer and the two-argument mix (inc/random.hpp:11-24): the FindBest
// seed of iteration `iter` is mix64(cfg.seed, iter) (inc/reconstruct.hpp:168)
inline std::uint64_t mix64(std::uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
inline std::uint64_t mix64(std::uint64_t a, std::uint64_t b) { return mix64(a ^ mix64(b)); }

inline std::uint64_t pair_key(NodeId a, NodeId b) {
    if (a > b) std::swap(a, b);
    return (static_cast<std::uint64_t>(static_cast<std::uint32_t>(a)) << 32) | static_cast<std::uint32_t>(b);
}

// ---------------------------------------------------------------- SampleMatrix
class SampleMatrix {
public:
    SampleMatrix(NodeId n, int m) : n_(n), m_(m) {
        if (n < 1 || m < 0) throw std::invalid_argument("SampleMatrix: bad dimensions");
        values_.assign(static_cast<std::size_t>(n) * static_cast<std::size_t>(m), 0.0);
    }
    NodeId num_nodes() const { return n_; }
    int num_samples() const { return m_; }
    double operator()(NodeId i, int m) const { return values_[static_cast<std::size_t>(i) * m_ + m]; }
    void set(NodeId i, int m, double v) {
        values_[static_cast<std::size_t>(i) * m_ + m] = v;
        ++version_;
    }
    std::span<const double> row(NodeId i) const {
        return {values_.data() + static_cast<std::size_t>(i) * m_, static_cast<std::size_t>(m_)};
    }
    bool spin_valued() const {
        for (double v : values_)
            if (v != 1.0 && v != -1.0) return false;
        return true;
    }
    const double* data() const { return values_.data(); }
    std::uint64_t version() const { return version_; }

private:
    NodeId n_;
    int m_;
    std::vector<double> values_;
    std::uint64_t version_ = 1;
};

// ---------------------------------------------------------------- SparseWeights
class SparseWeights {
public:
    explicit SparseWeights(NodeId n, int samples = 0) : n_(n), samples_(samples) {
        if (n < 1 || samples < 0) throw std::invalid_argument("SparseWeights: bad dimensions");
        rows_.resize(static_cast<std::size_t>(n));
        theta_.assign(static_cast<std::size_t>(n), 0.0);
        sums_.assign(static_cast<std::size_t>(n) * static_cast<std::size_t>(samples), 0.0);
    }
    NodeId num_nodes() const { return n_; }
    int num_samples() const { return samples_; }
    std::size_t edge_count() const { return edges_; }
    double weight(NodeId i, NodeId j) const {
        check_pair(i, j);
        if (i > j) std::swap(i, j);
        const auto& r = rows_[static_cast<std::size_t>(i)];
        auto it = r.find(j);
        return it == r.end() ? 0.0 : it->second;
    }
    bool has_edge(NodeId i, NodeId j) const {
        if (i > j) std::swap(i, j);
        return rows_[static_cast<std::size_t>(i)].count(j) != 0;
    }
    // set_edge (inc/sparse_weights.hpp:54-85), host side; mirrored to the device lazily
    void set_edge(NodeId i, NodeId j, double w, const SampleMatrix& X) {
        check_pair(i, j);
        if (i == j) throw std::invalid_argument("set_edge: diagonal entries live in theta");
        if (X.num_nodes() != n_ || X.num_samples() != samples_)
            throw std::invalid_argument("set_edge: sample matrix shape mismatch");
        if (i > j) std::swap(i, j);
        auto& r = rows_[static_cast<std::size_t>(i)];
        auto it = r.find(j);
        const double old = it == r.end() ? 0.0 : it->second;
        const double delta = w - old;
        if (delta != 0.0) {
            double* si = sums_.data() + static_cast<std::size_t>(i) * samples_;
            double* sj = sums_.data() + static_cast<std::size_t>(j) * samples_;
            const auto xi = X.row(i), xj = X.row(j);
            for (int m = 0; m < samples_; ++m) {
                si[m] += delta * xj[m];
                sj[m] += delta * xi[m];
            }
        }
        if (w == 0.0) {
            if (it != r.end()) {
                r.erase(it);
                --edges_;
            }
        } else if (it == r.end()) {
            r.emplace(j, w);
            ++edges_;
        } else {
            it->second = w;
        }
        ++version_;
    }
    double theta(NodeId i) const { return theta_[static_cast<std::size_t>(i)]; }
    void set_theta(NodeId i, double v) {
        theta_[static_cast<std::size_t>(i)] = v;
        ++version_;
    }
    double sum(NodeId i, int m) const { return sums_[static_cast<std::size_t>(i) * samples_ + m]; }
    std::span<const double> sums_row(NodeId i) const {
        return {sums_.data() + static_cast<std::size_t>(i) * samples_, static_cast<std::size_t>(samples_)};
    }
    template <class Fn>
    void for_each_edge(Fn&& fn) const {
        for (NodeId i = 0; i < n_; ++i)
            for (const auto& [j, w] : rows_[static_cast<std::size_t>(i)]) fn(i, j, w);
    }
    std::vector<CandidateEdge> sorted_edges() const {
        std::vector<CandidateEdge> out;
        out.reserve(edges_);
        for (NodeId i = 0; i < n_; ++i) {
            std::vector<std::pair<NodeId, double>> r(rows_[i].begin(), rows_[i].end());
            std::sort(r.begin(), r.end());
            for (const auto& [j, w] : r) out.push_back({i, j, w});
        }
        return out;
    }
    std::uint64_t version() const { return version_; }

    // device write-back (PseudoLikelihood only): replaces edges, theta and sums
    void assign_from_device(const std::vector<double>& th, const std::vector<std::int32_t>& ei,
                            const std::vector<std::int32_t>& ej, const std::vector<double>& w,
                            std::vector<double>&& sums) {
        for (auto& r : rows_) r.clear();
        edges_ = 0;
        for (std::size_t t = 0; t < ei.size(); ++t) {
            rows_[static_cast<std::size_t>(ei[t])].emplace(ej[t], w[t]);
            ++edges_;
        }
        theta_ = th;
        sums_ = std::move(sums);
        ++version_;
    }

private:
    void check_pair(NodeId i, NodeId j) const {
        if (i < 0 || j < 0 || i >= n_ || j >= n_) throw std::out_of_range("node id out of range");
    }
    NodeId n_;
    int samples_;
    std::vector<std::unordered_map<NodeId, double>> rows_;
    std::vector<double> theta_;
    std::vector<double> sums_;
    std::size_t edges_ = 0;
    std::uint64_t version_ = 1;
};

// ---------------------------------------------------------------- model (inc/model.hpp)
enum class ModelKind { ising, gaussian };
enum class DistanceMode { exact, gradient };

struct EdgeOpt {
    double w;
    double gain;
    bool warning;
};

class PseudoLikelihood;

// DistanceCache (inc/model.hpp:36-97): the cache itself lives on the device with the
// model's state; this handle carries the generation the caller opened.
class DistanceCache {
public:
    explicit DistanceCache(unsigned = 64) {}
    void begin_generation() { ++gen_; }
    std::uint64_t generation() const { return gen_; }
    std::uint64_t hits() const;
    std::uint64_t misses() const;

private:
    friend class PseudoLikelihood;
    std::uint64_t gen_ = 0;
    const PseudoLikelihood* bound_ = nullptr;
};

class PseudoLikelihood {
public:
    static constexpr double kThetaMaxIsing = 20.0;
    static constexpr double kThetaMinGaussian = 1e-8;
    static constexpr double kArgTol = 1e-8;

    PseudoLikelihood(ModelKind kind, double lambda, const SampleMatrix& X, SparseWeights& state, int device = 0)
        : kind_(kind), lambda_(lambda), x_(&X), state_(&state) {
        if (lambda < 0.0) throw std::invalid_argument("lambda must be >= 0");
        if (X.num_nodes() != state.num_nodes() || X.num_samples() != state.num_samples())
            throw std::invalid_argument("model: sample matrix and state shapes differ");
        if (kind == ModelKind::ising && !X.spin_valued())
            throw std::invalid_argument("ising model requires +/-1 data");
        if (kind == ModelKind::gaussian)
            for (NodeId i = 0; i < state.num_nodes(); ++i)
                if (!(state.theta(i) > 0.0)) throw std::invalid_argument("gaussian model requires theta > 0");
        nrg_ctx* c = nullptr;
        detail::check(nrg_create(&c, X.num_nodes(), X.num_samples(), kind == ModelKind::ising ? NRG_ISING : NRG_GAUSSIAN,
                                 lambda, device));
        ctx_.reset(c);
        detail::check(nrg_upload_samples(c, X.data()));
        x_version_ = X.version();
        upload_state();
    }

    ModelKind kind() const { return kind_; }
    double lambda() const { return lambda_; }
    const SampleMatrix& samples() const { return *x_; }
    SparseWeights& state() { return *state_; }
    const SparseWeights& state() const { return *state_; }
    nrg_ctx* context() const {
        sync_to_device();
        return ctx_.get();
    }

    double log_posterior() const {
        double v = 0.0;
        detail::check(nrg_log_posterior(context(), &v));
        return v;
    }
    double edge_gradient(NodeId i, NodeId j) const {
        double g = 0.0;
        detail::check(nrg_edge_gradient(context(), 1, &i, &j, &g));
        return g;
    }
    EdgeOpt optimize_edge(NodeId i, NodeId j) const {
        double w = 0.0, gain = 0.0;
        std::uint8_t warn = 0;
        detail::check(nrg_optimize_edge(context(), 1, &i, &j, &w, &gain, &warn));
        return {w, gain, warn != 0};
    }
    double optimize_theta(NodeId i) const {
        std::vector<double> th(static_cast<std::size_t>(state_->num_nodes()));
        detail::check(nrg_optimize_theta(context(), th.data()));
        return th[static_cast<std::size_t>(i)];
    }
    std::uint64_t likelihood_evals() const { return counters()[2]; }
    std::uint64_t warning_count() const { return counters()[3]; }

    // opens the device generation matching the caller's DistanceCache
    void use_cache(DistanceCache& cache) const {
        if (cache.bound_ != this || cache.gen_ != seen_gen_) {
            detail::check(nrg_begin_generation(context()));
            cache.bound_ = this;
            seen_gen_ = cache.gen_;
        }
    }
    // device-side mutation happened: bring the caller's SparseWeights up to date
    void pull_state() const {
        const NodeId n = state_->num_nodes();
        const int M = state_->num_samples();
        std::vector<double> th(static_cast<std::size_t>(n));
        std::uint64_t ne = 0;
        detail::check(nrg_get_state(ctx_.get(), th.data(), 0, nullptr, nullptr, nullptr, &ne));
        std::vector<std::int32_t> ei(ne), ej(ne);
        std::vector<double> w(ne);
        detail::check(nrg_get_state(ctx_.get(), th.data(), ne, ei.data(), ej.data(), w.data(), &ne));
        if (ne < ei.size()) {  // the count call is an upper bound
            ei.resize(ne);
            ej.resize(ne);
            w.resize(ne);
        }
        std::vector<double> sums(static_cast<std::size_t>(n) * static_cast<std::size_t>(M));
        detail::check(nrg_get_sums(ctx_.get(), sums.data()));
        state_->assign_from_device(th, ei, ej, w, std::move(sums));
        state_version_ = state_->version();
    }
    std::vector<std::uint64_t> counters() const {
        std::vector<std::uint64_t> v(4);
        detail::check(nrg_counters(ctx_.get(), &v[0], &v[1], &v[2], &v[3]));
        return v;
    }

private:
    struct CtxDel {
        void operator()(nrg_ctx* c) const { nrg_destroy(c); }
    };
    void upload_state() const {
        const NodeId n = state_->num_nodes();
        std::vector<double> th(static_cast<std::size_t>(n));
        for (NodeId i = 0; i < n; ++i) th[i] = state_->theta(i);
        detail::check(nrg_reset_state(ctx_.get()));
        detail::check(nrg_set_theta(ctx_.get(), th.data()));
        const auto e = state_->sorted_edges();
        std::vector<std::int32_t> ei(e.size()), ej(e.size());
        std::vector<double> w(e.size());
        for (std::size_t t = 0; t < e.size(); ++t) {
            ei[t] = e[t].i;
            ej[t] = e[t].j;
            w[t] = e[t].dist;
        }
        if (!e.empty()) detail::check(nrg_set_edges(ctx_.get(), e.size(), ei.data(), ej.data(), w.data()));
        state_version_ = state_->version();
    }
    void sync_to_device() const {
        if (x_->version() != x_version_) {
            detail::check(nrg_upload_samples(ctx_.get(), x_->data()));
            x_version_ = x_->version();
            state_version_ = 0;
        }
        if (state_->version() != state_version_) upload_state();
    }

    ModelKind kind_;
    double lambda_;
    const SampleMatrix* x_;
    SparseWeights* state_;
    std::unique_ptr<nrg_ctx, CtxDel> ctx_;
    mutable std::uint64_t x_version_ = 0, state_version_ = 0, seen_gen_ = ~0ull;
};

inline std::uint64_t DistanceCache::hits() const { return bound_ ? bound_->counters()[1] : 0; }
inline std::uint64_t DistanceCache::misses() const { return bound_ ? bound_->counters()[0] : 0; }

inline double distance(const PseudoLikelihood& model, NodeId i, NodeId j, DistanceMode mode, DistanceCache& cache) {
    model.use_cache(cache);
    double d = 0.0;
    detail::check(nrg_distance(model.context(), mode == DistanceMode::exact ? NRG_EXACT : NRG_GRADIENT, 1, &i, &j, &d));
    return d;
}

// ModelDistance (inc/model.hpp:389-400): the device-backed distance of the searches
class ModelDistance {
public:
    ModelDistance(const PseudoLikelihood& model, DistanceCache& cache, DistanceMode mode)
        : model_(&model), cache_(&cache), mode_(mode) {}
    double operator()(NodeId i, NodeId j) const { return distance(*model_, i, j, mode_, *cache_); }
    DistanceCache& cache() const { return *cache_; }
    const PseudoLikelihood& model() const { return *model_; }
    int device_mode() const { return mode_ == DistanceMode::exact ? NRG_EXACT : NRG_GRADIENT; }

private:
    const PseudoLikelihood* model_;
    DistanceCache* cache_;
    DistanceMode mode_;
};

// Device-resident TableMetric (test_findbest.cpp:20-37): d(i,j) = table[min*n + max]
class DeviceTableDistance {
public:
    DeviceTableDistance(std::vector<double> table, std::size_t n, int device = 0) : n_(n), table_(std::move(table)) {
        nrg_ctx* c = nullptr;
        detail::check(nrg_create(&c, static_cast<std::int32_t>(n), 1, NRG_ISING, 0.0, device));
        ctx_.reset(c);
        std::vector<double> ones(n, 1.0);
        detail::check(nrg_upload_samples(c, ones.data()));
        detail::check(nrg_set_table(c, n, table_.data()));
    }
    double operator()(NodeId i, NodeId j) const {
        return table_[static_cast<std::size_t>(std::min(i, j)) * n_ + static_cast<std::size_t>(std::max(i, j))];
    }
    nrg_ctx* context() const { return ctx_.get(); }

private:
    struct CtxDel {
        void operator()(nrg_ctx* c) const { nrg_destroy(c); }
    };
    std::size_t n_;
    std::vector<double> table_;
    std::unique_ptr<nrg_ctx, CtxDel> ctx_;
};

inline SparseWeights make_empty_state(ModelKind kind, const SampleMatrix& X) {
    SparseWeights s(X.num_nodes(), X.num_samples());
    if (kind == ModelKind::gaussian) {
        const int M = X.num_samples();
        for (NodeId i = 0; i < X.num_nodes(); ++i) {
            double a = 0.0;
            for (int m = 0; m < M; ++m) a += X(i, m) * X(i, m);
            const double rms = M > 0 ? std::sqrt(a / M) : 1.0;
            s.set_theta(i, std::max(rms, PseudoLikelihood::kThetaMinGaussian));
        }
    }
    return s;
}

// ---------------------------------------------------------------- kNN (inc/knn.hpp)
struct KnnEntry {
    NodeId id;
    double dist;
};

// KnnGraph view: per-node out-neighbours, sorted by (dist, id) (the reference keeps a
// max-heap; only the set is observable, test_knn.cpp:154-179)
class KnnGraph {
public:
    KnnGraph(std::vector<NodeId> nodes, int k) : nodes_(std::move(nodes)), k_(k), entries_(nodes_.size() * k) {}
    std::size_t size() const { return nodes_.size(); }
    int k() const { return k_; }
    const std::vector<NodeId>& nodes() const { return nodes_; }
    std::span<const KnnEntry> neighbors(std::size_t local) const {
        return {entries_.data() + local * k_, static_cast<std::size_t>(k_)};
    }
    std::span<const KnnEntry> all_entries() const { return {entries_.data(), entries_.size()}; }
    const KnnEntry& worst(std::size_t local) const { return entries_[local * k_ + (k_ - 1)]; }
    bool contains(std::size_t local, NodeId id) const {
        for (const auto& e : neighbors(local))
            if (e.id == id) return true;
        return false;
    }
    std::vector<KnnEntry>& raw() { return entries_; }

private:
    std::vector<NodeId> nodes_;
    int k_;
    std::vector<KnnEntry> entries_;
};

struct KnnParams {
    double eps = 1e-3;
    int threads = 1;
    std::uint64_t seed = 0;
    int max_sweeps = 100;
    int scan_floor = 8;
    int width_floor = 4;
    bool reverse = false;  // extension: reverse-list NNDescent
};

struct KnnResult {
    KnnGraph graph;
    int sweeps = 0;
    std::vector<double> sweep_churn;
    int sweep_count() const { return sweeps; }
};

namespace detail {
template <class Dist>
constexpr bool is_device_distance_v = std::is_same_v<std::remove_cvref_t<Dist>, ModelDistance> ||
                                      std::is_same_v<std::remove_cvref_t<Dist>, DeviceTableDistance>;

template <class Dist>
std::pair<nrg_ctx*, int> device_of(Dist&& d) {
    using D = std::remove_cvref_t<Dist>;
    if constexpr (std::is_same_v<D, ModelDistance>) {
        d.model().use_cache(d.cache());
        return {d.model().context(), d.device_mode()};
    } else {
        return {d.context(), NRG_TABLE};
    }
}

template <class Dist>
KnnResult knn_call(int k, std::span<const NodeId> nodes, Dist&& d, const KnnParams& p, bool exhaustive) {
    static_assert(is_device_distance_v<Dist>,
                  "netrec_b200 runs the search on the GPU: pass a ModelDistance or DeviceTableDistance");
    auto [ctx, mode] = device_of(d);
    nrg_knn_params kp{p.eps, p.seed, p.max_sweeps, p.scan_floor, p.width_floor, p.threads, p.reverse ? 1 : 0, 0};
    const std::size_t n = nodes.size();
    const int kk = std::max(k, 1);
    std::vector<std::int32_t> ids(n * kk);
    std::vector<double> dists(n * kk), churn(static_cast<std::size_t>(std::max(p.max_sweeps, 1)));
    std::int32_t k_out = 0, sweeps = 0, nchurn = 0;
    check(nrg_find_knn(ctx, mode, k, nodes.data(), n, &kp, exhaustive ? 1 : 0, ids.data(), dists.data(), &k_out,
                       &sweeps, churn.data(), static_cast<std::int32_t>(churn.size()), &nchurn));
    KnnResult r{KnnGraph(std::vector<NodeId>(nodes.begin(), nodes.end()), k_out), sweeps, {}};
    for (std::size_t t = 0; t < n * static_cast<std::size_t>(k_out); ++t) r.graph.raw()[t] = {ids[t], dists[t]};
    r.sweep_churn.assign(churn.begin(), churn.begin() + nchurn);
    return r;
}
}  // namespace detail

template <class Dist>
KnnResult find_knn(int k, std::span<const NodeId> nodes, Dist&& d, const KnnParams& p = {}) {
    return detail::knn_call(k, nodes, d, p, false);
}
template <class Dist>
KnnResult find_knn_exhaustive(int k, std::span<const NodeId> nodes, Dist&& d, int threads = 1) {
    KnnParams p;
    p.threads = threads;
    return detail::knn_call(k, nodes, d, p, true);
}

// ---------------------------------------------------------------- FindBest (inc/find_best.hpp)
struct TraceLevel {
    int level;
    std::size_t nodes;
    int k;
    bool exhaustive;
    int knn_sweeps;
    std::size_t dedup_size;
};
struct RecursionTrace {
    std::vector<TraceLevel> levels;
    bool halving_ok() const {
        for (std::size_t t = 0; t + 1 < levels.size(); ++t)
            if (levels[t + 1].nodes * 2 > levels[t].nodes) return false;
        return true;
    }
};
struct BestPairsResult {
    std::vector<CandidateEdge> pairs;
    RecursionTrace trace;
    bool short_count = false;
};
struct FindBestParams {
    double knn_eps = 1e-3;
    int threads = 1;
    std::uint64_t seed = 0;
    bool reverse = false;  // extension: reverse-list NNDescent
};

namespace detail {
template <class Dist>
BestPairsResult fb_call(std::size_t m, std::span<const NodeId> s, Dist&& d, const FindBestParams& p, bool exhaustive) {
    static_assert(is_device_distance_v<Dist>,
                  "netrec_b200 runs the search on the GPU: pass a ModelDistance or DeviceTableDistance");
    auto [ctx, mode] = device_of(d);
    nrg_fb_params fp{p.knn_eps, p.seed, p.threads, p.reverse ? 1 : 0};
    const std::size_t total = s.size() * (s.size() > 0 ? s.size() - 1 : 0) / 2;
    std::vector<nrg_pair> out(std::min<std::size_t>(m, total) + 1);
    std::vector<nrg_trace_level> tr(64);
    std::uint64_t nout = 0;
    std::int32_t nl = 0, sc = 0;
    check(nrg_find_best(ctx, mode, m, s.data(), s.size(), &fp, exhaustive ? 1 : 0, out.data(), out.size(), &nout,
                        tr.data(), 64, &nl, &sc));
    BestPairsResult r;
    r.pairs.resize(nout);
    for (std::uint64_t t = 0; t < nout; ++t) r.pairs[t] = {out[t].i, out[t].j, out[t].dist};
    for (int t = 0; t < nl; ++t)
        r.trace.levels.push_back({tr[t].level, tr[t].nodes, tr[t].k, tr[t].exhaustive != 0, tr[t].knn_sweeps,
                                  tr[t].dedup_size});
    r.short_count = sc != 0;
    return r;
}
}  // namespace detail

template <class Dist>
BestPairsResult find_best(std::size_t m, std::span<const NodeId> s, Dist&& d, const FindBestParams& p = {}) {
    return detail::fb_call(m, s, d, p, false);
}
template <class Dist>
BestPairsResult find_best_exhaustive(std::size_t m, std::span<const NodeId> s, Dist&& d, int threads = 1) {
    FindBestParams p;
    p.threads = threads;
    return detail::fb_call(m, s, d, p, true);
}

inline std::vector<double> recall_curve(const BestPairsResult& exact, const BestPairsResult& approx) {
    if (exact.pairs.size() != approx.pairs.size()) throw std::invalid_argument("recall_curve: result lengths differ");
    std::vector<double> out(exact.pairs.size());
    if (!out.empty())
        detail::check(nrg_recall_curve(out.size(), reinterpret_cast<const nrg_pair*>(exact.pairs.data()),
                                       reinterpret_cast<const nrg_pair*>(approx.pairs.data()), out.data()));
    return out;
}

// ---------------------------------------------------------------- driver (inc/reconstruct.hpp)
struct IterationRecord {
    int iter;
    double delta;
    double seconds;
    std::size_t candidates;
    double objective;
};
struct ConvergenceTrace {
    std::vector<IterationRecord> iterations;
};
struct ReconstructionConfig {
    double kappa = 1.0;
    double eps = -1.0;
    int max_iters = 1000;
    DistanceMode mode = DistanceMode::exact;
    double knn_eps = 1e-3;
    int threads = 1;
    std::uint64_t seed = 0;
    std::function<void(int iter, std::vector<CandidateEdge>&)> candidate_hook;
    bool reverse = false;  // extension: reverse-list NNDescent
};
struct ReconstructionResult {
    bool converged = false;
    ConvergenceTrace trace;
};

namespace detail {
inline double apply_edge_updates(PseudoLikelihood& model, const std::vector<CandidateEdge>& candidates, int = 1) {
    double delta = 0.0;
    check(nrg_apply_updates(model.context(), reinterpret_cast<const nrg_pair*>(candidates.data()), candidates.size(),
                            &delta));
    model.pull_state();
    return delta;
}
inline void theta_pass(PseudoLikelihood& model, int = 1) {
    check(nrg_theta_pass(model.context()));
    model.pull_state();
}
}  // namespace detail

inline ReconstructionResult reconstruct_gcd(PseudoLikelihood& model, const ReconstructionConfig& cfg) {
    if (!(cfg.kappa > 0.0)) throw std::invalid_argument("reconstruct_gcd: kappa must be > 0");
    const NodeId n = model.state().num_nodes();
    const double eps = cfg.eps > 0.0 ? cfg.eps : 1e-6 * n;
    ReconstructionResult res;
    nrg_gcd_cfg g{cfg.kappa, cfg.eps, 1, cfg.mode == DistanceMode::exact ? NRG_EXACT : NRG_GRADIENT, cfg.knn_eps,
                  cfg.seed, cfg.threads, cfg.reverse ? 1 : 0};
    nrg_ctx* ctx = model.context();
    const std::size_t m = static_cast<std::size_t>(std::max(1.0, std::nearbyint(cfg.kappa * static_cast<double>(n))));
    std::vector<CandidateEdge> cands(m + 1);
    for (int iter = 1; iter <= cfg.max_iters; ++iter) {
        nrg_iter_record r{};
        if (!cfg.candidate_hook) {
            detail::check(nrg_gcd_iteration(ctx, &g, iter, &r, nullptr, 0, nullptr));
        } else {
            // the hook may edit the candidates between FindBest and the updates (:170)
            const auto t0 = std::chrono::steady_clock::now();
            detail::check(nrg_begin_generation(ctx));
            std::vector<NodeId> all(static_cast<std::size_t>(n));
            std::iota(all.begin(), all.end(), 0);
            nrg_fb_params fp{cfg.knn_eps, 0, cfg.threads, cfg.reverse ? 1 : 0};
            fp.seed = mix64(cfg.seed, static_cast<std::uint64_t>(iter));
            std::uint64_t nout = 0;
            detail::check(nrg_find_best(ctx, g.mode, m, all.data(), all.size(), &fp, 0,
                                        reinterpret_cast<nrg_pair*>(cands.data()), cands.size(), &nout, nullptr, 0,
                                        nullptr, nullptr));
            std::vector<CandidateEdge> v(cands.begin(), cands.begin() + static_cast<std::ptrdiff_t>(nout));
            cfg.candidate_hook(iter, v);
            double delta = 0.0;
            detail::check(nrg_apply_updates(ctx, reinterpret_cast<const nrg_pair*>(v.data()), v.size(), &delta));
            detail::check(nrg_theta_pass(ctx));
            const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            double obj = 0.0;
            detail::check(nrg_log_posterior(ctx, &obj));
            r = {iter, 0, delta, secs, v.size(), obj};
        }
        res.trace.iterations.push_back({r.iter, r.delta, r.seconds, static_cast<std::size_t>(r.candidates), r.objective});
        if (r.delta < eps) {
            res.converged = true;
            break;
        }
    }
    model.pull_state();
    return res;
}

/// Binary sample / state files: the fast counterparts of the text
/// formats in inc/io.hpp (samples_to_text / weights_to_text and their readers).
inline void write_samples_binary(const std::string& path, const SampleMatrix& X, bool ising) {
    detail::check(nrg_write_samples_file(path.c_str(), X.num_nodes(), X.num_samples(), ising ? 0 : 1, X.data()));
}
inline SampleMatrix read_samples_binary(const std::string& path) {
    int32_t n = 0, m = 0, kind = 0;
    detail::check(nrg_read_samples_info(path.c_str(), &n, &m, &kind));
    std::vector<double> v(static_cast<std::size_t>(n) * static_cast<std::size_t>(m));
    detail::check(nrg_read_samples_file(path.c_str(), v.data()));
    SampleMatrix X(n, m);
    for (NodeId i = 0; i < n; ++i)
        for (int t = 0; t < m; ++t) X.set(i, t, v[static_cast<std::size_t>(i) * m + t]);
    return X;
}
inline void write_weights_binary(const std::string& path, const SparseWeights& W) {
    const NodeId n = W.num_nodes();
    std::vector<double> th(static_cast<std::size_t>(n)), w;
    std::vector<int32_t> ei, ej;
    for (NodeId i = 0; i < n; ++i) th[static_cast<std::size_t>(i)] = W.theta(i);
    W.for_each_edge([&](NodeId i, NodeId j, double v) {
        ei.push_back(i);
        ej.push_back(j);
        w.push_back(v);
    });
    detail::check(nrg_write_state_file(path.c_str(), n, th.data(), ei.size(), ei.data(), ej.data(), w.data()));
}
/// rebuilds the sums against X (set_edge per stored coupling, inc/sparse_weights.hpp:54-85)
inline SparseWeights read_weights_binary(const std::string& path, const SampleMatrix& X) {
    int32_t n = 0;
    uint64_t ne = 0;
    detail::check(nrg_read_state_info(path.c_str(), &n, &ne));
    std::vector<double> th(static_cast<std::size_t>(n)), w(ne + 1);
    std::vector<int32_t> ei(ne + 1), ej(ne + 1);
    detail::check(nrg_read_state_file(path.c_str(), th.data(), ei.data(), ej.data(), w.data()));
    SparseWeights W(n, X.num_samples());
    for (NodeId i = 0; i < n; ++i) W.set_theta(i, th[static_cast<std::size_t>(i)]);
    for (uint64_t e = 0; e < ne; ++e) W.set_edge(ei[e], ej[e], w[e], X);
    return W;
}

/// reconstruct_cd (inc/reconstruct.hpp:185-207) on the device
inline ReconstructionResult reconstruct_cd(PseudoLikelihood& model, double eps = -1.0, int max_iters = 1000,
                                           int threads = 1) {
    std::vector<nrg_iter_record> recs(static_cast<std::size_t>(std::max(max_iters, 1)));
    int32_t ni = 0, cv = 0;
    detail::check(nrg_reconstruct_cd(model.context(), eps, max_iters, threads, recs.data(),
                                     static_cast<int32_t>(recs.size()), &ni, &cv));
    model.pull_state();
    ReconstructionResult res;
    res.converged = cv != 0;
    for (int t = 0; t < ni; ++t) {
        const auto& r = recs[static_cast<std::size_t>(t)];
        res.trace.iterations.push_back({r.iter, r.delta, r.seconds, static_cast<std::size_t>(r.candidates), r.objective});
    }
    return res;
}

}  // namespace netrec

#endif
