// tests/cpp/test_dropin.cpp — the drop-in C++ API (include/netrec_b200/netrec.hpp) used
// the way the reference's own tests use netrec (proj/tests/test_model.cpp,
// test_knn.cpp, test_findbest.cpp): same types, same calls, GPU underneath.
// Prints one line per case; exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <numeric>
#include <random>
#include <set>
#include <vector>

#include "netrec_b200/netrec.hpp"

using namespace netrec;

static int failures = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
            ++failures;                                                          \
        }                                                                        \
    } while (0)

static SampleMatrix random_spins(NodeId n, int M, unsigned seed) {
    SampleMatrix x(n, M);
    std::mt19937_64 rng(seed);
    for (NodeId i = 0; i < n; ++i)
        for (int m = 0; m < M; ++m) x.set(i, m, (rng() & 1) ? 1.0 : -1.0);
    return x;
}

// correlated spins: node i copies node i-1 with probability 0.8
static SampleMatrix chain_spins(NodeId n, int M, unsigned seed) {
    SampleMatrix x(n, M);
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    for (int m = 0; m < M; ++m) {
        double prev = (rng() & 1) ? 1.0 : -1.0;
        for (NodeId i = 0; i < n; ++i) {
            const double v = (i > 0 && u(rng) < 0.8) ? prev : ((rng() & 1) ? 1.0 : -1.0);
            x.set(i, m, v);
            prev = v;
        }
    }
    return x;
}

static std::vector<NodeId> iota_nodes(std::size_t n) {
    std::vector<NodeId> v(n);
    std::iota(v.begin(), v.end(), 0);
    return v;
}

int main() {
    {  // test_model.cpp:110-118
        const NodeId n = 40;
        const int M = 30;
        SampleMatrix x = random_spins(n, M, 1);
        SparseWeights w(n, M);
        PseudoLikelihood model(ModelKind::ising, 1.0, x, w);
        CHECK(std::fabs(model.log_posterior() + n * M * std::log(2.0)) <= 1e-12 * n * M);
        std::printf("ok   ising empty-state log-posterior\n");
    }
    {  // distance symmetry + memoization (test_model.cpp:255-310)
        SampleMatrix x = chain_spins(30, 200, 2);
        SparseWeights w = make_empty_state(ModelKind::ising, x);
        PseudoLikelihood model(ModelKind::ising, 5.0, x, w);
        DistanceCache cache;
        cache.begin_generation();
        const ModelDistance d(model, cache, DistanceMode::exact);
        for (NodeId i = 0; i < 10; ++i)
            for (NodeId j = i + 1; j < 12; ++j) CHECK(d(i, j) == d(j, i));
        const EdgeOpt r = model.optimize_edge(3, 4);
        CHECK(r.w > 0.0 && r.gain > 0.0);
        CHECK(std::fabs(-(model.log_posterior() + r.gain) - d(3, 4)) <= 1e-9 * std::fabs(d(3, 4)));
        std::printf("ok   distance symmetric, memoized, equals -(base + gain)\n");
    }
    {  // TableMetric kNN invariants (test_knn.cpp:83-104)
        const std::size_t n = 64;
        std::mt19937_64 rng(17);
        std::normal_distribution<double> nd;
        std::vector<double> t(n * n, 0.0);
        for (std::size_t i = 0; i < n; ++i)
            for (std::size_t j = i + 1; j < n; ++j) t[i * n + j] = nd(rng);
        const DeviceTableDistance d(t, n);
        const auto nodes = iota_nodes(n);
        for (std::uint64_t seed = 0; seed < 4; ++seed) {
            KnnParams p;
            p.seed = seed;
            const KnnResult r = find_knn(6, nodes, d, p);
            for (std::size_t li = 0; li < n; ++li) {
                std::set<NodeId> ids;
                for (const auto& e : r.graph.neighbors(li)) {
                    CHECK(e.id != nodes[li]);
                    CHECK(e.dist == d(nodes[li], e.id));
                    ids.insert(e.id);
                }
                CHECK(ids.size() == 6u);
            }
        }
        // base case == exhaustive (test_findbest.cpp:57-65)
        const BestPairsResult a = find_best(n * n / 4, nodes, d);
        const BestPairsResult b = find_best_exhaustive(n * n / 4, nodes, d);
        CHECK(a.pairs.size() == b.pairs.size());
        for (std::size_t t2 = 0; t2 < a.pairs.size() && t2 < b.pairs.size(); ++t2)
            CHECK(a.pairs[t2].i == b.pairs[t2].i && a.pairs[t2].j == b.pairs[t2].j && a.pairs[t2].dist == b.pairs[t2].dist);
        const BestPairsResult c = find_best(40, nodes, d, FindBestParams{});
        CHECK(c.trace.halving_ok());
        for (std::size_t t2 = 1; t2 < c.pairs.size(); ++t2) CHECK(candidate_less(c.pairs[t2 - 1], c.pairs[t2]));
        std::printf("ok   TableMetric kNN invariants, FindBest base case, sorted pairs\n");
    }
    {  // reconstruct_gcd with a candidate hook (inc/reconstruct.hpp:148-181)
        const NodeId n = 200;
        const int M = 400;
        SampleMatrix x = chain_spins(n, M, 3);
        SparseWeights w = make_empty_state(ModelKind::ising, x);
        PseudoLikelihood model(ModelKind::ising, 2.0 * std::sqrt(M * std::log(n)), x, w);
        const double before = model.log_posterior();
        ReconstructionConfig cfg;
        cfg.kappa = 1.0;
        cfg.max_iters = 8;
        cfg.seed = 5;
        int hooked = 0;
        cfg.candidate_hook = [&](int, std::vector<CandidateEdge>& v) { hooked += v.empty() ? 0 : 1; };
        const ReconstructionResult res = reconstruct_gcd(model, cfg);
        CHECK(hooked == static_cast<int>(res.trace.iterations.size()));
        CHECK(res.trace.iterations.back().objective > before);
        // the caller's SparseWeights now holds the device state: chain edges recovered
        std::size_t chain = 0;
        for (NodeId i = 1; i < n; ++i) chain += w.has_edge(i - 1, i) ? 1 : 0;
        CHECK(chain > static_cast<std::size_t>(0.9 * (n - 1)));
        CHECK(std::fabs(model.log_posterior() - res.trace.iterations.back().objective) <=
              1e-9 * std::fabs(res.trace.iterations.back().objective));
        std::printf("ok   reconstruct_gcd: %zu iterations, %zu edges, chain recall %.3f\n", res.trace.iterations.size(),
                    w.edge_count(), chain / double(n - 1));
    }
    {  // binary sample / weight files and reconstruct_cd
        const int n = 40, M = 64;
        SampleMatrix x(n, M);
        for (int i = 0; i < n; ++i)
            for (int m = 0; m < M; ++m) x.set(i, m, ((i * 7 + m * 3 + i * m) % 5) < 2 ? 1.0 : -1.0);
        SparseWeights w(n, M);
        w.set_edge(1, 5, 0.25, x);
        w.set_edge(7, 3, -0.5, x);
        w.set_theta(2, 0.125);
        const std::string sp = "/tmp/nrg_dropin_samples.bin", wp = "/tmp/nrg_dropin_weights.bin";
        write_samples_binary(sp, x, true);
        write_weights_binary(wp, w);
        const SampleMatrix y = read_samples_binary(sp);
        SparseWeights v = read_weights_binary(wp, y);
        bool same = y.num_nodes() == n && y.num_samples() == M;
        for (int i = 0; i < n && same; ++i)
            for (int m = 0; m < M; ++m) same = same && y.row(i)[m] == x.row(i)[m];
        CHECK(same);
        CHECK(v.edge_count() == 2 && v.weight(1, 5) == 0.25 && v.weight(3, 7) == -0.5 && v.theta(2) == 0.125);
        for (int i = 0; i < n; ++i)
            for (int m = 0; m < M; ++m) CHECK(v.sums_row(i)[m] == w.sums_row(i)[m]);
        PseudoLikelihood model(ModelKind::ising, 10.0, y, v);
        const ReconstructionResult r = reconstruct_cd(model, -1.0, 5);
        CHECK(!r.trace.iterations.empty() && r.trace.iterations[0].candidates == static_cast<std::size_t>(n * (n - 1) / 2));
        std::printf("ok   binary sample/weight files round-trip; reconstruct_cd %zu sweeps\n", r.trace.iterations.size());
    }
    {  // exception types (inc/model.hpp:115-123, inc/knn.hpp:153-155)
        SampleMatrix x(4, 3);
        SparseWeights w(4, 3);
        bool threw = false;
        try {
            PseudoLikelihood m(ModelKind::ising, 1.0, x, w);  // zeros are not spins
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        std::printf("ok   validation errors map to the reference's exception types\n");
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
    return failures;
}
