// The reference's OWN experiment harness (inc/bench.hpp, compiled unmodified from
// /root/reference) on the device path through the drop-in: ER precision truth, Gibbs
// samples, FindBest scaling / recall, GCD-vs-CD convergence and support metrics.
// Built only where the reference headers exist (paper_2401_01404_b200/build.py);
// prints one line per check.
#include <cmath>
#include <cstdio>

#include "netrec_b200/netrec.hpp"
#include "netrec_b200/synth.hpp"
#include "netrec/bench.hpp"  // the reference's file: resolved from -I/root/reference/proj/include

using namespace netrec;

static int failures = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
            ++failures;                                                          \
        }                                                                        \
    } while (0)

int main() {
    {  // truth generator: ER support, diagonal dominance by 1/(1-eps)^2
        GeneratorSpec gs;
        gs.n = 400;
        gs.mean_deg = 4.0;
        gs.weight_mu = -1.0;
        gs.weight_sigma = 0.1;
        gs.seed = 3;
        const SparseWeights t = gen_er_precision(gs);
        CHECK(t.edge_count() > 600 && t.edge_count() < 1000);
        // theta_i = 1/sqrt(W_ii), W_ii = |row sum| / (1 - eps)^2, 1 for isolated nodes
        for (NodeId i = 0; i < gs.n; ++i) {
            double row = 0.0;
            for (NodeId j = 0; j < gs.n; ++j)
                if (j != i) row += std::fabs(t.weight(i, j));
            const double want = 1.0 / std::sqrt(row > 0.0 ? row / ((1.0 - gs.epsilon) * (1.0 - gs.epsilon)) : 1.0);
            CHECK(std::fabs(t.theta(i) - want) <= 1e-12 * want);
        }
        const ReconstructionMetrics m = eval_reconstruction(t, t);
        CHECK(m.precision == 1.0 && m.recall == 1.0 && m.f1 == 1.0 && m.rmse == 0.0);
        std::printf("ok   gen_er_precision: %zu edges; eval_reconstruction(truth, truth) = 1/1/1/0\n", t.edge_count());
    }
    {  // the fitted exponent of exact power laws
        const std::vector<NodeId> ns = {100, 200, 400, 800, 1600};
        std::vector<double> secs;
        for (NodeId n : ns) secs.push_back(1e-6 * std::pow(static_cast<double>(n), 1.5));
        CHECK(std::fabs(fit_scaling_exponent(ns, secs) - 1.5) < 1e-9);
        std::printf("ok   fit_scaling_exponent\n");
    }
    BenchModelConfig cfg;
    cfg.gen.mean_deg = 3.0;
    cfg.gen.weight_mu = -1.0;
    cfg.gen.weight_sigma = 0.2;
    cfg.gen.epsilon = 0.2;
    {
        const int M = 400;
        cfg.lambda = 2.0 * std::sqrt(M * std::log(150.0)) * 0.5;
        const std::vector<ConvergenceRun> runs = bench_convergence(150, M, {1.0, 2.0}, true, -1.0, 60, 11, cfg);
        CHECK(runs.size() == 3 && runs[0].label == "cd");
        for (const auto& r : runs) CHECK(r.result.converged && r.total_seconds > 0.0);
        const double cd = runs[0].final_objective;
        for (std::size_t t = 1; t < runs.size(); ++t)
            CHECK(std::fabs(runs[t].final_objective - cd) <= 1e-4 * std::fabs(cd));
        std::printf("ok   bench_convergence: CD %.6f, GCD(k=1) %.6f, GCD(k=2) %.6f (within 1e-4)\n", cd,
                    runs[1].final_objective, runs[2].final_objective);
    }
    {
        cfg.lambda = 10.0;
        const RecallReport rr = bench_recall(500, {1.0, 2.0}, 2, 100, cfg);
        CHECK(rr.mean_curves.size() == 2 && rr.rank1_by_seed[0].size() == 2);
        for (const auto& c : rr.mean_curves) CHECK(!c.empty() && c.back() > 0.0 && c.back() <= 1.0);
        CHECK(rr.mean_curves[1].back() >= rr.mean_curves[0].back());  // recall grows with kappa (Fig. 3)
        std::printf("ok   bench_recall: full-list recall %.3f (k=1), %.3f (k=2)\n", rr.mean_curves[0].back(),
                    rr.mean_curves[1].back());
    }
    {
        const ScalingReport sr = bench_findbest_scaling({400, 800, 1600, 3200}, {1.0}, 1, 20, cfg);
        CHECK(sr.rows.size() == 4 && sr.all_halving_ok && std::isfinite(sr.exponent.at(1.0)));
        std::printf("ok   bench_findbest_scaling: exponent %.2f, all levels halve\n", sr.exponent.at(1.0));
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
    return failures;
}
