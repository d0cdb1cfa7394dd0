import os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np
import paper_2401_01404_b200 as P
import oracle_lib as O
for (n, M) in [(300, 256), (600, 300), (2000, 1000)]:
    m = P.Model(n, M, P.NRG_ISING, O.ising_lambda(n, M))
    m.generate_ising(mean_deg=4.0, seed=3)
    m.gcd_iteration(0, kappa=2.0, seed=3)
    nodes = np.arange(n, dtype=np.int32); tot = n * (n - 1) // 2
    os.environ.pop("NRG_NO_TC", None)
    m.begin_generation(); m.reset_counters()
    t = time.perf_counter(); a, _, _ = m.find_best(P.NRG_EXACT, tot, nodes, exhaustive=True); ta = time.perf_counter() - t
    st = m.kernel_stats()
    os.environ["NRG_NO_TC"] = "1"
    m.begin_generation(); m.reset_counters()
    t = time.perf_counter(); b, _, _ = m.find_best(P.NRG_EXACT, tot, nodes, exhaustive=True); tb = time.perf_counter() - t
    same = np.array_equal(a["i"], b["i"]) and np.array_equal(a["j"], b["j"]) and np.array_equal(a["dist"], b["dist"])
    nd = int(np.sum(a["dist"] != b["dist"]))
    print(n, M, "tc_launches", st["tc_launches"], "equal", same, "ndiff", nd, "t_tc %.3f t_cc %.3f" % (ta, tb), flush=True)
