"""Comparison helpers with the parity tolerances of BASELINE.json north_star /
SURVEY.md §8c, written once so every test states the same bar:

  * w*        : |dw| <= 1e-4 absolute
  * gain      : |dgain| <= 1e-5 * max(|gain_ref|, 1e-8 * M)
  * dist      : |ddist| <= 1e-5 * |dist_ref| (relative) — and the gain check above
  * couplings after updates on the same candidates: identical support, |dw| <= 1e-4
"""
from __future__ import annotations

import numpy as np

W_TOL = 1e-4
GAIN_REL = 1e-5


def gain_ok(g, g_ref, M):
    g, g_ref = np.asarray(g), np.asarray(g_ref)
    tol = GAIN_REL * np.maximum(np.abs(g_ref), 1e-8 * M)
    return np.abs(g - g_ref) <= tol


def assert_gains(g, g_ref, M, what="gain"):
    ok = gain_ok(g, g_ref, M)
    if not ok.all():
        bad = np.flatnonzero(~ok)[:10]
        raise AssertionError(f"{what}: {(~ok).sum()} of {len(ok)} outside tolerance; "
                             f"first {bad}: {np.asarray(g)[bad]} vs {np.asarray(g_ref)[bad]}")


def assert_w(w, w_ref, what="w*", tol=W_TOL):
    d = np.abs(np.asarray(w) - np.asarray(w_ref))
    if not (d <= tol).all():
        bad = np.flatnonzero(d > tol)[:10]
        raise AssertionError(f"{what}: max |dw| {d.max():.3g}; first {bad}: "
                             f"{np.asarray(w)[bad]} vs {np.asarray(w_ref)[bad]}")


def assert_rel(a, b, rel, what):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    d = np.abs(a - b) / np.maximum(np.abs(b), 1e-300)
    if not (d <= rel).all():
        i = int(np.argmax(d))
        raise AssertionError(f"{what}: max rel diff {d.max():.3g} at {i}: {a.flat[i]!r} vs {b.flat[i]!r}")


def edge_dict(ei, ej, w):
    return {(int(min(a, b)), int(max(a, b))): float(x) for a, b, x in zip(ei, ej, w)}


def assert_same_couplings(state, ref_state, tol=W_TOL, allow_support_diff=0):
    """Same support (up to `allow_support_diff` near-kink flips with |w| <= tol) and
    couplings within tol."""
    a = edge_dict(*state[1:4])
    b = edge_dict(*ref_state[1:4])
    only = [k for k in set(a) ^ set(b) if abs(a.get(k, 0.0)) > tol or abs(b.get(k, 0.0)) > tol]
    assert len(only) <= allow_support_diff, f"support differs on {len(only)} edges: {only[:10]}"
    worst = max((abs(a.get(k, 0.0) - b.get(k, 0.0)) for k in set(a) | set(b)), default=0.0)
    assert worst <= tol, f"coupling mismatch {worst:.3g}"


def row_sets(ids):
    return [set(map(int, r)) for r in np.asarray(ids)]


def knn_recall(approx_ids, exact_ids):
    """Per-node recall (test_knn.cpp:45-57)."""
    sa, se = row_sets(approx_ids), row_sets(exact_ids)
    k = np.asarray(exact_ids).shape[1]
    return float(np.mean([len(a & e) / k for a, e in zip(sa, se)]))


def pairs_equal(a, b):
    """same_pairs (test_findbest.cpp:45-53): bitwise identity of (i, j, dist)."""
    return (len(a) == len(b) and (np.asarray(a["i"]) == np.asarray(b["i"])).all()
            and (np.asarray(a["j"]) == np.asarray(b["j"])).all()
            and (np.asarray(a["dist"]) == np.asarray(b["dist"])).all())


def near_tie_tol(d_cut, base, M):
    """Window around a cut distance inside which two implementations may order pairs
    differently: the north_star gain tolerance at the cut's gain plus the rounding of
    dist = -(base + gain) (a few ulps of base)."""
    g_cut = -d_cut - base
    return 1e-5 * max(abs(g_cut), 1e-8 * M) + 4 * float(np.spacing(abs(base)))


def _offset(pairs_a, pairs_b):
    """Largest |d_a - d_b| over the entries both sides hold: the two implementations'
    distances of one pair differ by the rounding of their fp64 base (the generation's
    log_posterior, summed in different orders) -- a constant-size shift, asserted to be
    within 1e-9 relative."""
    off = 0.0
    for k in pairs_a.keys() & pairs_b.keys():
        a, b = pairs_a[k], pairs_b[k]
        assert abs(a - b) <= 1e-9 * abs(b), f"entry {k}: {a!r} vs {b!r}"
        off = max(off, abs(a - b))
    return off


def assert_rows_tie_aware(ids_a, d_a, ids_b, d_b, base, M, what="kNN rows"):
    """Per-node kNN rows of two implementations: shared neighbours carry the same
    distance (1e-9 relative), and every neighbour in one row but not the other is a
    near-tie at the other row's k-th distance: within the north_star gain tolerance plus
    the measured cross-implementation offset of the distances.  Returns the number of
    rows that differ."""
    rows = []
    off = 0.0
    for r in range(len(ids_a)):
        ra = {int(x): float(d) for x, d in zip(ids_a[r], d_a[r])}
        rb = {int(x): float(d) for x, d in zip(ids_b[r], d_b[r])}
        off = max(off, _offset(ra, rb))
        rows.append((ra, rb))
    diff_rows = 0
    for r, (ra, rb) in enumerate(rows):
        if ra.keys() == rb.keys():
            continue
        diff_rows += 1
        cut_a, cut_b = max(ra.values()), max(rb.values())
        tol = near_tie_tol(max(cut_a, cut_b), base, M) + off
        # an entry only one side kept must sit at the other side's cut (a tie there)
        worst = max([cut_b - ra[k] for k in ra.keys() - rb.keys()] + [cut_a - rb[k] for k in rb.keys() - ra.keys()])
        assert worst <= tol, (f"{what}: row {r} differs beyond a near-tie ({worst:.3g} > {tol:.3g}): "
                              f"{sorted(ra.items(), key=lambda t: t[1])} vs {sorted(rb.items(), key=lambda t: t[1])}")
    return diff_rows


def assert_lists_tie_aware(a, b, base, M, what="candidate lists"):
    """Two FindBest pair lists (sorted by (dist, i, j)): same length, shared pairs with
    the same distance (1e-9 relative), every pair in the symmetric difference a
    near-tie at the other list's cut.  Returns the size of the symmetric difference."""
    assert len(a) == len(b), (len(a), len(b))
    ka = {(int(x), int(y)): float(d) for x, y, d in zip(a["i"], a["j"], a["dist"])}
    kb = {(int(x), int(y)): float(d) for x, y, d in zip(b["i"], b["j"], b["dist"])}
    off = _offset(ka, kb)
    only_a, only_b = ka.keys() - kb.keys(), kb.keys() - ka.keys()
    if only_a or only_b:
        cut_a, cut_b = float(a["dist"][-1]), float(b["dist"][-1])
        tol = near_tie_tol(max(cut_a, cut_b), base, M) + off
        bad = [(k, ka[k]) for k in only_a if cut_b - ka[k] > tol] + [(k, kb[k]) for k in only_b if cut_a - kb[k] > tol]
        assert not bad, (f"{what}: {len(bad)} of {len(only_a) + len(only_b)} differing pairs are not near-ties at "
                         f"the cut ({cut_a!r} / {cut_b!r}): {bad[:6]}")
    return len(only_a) + len(only_b)
