"""GPU parity of the TGT+ AESC estimator (aesc.hpp) against the reference's
golden vectors and the CPU oracle.

Integer decisions (tau, tau~, pair/step counts, lambda_hat) must be bit-exact.
Float64 estimates must agree within |gpu - ref| <= 1e-9 * |ref| + 1e-15: the
GPU sums landing probabilities in ascending-neighbour order (the reference
pushes in discovery order) and reduces walk pairs with a tree (the reference
folds left), so only summation order differs (SURVEY §7 hard part 2).
"""
import ast

import numpy as np
import pytest

from conftest import golden_graph

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-9, 1e-15


def close(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return bool(np.all(np.abs(a - b) <= RTOL * np.abs(b) + ATOL))


def worst(a, b):
    return float(np.max(np.abs(a - b) / (np.abs(b) + 1e-300))) if len(a) else 0.0


def cfg_from(sb, kw):
    c = sb.AescConfig()
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def test_aesc_matches_reference_goldens(golden, sb):
    i = 0
    while f"aesc/{i}/graph" in golden:
        gname = str(golden[f"aesc/{i}/graph"])
        kw = ast.literal_eval(str(golden[f"aesc/{i}/kw"]))
        g = golden_graph(golden, gname)
        est = sb.aesc(g, cfg_from(sb, kw))
        lam, pairs, steps = golden[f"aesc/{i}/stats"]
        assert est.plan.lambda_hat == lam, (gname, kw)
        assert np.array_equal(est.plan.tau, golden[f"aesc/{i}/tau"])
        assert np.array_equal(est.plan.tau_tilde, golden[f"aesc/{i}/tau_tilde"]), (gname, kw)
        assert est.total_walk_pairs == int(pairs) and est.total_walk_steps == int(steps)
        assert close(est.g_hat, golden[f"aesc/{i}/g_hat"]), (gname, kw, worst(est.g_hat, golden[f"aesc/{i}/g_hat"]))
        assert close(est.s_hat, golden[f"aesc/{i}/s_hat"]), (gname, kw)
        i += 1
    assert i >= 10


def test_truncation_plans_match_reference(golden, sb):
    i = 0
    while f"plan/{i}/spec" in golden:
        eps, om, tmax, pe = golden[f"plan/{i}/spec"]
        g = golden_graph(golden, str(golden[f"plan/{i}/graph"]))
        p = sb.truncated_lengths(g, eps, int(om), int(tmax), bool(pe))
        lam, cl = golden[f"plan/{i}/lambda"]
        assert p.lambda_hat == lam and p.clamped == bool(cl)
        assert np.array_equal(p.tau, golden[f"plan/{i}/tau"])
        i += 1


def test_propagation_matches_reference(golden, sb):
    for key in golden:
        if key.startswith("prop/") and key.endswith("/prob"):
            _, gname, src, eps, cap, _ = key.split("/")
            base = key[: -len("/prob")]
            g = golden_graph(golden, gname)
            plan = sb.TruncationPlan(golden[base + "/tau"])
            lp, depth = sb.propagate_landing_probabilities(g, int(src), plan, float(eps), 0.05,
                                                           int(cap))
            assert depth == int(golden[base + "/depth"][0]) and lp.depth == depth
            want = golden[key]
            assert np.array_equal(np.nonzero(want)[0], lp.support)
            assert close(lp.dense(g.n), want), key
            assert abs(lp.sum() - 1.0) <= 1e-12


def test_propagation_star_and_fig1(sb):
    # test_aesc.cpp:89-117 (depth 2 of fig1 from A: {1/3, 1/6, 1/6, 1/3})
    g = sb.fig1()
    plan = sb.TruncationPlan(np.full(g.m, 3, np.uint32))
    lp, d = sb.propagate_landing_probabilities(g, 0, plan, 0.05, 0.05, switch_depth_cap=2)
    assert d == 2
    assert np.allclose(lp.dense(4), [1 / 3, 1 / 6, 1 / 6, 1 / 3], rtol=1e-14)
    s5 = sb.star(5)
    lp, d = sb.propagate_landing_probabilities(s5, 0, sb.TruncationPlan(np.full(5, 3, np.uint32)),
                                               0.05, 0.05, switch_depth_cap=1)
    assert d == 1 and lp.prob_of(0) == 0.0
    assert np.allclose([lp.prob_of(v) for v in range(1, 6)], 0.2, rtol=1e-15)


def test_estimate_edge_contract(sb):
    # test_aesc.cpp:154-181
    g = sb.fig1()
    empty = sb.LandingProbs(depth=1)
    assert sb.estimate_edge(g, 0, 1, empty, 3, 50, sb.WalkMode.Saba, 7) == 0.0
    p2 = sb.path(2)
    lp = sb.LandingProbs(0, 1, np.array([0, 1], np.uint32), np.array([0.5, 0.5]))
    assert abs(sb.estimate_edge(p2, 0, 1, lp, 4, 64, sb.WalkMode.Saba, 3)) <= 1e-12
    with pytest.raises(ValueError):
        sb.estimate_edge(g, 0, 1, empty, 0, 5, sb.WalkMode.Saba, 1)
    with pytest.raises(ValueError):
        sb.estimate_edge(g, 0, 1, empty, 1, 0, sb.WalkMode.Saba, 1)


def test_estimate_edge_matches_reference(sb):
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        pytest.skip("compiled reference not available")
    R = Reference()
    g = sb.make_scale_free(300, 4, 5)
    rg = R.from_csr(g.offsets, g.adjacency)
    tau, _, _ = R.truncated_lengths(rg, 0.05)
    prob, depth = R.propagate(rg, 11, tau, 0.1, 0.05)
    lp = sb.LandingProbs(11, depth, np.nonzero(prob)[0].astype(np.uint32), prob[prob != 0])
    for vj, te, nreq, seed in ((int(g.neighbors(11)[0]), 5, 5000, 99), (int(g.neighbors(11)[1]), 9, 3000, 7)):
        want = R.estimate_edge(rg, 11, vj, prob, depth, te, nreq, 3, seed)
        got = sb.estimate_edge(g, 11, vj, lp, te, nreq, sb.WalkMode.Saba, seed)
        assert abs(got - want) <= RTOL * abs(want) + ATOL, (got, want)


def exact_sc(g):
    """Effective resistance per edge via the Laplacian pseudo-inverse (small n)."""
    n = g.n
    L = np.zeros((n, n))
    e = g.edges()
    for u, v in e:
        L[u, v] -= 1
        L[v, u] -= 1
        L[u, u] += 1
        L[v, v] += 1
    Lp = np.linalg.pinv(L)
    return np.array([Lp[u, u] + Lp[v, v] - 2 * Lp[u, v] for u, v in e])


def test_epsilon_contract_small_graphs(sb):
    # test_aesc.cpp:183-223 (exact values from the Laplacian pseudo-inverse)
    assert np.allclose(sb.aesc(sb.triangle(), sb.AescConfig(epsilon=0.05)).s_hat, 2 / 3, atol=0.05)
    assert np.all(np.abs(sb.aesc(sb.star(5), sb.AescConfig(epsilon=0.05)).s_hat - 1) <= 0.05)
    for g in (sb.fig1(), sb.path(5), sb.complete(4), sb.grid3x3(), sb.petersen()):
        ex = exact_sc(g)
        for mode in (sb.WalkMode.Hash, sb.WalkMode.Saba):
            est = sb.aesc(g, sb.AescConfig(epsilon=0.05, mode=mode))
            assert np.all(np.abs(est.s_hat - ex) <= 0.05)
    p3 = sb.path(3)
    est = sb.aesc(p3, sb.AescConfig(epsilon=0.05, switch_depth_cap=0))  # test_aesc.cpp:225-238
    assert est.total_walk_pairs > 0 and np.all(np.abs(est.s_hat - 1.0) <= 0.05)


def test_mode_equivalence_and_determinism(sb):
    # test_aesc.cpp:265-308: hash == saba bitwise; reruns bitwise
    for g in (sb.fig1(), sb.path(5), sb.grid3x3()):
        cfg = sb.AescConfig(epsilon=0.05, max_truncation=5, switch_depth_cap=1, master_seed=20240917)
        a = sb.aesc(g, cfg)
        cfg.mode = sb.WalkMode.Hash
        b = sb.aesc(g, cfg)
        assert a.total_walk_pairs > 0
        assert np.array_equal(a.s_hat, b.s_hat)
        c = sb.aesc(g, cfg)
        assert np.array_equal(b.s_hat, c.s_hat)


def test_symmetrisation(sb):
    g = sb.fig1()
    est = sb.aesc(g, sb.AescConfig())
    for e, (u, v) in enumerate(g.edges()):
        assert est.s_hat[e] == est.g_hat[g.slot_of(u, v)] + est.g_hat[g.slot_of(v, u)]


def test_rejects_bad_inputs(sb):
    g = sb.triangle()
    with pytest.raises(ValueError):
        sb.aesc(g, sb.AescConfig(epsilon=0.0))
    with pytest.raises(ValueError):
        sb.aesc(g, sb.AescConfig(delta=1.5))
    with pytest.raises(ValueError):
        sb.aesc(g, sb.AescConfig(mode=sb.WalkMode.Naive))
    with pytest.raises(RuntimeError):
        sb.aesc(sb.Graph.from_edges(4, [(0, 1), (2, 3)]), sb.AescConfig())


def test_rmat_full_aesc_matches_oracle(sb, oracle):
    """A cfg3-shaped graph at small scale (R-MAT s10 ef8 LCC, eps 0.1,
    delta 0.01): the whole estimator, every source, against the oracle."""
    g = sb.make_rmat(10, 8, seed=3)
    est = sb.aesc(g, sb.AescConfig(epsilon=0.1, delta=0.01))
    ref = oracle.aesc(g.offsets, g.adjacency, epsilon=0.1, delta=0.01)
    assert est.plan.lambda_hat == ref.lambda_hat
    assert np.array_equal(est.plan.tau_tilde, ref.tau_tilde)
    assert est.total_walk_pairs == ref.total_walk_pairs > 0
    assert close(est.g_hat, ref.g_hat), worst(est.g_hat, ref.g_hat)
    assert close(est.s_hat, ref.s_hat)


def test_hub_rows_every_path_matches_oracle(sb, oracle):
    """Rows above the 256-neighbour piece threshold on every propagation path:
    a graph of hub rows only (a ring of eight K_258: every degree >= 257, so
    dense depths have no light-row work list and the pieces kernel takes every
    hub row), and hubs joined by light rows (sparse depths list the heavy
    candidates, dense depths hand pieces out with the light rows)."""
    k, c = 258, 8
    pairs = []
    for q in range(c):
        b = q * k
        pairs += [(b + u, b + v) for u in range(k) for v in range(u + 1, k)]
        pairs.append((b + k - 1, ((q + 1) % c) * k))
    hubs = sb.Graph.from_edges(k * c, pairs)
    assert int(np.diff(hubs.offsets).min()) > 256
    rng = np.random.default_rng(11)
    spokes = [(h, int(x)) for h in range(4) for x in rng.choice(np.arange(4, 3000), 400, replace=False)]
    mixed = sb.Graph.from_edges(3000, spokes + [(v, v + 1) for v in range(3, 2999)])
    for g, eps in ((hubs, 0.2), (mixed, 0.1)):
        assert g.max_degree() > 256
        src = np.arange(0, g.n, max(1, g.n // (8 if g is hubs else 96)), dtype=np.uint32)
        est = sb.aesc(g, sb.AescConfig(epsilon=eps, delta=0.05), sources=src)
        ref = oracle.aesc(g.offsets, g.adjacency, epsilon=eps, delta=0.05, sources=src)
        assert np.array_equal(est.plan.tau_tilde[src], ref.tau_tilde[src])
        assert est.total_walk_pairs == ref.total_walk_pairs
        assert close(est.g_hat, ref.g_hat), worst(est.g_hat, ref.g_hat)


def test_source_subset_and_shards(sb, oracle):
    g = sb.make_rmat(12, 8, seed=5)
    src = np.array([0, 1, 2, 7, 100, 513, g.n - 1], np.uint32)
    cfg = sb.AescConfig(epsilon=0.1, delta=0.01)
    est = sb.aesc(g, cfg, sources=src)
    ref = oracle.aesc(g.offsets, g.adjacency, epsilon=0.1, delta=0.01, sources=src)
    assert np.array_equal(est.plan.tau_tilde[src], ref.tau_tilde[src])
    assert close(est.g_hat, ref.g_hat), worst(est.g_hat, ref.g_hat)
    acc = np.zeros_like(est.g_hat)
    for i in range(3):
        acc += sb.aesc(g, cfg, sources=src, shard_index=i, shard_count=3).g_hat
    assert np.array_equal(acc, est.g_hat)  # GPU-count invariance is bitwise
