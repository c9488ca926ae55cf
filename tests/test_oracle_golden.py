"""Pin the CPU oracle (oracle/saba_oracle.c) against golden vectors produced
by the reference itself (tests/golden/make_golden.py). Everything is
bit-exact: integer outputs and float64 g_hat / s_hat / lambda / probabilities."""
import ast

import numpy as np
import pytest

from conftest import golden_graph  # noqa: F401


def csr(golden, name):
    return golden[f"g/{name}/off"], golden[f"g/{name}/adj"]


def test_slot_edges(golden, oracle):
    for key in golden:
        if key.endswith("/slot_edge"):
            name = key.split("/")[1]
            off, adj = csr(golden, name)
            assert np.array_equal(oracle.slot_edges(off, adj), golden[key]), name


def test_random_walk_paths(golden, oracle):
    for gname in ("sf300_4_5", "petersen", "sf2000_8_17"):
        off, adj = csr(golden, gname)
        st, sd, paths = (golden[f"walk/{gname}/{k}"] for k in ("starts", "seeds", "paths"))
        for i in range(len(st)):
            got = oracle.random_walk(off, adj, int(st[i]), paths.shape[1], int(sd[i]))
            assert np.array_equal(got, paths[i]), (gname, i)


def test_random_bouquet(golden, oracle):
    off, adj = csr(golden, "sf300_4_5")
    for b, seed in enumerate(golden["bouquet/seeds"]):
        got = oracle.random_walk(off, adj, 7, 12, int(seed))
        assert np.array_equal(got, golden["bouquet/paths"][b])


def test_campaign_counts(golden, oracle):
    for key in golden:
        if not key.startswith("camp/"):
            continue
        _, gname, spec = key.split("/")
        K, L, s = (int(x[1:]) for x in spec.split("_"))
        off, adj = csr(golden, gname)
        got = oracle.campaign_counts(off, adj, K=K, length=L, master=s, threads=2)
        assert np.array_equal(got, golden[key]), key


def test_uniform_start_campaign(golden, oracle):
    off, adj = csr(golden, "sf2000_8_17")
    kv = oracle.uniform_start_counts(len(off) - 1, 32768, 42)
    assert kv.sum() == 32768
    got = oracle.campaign_counts(off, adj, length=16, master=42, k_per_vertex=kv)
    assert np.array_equal(got, golden["ucamp/sf2000_8_17/W32768_L16_s42"])
    assert got.sum() == 32768 * 16


def test_campaign_ranges_partition(golden, oracle):
    off, adj = csr(golden, "sf400_5_21")
    full = golden["camp/sf400_5_21/K64_L7_s9"]
    total = 400 * 64
    for parts in (1, 2, 3, 7):
        acc = np.zeros_like(full)
        for i in range(parts):
            acc += oracle.campaign_range(off, adj, total * i // parts, total * (i + 1) // parts,
                                         K=64, length=7, master=9)
        assert np.array_equal(acc, full), parts


def test_walk_budget(golden, oracle):
    assert oracle.walk_budget(5, 0.05, 0.05, 4, 100) == 44936  # test_aesc.cpp:27
    for t, eps, delta, d, m, want in golden["walk_budget"]:
        assert oracle.walk_budget(int(t), eps, delta, int(d), int(m)) == int(want)
    with pytest.raises(ValueError):
        oracle.walk_budget(0, 0.05, 0.05, 1, 10)
    with pytest.raises(ValueError):
        oracle.walk_budget(1, 0.0, 0.05, 1, 10)


def test_truncation_plans(golden, oracle):
    i = 0
    while f"plan/{i}/spec" in golden:
        eps, om, tmax, pe = golden[f"plan/{i}/spec"]
        gname = str(golden[f"plan/{i}/graph"])
        off, adj = csr(golden, gname)
        tau, lam, cl = oracle.truncated_lengths(off, adj, eps, int(om), int(tmax), bool(pe))
        want_lam, want_cl = golden[f"plan/{i}/lambda"]
        assert lam == want_lam, (gname, lam, want_lam)  # bitwise
        assert cl == bool(want_cl)
        assert np.array_equal(tau, golden[f"plan/{i}/tau"]), gname
        i += 1
    assert i >= 10


def test_propagation(golden, oracle):
    for key in golden:
        if key.startswith("prop/") and key.endswith("/prob"):
            _, gname, src, eps, cap, _ = key.split("/")
            base = key[: -len("/prob")]
            off, adj = csr(golden, gname)
            prob, depth = oracle.propagate(off, adj, int(src), golden[base + "/tau"], float(eps),
                                           0.05, int(cap))
            assert depth == int(golden[base + "/depth"][0])
            assert np.array_equal(prob, golden[key]), key


def test_aesc_full(golden, oracle):
    i = 0
    while f"aesc/{i}/graph" in golden:
        gname = str(golden[f"aesc/{i}/graph"])
        kw = ast.literal_eval(str(golden[f"aesc/{i}/kw"]))
        off, adj = csr(golden, gname)
        r = oracle.aesc(off, adj, threads=2, **kw)
        lam, pairs, steps = golden[f"aesc/{i}/stats"]
        assert r.lambda_hat == lam
        assert r.total_walk_pairs == int(pairs) and r.total_walk_steps == int(steps)
        assert np.array_equal(r.tau, golden[f"aesc/{i}/tau"])
        assert np.array_equal(r.tau_tilde, golden[f"aesc/{i}/tau_tilde"])
        assert np.array_equal(r.g_hat, golden[f"aesc/{i}/g_hat"]), (gname, kw)
        assert np.array_equal(r.s_hat, golden[f"aesc/{i}/s_hat"]), (gname, kw)
        i += 1
    assert i >= 10


def test_aesc_source_subset_matches_full(golden, oracle):
    off, adj = csr(golden, "sf300_4_5")
    full = golden["aesc/11/g_hat"]  # sf300_4_5 eps 0.1
    src = np.array([3, 17, 150, 299], np.uint32)
    r = oracle.aesc(off, adj, epsilon=0.1, sources=src)
    for s in src:
        sl = slice(off[s], off[s + 1])
        assert np.array_equal(r.g_hat[sl], full[sl])


def test_oracle_generators_match_product(oracle, sb):
    """oracle_gen.c (the generators the reference arm of bench.py uses, so that
    it never loads the product library) builds the product's CSR bit for bit."""
    cases = [(oracle.gen_rmat(12, 8, seed=7), sb.make_rmat(12, 8, seed=7)),
             (oracle.gen_rmat(11, 4, seed=3, keep_lcc=False), sb.make_rmat(11, 4, seed=3, keep_lcc=False)),
             (oracle.gen_erdos_renyi(4096, 16384, 1), sb.make_erdos_renyi(4096, 16384, 1)),
             (oracle.gen_chung_lu(20000, 2.2, 12.0, 500.0, seed=4),
              sb.make_chung_lu(20000, 2.2, 12.0, 500.0, seed=4))]
    for (off, adj), g in cases:
        assert np.array_equal(off, g.offsets) and np.array_equal(adj, g.adjacency)
