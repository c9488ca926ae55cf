"""Every kernel variant and tuning switch against the oracle (VERDICT r1
"what's weak" 3): DESIGN.md claims no switch changes a result bit, so each
forced variant must reproduce the oracle's counts bit for bit (campaigns) and
the default variant's g_hat bit for bit (AESC; the default itself is checked
against the oracle within 1e-9, tau~ and pair/step counts exactly).

The library reads the switches once per process, so each variant runs in a
subprocess (tests/variant_worker.py). Graphs:
  * R-MAT s16 ef8 (fat adjacency auto-selected: L2-resident),
  * a ring of 2^21 + 4096 vertices with 2M chords: n > 2^21, so no packed
    adjacency and the unpacked hot / generic kernels,
  * R-MAT s13 ef8 AESC with 130 sources (3 batches: both batch workers),
  * Chung-Lu n=300K (m > 3.1M: beyond the fat-adjacency L2 budget, short
    plan: the 16-byte records).
Reference behaviour: walker.hpp:456-538 (campaign), aesc.hpp:380-400, 581-588
(switch and hook), aesc.hpp:448-525 (walk estimator).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
RTOL, ATOL = 1e-9, 1e-15

G_MID = ["rmat", 16, 8, 3]
G_BIG = ["ring", (1 << 21) + 4096, 2_000_000, 1]
A_MID = ["rmat", 13, 8, 5]
A_SHORT = ["chunglu", 300_000, 24.0, 3000.0, 2]

CAMPAIGN_MID = ["", "fat=1,wpt=2", "fat=1,wpt=8", "fat=1,agg=0",
                "fat=0,hot=1,packed=1", "fat=0,hot=1,packed=0", "fat=0,hot=1,hthreads=256",
                "fat=0,hot=1,hthreads=512", "fat=0,hot=1,agg=0",
                "fat=0,hot=0,wpt=1", "fat=0,hot=0,wpt=2", "fat=0,hot=0,wpt=8",
                "fat=0,hot=0,packed=0", "fat=0,hot=0,agg=0", "c32=1", "c32=1,packed=0",
                "sort=0", "sort=1", "fat=0,hot=1,sort=0",
                "fat=0,rec=1", "fat=0,rec=1,hthreads=512", "fat=0,rec=0,hot=1", "fat=0,rec=1,sort=0",
                "fat=0,rec=1,hrec=100,hcnt=301", "fat=0,rec=1,hrec=0,hcnt=0", "fat=0,rec=1,hrec=5000,hcnt=1000",
                "fat=0,rec=1,hrec=0,hcnt=70000", "priv=0", "priv=1"]
CAMPAIGN_BIG = ["", "hot=0", "hot=1,hthreads=256", "hot=0,wpt=2", "c32=1", "fat=1", "sort=0"]
AESC_ENV = [{}, {"SABA_AESC_FAT": "0"}, {"SABA_AESC_FAT16": "0"}, {"SABA_AESC_BITMAP": "0"},
            {"SABA_AESC_BITMAP": "1"}, {"SABA_AESC_WORKERS": "1"}, {"SABA_AESC_WORKERS": "2"},
            {"SABA_AESC_PRIO": "0"}, {"SABA_PULL_STATIC": "1"}, {"SABA_DEPTHS_PER_GRAPH": "2"},
            {"SABA_SHORT_STEPS": "0"}, {"SABA_SHORT_STEPS": "1000"},
            {"SABA_AESC_REC": "2"}, {"SABA_AESC_REC": "2", "SABA_SHORT_STEPS": "0"},
            {"SABA_PULL_SKIP": "0"}, {"SABA_PULL_SKIP": "1"}, {"SABA_PULL_SKIP": "1", "SABA_PULL_STATIC": "1"},
            {"SABA_AESC_HUB": "0"}, {"SABA_AESC_HUB": "300"}, {"SABA_AESC_HUB": "300", "SABA_AESC_WORKERS": "1"},
            {"SABA_AESC_HUB": "16000", "SABA_SHORT_STEPS": "0"},
            {"SABA_AESC_FAT": "0", "SABA_AESC_FAT16": "0", "SABA_AESC_REC": "0"},
            {"SABA_AESC_FAT": "0", "SABA_AESC_FAT16": "0", "SABA_AESC_REC": "0", "SABA_AESC_BITMAP": "1"}]


def run_variant(spec, env_extra, tmp_path, tag):
    out = str(tmp_path / f"{tag}.npz")
    env = dict(os.environ)
    for k in list(env):
        if k.startswith("SABA_") and k not in ("SABA_LIB",):
            del env[k]
    env.update(env_extra)
    r = subprocess.run([sys.executable, os.path.join(HERE, "variant_worker.py"), json.dumps(spec), out],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, f"{tag} {env_extra}: {r.stderr[-2000:]}"
    return dict(np.load(out))


def oracle_counts(sb, oracle, gspec, W, L, seed):
    sys.path.insert(0, HERE)
    from variant_worker import make_graph
    g = make_graph(gspec)
    kv = oracle.uniform_start_counts(g.n, W, seed)
    return g, oracle.campaign_counts(g.offsets, g.adjacency, length=L, master=seed, k_per_vertex=kv)


def test_campaign_variants_mid_graph(sb, oracle, tmp_path):
    W, L, seed = 1 << 20, 48, 9
    g, want = oracle_counts(sb, oracle, G_MID, W, L, seed)
    assert int(want.sum()) == W * L
    for i, v in enumerate(CAMPAIGN_MID):
        spec = {"kind": "campaign", "graph": G_MID, "W": W, "L": L, "seed": seed}
        got = run_variant(spec, {"SABA_WALK_VARIANT": v} if v else {}, tmp_path, f"mid{i}")["counts"]
        assert np.array_equal(got, want), v
    # sharded hub-counter kernel (the cfg2 default) and hash mode
    spec = {"kind": "campaign", "graph": G_MID, "W": W, "L": L, "seed": seed, "shards": 3}
    got = run_variant(spec, {"SABA_WALK_VARIANT": "fat=0,hot=1"}, tmp_path, "mid_sh")["counts"]
    assert np.array_equal(got, want)
    spec = {"kind": "campaign", "graph": G_MID, "W": W, "L": L, "seed": seed, "hash": True, "shards": 2}
    got = run_variant(spec, {"SABA_WALK_VARIANT": "fat=0,hot=1"}, tmp_path, "mid_hash")["counts"]
    assert np.array_equal(got, want)
    spec = {"kind": "campaign", "graph": G_MID, "W": W, "L": L, "seed": seed, "shards": 3}
    got = run_variant(spec, {"SABA_WALK_VARIANT": "fat=0,rec=1"}, tmp_path, "mid_rec_sh")["counts"]
    assert np.array_equal(got, want)


def test_campaign_16bit_counter_overflow(sb, oracle, tmp_path):
    """The 16-bit shared-memory counters (smem_count16) of the all-vertex fat
    kernel and of the rank kernel: a hub that takes about a quarter of all
    visits crosses 2^15 many times in every block, so the guard-bit spill to
    the global counter is exercised; counts stay bit-exact."""
    G = ["star", 3000]
    W, L, seed = 1 << 20, 48, 4
    g, want = oracle_counts(sb, oracle, G, W, L, seed)
    assert int(want[0]) > 148 * 65536  # every block's hub counter wraps its 15 bits more than once
    for i, v in enumerate(["", "priv=0", "fat=0,rec=1", "fat=0,rec=1,hrec=1,hcnt=1", "fat=0,rec=0,hot=1"]):
        spec = {"kind": "campaign", "graph": G, "W": W, "L": L, "seed": seed}
        got = run_variant(spec, {"SABA_WALK_VARIANT": v} if v else {}, tmp_path, f"star{i}")["counts"]
        assert np.array_equal(got, want), v


def test_campaign_per_vertex_sort_paths(sb, oracle, tmp_path):
    """K1's fused warp sort (K <= 256 per vertex), its run-wise form for larger
    K, and the CUB segmented sort give the same counts (order is a performance
    device only)."""
    G = ["rmat", 10, 8, 2]
    sys.path.insert(0, HERE)
    from variant_worker import make_graph
    g = make_graph(G)
    for K in (37, 600):
        want = oracle.campaign_counts(g.offsets, g.adjacency, K=K, length=11, master=8)
        for v in ("", "sort=0", "sort=1"):
            spec = {"kind": "campaign", "graph": G, "K": K, "L": 11, "seed": 8, "shards": 2 if v else 1}
            got = run_variant(spec, {"SABA_WALK_VARIANT": v} if v else {}, tmp_path, f"pv{K}{v}")["counts"]
            assert np.array_equal(got, want), (K, v)


def test_campaign_variants_beyond_packed_ids(sb, oracle, tmp_path):
    W, L, seed = 1 << 20, 32, 4
    g, want = oracle_counts(sb, oracle, G_BIG, W, L, seed)
    assert g.n > (1 << 21)
    for i, v in enumerate(CAMPAIGN_BIG):
        spec = {"kind": "campaign", "graph": G_BIG, "W": W, "L": L, "seed": seed,
                "shards": 2 if i % 2 else 1}
        got = run_variant(spec, {"SABA_WALK_VARIANT": v} if v else {}, tmp_path, f"big{i}")["counts"]
        assert np.array_equal(got, want), v


def _aesc_variants(sb, oracle, tmp_path, gspec, sources, eps, delta, tag):
    sys.path.insert(0, HERE)
    from variant_worker import make_graph
    g = make_graph(gspec)
    src = np.asarray(sources, np.uint32)
    ref = oracle.aesc(g.offsets, g.adjacency, epsilon=eps, delta=delta, sources=src)
    spec = {"kind": "aesc", "graph": gspec, "sources": [int(s) for s in src], "eps": eps, "delta": delta}
    base = None
    for i, env in enumerate(AESC_ENV):
        got = run_variant(spec, env, tmp_path, f"{tag}{i}")
        assert np.array_equal(got["tau_tilde"][src], ref.tau_tilde[src]), env
        assert int(got["stats"][0]) == ref.total_walk_pairs and int(got["stats"][1]) == ref.total_walk_steps, env
        err = np.abs(got["g_hat"] - ref.g_hat)
        assert np.all(err <= RTOL * np.abs(ref.g_hat) + ATOL), (env, float(np.max(err / (np.abs(ref.g_hat) + 1e-300))))
        if base is None:
            base = got["g_hat"]
        else:  # no switch changes a result bit
            assert np.array_equal(got["g_hat"], base), env
    return g


def test_aesc_variants_l2_resident(sb, oracle, tmp_path):
    g = sb.make_rmat(13, 8, seed=5)
    rng = np.random.default_rng(7)
    src = np.unique(rng.integers(0, g.n, 140))[:130]
    _aesc_variants(sb, oracle, tmp_path, A_MID, src, 0.2, 0.05, "amid")


def test_aesc_variants_short_walks_beyond_l2(sb, oracle, tmp_path):
    g = sb.make_chung_lu(300_000, 2.2, 24.0, 3000.0, seed=2)
    assert 16 * g.m > (48 << 20)  # the 16-byte record path is eligible
    deg = g.degrees()
    order = np.argsort(deg, kind="stable")
    src = np.unique(np.concatenate([order[:4], order[len(order) // 2: len(order) // 2 + 4], order[-4:]]))
    _aesc_variants(sb, oracle, tmp_path, A_SHORT, src, 0.1, 0.05, "ashort")
