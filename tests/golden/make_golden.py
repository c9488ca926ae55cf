"""Regenerate tests/golden/golden.npz from the REFERENCE ITSELF.

Every vector here is produced by the unmodified reference headers
(/root/reference/proj/include/saba, compiled by oracle/Makefile into
oracle/_ref/libsaba_ref.so via oracle/ref_driver.cpp). The reference's own
test fixtures are reproduced by construction (graphs.hpp:15-60 named graphs,
gen.hpp generators with the seeds the reference tests use).

    python tests/golden/make_golden.py      # needs oracle/_ref (this container)
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference, build  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def named_edges():
    tri = [(0, 1), (1, 2), (0, 2)]
    path = lambda n: [(v, v + 1) for v in range(n - 1)]  # noqa: E731
    star = lambda k: [(0, v) for v in range(1, k + 1)]  # noqa: E731
    comp = lambda n: [(u, v) for u in range(n) for v in range(u + 1, n)]  # noqa: E731
    fig1 = [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)]
    grid = []
    for r in range(3):
        for c in range(3):
            v = 3 * r + c
            if c + 1 < 3:
                grid.append((v, v + 1))
            if r + 1 < 3:
                grid.append((v, v + 3))
    pet = []
    for i in range(5):
        pet += [(i, (i + 1) % 5), (i, i + 5), (5 + i, 5 + (i + 2) % 5)]
    return {"triangle": (3, tri), "P2": (2, path(2)), "P3": (3, path(3)), "P5": (5, path(5)),
            "P100": (100, path(100)), "S5": (6, star(5)), "K4": (4, comp(4)), "K9": (9, comp(9)),
            "K20": (20, comp(20)), "fig1": (4, fig1), "grid3x3": (9, grid), "petersen": (10, pet)}


def main():
    build(quiet=False)
    R = Reference()
    G = {}
    for name, (n, e) in named_edges().items():
        G[name] = R.from_edges(n, e)
    G["sf300_4_5"] = R.scale_free(300, 4, 5)
    G["sf400_5_21"] = R.scale_free(400, 5, 21)
    G["sf300_3_2"] = R.scale_free(300, 3, 2)
    G["sf2000_8_17"] = R.scale_free(2000, 8, 17)
    G["rc120_150_31"] = R.random_connected(120, 150, 31)
    G["rc40_30_13"] = R.random_connected(40, 30, 13)
    out = {}
    for name, g in G.items():
        off, adj, se = g.csr()
        out[f"g/{name}/off"] = off
        out[f"g/{name}/adj"] = adj
        out[f"g/{name}/slot_edge"] = se

    # walks: random_walk (walker.hpp:283) on sf300_4_5 / petersen
    rng = np.random.default_rng(7)
    for gname, L in (("sf300_4_5", 12), ("petersen", 6), ("sf2000_8_17", 33)):
        g = G[gname]
        starts = rng.integers(0, g.n, 64).astype(np.uint32)
        seeds = rng.integers(0, 2**32, 64, dtype=np.uint64).astype(np.uint32)
        paths = np.stack([R.random_walk(g, int(s), L, int(sd)) for s, sd in zip(starts, seeds)])
        out[f"walk/{gname}/starts"], out[f"walk/{gname}/seeds"] = starts, seeds
        out[f"walk/{gname}/paths"] = paths
    # random_bouquet (test_walker.cpp:78-88): start 7, L 12, width 8, master 99
    seeds, paths = R.random_bouquet(G["sf300_4_5"], 7, 12, 8, 99)
    out["bouquet/seeds"], out["bouquet/paths"] = seeds, paths

    # campaigns (run_walk_campaign, saba mode) — shapes from test_walker.cpp
    camp = [("sf400_5_21", 64, 7, 9), ("fig1", 13, 4, 42), ("sf2000_8_17", 32, 10, 17),
            ("petersen", 16, 6, 99), ("P2", 64, 5, 42)]
    for gname, K, L, seed in camp:
        c, _, steps = R.campaign(G[gname], K, L, mode=3, threads=4, master=seed)
        out[f"camp/{gname}/K{K}_L{L}_s{seed}"] = c
    # uniform-start campaign on sf2000_8_17 (the SURVEY §8d mapping)
    c, _, _ = R.campaign_kv(G["sf2000_8_17"], 16, W=32768, master=42, threads=4)
    out["ucamp/sf2000_8_17/W32768_L16_s42"] = c

    # branching statistics (test_walker.cpp:207-282 shapes)
    stats = [("P2", 64, 5, 3, 8, 42), ("K9", 4096, 2, 2, 8, 42), ("sf2000_8_17", 2048, 10, 3, 8, 42),
             ("sf2000_8_17", 2048, 10, 2, 8, 42), ("sf400_5_21", 64, 7, 3, 16, 9),
             ("sf400_5_21", 13, 7, 3, 8, 9)]
    for gname, K, L, mode, lanes, seed in stats:
        hist, step, total, samples, mdeg, mean = R.campaign_stats(G[gname], K, L, mode, lanes,
                                                                  threads=4, master=seed)
        key = f"stats/{gname}/K{K}_L{L}_m{mode}_b{lanes}_s{seed}"
        out[key + "/hist"], out[key + "/per_step"] = hist, step
        out[key + "/scalars"] = np.array([total, samples, mdeg, mean], np.float64)

    # rng_stream (test_stream.cpp:75-104 and variants)
    for gname, starts, K, L, sel, seed in (("petersen", [3], 16, 6, 2, 99), ("petersen", [3], 16, 6, 1, 99),
                                           ("fig1", [0, 1, 2], 3, 4, 2, 7),
                                           ("sf300_4_5", [5, 17, 250], 32, 8, 2, 7)):
        w = R.rng_stream(G[gname], starts, K, L, sel, seed)
        key = f"stream/{gname}/{'-'.join(map(str, starts))}/K{K}_L{L}_sel{sel}_s{seed}"
        out[key] = w

    # walk budget (test_aesc.cpp:27 and a grid)
    wb = []
    for t in (1, 5, 13, 97):
        for eps in (0.01, 0.05, 0.1):
            for d in (1, 4, 77):
                for m in (100, 477534):
                    wb.append((t, eps, 0.05, d, m, R.walk_budget(t, eps, 0.05, d, m)))
    out["walk_budget"] = np.array(wb, dtype=np.float64)

    # truncation plans (test_aesc.cpp:49-86)
    plans = [("petersen", 0.005, 30, 128, 0), ("petersen", 0.01, 30, 128, 0),
             ("petersen", 0.05, 30, 128, 0), ("petersen", 0.2, 30, 128, 0),
             ("K20", 0.05, 30, 128, 0), ("P100", 0.05, 60, 128, 0), ("triangle", 0.05, 40, 128, 0),
             ("P3", 0.05, 40, 128, 0), ("sf300_3_2", 0.05, 30, 128, 0),
             ("sf300_3_2", 0.05, 30, 128, 1), ("sf2000_8_17", 0.025, 30, 128, 0),
             ("grid3x3", 0.05, 30, 128, 0)]
    for i, (gname, eps, om, tmax, pe) in enumerate(plans):
        tau, lam, cl = R.truncated_lengths(G[gname], eps, om, tmax, bool(pe))
        out[f"plan/{i}/spec"] = np.array([eps, om, tmax, pe], np.float64)
        out[f"plan/{i}/graph"] = np.array(gname)
        out[f"plan/{i}/tau"] = tau
        out[f"plan/{i}/lambda"] = np.array([lam, float(cl)])

    # propagation (test_aesc.cpp:142-151 and a deeper one)
    for gname, src, eps, cap in (("fig1", 0, 0.025, -1), ("rc40_30_13", 7, 0.05, -1),
                                 ("sf300_4_5", 11, 0.1, -1), ("sf300_4_5", 3, 0.1, 2)):
        tau, _, _ = R.truncated_lengths(G[gname], eps / 2, 30)
        prob, depth = R.propagate(G[gname], src, tau, eps, 0.05, cap)
        key = f"prop/{gname}/{src}/{eps}/{cap}"
        out[key + "/prob"] = prob
        out[key + "/depth"] = np.array([depth])
        out[key + "/tau"] = tau

    # full aesc (test_aesc.cpp:183-318 shapes)
    runs = [
        ("triangle", dict(epsilon=0.05)), ("S5", dict(epsilon=0.05)), ("fig1", dict(epsilon=0.01)),
        ("fig1", dict(epsilon=0.05)), ("P3", dict(epsilon=0.05, switch_depth_cap=0)),
        ("fig1", dict(epsilon=0.05, max_truncation=5, switch_depth_cap=1, master_seed=20240917)),
        ("P5", dict(epsilon=0.05, max_truncation=5, switch_depth_cap=1, master_seed=20240917)),
        ("grid3x3", dict(epsilon=0.05, master_seed=7, switch_depth_cap=1, max_truncation=5)),
        ("petersen", dict(epsilon=0.05)), ("K4", dict(epsilon=0.05)), ("P5", dict(epsilon=0.05)),
        ("sf300_4_5", dict(epsilon=0.1)),
        ("sf300_4_5", dict(epsilon=0.1, switch_depth_cap=3, max_truncation=9)),
        ("rc120_150_31", dict(epsilon=0.1, delta=0.01)),
    ]
    for i, (gname, kw) in enumerate(runs):
        r = R.aesc(G[gname], threads=4, **kw)
        key = f"aesc/{i}"
        out[key + "/graph"] = np.array(gname)
        out[key + "/kw"] = np.array(repr(kw))
        out[key + "/g_hat"], out[key + "/s_hat"] = r.g_hat, r.s_hat
        out[key + "/tau"], out[key + "/tau_tilde"] = r.tau, r.tau_tilde
        out[key + "/stats"] = np.array([r.lambda_hat, r.total_walk_pairs, r.total_walk_steps],
                                       np.float64)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(out)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
