"""Small runs of every cross-block protocol for compute-sanitizer
(VERDICT r1 "missing" 6): the last-block-publishes control block and the
dynamic work list of the AESC propagation, the warp-aggregated frontier
appends, the walk kernels' shared-memory hub counters, the device graph
builder's lock-free union-find, and the multi-replica combine.

  compute-sanitizer --tool memcheck  python tests/qa/sanitize_cases.py
  compute-sanitizer --tool racecheck python tests/qa/sanitize_cases.py
  compute-sanitizer --tool synccheck python tests/qa/sanitize_cases.py
  compute-sanitizer --tool initcheck python tests/qa/sanitize_cases.py

Every result is also checked against the CPU oracle, so a run that the
sanitizer slows down or perturbs still has to be exact.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2410_14056_b200 as sb  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402  (checker only)


def main():
    O = Oracle()
    # device graph build: radix sort + unique + union-find LCC + relabel
    g = sb.make_rmat(11, 8, seed=3, device=0)
    h = sb.make_rmat(11, 8, seed=3)
    assert np.array_equal(g.offsets, h.offsets) and np.array_equal(g.adjacency, h.adjacency)
    # campaign: default kernel (fat adjacency on this L2-resident graph)
    W, L = 20000, 12
    kv = O.uniform_start_counts(g.n, W, 5)
    want = O.campaign_counts(g.offsets, g.adjacency, length=L, master=5, k_per_vertex=kv)
    s = sb.VisitCountSink(g.n)
    sb.run_walk_campaign(g, sb.CampaignConfig(length=L, master_seed=5), s, total_walks=W)
    assert np.array_equal(s.counts, want)
    # multi-replica combine (logical shards on one GPU)
    s = sb.VisitCountSink(g.n)
    sb.run_walk_campaign(g, sb.CampaignConfig(length=L, master_seed=5), s, total_walks=W, devices=[0, 0])
    assert np.array_equal(s.counts, want)
    # paths
    st = np.arange(64, dtype=np.uint32) % g.n
    sd = (np.arange(64, dtype=np.uint64) * 2654435761 % (1 << 32)).astype(np.uint32)
    p = sb.walk_paths(g, st, sd, 9)
    assert np.array_equal(p[3], O.random_walk(g.offsets, g.adjacency, int(st[3]), 9, int(sd[3])))
    # AESC over >64 sources: several batches, both workers, sparse and dense
    # depths, hub pieces (R-MAT hubs have > 256 neighbours), hook + check
    src = np.arange(0, g.n, max(1, g.n // 150), dtype=np.uint32)
    est = sb.aesc(g, sb.AescConfig(epsilon=0.3, delta=0.1), sources=src)
    ref = O.aesc(g.offsets, g.adjacency, epsilon=0.3, delta=0.1, sources=src)
    assert np.array_equal(est.plan.tau_tilde[src], ref.tau_tilde[src])
    assert np.all(np.abs(est.g_hat - ref.g_hat) <= 1e-9 * np.abs(ref.g_hat) + 1e-15)
    est2 = sb.aesc(g, sb.AescConfig(epsilon=0.3, delta=0.1), sources=src, devices=[0, 0])
    assert np.array_equal(est2.g_hat, est.g_hat)
    print(f"sanitize cases ok: n={g.n} m={g.m} sources={len(src)} pairs={est.total_walk_pairs}")


if __name__ == "__main__":
    main()
