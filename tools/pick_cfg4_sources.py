"""Cheap non-hub cfg4 sources for the compiled-reference parity test: run the
GPU estimator on the first 256 sources of bench.py's permutation, then rank
the non-hub ones (degree <= 64, tau~ >= 2) by their walk work
sum_slots 2 * n_req(tau - tau~) * (tau - tau~) (aesc.hpp:103-110, 478-496)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_14056_b200 as sb  # noqa: E402

g = sb.make_rmat(22, 16, seed=1, device=0)
src = bench.subset_sources(g.n, 256)
cfg = sb.AescConfig(epsilon=0.05, delta=0.01)
est = sb.aesc(g, cfg, sources=src)
deg = g.degrees()
tau = int(est.plan.tau[0])
rows = []
for s in src:
    d, tt = int(deg[s]), int(est.plan.tau_tilde[s])
    if d > 64 or tt < 2 or tt >= tau:
        continue
    te = tau - tt
    steps = d * 2 * sb.walk_budget(te, 0.05, 0.01, d, g.m) * te
    rows.append((steps, int(s), d, tt))
rows.sort()
for r in rows[:12]:
    print(f"source {r[1]:8d} degree {r[2]:3d} tau~ {r[3]:3d} walk steps {r[0]:.3e}")
print("max degree", int(deg.max()), "tau", tau, "pairs(256)", est.total_walk_pairs)
