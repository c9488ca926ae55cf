"""Run the GPU AESC estimator on a BASELINE AESC config (profiling / timing
helper; bench.py --workload cfg3|cfg4|cfg5 is the reported measurement)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2410_14056_b200 as sb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--sources", type=int, default=0, help="0 = all")
ap.add_argument("--reps", type=int, default=2, help="timed runs; the last one is reported")
a = ap.parse_args()
t = time.time()
if a.workload == "cfg3":
    g, eps, delta = sb.make_rmat(16, 8, seed=1), 0.1, 0.01
elif a.workload == "cfg4":
    g, eps, delta = sb.make_rmat(22, 16, seed=1), 0.05, 0.01
else:
    g, eps, delta = sb.make_chung_lu(3_000_000, 2.2, 78.0, 30000.0, seed=1), 0.01, 0.01
print(f"graph {a.workload}: n={g.n} m={g.m} dmax={g.max_degree()} built in {time.time()-t:.1f}s",
      flush=True)
src = None
if a.sources:
    perm = np.argsort(sb.counter_hash(0x5355425345, np.arange(g.n, dtype=np.uint64)), kind="stable")
    src = np.sort(perm[: a.sources]).astype(np.uint32)
cfg = sb.AescConfig(epsilon=eps, delta=delta)
for _ in range(a.reps):
    t = time.time()
    est = sb.aesc(g, cfg, sources=src)
    wall = time.time() - t
tt = est.plan.tau_tilde if src is None else est.plan.tau_tilde[src]
print(f"aesc: wall {wall:.2f}s est.seconds {est.seconds:.2f}s plan {est.plan_seconds:.2f}s "
      f"prop {est.propagation_ms/1e3:.2f}s walk {est.walk_ms/1e3:.2f}s lambda {est.plan.lambda_hat:.4f} "
      f"tau {est.plan.max_tau} tau~[min/med/max] {tt.min()}/{int(np.median(tt))}/{tt.max()} "
      f"pairs {est.total_walk_pairs:.3e} steps {est.total_walk_steps:.3e} "
      f"-> {est.total_walk_steps/max(est.walk_ms*1e-3,1e-9):.3e} walk steps/s launches {est.launches}",
      flush=True)
import json  # noqa: E402
print("AESC_JSON " + json.dumps({"workload": a.workload, "sources": int(a.sources), "walk_steps": est.total_walk_steps,
                                 "walk_pairs": est.total_walk_pairs, "edge_visits": est.edge_visits,
                                 "propagation_ms": est.propagation_ms, "walk_ms": est.walk_ms, "wall_s": wall}),
      flush=True)
