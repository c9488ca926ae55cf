"""One full-graph run of the compiled reference on BASELINE config 3 (every
one of the ~40K sources, OpenMP over all host cores: the reference's own
aesc(), aesc.hpp:636-708), then the GPU estimator on the same graph, compared
slot by slot: the full-graph parity check and the measured (not
extrapolated) CPU wall time.

Writes gpurun_out/aesc_cpu_full.json (copied to profiles/ by hand)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle.oracle import Reference  # noqa: E402

spec, eps, delta, _, _ = bench.AESC_WORKLOADS["cfg3"]
off, adj = bench.ref_graph(spec)
R = Reference()
rg = R.from_csr(off, adj)
t0 = time.time()
r = R.aesc(rg, epsilon=eps, delta=delta)
wall = time.time() - t0
print(f"reference full cfg3: {r.seconds:.1f} s (aesc() timer), wall {wall:.1f} s, cores {R.max_threads()}", flush=True)

import paper_2410_14056_b200 as sb  # noqa: E402  (after the CPU run: not loaded during it)
g = sb.make_rmat(16, 8, seed=1, device=0)
assert np.array_equal(g.offsets, off) and np.array_equal(g.adjacency, adj)
est = sb.aesc(g, sb.AescConfig(epsilon=eps, delta=delta))
err = np.abs(est.g_hat - r.g_hat)
nz = r.g_hat != 0
rel = err[nz] / np.abs(r.g_hat[nz])
serr = np.abs(est.s_hat - r.s_hat)
out = {"cfg3": {"seconds": r.seconds, "wall_seconds": wall, "cores": R.max_threads(), "kind": "reference",
                "what": "oracle/_ref aesc() on the full cfg3 graph, every source (OpenMP, all host cores)",
                "n": int(len(off) - 1), "m": int(len(adj) // 2), "lambda_hat": r.lambda_hat,
                "pairs": r.total_walk_pairs, "steps": r.total_walk_steps,
                "gpu_seconds": est.seconds, "gpu_pairs": est.total_walk_pairs,
                "tau_tilde_equal": bool(np.array_equal(est.plan.tau_tilde, r.tau_tilde)),
                "tau_equal": bool(np.array_equal(est.plan.tau, r.tau)),
                "pairs_equal": est.total_walk_pairs == r.total_walk_pairs,
                "steps_equal": est.total_walk_steps == r.total_walk_steps,
                "g_hat_worst_rel": float(rel.max()), "g_hat_worst_abs": float(err.max()),
                "s_hat_worst_abs": float(serr.max()),
                "s_hat_worst_rel": float((serr / np.abs(r.s_hat)).max()),
                "within_1e-9": bool(np.all(err <= 1e-9 * np.abs(r.g_hat) + 1e-15)),
                "srchash": bench.lib_build_hash()}}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "aesc_cpu_full.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
