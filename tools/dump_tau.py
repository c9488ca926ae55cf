"""Dump tau~ of every cfg3 source (batch-efficiency analysis of propagation)."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_14056_b200 as sb  # noqa: E402
g = sb.make_rmat(16, 8, seed=1)
est = sb.aesc(g, sb.AescConfig(epsilon=0.1, delta=0.01))
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/tau_cfg3.npz", tau_tilde=est.plan.tau_tilde, deg=np.diff(g.offsets))
print("saved", est.seconds)
