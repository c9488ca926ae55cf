"""Phase trace of one end-to-end cfg3 AESC call through the public API from a
pinned host CSR (the bench's e2e path): SABA_TRACE=1 python tools/e2e_trace_cfg3.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_14056_b200 as sb  # noqa: E402

g = sb.make_rmat(16, 8, seed=1, device=0)
ge = sb.Graph(torch.from_numpy(g.offsets).pin_memory().numpy(),
              torch.from_numpy(g.adjacency).pin_memory().numpy(), _trusted=True)
cfg = sb.AescConfig(epsilon=0.1, delta=0.01)
for i in range(3):
    t = time.perf_counter()
    est = sb.aesc(ge, cfg)
    ge.release_device()
    print(f"e2e call {i}: {time.perf_counter() - t:.3f} s (est.seconds {est.seconds:.3f})", file=sys.stderr,
          flush=True)
