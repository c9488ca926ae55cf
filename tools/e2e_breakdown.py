"""Phase breakdown of the bench's e2e leg (cfg2): graph replica creation
(H2D + derived layouts), campaign (prep + walk + D2H), release."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_14056_b200 as sb  # noqa: E402

spec, walks, L = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
g = bench.make_graph(sb, spec, 0)
cfg = sb.CampaignConfig(length=L, master_seed=bench.MASTER_SEED)
ge = sb.Graph(torch.from_numpy(g.offsets).pin_memory().numpy(),
              torch.from_numpy(g.adjacency).pin_memory().numpy(), _trusted=True)
for i in range(6):
    t0 = time.perf_counter()
    ge.device_handle(0)
    t1 = time.perf_counter()
    sink = sb.VisitCountSink(g.n)
    rep = sb.run_walk_campaign(ge, cfg, sink, total_walks=walks)
    t2 = time.perf_counter()
    ge.release_device()
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):7.2f} ms  campaign {1e3*(t2-t1):7.2f} ms (device {1e3*rep.seconds:6.2f},"
          f" walk {rep.walk_kernel_ms:6.2f})  release {1e3*(t3-t2):6.2f} ms  total {1e3*(t3-t0):7.2f}")
