"""Run a few cfg-shaped campaigns for ncu (profiling helper; not a bench)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_14056_b200 as sb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--mode", default="saba")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
if a.workload == "cfg2":
    g, W, L = sb.make_rmat(20, 16, seed=1), 1 << 24, 128
else:
    g, W, L = sb.make_erdos_renyi(65536, 524288, 1), 1 << 20, 64
cfg = sb.CampaignConfig(length=L, master_seed=42,
                        mode=sb.WalkMode.Saba if a.mode == "saba" else sb.WalkMode.Hash)
counts = torch.zeros(g.n, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(a.reps):
    flush.zero_()
    counts.zero_()
    r = sb.run_walk_campaign_device(g, cfg, counts.data_ptr(), torch.cuda.current_stream().cuda_stream,
                                    total_walks=W, timing=True)
    print(f"walk_kernel_ms={r.walk_kernel_ms:.3f} total_ms={r.seconds*1e3:.3f}")
torch.cuda.synchronize()
assert int(counts.sum()) == W * L
