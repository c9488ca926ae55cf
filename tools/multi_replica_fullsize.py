"""Full-size check of the in-library multi-device path on one GPU (QA helper):
the cfg2 campaign over 8 logical replicas (device list [0]*8: eight shards,
one combine) and the cfg3 AESC over 2 must reproduce the single-device
checksums bench.py prints (counts_sha256_16 / s_hat_sha256_16)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_14056_b200 as sb  # noqa: E402

spec, walks, L = bench.WORKLOADS["cfg2"]
g = bench.make_graph(sb, spec, 0)
cfg = sb.CampaignConfig(length=L, master_seed=bench.MASTER_SEED)
one = sb.VisitCountSink(g.n)
sb.run_walk_campaign(g, cfg, one, total_walks=walks)
for R in (2, 8):
    many = sb.VisitCountSink(g.n)
    t = time.time()
    rep = sb.run_walk_campaign(g, cfg, many, total_walks=walks, devices=[0] * R)
    print(f"cfg2 campaign, {R} logical replicas on one GPU: counts checksum {bench.counts_checksum(many.counts)} "
          f"(single device {bench.counts_checksum(one.counts)}), equal {bool((many.counts == one.counts).all())}, "
          f"{time.time() - t:.2f} s wall, kernel {rep.kernel}", flush=True)
    assert (many.counts == one.counts).all()

spec, eps, delta, _, _ = bench.AESC_WORKLOADS["cfg3"]
g3 = bench.make_graph(sb, spec, 0)
acfg = sb.AescConfig(epsilon=eps, delta=delta, threads=1)
e1 = sb.aesc(g3, acfg)
e2 = sb.aesc(g3, acfg, devices=[0, 0])
print(f"cfg3 AESC, 2 logical replicas on one GPU: s_hat checksum {bench.f64_checksum(e2.s_hat)} "
      f"(single device {bench.f64_checksum(e1.s_hat)}), bit-identical {bool((e2.s_hat == e1.s_hat).all())}, "
      f"tau~ equal {bool((e2.plan.tau_tilde == e1.plan.tau_tilde).all())}, pairs {e2.total_walk_pairs} == {e1.total_walk_pairs}",
      flush=True)
assert (e2.s_hat == e1.s_hat).all() and e2.total_walk_pairs == e1.total_walk_pairs
print("multi-replica full-size check ok")
