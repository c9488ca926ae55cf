"""Multi-device execution inside the library (SURVEY §8b threading, §8e).

The reference's results do not depend on its thread count
(test_walker.cpp:152-158, test_aesc.cpp:292-308, README.md:114-120); here
`threads` becomes a GPU count. One GPU is available to the tests, so the N>1
paths run as N logical shards — one replica and one host thread each — on the
same device (a device list with repeats), through the same code that shards
over distinct GPUs; only the combine differs (peer copies + add instead of the
NCCL reduce), and both are exact sums. Results must be bit-identical to one
device.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_campaign_device_lists_bit_identical(sb):
    g = sb.make_rmat(13, 8, seed=4)
    cfg = sb.CampaignConfig(length=24, master_seed=17)
    one = sb.VisitCountSink(g.n)
    rep1 = sb.run_walk_campaign(g, cfg, one, total_walks=300_000)
    for devs in ([0, 0], [0, 0, 0], [0, 0, 0, 0, 0]):
        s = sb.VisitCountSink(g.n)
        rep = sb.run_walk_campaign(g, cfg, s, total_walks=300_000, devices=devs)
        assert np.array_equal(s.counts, one.counts), devs
        assert rep.total_steps == rep1.total_steps and rep.shard_walks == 300_000
    # per-vertex campaign, and an outer shard split further over replicas
    cfg2 = sb.CampaignConfig(walks_per_vertex=7, length=9, master_seed=3)
    a = sb.VisitCountSink(g.n)
    sb.run_walk_campaign(g, cfg2, a)
    acc = np.zeros(g.n, np.uint64)
    for i in range(2):
        s = sb.VisitCountSink(g.n)
        sb.run_walk_campaign(g, cfg2, s, shard_index=i, shard_count=2, devices=[0, 0, 0])
        acc += s.counts
    assert np.array_equal(acc, a.counts)


def test_aesc_device_lists_bit_identical(sb):
    g = sb.make_rmat(12, 8, seed=6)
    cfg = sb.AescConfig(epsilon=0.15, delta=0.05)
    one = sb.aesc(g, cfg)
    assert one.replicas == 1
    for w in (1, 2):  # batch workers per device (AescConfig.workers): same bits
        ew = sb.aesc(g, sb.AescConfig(epsilon=0.15, delta=0.05, workers=w))
        assert ew.workers == w and np.array_equal(ew.g_hat, one.g_hat) and np.array_equal(ew.s_hat, one.s_hat)
        assert ew.walk_kernel_ms > 0
    for devs in ([0, 0], [0, 0, 0]):
        est = sb.aesc(g, cfg, devices=devs)
        assert est.replicas == len(devs)
        assert np.array_equal(est.g_hat, one.g_hat), devs
        assert np.array_equal(est.s_hat, one.s_hat), devs
        assert np.array_equal(est.plan.tau_tilde, one.plan.tau_tilde)
        assert est.total_walk_pairs == one.total_walk_pairs and est.total_walk_steps == one.total_walk_steps
        assert est.edge_visits == one.edge_visits > 0
    # a source subset over replicas, plus outer shards
    src = np.arange(3, g.n, 11, dtype=np.uint32)
    sub = sb.aesc(g, cfg, sources=src)
    acc = np.zeros_like(sub.g_hat)
    for i in range(3):
        acc += sb.aesc(g, cfg, sources=src, shard_index=i, shard_count=3, devices=[0, 0]).g_hat
    assert np.array_equal(acc, sub.g_hat)


def test_aesc_device_symmetrise_matches_host_api(sb):
    torch = pytest.importorskip("torch")
    g = sb.make_rmat(11, 8, seed=8)
    cfg = sb.AescConfig(epsilon=0.15, delta=0.05)
    ref = sb.aesc(g, cfg)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    total = torch.zeros(2 * g.m, dtype=torch.float64, device=dev)
    part = torch.empty(2 * g.m, dtype=torch.float64, device=dev)
    tt = np.zeros(g.n, np.uint32)
    for i in range(3):  # three "ranks", summed like an NCCL all-reduce
        est = sb.aesc_device(g, cfg, part.data_ptr(), stream.cuda_stream, shard_index=i, shard_count=3)
        total += part
        tt += est.plan.tau_tilde
    s_hat = torch.empty(g.m, dtype=torch.float64, device=dev)
    sb.symmetrise(g, total.data_ptr(), s_hat.data_ptr(), stream.cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(total.cpu().numpy(), ref.g_hat)
    assert np.array_equal(s_hat.cpu().numpy(), ref.s_hat)
    assert np.array_equal(tt, ref.plan.tau_tilde)


def test_repeated_sources_are_idempotent(sb, oracle):
    """a repeated source must not double its slots' estimates."""
    g = sb.make_rmat(11, 8, seed=2)
    cfg = sb.AescConfig(epsilon=0.15, delta=0.05)
    src = np.array([5, 9, 5, 100, 9, 9, 31], np.uint32)
    est = sb.aesc(g, cfg, sources=src)
    uniq = sb.aesc(g, cfg, sources=np.unique(src))
    assert np.array_equal(est.g_hat, uniq.g_hat)
    ref = oracle.aesc(g.offsets, g.adjacency, epsilon=0.15, delta=0.05, sources=np.unique(src))
    assert np.all(np.abs(est.g_hat - ref.g_hat) <= 1e-9 * np.abs(ref.g_hat) + 1e-15)
    assert est.total_walk_pairs == ref.total_walk_pairs


def test_device_campaign_across_streams_with_growing_workspace(sb):
    """a second asynchronous call on another stream with a larger
    configuration must not free workspaces the first call's kernels still use."""
    torch = pytest.importorskip("torch")
    g = sb.make_rmat(13, 8, seed=9)
    dev = torch.device("cuda", 0)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    small, big = 200_000, 3_000_000
    cfg = sb.CampaignConfig(length=40, master_seed=5)
    want_small, want_big = sb.VisitCountSink(g.n), sb.VisitCountSink(g.n)
    sb.run_walk_campaign(g, cfg, want_small, total_walks=small)
    sb.run_walk_campaign(g, cfg, want_big, total_walks=big)
    for _ in range(3):
        a = torch.zeros(g.n, dtype=torch.int64, device=dev)
        b = torch.zeros(g.n, dtype=torch.int64, device=dev)
        torch.cuda.synchronize()
        g.release_device()  # fresh handle: the big call must grow every workspace
        sb.run_walk_campaign_device(g, cfg, a.data_ptr(), s1.cuda_stream, total_walks=small)
        sb.run_walk_campaign_device(g, cfg, b.data_ptr(), s2.cuda_stream, total_walks=big)
        torch.cuda.synchronize()
        assert np.array_equal(a.cpu().numpy().astype(np.uint64), want_small.counts)
        assert np.array_equal(b.cpu().numpy().astype(np.uint64), want_big.counts)


def test_bench_two_ranks_gloo_on_one_gpu(oracle):
    """bench.py's world>1 branches: two torchrun ranks
    share the GPU through the gloo backend; the all-reduced counts must equal
    the oracle's for the doubled (weak-scaling) workload."""
    import json
    import os
    import socket
    import subprocess
    import sys

    from conftest import ROOT
    sys.path.insert(0, ROOT)
    import bench

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--workload", "cfg1", "--steps", "2", "--warmup", "1", "--dist-backend", "gloo",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["walks_total"] == 2 << 20
    off, adj = oracle.gen_erdos_renyi(65536, 524288, bench.GRAPH_SEED)
    kv = oracle.uniform_start_counts(len(off) - 1, 2 << 20, bench.MASTER_SEED)
    want = oracle.campaign_counts(off, adj, length=64, master=bench.MASTER_SEED, k_per_vertex=kv)
    assert line["checksum"]["counts_sha256_16"] == bench.counts_checksum(want)
