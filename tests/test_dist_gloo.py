"""Multi-rank decomposition on CPU (gloo, world_size 2, 127.0.0.1).

The GPU path shards (a) campaigns by contiguous ranges of the flattened
(vertex, k) walk list and (b) AESC by cost-stratified sources
(saba_aesc_shard_sources: ascending degree, snake-dealt), then combines with
one all-reduce. Here each rank evaluates its shard with the CPU
oracle — the GPU kernels compute the same shards bit-exactly (see
test_walks_gpu / test_aesc_gpu) — and the combine runs through
torch.distributed exactly as bench.py does. The sums must equal the
unsharded results bit for bit.
"""
import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2410_14056_b200 as sb
    from oracle.oracle import Oracle

    O = Oracle()
    g = sb.make_rmat(11, 8, seed=9)
    # (a) campaign: uniform starts, contiguous walk-list ranges (campaign.cu)
    W, L = 40000, 12
    kv = O.uniform_start_counts(g.n, W, 42)
    r0, r1 = sb.campaign_shard_range(W, rank, world)
    part = O.campaign_range(g.offsets, g.adjacency, r0, r1, length=L, master=42, k_per_vertex=kv)
    t = torch.from_numpy(part.view(np.int64).copy())
    dist.all_reduce(t)
    # (b) AESC: cost-stratified source shards (aesc.cu shard_sources)
    src = np.arange(0, g.n, 7, dtype=np.uint32)
    mine = sb.aesc_shard_sources(g, src, rank, world)
    est = O.aesc(g.offsets, g.adjacency, epsilon=0.1, delta=0.01, sources=mine, threads=1)
    gh = torch.from_numpy(est.g_hat.copy())
    dist.all_reduce(gh)
    if rank == 0:
        np.save(os.path.join(out_dir, "counts.npy"), t.numpy().view(np.uint64))
        np.save(os.path.join(out_dir, "g_hat.npy"), gh.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_sum_to_unsharded(tmp_path, oracle, sb):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    g = sb.make_rmat(11, 8, seed=9)
    kv = oracle.uniform_start_counts(g.n, 40000, 42)
    full = oracle.campaign_counts(g.offsets, g.adjacency, length=12, master=42, k_per_vertex=kv)
    assert np.array_equal(np.load(tmp_path / "counts.npy"), full)
    src = np.arange(0, g.n, 7, dtype=np.uint32)
    ref = oracle.aesc(g.offsets, g.adjacency, epsilon=0.1, delta=0.01, sources=src, threads=1)
    assert np.array_equal(np.load(tmp_path / "g_hat.npy"), ref.g_hat)


def test_shard_helpers_partition(sb):
    for total in (1, 7, 1000, 16777216):
        for world in (1, 2, 3, 8):
            rs = [sb.campaign_shard_range(total, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
    g = sb.make_rmat(10, 8, seed=3)
    src = np.arange(0, g.n, 3, dtype=np.uint32)
    for world in (1, 2, 3, 8):
        parts = [sb.aesc_shard_sources(g, src, r, world) for r in range(world)]
        assert sorted(np.concatenate(parts).tolist()) == src.tolist()
        # cost-stratified: every shard's degree profile is the same up to one source per class
        if world > 1:
            sums = [int(g.degrees()[p].sum()) for p in parts]
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
            assert max(sums) - min(sums) <= 2 * int(g.degrees().max())
    # repeated sources run once (a repeat is idempotent in the reference's per-source loop)
    rep = np.array([5, 5, 9, 1, 9], np.uint32)
    assert sb.aesc_shard_sources(g, rep, 0, 1).tolist() == [1, 5, 9]
    everything = sum(len(sb.aesc_shard_sources(g, None, r, 4)) for r in range(4))
    assert everything == g.n
