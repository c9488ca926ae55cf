"""Subprocess body of tests/test_variants_gpu.py.

The tuning switches (SABA_WALK_VARIANT, SABA_AESC_*, SABA_PULL_STATIC,
SABA_DEPTHS_PER_GRAPH) are read once per process by libsaba_cuda.so, so every
forced variant runs in its own interpreter: this script builds the named graph,
runs the GPU path and writes its outputs to an .npz for the parent test to
compare against the oracle. It never imports oracle/.

usage: python variant_worker.py <spec-json> <out.npz>
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2410_14056_b200 as sb  # noqa: E402


def make_graph(spec):
    kind = spec[0]
    if kind == "rmat":
        return sb.make_rmat(spec[1], spec[2], seed=spec[3])
    if kind == "chunglu":
        return sb.make_chung_lu(spec[1], 2.2, spec[2], spec[3], seed=spec[4])
    if kind == "ring":  # n > 2^21: the unpacked adjacency paths
        n, chords, seed = spec[1], spec[2], spec[3]
        rng = np.random.default_rng(seed)
        a = np.arange(n, dtype=np.uint32)
        ring = np.stack([a, (a + 1) % n], 1)
        extra = rng.integers(0, n, size=(chords, 2)).astype(np.uint32)
        return sb.Graph.from_edges(n, np.concatenate([ring, extra]))
    if kind == "star":  # one hub next to every vertex of a ring: its counter overflows 16 bits in every block
        n = spec[1]
        a = np.arange(1, n, dtype=np.uint32)
        hub = np.stack([np.zeros(n - 1, np.uint32), a], 1)
        ring = np.stack([a, np.where(a + 1 < n, a + 1, 1).astype(np.uint32)], 1)
        return sb.Graph.from_edges(n, np.concatenate([hub, ring]))
    raise ValueError(kind)


def main():
    spec = json.loads(sys.argv[1])
    out = sys.argv[2]
    g = make_graph(spec["graph"])
    res = {}
    if spec["kind"] == "campaign":
        cfg = sb.CampaignConfig(length=spec["L"], master_seed=spec["seed"],
                                mode=sb.WalkMode.Hash if spec.get("hash") else sb.WalkMode.Saba)
        parts = spec.get("shards", 1)
        acc = np.zeros(g.n, np.uint64)
        if spec.get("K"):  # per-vertex campaign (walker.hpp:456-538)
            cfg.walks_per_vertex = spec["K"]
        for i in range(parts):
            sink = sb.VisitCountSink(g.n)
            sb.run_walk_campaign(g, cfg, sink, total_walks=spec.get("W", 0), shard_index=i, shard_count=parts)
            acc += sink.counts
        res["counts"] = acc
    else:
        src = np.asarray(spec["sources"], np.uint32)
        est = sb.aesc(g, sb.AescConfig(epsilon=spec["eps"], delta=spec["delta"]), sources=src)
        res["g_hat"] = est.g_hat
        res["tau_tilde"] = est.plan.tau_tilde
        res["stats"] = np.array([est.total_walk_pairs, est.total_walk_steps], np.uint64)
    np.savez(out, **res)


if __name__ == "__main__":
    main()
