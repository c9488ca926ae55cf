"""bench.py's reference arm (the vs-reference ratio must be
creditable): it runs on the host only, loads oracle/ and never the product
library, runs the full workload, prints the same `config` as the GPU arm and
a checksum of the visit counts that equals the oracle's."""
import json
import os
import subprocess
import sys

import numpy as np

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_reference_arm_cfg1_full_workload(oracle):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                        "cfg1", "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                       env={**os.environ, "OMP_NUM_THREADS": "8"})
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "walk steps/sec (Bouquets)"
    off, adj = oracle.gen_erdos_renyi(65536, 524288, bench.GRAPH_SEED)
    assert line["config"] == bench.walk_config("cfg1", len(off) - 1, len(adj) // 2, 1, "nccl")
    W, L = bench.WORKLOADS["cfg1"][1:]
    kv = oracle.uniform_start_counts(len(off) - 1, W, bench.MASTER_SEED)
    want = oracle.campaign_counts(off, adj, length=L, master=bench.MASTER_SEED, k_per_vertex=kv)
    assert line["checksum"]["counts_sha256_16"] == bench.counts_checksum(want)
    assert line["checksum"]["total_visits"] == W * L
    assert line["e2e"]["value"] == line["value"] == line["cpu_baseline"]["value"]


def test_subset_permutation_matches_product_hash(sb):
    n = 5000
    keys = sb.counter_hash(bench.SUBSET_TAG, np.arange(n, dtype=np.uint64))
    assert np.array_equal(bench.subset_sources(n, 64), np.argsort(keys, kind="stable")[:64].astype(np.uint32))
