"""Graph ingest timing: Graph::from_edges and the BASELINE
generators on the device (csrc/graph_build.cu) vs the host builders and the
reference's own Graph::from_edges (oracle/_ref, std::sort, graph.hpp:86-105).
Every device result is checked equal to the host result before it is timed.

    python tests/qa/graph_build_bench.py > profiles/r01_graph_build.txt
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_2410_14056_b200 as sb  # noqa: E402


def timed(f, reps=2):
    best, out = float("inf"), None
    for _ in range(reps):
        t = time.perf_counter()
        out = f()
        best = min(best, time.perf_counter() - t)
    return best, out


def same(a, b):
    return np.array_equal(a.offsets, b.offsets) and np.array_equal(a.adjacency, b.adjacency)


def main():
    cores = os.cpu_count()
    # from_edges on cfg4-sized raw input: 67M pairs (R-MAT s22 ef16 sample count)
    # over 2^22 ids, ~3% self-loops and duplicates
    rng = np.random.default_rng(7)
    n, count = 1 << 22, 16 << 22
    pairs = rng.integers(0, n, size=(count, 2), dtype=np.uint32)
    pairs[::37, 1] = pairs[::37, 0]
    dup = pairs[1::29]
    dup[:] = pairs[0::29][: len(dup)]  # repeated pairs
    td, gd = timed(lambda: sb.Graph.from_edges(0, pairs, device=0))
    th, gh = timed(lambda: sb.Graph.from_edges(0, pairs), reps=1)
    assert same(gd, gh)
    row = {"what": "Graph::from_edges", "input": f"{count} pairs over {n} ids (loops, duplicates)",
           "n": gd.n, "m": gd.m, "device_s": round(td, 3), "host_s": round(th, 3), "host_cores": cores}
    try:
        from oracle.oracle import Reference, reference_available
        if reference_available():
            R = Reference()
            tr, _ = timed(lambda: R.from_edges(0, pairs), reps=1)
            row["reference_s"] = round(tr, 3)
            row["reference"] = "oracle/_ref Graph::from_edges (std::sort, 1 thread)"
    except Exception as e:  # the reference shim is optional here
        row["reference_error"] = str(e)
    print(json.dumps(row), flush=True)
    del pairs

    for name, f in [("cfg2 R-MAT s20 ef16 LCC", lambda d: sb.make_rmat(20, 16, seed=1, device=d)),
                    ("cfg4 R-MAT s22 ef16 LCC", lambda d: sb.make_rmat(22, 16, seed=1, device=d)),
                    ("cfg5 Chung-Lu n=3M LCC", lambda d: sb.make_chung_lu(3_000_000, seed=1, device=d))]:
        td, gd = timed(lambda: f(0))
        th, gh = timed(lambda: f(None), reps=1)
        assert same(gd, gh), name
        print(json.dumps({"what": "generator", "graph": name, "n": gd.n, "m": gd.m,
                          "device_s": round(td, 3), "host_s": round(th, 3), "host_cores": cores,
                          "identical_csr": True}), flush=True)


if __name__ == "__main__":
    main()
