"""Randomised campaign parity sweep (GPU, profiling/QA helper; not part of the
test suite): a fixed list of seeded cases — graph family, size, walks, length,
mode, shard count — is run by every K2 variant (one process per variant: the
library reads SABA_WALK_VARIANT once) and every variant's counts must equal
the CPU oracle's, bit for bit.

  python tests/qa/fuzz_campaign.py            # driver: spawns the variants, compares, prints a summary
  python tests/qa/fuzz_campaign.py --worker   # one variant (env SABA_WALK_VARIANT), JSON of count digests
"""
import argparse
import hashlib
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

VARIANTS = ["", "rec=0", "fat=0", "fat=0,rec=0", "fat=0,rec=0,hot=0", "priv=0", "fat=0,hrec=7,hcnt=13",
            "fat=0,hrec=0,hcnt=0", "fat=0,hthreads=512", "fat=0,c32=1", "fat=0,packed=0", "fat=0,rec=0,hcount=5"]


def cases(n_cases):
    rng = np.random.default_rng(20241021)
    out = []
    for i in range(n_cases):
        fam = ["rmat", "er", "star", "chunglu"][int(rng.integers(0, 4))]
        c = {"id": i, "fam": fam, "gseed": int(rng.integers(1, 1000)), "seed": int(rng.integers(1, 1 << 30)),
             "L": int(rng.integers(1, 70)), "hash": bool(rng.integers(0, 2)), "shards": int(rng.integers(1, 4))}
        if fam == "rmat":
            c["scale"] = int(rng.integers(7, 15))
            c["ef"] = int(rng.integers(2, 12))
        elif fam == "er":
            c["n"] = int(rng.integers(50, 40000))
            c["deg"] = int(rng.integers(3, 20))
        elif fam == "star":
            c["n"] = int(rng.integers(5, 5000))
        else:
            c["n"] = int(rng.integers(2000, 120000))
            c["mean"] = float(rng.uniform(4, 30))
        if rng.integers(0, 4) == 0:
            c["K"] = int(rng.integers(1, 40))  # per-vertex campaign
        else:
            c["W"] = int(rng.integers(100, 1_500_000))
        out.append(c)
    return out


def make_graph(sb, c):
    if c["fam"] == "rmat":
        return sb.make_rmat(c["scale"], c["ef"], seed=c["gseed"])
    if c["fam"] == "er":
        g = sb.make_erdos_renyi(c["n"], c["n"] * c["deg"] // 2, c["gseed"])
        # campaigns need degree >= 1 everywhere: add a ring
        a = np.arange(g.n, dtype=np.uint32)
        ring = np.stack([a, (a + 1) % g.n], 1)
        edges = []
        for v in range(g.n):
            nb = g.adjacency[g.offsets[v]:g.offsets[v + 1]]
            edges.append(np.stack([np.full(len(nb), v, np.uint32), nb], 1))
        return sb.Graph.from_edges(g.n, np.concatenate(edges + [ring]))
    if c["fam"] == "star":
        n = c["n"]
        a = np.arange(1, n, dtype=np.uint32)
        hub = np.stack([np.zeros(n - 1, np.uint32), a], 1)
        ring = np.stack([a, np.where(a + 1 < n, a + 1, 1).astype(np.uint32)], 1)
        return sb.Graph.from_edges(n, np.concatenate([hub, ring]))
    return sb.make_chung_lu(c["n"], 2.2, c["mean"], 2000.0, seed=c["gseed"])


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def worker(n_cases, use_oracle):
    import paper_2410_14056_b200 as sb
    res = {}
    O = None
    if use_oracle:
        from oracle.oracle import Oracle, Reference  # checkers only
        O = Oracle()
        R = Reference() if use_oracle == "ref" else None
    for c in cases(n_cases):
        g = make_graph(sb, c)
        if use_oracle:
            if R is not None:  # the reference headers compiled in place (oracle/_ref)
                rg = R.from_csr(g.offsets, g.adjacency)
                if "K" in c:
                    want = R.campaign(rg, c["K"], c["L"], master=c["seed"])[0]
                else:
                    want = R.campaign_kv(rg, c["L"], W=c["W"], master=c["seed"])[0]
            elif "K" in c:
                want = O.campaign_counts(g.offsets, g.adjacency, K=c["K"], length=c["L"], master=c["seed"])
            else:
                kv = O.uniform_start_counts(g.n, c["W"], c["seed"])
                want = O.campaign_counts(g.offsets, g.adjacency, length=c["L"], master=c["seed"], k_per_vertex=kv)
            res[str(c["id"])] = {"digest": digest(want), "n": int(g.n), "m": int(g.m)}
            continue
        cfg = sb.CampaignConfig(length=c["L"], master_seed=c["seed"],
                                mode=sb.WalkMode.Hash if c["hash"] else sb.WalkMode.Saba)
        if "K" in c:
            cfg.walks_per_vertex = c["K"]
        acc = np.zeros(g.n, np.uint64)
        kern = ""
        for i in range(c["shards"]):
            sink = sb.VisitCountSink(g.n)
            rep = sb.run_walk_campaign(g, cfg, sink, total_walks=c.get("W", 0), shard_index=i, shard_count=c["shards"])
            acc += sink.counts
            kern = rep.kernel
        res[str(c["id"])] = {"digest": digest(acc), "kernel": kern}
    print("FUZZ_JSON " + json.dumps(res))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worker", action="store_true")
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--checker", default="oracle", choices=["oracle", "ref"],
                    help="oracle = the C restatement, ref = the compiled reference (oracle/_ref)")
    ap.add_argument("--cases", type=int, default=40)
    a = ap.parse_args()
    if a.worker:
        worker(a.cases, a.checker if a.oracle else "")
        return

    def run(env_extra, extra):
        env = dict(os.environ)
        env.pop("SABA_WALK_VARIANT", None)
        env.update(env_extra)
        r = subprocess.run([sys.executable, __file__, "--worker", "--cases", str(a.cases)] + extra, env=env,
                           capture_output=True, text=True)
        if r.returncode != 0:
            print(r.stderr[-3000:])
            raise SystemExit(1)
        line = [x for x in r.stdout.splitlines() if x.startswith("FUZZ_JSON ")][-1]
        return json.loads(line[len("FUZZ_JSON "):])

    want = run({}, ["--oracle", "--checker", a.checker])
    bad = 0
    for v in VARIANTS:
        got = run({"SABA_WALK_VARIANT": v} if v else {}, [])
        kernels = {}
        for k, w in want.items():
            kernels[got[k]["kernel"]] = kernels.get(got[k]["kernel"], 0) + 1
            if got[k]["digest"] != w["digest"]:
                bad += 1
                print(f"MISMATCH variant [{v}] case {k}: {cases(a.cases)[int(k)]}")
        print(f"variant [{v}]: {len(want)} cases equal to the checker; kernels {kernels}")
    print("fuzz campaign:", "FAILED" if bad else "ok", f"({len(VARIANTS)} variants x {len(want)} cases, checker: "
          f"{'the compiled reference' if a.checker == 'ref' else 'the C oracle'})")
    raise SystemExit(1 if bad else 0)


if __name__ == "__main__":
    main()
