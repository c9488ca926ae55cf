"""Randomised AESC parity sweep (GPU, QA helper; not part of the test suite):
seeded small cases — graph family and size, epsilon, delta, per-edge tau,
switch-depth cap, source subset or the whole graph — under a few library
switches (one process each) against the CPU oracle: tau~ and pair / step
counts equal, g_hat (and s_hat for whole-graph runs) within 1e-9 relative.

  python tests/qa/fuzz_aesc.py              # driver
  python tests/qa/fuzz_aesc.py --worker     # one switch set (from the environment)
"""
import argparse
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

RTOL, ATOL = 1e-9, 1e-15
ENVS = [{}, {"SABA_AESC_WORKERS": "1"}, {"SABA_AESC_FAT": "0"}, {"SABA_AESC_HUB": "500"},
        {"SABA_AESC_BITMAP": "1"}, {"SABA_SHORT_STEPS": "0"}, {"SABA_PULL_SKIP": "1"},
        {"SABA_AESC_FAT": "0", "SABA_AESC_FAT16": "0"}]


def cases(n_cases):
    rng = np.random.default_rng(7102024)
    out = []
    for i in range(n_cases):
        fam = ["rmat", "sf", "star", "chunglu"][int(rng.integers(0, 4))]
        c = {"id": i, "fam": fam, "gseed": int(rng.integers(1, 1000)), "seed": int(rng.integers(1, 1 << 30)),
             "eps": float(rng.choice([0.5, 0.3, 0.2])), "delta": float(rng.choice([0.1, 0.01])),
             "per_edge": bool(rng.integers(0, 2)), "cap": int(rng.choice([-1, -1, 0, 2, 5]))}
        if fam == "rmat":
            c["scale"] = int(rng.integers(6, 11))
            c["ef"] = int(rng.integers(3, 10))
        elif fam == "sf":
            c["n"] = int(rng.integers(30, 1500))
            c["k"] = int(rng.integers(2, 6))
        elif fam == "star":
            c["n"] = int(rng.integers(5, 400))
        else:
            c["n"] = int(rng.integers(500, 4000))
            c["mean"] = float(rng.uniform(4, 16))
        c["nsrc"] = int(rng.choice([0, 3, 70, 150]))  # 0 = whole graph (s_hat too)
        out.append(c)
    return out


def make_graph(sb, c):
    if c["fam"] == "rmat":
        return sb.make_rmat(c["scale"], c["ef"], seed=c["gseed"])
    if c["fam"] == "sf":
        return sb.make_scale_free(c["n"], c["k"], c["gseed"])
    if c["fam"] == "star":
        n = c["n"]
        a = np.arange(1, n, dtype=np.uint32)
        hub = np.stack([np.zeros(n - 1, np.uint32), a], 1)
        ring = np.stack([a, np.where(a + 1 < n, a + 1, 1).astype(np.uint32)], 1)
        return sb.Graph.from_edges(n, np.concatenate([hub, ring]))
    return sb.make_chung_lu(c["n"], 2.2, c["mean"], 300.0, seed=c["gseed"])


def sources_of(c, n):
    if c["nsrc"] == 0:
        return None
    rng = np.random.default_rng(c["seed"])
    return np.sort(rng.choice(n, size=min(n, c["nsrc"]), replace=False)).astype(np.uint32)


def worker(n_cases, use_oracle, out_path):
    import paper_2410_14056_b200 as sb
    res = {}
    O = None
    if use_oracle:
        from oracle.oracle import Oracle, Reference  # checkers only
        O = Oracle()
        R = Reference() if use_oracle == "ref" else None
    for c in cases(n_cases):
        g = make_graph(sb, c)
        src = sources_of(c, g.n)
        if use_oracle:
            try:
                if R is not None:  # the reference headers compiled in place (oracle/_ref)
                    r = R.aesc(R.from_csr(g.offsets, g.adjacency), epsilon=c["eps"], delta=c["delta"],
                               master_seed=c["seed"], per_edge_tau=c["per_edge"], switch_depth_cap=c["cap"],
                               sources=src)
                else:
                    r = O.aesc(g.offsets, g.adjacency, epsilon=c["eps"], delta=c["delta"], master_seed=c["seed"],
                               per_edge_tau=c["per_edge"], switch_depth_cap=c["cap"], sources=src)
            except (ValueError, RuntimeError) as e:  # e.g. a walk budget beyond 2^63 (aesc.hpp:117-126)
                res[f"e{c['id']}"] = np.array([1 if isinstance(e, ValueError) else 2])
                continue
            res[f"g{c['id']}"] = r.g_hat
            if r.s_hat is not None:
                res[f"s{c['id']}"] = r.s_hat
            res[f"t{c['id']}"] = r.tau_tilde
            res[f"c{c['id']}"] = np.array([r.total_walk_pairs, r.total_walk_steps], np.uint64)
            continue
        cfg = sb.AescConfig(epsilon=c["eps"], delta=c["delta"], master_seed=c["seed"],
                            per_edge_tau=c["per_edge"], switch_depth_cap=c["cap"])
        try:
            e = sb.aesc(g, cfg, sources=src)
        except (ValueError, RuntimeError) as x:
            res[f"e{c['id']}"] = np.array([1 if isinstance(x, ValueError) else 2])
            continue
        res[f"g{c['id']}"] = e.g_hat
        if src is None:
            res[f"s{c['id']}"] = e.s_hat
        res[f"t{c['id']}"] = e.plan.tau_tilde
        res[f"c{c['id']}"] = np.array([e.total_walk_pairs, e.total_walk_steps], np.uint64)
    np.savez(out_path, **res)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worker", action="store_true")
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--checker", default="oracle", choices=["oracle", "ref"],
                    help="oracle = the C restatement, ref = the compiled reference (oracle/_ref)")
    ap.add_argument("--cases", type=int, default=30)
    ap.add_argument("--out", default="/tmp/fuzz_aesc.npz")
    a = ap.parse_args()
    if a.worker:
        worker(a.cases, a.checker if a.oracle else "", a.out)
        return

    def run(env_extra, extra, tag):
        env = {k: v for k, v in os.environ.items() if not (k.startswith("SABA_") and k != "SABA_LIB")}
        env.update(env_extra)
        out = f"/tmp/fuzz_aesc_{tag}.npz"
        r = subprocess.run([sys.executable, __file__, "--worker", "--cases", str(a.cases), "--out", out] + extra,
                           env=env, capture_output=True, text=True)
        if r.returncode != 0:
            print(r.stderr[-3000:])
            raise SystemExit(1)
        return dict(np.load(out))

    want = run({}, ["--oracle", "--checker", a.checker], "oracle")
    cs = cases(a.cases)
    bad = 0
    for i, envx in enumerate(ENVS):
        got = run(envx, [], f"v{i}")
        worst = 0.0
        for c in cs:
            k = c["id"]
            if f"e{k}" in want or f"e{k}" in got:  # both must fail, with the same exception class
                if not (f"e{k}" in want and f"e{k}" in got and np.array_equal(want[f"e{k}"], got[f"e{k}"])):
                    bad += 1
                    print(f"MISMATCH (error behaviour) env {envx} case {c}")
                continue
            ok = np.array_equal(got[f"c{k}"], want[f"c{k}"])
            tg, tw = got[f"t{k}"], want[f"t{k}"]
            if c["nsrc"]:
                nz = np.flatnonzero(tw)
                ok = ok and np.array_equal(tg[nz], tw[nz])
            else:
                ok = ok and np.array_equal(tg, tw)
            for key in (f"g{k}", f"s{k}"):
                if key in want:
                    d = np.abs(got[key] - want[key])
                    ok = ok and bool(np.all(d <= RTOL * np.abs(want[key]) + ATOL))
                    nzv = np.abs(want[key]) > 1e-12  # below that the absolute term of the tolerance decides
                    if nzv.any():
                        worst = max(worst, float((d[nzv] / np.abs(want[key][nzv])).max()))
            if not ok:
                bad += 1
                print(f"MISMATCH env {envx} case {c}")
        print(f"env {envx}: {len(cs)} cases within 1e-9 of the checker (counts and tau~ equal); worst rel {worst:.2e} over |ref| > 1e-12")
    nerr = sum(1 for k in want if k.startswith("e"))
    print("fuzz aesc:", "FAILED" if bad else "ok", f"({len(ENVS)} switch sets x {len(cs)} cases, {nerr} of them "
          f"rejected alike by the checker and the GPU path; checker: "
          f"{'the compiled reference' if a.checker == 'ref' else 'the C oracle'})")
    raise SystemExit(1 if bad else 0)


if __name__ == "__main__":
    main()
