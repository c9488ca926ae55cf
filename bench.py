#!/usr/bin/env python3
"""Bouquets walk-campaign and TGT+ AESC benchmark (BASELINE.json metric
"walk steps/sec (Bouquets) and TGT+ all-edges SC wall time").

Default (N=1, BASELINE configs[1]): R-MAT a,b,c = 0.57,0.19,0.19, scale 20,
edge factor 16, symmetrised/deduplicated/loop-free, largest connected
component; 16,777,216 walks of length 128 from uniform-random starts, Saba
(seed-sorted bouquets), uint64 per-vertex visit counts. A "step" of this
benchmark is one whole campaign; the metric counts walk steps (L-1 per walk),
as the reference does (walker.hpp:523, bench.hpp:166-168). The default line
also carries `aesc_cfg3`: the second BASELINE metric (TGT+ all-edges SC wall
time, configs[2], every source) with its own roofline, e2e, cpu_baseline and
clocks.

Multi-GPU (torchrun, one rank per GPU): weak scaling — N x 16,777,216 walks,
the flattened (vertex, k) walk list cut into N contiguous ranges (one per
rank), CSR replicated, one all-reduce of the int64 counts (NCCL; or gloo with
--dist-backend gloo, which also lets N ranks share one GPU for testing).

--impl reference: the reference's own CPU implementation (oracle/_ref: the
reference headers compiled unchanged, OpenMP over all host threads) on the
SAME workload (every walk), rank 0 only. That process loads only oracle/
(the graph comes from oracle_gen.c, the BASELINE generators restated in C and
pinned bit-for-bit to the product's), prints the same `config`, and both arms
print a checksum of the visit counts so cross-arm parity is visible.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (generator spec, walks per GPU, length)
    "cfg2": (("rmat", 20, 16), 1 << 24, 128),
    "cfg1": (("er", 65536, 524288), 1 << 20, 64),
}
AESC_WORKLOADS = {
    # name: (graph spec, epsilon, delta, sources per GPU (0 = all), CPU sample sources)
    "cfg3": (("rmat", 16, 8), 0.1, 0.01, 0, 64),
    "cfg4": (("rmat", 22, 16), 0.05, 0.01, 512, 16),
    "cfg5": (("chunglu", 3_000_000), 0.01, 0.01, 8192, 64),
}
BYTES_PER_STEP = 64       # one 32 B sector for {base,deg} + one for adj[base+idx]
BYTES_PER_EDGE_VISIT = 12  # propagation: 4 B adjacency + 8 B p/d per edge-visit
MASTER_SEED = 42
GRAPH_SEED = 1
SUBSET_TAG = 0x5355425345  # "SUBSE": fixed source permutation of the subset protocol


# ----------------------------------------------------------------- shared

def gen_desc(spec):
    if spec[0] == "rmat":
        return f"R-MAT(0.57,0.19,0.19) scale {spec[1]} ef {spec[2]} LCC"
    if spec[0] == "er":
        return f"Erdos-Renyi G(n={spec[1]}, m={spec[2]})"
    return f"Chung-Lu n={spec[1]} gamma 2.2 mean 78 cap 30000 LCC"


def walk_config(name, n, m, world, backend):
    """The `config` both arms print (identical by construction)."""
    spec, walks, L = WORKLOADS[name]
    return {"workload": f"{name}: {gen_desc(spec)} (n={n}, m={m}); {walks} uniform-start walks x L={L} per GPU",
            "mode": "saba", "lanes": 8, "master_seed": MASTER_SEED, "graph_seed": GRAPH_SEED,
            "walks_total": walks * world, "length": L,
            "parallelism": f"walk-range shards x{world}, CSR replicated, {backend} all-reduce of counts",
            "l2": "flushed between timed steps (256 MiB write, outside the events)"}


def aesc_config(name, n, m, world, label):
    spec, eps, delta, _, _ = AESC_WORKLOADS[name]
    return {"workload": f"{name}: {gen_desc(spec)} (n={n}, m={m}) eps={eps} delta={delta}",
            "sources": label, "master_seed": MASTER_SEED, "graph_seed": GRAPH_SEED,
            "parallelism": f"cost-stratified source shards x{world}, CSR replicated, all-reduce of g_hat"}


def counts_checksum(counts) -> str:
    return hashlib.sha256(np.ascontiguousarray(counts, "<u8").tobytes()).hexdigest()[:16]


def f64_checksum(x) -> str:
    return hashlib.sha256(np.ascontiguousarray(x, "<f8").tobytes()).hexdigest()[:16]


def subset_sources(n, count):
    """First `count` vertices of a fixed counter_hash permutation.
    counter_hash(m, i) = mix64(m + (i+1) * 0x9e3779b97f4a7c15) (common.hpp:24-36)
    in numpy, so both arms compute it without either library."""
    idx = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(SUBSET_TAG) + (idx + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        keys = z ^ (z >> np.uint64(31))
    return np.argsort(keys, kind="stable")[:count].astype(np.uint32)


def read_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def lib_build_hash():
    try:
        with open(os.path.join(ROOT, "paper_2410_14056_b200", "libsaba_cuda.so.srchash")) as f:
            return f.read().strip()
    except OSError:
        return None


def read_profile_json(name, key):
    """Per-config ncu figures recorded under profiles/ (with the source hash
    of the build they were captured on)."""
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            d = json.load(f)
    except Exception:
        return None
    e = d.get(key)
    if isinstance(e, dict):
        e = dict(e)
        e["same_build"] = e.get("srchash") is not None and e.get("srchash") == lib_build_hash()
    return e


# L2-resident random-sector ceiling measured on this pool's B200 by
# tools/gather_ceiling.cu (profiles/r01_gather_ceiling.txt): 2.84e11 random
# 4 B gathers/s at a 32 MB working set = 9,083 GB/s in 32 B sectors.
L2_RANDOM_SECTOR_GBS = 9082.8


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed
    region by an NVML thread every 5 ms (nvidia-smi's own startup is longer
    than a short timed region)."""

    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
             ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, device, period=0.005):
        self.device, self.period = device, period
        self.rows, self.max_mhz, self.err = [], None, None
        self._stop = None
        self._thr = None

    def _run(self, nv, h):
        reasons_fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = reasons_fn(h)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                self.rows.append((sm, rs, pw))
            except Exception as e:  # noqa: BLE001
                self.err = str(e)
            self._stop.wait(self.period)

    def __enter__(self):
        import threading
        try:
            import pynvml as nv
            nv.nvmlInit()
            idx = self.device
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis and vis.split(",")[0].strip().isdigit():
                idx = int(vis.split(",")[self.device].strip())
            h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self._nv = nv
            self._stop = threading.Event()
            self._thr = threading.Thread(target=self._run, args=(nv, h), daemon=True)
            self._thr.start()
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml unavailable: {e}"
        return self

    def __exit__(self, *a):
        if self._thr:
            self._stop.set()
            self._thr.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"],
                    "samples": 0, "error": self.err}
        nv = self._nv
        sm = [r[0] for r in self.rows]
        reasons = sorted({name for _, rs, _ in self.rows for name, attr in self.NAMES
                          if rs & getattr(nv, attr, 0)})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "sm_mhz_min": min(sm),
                "power_w_max": max(r[2] for r in self.rows), "source": "nvml, 5 ms"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return int(os.environ.get("RANK", "0")), ws, int(os.environ.get("LOCAL_RANK", "0"))


# ---------------------------------------------------------- reference arm
# Loads oracle/ only (no product library): graphs from oracle_gen.c, the
# reference's own walk / AESC code from oracle/_ref.

def ref_graph(spec):
    from oracle.oracle import Oracle
    O = Oracle()
    if spec[0] == "rmat":
        return O.gen_rmat(spec[1], spec[2], 0.57, 0.19, 0.19, seed=GRAPH_SEED, keep_lcc=True)
    if spec[0] == "er":
        return O.gen_erdos_renyi(spec[1], spec[2], GRAPH_SEED)
    return O.gen_chung_lu(spec[1], 2.2, 78.0, 30000.0, seed=GRAPH_SEED, keep_lcc=True)


def reference_lib():
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        from oracle.oracle import build
        build()
    return Reference()


def cpu_campaign(R, rg, walks, L, threads=0):
    """One full campaign of the workload through the reference
    (campaign_vertex_scaled per start vertex, walker.hpp:430-449, OpenMP)."""
    counts, sec, steps = R.campaign_kv(rg, L, W=walks, sorted_=True, lanes=8, threads=threads,
                                       master=MASTER_SEED, vertex_stride=1, vertex_phase=0)
    return counts, sec, steps


def cpu_aesc_sample(R, off, adj, n, eps, delta, cpu_sources):
    """oracle/_ref aesc_source over the first `cpu_sources` sources of the
    subset permutation (OpenMP over sources), extrapolated to every source."""
    rg = R.from_csr(off, adj)
    cs = subset_sources(n, cpu_sources)
    r = R.aesc(rg, epsilon=eps, delta=delta, sources=cs)
    return {"value": r.seconds * n / cpu_sources + r.plan_seconds, "unit": "s",
            "cores": R.max_threads(), "kind": "reference",
            "sample": f"oracle/_ref aesc_source over {cpu_sources} sources of the fixed permutation "
                      f"({r.seconds:.2f} s + plan {r.plan_seconds:.2f} s), extrapolated x{n / cpu_sources:.1f}"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    spec, walks, L = WORKLOADS[args.workload]
    off, adj = ref_graph(spec)
    n, m = len(off) - 1, len(adj) // 2
    R = reference_lib()
    rg = R.from_csr(off, adj)
    total = walks * world
    secs, counts = [], None
    for i in range(args.warmup + args.steps):
        counts, sec, steps = cpu_campaign(R, rg, total, L)
        assert steps == total * (L - 1)
        if i >= args.warmup:
            secs.append(sec)
    ms = 1e3 * sum(secs) / len(secs)
    value = total * (L - 1) / (ms * 1e-3)
    cores = R.max_threads()
    out = {"impl": "reference", "metric": "walk steps/sec (Bouquets)", "value": value,
           "unit": "steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "u32", "data": "synthetic",
           "config": walk_config(args.workload, n, m, world, args.dist_backend),
           "checksum": {"counts_sha256_16": counts_checksum(counts), "total_visits": int(counts.sum())},
           "cpu_baseline": {"value": value, "unit": "steps/s", "cores": cores, "kind": "reference",
                            "sample": f"the full workload every step ({total} walks x L={L}; "
                                      "campaign_vertex_scaled per start vertex, the reference's own timer)"},
           "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    assert "paper_2410_14056_b200" not in sys.modules, "the reference arm must not load the product"
    if args.workload == "cfg2" and world == 1 and not args.no_aesc:
        spec3, eps, delta, _, cpu_sources = AESC_WORKLOADS["cfg3"]
        o3, a3 = ref_graph(spec3)
        out["aesc_cfg3"] = {"cpu_baseline": cpu_aesc_sample(R, o3, a3, len(o3) - 1, eps, delta, cpu_sources)}
    print(json.dumps(out))


def run_aesc_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    spec, eps, delta, per_gpu, cpu_sources = AESC_WORKLOADS[args.workload]
    off, adj = ref_graph(spec)
    n, m = len(off) - 1, len(adj) // 2
    R = reference_lib()
    cpu = cpu_aesc_sample(R, off, adj, n, eps, delta, cpu_sources)
    label = f"all {n} sources" if not per_gpu else \
        f"{per_gpu * world} sources of {n} (fixed permutation), extrapolated x{n / (per_gpu * world):.1f}"
    print(json.dumps({
        "impl": "reference", "metric": "TGT+ all-edges SC wall time", "value": cpu["value"],
        "unit": "s", "n_gpus": world, "steps": 1, "warmup": 0, "ms_per_step": cpu["value"] * 1e3,
        "higher_is_better": False, "scaling": "weak" if per_gpu else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": aesc_config(args.workload, n, m, world, label),
        "cpu_baseline": cpu,
        "e2e": {"value": cpu["value"], "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


# --------------------------------------------------------------- our arm

def init_dist(args, local):
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    ndev = torch.cuda.device_count()
    dev_index = local % max(ndev, 1)  # gloo mode may put several ranks on one GPU
    torch.cuda.set_device(dev_index)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group("gloo")
    return dev_index


def all_reduce(t, args, op=None):
    """Sum (or op) across ranks: on the device with NCCL, via host with gloo."""
    import torch.distributed as dist
    op = op or dist.ReduceOp.SUM
    if args.dist_backend == "nccl" or t.device.type == "cpu":
        dist.all_reduce(t, op=op)
        return t
    h = t.cpu()
    dist.all_reduce(h, op=op)
    t.copy_(h)
    return t


def make_graph(sb, spec, device):
    if spec[0] == "rmat":
        return sb.make_rmat(spec[1], spec[2], 0.57, 0.19, 0.19, seed=GRAPH_SEED, keep_lcc=True, device=device)
    if spec[0] == "er":
        return sb.make_erdos_renyi(spec[1], spec[2], GRAPH_SEED)
    return sb.make_chung_lu(spec[1], 2.2, 78.0, 30000.0, seed=GRAPH_SEED, keep_lcc=True, device=device)


K2_DESCR = {
    "walk_count_rank_kernel": "walk_count_rank_kernel (degree-ranked records, packed rank adjacency; the top "
                              "records and 16-bit visit counters in shared memory)",
    "walk_count_hot_kernel": "walk_count_hot_kernel (packed adjacency, shared-memory hub counters)",
    "walk_count_fat_priv_kernel": "walk_count_fat_priv_kernel (one fat gather per step; every vertex's 16-bit "
                                  "counter in shared memory)",
    "walk_count_fat_kernel": "walk_count_fat_kernel (one fat gather per step, L2 reductions)",
    "walk_count_kernel": "walk_count_kernel (csr + neighbour gathers, L2 reductions)",
}


def walk_roofline(args, kern_ms, steps_per_rank, ms_per_step, kernel):
    peak, peak_src = read_peak()
    achieved = steps_per_rank * BYTES_PER_STEP / (kern_ms * 1e-3) / 1e9
    traffic = read_profile_json("ncu_traffic.json", args.workload)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic.get("dram_bytes_per_launch") if isinstance(traffic, dict) else traffic,
            "traffic_detail": traffic,
            "kernel_ms": kern_ms, "step_share": kern_ms / ms_per_step,
            "bytes_per_step": BYTES_PER_STEP, "peak_source": peak_src,
            "model": "achieved = steps x 64 B (one 32 B sector for {base,deg} + one for the neighbour id, "
                     "SURVEY §8d) / K2 launch time (CUDA events on the launch stream)"}
    roof["kernel"] = "K2 " + K2_DESCR.get(kernel, kernel)
    if roof["frac"] > 1.0 and "fat" in kernel:
        roof["note"] = ("frac > 1: the 64 B/step model charges every step two DRAM sectors, while this kernel takes "
                        "one gather per step from an L2-resident array and counts in shared memory; HBM is not the "
                        "bound, see `l2`")
    elif roof["frac"] > 1.0:
        roof["note"] = ("frac > 1: the 64 B/step model charges every step two DRAM sectors, while the records and "
                        "counters of the highest-degree vertices are served from shared memory and part of the "
                        "neighbour sectors hit in L2; `traffic` is the DRAM bytes ncu measured per launch")
    if args.workload == "cfg1":
        # the cfg1 CSR (4.5 MB) is L2-resident: HBM is not the bound, L2
        # random-sector throughput is (SURVEY §8d asks for it beside HBM)
        # L2 sector bytes per step as ncu measured them on this kernel
        # (profiles/ncu_traffic.json); without a capture, one 32 B sector per
        # gather: the fat kernels take one gather per step, the others two
        per_step = traffic.get("l2_sector_bytes_per_step") if isinstance(traffic, dict) else None
        src = "ncu lts__t_sectors_srcunit_tex per step (profiles/ncu_traffic.json)"
        if not per_step:
            per_step = 32.0 if "fat" in kernel else 64.0
            src = "algorithmic: one 32 B sector per gather"
        l2 = steps_per_rank * per_step / (kern_ms * 1e-3) / 1e9
        roof["l2"] = {"achieved_sector_gbs": l2, "ceiling_gbs": L2_RANDOM_SECTOR_GBS,
                      "frac": l2 / L2_RANDOM_SECTOR_GBS, "sector_bytes_per_step": per_step,
                      "sector_bytes_source": src,
                      "ceiling_source": "tools/gather_ceiling.cu random 32 B-sector gathers, 32 MB working "
                                        "set (profiles/r01_gather_ceiling.txt)"}
    return roof


def run_ours(args):
    import torch

    import paper_2410_14056_b200 as sb

    rank, world, local = dist_env()
    dev_index = init_dist(args, local)
    dev = torch.device("cuda", dev_index)
    spec, walks, L = WORKLOADS[args.workload]
    g = make_graph(sb, spec, dev_index)
    cfg = sb.CampaignConfig(length=L, master_seed=MASTER_SEED)
    total_walks = walks * world
    steps_per_rank = walks * (L - 1)

    counts = torch.zeros(g.n, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    g.device_handle(dev_index)

    def one_step(timing):
        counts.zero_()
        rep = sb.run_walk_campaign_device(g, cfg, counts.data_ptr(), stream.cuda_stream,
                                          total_walks=total_walks, shard_index=rank,
                                          shard_count=world, device=dev_index, timing=timing)
        if world > 1:
            all_reduce(counts, args)
        return rep

    for _ in range(args.warmup):
        flush.zero_()
        one_step(False)
    torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    walk_ms, launches = [], 0
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev_index) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            starts[i].record(stream)
            rep = one_step(True)
            ends[i].record(stream)
            walk_ms.append(rep.walk_kernel_ms)
            launches += rep.launches
            k2_kernel = rep.kernel
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        all_reduce(tot, args, dist.ReduceOp.MAX)
    ms_per_step = tot.item() / args.steps
    value = total_walks * (L - 1) / (ms_per_step * 1e-3)

    final = counts.cpu().numpy().view(np.uint64).copy()
    assert int(final.sum()) == total_walks * L, (int(final.sum()), total_walks * L)
    # share of all visits that fell on vertices whose counters sat in shared
    # memory (the highest-degree ranks, ties by id, as the device orders them)
    n_rec, n_cnt = sb.campaign_tables(g, dev_index)
    deg = np.diff(g.offsets.astype(np.int64))
    by_rank = np.argsort(-deg, kind="stable")
    tables = {"records": n_rec, "counters": n_cnt,
              "visits_on_shared_counters_frac": float(final[by_rank[:n_cnt]].sum()) / float(final.sum()),
              "departures_from_shared_records_frac": float(final[by_rank[:n_rec]].sum()) / float(final.sum())}

    # end to end through the public API with host buffers (pinned CSR in,
    # host counts out); every step re-creates the device replica (H2D).
    pin_off = torch.from_numpy(g.offsets).pin_memory().numpy()
    pin_adj = torch.from_numpy(g.adjacency).pin_memory().numpy()
    ge = sb.Graph(pin_off, pin_adj, _trusted=True)
    e2e_t = []
    for i in range(args.warmup + args.steps):
        if world > 1:
            dist.barrier()
        # device events bracket the whole blocking API call (H2D, walks, D2H)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        sink = sb.VisitCountSink(g.n)
        sb.run_walk_campaign(ge, cfg, sink, total_walks=total_walks, shard_index=rank,
                             shard_count=world, device=dev_index)
        if world > 1:
            ct = torch.from_numpy(sink.counts.view(np.int64)).to(dev)
            all_reduce(ct, args)
            sink.counts[:] = ct.cpu().numpy().view(np.uint64)
        ge.release_device()
        e1.record(stream)
        e1.synchronize()
        if i >= args.warmup:
            e2e_t.append(e0.elapsed_time(e1) * 1e-3)
    assert np.array_equal(sink.counts, final), "e2e counts differ from the device-resident run"
    e2e_tot = torch.tensor([sum(e2e_t)], dtype=torch.float64, device=dev)
    if world > 1:
        all_reduce(e2e_tot, args, dist.ReduceOp.MAX)
    e2e_value = total_walks * (L - 1) / (e2e_tot.item() / args.steps)

    if rank == 0:
        kern_ms = statistics.mean(walk_ms)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            R = reference_lib()
            cnt, sec, steps = cpu_campaign(R, R.from_csr(g.offsets, g.adjacency), total_walks, L)
            assert np.array_equal(cnt, final), "CPU reference counts differ from the GPU counts"
            cpu = {"value": steps / sec, "unit": "steps/s", "cores": R.max_threads(), "kind": "reference",
                   "sample": f"oracle/_ref (reference headers, OpenMP) on the full workload: {steps} steps "
                             f"in {sec:.2f} s; counts equal to the GPU's (checked)"}
        out = {
            "metric": "walk steps/sec (Bouquets)", "value": value, "unit": "steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": walk_config(args.workload, g.n, g.m, world, args.dist_backend),
            "checksum": {"counts_sha256_16": counts_checksum(final), "total_visits": int(final.sum())},
            "roofline": dict(walk_roofline(args, kern_ms, steps_per_rank, ms_per_step, k2_kernel),
                             shared_tables=tables),
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "steps/s",
                    "h2d_bytes_per_step": int(g.offsets.nbytes + g.adjacency.nbytes),
                    "d2h_bytes_per_step": int(g.n * 8)},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if world == 1 and args.workload == "cfg2" and not args.no_aesc:
            out["aesc_cfg3"] = aesc_block(sb, args, "cfg3", dev_index)
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def aesc_roofline(name, est, wall_s):
    """Per-phase model (an honest AESC roofline):
    * propagation: the reference's edge-visits (sum over sources and depths of
      the support degree sum, counted exactly on the device) x 12 B, over the
      propagation's CUDA-event time;
    * walks: DRAM bytes and L2 sectors per walk step measured by ncu on this
      build for this config (profiles/aesc_walk_traffic.json), x steps, over
      the walk kernels' own CUDA-event time (events around every launch).
    `est` should come from a one-worker run (AescConfig.workers=1): with two
    batch workers the phases of different batches overlap and each phase's
    event time includes the other's interference."""
    peak, peak_src = read_peak()
    prop_s, walk_s = est.propagation_ms * 1e-3, (est.walk_kernel_ms or est.walk_ms) * 1e-3
    prop_bytes = est.edge_visits * BYTES_PER_EDGE_VISIT
    prop_gbs = prop_bytes / prop_s / 1e9 if prop_s > 0 else 0.0
    tr = read_profile_json("aesc_walk_traffic.json", name) or {}
    walk = {"steps": est.total_walk_steps, "seconds": walk_s,
            "steps_per_s": est.total_walk_steps / walk_s if walk_s > 0 else 0.0}
    dram_gbs = None
    if tr.get("dram_bytes_per_step") is not None and walk_s > 0:
        dram_gbs = tr["dram_bytes_per_step"] * est.total_walk_steps / walk_s / 1e9
        walk.update({"dram_bytes_per_step": tr["dram_bytes_per_step"], "achieved_dram_gbs": dram_gbs,
                     "dram_frac": dram_gbs / peak})
    l2 = None
    if tr.get("l2_sector_bytes_per_step") is not None and walk_s > 0:
        l2 = tr["l2_sector_bytes_per_step"] * est.total_walk_steps / walk_s / 1e9
        walk.update({"l2_sector_bytes_per_step": tr["l2_sector_bytes_per_step"], "achieved_l2_gbs": l2,
                     "l2_frac_of_random_sector_ceiling": l2 / L2_RANDOM_SECTOR_GBS})
    walk["traffic_source"] = tr or None
    phases = {"propagation": {"edge_visits": est.edge_visits, "bytes_per_edge_visit": BYTES_PER_EDGE_VISIT,
                              "seconds": prop_s, "achieved_gbs": prop_gbs, "frac": prop_gbs / peak},
              "walk": walk}
    # the dominant kernel is the walk (K4) whenever it holds most device time
    if dram_gbs is not None and walk_s >= prop_s:
        roof = {"bound": "hbm", "achieved": dram_gbs, "peak": peak, "unit": "GB/s", "frac": dram_gbs / peak,
                "traffic": tr.get("dram_bytes_per_launch"), "kernel": "aesc_walk_sorted (K4 walk phase)",
                "model": "ncu-measured DRAM bytes per walk step (this build, this config) x walk steps / "
                         "K4 kernel time"}
        if l2 is not None:
            # L2-resident configs (cfg3): the walk is bound by L2 random-sector
            # throughput, not HBM; the ceiling is measured (gather_ceiling.cu)
            roof["l2"] = {"achieved_sector_gbs": l2, "ceiling_gbs": L2_RANDOM_SECTOR_GBS,
                          "frac": l2 / L2_RANDOM_SECTOR_GBS,
                          "ceiling_source": "tools/gather_ceiling.cu random 32 B-sector gathers, 32 MB working set "
                                            "(profiles/r01_gather_ceiling.txt)"}
    else:
        roof = {"bound": "hbm", "achieved": prop_gbs, "peak": peak, "unit": "GB/s", "frac": prop_gbs / peak,
                "traffic": None, "kernel": "aesc_pull (K3 propagation)",
                "model": "edge-visits x 12 B (SURVEY §8d) / K3 phase time"}
    roof.update({"peak_source": peak_src, "phases": phases, "wall_s": wall_s})
    return roof


def aesc_block(sb, args, name, dev_index):
    """BASELINE's second metric on `name` (cfg3: every source), 1 warm-up +
    1 timed device run + 1 end-to-end run, clocks sampled during the timed run."""
    import torch
    spec, eps, delta, _, cpu_sources = AESC_WORKLOADS[name]
    g = make_graph(sb, spec, dev_index)
    cfg = sb.AescConfig(epsilon=eps, delta=delta, threads=1)
    sb.aesc(g, cfg, device=dev_index)  # warm-up
    stream = torch.cuda.current_stream(dev_index)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev_index)
    with ClockSampler(dev_index) as clk:
        e0.record(stream)
        est = sb.aesc(g, cfg, device=dev_index)
        e1.record(stream)
        e1.synchronize()
    wall = e0.elapsed_time(e1) * 1e-3
    # end to end: pinned host CSR in (device replica rebuilt), g_hat + s_hat out
    pin_off = torch.from_numpy(g.offsets).pin_memory().numpy()
    pin_adj = torch.from_numpy(g.adjacency).pin_memory().numpy()
    ge = sb.Graph(pin_off, pin_adj, _trusted=True)
    torch.cuda.synchronize(dev_index)
    e0.record(stream)
    est2 = sb.aesc(ge, cfg, device=dev_index)
    ge.release_device()
    e1.record(stream)
    e1.synchronize()
    e2e = e0.elapsed_time(e1) * 1e-3
    assert np.array_equal(est2.s_hat, est.s_hat), "e2e AESC differs from the device run"
    # roofline run: one batch worker, so each phase's CUDA-event time is its own
    cfg1 = sb.AescConfig(epsilon=eps, delta=delta, threads=1, workers=1)
    est1 = sb.aesc(g, cfg1, device=dev_index)
    assert np.array_equal(est1.s_hat, est.s_hat), "the one-worker run differs"
    res = {"metric": "TGT+ all-edges SC wall time", "value": wall, "unit": "s", "higher_is_better": False,
           "steps": 1, "warmup": 1, "dtype": "f64",
           "config": aesc_config(name, g.n, g.m, 1, f"all {g.n} sources"),
           "checksum": {"s_hat_sha256_16": f64_checksum(est.s_hat), "s_hat_sum": float(est.s_hat.sum())},
           "stats": {"walk_pairs": est.total_walk_pairs, "walk_steps": est.total_walk_steps,
                     "edge_visits": est.edge_visits, "lambda_hat": est.plan.lambda_hat,
                     "tau": int(est.plan.max_tau), "plan_s": est.plan_seconds,
                     "propagation_s": est.propagation_ms * 1e-3, "walk_s": est.walk_ms * 1e-3},
           "roofline": dict(aesc_roofline(name, est1, wall), roofline_run={
               "workers": est1.workers, "seconds": est1.seconds, "propagation_s": est1.propagation_ms * 1e-3,
               "walk_kernel_s": est1.walk_kernel_ms * 1e-3, "walk_phase_s": est1.walk_ms * 1e-3}),
           "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(g.offsets.nbytes + g.adjacency.nbytes),
                   "d2h_bytes_per_step": int(est.g_hat.nbytes + est.s_hat.nbytes)},
           "gpu_launches": int(est.launches), "clocks": clk.summary()}
    if not args.no_cpu_baseline:
        try:
            R = reference_lib()
            res["cpu_baseline"] = cpu_aesc_sample(R, g.offsets, g.adjacency, g.n, eps, delta, cpu_sources)
            res["cpu_baseline"]["full_run"] = read_profile_json("aesc_cpu_full.json", name)
        except Exception as e:  # noqa: BLE001
            res["cpu_baseline"] = {"unavailable": str(e)}
    return res


def run_aesc_bench(args):
    """TGT+ AESC wall time (BASELINE metric 2). Full graph for cfg3; cfg4/cfg5
    on a fixed source subset extrapolated x n/|subset| (the paper's own Orkut
    protocol), as SURVEY §8d prescribes. N ranks: each runs its
    cost-stratified shard with g_hat left on the device (saba_cu_aesc_device),
    one all-reduce of g_hat (exact: one writer per slot), then K5 on the
    device for full runs."""
    import torch

    import paper_2410_14056_b200 as sb

    rank, world, local = dist_env()
    dev_index = init_dist(args, local)
    dev = torch.device("cuda", dev_index)
    spec, eps, delta, per_gpu, cpu_sources = AESC_WORKLOADS[args.workload]
    g = make_graph(sb, spec, dev_index)
    cfg = sb.AescConfig(epsilon=eps, delta=delta, threads=1)
    if per_gpu:
        sources = subset_sources(g.n, per_gpu * world)
        label = f"{per_gpu * world} sources of {g.n} (fixed permutation), extrapolated x{g.n / (per_gpu * world):.1f}"
    else:
        sources = None
        label = f"all {g.n} sources"
    g.device_handle(dev_index)
    stream = torch.cuda.current_stream(dev)
    g_hat = torch.empty(2 * g.m, dtype=torch.float64, device=dev)
    s_hat = torch.empty(g.m, dtype=torch.float64, device=dev)

    def one(graph):
        # CUDA events on the current stream bracket the whole (blocking) call,
        # host planning included: the device-timeline span of one AESC run
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        est = sb.aesc_device(graph, cfg, g_hat.data_ptr(), stream.cuda_stream, sources=sources,
                             shard_index=rank, shard_count=world, device=dev_index)
        if world > 1:
            all_reduce(g_hat, args)  # each slot has one writer: the sum is exact
        if sources is None:
            sb.symmetrise(graph, g_hat.data_ptr(), s_hat.data_ptr(), stream.cuda_stream, device=dev_index)
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) * 1e-3, est

    for _ in range(args.warmup):
        one(g)
    times, ests = [], []
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev_index) as clk:
        for _ in range(args.steps):
            dt, est = one(g)
            times.append(dt)
            ests.append(est)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    tot = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    if world > 1:
        all_reduce(tot, args, dist.ReduceOp.MAX)
    measured = tot.item() / args.steps
    scale = g.n / len(sources) if sources is not None else 1.0
    # per-call costs (the truncation plan, and the setup between the plan and
    # the first batch: slot records, workspaces, tau upload) are paid once by
    # a full run too, so only the rest (the batches) is scaled by n/|sources|
    plan_s = ests[-1].plan_seconds
    setup_s = ests[-1].setup_seconds
    one_time = min(measured, plan_s + setup_s)
    full_estimate = one_time + (measured - one_time) * scale
    gh = g_hat.cpu().numpy()
    sh = s_hat.cpu().numpy() if sources is None else None
    # end to end: the public API from pinned host CSR (graph upload inside),
    # g_hat (and s_hat) back to host
    pin_off = torch.from_numpy(g.offsets).pin_memory().numpy()
    pin_adj = torch.from_numpy(g.adjacency).pin_memory().numpy()
    ge = sb.Graph(pin_off, pin_adj, _trusted=True)
    e2e = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        one(ge)
        host = g_hat.cpu()
        if sources is None:
            s_hat.cpu()
        ge.release_device()
        e1.record(stream)
        e1.synchronize()
        e2e.append(e0.elapsed_time(e1) * 1e-3)
    assert np.array_equal(host.numpy(), gh), "e2e g_hat differs from the device run"
    # roofline run of this rank's shard with one batch worker (phase times not overlapped)
    est1 = sb.aesc_device(g, sb.AescConfig(epsilon=eps, delta=delta, threads=1, workers=1), g_hat.data_ptr(),
                          stream.cuda_stream, sources=sources, shard_index=rank, shard_count=world,
                          device=dev_index)
    e2e_t = torch.tensor([sum(e2e)], dtype=torch.float64, device=dev)
    edge_visits = torch.tensor([float(ests[-1].edge_visits)], dtype=torch.float64, device=dev)
    if world > 1:
        all_reduce(e2e_t, args, dist.ReduceOp.MAX)
    if rank == 0:
        est = ests[-1]
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_aesc_sample(reference_lib(), g.offsets, g.adjacency, g.n, eps, delta, cpu_sources)
                cpu["full_run"] = read_profile_json("aesc_cpu_full.json", args.workload)
            except Exception as e:  # noqa: BLE001
                cpu = {"unavailable": str(e)}
        config = aesc_config(args.workload, g.n, g.m, world, label)
        config.update({"measured_seconds": measured,
                       "extrapolation": "one_time + (measured - one_time) * n/|sources|, one_time = plan_s + setup_s"
                       if sources is not None else "none", "plan_s": plan_s, "setup_s": setup_s,
                       "lambda_hat": est.plan.lambda_hat, "tau": int(est.plan.max_tau)})
        out = {
            "metric": "TGT+ all-edges SC wall time", "value": full_estimate, "unit": "s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": measured * 1e3, "higher_is_better": False,
            "scaling": "weak" if per_gpu else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config,
            "checksum": {"g_hat_sha256_16": f64_checksum(gh),
                         **({"s_hat_sha256_16": f64_checksum(sh)} if sh is not None else {})},
            "stats": {"walk_pairs_rank0": est.total_walk_pairs, "walk_steps_rank0": est.total_walk_steps,
                      "edge_visits_rank0": est.edge_visits, "plan_s": est.plan_seconds,
                      "propagation_s_rank0": est.propagation_ms * 1e-3, "walk_s_rank0": est.walk_ms * 1e-3},
            "roofline": dict(aesc_roofline(args.workload, est1, measured), roofline_run={
                "workers": est1.workers, "seconds": est1.seconds, "propagation_s": est1.propagation_ms * 1e-3,
                "walk_kernel_s": est1.walk_kernel_ms * 1e-3, "walk_phase_s": est1.walk_ms * 1e-3,
                "rank": 0}),
            "cpu_baseline": cpu,
            # the e2e-only work (pinned CSR upload, device replica build) is a
            # per-run cost: added once, not multiplied by the extrapolation
            "e2e": {"value": full_estimate + max(0.0, e2e_t.item() / args.steps - measured), "unit": "s",
                    "h2d_bytes_per_step": int(g.offsets.nbytes + g.adjacency.nbytes),
                    "d2h_bytes_per_step": int(gh.nbytes + (sh.nbytes if sh is not None else 0))},
            "gpu_launches": int(est.launches) * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 20 for walk campaigns, 2 for AESC workloads)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="saba", choices=["saba", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS) + sorted(AESC_WORKLOADS))
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="collective backend for N>1 (gloo: host all-reduce; N ranks may share one GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-aesc", action="store_true", help="skip the cfg3 AESC block of the default run")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 2 if args.workload in AESC_WORKLOADS else 20
    if args.workload in AESC_WORKLOADS:
        if args.impl == "reference":
            run_aesc_reference(args)
            return
        run_aesc_bench(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
