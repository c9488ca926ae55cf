"""TGT+ all-edges spanning centrality (aesc.hpp) over the sm_100a estimator.

Reference surface mirrored: AescConfig 40-53, TruncationPlan 55-61,
LandingProbs 63-79, CentralityEstimate 86-95, walk_budget 117-126,
truncated_lengths 210-248, propagate_landing_probabilities 406-422,
estimate_edge 533-553, aesc 636-708, write_centrality_tsv 713-734.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .graph import Graph
from .walker import HashSpec, WalkMode


@dataclass
class AescConfig:
    epsilon: float = 0.05
    delta: float = 0.05
    power_iterations: int = 30
    candidate_nodes: int = 0
    mode: WalkMode = WalkMode.Saba
    master_seed: int = 42
    threads: int = 0
    lanes: int = 8
    max_truncation: int = 128
    per_edge_tau: bool = False
    switch_depth_cap: int = -1
    hash: HashSpec = field(default_factory=HashSpec)
    workers: int = 0  # extension: batch workers per device (0 = auto); never changes results

    def to_c(self) -> L.AescConfigC:
        return L.AescConfigC(self.epsilon, self.delta, self.power_iterations, self.candidate_nodes,
                             int(self.mode), self.threads, self.master_seed, self.lanes,
                             self.max_truncation, int(self.per_edge_tau), self.workers,
                             self.switch_depth_cap, self.hash.multiplier)


@dataclass
class TruncationPlan:
    tau: np.ndarray
    tau_tilde: np.ndarray | None = None
    lambda_hat: float = 0.0
    clamped: bool = False
    max_tau: int = 0


@dataclass
class LandingProbs:
    source: int = 0
    depth: int = 0
    support: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    prob: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))

    def prob_of(self, v: int) -> float:
        i = int(np.searchsorted(self.support, v))
        return float(self.prob[i]) if i < len(self.support) and self.support[i] == v else 0.0

    def sum(self) -> float:
        s = 0.0
        for p in self.prob:  # sequential, like aesc.hpp:74-78
            s += float(p)
        return s

    def dense(self, n: int) -> np.ndarray:
        d = np.zeros(n, np.float64)
        d[self.support] = self.prob
        return d


@dataclass
class CentralityEstimate:
    s_hat: np.ndarray | None
    g_hat: np.ndarray
    config: AescConfig
    plan: TruncationPlan
    bipartite: bool = False
    total_walk_pairs: int = 0
    total_walk_steps: int = 0
    seconds: float = 0.0
    # device detail
    propagation_ms: float = 0.0
    walk_ms: float = 0.0
    plan_seconds: float = 0.0
    edge_visits: int = 0
    launches: int = 0
    replicas: int = 1
    workers: int = 1
    walk_kernel_ms: float = 0.0
    setup_seconds: float = 0.0


def walk_budget(tau_effective: int, epsilon: float, delta: float, degree: int,
                edge_count: int) -> int:
    out = C.c_uint64()
    L.check(L.lib().saba_cu_walk_budget(tau_effective, epsilon, delta, degree, edge_count,
                                        C.byref(out)), "walk_budget")
    return out.value


def truncated_lengths(g: Graph, epsilon: float, power_iterations: int,
                      max_truncation: int = 128, per_edge: bool = False,
                      device: int = 0) -> TruncationPlan:
    tau = np.zeros(g.m, np.uint32)
    lam = C.c_double()
    cl = C.c_int()
    L.check(L.lib().saba_cu_truncated_lengths(g.device_handle(device), epsilon, power_iterations,
                                              max_truncation, int(per_edge), L.ptr(tau, L.u32p),
                                              C.byref(lam), C.byref(cl)), "truncated_lengths")
    return TruncationPlan(tau, None, lam.value, bool(cl.value), int(tau.max()) if len(tau) else 0)


def _is_connected(g: Graph) -> bool:
    n = g.n
    if n == 0:
        return False
    seen = np.zeros(n, bool)
    seen[0] = True
    frontier = np.array([0], np.int64)
    while len(frontier):
        nb = np.concatenate([g.adjacency[g.offsets[u]:g.offsets[u + 1]] for u in frontier]) \
            if len(frontier) < 64 else g.adjacency[np.concatenate(
                [np.arange(g.offsets[u], g.offsets[u + 1]) for u in frontier])]
        nb = np.unique(nb)
        nb = nb[~seen[nb]]
        seen[nb] = True
        frontier = nb.astype(np.int64)
    return bool(seen.all())


def aesc(g: Graph, cfg: AescConfig, *, sources=None, shard_index: int = 0, shard_count: int = 1,
         device: int = 0, devices=None) -> CentralityEstimate:
    """aesc.hpp:636-708 on one B200. `sources` restricts the estimator to a
    source subset (SURVEY §8d protocol), deduplicated; shard `shard_index`
    of `shard_count` runs the sources aesc_shard_sources() returns. `devices`
    (a list, repeats allowed) runs the call over one replica per entry
    (Graph.device_group) with one combine of g_hat: identical results."""
    n, m = g.n, g.m
    g_hat = np.zeros(2 * m, np.float64)
    full = sources is None and shard_count == 1
    s_hat = np.zeros(m, np.float64) if full else None
    tau = np.zeros(m, np.uint32)
    tt = np.zeros(n, np.uint32)
    src = None if sources is None else np.ascontiguousarray(sources, np.uint32)
    rep = L.AescReportC()
    c = cfg.to_c()
    h = g.device_group(devices) if devices is not None else g.device_handle(device)
    L.check(L.lib().saba_cu_aesc(h, C.byref(c), L.ptr(src, L.u32p),
                                 0 if src is None else len(src), shard_index, shard_count,
                                 L.ptr(g_hat, L.f64p), L.ptr(s_hat, L.f64p), L.ptr(tau, L.u32p),
                                 L.ptr(tt, L.u32p), C.byref(rep)), "aesc")
    plan = TruncationPlan(tau, tt, rep.lambda_hat, bool(rep.clamped), rep.max_tau)
    return CentralityEstimate(s_hat, g_hat, cfg, plan, bool(rep.bipartite), rep.total_walk_pairs,
                              rep.total_walk_steps, rep.seconds, rep.propagation_ms, rep.walk_ms,
                              rep.plan_seconds, rep.edge_visits, rep.launches, rep.replicas, rep.workers,
                              rep.walk_kernel_ms, rep.setup_seconds)


def aesc_device(g: Graph, cfg: AescConfig, g_hat_dev_ptr: int, stream_ptr: int = 0, *, sources=None,
                shard_index: int = 0, shard_count: int = 1, device: int = 0) -> CentralityEstimate:
    """aesc() leaving g_hat (2m float64) in a caller-owned device buffer on
    `device` (e.g. a torch tensor's data_ptr()), zero outside this shard's
    slots, so one-process-per-GPU callers can all-reduce it (exact: one
    writer per slot) and form s_hat with symmetrise(). The returned estimate
    carries the plan, tau~ and counters; its g_hat/s_hat are None."""
    n, m = g.n, g.m
    tau = np.zeros(m, np.uint32)
    tt = np.zeros(n, np.uint32)
    src = None if sources is None else np.ascontiguousarray(sources, np.uint32)
    rep = L.AescReportC()
    c = cfg.to_c()
    L.check(L.lib().saba_cu_aesc_device(g.device_handle(device), C.byref(c), L.ptr(src, L.u32p),
                                        0 if src is None else len(src), shard_index, shard_count,
                                        C.c_void_p(g_hat_dev_ptr), L.ptr(tau, L.u32p), L.ptr(tt, L.u32p),
                                        C.c_void_p(stream_ptr), C.byref(rep)), "aesc_device")
    plan = TruncationPlan(tau, tt, rep.lambda_hat, bool(rep.clamped), rep.max_tau)
    return CentralityEstimate(None, None, cfg, plan, bool(rep.bipartite), rep.total_walk_pairs,
                              rep.total_walk_steps, rep.seconds, rep.propagation_ms, rep.walk_ms,
                              rep.plan_seconds, rep.edge_visits, rep.launches, rep.replicas, rep.workers,
                              rep.walk_kernel_ms, rep.setup_seconds)


def symmetrise(g: Graph, g_hat_dev_ptr: int, s_hat_dev_ptr: int, stream_ptr: int = 0,
               device: int = 0) -> None:
    """K5 on device buffers: s_hat[e] = g_hat[u->v] + g_hat[v->u]
    (aesc.hpp:702-706), enqueued on `stream_ptr`."""
    L.check(L.lib().saba_cu_symmetrise(g.device_handle(device), C.c_void_p(g_hat_dev_ptr),
                                       C.c_void_p(s_hat_dev_ptr), C.c_void_p(stream_ptr)), "symmetrise")


def propagate_landing_probabilities(g: Graph, source: int, plan: TruncationPlan, epsilon: float,
                                    delta: float, switch_depth_cap: int = -1, device: int = 0):
    """aesc.hpp:406-422 -> (LandingProbs at tau~, tau~)."""
    prob = np.zeros(g.n, np.float64)
    depth = C.c_uint32()
    tau = np.ascontiguousarray(plan.tau, np.uint32)
    L.check(L.lib().saba_cu_propagate(g.device_handle(device), source, L.ptr(tau, L.u32p), epsilon,
                                      delta, switch_depth_cap, L.ptr(prob, L.f64p), C.byref(depth)),
            "propagate")
    support = np.nonzero(prob)[0].astype(np.uint32)
    return LandingProbs(source, depth.value, support, prob[support]), depth.value


def estimate_edge(g: Graph, v_i: int, v_j: int, landing: LandingProbs, tau_eff: int, n_req: int,
                  mode: WalkMode, edge_seed: int, lanes: int = 8, hash: HashSpec = HashSpec(),
                  device: int = 0) -> float:
    """aesc.hpp:533-553."""
    prob = landing.dense(g.n)
    out = C.c_double()
    L.check(L.lib().saba_cu_estimate_edge(g.device_handle(device), v_i, v_j, L.ptr(prob, L.f64p),
                                          tau_eff, n_req, int(mode), edge_seed, lanes,
                                          hash.multiplier, C.byref(out)), "estimate_edge")
    return out.value


def write_centrality_tsv(out, g: Graph, values) -> None:
    """aesc.hpp:713-734: `u<TAB>v<TAB>%.6g`, ascending (u, v)."""
    values = np.asarray(values)
    if len(values) != g.m:
        raise ValueError("write_centrality_tsv: value count != edge count")
    e = g.edges()
    order = np.lexsort((e[:, 1], e[:, 0]))
    for i in order:
        out.write(f"{int(e[i, 0])}\t{int(e[i, 1])}\t{values[i]:.6g}\n")


def aesc_shard_sources(g: Graph, sources, shard_index: int, shard_count: int) -> np.ndarray:
    """The distinct sources shard `shard_index` of `shard_count` runs
    (sources=None: every vertex), exactly as saba_cu_aesc cuts them:
    ascending degree — a source's walk work falls as ~tau^3/d — dealt to the
    shards in snake order, so every shard gets the same cost profile.
    Host-only (no device needed)."""
    if not 0 <= shard_index < shard_count:
        raise ValueError("bad shard index/count")
    src = None if sources is None else np.ascontiguousarray(sources, np.uint32)
    cnt = C.c_uint64()
    args = (L.ptr(g.offsets, L.u32p), g.n, L.ptr(src, L.u32p), 0 if src is None else len(src),
            shard_index, shard_count)
    L.check(L.lib().saba_aesc_shard_sources(*args, None, C.byref(cnt)), "aesc_shard_sources")
    out = np.zeros(cnt.value, np.uint32)
    L.check(L.lib().saba_aesc_shard_sources(*args, L.ptr(out, L.u32p), C.byref(cnt)), "aesc_shard_sources")
    return out
