"""TEST INFRASTRUCTURE ONLY — ctypes front-ends for the parity oracle.

* ``Oracle``     -> oracle/_build/liboracle.so, the C restatement
                    (oracle/saba_oracle.c) of the reference hot path.
* ``Reference``  -> oracle/_ref/libsaba_ref.so, the reference headers compiled
                    unchanged (oracle/ref_driver.cpp); absent where neither
                    /root/reference nor a prebuilt copy exists.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
module. The product (paper_2410_14056_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsaba_ref.so")

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def build(quiet: bool = True) -> None:
    """Compile the oracle (and the reference shim where the reference exists)."""
    subprocess.run(["make", "-C", HERE, "-s"] if quiet else ["make", "-C", HERE],
                   check=True, stdout=subprocess.DEVNULL if quiet else None)


class _OracleCfg(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("delta", C.c_double),
                ("power_iterations", C.c_uint32), ("master_seed", C.c_uint64),
                ("max_truncation", C.c_uint32), ("per_edge_tau", C.c_int),
                ("switch_depth_cap", C.c_int64), ("hash_multiplier", C.c_uint64),
                ("threads", C.c_int)]


class _Csr(C.Structure):
    _fields_ = [("n", C.c_uint32), ("m", C.c_uint64), ("off", C.POINTER(C.c_uint32)),
                ("adj", C.POINTER(C.c_uint32))]


class _RefCfg(C.Structure):
    _fields_ = _OracleCfg._fields_ + [("mode", C.c_int), ("lanes", C.c_uint32)]


@dataclass
class AescResult:
    g_hat: np.ndarray
    s_hat: np.ndarray | None
    tau: np.ndarray
    tau_tilde: np.ndarray
    lambda_hat: float
    total_walk_pairs: int
    total_walk_steps: int
    seconds: float = 0.0
    plan_seconds: float = 0.0


DEFAULT_MULT = 0xC6A4A7935BD1E995


class Oracle:
    """The C restatement (saba_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.lib = L
        L.oracle_mix64.restype = C.c_uint64
        L.oracle_mix64.argtypes = [C.c_uint64]
        L.oracle_counter_hash.restype = C.c_uint64
        L.oracle_counter_hash.argtypes = [C.c_uint64, C.c_uint64]
        L.oracle_substream.restype = C.c_uint64
        L.oracle_substream.argtypes = [C.c_uint64, C.c_uint64]
        L.oracle_hash_state.restype = C.c_uint32
        L.oracle_hash_state.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
        L.oracle_scaled_index.restype = C.c_uint32
        L.oracle_scaled_index.argtypes = [C.c_uint32, C.c_uint32]
        L.oracle_random_walk.argtypes = [u32p, u32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_uint64, u32p]
        L.oracle_campaign_counts.argtypes = [u32p, u32p, C.c_uint32, u64p, C.c_uint64,
                                             C.c_uint32, C.c_uint64, C.c_uint64, C.c_int, u64p]
        L.oracle_campaign_range.argtypes = [u32p, u32p, C.c_uint32, u64p, C.c_uint64, C.c_uint32,
                                            C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        L.oracle_uniform_start_counts.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, u64p]
        L.oracle_is_connected.restype = C.c_int
        L.oracle_is_connected.argtypes = [u32p, u32p, C.c_uint32]
        L.oracle_slot_edges.argtypes = [u32p, u32p, C.c_uint32, u32p]
        L.oracle_truncated_lengths.restype = C.c_int
        L.oracle_truncated_lengths.argtypes = [u32p, u32p, C.c_uint32, C.c_uint64, C.c_double,
                                               C.c_uint32, C.c_uint32, C.c_int, u32p, f64p,
                                               C.POINTER(C.c_int)]
        L.oracle_walks_needed_raw.restype = C.c_double
        L.oracle_walks_needed_raw.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_uint32,
                                              C.c_uint64]
        L.oracle_walk_budget.restype = C.c_int
        L.oracle_walk_budget.argtypes = [C.c_uint32, C.c_double, C.c_double, C.c_uint32,
                                         C.c_uint64, u64p]
        L.oracle_propagate.argtypes = [u32p, u32p, C.c_uint32, C.c_uint64, C.c_uint32, u32p, u32p,
                                       C.c_double, C.c_double, C.c_int64, f64p, u32p]
        L.oracle_csr_free.argtypes = [C.POINTER(_Csr)]
        L.oracle_gen_erdos_renyi.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, C.POINTER(_Csr)]
        L.oracle_gen_rmat.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                      C.c_uint64, C.c_int, C.POINTER(_Csr)]
        L.oracle_gen_chung_lu.argtypes = [C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                          C.c_int, C.POINTER(_Csr)]
        L.oracle_aesc.restype = C.c_int
        L.oracle_aesc.argtypes = [u32p, u32p, C.c_uint32, C.c_uint64, C.POINTER(_OracleCfg),
                                  u32p, C.c_uint64, f64p, f64p, u32p, u32p, f64p, u64p, u64p]

    # -- BASELINE graphs (oracle_gen.c): (offsets, adjacency) numpy arrays
    def _csr(self, fn, *args):
        c = _Csr()
        _raise(fn(*args, C.byref(c)), fn.__name__)
        try:
            off = np.ctypeslib.as_array(c.off, shape=(c.n + 1,)).copy()
            adj = np.ctypeslib.as_array(c.adj, shape=(max(2 * c.m, 1),))[: 2 * c.m].copy()
        finally:
            self.lib.oracle_csr_free(C.byref(c))
        return off, adj

    def gen_erdos_renyi(self, n, m, seed):
        return self._csr(self.lib.oracle_gen_erdos_renyi, n, m, seed)

    def gen_rmat(self, scale, edge_factor, a=0.57, b=0.19, c=0.19, seed=1, keep_lcc=True):
        return self._csr(self.lib.oracle_gen_rmat, scale, edge_factor, a, b, c, seed, int(keep_lcc))

    def gen_chung_lu(self, n, gamma=2.2, mean_degree=78.0, max_degree=30000.0, seed=1, keep_lcc=True):
        return self._csr(self.lib.oracle_gen_chung_lu, n, gamma, mean_degree, max_degree, seed,
                         int(keep_lcc))

    # -- primitives
    def mix64(self, x): return self.lib.oracle_mix64(x)
    def counter_hash(self, m, i): return self.lib.oracle_counter_hash(m, i)
    def substream(self, m, t): return self.lib.oracle_substream(m, t)
    def hash_state(self, v, l, mult=DEFAULT_MULT): return self.lib.oracle_hash_state(mult, v, l)
    def scaled_index(self, raw, d): return self.lib.oracle_scaled_index(raw, d)

    # -- walks
    def random_walk(self, off, adj, start, length, seed, mult=DEFAULT_MULT):
        out = np.zeros(length, np.uint32)
        self.lib.oracle_random_walk(_p(off, u32p), _p(adj, u32p), start, length, seed, mult,
                                    _p(out, u32p))
        return out

    def campaign_counts(self, off, adj, K=0, length=10, master=42, mult=DEFAULT_MULT,
                        k_per_vertex=None, threads=0):
        n = len(off) - 1
        out = np.zeros(n, np.uint64)
        kpv = None if k_per_vertex is None else np.ascontiguousarray(k_per_vertex, np.uint64)
        self.lib.oracle_campaign_counts(_p(off, u32p), _p(adj, u32p), n, _p(kpv, u64p), K, length,
                                        master, mult, threads, _p(out, u64p))
        return out

    def campaign_range(self, off, adj, r0, r1, K=0, length=10, master=42, mult=DEFAULT_MULT,
                       k_per_vertex=None):
        n = len(off) - 1
        out = np.zeros(n, np.uint64)
        kpv = None if k_per_vertex is None else np.ascontiguousarray(k_per_vertex, np.uint64)
        self.lib.oracle_campaign_range(_p(off, u32p), _p(adj, u32p), n, _p(kpv, u64p), K, length,
                                       master, mult, r0, r1, _p(out, u64p))
        return out

    def uniform_start_counts(self, n, W, master=42):
        out = np.zeros(n, np.uint64)
        self.lib.oracle_uniform_start_counts(n, W, master, _p(out, u64p))
        return out

    # -- aesc pieces
    def is_connected(self, off, adj):
        return bool(self.lib.oracle_is_connected(_p(off, u32p), _p(adj, u32p), len(off) - 1))

    def slot_edges(self, off, adj):
        out = np.zeros(len(adj), np.uint32)
        self.lib.oracle_slot_edges(_p(off, u32p), _p(adj, u32p), len(off) - 1, _p(out, u32p))
        return out

    def truncated_lengths(self, off, adj, eps, omega=30, tau_max=128, per_edge=False):
        m = len(adj) // 2
        tau = np.zeros(m, np.uint32)
        lam = C.c_double()
        cl = C.c_int()
        rc = self.lib.oracle_truncated_lengths(_p(off, u32p), _p(adj, u32p), len(off) - 1, m, eps,
                                               omega, tau_max, int(per_edge), _p(tau, u32p),
                                               C.byref(lam), C.byref(cl))
        _raise(rc, "truncated_lengths")
        return tau, lam.value, bool(cl.value)

    def walks_needed_raw(self, tau_eff, eps, delta, d, m):
        return self.lib.oracle_walks_needed_raw(tau_eff, eps, delta, d, m)

    def walk_budget(self, tau_eff, eps, delta, d, m):
        out = C.c_uint64()
        _raise(self.lib.oracle_walk_budget(tau_eff, eps, delta, d, m, C.byref(out)), "walk_budget")
        return out.value

    def propagate(self, off, adj, source, tau, eps, delta, cap=-1):
        n = len(off) - 1
        m = len(adj) // 2
        se = self.slot_edges(off, adj)
        prob = np.zeros(n, np.float64)
        depth = C.c_uint32()
        tau = np.ascontiguousarray(tau, np.uint32)
        self.lib.oracle_propagate(_p(off, u32p), _p(adj, u32p), n, m, source, _p(tau, u32p),
                                  _p(se, u32p), eps, delta, cap, _p(prob, f64p), C.byref(depth))
        return prob, depth.value

    def aesc(self, off, adj, epsilon=0.05, delta=0.05, power_iterations=30, master_seed=42,
             max_truncation=128, per_edge_tau=False, switch_depth_cap=-1,
             hash_multiplier=DEFAULT_MULT, threads=0, sources=None) -> AescResult:
        n = len(off) - 1
        m = len(adj) // 2
        cfg = _OracleCfg(epsilon, delta, power_iterations, master_seed, max_truncation,
                         int(per_edge_tau), switch_depth_cap, hash_multiplier, threads)
        g = np.zeros(2 * m, np.float64)
        s = np.zeros(m, np.float64) if sources is None else None
        tau = np.zeros(m, np.uint32)
        tt = np.zeros(n, np.uint32)
        lam = C.c_double()
        pairs = C.c_uint64()
        steps = C.c_uint64()
        src = None if sources is None else np.ascontiguousarray(sources, np.uint32)
        rc = self.lib.oracle_aesc(_p(off, u32p), _p(adj, u32p), n, m, C.byref(cfg), _p(src, u32p),
                                  0 if src is None else len(src), _p(g, f64p), _p(s, f64p),
                                  _p(tau, u32p), _p(tt, u32p), C.byref(lam), C.byref(pairs),
                                  C.byref(steps))
        _raise(rc, "aesc")
        return AescResult(g, s, tau, tt, lam.value, pairs.value, steps.value)


def _raise(rc, what, msg=""):
    if rc == 1:
        raise ValueError(f"{what}: invalid argument {msg}")
    if rc == 2:
        raise RuntimeError(f"{what}: data error {msg}")
    if rc:
        raise RuntimeError(f"{what}: error {rc} {msg}")


class RefGraph:
    def __init__(self, ref: "Reference", handle):
        self.ref, self.h = ref, handle

    def __del__(self):
        try:
            self.ref.lib.ref_graph_free(self.h)
        except Exception:
            pass

    @property
    def n(self): return self.ref.lib.ref_graph_n(self.h)

    @property
    def m(self): return self.ref.lib.ref_graph_m(self.h)

    def csr(self):
        off = np.zeros(self.n + 1, np.uint32)
        adj = np.zeros(2 * self.m, np.uint32)
        se = np.zeros(2 * self.m, np.uint32)
        self.ref.lib.ref_graph_csr(self.h, _p(off, u32p), _p(adj, u32p), _p(se, u32p))
        return off, adj, se

    def edges(self):
        uv = np.zeros(2 * self.m, np.uint32)
        self.ref.lib.ref_graph_edges(self.h, _p(uv, u32p))
        return uv.reshape(-1, 2)


class Reference:
    """The unmodified reference headers behind oracle/ref_driver.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.lib = L
        L.ref_last_error.restype = C.c_char_p
        vpp = C.POINTER(C.c_void_p)
        L.ref_graph_from_edges.argtypes = [C.c_uint32, u32p, C.c_uint64, vpp]
        L.ref_graph_from_csr.argtypes = [C.c_uint32, u32p, u32p, vpp]
        L.ref_gen_scale_free.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, vpp]
        L.ref_gen_random_connected.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, vpp]
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_graph_n.restype = C.c_uint32
        L.ref_graph_n.argtypes = [C.c_void_p]
        L.ref_graph_m.restype = C.c_uint64
        L.ref_graph_m.argtypes = [C.c_void_p]
        L.ref_graph_csr.argtypes = [C.c_void_p, u32p, u32p, u32p]
        L.ref_graph_edges.argtypes = [C.c_void_p, u32p]
        L.ref_random_walk.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                      u32p]
        L.ref_random_bouquet.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_uint64, C.c_uint64, u32p, u32p]
        L.ref_campaign.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_uint32,
                                   C.c_int, C.c_uint64, C.c_uint64, u64p, f64p, u64p]
        L.ref_campaign_kv.argtypes = [C.c_void_p, u64p, C.c_uint64, C.c_uint32, C.c_int,
                                      C.c_uint32, C.c_int, C.c_uint64, C.c_uint64, C.c_uint32,
                                      C.c_uint32, u64p, f64p, u64p]
        L.ref_campaign_stats.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_uint32,
                                         C.c_int, C.c_uint64, C.c_uint64, u64p, u64p, u64p, f64p, f64p]
        L.ref_max_threads.restype = C.c_int
        L.ref_walk_budget.argtypes = [C.c_uint32, C.c_double, C.c_double, C.c_uint32, C.c_uint64,
                                      u64p]
        L.ref_truncated_lengths.argtypes = [C.c_void_p, C.c_double, C.c_uint32, C.c_uint32,
                                            C.c_int, u32p, f64p, C.POINTER(C.c_int)]
        L.ref_propagate.argtypes = [C.c_void_p, C.c_uint32, u32p, C.c_double, C.c_double,
                                    C.c_int64, f64p, u32p]
        L.ref_estimate_edge.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, f64p, C.c_uint32,
                                        C.c_uint32, C.c_uint64, C.c_int, C.c_uint64, C.c_uint32,
                                        C.c_uint64, f64p]
        L.ref_aesc.argtypes = [C.c_void_p, C.POINTER(_RefCfg), f64p, f64p, u32p, u32p, f64p,
                               u64p, u64p, f64p]
        L.ref_aesc_sources.argtypes = [C.c_void_p, C.POINTER(_RefCfg), u32p, C.c_uint64, f64p,
                                       u32p, u32p, f64p, u64p, u64p, f64p, f64p]

    def _chk(self, rc, what):
        if rc:
            _raise(rc, what, self.lib.ref_last_error().decode())

    def _graph(self, fn, *args):
        h = C.c_void_p()
        self._chk(fn(*args, C.byref(h)), fn.__name__)
        return RefGraph(self, h)

    def from_edges(self, n_hint, pairs):
        pairs = np.ascontiguousarray(np.asarray(pairs, np.uint32).reshape(-1, 2))
        return self._graph(self.lib.ref_graph_from_edges, n_hint, _p(pairs, u32p), len(pairs))

    def from_csr(self, off, adj):
        return self._graph(self.lib.ref_graph_from_csr, len(off) - 1, _p(off, u32p),
                           _p(adj, u32p))

    def scale_free(self, n, attach, seed):
        return self._graph(self.lib.ref_gen_scale_free, n, attach, seed)

    def random_connected(self, n, extra, seed):
        return self._graph(self.lib.ref_gen_random_connected, n, extra, seed)

    def max_threads(self):
        return self.lib.ref_max_threads()

    def random_walk(self, g, start, length, seed, mult=DEFAULT_MULT):
        out = np.zeros(length, np.uint32)
        self._chk(self.lib.ref_random_walk(g.h, start, length, seed, mult, _p(out, u32p)),
                  "random_walk")
        return out

    def random_bouquet(self, g, start, length, width, master, mult=DEFAULT_MULT):
        seeds = np.zeros(width, np.uint32)
        paths = np.zeros((width, length), np.uint32)
        self._chk(self.lib.ref_random_bouquet(g.h, start, length, width, master, mult,
                                              _p(seeds, u32p), _p(paths, u32p)), "random_bouquet")
        return seeds, paths

    def campaign(self, g, K, L, mode=3, lanes=8, threads=0, master=42, mult=DEFAULT_MULT):
        out = np.zeros(g.n, np.uint64)
        sec = C.c_double()
        steps = C.c_uint64()
        self._chk(self.lib.ref_campaign(g.h, K, L, mode, lanes, threads, master, mult,
                                        _p(out, u64p), C.byref(sec), C.byref(steps)), "campaign")
        return out, sec.value, steps.value

    def rng_stream(self, g, starts, K, L, selector=2, master=42, mult=DEFAULT_MULT):
        st = np.ascontiguousarray(starts, np.uint32)
        words = np.zeros(max(len(st) * K * max(L - 1, 0), 1), np.uint32)
        nw = C.c_uint64()
        fn = self.lib.ref_rng_stream
        fn.argtypes = [C.c_void_p, u32p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_int, C.c_uint64,
                       C.c_uint64, u32p, u64p]
        self._chk(fn(g.h, _p(st, u32p), len(st), K, L, selector, master, mult, _p(words, u32p),
                     C.byref(nw)), "rng_stream")
        return words[: nw.value]

    def campaign_stats(self, g, K, L, mode=3, lanes=8, threads=0, master=42, mult=DEFAULT_MULT):
        hist = np.zeros(lanes + 1, np.uint64)
        step = np.zeros(L - 1, np.uint64)
        out4 = np.zeros(4, np.uint64)
        md = C.c_double()
        mean = C.c_double()
        self._chk(self.lib.ref_campaign_stats(g.h, K, L, mode, lanes, threads, master, mult,
                                              _p(hist, u64p), _p(step, u64p), _p(out4, u64p),
                                              C.byref(md), C.byref(mean)), "campaign_stats")
        return hist, step, int(out4[0]), int(out4[1]), md.value, mean.value

    def campaign_kv(self, g, L, W=0, k_per_vertex=None, sorted_=True, lanes=8, threads=0,
                    master=42, mult=DEFAULT_MULT, vertex_stride=1, vertex_phase=0):
        out = np.zeros(g.n, np.uint64)
        sec = C.c_double()
        steps = C.c_uint64()
        kpv = None if k_per_vertex is None else np.ascontiguousarray(k_per_vertex, np.uint64)
        self._chk(self.lib.ref_campaign_kv(g.h, _p(kpv, u64p), W, L, int(sorted_), lanes, threads,
                                           master, mult, vertex_stride, vertex_phase,
                                           _p(out, u64p), C.byref(sec), C.byref(steps)),
                  "campaign_kv")
        return out, sec.value, steps.value

    def walk_budget(self, tau_eff, eps, delta, d, m):
        out = C.c_uint64()
        self._chk(self.lib.ref_walk_budget(tau_eff, eps, delta, d, m, C.byref(out)), "walk_budget")
        return out.value

    def truncated_lengths(self, g, eps, omega=30, tau_max=128, per_edge=False):
        tau = np.zeros(g.m, np.uint32)
        lam = C.c_double()
        cl = C.c_int()
        self._chk(self.lib.ref_truncated_lengths(g.h, eps, omega, tau_max, int(per_edge),
                                                 _p(tau, u32p), C.byref(lam), C.byref(cl)),
                  "truncated_lengths")
        return tau, lam.value, bool(cl.value)

    def propagate(self, g, source, tau, eps, delta, cap=-1):
        prob = np.zeros(g.n, np.float64)
        depth = C.c_uint32()
        tau = np.ascontiguousarray(tau, np.uint32)
        self._chk(self.lib.ref_propagate(g.h, source, _p(tau, u32p), eps, delta, cap,
                                         _p(prob, f64p), C.byref(depth)), "propagate")
        return prob, depth.value

    def estimate_edge(self, g, vi, vj, prob_dense, depth, tau_eff, n_req, mode=3, edge_seed=1,
                      lanes=8, mult=DEFAULT_MULT):
        out = C.c_double()
        prob_dense = np.ascontiguousarray(prob_dense, np.float64)
        self._chk(self.lib.ref_estimate_edge(g.h, vi, vj, _p(prob_dense, f64p), depth, tau_eff,
                                             n_req, mode, edge_seed, lanes, mult, C.byref(out)),
                  "estimate_edge")
        return out.value

    def _cfg(self, epsilon, delta, power_iterations, master_seed, max_truncation, per_edge_tau,
             switch_depth_cap, hash_multiplier, threads, mode, lanes):
        return _RefCfg(epsilon, delta, power_iterations, master_seed, max_truncation,
                       int(per_edge_tau), switch_depth_cap, hash_multiplier, threads, mode, lanes)

    def aesc(self, g, epsilon=0.05, delta=0.05, power_iterations=30, master_seed=42,
             max_truncation=128, per_edge_tau=False, switch_depth_cap=-1,
             hash_multiplier=DEFAULT_MULT, threads=0, mode=3, lanes=8, sources=None):
        cfg = self._cfg(epsilon, delta, power_iterations, master_seed, max_truncation,
                        per_edge_tau, switch_depth_cap, hash_multiplier, threads, mode, lanes)
        n, m = g.n, g.m
        gh = np.zeros(2 * m, np.float64)
        tau = np.zeros(m, np.uint32)
        tt = np.zeros(n, np.uint32)
        lam = C.c_double()
        pairs = C.c_uint64()
        steps = C.c_uint64()
        sec = C.c_double()
        if sources is None:
            sh = np.zeros(m, np.float64)
            self._chk(self.lib.ref_aesc(g.h, C.byref(cfg), _p(gh, f64p), _p(sh, f64p),
                                        _p(tau, u32p), _p(tt, u32p), C.byref(lam), C.byref(pairs),
                                        C.byref(steps), C.byref(sec)), "aesc")
            return AescResult(gh, sh, tau, tt, lam.value, pairs.value, steps.value, sec.value)
        src = np.ascontiguousarray(sources, np.uint32)
        psec = C.c_double()
        self._chk(self.lib.ref_aesc_sources(g.h, C.byref(cfg), _p(src, u32p), len(src),
                                            _p(gh, f64p), _p(tau, u32p), _p(tt, u32p),
                                            C.byref(lam), C.byref(pairs), C.byref(steps),
                                            C.byref(sec), C.byref(psec)), "aesc_sources")
        return AescResult(gh, None, tau, tt, lam.value, pairs.value, steps.value, sec.value,
                          psec.value)


def reference_available() -> bool:
    return os.path.exists(REF_SO)
