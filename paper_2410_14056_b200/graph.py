"""Graph: immutable CSR of a simple undirected graph (graph.hpp:28-247).

Host CSR arrays are numpy; device replicas (K0: packed {base, degree} +
adjacency) are created lazily per CUDA device through the C ABI and cached,
mirroring the immutability contract of the reference (graph.hpp:24-27).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L


class _HostCsr:
    """Owns a saba_hgraph handle; the numpy views of its CSR keep it alive
    (no copy of the up-to-GB adjacency out of the library)."""

    def __init__(self, h):
        self.h = h
        self._free = L.lib().saba_hgraph_free  # bound now: usable during interpreter shutdown

    def __del__(self):
        if self.h:
            self._free(self.h)
            self.h = None

    def view(self, ptr, count):
        if count == 0:
            return np.zeros(0, np.uint32)
        buf = (C.c_uint32 * count).from_address(C.addressof(ptr.contents))
        buf._owner = self  # the ctypes buffer (the array's base) pins the handle
        return np.frombuffer(buf, dtype=np.uint32)


def _from_handle(h) -> "Graph":
    lib = L.lib()
    owner = _HostCsr(h)
    n = lib.saba_hgraph_vertex_count(h)
    m = lib.saba_hgraph_edge_count(h)
    po, pa = L.u32p(), L.u32p()
    L.check(lib.saba_hgraph_data(h, C.byref(po), C.byref(pa)), "csr")
    return Graph(owner.view(po, n + 1), owner.view(pa, 2 * m), _trusted=True)


def _gen(fn, *args) -> "Graph":
    h = C.c_void_p()
    L.check(fn(*args, C.byref(h)), fn.__name__)
    return _from_handle(h)


class Graph:
    """CSR graph with the reference's accessors (graph.hpp:30-80)."""

    def __init__(self, offsets, adjacency, _trusted: bool = False):
        off = np.ascontiguousarray(offsets, dtype=np.uint32)
        adj = np.ascontiguousarray(adjacency, dtype=np.uint32)
        if not _trusted:
            h = C.c_void_p()
            L.check(L.lib().saba_hgraph_from_csr(len(off) - 1, L.ptr(off, L.u32p),
                                                 L.ptr(adj, L.u32p), C.byref(h)), "from_csr")
            L.lib().saba_hgraph_free(h)
        self.offsets = off
        self.adjacency = adj
        self._dev = {}
        self._slot_edge = None

    # -- construction (graph.hpp:86-105; gen.hpp; BASELINE generators)
    @staticmethod
    def from_edges(n_hint: int, pairs, device: int | None = None, keep_lcc: bool = False) -> "Graph":
        """graph.hpp:86-105. device=None canonicalises on the host; a CUDA
        device index runs the device pipeline (graph_build.cu), which returns
        the identical CSR; keep_lcc additionally keeps the largest component."""
        p = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint32).reshape(-1, 2))
        if device is not None:
            return _gen(L.lib().saba_cu_graph_from_edges, n_hint, L.ptr(p, L.u32p), len(p),
                        int(keep_lcc), int(device))
        g = _gen(L.lib().saba_hgraph_from_edges, n_hint, L.ptr(p, L.u32p), len(p))
        return largest_component(g) if keep_lcc else g

    @staticmethod
    def from_csr(offsets, adjacency) -> "Graph":
        return Graph(offsets, adjacency)

    # -- accessors
    def vertex_count(self) -> int:
        return len(self.offsets) - 1

    def edge_count(self) -> int:
        return len(self.adjacency) // 2

    @property
    def n(self) -> int:
        return self.vertex_count()

    @property
    def m(self) -> int:
        return self.edge_count()

    def degree(self, u: int) -> int:
        if not 0 <= u < self.n:
            raise ValueError("degree: vertex out of range")
        return int(self.offsets[u + 1] - self.offsets[u])

    def degrees(self) -> np.ndarray:
        return np.diff(self.offsets).astype(np.uint32)

    def neighbors(self, u: int) -> np.ndarray:
        if not 0 <= u < self.n:
            raise ValueError("neighbors: vertex out of range")
        return self.adjacency[self.offsets[u]:self.offsets[u + 1]]

    def has_edge(self, u: int, v: int) -> bool:
        nb = self.neighbors(u)
        i = np.searchsorted(nb, v)
        return bool(i < len(nb) and nb[i] == v)

    def slot_of(self, u: int, v: int) -> int:
        nb = self.neighbors(u)
        i = int(np.searchsorted(nb, v))
        if i >= len(nb) or nb[i] != v:
            raise ValueError("slot_of: not an edge")
        return int(self.offsets[u]) + i

    def max_degree(self) -> int:
        return int(self.degrees().max()) if self.n else 0

    def edges(self) -> np.ndarray:
        """(m, 2) endpoints u < v in edge-id order (graph.hpp:75, 92-100)."""
        deg = self.degrees()
        u = np.repeat(np.arange(self.n, dtype=np.uint32), deg)
        keep = self.adjacency > u
        return np.stack([u[keep], self.adjacency[keep]], axis=1)

    def slot_edges(self) -> np.ndarray:
        """Directed slot -> undirected edge id (graph.hpp:72)."""
        if self._slot_edge is None:
            deg = self.degrees()
            u = np.repeat(np.arange(self.n, dtype=np.int64), deg)
            a = self.adjacency.astype(np.int64)
            fwd = a > u
            se = np.zeros(len(a), np.uint32)
            se[fwd] = np.arange(int(fwd.sum()), dtype=np.uint32)
            # reverse slot (v->u) takes the id of (u->v): position of u in v's slice
            rev = np.nonzero(~fwd)[0]
            key_fwd = u[fwd] * self.n + a[fwd]  # sorted ascending (CSR order)
            key_rev = a[rev] * self.n + u[rev]
            se[rev] = se[fwd][np.searchsorted(key_fwd, key_rev)]
            self._slot_edge = se
        return self._slot_edge

    def is_connected(self) -> bool:
        from .aesc import _is_connected
        return _is_connected(self)

    def nbytes(self) -> int:
        return self.offsets.nbytes + self.adjacency.nbytes

    # -- device replicas (K0)
    def device_handle(self, device: int = 0):
        h = self._dev.get(device)
        if h is None:
            h = C.c_void_p()
            L.check(L.lib().saba_cu_graph_create(L.ptr(self.offsets, L.u32p),
                                                 L.ptr(self.adjacency, L.u32p), self.n,
                                                 len(self.adjacency), device, C.byref(h)),
                    "graph_create")
            self._dev[device] = h
        return h

    def device_group(self, devices) -> C.c_void_p:
        """One replica per entry of `devices` behind a single handle
        (saba_cu_graph_create_multi; repeats = logical shards on one GPU).
        Campaigns and AESC on it run one shard per replica and combine once;
        results are identical to one device."""
        devices = tuple(int(d) for d in devices)
        if len(devices) == 1:
            return self.device_handle(devices[0])
        h = self._dev.get(devices)
        if h is None:
            h = C.c_void_p()
            arr = (C.c_int * len(devices))(*devices)
            L.check(L.lib().saba_cu_graph_create_multi(L.ptr(self.offsets, L.u32p),
                                                       L.ptr(self.adjacency, L.u32p), self.n,
                                                       len(self.adjacency), arr, len(devices),
                                                       C.byref(h)), "graph_create_multi")
            self._dev[devices] = h
        return h

    def release_device(self) -> None:
        for h in self._dev.values():
            L.lib().saba_cu_graph_destroy(h)
        self._dev.clear()

    def __del__(self):
        try:
            self.release_device()
        except Exception:
            pass

    def __repr__(self) -> str:
        return f"Graph(n={self.n}, m={self.m})"


# -- generators ------------------------------------------------------------
def make_erdos_renyi(n: int, m: int, seed: int) -> Graph:
    """G(n, m) with exactly m distinct non-loop pairs (BASELINE config 1)."""
    return _gen(L.lib().saba_gen_erdos_renyi, n, m, seed)


def make_rmat(scale: int, edge_factor: int, a: float = 0.57, b: float = 0.19, c: float = 0.19,
              seed: int = 1, keep_lcc: bool = True, device: int | None = None) -> Graph:
    """R-MAT, symmetrised/deduplicated/loop-free, LCC (BASELINE configs 2-4).
    device: build on that CUDA device (same graph, bit for bit)."""
    if device is not None:
        return _gen(L.lib().saba_cu_gen_rmat, scale, edge_factor, a, b, c, seed, int(keep_lcc),
                    int(device))
    return _gen(L.lib().saba_gen_rmat, scale, edge_factor, a, b, c, seed, int(keep_lcc))


def make_chung_lu(n: int, gamma: float = 2.2, mean_degree: float = 78.0,
                  max_degree: float = 30000.0, seed: int = 1, keep_lcc: bool = True,
                  device: int | None = None) -> Graph:
    """Chung–Lu power law, LCC (BASELINE config 5). device: build on that CUDA
    device (alias table on the host, samples/canonicalisation/LCC on the GPU)."""
    if device is not None:
        return _gen(L.lib().saba_cu_gen_chung_lu, n, gamma, mean_degree, max_degree, seed,
                    int(keep_lcc), int(device))
    return _gen(L.lib().saba_gen_chung_lu, n, gamma, mean_degree, max_degree, seed, int(keep_lcc))


def make_scale_free(n: int, attach: int, seed: int) -> Graph:
    """gen.hpp:17-44."""
    return _gen(L.lib().saba_gen_scale_free, n, attach, seed)


def make_random_connected(n: int, extra: int, seed: int) -> Graph:
    """gen.hpp:48-69."""
    return _gen(L.lib().saba_gen_random_connected, n, extra, seed)


def largest_component(g: Graph) -> Graph:
    h = C.c_void_p()
    hin = C.c_void_p()
    L.check(L.lib().saba_hgraph_from_csr(g.n, L.ptr(g.offsets, L.u32p), L.ptr(g.adjacency, L.u32p),
                                         C.byref(hin)), "from_csr")
    try:
        L.check(L.lib().saba_hgraph_largest_component(hin, C.byref(h)), "largest_component")
    finally:
        L.lib().saba_hgraph_free(hin)
    return _from_handle(h)


# named test graphs (tests/support/graphs.hpp:15-60)
def triangle() -> Graph: return Graph.from_edges(3, [(0, 1), (1, 2), (0, 2)])
def path(n: int) -> Graph: return Graph.from_edges(n, [(v, v + 1) for v in range(n - 1)])
def star(leaves: int) -> Graph: return Graph.from_edges(leaves + 1, [(0, v) for v in range(1, leaves + 1)])
def complete(n: int) -> Graph: return Graph.from_edges(n, [(u, v) for u in range(n) for v in range(u + 1, n)])
def fig1() -> Graph: return Graph.from_edges(4, [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)])


def grid3x3() -> Graph:
    e = []
    for r in range(3):
        for c in range(3):
            v = 3 * r + c
            if c + 1 < 3:
                e.append((v, v + 1))
            if r + 1 < 3:
                e.append((v, v + 3))
    return Graph.from_edges(9, e)


def petersen() -> Graph:
    e = []
    for i in range(5):
        e += [(i, (i + 1) % 5), (i, i + 5), (5 + i, 5 + (i + 2) % 5)]
    return Graph.from_edges(10, e)
