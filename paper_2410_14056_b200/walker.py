"""Walk engine front end: the reference's walker.hpp / rng.hpp API over the
sm_100a kernels (include/saba_cuda.h).

Reference surface mirrored (walker.hpp / rng.hpp line numbers):
  WalkMode 30, SelectorKind rng.hpp:65, HashSpec rng.hpp:20-31, SeedSet /
  gen_seeds / gen_sorted_seeds rng.hpp:97-123, Walk 54-58, random_walk 283-302,
  random_bouquet 306-338, VisitCountSink 352-365, CampaignConfig 367-376,
  CampaignReport 383-391, run_walk_campaign 456-538.
Saba and Hash run the same kernels (they produce identical walks,
walker.hpp:25-26); Naive / VectorMod are CPU LCG baselines with different
walks and are rejected (ValueError) — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .graph import Graph

DEFAULT_HASH_MULTIPLIER = 0xC6A4A7935BD1E995
START_TAG = 0x5354415254  # uniform-start stream tag


class WalkMode(enum.IntEnum):
    Naive = 0
    VectorMod = 1
    Hash = 2
    Saba = 3


class SelectorKind(enum.IntEnum):
    NaiveMod = 0
    XorMod = 1
    Scaled = 2


@dataclass
class HashSpec:
    multiplier: int = DEFAULT_HASH_MULTIPLIER

    def state(self, vertex: int, step: int) -> int:
        return int(hash_state(np.uint32(vertex), np.uint32(step), self.multiplier))


# -- vectorised host restatements of the integer primitives (common.hpp:24-41,
#    rng.hpp:23-30, 61-63); used for seed sets and cheap host-side bookkeeping.
_M64 = (1 << 64) - 1


def mix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def counter_hash(master, index):
    with np.errstate(over="ignore"):
        i = np.asarray(index, dtype=np.uint64)
        return mix64(np.uint64(master) + (i + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15))


def substream(master, tag):
    with np.errstate(over="ignore"):
        return mix64(np.uint64(master) ^ mix64(np.asarray(tag, np.uint64) + np.uint64(0x632BE59BD9B4E019)))


def hash_state(vertex, step, multiplier=DEFAULT_HASH_MULTIPLIER):
    with np.errstate(over="ignore"):
        x = (np.asarray(vertex, np.uint64) << np.uint64(32)) | np.asarray(step, np.uint64)
        mu = np.uint64(multiplier)
        x = x * mu
        x ^= x >> np.uint64(47)
        x = x * mu
        x ^= x >> np.uint64(47)
        return (x >> np.uint64(32)).astype(np.uint32)


def scaled_index(raw, degree):
    return ((np.asarray(raw, np.uint64) * np.asarray(degree, np.uint64)) >> np.uint64(32)).astype(np.uint32)


class SeedOrdering(enum.IntEnum):
    AsGenerated = 0
    Sorted = 1


@dataclass
class SeedSet:
    seeds: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    ordering: SeedOrdering = SeedOrdering.AsGenerated
    master_seed: int = 0


def gen_seeds(count: int, master_seed: int, ordering: SeedOrdering) -> SeedSet:
    """rng.hpp:108-117: seed_i = counter_hash(master, i) >> 32."""
    if count < 1:
        raise ValueError("gen_seeds: count must be >= 1")
    s = (counter_hash(master_seed, np.arange(count, dtype=np.uint64)) >> np.uint64(32)).astype(np.uint32)
    if ordering == SeedOrdering.Sorted:
        s = np.sort(s)
    return SeedSet(s, ordering, master_seed)


def gen_sorted_seeds(count: int, master_seed: int) -> SeedSet:
    return gen_seeds(count, master_seed, SeedOrdering.Sorted)


@dataclass
class Walk:
    vertices: np.ndarray
    walk_id: int = 0
    seed: int = 0


def _require_scaled(selector: SelectorKind) -> None:
    if selector != SelectorKind.Scaled:
        raise ValueError("selector not supported on GPU (only the Bouquets scaled-hash selector)")


def walk_paths(g: Graph, starts, seeds, length: int, hash: HashSpec = HashSpec(),
               device: int = 0) -> np.ndarray:
    """Materialise many walks at once: paths[i, l] (K2 without the sink)."""
    st = np.ascontiguousarray(starts, np.uint32)
    sd = np.ascontiguousarray(seeds, np.uint32)
    if st.shape != sd.shape:
        raise ValueError("starts and seeds must have the same length")
    if length < 1:
        raise ValueError("walk length must be >= 1")
    out = np.zeros((len(st), length), np.uint32)
    L.check(L.lib().saba_cu_walk_paths(g.device_handle(device), L.ptr(st, L.u32p), L.ptr(sd, L.u32p),
                                       len(st), length, hash.multiplier, L.ptr(out, L.u32p)),
            "walk_paths")
    return out


def random_walk(g: Graph, start: int, length: int, selector: SelectorKind, seed: int,
                hash: HashSpec = HashSpec(), device: int = 0) -> Walk:
    """walker.hpp:283-302."""
    _require_scaled(selector)
    p = walk_paths(g, [start], [seed], length, hash, device)
    return Walk(p[0], 0, seed)


def random_bouquet(g: Graph, start: int, length: int, width: int, seeds: SeedSet,
                   selector: SelectorKind, hash: HashSpec = HashSpec(), device: int = 0):
    """walker.hpp:306-338: width lockstep walks from `start`, one per seed."""
    if not 1 <= width <= 64:
        raise ValueError("bouquet width must be in [1, 64]")
    if len(seeds.seeds) < width:
        raise ValueError("seed set smaller than bouquet width")
    _require_scaled(selector)
    sd = np.asarray(seeds.seeds[:width], np.uint32)
    p = walk_paths(g, np.full(width, start, np.uint32), sd, length, hash, device)
    return [Walk(p[b], b, int(sd[b])) for b in range(width)]


class VisitCountSink:
    """walker.hpp:352-365: per-vertex uint64 visit counts."""

    def __init__(self, n: int):
        self.counts = np.zeros(n, np.uint64)


@dataclass
class CampaignConfig:
    walks_per_vertex: int = 2048
    length: int = 10
    mode: WalkMode = WalkMode.Saba
    lanes: int = 8
    threads: int = 0
    master_seed: int = 42
    collect_stats: bool = False
    hash: HashSpec = field(default_factory=HashSpec)


@dataclass
class BranchingStats:
    """walker.hpp:111-118."""
    lanes: int = 0
    histogram: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    samples: int = 0
    mean: float = 0.0
    p1: int = 0
    p10: int = 0
    p25: int = 0
    mean_candidate_degree: float = 0.0


@dataclass
class DistinctProxy:
    per_step: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    total: int = 0


def branching_stats(histogram) -> BranchingStats:
    """Percentiles (ceil(q * total)-th, 1-based) and mean of a distinct-lanes
    histogram (walker.hpp:122-151)."""
    h = np.asarray(histogram, np.uint64)
    total = int(h.sum())
    if total == 0:
        raise ValueError("branching_stats: empty trace")
    weighted = 0.0
    for c, x in enumerate(h):  # same accumulation order as the reference
        weighted += float(c) * float(x)
    cum = np.cumsum(h.astype(np.int64))

    def pct(q):
        rank = max(1, int(np.ceil(q * float(total))))
        return int(np.searchsorted(cum, rank))

    return BranchingStats(max(len(h) - 1, 0), h.copy(), total, weighted / float(total),
                          pct(0.01), pct(0.10), pct(0.25))


@dataclass
class CampaignReport:
    seconds: float = 0.0
    total_steps: int = 0
    total_events: int = 0
    threads_used: int = 1
    has_stats: bool = False
    walk_kernel_ms: float = 0.0
    launches: int = 0
    shard_walks: int = 0
    kernel: str = ""  # K2 variant that ran (SABA_K2_* in include/saba_cuda.h)
    branching: BranchingStats | None = None
    proxy: DistinctProxy | None = None


K2_KERNELS = {0: "", 1: "walk_count_kernel", 2: "walk_count_fat_kernel", 3: "walk_count_hot_kernel",
              4: "walk_count_rank_kernel", 5: "walk_count_fat_priv_kernel"}


def _cfg_c(cfg: CampaignConfig, total_walks: int, shard_index: int, shard_count: int):
    return L.CampaignConfigC(cfg.walks_per_vertex if not total_walks else 0, total_walks, cfg.length,
                             cfg.lanes, int(cfg.mode), cfg.threads, cfg.master_seed,
                             cfg.hash.multiplier, shard_index, shard_count)


def _report(r: L.CampaignReportC) -> CampaignReport:
    return CampaignReport(r.seconds, r.total_steps, r.total_events, 1, False, r.walk_kernel_ms,
                          r.launches, r.shard_walks, K2_KERNELS.get(r.kernel, str(r.kernel)))


class _PinnedCounts:
    """A page-locked uint64[n] landing buffer (saba_cu_pinned_alloc): the
    campaign's counts arrive by direct DMA instead of a staged copy."""

    def __init__(self, n: int):
        self.n = n
        p = C.c_void_p()
        L.check(L.lib().saba_cu_pinned_alloc(8 * max(n, 1), C.byref(p)), "pinned_alloc")
        self._p = p
        self.array = np.frombuffer((C.c_uint64 * max(n, 1)).from_address(p.value), dtype=np.uint64)[:n]

    def __del__(self):
        try:
            self.array = None
            L.lib().saba_cu_pinned_free(self._p)
        except Exception:  # interpreter shutdown
            pass


_scratch = threading.local()


def _scratch_counts(n: int) -> np.ndarray:
    """Per-thread landing buffer for a campaign's counts, page-locked and
    reused from call to call (every entry is rewritten by each call)."""
    buf = getattr(_scratch, "buf", None)
    if buf is None or buf.n != n:
        buf = _PinnedCounts(n)
        _scratch.buf = buf
    return buf.array


def run_walk_campaign(g: Graph, cfg: CampaignConfig, sink: VisitCountSink, *,
                      total_walks: int = 0, shard_index: int = 0, shard_count: int = 1,
                      device: int = 0, devices=None) -> CampaignReport:
    """walker.hpp:456-538 on one B200.

    total_walks > 0 selects the uniform-random-start campaign
    instead of `walks_per_vertex` walks from every vertex. With sharding,
    only walk range `shard_index` of `shard_count` runs; the shards' counts
    sum to the unsharded counts exactly. `devices` (a list, repeats allowed)
    spreads the call over one replica per entry (Graph.device_group), one
    shard each, combined on the first: identical counts.
    """
    if not isinstance(sink, VisitCountSink):
        raise TypeError("the GPU campaign supports VisitCountSink only")
    if len(sink.counts) != g.n:
        raise ValueError("sink size != vertex count")
    counts = _scratch_counts(g.n)  # every entry is written by the call
    rep = L.CampaignReportC()
    c = _cfg_c(cfg, total_walks, shard_index, shard_count)
    h = g.device_group(devices) if devices is not None else g.device_handle(device)
    L.check(L.lib().saba_cu_walk_campaign(h, C.byref(c), L.ptr(counts, L.u64p), C.byref(rep)),
            "walk_campaign")
    np.add(sink.counts, counts, out=sink.counts)  # VisitCountSink::absorb (walker.hpp:360-364)
    out = _report(rep)
    # the reference collects stats in lane modes with L > 1 (walker.hpp:471)
    if cfg.collect_stats and cfg.length > 1:
        out.branching, out.proxy = collect_branching(g, cfg, total_walks=total_walks,
                                                     device=device)
        out.has_stats = True
    return out


def rng_stream(g: Graph, starts, walks_per_vertex: int = 1, length: int = 2,
               selector: SelectorKind = SelectorKind.Scaled, master_seed: int = 42,
               hash: HashSpec = HashSpec(), device: int = 0) -> bytes:
    """stream.hpp:29-83: the raw pre-selection words seed ^ h(cur, l) as
    little-endian bytes, step-major per start (Dieharder export)."""
    st = np.ascontiguousarray(starts, np.uint32)
    nw = C.c_uint64()
    total = len(st) * max(walks_per_vertex, 0) * max(length - 1, 0)
    words = np.zeros(max(total, 1), np.uint32)
    L.check(L.lib().saba_cu_rng_stream(g.device_handle(device), L.ptr(st, L.u32p), len(st),
                                       walks_per_vertex, length, int(selector), master_seed,
                                       hash.multiplier, L.ptr(words, L.u32p), C.byref(nw)),
            "rng_stream")
    return words[: nw.value].astype("<u4").tobytes()


def collect_branching(g: Graph, cfg: CampaignConfig, *, total_walks: int = 0, device: int = 0,
                      shard_index: int = 0, shard_count: int = 1, raw: bool = False):
    """Branching statistics of the campaign's bouquets (walker.hpp:64-109,
    526-536) computed on the GPU (the reference's untimed stats pass,
    bench.hpp:171-178). A shard covers the start vertices v with
    v % shard_count == shard_index; with raw=True the integer arrays
    (histogram, per_step, totals) come back so that shards can be summed."""
    hist = np.zeros(cfg.lanes + 1, np.uint64)
    step = np.zeros(cfg.length - 1, np.uint64)
    tot = np.zeros(4, np.uint64)
    c = _cfg_c(cfg, total_walks, shard_index, shard_count)
    L.check(L.lib().saba_cu_branching_stats(g.device_handle(device), C.byref(c), L.ptr(hist, L.u64p),
                                            L.ptr(step, L.u64p), L.ptr(tot, L.u64p)),
            "branching_stats")
    if raw:
        return hist, step, tot
    st = branching_stats(hist)
    st.mean_candidate_degree = float(tot[3]) / float(tot[2]) if tot[2] else 0.0
    return st, DistinctProxy(step, int(tot[0]))


def run_walk_campaign_device(g: Graph, cfg: CampaignConfig, counts_dev_ptr: int, stream_ptr: int = 0,
                             *, total_walks: int = 0, shard_index: int = 0, shard_count: int = 1,
                             device: int = 0, timing: bool = False) -> CampaignReport:
    """Device-resident campaign: accumulates into a device uint64[n] buffer
    (e.g. a torch tensor's data_ptr()) on `stream_ptr`; asynchronous unless
    timing=True."""
    rep = L.CampaignReportC()
    c = _cfg_c(cfg, total_walks, shard_index, shard_count)
    L.check(L.lib().saba_cu_walk_campaign_device(g.device_handle(device), C.byref(c),
                                                 C.c_void_p(counts_dev_ptr), C.c_void_p(stream_ptr),
                                                 int(timing), C.byref(rep)), "walk_campaign_device")
    return _report(rep)


def campaign_tables(g: Graph, device: int = 0):
    """(records, counters): how many of the highest-degree vertices had their
    record / visit counter in shared memory in the handle's last campaign."""
    r, c = C.c_uint32(0), C.c_uint32(0)
    L.check(L.lib().saba_cu_campaign_tables(g.device_handle(device), C.byref(r), C.byref(c)), "campaign_tables")
    return int(r.value), int(c.value)


def uniform_start_counts(n: int, total_walks: int, master_seed: int = 42) -> np.ndarray:
    """K_v of the uniform-start campaign (host restatement for bookkeeping)."""
    s = substream(master_seed, START_TAG)
    out = np.zeros(n, np.uint64)
    chunk = 1 << 24
    for a in range(0, total_walks, chunk):
        w = np.arange(a, min(total_walks, a + chunk), dtype=np.uint64)
        v = scaled_index((counter_hash(s, w) >> np.uint64(32)).astype(np.uint32), n)
        out += np.bincount(v, minlength=n).astype(np.uint64)
    return out


def campaign_shard_range(total_walks: int, shard_index: int, shard_count: int):
    """Walk-list range [r0, r1) of one shard: the partition campaign.cu uses
    (contiguous ranges of the flattened (vertex, k) list)."""
    if not 0 <= shard_index < shard_count:
        raise ValueError("bad shard index/count")
    return (total_walks * shard_index // shard_count,
            total_walks * (shard_index + 1) // shard_count)
