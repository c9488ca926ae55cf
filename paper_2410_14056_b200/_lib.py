"""ctypes binding of libsaba_cuda.so (include/saba_cuda.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2410_14056_b200/csrc``). There is no fallback: if it is missing, import
of the compute entry points fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SABA_LIB points at an experiment build of the same library (tools/build_variant.sh)
LIB_PATH = os.environ.get("SABA_LIB") or os.path.join(HERE, "libsaba_cuda.so")

SABA_OK, SABA_EINVAL, SABA_EDATA, SABA_ECUDA = 0, 1, 2, 3

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)


class CudaError(RuntimeError):
    """A CUDA failure inside libsaba_cuda (SABA_ECUDA)."""


class CampaignConfigC(C.Structure):
    _fields_ = [("walks_per_vertex", C.c_uint64), ("total_walks", C.c_uint64),
                ("length", C.c_uint32), ("lanes", C.c_uint32), ("mode", C.c_int32),
                ("threads", C.c_int32), ("master_seed", C.c_uint64),
                ("hash_multiplier", C.c_uint64), ("shard_index", C.c_uint32),
                ("shard_count", C.c_uint32)]


class CampaignReportC(C.Structure):
    _fields_ = [("seconds", C.c_double), ("total_steps", C.c_uint64),
                ("total_events", C.c_uint64), ("shard_walks", C.c_uint64),
                ("shard_steps", C.c_uint64), ("walk_kernel_ms", C.c_double),
                ("launches", C.c_uint32), ("kernel", C.c_uint32)]


class AescConfigC(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("delta", C.c_double),
                ("power_iterations", C.c_uint32), ("candidate_nodes", C.c_uint32),
                ("mode", C.c_int32), ("threads", C.c_int32), ("master_seed", C.c_uint64),
                ("lanes", C.c_uint32), ("max_truncation", C.c_uint32),
                ("per_edge_tau", C.c_int32), ("workers", C.c_int32),
                ("switch_depth_cap", C.c_int64), ("hash_multiplier", C.c_uint64)]


class AescReportC(C.Structure):
    _fields_ = [("seconds", C.c_double), ("plan_seconds", C.c_double),
                ("propagation_ms", C.c_double), ("walk_ms", C.c_double),
                ("total_walk_pairs", C.c_uint64), ("total_walk_steps", C.c_uint64),
                ("edge_visits", C.c_uint64), ("sources", C.c_uint64),
                ("lambda_hat", C.c_double), ("bipartite", C.c_int32), ("clamped", C.c_int32),
                ("max_tau", C.c_uint32), ("launches", C.c_uint32), ("replicas", C.c_uint32),
                ("workers", C.c_uint32), ("walk_kernel_ms", C.c_double), ("setup_seconds", C.c_double)]


vp = C.c_void_p
vpp = C.POINTER(C.c_void_p)

# name -> (restype, argtypes); every symbol include/saba_cuda.h declares
SIGNATURES = {
    "saba_cu_last_error": (C.c_char_p, []),
    "saba_cu_version": (C.c_char_p, []),
    "saba_cu_device_count": (C.c_int, []),
    "saba_cu_pinned_alloc": (C.c_int, [C.c_uint64, C.POINTER(C.c_void_p)]),
    "saba_cu_pinned_free": (C.c_int, [C.c_void_p]),
    "saba_hgraph_from_edges": (C.c_int, [C.c_uint32, u32p, C.c_uint64, vpp]),
    "saba_hgraph_from_csr": (C.c_int, [C.c_uint32, u32p, u32p, vpp]),
    "saba_gen_erdos_renyi": (C.c_int, [C.c_uint32, C.c_uint64, C.c_uint64, vpp]),
    "saba_gen_rmat": (C.c_int, [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                C.c_uint64, C.c_int, vpp]),
    "saba_gen_chung_lu": (C.c_int, [C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                    C.c_int, vpp]),
    "saba_gen_scale_free": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, vpp]),
    "saba_gen_random_connected": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, vpp]),
    "saba_hgraph_largest_component": (C.c_int, [vp, vpp]),
    "saba_cu_graph_from_edges": (C.c_int, [C.c_uint32, u32p, C.c_uint64, C.c_int, C.c_int, vpp]),
    "saba_cu_gen_rmat": (C.c_int, [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                   C.c_uint64, C.c_int, C.c_int, vpp]),
    "saba_cu_gen_chung_lu": (C.c_int, [C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                       C.c_int, C.c_int, vpp]),
    "saba_hgraph_vertex_count": (C.c_uint32, [vp]),
    "saba_hgraph_edge_count": (C.c_uint64, [vp]),
    "saba_hgraph_csr": (C.c_int, [vp, u32p, u32p]),
    "saba_hgraph_data": (C.c_int, [vp, C.POINTER(u32p), C.POINTER(u32p)]),
    "saba_hgraph_free": (None, [vp]),
    "saba_cu_graph_create": (C.c_int, [u32p, u32p, C.c_uint32, C.c_uint64, C.c_int, vpp]),
    "saba_cu_graph_create_multi": (C.c_int, [u32p, u32p, C.c_uint32, C.c_uint64, C.POINTER(C.c_int),
                                             C.c_int, vpp]),
    "saba_cu_graph_replica_count": (C.c_int, [vp]),
    "saba_cu_graph_destroy": (C.c_int, [vp]),
    "saba_cu_graph_vertex_count": (C.c_uint32, [vp]),
    "saba_cu_graph_edge_count": (C.c_uint64, [vp]),
    "saba_cu_walk_paths": (C.c_int, [vp, u32p, u32p, C.c_uint64, C.c_uint32, C.c_uint64, u32p]),
    "saba_cu_walk_campaign": (C.c_int, [vp, C.POINTER(CampaignConfigC), u64p,
                                        C.POINTER(CampaignReportC)]),
    "saba_cu_walk_campaign_device": (C.c_int, [vp, C.POINTER(CampaignConfigC), C.c_void_p,
                                               C.c_void_p, C.c_int,
                                               C.POINTER(CampaignReportC)]),
    "saba_cu_campaign_tables": (C.c_int, [vp, u32p, u32p]),
    "saba_cu_branching_stats": (C.c_int, [vp, C.POINTER(CampaignConfigC), u64p, u64p, u64p]),
    "saba_cu_rng_stream": (C.c_int, [vp, u32p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_int,
                                     C.c_uint64, C.c_uint64, u32p, u64p]),
    "saba_cu_walk_budget": (C.c_int, [C.c_uint32, C.c_double, C.c_double, C.c_uint32,
                                      C.c_uint64, u64p]),
    "saba_cu_truncated_lengths": (C.c_int, [vp, C.c_double, C.c_uint32, C.c_uint32, C.c_int,
                                            u32p, f64p, C.POINTER(C.c_int)]),
    "saba_cu_aesc": (C.c_int, [vp, C.POINTER(AescConfigC), u32p, C.c_uint64, C.c_uint32,
                               C.c_uint32, f64p, f64p, u32p, u32p, C.POINTER(AescReportC)]),
    "saba_cu_aesc_device": (C.c_int, [vp, C.POINTER(AescConfigC), u32p, C.c_uint64, C.c_uint32,
                                      C.c_uint32, C.c_void_p, u32p, u32p, C.c_void_p,
                                      C.POINTER(AescReportC)]),
    "saba_cu_symmetrise": (C.c_int, [vp, C.c_void_p, C.c_void_p, C.c_void_p]),
    "saba_aesc_shard_sources": (C.c_int, [u32p, C.c_uint32, u32p, C.c_uint64, C.c_uint32, C.c_uint32,
                                          u32p, u64p]),
    "saba_cu_propagate": (C.c_int, [vp, C.c_uint32, u32p, C.c_double, C.c_double, C.c_int64,
                                    f64p, u32p]),
    "saba_cu_estimate_edge": (C.c_int, [vp, C.c_uint32, C.c_uint32, f64p, C.c_uint32,
                                        C.c_uint64, C.c_int, C.c_uint64, C.c_uint32, C.c_uint64,
                                        f64p]),
}

_lib = None


def lib():
    """Load libsaba_cuda.so once (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(there is no CPU fallback for the sm_100a path)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI status to the reference's exception split (common.hpp:13-21)."""
    if rc == SABA_OK:
        return
    msg = lib().saba_cu_last_error().decode()
    if rc == SABA_EINVAL:
        raise ValueError(msg or what)
    if rc == SABA_ECUDA:
        raise CudaError(msg or what)
    raise RuntimeError(msg or what)


def ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)
