"""Full-size parity against the COMPILED REFERENCE (oracle/_ref: the
reference headers compiled unchanged, VERDICT r1 "weak" 1-2).

* cfg1, cfg2: every visit count of the BASELINE campaigns equals the
  reference's own campaign_vertex_scaled per start vertex (walker.hpp:430-449)
  bit for bit, unsharded and sharded.
* cfg3, cfg4, cfg5: AESC on the BASELINE graphs for source samples (64
  sources of cfg3, a hub and two non-hub cfg4 sources, 16 of cfg5) against the
  reference's aesc_source (aesc.hpp:561-629): lambda_hat, tau, tau~, pair and
  step counts bit-exact, g_hat within 1e-9 relative. The worst relative and
  absolute g_hat errors are reported as ParityMargin warnings (they appear in
  pytest's warnings summary).
"""
import warnings

import numpy as np
import pytest

from conftest import ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

RTOL, ATOL = 1e-9, 1e-15


class ParityMargin(UserWarning):
    pass


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref (the compiled reference) is not built here")
    return Reference()


def _bench_sources(n, count):
    import sys
    sys.path.insert(0, ROOT)
    import bench
    return np.sort(bench.subset_sources(n, count))


def _campaign(sb, g, W, L, seed, **kw):
    s = sb.VisitCountSink(g.n)
    sb.run_walk_campaign(g, sb.CampaignConfig(length=L, master_seed=seed, **kw.pop("cfg", {})), s,
                         total_walks=W, **kw)
    return s.counts


def _check_campaign(sb, ref, g, W, L, shards):
    rg = ref.from_csr(g.offsets, g.adjacency)
    want, _, steps = ref.campaign_kv(rg, L, W=W, sorted_=True, lanes=8, master=42, vertex_stride=1)
    assert steps == W * (L - 1) and int(want.sum()) == W * L
    got = _campaign(sb, g, W, L, 42)
    assert np.array_equal(got, want)
    for parts in shards:
        acc = np.zeros(g.n, np.uint64)
        for i in range(parts):
            acc += _campaign(sb, g, W, L, 42, shard_index=i, shard_count=parts)
        assert np.array_equal(acc, want), parts
    return want


def test_cfg1_counts_equal_compiled_reference(sb, ref):
    g = sb.make_erdos_renyi(65536, 524288, 1)
    _check_campaign(sb, ref, g, 1 << 20, 64, (2, 4))


def test_cfg2_counts_equal_compiled_reference(sb, ref):
    """R-MAT s20 ef16 LCC, 16,777,216 uniform walks of 128 (2^31 visits): the
    hub-counter kernel, its 2-shard split and Hash mode."""
    g = sb.make_rmat(20, 16, seed=1, device=0)
    want = _check_campaign(sb, ref, g, 1 << 24, 128, (2,))
    h = _campaign(sb, g, 1 << 24, 128, 42, cfg={"mode": sb.WalkMode.Hash})
    assert np.array_equal(h, want)


def _check_aesc(sb, ref, g, eps, delta, src, tag):
    src = np.asarray(src, np.uint32)
    cfg = sb.AescConfig(epsilon=eps, delta=delta)
    est = sb.aesc(g, cfg, sources=src)
    r = ref.aesc(ref.from_csr(g.offsets, g.adjacency), epsilon=eps, delta=delta, sources=src)
    assert est.plan.lambda_hat == r.lambda_hat
    assert np.array_equal(est.plan.tau, r.tau)
    assert np.array_equal(est.plan.tau_tilde[src], r.tau_tilde[src])
    assert est.total_walk_pairs == r.total_walk_pairs > 0
    assert est.total_walk_steps == r.total_walk_steps
    err = np.abs(est.g_hat - r.g_hat)
    rel = err / np.maximum(np.abs(r.g_hat), 1e-300)
    mask = r.g_hat != 0
    worst_rel = float(rel[mask].max()) if mask.any() else 0.0
    warnings.warn(ParityMargin(f"{tag}: {len(src)} sources vs compiled reference: worst rel {worst_rel:.3e}, "
                               f"worst abs {float(err.max()):.3e}, tau~ {sorted(set(r.tau_tilde[src].tolist()))[:8]}, "
                               f"pairs {r.total_walk_pairs}"))
    assert np.all(err <= RTOL * np.abs(r.g_hat) + ATOL), (tag, worst_rel)


def test_cfg3_64_sources_match_compiled_reference(sb, ref):
    g = sb.make_rmat(16, 8, seed=1, device=0)
    _check_aesc(sb, ref, g, 0.1, 0.01, _bench_sources(g.n, 64), "cfg3")


def test_cfg5_16_sources_match_compiled_reference(sb, ref):
    g = sb.make_chung_lu(3_000_000, 2.2, 78.0, 30000.0, seed=1, device=0)
    _check_aesc(sb, ref, g, 0.01, 0.01, _bench_sources(g.n, 16), "cfg5")


def test_cfg4_hub_and_nonhub_sources_match_compiled_reference(sb, ref):
    """cfg4 (R-MAT s22 ef16 LCC, eps 0.05): the highest-degree source among the
    first 256 of the bench permutation (a hub: it switches after one depth),
    and two NON-hub sources (degree between 0.1% and 1% of the maximum, tau~ >= 2)
    from the first 4096 of the permutation — the two with the least walk work,
    sum_slots 2 n_req(tau - tau~) (tau - tau~) (aesc.hpp:103-110, 478-496), from
    the GPU's tau~, so the reference finishes them in minutes (low-degree
    sources cost ~1e10 reference steps each: tools/pick_cfg4_sources.py)."""
    g = sb.make_rmat(22, 16, seed=1, device=0)
    deg = np.diff(g.offsets).astype(np.int64)
    cand = _bench_sources(g.n, 256)
    hub = int(cand[np.argmax(deg[cand])])
    _check_aesc(sb, ref, g, 0.05, 0.01, [hub], "cfg4 hub")
    wide = _bench_sources(g.n, 4096)
    band = wide[(deg[wide] >= deg.max() // 1000) & (deg[wide] <= deg.max() // 100)]
    est = sb.aesc(g, sb.AescConfig(epsilon=0.05, delta=0.01), sources=band)
    tau = int(est.plan.tau[0])
    cost = []
    for s in band:
        d, tt = int(deg[s]), int(est.plan.tau_tilde[s])
        if 2 <= tt < tau and d <= deg.max() // 100:
            te = tau - tt
            cost.append((d * 2 * sb.walk_budget(te, 0.05, 0.01, d, g.m) * te, int(s)))
    nonhub = sorted(s for _, s in sorted(cost)[:2])
    assert len(nonhub) == 2
    _check_aesc(sb, ref, g, 0.05, 0.01, nonhub, "cfg4 non-hub")
