"""GPU parity of the Bouquets walk engine against the oracle and the
reference's golden vectors. Integer outputs are compared bit-exactly."""
import numpy as np
import pytest

from conftest import golden_graph

pytestmark = pytest.mark.gpu


def test_random_walk_matches_reference_paths(golden, sb):
    for gname in ("sf300_4_5", "petersen", "sf2000_8_17"):
        g = golden_graph(golden, gname)
        st, sd, paths = (golden[f"walk/{gname}/{k}"] for k in ("starts", "seeds", "paths"))
        got = sb.walk_paths(g, st, sd, paths.shape[1])
        assert np.array_equal(got, paths), gname
        w = sb.random_walk(g, int(st[0]), paths.shape[1], sb.SelectorKind.Scaled, int(sd[0]))
        assert np.array_equal(w.vertices, paths[0])


def test_random_bouquet_lanes_replay_walks(golden, sb):
    g = golden_graph(golden, "sf300_4_5")
    seeds = sb.gen_sorted_seeds(8, 99)  # test_walker.cpp:78-88
    assert np.array_equal(seeds.seeds, golden["bouquet/seeds"])
    walks = sb.random_bouquet(g, 7, 12, 8, seeds, sb.SelectorKind.Scaled)
    for b in range(8):
        assert np.array_equal(walks[b].vertices, golden["bouquet/paths"][b])
        solo = sb.random_walk(g, 7, 12, sb.SelectorKind.Scaled, int(seeds.seeds[b]))
        assert np.array_equal(walks[b].vertices, solo.vertices)
    eq = sb.SeedSet(np.array([123456, 123456], np.uint32))
    w2 = sb.random_bouquet(g, 1, 9, 2, eq, sb.SelectorKind.Scaled)
    assert np.array_equal(w2[0].vertices, w2[1].vertices)


def test_random_walk_basics_and_errors(sb):
    f = sb.fig1()
    assert list(sb.random_walk(f, 2, 1, sb.SelectorKind.Scaled, 77).vertices) == [2]
    assert list(sb.random_walk(sb.path(2), 0, 3, sb.SelectorKind.Scaled, 123).vertices) == [0, 1, 0]
    with pytest.raises(ValueError):
        sb.random_walk(f, 0, 0, sb.SelectorKind.Scaled, 1)
    iso = sb.Graph.from_edges(3, [(0, 1)])
    with pytest.raises(ValueError):
        sb.random_walk(iso, 2, 2, sb.SelectorKind.Scaled, 1)
    assert len(sb.random_walk(iso, 2, 1, sb.SelectorKind.Scaled, 1).vertices) == 1


def test_paths_match_oracle_random(sb, oracle):
    g = sb.make_rmat(14, 8, seed=11)
    rng = np.random.default_rng(3)
    st = rng.integers(0, g.n, 4096).astype(np.uint32)
    sd = rng.integers(0, 2**32, 4096, dtype=np.uint64).astype(np.uint32)
    got = sb.walk_paths(g, st, sd, 40)
    for i in range(0, 4096, 97):
        assert np.array_equal(got[i], oracle.random_walk(g.offsets, g.adjacency, int(st[i]), 40,
                                                         int(sd[i])))
    # every consecutive pair is an edge (test_walker.cpp:166-189)
    a, b = got[:, :-1].ravel(), got[:, 1:].ravel()
    pos = np.searchsorted(g.adjacency, b)  # cheap check via per-vertex slices
    for x, y in list(zip(a[:2000], b[:2000])):
        assert g.has_edge(int(x), int(y))


def _camp(sb, g, K, L, seed, mode=None, lanes=8, **kw):
    cfg = sb.CampaignConfig(walks_per_vertex=K, length=L, master_seed=seed, lanes=lanes,
                            mode=mode if mode is not None else sb.WalkMode.Saba)
    sink = sb.VisitCountSink(g.n)
    rep = sb.run_walk_campaign(g, cfg, sink, **kw)
    return sink.counts, rep


def test_campaign_counts_match_reference(golden, sb):
    for key in golden:
        if not key.startswith("camp/"):
            continue
        _, gname, spec = key.split("/")
        K, L, s = (int(x[1:]) for x in spec.split("_"))
        g = golden_graph(golden, gname)
        got, rep = _camp(sb, g, K, L, s)
        assert np.array_equal(got, golden[key]), key
        assert rep.total_steps == g.n * K * (L - 1)
        assert rep.total_events == g.n * K * L


def test_campaign_modes_lanes_shards_invariant(golden, sb):
    g = golden_graph(golden, "sf400_5_21")
    want = golden["camp/sf400_5_21/K64_L7_s9"]
    h, _ = _camp(sb, g, 64, 7, 9, mode=sb.WalkMode.Hash)
    assert np.array_equal(h, want)  # hash == saba (test_walker.cpp:147-151)
    l16, _ = _camp(sb, g, 64, 7, 9, lanes=16)
    assert np.array_equal(l16, want)
    for parts in (2, 3, 8):
        acc = np.zeros_like(want)
        for i in range(parts):
            c, rep = _camp(sb, g, 64, 7, 9, shard_index=i, shard_count=parts)
            acc += c
        assert np.array_equal(acc, want), parts


def test_uniform_start_campaign_matches_reference(golden, sb):
    g = golden_graph(golden, "sf2000_8_17")
    cfg = sb.CampaignConfig(length=16, master_seed=42)
    sink = sb.VisitCountSink(g.n)
    rep = sb.run_walk_campaign(g, cfg, sink, total_walks=32768)
    assert np.array_equal(sink.counts, golden["ucamp/sf2000_8_17/W32768_L16_s42"])
    assert rep.total_steps == 32768 * 15


def test_campaign_validation(sb):
    # test_walker.cpp:284-300
    g = sb.triangle()
    sink = sb.VisitCountSink(3)
    for kw in (dict(walks_per_vertex=0), dict(walks_per_vertex=1, length=0),
               dict(walks_per_vertex=1, length=2, lanes=7),
               dict(walks_per_vertex=1, length=2, mode=sb.WalkMode.Naive)):
        with pytest.raises(ValueError):
            sb.run_walk_campaign(g, sb.CampaignConfig(**kw), sink)
    iso = sb.Graph.from_edges(4, [(0, 1), (1, 2), (0, 2)])
    with pytest.raises(ValueError):
        sb.run_walk_campaign(iso, sb.CampaignConfig(walks_per_vertex=1, length=2),
                             sb.VisitCountSink(4))
    # L = 1: one event per walk, no steps (test_walker.cpp:106-119)
    c, rep = _camp(sb, sb.fig1(), 1, 1, 42)
    assert list(c) == [1, 1, 1, 1] and rep.total_steps == 0
    c, rep = _camp(sb, sb.fig1(), 13, 4, 42)
    assert c.sum() == 4 * 13 * 4


def test_cfg1_full_size_bit_exact(sb, oracle):
    """BASELINE config 1 at full size: ER n=65,536 m=524,288, 1,048,576
    uniform-start walks of length 64 — counts equal the oracle bit for bit."""
    g = sb.make_erdos_renyi(65536, 524288, 1)
    W, L = 1 << 20, 64
    sink = sb.VisitCountSink(g.n)
    sb.run_walk_campaign(g, sb.CampaignConfig(length=L, master_seed=42), sink, total_walks=W)
    kv = oracle.uniform_start_counts(g.n, W, 42)
    want = oracle.campaign_counts(g.offsets, g.adjacency, length=L, master=42, k_per_vertex=kv)
    assert np.array_equal(sink.counts, want)
    assert int(sink.counts.sum()) == W * L
    # sharded (2 and 4 "GPUs") sums are identical
    for parts in (2, 4):
        acc = np.zeros(g.n, np.uint64)
        for i in range(parts):
            s = sb.VisitCountSink(g.n)
            sb.run_walk_campaign(g, sb.CampaignConfig(length=L, master_seed=42), s,
                                 total_walks=W, shard_index=i, shard_count=parts)
            acc += s.counts
        assert np.array_equal(acc, want)


def test_device_variant_matches_host_variant(sb):
    torch = pytest.importorskip("torch")
    g = sb.make_rmat(14, 8, seed=2)
    cfg = sb.CampaignConfig(length=32, master_seed=5)
    sink = sb.VisitCountSink(g.n)
    sb.run_walk_campaign(g, cfg, sink, total_walks=200000)
    counts = torch.zeros(g.n, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    sb.run_walk_campaign_device(g, cfg, counts.data_ptr(), st.cuda_stream, total_walks=200000)
    torch.cuda.synchronize()
    assert np.array_equal(counts.cpu().numpy().astype(np.uint64), sink.counts)


def test_branching_statistics_match_reference(golden, sb):
    """BranchCollector output (walker.hpp:64-109) of the reference's campaign
    with collect_stats, rebuilt on the GPU bouquet for bouquet."""
    n = 0
    for key in golden:
        if not (key.startswith("stats/") and key.endswith("/hist")):
            continue
        base = key[: -len("/hist")]
        _, gname, spec = base.split("/")
        K, L, mode, lanes, seed = (int(x[1:]) for x in spec.split("_"))
        g = golden_graph(golden, gname)
        cfg = sb.CampaignConfig(walks_per_vertex=K, length=L, mode=sb.WalkMode(mode), lanes=lanes,
                                master_seed=seed, collect_stats=True)
        rep = sb.run_walk_campaign(g, cfg, sb.VisitCountSink(g.n))
        total, samples, mdeg, mean = golden[base + "/scalars"]
        assert rep.has_stats
        assert np.array_equal(rep.branching.histogram, golden[key]), base
        assert np.array_equal(rep.proxy.per_step, golden[base + "/per_step"]), base
        assert rep.proxy.total == int(total) and rep.branching.samples == int(samples)
        assert rep.branching.mean_candidate_degree == mdeg and rep.branching.mean == mean
        n += 1
    assert n >= 6
    # test_walker.cpp:227-241: forced lanes -> one distinct vertex per step
    p2 = sb.path(2)
    rep = sb.run_walk_campaign(p2, sb.CampaignConfig(walks_per_vertex=64, length=5, collect_stats=True),
                               sb.VisitCountSink(2))
    assert rep.branching.mean == 1.0 and rep.branching.p1 == 1 and rep.branching.p25 == 1


def test_branching_statistics_shards_add_up(golden, sb):
    """Vertex-striped shards of the statistics pass sum to the unsharded one."""
    g = golden_graph(golden, "sf2000_8_17")
    cfg = sb.CampaignConfig(walks_per_vertex=24, length=9, lanes=8, collect_stats=True)
    for total in (0, 50_000):
        whole = sb.collect_branching(g, cfg, total_walks=total, raw=True)
        for S in (2, 5):
            parts = [sb.collect_branching(g, cfg, total_walks=total, shard_index=i, shard_count=S, raw=True)
                     for i in range(S)]
            for k in range(3):
                assert np.array_equal(sum(p[k] for p in parts), whole[k]), (total, S, k)


def test_saba_clusters_bouquets(golden, sb):
    """test_walker.cpp:259-282: sorted seeds give fewer distinct lanes."""
    g = golden_graph(golden, "sf2000_8_17")
    run = lambda m: sb.run_walk_campaign(  # noqa: E731
        g, sb.CampaignConfig(walks_per_vertex=2048, length=10, mode=m, collect_stats=True),
        sb.VisitCountSink(g.n))
    h, s = run(sb.WalkMode.Hash), run(sb.WalkMode.Saba)
    assert s.branching.mean < h.branching.mean
    assert s.proxy.per_step[0] <= h.proxy.per_step[0]


def test_campaign_report_names_the_kernel(sb, oracle):
    """The campaign report says which K2 variant ran (saba_cuda.h SABA_K2_*):
    a small graph takes the all-vertex shared-counter kernel, a graph beyond
    the fat adjacency's L2 budget the degree-ranked one, and a length-1
    campaign launches no walk kernel. Counts stay the oracle's either way."""
    small = sb.make_rmat(12, 8, seed=5)
    sink = sb.VisitCountSink(small.n)
    rep = sb.run_walk_campaign(small, sb.CampaignConfig(length=9, master_seed=2), sink, total_walks=20000)
    assert rep.kernel == "walk_count_fat_priv_kernel"
    assert sb.campaign_tables(small) == (0, small.n)  # every vertex's counter in shared memory
    kv = oracle.uniform_start_counts(small.n, 20000, 2)
    assert np.array_equal(sink.counts, oracle.campaign_counts(small.offsets, small.adjacency, length=9, master=2,
                                                              k_per_vertex=kv))
    sink1 = sb.VisitCountSink(small.n)
    rep1 = sb.run_walk_campaign(small, sb.CampaignConfig(length=1, master_seed=2), sink1, total_walks=20000)
    assert rep1.kernel == "" and int(sink1.counts.sum()) == 20000
    big = sb.make_chung_lu(300_000, 2.2, 24.0, 3000.0, seed=2)  # 16 m > 48 MiB: no fat adjacency
    sinkb = sb.VisitCountSink(big.n)
    repb = sb.run_walk_campaign(big, sb.CampaignConfig(length=17, master_seed=6), sinkb, total_walks=300000)
    assert repb.kernel == "walk_count_rank_kernel"
    assert sb.campaign_tables(big) == (2560, 22016)  # the 63 KB default split (records, 16-bit counters)
    kvb = oracle.uniform_start_counts(big.n, 300000, 6)
    assert np.array_equal(sinkb.counts, oracle.campaign_counts(big.offsets, big.adjacency, length=17, master=6,
                                                               k_per_vertex=kvb))
