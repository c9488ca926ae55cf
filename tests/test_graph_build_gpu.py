"""Device graph ingest (csrc/graph_build.cu) against the
reference's own Graph::from_edges (oracle/_ref, graph.hpp:86-105) and the host
builders: the CSR must be identical, array for array."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref not built")
    return Reference()


def same_csr(a, b):
    return np.array_equal(a.offsets, b.offsets) and np.array_equal(a.adjacency, b.adjacency)


def messy_pairs(rng, n, count):
    p = rng.integers(0, n, size=(count, 2), dtype=np.uint32)
    p[::7, 1] = p[::7, 0]                      # self-loops
    p = np.concatenate([p, p[::3, ::-1], p[::5]])  # reversed and plain duplicates
    return p[rng.permutation(len(p))]


@pytest.mark.parametrize("n,count,n_hint", [(50, 200, 0), (1000, 5000, 1200), (70000, 400000, 0),
                                            (3, 1, 0)])
def test_from_edges_matches_reference(sb, ref, n, count, n_hint):
    rng = np.random.default_rng(n + count)
    pairs = messy_pairs(rng, n, count)
    r_off, r_adj, _ = ref.from_edges(n_hint, pairs).csr()
    dev = sb.Graph.from_edges(n_hint, pairs, device=0)
    host = sb.Graph.from_edges(n_hint, pairs)
    assert np.array_equal(dev.offsets, r_off) and np.array_equal(dev.adjacency, r_adj)
    assert same_csr(dev, host)


def test_from_edges_edge_cases(sb, ref):
    # no pairs: n_hint isolated vertices; loops only: n still counts them
    g = sb.Graph.from_edges(5, np.zeros((0, 2), np.uint32), device=0)
    assert g.n == 5 and g.m == 0 and np.array_equal(g.offsets, np.zeros(6, np.uint32))
    loops = np.array([[4, 4], [9, 9]], np.uint32)
    g = sb.Graph.from_edges(0, loops, device=0)
    r_off, r_adj, _ = ref.from_edges(0, loops).csr()
    assert g.n == 10 and g.m == 0 and np.array_equal(g.offsets, r_off)
    with pytest.raises(RuntimeError):  # check_data(n > 0) (graph.hpp:95)
        sb.Graph.from_edges(0, np.zeros((0, 2), np.uint32), device=0)


def test_largest_component_matches_host(sb):
    rng = np.random.default_rng(5)
    # several components, two of the largest size (ties go to the one holding
    # the smallest vertex, the host BFS's first find), isolated vertices
    blocks, base = [], 0
    for size in (40, 300, 17, 300, 2, 1):
        ids = base + rng.permutation(size)
        blocks.append(np.stack([ids[:-1], ids[1:]], 1))
        extra = rng.integers(0, size, size=(size, 2)) + base
        blocks.append(extra)
        base += size
    perm = rng.permutation(base).astype(np.uint32)  # scatter the components over the id range
    pairs = perm[np.concatenate(blocks)]
    dev = sb.Graph.from_edges(base + 3, pairs, device=0, keep_lcc=True)
    host = sb.Graph.from_edges(base + 3, pairs, keep_lcc=True)
    assert dev.n == 300 and same_csr(dev, host)


@pytest.mark.parametrize("scale,ef,lcc", [(10, 4, True), (12, 16, False), (16, 8, True)])
def test_rmat_device_matches_host(sb, scale, ef, lcc):
    assert same_csr(sb.make_rmat(scale, ef, seed=3, keep_lcc=lcc, device=0),
                    sb.make_rmat(scale, ef, seed=3, keep_lcc=lcc))


@pytest.mark.parametrize("n", [2000, 100000])
def test_chung_lu_device_matches_host(sb, n):
    assert same_csr(sb.make_chung_lu(n, seed=2, device=0), sb.make_chung_lu(n, seed=2))


def test_baseline_graphs_device_matches_host(sb):
    # cfg2 (R-MAT s20 ef16) and cfg4 (R-MAT s22 ef16), LCC, seed 1 as in bench.py
    for scale in (20, 22):
        dev = sb.make_rmat(scale, 16, seed=1, device=0)
        host = sb.make_rmat(scale, 16, seed=1)
        assert same_csr(dev, host), scale
