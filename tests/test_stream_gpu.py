"""rng_stream (stream.hpp:29-83) on the GPU against the reference's bytes,
plus the word-by-word restatement of test_stream.cpp:75-104."""
import numpy as np
import pytest

from conftest import golden_graph

pytestmark = pytest.mark.gpu


def test_stream_matches_reference_bytes(golden, sb):
    n = 0
    for key in golden:
        if not key.startswith("stream/"):
            continue
        _, gname, starts, spec = key.split("/")
        K, L, sel, seed = (int(x.lstrip("KLsel")) for x in spec.split("_"))
        g = golden_graph(golden, gname)
        got = sb.rng_stream(g, [int(s) for s in starts.split("-")], K, L, sb.SelectorKind(sel), seed)
        assert got == golden[key].astype("<u4").tobytes(), key
        n += 1
    assert n >= 4


def test_stream_words_restated(golden, sb):
    # test_stream.cpp:75-104: word (l-1)*K + k == seed_k ^ h(cur, l)
    g = golden_graph(golden, "petersen")
    K, L = 16, 6
    words = np.frombuffer(sb.rng_stream(g, [3], K, L, sb.SelectorKind.Scaled, 99), "<u4")
    vseed = sb.substream(99, 3)
    h = sb.HashSpec()
    for k in range(K):
        seed = int(sb.counter_hash(vseed, k)) >> 32
        cur = 3
        for l in range(1, L):
            raw = seed ^ h.state(cur, l)
            assert int(words[(l - 1) * K + k]) == raw
            cur = int(g.neighbors(cur)[int(sb.scaled_index(raw, g.degree(cur)))])


def test_stream_contract(sb):
    g = sb.triangle()
    assert sb.rng_stream(g, [0], 1, 2) != b"" and len(sb.rng_stream(g, [0], 100, 5)) == 1600
    assert sb.rng_stream(g, [0], 5, 1) == b""  # length 1 emits nothing
    with pytest.raises(ValueError):
        sb.rng_stream(g, [], 1, 2)
    with pytest.raises(ValueError):
        sb.rng_stream(g, [0], 0, 2)
