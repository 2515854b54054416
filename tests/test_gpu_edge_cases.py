"""GPU parity on the edge cases the reference permits and on its error
behaviour, plus the tie-detection / exact-redo machinery of the CRCW path."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.util import assert_same_result, to_hb_graph, to_hb_stream

pytestmark = pytest.mark.gpu
VARIANTS = ["crcw", "crew"]


def _run(hb, g, s, variant, **kw):
    return hb.run_variant(to_hb_graph(g), to_hb_stream(s), hb.ParallelConfig(variant=variant, **kw))


@pytest.mark.parametrize("variant", VARIANTS)
def test_known_answers(hb, port, variant):
    """test_seq.cpp:7-65 / test_par.cpp:9-30 through the device path."""
    z = lambda seed: po.Stream(seed=seed, noise_high=0.0)  # noqa: E731
    r = _run(hb, po.graph_from_edge_lists([[0, 1]]), z(1), variant)
    assert r.matching.matched_edges.tolist() == [0] and r.report.rounds == 1 and r.matching.total_weight == 1.0
    r = _run(hb, port.tight_family(3, 0.1), z(5), variant)
    assert r.matching.matched_edges.tolist() == [3] and abs(r.matching.total_weight - 1.1) < 1e-12
    r = _run(hb, port.tight_family(4, 0.25), z(9), variant)
    assert r.matching.matched_edges.tolist() == [4]
    r = _run(hb, po.graph_from_edge_lists([[0, 1], [1, 2], [2, 3]], [5, 9, 5]), z(1), variant)
    assert r.matching.matched_edges.tolist() == [1] and r.report.deactivated_per_round == [2]
    spokes = 9
    star = po.graph_from_edge_lists([[0, i + 1] for i in range(spokes)], [1.0 + i for i in range(spokes)])
    r = _run(hb, star, z(3), variant)
    assert r.matching.matched_edges.tolist() == [spokes - 1] and r.report.deactivated_per_round == [spokes - 1]
    r = _run(hb, po.graph_from_edge_lists([[0, 1], [2, 3]], [4, 2]), z(1), variant)
    assert r.matching.matched_edges.tolist() == [0, 1] and r.report.rounds == 1


@pytest.mark.parametrize("variant", VARIANTS)
def test_empty_and_degenerate_instances(hb, port, variant):
    empty = po.Graph(5, 0, np.zeros(6, dtype=np.uint64), np.zeros(0, dtype=np.uint32), np.zeros(1, dtype=np.uint64),
                     np.zeros(0, dtype=np.uint32), np.zeros(0))
    r = _run(hb, empty, po.Stream(), variant)
    assert r.report.rounds == 0 and len(r.matching.matched_edges) == 0 and r.matching.total_weight == 0.0
    # size-1 edges, parallel (identical) edges, isolated vertices (kept), one vertex shared by all
    g = po.graph_from_edge_lists([[3], [3], [0, 1], [0, 1], [0, 1], [2], [5, 6, 7], [7]], n=10)
    for s in (po.Stream(seed=4), po.Stream(seed=4, noise_high=0.0), po.Stream(seed=2, mode=po.MODE_REPLACE_UNIFORM)):
        assert_same_result(_run(hb, g, s, variant), port.local_max(g, s), f"degenerate {s}")


@pytest.mark.parametrize("variant", VARIANTS)
def test_large_and_ragged_edges(hb, port, variant):
    """Edge sizes from 1 to 4096 in one instance: thread-per-edge and warp-per-edge classes."""
    rng = np.random.default_rng(3)
    n = 6000
    sizes = [1, 2, 3, 31, 32, 33, 64, 65, 100, 1000, 4096, 4095, 2, 2, 5, 7] + rng.integers(1, 40, 400).tolist()
    lists = [rng.choice(n, size=s, replace=False).tolist() for s in sizes]
    g = po.graph_from_edge_lists(lists, rng.integers(1, 50, len(lists)).astype(float), n=n)
    for s in (po.Stream(seed=6), po.Stream(seed=6, noise_high=0.0), po.Stream(seed=6, kind=po.GEN_PARK_MILLER)):
        want = port.local_max(g, s)
        assert_same_result(_run(hb, g, s, variant), want, f"ragged {s}")
        if variant == "crcw":
            assert_same_result(_run(hb, g, s, variant, tie_mode="exact"), want, f"ragged exact {s}")
            assert_same_result(_run(hb, g, s, variant, loop_mode="host"), want, f"ragged host {s}")


@pytest.mark.parametrize("variant", VARIANTS)
def test_round_cap_carries_partial_result(hb, port, variant):
    """test_par.cpp:86-99 / test_seq.cpp:115-134."""
    g = po.graph_from_edge_lists([[i, i + 1] for i in range(12)], [1.0 + i for i in range(12)])
    s = po.Stream(seed=1, noise_high=0.0)
    want = port.local_max(g, s, max_rounds=2)
    assert want.status == po.ROUND_LIMIT
    with pytest.raises(hb.RoundLimitError) as ei:
        _run(hb, g, s, variant, max_rounds=2)
    err = ei.value
    assert err.report.rounds == 2
    assert np.array_equal(err.partial.matched_edges, want.matched_edges)
    assert err.report.matched_per_round_count == want.per_round_matched
    assert err.report.deactivated_per_round == want.per_round_deactivated
    # one more round than needed is not an error
    full = port.local_max(g, s)
    assert_same_result(_run(hb, g, s, variant, max_rounds=full.rounds), full)


def test_input_errors(hb, port):
    g = po.graph_from_edge_lists([[0, 1], [1, 2]])
    with pytest.raises(hb.InputError):  # weight_stream.hpp:96-100
        _run(hb, g, po.Stream(noise_low=-1.0), "crcw")
    with pytest.raises(hb.InputError):
        _run(hb, g, po.Stream(noise_low=2.0, noise_high=1.0), "crew")
    with pytest.raises(hb.InputError):  # local_max_par.hpp:615
        hb.run_variant(to_hb_graph(g), hb.WeightStream(), hb.ParallelConfig(variant=7))
    bad = to_hb_graph(g)
    bad.edge_members = np.array([0, 1, 1, 9], dtype=np.uint32)  # vertex id out of range
    with pytest.raises(hb.InputError):
        hb.run_variant(bad, hb.WeightStream())
    bad = to_hb_graph(g)
    bad.base_weights = np.array([1.0, 0.0])  # hypergraph.hpp:104
    with pytest.raises(hb.InputError):
        hb.run_variant(bad, hb.WeightStream())


def test_tie_detection_and_exact_redo(hb, port):
    """Weights that collide in the 64-bit key force the tie flag; the redone round must be exact.
    park-miller has only 2^31 noise values, and a huge flat star makes equal maxima certain."""
    # many parallel edges with identical base weight and a 31-bit generator under uniform mode:
    # equal weights are common, the order is decided by (tie_hash, id)
    rng = np.random.default_rng(0)
    hub_edges = [[0, 1 + i] for i in range(3000)]
    extra = [rng.choice(3001, size=3, replace=False).tolist() for _ in range(2000)]
    g = po.graph_from_edge_lists(hub_edges + extra, n=3001)
    # two-level noise: width so small that weights collapse onto a handful of doubles
    s = po.Stream(seed=5, kind=po.GEN_PARK_MILLER, noise_low=0.0, noise_high=2.0 ** -50)
    want = port.local_max(g, s)
    got = hb.run_variant(to_hb_graph(g), to_hb_stream(s), hb.ParallelConfig(variant="crcw", loop_mode="graph"))
    assert_same_result(got, want, "collapsed weights")
    assert got.report.tie_redo_rounds >= 1  # the fast path saw equal keys and fell back
    got_host = hb.run_variant(to_hb_graph(g), to_hb_stream(s), hb.ParallelConfig(variant="crcw", loop_mode="host"))
    assert_same_result(got_host, want, "collapsed weights, host loop")
    assert_same_result(hb.run_variant(to_hb_graph(g), to_hb_stream(s), hb.ParallelConfig(variant="crew")), want)


def test_weights_spanning_many_binades_use_the_exact_path(hb, port):
    """bits(w_max) - bits(w_min) needs more than 62 bits: no tagged 64-bit key exists."""
    rng = np.random.default_rng(1)
    g = port.generate_random(400, 900, 2, 4, 3)
    g.base_weights = np.exp(rng.uniform(-600, 600, g.m))
    for s in (po.Stream(seed=2), po.Stream(seed=2, noise_high=0.0)):
        assert_same_result(_run(hb, g, s, "crcw"), port.local_max(g, s), f"wide {s}")
        assert_same_result(_run(hb, g, s, "crew"), port.local_max(g, s), f"wide crew {s}")


def test_non_integer_weights_sum_in_id_order(hb, port):
    """total_weight must be the ascending-id sequential sum (local_max_seq.hpp:79), bit for bit."""
    rng = np.random.default_rng(5)
    g = port.generate_random(3000, 5000, 2, 3, 9)
    g.base_weights = rng.random(g.m) * 10 + 0.1
    for variant in VARIANTS:
        s = po.Stream(seed=3)
        want = port.local_max(g, s)
        got = _run(hb, g, s, variant)
        assert_same_result(got, want)
        seq_sum = 0.0
        for e in want.matched_edges:
            seq_sum += g.base_weights[e]
        assert got.matching.total_weight == seq_sum


def test_many_rounds_epoch_wrap(hb, port):
    """A path with geometrically increasing weights needs about one round per two edges, and its
    weights span ~90 binades: the 59-bit payload leaves room for only 30 distinct round tags, so
    the tags wrap several times (ST_EPOCH) before the matching is maximal."""
    k = 150
    g = po.graph_from_edge_lists([[i, i + 1] for i in range(k)], [1e-6 * 1.5 ** i for i in range(k)])
    z = po.Stream(seed=1, noise_high=0.0)
    want = port.local_max(g, z, max_rounds=400)
    assert want.rounds >= 70
    for loop in ("host", "graph"):
        got = hb.run_variant(to_hb_graph(g), to_hb_stream(z), hb.ParallelConfig(variant="crcw", loop_mode=loop,
                                                                                max_rounds=400))
        assert_same_result(got, want, f"long chain {loop}")
        if loop == "graph":
            assert got.report.graph_launches >= 3  # one relaunch per tag epoch
    assert_same_result(hb.run_variant(to_hb_graph(g), to_hb_stream(z), hb.ParallelConfig(variant="crew", max_rounds=400)),
                       want, "long chain crew")


@pytest.mark.parametrize("d", [2, 4, 8])
@pytest.mark.parametrize("resident", [False, True])
def test_ties_on_the_uniform_kernels(hb, port, d, resident):
    """Equal 64-bit keys on the uniform-size sweeps (round-1 pipelined kernel with the deferred tie
    check, later-round kernels, d = 8 without deferral), both for the caller's edge order (one-shot
    call) and for the first-pin sorted resident instance: detected, redone exactly, same result."""
    g = port.syn_generate(po.SYN_UNIFORM, n=600, m=6000, d=d, seed=11 + d)
    s = po.Stream(seed=5, kind=po.GEN_PARK_MILLER, noise_low=0.0, noise_high=2.0 ** -50)
    want = port.local_max(g, s)
    for loop in ("graph", "host"):
        cfg = hb.ParallelConfig(variant="crcw", loop_mode=loop)
        if resident:
            with hb.DeviceHypergraph.upload(to_hb_graph(g)) as dg:
                got = dg.match(to_hb_stream(s), cfg)
        else:
            got = hb.run_variant(to_hb_graph(g), to_hb_stream(s), cfg)
        assert_same_result(got, want, f"uniform d={d} resident={resident} {loop}")
        assert got.report.tie_redo_rounds >= 1
