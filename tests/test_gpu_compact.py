"""compact (local_max_par.hpp:350-454) on the device against the reference's own compact
(oracle/_ref): the cases of tests/test_par.cpp:101-158 and acceptance criterion 9, plus flags taken
from real matching rounds on a larger instance."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.util import to_hb_graph, to_hb_stream

pytestmark = pytest.mark.gpu


def _same(got, want_graph, want_vmap, want_emap, what=""):
    g = got.graph
    assert (g.num_vertices, g.num_edges) == (want_graph.n, want_graph.m), what
    for a, b in ((g.vertex_offsets, want_graph.vertex_offsets), (g.vertex_incidence, want_graph.vertex_incidence),
                 (g.edge_offsets, want_graph.edge_offsets), (g.edge_members, want_graph.edge_members),
                 (g.base_weights, want_graph.base_weights), (got.vertex_map, want_vmap), (got.edge_map, want_emap)):
        assert np.array_equal(np.asarray(a), np.asarray(b)), what


def test_identity_and_empty(hb, port):
    g = port.generate_random(20, 25, 2, 4, 5)  # test_par.cpp:101-108
    h = to_hb_graph(g, with_incidence=True)
    c = hb.compact(h, np.ones(g.n, np.uint8), np.ones(g.m, np.uint8))
    _same(c, g, np.arange(g.n, dtype=np.uint32), np.arange(g.m, dtype=np.uint32), "identity")
    t = port.tight_family(3, 0.1)  # :110-117
    c = hb.compact(to_hb_graph(t, with_incidence=True), np.zeros(t.n, np.uint8), np.zeros(t.m, np.uint8))
    assert c.graph.num_vertices == 0 and c.graph.num_edges == 0
    assert c.graph.vertex_offsets.tolist() == [0] and c.graph.edge_offsets.tolist() == [0]


def test_random_flag_sets_equal_the_reference(hb, port, ref):
    rng = np.random.default_rng(17)  # test_par.cpp:119-150
    for trial in range(100):
        g = port.generate_random(25, 30, 2, 4, 300 + trial)
        if trial % 2:
            g.base_weights = port.random_weights_1_100(g.m, trial)
        v_active = (rng.integers(0, 4, g.n) != 0).astype(np.uint8)
        e_active = np.zeros(g.m, np.uint8)
        for e in range(g.m):
            members = g.edge_members[int(g.edge_offsets[e]):int(g.edge_offsets[e + 1])]
            e_active[e] = 1 if (rng.integers(0, 5) != 0 and v_active[members].all()) else 0
        rc, wg, wv, we, wc = ref.compact(g, v_active, e_active, workers=1 + trial % 4)
        assert rc == po.OK
        got = hb.compact(to_hb_graph(g, with_incidence=True), v_active, e_active)
        _same(got, wg, wv, we, f"trial {trial}")
        assert [got.work.total_edge_visits, got.work.total_pin_visits, got.work.prefix_sum_invocations,
                got.work.compactions] == wc


def test_precondition_error(hb, port, ref):
    g = po.graph_from_edge_lists([[0, 1], [1, 2]])  # test_par.cpp:152-158
    v_active, e_active = np.array([1, 0, 1], np.uint8), np.array([1, 0], np.uint8)
    assert ref.compact(g, v_active, e_active)[0] == po.INPUT_ERROR
    with pytest.raises(hb.InputError):
        hb.compact(to_hb_graph(g, with_incidence=True), v_active, e_active)


def test_flags_of_real_rounds_on_a_larger_instance(hb, port, ref):
    """acceptance criterion 9 style: the active part after 1 and after 2 matching rounds of a
    200 K-edge instance, compacted on the device and by the reference."""
    g = port.generate_random(150000, 200000, 2, 6, 9)
    g.base_weights = port.random_weights_1_100(g.m, 4)
    s = po.Stream(seed=8)
    for cap in (1, 2):
        part = port.local_max(g, s, max_rounds=cap)
        covered = np.zeros(g.n, bool)
        for e in part.matched_edges:
            covered[g.edge_members[int(g.edge_offsets[e]):int(g.edge_offsets[e + 1])]] = True
        sizes = np.diff(g.edge_offsets).astype(np.int64)
        touched = np.add.reduceat(covered[g.edge_members].astype(np.int64), g.edge_offsets[:-1].astype(np.int64))
        e_active = (touched == 0).astype(np.uint8)
        assert sizes.min() >= 1
        v_active = (~covered).astype(np.uint8)
        rc, wg, wv, we, wc = ref.compact(g, v_active, e_active, workers=4)
        assert rc == po.OK and wg.m < g.m
        got = hb.compact(to_hb_graph(g, with_incidence=True), v_active, e_active)
        _same(got, wg, wv, we, f"after {cap} round(s)")
        assert got.work.total_pin_visits == wc[1]
