"""GPU parity of the loader: device-side synthetic generators vs their CPU restatement
(oracle/hlm_oracle.c orc_syn_*), upload/download round trips, device verify vs oracle verify."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.util import assert_same_result, to_hb_graph, to_hb_stream

pytestmark = pytest.mark.gpu

CASES = [
    ("uniform", po.SYN_UNIFORM, dict(n=5000, m=20000, d=4), False),
    ("uniform", po.SYN_UNIFORM, dict(n=3000, m=9000, d=8), True),
    ("uniform", po.SYN_UNIFORM, dict(n=200, m=3000, d=3), True),
    ("rmat", po.SYN_RMAT, dict(scale=12, m=60000), True),
    ("powerlaw", po.SYN_POWERLAW, dict(n=20000, m=40000), False),
    ("netlist", po.SYN_NETLIST, dict(n=30000, m=60000), True),
]


@pytest.mark.parametrize("family,fam_id,kw,intw", CASES)
def test_generator_matches_cpu_restatement(hb, port, family, fam_id, kw, intw):
    want = port.syn_generate(fam_id, seed=5, int_weights=intw, **kw)
    with hb.DeviceHypergraph.generate(family, seed=5, int_weights=intw, **kw) as dg:
        got = dg.download(with_incidence=True)
        info = dg.info()
        assert (got.num_vertices, got.num_edges) == (want.n, want.m)
        assert np.array_equal(got.edge_offsets, want.edge_offsets)
        assert np.array_equal(got.edge_members, want.edge_members)
        assert np.array_equal(got.base_weights, want.base_weights)
        # incidence lists: same sets per vertex (order inside a list is unspecified)
        assert np.array_equal(got.vertex_offsets, want.vertex_offsets)
        order = np.lexsort((got.vertex_incidence, np.repeat(np.arange(want.n), np.diff(want.vertex_offsets).astype(np.int64))))
        assert np.array_equal(got.vertex_incidence[order], want.vertex_incidence)
        if family == "netlist":
            assert info.num_large_edges > 0 and info.max_edge_size > 32
        # matching on the generated instance == oracle on the CPU-generated one
        for s in (po.Stream(seed=3), po.Stream(seed=3, noise_high=0.0)):
            ref = port.local_max(want, s)
            res = dg.match(to_hb_stream(s), hb.ParallelConfig(variant="crcw"))
            assert_same_result(res, ref, f"{family} {s}")
            v = dg.verify(res.matching.matched_edges)
            assert v.valid() and v.weight == ref.total_weight
            assert port.verify(want, ref.matched_edges)[:2] == (True, True)


def test_edge_shards_concatenate_to_the_whole_instance(hb, port):
    """Counter-based generation: shard [b, b+k) of an instance equals rows b..b+k of the whole."""
    whole = port.syn_generate(po.SYN_UNIFORM, n=4000, m=10000, d=8, seed=9)
    parts = []
    for b, k in ((0, 3000), (3000, 3000), (6000, 4000)):
        with hb.DeviceHypergraph.generate("uniform", n=4000, m=10000, d=8, seed=9, edge_begin=b, m_local=k) as dg:
            parts.append(dg.download().edge_members)
    assert np.array_equal(np.concatenate(parts), whole.edge_members)


def test_upload_download_roundtrip_and_reorder_invariance(hb, port, monkeypatch):
    g = port.generate_random(3000, 8000, 4, 4, 11)
    g.base_weights = port.random_weights_1_100(g.m, 4)
    s = po.Stream(seed=8)
    want = port.local_max(g, s)
    for reorder in ("1", "0"):
        monkeypatch.setenv("HLM_B200_REORDER", reorder)
        with hb.DeviceHypergraph.upload(to_hb_graph(g)) as dg:
            back = dg.download()
            assert np.array_equal(back.edge_offsets, g.edge_offsets)
            assert np.array_equal(back.edge_members, g.edge_members)
            assert np.array_equal(back.base_weights, g.base_weights)
            assert_same_result(dg.match(to_hb_stream(s)), want, f"reorder={reorder}")


def test_verify_flags_bad_matchings(hb, port):
    g = port.generate_random(500, 900, 2, 5, 2)
    want = port.local_max(g, po.Stream())
    with hb.DeviceHypergraph.upload(to_hb_graph(g)) as dg:
        ok = dg.verify(want.matched_edges)
        assert ok.valid() and ok.weight == want.total_weight
        fewer = dg.verify(want.matched_edges[:-1])  # still disjoint, no longer maximal
        assert fewer.disjoint and not fewer.maximal
        assert (fewer.disjoint, fewer.maximal) == port.verify(g, want.matched_edges[:-1])[:2]
        # add an edge that shares a vertex with a matched one
        matched = set(want.matched_edges.tolist())
        extra = next(e for e in range(g.m) if e not in matched)
        both = np.sort(np.append(want.matched_edges, extra)).astype(np.uint32)
        bad = dg.verify(both)
        assert not bad.disjoint
        assert (bad.disjoint, bad.maximal) == port.verify(g, both)[:2]
        dup = dg.verify(np.append(want.matched_edges, want.matched_edges[0]).astype(np.uint32))
        assert not dup.disjoint
        with pytest.raises(hb.InputError):
            dg.verify(np.array([g.m], dtype=np.uint32))
