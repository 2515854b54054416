"""GPU parity of the one-shot drop-in call (hlm_b200_match_host) across the loader's paths:
host-assisted (uniformity scan of the offsets and one-byte packing of the weights on the host
cores while the pins cross PCIe) vs the plain upload, and resident (first-pin sorted) vs one-shot
(caller's edge order).  Every path must give the oracle's result bit for bit."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.util import assert_same_result, to_hb_graph, to_hb_stream

pytestmark = pytest.mark.gpu


def _variants(port):
    """(name, graph) pairs that take the different branches of the loader."""
    out = []
    g = port.syn_generate(po.SYN_RMAT, scale=13, m=60000, seed=3, int_weights=True)
    out.append(("uniform d=2, weights 1..100: offsets skipped, weights packed", g))
    g2 = port.syn_generate(po.SYN_RMAT, scale=13, m=60000, seed=3, int_weights=True)
    g2.base_weights = g2.base_weights.copy()
    g2.base_weights[12345] = 0.5  # not an integer: the weights go up as doubles
    out.append(("uniform, one fractional weight: weights raw", g2))
    g3 = port.syn_generate(po.SYN_RMAT, scale=13, m=60000, seed=3, int_weights=True)
    g3.base_weights = g3.base_weights.copy()
    g3.base_weights[59999] = 256.0  # outside one byte
    out.append(("uniform, weight 256: weights raw", g3))
    g4 = port.syn_generate(po.SYN_UNIFORM, n=20000, m=50000, d=4, seed=5, int_weights=False)
    out.append(("uniform d=4, unit weights: packed then folded to a constant", g4))
    g5 = port.syn_generate(po.SYN_NETLIST, n=30000, m=50000, seed=2, int_weights=True)
    out.append(("ragged sizes: 16-bit sizes instead of offsets, weights packed", g5))
    g7 = port.generate_random(70000, 3, 2, 5, 9)
    lists7 = [list(g7.edge_members[int(g7.edge_offsets[e]):int(g7.edge_offsets[e + 1])]) for e in range(g7.m)]
    lists7.append(list(range(66000)))  # one edge of 66 000 pins: does not fit 16 bits, offsets raw
    lists7 += [[e % 70000, (e * 7 + 1) % 70000 if (e * 7 + 1) % 70000 != e % 70000 else (e + 2) % 70000] for e in range(3000)]
    out.append(("ragged with a 66 000-pin edge: offsets raw", po.graph_from_edge_lists(lists7, [1.0] * len(lists7), n=70000)))
    g8 = port.generate_random(30000, 80000, 2, 2, 4)
    lists8 = [list(g8.edge_members[int(g8.edge_offsets[e]):int(g8.edge_offsets[e + 1])]) for e in range(g8.m)]
    for e in range(70000, 70050):  # uniform for the first 70 000 edges (beyond the loader's look-ahead), then ragged
        v = 0
        while v in lists8[e]:
            v += 1
        lists8[e].append(v)
    out.append(("uniform prefix, ragged later: offsets raw", po.graph_from_edge_lists(lists8, [1.0] * g8.m, n=g8.n)))
    g6 = port.generate_random(30000, 50000, 3, 3, 4)
    lists = [list(g6.edge_members[int(g6.edge_offsets[e]):int(g6.edge_offsets[e + 1])]) for e in range(g6.m)]
    extra = 0
    while extra in lists[-1]:
        extra += 1
    lists[-1].append(extra)  # only the LAST edge breaks uniformity
    out.append(("uniform except the last edge: offsets raw", po.graph_from_edge_lists(lists, [1.0] * g6.m, n=g6.n)))
    return out


@pytest.mark.parametrize("assist", [True, False])
def test_one_shot_call_on_every_loader_path(hb, port, monkeypatch, assist):
    if assist:
        monkeypatch.setenv("HLM_B200_ASSIST_MIN_EDGES", "1000")
    else:
        monkeypatch.setenv("HLM_B200_NO_HOST_ASSIST", "1")
    streams = [po.Stream(seed=5), po.Stream(seed=5, noise_high=0.0)]
    for name, g in _variants(port):
        for s in streams:
            want = port.local_max(g, s)
            got = hb.run_variant(to_hb_graph(g), to_hb_stream(s))
            assert_same_result(got, want, f"{name} assist={assist} {s}")
            expect_bytes = g.edge_members.nbytes + g.edge_offsets.nbytes + g.base_weights.nbytes
            if assist and name.startswith("uniform d="):
                assert got.report.h2d_bytes == g.edge_members.nbytes + g.m  # pins + one byte per weight
            elif assist and "16-bit sizes" in name:
                assert got.report.h2d_bytes == g.edge_members.nbytes + 2 * g.m + g.m  # pins + sizes + weight codes
            elif assist and "offsets raw" in name and "last edge" not in name:
                assert got.report.h2d_bytes >= g.edge_members.nbytes + g.edge_offsets.nbytes
            elif not assist:
                assert got.report.h2d_bytes == expect_bytes


def test_host_assist_rejects_bad_pins(hb, port, monkeypatch):
    monkeypatch.setenv("HLM_B200_ASSIST_MIN_EDGES", "1000")
    g = port.syn_generate(po.SYN_UNIFORM, n=5000, m=20000, d=2, seed=1, int_weights=True)
    g.edge_members = g.edge_members.copy()
    g.edge_members[777] = 5000  # == n: out of range
    with pytest.raises(hb.InputError):
        hb.run_variant(to_hb_graph(g), hb.WeightStream())


def test_resident_and_one_shot_agree_at_scale(hb):
    """2^22 edges (the default host-assist threshold): the resident path (first-pin sorted) and
    the one-shot path (caller order, host-assisted loader) must return the same matching."""
    dg = hb.DeviceHypergraph.generate("rmat", scale=18, m=1 << 22, seed=7, int_weights=True)
    s = hb.WeightStream(seed=3)
    a = dg.match(s)
    host = dg.download()
    dg.release()
    b = hb.run_variant(host, s)
    assert np.array_equal(a.matching.matched_edges, b.matching.matched_edges)
    assert a.report.matched_per_round_count == b.report.matched_per_round_count
    assert a.report.deactivated_per_round == b.report.deactivated_per_round
    assert a.matching.total_weight == b.matching.total_weight
    assert b.report.h2d_bytes == host.edge_members.nbytes + host.num_edges
