"""run_variant (local_max_par.hpp:586) with every Variant the device accepts: seq, crcw, crew and
work_optimal return the same matching (test_par.cpp:32-55) and their WorkCounters must equal what
the UNMODIFIED reference reports for that variant on the same input (oracle/_ref, prebuilt here
and shipped to the GPU box), on uniform and ragged instances, including large edges."""
import pytest

from oracle import pyoracle as po
from tests.util import assert_same_result, to_hb_graph, to_hb_stream

pytestmark = pytest.mark.gpu

VARIANTS = [("seq", po.VARIANT_SEQ), ("crcw", po.VARIANT_CRCW), ("crew", po.VARIANT_CREW),
            ("work_optimal", po.VARIANT_WORK_OPTIMAL)]


def _instances(port):
    yield "uniform d=4", port.syn_generate(po.SYN_UNIFORM, n=3000, m=5000, d=4, seed=3, int_weights=True)
    yield "graph d=2", port.syn_generate(po.SYN_RMAT, scale=10, m=8000, seed=2, int_weights=True)
    yield "ragged 2..5", port.generate_random(2000, 3500, 2, 5, 7)
    yield "power-law 2..64 (large edges)", port.syn_generate(po.SYN_POWERLAW, n=4000, m=6000, seed=5)
    yield "netlist <= 4096", port.syn_generate(po.SYN_NETLIST, n=9000, m=12000, seed=6, int_weights=True)


def test_every_variant_matches_the_reference_including_work_counters(hb, port, ref):
    for name, g in _instances(port):
        for s in (po.Stream(seed=4), po.Stream(seed=4, noise_high=0.0)):
            want = port.local_max(g, s)
            for vname, vid in VARIANTS:
                got = hb.run_variant(to_hb_graph(g), to_hb_stream(s), hb.ParallelConfig(variant=vname))
                assert_same_result(got, want, f"{name} {vname} {s}")
                theirs = ref.local_max(g, s, variant=vid, workers=2)
                assert theirs.rounds == got.report.rounds
                assert got.report.work.total_edge_visits == theirs.edge_visits, f"{name} {vname}: edge visits"
                assert got.report.work.total_pin_visits == theirs.pin_visits, f"{name} {vname}: pin visits"
                if vname == "work_optimal":
                    assert got.report.work.prefix_sum_invocations == 4 * got.report.rounds  # local_max_par.hpp:450
                    assert got.report.work.compactions == got.report.rounds
                else:
                    assert got.report.work.prefix_sum_invocations == 0 and got.report.work.compactions == 0


def test_work_optimal_counters_config1_golden(hb, port):
    """the reference's opt counters on config 1 are 32 344 460 pin / 5 470 808 edge
    visits (seq / crcw: 60 000 000 / 15 000 000; crew: 80 000 000 / 25 000 000)."""
    g = port.generate_random(1000000, 1000000, 4, 4, 1)
    h = to_hb_graph(g)
    expect = {"work_optimal": (32344460, 5470808), "crcw": (60000000, 15000000), "seq": (60000000, 15000000),
              "crew": (80000000, 25000000)}
    for vname, (pins, edges) in expect.items():
        got = hb.run_variant(h, hb.WeightStream(), hb.ParallelConfig(variant=vname))
        assert po.fnv1a_ids(got.matching.matched_edges) == 0x5F60F5D9FB1486B9
        assert got.report.work.total_pin_visits == pins, vname
        assert got.report.work.total_edge_visits == edges, vname


def test_work_optimal_round_cap(hb, port):
    g = port.generate_random(2000, 3500, 2, 5, 7)
    s = po.Stream(seed=2)
    want = port.local_max(g, s, max_rounds=2)
    assert want.status == po.ROUND_LIMIT
    with pytest.raises(hb.RoundLimitError) as ei:
        hb.run_variant(to_hb_graph(g), to_hb_stream(s), hb.ParallelConfig(variant="work_optimal", max_rounds=2))
    assert list(ei.value.partial.matched_edges) == list(want.matched_edges)
