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


def test_greedy_variant_equals_greedy_sorted(hb, port, ref):
    """run_variant(Variant::greedy) (local_max_par.hpp:597-612 -> greedy_sorted, local_max_seq.hpp:130):
    the device reaches the same matching by iterating the static (weight desc, id asc) order to its
    fixpoint; matched set, total weight (summed in scan order), the one-round report and the work
    counters must equal the reference's."""
    import numpy as np

    rng = np.random.default_rng(3)
    cases = list(_instances(port))
    g = port.generate_random(3000, 5000, 2, 4, 21)
    g.base_weights = rng.random(g.m) * 10 + 0.1          # real weights: the FP sum order matters
    cases.append(("real weights", g))
    g = port.generate_random(3000, 5000, 2, 4, 22)
    g.base_weights = rng.integers(1, 4, g.m).astype(np.float64)  # heavy ties: decided by the lower id
    cases.append(("three weight classes", g))
    g = po.graph_from_edge_lists([[i, i + 1] for i in range(300)])  # unit path: dependency depth 150
    cases.append(("unit path", g))
    # long dependency chains: after 64 rounds the rest is finished by the ordered scan (hlm_greedy.cu)
    g = po.graph_from_edge_lists([[i, i + 1] for i in range(20000)])
    cases.append(("long unit path", g))
    side = 120  # unit-weight mesh in natural order (what a METIS grid graph looks like)
    mesh = [[r * side + c, r * side + c + 1] for r in range(side) for c in range(side - 1)]
    mesh += [[r * side + c, (r + 1) * side + c] for r in range(side - 1) for c in range(side)]
    cases.append(("unit mesh", po.graph_from_edge_lists(mesh)))
    g = po.graph_from_edge_lists([[i, i + 1, i + 2] for i in range(15000)])
    g.base_weights = (np.arange(g.m)[::-1] % 7 + 1).astype(np.float64) * 0.5  # weight classes along a 3-uniform chain
    cases.append(("weighted 3-uniform chain", g))
    for name, g in cases:
        want = ref.local_max(g, po.Stream(), variant=po.VARIANT_GREEDY)
        got = hb.run_variant(to_hb_graph(g), hb.WeightStream(), hb.ParallelConfig(variant="greedy"))
        assert_same_result(got, want, f"greedy {name}")
        assert got.report.rounds == 1 and got.report.work.rounds == 1
        assert got.report.work.total_edge_visits == want.edge_visits == g.m
        assert got.report.work.total_pin_visits == want.pin_visits == g.kappa
        with hb.DeviceHypergraph.upload(to_hb_graph(g)) as dg:  # resident (renumbered, sorted) instance
            again = dg.match(hb.WeightStream(), hb.ParallelConfig(variant="greedy"))
            assert_same_result(again, want, f"greedy resident {name}")
            v = dg.verify(again.matching.matched_edges)
            assert v.disjoint and v.maximal


def test_a_generous_round_cap_is_accepted(hb, port):
    """The reference takes any uint32 max_rounds; a cap used as "unlimited" must run, not be refused."""
    g = port.generate_random(2000, 4000, 2, 4, 5)
    s = po.Stream(seed=3)
    want = port.local_max(g, s)
    for variant in ("crcw", "crew", "auto"):
        got = hb.run_variant(to_hb_graph(g), to_hb_stream(s), hb.ParallelConfig(variant=variant, max_rounds=1_000_000))
        assert_same_result(got, want, f"max_rounds 1e6 {variant}")


def test_quality_band_vs_greedy_acceptance_criterion_7(hb, port):
    """acceptance.cpp:261-289 on the device: 100 instances (m = 50 .. 10^4, integer weights 1-100,
    default [0,100) noise): geometric mean of crcw weight / greedy weight >= 0.85."""
    import math

    logs, worst = 0.0, 1.0
    for i in range(100):
        m = int(50.0 * 10.0 ** (2.30103 * i / 99.0))
        g = port.generate_random(max(6, m), m, 2, 2 if i % 2 == 0 else 5, 80000 + i)
        g.base_weights = port.random_weights_1_100(g.m, 7 * i + 1)
        h = to_hb_graph(g)
        crcw = hb.run_variant(h, hb.WeightStream(seed=300 + i), hb.ParallelConfig(variant="crcw"))
        greedy = hb.run_variant(h, hb.WeightStream(), hb.ParallelConfig(variant="greedy"))
        ratio = crcw.matching.total_weight / greedy.matching.total_weight
        logs += math.log(ratio)
        worst = min(worst, ratio)
    geomean = math.exp(logs / 100)
    assert geomean >= 0.85, (geomean, worst)


def test_auto_is_crcw_to_the_caller_on_either_engine(hb, port, ref, monkeypatch):
    """HLM_B200_VARIANT_AUTO (B200 extension): same matching, report and WorkCounters as crcw, whichever
    engine the library picks (forced both ways here), on resident instances and through the one-shot
    call (which always takes the CRCW kernels)."""
    for name, g in _instances(port):
        s = po.Stream(seed=9)
        want = port.local_max(g, s)
        theirs = ref.local_max(g, s, variant=po.VARIANT_CRCW, workers=2)
        one_shot = hb.run_variant(to_hb_graph(g), to_hb_stream(s), hb.ParallelConfig(variant="auto"))
        assert_same_result(one_shot, want, f"{name} auto one-shot")
        dg = hb.DeviceHypergraph.upload(to_hb_graph(g))
        for forced in (None, "crcw", "crew"):
            if forced is None:
                monkeypatch.delenv("HLM_B200_AUTO", raising=False)
            else:
                monkeypatch.setenv("HLM_B200_AUTO", forced)
            got = dg.match(to_hb_stream(s), hb.ParallelConfig(variant="auto"))
            assert_same_result(got, want, f"{name} auto forced={forced}")
            assert got.report.work.total_edge_visits == theirs.edge_visits, f"{name} auto {forced}: edge visits"
            assert got.report.work.total_pin_visits == theirs.pin_visits, f"{name} auto {forced}: pin visits"
        dg.release()


def test_vertex_owned_run_finished_by_the_crcw_kernels(hb, port, monkeypatch):
    """variant auto on the vertex-owned engine hands the last rounds to the CRCW kernels once few edges are
    alive (hlm_crew2.inc -> crcw_tail).  Forced early here (hand-over before round 3) on instances with
    ragged and large edges, integer and real weights, and on streams whose ties send the tail's rounds
    through the exact path: matching, rounds and per-round report must equal the oracle's."""
    monkeypatch.setenv("HLM_B200_AUTO", "crew")
    monkeypatch.setenv("HLM_B200_CREW_TAIL", "100000")  # percent of n alive pins: always true from round 2 on
    cases = [
        ("netlist", po.SYN_NETLIST, dict(n=60_000, m=120_000), True),
        # (above 4 M pins: smaller 8-uniform instances belong to the CRCW engine and are loaded in its edge order)
        ("uniform", po.SYN_UNIFORM, dict(n=280_000, m=560_000, d=8), False),
        ("powerlaw", po.SYN_POWERLAW, dict(n=50_000, m=100_000), False),
    ]
    streams = [po.Stream(seed=4), po.Stream(seed=4, noise_high=0.0), po.Stream(seed=8, kind=po.GEN_PARK_MILLER, noise_high=2.0 ** -50),
               po.Stream(seed=2, mode=po.MODE_REPLACE_UNIFORM)]
    for family, fam_id, kw, intw in cases:
        g = port.syn_generate(fam_id, seed=6, int_weights=intw, **kw)
        dg = hb.DeviceHypergraph.generate(family, seed=6, int_weights=intw, **kw)
        for s in streams:
            want = port.local_max(g, s)
            for loop in ("graph", "host"):
                got = dg.match(to_hb_stream(s), hb.ParallelConfig(variant="auto", loop_mode=loop))
                assert_same_result(got, want, f"{family} tail {loop} {s}")
                assert "crcw from round 3" in got.report.engine, got.report.engine
            # the round cap hit inside the tail: partial matching and report of exactly 3 rounds
            capped = port.local_max(g, s, max_rounds=3)
            if capped.status == po.ROUND_LIMIT:
                import pytest

                with pytest.raises(hb.RoundLimitError) as ei:
                    dg.match(to_hb_stream(s), hb.ParallelConfig(variant="auto", max_rounds=3))
                assert list(ei.value.partial.matched_edges) == list(capped.matched_edges)
                assert ei.value.report.deactivated_per_round == capped.per_round_deactivated
        dg.release()


def test_round_cap_with_ties_on_every_engine(hb, port):
    """A tie seen by the sweep that follows the last allowed round must not commit anything (the sweep only counts
    what that round deactivated): round cap + tie-prone streams on crcw, crew and auto."""
    g = port.generate_random(4000, 9000, 2, 5, 12)
    for s in (po.Stream(seed=5, noise_high=0.0), po.Stream(seed=5, kind=po.GEN_PARK_MILLER, noise_high=2.0 ** -50)):
        for cap in (1, 2, 3):
            want = port.local_max(g, s, max_rounds=cap)
            if want.status != po.ROUND_LIMIT:
                continue
            for variant in ("crcw", "crew", "auto"):
                with pytest.raises(hb.RoundLimitError) as ei:
                    hb.run_variant(to_hb_graph(g), to_hb_stream(s), hb.ParallelConfig(variant=variant, max_rounds=cap))
                assert list(ei.value.partial.matched_edges) == list(want.matched_edges), (variant, cap)
                assert ei.value.report.matched_per_round_count == want.per_round_matched
                assert ei.value.report.deactivated_per_round == want.per_round_deactivated
