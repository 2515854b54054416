"""The one-launch kernel of small instances (uniform d = 2 / 4 / 8, or ragged sizes: k_rounds_fused): initialisation,
every round and the result assembly in one cooperative launch.  It must give what the oracle gives --
matching, rounds, per-round counts, total weight -- on every path through it: integer weights (summed on the
device), unit weights, real weights (assembly on the usual path), ties (the kernel hands the round to the
exact redo and is relaunched), the round cap, the round record switched off; and it must be what actually
ran (one kernel launch per matching)."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.util import assert_same_result, to_hb_graph, to_hb_stream

pytestmark = pytest.mark.gpu


def _weighted(port, g):
    g.base_weights = port.random_weights_1_100(g.m, 3)
    return g


def _cases(port):
    yield "4-uniform, unit weights", port.generate_random(30_000, 30_000, 4, 4, 1), True
    yield "2-uniform graph, weights 1-100", port.syn_generate(po.SYN_RMAT, scale=13, m=60_000, seed=2, int_weights=True), True
    yield "8-uniform, weights 1-100", port.syn_generate(po.SYN_UNIFORM, n=20_000, m=30_000, d=8, seed=3, int_weights=True), True
    # real weights: rounds in the kernel, the ordered FP64 sum needs the usual assembly (3 more kernels)
    real = port.syn_generate(po.SYN_UNIFORM, n=9_000, m=20_000, d=4, seed=5)
    real.base_weights[:] = 0.25 + np.random.default_rng(11).random(real.m) * 7.5
    yield "4-uniform, real weights", real, None
    yield "one edge", port.generate_random(4, 1, 4, 4, 1), True
    yield "ragged 2..5", port.generate_random(2000, 3500, 2, 5, 7), True
    yield "ragged 1..30, weights 1-100", _weighted(port, port.generate_random(30_000, 20_000, 1, 30, 5)), True
    yield "power-law 2..64 (edges above 32 pins: warp per edge)", port.syn_generate(po.SYN_POWERLAW, n=4000, m=6000, seed=5), True
    yield "netlist <= 4096, weights 1-100", port.syn_generate(po.SYN_NETLIST, n=9000, m=12000, seed=6, int_weights=True), True
    yield "3-uniform (the ragged form)", port.generate_random(3000, 4000, 3, 3, 2), True
    yield "40-uniform (every edge a warp's)", port.generate_random(30_000, 2000, 40, 40, 2), True


STREAMS = [po.Stream(seed=1), po.Stream(seed=4, noise_high=0.0),  # every key of a weight class ties
           po.Stream(seed=8, kind=po.GEN_PARK_MILLER, noise_high=2.0 ** -50),
           po.Stream(seed=2, mode=po.MODE_REPLACE_UNIFORM), po.Stream(seed=3, kind=po.GEN_SPLITMIX)]


def test_one_launch_matching_equals_the_oracle(hb, port):
    for name, g, eligible in _cases(port):
        dg = hb.DeviceHypergraph.upload(to_hb_graph(g))
        for s in STREAMS:
            want = port.local_max(g, s)
            got = dg.match(to_hb_stream(s), hb.ParallelConfig(variant="crcw", loop_mode="graph"))
            assert_same_result(got, want, f"{name} {s}")
            if eligible and got.report.tie_redo_rounds == 0:
                assert got.report.kernel_launches == 1, (name, got.report.kernel_launches)
            if eligible is not True:
                assert got.report.kernel_launches > 1
            # the round record switched off: same ids, no round array
            bare = dg.match(to_hb_stream(s), hb.ParallelConfig(variant="crcw", loop_mode="graph", want_round_of=False))
            assert np.array_equal(bare.matching.matched_edges, got.matching.matched_edges)
            assert bare.matching.total_weight == got.matching.total_weight
            # the host-driven loop of the stand-alone kernels on the same instance
            host = dg.match(to_hb_stream(s), hb.ParallelConfig(variant="crcw", loop_mode="host"))
            assert_same_result(host, want, f"{name} host loop {s}")
        dg.release()


def test_one_launch_matching_round_cap_and_repeat(hb, port):
    g = port.generate_random(30_000, 30_000, 4, 4, 1)
    dg = hb.DeviceHypergraph.upload(to_hb_graph(g))
    for s in (po.Stream(seed=1), po.Stream(seed=4, noise_high=0.0)):
        for cap in (1, 2, 3):
            want = port.local_max(g, s, max_rounds=cap)
            assert want.status == po.ROUND_LIMIT
            with pytest.raises(hb.RoundLimitError) as ei:
                dg.match(to_hb_stream(s), hb.ParallelConfig(variant="crcw", max_rounds=cap))
            assert list(ei.value.partial.matched_edges) == list(want.matched_edges)
            assert ei.value.report.matched_per_round_count == want.per_round_matched
            assert ei.value.report.deactivated_per_round == want.per_round_deactivated
        # the instance's scratch is reused call after call: a capped run must leave nothing behind
        want = port.local_max(g, s)
        for _ in range(3):
            got = dg.match(to_hb_stream(s), hb.ParallelConfig(variant="auto"))
            assert_same_result(got, want, f"repeat {s}")
    dg.release()


def test_one_launch_kernel_switched_off_gives_the_same(hb, port, monkeypatch):
    g = port.syn_generate(po.SYN_UNIFORM, n=20_000, m=40_000, d=4, seed=9, int_weights=True)
    dg = hb.DeviceHypergraph.upload(to_hb_graph(g))
    s = po.Stream(seed=6)
    fused = dg.match(to_hb_stream(s), hb.ParallelConfig(variant="crcw"))
    assert fused.report.kernel_launches == 1
    monkeypatch.setenv("HLM_B200_FUSED_MAX_PINS", "0")
    graph = dg.match(to_hb_stream(s), hb.ParallelConfig(variant="crcw"))
    assert graph.report.kernel_launches > 1
    monkeypatch.setenv("HLM_B200_FUSED_MAX_PINS", str(1 << 40))
    monkeypatch.setenv("HLM_B200_NO_FUSED_RESULT", "1")  # rounds in the kernel, assembly by the usual kernels
    mixed = dg.match(to_hb_stream(s), hb.ParallelConfig(variant="crcw"))
    for other in (graph, mixed):
        assert np.array_equal(other.matching.matched_edges, fused.matching.matched_edges)
        assert np.array_equal(other.report.matched_round, fused.report.matched_round)
        assert other.report.matched_per_round_count == fused.report.matched_per_round_count
        assert other.report.deactivated_per_round == fused.report.deactivated_per_round
        assert other.matching.total_weight == fused.matching.total_weight
    dg.release()


def test_refused_cooperative_launch_falls_back_to_the_graph_loop(hb, port, monkeypatch):
    """An SM-limited context (MPS share, green context) can refuse the cooperative launch: the instance then
    runs on the CUDA-graph loop, in that call and in every later one, with the same result."""
    g = port.syn_generate(po.SYN_UNIFORM, n=20_000, m=40_000, d=4, seed=9, int_weights=True)
    s = po.Stream(seed=6)
    want = port.local_max(g, s)
    dg = hb.DeviceHypergraph.upload(to_hb_graph(g))
    monkeypatch.setenv("HLM_B200_FUSED_REFUSE", "1")
    got = dg.match(to_hb_stream(s), hb.ParallelConfig(variant="crcw"))
    assert_same_result(got, want, "refused launch")
    assert got.report.kernel_launches > 1
    monkeypatch.delenv("HLM_B200_FUSED_REFUSE")
    again = dg.match(to_hb_stream(s), hb.ParallelConfig(variant="crcw"))  # stays on the graph loop
    assert_same_result(again, want, "after a refused launch")
    assert again.report.kernel_launches > 1
    dg.release()
