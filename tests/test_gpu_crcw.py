"""GPU parity: the CUDA CRCW path through the C-ABI vs the CPU oracle, bit-exact."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.util import assert_same_result, to_hb_graph, to_hb_stream

pytestmark = pytest.mark.gpu


def _streams(seed):
    return [
        po.Stream(seed=seed),
        po.Stream(seed=seed, mode=po.MODE_REPLACE_UNIFORM),
        po.Stream(seed=seed, noise_high=0.0),
        po.Stream(seed=seed, kind=po.GEN_PARK_MILLER),
        po.Stream(seed=seed, kind=po.GEN_SPLITMIX, noise_low=1.0, noise_high=3.5),
        po.Stream(seed=seed, kind=po.GEN_PARK_MILLER, mode=po.MODE_REPLACE_UNIFORM),
    ]


@pytest.mark.parametrize("loop_mode", ["host", "graph"])
@pytest.mark.parametrize("tie_mode", ["auto", "exact"])
def test_random_corpus_matches_oracle(hb, port, loop_mode, tie_mode):
    """test_par.cpp:32-55 on the device: matched set, rounds and per-round sets == sequential."""
    for seed in range(1, 13):
        g = port.generate_random(40 + 30 * seed, 60 + 50 * seed, 2, 4, seed)
        if seed % 3 == 0:
            g.base_weights = port.random_weights_1_100(g.m, seed)
        for s in _streams(seed * 7):
            want = port.local_max(g, s)
            got = hb.run_variant(to_hb_graph(g), to_hb_stream(s),
                                 hb.ParallelConfig(variant="crcw", loop_mode=loop_mode, tie_mode=tie_mode))
            assert_same_result(got, want, f"seed {seed} stream {s}")


def test_config1_golden(hb, port):
    """BASELINE config 1 against the reference-generated golden."""
    g = port.generate_random(1000000, 1000000, 4, 4, 1)
    got = hb.run_variant(to_hb_graph(g), hb.WeightStream())
    assert got.report.rounds == 5
    assert got.report.matched_per_round_count == [62600, 46336, 28540, 6717, 306]
    assert got.report.deactivated_per_round == [649722, 171213, 32049, 2468, 49]
    assert po.fnv1a_ids(got.matching.matched_edges) == 0x5F60F5D9FB1486B9
    assert got.matching.total_weight == 144499.0


def test_crew_matches_oracle(hb, port):
    """local_max_crew (local_max_par.hpp:258) on the device: natively exact comparator."""
    for seed in range(1, 11):
        g = port.generate_random(50 + 40 * seed, 80 + 70 * seed, 1 if seed % 4 == 0 else 2, 5, seed)
        if seed % 2 == 0:
            g.base_weights = port.random_weights_1_100(g.m, seed)
        elif seed % 4 == 1:  # fractional weights: the caller's f64 array is read per incidence entry
            g.base_weights = np.asarray(port.random_weights_1_100(g.m, seed), dtype=np.float64) * 0.37 + 0.11
        for s in _streams(seed * 3):
            want = port.local_max(g, s)
            got = hb.run_variant(to_hb_graph(g), to_hb_stream(s), hb.ParallelConfig(variant="crew"))
            assert_same_result(got, want, f"crew seed {seed} stream {s}")
            # WorkCounters follow the reference's crew formulas (5 m and 4 kappa per round)
            assert got.report.work.total_edge_visits == 5 * g.m * want.rounds
            assert got.report.work.total_pin_visits == 4 * g.kappa * want.rounds


def test_config1_all_stream_modes_both_variants(hb, port):
    import json
    import os

    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "config1.json")))["cases"]
    g = port.generate_random(1000000, 1000000, 4, 4, 1)
    ints = port.random_weights_1_100(g.m, 1)
    for variant in ("crcw", "crew"):
        for name, case in gold.items():
            hg = to_hb_graph(g)
            if case["weights_seed"] is not None:
                hg.base_weights = ints
            st = case["stream"]
            s = po.Stream(seed=st["seed"], kind=st["kind"], mode=st["mode"], noise_low=st["noise_low"],
                          noise_high=st["noise_high"])
            got = hb.run_variant(hg, to_hb_stream(s), hb.ParallelConfig(variant=variant))
            assert got.report.rounds == case["rounds"], (variant, name)
            assert got.report.matched_per_round_count == case["per_round_matched"], (variant, name)
            assert got.report.deactivated_per_round == case["per_round_deactivated"], (variant, name)
            assert format(po.fnv1a_ids(got.matching.matched_edges), "016x") == case["fnv1a"], (variant, name)
            assert got.matching.total_weight == case["total_weight"], (variant, name)
