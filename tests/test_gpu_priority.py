"""GPU parity of the priority stream: the device code the kernels use (hlm_priority.cuh) must
reproduce WeightStream::weight / tie_hash (weight_stream.hpp:78,86) bit for bit -- no FMA
contraction, IEEE division for park-miller, the same u64 -> f64 conversion."""
import json
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from tests.util import to_hb_stream

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_stream_bits_match_reference_goldens(hb):
    gold = json.load(open(os.path.join(GOLDEN, "stream_bits.json")))
    for case in gold["cases"]:
        st = case["stream"]
        s = po.Stream(seed=st["seed"], kind=st["kind"], mode=st["mode"], noise_low=st["noise_low"],
                      noise_high=st["noise_high"])
        w, t = hb.eval_stream(to_hb_stream(s), case["edges"], case["rounds"], case["base"])
        assert [format(x, "016x") for x in w.view(np.uint64)] == case["weight_bits"]
        assert [format(x, "016x") for x in t] == case["tie_hash"]


@pytest.mark.parametrize("kind", [po.GEN_XORSHIFT, po.GEN_PARK_MILLER, po.GEN_SPLITMIX])
@pytest.mark.parametrize("mode", [po.MODE_PERTURB_BASE, po.MODE_REPLACE_UNIFORM])
def test_stream_bits_match_oracle_on_a_million_pairs(hb, port, kind, mode):
    rng = np.random.default_rng(kind * 7 + mode)
    cnt = 1 << 20
    e = rng.integers(0, 2**32 - 1, cnt, dtype=np.uint64).astype(np.uint32)
    r = rng.integers(1, 189, cnt).astype(np.uint32)
    b = np.where(rng.random(cnt) < 0.5, rng.integers(1, 101, cnt).astype(np.float64), rng.random(cnt) * 1e3 + 1e-9)
    for lo, hi in ((0.0, 100.0), (0.0, 0.0), (0.125, 0.3), (7.0, 7.0)):
        s = po.Stream(seed=0x9E3779B97F4A7C15 ^ kind, kind=kind, mode=mode, noise_low=lo, noise_high=hi)
        w0, t0 = port.eval_stream(s, e, r, b)
        w1, t1 = hb.eval_stream(to_hb_stream(s), e, r, b)
        assert np.array_equal(w0.view(np.uint64), w1.view(np.uint64)), (kind, mode, lo, hi)
        assert np.array_equal(t0, t1)
