"""Edge-partitioned matching: k virtual ranks on ONE GPU run the real multi-GPU protocol (same
kernels, same step-level C-ABI, collectives replaced by element-wise ops between the shards'
buffers).  The result must not depend on k (the reference's invariant: independent of workers,
test_par.cpp:32-55) and must equal the oracle on the unpartitioned instance."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.util import assert_same_result, to_hb_stream

pytestmark = pytest.mark.gpu

FAMILIES = [
    ("uniform", po.SYN_UNIFORM, dict(n=6000, m=20000, d=8), False),
    ("uniform", po.SYN_UNIFORM, dict(n=9000, m=15000, d=4), True),
    ("rmat", po.SYN_RMAT, dict(scale=11, m=30000), True),
    ("powerlaw", po.SYN_POWERLAW, dict(n=8000, m=12000), False),
    ("netlist", po.SYN_NETLIST, dict(n=9000, m=15000), True),
]


@pytest.mark.parametrize("family,fam_id,kw,intw", FAMILIES)
def test_shard_count_never_changes_the_matching(hb, port, family, fam_id, kw, intw):
    from paper_2602_22976_b200 import multi_gpu

    g = port.syn_generate(fam_id, seed=4, int_weights=intw, **kw)
    streams = [po.Stream(seed=9), po.Stream(seed=9, noise_high=0.0), po.Stream(seed=2, mode=po.MODE_REPLACE_UNIFORM)]
    for s in streams:
        want = port.local_max(g, s)
        for world in (1, 2, 3, 8):
            sm = multi_gpu.virtual_cluster(family, world, seed=4, int_weights=intw, **kw)
            got = sm.match(to_hb_stream(s), hb.ParallelConfig(variant="crcw"))
            assert_same_result(got, want, f"{family} world={world} {s}")
            for tie_mode in (("exact",) if world == 2 else ()):
                got = sm.match(to_hb_stream(s), hb.ParallelConfig(variant="crcw", tie_mode=tie_mode))
                assert_same_result(got, want, f"{family} world={world} exact {s}")
            for e in sm.engines:
                e.shard.release()


def test_cross_shard_ties_take_the_exact_path(hb, port):
    """Collapsed weights: equal maxima held by edges of different shards are invisible to the
    local atomics; the claimant count must catch them."""
    from paper_2602_22976_b200 import multi_gpu

    kw = dict(n=3000, m=12000, d=2)
    g = port.syn_generate(po.SYN_UNIFORM, seed=6, **kw)
    s = po.Stream(seed=5, kind=po.GEN_PARK_MILLER, noise_low=0.0, noise_high=2.0 ** -50)
    want = port.local_max(g, s)
    for world in (2, 4):
        sm = multi_gpu.virtual_cluster("uniform", world, seed=6, **kw)
        got = sm.match(to_hb_stream(s))
        assert_same_result(got, want, f"ties world={world}")
        assert got.report.tie_redo_rounds >= 1
        for e in sm.engines:
            e.shard.release()


def test_round_cap_in_sharded_runs(hb, port):
    from paper_2602_22976_b200 import multi_gpu

    kw = dict(n=2000, m=6000, d=3)
    g = port.syn_generate(po.SYN_UNIFORM, seed=2, **kw)
    s = po.Stream(seed=1)
    want = port.local_max(g, s, max_rounds=2)
    assert want.status == po.ROUND_LIMIT
    sm = multi_gpu.virtual_cluster("uniform", 2, seed=2, **kw)
    with pytest.raises(hb.RoundLimitError) as ei:
        sm.match(to_hb_stream(s), hb.ParallelConfig(max_rounds=2))
    assert np.array_equal(ei.value.partial.matched_edges, want.matched_edges)
    assert ei.value.report.deactivated_per_round == want.per_round_deactivated
