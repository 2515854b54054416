"""CPU tests (gloo, world_size 2) of the multi-rank protocol in paper_2602_22976_b200/multi_gpu.py:
sharding, the three all-reduces per round, the exact-tie levels, ordered weight fold, result
assembly.  The CUDA step engine is replaced by tests/fake_engine.py (numpy + oracle stream) because
there is no GPU here; the same protocol runs on real kernels in tests/test_gpu_multi.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pyoracle as po


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _instance(kind):
    orc = po.Oracle("port")
    if kind == "hyper":
        g = orc.generate_random(300, 700, 2, 5, 3)
        g.base_weights = orc.random_weights_1_100(g.m, 5)
        return g, po.Stream(seed=7)
    if kind == "ties":
        g = orc.syn_generate(po.SYN_UNIFORM, n=200, m=900, d=2, seed=6)
        return g, po.Stream(seed=5, kind=po.GEN_PARK_MILLER, noise_low=0.0, noise_high=2.0 ** -50)
    g = orc.generate_random(400, 600, 2, 3, 8)
    g.base_weights = np.random.default_rng(1).random(g.m) * 9 + 0.5  # non-integer: ordered weight fold matters
    return g, po.Stream(seed=2)


def _worker(rank, world, port, kind, max_rounds, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2602_22976_b200 as hb
        from paper_2602_22976_b200 import multi_gpu
        from tests.fake_engine import FakeEngine

        g, s = _instance(kind)
        b, k = multi_gpu.shard_bounds(g.m, world, rank)
        sm = multi_gpu.ShardedMatcher([FakeEngine(g, b, k)], g.m, g.kappa, multi_gpu.Collectives(dist))
        ws = hb.WeightStream(s.seed, {0: "xorshift", 1: "park_miller", 2: "splitmix"}[s.kind],
                             {0: "perturb_base", 1: "replace_uniform"}[s.mode], s.noise_low, s.noise_high)
        try:
            res = sm.match(ws, hb.ParallelConfig(max_rounds=max_rounds))
            payload = ("ok", res.matching.matched_edges, res.report.matched_round, res.report.matched_per_round_count,
                       res.report.deactivated_per_round, res.matching.total_weight, res.report.rounds)
        except hb.RoundLimitError as e:
            payload = ("limit", e.partial.matched_edges, e.report.matched_round, e.report.matched_per_round_count,
                       e.report.deactivated_per_round, e.partial.total_weight, e.report.rounds)
        out.put((rank, payload))
    finally:
        dist.destroy_process_group()


def _run(kind, world=2, max_rounds=0):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, max_rounds, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


@pytest.mark.parametrize("kind", ["hyper", "ties", "real_weights"])
def test_two_ranks_reproduce_the_oracle(kind):
    g, s = _instance(kind)
    want = po.Oracle("port").local_max(g, s)
    results = _run(kind)
    for rank, (tag, matched, round_of, prm, prd, weight, rounds) in results.items():
        assert tag == "ok"
        assert np.array_equal(matched, want.matched_edges), (kind, rank)
        assert np.array_equal(round_of.astype(np.uint32), want.matched_round)
        assert prm == want.per_round_matched and prd == want.per_round_deactivated
        assert rounds == want.rounds
        assert weight == want.total_weight  # bit-exact: folded across ranks in id order


def test_round_cap_across_ranks():
    g, s = _instance("hyper")
    want = po.Oracle("port").local_max(g, s, max_rounds=2)
    assert want.status == po.ROUND_LIMIT
    for rank, (tag, matched, _, prm, prd, _, rounds) in _run("hyper", max_rounds=2).items():
        assert tag == "limit" and rounds == 2
        assert np.array_equal(matched, want.matched_edges)
        assert prm == want.per_round_matched and prd == want.per_round_deactivated


def test_shard_bounds_cover_the_edge_range():
    from paper_2602_22976_b200 import multi_gpu

    for m in (0, 1, 7, 100, 2_000_000_000):
        for world in (1, 2, 3, 8):
            spans = [multi_gpu.shard_bounds(m, world, r) for r in range(world)]
            assert sum(k for _, k in spans) == m
            pos = 0
            for b, k in spans:
                assert b == pos or k == 0
                pos += k
