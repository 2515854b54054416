"""CPU tests (gloo, world_size 2) of the multi-rank path: the round protocol of csrc/hlm_shard.inc restated
in numpy (tests/shard_model.py) with its collectives carried by torch.distributed, the plumbing of
paper_2602_22976_b200/multi_gpu.py that runs on every rank (edge blocks, the 128-byte communicator id
travelling from rank 0), the ordered weight fold and the result assembly.  The CUDA kernels and the C++
round driver run in tests/test_gpu_multi.py."""
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
    if kind == "zero_noise":
        g = orc.generate_random(300, 800, 2, 4, 9)
        return g, po.Stream(seed=3, noise_high=0.0)
    g = orc.generate_random(400, 600, 2, 3, 8)
    g.base_weights = np.random.default_rng(1).random(g.m) * 9 + 0.5  # non-integer: ordered weight fold matters
    return g, po.Stream(seed=2)


def _worker(rank, world, port, kind, max_rounds, exact, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_22976_b200 import multi_gpu
        from tests.shard_model import ShardModel

        def allreduce(op):
            def f(a):
                t = torch.from_numpy(np.ascontiguousarray(a))
                dist.all_reduce(t, op=op)
                return t.numpy()
            return f

        # the communicator id: made by rank 0, identical on every rank afterwards
        uid = multi_gpu.Communicator.exchange_unique_id(dist, lambda: bytes(range(128)))
        assert uid == bytes(range(128))
        g, s = _instance(kind)
        b, k = multi_gpu.shard_bounds(g.m, world, rank)
        res = ShardModel(g, b, k, s, allreduce(dist.ReduceOp.MAX), allreduce(dist.ReduceOp.SUM), max_rounds, exact).run()
        # ordered weight fold: rank q continues the sum of the ranks below it (local_max_seq.hpp:79)
        acc = torch.zeros(1, dtype=torch.float64)
        for q in range(world):
            if rank == q:
                tw = float(acc.item())
                for w in res["weights"]:
                    tw += float(w)
                acc[0] = tw
            dist.broadcast(acc, src=q)
        # the slices of all ranks in rank order
        parts = [None] * world
        dist.all_gather_object(parts, (res["matched"], res["round_of"]))
        matched = np.concatenate([p[0] for p in parts])
        round_of = np.concatenate([p[1] for p in parts])
        out.put((rank, ("limit" if res["limit"] else "ok", matched, round_of, res["per_round_matched"],
                        res["per_round_deactivated"], float(acc.item()), res["rounds"], res["live"], res["bytes"],
                        res["tie_redos"])))
    finally:
        dist.destroy_process_group()


def _run(kind, world=2, max_rounds=0, exact=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, max_rounds, exact, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


@pytest.mark.parametrize("kind,exact", [("hyper", False), ("ties", False), ("zero_noise", False), ("real_weights", False),
                                        ("hyper", True)])
def test_two_ranks_reproduce_the_oracle(kind, exact):
    g, s = _instance(kind)
    want = po.Oracle("port").local_max(g, s)
    results = _run(kind, exact=exact)
    for rank, (tag, matched, round_of, prm, prd, weight, rounds, live, moved, redos) in results.items():
        assert tag == "ok"
        assert np.array_equal(matched, want.matched_edges), (kind, rank)
        assert np.array_equal(round_of.astype(np.uint32), want.matched_round)
        assert prm == want.per_round_matched and prd == want.per_round_deactivated
        assert rounds == want.rounds
        assert weight == want.total_weight  # bit-exact: folded across ranks in id order
        assert live[0] == g.n and live == sorted(live, reverse=True)  # the exchange shrinks with the live set
        if kind in ("ties", "zero_noise"):
            assert redos >= 1
        if kind == "hyper" and not exact:
            assert redos == 0 and moved == sorted(moved, reverse=True)


def test_round_cap_across_ranks():
    g, s = _instance("hyper")
    want = po.Oracle("port").local_max(g, s, max_rounds=2)
    assert want.status == po.ROUND_LIMIT
    for rank, (tag, matched, _, prm, prd, _, rounds, _, _, _) in _run("hyper", max_rounds=2).items():
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
