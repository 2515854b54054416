"""Run by tests/test_gpu_multi.py under torchrun with 2 or 3 ranks ON ONE GPU: every process holds one edge
shard and the library's multi-rank round driver (hlm_b200_match_sharded, nranks > 1: global edge count, key /
bitmap / counter all-reduces, tie redo decided on reduced data, the rank-by-rank weight chain) joins them
through tests/cpp/shm_nccl.cpp, a stand-in for libnccl.so.2 over shared memory (NCCL itself refuses two ranks
on one device).  The concatenated slices must equal the oracle's matching of the whole instance."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2602_22976_b200 as hb  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from paper_2602_22976_b200 import multi_gpu  # noqa: E402
from tests.util import to_hb_graph, to_hb_stream  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    assert os.environ.get("HLM_B200_NCCL_LIB", "").endswith("libshm_nccl.so")
    dist.init_process_group("gloo")  # carries the 128-byte id only
    comm = multi_gpu.Communicator.from_torch(dist, 0)
    assert comm.nccl_version() == 99999  # the stand-in, not NCCL
    port = po.Oracle("port")
    real = port.syn_generate(po.SYN_POWERLAW, n=9000, m=15000, seed=5)
    real.base_weights[:] = 0.25 + np.random.default_rng(3).random(real.m) * 7.5  # the ordered FP64 sum crosses ranks
    cases = [("uniform, weights 1-100", port.syn_generate(po.SYN_UNIFORM, n=20000, m=60000, d=4, seed=8, int_weights=True)),
             ("power-law 2..64, real weights", real),
             ("netlist <= 4096", port.syn_generate(po.SYN_NETLIST, n=9000, m=12000, seed=6, int_weights=True)),
             ("five edges", port.generate_random(50, 5, 2, 3, 1))]
    streams = [po.Stream(seed=4), po.Stream(seed=4, noise_high=0.0),  # every weight class ties, on every rank
               po.Stream(seed=2, mode=po.MODE_REPLACE_UNIFORM)]
    for name, g in cases:
        b, k = multi_gpu.shard_bounds(g.m, world, rank)
        shards = multi_gpu.upload_shards(to_hb_graph(g), world, 0, only_rank=rank)
        for s in streams:
            for ties in ("auto", "exact"):
                want = port.local_max(g, s)
                if os.environ.get("HLM_TEST_VERBOSE"):
                    print(f"[{rank}] {name} {s} ties={ties}: want rounds {want.rounds} matched {want.per_round_matched} deact {want.per_round_deactivated}", flush=True)
                got, rep = multi_gpu.match_sharded(shards, to_hb_stream(s), hb.ParallelConfig(tie_mode=ties), comm)
                mine = want.matched_edges[(want.matched_edges >= b) & (want.matched_edges < b + k)]
                what = f"{name} {s} ties={ties} rank {rank}/{world}"
                assert np.array_equal(got.matching.matched_edges, mine), what + ": slice differs"
                assert got.report.rounds == want.rounds, what
                assert got.report.matched_per_round_count == want.per_round_matched, what
                assert got.report.deactivated_per_round == want.per_round_deactivated, what
                assert got.matching.total_weight == want.total_weight, what + f": {got.matching.total_weight} != {want.total_weight}"
                assert rep["num_processes"] == world and rep["nccl_calls"] > 0
        # the round cap, hit on every rank in the same round
        s = po.Stream(seed=4)
        capped = port.local_max(g, s, max_rounds=2)
        if capped.status == po.ROUND_LIMIT:
            try:
                multi_gpu.match_sharded(shards, to_hb_stream(s), hb.ParallelConfig(max_rounds=2), comm)
                raise AssertionError("no round-limit error")
            except hb.RoundLimitError as ex:
                mine = capped.matched_edges[(capped.matched_edges >= b) & (capped.matched_edges < b + k)]
                assert list(ex.partial.matched_edges) == list(mine)
        for sh in shards:
            sh.release()
    dist.barrier()
    if rank == 0:
        print(f"multi-rank parity over shared memory, {world} ranks: ok")
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
