"""Run by tests/test_gpu_multi.py under torchrun with 2 ranks (needs 2 GPUs): every rank holds one
edge shard, the library's round driver joins them over NCCL, and the concatenated slices must equal
the oracle's matching of the whole instance."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2602_22976_b200 as hb  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from paper_2602_22976_b200 import multi_gpu  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = multi_gpu.Communicator.from_torch(dist, local)
    port = po.Oracle("port")
    kw = dict(n=20000, m=60000, d=4)
    g = port.syn_generate(po.SYN_UNIFORM, seed=8, int_weights=True, **kw)
    for s, hs in ((po.Stream(seed=4), hb.WeightStream(seed=4)),
                  (po.Stream(seed=4, noise_high=0.0), hb.WeightStream(seed=4, noise_high=0.0))):
        want = port.local_max(g, s)
        b, k = multi_gpu.shard_bounds(kw["m"], world, rank)
        shard = hb.DeviceHypergraph.generate("uniform", seed=8, int_weights=True, edge_begin=b, m_local=k, device=local, **kw)
        got, rep = multi_gpu.match_sharded([shard], hs, hb.ParallelConfig(), comm)
        mine = want.matched_edges[(want.matched_edges >= b) & (want.matched_edges < b + k)]
        assert np.array_equal(got.matching.matched_edges, mine), "slice differs"
        assert got.report.rounds == want.rounds
        assert got.report.matched_per_round_count == want.per_round_matched
        assert got.report.deactivated_per_round == want.per_round_deactivated
        assert got.matching.total_weight == want.total_weight
        assert rep["num_processes"] == world
        shard.release()
    dist.barrier()
    if rank == 0:
        print("two-rank parity: ok")
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
