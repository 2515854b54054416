"""Single-rank timing of the edge-partitioned driver: python scripts/shard_perf.py n m d [world] [nccl] [reps]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2602_22976_b200 as hb
from paper_2602_22976_b200 import multi_gpu as mg
n, m, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
world = int(sys.argv[4]) if len(sys.argv) > 4 else 1
nccl = len(sys.argv) > 5 and sys.argv[5] == "1"
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 4
# a shard of the instance with m * world edges: [0, m) of it, as rank 0 of `world` would hold
g = hb.DeviceHypergraph.generate("uniform", n=n, m=m * world, d=d, seed=1, edge_begin=0, m_local=m)
comm = mg.Communicator.create(None, 0, 1, 0) if nccl else None
ws = hb.WeightStream()
for i in range(reps):
    t0 = time.perf_counter()
    res, rep = mg.match_sharded([g], ws, hb.ParallelConfig(), comm)
    dt = (time.perf_counter() - t0) * 1e3
    print(f"rep {i}: {dt:.1f} ms wall, device {res.report.device_ms:.1f} ms, rounds {rep['rounds']} matched {len(res.matching.matched_edges)} "
          f"live {rep['live_vertices_per_round']} bytes/round {rep['collective_bytes_per_round']} launches {rep['kernel_launches']}", flush=True)
v = g.verify(res.matching.matched_edges)
print("verify", v)
