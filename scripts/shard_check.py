import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2602_22976_b200 as hb
from paper_2602_22976_b200 import multi_gpu as mg
fam, spec = sys.argv[1], dict(n=int(sys.argv[2]), m=int(sys.argv[3]), d=int(sys.argv[4]), seed=1, int_weights=False)
worlds = [int(x) for x in sys.argv[5].split(",")]
full = hb.DeviceHypergraph.generate(fam, **spec)
for ws in (hb.WeightStream(), hb.WeightStream(noise_high=0.0)):
    ref = full.match(ws, hb.ParallelConfig(variant="crew"))
    print("single crew", ref.report.rounds, len(ref.matching.matched_edges), ref.report.matched_per_round_count, ref.report.deactivated_per_round)
    for w in worlds:
        shards = mg.generate_shards(fam, w, **spec)
        # "nonccl" as 6th argument: co-located exchange only (racecheck cannot follow NCCL's kernels)
        for comm in ((None,) if len(sys.argv) > 6 and sys.argv[6] == "nonccl" else (None, mg.Communicator.create(None, 0, 1, 0))):
            for tie in ("auto", "exact"):
                t0 = time.time()
                res, rep = mg.match_sharded(shards, ws, hb.ParallelConfig(tie_mode=tie), comm)
                ok = (np.array_equal(res.matching.matched_edges, ref.matching.matched_edges) and res.report.rounds == ref.report.rounds
                      and res.report.matched_per_round_count == ref.report.matched_per_round_count
                      and res.report.deactivated_per_round == ref.report.deactivated_per_round
                      and res.matching.total_weight == ref.matching.total_weight)
                print(f"world {w} nccl {comm is not None} ties {tie}: ok={ok} rounds {rep['rounds']} redo {rep['tie_redo_rounds']} syncs {rep['host_syncs']} "
                      f"live {rep['live_vertices_per_round']} bytes {rep['collective_bytes_per_round']} nccl_calls {rep['nccl_calls']} {1e3*(time.time()-t0):.1f} ms")
                assert ok
