"""One-shot call on a config-1-size instance (uniform d=4, n=1M, m=1M): where do the fixed costs go?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2602_22976_b200 as hb
dg = hb.DeviceHypergraph.generate("uniform", n=1_000_000, m=1_000_000, d=4, seed=1)
host = dg.download(pinned=False)
dg.release()
for loop in ("auto", "host"):
    for rep in range(6):
        if rep == 5:
            os.environ["HLM_B200_TRACE"] = "1"
        else:
            os.environ.pop("HLM_B200_TRACE", None)
        t0 = time.perf_counter()
        r = hb.run_variant(host, hb.WeightStream(), hb.ParallelConfig(loop_mode=loop))
        print("loop=%s e2e %.3f ms  device %.3f ms  wall(match) %.3f rounds %d" % (loop, (time.perf_counter() - t0) * 1e3, r.report.device_ms, r.report.wall_time_ms, r.report.rounds), flush=True)
