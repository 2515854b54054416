"""One small CREW matching checked against CRCW (sanitizer target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2602_22976_b200 as hb
for spec in (dict(family="uniform", n=20000, m=40000, d=8, seed=3), dict(family="powerlaw", n=30000, m=60000, seed=2),
             dict(family="rmat", scale=12, m=1 << 16, seed=1, int_weights=True)):
    dg = hb.DeviceHypergraph.generate(**spec)
    print("generated", spec["family"], flush=True)
    a = dg.match(hb.WeightStream(), hb.ParallelConfig(variant=os.environ.get("FIRST_VARIANT", "crcw"), loop_mode=os.environ.get("LOOP", "auto")))
    print("first done", flush=True)
    b = dg.match(hb.WeightStream(), hb.ParallelConfig(variant="crew"))
    same = np.array_equal(np.asarray(a.matching.matched_edges), np.asarray(b.matching.matched_edges))
    print(spec["family"], "rounds", a.report.rounds, b.report.rounds, "same" if same else "DIFFERENT", flush=True)
    assert same and a.report.rounds == b.report.rounds
    dg.release()
