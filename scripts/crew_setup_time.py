"""Cost of the first CREW / auto matching on a resident instance (builds the incidence side and the
CREW work arrays) against the following ones."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_22976_b200 as hb
from crew_perf import CASES  # noqa
for name in sys.argv[1:] or ["c3", "u8", "c4"]:
    dg = hb.DeviceHypergraph.generate(**CASES[name])
    dg.match(hb.WeightStream(), hb.ParallelConfig(variant="crcw"))
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        r = dg.match(hb.WeightStream(), hb.ParallelConfig(variant="crew"))
        ts.append((time.perf_counter() - t0) * 1e3)
    print(name, "first crew call %.1f ms, then %.1f / %.1f ms (device %.1f ms)" % (ts[0], ts[1], ts[2], r.report.device_ms), flush=True)
    dg.release()
