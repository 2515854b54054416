"""Config 1: variant auto forced onto either engine (HLM_B200_AUTO), device ms."""
import os, sys
sys.path.insert(0, ".")
import paper_2602_22976_b200 as hb
host = hb.generate_random(1_000_000, 1_000_000, 4, 4, 1)
for forced in ("crcw", "crew"):
    os.environ["HLM_B200_AUTO"] = forced
    dg = hb.DeviceHypergraph.upload(host)
    best = 1e9
    for _ in range(30):
        r = dg.match(hb.WeightStream(), hb.ParallelConfig(variant="auto", loop_mode="graph"))
        best = min(best, r.report.device_ms)
    print(forced, r.report.engine, "device ms %.3f" % best, "rounds", r.report.rounds, "launches", r.report.kernel_launches)
    dg.release()
