"""Config 1 (reference generate_random 4-uniform, n = m = 1M): per-variant time, graph vs host loop."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2602_22976_b200 as hb
host = hb.generate_random(1_000_000, 1_000_000, 4, 4, 1)
dg = hb.DeviceHypergraph.upload(host)
ws = hb.WeightStream()
for variant in ("crcw", "crew"):
    for loop in ("graph", "host"):
        cfg = hb.ParallelConfig(variant=variant, loop_mode=loop)
        for _ in range(5):
            r = dg.match(ws, cfg)
        ts, ds = [], []
        for _ in range(20):
            t = time.perf_counter()
            r = dg.match(ws, cfg)
            ts.append((time.perf_counter() - t) * 1e3)
            ds.append(r.report.device_ms)
        print(f"{variant:5s} {loop:5s} wall best {min(ts):.3f} median {sorted(ts)[10]:.3f} ms; device best {min(ds):.3f} ms; rounds {r.report.rounds} launches {r.report.kernel_launches}")
