"""Where the time of a small matching goes: per-round kernel times (host loop, CUDA events) against the
device time of the whole call, for config 1 and for a nearly empty instance (the fixed cost)."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2602_22976_b200 as hb
ws = hb.WeightStream()
for (n, m, d) in ((1000, 1000, 4), (1_000_000, 1_000_000, 4)):
    host = hb.generate_random(n, m, d, d, 1)
    dg = hb.DeviceHypergraph.upload(host)
    for variant in ("crcw", "crew"):
        cfg = hb.ParallelConfig(variant=variant, loop_mode="host", kernel_times=True)
        for _ in range(3):
            r = dg.match(ws, cfg)
        f, c = r.report.round_filter_ms, r.report.round_check_ms
        print(f"m={m} {variant} host loop: device {r.report.device_ms:.3f} ms; sweep {[round(x*1e3) for x in f]} us; check {[round(x*1e3) for x in c]} us; sum {sum(f)+sum(c):.3f} ms")
        cfg = hb.ParallelConfig(variant=variant, loop_mode="graph")
        for _ in range(5):
            r = dg.match(ws, cfg)
        ds, wl = [], []
        for _ in range(30):
            t = time.perf_counter()
            r = dg.match(ws, cfg)
            wl.append((time.perf_counter() - t) * 1e3)
            ds.append(r.report.device_ms)
        print(f"m={m} {variant} graph: device best {min(ds):.3f} med {sorted(ds)[15]:.3f}; wall best {min(wl):.3f} ms; launches {r.report.kernel_launches}", flush=True)
    dg.release()
