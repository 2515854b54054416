"""Config 2: per-round sweep / check times (host loop, CUDA events, best of 3) and the graph-loop time."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2602_22976_b200 as hb
dg = hb.DeviceHypergraph.generate("rmat", scale=24, m=1 << 28, seed=1, int_weights=True)
ws = hb.WeightStream()
f = c = None
for _ in range(3):
    r = dg.match(ws, hb.ParallelConfig(variant="crcw", loop_mode="host", kernel_times=True))
    a, b = np.array(r.report.round_filter_ms), np.array(r.report.round_check_ms)
    f = a if f is None else np.minimum(f, a); c = b if c is None else np.minimum(c, b)
print("sweep", [round(float(x), 3) for x in f], "sum", round(float(f.sum()), 3))
print("check", [round(float(x), 3) for x in c], "sum", round(float(c.sum()), 3))
ds = []
for _ in range(10):
    ds.append(dg.match(ws, hb.ParallelConfig(variant="crcw")).report.device_ms)
print("graph loop device ms: best", round(min(ds), 3), "median", round(sorted(ds)[5], 3))
