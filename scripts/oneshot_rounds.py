import sys; sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2602_22976_b200 as hb
dg = hb.DeviceHypergraph.generate("rmat", scale=24, m=1 << 28, seed=1, int_weights=True)
host = dg.download(pinned=True)
dg.release()
for _ in range(3):
    r = hb.run_variant(host, hb.WeightStream(), hb.ParallelConfig(kernel_times=True))
print("device ms", r.report.device_ms)
print("filter", np.round(np.array(r.report.round_filter_ms), 3).tolist(), "sum", float(np.sum(r.report.round_filter_ms)))
print("check ", np.round(np.array(r.report.round_check_ms), 3).tolist(), "sum", float(np.sum(r.report.round_check_ms)))
