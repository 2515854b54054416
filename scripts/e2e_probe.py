import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_22976_b200 as hb
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
dg = hb.DeviceHypergraph.generate("rmat", scale=scale, m=1 << (scale + 4), seed=1, int_weights=True)
for pinned in (True, False):
    host = dg.download(pinned=pinned)
    nbytes = host.edge_offsets.nbytes + host.edge_members.nbytes + host.base_weights.nbytes
    for rep in range(2):
        t0 = time.perf_counter(); g2 = hb.DeviceHypergraph.upload(host); t1 = time.perf_counter()
        r = g2.match(hb.WeightStream()); t2 = time.perf_counter()
        r = g2.match(hb.WeightStream()); t3 = time.perf_counter()
        g2.release(); t4 = time.perf_counter()
        print(f"pinned={pinned} upload {1e3*(t1-t0):.1f} ms ({nbytes/(t1-t0)/1e9:.1f} GB/s)  first match {1e3*(t2-t1):.1f}  second match {1e3*(t3-t2):.1f} (device {r.report.device_ms:.1f})  release {1e3*(t4-t3):.1f}")
    # raw torch copy for reference
    t = torch.from_numpy(host.edge_members.view(np.int32))
    torch.cuda.synchronize(); t0 = time.perf_counter(); d = t.cuda(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"  torch H2D of pins: {t.numel()*4/(t1-t0)/1e9:.1f} GB/s")
    del host
