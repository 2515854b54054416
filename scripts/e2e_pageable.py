"""e2e through hlm_b200_match_host from page-locked and from pageable arrays (config 2 by default)."""
import sys, time, os
sys.path.insert(0, ".")
import numpy as np
import paper_2602_22976_b200 as hb
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
dg = hb.DeviceHypergraph.generate("rmat", scale=scale, m=1 << (scale + 4), seed=1, int_weights=True)
ref = dg.match(hb.WeightStream(), hb.ParallelConfig(variant="auto"))
host = dg.download(pinned=True)
dg.release()
page = hb.Hypergraph(host.num_vertices, host.num_edges, None, None, np.array(host.edge_offsets), np.array(host.edge_members), np.array(host.base_weights))
for name, h in (("pinned", host), ("pageable", page), ("pageable", page)):
    ts = []
    for i in range(6):
        t = time.perf_counter()
        r = hb.run_variant(h, hb.WeightStream(), hb.ParallelConfig(variant="auto"))
        ts.append((time.perf_counter() - t) * 1e3)
    assert np.array_equal(r.matching.matched_edges, ref.matching.matched_edges)
    print(name, " ".join(f"{x:.1f}" for x in ts), "ms; h2d", r.report.h2d_bytes)
