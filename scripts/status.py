"""Round status table: every BASELINE config shape on one B200 (resident instance, CUDA-graph loop,
best of 6), verified on the device (disjoint + maximal).  Output goes to profiles/status_*.txt."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_22976_b200 as hb  # noqa: E402

CASES = [
    ("c1-shape uniform d=4 n=1M m=1M", dict(family="uniform", n=1_000_000, m=1_000_000, d=4, seed=1), ("crcw", "crew", "auto")),
    ("c2 RMAT scale 24, 2^28 edges, w 1-100", dict(family="rmat", scale=24, m=1 << 28, seed=1, int_weights=True), ("crcw", "crew", "auto")),
    ("c2/16 RMAT scale 20, 2^24 edges", dict(family="rmat", scale=20, m=1 << 24, seed=1, int_weights=True), ("crcw", "crew", "auto")),
    ("c3 power-law n=50M m=100M sizes 2-64", dict(family="powerlaw", n=50_000_000, m=100_000_000, seed=1), ("crcw", "crew", "auto")),
    ("c3/10 power-law n=5M m=10M", dict(family="powerlaw", n=5_000_000, m=10_000_000, seed=1), ("crcw", "crew", "auto")),
    ("c4 netlist n=10M m=20M sizes <= 4096, w 1-100", dict(family="netlist", n=10_000_000, m=20_000_000, seed=1, int_weights=True), ("crcw", "crew", "auto")),
    ("c5 shard shape: 8-uniform n=125M m=250M", dict(family="uniform", n=125_000_000, m=250_000_000, d=8, seed=1), ("crcw", "crew", "auto")),
]

print(f"{'workload':48s} {'variant':5s} {'pins':>12s} {'rounds':>6s} {'|M|':>10s} {'device ms':>10s} {'G pins/s':>9s} {'ties':>4s} verify")
for name, spec, variants in CASES:
    t0 = time.time()
    dg = hb.DeviceHypergraph.generate(**spec)
    info = dg.info()
    for variant in variants:
        best = None
        for _ in range(6):
            r = dg.match(hb.WeightStream(), hb.ParallelConfig(variant=variant, loop_mode="graph"))
            if best is None or r.report.device_ms < best.report.device_ms:
                best = r
        v = dg.verify(best.matching.matched_edges)
        print(f"{name:48s} {variant:5s} {info.num_pins:12d} {best.report.rounds:6d} {len(best.matching.matched_edges):10d} "
              f"{best.report.device_ms:10.3f} {info.num_pins / best.report.device_ms / 1e6:9.2f} {best.report.tie_redo_rounds:4d} "
              f"{'ok' if v.valid() else 'FAILED'}", flush=True)
    dg.release()
