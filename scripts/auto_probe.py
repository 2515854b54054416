import sys; sys.path.insert(0, "/root/repo")
import paper_2602_22976_b200 as hb
for name, spec in (("u4 n=32M m=64M d=4", dict(family="uniform", n=32_000_000, m=64_000_000, d=4, seed=1)),
                   ("u4b n=24M m=96M d=4", dict(family="uniform", n=24_000_000, m=96_000_000, d=4, seed=1)),
                   ("rmat22 2^26 edges", dict(family="rmat", scale=22, m=1 << 26, seed=1, int_weights=True)),
                   ("c2", dict(family="rmat", scale=24, m=1 << 28, seed=1, int_weights=True))):
    dg = hb.DeviceHypergraph.generate(**spec)
    for v in ("crcw", "crew", "auto"):
        best = min(dg.match(hb.WeightStream(), hb.ParallelConfig(variant=v, loop_mode="graph")).report.device_ms for _ in range(4))
        print(name, v, round(best, 3), flush=True)
    dg.release()
