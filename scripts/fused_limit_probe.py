"""Where the one-launch kernel stops paying: graph loop vs fused (forced) vs vertex-owned on growing instances."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2602_22976_b200 as hb
ws = hb.WeightStream()
def best(dg, variant, fused):
    os.environ["HLM_B200_FUSED_MAX_PINS"] = str(1 << 40) if fused else "0"
    cfg = hb.ParallelConfig(variant=variant)
    for _ in range(3): dg.match(ws, cfg)
    return min(dg.match(ws, cfg).report.device_ms for _ in range(10))
cases = [("uniform", dict(n=10_000_000, m=10_000_000, d=4, seed=1)), ("uniform", dict(n=12_000_000, m=12_000_000, d=4, seed=1)),
         ("uniform", dict(n=14_000_000, m=14_000_000, d=4, seed=1)), ("uniform", dict(n=6_000_000, m=16_000_000, d=4, seed=1)),
         ("uniform", dict(n=12_000_000, m=24_000_000, d=2, seed=1)), ("uniform", dict(n=15_000_000, m=30_000_000, d=2, seed=1)),
         ("uniform", dict(n=8_000_000, m=32_000_000, d=2, seed=1)), ("rmat", dict(scale=21, m=1 << 25, seed=1, int_weights=True)),
         ("rmat", dict(scale=23, m=1 << 25, seed=1, int_weights=True))]
if len(sys.argv) > 1:
    cases = eval(sys.argv[1])
for fam, spec in cases:
    dg = hb.DeviceHypergraph.generate(fam, **spec)
    info = dg.info()
    g, f, c = best(dg, "crcw", False), best(dg, "crcw", True), best(dg, "crew", True)
    print(f"{fam} {spec}: pins {info.num_pins/1e6:.0f} M  graph {g:.3f}  fused {f:.3f}  vertex-owned {c:.3f} ms", flush=True)
    dg.release()
