"""First vertex-owned matching of a resident instance (incidence build etc.): phase trace on stderr."""
import os, sys, time
sys.path.insert(0, ".")
import paper_2602_22976_b200 as hb
which = sys.argv[1] if len(sys.argv) > 1 else "u8"
spec = {"u8": ("uniform", dict(n=125_000_000, m=250_000_000, d=8, seed=1)),
        "c3": ("powerlaw", dict(n=50_000_000, m=100_000_000, seed=1)),
        "c4": ("netlist", dict(n=10_000_000, m=20_000_000, seed=1, int_weights=True))}[which]
ws = hb.WeightStream()
if len(sys.argv) > 2:  # warm the memory pool first: same instance, matched and released
    dg = hb.DeviceHypergraph.generate(spec[0], **spec[1])
    dg.match(ws, hb.ParallelConfig(variant="crew"))
    dg.release()
    print("-- pool warm", file=sys.stderr)
dg = hb.DeviceHypergraph.generate(spec[0], **spec[1])
os.environ["HLM_B200_TRACE"] = "1"
t = time.perf_counter()
r = dg.match(ws, hb.ParallelConfig(variant="crew"))
print(f"first call wall {(time.perf_counter()-t)*1e3:.1f} ms device {r.report.device_ms:.2f}", file=sys.stderr)
t = time.perf_counter()
r = dg.match(ws, hb.ParallelConfig(variant="crew"))
print(f"second call wall {(time.perf_counter()-t)*1e3:.1f} ms device {r.report.device_ms:.2f}", file=sys.stderr)
