"""Per-round kernel times of variant auto on the shard shape / config 3 (host loop, CUDA events), hand-over included."""
import os, sys, time
sys.path.insert(0, ".")
import paper_2602_22976_b200 as hb
which = sys.argv[1] if len(sys.argv) > 1 else "u8"
spec = {"u8": ("uniform", dict(n=125_000_000, m=250_000_000, d=8, seed=1)),
        "c3": ("powerlaw", dict(n=50_000_000, m=100_000_000, seed=1)),
        "c4": ("netlist", dict(n=10_000_000, m=20_000_000, seed=1, int_weights=True))}[which]
dg = hb.DeviceHypergraph.generate(spec[0], **spec[1])
ws = hb.WeightStream()
for _ in range(2):
    r = dg.match(ws, hb.ParallelConfig(variant="auto"))
print(f"auto graph: device {r.report.device_ms:.2f} ms engine {r.report.engine}")
os.environ["HLM_B200_CREW_TIMES"] = "1"
os.environ["HLM_B200_TRACE"] = "1"
r = dg.match(ws, hb.ParallelConfig(variant="auto", loop_mode="host", kernel_times=True))
print(f"auto host loop: device {r.report.device_ms:.2f} ms rounds {r.report.rounds}")
print("sweep ms", [round(x, 3) for x in (r.report.round_filter_ms or [])])
print("check ms", [round(x, 3) for x in (r.report.round_check_ms or [])])
print("matched", r.report.matched_per_round_count)
print("deact", r.report.deactivated_per_round)
