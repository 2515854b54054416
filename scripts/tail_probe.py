"""Per-round kernel times of variant auto (vertex-owned rounds, then the CRCW tail) on a named case."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import paper_2602_22976_b200 as hb
from crew_perf import CASES
name = sys.argv[1] if len(sys.argv) > 1 else "u8"
dg = hb.DeviceHypergraph.generate(**CASES[name])
cfg = hb.ParallelConfig(variant="auto", loop_mode="host", kernel_times=True)
for _ in range(2):
    r = dg.match(hb.WeightStream(), cfg)
print(name, r.report.engine, "device ms", round(r.report.device_ms, 2))
act = dg.info().num_edges
for q in range(r.report.rounds):
    print(f"round {q+1}: active {act:>10d} sweep {r.report.round_filter_ms[q]:.3f} rest {r.report.round_check_ms[q]:.3f}")
    act -= r.report.matched_per_round_count[q] + r.report.deactivated_per_round[q]
