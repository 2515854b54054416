"""Per-round kernel times of the compacting CREW variant (HLM_B200_CREW_TIMES=1 prints them on stderr)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_22976_b200 as hb
from crew_perf import CASES  # noqa
name = sys.argv[1] if len(sys.argv) > 1 else "u8"
dg = hb.DeviceHypergraph.generate(**CASES[name])
dg.match(hb.WeightStream(), hb.ParallelConfig(variant="crew"))
os.environ["HLM_B200_CREW_TIMES"] = "1"
r = dg.match(hb.WeightStream(), hb.ParallelConfig(variant="crew"))
print(name, "device ms", r.report.device_ms, "rounds", r.report.rounds)
