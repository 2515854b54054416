"""ncu target: one CREW matching of a named case (scripts/crew_perf.py CASES); profile with
ncu -k regex:k_c2_ ... python scripts/crew_ncu_target.py u8s"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_22976_b200 as hb
from crew_perf import CASES  # noqa
name = sys.argv[1] if len(sys.argv) > 1 else "u8s"
dg = hb.DeviceHypergraph.generate(**CASES[name])
r = dg.match(hb.WeightStream(), hb.ParallelConfig(variant="crew"))
print(name, "device ms", r.report.device_ms, "rounds", r.report.rounds)
