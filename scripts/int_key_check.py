"""KM 4 (integer noise compare) against the FP key: same matchings; forced fallbacks (huge delta) too."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2602_22976_b200 as hb
spec = dict(family="uniform", n=2_000_000, m=4_000_000, d=8, seed=3)
dg = hb.DeviceHypergraph.generate(**spec)
for ws in (hb.WeightStream(seed=5), hb.WeightStream(seed=5, noise_low=3.0, noise_high=3.5), hb.WeightStream(seed=9, noise_high=1e-3)):
    os.environ["HLM_B200_CREW_INT_KEY"] = "0"
    ref = dg.match(ws, hb.ParallelConfig(variant="crew"))
    for val in ("1", "4503599627370496", "1000000000000"):
        os.environ["HLM_B200_CREW_INT_KEY"] = val
        got = dg.match(ws, hb.ParallelConfig(variant="crew"))
        ok = np.array_equal(got.matching.matched_edges, ref.matching.matched_edges) and got.report.matched_per_round_count == ref.report.matched_per_round_count
        print(ws, "int_key", val, "ok" if ok else "MISMATCH", got.report.rounds, got.report.device_ms)
        assert ok
crcw = dg.match(hb.WeightStream(seed=5), hb.ParallelConfig(variant="crcw"))
os.environ["HLM_B200_CREW_INT_KEY"] = "1"
got = dg.match(hb.WeightStream(seed=5), hb.ParallelConfig(variant="crew"))
assert np.array_equal(got.matching.matched_edges, crcw.matching.matched_edges)
print("crcw == crew(int)")
