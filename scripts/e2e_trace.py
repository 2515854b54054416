"""Phase times of the one-shot drop-in call on config 2 (HLM_B200_TRACE=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_22976_b200 as hb
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
dg = hb.DeviceHypergraph.generate("rmat", scale=scale, m=1 << (scale + 4), seed=1, int_weights=True)
host = dg.download(pinned=True)
dg.release()
for rep in range(3):
    os.environ["HLM_B200_TRACE"] = "1" if rep == 2 else ""
    if rep != 2:
        os.environ.pop("HLM_B200_TRACE", None)
    t0 = time.perf_counter()
    r = hb.run_variant(host, hb.WeightStream())
    print("e2e %.2f ms  device %.2f ms  rounds %d" % ((time.perf_counter() - t0) * 1e3, r.report.device_ms, r.report.rounds), flush=True)
