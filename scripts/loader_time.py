import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_22976_b200 as hb
for rep in range(3):
    t0 = time.perf_counter()
    dg = hb.DeviceHypergraph.generate("rmat", scale=24, m=1 << 28, seed=1, int_weights=True)
    t1 = time.perf_counter()
    dg.release()
    print("generate + loader passes: %.1f ms (HLM_B200_RENUMBER=%s HLM_B200_REORDER=%s)" % ((t1 - t0) * 1e3, os.environ.get("HLM_B200_RENUMBER"), os.environ.get("HLM_B200_REORDER")), flush=True)
