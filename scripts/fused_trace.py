"""Phase times inside k_rounds_fused (analysis build: HLM_NVCC_EXTRA=-DHLM_FUSED_TRACE, HLM_B200_TRACE=1)."""
import os, sys
sys.path.insert(0, ".")
import paper_2602_22976_b200 as hb
ws = hb.WeightStream()
for (n, m, d) in (((1_000_000, 1_000_000, 4),) if len(sys.argv) > 1 else ((1000, 1000, 4), (1_000_000, 1_000_000, 4))):
    host = hb.generate_random(n, m, d, d, 1)
    dg = hb.DeviceHypergraph.upload(host)
    cfg = hb.ParallelConfig(variant="crcw", loop_mode="graph")
    os.environ.pop("HLM_B200_TRACE", None)
    for _ in range(5):
        try: dg.match(ws, cfg)
        except Exception: pass
    print(f"-- n={n} m={m} d={d}", file=sys.stderr, flush=True)
    os.environ["HLM_B200_TRACE"] = "1"
    try: r = dg.match(ws, cfg)
    except Exception as ex:
        print("failed", type(ex).__name__, file=sys.stderr); continue
    os.environ.pop("HLM_B200_TRACE", None)
    print(f"device {r.report.device_ms:.3f} ms rounds {r.report.rounds}", file=sys.stderr, flush=True)
    dg.release()
