"""Fused all-rounds kernel (k_rounds_fused) against the CUDA-graph loop on small uniform instances:
same matching / per-round report, device time of both."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2602_22976_b200 as hb

def run(dg, ws, fused, variant="crcw"):
    os.environ["HLM_B200_FUSED_MAX_PINS"] = str(1 << 40) if fused else "0"
    cfg = hb.ParallelConfig(variant=variant, loop_mode="graph")
    for _ in range(5):
        r = dg.match(ws, cfg)
    ds = []
    for _ in range(30):
        r = dg.match(ws, cfg)
        ds.append(r.report.device_ms)
    return r, min(ds), sorted(ds)[15]

ws = hb.WeightStream()
if len(sys.argv) > 1 and sys.argv[1] == "ragged":
    for (n, m, lo, hi) in ((3000, 5000, 2, 5), (200_000, 300_000, 2, 5), (1_000_000, 1_000_000, 2, 8), (500_000, 1_000_000, 1, 30),
                           (2_000_000, 2_000_000, 3, 5)):
        dg = hb.DeviceHypergraph.upload(hb.generate_random(n, m, lo, hi, 1))
        a, ta, _ = run(dg, ws, False)
        b, tb, _ = run(dg, ws, True)
        c, tc, _ = run(dg, ws, True, "crew")
        same = (np.array_equal(a.matching.matched_edges, b.matching.matched_edges)
                and a.report.matched_per_round_count == b.report.matched_per_round_count
                and a.report.deactivated_per_round == b.report.deactivated_per_round
                and a.report.work.total_pin_visits == b.report.work.total_pin_visits)
        print(f"ragged n={n} m={m} sizes {lo}..{hi}: pins {dg.info().num_pins} same={same} graph {ta:.3f} fused {tb:.3f} vertex-owned {tc:.3f} ms launches {a.report.kernel_launches}/{b.report.kernel_launches}", flush=True)
        dg.release()
    for fam, spec in (("powerlaw", dict(n=30_000, m=60_000, seed=1)), ("powerlaw", dict(n=500_000, m=1_000_000, seed=1)),
                      ("netlist", dict(n=50_000, m=100_000, seed=1, int_weights=True)), ("netlist", dict(n=500_000, m=1_000_000, seed=1, int_weights=True)),
                      ("netlist", dict(n=900_000, m=1_800_000, seed=1, int_weights=True))):
        os.environ["HLM_B200_REORDER"] = "0"
        dg = hb.DeviceHypergraph.generate(fam, **spec)
        a, ta, _ = run(dg, ws, False)
        b, tb, _ = run(dg, ws, True)
        c, tc, _ = run(dg, ws, True, "crew")
        same = (np.array_equal(a.matching.matched_edges, b.matching.matched_edges) and np.array_equal(c.matching.matched_edges, b.matching.matched_edges)
                and a.report.matched_per_round_count == b.report.matched_per_round_count
                and a.report.deactivated_per_round == b.report.deactivated_per_round
                and a.report.work.total_pin_visits == b.report.work.total_pin_visits)
        print(f"ragged {fam} {spec}: pins {dg.info().num_pins} same={same} graph {ta:.3f} fused {tb:.3f} vertex-owned {tc:.3f} ms launches {a.report.kernel_launches}/{b.report.kernel_launches}", flush=True)
        dg.release()
    sys.exit(0)
for (n, m, d) in ((1000, 1000, 4), (1_000_000, 1_000_000, 4), (100_000, 300_000, 2), (250_000, 250_000, 8), (2_000_000, 2_000_000, 4), (2_000_000, 8_000_000, 2), (500_000, 1_000_000, 8), (4_000_000, 4_000_000, 2)):
    host = hb.generate_random(n, m, d, d, 1)
    dg = hb.DeviceHypergraph.upload(host)
    b, tb, mb = run(dg, ws, True)
    if len(sys.argv) > 1:
        print(f"n={n} m={m} d={d}: rounds {b.report.rounds} fused {tb:.3f} (med {mb:.3f}) ms", flush=True)
        dg.release()
        continue
    a, ta, ma = run(dg, ws, False)
    same = (np.array_equal(a.matching.matched_edges, b.matching.matched_edges)
            and a.report.matched_per_round_count == b.report.matched_per_round_count
            and a.report.deactivated_per_round == b.report.deactivated_per_round
            and a.matching.total_weight == b.matching.total_weight)
    c, tc, mc = run(dg, ws, True, "crew")
    d_, td, md = run(dg, ws, True, "auto")
    print(f"     vertex-owned {tc:.3f} ms, auto {td:.3f} ms (engine {d_.report.engine})")
    print(f"n={n} m={m} d={d}: same={same} rounds {a.report.rounds}/{b.report.rounds} graph {ta:.3f} (med {ma:.3f}) fused {tb:.3f} (med {mb:.3f}) ms launches {a.report.kernel_launches}/{b.report.kernel_launches}", flush=True)
    dg.release()
