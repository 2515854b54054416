"""Quick on-GPU probe: timings of the matching on the BASELINE configs (not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2602_22976_b200 as hb
from oracle import pyoracle as po

def run(name, g, stream=hb.WeightStream(), reps=5, **cfg):
    if PROF:
        reps = 1
        cfg["loop_mode"] = "host"
    info = g.info()
    best = None
    for i in range(reps):
        r = g.match(stream, hb.ParallelConfig(**cfg))
        if best is None or r.report.device_ms < best.report.device_ms:
            best = r
    rep = best.report
    print(f"{name} {cfg}: n={info.num_vertices} m={info.num_edges} pins={info.num_pins} d={info.uniform_size} "
          f"rounds={rep.rounds} |M|={len(best.matching.matched_edges)} device_ms={rep.device_ms:.3f} wall_ms={rep.wall_time_ms:.3f} "
          f"Gpins/s={info.num_pins/rep.device_ms/1e6:.2f} launches={rep.kernel_launches} graphs={rep.graph_launches} ties={rep.tie_redo_rounds} "
          f"swept={rep.device_edge_visits}", flush=True)
    return best

which = sys.argv[1:] or ["c1", "c2s", "c2"]
PROF = os.environ.get("HLM_PROF") == "1"
orc = po.Oracle("port")
if "c1" in which:
    g = orc.generate_random(1000000, 1000000, 4, 4, 1)
    dg = hb.DeviceHypergraph.upload(hb.Hypergraph(g.n, g.m, None, None, g.edge_offsets, g.edge_members, g.base_weights))
    run("C1", dg, loop_mode="host")
    r = run("C1", dg, loop_mode="graph")
    print(r.report.matched_per_round_count, hex(po.fnv1a_ids(r.matching.matched_edges)))
    run("C1 zero-noise", dg, stream=hb.WeightStream(noise_high=0.0), loop_mode="graph")
    run("C1 exact", dg, tie_mode="exact")
    dg.release()
if "c2s" in which:
    t = time.time(); dg = hb.DeviceHypergraph.generate("rmat", scale=20, m=1 << 24, seed=1, int_weights=True); print("gen", time.time() - t)
    run("RMAT20", dg, loop_mode="graph")
    dg.release()
if "c2" in which:
    t = time.time(); dg = hb.DeviceHypergraph.generate("rmat", scale=24, m=1 << 28, seed=1, int_weights=True); print("gen", time.time() - t)
    run("C2", dg, loop_mode="host", reps=3)
    r = run("C2", dg, loop_mode="graph", reps=3)
    print(r.report.matched_per_round_count, r.report.deactivated_per_round)
    v = dg.verify(r.matching.matched_edges); print("verify", v)
    dg.release()
if "c3" in which:
    t = time.time(); dg = hb.DeviceHypergraph.generate("powerlaw", n=50_000_000, m=100_000_000, seed=1); print("gen", time.time() - t)
    r = run("C3", dg, loop_mode="graph", reps=3)
    print(r.report.matched_per_round_count)
    print("verify", dg.verify(r.matching.matched_edges))
    dg.release()
if "c4" in which:
    t = time.time(); dg = hb.DeviceHypergraph.generate("netlist", n=10_000_000, m=20_000_000, seed=1, int_weights=True); print("gen", time.time() - t)
    r = run("C4", dg, loop_mode="graph", reps=3)
    print(r.report.matched_per_round_count)
    print("verify", dg.verify(r.matching.matched_edges))
    dg.release()
