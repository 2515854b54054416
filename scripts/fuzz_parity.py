"""Randomised parity soak: many small and a few medium instances x stream modes x every engine (CRCW graph / host
loop, exact ties, vertex-owned, vertex-owned handed over to CRCW early, edge-partitioned with 2-4 co-located
shards, host arrays over several blocks) against the CPU oracle.  Test infrastructure (imports oracle/).

    python scripts/fuzz_parity.py [seconds] [seed]     -> summary line per engine, non-zero exit on any mismatch
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2602_22976_b200 as hb  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from paper_2602_22976_b200 import multi_gpu  # noqa: E402
from tests.util import to_hb_graph, to_hb_stream  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
port = po.Oracle("port")
counts, bad = {}, []


def same(got, want):
    return (np.array_equal(got.matching.matched_edges, want.matched_edges) and got.report.rounds == want.rounds
            and got.report.matched_per_round_count == want.per_round_matched
            and got.report.deactivated_per_round == want.per_round_deactivated
            and got.matching.total_weight == want.total_weight
            and (got.report.matched_round is None
                 or np.array_equal(got.report.matched_round.astype(np.uint32), want.matched_round)))


def rand_stream():
    kind = int(rng.integers(0, 3))
    mode = int(rng.integers(0, 2))
    lo = float(rng.choice([0.0, 0.0, 1.5, 100.0]))
    width = float(rng.choice([0.0, 2.0 ** -50, 1e-3, 1.0, 100.0, 1e6]))
    return po.Stream(seed=int(rng.integers(0, 2 ** 62)), kind=kind, mode=mode, noise_low=lo, noise_high=lo + width)


def rand_graph(medium):
    if medium:
        n, m = int(rng.integers(20_000, 60_000)), int(rng.integers(70_000, 140_000))
    else:
        n, m = int(rng.integers(2, 3000)), int(rng.integers(1, 5000))
    lo = int(rng.integers(1, 4))
    hi = min(n, lo + int(rng.choice([0, 1, 3, 8, 40])))
    lo = min(lo, hi)
    if rng.random() < 0.3:  # uniform 2 / 4 / 8: the one-launch kernel of small instances (k_rounds_fused)
        lo = hi = min(n, int(rng.choice([2, 4, 8])))
    g = port.generate_random(n, m, lo, hi, int(rng.integers(0, 2 ** 31)))
    w = int(rng.integers(0, 4))
    if w == 1:
        g.base_weights = port.random_weights_1_100(g.m, int(rng.integers(0, 1000)))
    elif w == 2:
        g.base_weights = rng.random(g.m) * float(rng.choice([1.0, 1e-3, 1e6])) + 1e-9
    elif w == 3:
        g.base_weights = rng.integers(1, 3, g.m).astype(np.float64)
    return g


def check(name, got, want, what):
    counts[name] = counts.get(name, 0) + 1
    if not same(got, want):
        bad.append((name, what))
        print("MISMATCH", name, what, flush=True)


t_end = time.time() + budget
it = 0
while time.time() < t_end and not bad:
    it += 1
    medium = it % 25 == 0
    g = rand_graph(medium)
    s = rand_stream()
    want = port.local_max(g, s)
    hs, hg = to_hb_stream(s), to_hb_graph(g)
    what = f"it {it} n={g.n} m={g.m} kappa={g.kappa} stream={s}"
    dg = hb.DeviceHypergraph.upload(hg)
    os.environ.pop("HLM_B200_AUTO", None)
    os.environ.pop("HLM_B200_CREW_TAIL", None)
    r = dg.match(hs, hb.ParallelConfig(variant="crcw", loop_mode="graph"))
    check("crcw graph", r, want, what)
    if r.report.kernel_launches == 1:
        check("crcw graph, one launch", r, want, what)
        check("crcw graph, one launch, no round record",
              dg.match(hs, hb.ParallelConfig(variant="crcw", loop_mode="graph", want_round_of=False)), want, what)
    check("crcw host", dg.match(hs, hb.ParallelConfig(variant="crcw", loop_mode="host")), want, what)
    check("crcw exact ties", dg.match(hs, hb.ParallelConfig(variant="crcw", tie_mode="exact")), want, what)
    check("crew graph", dg.match(hs, hb.ParallelConfig(variant="crew")), want, what)
    check("crew host", dg.match(hs, hb.ParallelConfig(variant="crew", loop_mode="host")), want, what)
    dg.release()
    if medium:
        # the vertex-owned engine on the caller's edge order, handed over to the CRCW kernels before round 3
        os.environ["HLM_B200_AUTO"] = "crew"
        os.environ["HLM_B200_CREW_TAIL"] = "100000"
        os.environ["HLM_B200_REORDER"] = "0"
        dg = hb.DeviceHypergraph.upload(hg)
        os.environ.pop("HLM_B200_REORDER", None)
        for loop in ("graph", "host"):
            r = dg.match(hs, hb.ParallelConfig(variant="auto", loop_mode=loop))
            check("vertex-owned, crcw tail", r, want, what)
            if want.rounds >= 3 and "crcw from round" not in r.report.engine:
                bad.append(("vertex-owned, crcw tail", "no hand-over: " + r.report.engine))
        dg.release()
        os.environ.pop("HLM_B200_AUTO", None)
        os.environ.pop("HLM_B200_CREW_TAIL", None)
        shards = multi_gpu.upload_shards(hg, 1)
        r, _ = multi_gpu.match_sharded(shards, hs)
        check("sharded x1", r, want, what)
        for sh in shards:
            sh.release()
    world = int(rng.integers(2, 5))
    shards = multi_gpu.upload_shards(hg, world)
    r, _ = multi_gpu.match_sharded(shards, hs, hb.ParallelConfig(tie_mode="exact" if it % 3 == 0 else "auto"))
    check("sharded co-located", r, want, what)
    for sh in shards:
        sh.release()
    if it % 4 == 0:
        check("host arrays, num_gpus", hb.run_variant(hg, hs, hb.ParallelConfig(num_gpus=int(rng.integers(2, 6)))), want, what)
    if it % 5 == 0:
        # the host-assisted loader on small instances (threshold lowered): uniformity scan, weight codes, 16-bit sizes
        os.environ["HLM_B200_ASSIST_MIN_EDGES"] = "2"
        check("host arrays, assisted loader", hb.run_variant(hg, hs, hb.ParallelConfig(variant="auto")), want, what)
        os.environ.pop("HLM_B200_ASSIST_MIN_EDGES", None)
print(f"{it} instances in {budget:.0f} s")
for k, v in sorted(counts.items()):
    print(f"  {k:28s} {v} matchings compared with the oracle: {'ok' if not any(b[0] == k for b in bad) else 'MISMATCH'}")
sys.exit(1 if bad else 0)
