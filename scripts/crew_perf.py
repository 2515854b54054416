"""CREW (compacting, vertex-owned) vs CREW (soft deletion) vs CRCW on the config shapes: device ms, verified."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2602_22976_b200 as hb  # noqa: E402

CASES = {
    "c1": dict(family="uniform", n=1_000_000, m=1_000_000, d=4, seed=1),
    "c2s": dict(family="rmat", scale=20, m=1 << 24, seed=1, int_weights=True),
    "c3s": dict(family="powerlaw", n=5_000_000, m=10_000_000, seed=1),
    "c4": dict(family="netlist", n=10_000_000, m=20_000_000, seed=1, int_weights=True),
    "u8s": dict(family="uniform", n=12_500_000, m=25_000_000, d=8, seed=1),
    "u8": dict(family="uniform", n=125_000_000, m=250_000_000, d=8, seed=1),
    "c3": dict(family="powerlaw", n=50_000_000, m=100_000_000, seed=1),
    "c2": dict(family="rmat", scale=24, m=1 << 28, seed=1, int_weights=True),
}
def main(which):
  for name in which:
      dg = hb.DeviceHypergraph.generate(**CASES[name])
      info = dg.info()
      ref = None
      for label, variant, soft in (("crcw", "crcw", "0"), ("crew", "crew", "0"), ("crew-soft", "crew", "1")):
          if label == "crew-soft" and name in ("u8", "c3", "c2"):
              continue
          os.environ["HLM_B200_CREW_SOFT"] = soft
          best = None
          for _ in range(4):
              r = dg.match(hb.WeightStream(), hb.ParallelConfig(variant=variant, loop_mode="graph"))
              if best is None or r.report.device_ms < best.report.device_ms:
                  best = r
          ids = np.asarray(best.matching.matched_edges)
          if ref is None:
              ref = (ids.copy(), best.report.rounds, list(best.report.matched_per_round_count), list(best.report.deactivated_per_round))
              same = "ref"
          else:
              same = "same" if (np.array_equal(ids, ref[0]) and best.report.rounds == ref[1] and
                                list(best.report.matched_per_round_count) == ref[2] and
                                list(best.report.deactivated_per_round) == ref[3]) else "DIFFERENT"
          print(f"{name:4s} {label:9s} pins {info.num_pins:11d} rounds {best.report.rounds:2d} |M| {len(ids):9d} "
                f"device ms {best.report.device_ms:9.3f}  G pins/s {info.num_pins / best.report.device_ms / 1e6:7.2f}  {same}", flush=True)
      dg.release()


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2s", "c3s", "c4", "u8s"])
