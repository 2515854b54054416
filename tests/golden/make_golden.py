#!/usr/bin/env python
"""Generates tests/golden/*.json from the UNMODIFIED reference (oracle/_ref/libhlm_ref.so, built
by `make -C oracle ref` from /root/reference).  Run in the build container:

    python tests/golden/make_golden.py

The fixtures pin the CPU oracle (tests/test_oracle_pinned.py) and the CUDA path
(tests/test_gpu_*.py) on the GPU box, where /root/reference does not exist.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as po  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sdict(s: po.Stream):
    return {"seed": s.seed, "kind": s.kind, "mode": s.mode, "noise_low": s.noise_low, "noise_high": s.noise_high}


def all_variants_agree(ref, g, s, workers=(1, 8)):
    seq = ref.local_max(g, s, variant=po.VARIANT_SEQ)
    for v in (po.VARIANT_CRCW, po.VARIANT_CREW, po.VARIANT_WORK_OPTIMAL):
        for w in workers:
            r = ref.local_max(g, s, variant=v, workers=w)
            assert np.array_equal(r.matched_edges, seq.matched_edges) and r.rounds == seq.rounds
            assert np.array_equal(r.matched_round, seq.matched_round)
    return seq


def main():
    ref = po.Oracle("reference")

    # ---- stream bit patterns ----
    rng = np.random.default_rng(20260222)
    cases = []
    for kind in (po.GEN_XORSHIFT, po.GEN_PARK_MILLER, po.GEN_SPLITMIX):
        for mode in (po.MODE_PERTURB_BASE, po.MODE_REPLACE_UNIFORM):
            for lo, hi in ((0.0, 100.0), (0.0, 0.0), (0.5, 0.75)):
                s = po.Stream(seed=int(rng.integers(1, 2**62)), kind=kind, mode=mode, noise_low=lo, noise_high=hi)
                e = np.concatenate([rng.integers(0, 2**32 - 1, 20, dtype=np.uint64).astype(np.uint32),
                                    np.array([0, 1, 2**32 - 2], dtype=np.uint32)])
                r = np.concatenate([rng.integers(1, 190, 20).astype(np.uint32), np.array([1, 188, 7], dtype=np.uint32)])
                b = np.concatenate([rng.integers(1, 101, 12).astype(np.float64), rng.random(11) * 50 + 0.001])
                w, t = ref.eval_stream(s, e, r, b)
                cases.append({"stream": sdict(s), "edges": e.tolist(), "rounds": r.tolist(), "base": b.tolist(),
                              "weight_bits": [format(x, "016x") for x in w.view(np.uint64)],
                              "tie_hash": [format(x, "016x") for x in t]})
    with open(os.path.join(HERE, "stream_bits.json"), "w") as f:
        json.dump({"source": "oracle/_ref (reference weight_stream.hpp)", "cases": cases}, f)

    # ---- small corpus ----
    cases = []
    for seed in range(1, 41):
        n, m = 30 + 17 * seed, 40 + 29 * seed
        lo, hi = (2, 4) if seed % 4 else (1, 6)
        inst = {"n": n, "m": m, "min_size": lo, "max_size": hi, "seed": seed,
                "weights_seed": seed if seed % 3 == 0 else None}
        g = ref.generate_random(n, m, lo, hi, seed)
        if inst["weights_seed"] is not None:
            g.base_weights = ref.random_weights_1_100(g.m, seed)
        streams = [po.Stream(seed=seed * 7), po.Stream(seed=seed * 7, mode=po.MODE_REPLACE_UNIFORM),
                   po.Stream(seed=seed, noise_high=0.0), po.Stream(seed=seed, kind=po.GEN_PARK_MILLER),
                   po.Stream(seed=seed, kind=po.GEN_SPLITMIX, noise_low=1.0, noise_high=3.5)]
        s = streams[seed % len(streams)]
        r = all_variants_agree(ref, g, s)
        cases.append({"instance": inst, "n_after_drop": g.n, "kappa": g.kappa, "stream": sdict(s), "rounds": r.rounds,
                      "per_round_matched": r.per_round_matched, "per_round_deactivated": r.per_round_deactivated,
                      "matched_edges": r.matched_edges.tolist(), "total_weight": r.total_weight})
    with open(os.path.join(HERE, "small_corpus.json"), "w") as f:
        json.dump({"source": "oracle/_ref run_variant (seq == crcw == crew == work_optimal, workers 1 and 8)",
                   "cases": cases}, f)

    # ---- BASELINE config 1 in every stream mode ----
    g = ref.generate_random(1_000_000, 1_000_000, 4, 4, 1)
    unit = g.base_weights
    ints = ref.random_weights_1_100(g.m, 1)
    modes = {
        "default": (po.Stream(), None),
        "uniform": (po.Stream(mode=po.MODE_REPLACE_UNIFORM), None),
        "zero_noise": (po.Stream(noise_high=0.0), None),
        "park_miller": (po.Stream(kind=po.GEN_PARK_MILLER), None),
        "splitmix": (po.Stream(kind=po.GEN_SPLITMIX), None),
        "int_weights": (po.Stream(), 1),
        "int_weights_zero_noise": (po.Stream(noise_high=0.0), 1),
    }
    out = {}
    for name, (s, wseed) in modes.items():
        g.base_weights = unit if wseed is None else ints
        r = all_variants_agree(ref, g, s, workers=(8,))
        out[name] = {"stream": sdict(s), "weights_seed": wseed, "rounds": r.rounds, "num_matched": len(r.matched_edges),
                     "per_round_matched": r.per_round_matched, "per_round_deactivated": r.per_round_deactivated,
                     "fnv1a": format(po.fnv1a_ids(r.matched_edges), "016x"), "total_weight": r.total_weight}
        print(name, out[name]["rounds"], out[name]["num_matched"], out[name]["fnv1a"], flush=True)
    with open(os.path.join(HERE, "config1.json"), "w") as f:
        json.dump({"source": "oracle/_ref on generate_random{1e6,1e6,4,4,seed 1}", "n": g.n, "kappa": g.kappa,
                   "cases": out}, f, indent=1)


if __name__ == "__main__":
    main()
