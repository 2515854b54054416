#!/usr/bin/env python
"""bench.py -- headline benchmark of the B200-native local-max hypergraph matching (HLM).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2] [--configs all|none]

Metric (BASELINE.json): pins/s and ms to a maximal matching on synthetic hypergraphs, next to the
HBM roofline and the reference CPU implementation.  One "step" = one complete matching (all
rounds, result assembled and copied back) of the workload instance.

* value        -- whole-job pins/s with the instance already resident in HBM (paper protocol,
                  PAPER.md:316-319: load + H2D excluded, per-round noise generation included),
                  timed with CUDA events on the launching stream around exactly K steps.
* e2e          -- the same metric through the drop-in call hlm_b200_match_host (C-ABI, host
                  buffers): H2D of the CSR, loader kernels, matching, result D2H -- from page-locked
                  arrays (the contract's number) and from ordinary pageable ones (`e2e.pageable`: what a
                  caller holding std::vector storage gets).
* roofline     -- dominant kernel (the round sweep) algorithmic bytes / its CUDA-event time vs the
                  measured HBM copy bandwidth (MEASURED_PEAKS.json); `traffic` = DRAM bytes per launch
                  from the ncu capture of the same workload (profiles/traffic_r02.json).
* configs      -- every BASELINE config that fits one GPU (c1 .. c4 and the single-GPU shard shape of c5),
                  each run with variant "auto": ms, pins/s, rounds, whole-job and dominant-kernel fraction
                  of the HBM roofline.
* cpu_baseline -- the unmodified reference (oracle/_ref) on the SAME instance when host memory allows
                  (single-core local_max_sequential and all-core local_max_crcw), else on a bounded sample.

`--impl reference` times the reference's own CPU implementation (oracle/_ref, local_max_crcw, all
cores) on the same configuration.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pins_per_sec_to_maximal_matching"
UNIT = "pins/s"

WORKLOADS = {
    # BASELINE.json configs[0]: the reference's own CPU-runnable case (reference generator, host -> upload)
    "c1": dict(desc="config 1: generate_random 4-uniform, n=1M (981682 after dropping unused), m=1M, unit weights, seed 1",
               family="reference_random", n=1_000_000, m=1_000_000, d=4, seed=1, int_weights=False),
    # BASELINE.json configs[1]: the configuration the metric is quoted on at N = 1
    "c2": dict(desc="config 2: RMAT graph (d=2) scale 24, 2^28 edges, integer weights 1-100, seed 1; "
                    "default stream (xorshift, noise [0,100), seed 1)",
               family="rmat", scale=24, m=1 << 28, seed=1, int_weights=True,
               sample=dict(family="rmat", scale=20, m=1 << 24, seed=1, int_weights=True),
               sample_desc="same generator at scale 20, 2^24 edges (1/16 of the pins)"),
    "c2s": dict(desc="RMAT scale 20, 2^24 edges (smoke-size)", family="rmat", scale=20, m=1 << 24, seed=1,
                int_weights=True, sample=dict(family="rmat", scale=16, m=1 << 20, seed=1, int_weights=True),
                sample_desc="scale 16, 2^20 edges"),
    "c3": dict(desc="config 3: power-law hypergraph n=50M, m=100M, sizes 2-64, unit weights, seed 1",
               family="powerlaw", n=50_000_000, m=100_000_000, seed=1, int_weights=False,
               sample=dict(family="powerlaw", n=2_500_000, m=5_000_000, seed=1, int_weights=False),
               sample_desc="same generator at n=2.5M, m=5M (1/20)"),
    "c4": dict(desc="config 4: netlist-like hypergraph n=10M, m=20M, edge sizes up to 4096, weights 1-100",
               family="netlist", n=10_000_000, m=20_000_000, seed=1, int_weights=True,
               sample=dict(family="netlist", n=1_000_000, m=2_000_000, seed=1, int_weights=True),
               sample_desc="same generator at n=1M, m=2M (1/10)"),
    # BASELINE.json configs[4] does not fit one GPU; this is the shard one of its 8 GPUs holds at weak scaling
    "c5s": dict(desc="config 5, single-GPU shard shape: 8-uniform n=125M, m=250M (2 G pins), unit weights, seed 1",
                family="uniform", n=125_000_000, m=250_000_000, d=8, seed=1, int_weights=False,
                sample=dict(family="uniform", n=1_250_000, m=2_500_000, d=8, seed=1, int_weights=False),
                sample_desc="same generator at n=1.25M, m=2.5M (1/100)"),
}
CONFIG_ORDER = ["c1", "c2", "c3", "c4", "c5s"]


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def begin(self):
        """The timed region starts here (nvidia-smi was started earlier: it needs ~0.2 s to come up)."""
        self.t_begin = time.time()

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        t_begin = getattr(self, "t_begin", 0.0)
        window = [ln for t, ln in self.lines if t >= t_begin]
        if len(window) < 3:  # a very short region: the samples around it
            window = [ln for t, ln in self.lines if t >= t_begin - 0.2]
        for ln in window:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), p[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        top = sorted(sm)[len(sm) // 2:]  # samples under load = the upper half
        return {"sm_mhz": sorted(top)[len(top) // 2], "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def algorithmic_bytes(kappa, m, n, d_uniform, per_round_matched, per_round_deact):
    """SURVEY.md 8(d) / DESIGN.md: bytes the path must move per round with B200 element sizes
    (bytes_r = 29 kappa_r + 13 m_r + 8 n_r).  Returns the whole-job total and its split over the launches
    of the two engines:
      CRCW   sweep(r) = 5 kappa_{r-1} + 12 kappa_r + 12 m_r   (invalidate of r-1 + compact + vertex-max of r)
             check(r) = 12 kappa_r + 13 m_r
      vertex-owned (crew kernels)
             sweep(r) = 12 kappa_r + 8 n_r                    (vertex-max over the incidence lists)
             rest(r)  = 17 kappa_r + 13 m_r                   (agreement + invalidate)
    For ragged instances kappa_r and n_r use the mean edge size (the device does not report them)."""
    rounds = len(per_round_matched)
    m_r, n_r = [], []
    act, live = m, n
    avg = kappa / max(1, m)
    for q in range(rounds):
        m_r.append(act)
        n_r.append(max(0, live))
        act -= per_round_matched[q] + per_round_deact[q]
        live -= int((d_uniform or avg) * per_round_matched[q])
    k_r = [x * (d_uniform if d_uniform else avg) for x in m_r]
    total = sum(29 * k + 13 * mm + 8 * nn for k, mm, nn in zip(k_r, m_r, n_r))
    filt, chk = [], []
    for q in range(rounds + 1):
        k_prev = k_r[q - 1] if q >= 1 else 0
        k_cur = k_r[q] if q < rounds else 0
        m_cur = m_r[q] if q < rounds else 0
        filt.append(5 * k_prev + 12 * k_cur + 12 * m_cur)
        chk.append(12 * k_cur + 13 * m_cur)
    vsweep = [12 * k + 8 * nn for k, nn in zip(k_r, n_r)]
    vrest = [17 * k + 13 * mm for k, mm in zip(k_r, m_r)]
    return total, filt, chk, vsweep, vrest


def host_mem_available_gb():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) / 1e6
    except OSError:
        pass
    return 0.0


def oracle_instance(po, gen, spec):
    """The workload instance on the host, from the checker's generators (bit-identical to the device ones)."""
    if spec["family"] == "reference_random":
        return gen.generate_random(spec["n"], spec["m"], spec["d"], spec["d"], spec["seed"])
    fam = {"uniform": po.SYN_UNIFORM, "rmat": po.SYN_RMAT, "powerlaw": po.SYN_POWERLAW, "netlist": po.SYN_NETLIST}[spec["family"]]
    return gen.syn_generate(fam, n=spec.get("n", 0), m=spec["m"], d=spec.get("d", 0), scale=spec.get("scale", 0),
                            seed=spec["seed"], int_weights=spec["int_weights"])


def full_config_fits(wl):
    """Host bytes of the reference's Hypergraph for the whole workload (both CSR sides) plus the run state."""
    if wl["family"] == "rmat":
        kappa, m, n = 2 * wl["m"], wl["m"], 1 << wl["scale"]
    elif wl["family"] in ("uniform", "reference_random"):
        kappa, m, n = wl["d"] * wl["m"], wl["m"], wl["n"]
    else:
        kappa, m, n = 7 * wl["m"], wl["m"], wl["n"]
    need = (kappa * 8 + m * 16 + n * 8) * 2.2 + m * 40 + n * 16  # checker copy + reference copy + run state
    return need / 1e9 + 6 < host_mem_available_gb(), need / 1e9


def reference_arm(args, wl):
    """`--impl reference`: the reference's own CPU implementation on this box's host cores, on the SAME
    configuration as this repo's arm whenever it fits host memory (config 2: 8.6 GB of Hypergraph)."""
    import numpy as np  # noqa: F401

    from oracle import pyoracle as po
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    kind = "reference" if po.reference_available() else "port"
    orc = po.Oracle(kind)
    gen = po.Oracle("port")
    sample_desc, same = None, True
    if args.gpus > 1:
        # the N > 1 arm of this repo runs the config-5 shape (multi_gpu.bench_main); the whole instance
        # (n = 125 M x N, m = 250 M x N) does not fit host memory at N = 8, so: 1/128 of it
        per_m = int(os.environ.get("HLM_BENCH_MG_EDGES", 250_000_000))
        per_n = int(os.environ.get("HLM_BENCH_MG_VERTICES", 125_000_000))
        n5, m5 = per_n * args.gpus, per_m * args.gpus
        wl = dict(desc=f"config 5 shape: 8-uniform, n={n5}, m={m5} edge-partitioned over {args.gpus} GPUs "
                       f"({per_m} edges per GPU), unit weights, default stream")
        spec = dict(family="uniform", n=max(1000, n5 // 128), m=max(1000, m5 // 128), d=8, seed=1, int_weights=False)
        sample_desc, same = "same generator at 1/128 of the vertices and edges", False
    else:
        fits, need_gb = full_config_fits(wl)
        if fits and os.environ.get("HLM_BENCH_REF_SAMPLE") != "1":
            spec = wl
        else:
            spec = wl["sample"]
            sample_desc, same = wl["sample_desc"] + f" (the full instance needs {need_gb:.0f} GB of host memory)", False
    t_gen = time.perf_counter()
    g = oracle_instance(po, gen, spec)
    t_gen = time.perf_counter() - t_gen
    stream = po.Stream()
    cores = orc.hardware_workers() if kind == "reference" else 1
    if kind == "reference":
        h = orc.graph_handle(g)
        run = lambda: orc.run_handle(h, stream, po.VARIANT_CRCW, cores)  # noqa: E731
    else:
        run = lambda: orc.local_max(g, stream)  # noqa: E731
    # bounded: the whole arm must end within a few minutes whatever --steps says
    budget_s = float(os.environ.get("HLM_BENCH_REF_BUDGET_S", 150))
    t0 = time.perf_counter()
    first = run()
    per_run = max(1e-3, time.perf_counter() - t0)
    warm = 1 + (1 if args.warmup >= 2 and per_run * 3 < budget_s else 0)
    if warm == 2:
        run()
    steps = max(1, min(args.steps, int((budget_s - per_run * warm) / per_run)))
    times = []
    t0 = time.perf_counter()
    for _ in range(steps):
        times.append(run().wall_ms)
    wall = time.perf_counter() - t0
    ms = sum(times) / len(times)
    value = g.kappa / (ms * 1e-3)
    sample = sample_desc or "the whole configuration (same instance as this repo's arm)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "steps_requested": args.steps, "warmup": warm, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl["desc"], "same_config": same, "sample": sample, "variant": "crcw",
                       "pins": int(g.kappa), "edges": int(g.m), "vertices": int(g.n), "rounds": int(first.rounds),
                       "timing": "report.wall_time_ms of the reference (load excluded)", "wall_s": wall,
                       "instance_generation_s": t_gen, "best_ms": min(times)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(wl, want=None):
    """The unmodified reference (or the C port) timed beside the GPU run: on the SAME instance when host
    memory allows -- single-core local_max_sequential (the "x over single core" denominator) and all-core
    local_max_crcw -- else on a bounded scaled-down sample.  `want`: the GPU result to compare with."""
    from oracle import pyoracle as po
    kind = "reference" if po.reference_available() else "port"
    orc = po.Oracle(kind)
    gen = po.Oracle("port")
    fits, need_gb = full_config_fits(wl)
    full = fits and kind == "reference" and os.environ.get("HLM_BENCH_CPU_SAMPLE") != "1"
    spec = wl if full else wl["sample"]
    g = oracle_instance(po, gen, spec)
    stream = po.Stream()
    sample = ("the whole configuration (same instance)" if full else wl["sample_desc"])
    out = {"unit": UNIT, "kind": kind, "sample": sample + "; local_max_sequential", "sample_pins": int(g.kappa),
           "same_config": bool(full)}
    if kind == "reference":
        h = orc.graph_handle(g)
        ncores = orc.hardware_workers()
        allc = orc.run_handle(h, stream, po.VARIANT_CRCW, ncores)
        seq = orc.run_handle(h, stream, po.VARIANT_SEQ, 1).wall_ms
        if not full:
            seq = min(seq, orc.run_handle(h, stream, po.VARIANT_SEQ, 1).wall_ms)
            one = orc.run_handle(h, stream, po.VARIANT_CRCW, 1)
            out["crcw_1core"] = {"value": g.kappa / (one.wall_ms * 1e-3), "ms": one.wall_ms}
        orc.graph_release(h)
        out.update(value=g.kappa / (seq * 1e-3), cores=1, seq_ms=seq,
                   crcw_allcores={"value": g.kappa / (allc.wall_ms * 1e-3), "ms": allc.wall_ms, "cores": ncores},
                   rounds=allc.rounds)
        if full and want is not None:
            import numpy as np

            out["gpu_result_identical"] = bool(
                np.array_equal(want.matching.matched_edges, allc.matched_edges) and want.report.rounds == allc.rounds
                and want.report.matched_per_round_count == allc.per_round_matched
                and want.report.deactivated_per_round == allc.per_round_deactivated
                and want.matching.total_weight == allc.total_weight)
    else:
        r = orc.local_max(g, stream)
        out.update(value=g.kappa / (r.wall_ms * 1e-3), cores=1, seq_ms=r.wall_ms)
    return out


def make_instance(hb, wl, device):
    if wl["family"] == "reference_random":
        host = hb.generate_random(wl["n"], wl["m"], wl["d"], wl["d"], wl["seed"])
        return hb.DeviceHypergraph.upload(host, device)
    return hb.DeviceHypergraph.generate(wl["family"], n=wl.get("n", 0), m=wl["m"], d=wl.get("d", 0), scale=wl.get("scale", 0),
                                        seed=wl["seed"], int_weights=wl["int_weights"], device=device)


def measure(hb, torch, np, dg, wl, steps, warmup, tstream, hbm_gbs):
    """One workload, instance resident: K timed matchings (variant auto, one CUDA-graph launch per matching
    where the engine has one), then a pass with CUDA events around every round kernel for the roofline."""
    info = dg.info()
    kappa, m, n = int(info.num_pins), int(info.num_edges), int(info.num_vertices)
    stream = hb.WeightStream()
    cfg = hb.ParallelConfig(variant="auto", loop_mode="graph")
    dg.set_stream(tstream.cuda_stream)
    for _ in range(max(3, warmup)):
        res = dg.match(stream, cfg)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches, dev_ms = 0, []
    ev0.record(tstream)
    for _ in range(steps):
        res = dg.match(stream, cfg)
        launches += res.report.kernel_launches
        dev_ms.append(res.report.device_ms)
    ev1.record(tstream)
    torch.cuda.synchronize()
    total_ms = ev0.elapsed_time(ev1)
    ms_per_step = total_ms / steps
    crcw_engine = res.report.engine == "crcw"
    # per-kernel times: host-driven loop, CUDA events around every launch, best of 3
    prof_cfg = hb.ParallelConfig(variant="auto", loop_mode="host", kernel_times=True)
    sweep_ms = rest_ms = None
    for _ in range(3):
        pres = dg.match(stream, prof_cfg)
        f, c = np.array(pres.report.round_filter_ms), np.array(pres.report.round_check_ms)
        sweep_ms = f if sweep_ms is None else np.minimum(sweep_ms, f)
        rest_ms = c if rest_ms is None else np.minimum(rest_ms, c)
    rep = res.report
    total_bytes, fb, cb, vs, vr = algorithmic_bytes(kappa, m, n, int(info.uniform_size), rep.matched_per_round_count,
                                                    rep.deactivated_per_round)
    if crcw_engine:
        sweep_bytes = fb
        d = int(info.uniform_size)
        kernel = ((f"round sweep of the CRCW engine: k_sweep_uniform<{d},1,1> (round 1), "
                   + ("k_sweep_uniform_dense<2>" if d == 2 else f"k_sweep_uniform_simple<{d}>" if d == 4 else f"k_sweep_uniform<{d},1,0>")
                   + " (later rounds)") if d in (2, 4, 8) else
                  "round sweep of the CRCW engine: k_filter_vmax_small / k_filter_vmax_large") + \
            ": invalidate + compact + key + vertex-max atomics"
    else:
        # vertex-owned rounds: the vertex-max sweep over the incidence lists; after the hand-over (if any) the
        # CRCW round sweep, each with its own share of the algorithmic bytes
        sw = res.report.engine_switch_round or (len(vs) + 1)
        sweep_bytes = [vs[q] if q + 1 < sw else fb[q] for q in range(len(vs))]
        kernel = ("vertex-max sweep of the vertex-owned engine: k_c2_argmax_light<MODE,KM> (+ k_c2_argmax_task / "
                  "k_c2_argmax_heavy for lists > 256 entries): list walk + alive filter + key + argmax + compaction"
                  + (f"; from round {sw} the CRCW round sweep (few edges left)" if res.report.engine_switch_round else ""))
    nl = len(sweep_bytes)
    sweep_total_ms = float(sweep_ms[:nl].sum())
    rest_total_ms = float(rest_ms[:nl].sum())
    achieved = sum(sweep_bytes) / (sweep_total_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": hbm_gbs, "unit": "GB/s",
                "frac": achieved / hbm_gbs, "traffic": None, "launches_per_step": nl,
                "algorithmic_bytes_per_launch": sum(sweep_bytes) / nl, "avg_launch_ms": sweep_total_ms / nl,
                "share_of_step": sweep_total_ms / max(1e-9, sweep_total_ms + rest_total_ms),
                "share_source": "host-driven pass of the same kernels (CUDA events around every launch); the timed "
                                "steps run them from one CUDA graph where the engine has one",
                "round1_frac": sweep_bytes[0] / (float(sweep_ms[0]) * 1e-3) / 1e9 / hbm_gbs,
                "whole_job": {"algorithmic_bytes": total_bytes, "achieved": total_bytes / (ms_per_step * 1e-3) / 1e9,
                              "frac": total_bytes / (ms_per_step * 1e-3) / 1e9 / hbm_gbs}}
    out = dict(kappa=kappa, m=m, n=n, ms_per_step=ms_per_step, total_ms=total_ms, value=kappa * steps / (total_ms * 1e-3),
               launches=int(launches), dev_ms=float(np.mean(dev_ms)), res=res, roofline=roofline,
               engine=res.report.engine + (" (ONE cooperative kernel launch per matching: k_rounds_fused = state reset, "
                                           "all rounds, result assembly)" if res.report.kernel_launches == 1
                                           else " (one CUDA-graph launch per matching)"))
    return out


def config_entry(name, wl, r):
    rep = r["res"].report
    return {"name": name, "workload": wl["desc"], "pins": r["kappa"], "edges": r["m"], "vertices": r["n"],
            "variant": "auto", "engine": r["engine"], "rounds": rep.rounds, "matched": int(len(r["res"].matching.matched_edges)),
            "ms": r["ms_per_step"], "device_ms": r["dev_ms"], "pins_per_s": r["value"], "whole_job_frac": r["roofline"]["whole_job"]["frac"],
            "dominant_kernel": r["roofline"]["kernel"].split(":")[0], "dominant_frac": r["roofline"]["frac"],
            "dominant_round1_frac": r["roofline"]["round1_frac"], "dominant_share_of_step": r["roofline"]["share_of_step"],
            "algorithmic_bytes": r["roofline"]["whole_job"]["algorithmic_bytes"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=os.environ.get("HLM_BENCH_WORKLOAD", "c2"))
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--configs", default=os.environ.get("HLM_BENCH_CONFIGS", "all"), choices=["all", "none"],
                    help="also run the other BASELINE configs (5 steps each) and report them in `configs`")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]

    if args.impl == "reference":
        reference_arm(args, wl)
        return

    import numpy as np
    import torch

    import paper_2602_22976_b200 as hb

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device: the matching path has no CPU fallback")
    # HLM_BENCH_ONE_GPU=1: dry run of the N-rank path on a box with one device (tests/test_gpu_multi.py): every
    # rank uses device 0, gloo carries the communicator id, and HLM_B200_NCCL_LIB must name a transport that
    # accepts several ranks per device (NCCL does not).  Not a measurement.
    one_gpu = os.environ.get("HLM_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    # HLM_BENCH_FORCE_MG=1 runs the edge-partitioned (multi-GPU) driver even with one rank: the only
    # way to exercise that code path on a single-GPU box
    sharded = world > 1 or os.environ.get("HLM_BENCH_FORCE_MG") == "1"
    hbm_gbs, peak_src = load_peaks()
    if sharded:
        import torch.distributed as dist_mod

        # NCCL writes its version line to stdout: everything but the one JSON line goes to stderr
        sys.stdout.flush()
        json_fd = os.dup(1)
        os.dup2(2, 1)

        def emit(text):
            sys.stdout.flush()
            os.write(json_fd, (text + "\n").encode())

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        if one_gpu:
            dist_mod.init_process_group("gloo")
        else:
            dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        from paper_2602_22976_b200 import multi_gpu

        multi_gpu.bench_main(args, wl, rank, world, local_rank, dist_mod,
                             extras=dict(emit=emit, sampler=ClockSampler(local_rank) if rank == 0 else None,
                                         algorithmic_bytes=lambda *a: algorithmic_bytes(*a)[:3], hbm_gbs=hbm_gbs,
                                         peak_src=peak_src))
        dist_mod.destroy_process_group()
        return

    tstream = torch.cuda.Stream()  # a real (non-legacy) stream: the library launches on it
    torch.cuda.set_stream(tstream)
    dg = make_instance(hb, wl, local_rank)
    sampler = ClockSampler(local_rank)
    sampler.start()  # before the warm-up: nvidia-smi needs a moment before its first line
    time.sleep(0.3)
    sampler.begin()
    r = measure(hb, torch, np, dg, wl, args.steps, args.warmup, tstream, hbm_gbs)
    clocks = sampler.stop()
    res, rep = r["res"], r["res"].report
    kappa, m, n = r["kappa"], r["m"], r["n"]
    roofline = r["roofline"]
    roofline["peak_source"] = peak_src
    roofline["note"] = ("the sweeps are bound by the SM's sector rate for uncoalesced accesses (1 sector/clk/SM = "
                        "285-300 G random 4-byte gathers/s measured, scripts/micro/gather_bench.cu), not by HBM")
    traffic_file = os.path.join(ROOT, "profiles", "traffic_r02.json")
    if os.path.exists(traffic_file):
        with open(traffic_file) as f:
            t = json.load(f).get(args.workload, {})
        roofline["traffic"] = t.get("sweep_bytes_per_launch")
        roofline["traffic_source"] = "profiles/traffic_r02.json: dram__bytes_read.sum + dram__bytes_write.sum of the sweep " \
                                     "launches, ncu --set full capture of this workload"

    # ---- e2e: host buffers through the drop-in C-ABI call ----
    host = dg.download(pinned=True)
    h2d = host.edge_offsets.nbytes + host.edge_members.nbytes + host.base_weights.nbytes
    dg.release()
    torch.cuda.synchronize()
    e2e_cfg = hb.ParallelConfig(variant="auto")  # the call a user makes (variant auto = crcw to the caller)
    e2e_steps = max(1, min(args.e2e_steps, args.steps))

    def e2e_leg(h, warm=3):
        for _ in range(warm):  # warm: the first calls still grow the memory pools; the result stays bound like in the
            # timed loop, so the second set of page-locked result arrays is allocated here, not there
            er = hb.run_variant(h, hb.WeightStream(), e2e_cfg, device=local_rank)
        each = []
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            t1 = time.perf_counter()
            er = hb.run_variant(h, hb.WeightStream(), e2e_cfg, device=local_rank)
            each.append(round((time.perf_counter() - t1) * 1e3, 2))
        return (time.perf_counter() - t0) / e2e_steps, each, er

    e2e_s, e2e_each, eres = e2e_leg(host)
    d2h = int(eres.matching.matched_edges.nbytes + eres.report.matched_round.nbytes + 8 * eres.report.rounds)
    assert np.array_equal(eres.matching.matched_edges, res.matching.matched_edges)
    e2e = {"value": kappa / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(eres.report.h2d_bytes),
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3, "steps": e2e_steps, "warmup": 3,
           "ms_each": e2e_each, "host_input_bytes": int(h2d), "host_memory": "page-locked",
           "call": "hlm_b200_match_host (host scan/pack of offsets+weights || pin upload, loader kernels, matching, "
                   "result copy)"}
    if os.environ.get("HLM_BENCH_PAGEABLE", "1") == "1":
        # the same call on ordinary (pageable) arrays: what a caller holding std::vector storage gets
        pageable = hb.Hypergraph(host.num_vertices, host.num_edges, None, None, np.array(host.edge_offsets, copy=True),
                                 np.array(host.edge_members, copy=True), np.array(host.base_weights, copy=True))
        # (five warm calls: freshly written pageable arrays keep getting faster for several passes on some
        # boxes -- page migration / huge-page collapse behind the copy -- 113, 101, 84, 82, 78 ms seen)
        p_s, p_each, pres = e2e_leg(pageable, warm=5)
        assert np.array_equal(pres.matching.matched_edges, res.matching.matched_edges)
        e2e["pageable"] = {"value": kappa / p_s, "ms_per_step": p_s * 1e3, "ms_each": p_each,
                           "h2d_bytes_per_step": int(pres.report.h2d_bytes), "warmup": 5,
                           "host_memory": "pageable (numpy / std::vector)"}
        del pageable
    del host

    line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": r["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64 keys (f64 weights, u32 ids)",
            "data": "synthetic",
            "config": {"workload": wl["desc"], "pins": kappa, "edges": m, "vertices": n, "variant": "auto",
                       "engine": r["engine"], "rounds": rep.rounds, "matched": int(len(res.matching.matched_edges)),
                       "l2_policy": "inputs larger than L2 (pins %.1f GB); no flush" % (kappa * 4 / 1e9),
                       "device_ms_per_step_lib_events": r["dev_ms"],
                       "matched_per_round": rep.matched_per_round_count},
            "clocks": clocks, "e2e": e2e, "gpu_launches": r["launches"], "roofline": roofline}

    # ---- the other BASELINE configs (variant auto each), 5 steps apiece ----
    if args.configs == "all":
        entries = {args.workload: config_entry(args.workload, wl, r)}
        for name in CONFIG_ORDER:
            if name in entries:
                continue
            try:
                g2 = make_instance(hb, WORKLOADS[name], local_rank)
                r2 = measure(hb, torch, np, g2, WORKLOADS[name], 5, 3, tstream, hbm_gbs)
                if r2["ms_per_step"] < 2.0:  # a sub-millisecond matching: five calls time the first-call effects
                    r2 = measure(hb, torch, np, g2, WORKLOADS[name], 50, 5, tstream, hbm_gbs)
                entries[name] = config_entry(name, WORKLOADS[name], r2)
                entries[name]["steps"] = 50 if r2["ms_per_step"] < 2.0 else 5
                # the same config through the drop-in call on host arrays (page-locked), where the download is
                # cheap enough for a side line: 2 warm + 3 timed calls of hlm_b200_match_host
                if r2["kappa"] <= 1_000_000_000 and os.environ.get("HLM_BENCH_CONFIG_E2E", "1") == "1":
                    h2 = g2.download(pinned=True)
                    g2.release()
                    for _ in range(2):
                        er2 = hb.run_variant(h2, hb.WeightStream(), hb.ParallelConfig(variant="auto"), device=local_rank)
                    t_each = []
                    for _ in range(3):
                        t1 = time.perf_counter()
                        er2 = hb.run_variant(h2, hb.WeightStream(), hb.ParallelConfig(variant="auto"), device=local_rank)
                        t_each.append((time.perf_counter() - t1) * 1e3)
                    assert np.array_equal(er2.matching.matched_edges, r2["res"].matching.matched_edges)
                    entries[name]["e2e_ms"] = float(np.mean(t_each))
                    entries[name]["e2e_h2d_bytes"] = int(er2.report.h2d_bytes)
                    entries[name]["e2e_engine"] = er2.report.engine
                    del h2, er2
                else:
                    g2.release()
                del r2
            except Exception as exc:  # one config must not cost the headline line
                entries[name] = {"name": name, "workload": WORKLOADS[name]["desc"], "failed": str(exc)}
            torch.cuda.synchronize()
        line["configs"] = [entries[k] for k in CONFIG_ORDER if k in entries] + \
                          [v for k, v in entries.items() if k not in CONFIG_ORDER]
    if not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(wl, res)
            seq_ms = line["cpu_baseline"].get("seq_ms")
            if seq_ms and line["cpu_baseline"].get("same_config"):
                line["cpu_baseline"]["speedup_vs_single_core"] = {"resident": seq_ms / r["ms_per_step"],
                                                                  "e2e": seq_ms / (e2e_s * 1e3)}
        except Exception as exc:  # the checker is optional at bench time, the GPU numbers are not
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                                    "sample": f"failed: {exc}"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
