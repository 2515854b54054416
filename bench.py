#!/usr/bin/env python
"""bench.py -- headline benchmark of the B200-native local-max hypergraph matching (HLM).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2]

Metric (BASELINE.json): pins/s and ms to a maximal matching on synthetic hypergraphs, next to the
HBM roofline and the reference CPU implementation.  One "step" = one complete matching (all
rounds, result assembled and copied back) of the workload instance.

* value        -- whole-job pins/s with the instance already resident in HBM (paper protocol,
                  PAPER.md:316-319: load + H2D excluded, per-round noise generation included),
                  timed with CUDA events on the launching stream around exactly K steps.
* e2e          -- the same metric through the drop-in call hlm_b200_match_host (C-ABI, host
                  buffers): H2D of the CSR from pinned memory, loader kernels, matching, result D2H.
* roofline     -- dominant kernel (the round sweep: k_sweep_uniform in round 1, k_sweep_uniform_simple
                  afterwards) algorithmic bytes / its CUDA-event time vs the measured HBM copy
                  bandwidth (MEASURED_PEAKS.json); `traffic` = DRAM bytes per launch from the ncu
                  capture of the same workload (profiles/traffic_r01.json).
* cpu_baseline -- the unmodified reference (oracle/_ref) on a bounded sample of the workload,
                  timed on this box's host cores.

Prints ONE JSON line on rank 0.
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
}


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
    """SURVEY.md 8(d) / DESIGN.md: bytes the path must move per round with B200 element sizes.
    Returns (total_bytes, filter_bytes_per_launch[], check_bytes_per_launch[])."""
    rounds = len(per_round_matched)
    m_r, n_r = [], []
    act, live = m, n
    for q in range(rounds):
        m_r.append(act)
        n_r.append(live)
        act -= per_round_matched[q] + per_round_deact[q]
        live -= (d_uniform or 0) * per_round_matched[q]
    avg = kappa / max(1, m)
    k_r = [x * (d_uniform if d_uniform else avg) for x in m_r]
    total = sum(29 * k + 13 * mm + 8 * nn for k, mm, nn in zip(k_r, m_r, n_r))
    filt, chk = [], []
    for q in range(rounds + 1):
        k_prev = k_r[q - 1] if q >= 1 else 0
        k_cur = k_r[q] if q < rounds else 0
        m_cur = m_r[q] if q < rounds else 0
        # invalidate sweep of the previous round (pin id + dead flag) + vertex-max of this round
        filt.append(5 * k_prev + 12 * k_cur + 12 * m_cur)
        chk.append(12 * k_cur + 13 * m_cur)
    return total, filt, chk


def reference_arm(args, wl):
    """`--impl reference`: the reference's own CPU implementation on this box's host cores."""
    import numpy as np  # noqa: F401

    from oracle import pyoracle as po
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    kind = "reference" if po.reference_available() else "port"
    orc = po.Oracle(kind)
    gen = po.Oracle("port")
    if args.gpus > 1:
        # the N > 1 arm of this repo runs the config-5 shape (multi_gpu.bench_main): the same here,
        # 1/128 of it (the whole instance does not fit host memory, nor a few minutes of CPU time)
        per_m = int(os.environ.get("HLM_BENCH_MG_EDGES", 250_000_000))
        per_n = int(os.environ.get("HLM_BENCH_MG_VERTICES", 125_000_000))
        n5, m5 = per_n * args.gpus, per_m * args.gpus
        wl = dict(desc=f"config 5 shape: 8-uniform, n={n5}, m={m5} edge-partitioned over {args.gpus} GPUs "
                       f"({per_m} edges per GPU), unit weights, default stream",
                  sample=dict(family="uniform", n=max(1000, n5 // 128), m=max(1000, m5 // 128), d=8, seed=1, int_weights=False),
                  sample_desc="same generator at 1/128 of the vertices and edges")
    s = wl["sample"]
    fam = {"uniform": po.SYN_UNIFORM, "rmat": po.SYN_RMAT, "powerlaw": po.SYN_POWERLAW, "netlist": po.SYN_NETLIST}[s["family"]]
    g = gen.syn_generate(fam, n=s.get("n", 0), m=s["m"], d=s.get("d", 0), scale=s.get("scale", 0), seed=s["seed"],
                         int_weights=s["int_weights"])
    stream = po.Stream()
    cores = orc.hardware_workers() if kind == "reference" else 1
    times = []
    if kind == "reference":
        h = orc.graph_handle(g)
        run = lambda: orc.run_handle(h, stream, po.VARIANT_CRCW, cores)  # noqa: E731
    else:
        run = lambda: orc.local_max(g, stream)  # noqa: E731
    for _ in range(args.warmup if args.warmup < 2 else 1):
        run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = run()
        times.append(r.wall_ms)
    wall = time.perf_counter() - t0
    ms = sum(times) / len(times)
    value = g.kappa / (ms * 1e-3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl["desc"], "sample": wl["sample_desc"], "variant": "crcw", "timing":
                       "report.wall_time_ms of the reference (load excluded)", "wall_s": wall},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": wl["sample_desc"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(wl):
    """Bounded CPU sample: the unmodified reference (or the C port) on a scaled-down instance."""
    from oracle import pyoracle as po
    kind = "reference" if po.reference_available() else "port"
    orc = po.Oracle(kind)
    gen = po.Oracle("port")
    s = wl["sample"]
    fam = {"uniform": po.SYN_UNIFORM, "rmat": po.SYN_RMAT, "powerlaw": po.SYN_POWERLAW, "netlist": po.SYN_NETLIST}[s["family"]]
    g = gen.syn_generate(fam, n=s.get("n", 0), m=s["m"], d=s.get("d", 0), scale=s.get("scale", 0), seed=s["seed"],
                         int_weights=s["int_weights"])
    stream = po.Stream()
    out = {"unit": UNIT, "kind": kind, "sample": wl["sample_desc"] + "; local_max_sequential, best of 2",
           "sample_pins": g.kappa}
    if kind == "reference":
        h = orc.graph_handle(g)
        seq = min(orc.run_handle(h, stream, po.VARIANT_SEQ, 1).wall_ms for _ in range(2))
        ncores = orc.hardware_workers()
        allc = orc.run_handle(h, stream, po.VARIANT_CRCW, ncores)
        one = orc.run_handle(h, stream, po.VARIANT_CRCW, 1)
        orc.graph_release(h)
        out.update(value=g.kappa / (seq * 1e-3), cores=1, seq_ms=seq,
                   crcw_1core={"value": g.kappa / (one.wall_ms * 1e-3), "ms": one.wall_ms},
                   crcw_allcores={"value": g.kappa / (allc.wall_ms * 1e-3), "ms": allc.wall_ms, "cores": ncores},
                   rounds=allc.rounds)
        ref_result = allc
    else:
        r = orc.local_max(g, stream)
        out.update(value=g.kappa / (r.wall_ms * 1e-3), cores=1, seq_ms=r.wall_ms)
        ref_result = r
    return out, g, ref_result


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=os.environ.get("HLM_BENCH_WORKLOAD", "c2"))
    ap.add_argument("--e2e-steps", type=int, default=5)
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
    torch.cuda.set_device(local_rank)
    dist = None
    # HLM_BENCH_FORCE_MG=1 runs the edge-partitioned (multi-GPU) driver even with one rank: the only
    # way to exercise that code path on a single-GPU box
    sharded = world > 1 or os.environ.get("HLM_BENCH_FORCE_MG") == "1"
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
        dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist = dist_mod
        from paper_2602_22976_b200 import multi_gpu

        hbm_gbs, peak_src = load_peaks()
        multi_gpu.bench_main(args, wl, rank, world, local_rank, dist,
                             extras=dict(emit=emit, sampler=ClockSampler(local_rank) if rank == 0 else None,
                                         algorithmic_bytes=algorithmic_bytes, hbm_gbs=hbm_gbs, peak_src=peak_src))
        dist_mod.destroy_process_group()
        return

    hbm_gbs, peak_src = load_peaks()
    spec = {k: wl[k] for k in ("family", "seed", "int_weights") if k in wl}
    dg = hb.DeviceHypergraph.generate(wl["family"], n=wl.get("n", 0), m=wl["m"], d=wl.get("d", 0),
                                      scale=wl.get("scale", 0), seed=wl["seed"], int_weights=wl["int_weights"],
                                      device=local_rank)
    info = dg.info()
    kappa, m, n = int(info.num_pins), int(info.num_edges), int(info.num_vertices)
    stream = hb.WeightStream()
    cfg = hb.ParallelConfig(variant="crcw", loop_mode="graph")
    tstream = torch.cuda.Stream()  # a real (non-legacy) stream: the library launches on it
    torch.cuda.set_stream(tstream)
    dg.set_stream(tstream.cuda_stream)

    sampler = ClockSampler(local_rank)
    sampler.start()  # before the warm-up: nvidia-smi needs a moment before its first line
    for _ in range(max(3, args.warmup)):
        res = dg.match(stream, cfg)
    torch.cuda.synchronize()
    sampler.begin()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    dev_ms = []
    ev0.record(tstream)
    for _ in range(args.steps):
        res = dg.match(stream, cfg)
        launches += res.report.kernel_launches
        dev_ms.append(res.report.device_ms)
    ev1.record(tstream)
    torch.cuda.synchronize()
    total_ms = ev0.elapsed_time(ev1)
    ms_per_step = total_ms / args.steps
    value = kappa * args.steps / (total_ms * 1e-3)

    # ---- per-kernel times (host loop, CUDA events around every round kernel) -> roofline ----
    prof_cfg = hb.ParallelConfig(variant="crcw", loop_mode="host", kernel_times=True)
    filt_ms = chk_ms = None
    for _ in range(3):
        pres = dg.match(stream, prof_cfg)
        f, c = np.array(pres.report.round_filter_ms), np.array(pres.report.round_check_ms)
        filt_ms = f if filt_ms is None else np.minimum(filt_ms, f)
        chk_ms = c if chk_ms is None else np.minimum(chk_ms, c)
    clocks = sampler.stop()
    rep = res.report
    total_bytes, fb, cb = algorithmic_bytes(kappa, m, n, int(info.uniform_size), rep.matched_per_round_count,
                                            rep.deactivated_per_round)
    filt_total_ms, chk_total_ms = float(filt_ms.sum()), float(chk_ms.sum())
    n_launch = len(fb)
    achieved = sum(fb) / (filt_total_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm",
                "kernel": "round sweep: k_sweep_uniform<2,1,1> (round 1) + k_sweep_uniform_simple<2,1> (later rounds): "
                          "invalidate + compact + key + vertex-max atomics",
                "achieved": achieved, "peak": hbm_gbs, "peak_source": peak_src, "unit": "GB/s",
                "frac": achieved / hbm_gbs, "traffic": None,
                "launches_per_step": n_launch, "algorithmic_bytes_per_launch": sum(fb) / n_launch,
                "avg_launch_ms": filt_total_ms / n_launch,
                "share_of_step": filt_total_ms / (filt_total_ms + chk_total_ms),
                "round1_frac": fb[0] / (float(filt_ms[0]) * 1e-3) / 1e9 / hbm_gbs,
                "check_kernel": {"achieved": sum(cb) / (chk_total_ms * 1e-3) / 1e9,
                                 "frac": sum(cb) / (chk_total_ms * 1e-3) / 1e9 / hbm_gbs},
                "note": "the sweeps are bound by the SM's sector rate for uncoalesced accesses (1 sector/clk/SM = "
                        "285-300 G random 4-byte gathers/s measured, scripts/micro/gather_bench.cu), not by HBM",
                "whole_job": {"algorithmic_bytes": total_bytes, "achieved": total_bytes / (ms_per_step * 1e-3) / 1e9,
                              "frac": total_bytes / (ms_per_step * 1e-3) / 1e9 / hbm_gbs}}
    traffic_file = os.path.join(ROOT, "profiles", "traffic_r01.json")
    if os.path.exists(traffic_file):
        with open(traffic_file) as f:
            roofline["traffic"] = json.load(f).get(args.workload, {}).get("filter_bytes_per_launch")

    # ---- e2e: host buffers through the drop-in C-ABI call ----
    host = dg.download(pinned=True)
    h2d = host.edge_offsets.nbytes + host.edge_members.nbytes + host.base_weights.nbytes
    dg.release()
    torch.cuda.synchronize()
    e2e_cfg = hb.ParallelConfig(variant="crcw")  # the call a user makes: default loop mode (host loop for one matching)
    for _ in range(3):  # warm: the first calls still grow the memory pools (16-40 ms of device time instead of 9);
        # the result stays bound like in the timed loop, so the second set of page-locked result arrays
        # (the previous result is still alive when the next call returns) is allocated here, not there
        eres = hb.run_variant(host, stream, e2e_cfg, device=local_rank)
    e2e_steps = max(1, min(args.e2e_steps, args.steps))
    t0 = time.perf_counter()
    e2e_each = []
    for _ in range(e2e_steps):
        t1 = time.perf_counter()
        eres = hb.run_variant(host, stream, e2e_cfg, device=local_rank)
        e2e_each.append(round((time.perf_counter() - t1) * 1e3, 2))
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    d2h = int(eres.matching.matched_edges.nbytes + eres.report.matched_round.nbytes + 8 * eres.report.rounds)
    assert np.array_equal(eres.matching.matched_edges, res.matching.matched_edges)
    e2e = {"value": kappa / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(eres.report.h2d_bytes),
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3, "steps": e2e_steps, "warmup": 3,
           "ms_each": e2e_each,
           "host_input_bytes": int(h2d),
           "call": "hlm_b200_match_host (host scan/pack of offsets+weights || pin upload, loader kernels, matching, "
                   "result copy), pinned host CSR"}
    del host

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64 keys (f64 weights, u32 ids)",
            "data": "synthetic",
            "config": {"workload": wl["desc"], "pins": kappa, "edges": m, "vertices": n, "variant": "crcw",
                       "loop": "CUDA-graph WHILE", "rounds": rep.rounds, "matched": int(len(res.matching.matched_edges)),
                       "l2_policy": "inputs larger than L2 (pins %.1f GB); no flush" % (kappa * 4 / 1e9),
                       "device_ms_per_step_lib_events": float(np.mean(dev_ms)),
                       "matched_per_round": rep.matched_per_round_count},
            "clocks": clocks, "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline}
    if not args.no_cpu:
        try:
            cb_out, _, _ = cpu_baseline(wl)
            line["cpu_baseline"] = cb_out
        except Exception as exc:  # the checker is optional at bench time, the GPU numbers are not
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                                    "sample": f"failed: {exc}"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
