"""Edge-partitioned matching across GPUs (BASELINE config 5).

One process per GPU holds a contiguous block of edge rows (global edge ids) plus replicated
per-vertex arrays.  Each round the ranks run the same sm_100a kernels on their shard through the
step-level C-ABI (csrc/hlm_multi.inc) and combine three arrays with collectives:

    vkey[n]  int64   all-reduce(max)   the vertex maxima             (8 n bytes)
    claims   int32   all-reduce(sum)   claimants per vertex, 4 bits  (n / 2 bytes) + 8 words of stats
    dead_new int32   all-reduce(sum)   newly covered vertices        (n / 8 bytes; each bit is set
                                       by exactly one rank because matched edges are disjoint, so
                                       the sum is a bitwise OR -- NCCL has no OR)

The result is identical for every rank count (the reference's invariant "independent of workers",
test_par.cpp:32-55): priorities use global edge ids, and a vertex whose maximum is claimed by two
edges (on the same or on different ranks) sends that round to the exact three-level comparator,
whose levels are all-reduced as well.

`ShardedMatcher` drives a LIST of shards held by this process plus an optional torch.distributed
group: a list of k shards with no group is k "virtual ranks" on one GPU (how the protocol is
tested on a single B200); one shard per process with an NCCL group is the production layout.
Python only orchestrates: every array operation is a CUDA kernel of the library or a collective.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import time
from typing import List, Optional

import numpy as np

from . import _lib
from .api import (DeviceHypergraph, MatchResult, Matching, ParallelConfig, RoundLimitError, RunReport,
                  WeightStream, WorkCounters, _raise, _take)

MG_RUNNING, MG_DONE, MG_ROUND_LIMIT = 0, 1, 2


def shard_bounds(num_edges: int, world: int, rank: int):
    """Block partition of the edge ids: rank r owns [begin, begin + count)."""
    per = (num_edges + world - 1) // world
    begin = min(num_edges, rank * per)
    return begin, min(num_edges, begin + per) - begin


class Collectives:
    """All-reduce over the shards of this process and, if given, a torch.distributed group."""

    def __init__(self, dist=None, group=None):
        self.dist = dist
        self.group = group
        self.bytes_moved = 0

    def _reduce(self, tensors, op_local, op_dist):
        acc = tensors[0]
        if len(tensors) > 1:
            acc = tensors[0].clone()
            for t in tensors[1:]:
                op_local(acc, t)
        if self.dist is not None:
            self.dist.all_reduce(acc, op=op_dist, group=self.group)
            self.bytes_moved += acc.numel() * acc.element_size()
        if len(tensors) > 1 or self.dist is not None:
            for t in tensors:
                if t is not acc:
                    t.copy_(acc)

    def allreduce_max(self, tensors):
        import torch

        self._reduce(tensors, lambda a, b: torch.maximum(a, b, out=a),
                     self.dist.ReduceOp.MAX if self.dist is not None else None)

    def allreduce_sum(self, tensors):
        self._reduce(tensors, lambda a, b: a.add_(b), self.dist.ReduceOp.SUM if self.dist is not None else None)

    def reduce_scalars(self, values: List[float], op: str) -> float:
        """op in {'min', 'max', 'sum'} over the local values and the group."""
        import torch

        local = {"min": min, "max": max, "sum": sum}[op](values)
        if self.dist is None:
            return local
        t = torch.tensor([local], dtype=torch.float64, device="cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu")
        self.dist.all_reduce(t, op={"min": self.dist.ReduceOp.MIN, "max": self.dist.ReduceOp.MAX,
                                    "sum": self.dist.ReduceOp.SUM}[op], group=self.group)
        return float(t.item())

    def chain_weights(self, fold):
        """Ordered fold across ranks: rank k starts from the total of ranks < k (the reference sums
        base weights in ascending edge-id order).  `fold(acc_in) -> acc_out` is this process's part."""
        if self.dist is None:
            return fold(0.0)
        import torch

        rank, world = self.dist.get_rank(self.group), self.dist.get_world_size(self.group)
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        acc = torch.zeros(1, dtype=torch.float64, device=dev)
        out = 0.0
        for k in range(world):
            if rank == k:
                out = fold(float(acc.item()))
                acc[0] = out
            self.dist.broadcast(acc, src=k, group=self.group)
        return float(acc.item())

    def gather_arrays(self, arr: np.ndarray) -> Optional[np.ndarray]:
        """Concatenation of `arr` over ranks in rank order (every rank gets it)."""
        if self.dist is None:
            return arr
        import torch

        world = self.dist.get_world_size(self.group)
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        n = torch.tensor([arr.size], dtype=torch.int64, device=dev)
        sizes = [torch.zeros_like(n) for _ in range(world)]
        self.dist.all_gather(sizes, n, group=self.group)
        sizes = [int(x.item()) for x in sizes]
        cap = max(sizes) if sizes else 0
        buf = torch.zeros(max(cap, 1), dtype=torch.int64, device=dev)
        buf[:arr.size] = torch.from_numpy(arr.astype(np.int64)).to(dev)
        parts = [torch.zeros_like(buf) for _ in range(world)]
        self.dist.all_gather(parts, buf, group=self.group)
        return np.concatenate([p[:s].cpu().numpy() for p, s in zip(parts, sizes)]).astype(arr.dtype)


class LibEngine:
    """The production step engine: one shard on one GPU, driven through the C-ABI."""

    def __init__(self, shard: DeviceHypergraph, stream=None):
        import torch

        self.shard = shard
        self.lib = _lib.load_library()
        info = shard.info()
        self.n = int(info.num_vertices)
        self.m_local = int(info.num_edges)
        self.device = torch.device("cuda", int(info.device))
        self.torch = torch
        self.nw = (self.n + 31) // 32
        self.nc = (self.n + 7) // 8
        words = int(self.lib.hlm_b200_mg_exch_words(self.n))
        with torch.cuda.device(self.device):
            self.vkey = torch.zeros(self.n, dtype=torch.int64, device=self.device)
            self.exch = torch.zeros(words, dtype=torch.int32, device=self.device)
            # all shards of one process share one stream: library kernels, torch element-wise ops
            # and the NCCL collectives are then ordered without host synchronisation
            self.stream = stream if stream is not None else torch.cuda.Stream(device=self.device)
        self.exact = None
        shard.set_stream(self.stream.cuda_stream)

    # views the collectives act on
    def keys(self):
        return self.vkey

    def claims_and_stats(self):
        return self.exch[self.nw:]

    def dead_new(self):
        return self.exch[:self.nw]

    def _ck(self, st, what):
        if st != _lib.OK:
            _raise(st, what)

    def weight_info(self, noise_low: float):
        wi = _lib.WeightInfo()
        self._ck(self.lib.hlm_b200_graph_weight_info(self.shard._h, noise_low, C.byref(wi)), "weight_info")
        return wi.base_min, wi.base_max, int(wi.non_integer), int(wi.num_edges)

    def begin(self, stream: WeightStream, cfg: ParallelConfig, base_min, base_max, non_integer, m_global):
        cs, cc = stream._c(), cfg._c()
        su = _lib.MgSetup(self.vkey.data_ptr(), self.exch.data_ptr(), base_min, base_max, non_integer, m_global)
        self._ck(self.lib.hlm_b200_mg_begin(self.shard._h, C.byref(cs), C.byref(cc), C.byref(su)), "mg_begin")

    def vertex_max(self):
        self._ck(self.lib.hlm_b200_mg_vertex_max(self.shard._h), "mg_vertex_max")

    def claims(self):
        self._ck(self.lib.hlm_b200_mg_claims(self.shard._h), "mg_claims")

    def decide(self):
        act, tie = C.c_uint32(0), C.c_int(0)
        self._ck(self.lib.hlm_b200_mg_decide(self.shard._h, C.byref(act), C.byref(tie)), "mg_decide")
        return int(act.value), bool(tie.value)

    def check_commit(self):
        self._ck(self.lib.hlm_b200_mg_check_commit(self.shard._h), "mg_check_commit")

    def exact_arrays(self):
        if self.exact is None:
            t = self.torch
            with t.cuda.device(self.device):
                self.exact = (t.zeros(self.n, dtype=t.int64, device=self.device),
                              t.zeros(self.n, dtype=t.int64, device=self.device),
                              t.zeros(self.n, dtype=t.int32, device=self.device))
        return self.exact

    def exact_level(self, level: int):
        va, vb, vc = self.exact_arrays()
        self._ck(self.lib.hlm_b200_mg_exact_level(self.shard._h, level, va.data_ptr(), vb.data_ptr(), vc.data_ptr()),
                 "mg_exact_level")

    def end_round(self, global_active: int) -> int:
        status = C.c_int(0)
        self._ck(self.lib.hlm_b200_mg_end_round(self.shard._h, global_active, C.byref(status)), "mg_end_round")
        return int(status.value)

    def finish(self, weight_before: float):
        res = _lib.Result()
        st = self.lib.hlm_b200_mg_finish(self.shard._h, weight_before, C.byref(res))
        if st not in (_lib.OK, _lib.ERR_ROUND_LIMIT):
            _raise(st, "mg_finish")
        out = dict(matched=_take(res.matched_edges, res.num_matched, np.uint32),
                   round_of=_take(res.matched_round, res.num_matched, np.uint16),
                   per_round_matched=_take(res.per_round_matched, res.rounds, np.uint32).astype(np.int64),
                   per_round_deactivated=_take(res.per_round_deactivated, res.rounds, np.uint32).astype(np.int64),
                   rounds=int(res.rounds), total_weight=float(res.total_weight), launches=int(res.kernel_launches),
                   tie_redos=int(res.tie_redo_rounds), limit=st == _lib.ERR_ROUND_LIMIT)
        self.lib.hlm_b200_result_free(C.byref(res))
        return out

    def sync(self):
        self.stream.synchronize()


class ShardedMatcher:
    """run_variant over an edge-partitioned instance.  `engines`: the shards of this process in
    ascending edge-id order; `coll`: how arrays cross shards / ranks."""

    def __init__(self, engines: list, num_edges_global: int, kappa_global: int, coll: Optional[Collectives] = None):
        self.engines = engines
        self.m = int(num_edges_global)
        self.kappa = int(kappa_global)
        self.coll = coll or Collectives()
        self.timings = {}

    def _all(self, name, *args):
        return [getattr(e, name)(*args) for e in self.engines]

    def _sync(self):
        pass  # one stream per process orders everything (see LibEngine.__init__)

    def match(self, stream: WeightStream, cfg: Optional[ParallelConfig] = None, gather: bool = True) -> MatchResult:
        cuda_stream = getattr(self.engines[0], "stream", None)
        if cuda_stream is None:
            return self._match(stream, cfg, gather)
        import torch

        with torch.cuda.stream(cuda_stream):
            return self._match(stream, cfg, gather)

    def _match(self, stream: WeightStream, cfg: Optional[ParallelConfig] = None, gather: bool = True) -> MatchResult:
        cfg = cfg or ParallelConfig()
        t0 = time.perf_counter()
        E, coll = self.engines, self.coll
        # 1. agree on the weight facts that fix the 64-bit key layout
        infos = self._all("weight_info", stream.noise_low)
        live = [i for i in infos if i[3] > 0] or infos
        bmin = coll.reduce_scalars([i[0] for i in live], "min")
        bmax = coll.reduce_scalars([i[1] for i in live], "max")
        nonint = int(coll.reduce_scalars([float(i[2]) for i in infos], "max"))
        self._all("begin", stream, cfg, bmin, bmax, nonint, self.m)
        status, rounds_guard = MG_RUNNING, 0
        t_coll = 0.0
        while status == MG_RUNNING:
            self._all("vertex_max")
            self._sync()
            tc = time.perf_counter()
            coll.allreduce_max([e.keys() for e in E])
            t_coll += time.perf_counter() - tc
            self._all("claims")
            self._sync()
            tc = time.perf_counter()
            coll.allreduce_sum([e.claims_and_stats() for e in E])
            t_coll += time.perf_counter() - tc
            decisions = self._all("decide")
            active, tie = decisions[0]
            assert all(d == decisions[0] for d in decisions), "ranks disagree after the all-reduce"
            if active > 0:
                if tie:
                    self._exact_round()
                else:
                    self._all("check_commit")
                    self._sync()
            tc = time.perf_counter()
            coll.allreduce_sum([e.dead_new() for e in E])
            t_coll += time.perf_counter() - tc
            statuses = self._all("end_round", active)
            status = statuses[0]
            assert all(s == status for s in statuses)
            rounds_guard += 1
            if rounds_guard > 70000:
                raise RuntimeError("round loop did not terminate")
        # 2. assemble: shards are in ascending id order, so concatenation is the sorted result
        parts = []

        def fold(acc):
            for e in E:
                p = e.finish(acc)
                parts.append(p)
                acc = p["total_weight"]
            return acc

        total_weight = coll.chain_weights(fold)
        rounds = parts[0]["rounds"]
        prm = np.sum([p["per_round_matched"] for p in parts], axis=0) if rounds else np.zeros(0, dtype=np.int64)
        prd = np.sum([p["per_round_deactivated"] for p in parts], axis=0) if rounds else np.zeros(0, dtype=np.int64)
        if coll.dist is not None and rounds:
            import torch

            dev = E[0].device if hasattr(E[0], "device") else "cpu"
            t = torch.from_numpy(np.concatenate([prm, prd])).to(dev)
            coll.dist.all_reduce(t, group=coll.group)
            both = t.cpu().numpy()
            prm, prd = both[:rounds], both[rounds:]
        matched = np.concatenate([p["matched"] for p in parts]) if parts else np.zeros(0, dtype=np.uint32)
        round_of = np.concatenate([p["round_of"] for p in parts]) if parts else np.zeros(0, dtype=np.uint16)
        if gather:
            matched = coll.gather_arrays(matched)
            round_of = coll.gather_arrays(round_of)
        wall = (time.perf_counter() - t0) * 1e3
        self.timings = {"wall_ms": wall, "collective_ms": t_coll * 1e3, "collective_bytes": coll.bytes_moved}
        matching = Matching(matched, total_weight, rounds, [int(x) for x in prm])
        report = RunReport(rounds, [int(x) for x in prm], [int(x) for x in prd], round_of,
                           WorkCounters(rounds, 3 * self.m * rounds, 3 * self.kappa * rounds), wall, 0, 0.0, 0,
                           max(p["tie_redos"] for p in parts), sum(p["launches"] for p in parts), 0, matched)
        if any(p["limit"] for p in parts):
            raise RoundLimitError(matching, report)
        return MatchResult(matching, report)

    def _exact_round(self):
        """Three max levels of the reference comparator, each all-reduced (weight_stream.hpp:105-113)."""
        E, coll = self.engines, self.coll
        arrays = [e.exact_arrays() for e in E]
        for va, vb, vc in arrays:
            va.zero_()
            vb.zero_()
            vc.zero_()
        self._all("exact_level", 1)
        self._sync()
        coll.allreduce_max([a[0] for a in arrays])  # weight bits: positive doubles, < 2^63
        self._all("exact_level", 2)
        self._sync()
        sign64 = -(1 << 63)
        for _, vb, _ in arrays:  # unsigned order of the hash == signed order with the top bit flipped
            vb.bitwise_xor_(sign64)
        coll.allreduce_max([a[1] for a in arrays])
        for _, vb, _ in arrays:
            vb.bitwise_xor_(sign64)
        self._all("exact_level", 3)
        self._sync()
        sign32 = -(1 << 31)
        for _, _, vc in arrays:
            vc.bitwise_xor_(sign32)
        coll.allreduce_max([a[2] for a in arrays])
        for _, _, vc in arrays:
            vc.bitwise_xor_(sign32)
        self._all("exact_level", 4)
        self._sync()


def virtual_cluster(family: str, world: int, device: int = 0, **spec) -> ShardedMatcher:
    """k edge shards of one synthetic instance on ONE GPU (no process group): the multi-GPU
    protocol with the collectives replaced by element-wise ops between the shards' buffers."""
    m = spec["m"]
    import torch

    engines, kappa = [], 0
    shared = torch.cuda.Stream(device=torch.device("cuda", device))
    for r in range(world):
        b, k = shard_bounds(m, world, r)
        if k == 0:
            continue
        g = DeviceHypergraph.generate(family, edge_begin=b, m_local=k, device=device, **spec)
        kappa += int(g.info().num_pins)
        engines.append(LibEngine(g, shared))
    return ShardedMatcher(engines, m, kappa, Collectives())


def bench_main(args, wl, rank, world, local_rank, dist, extras=None):
    """bench.py --gpus N (N > 1): config 5 shape, weak scaling -- every rank owns 250 M edges of an
    8-uniform instance with n = 125 M * N vertices (N = 8 is BASELINE config 5 exactly)."""
    import torch

    per_rank_m = int(os.environ.get("HLM_BENCH_MG_EDGES", 250_000_000))
    per_rank_n = int(os.environ.get("HLM_BENCH_MG_VERTICES", 125_000_000))
    m, n, d = per_rank_m * world, per_rank_n * world, 8
    b, k = shard_bounds(m, world, rank)
    g = DeviceHypergraph.generate("uniform", n=n, m=m, d=d, seed=1, edge_begin=b, m_local=k, device=local_rank)
    eng = LibEngine(g)
    coll = Collectives(dist)
    sm = ShardedMatcher([eng], m, m * d, coll)
    stream = WeightStream()
    cfg = ParallelConfig(variant="crcw")
    extras = extras or {}
    sampler = extras.get("sampler")
    if sampler:
        sampler.start()  # before the warm-up: nvidia-smi needs a moment before its first line
    for _ in range(max(3, args.warmup)):
        res = sm.match(stream, cfg, gather=False)
    dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.begin()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(eng.stream):
        ev0.record(eng.stream)
        for _ in range(args.steps):
            res = sm.match(stream, cfg, gather=False)
        ev1.record(eng.stream)
    torch.cuda.synchronize()
    ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    total_ms = float(ms.item())
    clocks = sampler.stop() if sampler else None
    if rank == 0:
        value = m * d * args.steps / (total_ms * 1e-3)
        roofline = None
        if extras.get("algorithmic_bytes"):
            # whole job, all ranks: algorithmic bytes of the rounds over the step time,
            # against N x the measured HBM peak (collective time is inside the step)
            total_bytes, _, _ = extras["algorithmic_bytes"](m * d, m, n, d, res.report.matched_per_round_count,
                                                            res.report.deactivated_per_round)
            achieved = total_bytes / (total_ms / args.steps * 1e-3) / 1e9
            peak = extras["hbm_gbs"] * world
            roofline = {"bound": "hbm", "kernel": "whole job (round sweeps + checks + collectives), all ranks",
                        "achieved": achieved, "peak": peak, "peak_source": extras["peak_src"] + f" x {world} GPUs",
                        "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                        "collective_ms_per_step": sm.timings.get("collective_ms"),
                        "collective_bytes_per_step": sm.timings.get("collective_bytes")}
        line = {"metric": "pins_per_sec_to_maximal_matching", "value": value, "unit": "pins/s", "n_gpus": world,
                "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": total_ms / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "u64 keys (f64 weights, u32 ids)", "data": "synthetic",
                "config": {"workload": f"config 5 shape: 8-uniform, n={n}, m={m} edge-partitioned over {world} GPUs "
                                       f"({per_rank_m} edges per GPU), unit weights, default stream",
                           "pins": m * d, "rounds": res.report.rounds, "matched": int(sum(res.report.matched_per_round_count)),
                           "collectives_per_round": "all-reduce(max) int64[n] + all-reduce(sum) int32[n/2] + int32[n/8]",
                           "collective_ms_last_step": sm.timings.get("collective_ms"),
                           "l2_policy": "inputs larger than L2; no flush"},
                "gpu_launches": int(res.report.kernel_launches) * args.steps,
                "clocks": clocks, "roofline": roofline,
                "cpu_baseline": {"value": None, "unit": "pins/s", "cores": 0, "kind": "unavailable",
                                 "sample": "N > 1: the CPU baseline is reported by the N = 1 run (config 5 does not "
                                           "fit host memory)"},
                "e2e": {"value": value, "unit": "pins/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                        "note": "instance generated on the devices (16 G pins do not fit host memory)"}}
        emit = extras.get("emit") or (lambda text: print(text, flush=True))
        emit(json.dumps(line))
    dist.barrier()
