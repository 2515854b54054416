"""Edge-partitioned matching across GPUs (BASELINE config 5).

One process per GPU holds a contiguous block of edge rows (global edge ids) and the incidence lists of
its own edges; per-vertex state is replicated.  The round loop, the collectives (NCCL, bound by the
library at run time) and the tie handling all live inside libhlm_b200.so behind ONE call,
hlm_b200_match_sharded (csrc/hlm_shard.inc has the protocol).  Per round the ranks combine

    lkey[L_r]  uint64  all-reduce(max)   local maxima of the L_r still-live vertices   (8 L_r bytes)
    covered    uint32  all-reduce(sum)   newly covered vertices + 8 statistics words    (n / 8 bytes;
                                         bits are disjoint over ranks, so the sum is an OR)
    alive      uint32  all-reduce(sum)   4 words: alive edges (termination)

and the host waits for the device once per round.  The result is identical for every rank count (the
reference's invariant "independent of workers", test_par.cpp:32-55): priorities use global edge ids,
and a vertex whose maximum weight sits on two ranks sends the round through the reference comparator
level by level (tie hash, then id), each level all-reduced.

Python here is plumbing only: it makes the communicator (torch.distributed carries the 128-byte NCCL
id to the other ranks) and marshals the call.  Several shards handed over by ONE process and sitting
on one GPU are "virtual ranks": the same kernels and the same loop, which is how the path is tested
on a single B200.
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
                  WeightStream, WorkCounters, _borrow, _raise, _take)

def shard_bounds(num_edges: int, world: int, rank: int):
    """Block partition of the edge ids: rank r owns [begin, begin + count)."""
    per = (num_edges + world - 1) // world
    begin = min(num_edges, rank * per)
    return begin, min(num_edges, begin + per) - begin


class Communicator:
    """One rank of the NCCL communicator the library's round driver uses (hlm_b200_comm).  The 128-byte
    unique id is made by rank 0 and shipped to the others by whatever the caller has -- here a
    torch.distributed broadcast; the data path itself never goes through torch."""

    def __init__(self, handle, rank: int, world: int):
        self._h, self.rank, self.world = handle, rank, world

    @staticmethod
    def exchange_unique_id(dist, make_id, group=None) -> bytes:
        """rank 0: make_id() -> 128 bytes; everyone: the same bytes (any backend)."""
        import torch

        rank = dist.get_rank(group)
        dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        buf = torch.zeros(_lib.UNIQUE_ID_BYTES, dtype=torch.uint8, device=dev)
        if rank == 0:
            raw = make_id()
            assert len(raw) == _lib.UNIQUE_ID_BYTES
            buf.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
        dist.broadcast(buf, src=0, group=group)
        return bytes(buf.cpu().numpy().tobytes())

    @classmethod
    def from_torch(cls, dist, device: int, group=None) -> "Communicator":
        lib = _lib.load_library()

        def make_id():
            raw = (C.c_uint8 * _lib.UNIQUE_ID_BYTES)()
            st = lib.hlm_b200_comm_unique_id(raw)
            if st != _lib.OK:
                _raise(st, "hlm_b200_comm_unique_id")
            return bytes(raw)

        uid = cls.exchange_unique_id(dist, make_id, group)
        return cls.create(uid, dist.get_rank(group), dist.get_world_size(group), device)

    @classmethod
    def create(cls, uid: Optional[bytes], rank: int, world: int, device: int) -> "Communicator":
        lib = _lib.load_library()
        out = C.c_void_p()
        raw = (C.c_uint8 * _lib.UNIQUE_ID_BYTES).from_buffer_copy(uid) if uid is not None else None
        st = lib.hlm_b200_comm_create(raw, rank, world, device, C.byref(out))
        if st != _lib.OK:
            _raise(st, "hlm_b200_comm_create")
        return cls(out.value, rank, world)

    def nccl_version(self) -> int:
        v = C.c_int(0)
        _lib.load_library().hlm_b200_comm_info(self._h, None, None, None, C.byref(v))
        return int(v.value)

    def destroy(self):
        if self._h:
            _lib.load_library().hlm_b200_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class _ShardResults:
    """Keeps the hlm_b200_result array of a sharded call alive while numpy views of it exist."""

    def __init__(self, results, rep):
        self.results, self.rep = results, rep

    def __del__(self):
        try:
            lib = _lib.load_library()
            for r in self.results:
                lib.hlm_b200_result_free(C.byref(r))
            lib.hlm_b200_shard_report_free(C.byref(self.rep))
        except Exception:
            pass


def match_sharded(shards: List[DeviceHypergraph], stream: WeightStream, cfg: Optional[ParallelConfig] = None,
                  comm: Optional[Communicator] = None):
    """hlm_b200_match_sharded: the round loop, the collectives and the tie handling run inside the library.
    Returns (MatchResult over the LOCAL slices concatenated -- global ids, global rounds / per-round
    counts / total_weight --, shard report as a dict)."""
    cfg = cfg or ParallelConfig()
    lib = _lib.load_library()
    k = len(shards)
    handles = (C.c_void_p * k)(*[s._h for s in shards])
    results = (_lib.Result * k)()
    rep = _lib.ShardReport()
    cs, cc = stream._c(), cfg._c()
    st = lib.hlm_b200_match_sharded(handles, k, comm._h if comm else None, C.byref(cs), C.byref(cc), results,
                                    C.byref(rep))
    owner = _ShardResults(results, rep)  # frees the C results when the last view of them is gone
    if st not in (_lib.OK, _lib.ERR_ROUND_LIMIT):
        _raise(st, "hlm_b200_match_sharded")
    rounds = int(rep.rounds)
    # views of the library's page-locked result arrays: no copy for one shard, one concatenation otherwise
    ids = [_borrow(owner, r.matched_edges, r.num_matched, C.c_uint32, np.uint32) for r in results]
    rnd = [_borrow(owner, r.matched_round, r.num_matched, C.c_uint16, np.uint16) for r in results]
    matched = ids[0] if k == 1 else np.concatenate(ids)
    round_of = rnd[0] if k == 1 else np.concatenate(rnd)
    prm = _take(results[0].per_round_matched, rounds, np.uint32).tolist()
    prd = _take(results[0].per_round_deactivated, rounds, np.uint32).tolist()
    report = dict(rounds=rounds, num_local_shards=int(rep.num_local_shards), num_processes=int(rep.num_processes),
                  tie_redo_rounds=int(rep.tie_redo_rounds), host_syncs=int(rep.host_syncs),
                  kernel_launches=int(rep.kernel_launches), nccl_calls=int(rep.nccl_calls),
                  num_edges_global=int(rep.num_edges_global), collective_bytes=int(rep.collective_bytes),
                  collective_bytes_per_round=_take(rep.collective_bytes_per_round, rounds, np.uint64).tolist(),
                  live_vertices_per_round=_take(rep.live_vertices_per_round, rounds, np.uint32).tolist())
    matching = Matching(matched, float(results[0].total_weight), rounds, prm)
    rr = RunReport(rounds, prm, prd, round_of,
                   WorkCounters(rounds, sum(int(r.total_edge_visits) for r in results),
                                sum(int(r.total_pin_visits) for r in results)),
                   float(results[0].wall_time_ms), 0, max(float(r.device_ms) for r in results), 0,
                   int(rep.tie_redo_rounds), int(rep.kernel_launches), 0, matched)
    if st == _lib.ERR_ROUND_LIMIT:
        raise RoundLimitError(matching, rr)
    return MatchResult(matching, rr), report


def generate_shards(family: str, world: int, device: int = 0, **spec) -> List[DeviceHypergraph]:
    """k edge shards of one synthetic instance on ONE GPU ("virtual ranks")."""
    out = []
    for r in range(world):
        b, k = shard_bounds(spec["m"], world, r)
        if k:
            out.append(DeviceHypergraph.generate(family, edge_begin=b, m_local=k, device=device, **spec))
    return out


def upload_shards(h, world: int, device: int = 0, only_rank: Optional[int] = None) -> List[DeviceHypergraph]:
    """The edge rows of a host Hypergraph cut into `world` blocks, each loaded as a shard on `device`
    (only_rank: just that rank's block -- one process per rank)."""
    lib = _lib.load_library()
    out = []
    eo = np.ascontiguousarray(h.edge_offsets, dtype=np.uint64)
    pins = np.ascontiguousarray(h.edge_members, dtype=np.uint32)
    base = np.ascontiguousarray(h.base_weights, dtype=np.float64)
    for r in (range(world) if only_rank is None else [only_rank]):
        b, k = shard_bounds(h.num_edges, world, r)
        if not k:
            continue
        off = np.ascontiguousarray(eo[b:b + k + 1] - eo[b])
        rows = pins[int(eo[b]):int(eo[b + k])]
        view = _lib.CsrView(h.num_vertices, k, None, None, off.ctypes.data, rows.ctypes.data if rows.size else None,
                            base[b:b + k].ctypes.data)
        handle = C.c_void_p()
        st = lib.hlm_b200_graph_upload_shard(C.byref(view), b, device, C.byref(handle))
        if st != _lib.OK:
            _raise(st, "hlm_b200_graph_upload_shard")
        out.append(DeviceHypergraph(handle.value))
    return out


def bench_main(args, wl, rank, world, local_rank, dist, extras=None):
    """bench.py --gpus N (N > 1, or HLM_BENCH_FORCE_MG=1 on one GPU): config 5 shape, weak scaling -- every
    rank owns 250 M edges of an 8-uniform instance with n = 125 M * N vertices (N = 8 is BASELINE config 5
    exactly).  One call of hlm_b200_match_sharded per step."""
    import torch

    per_rank_m = int(os.environ.get("HLM_BENCH_MG_EDGES", 250_000_000))
    per_rank_n = int(os.environ.get("HLM_BENCH_MG_VERTICES", 125_000_000))
    m, n, d = per_rank_m * world, per_rank_n * world, 8
    b, k = shard_bounds(m, world, rank)
    g = DeviceHypergraph.generate("uniform", n=n, m=m, d=d, seed=1, edge_begin=b, m_local=k, device=local_rank)
    comm = Communicator.from_torch(dist, local_rank)
    tstream = torch.cuda.Stream()
    g.set_stream(tstream.cuda_stream)
    stream = WeightStream()
    cfg = ParallelConfig()
    extras = extras or {}
    sampler = extras.get("sampler")
    if sampler:
        sampler.start()  # before the warm-up: nvidia-smi needs a moment before its first line
    for _ in range(max(3, args.warmup)):
        res, rep = match_sharded([g], stream, cfg, comm)
    dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.begin()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    ev0.record(tstream)
    for _ in range(args.steps):
        res, rep = match_sharded([g], stream, cfg, comm)
        launches += rep["kernel_launches"]
    ev1.record(tstream)
    torch.cuda.synchronize()
    ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
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
            roofline = {"bound": "hbm", "kernel": "whole job (vertex-owned sweeps + candidate checks + collectives), all ranks",
                        "achieved": achieved, "peak": peak, "peak_source": extras["peak_src"] + f" x {world} GPUs",
                        "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                        "algorithmic_bytes": total_bytes}
        line = {"metric": "pins_per_sec_to_maximal_matching", "value": value, "unit": "pins/s", "n_gpus": world,
                "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": total_ms / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "u64 keys (f64 weights, u32 ids)", "data": "synthetic",
                "config": {"workload": f"config 5 shape: 8-uniform, n={n}, m={m} edge-partitioned over {world} GPUs "
                                       f"({per_rank_m} edges per GPU), unit weights, default stream",
                           "pins": m * d, "rounds": res.report.rounds, "matched": int(sum(res.report.matched_per_round_count)),
                           "driver": "hlm_b200_match_sharded (C++ round loop, NCCL %d bound by dlopen)" % comm.nccl_version(),
                           "collectives_per_round": "all-reduce(max) uint64[live vertices] + all-reduce(sum) uint32[n/32 + 8] "
                                                    "+ all-reduce(sum) uint32[4]",
                           "collective_bytes_per_round": rep["collective_bytes_per_round"],
                           "live_vertices_per_round": rep["live_vertices_per_round"],
                           "host_syncs_per_step": rep["host_syncs"], "nccl_calls_per_step": rep["nccl_calls"],
                           "l2_policy": "inputs larger than L2; no flush"},
                "gpu_launches": int(launches),
                "clocks": clocks, "roofline": roofline,
                "cpu_baseline": {"value": None, "unit": "pins/s", "cores": 0, "kind": "unavailable",
                                 "sample": "N > 1: the CPU baseline is reported by the N = 1 run (config 5 does not "
                                           "fit host memory)"},
                "e2e": {"value": value, "unit": "pins/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": int(res.matching.matched_edges.nbytes * 1.5),
                        "note": "instance generated on the devices (16 G pins do not fit host memory); the result "
                                "slices are copied to the host inside the timed region"}}
        emit = extras.get("emit") or (lambda text: print(text, flush=True))
        emit(json.dumps(line))
    dist.barrier()
    comm.destroy()
