"""Host-side mirror of the reference's matching API (proj/include/hlm/), over the C-ABI.

Same names, argument meaning and error behaviour as the reference:

* ``Hypergraph``      -- hypergraph.hpp:19-27 (five arrays, numpy)
* ``WeightStream``    -- weight_stream.hpp:56-61
* ``ParallelConfig``  -- local_max_par.hpp:36-42 (``workers`` / ``grain`` accepted and ignored)
* ``run_variant`` / ``local_max_crcw`` / ``local_max_crew`` -- local_max_par.hpp:586,190,258
* ``verify_matching`` -- exact.hpp:115-140
* ``InputError`` / ``RoundLimitError`` -- common.hpp:18, matching.hpp:77-85

All work is done by libhlm_b200.so on the GPU; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib

GENERATOR_KINDS = {"xorshift": 0, "park_miller": 1, "splitmix": 2}
WEIGHT_MODES = {"perturb_base": 0, "replace_uniform": 1}
VARIANTS = {"seq": 0, "crcw": 1, "crew": 2, "work_optimal": 3, "opt": 3, "greedy": 4,
            "auto": 5}  # auto: B200 extension -- crcw to the caller, engine chosen by the library
LOOP_MODES = {"auto": 0, "host": 1, "graph": 2}
TIE_MODES = {"auto": 0, "exact": 1}
SYN_FAMILIES = {"uniform": 0, "rmat": 1, "powerlaw": 2, "netlist": 3}


class InputError(ValueError):
    """hlm::input_error (common.hpp:18)."""


class RoundLimitError(RuntimeError):
    """hlm::round_limit_error (matching.hpp:77-85): carries the partial matching and report."""

    def __init__(self, partial: "Matching", report: "RunReport"):
        super().__init__(f"round limit exceeded with {report.rounds} rounds used")
        self.partial = partial
        self.report = report


class DeviceError(RuntimeError):
    """CUDA failure or no device: the library has no CPU fallback."""


@dataclass
class Hypergraph:
    num_vertices: int
    num_edges: int
    vertex_offsets: Optional[np.ndarray]
    vertex_incidence: Optional[np.ndarray]
    edge_offsets: np.ndarray
    edge_members: np.ndarray
    base_weights: np.ndarray

    def pin_count(self) -> int:
        return int(self.edge_members.shape[0])


@dataclass
class WeightStream:
    seed: int = 1
    kind: str = "xorshift"
    mode: str = "perturb_base"
    noise_low: float = 0.0
    noise_high: float = 100.0

    def _c(self) -> _lib.Stream:
        kind = GENERATOR_KINDS[self.kind] if isinstance(self.kind, str) else int(self.kind)
        mode = WEIGHT_MODES[self.mode] if isinstance(self.mode, str) else int(self.mode)
        return _lib.Stream(self.seed & 0xFFFFFFFFFFFFFFFF, kind, mode, self.noise_low, self.noise_high)


@dataclass
class ParallelConfig:
    workers: int = 0          # ignored: the device decides its own parallelism
    variant: str = "crcw"
    grain: int = 1024         # ignored
    max_rounds: int = 0
    assert_exclusive_writes: bool = False  # see DESIGN.md (compute-sanitizer racecheck)
    loop_mode: str = "auto"   # B200 extension: "host" | "graph"
    tie_mode: str = "auto"    # B200 extension: "exact" forces the three-level comparator
    want_round_of: bool = True
    kernel_times: bool = False  # B200 extension (host loop): CUDA-event time of each round kernel
    num_gpus: int = 0         # B200 extension (run_variant with host arrays): edge blocks over k devices

    def _c(self) -> _lib.Config:
        if isinstance(self.variant, str):
            if self.variant not in VARIANTS:
                raise InputError("unknown variant")  # local_max_par.hpp:615
            variant = VARIANTS[self.variant]
        else:
            variant = int(self.variant)
        flags = (0 if self.want_round_of else 1) | (2 if self.kernel_times else 0)
        return _lib.Config(variant, self.max_rounds, LOOP_MODES[self.loop_mode], TIE_MODES[self.tie_mode], flags,
                           int(self.num_gpus))


@dataclass
class Matching:
    matched_edges: np.ndarray
    total_weight: float = 0.0
    rounds_used: int = 0
    per_round_matched: List[int] = field(default_factory=list)


@dataclass
class WorkCounters:
    rounds: int = 0
    total_edge_visits: int = 0
    total_pin_visits: int = 0
    prefix_sum_invocations: int = 0
    compactions: int = 0


@dataclass
class RunReport:
    rounds: int = 0
    matched_per_round_count: List[int] = field(default_factory=list)
    deactivated_per_round: List[int] = field(default_factory=list)
    matched_round: Optional[np.ndarray] = None   # round of matched_edges[i]; see matched_per_round
    work: WorkCounters = field(default_factory=WorkCounters)
    wall_time_ms: float = 0.0
    write_conflicts: int = 0
    # B200 extensions
    device_ms: float = 0.0
    device_edge_visits: int = 0
    tie_redo_rounds: int = 0
    kernel_launches: int = 0
    graph_launches: int = 0
    _matched_edges: Optional[np.ndarray] = None
    round_filter_ms: Optional[List[float]] = None
    round_check_ms: Optional[List[float]] = None
    h2d_bytes: int = 0  # run_variant (host arrays in): bytes the loader moved host -> device
    engine: str = ""    # which kernels ran: "crcw" | "vertex-owned" | "vertex-owned, crcw from round k" | "sharded"
    engine_switch_round: int = 0

    @property
    def matched_per_round(self) -> List[np.ndarray]:
        """RunReport::matched_per_round (matching.hpp:39): ascending ids per round."""
        if self.matched_round is None:
            raise ValueError("run with want_round_of=True to get per-round id lists")
        return [self._matched_edges[self.matched_round == r + 1] for r in range(self.rounds)]


@dataclass
class MatchResult:
    matching: Matching
    report: RunReport


@dataclass
class VerificationReport:
    disjoint: bool
    maximal: bool
    weight: float

    def valid(self) -> bool:
        return self.disjoint and self.maximal


def _raise(status: int, what: str):
    msg = f"{what}: {_lib.last_error()}"
    if status == _lib.ERR_INPUT:
        raise InputError(msg)
    if status == _lib.ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if status == _lib.ERR_NOMEM:
        raise MemoryError(msg)
    raise DeviceError(msg)  # ERR_CUDA, ERR_NCCL


def _take(ptr, count, dtype):
    if count == 0 or not ptr:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(int(count),)).astype(dtype, copy=True)


class _ResultOwner:
    """Keeps an hlm_b200_result alive while numpy views of its arrays exist (no copy of the
    matched ids: they stay in the library's page-locked result buffers until garbage-collected)."""

    def __init__(self, res: _lib.Result):
        self.res = res

    def __del__(self):
        try:
            _lib.load_library().hlm_b200_result_free(C.byref(self.res))
        except Exception:
            pass


def _borrow(owner: _ResultOwner, ptr, count, ctype, dtype):
    if count == 0 or not ptr:
        return np.zeros(0, dtype=dtype)
    buf = (ctype * int(count)).from_address(C.addressof(ptr.contents))
    buf._owner = owner  # the view keeps the buffer object, the buffer object keeps the result
    return np.frombuffer(buf, dtype=dtype)


def _convert(status: int, res: _lib.Result) -> MatchResult:
    owner = _ResultOwner(res)
    if status not in (_lib.OK, _lib.ERR_ROUND_LIMIT):
        _raise(status, "hlm_b200_match")
    matched = _borrow(owner, res.matched_edges, res.num_matched, C.c_uint32, np.uint32)
    round_of = _borrow(owner, res.matched_round, res.num_matched, C.c_uint16, np.uint16) if res.matched_round else None
    prm = _take(res.per_round_matched, res.rounds, np.uint32).tolist()
    prd = _take(res.per_round_deactivated, res.rounds, np.uint32).tolist()
    matching = Matching(matched, float(res.total_weight), int(res.rounds), prm)
    report = RunReport(int(res.rounds), prm, prd, round_of,
                       WorkCounters(int(res.rounds), int(res.total_edge_visits), int(res.total_pin_visits),
                                    int(res.prefix_sum_invocations), int(res.compactions)),
                       float(res.wall_time_ms), int(res.write_conflicts), float(res.device_ms),
                       int(res.device_edge_visits), int(res.tie_redo_rounds), int(res.kernel_launches),
                       int(res.graph_launches), matched,
                       _take(res.round_filter_ms, res.rounds + 1, np.float32).tolist() if res.round_filter_ms else None,
                       _take(res.round_check_ms, res.rounds + 1, np.float32).tolist() if res.round_check_ms else None,
                       int(res.h2d_bytes),
                       {1: "crcw", 2: "vertex-owned", 3: f"vertex-owned, crcw from round {int(res.engine_switch_round)}",
                        4: "sharded"}.get(int(res.engine), ""), int(res.engine_switch_round))
    if status == _lib.ERR_ROUND_LIMIT:
        raise RoundLimitError(matching, report)
    return MatchResult(matching, report)


def _view(h: Hypergraph, keep: list) -> _lib.CsrView:
    def ptr(a, dtype):
        if a is None:
            return None
        arr = np.ascontiguousarray(a, dtype=dtype)
        keep.append(arr)
        return arr.ctypes.data

    return _lib.CsrView(h.num_vertices, h.num_edges, ptr(h.vertex_offsets, np.uint64),
                        ptr(h.vertex_incidence, np.uint32), ptr(h.edge_offsets, np.uint64),
                        ptr(h.edge_members, np.uint32), ptr(h.base_weights, np.float64))


class DeviceHypergraph:
    """An instance resident in HBM (the loader's output).  Reusable across matchings, so a bench
    can time the matching alone with inputs already on the device, as the paper's protocol does
    (PAPER.md:316-319)."""

    def __init__(self, handle: int):
        self._h = handle

    @classmethod
    def upload(cls, h: Hypergraph, device: int = 0) -> "DeviceHypergraph":
        lib = _lib.load_library()
        keep: list = []
        view = _view(h, keep)
        out = C.c_void_p()
        st = lib.hlm_b200_graph_upload(C.byref(view), device, C.byref(out))
        if st != _lib.OK:
            _raise(st, "hlm_b200_graph_upload")
        return cls(out.value)

    @classmethod
    def generate(cls, family: str, n: int = 0, m: int = 0, d: int = 0, scale: int = 0, seed: int = 1,
                 int_weights: bool = False, edge_begin: int = 0, m_local: int = 0,
                 device: int = 0) -> "DeviceHypergraph":
        lib = _lib.load_library()
        spec = _lib.SynSpec(SYN_FAMILIES[family], n, m, d, scale, seed, 1 if int_weights else 0, edge_begin,
                            m_local)
        out = C.c_void_p()
        st = lib.hlm_b200_graph_generate(C.byref(spec), device, C.byref(out))
        if st != _lib.OK:
            _raise(st, "hlm_b200_graph_generate")
        return cls(out.value)

    def info(self) -> _lib.GraphInfo:
        info = _lib.GraphInfo()
        _lib.load_library().hlm_b200_graph_info_get(self._h, C.byref(info))
        return info

    def download(self, with_incidence: bool = False, pinned: bool = False) -> Hypergraph:
        info = self.info()
        n, m, k = info.num_vertices, info.num_edges, info.num_pins

        def buf(count, dtype):
            if pinned:
                import torch

                t = torch.empty(int(count), dtype=getattr(torch, np.dtype(dtype).name), pin_memory=True)
                return t.numpy()
            return np.empty(int(count), dtype=dtype)

        # torch has no uint64/uint32 pinned dtypes in older versions; use same-width ints then view
        def ubuf(count, dtype):
            if pinned:
                signed = {np.dtype(np.uint64): np.int64, np.dtype(np.uint32): np.int32}[np.dtype(dtype)]
                return buf(count, signed).view(dtype)
            return np.empty(int(count), dtype=dtype)

        eoff = ubuf(m + 1, np.uint64)
        pins = ubuf(k, np.uint32)
        base = buf(m, np.float64)
        voff = ubuf(n + 1, np.uint64) if with_incidence else None
        vinc = ubuf(k, np.uint32) if with_incidence else None
        st = _lib.load_library().hlm_b200_graph_download(
            self._h, voff.ctypes.data if with_incidence else None, vinc.ctypes.data if with_incidence else None,
            eoff.ctypes.data, pins.ctypes.data, base.ctypes.data)
        if st != _lib.OK:
            _raise(st, "hlm_b200_graph_download")
        return Hypergraph(n, m, voff, vinc, eoff, pins, base)

    def match(self, stream: WeightStream, cfg: Optional[ParallelConfig] = None) -> MatchResult:
        cfg = cfg or ParallelConfig()
        cs, cc = stream._c(), cfg._c()
        res = _lib.Result()
        st = _lib.load_library().hlm_b200_match(self._h, C.byref(cs), C.byref(cc), C.byref(res))
        return _convert(st, res)

    def verify(self, matched_edges) -> VerificationReport:
        ids = np.ascontiguousarray(matched_edges, dtype=np.uint32)
        dis, mx, w = C.c_int(0), C.c_int(0), C.c_double(0.0)
        st = _lib.load_library().hlm_b200_verify(self._h, ids.ctypes.data if ids.size else None, ids.size,
                                                  C.byref(dis), C.byref(mx), C.byref(w))
        if st != _lib.OK:
            _raise(st, "hlm_b200_verify")
        return VerificationReport(bool(dis.value), bool(mx.value), float(w.value))

    def set_stream(self, cuda_stream: Optional[int]):
        """Run this instance's work on the given cudaStream_t handle (e.g.
        ``torch.cuda.current_stream().cuda_stream``) so the caller's events bracket it."""
        _lib.load_library().hlm_b200_graph_set_stream(self._h, cuda_stream)

    def release(self):
        if self._h:
            _lib.load_library().hlm_b200_graph_release(self._h)
            self._h = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.release()


def run_variant(h: Hypergraph, stream: WeightStream, cfg: Optional[ParallelConfig] = None,
                device: int = 0) -> MatchResult:
    """run_variant (local_max_par.hpp:586): host arrays in, MatchResult out (upload + match)."""
    cfg = cfg or ParallelConfig()
    lib = _lib.load_library()
    keep: list = []
    view = _view(h, keep)
    cs, cc = stream._c(), cfg._c()
    res = _lib.Result()
    st = lib.hlm_b200_match_host(C.byref(view), C.byref(cs), C.byref(cc), device, C.byref(res))
    return _convert(st, res)


def local_max_crcw(h: Hypergraph, stream: WeightStream, cfg: Optional[ParallelConfig] = None) -> MatchResult:
    cfg = cfg or ParallelConfig()
    cfg.variant = "crcw"
    return run_variant(h, stream, cfg)


def local_max_crew(h: Hypergraph, stream: WeightStream, cfg: Optional[ParallelConfig] = None) -> MatchResult:
    cfg = cfg or ParallelConfig()
    cfg.variant = "crew"
    return run_variant(h, stream, cfg)


def verify_matching(h: Hypergraph, m: Matching, device: int = 0) -> VerificationReport:
    """verify_matching (exact.hpp:115-140) on the device."""
    with DeviceHypergraph.upload(h, device) as g:
        return g.verify(m.matched_edges)


def default_max_rounds(num_edges: int) -> int:
    return int(_lib.load_library().hlm_b200_default_max_rounds(num_edges))


def eval_stream(stream: WeightStream, edges, rounds, base=None, device: int = 0):
    """WeightStream::weight / tie_hash evaluated by the device code (bit-exactness tests)."""
    edges = np.ascontiguousarray(edges, dtype=np.uint32)
    rounds = np.ascontiguousarray(rounds, dtype=np.uint32)
    w = np.empty(edges.size, dtype=np.float64)
    t = np.empty(edges.size, dtype=np.uint64)
    b = None
    if base is not None:
        base = np.ascontiguousarray(base, dtype=np.float64)
        b = base.ctypes.data
    cs = stream._c()
    st = _lib.load_library().hlm_b200_eval_stream(C.byref(cs), edges.ctypes.data, rounds.ctypes.data, b, edges.size,
                                                   w.ctypes.data, t.ctypes.data, device)
    if st != _lib.OK:
        _raise(st, "hlm_b200_eval_stream")
    return w, t


# ---- text formats (io.hpp of the reference), parsed / written on the host by the library ----------
DEGREE_ZERO = {"reject": 0, "drop_and_renumber": 1, "drop": 1}


def _take_host_graph(hg: _lib.HostGraph) -> Hypergraph:
    n, m = int(hg.num_vertices), int(hg.num_edges)
    kappa = int(hg.edge_offsets[m]) if m else 0
    try:
        return Hypergraph(n, m, _take(hg.vertex_offsets, n + 1, np.uint64), _take(hg.vertex_incidence, kappa, np.uint32),
                          _take(hg.edge_offsets, m + 1, np.uint64), _take(hg.edge_members, kappa, np.uint32),
                          _take(hg.base_weights, m, np.float64))
    finally:
        _lib.load_library().hlm_b200_host_graph_free(C.byref(hg))


def _parse(fn_name: str, text, degree_zero: str, warnings: Optional[list]) -> Hypergraph:
    data = text.encode() if isinstance(text, str) else bytes(text)
    hg = _lib.HostGraph()
    st = getattr(_lib.load_library(), fn_name)(data, len(data), DEGREE_ZERO[degree_zero], C.byref(hg))
    if st != _lib.OK:
        _raise(st, fn_name)
    if warnings is not None and hg.num_warnings:
        warnings.append("vertex weights present but ignored; matching does not use them")
    return _take_host_graph(hg)


def parse_hgr(text, degree_zero: str = "reject", warnings: Optional[list] = None) -> Hypergraph:
    """parse_hgr (io.hpp:79-137): hMetis .hgr text -> Hypergraph; raises InputError like the reference."""
    return _parse("hlm_b200_parse_hgr", text, degree_zero, warnings)


def parse_metis_graph(text, degree_zero: str = "reject") -> Hypergraph:
    """parse_metis_graph (io.hpp:176-231): METIS graph text -> 2-uniform Hypergraph."""
    return _parse("hlm_b200_parse_metis_graph", text, degree_zero, None)


def generate_random(num_vertices: int, num_edges: int, min_edge_size: int = 2, max_edge_size: int = 3,
                    seed: int = 1) -> Hypergraph:
    """generate_random (generators.hpp:65-93), RandomInstanceSpec's fields and defaults (:56-62)."""
    hg = _lib.HostGraph()
    st = _lib.load_library().hlm_b200_generate_random(num_vertices, num_edges, min_edge_size, max_edge_size,
                                                      seed & 0xFFFFFFFFFFFFFFFF, C.byref(hg))
    if st != _lib.OK:
        _raise(st, "hlm_b200_generate_random")
    return _take_host_graph(hg)


def generate_tight_family(d: int, epsilon: float) -> Hypergraph:
    """generate_tight_family (generators.hpp:37-54)."""
    hg = _lib.HostGraph()
    st = _lib.load_library().hlm_b200_generate_tight_family(d, epsilon, C.byref(hg))
    if st != _lib.OK:
        _raise(st, "hlm_b200_generate_tight_family")
    return _take_host_graph(hg)


def random_weights_1_100(num_edges: int, seed: int) -> np.ndarray:
    """random_weights_1_100 (generators.hpp:96-101)."""
    out = np.empty(num_edges, dtype=np.float64)
    st = _lib.load_library().hlm_b200_random_weights_1_100(num_edges, seed & 0xFFFFFFFFFFFFFFFF,
                                                           out.ctypes.data if num_edges else None)
    if st != _lib.OK:
        _raise(st, "hlm_b200_random_weights_1_100")
    return out


def _text_out(st: int, what: str, ptr: C.c_void_p, length: C.c_size_t) -> str:
    if st != _lib.OK:
        _raise(st, what)
    try:
        return C.string_at(ptr.value, length.value).decode()
    finally:
        _lib.load_library().hlm_b200_text_free(ptr)


def write_hgr(h: Hypergraph) -> str:
    """write_hgr (io.hpp:146-171): weights in shortest round-trip form, integral ones as integers."""
    keep: list = []
    view = _view(h, keep)
    ptr, length = C.c_void_p(), C.c_size_t()
    st = _lib.load_library().hlm_b200_write_hgr(C.byref(view), C.byref(ptr), C.byref(length))
    return _text_out(st, "hlm_b200_write_hgr", ptr, length)


def write_matching(m: Matching) -> str:
    """write_matching (io.hpp:240-247)."""
    ids = np.ascontiguousarray(m.matched_edges, dtype=np.uint32)
    ptr, length = C.c_void_p(), C.c_size_t()
    st = _lib.load_library().hlm_b200_write_matching(ids.ctypes.data if ids.size else None, ids.size,
                                                      float(m.total_weight), int(m.rounds_used), C.byref(ptr),
                                                      C.byref(length))
    return _text_out(st, "hlm_b200_write_matching", ptr, length)


def parse_matching(text) -> np.ndarray:
    """parse_matching (io.hpp:249-257): edge ids, one or more per content line."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    ptr, count = C.c_void_p(), C.c_uint64()
    lib = _lib.load_library()
    st = lib.hlm_b200_parse_matching(data, len(data), C.byref(ptr), C.byref(count))
    if st != _lib.OK:
        _raise(st, "hlm_b200_parse_matching")
    try:
        if count.value == 0:
            return np.zeros(0, dtype=np.uint32)
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint32)), shape=(count.value,)).copy()
    finally:
        lib.hlm_b200_text_free(ptr)


def load_instance_file(path: str, metis: bool = False, degree_zero: str = "reject") -> Hypergraph:
    """load_instance_file (io.hpp:259-264)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as exc:
        raise IOError(f"cannot open instance file {path}") from exc  # hlm::io_error
    return parse_metis_graph(data, degree_zero) if metis else parse_hgr(data, degree_zero)


@dataclass
class CompactResult:
    """CompactResult (local_max_par.hpp:340-344) plus what one compaction adds to the WorkCounters."""
    graph: Hypergraph
    vertex_map: np.ndarray  # old id -> new id or 0xFFFFFFFF
    edge_map: np.ndarray
    work: WorkCounters


def compact(h: Hypergraph, vertex_active, edge_active, device: int = 0) -> CompactResult:
    """compact (local_max_par.hpp:350-454) on the device; needs both CSR sides of `h`."""
    lib = _lib.load_library()
    keep: list = []
    view = _view(h, keep)
    va = np.ascontiguousarray(vertex_active, dtype=np.uint8)
    ea = np.ascontiguousarray(edge_active, dtype=np.uint8)
    if va.size != h.num_vertices or ea.size != h.num_edges:
        raise InputError("activity flag arrays do not match the hypergraph")
    hg, vm, em, wk = _lib.HostGraph(), C.c_void_p(), C.c_void_p(), _lib.CompactWork()
    st = lib.hlm_b200_compact(C.byref(view), va.ctypes.data if va.size else None, ea.ctypes.data if ea.size else None,
                              device, C.byref(hg), C.byref(vm), C.byref(em), C.byref(wk))
    if st != _lib.OK:
        _raise(st, "hlm_b200_compact")
    try:
        vmap = _take(C.cast(vm, C.POINTER(C.c_uint32)), h.num_vertices, np.uint32)
        emap = _take(C.cast(em, C.POINTER(C.c_uint32)), h.num_edges, np.uint32)
    finally:
        lib.hlm_b200_text_free(vm)
        lib.hlm_b200_text_free(em)
    return CompactResult(_take_host_graph(hg), vmap, emap,
                         WorkCounters(0, int(wk.total_edge_visits), int(wk.total_pin_visits),
                                      int(wk.prefix_sum_invocations), int(wk.compactions)))
