"""ctypes loader for the test-only CPU checker (oracle/).

TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, bench.py's cpu_baseline /
``--impl reference`` legs and ``__graft_entry__.smoke()`` may import this module.
The product package (paper_2602_22976_b200) never does.

Two back ends with the same Python surface:

* ``Oracle("port")``       -- oracle/_build/libhlm_oracle.so, the plain-C restatement
  (hlm_oracle.c), always available (built by ``make -C oracle``).
* ``Oracle("reference")``  -- oracle/_ref/libhlm_ref.so, the UNMODIFIED reference headers
  compiled by ``make -C oracle ref`` in the build container (prebuilt file travels to the GPU
  box; it cannot be rebuilt there because /root/reference does not exist there).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(_HERE, "_build", "libhlm_oracle.so")
REF_LIB = os.path.join(_HERE, "_ref", "libhlm_ref.so")

GEN_XORSHIFT, GEN_PARK_MILLER, GEN_SPLITMIX = 0, 1, 2
MODE_PERTURB_BASE, MODE_REPLACE_UNIFORM = 0, 1
OK, INPUT_ERROR, ROUND_LIMIT = 0, 1, 2
VARIANT_SEQ, VARIANT_CRCW, VARIANT_CREW, VARIANT_WORK_OPTIMAL, VARIANT_GREEDY = 0, 1, 2, 3, 4
SYN_UNIFORM, SYN_RMAT, SYN_POWERLAW, SYN_NETLIST = 0, 1, 2, 3


class CStream(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("kind", C.c_int32), ("mode", C.c_int32),
                ("noise_low", C.c_double), ("noise_high", C.c_double)]


class CGraph(C.Structure):
    _fields_ = [("n", C.c_uint32), ("m", C.c_uint32),
                ("vertex_offsets", C.c_void_p), ("vertex_incidence", C.c_void_p),
                ("edge_offsets", C.c_void_p), ("edge_members", C.c_void_p),
                ("base_weights", C.c_void_p)]


class COwnedGraph(C.Structure):
    _fields_ = [("n", C.c_uint32), ("m", C.c_uint32), ("kappa", C.c_uint64),
                ("vertex_offsets", C.POINTER(C.c_uint64)), ("vertex_incidence", C.POINTER(C.c_uint32)),
                ("edge_offsets", C.POINTER(C.c_uint64)), ("edge_members", C.POINTER(C.c_uint32)),
                ("base_weights", C.POINTER(C.c_double))]


class CResult(C.Structure):
    _fields_ = [("matched_edges", C.POINTER(C.c_uint32)), ("matched_round", C.POINTER(C.c_uint32)),
                ("num_matched", C.c_uint64), ("total_weight", C.c_double), ("rounds", C.c_uint32),
                ("per_round_matched", C.POINTER(C.c_uint32)),
                ("per_round_deactivated", C.POINTER(C.c_uint32)),
                ("edge_visits", C.c_uint64), ("pin_visits", C.c_uint64), ("wall_ms", C.c_double)]


class CSynSpec(C.Structure):
    _fields_ = [("family", C.c_int32), ("n", C.c_uint32), ("m", C.c_uint32), ("d", C.c_uint32),
                ("scale", C.c_uint32), ("seed", C.c_uint64), ("int_weights", C.c_int32)]


@dataclass
class Stream:
    """hlm::WeightStream (weight_stream.hpp:56-61)."""
    seed: int = 1
    kind: int = GEN_XORSHIFT
    mode: int = MODE_PERTURB_BASE
    noise_low: float = 0.0
    noise_high: float = 100.0

    def c(self) -> CStream:
        return CStream(self.seed & 0xFFFFFFFFFFFFFFFF, self.kind, self.mode, self.noise_low,
                       self.noise_high)


@dataclass
class Graph:
    """hlm::Hypergraph (hypergraph.hpp:19-27) as numpy arrays."""
    n: int
    m: int
    vertex_offsets: np.ndarray
    vertex_incidence: np.ndarray
    edge_offsets: np.ndarray
    edge_members: np.ndarray
    base_weights: np.ndarray

    @property
    def kappa(self) -> int:
        return int(self.edge_members.shape[0])

    def c(self) -> CGraph:
        return CGraph(self.n, self.m, self.vertex_offsets.ctypes.data, self.vertex_incidence.ctypes.data,
                      self.edge_offsets.ctypes.data, self.edge_members.ctypes.data,
                      self.base_weights.ctypes.data)


@dataclass
class Result:
    status: int
    matched_edges: np.ndarray
    matched_round: np.ndarray
    total_weight: float
    rounds: int
    per_round_matched: list
    per_round_deactivated: list
    edge_visits: int = 0
    pin_visits: int = 0
    wall_ms: float = 0.0
    extra: dict = field(default_factory=dict)

    def matched_per_round(self):
        return [self.matched_edges[self.matched_round == r + 1] for r in range(self.rounds)]


def fnv1a_ids(ids: np.ndarray) -> int:
    """FNV-1a-64 over the little-endian bytes of each uint32 id."""
    arr = np.ascontiguousarray(ids, dtype="<u4")
    lib = _load(PORT_LIB, build=True)
    lib.orc_fnv1a_ids.restype = C.c_uint64
    lib.orc_fnv1a_ids.argtypes = [C.c_void_p, C.c_uint64]
    return int(lib.orc_fnv1a_ids(arr.ctypes.data if arr.size else None, arr.size))


_LIBS: dict = {}


def build_port() -> str:
    subprocess.run(["make", "-C", _HERE, "-s"], check=True, stdout=subprocess.DEVNULL)
    return PORT_LIB


def build_reference(reference_root: str = "/root/reference") -> str | None:
    """Compile oracle/_ref from the reference tree if (and only if) that tree is present."""
    if not os.path.isdir(os.path.join(reference_root, "proj", "include", "hlm")):
        return REF_LIB if os.path.exists(REF_LIB) else None
    subprocess.run(["make", "-C", _HERE, "-s", "ref", f"REFERENCE={reference_root}"], check=True,
                   stdout=subprocess.DEVNULL)
    return REF_LIB


def _load(path: str, build: bool = False):
    if path in _LIBS:
        return _LIBS[path]
    if build and path == PORT_LIB:
        src = os.path.join(_HERE, "hlm_oracle.c")
        if (not os.path.exists(path)) or os.path.getmtime(path) < os.path.getmtime(src):
            build_port()
    lib = C.CDLL(path)
    _LIBS[path] = lib
    return lib


def reference_available() -> bool:
    return os.path.exists(REF_LIB)


def _take(ptr, count, dtype):
    if count == 0 or not ptr:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(int(count),)).astype(dtype, copy=True)


def _own_graph(og: COwnedGraph) -> Graph:
    n, m, k = og.n, og.m, og.kappa
    return Graph(n, m, _take(og.vertex_offsets, n + 1, np.uint64), _take(og.vertex_incidence, k, np.uint32),
                 _take(og.edge_offsets, m + 1, np.uint64), _take(og.edge_members, k, np.uint32),
                 _take(og.base_weights, m, np.float64))


def _own_result(status: int, r: CResult) -> Result:
    return Result(status, _take(r.matched_edges, r.num_matched, np.uint32),
                  _take(r.matched_round, r.num_matched, np.uint32), float(r.total_weight), int(r.rounds),
                  _take(r.per_round_matched, r.rounds, np.uint32).tolist(),
                  _take(r.per_round_deactivated, r.rounds, np.uint32).tolist(),
                  int(r.edge_visits), int(r.pin_visits), float(r.wall_ms))


class Oracle:
    def __init__(self, kind: str = "port"):
        assert kind in ("port", "reference")
        self.kind = kind
        if kind == "port":
            self.lib = _load(PORT_LIB, build=True)
            self.p = "orc_"
        else:
            if not os.path.exists(REF_LIB):
                raise FileNotFoundError(f"{REF_LIB} missing: run `make -C oracle ref` where /root/reference exists")
            self.lib = _load(REF_LIB)
            self.p = "ref_"
        self._port = _load(PORT_LIB, build=True)

    def _fn(self, name, restype=C.c_int, argtypes=None):
        f = getattr(self.lib, self.p + name)
        f.restype = restype
        if argtypes is not None:
            f.argtypes = argtypes
        return f

    # ---- priority stream ----
    def eval_stream(self, stream: Stream, edges, rounds, base=None):
        edges = np.ascontiguousarray(edges, dtype=np.uint32)
        rounds = np.ascontiguousarray(rounds, dtype=np.uint32)
        cnt = edges.size
        w = np.empty(cnt, dtype=np.float64)
        t = np.empty(cnt, dtype=np.uint64)
        bptr = None
        if base is not None:
            base = np.ascontiguousarray(base, dtype=np.float64)
            bptr = base.ctypes.data
        cs = stream.c()
        f = self._fn("eval_stream", None, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                           C.c_void_p, C.c_void_p])
        f(C.addressof(cs), edges.ctypes.data, rounds.ctypes.data, bptr, cnt, w.ctypes.data, t.ctypes.data)
        return w, t

    def tie_break(self, wa, ida, wb, idb, stream: Stream, rnd: int) -> int:
        cs = stream.c()
        f = self._fn("tie_break", C.c_int, [C.c_double, C.c_uint32, C.c_double, C.c_uint32, C.c_void_p, C.c_uint32])
        return int(f(wa, ida, wb, idb, C.addressof(cs), rnd))

    def default_max_rounds(self, m: int) -> int:
        return int(self._fn("default_max_rounds", C.c_uint32, [C.c_uint32])(m))

    # ---- instance sources ----
    def generate_random(self, n, m, min_size, max_size, seed) -> Graph:
        og = COwnedGraph()
        rc = self._fn("generate_random", C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                                    C.c_void_p])(n, m, min_size, max_size, seed, C.addressof(og))
        if rc != OK:
            raise ValueError("generate_random: input error")
        g = _own_graph(og)
        self._fn("free_graph", None, [C.c_void_p])(C.addressof(og))
        return g

    def random_weights_1_100(self, m, seed) -> np.ndarray:
        out = np.empty(m, dtype=np.float64)
        self._fn("random_weights_1_100", None, [C.c_uint32, C.c_uint64, C.c_void_p])(m, seed, out.ctypes.data)
        return out

    def tight_family(self, d, eps) -> Graph:
        og = COwnedGraph()
        rc = self._fn("tight_family", C.c_int, [C.c_uint32, C.c_double, C.c_void_p])(d, eps, C.addressof(og))
        if rc != OK:
            raise ValueError("tight_family: input error")
        g = _own_graph(og)
        self._fn("free_graph", None, [C.c_void_p])(C.addressof(og))
        return g

    # ---- matcher ----
    def local_max(self, g: Graph, stream: Stream, max_rounds: int = 0, variant: int = VARIANT_SEQ,
                  workers: int = 1) -> Result:
        res = CResult()
        cs = stream.c()
        if self.kind == "port":
            cg = g.c()
            f = self._fn("local_max", C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p])
            rc = f(C.addressof(cg), C.addressof(cs), max_rounds, C.addressof(res))
            out = _own_result(rc, res)
            self._fn("free_result", None, [C.c_void_p])(C.addressof(res))
            return out
        h = self.graph_handle(g)
        try:
            return self.run_handle(h, stream, variant, workers, max_rounds)
        finally:
            self.graph_release(h)

    # reference only: keep the hlm::Hypergraph alive across timed runs
    def graph_handle(self, g: Graph):
        assert self.kind == "reference"
        f = self._fn("graph_create", C.c_void_p, [C.c_uint32, C.c_uint32] + [C.c_void_p] * 5)
        return f(g.n, g.m, g.vertex_offsets.ctypes.data, g.vertex_incidence.ctypes.data,
                 g.edge_offsets.ctypes.data, g.edge_members.ctypes.data, g.base_weights.ctypes.data)

    def graph_release(self, h):
        self._fn("graph_destroy", None, [C.c_void_p])(h)

    def run_handle(self, h, stream: Stream, variant=VARIANT_SEQ, workers=1, max_rounds=0) -> Result:
        res = CResult()
        cs = stream.c()
        f = self._fn("run", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint, C.c_uint32, C.c_void_p])
        rc = f(h, variant, C.addressof(cs), workers, max_rounds, C.addressof(res))
        out = _own_result(rc, res)
        self._fn("free_result", None, [C.c_void_p])(C.addressof(res))
        return out

    # ---- reference only: io.hpp (text formats), for the parity tests of the library's parsers ----
    def parse_text(self, which: str, text, degree_zero: int = 0):
        """which: 'hgr' | 'metis'.  Returns (status, Graph or None, number of warnings)."""
        assert self.kind == "reference"
        data = text.encode() if isinstance(text, str) else bytes(text)
        og = COwnedGraph()
        nw = C.c_uint32(0)
        if which == "hgr":
            f = self._fn("parse_hgr", C.c_int, [C.c_char_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p])
            rc = f(data, len(data), degree_zero, C.addressof(og), C.addressof(nw))
        else:
            f = self._fn("parse_metis_graph", C.c_int, [C.c_char_p, C.c_size_t, C.c_int, C.c_void_p])
            rc = f(data, len(data), degree_zero, C.addressof(og))
        if rc != OK:
            return rc, None, 0
        g = _own_graph(og)
        self._fn("free_graph", None, [C.c_void_p])(C.addressof(og))
        return rc, g, int(nw.value)

    def _text(self, ptr, length) -> str:
        try:
            return C.string_at(ptr, length.value).decode()
        finally:
            self._fn("free_text", None, [C.c_void_p])(ptr)

    def write_hgr(self, g: Graph) -> str:
        h = self.graph_handle(g)
        try:
            length = C.c_size_t()
            ptr = self._fn("write_hgr", C.c_void_p, [C.c_void_p, C.c_void_p])(h, C.addressof(length))
            return self._text(ptr, length)
        finally:
            self.graph_release(h)

    def write_matching(self, matched, total_weight: float, rounds: int) -> str:
        ids = np.ascontiguousarray(matched, dtype=np.uint32)
        length = C.c_size_t()
        f = self._fn("write_matching", C.c_void_p, [C.c_void_p, C.c_uint64, C.c_double, C.c_uint32, C.c_void_p])
        return self._text(f(ids.ctypes.data if ids.size else None, ids.size, total_weight, rounds, C.addressof(length)), length)

    def parse_matching(self, text):
        data = text.encode() if isinstance(text, str) else bytes(text)
        ptr, cnt = C.POINTER(C.c_uint32)(), C.c_uint64()
        f = self._fn("parse_matching", C.c_int, [C.c_char_p, C.c_size_t, C.c_void_p, C.c_void_p])
        rc = f(data, len(data), C.addressof(ptr), C.addressof(cnt))
        if rc != OK:
            return rc, None
        out = _take(ptr, cnt.value, np.uint32)
        self._fn("free_text", None, [C.c_void_p])(C.cast(ptr, C.c_void_p))
        return rc, out

    def compact(self, g: Graph, vertex_active, edge_active, workers: int = 2):
        """reference only: (status, Graph, vertex_map, edge_map, [edge visits, pin visits, scans, compactions])"""
        assert self.kind == "reference"
        va = np.ascontiguousarray(vertex_active, dtype=np.uint8)
        ea = np.ascontiguousarray(edge_active, dtype=np.uint8)
        vmap, emap = np.empty(g.n, dtype=np.uint32), np.empty(g.m, dtype=np.uint32)
        counters = np.zeros(4, dtype=np.uint64)
        og = COwnedGraph()
        h = self.graph_handle(g)
        try:
            f = self._fn("compact", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_void_p])
            rc = f(h, va.ctypes.data, ea.ctypes.data, workers, C.addressof(og), vmap.ctypes.data, emap.ctypes.data,
                   counters.ctypes.data)
        finally:
            self.graph_release(h)
        if rc != OK:
            return rc, None, None, None, None
        out = _own_graph(og)
        self._fn("free_graph", None, [C.c_void_p])(C.addressof(og))
        return rc, out, vmap, emap, counters.tolist()

    def hardware_workers(self) -> int:
        if self.kind == "reference":
            return int(self._fn("hardware_workers", C.c_uint, [])())
        return 1

    def verify(self, g: Graph, matched) -> tuple:
        matched = np.ascontiguousarray(matched, dtype=np.uint32)
        dis, mx, w = C.c_int(0), C.c_int(0), C.c_double(0)
        if self.kind == "port":
            cg = g.c()
            f = self._fn("verify_matching", C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                                       C.c_void_p])
            rc = f(C.addressof(cg), matched.ctypes.data, matched.size, C.byref(dis), C.byref(mx), C.byref(w))
        else:
            h = self.graph_handle(g)
            f = self._fn("verify", C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p])
            rc = f(h, matched.ctypes.data, matched.size, C.byref(dis), C.byref(mx), C.byref(w))
            self.graph_release(h)
        if rc != OK:
            raise ValueError("verify: matching references an edge out of range")
        return bool(dis.value), bool(mx.value), float(w.value)

    # ---- synthetic bench instances (port only; the reference has no such generators) ----
    def syn_generate(self, family, n=0, m=0, d=0, scale=0, seed=1, int_weights=False) -> Graph:
        lib = self._port
        spec = CSynSpec(family, n, m, d, scale, seed, 1 if int_weights else 0)
        og = COwnedGraph()
        lib.orc_syn_generate.restype = C.c_int
        lib.orc_syn_generate.argtypes = [C.c_void_p, C.c_void_p]
        rc = lib.orc_syn_generate(C.addressof(spec), C.addressof(og))
        if rc != OK:
            raise ValueError("syn_generate: input error")
        g = _own_graph(og)
        lib.orc_free_graph.argtypes = [C.c_void_p]
        lib.orc_free_graph(C.addressof(og))
        return g


def graph_from_edge_lists(lists, weights=None, n=None) -> Graph:
    """Small helper for literal test instances (hypergraph.hpp:78 without the degree-0 policy)."""
    m = len(lists)
    sizes = np.array([len(x) for x in lists], dtype=np.uint64)
    eoff = np.zeros(m + 1, dtype=np.uint64)
    np.cumsum(sizes, out=eoff[1:])
    pins = np.array([v for x in lists for v in x], dtype=np.uint32)
    if n is None:
        n = int(pins.max()) + 1 if pins.size else 0
    base = np.ones(m, dtype=np.float64) if weights is None else np.asarray(weights, dtype=np.float64)
    voff = np.zeros(n + 1, dtype=np.uint64)
    vinc = np.zeros(pins.size, dtype=np.uint32)
    lib = _load(PORT_LIB, build=True)
    lib.orc_build_incidence.restype = C.c_int
    lib.orc_build_incidence.argtypes = [C.c_uint32, C.c_uint32] + [C.c_void_p] * 4
    rc = lib.orc_build_incidence(n, m, eoff.ctypes.data, pins.ctypes.data, voff.ctypes.data, vinc.ctypes.data)
    if rc != OK:
        raise ValueError("vertex id out of range")
    return Graph(n, m, voff, vinc, eoff, pins, base)


def graph_from_csr(n, m, edge_offsets, edge_members, base_weights) -> Graph:
    """Completes an edge-side CSR with the vertex-incidence side (hypergraph.hpp:144-151)."""
    eoff = np.ascontiguousarray(edge_offsets, dtype=np.uint64)
    pins = np.ascontiguousarray(edge_members, dtype=np.uint32)
    base = np.ascontiguousarray(base_weights, dtype=np.float64)
    voff = np.zeros(n + 1, dtype=np.uint64)
    vinc = np.zeros(pins.size, dtype=np.uint32)
    lib = _load(PORT_LIB, build=True)
    lib.orc_build_incidence.restype = C.c_int
    lib.orc_build_incidence.argtypes = [C.c_uint32, C.c_uint32] + [C.c_void_p] * 4
    rc = lib.orc_build_incidence(n, m, eoff.ctypes.data, pins.ctypes.data, voff.ctypes.data, vinc.ctypes.data)
    if rc != OK:
        raise ValueError("vertex id out of range")
    return Graph(n, m, voff, vinc, eoff, pins, base)
