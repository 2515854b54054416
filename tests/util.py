"""Shared helpers for the parity tests (test infrastructure; may import oracle/)."""
import numpy as np

import paper_2602_22976_b200 as hb
from oracle import pyoracle as po

KIND_NAMES = {po.GEN_XORSHIFT: "xorshift", po.GEN_PARK_MILLER: "park_miller", po.GEN_SPLITMIX: "splitmix"}
MODE_NAMES = {po.MODE_PERTURB_BASE: "perturb_base", po.MODE_REPLACE_UNIFORM: "replace_uniform"}


def to_hb_graph(g: po.Graph, with_incidence: bool = False) -> hb.Hypergraph:
    return hb.Hypergraph(g.n, g.m, g.vertex_offsets if with_incidence else None,
                         g.vertex_incidence if with_incidence else None, g.edge_offsets, g.edge_members,
                         g.base_weights)


def to_hb_stream(s: po.Stream) -> hb.WeightStream:
    return hb.WeightStream(s.seed, KIND_NAMES[s.kind], MODE_NAMES[s.mode], s.noise_low, s.noise_high)


def from_hb_graph(h: hb.Hypergraph) -> po.Graph:
    """hb.Hypergraph (e.g. a download of a device-generated instance) -> oracle graph with a
    host-built incidence side."""
    g = po.Graph(h.num_vertices, h.num_edges, np.zeros(h.num_vertices + 1, dtype=np.uint64),
                 np.zeros(h.edge_members.size, dtype=np.uint32), np.ascontiguousarray(h.edge_offsets),
                 np.ascontiguousarray(h.edge_members), np.ascontiguousarray(h.base_weights))
    lists_g = po.graph_from_csr(g.n, g.m, g.edge_offsets, g.edge_members, g.base_weights)
    return lists_g


def assert_same_result(got: hb.MatchResult, want: po.Result, what: str = ""):
    assert got.report.rounds == want.rounds, f"{what}: rounds {got.report.rounds} != {want.rounds}"
    assert got.report.matched_per_round_count == want.per_round_matched, f"{what}: per-round matched"
    assert got.report.deactivated_per_round == want.per_round_deactivated, f"{what}: per-round deactivated"
    assert np.array_equal(got.matching.matched_edges, want.matched_edges), f"{what}: matched set differs"
    if got.report.matched_round is not None:
        assert np.array_equal(got.report.matched_round.astype(np.uint32), want.matched_round), f"{what}: round of match"
    # bit-exact: same ids summed in the same order
    assert got.matching.total_weight == want.total_weight, f"{what}: weight {got.matching.total_weight} != {want.total_weight}"
