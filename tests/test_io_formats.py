"""Text formats of the library (hMetis .hgr, METIS graphs, matching files; host only, no GPU):
the literal cases of the reference's tests/test_io.cpp, and differential runs against the
reference's own io.hpp (oracle/_ref) on well-formed, perturbed and malformed texts: the same
inputs must be accepted and rejected, with identical CSR arrays and identical texts out."""
import numpy as np
import pytest

from oracle import pyoracle as po


def _same_graph(h, g: po.Graph, what=""):
    assert (h.num_vertices, h.num_edges) == (g.n, g.m), what
    for a, b in ((h.vertex_offsets, g.vertex_offsets), (h.vertex_incidence, g.vertex_incidence),
                 (h.edge_offsets, g.edge_offsets), (h.edge_members, g.edge_members), (h.base_weights, g.base_weights)):
        assert np.array_equal(np.asarray(a), np.asarray(b)), what


def _to_hb(hb, g: po.Graph):
    return hb.Hypergraph(g.n, g.m, g.vertex_offsets, g.vertex_incidence, g.edge_offsets, g.edge_members, g.base_weights)


def test_known_answers_of_test_io_cpp(hb, port):
    h = hb.parse_hgr("1 2\n1 2\n")  # test_io.cpp:9-16
    assert (h.num_vertices, h.num_edges) == (2, 1)
    assert h.edge_members.tolist() == [0, 1] and h.base_weights.tolist() == [1.0]
    h = hb.parse_hgr("4 6 1\n1 1 4\n1 2 5\n1 3 6\n1.1 1 2 3\n")  # :18-21: the tight family d = 3, eps = 0.1
    _same_graph(h, port.tight_family(3, 0.1), "tight family")
    h = hb.parse_hgr("% a comment\n\n2 4 1\n% another\n3 1 2\n\n5 3 4\n")  # :23-27
    assert h.num_edges == 2 and h.base_weights.tolist() == [3.0, 5.0]
    warnings = []
    h = hb.parse_hgr("1 2 11\n2 1 2\n7\n9\n", warnings=warnings)  # :29-37
    assert h.num_edges == 1 and h.base_weights.tolist() == [2.0] and len(warnings) == 1
    for bad in ["", "x y\n", "1 2 7\n1 2\n", "2 2\n1 2\n", "1 2\n1 3\n", "1 2\n0 1\n", "1 2 1\n1\n", "1 2 1\n0 1 2\n",
                "1 2 1\n-1 1 2\n", "1 2\n1 2\n1 2\n", "1 4\n1 2\n"]:  # :39-51
        with pytest.raises(hb.InputError):
            hb.parse_hgr(bad)
    h = hb.parse_metis_graph("3 3\n2 3\n1 3\n1 2\n")  # :69-75
    assert h.num_edges == 3 and h.edge_members.size == 6
    assert hb.parse_metis_graph("3 2\n2\n1 3\n2\n").num_edges == 2  # :77-82
    grid = "9 12\n2 4\n1 3 5\n2 6\n1 5 7\n2 4 6 8\n3 5 9\n4 8\n5 7 9\n6 8\n"  # :84-95
    assert hb.parse_metis_graph(grid).num_edges == 12
    for bad in ["2 1\n2\n\n", "2 1\n1 2\n1\n", "3 5\n2\n1 3\n2\n", "2 1 1\n2\n1\n"]:  # :97-102
        with pytest.raises(hb.InputError):
            hb.parse_metis_graph(bad)
    assert hb.parse_hgr("1 4\n1 2\n", degree_zero="drop_and_renumber").num_vertices == 2


def test_round_trip_and_writer_equal_the_reference(hb, port, ref):
    """test_io.cpp:53-67 (100 random instances, three weight styles) + byte-identical writer output."""
    for seed in range(1, 101):
        g = port.generate_random(20, 15, 1, 4, seed)
        if seed % 3 == 0:
            g.base_weights = port.random_weights_1_100(g.m, seed)
        if seed % 3 == 1:
            g.base_weights = np.array([0.25 + 0.125 * (e % 7) + (seed % 5) * 1e-3 for e in range(g.m)])
        text = hb.write_hgr(_to_hb(hb, g))
        assert text == ref.write_hgr(g), f"seed {seed}"
        _same_graph(hb.parse_hgr(text), g, f"round trip seed {seed}")
    ids = np.array([3, 17, 4000000000], dtype=np.uint32)
    assert hb.write_matching(hb.Matching(ids, 123.4567891, 7)) == ref.write_matching(ids, 123.4567891, 7)
    assert hb.write_matching(hb.Matching(np.zeros(0, np.uint32), 0.0, 0)) == ref.write_matching([], 0.0, 0)
    text = "% weight 1\n% size 2\n5 9\n\n  12\t13 \r\n"
    assert hb.parse_matching(text).tolist() == ref.parse_matching(text)[1].tolist() == [5, 9, 12, 13]
    with pytest.raises(hb.InputError):
        hb.parse_matching("1 x\n")
    assert ref.parse_matching("1 x\n")[0] == po.INPUT_ERROR


def _mutations(rng, text: str):
    """Small perturbations of a well-formed text: most break it, some do not."""
    lines = text.split("\n")
    yield "\n".join(lines[:-2])                       # truncated
    yield text + "7 7\n"                             # trailing content
    yield text.replace(" ", "\t")                   # tabs
    yield text.replace("\n", "\r\n")                # CRLF
    yield "% c\n\n" + text.replace("\n", "\n% x\n", 2)  # comments and blank lines
    for _ in range(12):
        i = int(rng.integers(0, len(text)))
        c = "0123456789 -.x%\n"[int(rng.integers(0, 16))]
        yield text[:i] + c + text[i + 1:]            # one character replaced
        yield text[:i] + c + text[i:]                # one character inserted
        yield text[:i] + text[i + 1:]                # one character deleted


def test_differential_against_the_reference_parsers(hb, port, ref):
    rng = np.random.default_rng(7)
    checked = rejected = 0
    for seed in range(1, 25):
        g = port.generate_random(12, 10, 1, 4, seed)
        if seed % 2:
            g.base_weights = port.random_weights_1_100(g.m, seed) * (0.5 if seed % 4 == 1 else 1.0)
        base = ref.write_hgr(g)
        if seed % 5 == 0:  # a vertex-weight block
            base = base.replace("\n", " 1\n", 1) if " 1\n" not in base.split("\n")[0] + "\n" else base
            base = base.split("\n", 1)[0].replace(" 1", " 11") + "\n" + base.split("\n", 1)[1] + "".join("3\n" for _ in range(g.n))
        for text in [base, *_mutations(rng, base)]:
            for dz in (0, 1):
                rc, want, nwarn = ref.parse_text("hgr", text, dz)
                warnings = []
                try:
                    got = hb.parse_hgr(text, degree_zero="drop" if dz else "reject", warnings=warnings)
                except hb.InputError:
                    assert rc == po.INPUT_ERROR, f"library rejects what the reference accepts: {text!r}"
                    rejected += 1
                    continue
                assert rc == po.OK, f"library accepts what the reference rejects: {text!r}"
                _same_graph(got, want, repr(text))
                assert len(warnings) == nwarn
                checked += 1
    assert checked > 200 and rejected > 200
    # METIS graphs: random symmetric adjacency, then perturbed
    checked = rejected = 0
    for seed in range(1, 25):
        n = 9
        adj = rng.random((n, n)) < 0.3
        adj = np.triu(adj, 1)
        adj = adj | adj.T
        m = int(adj.sum() // 2)
        base = f"{n} {m}\n" + "".join(" ".join(str(v + 1) for v in np.nonzero(adj[u])[0]) + "\n" for u in range(n))
        for text in [base, *_mutations(rng, base)]:
            for dz in (0, 1):
                rc, want, _ = ref.parse_text("metis", text, dz)
                try:
                    got = hb.parse_metis_graph(text, degree_zero="drop" if dz else "reject")
                except hb.InputError:
                    assert rc == po.INPUT_ERROR, f"library rejects what the reference accepts: {text!r}"
                    rejected += 1
                    continue
                assert rc == po.OK, f"library accepts what the reference rejects: {text!r}"
                _same_graph(got, want, repr(text))
                checked += 1
    assert checked > 100 and rejected > 200


def test_load_instance_file(hb, tmp_path):
    p = tmp_path / "tiny.hgr"
    p.write_text("2 3\n1 2\n2 3\n")
    h = hb.load_instance_file(str(p))
    assert h.num_edges == 2 and h.edge_members.tolist() == [0, 1, 1, 2]
    with pytest.raises(IOError):
        hb.load_instance_file(str(tmp_path / "missing.hgr"))
