"""tools/hlm_b200_cli.cpp: the reference's command-line harness (proj/tools/hlm_app.hpp) on libhlm_b200.so.
The cases are the reference's own (proj/tests/test_cli.cpp) minus the exact oracle, which is out of scope:
same subcommands and flags, same CSV schema, same exit codes."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2602_22976_b200", "lib", "hlm_b200_cli")
HEADER = "instance,variant,workers,seed,generator,repeat,rounds,size,weight,time_ms,edge_visits,pin_visits,ratio_vs_oracle"


def cli(*args):
    return subprocess.run([CLI, *[str(a) for a in args]], capture_output=True, text=True, timeout=300)


def lines_of(path):
    with open(path) as f:
        return [ln for ln in f.read().splitlines() if ln]


@pytest.fixture(scope="module", autouse=True)
def built(hb):
    import __graft_entry__ as ge

    ge.build_cli()
    assert os.path.exists(CLI)


def test_generate_writes_the_reference_instances(hb, port, tmp_path):
    """generate tight / random (test_cli.cpp:45-52,83-86): the files parse back to the reference's instances."""
    out = tmp_path / "tight.hgr"
    r = cli("generate", "tight", "--d", 3, "--epsilon", 0.1, "--out", out)
    assert r.returncode == 0 and "n=6 m=4 kappa=9" in r.stdout
    h = hb.parse_hgr(out.read_text())
    t = hb.generate_tight_family(3, 0.1)
    assert np.array_equal(h.edge_members, t.edge_members) and np.array_equal(h.base_weights, t.base_weights)
    rnd = tmp_path / "rnd.hgr"
    assert cli("generate", "random", "--n", 60, "--m", 80, "--min-size", 2, "--max-size", 4, "--seed", 5, "--weights",
               "random", "--out", rnd).returncode == 0
    want = port.generate_random(60, 80, 2, 4, 5)
    got = hb.parse_hgr(rnd.read_text())
    assert np.array_equal(got.edge_offsets, want.edge_offsets) and np.array_equal(got.edge_members, want.edge_members)
    assert np.array_equal(got.base_weights, port.random_weights_1_100(want.m, 1))


def test_bad_invocations_exit_nonzero(tmp_path):
    """test_cli.cpp:67-71 plus the flag checks CLI11 does for the reference."""
    assert cli("run", "--instance", "/nonexistent.hgr").returncode != 0
    assert cli("run", "--bogus").returncode != 0
    assert cli().returncode != 0
    assert cli("run", "--instance", "x.hgr", "--variant", "fastest").returncode != 0
    assert cli("generate", "random", "--n", 5, "--out", tmp_path / "x.hgr").returncode != 0  # --m missing
    assert cli("generate", "random", "--n", 5, "--m", 5, "--min-size", 9, "--max-size", 3, "--out", tmp_path / "x.hgr").returncode == 1
    assert cli("oracle", "--instance", "x.hgr").returncode == 2
    assert cli("--help").returncode == 0


@pytest.mark.gpu
def test_run_verify_round_trip(tmp_path):
    """test_cli.cpp:40-65: tight family, zero noise -> the heavy edge alone: size 1, weight 1.100000."""
    inst, matching, csv = tmp_path / "tight.hgr", tmp_path / "m.txt", tmp_path / "run.csv"
    assert cli("generate", "tight", "--d", 3, "--epsilon", 0.1, "--out", inst).returncode == 0
    r = cli("run", "--instance", inst, "--noise", "0:0", "--variant", "crcw", "--oracle", "--emit-matching", matching, "--csv", csv)
    assert r.returncode == 0, r.stderr
    rows = lines_of(csv)
    assert len(rows) == 2 and rows[0] == HEADER
    assert ",1,1.100000," in rows[1]
    assert rows[1].endswith(",")  # ratio_vs_oracle stays blank: the exact search is not part of the library
    assert r.stdout.splitlines()[0] == HEADER
    v = cli("verify", "--instance", inst, "--matching", matching)
    assert v.returncode == 0 and "disjoint: yes" in v.stdout and "maximal: yes" in v.stdout and "weight: 1.100000" in v.stdout


@pytest.mark.gpu
def test_variants_agree_through_the_cli(port, tmp_path):
    """test_cli.cpp:73-101, with the oracle's answer on top: every variant, same size and weight."""
    from oracle import pyoracle as po

    inst, csv = tmp_path / "rnd.hgr", tmp_path / "both.csv"
    assert cli("generate", "random", "--n", 60, "--m", 80, "--min-size", 2, "--max-size", 4, "--seed", 5, "--weights",
               "random", "--out", inst).returncode == 0
    for variant in ("seq", "crcw", "crew", "opt", "auto"):
        r = cli("run", "--instance", inst, "--variant", variant, "--seed", 9, "--csv", csv)
        assert r.returncode == 0, r.stderr
    rows = lines_of(csv)
    assert len(rows) == 6
    g = port.generate_random(60, 80, 2, 4, 5)
    g.base_weights = port.random_weights_1_100(g.m, 1)
    want = port.local_max(g, po.Stream(seed=9))
    for row in rows[1:]:
        f = row.split(",")
        assert int(f[6]) == want.rounds and int(f[7]) == len(want.matched_edges) and float(f[8]) == want.total_weight
    # two shards on the one device: the same row
    r = cli("run", "--instance", inst, "--variant", "crcw", "--seed", 9, "--gpus", 2)
    f = r.stdout.splitlines()[1].split(",")
    assert r.returncode == 0 and int(f[7]) == len(want.matched_edges) and float(f[8]) == want.total_weight


@pytest.mark.gpu
def test_bench_rows_means_and_geomeans(tmp_path):
    """test_cli.cpp:103-127: header + 2 instances x 2 variants x 3 repeats + 4 mean rows + 2 geomean rows; a missing
    instance keeps its blank rows and turns the exit code to 1 without stopping the batch (hlm_app.hpp:228-231)."""
    a, b, csv = tmp_path / "a.hgr", tmp_path / "b.hgr", tmp_path / "bench.csv"
    assert cli("generate", "random", "--n", 30, "--m", 40, "--seed", 1, "--out", a).returncode == 0
    assert cli("generate", "random", "--n", 30, "--m", 40, "--seed", 2, "--out", b).returncode == 0
    r = cli("bench", "--instances", a, b, "--variants", "crcw,greedy", "--repeats", 3, "--csv", csv)
    assert r.returncode == 0, r.stderr
    rows = lines_of(csv)
    assert len(rows) == 1 + 12 + 4 + 2
    assert sum(",mean," in ln for ln in rows) == 4
    assert sum(ln.startswith("geomean,") for ln in rows) == 2
    r = cli("bench", "--instances", a, tmp_path / "missing.hgr", "--repeats", 2)
    out = [ln for ln in r.stdout.splitlines() if ln]
    assert r.returncode == 1 and len(out) == 1 + 4 + 1 + 1
    assert sum(ln.endswith(",,,,,,,") for ln in out) == 2  # the failed runs: measurements blank, schema unchanged


@pytest.mark.gpu
def test_verify_exit_codes(tmp_path):
    """test_cli.cpp:129-150: a triangle of pair edges; the empty matching is not maximal, {0, 1} not disjoint."""
    inst = tmp_path / "tri.hgr"
    inst.write_text("3 3 1\n5 1 2\n4 2 3\n3 1 3\n")
    empty, overlap, good = tmp_path / "empty.txt", tmp_path / "overlap.txt", tmp_path / "good.txt"
    empty.write_text("% nothing matched\n")
    overlap.write_text("0\n1\n")
    good.write_text("0\n")
    r = cli("verify", "--instance", inst, "--matching", empty)
    assert r.returncode == 1 and "maximal: NO" in r.stdout
    r = cli("verify", "--instance", inst, "--matching", overlap)
    assert r.returncode == 1 and "disjoint: NO" in r.stdout
    r = cli("verify", "--instance", inst, "--matching", good)
    assert r.returncode == 0 and "weight: 5.000000" in r.stdout
