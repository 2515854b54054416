"""Edge-partitioned matching through hlm_b200_match_sharded (the round driver, the collectives and the
tie handling live inside the library).  k shards on ONE GPU ("virtual ranks") run the same kernels and
the same host loop as k GPUs; with a one-rank communicator every collective really goes through NCCL.
The result must not depend on k (the reference's invariant: independent of workers,
test_par.cpp:32-55) and must equal the oracle on the unpartitioned instance."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.util import assert_same_result, to_hb_graph, to_hb_stream

pytestmark = pytest.mark.gpu

FAMILIES = [
    ("uniform", po.SYN_UNIFORM, dict(n=6000, m=20000, d=8), False),
    ("uniform", po.SYN_UNIFORM, dict(n=9000, m=15000, d=4), True),
    ("rmat", po.SYN_RMAT, dict(scale=11, m=30000), True),
    ("powerlaw", po.SYN_POWERLAW, dict(n=8000, m=12000), False),
    ("netlist", po.SYN_NETLIST, dict(n=9000, m=15000), True),
]


def _release(shards):
    for s in shards:
        s.release()


@pytest.mark.parametrize("family,fam_id,kw,intw", FAMILIES)
def test_shard_count_never_changes_the_matching(hb, port, family, fam_id, kw, intw):
    from paper_2602_22976_b200 import multi_gpu

    g = port.syn_generate(fam_id, seed=4, int_weights=intw, **kw)
    streams = [po.Stream(seed=9), po.Stream(seed=9, noise_high=0.0), po.Stream(seed=2, mode=po.MODE_REPLACE_UNIFORM)]
    for s in streams:
        want = port.local_max(g, s)
        for world in (1, 2, 3, 8):
            shards = multi_gpu.generate_shards(family, world, seed=4, int_weights=intw, **kw)
            got, rep = multi_gpu.match_sharded(shards, to_hb_stream(s), hb.ParallelConfig())
            assert_same_result(got, want, f"{family} world={world} {s}")
            assert rep["host_syncs"] == rep["rounds"] + rep["tie_redo_rounds"]
            # the exchange shrinks with the live-vertex set
            live = rep["live_vertices_per_round"]
            assert live == sorted(live, reverse=True) and live[0] == g.n
            if world == 2:
                got, rep = multi_gpu.match_sharded(shards, to_hb_stream(s), hb.ParallelConfig(tie_mode="exact"))
                assert_same_result(got, want, f"{family} world={world} exact {s}")
                assert rep["tie_redo_rounds"] == 0
            _release(shards)


def test_collectives_through_nccl(hb, port):
    """A one-rank communicator: the same loop with every all-reduce issued to NCCL (dlopen'ed)."""
    from paper_2602_22976_b200 import multi_gpu

    kw = dict(n=5000, m=16000, d=4)
    g = port.syn_generate(po.SYN_UNIFORM, seed=3, **kw)
    comm = multi_gpu.Communicator.create(None, 0, 1, 0)
    assert comm.nccl_version() >= 21800
    for s in (po.Stream(seed=7), po.Stream(seed=7, noise_high=0.0)):
        want = port.local_max(g, s)
        for world in (1, 3):
            shards = multi_gpu.generate_shards("uniform", world, seed=3, **kw)
            got, rep = multi_gpu.match_sharded(shards, to_hb_stream(s), hb.ParallelConfig(), comm)
            assert_same_result(got, want, f"nccl world={world} {s}")
            assert rep["nccl_calls"] >= 3 * rep["rounds"]
            assert rep["collective_bytes"] == sum(rep["collective_bytes_per_round"])
            _release(shards)
    comm.destroy()


def test_cross_shard_ties_take_the_exact_path(hb, port):
    """Collapsed weights: equal maxima held by edges of different shards; the owner count must catch
    them and the round must be resolved by the three-level comparator across shards."""
    from paper_2602_22976_b200 import multi_gpu

    kw = dict(n=3000, m=12000, d=2)
    g = port.syn_generate(po.SYN_UNIFORM, seed=6, **kw)
    s = po.Stream(seed=5, kind=po.GEN_PARK_MILLER, noise_low=0.0, noise_high=2.0 ** -50)
    want = port.local_max(g, s)
    for world in (2, 4):
        shards = multi_gpu.generate_shards("uniform", world, seed=6, **kw)
        got, rep = multi_gpu.match_sharded(shards, to_hb_stream(s))
        assert_same_result(got, want, f"ties world={world}")
        assert rep["tie_redo_rounds"] >= 1
        _release(shards)


def test_round_cap_in_sharded_runs(hb, port):
    from paper_2602_22976_b200 import multi_gpu

    kw = dict(n=2000, m=6000, d=3)
    g = port.syn_generate(po.SYN_UNIFORM, seed=2, **kw)
    s = po.Stream(seed=1)
    want = port.local_max(g, s, max_rounds=2)
    assert want.status == po.ROUND_LIMIT
    shards = multi_gpu.generate_shards("uniform", 2, seed=2, **kw)
    with pytest.raises(hb.RoundLimitError) as ei:
        multi_gpu.match_sharded(shards, to_hb_stream(s), hb.ParallelConfig(max_rounds=2))
    assert np.array_equal(ei.value.partial.matched_edges, want.matched_edges)
    assert ei.value.report.deactivated_per_round == want.per_round_deactivated
    _release(shards)


def test_host_arrays_over_several_gpus(hb, port):
    """run_variant(num_gpus = k) -- hlm_b200_config.num_gpus: the drop-in call cuts the caller's CSR into
    k edge blocks (co-located on the visible devices) and returns the one result."""
    from paper_2602_22976_b200 import multi_gpu

    g = port.generate_random(4000, 9000, 2, 9, 5)
    g.base_weights = port.random_weights_1_100(g.m, 2) * 0.37  # non-integer: ordered FP64 sum across shards
    for s in (po.Stream(seed=3), po.Stream(seed=3, noise_high=0.0)):
        want = port.local_max(g, s)
        for k in (2, 5):
            got = hb.run_variant(to_hb_graph(g), to_hb_stream(s), hb.ParallelConfig(num_gpus=k))
            assert_same_result(got, want, f"num_gpus={k} {s}")
        shards = multi_gpu.upload_shards(to_hb_graph(g), 3)
        got, _ = multi_gpu.match_sharded(shards, to_hb_stream(s))
        assert_same_result(got, want, f"uploaded shards {s}")
        _release(shards)


def test_sharded_call_rejects_what_it_cannot_do(hb, port):
    from paper_2602_22976_b200 import multi_gpu

    shards = multi_gpu.generate_shards("uniform", 2, n=2000, m=5000, d=3, seed=1)
    with pytest.raises(NotImplementedError):
        multi_gpu.match_sharded(shards, hb.WeightStream(), hb.ParallelConfig(variant="greedy"))
    with pytest.raises(hb.InputError):
        multi_gpu.match_sharded(shards, hb.WeightStream(noise_low=2.0, noise_high=1.0))
    with pytest.raises(hb.InputError):  # shards of different instances
        other = multi_gpu.generate_shards("uniform", 2, n=3000, m=5000, d=3, seed=1)
        multi_gpu.match_sharded([shards[0], other[1]], hb.WeightStream())
    whole = hb.DeviceHypergraph.generate("powerlaw", n=3000, m=6000, seed=1)  # loaded whole: vertices renumbered
    with pytest.raises(hb.InputError):
        multi_gpu.match_sharded([whole, shards[1]], hb.WeightStream())
    _release(shards + other + [whole])


def test_two_real_ranks_when_two_gpus_are_visible(hb, port, tmp_path):
    """Two processes, two GPUs, NCCL between them; skipped on a one-GPU box."""
    from paper_2602_22976_b200 import _lib

    if _lib.load_library().hlm_b200_device_count() < 2:
        pytest.skip("needs two visible GPUs")
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29533",
                          os.path.join(root, "tests", "two_rank_check.py")], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "two-rank parity: ok" in out.stdout


def _shm_nccl_lib():
    """tests/cpp/shm_nccl.cpp -> tests/cpp/_build/libshm_nccl.so (nvcc: static cudart, like the library)."""
    import os
    import shutil
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = os.path.join(root, "tests", "cpp", "shm_nccl.cpp")
    out = os.path.join(root, "tests", "cpp", "_build", "libshm_nccl.so")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
        os.makedirs(os.path.dirname(out), exist_ok=True)
        subprocess.run([nvcc, "-shared", "-Xcompiler", "-fPIC", "-O2", "-std=c++17", "-x", "cu", src, "-o", out, "-lrt"], check=True)
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_multi_rank_driver_between_processes_on_one_gpu(hb, port, world):
    """The nranks > 1 path of hlm_b200_match_sharded between real processes: NCCL refuses two ranks on one
    device, so the collectives go through a shared-memory stand-in for libnccl.so.2 (HLM_B200_NCCL_LIB);
    everything above the twelve bound calls is the product's code.  tests/multi_rank_shm_check.py compares
    every rank's slice with the oracle (ragged and uniform instances, real weights, ties, the round cap)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HLM_B200_NCCL_LIB=_shm_nccl_lib(), CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0])
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
                          "--master-addr", "127.0.0.1", "--master-port", str(29540 + world),
                          os.path.join(root, "tests", "multi_rank_shm_check.py")], capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-6000:]
    assert f"multi-rank parity over shared memory, {world} ranks: ok" in out.stdout


def test_bench_scaling_arm_end_to_end_with_two_ranks_on_one_gpu(hb):
    """`bench.py --gpus 2` exactly as the driver launches it (torchrun, one rank per process), shrunk to a
    test size and pointed at the shared-memory transport: the JSON line of the N > 1 arm must come out, once,
    from rank 0, with the whole-job pin count and the per-round exchange report."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HLM_B200_NCCL_LIB=_shm_nccl_lib(), HLM_BENCH_ONE_GPU="1", HLM_BENCH_MG_EDGES="200000",
               HLM_BENCH_MG_VERTICES="100000")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29547", os.path.join(root, "bench.py"),
                          "--gpus", "2", "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-6000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["steps"] == 2
    assert line["config"]["pins"] == 2 * 200000 * 8
    assert line["value"] > 0 and line["gpu_launches"] > 0
    moved = line["config"]["collective_bytes_per_round"]
    assert moved == sorted(moved, reverse=True) and len(moved) == line["config"]["rounds"]
    assert line["config"]["matched"] > 0 and line["roofline"]["frac"] > 0
