"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every symbol that
include/hlm_b200.h declares, and fails loudly (no CPU fallback) when there is no CUDA device."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "hlm_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hlm_b200_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_are_exported(hb):
    from paper_2602_22976_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/hlm_b200.h but not exported"
    # the Python binding covers the same set
    assert sorted(_lib.SYMBOLS) == declared
    assert lib.hlm_b200_abi_version() == 3


def test_struct_layouts_match_the_header(hb, tmp_path):
    """sizeof of the ctypes mirrors == sizeof the C compiler computes from include/hlm_b200.h."""
    import subprocess

    from paper_2602_22976_b200 import _lib

    src = tmp_path / "sizes.c"
    src.write_text('#include <stdio.h>\n#include "hlm_b200.h"\nint main(void){printf("%zu %zu %zu %zu %zu %zu %zu\\n",'
                   "sizeof(hlm_b200_csr_view),sizeof(hlm_b200_stream),sizeof(hlm_b200_config),"
                   "sizeof(hlm_b200_syn_spec),sizeof(hlm_b200_graph_info),sizeof(hlm_b200_result),"
                   "sizeof(hlm_b200_shard_report));return 0;}\n")
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    sizes = [int(x) for x in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()]
    mirrors = [_lib.CsrView, _lib.Stream, _lib.Config, _lib.SynSpec, _lib.GraphInfo, _lib.Result, _lib.ShardReport]
    assert sizes == [ctypes.sizeof(m) for m in mirrors]


def test_default_max_rounds_needs_no_device(hb):
    assert hb.default_max_rounds(0) == 64 + 4 * 1
    assert hb.default_max_rounds(1_000_000) == 144
    assert hb.default_max_rounds(1 << 28) == 180


def test_no_cpu_fallback(hb):
    """Without a GPU every compute entry point must fail with a device error, never compute."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    h = hb.Hypergraph(2, 1, None, None, np.array([0, 2], dtype=np.uint64), np.array([0, 1], dtype=np.uint32),
                      np.ones(1))
    with pytest.raises(hb.DeviceError):
        hb.run_variant(h, hb.WeightStream())
    with pytest.raises(hb.DeviceError):
        hb.DeviceHypergraph.generate("uniform", n=10, m=10, d=2)
    with pytest.raises(hb.DeviceError):
        hb.eval_stream(hb.WeightStream(), [0], [1])


def test_product_code_never_touches_the_oracle():
    """The oracle is test infrastructure: nothing under the package may import, link or dlopen it."""
    pkg = os.path.join(ROOT, "paper_2602_22976_b200")
    for base, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".hpp", ".cpp")):
                text = open(os.path.join(base, f), errors="ignore").read()
                for pat in (r"^\s*(from|import)\s+oracle", r"#\s*include\s*[<\"].*oracle", r"(CDLL|dlopen)\(.*oracle",
                            r"libhlm_(ref|oracle)\.so"):
                    assert not re.search(pat, text, flags=re.M), (f, pat)
    for f in ("include/hlm_b200.h",):
        assert "pyoracle" not in open(os.path.join(ROOT, f)).read()
