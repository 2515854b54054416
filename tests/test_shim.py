"""include/hlm_b200.hpp: the C++ shim with the reference's signatures.

CPU part (here): it compiles and links against the UNMODIFIED reference headers + libhlm_b200.so
(needs /root/reference; the binary lands in tests/cpp/_build/, which travels to the GPU box).
GPU part: run the prebuilt binary -- the reference's own call sites with hlm::b200:: swapped in
must reproduce local_max_sequential exactly."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "cpp", "_build")
EXE = os.path.join(BUILD, "shim_parity")
REF_INC = "/root/reference/proj/include"


def test_shim_compiles_against_reference_headers(hb):
    if not os.path.isdir(REF_INC):
        pytest.skip("reference headers not present on this machine")
    from paper_2602_22976_b200 import _lib

    os.makedirs(BUILD, exist_ok=True)
    libdir = os.path.dirname(_lib.LIB_PATH)
    cmd = ["g++", "-std=c++20", "-O2", "-pthread", "-ffp-contract=off", "-I", REF_INC, "-I",
           os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp", "shim_parity.cpp"), "-o", EXE,
           "-L", libdir, "-lhlm_b200", "-Wl,-rpath,$ORIGIN/../../../paper_2602_22976_b200/lib"]
    subprocess.run(cmd, check=True)
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_shim_reproduces_reference_on_gpu():
    if not os.path.exists(EXE):
        pytest.skip("tests/cpp/_build/shim_parity was not prebuilt (needs the reference headers)")
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "shim parity: ok" in out.stdout
