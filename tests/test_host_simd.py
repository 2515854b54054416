"""The loader's host loops (csrc/hlm_host_simd.cpp): AVX2 forms == scalar forms on edge cases.
Pure host code, compiled here with g++ and run on the CPU."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2602_22976_b200", "csrc")


def _build(tmp_path):
    exe = tmp_path / "host_simd_check"
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", CSRC, os.path.join(ROOT, "tests", "cpp", "host_simd_check.cpp"),
                    os.path.join(CSRC, "hlm_host_simd.cpp"), "-o", str(exe)], check=True)
    return str(exe)


def test_simd_loops_match_scalar(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert ": ok" in out.stdout


def test_scalar_dispatch_switch(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120, env={**os.environ, "HLM_B200_HOST_SIMD": "0"})
    assert out.returncode == 0 and "host simd (scalar): ok" in out.stdout
