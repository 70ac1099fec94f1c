"""The C++ host API (include/moeprism/moe_layer.hpp) and its drop-in
partitioned_forward: compiled here (CPU) and run on the GPU, where it executes
the reference's expert KATs (proj/tests/test_expert.cpp) and acceptance C1."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_2510_19366_b200"


def _build(out: Path):
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "test_dropin.cpp"),
           f"-L{PKG}", "-lmoeprism_b200", f"-Wl,-rpath,{PKG}", "-o", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_cpp_header_compiles_and_links(tmp_path):
    _build(tmp_path / "test_dropin")


@pytest.mark.gpu
def test_cpp_dropin_on_gpu(tmp_path, cuda_lib):
    exe = tmp_path / "test_dropin"
    _build(exe)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASSED" in r.stdout
