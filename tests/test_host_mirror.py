"""The C++ host mirror (paper_2604_03960_b200/host/adaptchi_b200.hpp) compiles
against the C-ABI (CPU) and passes the reference-style C++ tests on the GPU
(tests/cpp/test_host_mirror.cpp, cases from /root/reference/proj/tests/*.cpp)."""
import os
import shutil
import subprocess

import pytest

from paper_2604_03960_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_host_mirror.cpp")


def _compile(out):
    lib_dir = os.path.dirname(abi.LIB_PATH)
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-Werror", SRC, "-L" + lib_dir,
           "-ladaptchi_b200", "-Wl,-rpath," + lib_dir, "-o", out]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


@pytest.mark.skipif(shutil.which("g++") is None, reason="no host C++ compiler")
def test_host_mirror_compiles_and_links(tmp_path):
    abi.load()
    _compile(str(tmp_path / "t"))
    assert os.path.exists(tmp_path / "t")


@pytest.mark.gpu
def test_host_mirror_reference_cases(tmp_path, oracle):
    exe = str(tmp_path / "t")
    _compile(exe)
    e_heis = oracle.exact_ground_energy(abi.model_spec(8))
    e_tfim = oracle.exact_ground_energy(abi.model_spec(8, family=abi.TRANSVERSE_ISING, h=1.0))
    p = subprocess.run([exe, repr(e_heis), repr(e_tfim)], capture_output=True, text=True,
                       timeout=600)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failures" in p.stdout
