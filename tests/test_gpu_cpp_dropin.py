"""Compile tests/cpp/test_dropin.cpp against include/tqsb/reconstruct.hpp and
libtqsb.so (the C++ drop-in for tqs::reconstruct) and run it on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "test_dropin")
    libdir = os.path.join(ROOT, "paper_2205_02646_b200")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-o", exe,
                    "-L", libdir, "-l:libtqsb.so", f"-Wl,-rpath,{libdir}"], check=True)
    return exe


def test_dropin_header_compiles(tmp_path):
    """CPU check: the drop-in header and the C ABI link cleanly."""
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_dropin_reference_pipeline_cases(tmp_path, need_gpu):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
