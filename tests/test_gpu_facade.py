"""Builds tests/cpp/test_facade.cpp against the C++ facade + C ABI and runs it on the GPU
(the reference's own unit tests restated for the device path)."""
import pathlib
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parents[1]


def test_cpp_facade_reference_unit_tests(gpu, tmp_path):
    exe = tmp_path / "test_facade"
    libdir = ROOT / "paper_2508_08438_b200"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", str(ROOT / "include"), str(ROOT / "tests/cpp/test_facade.cpp"),
                    "-L", str(libdir), "-lsafekv_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
