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


def test_reference_unit_tests_against_dropin_facade(gpu):
    """The reference's own unit-test cases for the path (test_cache_index.cpp:96-118,334-388,463-471;
    test_monitor.cpp:14-186; test_detection.cpp:33-145), compiled unchanged against the drop-in
    facade include/safekv/ (tests/cpp/build_ref_unit.py, built where /root/reference exists)."""
    exe = ROOT / "tests" / "cpp" / "_ref_unit" / "ref_unit"
    if not exe.exists():
        pytest.skip("reference unit-test binary not built (tests/cpp/build_ref_unit.py needs /root/reference)")
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(out.stdout[-4000:])
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "0 failed cases" in out.stdout
