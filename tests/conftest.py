import os
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 CUDA device (runs through the C ABI on the GPU)")


def _ensure_built():
    lib = ROOT / "paper_2508_08438_b200" / "libsafekv_b200.so"
    orc = ROOT / "oracle" / "_ref" / "liboracle.so"
    ref = ROOT / "oracle" / "_ref" / "libsafekv_ref.so"
    gen = ROOT / "workload" / "libskv_gen.so"
    if not gen.exists():
        subprocess.run(["make", "-C", str(ROOT), "workload/libskv_gen.so"], check=True, capture_output=True)
    if not lib.exists():
        subprocess.run(["make", "-C", str(ROOT), "-j8", "paper_2508_08438_b200/libsafekv_b200.so"], check=True,
                       capture_output=True)
    if not orc.exists() and (ROOT / "oracle" / "safekv_oracle.c").exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "oracle"], check=False, capture_output=True)
    if not ref.exists() and pathlib.Path("/root/reference/proj/include").exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "ref"], check=False, capture_output=True)


_ensure_built()


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available() and torch.cuda.get_device_capability(0)[0] == 10
    except Exception:
        return False


@pytest.fixture(scope="session")
def ref():
    from refh import load_ref
    L = load_ref()
    if L is None:
        pytest.skip("reference harness oracle/_ref/libsafekv_ref.so not built (needs /root/reference)")
    return L


@pytest.fixture(scope="session")
def gpu():
    # -m gpu runs only on B200 boxes: a missing device is a failure, not a skip
    assert gpu_available(), "gpu-marked test needs an sm_100 device"
    return True
