"""Tier-1/2/3 DetectionPipeline + production index sink (reference detection.hpp:491-676) on the
drop-in facade vs the reference: tests/cpp/pipeline_parity.cpp compiled against include/safekv/
(device Tier-1 scan of each drain in one launch, labels landing in the device index) must print
the same transcript as the same source compiled against the reference headers
(oracle/_ref/pipeline_parity_ref, built by oracle/Makefile where /root/reference exists)."""
import pathlib
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parents[1]
REF_BIN = ROOT / "oracle" / "_ref" / "pipeline_parity_ref"
JSON_PARENT = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"


@pytest.fixture(scope="module")
def facade_bin(tmp_path_factory):
    exe = tmp_path_factory.mktemp("pipe") / "pipeline_parity"
    lib = ROOT / "paper_2508_08438_b200"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"), "-I", JSON_PARENT,
                    str(ROOT / "tests/cpp/pipeline_parity.cpp"), "-L", str(lib), "-lsafekv_b200",
                    f"-Wl,-rpath,{lib}", "-pthread", "-o", str(exe)], check=True)
    return exe


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("seed", [7, 2026])
def test_pipeline_transcript_matches_reference(gpu, facade_bin, seed, mode):
    if not REF_BIN.exists():
        pytest.skip("oracle/_ref/pipeline_parity_ref not built (needs /root/reference)")
    want = subprocess.run([str(REF_BIN), str(seed), str(mode)], capture_output=True, text=True, timeout=300)
    got = subprocess.run([str(facade_bin), str(seed), str(mode)], capture_output=True, text=True, timeout=600)
    assert want.returncode == 0 and got.returncode == 0, got.stderr[-2000:]
    w, g = want.stdout.splitlines(), got.stdout.splitlines()
    assert any(l.startswith("outcome") for l in w) and any("dropped" in l for l in w)
    for i, (a, b) in enumerate(zip(w, g)):
        assert a == b, f"line {i}: reference {a!r} != facade {b!r}"
    assert len(w) == len(g)
