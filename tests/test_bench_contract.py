"""The bench.py JSON contract: the reference arm runs on the host (CPU test, a tiny
sample), our arm on the GPU (a reduced batch via --prompts); both print one line with
the keys the driver reads."""
import json
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_contract(ref):
    j = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-sample", "32"], 600)
    if "unavailable" in j:
        pytest.skip(j["unavailable"])
    assert BASE_KEYS <= set(j) and j["impl"] == "reference"
    assert j["value"] > 0 and j["unit"] == "blocks/s" and j["higher_is_better"] is True
    assert j["cpu_baseline"]["kind"] == "reference" and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["value"] == j["value"]


@pytest.mark.gpu
def test_our_arm_contract(gpu):
    j = _run(["--steps", "3", "--warmup", "3", "--prompts", "4096", "--no-cpu-baseline"], 900)
    assert BASE_KEYS <= set(j) and "impl" not in j
    assert j["value"] > 0 and j["n_gpus"] == 1 and j["steps"] == 3 and j["warmup"] == 3
    r = j["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5 and r["peak"] > 0
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    e = j["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert j["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(j["clocks"])
