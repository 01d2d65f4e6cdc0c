"""CPU tests of the drop-in boundary: the C-ABI library loads, exports exactly the entry
points include/safekv_b200.h declares, host-only entry points work, and the device
entry points fail loudly (no CPU fallback) when no GPU is present."""
import ctypes as C
import pathlib
import re

import numpy as np
import pytest

from conftest import gpu_available
from paper_2508_08438_b200 import native as N
from paper_2508_08438_b200 import AdmissionEngine, CudaError
from workload import GenSpec, generate, generate_pool

ROOT = pathlib.Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "safekv_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(skv_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = N.load_library()
    decl = declared_symbols()
    assert len(decl) >= 25
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(N.SIGNATURES) == decl  # the binding covers the whole ABI


def test_struct_layouts_match_header(tmp_path):
    """Every ctypes mirror has the size and field offsets the C compiler gives the header."""
    import subprocess
    pairs = {"skv_event": N.Event, "skv_entry": N.Entry, "skv_config": N.Config, "skv_batch": N.Batch,
             "skv_admit_out": N.AdmitOut, "skv_stage_times": N.StageTimes,
             "skv_dfa_view": N.DfaView, "skv_cost_model": N.CostModel, "skv_rep_entry": N.RepEntry,
             "skv_rep_access": N.RepAccess}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "safekv_b200.h"', "int main(void){"]
    for cname, cls in pairs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            if f == "pad":
                continue
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for cname, cls in pairs.items():
        assert int(got[cname]) == C.sizeof(cls), cname
        for f, _ in cls._fields_:
            if f != "pad":
                assert int(got[f"{cname}.{f}"]) == getattr(cls, f).offset, f"{cname}.{f}"


def test_generator_struct_layout(tmp_path):
    """workload/skv_gen.h's spec struct matches its ctypes mirror."""
    import subprocess
    import workload as W
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "skv_gen.h"', "int main(void){",
             'printf("size %zu\\n", sizeof(skvgen_spec));']
    for f, _ in W._Spec._fields_:
        lines.append(f'printf("{f} %zu\\n", offsetof(skvgen_spec, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "gl.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "gl"
    subprocess.run(["gcc", "-I", str(ROOT / "workload"), str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    assert int(got["size"]) == C.sizeof(W._Spec)
    for f, _ in W._Spec._fields_:
        assert int(got[f]) == getattr(W._Spec, f).offset, f


def test_generator_is_not_in_the_product_library():
    """The bench/test generator lives in workload/ (and oracle/_ref for the reference arm),
    never in the product library."""
    lib = N.load_library()
    for name in ("skvgen_generate", "skv_generate", "skv_generate_pool"):
        assert not hasattr(lib, name), name


def test_reference_arm_generator_is_identical(ref):
    """The reference arm binds the generator from oracle/_ref/libsafekv_ref.so (compiled from
    the same source): both produce the same bytes."""
    import importlib
    import workload as W
    spec = GenSpec(n_prompts=40, prompt_tokens=2048, seed=7, prompt_id_base=123456)
    a = generate(spec)
    try:
        W.use_library(ROOT / "oracle" / "_ref" / "libsafekv_ref.so")
        b = generate(spec)
        pa = generate_pool(spec)
    finally:
        W.use_library()
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    for x, y in zip(pa, generate_pool(spec)):
        np.testing.assert_array_equal(x, y)


def test_no_cpu_fallback_without_gpu():
    if gpu_available():
        pytest.skip("GPU present")
    with pytest.raises(CudaError, match="no CUDA device"):
        AdmissionEngine(block_tokens=16)


def test_config_validation_precedes_device():
    from paper_2508_08438_b200 import ConfigError
    with pytest.raises(ConfigError):
        AdmissionEngine(block_tokens=0)


def test_generator_is_deterministic_and_shardable():
    spec = GenSpec(n_prompts=64, prompt_tokens=2048, seed=5)
    a = generate(spec)
    b = generate(spec, nthreads=3)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    half = GenSpec(n_prompts=32, prompt_tokens=2048, seed=5, prompt_id_base=32)
    c = generate(half)
    np.testing.assert_array_equal(c[0], a[0][32 * 2048:])
    np.testing.assert_array_equal(c[2], a[2][32:])
    tok = a[0].reshape(64, 2048)
    pool = generate_pool(spec)[0].reshape(256, 640)
    # every prompt starts with one of the pool prefixes (shared_fraction = 1)
    keys = {row.tobytes() for row in pool}
    assert all(row[:640].tobytes() in keys for row in tok)
    assert tok.max() < 256


def test_generator_primitives_match_reference(ref):
    """filler / make_secret restated from workload.hpp:155-266: the pool prefix of a
    reference-seeded SplitMix64 matches the reference generator byte for byte."""
    import ctypes as C2
    L = ref
    L.ref_filler.restype = C2.c_size_t
    L.ref_filler.argtypes = [C2.c_uint64, C2.c_size_t, C2.POINTER(C2.c_uint64), C2.c_char_p]
    L.ref_derive_seed.restype = C2.c_uint64
    L.ref_derive_seed.argtypes = [C2.c_uint64, C2.c_uint64]
    spec = GenSpec(n_prompts=1, prompt_tokens=2048, seed=1, pool_size=4, pool_tokens=640)
    pool = generate_pool(spec)[0].reshape(4, 640)
    for i in range(4):
        seed = C2.c_uint64(L.ref_derive_seed(1, 0x706F6F6C00000000 + i))
        buf = C2.create_string_buffer(640)
        L.ref_filler((1 << 40) + i, 640, C2.byref(seed), buf)
        assert pool[i].astype(np.uint8).tobytes() == buf.raw[:640]
