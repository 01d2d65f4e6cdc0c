#!/usr/bin/env python
"""Golden fixture of the SURVEY A.8 evaluation leak flag for config 1, from the UNMODIFIED
reference (oracle/_ref/libsafekv_ref.so): block b of request i leaks iff its reference label
(cfg1_expected.npz, Appendix-A batch 1 and 2) is Public and safekv::block_truth(req_i, 16 b,
16 (b + 1)).sensitive_alone (workload.hpp:137-147; the leak accounting of serving_sim.hpp:385-392).

    make -C oracle ref && python tests/golden/make_leak_golden.py   ->  cfg1_leak.npz
"""
import ctypes as C
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from refh import load_ref  # noqa: E402


def main():
    L = load_ref()
    assert L is not None, "build the reference harness first: make -C oracle ref"
    L.ref_workload_block_truth.restype = None
    L.ref_workload_block_truth.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t,
                                           C.POINTER(C.c_int), C.POINTER(C.c_int)]
    err = C.create_string_buffer(256)
    w = L.ref_workload_generate(0, 4, 1000, 0.05, 0.0, 0.3, 0.0, 2, err, len(err))
    wl = np.load(HERE / "cfg1_workload.npz")
    e = np.load(HERE / "cfg1_expected.npz")
    off = wl["offsets"].astype(np.int64)
    alone, withc = C.c_int(), C.c_int()
    sens = []
    for i in range(len(off) - 1):
        for b in range((off[i + 1] - off[i]) // 16):
            L.ref_workload_block_truth(w, i, 16 * b, 16 * (b + 1), C.byref(alone), C.byref(withc))
            sens.append(alone.value)
    L.ref_workload_free(w)
    sens = np.array(sens, np.uint8)
    out = {f"r{r}_leak": ((e[f"r{r}_label"] == 1) & (sens == 1)).astype(np.uint8) for r in (1, 2)}
    out["sensitive_alone"] = sens
    np.savez_compressed(HERE / "cfg1_leak.npz", **out)
    print({k: int(v.sum()) for k, v in out.items()})


if __name__ == "__main__":
    main()
