"""Host-side timeline of small-batch steps (config 1: the committed golden 1,000 x 112-token
workload, re-admitted on a warm index; config 5 shape: 4,096 x 2,048 tokens): host wall time of
each C-ABI call (through the Python binding) and device time between CUDA events recorded after
each call, to see whether the step is bound by its kernels or by host issue / synchronisation.
Diagnostic only (not a bench line)."""
import json, pathlib, sys, time
import numpy as np
import torch
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2508_08438_b200 import AdmissionEngine, EngineConfig
from paper_2508_08438_b200 import native as N

dev = torch.device("cuda", 0)


def run(name, tok, off, usr, own, steps=30, fresh=False, batches=None):
    n = len(off) - 1
    cfg = EngineConfig(block_tokens=16, window_tokens=32, index_capacity=1 << 24, max_prompts=max(n, 4096),
                       max_tokens=max(int(off[-1]), 1 << 20), max_window_entries=1 << 20)
    tk = [torch.from_numpy(t.astype(np.uint32).view(np.int32)).to(dev) for t in (batches or [tok])]
    of = torch.from_numpy(off.astype(np.uint64).view(np.int64)).to(dev)
    us = torch.from_numpy(usr.astype(np.uint64).view(np.int64)).to(dev)
    ow = torch.from_numpy(own.astype(np.uint8)).to(dev)
    rows = []
    with AdmissionEngine(cfg) as eng:
        s = torch.cuda.ExternalStream(eng.stream)
        for k in range(steps):
            t = tk[k % len(tk)]
            b = N.Batch(t.data_ptr(), of.data_ptr(), us.data_ptr(), ow.data_ptr(), n, int(off[-1]), 1)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            torch.cuda.synchronize()
            h = []
            ev[0].record(s); t0 = time.perf_counter()
            eng.admit_raw(b); h.append(time.perf_counter() - t0); ev[1].record(s)
            t0 = time.perf_counter(); eng.commit(); h.append(time.perf_counter() - t0); ev[2].record(s)
            t0 = time.perf_counter(); eng.epoch_pass(); h.append(time.perf_counter() - t0); ev[3].record(s)
            torch.cuda.synchronize()
            d = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
            if k >= 5:
                rows.append(h + d)
    r = np.median(np.array(rows), axis=0)
    out = {"workload": name, "host_us": {"admit": r[0] * 1e6, "commit": r[1] * 1e6, "epoch": r[2] * 1e6},
           "device_us": {"admit": r[3] * 1e3, "commit": r[4] * 1e3, "epoch": r[5] * 1e3},
           "step_device_us": float(sum(r[3:]) * 1e3), "step_host_us": float(sum(r[:3]) * 1e6)}
    print(json.dumps(out))


w = np.load(ROOT / "tests" / "golden" / "cfg1_workload.npz")
run("config 1 (golden, warm index)", w["tokens"], w["offsets"], w["users"], w["owners"])
rng = np.random.default_rng(5)
n, L = 4096, 2048
off = np.arange(n + 1, dtype=np.uint64) * L
usr = (np.arange(n) % 64 + 1).astype(np.uint64)
bs = [rng.integers(97, 123, n * L).astype(np.uint32) for _ in range(4)]
run("config-5 shape (4,096 x 2,048, fresh batches)", bs[0], off, usr, np.zeros(n, np.uint8), steps=24, batches=bs)
