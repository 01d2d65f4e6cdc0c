"""Where the end-to-end (host-buffer) config-2 step goes: raw pinned H2D / D2H bandwidth, then
per step the host wall time of each C-ABI call (admit with host outputs, prefetch of the next
host batch, commit, epoch) and the device time of the prefetch (H2D + stages 1-2).
Diagnostic only (not a bench number)."""
import pathlib
import sys
import time

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2508_08438_b200 import AdmissionEngine, EngineConfig  # noqa: E402
from paper_2508_08438_b200 import native as N  # noqa: E402
from workload import GenSpec, generate, generate_pool  # noqa: E402

dev = torch.device("cuda", 0)
# raw copy bandwidth from / to pinned memory
for mb in (16, 134):
    h = torch.empty(mb << 20, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    h2d = 10 * (mb << 20) / (e0.elapsed_time(e1) / 1e3) / 1e9
    e0.record()
    for _ in range(10):
        h.copy_(d, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    d2h = 10 * (mb << 20) / (e0.elapsed_time(e1) / 1e3) / 1e9
    print(f"pinned copy {mb} MiB: H2D {h2d:.1f} GB/s, D2H {d2h:.1f} GB/s")

n = 65536
spec = GenSpec(n_prompts=n, prompt_tokens=2048, n_users=64, pool_size=256, pool_tokens=640, pii_per_kib=1.0, seed=1)
host = []
for k in range(8):
    spec.prompt_id_base = (k + 1) * 100_000_000
    tok, off, users, owners = generate(spec)
    t8 = torch.empty(len(tok), dtype=torch.uint8, pin_memory=True)
    t8.numpy()[:] = tok
    pins = [torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).pin_memory() for a in (off, users, owners)]
    host.append((t8, *pins))
pool = generate_pool(spec)
B = n * 128
out_label = torch.empty(B, dtype=torch.uint8, pin_memory=True)
out_dec = torch.empty(B, dtype=torch.uint8, pin_memory=True)
out_match = torch.empty(n, dtype=torch.int32, pin_memory=True)
out_tier = torch.empty(n, dtype=torch.uint8, pin_memory=True)


def hb(k):
    t8, off, users, owners = host[k]
    return N.Batch(None, off.data_ptr(), users.data_ptr(), owners.data_ptr(), n, n * 2048, 0, t8.data_ptr())


cfg = EngineConfig(block_tokens=16, window_tokens=32, index_capacity=1 << 28, max_prompts=n, max_tokens=n * 2048,
                   max_window_entries=1 << 18)
with AdmissionEngine(cfg) as eng:
    eng.admit(*pool)
    eng.commit()
    eng.epoch_pass()
    eng.stage_raw(hb(0))
    eng.stage_raw(hb(1))
    eng.prefetch_raw(hb(0))
    for k in range(7):
        o = N.AdmitOut(None, None, out_label.data_ptr(), None, out_dec.data_ptr(), out_match.data_ptr(),
                       out_tier.data_ptr(), None, 0, 0, 0)
        t = [time.perf_counter()]
        eng.admit_raw(hb(k), o)
        t.append(time.perf_counter())
        pf = eng.times()["hash_scan_ms"]
        eng.prefetch_raw(hb(k + 1))
        t.append(time.perf_counter())
        eng.commit()
        if k + 2 < 8:
            eng.stage_raw(hb(k + 2))
        t.append(time.perf_counter())
        eng.epoch_pass()
        t.append(time.perf_counter())
        d = np.diff(t) * 1e3
        print(f"step {k}: host ms admit {d[0]:.3f} prefetch {d[1]:.3f} commit {d[2]:.3f} epoch {d[3]:.3f} "
              f"total {sum(d):.3f} | prefetch of this batch (H2D + stages 1-2, device) {pf:.3f} ms")
