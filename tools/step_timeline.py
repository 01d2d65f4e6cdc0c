"""Host-side timeline of the config-2 step (admit / prefetch / commit / epoch): host
wall time of each call and device time between CUDA events recorded after each call, to
see where the device idles on host synchronisation.  Diagnostic only."""
import sys, pathlib, time
import numpy as np
import torch
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2508_08438_b200 import AdmissionEngine, EngineConfig
from workload import GenSpec, generate, generate_pool
from paper_2508_08438_b200 import native as N

n = 65536
spec = GenSpec(n_prompts=n, prompt_tokens=2048, n_users=64, pool_size=256, pool_tokens=640, pii_per_kib=1.0, seed=1)
dev = torch.device("cuda", 0)
batches = []
for k in range(6):
    spec.prompt_id_base = (k + 1) * 100_000_000
    tok, off, users, owners = generate(spec)
    batches.append(tuple(torch.from_numpy(a.view(v)).to(dev) for a, v in
                         ((tok, np.int32), (off, np.int64), (users, np.int64), (owners, np.uint8))))
pool = generate_pool(spec)
cfg = EngineConfig(block_tokens=16, window_tokens=32, index_capacity=1 << 28, max_prompts=n, max_tokens=n * 2048,
                   max_window_entries=1 << 18)
with AdmissionEngine(cfg) as eng:
    eng.admit(*pool); eng.commit(); eng.epoch_pass()
    st = torch.cuda.Stream(device=dev, priority=0)
    def b(k):
        t, o, u, w = batches[k]
        return N.Batch(t.data_ptr(), o.data_ptr(), u.data_ptr(), w.data_ptr(), n, n * 2048, 1)
    s = torch.cuda.ExternalStream(eng.stream)
    for k in range(5):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        h = []
        ev[0].record(s); t0 = time.perf_counter()
        eng.admit_raw(b(k)); h.append(time.perf_counter() - t0); ev[1].record(s)
        t0 = time.perf_counter(); eng.prefetch_raw(b(k + 1)); h.append(time.perf_counter() - t0)
        t0 = time.perf_counter(); eng.commit(); h.append(time.perf_counter() - t0); ev[2].record(s)
        t0 = time.perf_counter(); eng.epoch_pass(); h.append(time.perf_counter() - t0); ev[3].record(s)
        torch.cuda.synchronize()
        d = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
        print(f"step {k}: host ms admit {h[0]*1e3:.3f} prefetch {h[1]*1e3:.3f} commit {h[2]*1e3:.3f} epoch {h[3]*1e3:.3f} | "
              f"device ms admit {d[0]:.3f} commit {d[1]:.3f} epoch {d[2]:.3f} total {sum(d):.3f}")
