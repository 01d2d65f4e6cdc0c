"""Eviction at config-2 scale: the per-batch cost of eviction bookkeeping (access epochs,
node ids) and the time of one evict() over the resulting index.  Prints one JSON line."""
import json, sys, pathlib, time
import numpy as np
import torch
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2508_08438_b200 import AdmissionEngine, EngineConfig
from workload import GenSpec, generate, generate_pool
from paper_2508_08438_b200 import native as N

n, nb_batches = 65536, 6
spec = GenSpec(n_prompts=n, prompt_tokens=2048, n_users=64, pool_size=256, pool_tokens=640, pii_per_kib=1.0, seed=1)
dev = torch.device("cuda", 0)
batches = []
for k in range(nb_batches):
    spec.prompt_id_base = (k + 1) * 100_000_000
    tok, off, users, owners = generate(spec)
    batches.append(tuple(torch.from_numpy(a.view(v)).to(dev) for a, v in
                         ((tok, np.int32), (off, np.int64), (users, np.int64), (owners, np.uint8))))
pool = generate_pool(spec)
out = {}
for evict_on in (False, True):
    cfg = EngineConfig(block_tokens=16, window_tokens=32, index_capacity=1 << 27, max_prompts=n,
                       max_tokens=n * 2048, max_window_entries=1 << 18)
    with AdmissionEngine(cfg) as eng:
        if evict_on:
            eng.enable_eviction()
        eng.admit(*pool); eng.commit(); eng.epoch_pass()
        ms = []
        for k in range(nb_batches):
            t, o, u, w = batches[k]
            b = N.Batch(t.data_ptr(), o.data_ptr(), u.data_ptr(), w.data_ptr(), n, n * 2048, 1)
            torch.cuda.synchronize(); t0 = time.perf_counter()
            eng.admit_raw(b); eng.commit(); eng.epoch_pass()
            torch.cuda.synchronize(); ms.append((time.perf_counter() - t0) * 1e3)
        out["step_ms_evict_" + ("on" if evict_on else "off")] = float(np.median(ms[1:]))
        if evict_on:
            live = eng.entry_count()
            torch.cuda.synchronize(); t0 = time.perf_counter()
            nev = eng.evict(live // 10)[0]
            torch.cuda.synchronize()
            out.update(evict_ms=(time.perf_counter() - t0) * 1e3, evicted=nev, live_entries=live,
                       index_slots=1 << 27)
print(json.dumps(out))
