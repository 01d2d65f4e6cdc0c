"""Stage-1/2 timing probe: repeated admits of one resident config-2 batch; prints the
CUDA-event hash_scan_ms of each admit (compare with an ncu launch list of this script)."""
import sys, pathlib
import numpy as np
import torch
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2508_08438_b200 import AdmissionEngine, EngineConfig
from workload import GenSpec, generate, generate_pool
from paper_2508_08438_b200 import native as N

n = 65536
spec = GenSpec(n_prompts=n, prompt_tokens=2048, n_users=64, pool_size=256, pool_tokens=640, pii_per_kib=1.0, seed=1)
tok, off, users, owners = generate(spec)
dev = torch.device("cuda", 0)
t = torch.from_numpy(tok.view(np.int32)).to(dev)
o = torch.from_numpy(off.view(np.int64)).to(dev)
u = torch.from_numpy(users.view(np.int64)).to(dev)
w = torch.from_numpy(owners).to(dev)
cfg = EngineConfig(block_tokens=16, window_tokens=32, index_capacity=1 << 25, max_prompts=n, max_tokens=n * 2048,
                   max_window_entries=1 << 18)
with AdmissionEngine(cfg) as eng:
    b = N.Batch(t.data_ptr(), o.data_ptr(), u.data_ptr(), w.data_ptr(), n, n * 2048, 1)
    res = []
    for k in range(8):
        eng.admit_raw(b)
        eng.commit()
        eng.epoch_pass()
        res.append(eng.times()["hash_scan_ms"])
    print("hash_scan_ms", [round(x, 4) for x in res])
    res = []
    for k in range(4):
        eng.prefetch_raw(b)
        eng.admit_raw(b)
        eng.commit()
        eng.epoch_pass()
        res.append(eng.times()["hash_scan_ms"])
    print("prefetched hash_scan_ms", [round(x, 4) for x in res])
