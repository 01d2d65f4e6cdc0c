"""Stage-1/2 timing probe: repeated admits (no commit: the index keeps only the pool, so every
admit sees the same lookups) of one resident config-2 batch; prints the CUDA-event
hash_scan_ms of each admit (compare with an ncu launch list of this script).
SKV_HS_GENERAL=1 selects the general kernel (k_hash_scan) instead of k_hash_scan16."""
import sys, pathlib
import numpy as np
import torch
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2508_08438_b200 import AdmissionEngine, EngineConfig
from workload import GenSpec, generate, generate_pool
from paper_2508_08438_b200 import native as N

n = 65536
spec = GenSpec(n_prompts=n, prompt_tokens=2048, n_users=64, pool_size=256, pool_tokens=640, pii_per_kib=1.0, seed=1,
               prompt_id_base=100_000_000)
tok, off, users, owners = generate(spec)
dev = torch.device("cuda", 0)
t = torch.from_numpy(tok.view(np.int32)).to(dev)
o = torch.from_numpy(off.view(np.int64)).to(dev)
u = torch.from_numpy(users.view(np.int64)).to(dev)
w = torch.from_numpy(owners).to(dev)
cfg = EngineConfig(block_tokens=16, window_tokens=32, index_capacity=1 << 25, max_prompts=n, max_tokens=n * 2048,
                   max_window_entries=1 << 18)
with AdmissionEngine(cfg) as eng:
    eng.admit(*generate_pool(spec))
    eng.commit()
    b = N.Batch(t.data_ptr(), o.data_ptr(), u.data_ptr(), w.data_ptr(), n, n * 2048, 1)
    res = []
    for k in range(12):
        eng.admit_raw(b)
        res.append(eng.times()["hash_scan_ms"])
        if k % 4 == 3:
            eng.epoch_pass()
    print("hash_scan_ms", [round(x, 4) for x in res])
    print("median_ms", float(np.median(res[2:])))
