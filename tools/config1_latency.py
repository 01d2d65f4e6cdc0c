"""Config 1 (BASELINE.json configs[0]: the smallest preset, 1,000 x 112-token prompts, 4 users,
7,000 blocks) is latency-bound: report microseconds per batch (device-resident inputs, CUDA
events around admit + commit + epoch), cold index (first batch) and warm (the same batch
again).  Inputs are the committed golden workload (tests/golden/cfg1_workload.npz, data only)."""
import json, pathlib, sys
import numpy as np
import torch
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2508_08438_b200 import AdmissionEngine, EngineConfig
from paper_2508_08438_b200 import native as N

w = np.load(ROOT / "tests" / "golden" / "cfg1_workload.npz")
dev = torch.device("cuda", 0)
tok = torch.from_numpy(w["tokens"].astype(np.uint32).view(np.int32)).to(dev)
off = torch.from_numpy(w["offsets"].astype(np.uint64).view(np.int64)).to(dev)
usr = torch.from_numpy(w["users"].astype(np.uint64).view(np.int64)).to(dev)
own = torch.from_numpy(w["owners"].astype(np.uint8)).to(dev)
n = len(w["offsets"]) - 1
cfg = EngineConfig(block_tokens=16, window_tokens=32, index_capacity=1 << 18, max_prompts=4096, max_tokens=1 << 20,
                   max_window_entries=1 << 15)
REPS = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 25
SKIP = 5 if REPS > 5 else 0
cold, warm = [], []
for rep in range(REPS):
    with AdmissionEngine(cfg) as eng:
        s = torch.cuda.ExternalStream(eng.stream)
        b = N.Batch(tok.data_ptr(), off.data_ptr(), usr.data_ptr(), own.data_ptr(), n, int(w["offsets"][-1]), 1)
        for out in (cold, warm):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            eng.admit_raw(b)
            eng.commit()
            eng.epoch_pass()
            e1.record(s)
            torch.cuda.synchronize()
            if rep >= SKIP:
                out.append(e0.elapsed_time(e1) * 1e3)
print(json.dumps({"workload": "config 1: 1000 x 112-token prompts (golden), B=16, W=32", "blocks": 7000,
                  "us_per_batch_cold_index": float(np.median(cold)), "us_per_batch_warm_index": float(np.median(warm))}))
