"""Cost of the replicated-layer sync per step: `world` engines in one
process on cuda:0 each admit their routed share of a workload batch, commit, then export / merge /
apply; prints the wall time of each phase (median over steps).  The all-gather is a host list here
(the bench uses NCCL device all-gathers); export and apply are the product calls."""
import sys, pathlib, time, json
import numpy as np
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench
from paper_2508_08438_b200 import AdmissionEngine, EngineConfig, merge_entries, split_batch
from workload import generate_pool, route

wl = int(sys.argv[1]) if len(sys.argv) > 1 else 6
world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
c = dict(bench.CONFIGS[wl], n_prompts=n)
D = c.get("rep_depth", 1)
B = c["block_tokens"]
cfg = EngineConfig(block_tokens=B, window_tokens=c["window_tokens"], index_capacity=1 << 26, max_prompts=n,
                   max_tokens=n * c["prompt_tokens"], max_window_entries=1 << 18)
engs = [AdmissionEngine(cfg) for _ in range(world)]
for e in engs:
    e.set_replicated_depth(D)
spec = bench.gen_spec(c, n)
pt, po, pu, pw = generate_pool(spec)
pr = route(pt, po, world, B, depth=D)
def step(tok, off, users, owners, gids):
    ranks = route(tok, off, world, B, prompt_ids=gids, depth=D)
    T = {}
    exps = []
    for r, e in enumerate(engs):
        sub = split_batch(tok, off, users, owners, ranks, r)
        e.admit(*sub)
        e.commit()
    t0 = time.perf_counter()
    for r, e in enumerate(engs):
        exps.append(e.replica_export(gids[ranks == r]))
    t1 = time.perf_counter()
    E = merge_entries([x[0] for x in exps])
    A = np.concatenate([x[1] for x in exps])
    t2 = time.perf_counter()
    for e in engs:
        e.replica_apply(E, A)
    t3 = time.perf_counter()
    for e in engs:
        e.epoch_pass()
    return {"export_ms": 1e3 * (t1 - t0) / world, "merge_ms": 1e3 * (t2 - t1), "apply_ms": 1e3 * (t3 - t2) / world,
            "n_ent": len(E), "n_acc": len(A)}
step(pt, po, pu, pw, np.arange(len(po) - 1, dtype=np.uint64))
res = []
for k in range(6):
    tok, off, users, owners, gids = bench.build_batch(c, wl, k, n, spec=spec)
    res.append(step(tok, off, users, owners, gids))
print(json.dumps({k: float(np.median([r[k] for r in res[1:]])) for k in res[0]}))
