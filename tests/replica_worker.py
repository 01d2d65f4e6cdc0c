"""One rank of the world-2 replicated-layer test (tests/test_gpu_replica.py): torch.distributed
(gloo) process, CUDA engine on cuda:0, ReplicaGroup over torch_allgather.  Rank 0 also runs the
unmodified reference over the whole stream and compares the merged events and the union of the
ranks' index dumps with it; writes {"ok": ...} to argv[1]."""
import json
import os
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2508_08438_b200 import (AdmissionEngine, EngineConfig, ReplicaGroup, merge_events, route,  # noqa: E402
                                   torch_allgather)
from replica_harness import ref_rows, replica_stream, split, union_exports  # noqa: E402

B, W, DEPTH = 4, 8, 44


def main(out_path):
    dist.init_process_group("gloo", init_method="env://")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 16, max_prompts=1024,
                       max_tokens=1 << 18, max_window_entries=1 << 14, u_pre_max=3, entropy_jump=0.1)
    stream = replica_stream(91, 5, 120, 90, B)
    res = {"ok": True, "batches": 0, "sizes": []}
    with AdmissionEngine(cfg) as eng:
        grp = ReplicaGroup(eng, DEPTH, torch_allgather())
        ref = None
        if rank == 0:
            from refh import RefEngine, RefRules, load_ref
            L = load_ref()
            ref = RefEngine(L, RefRules(L), B=B, W=W, jump=0.1, u_pre_max=3)
        for batch in stream:
            parts = split(batch, world, B, DEPTH, route)
            t, o, u, w, g, sel = parts[rank]
            got = eng.admit(t, o, u, w)
            eng.commit()
            grp.sync(g)
            _, ev = eng.epoch_pass()
            evs = [None] * world
            dist.all_gather_object(evs, [(e.h, e.d, e.action, e.entropy_now, e.entropy_prev, e.u_pre) for e in ev])
            dumps = [None] * world
            ex = eng.export()
            dist.all_gather_object(dumps, ex.tobytes())
            matched = [None] * world
            dist.all_gather_object(matched, (sel.tolist(), got.matched_blocks.tolist()))
            if rank == 0:
                exp = ref.admit(*batch[:4])
                ref.commit()
                _, ev_r = ref.epoch(cap=1 << 16)
                m = np.zeros(len(batch[4]), np.int64)
                for s_, mb in matched:
                    m[np.asarray(s_, np.int64)] = mb
                ok_m = np.array_equal(m, exp["matched_blocks"].astype(np.int64))
                merged = sorted({(e[0], e[1]): e for es in evs for e in es}.values())
                ok_e = [(e[0], e[1], e[2], e[5]) for e in merged] == [(e[0], e[1], e[2], e[5]) for e in ev_r] and \
                    all(abs(a[3] - b[3]) <= 1e-6 * abs(b[3]) and abs(a[4] - b[4]) <= 1e-6 * abs(b[4])
                        for a, b in zip(merged, ev_r))
                rows = union_exports([np.frombuffer(d, dtype=ex.dtype) for d in dumps])
                ok_i = rows == ref_rows(ref.export())
                res["ok"] = bool(res["ok"] and ok_m and ok_e and ok_i)
                res.setdefault("detail", []).append({"matched": bool(ok_m), "events": bool(ok_e), "index": bool(ok_i),
                                                     "n_events": len(ev_r)})
                res["sizes"].append(min(len(p[5]) for p in parts))
            res["batches"] += 1
        if ref is not None:
            ref.close()
    dist.barrier()
    dist.destroy_process_group()
    pathlib.Path(out_path).write_text(json.dumps(res))


if __name__ == "__main__":
    main(sys.argv[1])
