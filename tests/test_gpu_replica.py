"""The multi-GPU replicated layer on the CUDA path: entries at depth < D are
replicated on every rank, deeper ones owned by the rank skv_route_depth picks; after every commit
the ranks all-gather their replicated-layer exports (new entries, per (entry, user) accesses) and
apply the same merge.  A system-prompt stream (one dominant shared root) is split over 2 and 3
ranks: every rank's admit outputs, the merged epoch events and the union of the ranks' index
dumps must equal one engine over the whole stream -- and the unmodified reference.

  * in-process: the ranks are engines of one process on cuda:0, allgather = a list;
  * multi-process: world-2 torch.distributed (gloo) job, one process per rank sharing cuda:0,
    allgather = paper_2508_08438_b200.torch_allgather (the bench uses the same code over NCCL).
"""
import json
import os
import pathlib
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_2508_08438_b200 import AdmissionEngine, EngineConfig, merge_entries, merge_events, merge_replica, route
from refh import RefEngine, RefRules
from replica_harness import ref_rows, replica_stream, split, union_exports
from test_gpu_parity import check_events

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parents[1]


def _cfg(B, W):
    return EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 16, max_prompts=1024,
                        max_tokens=1 << 18, max_window_entries=1 << 14, u_pre_max=3, entropy_jump=0.1)


def _run_world(ref, world, depth, B=4, W=8, seed=71, n_batches=5, n_prompts=120, n_users=90, mode="raw_host"):
    stream = replica_stream(seed, n_batches, n_prompts, n_users, B)
    engines = [AdmissionEngine(_cfg(B, W)) for _ in range(world)]
    single = AdmissionEngine(_cfg(B, W))
    re_ = RefEngine(ref, RefRules(ref), B=B, W=W, jump=0.1, u_pre_max=3)
    try:
        for e in engines:
            e.set_replicated_depth(depth)
        sizes = []
        for k, batch in enumerate(stream):
            parts = split(batch, world, B, depth, route)
            sizes.append([len(p[5]) for p in parts])
            full = single.admit(*batch[:4])
            exp = re_.admit(*batch[:4])
            np.testing.assert_array_equal(full.matched_blocks, exp["matched_blocks"])
            for e, (t, o, u, w, g, sel) in zip(engines, parts):
                got = e.admit(t, o, u, w)
                np.testing.assert_array_equal(got.matched_blocks, full.matched_blocks[sel])
                np.testing.assert_array_equal(got.lowest_tier, full.lowest_tier[sel])
                # per-block outputs: the rank's prompts' blocks in the single engine's layout
                blk = np.concatenate([np.arange(full.block_offsets[p], full.block_offsets[p + 1]) for p in sel]
                                     ) if len(sel) else np.zeros(0, np.int64)
                for f in ("block_h", "block_d", "label", "decision", "rule_mask"):
                    np.testing.assert_array_equal(getattr(got, f), getattr(full, f)[blk], f)
            single.commit()
            re_.commit()
            exports = []
            for e, part in zip(engines, parts):
                e.commit()
                exports.append(e.replica_export(part[4], device=(mode == "raw_device")))
            E = merge_entries([x[0] for x in exports])
            if mode == "merged_host":  # merged on the host: the device merge must be idempotent
                A = merge_replica([], [x[1] for x in exports])[1]
            elif mode == "raw_host":
                A = np.concatenate([x[1] for x in exports])
            else:
                import torch
                A = torch.cat([x[1] for x in exports])
            for e in engines:
                e.replica_apply(E, A)
            ev_r = re_.epoch(cap=1 << 16)[1]
            ev_s = single.epoch_pass()[1]
            ev_w = merge_events([e.epoch_pass()[1] for e in engines])
            check_events(ev_s, ev_r)
            check_events(ev_w, ev_r)
            rows = union_exports([e.export() for e in engines])
            assert rows == ref_rows(re_.export())
        return sizes
    finally:
        for e in engines + [single]:
            e.close()
        re_.close()


@pytest.mark.parametrize("world,depth,mode", [(2, 8, "merged_host"), (3, 8, "raw_host"), (2, 44, "raw_device"),
                                              (3, 44, "raw_device"), (4, 1, "raw_host")])
def test_replicated_layer_in_process(ref, gpu, world, depth, mode):
    sizes = _run_world(ref, world, depth, mode=mode)
    # depth 44 > the shared system prompt (41.75 blocks at B=4): it no longer sends everything to one rank
    if depth == 44:
        assert all(min(s) > 0.2 * sum(s) / world for s in sizes), sizes


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_replicated_layer_world2_processes(ref, gpu, tmp_path):
    """Two processes (gloo, one rank per process, both on cuda:0) run the protocol through
    torch_allgather; rank 0 checks the merged results against the reference."""
    port = _free_port()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="2")
    procs = []
    for r in range(2):
        out = tmp_path / f"rank{r}.json"
        procs.append((subprocess.Popen([sys.executable, str(ROOT / "tests" / "replica_worker.py"), str(out)],
                                       env=dict(env, RANK=str(r), LOCAL_RANK=str(r)), cwd=ROOT,
                                       stdout=subprocess.PIPE, stderr=subprocess.STDOUT), out))
    for p, out in procs:
        o, _ = p.communicate(timeout=600)
        assert p.returncode == 0, o.decode()[-3000:]
    res = json.loads((tmp_path / "rank0.json").read_text())
    assert res["ok"], res
    assert res["batches"] == 5 and min(res["sizes"]) > 0
