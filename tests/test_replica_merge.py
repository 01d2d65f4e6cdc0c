"""CPU tests of the multi-GPU replicated layer's host logic:

* merge_replica's per-(entry, user) summaries -- lowest first prompt id, summed count -- replayed
  per entry in first-id order give exactly the AccessStats (access_stats.hpp:27-37, 64-user
  saturation included) of replaying every raw access in global order, whatever the split of the
  accesses over ranks;
* first-creator-wins across ranks (the lowest global prompt id per key);
* torch_allgather over a world-2 gloo job (two processes) returns every rank's records.
"""
import os
import pathlib
import socket
import subprocess
import sys

import numpy as np

from paper_2508_08438_b200 import REP_ACCESS, REP_ENTRY, merge_replica

ROOT = pathlib.Path(__file__).resolve().parents[1]


class Stats:  # restatement of AccessStats::record (test infrastructure)
    def __init__(self):
        self.hit, self.u, self.members = 0, 0, set()

    def record(self, user):
        self.hit += 1
        if user in self.members:
            return
        if len(self.members) < 64:
            self.members.add(user)
        self.u += 1


def replay_summaries(A):
    out = {}
    for r in A:
        k = (int(r["h"]), int(r["d"]))
        s = out.setdefault(k, Stats())
        s.hit += int(r["count"])
        u = int(r["user"])
        if u in s.members:
            continue
        if len(s.members) < 64:
            s.members.add(u)
            s.u += 1
        else:
            s.u += int(r["count"])
    return {k: (v.hit, v.u) for k, v in out.items()}


def test_access_summaries_replay_exactly():
    rng = np.random.default_rng(5)
    for trial in range(30):
        world = int(rng.integers(1, 5))
        n = int(rng.integers(1, 3000))
        keys = rng.integers(1, 6, n)            # few hot entries
        users = rng.integers(1, int(rng.integers(2, 200)), n)  # up to ~200 users -> saturation
        gids = np.sort(rng.choice(10 * n, n, replace=False))   # global prompt order
        ranks = rng.integers(0, world, n)
        truth = {}
        for k, u in zip(keys, users):
            truth.setdefault((int(k), 7), Stats()).record(int(u))
        truth = {k: (v.hit, v.u) for k, v in truth.items()}
        per_rank = []
        for r in range(world):
            sel = ranks == r
            agg = {}
            for k, u, g in zip(keys[sel], users[sel], gids[sel]):
                a = agg.setdefault((int(k), int(u)), [int(g), 0])
                a[0] = min(a[0], int(g))
                a[1] += 1
            arr = np.zeros(len(agg), REP_ACCESS)
            for i, ((k, u), (g, c)) in enumerate(agg.items()):
                arr[i] = (k, 7, u, g, c)
            per_rank.append(arr)
        _, A = merge_replica([], per_rank)
        assert replay_summaries(A) == truth, trial


def test_entries_first_creator_wins():
    rng = np.random.default_rng(6)
    E = []
    for r in range(3):
        e = np.zeros(4, REP_ENTRY)
        e["h"] = [1, 2, 3, 4]
        e["d"] = 9
        e["gid"] = rng.integers(0, 1000, 4)
        e["creator"] = 100 + r
        E.append(e)
    M, _ = merge_replica(E, [])
    assert len(M) == 4
    allg = np.stack([e["gid"] for e in E])
    for i in range(4):
        assert M["gid"][i] == allg[:, i].min()
        assert M["creator"][i] == 100 + int(np.argmin(allg[:, i]))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


WORKER = r'''
import sys, numpy as np, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
from paper_2508_08438_b200 import REP_ACCESS, torch_allgather
dist.init_process_group("gloo", init_method="env://")
r = dist.get_rank()
a = np.zeros(3 + 5 * r, REP_ACCESS); a["h"] = r + 1; a["count"] = np.arange(len(a))
got = torch_allgather()(a)
assert [len(x) for x in got] == [3, 8], [len(x) for x in got]
assert all((x["h"] == i + 1).all() for i, x in enumerate(got))
empty = torch_allgather()(np.zeros(0 if r == 0 else 2, REP_ACCESS))
assert [len(x) for x in empty] == [0, 2]
dist.destroy_process_group()
print("ok", r)
'''


def test_torch_allgather_gloo_world2(tmp_path):
    port = _free_port()
    src = tmp_path / "w.py"
    src.write_text(WORKER)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="2")
    ps = [subprocess.Popen([sys.executable, str(src), str(ROOT)], env=dict(env, RANK=str(r)), stdout=subprocess.PIPE,
                           stderr=subprocess.STDOUT) for r in range(2)]
    for p in ps:
        out, _ = p.communicate(timeout=300)
        assert p.returncode == 0, out.decode()[-2000:]
