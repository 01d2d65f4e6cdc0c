"""Multi-GPU partitioning (prefix-forest routing, skv_route) on CPU.

The multi-GPU design shards prompts by the root of their path in the prefix forest
(the key h_0 of the first full block): every index entry a prompt can match, insert,
record or relabel lies in that root's tree, so ranks own disjoint forests and the
admission path needs no data-path collective.  These tests check, with the C oracle as
the per-rank engine (test infrastructure), that the union of the per-rank results of a
world-size-2 `gloo` job equals one engine run over the whole batch sequence -- outputs
per prompt, index contents and monitor events -- and that the router and the routed
generator agree with their restatements.
"""
import os
import socket

import numpy as np
import pytest

from oracle_c import OracleEngine, lib as orc_lib
from paper_2508_08438_b200 import route, split_batch
from workload import GenSpec, generate
from workloads import make_batch, make_trunks

WORLD = 2
MASK = (1 << 64) - 1


def _rank_of_root_py(h0: int, world: int) -> int:
    z = (h0 + 0x9E3779B97F4A7C15) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    z ^= z >> 31
    return (z * world) >> 64


def test_route_matches_restatement():
    import ctypes as C
    L = orc_lib()
    L.orc_token_seq_digest.restype = C.c_uint64
    L.orc_token_seq_digest.argtypes = [C.c_void_p, C.c_size_t]
    L.orc_chain.restype = C.c_uint64
    L.orc_chain.argtypes = [C.c_uint64, C.c_uint64]
    rng = np.random.default_rng(3)
    tok, off, users, owners = make_batch(rng, make_trunks(rng, 8), 300, 4, wide_p=0.2)
    for world in (2, 3, 8):
        for B in (4, 16):
            ranks = route(tok, off, world, B)
            for p in range(len(off) - 1):
                a, b = int(off[p]), int(off[p + 1])
                if b - a < B:
                    exp = p % world
                else:
                    blk = np.ascontiguousarray(tok[a:a + B], np.uint32)
                    d0 = L.orc_token_seq_digest(blk.ctypes.data, B)
                    exp = _rank_of_root_py(L.orc_chain(0, d0), world)
                assert ranks[p] == exp
    # prompts sharing a first block always land together
    ranks = route(tok, off, 8, 16)
    first = {}
    for p in range(len(off) - 1):
        a, b = int(off[p]), int(off[p + 1])
        if b - a >= 16:
            k = tok[a:a + 16].tobytes()
            assert first.setdefault(k, ranks[p]) == ranks[p]


def test_routed_generator_is_a_filter_of_the_global_sequence():
    base = GenSpec(n_prompts=400, prompt_tokens=96, n_users=8, pool_size=6, pool_tokens=40, shared_fraction=0.7,
                   pii_per_kib=8.0, seed=9, prompt_id_base=1000)
    tok, off, users, owners, ids = generate(base, return_ids=True)
    np.testing.assert_array_equal(ids, np.arange(1000, 1400, dtype=np.uint64))
    ranks = route(tok, off, 3, 16, prompt_ids=ids)
    for r in range(3):
        want = np.flatnonzero(ranks == r)[:50]
        spec = GenSpec(**{**base.__dict__, "n_prompts": 50, "route_world": 3, "route_rank": r,
                          "route_block_tokens": 16})
        t2, o2, u2, w2, i2 = generate(spec, return_ids=True)
        np.testing.assert_array_equal(i2, ids[want])
        st, so, su, sw = split_batch(tok, off, users, owners, ranks, r)
        n_tok = int(so[len(want)])
        np.testing.assert_array_equal(t2, st[:n_tok])
        np.testing.assert_array_equal(u2, su[:len(want)])


def _batches(seed, n_batches, n_prompts, n_users):
    rng = np.random.default_rng(seed)
    trunks = make_trunks(rng, 16)
    return [make_batch(rng, trunks, n_prompts, n_users) for _ in range(n_batches)]


def _run(batches, B, W, rank=None, world=1, epoch_every=1):
    """Engine over the batches (or over this rank's routed share of each).  Returns
    per-prompt outputs keyed by global (batch, prompt), events per epoch, and the export."""
    eng = OracleEngine(B=B, W=W, jump=0.3, u_pre_max=1)
    per_prompt, events = {}, []
    try:
        for k, (tok, off, users, owners) in enumerate(batches):
            n = len(off) - 1
            if world > 1:
                ranks = route(tok, off, world, B)
                sel = np.flatnonzero(ranks == rank)
                sub = split_batch(tok, off, users, owners, ranks, rank)
            else:
                sel = np.arange(n)
                sub = (tok, off, users, owners)
            o = eng.admit(*sub)
            nb = ((sub[1][1:] - sub[1][:-1]) // B).astype(np.int64)
            bo = np.concatenate([[0], np.cumsum(nb)])
            for j, p in enumerate(sel):
                s, e = bo[j], bo[j + 1]
                per_prompt[(k, int(p))] = (int(o["matched_blocks"][j]), int(o["lowest_tier"][j]),
                                           o["block_h"][s:e].tolist(), o["mask"][s:e].tolist(),
                                           o["label"][s:e].tolist(), o["decision"][s:e].tolist())
            eng.commit()
            if (k + 1) % epoch_every == 0:
                ep, ev = eng.epoch()
                events.append((ep, ev))
        exp = eng.export()
    finally:
        eng.close()
    return per_prompt, events, {k: v.tolist() for k, v in exp.items()}


def _merge(results):
    per_prompt, events, export = {}, None, None
    for pp, ev, ex in results:
        per_prompt.update(pp)
        if events is None:
            events = [(ep, list(e)) for ep, e in ev]
            export = {k: list(v) for k, v in ex.items()}
        else:
            for i, (ep, e) in enumerate(ev):
                assert events[i][0] == ep  # epochs advance in lock step
                events[i][1].extend(e)
            for k in export:
                export[k].extend(ex[k])
    events = [(ep, sorted(e)) for ep, e in events]  # skv_epoch order: by (h, d)
    order = sorted(range(len(export["h"])), key=lambda i: (export["h"][i], export["d"][i]))
    export = {k: [v[i] for i in order] for k, v in export.items()}
    return per_prompt, events, export


def _worker(rank, world, port, seed, out_dir):
    import pickle

    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = _run(_batches(seed, 8, 120, 3), B=4, W=8, rank=rank, world=world)
        gathered = [None] * world
        dist.all_gather_object(gathered, res)
        if rank == 0:
            with open(os.path.join(out_dir, "merged.pkl"), "wb") as f:
                pickle.dump(_merge(gathered), f)
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("seed", [101, 102])
def test_gloo_world2_partition_equals_single_engine(tmp_path, seed):
    import pickle

    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(WORLD, _free_port(), seed, str(tmp_path)), nprocs=WORLD, join=True)
    with open(tmp_path / "merged.pkl", "rb") as f:
        per_prompt, events, export = pickle.load(f)
    pp1, ev1, ex1 = _run(_batches(seed, 8, 120, 3), B=4, W=8)
    assert per_prompt == pp1
    assert [(ep, sorted(e)) for ep, e in ev1] == events
    assert sum(len(e) for _, e in events) > 0  # the scenario exercises the monitor
    assert ex1 == export


def test_partition_in_process_many_ranks():
    """Same property for world sizes 3 and 8 (in-process), epochs every other batch."""
    batches = _batches(7, 6, 200, 6)
    single = _run(batches, B=4, W=8, epoch_every=2)
    for world in (3, 8):
        merged = _merge([_run(batches, B=4, W=8, rank=r, world=world, epoch_every=2) for r in range(world)])
        assert merged[0] == single[0]
        assert merged[1] == [(ep, sorted(e)) for ep, e in single[1]]
        assert merged[2] == single[2]
