"""Prefix-forest partitioning on the CUDA path: `world` engines (one per would-be GPU,
here all on cuda:0), each admitting its skv_route share of every batch, together equal
one engine over the whole batches -- per-prompt outputs, index exports and events."""
import numpy as np
import pytest

from paper_2508_08438_b200 import AdmissionEngine, EngineConfig, route, split_batch
from workloads import make_batch, make_trunks

pytestmark = pytest.mark.gpu


def _cfg(B, W):
    return EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 18, max_prompts=4096,
                        max_tokens=1 << 20, max_window_entries=1 << 15, entropy_jump=0.3, u_pre_max=1)


def _prompt_rows(res, B, offsets, sel):
    nb = ((offsets[1:] - offsets[:-1]) // B).astype(np.int64)
    bo = np.concatenate([[0], np.cumsum(nb)])
    rows = {}
    for j, p in enumerate(sel):
        s, e = bo[j], bo[j + 1]
        rows[int(p)] = (int(res.matched_blocks[j]), int(res.lowest_tier[j]), res.block_h[s:e].tolist(),
                        res.rule_mask[s:e].tolist(), res.label[s:e].tolist(), res.decision[s:e].tolist())
    return rows


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_engines_equal_single_engine(gpu, world):
    B, W = 4, 8
    rng = np.random.default_rng(200 + world)
    trunks = make_trunks(rng, 16)
    batches = [make_batch(rng, trunks, 200, 3) for _ in range(6)]
    single = AdmissionEngine(_cfg(B, W))
    parts = [AdmissionEngine(_cfg(B, W)) for _ in range(world)]
    fired = 0
    try:
        for k, (tok, off, users, owners) in enumerate(batches):
            r1 = single.admit(tok, off, users, owners)
            want = _prompt_rows(r1, B, off, np.arange(len(off) - 1))
            ranks = route(tok, off, world, B)
            got = {}
            for r, eng in enumerate(parts):
                sub = split_batch(tok, off, users, owners, ranks, r)
                got.update(_prompt_rows(eng.admit(*sub), B, sub[1], np.flatnonzero(ranks == r)))
            assert got == want
            single.commit()
            for eng in parts:
                eng.commit()
            ep1, ev1 = single.epoch_pass()
            evs = []
            for eng in parts:
                ep, ev = eng.epoch_pass()
                assert ep == ep1
                evs.extend(ev)
            key = lambda e: (e.h, e.d)
            assert sorted(((e.h, e.d, e.action, e.entropy_now, e.entropy_prev, e.u_pre) for e in evs)) == \
                [(e.h, e.d, e.action, e.entropy_now, e.entropy_prev, e.u_pre) for e in sorted(ev1, key=key)]
            fired += len(ev1)
            x1 = single.export()
            xs = np.concatenate([eng.export() for eng in parts])
            xs.sort(order=["h", "d"])
            np.testing.assert_array_equal(xs, x1)
        assert fired > 0
    finally:
        single.close()
        for eng in parts:
            eng.close()
