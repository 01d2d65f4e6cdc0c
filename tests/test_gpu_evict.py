"""GPU parity of eviction (RadixCacheIndex::evict / select_victim, cache_index.hpp:281-292,
697-728, untiered): after batches spread over several monitor epochs (distinct access
epochs), tier demotions (off-HBM entries never leave and pin their ancestors) and label
changes, evict(k) on the CUDA index and on the unmodified reference must free the same
number of entries and leave the same live index; later batches re-insert evicted keys
(tombstones revive as fresh nodes with new node ids) and every admit, event and index
dump must still match, through further evictions and a final over-ask (capacity
exhausted after freeing every candidate)."""
import numpy as np
import pytest

from paper_2508_08438_b200 import AdmissionEngine, CapacityExhausted, EngineConfig
from refh import RefEngine, RefRules
from test_gpu_parity import check_admit, check_events, check_index
from workloads import make_batch, make_trunks

pytestmark = pytest.mark.gpu


def _step(eng, re_, rs, batch, epoch=True):
    got = eng.admit(*batch)
    exp = re_.admit(*batch)
    check_admit(rs, got, exp)
    eng.commit()
    re_.commit()
    if epoch:
        ep_g, ev_g = eng.epoch_pass()
        ep_r, ev_r = re_.epoch(cap=1 << 16)
        assert ep_g == ep_r
        check_events(ev_g, ev_r)
    check_index(eng, re_)
    return got


def _evict(eng, re_, k):
    rc_r, n_r = re_.evict(k)
    try:
        n_g = eng.evict(k)[0]
        rc_g = 0
    except CapacityExhausted:
        n_g, rc_g = eng._evicted[0], 1
    assert (rc_g, n_g) == (rc_r, n_r)
    check_index(eng, re_)
    assert eng.entry_count() == len(re_.export()["h"])
    return n_g


@pytest.mark.parametrize("seed,tiered", [(11, False), (12, False), (13, True)])
def test_evict_parity(ref, gpu, seed, tiered):
    rng = np.random.default_rng(seed)
    trunks = make_trunks(rng, 8)
    B, W = 4, 8
    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 16, max_prompts=1024,
                       max_tokens=1 << 18, max_window_entries=1 << 14, u_pre_max=3, entropy_jump=0.1)
    with AdmissionEngine(cfg) as eng:
        eng.enable_eviction(tiered_demotion=tiered)
        re_ = RefEngine(ref, RefRules(ref), B=B, W=W, u_pre_max=3, jump=0.1)
        if tiered:
            re_.set_tiered()
        try:
            rs = eng.rules
            for k in range(4):
                batch = make_batch(rng, trunks, 60, 5)
                got = _step(eng, re_, rs, batch)
                if k == 1:  # demote a slice of the index off HBM (those never leave)
                    tiers = (rng.integers(0, 10, got.n_blocks) >= 8).astype(np.uint8)
                    eng.set_tiers(got.block_h, got.block_d, tiers, got.block_offsets)
                    re_.set_tiers(batch[0], batch[1], tiers)
                    check_index(eng, re_)
            total = eng.entry_count()
            if tiered:  # only leaves move (to DRAM), so ask for fewer than there are leaves
                assert _evict(eng, re_, 50) == 50
            else:
                assert _evict(eng, re_, total // 5) == total // 5
            for k in range(3):  # revivals, more epochs
                _step(eng, re_, rs, make_batch(rng, trunks, 60, 5), epoch=(k != 1))
            _evict(eng, re_, eng.entry_count() // 3)
            _step(eng, re_, rs, make_batch(rng, trunks, 40, 5))
            _evict(eng, re_, 10 ** 6)  # over-ask: frees every candidate, then capacity exhausted
            _step(eng, re_, rs, make_batch(rng, trunks, 40, 5))
        finally:
            re_.close()


def test_evict_speculative_node_ids(ref, gpu):
    """Batches without duplicate claims take the commit's speculative node ids (no exact
    pass); eviction order among equal-epoch, equal-label leaves then rests on them."""
    rng = np.random.default_rng(21)
    B, W = 4, 8
    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 16, max_prompts=1024,
                       max_tokens=1 << 18, max_window_entries=1 << 14)

    def unique_batch(n):
        toks, off = [], [0]
        for _ in range(n):
            t = rng.integers(ord("a"), ord("z") + 1, int(rng.integers(8, 80))).astype(np.uint32)
            if rng.random() < 0.3:  # some private tails
                t = np.concatenate([t, np.frombuffer(b"ssn 123-45-6789 ok", np.uint8).astype(np.uint32)])
            toks.append(t)
            off.append(off[-1] + len(t))
        return (np.concatenate(toks), np.array(off, np.uint64), rng.integers(1, 6, n).astype(np.uint64),
                np.zeros(n, np.uint8))

    with AdmissionEngine(cfg) as eng:
        eng.enable_eviction()
        re_ = RefEngine(ref, RefRules(ref), B=B, W=W)
        try:
            rs = eng.rules
            for _ in range(3):
                _step(eng, re_, rs, unique_batch(50), epoch=False)
            _evict(eng, re_, eng.entry_count() // 3)
            _step(eng, re_, rs, unique_batch(50))
            _evict(eng, re_, eng.entry_count() // 2)
        finally:
            re_.close()


def test_evict_revive_rematch_in_one_window(ref, gpu):
    """Entries touched in the current monitor window are evicted, re-inserted (revived as
    fresh nodes with empty windows) and matched again, all before the window's epoch: the
    revived entry's user set starts empty and its window is rolled once."""
    rng = np.random.default_rng(31)
    trunks = make_trunks(rng, 5)
    B, W = 4, 8
    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 16, max_prompts=1024,
                       max_tokens=1 << 18, max_window_entries=1 << 14, u_pre_max=3, entropy_jump=0.1)
    with AdmissionEngine(cfg) as eng:
        eng.enable_eviction()
        re_ = RefEngine(ref, RefRules(ref), B=B, W=W, u_pre_max=3, jump=0.1)
        try:
            rs = eng.rules
            batches = [make_batch(rng, trunks, 60, 7) for _ in range(3)]
            _step(eng, re_, rs, batches[0])                 # window 1 closes
            _step(eng, re_, rs, batches[1], epoch=False)    # window 2: touches entries
            _evict(eng, re_, eng.entry_count() // 2)        # ... evicts some of them
            _step(eng, re_, rs, batches[1], epoch=False)    # ... re-inserts (revives) them
            _step(eng, re_, rs, batches[1], epoch=False)    # ... and matches them again
            _step(eng, re_, rs, batches[2])                 # window 2 closes: events, roll
            _step(eng, re_, rs, batches[1])
        finally:
            re_.close()


def test_evict_drops_pending_batch(ref, gpu):
    """An evict between admit and commit drops the admitted batch: its commit (which would
    attach new blocks under entries the eviction may have freed) is a state error, the
    context stays consistent, and the batch can be admitted again."""
    from paper_2508_08438_b200 import StateError
    rng = np.random.default_rng(32)
    trunks = make_trunks(rng, 5)
    cfg = EngineConfig(block_tokens=4, window_tokens=8, index_capacity=1 << 14, max_prompts=256,
                       max_tokens=1 << 16, max_window_entries=1 << 12)
    with AdmissionEngine(cfg) as eng:
        eng.enable_eviction()
        re_ = RefEngine(ref, RefRules(ref), B=4, W=8)
        try:
            _step(eng, re_, eng.rules, make_batch(rng, trunks, 40, 4))
            batch = make_batch(rng, trunks, 40, 4)
            check_admit(eng.rules, eng.admit(*batch), re_.admit(*batch))
            _evict(eng, re_, 5)  # the reference evicts between two submits (records applied)
            with pytest.raises(StateError):
                eng.commit()
            _step(eng, re_, eng.rules, batch)  # admitted again, committed on both sides
        finally:
            re_.close()
