"""TierBudget-bounded HBM with insert-time make_room (reference cache_index.hpp:26-55, 152-205,
697-728, 801-806) under the batched serving contract A.9 (extending SURVEY Appendix A): each prompt's
matched path stays pinned from its lookup to the end of the batch's commit
(ServingSimulator::submit, serving_sim.hpp:195-215), the commit inserts the prompts in order and
every insert first evicts unpinned leaves in the reference's victim order until its new blocks
fit; an insert that cannot make room raises CapacityExhausted and its prompt is dropped.

The unmodified reference runs the same contract (oracle/ref_harness.cpp ref_engine_commit with
ref_engine_set_budget).  After every batch: admit outputs, dropped prompts, HBM usage, events and
the full index export must be equal -- under steady pressure (the budget a fraction of the
working set), with private prefixes other users walk but cannot see (evictions that cut a later
prompt's insert walk), with several batches per monitor epoch (victims of the current epoch
compete with the batch's own new nodes), and under a budget so small that inserts fail."""
import numpy as np
import pytest

from paper_2508_08438_b200 import AdmissionEngine, EngineConfig
from refh import RefEngine, RefRules
from test_gpu_parity import check_admit, check_events, check_index
from workloads import make_batch, make_trunks

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,budget,epoch_every,n_prompts,pii_p,drops_expected", [
    (21, 400, 1, 60, 0.08, False),  # steady pressure, an epoch per batch
    (22, 400, 3, 80, 0.3, True),    # many private prefixes walked by others; 3 batches per epoch
    (22, 250, 3, 80, 0.3, True),    # ... with a budget below one batch's new blocks: frequent drops
    (23, 200, 2, 60, 0.15, False),  # current-epoch victims compete with the batch's own new nodes
    (24, 90, 1, 40, 0.08, True),    # most inserts cannot make room (CapacityExhausted)
])
def test_budgeted_commit_parity(ref, gpu, seed, budget, epoch_every, n_prompts, pii_p, drops_expected):
    rng = np.random.default_rng(seed)
    trunks = make_trunks(rng, 6, pii_p=pii_p)
    B, W = 4, 8
    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 16, max_prompts=1024,
                       max_tokens=1 << 18, max_window_entries=1 << 14, u_pre_max=3, entropy_jump=0.1)
    with AdmissionEngine(cfg) as eng:
        eng.enable_eviction()
        eng.set_tier_budget(budget)
        rs = eng.rules
        re_ = RefEngine(ref, RefRules(ref), B=B, W=W, u_pre_max=3, jump=0.1)
        re_.set_budget(budget)
        try:
            drops = 0
            max_used = 0
            for k in range(12):
                batch = make_batch(rng, trunks, n_prompts, 5, pii_p=pii_p)
                got = eng.admit(*batch)
                exp = re_.admit(*batch)
                check_admit(rs, got, exp)
                eng.commit()
                re_.commit()
                np.testing.assert_array_equal(eng.last_drops(), re_.dropped())
                drops += len(re_.dropped())
                used, cap = eng.tier_usage()
                assert int(used[0]) == int(re_.budget_used()[0]) <= budget
                max_used = max(max_used, int(used[0]))
                if k % epoch_every == epoch_every - 1:
                    ep_g, ev_g = eng.epoch_pass()
                    ep_r, ev_r = re_.epoch(cap=1 << 16)
                    assert ep_g == ep_r
                    check_events(ev_g, ev_r)
                check_index(eng, re_)
            assert max_used > budget * 0.8  # the budget was binding
            assert (drops > 0) == drops_expected
        finally:
            re_.close()


@pytest.mark.parametrize("seed,budgets,epoch_every,n_prompts,pii_p,max_words", [
    (31, (200, 20, 10), 1, 60, 0.08, 12),   # DRAM and SSD fill: demotions cascade, SSD frees expose parents
    (32, (300, 15, 0), 2, 60, 0.3, 12),     # no SSD: a full DRAM frees its victim outright
    (33, (150, 0, 30), 1, 50, 0.1, 12),     # no DRAM: HBM victims are freed directly
    (34, (250, 30, 20), 3, 80, 0.15, 20),   # 3 batches per epoch, longer prompts
])
def test_budgeted_tiered_cascade_parity(ref, gpu, seed, budgets, epoch_every, n_prompts, pii_p, max_words):
    """Tiered demotion with bounded DRAM / SSD (evict_or_demote, cache_index.hpp:732-766): every
    make_room of the commit and every explicit evict cascade down the tiers exactly like the
    reference; tier usage, drops, per-entry tiers and the live index are compared every batch."""
    from paper_2508_08438_b200 import CapacityExhausted
    rng = np.random.default_rng(seed)
    trunks = make_trunks(rng, 6, pii_p=pii_p)
    B, W = 4, 8
    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 16, max_prompts=1024,
                       max_tokens=1 << 18, max_window_entries=1 << 14, u_pre_max=3, entropy_jump=0.1)
    with AdmissionEngine(cfg) as eng:
        eng.enable_eviction(tiered_demotion=True)
        eng.set_tier_budget(*budgets)
        rs = eng.rules
        re_ = RefEngine(ref, RefRules(ref), B=B, W=W, u_pre_max=3, jump=0.1)
        re_.set_budget(*budgets, tiered=True)
        try:
            lower_used = 0
            for k in range(12):
                batch = make_batch(rng, trunks, n_prompts, 5, pii_p=pii_p, max_words=max_words)
                got = eng.admit(*batch)
                exp = re_.admit(*batch)
                check_admit(rs, got, exp)
                eng.commit()
                re_.commit()
                np.testing.assert_array_equal(eng.last_drops(), re_.dropped())
                used, _ = eng.tier_usage()
                np.testing.assert_array_equal(used, re_.budget_used())
                lower_used = max(lower_used, int(used[1] + used[2]))
                if k % epoch_every == epoch_every - 1:
                    ep_g, ev_g = eng.epoch_pass()
                    ep_r, ev_r = re_.epoch(cap=1 << 16)
                    assert ep_g == ep_r
                    check_events(ev_g, ev_r)
                check_index(eng, re_)
                if k in (4, 8):  # explicit RadixCacheIndex::evict with the same cascade
                    rc_r, n_r = re_.evict(20)
                    try:
                        n_g, rc_g = eng.evict(20)[0], 0
                    except CapacityExhausted:
                        n_g, rc_g = eng._evicted[0], 1
                    assert (rc_g, n_g) == (rc_r, n_r)
                    np.testing.assert_array_equal(eng.tier_usage()[0], re_.budget_used())
                    check_index(eng, re_)
            assert (lower_used > 0) == (budgets[1] > 0)  # victims were demoted (freed outright without DRAM)
        finally:
            re_.close()
