"""GPU parity: the CUDA admission path (through the C ABI) against the reference
RadixCacheIndex / CompiledRuleSet / EntropyMonitor driven by the Appendix-A contract
(oracle/ref_harness.cpp).  Bit-exact on hashes, masks, labels, decisions, match lengths,
tiers, index contents and leakage events; entropies compared exactly (tolerance 1e-6
relative is the contract; IEEE FP64 division on both sides gives equality)."""
import numpy as np
import pytest

from paper_2508_08438_b200 import AdmissionEngine, EngineConfig, RuleSet
from refh import RefEngine, RefRules
from workloads import make_batch, make_trunks

pytestmark = pytest.mark.gpu

REL_TOL = 1e-6


def device_to_rule_masks(rs: RuleSet, masks: np.ndarray) -> np.ndarray:
    en = rs.enabled_rules()
    out = np.zeros(len(masks), np.uint64)
    for j, r in enumerate(en):
        out |= ((masks.astype(np.uint64) >> np.uint64(j)) & np.uint64(1)) << np.uint64(r)
    return out


def check_admit(rs, got, exp):
    assert got.n_blocks == len(exp["block_h"])
    np.testing.assert_array_equal(got.block_d, exp["block_d"], "block digests")
    np.testing.assert_array_equal(got.block_h, exp["block_h"], "chained keys")
    np.testing.assert_array_equal(device_to_rule_masks(rs, got.rule_mask), exp["mask"], "window verdict masks")
    np.testing.assert_array_equal(got.label, exp["label"], "labels")
    np.testing.assert_array_equal(got.matched_blocks, exp["matched_blocks"], "matched prefix lengths")
    np.testing.assert_array_equal(got.decision, exp["decision"], "owner/public decisions")
    np.testing.assert_array_equal(got.lowest_tier, exp["lowest_tier"], "lowest tier")


def check_events(got, exp):
    assert len(got) == len(exp)
    for g, e in zip(got, exp):
        assert (g.h, g.d, g.action, g.u_pre) == (e[0], e[1], e[2], e[5])
        assert g.entropy_now == pytest.approx(e[3], rel=REL_TOL, abs=0)
        assert g.entropy_prev == pytest.approx(e[4], rel=REL_TOL, abs=0)


def check_index(eng, ref_eng):
    g = eng.export()
    r = ref_eng.export()
    assert len(g) == len(r["h"])
    for k in ("h", "d", "creator", "label", "owner", "tier", "hit_cur", "u_cnt", "hit_pre", "u_pre"):
        np.testing.assert_array_equal(g[k].astype(np.uint64), r[k].astype(np.uint64), k)


def run_scenario(ref, seed, B, W, n_batches, n_prompts, n_users, jump=0.3, u_pre_max=1, epoch_every=1,
                 wide_p=0.0, rules_json=None, ev_cap=1 << 16):
    rng = np.random.default_rng(seed)
    trunks = make_trunks(rng, 12)
    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 18, max_prompts=4096,
                       max_tokens=1 << 20, max_window_entries=1 << 15, entropy_jump=jump, u_pre_max=u_pre_max)
    fired = 0
    with AdmissionEngine(cfg) as eng:
        rrules = RefRules(ref, rules_json)
        if rules_json is not None:
            eng.set_rules(RuleSet.from_json(rules_json))
        rs = eng.rules
        re_ = RefEngine(ref, rrules, B=B, W=W, jump=jump, u_pre_max=u_pre_max)
        try:
            for k in range(n_batches):
                batch = make_batch(rng, trunks, n_prompts, n_users, wide_p=wide_p)
                got = eng.admit(*batch)
                exp = re_.admit(*batch)
                check_admit(rs, got, exp)
                eng.commit()
                re_.commit()
                if (k + 1) % epoch_every == 0:
                    ep_g, ev_g = eng.epoch_pass(cap=ev_cap)
                    ep_r, ev_r = re_.epoch(cap=1 << 16)
                    assert ep_g == ep_r
                    check_events(ev_g, ev_r)
                    fired += len(ev_g)
                check_index(eng, re_)
        finally:
            re_.close()
    return fired


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_parity_b16_w32(ref, gpu, seed):
    run_scenario(ref, seed, B=16, W=32, n_batches=6, n_prompts=160, n_users=4)


@pytest.mark.parametrize("seed,ev_cap", [(11, 1 << 16), (12, 1)])
def test_parity_small_blocks_many_events(ref, gpu, seed, ev_cap):
    # B=4 makes deep trees, many shared entries and frequent monitor events; ev_cap=1: every
    # epoch overflows the caller's event buffer and the rest comes from skv_last_events
    fired = run_scenario(ref, seed, B=4, W=8, n_batches=8, n_prompts=120, n_users=3, ev_cap=ev_cap)
    assert fired > 0


def test_parity_epoch_every_3_batches(ref, gpu):
    run_scenario(ref, 21, B=8, W=16, n_batches=9, n_prompts=100, n_users=5, epoch_every=3)


def test_parity_saturating_user_sets(ref, gpu):
    # > 64 distinct users hit the same shared entries in one window: order-dependent
    # saturating distinct-user counts (access_stats.hpp:27-37)
    run_scenario(ref, 31, B=4, W=8, n_batches=4, n_prompts=600, n_users=150, epoch_every=2)


def test_parity_wide_tokens(ref, gpu):
    run_scenario(ref, 41, B=16, W=32, n_batches=3, n_prompts=100, n_users=4, wide_p=0.3)


def test_parity_monitor_config(ref, gpu):
    run_scenario(ref, 51, B=4, W=4, n_batches=6, n_prompts=100, n_users=6, jump=0.1, u_pre_max=3)


def test_parity_custom_rules(ref, gpu):
    rules = ('{"version": 7, "rules": ['
             '{"rule_id": "a", "category": "X", "kind": "regex", "pattern": "foo|ba[rz]+"},'
             '{"rule_id": "b", "category": "Y", "kind": "blacklist", "pattern": "alpha"},'
             '{"rule_id": "c", "category": "X", "kind": "regex", "pattern": "\\\\bkv\\\\b", "enabled": false},'
             '{"rule_id": "d", "category": "Z", "kind": "regex", "pattern": "^the|mail$"}]}')
    run_scenario(ref, 61, B=8, W=8, n_batches=4, n_prompts=120, n_users=4, rules_json=rules)
