"""GPU parity against committed golden vectors (generated from the unmodified reference by
tests/golden/make_golden.py) and against the C restatement oracle -- neither needs
/root/reference at run time."""
import json
import pathlib

import numpy as np
import pytest

from oracle_c import OracleEngine, OracleRules
from paper_2508_08438_b200 import AdmissionEngine, EngineConfig, RuleSet
from workloads import make_batch, make_trunks

pytestmark = pytest.mark.gpu
GOLD = pathlib.Path(__file__).resolve().parent / "golden"


def cfg(**kw):
    base = dict(block_tokens=16, window_tokens=32, index_capacity=1 << 18, max_prompts=4096, max_tokens=1 << 20,
                max_window_entries=1 << 15)
    base.update(kw)
    return EngineConfig(**base)


def test_config1_golden(gpu):
    """Config 1 (1000 x 112-token reference-generated prompts, 4 users): two admission
    rounds with commit + epoch, bit-exact against the reference's outputs."""
    w = np.load(GOLD / "cfg1_workload.npz")
    e = np.load(GOLD / "cfg1_expected.npz")
    assert int(w["digest"][0]) == 0x1FF5DFD735EC52B0  # reference canonical_bytes() pin
    tok = w["tokens"].astype(np.uint32)
    with AdmissionEngine(cfg()) as eng:
        rs = eng.rules
        for rnd in (1, 2):
            got = eng.admit(tok, w["offsets"], w["users"], w["owners"])
            np.testing.assert_array_equal(got.block_h, e[f"r{rnd}_block_h"])
            np.testing.assert_array_equal(got.block_d, e[f"r{rnd}_block_d"])
            np.testing.assert_array_equal(rs.to_rule_mask_array(got.rule_mask), e[f"r{rnd}_mask"])
            np.testing.assert_array_equal(got.label, e[f"r{rnd}_label"])
            np.testing.assert_array_equal(got.decision, e[f"r{rnd}_decision"])
            np.testing.assert_array_equal(got.matched_blocks, e[f"r{rnd}_matched_blocks"])
            np.testing.assert_array_equal(got.lowest_tier, e[f"r{rnd}_lowest_tier"])
            eng.commit()
            ep, ev = eng.epoch_pass()
            assert ep == int(e[f"r{rnd}_epoch"][0])
            assert [(x.h, x.d, x.action, x.u_pre) for x in ev] == [tuple(map(int, r)) for r in e[f"r{rnd}_events"]]
        x = eng.export()
        for k in ("h", "d", "creator", "label", "owner", "tier", "hit_cur", "u_cnt", "hit_pre", "u_pre"):
            np.testing.assert_array_equal(x[k].astype(np.uint64), e[f"export_{k}"].astype(np.uint64), k)


def test_tier1_scan_known_answers(gpu):
    """RuleEngine::tier1_scan known answers (test_detection.cpp:33-77) through the device."""
    kats = json.loads((GOLD / "scan_kats.json").read_text())
    with AdmissionEngine(cfg()) as eng:
        for k in kats["kats"] + kats["rule_corpus_500_77"][:100]:
            m = eng.tier1_scan(k["text"].encode("latin-1"))
            assert eng.rules.to_rule_mask(m) == k["mask"], k["text"]
            assert eng.rules.categories(m) == k["categories"], k["text"]


def test_token_seq_digest_device(gpu):
    import oracle_c
    L = oracle_c.lib()
    rng = np.random.default_rng(1)
    with AdmissionEngine(cfg()) as eng:
        for n in (0, 1, 7, 16, 33):
            t = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
            assert eng.token_seq_digest(t) == L.orc_token_seq_digest(t.ctypes.data, n)


@pytest.mark.parametrize("B,W", [(16, 32), (16, 16), (16, 40), (8, 4), (128, 32), (4, 0)])
def test_vs_c_oracle_ragged(gpu, B, W):
    """Ragged / empty / sub-block prompts, non-byte tokens, window shapes with and without
    the neighbour-shared context block, against the C restatement."""
    rng = np.random.default_rng(B * 1000 + W)
    trunks = make_trunks(rng, 10)
    orc = OracleEngine(OracleRules(), B=B, W=W)
    with AdmissionEngine(cfg(block_tokens=B, window_tokens=W)) as eng:
        for _ in range(4):
            batch = make_batch(rng, trunks, 300, 4, wide_p=0.05, max_words=120 if B >= 64 else 40)
            got = eng.admit(*batch)
            exp = orc.admit(*batch)
            np.testing.assert_array_equal(got.block_h, exp["block_h"])
            np.testing.assert_array_equal(eng.rules.to_rule_mask_array(got.rule_mask), exp["mask"])
            np.testing.assert_array_equal(got.label, exp["label"])
            np.testing.assert_array_equal(got.matched_blocks, exp["matched_blocks"])
            np.testing.assert_array_equal(got.decision, exp["decision"])
            eng.commit()
            orc.commit()
            _, ev = eng.epoch_pass()
            _, ev_o = orc.epoch()
            assert [(x.h, x.d, x.action) for x in ev] == [(x[0], x[1], x[2]) for x in ev_o]
    orc.close()


@pytest.mark.parametrize("W", [32, 16, 20])
def test_vs_c_oracle_aligned_dense(gpu, W):
    """Block-aligned prompts (the vectorised 16-token path of k_hash_scan) with dense PII:
    many windows accept, so the deferred exact-mask queue overflows and flushes."""
    B = 16
    rng = np.random.default_rng(7000 + W)
    trunks = make_trunks(rng, 10, pii_p=0.4)
    orc = OracleEngine(OracleRules(), B=B, W=W)
    with AdmissionEngine(cfg(block_tokens=B, window_tokens=W)) as eng:
        for _ in range(3):
            batch = make_batch(rng, trunks, 400, 4, pii_p=0.35, max_words=60, align=16)
            got = eng.admit(*batch)
            exp = orc.admit(*batch)
            np.testing.assert_array_equal(got.block_d, exp["block_d"])
            np.testing.assert_array_equal(got.block_h, exp["block_h"])
            np.testing.assert_array_equal(eng.rules.to_rule_mask_array(got.rule_mask), exp["mask"])
            np.testing.assert_array_equal(got.label, exp["label"])
            np.testing.assert_array_equal(got.matched_blocks, exp["matched_blocks"])
            eng.commit()
            orc.commit()
            eng.epoch_pass()
            orc.epoch()
    orc.close()


def test_large_batch_properties(gpu):
    """Config-2 sized batch (65,536 x 2,048): size-independent properties -- every prompt
    matches exactly its 40-block pool prefix (pool pre-inserted, Public), labels are a
    prefix-OR of the window masks, keys of identical pool prefixes coincide, and a
    sample of prompts agrees with the C oracle."""
    from workload import GenSpec, generate, generate_pool
    spec = GenSpec(n_prompts=65536, prompt_tokens=2048, seed=1)
    tok, off, users, owners = generate(spec)
    ptok, poff, pusers, powners = generate_pool(spec)
    with AdmissionEngine(cfg(max_prompts=65536, max_tokens=65536 * 2048, index_capacity=1 << 25,
                             max_window_entries=1 << 16)) as eng:
        eng.admit(ptok, poff, pusers, powners)
        eng.commit()
        eng.epoch_pass()
        got = eng.admit(tok, off, users, owners)
    nb = 128
    assert got.n_blocks == 65536 * nb
    assert (got.matched_blocks == 40).all()
    lab = got.label.reshape(-1, nb)
    sens = (got.rule_mask.reshape(-1, nb) != 0)
    np.testing.assert_array_equal(lab == 0, np.logical_or.accumulate(sens, axis=1))
    orc = OracleEngine(OracleRules(), B=16, W=32)
    orc.admit(ptok, poff, pusers, powners)
    orc.commit()
    orc.epoch()
    idx = np.arange(0, 65536, 4099)
    sub_tok = np.concatenate([tok[i * 2048:(i + 1) * 2048] for i in idx])
    sub_off = np.arange(len(idx) + 1, dtype=np.uint64) * 2048
    exp = orc.admit(sub_tok, sub_off, users[idx], owners[idx])
    sel = (idx[:, None] * nb + np.arange(nb)[None, :]).ravel()
    np.testing.assert_array_equal(got.block_h[sel], exp["block_h"])
    np.testing.assert_array_equal(eng.rules.to_rule_mask_array(got.rule_mask[sel]), exp["mask"])
    np.testing.assert_array_equal(got.label[sel], exp["label"])
    orc.close()


def _always_spans(w):
    cnt = w["truth_count"].astype(np.int64)
    keep = w["truth_sens"] == 0  # SpanSensitivity::Always
    so = np.zeros(len(cnt) + 1, np.uint32)
    owner = np.repeat(np.arange(len(cnt)), cnt)[keep]
    np.add.at(so, owner + 1, 1)
    return np.cumsum(so).astype(np.uint32), w["truth_begin"][keep], w["truth_end"][keep]


def test_leak_flags_config1(ref, gpu):
    """SURVEY A.8 leak flags on the device (skv_leak_flags) for config 1: with the default rules
    against the reference's golden (no planted secret leaks); with a rule set that knows only the
    SSN and e-mail templates, Public blocks over planted secrets do leak, and the device flags
    equal Public (reference labels under the same rules) AND block_truth.sensitive_alone."""
    from paper_2508_08438_b200 import RuleSet
    from refh import RefEngine, RefRules
    w = np.load(GOLD / "cfg1_workload.npz")
    lk = np.load(GOLD / "cfg1_leak.npz")
    tok = w["tokens"].astype(np.uint32)
    so, sb, se = _always_spans(w)
    with AdmissionEngine(cfg()) as eng:
        eng.admit(tok, w["offsets"], w["users"], w["owners"])
        flags, n = eng.leak_flags(so, sb, se)
        np.testing.assert_array_equal(flags, lk["r1_leak"])
        assert n == int(lk["r1_leak"].sum())
    rules = ('{"version": 3, "rules": ['
             '{"rule_id": "ssn", "category": "Identity Information", "kind": "regex", '
             '"pattern": "\\\\b\\\\d{3}-\\\\d{2}-\\\\d{4}\\\\b"},'
             '{"rule_id": "mail", "category": "Basic Information", "kind": "regex", '
             '"pattern": "[A-Za-z0-9._%+-]+@[A-Za-z0-9.-]+\\\\.[A-Za-z]{2,}"}]}')
    with AdmissionEngine(cfg()) as eng:
        eng.set_rules(RuleSet.from_json(rules))
        got = eng.admit(tok, w["offsets"], w["users"], w["owners"])
        re_ = RefEngine(ref, RefRules(ref, rules), B=16, W=32)
        try:
            exp = re_.admit(tok, w["offsets"], w["users"], w["owners"])
        finally:
            re_.close()
        np.testing.assert_array_equal(got.label, exp["label"])
        flags, n = eng.leak_flags(so, sb, se)
        want = ((exp["label"] == 1) & (lk["sensitive_alone"] == 1)).astype(np.uint8)
        np.testing.assert_array_equal(flags, want)
        assert n == int(want.sum()) > 0
