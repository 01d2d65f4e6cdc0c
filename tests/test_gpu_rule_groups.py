"""Rule sets larger than one device automaton: more than 16 enabled rules,
and automata beyond the 32 KB row region, run as consecutive rule groups (one scan pass each,
masks at their rules' bits).  Per-rule window masks, labels, matches, events and the index must
equal the unmodified reference (std::regex per rule) -- on both the B=16/W=32 kernel and the
general one (B=8)."""
import json

import numpy as np
import pytest

from paper_2508_08438_b200 import AdmissionEngine, EngineConfig, RuleSet
from refh import RefEngine, RefRules
from test_gpu_parity import check_admit, check_events, check_index

pytestmark = pytest.mark.gpu


def rule_sets():
    rng = np.random.default_rng(7)
    words = ["alpha", "beta", "cache", "kv", "block", "prefix", "user", "mail", "account", "number", "imei", "card"]
    many = []
    for i in range(28):
        w = words[i % len(words)]
        if i % 4 == 0:
            many.append({"rule_id": f"b{i}", "category": f"C{i % 5}", "kind": "blacklist", "pattern": f"{w.upper()}{i}"})
        else:
            many.append({"rule_id": f"r{i}", "category": f"C{i % 6}", "kind": "regex",
                         "pattern": f"\\b{w}[0-9]{{{1 + i % 3}}}\\b|x{i}y+z", "enabled": i % 9 != 5})
    lits = ["".join(rng.choice(list("abcdefgh"), 10)) for _ in range(300)]
    big = [{"rule_id": f"g{i}", "category": f"Big{i % 3}", "kind": "regex", "pattern": "|".join(lits[25 * i:25 * i + 25])}
           for i in range(12)]
    return {"many": (json.dumps({"version": 11, "rules": many}), words), "big": (json.dumps({"version": 12, "rules": big}), lits)}


def make_batch(rng, vocab, n_prompts, n_users):
    toks, offs, users = [], [0], []
    for _ in range(n_prompts):
        parts = []
        for _ in range(int(rng.integers(4, 40))):
            r = rng.random()
            w = vocab[rng.integers(len(vocab))]
            if r < 0.3:
                parts.append(w + str(int(rng.integers(0, 1000))))
            elif r < 0.4:
                parts.append(w.upper() + str(int(rng.integers(0, 30))))
            elif r < 0.5:
                parts.append(f"x{int(rng.integers(0, 30))}yyz")
            else:
                parts.append(w)
        t = np.frombuffer(" ".join(parts).encode(), np.uint8).astype(np.uint32)
        toks.append(t)
        offs.append(offs[-1] + len(t))
        users.append(1 + int(rng.integers(n_users)))
    return (np.concatenate(toks), np.array(offs, np.uint64), np.array(users, np.uint64),
            np.zeros(n_prompts, np.uint8))


@pytest.mark.parametrize("which,B,W", [("many", 16, 32), ("many", 8, 16), ("big", 16, 32), ("big", 8, 16)])
def test_rule_groups_parity(ref, gpu, which, B, W):
    text, vocab = rule_sets()[which]
    rs = RuleSet.from_json(text)
    assert rs.group_count() >= 2
    rng = np.random.default_rng(hash((which, B)) % 1000)
    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 16, max_prompts=512, max_tokens=1 << 18,
                       max_window_entries=1 << 14)
    with AdmissionEngine(cfg) as eng:
        eng.set_rules(rs)
        re_ = RefEngine(ref, RefRules(ref, text), B=B, W=W)
        try:
            flagged = 0
            for _ in range(3):
                batch = make_batch(rng, vocab, 160, 5)
                got = eng.admit(*batch)
                exp = re_.admit(*batch)
                check_admit(rs, got, exp)
                flagged += int((got.rule_mask != 0).sum())
                eng.commit()
                re_.commit()
                _, ev_g = eng.epoch_pass()
                _, ev_r = re_.epoch()
                check_events(ev_g, ev_r)
                check_index(eng, re_)
            assert flagged > 0
            # per-call tier1_scan across the groups
            for t in (b"alpha12 x3yyz", b"CARD11 kv", vocab[3].encode() + b" " + vocab[250 % len(vocab)].encode()):
                assert rs.to_rule_mask(eng.tier1_scan(t)) == RefRules(ref, text).mask(t)
        finally:
            re_.close()


def test_hot_reload_parity(ref, gpu):
    """Rule hot reload at batch boundaries (RuleEngine::load_rules, detection.hpp:238-241, 651-662):
    default -> 28-rule set -> large-automaton set -> default, the device (skv_set_rules) and the
    reference engine swapping the same snapshots between the same batches; every batch, epoch and
    index dump equal."""
    sets = rule_sets()
    vocab = sets["many"][1] + sets["big"][1][:40]
    seq = [None, sets["many"][0], sets["big"][0], None]
    rng = np.random.default_rng(99)
    cfg = EngineConfig(block_tokens=16, window_tokens=32, index_capacity=1 << 16, max_prompts=512, max_tokens=1 << 18,
                       max_window_entries=1 << 14)
    with AdmissionEngine(cfg) as eng:
        re_ = RefEngine(ref, RefRules(ref), B=16, W=32)
        try:
            for text in seq:
                rs = RuleSet.default() if text is None else RuleSet.from_json(text)
                eng.set_rules(rs)
                re_.set_rules(RefRules(ref, text))
                for _ in range(2):
                    batch = make_batch(rng, vocab, 120, 4)
                    check_admit(rs, eng.admit(*batch), re_.admit(*batch))
                    eng.commit()
                    re_.commit()
                    _, ev_g = eng.epoch_pass()
                    check_events(ev_g, re_.epoch()[1])
                    check_index(eng, re_)
        finally:
            re_.close()


def windows_of(tokens, offsets, B, W):
    """A.3 window texts: tokens[bB : min(L, (b+1)B + W)] of every full block, prompt-major."""
    out = []
    for p in range(len(offsets) - 1):
        t = tokens[int(offsets[p]):int(offsets[p + 1])].astype(np.uint8).tobytes()
        for b in range(len(t) // B):
            out.append(t[b * B:min(len(t), (b + 1) * B + W)])
    return out


@pytest.mark.parametrize("B,W", [(16, 32), (8, 16)])
def test_wide_rule_library_parity(ref, gpu, B, W):
    """A library of more than 32 enabled rules (three mask words) on both scan kernels: every
    window's full per-rule mask equals the reference's per-rule verdicts, the category list of a
    sample of windows equals the stock CompiledRuleSet::scan's (rule order, de-duplicated), and
    labels, matches, decisions, events and the index equal the reference engine's (one stock scan
    per window)."""
    from paper_2508_08438_b200 import combine_mask_words
    from test_rules_compiler import wide_library
    text, words = wide_library()
    rs = RuleSet.from_json(text)
    assert rs.mask_words() >= 3
    n_rules = rs.size()
    rr = RefRules(ref, text)
    vocab = [f"{w}{i}" for i, w in enumerate(words * 8)] + [f"{w.upper()}-{i}" for i, w in enumerate(words * 8)] + words
    rng = np.random.default_rng(B)
    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 16, max_prompts=512, max_tokens=1 << 18,
                       max_window_entries=1 << 14)
    with AdmissionEngine(cfg) as eng:
        eng.set_rules(rs)
        re_ = RefEngine(ref, rr, B=B, W=W)
        re_.set_stock_scan(True)
        try:
            hits_hi = 0
            for _ in range(3):
                batch = make_batch(rng, vocab, 120, 5)
                got = eng.admit(*batch)
                exp = re_.admit(*batch)
                assert got.rule_mask_words is not None and got.rule_mask_words.shape[0] == rs.mask_words()
                np.testing.assert_array_equal(got.rule_mask_words[0], got.rule_mask)
                dev = combine_mask_words(got.rule_mask_words)
                wins = windows_of(batch[0], batch[1], B, W)
                assert len(wins) == got.n_blocks
                for i, t in enumerate(wins):
                    assert rs.to_rule_mask(dev[i]) == rr.mask_wide(t, n_rules), (i, t)
                for i in range(0, len(wins), 7):
                    assert (dev[i] != 0, rs.categories(dev[i])) == rr.verdict(wins[i]), (i, wins[i])
                hits_hi += sum(1 for m in dev if m >> 32)
                np.testing.assert_array_equal(got.block_h, exp["block_h"])
                np.testing.assert_array_equal(np.array([m != 0 for m in dev], np.uint64), exp["mask"])
                for k in ("label", "decision", "matched_blocks", "lowest_tier"):
                    np.testing.assert_array_equal(getattr(got, k), exp[k], k)
                eng.commit()
                re_.commit()
                _, ev_g = eng.epoch_pass()
                check_events(ev_g, re_.epoch()[1])
                check_index(eng, re_)
            assert hits_hi > 0  # rules beyond the first mask word fired
            # per-call tier1_scan and the facade's batch scan across the words
            for t in wins[:64:5] + [b"acct13 Q7 q41abz", f"{words[1].upper()}-85 x".encode()]:
                m = eng.tier1_scan(t)
                assert rs.to_rule_mask(m) == rr.mask_wide(t, n_rules)
        finally:
            re_.close()
