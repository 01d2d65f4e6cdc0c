"""CPU tests: pin the C restatement oracle (oracle/safekv_oracle.c) against the
reference's own known answers (committed goldens generated from the unmodified
reference) and against the reference harness on randomized inputs."""
import json
import pathlib

import numpy as np
import pytest

from oracle_c import DEFAULT_RULES, OracleEngine, OracleRules
from workloads import make_batch, make_trunks

GOLD = pathlib.Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def orules():
    r = OracleRules()
    yield r
    r.close()


def categories(mask, rules=DEFAULT_RULES):
    cats = []
    for i, r in enumerate(rules):
        if mask >> i & 1 and r[1] not in cats:
            cats.append(r[1])
    return cats


def test_reference_known_answers(orules):
    """test_detection.cpp:33-77 (+ SURVEY App. B probes): verdict, categories, rule mask."""
    kats = json.loads((GOLD / "scan_kats.json").read_text())["kats"]
    for k in kats:
        m = orules.mask(k["text"].encode())
        assert m == k["mask"], k["text"]
        assert (m != 0) == k["sensitive"], k["text"]
        assert categories(m) == k["categories"], k["text"]
    by = {k["text"]: k for k in kats}
    assert by["my ssn is 123-45-6789"]["categories"] == ["Identity Information"]
    assert not by["the weather is nice"]["sensitive"]
    assert by["see (PROJECT-TITAN)."]["sensitive"] and not by["PROJECT-TITANIC is something else"]["sensitive"]


def test_rule_corpus_full_recall(orules):
    """generate_rule_corpus(500, 77) is fully flagged (test_workload.cpp:209-218)."""
    corpus = json.loads((GOLD / "scan_kats.json").read_text())["rule_corpus_500_77"]
    assert len(corpus) == 500
    for c in corpus:
        m = orules.mask(c["text"].encode("latin-1"))
        assert m == c["mask"] and m != 0


def test_disabled_rule_does_not_match():
    """test_detection.cpp:110-118"""
    r = OracleRules(rules=[("off", "X", "regex", "danger", False)])
    assert r.mask(b"danger zone") == 0
    r.close()


def test_duplicate_blacklist_last_writer_wins():
    r = OracleRules(rules=[("a", "X", "blacklist", "TERM", True), ("b", "Y", "blacklist", "TERM", False)])
    assert r.mask(b"a TERM b") == 0  # later disabled duplicate hides the term (detection.hpp:62,157-159)
    r.close()


def test_digest_structural():
    """test_core.cpp:31-45: equal sequences -> equal digests; a bit flip changes it."""
    import oracle_c
    L = oracle_c.lib()
    rng = np.random.default_rng(7)
    for _ in range(200):
        s = rng.integers(0, 256, rng.integers(0, 32)).astype(np.uint32)
        d = L.orc_token_seq_digest(s.ctypes.data, len(s))
        assert d == L.orc_token_seq_digest(s.copy().ctypes.data, len(s))
        if len(s):
            t = s.copy()
            t[rng.integers(len(t))] ^= 1
            assert d != L.orc_token_seq_digest(t.ctypes.data, len(t))


def test_digest_and_chain_vs_reference(ref):
    import oracle_c
    L = oracle_c.lib()
    rng = np.random.default_rng(3)
    for _ in range(300):
        s = rng.integers(0, 1 << 32, rng.integers(0, 40), dtype=np.uint64).astype(np.uint32)
        assert L.orc_token_seq_digest(s.ctypes.data, len(s)) == ref.ref_token_seq_digest(s.ctypes.data, len(s))
        a, b = int(rng.integers(0, 1 << 63)), int(rng.integers(0, 1 << 63))
        assert L.orc_chain(a, b) == ref.ref_chain(a, b)


def test_scan_vs_reference_adversarial(ref, orules):
    from refh import RefRules
    rr = RefRules(ref)
    rng = np.random.default_rng(9)
    alpha = b"0123456789-.:@()[] \t\n\r\v\fabcdefxyzABCDEFimeiaccountnoumbrPROJECT-TITAN,;!?\"'_%+\xe9\x80\x00"
    frags = [b"account number ", b"account no. ", b"imei ", b"PROJECT-TITAN", b"(PROJECT-TITAN).",
             b"my ssn is 123-45-6789", b"(415) 555-0134", b"415-555-0134", b"user99@mail01.com", b"10.4.77.3",
             b"4111-1111-1111-1111", b"0a:1b:2c:3d:4e:5f", b"490154203237518", b"123456"]
    for _ in range(5000):
        parts = []
        for _ in range(int(rng.integers(1, 6))):
            if rng.random() < 0.5:
                parts.append(frags[rng.integers(len(frags))])
            else:
                parts.append(bytes(alpha[i] for i in rng.integers(0, len(alpha), rng.integers(0, 8))))
        t = b"".join(parts)
        assert orules.mask(t) == rr.mask(t), t


@pytest.mark.parametrize("B,W,users", [(16, 32, 3), (4, 8, 3), (8, 16, 80)])
def test_engine_vs_reference(ref, orules, B, W, users):
    from refh import RefEngine, RefRules
    rng = np.random.default_rng(B * 100 + users)
    trunks = make_trunks(rng, 10)
    re_ = RefEngine(ref, RefRules(ref), B=B, W=W)
    oe = OracleEngine(orules, B=B, W=W)
    for k in range(5):
        batch = make_batch(rng, trunks, 200 if users < 50 else 400, users, wide_p=0.05)
        a, b = re_.admit(*batch), oe.admit(*batch)
        for key in a:
            np.testing.assert_array_equal(a[key], b[key], key)
        re_.commit()
        oe.commit()
        assert re_.epoch() == oe.epoch()
        xa, xb = re_.export(), oe.export()
        for key in xa:
            np.testing.assert_array_equal(xa[key], xb[key], key)
    re_.close()
    oe.close()


COST_MODELS = [
    dict(t_base_ms=10.0, c_prefill_ms=1.0, tier_penalty_ms=(0.0, 0.2, 0.5), noise_sigma_ms=0.0, seed=0),
    dict(t_base_ms=3.5, c_prefill_ms=0.7, tier_penalty_ms=(0.0, 0.13, 0.31), noise_sigma_ms=2.5, seed=99),
]


@pytest.mark.parametrize("model", COST_MODELS)
def test_ttft_and_reuse_vs_reference(ref, orules, model):
    """CostModel::ttft (serving_sim.hpp:50-56) and attribute_reuse (:313-324) on the
    C restatement vs the reference's own CostModel, over tiered, partly private indexes.
    Bit-exact without noise; with Box-Muller noise within 1e-12 relative (libm log/cos)."""
    from refh import RefEngine, RefRules
    B, W = 8, 16
    rng = np.random.default_rng(77)
    trunks = make_trunks(rng, 10)
    re_ = RefEngine(ref, RefRules(ref), B=B, W=W)
    oe = OracleEngine(orules, B=B, W=W)
    for k in range(4):
        batch = make_batch(rng, trunks, 150, 5)
        re_.admit(*batch)
        oe.admit(*batch)
        n = len(batch[1]) - 1
        rid = np.arange(1000 * k, 1000 * k + n, dtype=np.uint64)
        ta, ia, xa = re_.ttft(n, model, rid)
        tb, ib, xb = oe.ttft(n, model, rid)
        np.testing.assert_array_equal(ia, ib)
        np.testing.assert_array_equal(xa, xb)
        if model["noise_sigma_ms"] == 0:
            np.testing.assert_array_equal(ta, tb)
        else:
            np.testing.assert_allclose(ta, tb, rtol=1e-12, atol=0)
        re_.commit()
        oe.commit()
        # tier tags on a fresh share of the committed blocks
        nb = int(((batch[1][1:] - batch[1][:-1]) // B).sum())
        tiers = rng.integers(0, 3, nb).astype(np.uint8)
        re_.set_tiers(batch[0], batch[1], tiers)
        oe.set_tiers(batch[0], batch[1], tiers)
    re_.close()
    oe.close()


def test_monitor_burst_downgrade():
    """test_monitor.cpp:101-120 restated through the batch engine: a block used by one
    user in the previous window and by a cross-user burst now is downgraded to Private
    and its subtree hidden; entropy_prev = 1/20, entropy_now = 0.75 (6 users / 8 hits)."""
    B = 4
    oe = OracleEngine(OracleRules(rules=[]), B=B, W=0)
    blk = np.array([1, 2, 3, 4], np.uint32)
    two = np.array([1, 2, 3, 4, 5, 6, 7, 8], np.uint32)

    def batch(seqs, users):
        toks = np.concatenate(seqs).astype(np.uint32)
        offs = np.cumsum([0] + [len(s) for s in seqs]).astype(np.uint64)
        return toks, offs, np.array(users, np.uint64)

    oe.admit(*batch([two], [1]))  # victim inserts a 2-block chain (Public: no rules)
    oe.commit()
    oe.epoch()
    oe.admit(*batch([blk] * 20, [1] * 20))  # previous window: 20 hits, 1 user
    oe.commit()
    oe.epoch()
    oe.admit(*batch([blk] * 8, [10, 11, 12, 13, 14, 15, 10, 11]))  # burst: 6 users / 8 hits
    oe.commit()
    _, ev = oe.epoch()
    assert len(ev) == 1
    h, d, act, now, prev, upre = ev[0]
    assert act == 1 and now == pytest.approx(0.75) and prev == pytest.approx(1 / 20) and upre == 1
    o = oe.admit(*batch([two], [2]))  # other user: downgraded block and its child are invisible
    assert o["matched_blocks"][0] == 0
    o = oe.admit(*batch([two], [1]))  # creator still sees both
    assert o["matched_blocks"][0] == 2
    oe.close()


def test_monitor_saturation():
    """access_stats.hpp:27-37 / test_monitor.cpp:43-53: 64 users, then a repeated
    untracked user counts as new every time."""
    oe = OracleEngine(OracleRules(rules=[]), B=4, W=0)
    blk = np.array([9, 9, 9, 9], np.uint32)
    oe.admit(blk, np.array([0, 4], np.uint64), np.array([1], np.uint64))
    oe.commit()
    oe.epoch()
    users = list(range(1, 65)) + [1000, 1000]
    toks = np.tile(blk, len(users))
    offs = np.arange(0, 4 * len(users) + 1, 4).astype(np.uint64)
    oe.admit(toks, offs, np.array(users, np.uint64))
    x = oe.export()
    assert x["hit_cur"][0] == 66 and x["u_cnt"][0] == 66
    oe.close()


def test_leak_golden_matches_truth_spans():
    """the golden sensitive_alone flags (reference block_truth, tests/golden/
    make_leak_golden.py) are exactly 'the block overlaps a planted span of sensitivity Always'
    -- the span convention skv_leak_flags takes."""
    import numpy as np
    g = pathlib.Path(__file__).resolve().parent / "golden"
    w = np.load(g / "cfg1_workload.npz")
    lk = np.load(g / "cfg1_leak.npz")
    off = w["offsets"].astype(np.int64)
    cnt = w["truth_count"].astype(np.int64)
    so = np.concatenate([[0], np.cumsum(cnt)])
    mine = []
    for i in range(len(off) - 1):
        spans = [(int(w["truth_begin"][k]), int(w["truth_end"][k])) for k in range(so[i], so[i + 1])
                 if w["truth_sens"][k] == 0]
        for b in range((off[i + 1] - off[i]) // 16):
            lo, hi = 16 * b, 16 * (b + 1)
            mine.append(int(any(not (e <= lo or s >= hi) for s, e in spans)))
    assert np.array_equal(np.array(mine, np.uint8), lk["sensitive_alone"])
    assert lk["sensitive_alone"].sum() > 0
