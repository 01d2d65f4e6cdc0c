"""CPU tests of the host rule compiler (rule JSON -> search DFA tables) against the
reference's std::regex / TokenTrie semantics.  The compiled tables are executed here by
a small numpy DFA runner (test infrastructure only); the device runs the same tables."""
import json
import pathlib

import numpy as np
import pytest

from paper_2508_08438_b200 import CompileError, ParseError, RuleSet

GOLD = pathlib.Path(__file__).resolve().parent / "golden"


def run_dfa(dfa, texts):
    """Vectorised DFA execution: returns the device-order rule mask per text."""
    n = len(texts)
    L = max((len(t) for t in texts), default=0)
    arr = np.zeros((n, L), np.int64)
    lens = np.array([len(t) for t in texts])
    for i, t in enumerate(texts):
        arr[i, :len(t)] = np.frombuffer(t, np.uint8)
    cls = dfa["class_map"][arr]
    s = np.full(n, dfa["start"], np.int64)
    acc = np.zeros(n, np.uint64)
    C = dfa["n_classes"]
    for j in range(L):
        live = j < lens
        c = cls[:, j]
        acc |= np.where(live, dfa["acc"][s, c], 0).astype(np.uint64)
        s = np.where(live, dfa["next"][s, c], s)
    acc |= dfa["acc"][s, C].astype(np.uint64)
    return acc


def test_default_dfa_size():
    d = RuleSet.default().dfa()
    assert d["n_classes"] + 1 <= 64  # pre-scaled class bytes fit a u8
    assert d["n_states"] * (d["n_classes"] + 1) * 4 <= 65535  # 16-bit row offsets
    assert d["n_states"] <= d["dfa_states_unminimized"]


def test_default_rules_known_answers():
    rs = RuleSet.default()
    kats = json.loads((GOLD / "scan_kats.json").read_text())
    items = kats["kats"] + kats["rule_corpus_500_77"]
    texts = [k["text"].encode("latin-1") for k in items]
    masks = run_dfa(rs.dfa(), texts)
    for k, m in zip(items, masks.tolist()):
        assert rs.to_rule_mask(int(m)) == k["mask"], k["text"]
        assert rs.categories(int(m)) == k["categories"], k["text"]


def _adversarial(rng, n):
    alpha = b"0123456789-.:@()[] \t\n\r\v\fabcdefxyzABCDEFimeiaccountnoumbrPROJECT-TITAN,;!?\"'_%+\xe9\x80\x00"
    frags = [b"account number ", b"account no. ", b"account  no", b"imei ", b"PROJECT-TITAN", b"(PROJECT-TITAN).",
             b"PROJECT-TITANIC", b"my ssn is 123-45-6789", b"(415) 555-0134", b"415-555-0134",
             b"user99@mail01.com", b"a@b.co", b"10.4.77.3", b"4111-1111-1111-1111", b"0a:1b:2c:3d:4e:5f",
             b"490154203237518", b"123456", b"12345678901234567"]
    out = []
    for _ in range(n):
        parts = []
        for _ in range(int(rng.integers(1, 7))):
            if rng.random() < 0.5:
                parts.append(frags[rng.integers(len(frags))])
            else:
                parts.append(bytes(alpha[i] for i in rng.integers(0, len(alpha), rng.integers(0, 9))))
        t = bytearray(b"".join(parts))
        if rng.random() < 0.3 and t:
            for _ in range(int(rng.integers(1, 4))):
                t[rng.integers(len(t))] = alpha[rng.integers(len(alpha))]
        out.append(bytes(t))
    return out


def test_default_rules_vs_reference_adversarial(ref):
    from refh import RefRules
    rr = RefRules(ref)
    rs = RuleSet.default()
    texts = _adversarial(np.random.default_rng(7), 20000)
    masks = run_dfa(rs.dfa(), texts)
    bad = [t for t, m in zip(texts, masks.tolist()) if rs.to_rule_mask(int(m)) != rr.mask(t)]
    assert not bad, bad[:5]


CUSTOM = [
    r"foo|ba[rz]+", r"^the", r"mail$", r"\bkv\b", r"\Bcache", r"a{2,3}b?c*", r"(?:ab|cd){2}", r"[^a-z0-9 ]+x",
    r"[\d-]{3}", r"[\w.]+@", r"\d{1,}\.\d", r"x[-a]y", r"[a\-z]", r"[]a]", r"[^]", r"\x41B", r"a.b",
    r"[[:alpha:]]{3}[[:digit:]]", r"\s\S\w\W\d\D", r"q?", r"(a|)+b", r"(a*)*c", r"\cJ", r"[\b]", r"\0",
    r"[z-a]?" + "", r"[.-]", r"[a-]", r"$^", r"\bimei\s*\d{3}\b", r"[\x80-\xff]+", r"\x7f",
]


@pytest.mark.parametrize("pattern", CUSTOM)
def test_custom_regex_vs_reference(ref, pattern):
    from refh import RefRules
    cfg = json.dumps({"version": 3, "rules": [{"rule_id": "r", "category": "C", "kind": "regex",
                                               "pattern": pattern}]})
    try:
        rr = RefRules(ref, cfg)
    except ValueError:
        with pytest.raises(CompileError):
            RuleSet.from_json(cfg)
        return
    rs = RuleSet.from_json(cfg)
    rng = np.random.default_rng(abs(hash(pattern)) % (1 << 32))
    alpha = b"abcdxyzqABCDkvcachemail the foo bar baz 0123456789.-_@\n\r\t\v\x80\xe9\xff\x00]\\[^$\x7fJ\b"
    texts = [bytes(alpha[i] for i in rng.integers(0, len(alpha), rng.integers(0, 24))) for _ in range(3000)]
    texts += [b"", b"the foo", b"kv cache", b"aab", b"abab", b"cdcd", b"x-y", b"]", b"AB", b"imei 123", b"a\nb"]
    masks = run_dfa(rs.dfa(), texts)
    for t, m in zip(texts, masks.tolist()):
        assert rs.to_rule_mask(int(m)) == rr.mask(t), (pattern, t)


BAD = ["(", "a{2", "a{,3}", "*a", "a**{", "[a", "\\", "a{3,2}", "[\\w-z]", "(?=x)", "(?!x)", r"(a)\1", "a{x}",
       "[[:nope:]]", ")"]


@pytest.mark.parametrize("pattern", BAD)
def test_bad_or_unsupported_patterns_raise_compile_error(ref, pattern):
    cfg = json.dumps({"version": 1, "rules": [{"rule_id": "bad", "kind": "regex", "pattern": pattern}]})
    with pytest.raises(CompileError, match="bad"):
        RuleSet.from_json(cfg)


def test_load_rules_json_errors_and_warnings():
    """detection.hpp:222-280 / test_detection.cpp:79-108"""
    good = {"version": 2, "rules": [{"rule_id": "a", "category": "X", "kind": "regex", "pattern": "foo"},
                                    {"rule_id": "b", "category": "Y", "kind": "blacklist", "pattern": "BAR"},
                                    {"rule_id": "c", "category": "Z", "kind": "regex", "pattern": "qu+x"}]}
    rs = RuleSet.from_json(json.dumps(good))
    assert rs.size() == 3 and rs.version == 2
    bad = json.loads(json.dumps(good))
    bad["rules"][1]["pattern"] = "("
    bad["rules"][1]["kind"] = "regex"
    with pytest.raises(CompileError, match="b"):
        RuleSet.from_json(json.dumps(bad))
    dup = json.loads(json.dumps(good))
    dup["rules"][2]["rule_id"] = "a"
    with pytest.raises(CompileError, match="duplicate"):
        RuleSet.from_json(json.dumps(dup))
    unk = dict(good, surprise=1)
    w = RuleSet.from_json(json.dumps(unk)).warnings()
    assert len(w) == 1 and "surprise" in w[0]
    for txt in ["[]", '{"version": "x"}', '{"rules": {}}', '{"rules": [1]}', '{"rules": [{"rule_id": "a"}]}',
                '{"rules": [{"rule_id": "a", "pattern": "x", "kind": "glob"}]}', "not json"]:
        with pytest.raises(ParseError):
            RuleSet.from_json(txt)


def test_disabled_and_blacklist_semantics():
    cfg = {"version": 1, "rules": [
        {"rule_id": "off", "category": "X", "kind": "regex", "pattern": "danger", "enabled": False},
        {"rule_id": "t1", "category": "A", "kind": "blacklist", "pattern": "TERM"},
        {"rule_id": "t2", "category": "B", "kind": "blacklist", "pattern": "TERM", "enabled": False},
        {"rule_id": "t3", "category": "C", "kind": "blacklist", "pattern": "(x)"},
        {"rule_id": "t4", "category": "D", "kind": "blacklist", "pattern": "a b"},
        {"rule_id": "t5", "category": "E", "kind": "blacklist", "pattern": "Q.Q"}]}
    rs = RuleSet.from_json(json.dumps(cfg))
    texts = [b"danger zone", b"TERM", b"(x)", b"x", b"a b", b"(Q.Q).", b"Q.Q\x0bz", b"Q.Q\tz"]
    m = [rs.to_rule_mask(int(x)) for x in run_dfa(rs.dfa(), texts)]
    assert m == [0, 0, 0, 0, 0, 1 << 5, 0, 1 << 5]


def wide_library(n_rules=90, seed=5):
    """A rule library of more than 32 enabled rules (several mask words): regexes and blacklist
    terms over a small vocabulary, a handful disabled, categories shared across rules."""
    rng = np.random.default_rng(seed)
    words = ["acct", "iban", "pin", "token", "secret", "badge", "vin", "mrn", "npi", "dea", "swift", "sort"]
    rules = []
    for i in range(n_rules):
        w = words[i % len(words)]
        if i % 5 == 0:
            rules.append({"rule_id": f"bl{i}", "category": f"Cat{i % 7}", "kind": "blacklist",
                          "pattern": f"{w.upper()}-{i}"})
        else:
            rules.append({"rule_id": f"rx{i}", "category": f"Cat{(i * 3) % 11}", "kind": "regex",
                          "pattern": f"\\b{w}{i}[0-9]{{{1 + i % 3}}}\\b|q{i}[a-c]+z",
                          "enabled": i % 17 != 3})
    return json.dumps({"version": 21, "rules": rules}), words


def test_wide_rule_library_loads():
    """More than 32 enabled rules load as several mask words (the reference
    loads a library of any size, detection.hpp:222-242); the single-automaton view is refused."""
    text, _ = wide_library()
    rs = RuleSet.from_json(text)
    en = rs.enabled_rules()
    assert len(en) == sum(1 for r in json.loads(text)["rules"] if r.get("enabled", True))
    assert rs.mask_words() == (len(en) + 31) // 32 >= 3
    assert rs.group_count() >= rs.mask_words()
    with pytest.raises(CompileError):
        rs.dfa()
    assert RuleSet.default().mask_words() == 1


def test_rule_library_maximum():
    rules = [{"rule_id": f"t{i}", "category": "C", "kind": "blacklist", "pattern": f"TERM{i}"} for i in range(1025)]
    with pytest.raises(CompileError):
        RuleSet.from_json(json.dumps({"version": 1, "rules": rules}))
