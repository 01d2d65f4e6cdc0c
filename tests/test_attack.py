"""CPU tests of the batched attack campaign (paper_2508_08438_b200/attack.py, restating
adversary.hpp:83-279): the SplitMix64 / derive_seed restatement against the reference's
own, and every campaign scenario run through the C restatement (oracle/) and the
unmodified reference harness (oracle/_ref) with identical results."""
import ctypes as C

import pytest

from attack_backends import HarnessBackend
from attack_scenarios import SCENARIOS, plans_for, result_key
from oracle_c import OracleEngine, OracleRules
from paper_2508_08438_b200.attack import SplitMix64, derive_seed, run_campaign
from refh import RefEngine, RefRules


def test_rng_matches_reference(ref):
    ref.ref_derive_seed.restype = C.c_uint64
    ref.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
    for root, tag in [(0, 0), (7, 3), (1, 0x5EC7), (2**63 + 5, 2**40)]:
        assert derive_seed(root, tag) == ref.ref_derive_seed(root, tag)
    r = SplitMix64(12345)
    assert [r.next() for _ in range(3)] == [0x22118258A9D111A0, 0x346EDCE5F713F8ED, 0x1E9A57BC80E6721D]


def _run(name, backend_factory):
    rules, plans, st, ck = plans_for(name)
    m, res = run_campaign(backend_factory(rules), plans, st, **ck)
    return m, res


@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_campaign_restatement_matches_reference(ref, name):
    m_o, r_o = _run(name, lambda rules: HarnessBackend(OracleEngine(OracleRules(rules) if rules else OracleRules(),
                                                                    B=4, W=32)))
    re_ = None

    def mk(rules):
        nonlocal re_
        re_ = RefEngine(ref, RefRules(ref, rules), B=4, W=32)
        return HarnessBackend(re_)

    try:
        m_r, r_r = _run(name, mk)
    finally:
        re_.close()
    assert result_key(m_o, r_o) == result_key(m_r, r_r)
    d = m_r.to_dict()
    if name == "detected":
        assert d["defense_success_rate"] == 1.0
    elif name == "undetected":
        assert d["attack_success_rate"] == 1.0
    elif name == "monitored":
        assert d["leakage_events"] > 0 and d["downgraded_mid_attack"] == d["n_secrets"]
        assert d["attack_success_rate"] == 0.0
    elif name == "budget":
        assert d["budget_exhausted"] == d["n_secrets"] and d["probes_used"] == 28 * d["n_secrets"]
