"""GPU: the batched attack campaign through the CUDA admission path (TTFT from the
device epilogue) against the unmodified reference harness -- identical per-secret
results and metrics in every scenario -- and one campaign at scale (full 10^4-candidate
positions, one batch of 160k probes per position)."""
import time

import numpy as np
import pytest

from attack_backends import COST, HarnessBackend
from attack_scenarios import NO_DETECTION, SCENARIOS, plans_for, result_key
from paper_2508_08438_b200 import AdmissionEngine, EngineConfig, RuleSet
from paper_2508_08438_b200.attack import AttackSettings, EngineBackend, digit_secret_plans, run_campaign
from refh import RefEngine, RefRules

pytestmark = pytest.mark.gpu


def _engine(rules, max_prompts=1 << 12, max_tokens=1 << 20):
    eng = AdmissionEngine(EngineConfig(block_tokens=4, window_tokens=32, index_capacity=1 << 22,
                                       max_prompts=max_prompts, max_tokens=max_tokens,
                                       max_window_entries=1 << 18))
    if rules is not None:
        eng.set_rules(RuleSet.from_json(rules))
    return eng


@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_campaign_cuda_matches_reference(ref, gpu, name):
    rules, plans, st, ck = plans_for(name)
    with _engine(rules) as eng:
        m_g, r_g = run_campaign(EngineBackend(eng, COST), plans, st, **ck)
    re_ = RefEngine(ref, RefRules(ref, rules), B=4, W=32)
    try:
        m_r, r_r = run_campaign(HarnessBackend(re_), plans, st, **ck)
    finally:
        re_.close()
    assert result_key(m_g, r_g) == result_key(m_r, r_r)


def test_campaign_at_scale(gpu):
    """16 secrets x 10,000 candidates per 4-digit block: 160,000 probes per batch."""
    out = {}
    for label, rules in (("undetected", NO_DETECTION), ("detected", None)):
        plans = digit_secret_plans(16, 4, digits=8)
        with _engine(rules, max_prompts=1 << 18, max_tokens=1 << 24) as eng:
            t0 = time.perf_counter()
            m, _ = run_campaign(EngineBackend(eng, COST), plans, AttackSettings(n_identities=16))
            out[label] = (m, time.perf_counter() - t0)
    m_u, t_u = out["undetected"]
    m_d, _ = out["detected"]
    assert m_u.probes_used == 16 * 2 * 10_000
    assert m_u.attack_success_rate() == 1.0
    assert m_d.defense_success_rate() == 1.0
    print(f"\n[attack at scale] {m_u.probes_used} probes in {t_u:.2f} s "
          f"({m_u.probes_used / t_u / 1e3:.0f} k probes/s incl. host batching)")
