"""Attack-campaign scenarios shared by the CPU (restatement vs reference) and GPU
(CUDA vs reference) parity tests."""
from paper_2508_08438_b200.attack import AttackSettings, digit_secret_plans

NO_DETECTION = ('{"version": 1, "rules": [{"rule_id": "none", "category": "X", "kind": "blacklist", '
                '"pattern": "qqqqqqqqqqqq"}]}')

# name -> (rules json or None for the shipped set, plan kwargs, settings, campaign kwargs)
SCENARIOS = {
    # Tier-1 detection labels the account number Private: the attacker never hits
    "detected": (None, dict(n=3, block_tokens=4, digits=16, n_candidates=20), AttackSettings(), {}),
    # no detection, no owner reuse: public secret blocks are recovered block by block
    "undetected": (NO_DETECTION, dict(n=3, block_tokens=4, digits=16, n_candidates=20), AttackSettings(), {}),
    # no detection, the victims reuse their prompts: the entropy monitor fires on the probed
    # public blocks (concentrated history, then many identities) and downgrades them
    # mid-attack
    "monitored": (NO_DETECTION, dict(n=3, block_tokens=4, digits=16, n_candidates=20),
                  AttackSettings(n_identities=64, hit_threshold_ms=12.0), dict(victim_repeats=2)),
    # probe budget runs out inside the second position; CalibrationDiff identities
    "budget": (NO_DETECTION, dict(n=2, block_tokens=4, digits=12, n_candidates=16),
               AttackSettings(pollution="calibration", max_probes=28), {}),
}


def plans_for(name):
    rules, pk, st, ck = SCENARIOS[name]
    return rules, digit_secret_plans(**pk), st, ck


def result_key(m, res):
    """Everything a campaign reports, in comparable form."""
    return (m.to_dict(), [([r.tobytes() for r in x.recovered], x.per_position_correct, x.low_confidence,
                           x.probes_used, x.success, x.budget_exhausted, x.downgraded_mid_attack, x.stale_probes)
                          for x in res])
