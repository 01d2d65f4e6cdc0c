"""Test infrastructure: the reference harness (oracle/_ref) and the C restatement as
attack-campaign backends (paper_2508_08438_b200.attack.Backend)."""
import numpy as np

COST = dict(t_base_ms=10.0, c_prefill_ms=1.0, tier_penalty_ms=(0.0, 0.2, 0.5), noise_sigma_ms=0.0, seed=3)


class HarnessBackend:
    """RefEngine (reference) or OracleEngine (restatement): same interface."""

    def __init__(self, eng, cost=COST):
        self.eng, self.cost = eng, dict(cost)

    def admit(self, tokens, offsets, users):
        self.eng.admit(tokens, offsets, users, np.zeros(len(offsets) - 1, np.uint8))

    def ttft(self, n, request_ids):
        return self.eng.ttft(n, self.cost, request_ids)[0]

    def commit(self):
        self.eng.commit()

    def epoch(self):
        return len(self.eng.epoch(cap=1 << 16)[1])
