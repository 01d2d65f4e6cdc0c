"""GPU parity of the serving observables: the TTFT cost model and
the reuse attribution computed from the probe's per-block results, against the
reference's own CostModel::ttft (serving_sim.hpp:50-56) and attribute_reuse
(:313-324) run on the reference harness's matches.  Bit-exact without noise; with the
Box-Muller noise term within 1e-12 relative (device vs libm log/cos)."""
import numpy as np
import pytest

from paper_2508_08438_b200 import AdmissionEngine, EngineConfig
from paper_2508_08438_b200.native import ConfigError
from refh import RefEngine, RefRules
from workloads import make_batch, make_trunks

pytestmark = pytest.mark.gpu

MODELS = [
    dict(t_base_ms=10.0, c_prefill_ms=1.0, tier_penalty_ms=(0.0, 0.2, 0.5), noise_sigma_ms=0.0, seed=0),
    dict(t_base_ms=3.5, c_prefill_ms=0.7, tier_penalty_ms=(0.0, 0.13, 0.31), noise_sigma_ms=2.5, seed=99),
]


@pytest.mark.parametrize("model", MODELS)
@pytest.mark.parametrize("B,W", [(16, 32), (8, 16)])
def test_ttft_reuse_parity(ref, gpu, model, B, W):
    rng = np.random.default_rng(600 + B)
    trunks = make_trunks(rng, 10)
    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 18, max_prompts=4096,
                       max_tokens=1 << 20, max_window_entries=1 << 15)
    with AdmissionEngine(cfg) as eng:
        eng.set_cost_model(**model)
        re_ = RefEngine(ref, RefRules(ref), B=B, W=W)
        try:
            for k in range(4):
                batch = make_batch(rng, trunks, 200, 5)
                n = len(batch[1]) - 1
                got = eng.admit(*batch)
                exp = re_.admit(*batch)
                np.testing.assert_array_equal(got.matched_blocks, exp["matched_blocks"])
                rid = np.arange(5000 * k, 5000 * k + n, dtype=np.uint64)
                tg, ig, xg = eng.ttft(n, rid)
                tr, ir, xr = re_.ttft(n, model, rid)
                np.testing.assert_array_equal(ig, ir, "intra-user reuse tokens")
                np.testing.assert_array_equal(xg, xr, "inter-user reuse tokens")
                if model["noise_sigma_ms"] == 0:
                    np.testing.assert_array_equal(tg, tr, "ttft")
                else:
                    np.testing.assert_allclose(tg, tr, rtol=1e-12, atol=0)
                eng.commit()
                re_.commit()
                # demote a random share of this batch's blocks (tiers only move down)
                tiers = rng.integers(0, 3, got.n_blocks).astype(np.uint8)
                eng.set_tiers(got.block_h, got.block_d, tiers, got.block_offsets)
                re_.set_tiers(batch[0], batch[1], tiers)
        finally:
            re_.close()


def test_cost_model_validation(gpu):
    with AdmissionEngine(EngineConfig(max_prompts=16, max_tokens=1 << 12, index_capacity=1 << 12)) as eng:
        for bad in (dict(tier_penalty_ms=(0.0, 0.6, 0.5)), dict(c_prefill_ms=0.4), dict(noise_sigma_ms=-1.0)):
            with pytest.raises(ConfigError):
                eng.set_cost_model(**bad)
