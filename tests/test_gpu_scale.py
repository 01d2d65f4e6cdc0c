"""GPU parity at the bench's own shapes (VERDICT r01 "parity at scale"): the CUDA path and the
unmodified reference (oracle/_ref, RadixCacheIndex / CompiledRuleSet per-rule masks /
EntropyMonitor under the Appendix-A contract, stages 1-2 on every host thread) admit the SAME
batches bench.py times -- same generator, same global prompt ids, same pool / stored index --
and every output is compared after every step: per-block keys, digests, per-rule window masks,
labels and decisions; per-prompt match lengths and lowest tiers; the epoch's events; the full
index export (keys, creators, labels, owners, tiers, AccessStats windows).

  config 2: the 256 x 640 pool + 2 full 65,536 x 2,048-token batches (16.8 M blocks)
  config 5: 4 batches of 4,096 prompts, every 10th an attacker probe with rotating identities,
            an epoch after every batch
  config 4: B=128, 32,768-token queries over a 500 k-entry stored index with HBM/DRAM/SSD tags
  config 3: a 16,384-prompt routed shard (rank 5 of 8) of 4,096-token prompts, 256 users,
            mixed PII density (full config 3 is throughput-only on the CPU)
"""
import os

import numpy as np
import pytest

import bench
from paper_2508_08438_b200 import AdmissionEngine, EngineConfig
from refh import RefEngine, RefRules
from test_gpu_parity import check_admit, check_events, check_index
from workload import generate_pool

pytestmark = pytest.mark.gpu


def _engines(ref, c, cap_log2, window_log2=18):
    B, W = c["block_tokens"], c["window_tokens"]
    n = c["n_prompts"]
    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << cap_log2, max_prompts=max(n, 4096),
                       max_tokens=max(n, 4096) * c["prompt_tokens"], max_window_entries=1 << window_log2)
    eng = AdmissionEngine(cfg)
    re_ = RefEngine(ref, RefRules(ref), B=B, W=W, threads=os.cpu_count() or 1)
    return eng, re_


def _step(eng, re_, batch, epoch=True, export=True):
    batch = batch[:4]  # bench.build_batch also returns the global prompt ids
    got = eng.admit(*batch)
    exp = re_.admit(*batch)
    check_admit(eng.rules, got, exp)
    eng.commit()
    re_.commit()
    if epoch:
        ep_g, ev_g = eng.epoch_pass()
        ep_r, ev_r = re_.epoch(cap=1 << 20)
        assert ep_g == ep_r
        check_events(ev_g, ev_r)
    if export:
        check_index(eng, re_)
    return got, exp


def test_scale_config2_full_batches(ref, gpu):
    c = bench.CFG2
    eng, re_ = _engines(ref, c, 25)
    try:
        spec = bench.gen_spec(c, c["n_prompts"])
        pool = generate_pool(spec)
        _step(eng, re_, pool)
        matched = 0
        for k in range(2):
            got, _ = _step(eng, re_, bench.build_batch(c, 2, k, c["n_prompts"], spec=spec))
            assert got.n_blocks == 65536 * 128
            matched += int(got.matched_blocks.sum())
        assert matched >= 2 * 65536 * 40  # every prompt reuses its 40-block pool prefix
    finally:
        eng.close()
        re_.close()


def test_scale_config5_adversarial_mix(ref, gpu):
    c = bench.CFG5
    eng, re_ = _engines(ref, c, 24)
    try:
        spec = bench.gen_spec(c, c["n_prompts"])
        _step(eng, re_, generate_pool(spec))
        probes = 0
        for k in range(5):
            batch = bench.build_batch(c, 5, k, c["n_prompts"], spec=spec)
            probes += int((batch[2] >= 1_000_000).sum())
            _step(eng, re_, batch, epoch=True)  # K = 1: an epoch after every batch
        assert probes == 5 * 410
    finally:
        eng.close()
        re_.close()


def test_scale_config4_long_context_tiered(ref, gpu):
    c = dict(bench.CFG4)
    n_stored = 1953  # 1,953 x 256 blocks = 500 k entries
    eng, re_ = _engines(ref, dict(c, n_prompts=c["stored_chunk"]), 22, window_log2=20)
    try:
        chunks = bench.stored_sequences(c, n_stored)
        first = 0
        for t, o, u, w in chunks:
            got, _ = _step(eng, re_, (t, o, u, w), epoch=False, export=False)
            tiers = bench.stored_tiers(c, first, got.n_blocks)
            eng.set_tiers(got.block_h, got.block_d, tiers, got.block_offsets)
            re_.set_tiers(t, o, tiers)
            first += got.n_blocks
        assert first == n_stored * 256
        check_index(eng, re_)
        ep_g, _ = eng.epoch_pass()
        assert ep_g == re_.epoch()[0]
        stored_tok = np.concatenate([t for t, _, _, _ in chunks]).reshape(n_stored, c["prompt_tokens"])
        matched = 0
        for k in range(2):
            got, exp = _step(eng, re_, bench.build_batch(c, 4, k, 256, stored_tok=stored_tok))
            matched += int(got.matched_blocks.sum())
            # the slowest tier of a match (MatchResult::lowest_tier): SSD once it spans many blocks
            assert set(got.lowest_tier[got.matched_blocks > 8].tolist()) <= {2}
        assert matched > 2 * 256 * 16  # long visible matches (uniform prefix lengths, half the prefixes Public)
    finally:
        eng.close()
        re_.close()


def test_scale_config3_routed_shard(ref, gpu):
    c = dict(bench.CFG3, n_prompts=16384)
    eng, re_ = _engines(ref, c, 24)
    try:
        spec = bench.gen_spec(c, c["n_prompts"], world=8, rank=5)
        _step(eng, re_, generate_pool(spec, 5))
        for k in range(2):
            _step(eng, re_, bench.build_batch(c, 3, k, c["n_prompts"], spec=spec))
    finally:
        eng.close()
        re_.close()
