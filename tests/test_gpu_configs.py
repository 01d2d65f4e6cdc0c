"""Parity of the CUDA path against the reference on reduced-size instances of
BASELINE.json configs 3-5 (config 2 is the bench workload; config 1 is pinned by
test_gpu_golden.test_config1_golden).  Every admit output, every epoch's leakage events
and the whole index (creators, labels, tiers, window stats) must equal the UNMODIFIED
reference (oracle/_ref/libsafekv_ref.so) driven on the same inputs.

* config 3 -- 4k-token prompts over the shared pool, 256 users, mixed PII density
  (60% none / 30% one per 2 KiB / 10% one per 256 B, skv_gen_spec.pii_mix), prefix-forest
  routed shard of a 2-GPU world.
* config 4 -- long-context prompts in 128-token blocks over a pre-built tiered index:
  stored sequences tagged HBM/DRAM/SSD by derive_seed(seed, entry) mod 10 (0-1 / 2-4 /
  5-9), queried by random-length prefixes of the stored sequences + fresh text, so the
  matches are long and lowest_tier is mixed (cache_index.hpp:234-235).
* config 5 -- adversarial probing mix: victims with account-number secrets behind a
  shared system prompt; 10% attacker probes (identities >= 1,000,000 rotated over 4,
  adversary.hpp:30,88-90) of the form known prefix + recovered digits + candidate digit
  (adversary.hpp:114-116); monitor epoch after EVERY batch (K = 1).
"""
import ctypes as C

import numpy as np
import pytest

from paper_2508_08438_b200 import AdmissionEngine, EngineConfig
from workload import GenSpec, generate, generate_pool
from refh import RefEngine, RefRules
from test_gpu_parity import check_admit, check_events, check_index

pytestmark = pytest.mark.gpu


def _run(eng, re_, rs, batches, epoch_every=1):
    fired = 0
    for k, batch in enumerate(batches):
        got = eng.admit(*batch)
        exp = re_.admit(*batch)
        check_admit(rs, got, exp)
        eng.commit()
        re_.commit()
        if (k + 1) % epoch_every == 0:
            ep_g, ev_g = eng.epoch_pass()
            ep_r, ev_r = re_.epoch(cap=1 << 16)
            assert ep_g == ep_r
            check_events(ev_g, ev_r)
            fired += len(ev_g)
        check_index(eng, re_)
    return fired


def _cfg(**kw):
    base = dict(block_tokens=16, window_tokens=32, index_capacity=1 << 20, max_prompts=4096, max_tokens=1 << 22,
                max_window_entries=1 << 17)
    base.update(kw)
    return EngineConfig(**base)


def test_config3_mixed_density_routed_shard(ref, gpu):
    """Config 3 shape: the rank-1 shard of a 2-GPU routed stream (4,096-token prompts,
    256 users, mixed PII density) over its share of the shared-prefix pool."""
    spec = GenSpec(n_prompts=192, prompt_tokens=4096, n_users=256, pii_mix=1, seed=3, route_world=2, route_rank=1,
                   route_block_tokens=16)
    pool = generate_pool(spec, 1)
    batches = [pool]
    for k in range(3):
        spec.prompt_id_base = (k + 1) * 1_000_000
        batches.append(generate(spec))
    with AdmissionEngine(_cfg()) as eng:
        re_ = RefEngine(ref, RefRules(ref), B=16, W=32, threads=8)
        try:
            _run(eng, re_, eng.rules, batches)
        finally:
            re_.close()


def _letters(rng, n):
    return rng.integers(ord("a"), ord("z") + 1, n, dtype=np.uint32)


def _with_pii(rng, toks, per_kib):
    phrases = [b"my ssn is 123-45-6789 ", b"account number 48392057 ", b"email me at user99@mail01.com ",
               b"card number 4111-1111-1111-1111 ", b"imei 490154203237518 ", b"PROJECT-TITAN "]
    k = rng.poisson(per_kib * len(toks) / 1024)
    for _ in range(k):
        ph = np.frombuffer(phrases[rng.integers(len(phrases))], np.uint8).astype(np.uint32)
        at = int(rng.integers(0, max(1, len(toks) - len(ph))))
        toks[at:at + len(ph)] = ph
    return toks


def test_config4_long_context_tiered_index(ref, gpu):
    """Config 4 shape: 128-token blocks, W = 32, long prompts matched against a
    pre-built index whose entries carry HBM/DRAM/SSD tier tags."""
    B, W, L = 128, 32, 8192
    rng = np.random.default_rng(404)
    n_stored, n_query = 10, 40
    stored = [_with_pii(rng, _letters(rng, L), 0.5) for _ in range(n_stored)]
    s_tok = np.concatenate(stored).astype(np.uint32)
    s_off = np.arange(n_stored + 1, dtype=np.uint64) * L
    s_users = np.arange(1, n_stored + 1, dtype=np.uint64)
    s_own = (np.arange(n_stored) % 3 == 0).astype(np.uint8)
    # tier tag of stored entry e: derive_seed(seed, e) mod 10 -> 0-1 HBM, 2-4 DRAM, 5-9 SSD
    nb = (L // B) * n_stored
    ref.ref_derive_seed.restype = C.c_uint64
    ref.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
    r = np.array([ref.ref_derive_seed(404, e) % 10 for e in range(nb)], np.uint64)
    tiers = np.where(r < 2, 0, np.where(r < 5, 1, 2)).astype(np.uint8)
    q_tok, q_off, q_users = [], [0], []
    for q in range(n_query):
        k = int(rng.integers(n_stored))
        # uniform prefix length (config 4); every third query a short one, so that
        # lowest_tier (the slowest tier on the matched path) takes all three values
        cut = int(rng.integers(0, L + 1)) if q % 3 else int(rng.integers(0, 3 * B))
        t = np.concatenate([stored[k][:cut], _with_pii(rng, _letters(rng, L - cut), 1.0)])
        q_tok.append(t)
        q_off.append(q_off[-1] + len(t))
        q_users.append(int(rng.integers(1, n_stored + 3)))  # creators (owner hits on Private) and others
    query = (np.concatenate(q_tok).astype(np.uint32), np.array(q_off, np.uint64), np.array(q_users, np.uint64),
             (np.array(q_users) % 3 == 0).astype(np.uint8))
    with AdmissionEngine(_cfg(block_tokens=B, window_tokens=W)) as eng:
        re_ = RefEngine(ref, RefRules(ref), B=B, W=W, threads=8)
        try:
            got = eng.admit(s_tok, s_off, s_users, s_own)
            exp = re_.admit(s_tok, s_off, s_users, s_own)
            check_admit(eng.rules, got, exp)
            eng.commit()
            re_.commit()
            eng.set_tiers(got.block_h, got.block_d, tiers, got.block_offsets)
            re_.set_tiers(s_tok, s_off, tiers)
            check_index(eng, re_)
            got = eng.admit(*query)
            exp = re_.admit(*query)
            check_admit(eng.rules, got, exp)
            assert len(set(exp["lowest_tier"].tolist())) == 3, "queries should see all three tiers"
            assert (exp["matched_blocks"] > 8).sum() > n_query // 3, "queries should have long matches"
            eng.commit()
            re_.commit()
            ep_g, ev_g = eng.epoch_pass()
            ep_r, ev_r = re_.epoch(cap=1 << 16)
            assert ep_g == ep_r
            check_events(ev_g, ev_r)
            check_index(eng, re_)
        finally:
            re_.close()


def test_config5_adversarial_probing_epoch_every_batch(ref, gpu):
    """Config 5 shape: victims' secrets behind a shared prefix; attacker probes
    (rotating identities) walk the secret digit by digit; the monitor runs after every
    batch and must flag the probed public entries exactly as the reference does."""
    B, W = 4, 8  # small blocks: probes resolve near token granularity
    rng = np.random.default_rng(505)
    system = np.frombuffer(b"system: you are a helpful banking assistant. ", np.uint8).astype(np.uint32)
    secrets = [f"{int(rng.integers(10**7, 10**8))}" for _ in range(6)]
    victims = [np.concatenate([system, np.frombuffer(f"my account number {s} thanks".encode(), np.uint8)
                               .astype(np.uint32)]) for s in secrets]
    batches = []
    recovered = [0] * len(secrets)
    for k in range(8):
        toks, users = [], []
        for i in range(40):
            if i % 10 == 0:  # attacker probe: known prefix + recovered digits + candidate digit
                v = int(rng.integers(len(secrets)))
                n_rec = recovered[v]
                guess = secrets[v][:n_rec] + str(int(rng.integers(10)))
                recovered[v] = min(n_rec + 1, len(secrets[v]))
                t = np.concatenate([system, np.frombuffer(f"my account number {guess}".encode(), np.uint8)
                                    .astype(np.uint32)])
                toks.append(t)
                users.append(1_000_000 + (k * 4 + i // 10) % 4)
            else:  # benign traffic and the victims themselves
                v = int(rng.integers(len(secrets)))
                if rng.random() < 0.5:
                    toks.append(victims[v])
                    users.append(10 + v)
                else:
                    tail = np.frombuffer(f"question {int(rng.integers(1000))} about fees".encode(), np.uint8)
                    toks.append(np.concatenate([system, tail.astype(np.uint32)]))
                    users.append(100 + int(rng.integers(40)))
        off = np.zeros(len(toks) + 1, np.uint64)
        np.cumsum([len(t) for t in toks], out=off[1:])
        batches.append((np.concatenate(toks).astype(np.uint32), off, np.array(users, np.uint64),
                        np.zeros(len(toks), np.uint8)))
    with AdmissionEngine(_cfg(block_tokens=B, window_tokens=W)) as eng:
        re_ = RefEngine(ref, RefRules(ref), B=B, W=W)
        try:
            fired = _run(eng, re_, eng.rules, batches, epoch_every=1)
        finally:
            re_.close()
    assert fired > 0, "the probing mix should trip the entropy monitor"
