"""Degenerate inputs and capacity limits on the CUDA path: empty batches, batches of only
sub-block prompts, batch limits, an index driven past its capacity, and eviction on an
empty index -- each with the reference's behaviour where the reference has one."""
import numpy as np
import pytest

from paper_2508_08438_b200 import AdmissionEngine, ArgError, CapacityExhausted, EngineConfig, StateError
from refh import RefEngine, RefRules
from test_gpu_parity import check_admit, check_index

pytestmark = pytest.mark.gpu


def _cfg(**kw):
    base = dict(block_tokens=16, window_tokens=32, index_capacity=1 << 12, max_prompts=64, max_tokens=1 << 14,
                max_window_entries=1 << 10)
    base.update(kw)
    return EngineConfig(**base)


def _batch(lengths, seed=0, users=None):
    rng = np.random.default_rng(seed)
    toks = [rng.integers(ord("a"), ord("z") + 1, n).astype(np.uint32) for n in lengths]
    off = np.zeros(len(lengths) + 1, np.uint64)
    np.cumsum(lengths, out=off[1:])
    tok = np.concatenate(toks) if toks else np.zeros(0, np.uint32)
    u = np.arange(1, len(lengths) + 1, dtype=np.uint64) if users is None else users
    return tok, off, u, np.zeros(len(lengths), np.uint8)


@pytest.mark.parametrize("lengths", [[], [0, 0, 3], [15, 1, 7, 0]])
def test_empty_and_sub_block_batches(ref, gpu, lengths):
    with AdmissionEngine(_cfg()) as eng:
        re_ = RefEngine(ref, RefRules(ref), B=16, W=32)
        try:
            for k in range(2):
                b = _batch(lengths, seed=k)
                got = eng.admit(*b)
                exp = re_.admit(*b)
                assert got.n_blocks == 0
                check_admit(eng.rules, got, exp)
                assert eng.commit() == 0
                re_.commit()
                eng.epoch_pass()
                re_.epoch()
                check_index(eng, re_)
            assert eng.entry_count() == 0
        finally:
            re_.close()


def test_batch_limits_are_errors(gpu):
    with AdmissionEngine(_cfg(max_prompts=4, max_tokens=256)) as eng:
        with pytest.raises((ArgError, CapacityExhausted)):
            eng.admit(*_batch([16] * 5))          # more prompts than max_prompts
        with pytest.raises((ArgError, CapacityExhausted)):
            eng.admit(*_batch([200, 100]))        # more tokens than max_tokens
        got = eng.admit(*_batch([64, 64]))        # the engine still works
        assert got.n_blocks == 8
        assert eng.commit() == 8


def test_index_capacity_exhausted(gpu):
    """Commits beyond 7/8 of the slots fail loudly (no eviction is implied)."""
    with AdmissionEngine(_cfg(index_capacity=1 << 10, max_prompts=64, max_tokens=1 << 16)) as eng:
        with pytest.raises(CapacityExhausted):
            for k in range(20):
                eng.admit(*_batch([1024] * 4, seed=100 + k))
                eng.commit()
        assert eng.entry_count() <= (1 << 10)


def test_evict_on_empty_index(ref, gpu):
    with AdmissionEngine(_cfg()) as eng:
        eng.enable_eviction()
        with pytest.raises(CapacityExhausted):
            eng.evict(5)
        assert eng._evicted[0] == 0
    re_ = RefEngine(ref, RefRules(ref), B=16, W=32)
    try:
        assert re_.evict(5) == (1, 0)
    finally:
        re_.close()


def test_enable_eviction_after_inserts_is_an_error(gpu):
    with AdmissionEngine(_cfg()) as eng:
        eng.admit(*_batch([32, 48]))
        eng.commit()
        with pytest.raises(StateError):
            eng.enable_eviction()
