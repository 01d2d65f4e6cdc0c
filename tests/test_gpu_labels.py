"""GPU parity of asynchronous label landing: new entries committed as
PendingPrivate (visible to their creator only, cache_index.hpp:196-198) and labels landed
later with RadixCacheIndex::resolve_block semantics (cache_index.hpp:321-343): Public
spans label every block without propagation, Private/Restricted spans label the span's
top and every descendant.  Compared with the reference harness driven identically
(admit outputs, leakage events and the whole index export)."""
import numpy as np
import pytest

from paper_2508_08438_b200 import AdmissionEngine, EngineConfig
from paper_2508_08438_b200.native import ArgError
from refh import RefEngine, RefRules
from test_gpu_parity import check_admit, check_events, check_index
from workloads import make_batch, make_trunks

pytestmark = pytest.mark.gpu

LABELS = np.array([1, 0, 3], np.uint8)  # Public, Private, Restricted


@pytest.mark.parametrize("B,W", [(4, 8), (16, 32)])
def test_pending_then_resolve_parity(ref, gpu, B, W):
    rng = np.random.default_rng(900 + B)
    trunks = make_trunks(rng, 8)
    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 18, max_prompts=4096,
                       max_tokens=1 << 20, max_window_entries=1 << 15)
    with AdmissionEngine(cfg) as eng:
        eng.set_label_policy(True)
        re_ = RefEngine(ref, RefRules(ref), B=B, W=W)
        re_.set_pending(True)
        try:
            for k in range(6):
                batch = make_batch(rng, trunks, 150, 4)
                got = eng.admit(*batch)
                exp = re_.admit(*batch)
                check_admit(eng.rules, got, exp)
                eng.commit()
                re_.commit()
                check_index(eng, re_)  # new entries PendingPrivate on both sides
                # land labels for a random half of the batch's prompts, spans [f, n)
                n = len(batch[1]) - 1
                nb = np.diff(got.block_offsets.astype(np.int64))
                sel = rng.random(n) < 0.5
                first = np.array([int(rng.integers(0, m + 1)) for m in nb], np.uint32)
                first[~sel] = nb[~sel]  # empty span: nothing landed
                labels = LABELS[rng.integers(0, 3, n)]
                eng.resolve_blocks(got.block_h, got.block_d, got.block_offsets, first, labels)
                re_.resolve(batch[0], batch[1], first, labels)
                check_index(eng, re_)
                ep_g, ev_g = eng.epoch_pass()
                ep_r, ev_r = re_.epoch(cap=1 << 16)
                assert ep_g == ep_r
                check_events(ev_g, ev_r)
        finally:
            re_.close()


def test_resolve_rejects_bad_input(gpu):
    with AdmissionEngine(EngineConfig(block_tokens=4, window_tokens=0, max_prompts=16, max_tokens=1 << 12,
                                      index_capacity=1 << 12)) as eng:
        t = np.arange(8, dtype=np.uint32)
        got = eng.admit(t, np.array([0, 8], np.uint64), np.array([1], np.uint64))
        eng.commit()
        with pytest.raises(ArgError):  # PendingPrivate is not a landing label
            eng.resolve_blocks(got.block_h, got.block_d, got.block_offsets, np.zeros(1, np.uint32),
                               np.array([2], np.uint8))
        with pytest.raises(ArgError):  # a span whose blocks are not in the index
            eng.resolve_blocks(got.block_h + 1, got.block_d, got.block_offsets, np.zeros(1, np.uint32),
                               np.array([0], np.uint8))
