"""Cross-batch pipelining (skv_prefetch): an engine that stages batch k+1's digests and
window masks on its side stream while batch k commits must produce exactly the
outputs, index contents and events of the reference harness run without it."""
import ctypes as C

import numpy as np
import pytest

from paper_2508_08438_b200 import AdmissionEngine, EngineConfig
from paper_2508_08438_b200 import native as N
from refh import RefEngine, RefRules
from test_gpu_parity import check_events, check_index, device_to_rule_masks
from workloads import make_batch, make_trunks

pytestmark = pytest.mark.gpu


def _dev_batch(torch, dev, batch):
    tok, off, users, owners = batch
    t = torch.from_numpy(np.ascontiguousarray(tok).view(np.int32)).to(dev)
    o = torch.from_numpy(np.ascontiguousarray(off).view(np.int64)).to(dev)
    u = torch.from_numpy(np.ascontiguousarray(users).view(np.int64)).to(dev)
    w = torch.from_numpy(np.ascontiguousarray(owners)).to(dev)
    nb = N.Batch(t.data_ptr(), o.data_ptr(), u.data_ptr(), w.data_ptr(), len(off) - 1, len(tok), 1)
    return nb, (t, o, u, w)


def _admit_out(n_prompts, n_blocks_max):
    bufs = dict(block_h=np.zeros(n_blocks_max, np.uint64), block_d=np.zeros(n_blocks_max, np.uint64),
                label=np.zeros(n_blocks_max, np.uint8), rule_mask=np.zeros(n_blocks_max, np.uint32),
                decision=np.zeros(n_blocks_max, np.uint8), matched_blocks=np.zeros(n_prompts, np.uint32),
                lowest_tier=np.zeros(n_prompts, np.uint8))
    o = N.AdmitOut(*(bufs[k].ctypes.data for k in ("block_h", "block_d", "label", "rule_mask", "decision",
                                                   "matched_blocks", "lowest_tier")), None, 0, 0, 0)
    return o, bufs


@pytest.mark.parametrize("mode", ["device", "host"])
@pytest.mark.parametrize("seed,B,W", [(71, 16, 32), (72, 4, 8)])
def test_prefetch_pipeline_parity(ref, gpu, seed, B, W, mode):
    import torch
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(seed)
    trunks = make_trunks(rng, 12)
    batches = [make_batch(rng, trunks, 150, 4) for _ in range(6)]
    dbs = [_dev_batch(torch, dev, b) for b in batches] if mode == "device" else None
    torch.cuda.synchronize()
    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 18, max_prompts=4096,
                       max_tokens=1 << 20, max_window_entries=1 << 15, entropy_jump=0.3, u_pre_max=1)

    def prefetch(eng, k):
        if mode == "device":
            eng.prefetch_raw(dbs[k][0])
        else:
            eng.prefetch(*batches[k])

    def admit(eng, k):
        if mode == "host":
            r = eng.admit(*batches[k])
            return r.n_blocks, dict(block_h=r.block_h, block_d=r.block_d, label=r.label, rule_mask=r.rule_mask,
                                    decision=r.decision, matched_blocks=r.matched_blocks,
                                    lowest_tier=r.lowest_tier)
        o, got = _admit_out(len(batches[k][2]), len(batches[k][0]) // B + 1)
        eng.admit_raw(dbs[k][0], o)
        return o.n_blocks, got

    with AdmissionEngine(cfg) as eng:
        rs = eng.rules
        re_ = RefEngine(ref, RefRules(ref, None), B=B, W=W, jump=0.3, u_pre_max=1)
        try:
            prefetch(eng, 0)
            for k, batch in enumerate(batches):
                n, got = admit(eng, k)
                assert eng.times()["prefetched"] == 1
                if k + 1 < len(batches):
                    prefetch(eng, k + 1)  # overlaps this batch's commit
                exp = re_.admit(*batch)
                assert n == len(exp["block_h"])
                np.testing.assert_array_equal(got["block_d"][:n], exp["block_d"])
                np.testing.assert_array_equal(got["block_h"][:n], exp["block_h"])
                np.testing.assert_array_equal(device_to_rule_masks(rs, got["rule_mask"][:n]), exp["mask"])
                np.testing.assert_array_equal(got["label"][:n], exp["label"])
                np.testing.assert_array_equal(got["decision"][:n], exp["decision"])
                np.testing.assert_array_equal(got["matched_blocks"], exp["matched_blocks"])
                np.testing.assert_array_equal(got["lowest_tier"], exp["lowest_tier"])
                eng.commit()
                re_.commit()
                ep_g, ev_g = eng.epoch_pass()
                ep_r, ev_r = re_.epoch(cap=1 << 16)
                assert ep_g == ep_r
                check_events(ev_g, ev_r)
                check_index(eng, re_)
        finally:
            re_.close()


def test_prefetch_mismatch_is_dropped(gpu):
    """A prefetch for a different batch than the one admitted is discarded, and
    skv_set_rules drops a staged scan made under the previous rule snapshot."""
    import torch
    from paper_2508_08438_b200 import RuleSet
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    trunks = make_trunks(rng, 6)
    b0, b1 = make_batch(rng, trunks, 64, 3), make_batch(rng, trunks, 64, 3)
    d0, d1 = _dev_batch(torch, dev, b0), _dev_batch(torch, dev, b1)
    torch.cuda.synchronize()
    cfg = EngineConfig(block_tokens=16, window_tokens=32, index_capacity=1 << 16, max_prompts=1024,
                       max_tokens=1 << 18)
    with AdmissionEngine(cfg) as a, AdmissionEngine(cfg) as b:
        a.prefetch(*b1)
        ra = a.admit(*b0)          # a different batch: the staged b1 is dropped
        assert a.times()["prefetched"] == 0
        rb = b.admit(*b0)
        np.testing.assert_array_equal(ra.label, rb.label)
        a.commit(), b.commit()
        a.prefetch_raw(d1[0])
        a.set_rules(RuleSet.from_json('{"version": 2, "rules": ['
                                      '{"rule_id": "x", "category": "X", "kind": "regex", "pattern": "a"}]}'))
        o, got = _admit_out(64, len(b1[0]) // 16 + 1)
        a.admit_raw(d1[0], o)
        assert a.times()["prefetched"] == 0
        with AdmissionEngine(cfg) as c_:
            c_.set_rules(RuleSet.from_json('{"version": 2, "rules": ['
                                           '{"rule_id": "x", "category": "X", "kind": "regex", "pattern": "a"}]}'))
            c_.admit(*b0)
            c_.commit()
            rc = c_.admit(*b1)
            np.testing.assert_array_equal(got["rule_mask"][:o.n_blocks], rc.rule_mask)
            np.testing.assert_array_equal(got["label"][:o.n_blocks], rc.label)


def test_byte_token_batches(ref, gpu):
    """Byte tokens (skv_batch::token_bytes, the reference's ByteVocabulary) give exactly the
    TokenId path's results -- host and device batches, inline and prefetched."""
    import torch
    from paper_2508_08438_b200 import native as N
    from test_gpu_parity import check_admit, check_index
    rng = np.random.default_rng(77)
    trunks = make_trunks(rng, 8)
    batches = [make_batch(rng, trunks, 120, 5) for _ in range(4)]
    cfg = EngineConfig(block_tokens=16, window_tokens=32, index_capacity=1 << 16, max_prompts=1024,
                       max_tokens=1 << 18, max_window_entries=1 << 14)
    with AdmissionEngine(cfg) as a, AdmissionEngine(cfg) as b:
        re_ = RefEngine(ref, RefRules(ref), B=16, W=32)
        try:
            for k, (tok, off, users, owners) in enumerate(batches):
                t8 = tok.astype(np.uint8)
                if k % 2 == 0:  # host byte batch
                    got = a.admit(t8, off, users, owners)
                else:           # device byte batch, prefetched then admitted
                    dev = torch.device("cuda", 0)
                    dt = torch.from_numpy(t8.copy()).to(dev)
                    do = torch.from_numpy(off.view(np.int64)).to(dev)
                    du = torch.from_numpy(users.view(np.int64)).to(dev)
                    dw = torch.from_numpy(owners).to(dev)
                    bat = N.Batch(None, do.data_ptr(), du.data_ptr(), dw.data_ptr(), len(off) - 1, len(tok), 1,
                                  dt.data_ptr())
                    a.prefetch_raw(bat)
                    a.admit_raw(bat)
                    got = None
                exp_u32 = b.admit(tok, off, users, owners)
                exp = re_.admit(tok, off, users, owners)
                check_admit(b.rules, exp_u32, exp)
                if got is not None:
                    check_admit(a.rules, got, exp)
                a.commit()
                b.commit()
                re_.commit()
                check_index(a, re_)
        finally:
            re_.close()


@pytest.mark.parametrize("byte_tokens", [False, True])
@pytest.mark.parametrize("pattern", ["stage+prefetch", "stage-only", "mixed"])
def test_staged_host_pipeline_parity(ref, gpu, pattern, byte_tokens):
    """skv_stage (host-input copies queued ahead on the copy stream, two slots) under the
    end-to-end bench's call pattern -- admit(k), prefetch(k+1), commit(k), stage(k+2), epoch --
    and with staged batches admitted without a prefetch: outputs, events and the index equal
    the reference harness's after every batch."""
    B, W = 16, 32
    rng = np.random.default_rng(90 + len(pattern) + byte_tokens)
    trunks = make_trunks(rng, 12)
    batches = [make_batch(rng, trunks, 150, 4) for _ in range(7)]
    # the caller's host buffers, alive and unchanged until each batch's admit
    keep = []
    for tok, off, users, owners in batches:
        t = np.ascontiguousarray(tok, dtype=np.uint8 if byte_tokens else np.uint32)
        o, u, w = (np.ascontiguousarray(a) for a in (off, users, owners))
        keep.append((t, o.astype(np.uint64), u.astype(np.uint64), w.astype(np.uint8)))

    def hb(k):
        t, o, u, w = keep[k]
        if byte_tokens:
            return N.Batch(None, o.ctypes.data, u.ctypes.data, w.ctypes.data, len(o) - 1, len(t), 0, t.ctypes.data)
        return N.Batch(t.ctypes.data, o.ctypes.data, u.ctypes.data, w.ctypes.data, len(o) - 1, len(t), 0)

    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 18, max_prompts=4096,
                       max_tokens=1 << 20, max_window_entries=1 << 15, entropy_jump=0.3, u_pre_max=1)
    with AdmissionEngine(cfg) as eng:
        rs = eng.rules
        re_ = RefEngine(ref, RefRules(ref, None), B=B, W=W, jump=0.3, u_pre_max=1)
        try:
            eng.stage_raw(hb(0))
            eng.stage_raw(hb(1))
            if pattern != "stage-only":
                eng.prefetch_raw(hb(0))
            for k, batch in enumerate(batches):
                o, got = _admit_out(len(batch[2]), len(batch[0]) // B + 1)
                eng.admit_raw(hb(k), o)
                use_pf = pattern == "stage+prefetch" or (pattern == "mixed" and k % 3 != 1)
                if k + 1 < len(batches) and use_pf:
                    eng.prefetch_raw(hb(k + 1))
                exp = re_.admit(*batch)
                n = o.n_blocks
                assert n == len(exp["block_h"])
                np.testing.assert_array_equal(got["block_d"][:n], exp["block_d"])
                np.testing.assert_array_equal(got["block_h"][:n], exp["block_h"])
                np.testing.assert_array_equal(device_to_rule_masks(rs, got["rule_mask"][:n]), exp["mask"])
                np.testing.assert_array_equal(got["label"][:n], exp["label"])
                np.testing.assert_array_equal(got["decision"][:n], exp["decision"])
                np.testing.assert_array_equal(got["matched_blocks"], exp["matched_blocks"])
                np.testing.assert_array_equal(got["lowest_tier"], exp["lowest_tier"])
                eng.commit()
                re_.commit()
                if k + 2 < len(batches):
                    eng.stage_raw(hb(k + 2))
                ep_g, ev_g = eng.epoch_pass()
                ep_r, ev_r = re_.epoch(cap=1 << 16)
                assert ep_g == ep_r
                check_events(ev_g, ev_r)
                check_index(eng, re_)
        finally:
            re_.close()


@pytest.mark.parametrize("byte_tokens", [False, True])
def test_step_host_pipeline_parity(ref, gpu, byte_tokens):
    """skv_step with the end-to-end call pattern folded into one call per batch -- admit(k) with
    host outputs, prefetch(k+1), commit(k), stage(k+2), epoch, one synchronisation: the outputs
    (filled by the step's synchronisation), events and the index equal the reference harness's
    after every batch."""
    B, W = 16, 32
    rng = np.random.default_rng(404 + byte_tokens)
    trunks = make_trunks(rng, 12)
    batches = [make_batch(rng, trunks, 150, 4) for _ in range(7)]
    keep = []
    for tok, off, users, owners in batches:
        t = np.ascontiguousarray(tok, dtype=np.uint8 if byte_tokens else np.uint32)
        keep.append((t, off.astype(np.uint64), users.astype(np.uint64), owners.astype(np.uint8)))

    def hb(k):
        t, o, u, w = keep[k]
        if byte_tokens:
            return N.Batch(None, o.ctypes.data, u.ctypes.data, w.ctypes.data, len(o) - 1, len(t), 0, t.ctypes.data)
        return N.Batch(t.ctypes.data, o.ctypes.data, u.ctypes.data, w.ctypes.data, len(o) - 1, len(t), 0)

    cfg = EngineConfig(block_tokens=B, window_tokens=W, index_capacity=1 << 18, max_prompts=4096,
                       max_tokens=1 << 20, max_window_entries=1 << 15, entropy_jump=0.3, u_pre_max=1)
    with AdmissionEngine(cfg) as eng:
        rs = eng.rules
        re_ = RefEngine(ref, RefRules(ref, None), B=B, W=W, jump=0.3, u_pre_max=1)
        try:
            eng.stage_raw(hb(0))
            eng.stage_raw(hb(1))
            eng.prefetch_raw(hb(0))
            for k, batch in enumerate(batches):
                o, got = _admit_out(len(batch[2]), len(batch[0]) // B + 1)
                nxt = hb(k + 1) if k + 1 < len(batches) else None
                stg = hb(k + 2) if k + 2 < len(batches) else None
                _, ep_g, ev_g = eng.step_raw(hb(k), out=o, next_batch=nxt, stage=stg)
                exp = re_.admit(*batch)
                n = o.n_blocks
                assert n == len(exp["block_h"])
                np.testing.assert_array_equal(got["block_h"][:n], exp["block_h"])
                np.testing.assert_array_equal(device_to_rule_masks(rs, got["rule_mask"][:n]), exp["mask"])
                np.testing.assert_array_equal(got["label"][:n], exp["label"])
                np.testing.assert_array_equal(got["decision"][:n], exp["decision"])
                np.testing.assert_array_equal(got["matched_blocks"], exp["matched_blocks"])
                np.testing.assert_array_equal(got["lowest_tier"], exp["lowest_tier"])
                re_.commit()
                ep_r, ev_r = re_.epoch(cap=1 << 16)
                assert ep_g == ep_r
                check_events(ev_g, ev_r)
                check_index(eng, re_)
                assert eng.times()["prefetched"] == 1  # every batch was staged and prefetched
        finally:
            re_.close()
