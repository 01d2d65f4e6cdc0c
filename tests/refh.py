"""Test infrastructure: ctypes wrappers of the oracles.

* ``oracle/_ref/libsafekv_ref.so`` -- the UNMODIFIED reference headers compiled with
  oracle/ref_harness.cpp (built here from /root/reference; the prebuilt .so travels to
  the GPU box).
* ``oracle/_ref/liboracle.so`` -- the C restatement (oracle/safekv_oracle.c).

Only tests, __graft_entry__.smoke() and bench.py's CPU-baseline arm use this module.
"""
from __future__ import annotations

import ctypes as C
import pathlib

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
REF_SO = ROOT / "oracle" / "_ref" / "libsafekv_ref.so"
ORC_SO = ROOT / "oracle" / "_ref" / "liboracle.so"

u64p = C.POINTER(C.c_uint64)


def _p(a):
    return None if a is None else a.ctypes.data


def load_ref():
    if not REF_SO.exists():
        return None
    L = C.CDLL(str(REF_SO))
    vp, sz = C.c_void_p, C.c_size_t
    sig = {
        "ref_rules_default": (vp, []),
        "ref_rules_load": (vp, [C.c_char_p, sz, C.c_char_p, sz]),
        "ref_rules_free": (None, [vp]),
        "ref_rules_count": (C.c_uint32, [vp]),
        "ref_rules_verdict": (C.c_int, [vp, C.c_char_p, sz, C.c_char_p, sz]),
        "ref_rules_mask": (C.c_uint64, [vp, C.c_char_p, sz]),
        "ref_rules_mask_wide": (None, [vp, C.c_char_p, sz, vp, sz]),
        "ref_engine_set_stock_scan": (None, [vp, C.c_int]),
        "ref_scan_windows": (C.c_uint64, [vp, vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, vp, C.c_int]),
        "ref_token_seq_digest": (C.c_uint64, [vp, sz]),
        "ref_fnv1a64_bytes": (C.c_uint64, [vp, sz]),
        "ref_chain": (C.c_uint64, [C.c_uint64, C.c_uint64]),
        "ref_block_keys": (C.c_uint64, [vp, vp, C.c_uint32, C.c_uint32, vp, vp]),
        "ref_engine_create": (vp, [vp, C.c_uint32, C.c_uint32, C.c_double, C.c_uint64]),
        "ref_engine_free": (None, [vp]),
        "ref_engine_set_threads": (None, [vp, C.c_int]),
        "ref_engine_set_rules": (None, [vp, vp]),
        "ref_engine_admit": (C.c_int, [vp, vp, vp, vp, vp, C.c_uint32, vp, vp, vp, vp, vp, vp, vp]),
        "ref_engine_commit": (C.c_int, [vp]),
        "ref_engine_set_tiers": (C.c_int, [vp, vp, vp, C.c_uint32, vp]),
        "ref_engine_set_pending": (None, [vp, C.c_int]),
        "ref_engine_resolve": (C.c_int, [vp, vp, vp, C.c_uint32, vp, vp]),
        "ref_engine_ttft": (C.c_int, [vp, vp, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                      C.c_uint64, vp, vp, vp]),
        "ref_engine_epoch": (C.c_int, [vp, u64p, sz, vp, vp, vp, vp, vp, vp, C.POINTER(sz)]),
        "ref_engine_export": (sz, [vp, sz, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "ref_workload_generate": (vp, [C.c_int, C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                       C.c_double, C.c_uint64, C.c_char_p, sz]),
        "ref_workload_free": (None, [vp]),
        "ref_workload_count": (sz, [vp]),
        "ref_workload_digest": (C.c_uint64, [vp]),
        "ref_workload_text": (sz, [vp, sz, C.c_char_p, sz]),
        "ref_workload_user": (C.c_uint64, [vp, sz]),
        "ref_workload_owner": (C.c_uint8, [vp, sz]),
        "ref_workload_truth": (sz, [vp, sz, sz, vp, vp, vp]),
        "ref_rule_corpus": (sz, [sz, C.c_uint64, C.c_char_p, sz, vp]),
        "ref_engine_evict": (C.c_int, [vp, C.c_uint64, C.c_uint64, u64p]),
        "ref_engine_current_epoch": (C.c_uint64, [vp]),
        "ref_engine_set_tiered": (C.c_int, [vp, C.c_int]),
        "ref_engine_set_budget": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]),
        "ref_engine_dropped": (sz, [vp, vp, sz]),
        "ref_engine_budget_used": (None, [vp, vp]),
    }
    for n, (r, a) in sig.items():
        f = getattr(L, n)
        f.restype, f.argtypes = r, a
    return L


class RefRules:
    def __init__(self, L, json_text: str | None = None):
        self.L = L
        if json_text is None:
            self.h = L.ref_rules_default()
        else:
            raw = json_text.encode()
            err = C.create_string_buffer(512)
            self.h = L.ref_rules_load(raw, len(raw), err, len(err))
            if not self.h:
                raise ValueError(err.value.decode())

    def mask(self, text: bytes) -> int:
        return int(self.L.ref_rules_mask(self.h, text, len(text)))

    def mask_wide(self, text: bytes, n_rules: int) -> int:
        """Per-rule hit bits of every rule of the list (bit i = rule i), any library size."""
        w = np.zeros((n_rules + 63) // 64, np.uint64)
        self.L.ref_rules_mask_wide(self.h, text, len(text), w.ctypes.data, len(w))
        return sum(int(x) << (64 * i) for i, x in enumerate(w))

    def verdict(self, text: bytes) -> tuple[bool, list[str]]:
        buf = C.create_string_buffer(4096)
        s = self.L.ref_rules_verdict(self.h, text, len(text), buf, len(buf))
        v = buf.value.decode()
        return bool(s), (v.split("\n") if v else [])


class RefEngine:
    """Appendix A pipeline on the reference RadixCacheIndex + EntropyMonitor."""

    def __init__(self, L, rules: RefRules, B=16, W=32, jump=0.3, u_pre_max=1, threads=1):
        self.L, self.B = L, B
        self.rules = rules
        self.h = L.ref_engine_create(rules.h, B, W, jump, u_pre_max)
        L.ref_engine_set_threads(self.h, threads)

    def close(self):
        if self.h:
            self.L.ref_engine_free(self.h)
            self.h = None

    def set_stock_scan(self, on: bool = True):
        """One stock CompiledRuleSet::scan per window: mask = the window's sensitive flag."""
        self.L.ref_engine_set_stock_scan(self.h, 1 if on else 0)

    def set_rules(self, rules: "RefRules"):
        """Reload between batches (RuleEngine::load_rules swap, detection.hpp:238-241)."""
        self.rules = rules
        self.L.ref_engine_set_rules(self.h, rules.h)

    def admit(self, tokens, offsets, users, owners=None):
        tokens = np.ascontiguousarray(tokens, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        users = np.ascontiguousarray(users, np.uint64)
        n = len(offsets) - 1
        owners = np.zeros(n, np.uint8) if owners is None else np.ascontiguousarray(owners, np.uint8)
        nb = int(((offsets[1:] - offsets[:-1]) // self.B).sum()) if n else 0
        o = {k: np.zeros(nb, t) for k, t in (("block_h", np.uint64), ("block_d", np.uint64),
                                             ("mask", np.uint64), ("label", np.uint8), ("decision", np.uint8))}
        o["matched_blocks"] = np.zeros(n, np.uint32)
        o["lowest_tier"] = np.zeros(n, np.uint8)
        rc = self.L.ref_engine_admit(self.h, _p(tokens), _p(offsets), _p(users), _p(owners), n, _p(o["block_h"]),
                                     _p(o["block_d"]), _p(o["mask"]), _p(o["label"]), _p(o["decision"]),
                                     _p(o["matched_blocks"]), _p(o["lowest_tier"]))
        assert rc == 0
        return o

    def commit(self):
        assert self.L.ref_engine_commit(self.h) == 0

    def set_pending(self, pending: bool):
        self.L.ref_engine_set_pending(self.h, 1 if pending else 0)

    def resolve(self, tokens, offsets, first_block, labels):
        tokens = np.ascontiguousarray(tokens, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        fb = np.ascontiguousarray(first_block, np.uint32)
        lab = np.ascontiguousarray(labels, np.uint8)
        assert self.L.ref_engine_resolve(self.h, _p(tokens), _p(offsets), len(offsets) - 1, _p(fb), _p(lab)) == 0

    def ttft(self, n, model, request_ids=None):
        """CostModel::ttft + attribute_reuse of the last admit (model: dict of skv_cost_model fields)."""
        out = np.zeros(n, np.float64)
        intra = np.zeros(n, np.uint32)
        inter = np.zeros(n, np.uint32)
        rid = None if request_ids is None else np.ascontiguousarray(request_ids, np.uint64)
        pen = model["tier_penalty_ms"]
        assert self.L.ref_engine_ttft(self.h, _p(rid), model["t_base_ms"], model["c_prefill_ms"], pen[1], pen[2],
                                      model["noise_sigma_ms"], model["seed"], _p(out), _p(intra), _p(inter)) == 0
        return out, intra, inter

    def set_tiers(self, tokens, offsets, tiers):
        tokens = np.ascontiguousarray(tokens, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        tiers = np.ascontiguousarray(tiers, np.uint8)
        assert self.L.ref_engine_set_tiers(self.h, _p(tokens), _p(offsets), len(offsets) - 1, _p(tiers)) == 0

    def set_tiered(self, tiered=True):
        assert self.L.ref_engine_set_tiered(self.h, 1 if tiered else 0) == 0

    def set_budget(self, hbm, dram=0, ssd=0, tiered=False):
        """A.9: TierBudget::from_tokens(hbm, dram, ssd) in blocks, before any insert."""
        assert self.L.ref_engine_set_budget(self.h, hbm, dram, ssd, 1 if tiered else 0) == 0

    def dropped(self):
        n = self.L.ref_engine_dropped(self.h, None, 0)
        out = np.zeros(max(n, 1), np.uint32)
        self.L.ref_engine_dropped(self.h, _p(out), n)
        return out[:n]

    def budget_used(self):
        out = np.zeros(3, np.uint64)
        self.L.ref_engine_budget_used(self.h, _p(out))
        return out

    def evict(self, needed):
        """RadixCacheIndex::evict(needed, current epoch); (rc, nodes freed)."""
        ep = self.L.ref_engine_current_epoch(self.h)
        n = C.c_uint64()
        rc = self.L.ref_engine_evict(self.h, needed, ep, C.byref(n))
        return rc, int(n.value)

    def epoch(self, cap=1 << 16):
        ep = C.c_uint64()
        n = C.c_size_t()
        h = np.zeros(cap, np.uint64)
        d = np.zeros(cap, np.uint64)
        act = np.zeros(cap, np.uint8)
        now = np.zeros(cap, np.float64)
        prev = np.zeros(cap, np.float64)
        upre = np.zeros(cap, np.uint64)
        assert self.L.ref_engine_epoch(self.h, C.byref(ep), cap, _p(h), _p(d), _p(act), _p(now), _p(prev), _p(upre),
                                       C.byref(n)) == 0
        k = min(n.value, cap)
        ev = sorted(zip(h[:k].tolist(), d[:k].tolist(), act[:k].tolist(), now[:k].tolist(), prev[:k].tolist(),
                        upre[:k].tolist()))
        return int(ep.value), ev

    def export(self):
        n = self.L.ref_engine_export(self.h, 0, *([None] * 10))
        cols = {k: np.zeros(n, t) for k, t in (("h", np.uint64), ("d", np.uint64), ("creator", np.uint64),
                                               ("label", np.uint8), ("owner", np.uint8), ("tier", np.uint8),
                                               ("hit_cur", np.uint64), ("u_cnt", np.uint64),
                                               ("hit_pre", np.uint64), ("u_pre", np.uint64))}
        self.L.ref_engine_export(self.h, n, *[_p(cols[k]) for k in ("h", "d", "creator", "label", "owner", "tier",
                                                                      "hit_cur", "u_cnt", "hit_pre", "u_pre")])
        order = np.lexsort((cols["d"], cols["h"]))
        return {k: v[order] for k, v in cols.items()}


def reference_workload(L, scenario, n_users, n_requests, inter, intra, density, ctx, seed):
    err = C.create_string_buffer(256)
    w = L.ref_workload_generate(scenario, n_users, n_requests, inter, intra, density, ctx, seed, err, len(err))
    if not w:
        raise ValueError(err.value.decode())
    n = L.ref_workload_count(w)
    texts, users, owners, truth = [], [], [], []
    for i in range(n):
        ln = L.ref_workload_text(w, i, None, 0)
        buf = C.create_string_buffer(ln)
        L.ref_workload_text(w, i, buf, ln)
        texts.append(buf.raw[:ln])
        users.append(L.ref_workload_user(w, i))
        owners.append(L.ref_workload_owner(w, i))
        k = L.ref_workload_truth(w, i, 0, None, None, None)
        b = np.zeros(k, np.uint64)
        e = np.zeros(k, np.uint64)
        s = np.zeros(k, np.uint8)
        L.ref_workload_truth(w, i, k, _p(b), _p(e), _p(s))
        truth.append(list(zip(b.tolist(), e.tolist(), s.tolist())))
    digest = L.ref_workload_digest(w)
    L.ref_workload_free(w)
    return texts, users, owners, truth, digest
