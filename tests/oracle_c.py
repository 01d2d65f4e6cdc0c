"""Test infrastructure: ctypes wrapper of the C restatement oracle/_ref/liboracle.so
(oracle/safekv_oracle.c).  Same interface as refh.RefEngine."""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from refh import ORC_SO, _p

# The shipped Tier-1 rule set (reference detection.hpp:185-204 ==
# configs/privacy_pattern_config.json): (rule_id, category, kind, pattern).
DEFAULT_RULES = [
    ("ssn_dashed", "Identity Information", "regex", r"\b\d{3}-\d{2}-\d{4}\b"),
    ("phone_us", "Basic Information", "regex", r"\(\d{3}\)\s?\d{3}-\d{4}|\b\d{3}-\d{3}-\d{4}\b"),
    ("email", "Basic Information", "regex", r"[A-Za-z0-9._%+-]+@[A-Za-z0-9.-]+\.[A-Za-z]{2,}"),
    ("ipv4", "System/Network Identification", "regex", r"\b\d{1,3}\.\d{1,3}\.\d{1,3}\.\d{1,3}\b"),
    ("credit_card", "Financial Info", "regex", r"\b\d{4}[- ]\d{4}[- ]\d{4}[- ]\d{4}\b"),
    ("bank_account", "Financial Info", "regex", r"\baccount\s+(?:no|number)\.?\s*\d{6,}\b"),
    ("mac_address", "Hardware Device Information", "regex", r"\b[0-9A-Fa-f]{2}(?::[0-9A-Fa-f]{2}){5}\b"),
    ("imei", "Hardware Device Information", "regex", r"\bimei\s*\d{15}\b"),
    ("blk_project_codes", "Service Content Info", "blacklist", "PROJECT-TITAN"),
]

_L = None


def lib():
    global _L
    if _L is None:
        L = C.CDLL(str(ORC_SO))
        vp, sz = C.c_void_p, C.c_size_t
        sig = {
            "orc_rules_create": (vp, [C.c_uint32, C.POINTER(C.c_char_p), vp, vp, vp, C.c_char_p, sz]),
            "orc_rules_free": (None, [vp]),
            "orc_rules_mask": (C.c_uint64, [vp, C.c_char_p, sz]),
            "orc_fnv1a64": (C.c_uint64, [vp, sz]),
            "orc_token_seq_digest": (C.c_uint64, [vp, sz]),
            "orc_chain": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "orc_engine_create": (vp, [vp, C.c_uint32, C.c_uint32, C.c_double, C.c_uint64]),
            "orc_engine_free": (None, [vp]),
            "orc_engine_admit": (C.c_int, [vp, vp, vp, vp, vp, C.c_uint32, vp, vp, vp, vp, vp, vp, vp]),
            "orc_engine_commit": (C.c_int, [vp]),
            "orc_engine_set_tiers": (C.c_int, [vp, vp, vp, C.c_uint32, vp]),
            "orc_engine_ttft": (C.c_int, [vp, vp, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                          C.c_uint64, vp, vp, vp]),
            "orc_engine_epoch": (C.c_int, [vp, C.POINTER(C.c_uint64), sz, vp, vp, vp, vp, vp, vp,
                                           C.POINTER(sz)]),
            "orc_engine_export": (sz, [vp, sz, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _L = L
    return _L


def rules_from_json(text: str | None):
    if text is None:
        return [(r, c, k, p, True) for (r, c, k, p) in DEFAULT_RULES]
    j = json.loads(text)
    return [(r["rule_id"], r.get("category", ""), r.get("kind", "regex"), r["pattern"], r.get("enabled", True))
            for r in j["rules"]]


class OracleRules:
    def __init__(self, rules_json: str | None = None, rules=None):
        L = lib()
        rules = rules if rules is not None else rules_from_json(rules_json)
        self.rules = rules
        n = len(rules)
        pats = [r[3].encode("latin-1") for r in rules]
        arr = (C.c_char_p * max(n, 1))(*pats)
        lens = np.array([len(p) for p in pats] or [0], np.uint32)
        kinds = np.array([1 if r[2] == "blacklist" else 0 for r in rules] or [0], np.uint8)
        en = np.array([1 if r[4] else 0 for r in rules] or [0], np.uint8)
        err = C.create_string_buffer(256)
        self.h = L.orc_rules_create(n, arr, _p(lens), _p(kinds), _p(en), err, len(err))
        if not self.h:
            raise ValueError(err.value.decode())
        self._keep = (pats, arr, lens, kinds, en)

    def mask(self, text: bytes) -> int:
        return int(lib().orc_rules_mask(self.h, text, len(text)))

    def close(self):
        if self.h:
            lib().orc_rules_free(self.h)
            self.h = None


class OracleEngine:
    def __init__(self, rules: OracleRules | None = None, B=16, W=32, jump=0.3, u_pre_max=1):
        self.B = B
        self.rules = rules or OracleRules()
        self.h = lib().orc_engine_create(self.rules.h, B, W, jump, u_pre_max)

    def close(self):
        if self.h:
            lib().orc_engine_free(self.h)
            self.h = None

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
        assert lib().orc_engine_admit(self.h, _p(tokens), _p(offsets), _p(users), _p(owners), n, _p(o["block_h"]),
                                      _p(o["block_d"]), _p(o["mask"]), _p(o["label"]), _p(o["decision"]),
                                      _p(o["matched_blocks"]), _p(o["lowest_tier"])) == 0
        return o

    def commit(self):
        assert lib().orc_engine_commit(self.h) == 0

    def ttft(self, n, model, request_ids=None):
        out = np.zeros(n, np.float64)
        intra = np.zeros(n, np.uint32)
        inter = np.zeros(n, np.uint32)
        rid = None if request_ids is None else np.ascontiguousarray(request_ids, np.uint64)
        pen = model["tier_penalty_ms"]
        assert lib().orc_engine_ttft(self.h, _p(rid), model["t_base_ms"], model["c_prefill_ms"], pen[1], pen[2],
                                     model["noise_sigma_ms"], model["seed"], _p(out), _p(intra), _p(inter)) == 0
        return out, intra, inter

    def set_tiers(self, tokens, offsets, tiers):
        tokens = np.ascontiguousarray(tokens, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        tiers = np.ascontiguousarray(tiers, np.uint8)
        assert lib().orc_engine_set_tiers(self.h, _p(tokens), _p(offsets), len(offsets) - 1, _p(tiers)) == 0

    def epoch(self, cap=1 << 16):
        ep = C.c_uint64()
        n = C.c_size_t()
        h = np.zeros(cap, np.uint64)
        d = np.zeros(cap, np.uint64)
        act = np.zeros(cap, np.uint8)
        now = np.zeros(cap, np.float64)
        prev = np.zeros(cap, np.float64)
        upre = np.zeros(cap, np.uint64)
        assert lib().orc_engine_epoch(self.h, C.byref(ep), cap, _p(h), _p(d), _p(act), _p(now), _p(prev), _p(upre),
                                      C.byref(n)) == 0
        k = min(n.value, cap)
        ev = sorted(zip(h[:k].tolist(), d[:k].tolist(), act[:k].tolist(), now[:k].tolist(), prev[:k].tolist(),
                        upre[:k].tolist()))
        return int(ep.value), ev

    def export(self):
        L = lib()
        n = L.orc_engine_export(self.h, 0, *([None] * 10))
        cols = {k: np.zeros(n, t) for k, t in (("h", np.uint64), ("d", np.uint64), ("creator", np.uint64),
                                               ("label", np.uint8), ("owner", np.uint8), ("tier", np.uint8),
                                               ("hit_cur", np.uint64), ("u_cnt", np.uint64),
                                               ("hit_pre", np.uint64), ("u_pre", np.uint64))}
        L.orc_engine_export(self.h, n, *[_p(cols[k]) for k in ("h", "d", "creator", "label", "owner", "tier",
                                                                 "hit_cur", "u_cnt", "hit_pre", "u_pre")])
        order = np.lexsort((cols["d"], cols["h"]))
        return {k: v[order] for k, v in cols.items()}
