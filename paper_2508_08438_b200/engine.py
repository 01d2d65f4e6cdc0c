"""Host-side mirror of the reference interface for the admission path.

Python names follow the reference C++ API (``safekv::RuleEngine::tier1_scan``,
``RadixCacheIndex::match_prefix``, ``EntropyMonitor::epoch_pass`` ...), but every call
goes through the C ABI into the CUDA library; nothing is computed here beyond argument
marshalling.  The batch entry points implement the parity contract of SURVEY.md
Appendix A (phases L / C / E).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import native as N


def _ptr(a: Optional[np.ndarray]) -> Optional[int]:
    return None if a is None else a.ctypes.data


class RuleSet:
    """Immutable compiled rule snapshot (reference ``CompiledRuleSet``, detection.hpp:118-181)."""

    def __init__(self, handle: int):
        self._lib = N.load_library()
        self._h = C.c_void_p(handle)

    @classmethod
    def default(cls) -> "RuleSet":
        lib = N.load_library()
        h = C.c_void_p()
        N.raise_for(lib.skv_rules_default(C.byref(h)), "default rules")
        return cls(h.value)

    @classmethod
    def from_json(cls, text: str | bytes) -> "RuleSet":
        """``RuleEngine::load_rules_json`` (detection.hpp:222-242): ParseError / CompileError."""
        lib = N.load_library()
        raw = text.encode() if isinstance(text, str) else text
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = lib.skv_rules_from_json(raw, len(raw), C.byref(h), err, len(err))
        N.raise_for(rc, err.value.decode(errors="replace"))
        return cls(h.value)

    def __del__(self):
        try:
            if self._h:
                self._lib.skv_rules_free(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @property
    def version(self) -> int:
        return int(self._lib.skv_rules_version(self._h))

    def size(self) -> int:
        return int(self._lib.skv_rules_count(self._h))

    def rules(self) -> list[dict]:
        out = []
        for i in range(self.size()):
            rid, cat = C.c_char_p(), C.c_char_p()
            kind, en = C.c_int(), C.c_int()
            N.raise_for(self._lib.skv_rules_info(self._h, i, C.byref(rid), C.byref(cat), C.byref(kind),
                                                 C.byref(en)), "rules_info")
            out.append({"rule_id": rid.value.decode(), "category": cat.value.decode(),
                        "kind": "blacklist" if kind.value else "regex", "enabled": bool(en.value)})
        return out

    def warnings(self) -> list[str]:
        n = self._lib.skv_rules_warning_count(self._h)
        return [self._lib.skv_rules_warning(self._h, i).decode() for i in range(n)]

    def group_count(self) -> int:
        """Device automata the rule set runs as (one scan pass each)."""
        return int(self._lib.skv_rules_group_count(self._h))

    def enabled_rules(self) -> list[int]:
        n = self._lib.skv_rules_enabled_count(self._h)
        return [int(self._lib.skv_rules_enabled_rule(self._h, j)) for j in range(n)]

    def mask_words(self) -> int:
        """u32 words of a window's device mask (bit j = j-th enabled rule; > 32 enabled rules
        take more than one word)."""
        return int(self._lib.skv_rules_mask_words(self._h))

    def to_rule_mask(self, device_mask: int) -> int:
        """Device mask (bit j = j-th enabled rule) -> mask over rule-list positions."""
        m = 0
        for j, r in enumerate(self.enabled_rules()):
            if device_mask >> j & 1:
                m |= 1 << r
        return m

    def to_rule_mask_array(self, device_masks: np.ndarray) -> np.ndarray:
        out = np.zeros(len(device_masks), np.uint64)
        dm = np.asarray(device_masks).astype(np.uint64)
        for j, r in enumerate(self.enabled_rules()):
            out |= ((dm >> np.uint64(j)) & np.uint64(1)) << np.uint64(r)
        return out

    def categories(self, device_mask: int) -> list[str]:
        """Ordered, de-duplicated categories exactly as ``CompiledRuleSet::scan`` lists them
        (rule order of the hit rules, detection.hpp:160-166)."""
        rules = self.rules()
        rm = self.to_rule_mask(device_mask)
        cats: list[str] = []
        for i, r in enumerate(rules):
            if rm >> i & 1 and r["category"] not in cats:
                cats.append(r["category"])
        return cats

    def dfa(self) -> dict:
        v = N.DfaView()
        N.raise_for(self._lib.skv_rules_dfa(self._h, C.byref(v)), "dfa")
        S, Cn = v.n_states, v.n_classes
        return {
            "n_states": S, "n_classes": Cn, "start": v.start,
            "class_map": np.ctypeslib.as_array(v.class_map, shape=(256,)).copy(),
            "next": np.ctypeslib.as_array(v.next, shape=(S * Cn,)).reshape(S, Cn).copy(),
            "acc": np.ctypeslib.as_array(v.acc, shape=(S * (Cn + 1),)).reshape(S, Cn + 1).copy(),
            "nfa_states": v.nfa_states, "dfa_states_unminimized": v.dfa_states_unminimized,
        }


@dataclass
class AdmitResult:
    block_offsets: np.ndarray   # n_prompts + 1 (uint32)
    block_h: np.ndarray         # uint64 per block
    block_d: np.ndarray
    label: np.ndarray           # uint8 per block (0 Private, 1 Public)
    rule_mask: np.ndarray       # uint32 per block (bit j = j-th enabled rule; word 0 of the mask)
    decision: np.ndarray        # uint8 per block (0 miss, 1 public hit, 2 owner hit)
    matched_blocks: np.ndarray  # uint32 per prompt
    lowest_tier: np.ndarray     # uint8 per prompt
    n_blocks: int = 0
    matched_total: int = 0
    rule_mask_words: Optional[np.ndarray] = None  # [words, n_blocks] when > 32 rules are enabled


@dataclass
class AnomalyEvent:
    h: int
    d: int
    action: int
    owner: int
    entropy_now: float
    entropy_prev: float
    u_pre: int
    epoch: int


@dataclass
class EngineConfig:
    block_tokens: int = 16
    window_tokens: int = 32
    index_capacity: int = 1 << 20
    max_prompts: int = 1 << 16
    max_tokens: int = 1 << 24
    max_window_entries: int = 1 << 16
    entropy_jump: float = 0.3
    u_pre_max: int = 1
    max_users: int = 1 << 20
    device: int = 0


class AdmissionEngine:
    """Device-resident SafeKV admission context (index + monitor + rule DFA)."""

    def __init__(self, cfg: EngineConfig | None = None, **kw):
        self.cfg = cfg or EngineConfig(**kw)
        self._lib = N.load_library()
        c = N.Config()
        self._lib.skv_config_default(C.byref(c))
        for f, _ in N.Config._fields_:
            setattr(c, f, getattr(self.cfg, f))
        h = C.c_void_p()
        rc = self._lib.skv_create(C.byref(c), C.byref(h))
        if rc != N.SKV_OK:
            N.raise_for(rc, self._lib.skv_last_error(None).decode())
        self._h = h
        self.rules = RuleSet.default()

    def close(self):
        if getattr(self, "_h", None):
            self._lib.skv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _err(self) -> str:
        return self._lib.skv_last_error(self._h).decode(errors="replace")

    def _check(self, rc: int):
        N.raise_for(rc, self._err())

    @property
    def stream(self) -> int:
        return int(self._lib.skv_stream(self._h) or 0)

    def set_rules(self, rs: RuleSet):
        self._check(self._lib.skv_set_rules(self._h, rs.handle))
        self.rules = rs

    # --------------------------------------------------------------- phase L
    def admit(self, tokens: np.ndarray, offsets: np.ndarray, users: np.ndarray,
              owners: Optional[np.ndarray] = None) -> AdmitResult:
        """Phase L of one batch.  ``tokens`` as uint32 TokenIds, or as uint8 byte tokens (the
        reference's ByteVocabulary: a quarter of the host->device copy, skv_batch::token_bytes)."""
        as_bytes = isinstance(tokens, (bytes, bytearray)) or np.asarray(tokens).dtype == np.uint8
        tokens = np.ascontiguousarray(np.frombuffer(tokens, np.uint8) if isinstance(tokens, (bytes, bytearray))
                                      else tokens, dtype=np.uint8 if as_bytes else np.uint32)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        users = np.ascontiguousarray(users, dtype=np.uint64)
        if owners is not None:
            owners = np.ascontiguousarray(owners, dtype=np.uint8)
        n = len(offsets) - 1
        B = self.cfg.block_tokens
        nb = int(((offsets[1:] - offsets[:-1]) // B).sum()) if n > 0 else 0
        res = AdmitResult(
            block_offsets=np.zeros(n + 1, np.uint32), block_h=np.zeros(nb, np.uint64),
            block_d=np.zeros(nb, np.uint64), label=np.zeros(nb, np.uint8), rule_mask=np.zeros(nb, np.uint32),
            decision=np.zeros(nb, np.uint8), matched_blocks=np.zeros(n, np.uint32),
            lowest_tier=np.zeros(n, np.uint8))
        b = N.Batch(None if as_bytes else _ptr(tokens), _ptr(offsets), _ptr(users), _ptr(owners), n, len(tokens), 0,
                    _ptr(tokens) if as_bytes else None)
        o = N.AdmitOut(_ptr(res.block_h), _ptr(res.block_d), _ptr(res.label), _ptr(res.rule_mask),
                       _ptr(res.decision), _ptr(res.matched_blocks), _ptr(res.lowest_tier),
                       _ptr(res.block_offsets), 0, 0, 0)
        self._check(self._lib.skv_admit(self._h, C.byref(b), C.byref(o)))
        res.n_blocks, res.matched_total = int(o.n_blocks), int(o.matched_total)
        self._last_blocks = res.n_blocks
        if int(self._lib.skv_mask_words(self._h)) > 1:  # a rule library of more than 32 enabled rules
            res.rule_mask_words = self.last_rule_masks()
        return res

    def access_entropy(self, cap: int = 1 << 22) -> dict:
        """Diagnostic (``skv_access_entropy``; no reference counterpart): for every entry the last
        admitted batch matched, its accesses, distinct users and the Shannon entropy (bits) of the
        batch's accesses over users.  The monitor's leak flags use the reference predicate."""
        out = {k: np.zeros(cap, t) for k, t in (("h", np.uint64), ("d", np.uint64), ("accesses", np.uint64),
                                                ("users", np.uint64), ("bits", np.float64))}
        n = C.c_size_t()
        self._check(self._lib.skv_access_entropy(self._h, _ptr(out["h"]), _ptr(out["d"]), _ptr(out["accesses"]),
                                                 _ptr(out["users"]), _ptr(out["bits"]), cap, C.byref(n)))
        k = min(int(n.value), cap)
        return {key: v[:k] for key, v in out.items()}

    def set_graphs(self, on: bool) -> None:
        """CUDA-graph replay of small device-batch steps (``skv_set_graphs``; default on)."""
        self._check(self._lib.skv_set_graphs(self._h, 1 if on else 0))

    def admit_raw(self, batch: N.Batch, out: Optional[N.AdmitOut] = None) -> None:
        """Zero-copy entry point: device (or host) pointers supplied by the caller."""
        self._check(self._lib.skv_admit(self._h, C.byref(batch), C.byref(out) if out is not None else None))

    def prefetch(self, tokens: np.ndarray, offsets: np.ndarray, users: np.ndarray,
                 owners: Optional[np.ndarray] = None) -> None:
        """Cross-batch pipelining (skv_prefetch): start the H2D copy and stages 1-2 of the
        NEXT host batch on the engine's side stream; call between ``admit`` and ``commit``
        of the current batch.  The following ``admit`` of the same arrays consumes it.
        Arrays should already be contiguous with the ABI dtypes (uint32/uint64/uint64/uint8),
        ideally pinned, so that ``admit`` sees the same buffers."""
        arrs = (np.ascontiguousarray(tokens, dtype=np.uint32), np.ascontiguousarray(offsets, dtype=np.uint64),
                np.ascontiguousarray(users, dtype=np.uint64),
                None if owners is None else np.ascontiguousarray(owners, dtype=np.uint8))
        self._pf_keep = arrs  # the async copy reads these until the next admit
        b = N.Batch(_ptr(arrs[0]), _ptr(arrs[1]), _ptr(arrs[2]), _ptr(arrs[3]), len(arrs[1]) - 1, len(arrs[0]), 0)
        self._check(self._lib.skv_prefetch(self._h, C.byref(b)))

    def stage_raw(self, batch: N.Batch) -> None:
        """skv_stage: queue the host->device copy of a host batch ahead of its prefetch / admit."""
        self._check(self._lib.skv_stage(self._h, C.byref(batch)))

    def prefetch_raw(self, batch: N.Batch) -> None:
        """skv_prefetch with caller-owned (device or host) pointers."""
        self._check(self._lib.skv_prefetch(self._h, C.byref(batch)))

    # --------------------------------------------------------------- phase C

    def commit(self) -> int:
        n = C.c_uint64()
        self._check(self._lib.skv_commit(self._h, C.byref(n)))
        return int(n.value)

    # --------------------------------------------------------------- phase E
    def epoch_pass(self, cap: int = 1 << 16) -> tuple[int, list[AnomalyEvent]]:
        """advance_epoch + ``EntropyMonitor::epoch_pass`` (monitor.hpp:85-99): returns the
        epoch number and the fired events sorted by entry key."""
        buf = getattr(self, "_evbuf", None)
        if buf is None or len(buf) < cap:  # one event buffer per engine (no per-call 3 MB allocation)
            buf = self._evbuf = (N.Event * cap)()
        n = C.c_size_t()
        ep = C.c_uint64()
        self._check(self._lib.skv_epoch(self._h, buf, cap, C.byref(n), C.byref(ep)))
        if n.value > cap:  # the epoch is applied; fetch the whole list (skv_last_events)
            buf = self._evbuf = (N.Event * n.value)()
            self._check(self._lib.skv_last_events(self._h, buf, n.value, C.byref(n)))
        evs = [AnomalyEvent(e.h, e.d, e.action, e.owner, e.entropy_now, e.entropy_prev, e.u_pre, e.epoch)
               for e in buf[:n.value]]
        return int(ep.value), evs

    def step_raw(self, batch: N.Batch, out: Optional[N.AdmitOut] = None, next_batch: Optional[N.Batch] = None,
                 stage: Optional[N.Batch] = None, cap: int = 1 << 16) -> tuple[int, int, list[AnomalyEvent]]:
        """``skv_step``: admit (+ ``out``) -> prefetch ``next_batch`` -> commit -> stage ``stage`` ->
        epoch, one host synchronisation in the common case.  Returns (new entries, epoch, events)."""
        buf = getattr(self, "_evbuf", None)
        if buf is None or len(buf) < cap:
            buf = self._evbuf = (N.Event * cap)()
        sc = getattr(self, "_step_scalars", None)
        if sc is None:  # per-engine result scalars (a serving loop calls this once per batch)
            sc = self._step_scalars = (C.c_size_t(), C.c_uint64(), C.c_uint64())
        n, ep, nn = sc
        self._check(self._lib.skv_step(self._h, C.byref(batch), None if out is None else C.byref(out),
                                       None if next_batch is None else C.byref(next_batch),
                                       None if stage is None else C.byref(stage), C.byref(nn), buf, cap, C.byref(n),
                                       C.byref(ep)))
        if n.value > cap:
            buf = self._evbuf = (N.Event * n.value)()
            self._check(self._lib.skv_last_events(self._h, buf, n.value, C.byref(n)))
        evs = [AnomalyEvent(e.h, e.d, e.action, e.owner, e.entropy_now, e.entropy_prev, e.u_pre, e.epoch)
               for e in buf[:n.value]]
        return int(nn.value), int(ep.value), evs

    # --------------------------------------------------------------- misc
    # --------------------------------------------------------------- serving observables

    def set_cost_model(self, t_base_ms: float = 10.0, c_prefill_ms: float = 1.0,
                       tier_penalty_ms: Sequence[float] = (0.0, 0.2, 0.5), noise_sigma_ms: float = 0.0,
                       seed: int = 0) -> None:
        """``CostModel`` (serving_sim.hpp:25-57); raises ConfigError like CostModel::validate."""
        m = N.CostModel(t_base_ms, c_prefill_ms, (C.c_double * 3)(*tier_penalty_ms), noise_sigma_ms, seed)
        self._check(self._lib.skv_set_cost_model(self._h, C.byref(m)))

    def ttft(self, n_prompts: int, request_ids: Optional[np.ndarray] = None):
        """Per prompt of the last admit: (ttft_ms, intra_tokens, inter_tokens) --
        CostModel::ttft (serving_sim.hpp:50-56) and attribute_reuse (:313-324)."""
        out = np.zeros(n_prompts, np.float64)
        intra = np.zeros(n_prompts, np.uint32)
        inter = np.zeros(n_prompts, np.uint32)
        rid = None if request_ids is None else np.ascontiguousarray(request_ids, np.uint64)
        self._check(self._lib.skv_admit_ttft(self._h, _ptr(rid), _ptr(out), _ptr(intra), _ptr(inter), 0))
        return out, intra, inter

    def set_label_policy(self, pending: bool) -> None:
        """New entries start PendingPrivate until their labels are landed (resolve_blocks)."""
        self._check(self._lib.skv_set_label_policy(self._h, 1 if pending else 0))

    def resolve_blocks(self, h: np.ndarray, d: np.ndarray, block_offsets: np.ndarray, first_block: np.ndarray,
                       labels: np.ndarray) -> None:
        """``RadixCacheIndex::resolve_block`` (cache_index.hpp:321-343) of each prompt's
        classification span [first_block, n) with its label (Public: no propagation;
        Private/Restricted: span top + descendants)."""
        h = np.ascontiguousarray(h, np.uint64)
        d = np.ascontiguousarray(d, np.uint64)
        bo = np.ascontiguousarray(block_offsets, np.uint32)
        fb = np.ascontiguousarray(first_block, np.uint32)
        lab = np.ascontiguousarray(labels, np.uint8)
        self._check(self._lib.skv_resolve_blocks(self._h, _ptr(h), _ptr(d), _ptr(bo), len(bo) - 1, _ptr(fb),
                                                 _ptr(lab)))

    def set_tiers(self, h: np.ndarray, d: np.ndarray, tiers: np.ndarray, block_offsets: np.ndarray):
        """Tier tags (demote semantics) of the blocks of whole prompts, prompt-major as
        ``admit`` returns them (``AdmitResult.block_offsets``)."""
        h = np.ascontiguousarray(h, np.uint64)
        d = np.ascontiguousarray(d, np.uint64)
        tiers = np.ascontiguousarray(tiers, np.uint8)
        bo = np.ascontiguousarray(block_offsets, np.uint32)
        self._check(self._lib.skv_set_tiers(self._h, _ptr(h), _ptr(d), _ptr(bo), len(bo) - 1, _ptr(tiers)))

    def export(self) -> np.ndarray:
        cnt = int(self._lib.skv_entry_count(self._h))
        cap = max(cnt, 1)
        buf = (N.Entry * cap)()
        n = C.c_size_t()
        self._check(self._lib.skv_export(self._h, buf, cap, C.byref(n)))
        dt = np.dtype([("h", "<u8"), ("d", "<u8"), ("creator", "<u8"), ("label", "u1"), ("owner", "u1"),
                       ("tier", "u1"), ("hit_cur", "<u8"), ("u_cnt", "<u8"), ("hit_pre", "<u8"),
                       ("u_pre", "<u8")], align=True)
        assert dt.itemsize == C.sizeof(N.Entry)
        arr = np.frombuffer(bytes(buf), dtype=dt, count=min(n.value, cap)).copy()
        arr.sort(order=["h", "d"])
        return arr

    def enable_eviction(self, tiered_demotion: bool = False) -> None:
        """Per-entry access epochs and node ids for ``evict`` (before the first admit);
        with ``tiered_demotion`` victims move HBM -> DRAM instead of leaving."""
        self._check(self._lib.skv_enable_eviction(self._h, 1 if tiered_demotion else 0))

    def set_tier_budget(self, hbm_blocks: int, dram_blocks: int = 0, ssd_blocks: int = 0) -> None:
        """TierBudget (cache_index.hpp:26-55) in blocks with insert-time make_room (A.9):
        every commit inserts its prompts in order, each first evicting unpinned leaves until its
        new blocks fit (needs ``enable_eviction()``, before the first admit)."""
        self._check(self._lib.skv_set_tier_budget(self._h, hbm_blocks, dram_blocks, ssd_blocks))

    def tier_usage(self):
        """(used, capacity) blocks per tier (HBM, DRAM, SSD)."""
        u = np.zeros(3, np.uint64)
        c = np.zeros(3, np.uint64)
        self._check(self._lib.skv_tier_usage(self._h, _ptr(u), _ptr(c)))
        return u, c

    def last_drops(self) -> np.ndarray:
        """Prompts of the last commit whose insert could not make room (CapacityExhausted)."""
        n = C.c_size_t()
        self._check(self._lib.skv_last_drops(self._h, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), np.uint32)
        self._check(self._lib.skv_last_drops(self._h, _ptr(out), n.value, C.byref(n)))
        return out[:n.value]

    def evict(self, needed_blocks: int, epoch: int = 0):
        """RadixCacheIndex::evict (cache_index.hpp:281-292): frees ``needed_blocks`` entries
        in the reference's victim order; returns (n_evicted, victim h, victim d).  Raises
        CapacityExhausted (after freeing every candidate) when fewer could be freed."""
        n = C.c_uint64()
        cap = max(int(needed_blocks), 1)
        vh = np.zeros(cap, np.uint64)
        vd = np.zeros(cap, np.uint64)
        rc = self._lib.skv_evict(self._h, needed_blocks, epoch, C.byref(n), _ptr(vh), _ptr(vd), cap)
        self._evicted = (int(n.value), vh[:n.value], vd[:n.value])
        self._check(rc)
        return self._evicted

    # --------------------------------------------------------------- replicated layer (multi-GPU)
    def set_replicated_depth(self, depth: int) -> None:
        """Entries at depth < ``depth`` are replicated on every rank (before the first admit);
        see ReplicaGroup."""
        self._check(self._lib.skv_set_replicated_depth(self._h, depth))

    def replica_export(self, prompt_gids: np.ndarray, device: bool = False):
        """After ``commit``: (new replicated-layer entries as a REP_ENTRY array, the batch's
        replicated-layer accesses aggregated per (entry, user) as a REP_ACCESS array -- or, with
        ``device``, as a uint8 torch tensor in device memory); ``prompt_gids`` = global ids of the
        batch's prompts."""
        gids = np.ascontiguousarray(prompt_gids, np.uint64)
        ne, na = C.c_size_t(), C.c_size_t()
        ecap, acap = 1 << 12, 1 << 14
        while True:
            ents = np.zeros(ecap, REP_ENTRY)
            if device:
                import torch
                accs = torch.empty(acap * REP_ACCESS.itemsize, dtype=torch.uint8,
                                   device=torch.device("cuda", self.cfg.device))
                aptr = accs.data_ptr()
            else:
                accs = np.zeros(acap, REP_ACCESS)
                aptr = _ptr(accs)
            rc = self._lib.skv_replica_export(self._h, _ptr(gids), _ptr(ents), ecap, C.byref(ne), aptr, acap,
                                              C.byref(na), 1 if device else 0)
            if rc == N.SKV_ERR_CAPACITY and (ne.value > ecap or na.value > acap):
                ecap, acap = max(ecap, ne.value), max(acap, na.value)
                continue
            self._check(rc)
            return ents[:ne.value], accs[:na.value * (REP_ACCESS.itemsize if device else 1)]

    def replica_apply(self, ents: np.ndarray, accs) -> None:
        """Apply every rank's export: ``ents`` merged (``merge_replica``), ``accs`` the ranks'
        access exports concatenated (a REP_ACCESS array, or a uint8 torch tensor in device
        memory); the accesses are merged on the device."""
        ents = np.ascontiguousarray(ents, REP_ENTRY)
        if isinstance(accs, np.ndarray):
            accs = np.ascontiguousarray(accs, REP_ACCESS)
            rc = self._lib.skv_replica_apply(self._h, _ptr(ents), len(ents), _ptr(accs), len(accs), 0)
        else:  # a device tensor of raw REP_ACCESS records
            n = accs.numel() // REP_ACCESS.itemsize
            rc = self._lib.skv_replica_apply(self._h, _ptr(ents), len(ents), accs.data_ptr() if n else None, n, 1)
        self._check(rc)

    def leak_flags(self, span_off: np.ndarray, span_begin: np.ndarray, span_end: np.ndarray):
        """SURVEY A.8 leak flags of the last admit: (per-block flags, count).  Spans: the planted
        spans that are sensitive on their own, per prompt [span_off[p], span_off[p+1])."""
        so = np.ascontiguousarray(span_off, np.uint32)
        sb = np.ascontiguousarray(span_begin, np.uint64)
        se = np.ascontiguousarray(span_end, np.uint64)
        nb = getattr(self, "_last_blocks", None)
        flags = np.zeros(max(int(nb or 0), 1), np.uint8)
        n = C.c_uint64()
        self._check(self._lib.skv_leak_flags(self._h, _ptr(so), _ptr(sb), _ptr(se), _ptr(flags), C.byref(n)))
        return flags[:int(nb or 0)], int(n.value)

    def entry_count(self) -> int:
        return int(self._lib.skv_entry_count(self._h))

    def times(self) -> dict:
        return self.times_dict(self.times_raw())

    def times_raw(self) -> "N.StageTimes":
        """``skv_last_times`` as the raw struct (one ctypes call; ``times_dict`` converts)."""
        t = N.StageTimes()
        self._check(self._lib.skv_last_times(self._h, C.byref(t)))
        return t

    @staticmethod
    def times_dict(t: "N.StageTimes") -> dict:
        return {f: getattr(t, f) for f, _ in N.StageTimes._fields_}

    def tier1_scan(self, text: str | bytes) -> int:
        """``RuleEngine::tier1_scan`` (detection.hpp:217) as a batch of one on the device.
        Returns the device rule mask; ``self.rules.categories(mask)`` gives the verdict's
        category list and ``mask != 0`` its ``sensitive`` flag."""
        raw = text.encode("latin-1") if isinstance(text, str) else bytes(text)
        m = np.zeros(max(1, int(self._lib.skv_mask_words(self._h))), np.uint32)
        self._check(self._lib.skv_tier1_scan(self._h, raw, len(raw), _ptr(m)))
        return combine_mask_words(m[:, None])[0]

    def last_rule_masks(self, n_blocks: Optional[int] = None) -> np.ndarray:
        """The last admitted batch's full window masks, ``[mask words, n_blocks]`` uint32
        (word 0 is ``AdmitResult.rule_mask``); ``combine_mask_words`` gives one int per block.
        ``n_blocks``: the batch's block count (default: that of the last ``admit``)."""
        w = int(self._lib.skv_mask_words(self._h))
        nb = getattr(self, "_last_blocks", 0) if n_blocks is None else int(n_blocks)
        out = np.zeros((w, nb), np.uint32)
        self._check(self._lib.skv_last_rule_masks(self._h, _ptr(out), 0))
        return out

    def token_seq_digest(self, tokens: Sequence[int]) -> int:
        """``safekv::token_seq_digest`` (core.hpp:68-73) on the device."""
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.uint32))
        d = C.c_uint64()
        self._check(self._lib.skv_token_seq_digest(self._h, _ptr(t), len(t), C.byref(d)))
        return int(d.value)


def combine_mask_words(words: np.ndarray) -> list[int]:
    """``[mask words, n]`` uint32 device masks -> one Python int per window (bit j = j-th
    enabled rule, any number of words)."""
    words = np.asarray(words, np.uint32)
    out = [0] * words.shape[1]
    for w in range(words.shape[0]):
        nz = np.nonzero(words[w])[0]
        for i in nz:
            out[i] |= int(words[w, i]) << (32 * w)
    return out


# skv_rep_entry / skv_rep_access (include/safekv_b200.h)
REP_ENTRY = np.dtype([("h", "<u8"), ("d", "<u8"), ("ph", "<u8"), ("pd", "<u8"), ("creator", "<u8"), ("gid", "<u8"),
                      ("label", "u1"), ("owner", "u1"), ("pad", "u1", (6,))])
REP_ACCESS = np.dtype([("h", "<u8"), ("d", "<u8"), ("user", "<u8"), ("gid", "<u8"), ("count", "<u8")])
assert REP_ENTRY.itemsize == 56 and REP_ACCESS.itemsize == 40


def merge_replica(ents_list, accs_list):
    """The merge every rank applies (host, identical everywhere): of all ranks' new
    replicated-layer entries, the one per key with the lowest global prompt id (first creator
    wins, cache_index.hpp:164-168); of all accesses, per (key, user) the lowest first prompt id
    and the summed count, sorted by key then first prompt id (the global access order the
    entry's AccessStats replays)."""
    E = np.concatenate([np.asarray(e, REP_ENTRY) for e in ents_list]) if ents_list else np.zeros(0, REP_ENTRY)
    if len(E):
        E = E[np.lexsort((E["gid"], E["d"], E["h"]))]
        keep = np.ones(len(E), bool)
        keep[1:] = (E["h"][1:] != E["h"][:-1]) | (E["d"][1:] != E["d"][:-1])
        E = E[keep]
    A = np.concatenate([np.asarray(a, REP_ACCESS) for a in accs_list]) if accs_list else np.zeros(0, REP_ACCESS)
    if len(A):
        A = A[np.lexsort((A["gid"], A["user"], A["d"], A["h"]))]
        head = np.ones(len(A), bool)
        head[1:] = (A["h"][1:] != A["h"][:-1]) | (A["d"][1:] != A["d"][:-1]) | (A["user"][1:] != A["user"][:-1])
        starts = np.flatnonzero(head)
        counts = np.add.reduceat(A["count"], starts)
        A = A[starts].copy()  # the first row of a (key, user) group carries its lowest gid
        A["count"] = counts
        A = A[np.lexsort((A["gid"], A["d"], A["h"]))]
    return E, A


def merge_entries(ents_list):
    """The first-creator merge of all ranks' new replicated-layer entries: one per key, the
    lowest global prompt id (cache_index.hpp:164-168)."""
    return merge_replica(ents_list, [])[0]


def torch_allgather(group=None):
    """An allgather of numpy records over torch.distributed (NCCL: device tensors over NVLink;
    gloo: host tensors): returns every rank's array, in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")

    def ag(arr: np.ndarray):
        raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
        n = torch.tensor([raw.size], dtype=torch.int64, device=dev)
        sizes = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(sizes, n, group=group)
        sizes = [int(x.item()) for x in sizes]
        mx = max(max(sizes), 1)
        buf = torch.zeros(mx, dtype=torch.uint8, device=dev)
        if raw.size:
            buf[:raw.size] = torch.from_numpy(raw.copy()).to(dev)
        outs = [torch.empty(mx, dtype=torch.uint8, device=dev) for _ in range(world)]
        dist.all_gather(outs, buf, group=group)
        return [o[:sz].cpu().numpy().view(arr.dtype) for o, sz in zip(outs, sizes)]
    return ag


def torch_allgather_device(group=None):
    """NCCL allgather of a uint8 device tensor of records: every rank's records concatenated, in
    rank order, staying in device memory (NVLink; no host round trip of the data)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)

    def ag(t):
        n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
        sizes = torch.empty(world, dtype=torch.int64, device=t.device)
        dist.all_gather_into_tensor(sizes, n, group=group)
        sizes = sizes.tolist()
        mx = max(max(sizes), 1)
        buf = torch.zeros(mx, dtype=torch.uint8, device=t.device)
        buf[:t.numel()] = t
        out = torch.empty(world * mx, dtype=torch.uint8, device=t.device)
        dist.all_gather_into_tensor(out, buf, group=group)
        return torch.cat([out[i * mx:i * mx + sz] for i, sz in enumerate(sizes)])
    return ag


class ReplicaGroup:
    """Cross-rank merge of the replicated layer (north star: "each GPU holds a replica of the
    index, and new-entry inserts and entropy counters are merged across GPUs with NCCL").
    Per batch: ``engine.commit()`` then ``sync(prompt_gids)``; every rank applies the same merge,
    so replicated entries and their window statistics are identical on all ranks and equal one
    engine's over the whole batch.  With ``allgather_device`` (NCCL) the access records stay
    in device memory from the export through the all-gather to the device-side merge."""

    def __init__(self, engine: "AdmissionEngine", depth: int, allgather, allgather_device=None):
        self.engine, self.depth = engine, depth
        self.allgather, self.allgather_device = allgather, allgather_device
        engine.set_replicated_depth(depth)

    def sync(self, prompt_gids: np.ndarray):
        if self.allgather_device is not None:
            e, a = self.engine.replica_export(prompt_gids, device=True)
            E = merge_entries(self.allgather(e))
            A = self.allgather_device(a)
            self.engine.replica_apply(E, A)
            return len(E), A.numel() // REP_ACCESS.itemsize
        e, a = self.engine.replica_export(prompt_gids)
        E = merge_entries(self.allgather(e))
        A = self.allgather(a)
        A = np.concatenate(A) if A else np.zeros(0, REP_ACCESS)
        self.engine.replica_apply(E, A)
        return len(E), len(A)


def merge_events(events_per_rank):
    """Union of the ranks' epoch events (a replicated entry fires identically on every rank),
    sorted by key."""
    seen, out = set(), []
    for evs in events_per_rank:
        for e in evs:
            if (e.h, e.d) not in seen:
                seen.add((e.h, e.d))
                out.append(e)
    return sorted(out, key=lambda e: (e.h, e.d))


def route(tokens: np.ndarray, offsets: np.ndarray, world: int, block_tokens: int,
          prompt_ids: Optional[np.ndarray] = None, depth: int = 0) -> np.ndarray:
    """skv_route_depth: owning rank of every prompt (host).  Entries at depth < ``depth`` are
    replicated; deeper ones belong to the rank of their depth-``depth`` ancestor's key."""
    lib = N.load_library()
    tokens = np.ascontiguousarray(tokens, np.uint32)
    offsets = np.ascontiguousarray(offsets, np.uint64)
    n = len(offsets) - 1
    ids = None if prompt_ids is None else np.ascontiguousarray(prompt_ids, np.uint64)
    out = np.empty(n, np.uint32)
    N.raise_for(lib.skv_route_depth(_ptr(tokens), _ptr(offsets), n, block_tokens, depth, _ptr(ids), world, _ptr(out)),
                "route")
    return out


def split_batch(tokens, offsets, users, owners, ranks: np.ndarray, rank: int):
    """The sub-batch of the prompts routed to ``rank``, in their original (global) order."""
    tokens = np.asarray(tokens)
    offsets = np.asarray(offsets, np.uint64)
    sel = np.flatnonzero(ranks == rank)
    lens = (offsets[1:] - offsets[:-1])[sel]
    off = np.zeros(len(sel) + 1, np.uint64)
    np.cumsum(lens, out=off[1:])
    parts = [tokens[int(offsets[p]):int(offsets[p + 1])] for p in sel]
    tok = np.concatenate(parts).astype(np.uint32) if parts else np.zeros(0, np.uint32)
    own = None if owners is None else np.asarray(owners, np.uint8)[sel]
    return tok, off, np.asarray(users, np.uint64)[sel], own
