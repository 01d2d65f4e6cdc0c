"""Prompt-leakage attack campaign over the admission path, batched.

Restates the reference adversary (adversary.hpp:83-279: ``calibrate_threshold``,
``reconstruct``, ``score_attack``, ``run_attack_campaign``, ``CampaignMetrics``) for the
batch-snapshot admission contract: instead of one probe per
``ServingSimulator::submit``, every secret under attack probes all candidates of its
current position in ONE admission batch, so a campaign over S secrets with C candidates
per position costs one GPU batch of S x C prompts per position.  Inside a batch the
probes do not see each other's inserts (snapshot semantics); across batches they do,
exactly as the reference's sequential probes see earlier probes.

The attacker observes only TTFT (``CostModel::ttft``, serving_sim.hpp:50-56, computed on
the device by the probe epilogue); the decision logic per position is the reference's:
hit iff TTFT < threshold, pick the lowest-TTFT hit, else the overall argmin flagged
low-confidence; a position that runs cold after an earlier hit marks the attack
``downgraded_mid_attack``.  Identities rotate (FreshIdentity) or stay fixed
(CalibrationDiff); the threshold is the midpoint of a miss/hit calibration pair on
attacker-owned content unless fixed.

Block granularity.  The index matches whole blocks (the north star's unit), so a
candidate is observable only when it completes a block.  ``digit_secret_plans`` builds
plans whose secret starts at a block boundary and whose positions are whole blocks
(candidates = every digit string of that block's length) -- the block-granular form of
the reference's token-by-token search.  Token-granular plans work too; their unaligned
positions are simply unobservable (low confidence).

The backend is anything with ``admit / ttft / commit / epoch``: ``EngineBackend`` wraps
the CUDA ``AdmissionEngine``; the parity tests drive the same campaign through the
reference harness and compare results field by field.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Protocol, Sequence

import numpy as np

MASK64 = (1 << 64) - 1


class SplitMix64:
    """util.hpp SplitMix64 (next, next_below)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def next_below(self, bound: int) -> int:
        return self.next() % bound


def derive_seed(root: int, tag: int) -> int:
    """util.hpp derive_seed."""
    return SplitMix64(root ^ ((0x51A1C9E3B7D24F85 * (tag + 1)) & MASK64)).next()


@dataclass
class SecretPlan:
    """workload.hpp:78-86, with multi-token candidates (one position = one block when
    block-granular)."""
    secret_id: int
    victim: int                        # victim UserId
    victim_tokens: np.ndarray          # the victim's prompt (u32 tokens)
    known_prefix: np.ndarray           # what the attacker knows precedes the secret
    candidates: list                   # per position: u32 token arrays (a 2-D array when equal length)
    truth: list                        # per position: the true token array
    category: str = ""


@dataclass
class AttackSettings:
    """adversary.hpp:30-37 (schedule/jitter have no meaning without virtual time)."""
    n_identities: int = 4
    pollution: str = "fresh"           # "fresh" (FreshIdentity) | "calibration" (CalibrationDiff)
    hit_threshold_ms: float = -1.0     # < 0: calibrated per secret
    max_probes: int = (1 << 64) - 1
    seed: int = 7


@dataclass
class AttackResult:
    """adversary.hpp:39-48."""
    recovered: list = field(default_factory=list)
    per_position_correct: list = field(default_factory=list)
    low_confidence: list = field(default_factory=list)
    probes_used: int = 0
    success: bool = False
    budget_exhausted: bool = False
    downgraded_mid_attack: bool = False
    stale_probes: int = 0


@dataclass
class CampaignMetrics:
    """adversary.hpp:165-201."""
    n_secrets: int = 0
    fully_recovered: int = 0
    positions_total: int = 0
    positions_correct: int = 0
    probes_used: int = 0
    downgraded_mid_attack: int = 0
    stale_probes: int = 0
    budget_exhausted: int = 0
    correct_by_position: list = field(default_factory=list)
    batches: int = 0
    leakage_events: int = 0

    def attack_success_rate(self) -> float:
        return self.fully_recovered / self.n_secrets if self.n_secrets else 0.0

    def defense_success_rate(self) -> float:
        return 1.0 - self.attack_success_rate()

    def per_token_recovery_rate(self) -> float:
        return self.positions_correct / self.positions_total if self.positions_total else 0.0

    def to_dict(self) -> dict:
        return {"n_secrets": self.n_secrets, "fully_recovered": self.fully_recovered,
                "attack_success_rate": self.attack_success_rate(),
                "defense_success_rate": self.defense_success_rate(),
                "per_token_recovery_rate": self.per_token_recovery_rate(),
                "positions_total": self.positions_total, "positions_correct": self.positions_correct,
                "probes_used": self.probes_used, "downgraded_mid_attack": self.downgraded_mid_attack,
                "stale_probes": self.stale_probes, "budget_exhausted": self.budget_exhausted,
                "correct_by_position": list(self.correct_by_position), "batches": self.batches,
                "leakage_events": self.leakage_events}


class Backend(Protocol):
    def admit(self, tokens: np.ndarray, offsets: np.ndarray, users: np.ndarray) -> None: ...

    def ttft(self, n: int, request_ids: np.ndarray) -> np.ndarray: ...

    def commit(self) -> None: ...

    def epoch(self) -> int: ...


class EngineBackend:
    """The CUDA admission path as an attack backend (TTFT from the device epilogue)."""

    def __init__(self, engine, cost_model: Optional[dict] = None):
        self.eng = engine
        if cost_model:
            engine.set_cost_model(**cost_model)

    def admit(self, tokens, offsets, users):
        self.eng.admit(tokens, offsets, users, np.zeros(len(offsets) - 1, np.uint8))

    def ttft(self, n, request_ids):
        return self.eng.ttft(n, request_ids)[0]

    def commit(self):
        self.eng.commit()

    def epoch(self) -> int:
        return len(self.eng.epoch_pass()[1])


def _batch(seqs: Sequence[np.ndarray]):
    off = np.zeros(len(seqs) + 1, np.uint64)
    np.cumsum([len(s) for s in seqs], out=off[1:])
    tok = np.concatenate(seqs).astype(np.uint32) if seqs else np.zeros(0, np.uint32)
    return tok, off


class _Campaign:
    def __init__(self, backend: Backend, settings: AttackSettings, epoch_every: int):
        self.b, self.s, self.k = backend, settings, max(1, epoch_every)
        self.metrics = CampaignMetrics()

    def run_batch_flat(self, tok, off, users, rids) -> np.ndarray:
        self.b.admit(tok, off, np.asarray(users, np.uint64))
        t = self.b.ttft(len(off) - 1, np.asarray(rids, np.uint64))
        self.b.commit()
        self.metrics.batches += 1
        if self.metrics.batches % self.k == 0:
            self.metrics.leakage_events += self.b.epoch()
        return t

    def run_batch(self, seqs, users, rids=None) -> Optional[np.ndarray]:
        """One admission batch: admit, TTFT (when request ids are given), commit, and the
        monitor epoch every k batches."""
        tok, off = _batch(seqs)
        self.b.admit(tok, off, np.asarray(users, np.uint64))
        t = self.b.ttft(len(seqs), np.asarray(rids, np.uint64)) if rids is not None else None
        self.b.commit()
        self.metrics.batches += 1
        if self.metrics.batches % self.k == 0:
            self.metrics.leakage_events += self.b.epoch()
        return t


def run_campaign(backend: Backend, plans: Sequence[SecretPlan], settings: AttackSettings = AttackSettings(),
                 epoch_every: int = 1, benign: Sequence[tuple] = (), victim_repeats: int = 0):
    """run_attack_campaign (adversary.hpp:232-277), batched: the victims (and any benign
    traffic, as (tokens, user) pairs) are admitted first, then one batch in which every
    victim re-sends its prompt ``victim_repeats`` times (an owner's reuse: the
    concentrated access history -- few users, many hits -- the entropy monitor compares
    against, monitor.hpp:68-70), then every secret is attacked in
    lock-step, one batch per probing round.  Returns (metrics, per-secret results)."""
    cp = _Campaign(backend, settings, epoch_every)
    m = cp.metrics
    seqs = [np.asarray(t, np.uint32) for t, _ in benign] + [p.victim_tokens for p in plans]
    users = [u for _, u in benign] + [p.victim for p in plans]
    if seqs:
        cp.run_batch(seqs, users)
    if victim_repeats and plans:
        cp.run_batch([p.victim_tokens for p in plans for _ in range(victim_repeats)],
                     [p.victim for p in plans for _ in range(victim_repeats)])
    n = len(plans)
    res = [AttackResult() for _ in plans]
    rngs = [SplitMix64(derive_seed(settings.seed, p.secret_id)) for p in plans]
    ids = [[1000000 + p.secret_id * 64 + i for i in range(max(1, settings.n_identities))] for p in plans]
    probe_seq = [0] * n  # SimAttackerView::probe_seq_

    def rid(i):
        probe_seq[i] += 1
        return 10000000 + probe_seq[i] + plans[i].secret_id * 100000

    # calibrate_threshold: attacker-owned content, miss then hit under identities[0]
    thr = [settings.hit_threshold_ms] * n
    if settings.hit_threshold_ms < 0:
        cal = [i for i in range(n)]
        content = []
        for i in cal:
            L = len(plans[i].known_prefix) + len(plans[i].candidates)
            content.append(np.array([ord("a") + rngs[i].next_below(26) for _ in range(L)], np.uint32))
        live = [i for i in cal if len(content[i])]
        if live:
            t_miss = cp.run_batch([content[i] for i in live], [ids[i][0] for i in live], [rid(i) for i in live])
            t_hit = cp.run_batch([content[i] for i in live], [ids[i][0] for i in live], [rid(i) for i in live])
            for k, i in enumerate(live):
                thr[i] = 0.5 * (float(t_hit[k]) + float(t_miss[k]))
        for i in cal:
            if not len(content[i]):
                thr[i] = 0.0
    rotation = [0] * n
    had_hit = [False] * n
    active = [True] * n
    npos = max((len(p.candidates) for p in plans), default=0)
    for pos in range(npos):
        # one batch: every active secret's candidates for this position, built per secret
        # as a (candidates x tokens) block (known prefix + recovered blocks + candidate)
        toks, lens, users, rids, spans = [], [], [], [], []
        for i, p in enumerate(plans):
            if not active[i] or pos >= len(p.candidates):
                continue
            cand = p.candidates[pos]
            a = max(0, min(len(cand), settings.max_probes - res[i].probes_used))
            if a:
                base = np.concatenate([p.known_prefix] + [np.asarray(r, np.uint32) for r in res[i].recovered])
                if isinstance(cand, np.ndarray) and cand.ndim == 2:
                    blk = np.hstack([np.broadcast_to(base, (a, len(base))), cand[:a]])
                    toks.append(blk.ravel())
                    lens.append(np.full(a, blk.shape[1], np.uint64))
                else:
                    rows = [np.concatenate([base, np.asarray(cand[j], np.uint32)]) for j in range(a)]
                    toks.append(np.concatenate(rows))
                    lens.append(np.array([len(r) for r in rows], np.uint64))
                nid = len(ids[i])
                if settings.pollution == "fresh":
                    users.append(np.asarray(ids[i], np.uint64)[(rotation[i] + np.arange(a)) % nid])
                    rotation[i] += a
                else:
                    users.append(np.full(a, ids[i][0], np.uint64))
                rids.append(10000000 + probe_seq[i] + np.arange(1, a + 1, dtype=np.uint64) + plans[i].secret_id * 100000)
                probe_seq[i] += a
                spans.append((i, a))
            res[i].probes_used += a
            if a < len(cand):
                res[i].budget_exhausted = True
                active[i] = False
        if not spans:
            break
        tok = np.concatenate(toks).astype(np.uint32)
        off = np.zeros(sum(len(x) for x in lens) + 1, np.uint64)
        np.cumsum(np.concatenate(lens), out=off[1:])
        t = cp.run_batch_flat(tok, off, np.concatenate(users), np.concatenate(rids))
        k0 = 0
        for i, a in spans:
            tt = np.asarray(t[k0:k0 + a], np.float64)
            k0 += a
            if not active[i]:
                continue  # budget ran out inside this position: no pick (reconstruct returns)
            best_any = int(np.argmin(tt))  # first minimum, as the strict '<' scan
            hit = tt < thr[i]
            any_hit = bool(hit.any())
            if not any_hit and had_hit[i]:
                res[i].downgraded_mid_attack = True
                res[i].stale_probes += len(plans[i].candidates[pos])
            if any_hit:
                pick = int(np.flatnonzero(hit)[np.argmin(tt[hit])])
            else:
                pick = best_any
            res[i].low_confidence.append(not any_hit)
            res[i].recovered.append(np.asarray(plans[i].candidates[pos][pick], np.uint32))
            had_hit[i] = had_hit[i] or any_hit
    for i, p in enumerate(plans):
        score_attack(p, res[i])
        m.n_secrets += 1
        m.fully_recovered += 1 if res[i].success else 0
        m.positions_total += len(p.truth)
        if len(m.correct_by_position) < len(res[i].per_position_correct):
            m.correct_by_position += [0] * (len(res[i].per_position_correct) - len(m.correct_by_position))
        for k, ok in enumerate(res[i].per_position_correct):
            if ok:
                m.positions_correct += 1
                m.correct_by_position[k] += 1
        m.probes_used += res[i].probes_used
        m.downgraded_mid_attack += 1 if res[i].downgraded_mid_attack else 0
        m.stale_probes += res[i].stale_probes
        m.budget_exhausted += 1 if res[i].budget_exhausted else 0
    return m, res


def score_attack(plan: SecretPlan, res: AttackResult) -> None:
    """adversary.hpp:147-158."""
    res.per_position_correct = []
    ok_all = len(plan.truth) > 0
    for i, tr in enumerate(plan.truth):
        ok = i < len(res.recovered) and np.array_equal(res.recovered[i], np.asarray(tr, np.uint32))
        res.per_position_correct.append(ok)
        ok_all = ok_all and ok
    if not plan.truth:
        ok_all = True
    res.success = ok_all


def _text(s: str) -> np.ndarray:
    return np.frombuffer(s.encode(), np.uint8).astype(np.uint32)


def digit_secret_plans(n: int, block_tokens: int, digits: int = 8, seed: int = 1, first_id: int = 0,
                       position_tokens: Optional[int] = None, n_candidates: Optional[int] = None,
                       prefix: str = "system: you are a banking assistant. ", lead: str = "my account number ",
                       first_victim: int = 10):
    """Victims whose prompts carry an account-number secret (the account template of
    workload.hpp make_secret, matched by the shipped ``bank_account`` rule) right after a
    known prefix, padded (before the lead-in, so the rule still matches) so that the
    secret starts at a block boundary.  A position is ``position_tokens`` digits
    (default: one block); its candidates are every digit string of that length (10**k),
    or, with ``n_candidates``, an ascending deterministic subset of that size holding the
    truth (an attacker with a shortlist)."""
    k = position_tokens or block_tokens
    if digits % k:
        raise ValueError("digits must be a multiple of the position length")
    rng = SplitMix64(derive_seed(seed, 0x5EC7))
    plans = []
    for s in range(n):
        sid = first_id + s
        head = prefix + f"[{sid}] "
        pad = (-(len(head) + len(lead))) % block_tokens
        known = _text(head + "." * pad + lead)
        secret = "".join(str(rng.next_below(10)) for _ in range(digits))
        victim = np.concatenate([known, _text(secret), _text(" thanks")])
        cands, truth = [], []
        for q in range(digits // k):
            tv = int(secret[q * k:(q + 1) * k])
            if n_candidates is None or n_candidates >= 10 ** k:
                vals = list(range(10 ** k))
            else:
                pool = {tv}
                while len(pool) < n_candidates:
                    pool.add(rng.next_below(10 ** k))
                vals = sorted(pool)
            cands.append(np.array([[ord(c) for c in f"{v:0{k}d}"] for v in vals], np.uint32))
            truth.append(_text(secret[q * k:(q + 1) * k]))
        plans.append(SecretPlan(secret_id=sid, victim=first_victim + s, victim_tokens=victim, known_prefix=known,
                                candidates=cands, truth=truth, category="account"))
    return plans
