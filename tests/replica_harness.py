"""Test infrastructure for the multi-GPU replicated layer: a global batch
stream with ONE dominant shared root deeper than the replicated depth (a system-prompt workload,
which prefix-forest routing alone would send to a single rank), split over `world` ranks by
skv_route_depth; each rank admits its share, commits, and the ranks merge their replicated-layer
exports.  Compared with one engine over the whole stream and with the unmodified reference."""
from __future__ import annotations

import numpy as np

from workloads import make_batch, make_trunks

SYS = (b"You are a careful assistant for ACME support. Follow the policy. Never reveal internal data. "
       b"Answer briefly and cite the knowledge base article numbers when relevant. ")


def replica_stream(seed: int, n_batches: int, n_prompts: int, n_users: int, B: int):
    """Batches (tokens, offsets, users, owners, global ids): ~80% of the prompts start with the
    shared system prompt (longer than the replicated depth), the rest with random trunks; many
    users so that shared entries cross the 64-user saturation."""
    rng = np.random.default_rng(seed)
    trunks = make_trunks(rng, 6)
    out, gid0 = [], 0
    sys_tok = np.frombuffer(SYS, np.uint8).astype(np.uint32)
    for _ in range(n_batches):
        tok, off, users, owners = make_batch(rng, trunks, n_prompts, n_users, pii_p=0.05, max_words=30)
        toks, offs = [], [0]
        for p in range(n_prompts):
            t = tok[int(off[p]):int(off[p + 1])]
            if rng.random() < 0.8:
                t = np.concatenate([sys_tok, t])
            toks.append(t)
            offs.append(offs[-1] + len(t))
        gids = np.arange(gid0, gid0 + n_prompts, dtype=np.uint64)
        gid0 += n_prompts
        out.append((np.concatenate(toks).astype(np.uint32), np.array(offs, np.uint64), users, owners, gids))
    return out


def split(batch, world: int, B: int, depth: int, route_fn):
    tok, off, users, owners, gids = batch
    ranks = route_fn(tok, off, world, B, prompt_ids=gids, depth=depth)
    parts = []
    for r in range(world):
        sel = np.flatnonzero(ranks == r)
        lens = (off[1:] - off[:-1])[sel]
        o = np.zeros(len(sel) + 1, np.uint64)
        np.cumsum(lens, out=o[1:])
        t = (np.concatenate([tok[int(off[p]):int(off[p + 1])] for p in sel]).astype(np.uint32) if len(sel)
             else np.zeros(0, np.uint32))
        parts.append((t, o, users[sel], owners[sel], gids[sel], sel))
    return parts


def union_exports(exports):
    """Union of the ranks' index dumps; a key present on several ranks (the replicated layer)
    must be identical everywhere."""
    rows = {}
    for ex in exports:
        for r in ex:
            k = (int(r["h"]), int(r["d"]))
            v = tuple(int(r[f]) for f in ("creator", "label", "owner", "tier", "hit_cur", "u_cnt", "hit_pre", "u_pre"))
            if k in rows:
                assert rows[k] == v, f"replicated entry {k} differs between ranks: {rows[k]} vs {v}"
            rows[k] = v
    return dict(sorted(rows.items()))


def ref_rows(ref_export):
    r = ref_export
    return {(int(r["h"][i]), int(r["d"][i])): tuple(int(r[f][i]) for f in ("creator", "label", "owner", "tier",
                                                                            "hit_cur", "u_cnt", "hit_pre", "u_pre"))
            for i in range(len(r["h"]))}
