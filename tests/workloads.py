"""Seeded synthetic batches for parity tests (test infrastructure).

Prompts are built from a small set of shared "trunk" texts (so leading blocks collide
across prompts and users -> shared index entries, invisible private prefixes, intra-batch
duplicate inserts), random word suffixes, PII phrases from the reference's template
families (often straddling block boundaries or sitting in the right-context window),
ragged lengths (partial tail blocks, prompts shorter than one block, empty prompts),
and occasional non-byte token ids (>= 256).
"""
from __future__ import annotations

import numpy as np

PII = [b"my ssn is 123-45-6789", b"call me at (415) 555-0134", b"email me at user99@mail01.com",
       b"server at 10.4.77.3", b"card number 4111-1111-1111-1111", b"account number 48392057",
       b"device mac 0a:1b:2c:3d:4e:5f", b"imei 490154203237518", b"PROJECT-TITAN", b"(PROJECT-TITAN).",
       b"account no. 1234567", b"415-555-0134"]
WORDS = [b"alpha", b"beta", b"cache", b"kv", b"block", b"prefix", b"user", b"the", b"a", b"of", b"imei",
         b"account", b"number", b"no", b"10", b"4111", b"x", b"PROJECT-TITANIC", b"mail", b"@", b"."]


def _text(rng, n_words, pii_p):
    parts = []
    for _ in range(n_words):
        if rng.random() < pii_p:
            parts.append(PII[rng.integers(len(PII))])
        else:
            parts.append(WORDS[rng.integers(len(WORDS))])
    sep = [b" ", b" ", b" ", b"\n", b"\t", b", "]
    out = b""
    for p in parts:
        out += p + sep[rng.integers(len(sep))]
    return out


def make_trunks(rng, n_trunks, pii_p=0.15):
    return [_text(rng, int(rng.integers(0, 40)), pii_p) for _ in range(n_trunks)]


def make_batch(rng, trunks, n_prompts, n_users, business_p=0.3, pii_p=0.08, wide_p=0.0, max_words=40,
               user_base=1, align=0):
    """align > 0: every prompt length is cut down to a multiple of `align` tokens."""
    toks, offs, users, owners = [], [0], [], []
    for _ in range(n_prompts):
        r = rng.random()
        if r < 0.05:
            text = b""  # empty prompt
        elif r < 0.1:
            text = b"tiny"[: int(rng.integers(0, 4))]
        else:
            t = trunks[rng.integers(len(trunks))]
            cut = int(rng.integers(0, len(t) + 1)) if rng.random() < 0.3 else len(t)
            text = t[:cut] + _text(rng, int(rng.integers(0, max_words)), pii_p)
        arr = np.frombuffer(text, np.uint8).astype(np.uint32)
        if align:
            arr = arr[: len(arr) - len(arr) % align]
        if wide_p and len(arr) and rng.random() < wide_p:
            k = int(rng.integers(len(arr)))
            arr[k] = arr[k] | (int(rng.integers(1, 1 << 20)) << 8)
        toks.append(arr)
        offs.append(offs[-1] + len(arr))
        u = user_base + int(rng.integers(n_users))
        users.append(u)
        owners.append(1 if (u * 2654435761) % 1000 < business_p * 1000 else 0)
    tokens = np.concatenate(toks) if toks else np.zeros(0, np.uint32)
    return (tokens.astype(np.uint32), np.array(offs, np.uint64), np.array(users, np.uint64),
            np.array(owners, np.uint8))
