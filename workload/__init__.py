"""Bench / test workload generator (NOT product code): ctypes binding of workload/skv_gen.h.

The generator is compiled into ``workload/libskv_gen.so`` (used by our bench arm and the
tests) and, from the same source, into ``oracle/_ref/libsafekv_ref.so`` (used by the
reference arm of bench.py, which must not load the product library).  ``use_library``
selects which one this module binds.  Inputs are built from the reference's generator
primitives (SplitMix64 / derive_seed util.hpp:14-55, detail::filler workload.hpp:256-266,
detail::make_secret workload.hpp:182-241); every prompt is a pure function of
(seed, prompt id).
"""
from __future__ import annotations

import ctypes as C
import pathlib
from dataclasses import dataclass
from typing import Optional

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
GEN_SO = ROOT / "workload" / "libskv_gen.so"


class _Spec(C.Structure):
    _fields_ = [("n_prompts", C.c_uint64), ("prompt_tokens", C.c_uint64), ("n_users", C.c_uint64),
                ("first_user", C.c_uint64), ("pool_size", C.c_uint64), ("pool_tokens", C.c_uint64),
                ("shared_fraction", C.c_double), ("pii_per_kib", C.c_double), ("pii_mix", C.c_uint32),
                ("pad0_", C.c_uint32), ("seed", C.c_uint64), ("prompt_id_base", C.c_uint64),
                ("route_world", C.c_uint32), ("route_rank", C.c_uint32), ("route_block_tokens", C.c_uint32),
                ("route_depth", C.c_uint32), ("prompt_ids_out", C.c_void_p)]


_lib = None


def use_library(path: str | pathlib.Path | None = None) -> C.CDLL:
    """Bind the generator from ``path`` (default workload/libskv_gen.so)."""
    global _lib
    p = pathlib.Path(path) if path else GEN_SO
    if not p.exists():
        raise ImportError(f"{p} not found: build it with `make`")
    L = C.CDLL(str(p))
    vp = C.c_void_p
    for name, args in (("skvgen_generate", [C.POINTER(_Spec), vp, vp, vp, vp, C.c_int]),
                       ("skvgen_generate_pool", [C.POINTER(_Spec), vp, vp, vp, vp]),
                       ("skvgen_route", [vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, vp, C.c_uint32, vp])):
        f = getattr(L, name)
        f.restype, f.argtypes = C.c_int, args
    _lib = L
    return L


def _L() -> C.CDLL:
    return _lib if _lib is not None else use_library()


def _ptr(a):
    return None if a is None else a.ctypes.data


def _ok(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"{what}: status {rc}")


@dataclass
class GenSpec:
    n_prompts: int
    prompt_tokens: int
    n_users: int = 64
    first_user: int = 1
    pool_size: int = 256
    pool_tokens: int = 640
    shared_fraction: float = 1.0
    pii_per_kib: float = 1.0
    pii_mix: int = 0
    seed: int = 1
    prompt_id_base: int = 0
    # routed generation: the first n_prompts ids routed to route_rank (skv_route_depth)
    route_world: int = 1
    route_rank: int = 0
    route_block_tokens: int = 16
    route_depth: int = 0

    def native(self, ids_out: Optional[np.ndarray] = None) -> _Spec:
        return _Spec(self.n_prompts, self.prompt_tokens, self.n_users, self.first_user, self.pool_size,
                     self.pool_tokens, self.shared_fraction, self.pii_per_kib, self.pii_mix, 0, self.seed,
                     self.prompt_id_base, self.route_world, self.route_rank, self.route_block_tokens,
                     self.route_depth, _ptr(ids_out))


def generate(spec: GenSpec, nthreads: int = 0, tokens_out: Optional[np.ndarray] = None,
             return_ids: bool = False):
    """Deterministic synthetic batch (host): tokens, offsets, users, owners (+ global prompt ids)."""
    n, L = spec.n_prompts, spec.prompt_tokens
    tokens = tokens_out if tokens_out is not None else np.empty(n * L, np.uint32)
    offsets = np.empty(n + 1, np.uint64)
    users = np.empty(n, np.uint64)
    owners = np.empty(n, np.uint8)
    ids = np.empty(n, np.uint64)
    s = spec.native(ids)
    _ok(_L().skvgen_generate(C.byref(s), _ptr(tokens), _ptr(offsets), _ptr(users), _ptr(owners), nthreads),
        "generate")
    return (tokens, offsets, users, owners, ids) if return_ids else (tokens, offsets, users, owners)


def route(tokens, offsets, world: int, block_tokens: int, prompt_ids=None, depth: int = 0) -> np.ndarray:
    """The router's rank of every prompt (same arithmetic as the product's skv_route_depth)."""
    tokens = np.ascontiguousarray(tokens, np.uint32)
    offsets = np.ascontiguousarray(offsets, np.uint64)
    n = len(offsets) - 1
    ids = None if prompt_ids is None else np.ascontiguousarray(prompt_ids, np.uint64)
    out = np.empty(n, np.uint32)
    _ok(_L().skvgen_route(_ptr(tokens), _ptr(offsets), n, block_tokens, depth, _ptr(ids), world, _ptr(out)), "route")
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


def generate_pool(spec: GenSpec, rank: Optional[int] = None):
    """The shared-prefix pool; with ``rank`` (and spec.route_world > 1) only the prefixes
    routed to that rank."""
    n, L = spec.pool_size, spec.pool_tokens
    tokens = np.empty(n * L, np.uint32)
    offsets = np.empty(n + 1, np.uint64)
    users = np.empty(n, np.uint64)
    owners = np.empty(n, np.uint8)
    s = spec.native()
    _ok(_L().skvgen_generate_pool(C.byref(s), _ptr(tokens), _ptr(offsets), _ptr(users), _ptr(owners)),
        "generate_pool")
    if rank is None or spec.route_world <= 1:
        return tokens, offsets, users, owners
    ranks = route(tokens, offsets, spec.route_world, spec.route_block_tokens, depth=spec.route_depth)
    return split_batch(tokens, offsets, users, owners, ranks, rank)
