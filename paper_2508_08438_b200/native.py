"""ctypes binding of the C ABI declared in include/safekv_b200.h.

The shared library is built in-tree (``make``) into
``paper_2508_08438_b200/libsafekv_b200.so``.  Loading fails loudly if it is missing:
there is no Python or CPU implementation of the hot path behind this module.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

_HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = _HERE / "libsafekv_b200.so"

SKV_OK = 0
SKV_ERR_ARG = 1
SKV_ERR_PARSE = 2
SKV_ERR_COMPILE = 3
SKV_ERR_CONFIG = 4
SKV_ERR_CAPACITY = 5
SKV_ERR_STATE = 6
SKV_ERR_CUDA = 7
SKV_ERR_INTERNAL = 8

LABEL_PRIVATE, LABEL_PUBLIC, LABEL_PENDING, LABEL_RESTRICTED = 0, 1, 2, 3
TIER_HBM, TIER_DRAM, TIER_SSD = 0, 1, 2
MISS, PUBLIC_HIT, OWNER_HIT = 0, 1, 2
ACTION_NONE, ACTION_DOWNGRADE, ACTION_RESTRICT = 0, 1, 2


class SkvError(RuntimeError):
    """Base error; subclasses mirror safekv::Error (reference core.hpp:19-59)."""

    code = SKV_ERR_INTERNAL


class ArgError(SkvError):
    code = SKV_ERR_ARG


class ParseError(SkvError):
    code = SKV_ERR_PARSE


class CompileError(SkvError):
    code = SKV_ERR_COMPILE


class ConfigError(SkvError):
    code = SKV_ERR_CONFIG


class CapacityExhausted(SkvError):
    code = SKV_ERR_CAPACITY


class StateError(SkvError):
    code = SKV_ERR_STATE


class CudaError(SkvError):
    code = SKV_ERR_CUDA


_ERRORS = {c.code: c for c in (ArgError, ParseError, CompileError, ConfigError, CapacityExhausted, StateError,
                               CudaError)}


def raise_for(rc: int, msg: str) -> None:
    if rc != SKV_OK:
        raise _ERRORS.get(rc, SkvError)(f"[{rc}] {msg}")


class DfaView(C.Structure):
    _fields_ = [("n_states", C.c_uint32), ("n_classes", C.c_uint32), ("start", C.c_uint32),
                ("class_map", C.POINTER(C.c_uint8)), ("next", C.POINTER(C.c_uint16)),
                ("acc", C.POINTER(C.c_uint32)), ("nfa_states", C.c_uint32),
                ("dfa_states_unminimized", C.c_uint32)]


class Config(C.Structure):
    _fields_ = [("device", C.c_int), ("block_tokens", C.c_uint32), ("window_tokens", C.c_uint32),
                ("index_capacity", C.c_uint64), ("max_prompts", C.c_uint64), ("max_tokens", C.c_uint64),
                ("max_window_entries", C.c_uint64), ("entropy_jump", C.c_double), ("u_pre_max", C.c_uint64),
                ("max_users", C.c_uint64)]


class Batch(C.Structure):
    _fields_ = [("tokens", C.c_void_p), ("offsets", C.c_void_p), ("users", C.c_void_p), ("owners", C.c_void_p),
                ("n_prompts", C.c_uint32), ("n_tokens", C.c_uint64), ("on_device", C.c_int),
                ("token_bytes", C.c_void_p)]


class AdmitOut(C.Structure):
    _fields_ = [("block_h", C.c_void_p), ("block_d", C.c_void_p), ("label", C.c_void_p),
                ("rule_mask", C.c_void_p), ("decision", C.c_void_p), ("matched_blocks", C.c_void_p),
                ("lowest_tier", C.c_void_p), ("block_offsets", C.c_void_p), ("on_device", C.c_int),
                ("n_blocks", C.c_uint64), ("matched_total", C.c_uint64)]


class Event(C.Structure):
    _fields_ = [("h", C.c_uint64), ("d", C.c_uint64), ("action", C.c_uint8), ("owner", C.c_uint8),
                ("pad", C.c_uint8 * 6), ("entropy_now", C.c_double), ("entropy_prev", C.c_double),
                ("u_pre", C.c_uint64), ("epoch", C.c_uint64)]


class Entry(C.Structure):
    _fields_ = [("h", C.c_uint64), ("d", C.c_uint64), ("creator", C.c_uint64), ("label", C.c_uint8),
                ("owner", C.c_uint8), ("tier", C.c_uint8), ("hit_cur", C.c_uint64), ("u_cnt", C.c_uint64),
                ("hit_pre", C.c_uint64), ("u_pre", C.c_uint64)]


class StageTimes(C.Structure):
    _fields_ = [("hash_scan_ms", C.c_float), ("chain_probe_ms", C.c_float), ("record_ms", C.c_float),
                ("admit_total_ms", C.c_float), ("commit_ms", C.c_float), ("epoch_ms", C.c_float),
                ("matched_total", C.c_uint64), ("accesses", C.c_uint64), ("new_blocks", C.c_uint64),
                ("touched_entries", C.c_uint64), ("replayed_entries", C.c_uint64),
                ("kernels_launched", C.c_uint32), ("prefetched", C.c_uint32)]


class CostModel(C.Structure):
    _fields_ = [("t_base_ms", C.c_double), ("c_prefill_ms", C.c_double), ("tier_penalty_ms", C.c_double * 3),
                ("noise_sigma_ms", C.c_double), ("seed", C.c_uint64)]


class RepEntry(C.Structure):
    _fields_ = [("h", C.c_uint64), ("d", C.c_uint64), ("ph", C.c_uint64), ("pd", C.c_uint64), ("creator", C.c_uint64),
                ("gid", C.c_uint64), ("label", C.c_uint8), ("owner", C.c_uint8), ("pad", C.c_uint8 * 6)]


class RepAccess(C.Structure):
    _fields_ = [("h", C.c_uint64), ("d", C.c_uint64), ("user", C.c_uint64), ("gid", C.c_uint64),
                ("count", C.c_uint64)]


# name -> (restype, argtypes); this table is also the export list checked by the CPU tests
SIGNATURES = {
    "skv_rules_default": (C.c_int, [C.POINTER(C.c_void_p)]),
    "skv_rules_from_json": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]),
    "skv_rules_free": (None, [C.c_void_p]),
    "skv_rules_version": (C.c_uint64, [C.c_void_p]),
    "skv_rules_count": (C.c_uint32, [C.c_void_p]),
    "skv_rules_info": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p),
                                 C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "skv_rules_warning_count": (C.c_size_t, [C.c_void_p]),
    "skv_rules_warning": (C.c_char_p, [C.c_void_p, C.c_size_t]),
    "skv_rules_group_count": (C.c_uint32, [C.c_void_p]),
    "skv_rules_enabled_count": (C.c_uint32, [C.c_void_p]),
    "skv_rules_enabled_rule": (C.c_uint32, [C.c_void_p, C.c_uint32]),
    "skv_rules_mask_words": (C.c_uint32, [C.c_void_p]),
    "skv_mask_words": (C.c_uint32, [C.c_void_p]),
    "skv_set_graphs": (C.c_int, [C.c_void_p, C.c_int]),
    "skv_access_entropy": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_size_t, C.c_void_p]),
    "skv_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                           C.c_size_t, C.c_void_p, C.c_void_p]),
    "skv_last_rule_masks": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "skv_rules_dfa": (C.c_int, [C.c_void_p, C.POINTER(DfaView)]),
    "skv_config_default": (None, [C.POINTER(Config)]),
    "skv_create": (C.c_int, [C.POINTER(Config), C.POINTER(C.c_void_p)]),
    "skv_destroy": (C.c_int, [C.c_void_p]),
    "skv_last_error": (C.c_char_p, [C.c_void_p]),
    "skv_set_rules": (C.c_int, [C.c_void_p, C.c_void_p]),
    "skv_stream": (C.c_void_p, [C.c_void_p]),
    "skv_admit": (C.c_int, [C.c_void_p, C.POINTER(Batch), C.POINTER(AdmitOut)]),
    "skv_prefetch": (C.c_int, [C.c_void_p, C.POINTER(Batch)]),
    "skv_commit": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "skv_epoch": (C.c_int, [C.c_void_p, C.POINTER(Event), C.c_size_t, C.POINTER(C.c_size_t),
                            C.POINTER(C.c_uint64)]),
    "skv_last_events": (C.c_int, [C.c_void_p, C.POINTER(Event), C.c_size_t, C.POINTER(C.c_size_t)]),
    "skv_set_monitor_config": (C.c_int, [C.c_void_p, C.c_double, C.c_uint64]),
    "skv_set_label_policy": (C.c_int, [C.c_void_p, C.c_int]),
    "skv_resolve_blocks": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p,
                                     C.c_void_p]),
    "skv_set_tiers": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p]),
    "skv_export": (C.c_int, [C.c_void_p, C.POINTER(Entry), C.c_size_t, C.POINTER(C.c_size_t)]),
    "skv_entry_count": (C.c_uint64, [C.c_void_p]),
    "skv_enable_eviction": (C.c_int, [C.c_void_p, C.c_int]),
    "skv_evict": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p,
                            C.c_size_t]),
    "skv_last_times": (C.c_int, [C.c_void_p, C.POINTER(StageTimes)]),
    "skv_cost_model_default": (None, [C.POINTER(CostModel)]),
    "skv_set_cost_model": (C.c_int, [C.c_void_p, C.POINTER(CostModel)]),
    "skv_admit_ttft": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "skv_lookup": (C.c_int, [C.c_void_p, C.POINTER(Batch), C.POINTER(AdmitOut)]),
    "skv_insert": (C.c_int, [C.c_void_p, C.POINTER(Batch), C.POINTER(C.c_uint64)]),
    "skv_get_entries": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(Entry), C.c_void_p]),
    "skv_label_entries": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint8, C.c_int,
                                    C.POINTER(C.c_size_t)]),
    "skv_record_accesses": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    "skv_roll_entries": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    "skv_check_anomaly": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(Event),
                                    C.POINTER(C.c_int)]),
    "skv_leak_flags": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.POINTER(C.c_uint64)]),
    "skv_tier1_scan": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.c_void_p]),
    "skv_stage": (C.c_int, [C.c_void_p, C.c_void_p]),
    "skv_set_tier_budget": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64]),
    "skv_tier_usage": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "skv_last_drops": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "skv_tier1_scan_batch": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_uint32, C.c_void_p]),
    "skv_token_seq_digest": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_uint64)]),
    "skv_set_replicated_depth": (C.c_int, [C.c_void_p, C.c_uint32]),
    "skv_replica_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t),
                                     C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t), C.c_int]),
    "skv_replica_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_int]),
    "skv_route": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p]),
    "skv_route_depth": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p,
                                  C.c_uint32, C.c_void_p]),
}

_lib = None


def load_library(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load (once) the in-tree CUDA library.  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    p = pathlib.Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(f"{p} not found: build it with `make` (or __graft_entry__.build()); "
                          "there is no CPU fallback for the SafeKV admission path")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
