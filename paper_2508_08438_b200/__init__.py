"""B200-native SafeKV admission hot path (hash -> rule-tier scan -> privacy-aware index
lookup -> entropy monitor) behind the C ABI of include/safekv_b200.h."""
from .native import (ArgError, CapacityExhausted, CompileError, ConfigError, CudaError, ParseError, SkvError,
                     StateError, load_library)
from .engine import (REP_ACCESS, REP_ENTRY, AdmissionEngine, AdmitResult, AnomalyEvent, EngineConfig, ReplicaGroup,
                     combine_mask_words,
                     RuleSet, merge_entries, merge_events, merge_replica, route, split_batch, torch_allgather,
                     torch_allgather_device)

__all__ = [
    "combine_mask_words",
    "AdmissionEngine", "AdmitResult", "AnomalyEvent", "EngineConfig", "RuleSet", "route", "split_batch",
    "ReplicaGroup", "merge_replica", "merge_entries", "merge_events", "torch_allgather", "torch_allgather_device", "REP_ENTRY", "REP_ACCESS", "load_library", "SkvError", "ArgError", "ParseError", "CompileError", "ConfigError", "CapacityExhausted",
    "CudaError", "StateError",
]
