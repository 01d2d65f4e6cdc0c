"""B200-native SafeKV admission hot path (hash -> rule-tier scan -> privacy-aware index
lookup -> entropy monitor) behind the C ABI of include/safekv_b200.h."""
from .native import (ArgError, CapacityExhausted, CompileError, ConfigError, CudaError, ParseError, SkvError,
                     StateError, load_library)
from .engine import AdmissionEngine, AdmitResult, AnomalyEvent, EngineConfig, RuleSet, route, split_batch

__all__ = [
    "AdmissionEngine", "AdmitResult", "AnomalyEvent", "EngineConfig", "RuleSet", "route", "split_batch", "load_library", "SkvError", "ArgError", "ParseError", "CompileError", "ConfigError", "CapacityExhausted",
    "CudaError", "StateError",
]
