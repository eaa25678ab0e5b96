"""B200-native engine-side hot path of arXiv 2512.15834 (speculative tool calls).

Drop-in for the reference `spectool` engine surface: `EngineSim` (=`B200Engine`),
`EngineConfig`, `ToolCacheStore`, `CacheEntry`, `validate_draft`, `split_turn`,
the `EngineClient` caller, `run_engine_scenario`, the engine workload driver and
`create_app` (the `/cache-tool-output` endpoint). Phases execute on sm_100a
kernels through `libstb200.so` (see include/stb200.h).

Imports here are lazy-free and CPU-safe: nothing touches CUDA until an engine
builds its runtime.
"""

from .accounting import (
    EngineScenario,
    TurnFate,
    TurnProfile,
    time_engine_realized,
    time_prefix_cached_engine,
    time_tool_cache_engine,
    time_vanilla_engine,
    tool_cache_saving_terms,
)
from .domain import CanonicalKey, Token, TokenKind, ToolCall, canonical_key, extract_tool_call, render_tool_call
from .engine import B200Engine, CacheEntry, EngineConfig, EngineSim, ToolCacheStore, split_turn, validate_draft
from .errors import ConfigError, InvalidScenario, KernelError, KVCapacityError, SpectoolError
from .mocks import GenerationScript, SpecConfig, Speculator, ToolRuntime
from .orchestrator import AgentResult, AgentSetup, EngineClient, HopPolicy, run_engine_scenario
from .sim import Simulator
from .workload import WorkloadConfig, run_workload, throughput, time_saved

__all__ = [
    "AgentResult", "AgentSetup", "B200Engine", "CacheEntry", "CanonicalKey", "ConfigError", "EngineClient",
    "EngineConfig", "EngineScenario", "EngineSim", "GenerationScript", "HopPolicy", "InvalidScenario",
    "KVCapacityError", "KernelError", "Simulator", "SpecConfig", "Speculator", "SpectoolError", "Token",
    "TokenKind", "ToolCacheStore", "ToolCall", "ToolRuntime", "TurnFate", "TurnProfile", "WorkloadConfig",
    "canonical_key", "extract_tool_call", "render_tool_call", "run_engine_scenario", "run_workload",
    "split_turn", "throughput", "time_engine_realized", "time_prefix_cached_engine", "time_saved",
    "time_tool_cache_engine", "time_vanilla_engine", "tool_cache_saving_terms", "validate_draft",
]

__version__ = "0.1.0"
