"""B200-native engine-side hot path of arXiv 2512.15834 (speculative tool calls).

Drop-in for the reference `spectool` engine surface (`pkg/src/spectool/engine.py`,
`service.py`): `EngineSim` (= `B200Engine`), `EngineConfig`, `ToolCacheStore`,
`CacheEntry`, `validate_draft`, `split_turn` and `create_app` (the
`/cache-tool-output` endpoint), plus the token / tool-call vocabulary they read.
Phases execute on sm_100a kernels through `libstb200.so` (include/stb200.h,
DESIGN.md). Token identity is structural (kind value, text), so the reference's
own `Token` objects, scripts and clients drive this engine unchanged; its error
classes can be bridged with `errors.bridge(spectool.errors)`.

The caller side used to drive the engine in tests and the bench (Simulator,
EngineClient, workload fleets) is NOT part of this package: see `harness/`.

Imports here are CPU-safe: nothing touches CUDA until an engine builds its runtime.
"""

from .domain import CanonicalKey, Token, TokenKind, ToolCall, canonical_key, extract_tool_call, render_tool_call
from .engine import B200Engine, CacheEntry, EngineConfig, EngineSim, ToolCacheStore, split_turn, validate_draft
from .errors import ConfigError, InvalidScenario, KernelError, KVCapacityError, SpectoolError, bridge

__all__ = [
    "B200Engine", "CacheEntry", "CanonicalKey", "ConfigError", "EngineConfig", "EngineSim", "InvalidScenario",
    "KVCapacityError", "KernelError", "SpectoolError", "Token", "TokenKind", "ToolCacheStore", "ToolCall",
    "bridge", "canonical_key", "extract_tool_call", "render_tool_call", "split_turn", "validate_draft",
]

__version__ = "0.2.0"
