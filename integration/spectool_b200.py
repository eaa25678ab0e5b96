"""Reference-side binding: what a maintainer adds to the reference as `spectool/_b200.py`.

Swaps the reference's virtual-time `EngineSim` (`pkg/src/spectool/engine.py:172-401`) for
`B200Engine`, whose phases run on the sm_100a kernels, without touching any reference caller:

    import spectool._b200 as b200
    b200.install()                # every later `EngineSim(sim, config)` is the B200 engine

* `EngineSim(sim, config)` keeps the reference constructor; the runtime comes from
  `runtime_factory(config)` (default: the CUDA `EagerRuntime` of config C1 — one sequence per
  phase, exact virtual-time parity; pass a `BatchRuntime` builder for wall-clock throughput).
* the reference's own `Token` / `TokenKind` objects, `GenerationScript`s, `CacheEntry`s and
  clients flow through unchanged (token identity is structural in the B200 engine);
* `errors.bridge(spectool.errors)` makes every exception the engine raises an instance of the
  reference's same-named class (`errors.py:6-55`), so `except spectool.errors.ConfigError` and
  `pytest.raises(ConfigError)` in the reference callers and tests keep working.

`install()` rebinds the name in every reference module that imported it
(`spectool`, `spectool.engine`, `spectool.orchestrator` :34, `spectool.workload` :24); modules
imported afterwards (e.g. the reference tests' `from spectool.engine import EngineSim`) see it.
"""

from __future__ import annotations

import sys

from paper_2512_15834_b200 import errors as _errors
from paper_2512_15834_b200.engine import B200Engine

_runtime_factory = None


class EngineSim(B200Engine):
    """`spectool.engine.EngineSim` on the B200 runtime (same constructor). Tool calls are parsed
    and keyed by the reference's own `extract_tool_call` / `canonical_key` (set by `install`), so
    `on_emit` hands reference callers the reference's `ToolCall`."""

    def __init__(self, sim, config, runtime=None):
        if runtime is None and _runtime_factory is not None:
            runtime = _runtime_factory(config)
        super().__init__(sim, config, runtime=runtime)


def install(runtime_factory=None) -> type:
    """Rebind `EngineSim` across the reference package; returns the class installed."""
    global _runtime_factory
    _runtime_factory = runtime_factory
    import spectool
    import spectool.engine
    import spectool.errors

    import spectool.domain

    _errors.bridge(spectool.errors)
    EngineSim.parse_call = staticmethod(spectool.domain.extract_tool_call)
    EngineSim.key_of = staticmethod(spectool.domain.canonical_key)
    for name in ("spectool", "spectool.engine", "spectool.orchestrator", "spectool.workload"):
        mod = sys.modules.get(name)
        if mod is None:
            __import__(name)
            mod = sys.modules[name]
        mod.EngineSim = EngineSim
    return EngineSim
