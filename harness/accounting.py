"""Closed-form engine accounting (paper Eqs. 3-5), the virtual-time self-check.

Restates the engine half of `spectool/model.py`: `TurnProfile` (:49-64),
`EngineScenario` (:67-104), `time_vanilla_engine` (:156-165),
`time_prefix_cached_engine` (:173-182), `time_tool_cache_engine` (:185-204),
`TurnFate` / `time_engine_realized` (:207-235), `tool_cache_saving_terms`
(:238-246). The B200 engine in virtual-time mode must land on these numbers
exactly (to 1e-9), like the reference engine does.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

from paper_2512_15834_b200.errors import InvalidScenario


@dataclass(frozen=True)
class TurnProfile:
    reason_tokens: int
    call_tokens: int
    output_tokens: int
    tool_seconds: float

    def __post_init__(self) -> None:
        if self.reason_tokens < 0 or self.output_tokens < 0:
            raise InvalidScenario("token counts cannot be negative")
        if self.call_tokens < 1:
            raise InvalidScenario("a tool call is at least one token")
        if self.tool_seconds < 0:
            raise InvalidScenario("tool_seconds cannot be negative")


@dataclass(frozen=True)
class EngineScenario:
    dispatch_overhead: float
    prefill_rate: float
    decode_rate: float
    prompt_tokens: int
    turns: tuple[TurnProfile, ...]
    accept_rate: float = 0.0

    def __post_init__(self) -> None:
        object.__setattr__(self, "turns", tuple(self.turns))
        if min(self.dispatch_overhead, self.prefill_rate, self.decode_rate) < 0:
            raise InvalidScenario("rates and overhead cannot be negative")
        if self.prompt_tokens < 0:
            raise InvalidScenario("prompt_tokens cannot be negative")
        if not self.turns:
            raise InvalidScenario("an engine scenario needs at least one turn")
        if not 0.0 <= self.accept_rate <= 1.0:
            raise InvalidScenario("accept_rate must lie in [0, 1]")

    @property
    def turn_count(self) -> int:
        return len(self.turns)

    def prompt_lengths(self) -> list[int]:
        """Per-turn prompt length: history grows by call + output each turn."""
        out = [self.prompt_tokens]
        for p in self.turns[:-1]:
            out.append(out[-1] + p.call_tokens + p.output_tokens)
        return out


def _sums(s: EngineScenario) -> tuple[int, int, float]:
    return (sum(p.reason_tokens for p in s.turns), sum(p.call_tokens for p in s.turns),
            sum(p.tool_seconds for p in s.turns))


def _unique_prompt_tokens(s: EngineScenario) -> int:
    return s.prompt_tokens + sum(p.call_tokens + p.output_tokens for p in s.turns)


def time_vanilla_engine(s: EngineScenario) -> float:
    reason, calls, tools = _sums(s)
    return (2.0 * s.turn_count * s.dispatch_overhead + s.prefill_rate * sum(s.prompt_lengths())
            + s.decode_rate * (reason + calls) + tools)


def time_prefix_cached_engine(s: EngineScenario) -> float:
    reason, calls, tools = _sums(s)
    return (2.0 * s.turn_count * s.dispatch_overhead + s.prefill_rate * _unique_prompt_tokens(s)
            + s.decode_rate * (reason + calls) + tools)


def time_tool_cache_engine(s: EngineScenario) -> float:
    a, k = s.accept_rate, s.turn_count
    reason, calls, tools = _sums(s)
    return ((1.0 - a) * 2.0 * k * s.dispatch_overhead + s.prefill_rate * _unique_prompt_tokens(s)
            + s.decode_rate * (a * k + reason + (1.0 - a) * calls) + (1.0 - a) * tools)


class TurnFate(Enum):
    FULL_HIT = "full_hit"
    LATE_HIT = "late_hit"
    MISS = "miss"


def time_engine_realized(s: EngineScenario, fates: list[TurnFate]) -> float:
    if len(fates) != s.turn_count:
        raise InvalidScenario("fate vector length must equal turn count")
    total = s.prefill_rate * s.prompt_tokens
    for p, fate in zip(s.turns, fates):
        if fate is TurnFate.FULL_HIT:
            total += s.decode_rate * (p.reason_tokens + 1) + s.prefill_rate * (p.call_tokens + p.output_tokens)
        elif fate is TurnFate.LATE_HIT:
            total += s.decode_rate * (p.reason_tokens + p.call_tokens) + s.prefill_rate * p.output_tokens
        else:
            total += (s.decode_rate * (p.reason_tokens + p.call_tokens)
                      + s.prefill_rate * (p.call_tokens + p.output_tokens)
                      + 2.0 * s.dispatch_overhead + p.tool_seconds)
    return total


def tool_cache_saving_terms(s: EngineScenario) -> float:
    _, calls, tools = _sums(s)
    return 2.0 * s.turn_count * s.dispatch_overhead + s.decode_rate * (calls - s.turn_count) + tools
