"""Wall-clock agent fleets on the B200 engine (throughput mode).

A fleet is M agents, each working through scripted tasks back to back with
`EngineClient` (speculating, pushing tool outputs into the engine's cache) on
a `RealtimeLoop`; the engine runs a `BatchRuntime`, so every resident
sequence's decode shares one packed forward per step.

Trace shapes ("proposed" where BASELINE leaves it
open): C2 = Llama-3-8B, 32 agents, prompt 2048, reasoning 64-512 tokens, a
32-token call (`chunk_text`, as `build_scenario_script` does), tool outputs
64-1024 tokens, tool latency log-uniform 10 ms - 2 s seeded per (task, turn)
with `derived_rng` (`mocks.py:34-37`), draft latency 50 ms, accuracy 0.8.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass

from paper_2512_15834_b200.domain import TOOL_END, TOOL_START, Token, TokenKind, ToolCall, canonical_key
from paper_2512_15834_b200.engine import EngineConfig
from .mocks import GenerationScript, SpecConfig, ToolRuntime, derived_rng
from .orchestrator import AgentSetup, EngineClient, HopPolicy, chunk_text
from .sim import spawn
from .workload import TOOL_ROSTER, task_assignment


@dataclass(frozen=True)
class TraceSpec:
    prompt_tokens: int = 2048
    reason: tuple[int, int] = (64, 512)
    call_tokens: int = 32
    output: tuple[int, int] = (64, 1024)
    tool_latency: tuple[float, float] = (0.010, 2.0)
    tools: tuple[int, int] = (1, 5)
    closing: tuple[int, int] = (2, 6)
    draft_latency: float = 0.05
    accept_rate: float = 0.8
    seed: int = 0
    library: int = 64


def build_trace_task(spec: TraceSpec, index: int):
    """(script, fixtures {key: output text}, durations {key: seconds}) for task `index`."""
    rng = derived_rng(spec.seed, "c2_task", index)
    n_tools = spec.tools[0] + index % (spec.tools[1] - spec.tools[0] + 1)
    turns, fixtures, durations = [], {}, {}
    for j in range(n_tools):
        name = TOOL_ROSTER[rng.randrange(len(TOOL_ROSTER))]
        call = ToolCall.of(name, q=f"task{index} step{j}")
        payload = f"{call.name} {json.dumps(dict(call.args))}"
        body = [Token(TokenKind.TEXT, c) for c in chunk_text(payload, spec.call_tokens - 2)]
        reason = [Token(TokenKind.TEXT, "mull ")] * rng.randint(*spec.reason)
        turns.append(reason + [TOOL_START] + body + [TOOL_END])
        n_out = rng.randint(*spec.output)
        key = canonical_key(call)
        fixtures[key] = (f"{name}:{index}:{j}:" * n_out)[: 4 * n_out]  # token_estimate == n_out
        lo, hi = spec.tool_latency
        u = derived_rng(spec.seed, "tool_latency", index, j).random()
        durations[key] = math.exp(math.log(lo) + u * (math.log(hi) - math.log(lo)))
    turns.append([Token(TokenKind.TEXT, "answer ")] * rng.randint(*spec.closing) + [Token(TokenKind.EOS)])
    return GenerationScript(turns), fixtures, durations


class Fleet:
    """M agents cycling through the trace library against one engine."""

    def __init__(self, engine, loop, spec: TraceSpec, agents: int, agent_offset: int = 0):
        self.engine, self.loop, self.spec, self.agents = engine, loop, spec, agents
        self.offset = agent_offset
        self.library = [build_trace_task(spec, i) for i in range(spec.library)]
        fixtures, durations = {}, {}
        for _, f, d in self.library:
            fixtures.update(f)
            durations.update(d)
        self.tools = ToolRuntime(fixtures, mean=0.0, stddev=0.0, seed=spec.seed)
        self.tools.duration_map.update(durations)
        self.results = []
        self.completed = 0

    def start(self) -> None:
        for a in range(self.agents):
            spawn(self._agent(self.offset + a))

    def _agent(self, a: int):
        slot = 0
        while True:
            script = self.library[task_assignment(a, slot) % len(self.library)][0]
            setup = AgentSetup(script=script, runtime=self.tools, task_id=f"a{a}_s{slot}",
                               prompt_tokens=self.spec.prompt_tokens)
            client = EngineClient(self.loop, self.engine, setup,
                                  spec=SpecConfig(self.spec.draft_latency, self.spec.accept_rate, 1, self.spec.seed),
                                  hops=HopPolicy(), submit_to_engine=True)
            client.start()
            self.results.append(client.result)
            yield client.result.completion
            self.completed += 1
            slot += 1


ENGINE_MODES = {  # the paper's three engine variants (Eqs. 3-5; reference engine.py:245-255,374-387)
    "tool_cache": (True, True),   # tool output ingested in place into the resident sequence
    "prefix": (True, False),      # every tool call evicts down to the turn base, then re-prefills
    "vanilla": (False, False),    # every tool call evicts everything, then re-prefills it all
}


def engine_config(agents: int, mode: str = "tool_cache") -> EngineConfig:
    # rates are virtual-time charges; the wall-clock engine ignores them
    prefix, tool = ENGINE_MODES[mode]
    return EngineConfig(prefill_rate=0.0, decode_rate=0.0, batch_size=max(64, agents), prefix_cache=prefix,
                        tool_cache=tool)
