"""Fleet driver: M agents x scripted tasks against one engine (engine backend).

Restates the engine backend of `spectool/workload.py`: the 64-task library
(`build_task` :137-155), `WorkloadConfig` (:176-231), `task_assignment`
(:234-236), `_execute` with `backend="engine"` (:293-384), the paired
baseline twin (`run_workload` :387-392), `time_saved` / `throughput`
(:47-58) and `records_jsonl` (:461-479). The API backend (fixed-latency
completion endpoint, client-side speculation only) is outside the engine hot
path and rejected here.

In virtual time (the default `Simulator`) a run is event-for-event the
reference's, with every phase executed on the GPU. The wall-clock fleet used
for throughput lives in `runtime/fleet.py` and reuses `build_task` and
`task_assignment` so both see the same scripts.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field, replace

from paper_2512_15834_b200.domain import TOOL_END, TOOL_START, Token, TokenKind, ToolCall, canonical_key
from paper_2512_15834_b200.engine import EngineConfig
from paper_2512_15834_b200.errors import ConfigError, InvalidBaseline, InvalidWindow
from .mocks import GenerationScript, SpecConfig, ToolRuntime, derived_rng
from .orchestrator import AgentResult, AgentSetup, EngineClient, default_engine_factory, uniform_hops
from .sim import Simulator, spawn

MODES = ("baseline", "client_spec", "engine_spec")
BACKENDS = ("api", "engine")
TASK_LIBRARY_SIZE = 64
TOOL_ROSTER = ("web_search", "read_file", "run_query", "fetch_url", "list_dir", "get_weather", "calculate",
               "translate")


def time_saved(t_base: float, t_spec: float) -> float:
    if t_base <= 0:
        raise InvalidBaseline(f"baseline time must be positive, got {t_base!r}")
    return 100.0 * (t_base - t_spec) / t_base


def throughput(tokens: int, elapsed: float) -> float:
    if elapsed <= 0:
        raise InvalidWindow(f"window must be positive, got {elapsed!r}")
    return tokens / elapsed


@dataclass(frozen=True)
class TaskSpec:
    library_index: int
    script: GenerationScript
    fixtures: dict
    tool_turns: int


def build_task(library_index: int, seed: int = 0) -> TaskSpec:
    """1-5 tool turns of 4-24 reasoning tokens + a 3-token call; 2-6 closing tokens + EOS."""
    rng = derived_rng(seed, "task", library_index)
    n_tools = 1 + library_index % 5
    turns, fixtures = [], {}
    for j in range(n_tools):
        name = TOOL_ROSTER[rng.randrange(len(TOOL_ROSTER))]
        call = ToolCall.of(name, q=f"task{library_index} step{j}")
        reason = [Token(TokenKind.TEXT, "mull ")] * rng.randint(4, 24)
        span = [TOOL_START, Token(TokenKind.TEXT, f"{call.name} {json.dumps(dict(call.args))}"), TOOL_END]
        turns.append(reason + span)
        fixtures[canonical_key(call)] = f"{name} result {rng.randrange(1000)} for task {library_index} step {j}"
    turns.append([Token(TokenKind.TEXT, "answer ")] * rng.randint(2, 6) + [Token(TokenKind.EOS)])
    return TaskSpec(library_index, GenerationScript(turns), fixtures, n_tools)


def build_task_library(seed: int = 0, size: int = TASK_LIBRARY_SIZE) -> list[TaskSpec]:
    return [build_task(i, seed) for i in range(size)]


def verify_fixtures(tasks: list[TaskSpec], fixtures: dict) -> None:
    for task in tasks:
        for j in range(task.tool_turns):
            if canonical_key(task.script.tool_call_at(j)) not in fixtures:
                raise ConfigError(f"missing fixture for task {task.library_index} turn {j}")


@dataclass(frozen=True)
class WorkloadConfig:
    agents: int = 1
    tasks_per_agent: int = 32
    tool_mean: float = 1.0
    tool_stddev: float = 0.0
    gen_seconds: float = 2.0
    draft_seconds: float = 0.5
    accept_rate: float = 0.8
    samples: int = 1
    mode: str = "baseline"
    backend: str = "api"
    seed: int = 0
    repetitions: int = 5
    dispatch_overhead: float = 0.0
    prefill_rate: float = 0.001
    decode_rate: float = 0.02
    prompt_tokens: int = 256
    prefix_discount: float = 1.0

    def __post_init__(self) -> None:
        if self.agents < 1:
            raise ConfigError("need at least one agent")
        if self.tasks_per_agent < 1:
            raise ConfigError("need at least one task per agent")
        if self.mode not in MODES:
            raise ConfigError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.backend not in BACKENDS:
            raise ConfigError(f"backend must be one of {BACKENDS}, got {self.backend!r}")
        if self.mode == "engine_spec" and self.backend != "engine":
            raise ConfigError("engine_spec requires the engine backend")
        if not 0.0 <= self.accept_rate <= 1.0:
            raise ConfigError("accept_rate must lie in [0, 1]")
        if self.samples < 0:
            raise ConfigError("samples cannot be negative")
        if self.repetitions < 1:
            raise ConfigError("need at least one repetition")
        if min(self.tool_mean, self.gen_seconds, self.draft_seconds) <= 0:
            raise ConfigError("latencies must be positive")
        if self.tool_stddev < 0 or self.dispatch_overhead < 0:
            raise ConfigError("spread and overhead cannot be negative")

    def spec_config(self) -> SpecConfig:
        return SpecConfig(latency_seconds=self.draft_seconds, accuracy=self.accept_rate, samples=self.samples,
                          seed=self.seed)


def task_assignment(agent_index: int, slot: int) -> int:
    return (agent_index * 13 + slot) % TASK_LIBRARY_SIZE


@dataclass
class AgentSummary:
    agent_index: int
    elapsed: float
    tokens: int
    tool_turns: int
    hits: int

    @property
    def throughput(self) -> float:
        return throughput(self.tokens, self.elapsed)


@dataclass
class WorkloadRun:
    config: WorkloadConfig
    agents: list[AgentSummary]
    task_results: dict[str, AgentResult]
    usage: list
    fates: dict[str, list[str]] = field(default_factory=dict)
    paired_baseline: "WorkloadRun | None" = None
    engine: object = None

    @property
    def total_tool_turns(self) -> int:
        return sum(a.tool_turns for a in self.agents)

    @property
    def hit_rate(self) -> float:
        n = self.total_tool_turns
        return sum(a.hits for a in self.agents) / n if n else 0.0

    @property
    def mean_throughput(self) -> float:
        return sum(a.throughput for a in self.agents) / len(self.agents)

    def per_agent_time_saved(self) -> list[float]:
        if self.paired_baseline is None:
            return [0.0] * len(self.agents)
        return [time_saved(b.elapsed, m.elapsed) for b, m in zip(self.paired_baseline.agents, self.agents)]

    @property
    def mean_time_saved(self) -> float:
        saved = self.per_agent_time_saved()
        return sum(saved) / len(saved)


def engine_config_for(config: WorkloadConfig, **extra) -> EngineConfig:
    """The engine a workload builds (`workload.py:314-323`)."""
    return EngineConfig(prefill_rate=config.prefill_rate, decode_rate=config.decode_rate,
                        batch_size=max(64, config.agents), prefix_cache=True,
                        tool_cache=config.mode == "engine_spec", **extra)


def _execute(config: WorkloadConfig, engine_factory=None, sim=None, agent_ids=None) -> WorkloadRun:
    """Run the fleet; `agent_ids` restricts it to a shard of the agents (replicas:
    sessions are independent, so a shard's agents behave exactly as in the full run)."""
    if config.backend != "engine":
        raise ConfigError("only the engine backend is part of the B200 hot path")
    library = build_task_library(config.seed)
    fixtures: dict = {}
    for task in library:
        fixtures.update(task.fixtures)
    verify_fixtures(library, fixtures)
    runtime = ToolRuntime(fixtures, mean=config.tool_mean, stddev=config.tool_stddev, seed=config.seed)
    sim = sim if sim is not None else Simulator()
    usage: list = []
    results: dict[str, AgentResult] = {}
    fates: dict[str, list[str]] = {}
    agent_ids = list(range(config.agents)) if agent_ids is None else list(agent_ids)
    plan = [(a, f"a{a}_s{s}", library[task_assignment(a, s)]) for a in agent_ids
            for s in range(config.tasks_per_agent)]
    engine = (engine_factory or default_engine_factory)(sim, engine_config_for(config))

    def start_task(task_id: str, task: TaskSpec) -> AgentResult:
        setup = AgentSetup(script=task.script, runtime=runtime, task_id=task_id,
                           prompt_tokens=config.prompt_tokens, dispatch_overhead=config.dispatch_overhead,
                           usage=usage)
        client = EngineClient(sim, engine, setup, spec=None if config.mode == "baseline" else config.spec_config(),
                              hops=uniform_hops(config.dispatch_overhead),
                              submit_to_engine=config.mode == "engine_spec")
        client.start()
        return client.result

    def agent_loop(agent: int):
        for a, task_id, task in plan:
            if a != agent:
                continue
            result = start_task(task_id, task)
            results[task_id] = result
            yield result.completion
            fates[task_id] = list(engine.sequences[task_id].fates)

    for a in agent_ids:
        spawn(agent_loop(a))
    sim.run_until_idle()

    agents = []
    for a in agent_ids:
        mine = [results[t] for ag, t, _ in plan if ag == a]
        if not all(r.done for r in mine):
            raise ConfigError(f"agent {a} did not finish all tasks")
        agents.append(AgentSummary(a, max(r.finished_at for r in mine), sum(r.tokens_emitted for r in mine),
                                   sum(len(r.outcomes) for r in mine), sum(r.hits for r in mine)))
    return WorkloadRun(config, agents, results, usage, fates, engine=engine)


def run_workload(config: WorkloadConfig, engine_factory=None) -> WorkloadRun:
    run = _execute(config, engine_factory)
    if config.mode != "baseline":
        run.paired_baseline = _execute(replace(config, mode="baseline"), engine_factory)
    return run


def records_jsonl(run: WorkloadRun, label: str | None = None) -> str:
    lines = []
    for task_id in sorted(run.task_results):
        r = run.task_results[task_id]
        rec = {"task": task_id, "mode": r.mode, "seconds": r.total_seconds, "tool_turns": len(r.outcomes),
               "hits": r.hits, "tokens": r.tokens_emitted}
        if label is not None:
            rec["run"] = label
        if task_id in run.fates:
            rec["fates"] = run.fates[task_id]
        lines.append(json.dumps(rec, sort_keys=True, separators=(",", ":")))
    return "\n".join(lines) + "\n" if lines else ""
