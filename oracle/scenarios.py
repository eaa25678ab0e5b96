"""ORACLE (test infrastructure). Scenario drivers shared by the golden
generator (run against the REAL reference, `oracle/gen_golden.py`) and the
parity tests (run against the oracle engine and the B200 engine).

Each driver takes `api`, a namespace exposing the reference-shaped surface
(domain / engine / mocks / sim / orchestrator / workload names), plus an
`engine_factory(sim, config)`; it returns plain JSON-able dicts so results
from different implementations compare with `==`.

Scenarios mirror the reference's own known-answer tests:
  timelines   pkg/tests/test_engine.py:196-355 (vanilla, prefix, full / late /
              partial hit, expiry, per-token validation, batch-1 admission)
  windows     pkg/tests/test_orchestrator.py:276-340 (TWO_TURN, PINNED, uneven)
  clients     pkg/tests/test_orchestrator.py:410-443 (EngineClient 9.65/7.65/6.45)
  fleets      SURVEY §8 config C1 + pkg/tests/test_workload.py:222-277 shapes
"""

from __future__ import annotations

from types import SimpleNamespace


def reference_api():
    """The real reference (this container only: /root/reference)."""
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    from spectool import domain, engine, mocks, model, orchestrator, service, sim, workload

    return SimpleNamespace(domain=domain, engine=engine, mocks=mocks, model=model, orchestrator=orchestrator,
                           service=service, sim=sim, workload=workload, is_reference=True)


def product_api():
    from harness import accounting, mocks, orchestrator, sim, workload
    from paper_2512_15834_b200 import domain, engine, service

    return SimpleNamespace(domain=domain, engine=engine, mocks=mocks, model=accounting, orchestrator=orchestrator,
                           service=service, sim=sim, workload=workload, is_reference=False)


def _call_json(call):
    return {"name": call.name, "args": [[k, v] for k, v in call.args]}


class StubClient:
    """Records callbacks; resubmits after each emit with a fixed output size
    (same behaviour as the reference test helper, pkg/tests/test_engine.py:41-70)."""

    def __init__(self, sim, engine, output_tokens=1, resubmit_delay=0.0):
        self.sim, self.engine = sim, engine
        self.output_tokens, self.resubmit_delay = output_tokens, resubmit_delay
        self.log = []

    def on_turn_start(self, rid, turn):
        self.log.append(["turn_start", self.sim.now, rid, turn])

    def on_emit(self, rid, turn, span, call, base):
        self.log.append(["emit", self.sim.now, rid, turn, _call_json(call), base])
        prompt = base + len(span) + self.output_tokens
        self.sim.schedule(self.resubmit_delay, lambda: self.engine.resubmit(rid, prompt, turn_resolved=True))

    def on_ingest(self, rid, turn, entry):
        self.log.append(["ingest", self.sim.now, rid, turn, entry.output])

    def on_final(self, rid, tokens):
        self.log.append(["final", self.sim.now, rid, len(tokens)])


def _script(api, reason_counts, payloads, final_texts=()):
    D = api.domain
    turns = []
    for n, payload in zip(reason_counts, payloads):
        turns.append([D.Token(D.TokenKind.TEXT, "r")] * n
                     + [D.TOOL_START, D.Token(D.TokenKind.TEXT, f"lookup {payload}"), D.TOOL_END])
    turns.append([D.Token(D.TokenKind.TEXT, t) for t in final_texts] + [D.Token(D.TokenKind.EOS)])
    return api.mocks.GenerationScript(turns)


def _hit_entry(api, payload='{"q": 1}', output_tokens=4, key_args=None):
    D = api.domain
    call = D.ToolCall.of("lookup", **(key_args or {"q": 1}))
    return api.engine.CacheEntry("lookup", "result", key=D.canonical_key(call),
                                 call_tokens=[D.TOOL_START, D.Token(D.TokenKind.TEXT, f"lookup {payload}"), D.TOOL_END],
                                 output_tokens=output_tokens)


def _engine_snapshot(engine, clients):
    return {
        "events": list(engine.events),
        "fates": {rid: list(s.fates) for rid, s in sorted(engine.sequences.items())},
        "accepted": {rid: list(s.accepted_counts) for rid, s in sorted(engine.sequences.items())},
        "evictions": engine.evictions,
        "client_logs": [c.log for c in clients],
        "live_entries": {rid: engine.store.live_entries(rid) for rid in sorted(engine.sequences)}
        if engine.store is not None else None,
    }


TIMELINE_CASES = ("vanilla", "prefix", "full_hit", "late_hit", "partial_hit", "expired", "per_token", "batch1",
                  "two_turn_mixed", "long_reason_partial", "zero_output")


def run_timeline(api, case: str, engine_factory, prompt: int = 10):
    E, S = api.engine, api.sim
    cfg = {
        "vanilla": dict(prefill_rate=0.25, decode_rate=0.5, prefix_cache=False),
        "prefix": dict(prefill_rate=0.25, decode_rate=0.5, prefix_cache=True),
        "batch1": dict(prefill_rate=0.25, decode_rate=0.5, prefix_cache=False, batch_size=1),
        "per_token": dict(prefill_rate=0.25, decode_rate=0.5, tool_cache=True, validate_per_token=True),
    }.get(case, dict(prefill_rate=0.25, decode_rate=0.5, tool_cache=True))
    sim = S.Simulator()
    engine = engine_factory(sim, E.EngineConfig(**cfg))
    clients = []

    def new_client(**kw):
        c = StubClient(sim, engine, **kw)
        clients.append(c)
        return c

    if case == "batch1":
        engine.submit_request("a", _script(api, [2], ['{"q": 1}']), prompt, new_client())
        engine.submit_request("b", _script(api, [2], ['{"q": 1}']), prompt, new_client())
    elif case == "two_turn_mixed":
        # two tool turns: turn 0 fully validated + ingested, turn 1 misses (no entry for q=2)
        engine.submit_request("a", _script(api, [3, 5], ['{"q": 1}', '{"q": 2}'], ["done", "!"]), prompt,
                              new_client(output_tokens=7))
        engine.submit_tool_cache("a", _hit_entry(api, output_tokens=6))
    elif case == "long_reason_partial":
        # 20 reasoning tokens, wrong draft with the right key -> partial hit, then a second hit turn
        engine.submit_request("a", _script(api, [20, 0], ['{"q": 1}', '{"q": 3}'], ["x"]), prompt, new_client())
        e = _hit_entry(api, payload='{"q": 9}', output_tokens=18)
        engine.submit_tool_cache("a", e)
        sim.schedule(12.0, lambda: engine.submit_tool_cache(
            "a", _hit_entry(api, payload='{"q": 3}', output_tokens=3, key_args={"q": 3})))
    elif case == "zero_output":
        engine.submit_request("a", _script(api, [2], ['{"q": 1}']), prompt, new_client())
        engine.submit_tool_cache("a", _hit_entry(api, output_tokens=0))
    else:
        engine.submit_request("a", _script(api, [2], ['{"q": 1}']), prompt, new_client())
        if case in ("full_hit", "per_token"):
            engine.submit_tool_cache("a", _hit_entry(api))
        elif case == "late_hit":
            sim.schedule(3.75, lambda: engine.submit_tool_cache("a", _hit_entry(api)))
        elif case == "partial_hit":
            engine.submit_tool_cache("a", _hit_entry(api, payload='{"q": 2}'))
        elif case == "expired":
            e = _hit_entry(api)
            e.keep_alive = 0.5
            engine.submit_tool_cache("a", e)
    sim.run_until_idle()
    out = _engine_snapshot(engine, clients)
    out["now"] = sim.now
    return out, engine


def two_turn(api):
    M = api.model
    return M.EngineScenario(dispatch_overhead=0.05, prefill_rate=0.001, decode_rate=0.02, prompt_tokens=1000,
                            turns=(M.TurnProfile(100, 20, 200, 1.0), M.TurnProfile(100, 20, 200, 1.0)))


def uneven(api):
    M = api.model
    return M.EngineScenario(dispatch_overhead=0.01, prefill_rate=0.002, decode_rate=0.01, prompt_tokens=400,
                            turns=(M.TurnProfile(30, 10, 50, 0.4), M.TurnProfile(60, 12, 80, 2.2),
                                   M.TurnProfile(10, 8, 20, 0.9)))


WINDOW_CASES = (("two_turn", "vanilla", None), ("two_turn", "prefix_cache", None),
                ("two_turn", "tool_cache", [True, True]), ("two_turn", "tool_cache", [True, False]),
                ("two_turn", "tool_cache", [False, True]), ("two_turn", "tool_cache", [False, False]),
                ("uneven", "vanilla", None), ("uneven", "tool_cache", [True, False, True]))


def run_window(api, scen: str, mode: str, plan, engine_factory=None):
    s = two_turn(api) if scen == "two_turn" else uneven(api)
    O = api.orchestrator
    if api.is_reference:
        rep = O.run_engine_scenario(s, mode, hit_plan=plan)
    else:
        rep = O.run_engine_scenario(s, mode, hit_plan=plan, engine_factory=engine_factory)
    return {"measured": rep.measured_seconds, "fates": list(rep.fates), "events": list(rep.events),
            "evictions": rep.evictions, "submissions": rep.store_submissions,
            "transcript": O.transcript_jsonl(rep.result)}, rep


CLIENT_CASES = ("baseline", "client_spec", "tool_cache")


def run_client(api, case: str, engine_factory):
    D, E, Mk, O, S = api.domain, api.engine, api.mocks, api.orchestrator, api.sim
    script = Mk.GenerationScript([[D.Token(D.TokenKind.TEXT, "x"), D.Token(D.TokenKind.TEXT, "y"), D.TOOL_START,
                                   D.Token(D.TokenKind.TEXT, 'fetch {"page": 0}'), D.TOOL_END],
                                  [D.Token(D.TokenKind.EOS)]])
    call = D.ToolCall.of("fetch", page=0)
    runtime = Mk.ToolRuntime({D.canonical_key(call): "page 0 body"}, mean=0.0, stddev=0.0)
    runtime.duration_map[D.canonical_key(call)] = 2.0
    cfg = E.EngineConfig(prefill_rate=0.25, decode_rate=0.5, tool_cache=(case == "tool_cache"))
    spec = None if case == "baseline" else Mk.SpecConfig(latency_seconds=0.5, accuracy=1.0, samples=1, seed=3)
    sim = S.Simulator()
    engine = engine_factory(sim, cfg)
    setup = O.AgentSetup(script=script, runtime=runtime, task_id="job", prompt_tokens=10)
    client = O.EngineClient(sim, engine, setup, spec=spec, outcome_plan=None if spec is None else [True],
                            hops=O.uniform_hops(0.1), submit_to_engine=(case == "tool_cache"),
                            output_tokens_fn=lambda turn, out: 4)
    client.start()
    sim.run_until_idle()
    return {"total": client.result.total_seconds, "hits": client.result.hits, "events": list(engine.events),
            "evictions": engine.evictions, "transcript": O.transcript_jsonl(client.result)}, engine


FLEETS = {
    # the reference CPU run (4 agents x 8 tasks)
    "c1": dict(agents=4, tasks_per_agent=8, tool_mean=0.05, tool_stddev=0.02, draft_seconds=0.05, accept_rate=0.8,
               samples=1, mode="engine_spec", backend="engine", seed=7, repetitions=1, dispatch_overhead=0.05,
               prefill_rate=0.001, decode_rate=0.02, prompt_tokens=256),
    # pkg/tests/test_workload.py:222-237 shape
    "wl_spec": dict(agents=2, tasks_per_agent=3, tool_mean=0.2, tool_stddev=0.0, draft_seconds=0.5,
                    accept_rate=1.0, samples=1, mode="engine_spec", backend="engine", seed=5, repetitions=1,
                    dispatch_overhead=0.01, prefill_rate=0.001, decode_rate=0.1, prompt_tokens=256),
    "wl_client": dict(agents=2, tasks_per_agent=3, tool_mean=0.2, tool_stddev=0.0, draft_seconds=0.5,
                      accept_rate=1.0, samples=1, mode="client_spec", backend="engine", seed=5, repetitions=1,
                      dispatch_overhead=0.01, prefill_rate=0.001, decode_rate=0.1, prompt_tokens=256),
    "wl_base_b2": dict(agents=3, tasks_per_agent=2, tool_mean=0.3, tool_stddev=0.1, draft_seconds=0.2,
                       accept_rate=0.5, samples=2, mode="baseline", backend="engine", seed=9, repetitions=1,
                       dispatch_overhead=0.02, prefill_rate=0.001, decode_rate=0.05, prompt_tokens=64),
}


def run_fleet(api, name: str, engine_factory=None):
    W = api.workload
    cfg = W.WorkloadConfig(**FLEETS[name])
    if api.is_reference:
        made = []
        orig = W.EngineSim

        class Recording(orig):
            def __init__(self, *a, **k):
                super().__init__(*a, **k)
                made.append(self)

        W.EngineSim = Recording
        try:
            run = W._execute(cfg)
        finally:
            W.EngineSim = orig
        engine = made[0]
    else:
        run = W._execute(cfg, engine_factory)
        engine = run.engine
    return {
        "fates": {k: list(v) for k, v in sorted(run.fates.items())},
        "tokens": {k: r.tokens_emitted for k, r in sorted(run.task_results.items())},
        "seconds": {k: r.total_seconds for k, r in sorted(run.task_results.items())},
        "agents": [[a.elapsed, a.tokens, a.tool_turns, a.hits] for a in run.agents],
        "events": list(engine.events),
        "evictions": engine.evictions,
        "accepted": {rid: list(s.accepted_counts) for rid, s in sorted(engine.sequences.items())},
    }, engine


def domain_vectors(api):
    D, Mk, O, W = api.domain, api.mocks, api.orchestrator, api.workload
    calls = [D.ToolCall.of("search", q="cats"), D.ToolCall.of("f", b=1, a=2.0), D.ToolCall.of("g", x=True, y=None),
             D.ToolCall("h", (("é", "ü"), ("a", 1.5), ("Z", -3))), D.ToolCall.of("noargs"),
             D.ToolCall.of("n", v=float("inf")), D.ToolCall.of("s", t='quote"and\\slash')]
    out = {
        "keys": [D.canonical_key(c).hex for c in calls],
        "render": [[t.text for t in D.render_tool_call(c)] for c in calls],
        "perturb": [D.canonical_key(Mk.perturb_call(c)).hex for c in calls],
        "token_estimate": [D.token_estimate(s) for s in ["", "a", "abcd", "abcde", "ünïcode", "x" * 41]],
        "chunk": [O.chunk_text('step0 {"index": 0}', n) for n in (1, 3, 18, 25)],
        "rng": [Mk.derived_rng(7, "tool_latency", ("a0_s0", 0), "ab").random() for _ in range(1)]
        + [Mk.truncated_normal(Mk.derived_rng(s, "x"), 0.05, 0.02) for s in range(5)],
        "coins": [Mk.Speculator(Mk.SpecConfig(0.5, 0.8, 2, 7)).sample_correct(("a1_s3", t), i)
                  for t in range(4) for i in range(2)],
        "tasks": [[[[t.kind.value, t.text] for t in turn] for turn in W.build_task(i, 7).script.turns]
                  for i in (0, 1, 13, 63)],
        "assign": [W.task_assignment(a, s) for a in range(4) for s in range(8)],
    }
    return out


def service_vectors(api):
    from fastapi.testclient import TestClient

    E, Sv = api.engine, api.service
    import json

    clock = [0.0]
    store = E.ToolCacheStore(lambda: clock[0])
    client = TestClient(Sv.create_app(store=store, clock=lambda: clock[0], max_body_bytes=512))
    bodies = [
        [{"name": "search", "params": {"q": "cats"}, "output": "felines"}],
        [{"name": "whoami", "output": "alice"}],
        [{"name": "search", "params": {"q": "ok"}, "output": "fine"}, {"name": "search"}, 5,
         {"name": "", "output": "x"}, {"name": "a", "output": "b", "keep_alive": True},
         {"name": "a", "output": "b", "keep_alive": -1}, {"name": "a", "output": "b", "params": [1]},
         {"name": "a", "output": "b", "params": {"k": [1, 2]}}],
        {"not": "a list"},
    ]
    out = []
    for b in bodies:
        r = client.post("/cache-tool-output/r1", content=json.dumps(b))
        out.append([r.status_code, r.content.decode()])
    r = client.post("/cache-tool-output/r1", content=b"{bad json")
    out.append([r.status_code, r.content.decode()[:40]])
    r = client.post("/cache-tool-output/r1", content=json.dumps([{"name": "x", "output": "y" * 600}]))
    out.append([r.status_code, r.content.decode()])
    out.append([client.get("/healthz").status_code, client.get("/healthz").content.decode()])
    out.append(["live", store.live_entries("r1"), store.submissions])
    return out
