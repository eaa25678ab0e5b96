"""the /cache-tool-output endpoint bound to a *live* engine's
store (the reference's `serve` only builds a standalone store, cli.py:190-192).
A wire submission made while the sequence is decoding its reasoning turns the
call into a full hit: validated, ingested in place, never evicted."""

import json

from fastapi.testclient import TestClient

from oracle import scenarios as S
from paper_2512_15834_b200.engine import EngineConfig
from paper_2512_15834_b200.service import create_app
from harness.sim import Simulator
from stub_runtime import stub_factory

API = S.product_api()


def test_wire_submission_hits_live_engine():
    sim = Simulator()
    engine = stub_factory(sim, EngineConfig(prefill_rate=0.25, decode_rate=0.5, tool_cache=True))
    client = TestClient(create_app(engine.store))
    stub = S.StubClient(sim, engine)
    engine.submit_request("resp-1", S._script(API, [4], ['{"q": 1}']), 10, stub)

    def post():
        body = [{"name": "lookup", "params": {"q": 1}, "output": "x" * 40}]
        r = client.post("/cache-tool-output/resp-1", content=json.dumps(body))
        assert r.status_code == 200 and r.content == b'{"cached": 1}'

    sim.schedule(3.0, post)  # during reasoning (prefill ends 2.5, reasoning ends 4.5)
    sim.run_until_idle()
    seq = engine.sequences["resp-1"]
    assert seq.fates == ["full_hit"]
    assert seq.accepted_counts == [3]
    assert engine.evictions == 0
    assert any(e.endswith("phase=ingest tokens=10") for e in engine.events)  # ceil(40 bytes / 4)
    assert engine.store.live_entries("resp-1") == 0  # purged at the end


def test_wire_submission_after_span_is_a_miss():
    sim = Simulator()
    engine = stub_factory(sim, EngineConfig(prefill_rate=0.25, decode_rate=0.5, tool_cache=True))
    client = TestClient(create_app(engine.store))
    stub = S.StubClient(sim, engine)
    engine.submit_request("resp-2", S._script(API, [4], ['{"q": 1}']), 10, stub)
    sim.schedule(9.0, lambda: client.post("/cache-tool-output/resp-2",
                                          content=json.dumps([{"name": "lookup", "params": {"q": 1}, "output": "y"}])))
    sim.run_until_idle()
    assert engine.sequences["resp-2"].fates == ["miss"]
    assert engine.evictions == 1
