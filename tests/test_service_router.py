"""Per-replica routing of `POST /cache-tool-output/{response_id}` (sessions are
partitioned over G replica engines, each with its own ToolCacheStore shard; §8f row 2: the
endpoint bound to live engines). The router front door sends each submission to the store of
the replica that owns the response id — in process, or over HTTP to the replica process's own
endpoint, served here by real uvicorn server threads — with the reference's wire bytes
(`service.py:20-24,91-116`) either way."""

import json
import socket
import threading
import time

import httpx
import pytest
import uvicorn

from harness.sim import Simulator
from paper_2512_15834_b200.engine import EngineConfig, ToolCacheStore
from paper_2512_15834_b200.service import ReplicaRouter, create_app, create_router_app, fleet_owner
from oracle import scenarios as S
from stub_runtime import stub_factory

API = S.product_api()
BODY = [{"name": "lookup", "params": {"q": 1}, "output": "x" * 40}]


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class Server:
    """uvicorn in a daemon thread on 127.0.0.1."""

    def __init__(self, app):
        self.port = _free_port()
        self.server = uvicorn.Server(uvicorn.Config(app, host="127.0.0.1", port=self.port, log_level="warning"))
        self.thread = threading.Thread(target=self.server.run, daemon=True)

    def __enter__(self):
        self.thread.start()
        t0 = time.time()
        while not self.server.started:
            if time.time() - t0 > 20:
                raise RuntimeError("uvicorn did not start")
            time.sleep(0.02)
        return f"http://127.0.0.1:{self.port}"

    def __exit__(self, *exc):
        self.server.should_exit = True
        self.thread.join(timeout=10)


def test_router_owner_functions():
    r = ReplicaRouter(4, fleet_owner(8))
    assert [r.owner(f"a{a}_s3") for a in (0, 7, 8, 31)] == [0, 0, 1, 3]
    r.assign("a0_s0", 2)
    assert r.owner("a0_s0") == 2
    h = ReplicaRouter(3)
    assert all(0 <= h.owner(f"x{i}") < 3 for i in range(50))
    with pytest.raises(ValueError):
        r.assign("z", 4)


def test_router_in_process_replicas():
    from fastapi.testclient import TestClient

    stores = [ToolCacheStore(time.monotonic) for _ in range(3)]
    router = ReplicaRouter(3)
    router.assign("resp-a", 2)
    router.assign("resp-b", 0)
    client = TestClient(create_router_app(stores, router))
    r = client.post("/cache-tool-output/resp-a", content=json.dumps(BODY))
    assert r.status_code == 200 and r.content == b'{"cached": 1}'
    assert [s.live_entries("resp-a") for s in stores] == [0, 0, 1]
    r = client.post("/cache-tool-output/resp-b", content=json.dumps(BODY + [{"name": ""}]))
    assert r.content == b'{"cached": 1, "rejected": [{"index": 1, "error": "missing tool name"}]}'
    assert stores[0].live_entries("resp-b") == 1
    assert client.post("/cache-tool-output/resp-b", content=b"[").status_code == 400


def test_router_forwards_to_replica_servers():
    """Two replica endpoints (each create_app over its own store) and the router front door, all
    real uvicorn servers; submissions land only in the owning replica's store, replies verbatim."""
    stores = [ToolCacheStore(time.monotonic) for _ in range(2)]
    with Server(create_app(stores[0])) as u0, Server(create_app(stores[1], max_body_bytes=64)) as u1:
        router = ReplicaRouter(2, fleet_owner(4))
        with Server(create_router_app([u0, u1], router)) as front:
            with httpx.Client(base_url=front, timeout=10) as c:
                assert c.get("/healthz").json() == {"status": "ok", "replicas": 2}
                r = c.post("/cache-tool-output/a1_s0", content=json.dumps(BODY))  # agent 1 -> replica 0
                assert r.status_code == 200 and r.content == b'{"cached": 1}'
                r = c.post("/cache-tool-output/a5_s2", content=json.dumps([{"name": "t", "output": "o"}]))
                assert r.content == b'{"cached": 1}'  # agent 5 -> replica 1
                big = c.post("/cache-tool-output/a6_s0", content=json.dumps(BODY))  # > replica 1's 64-byte cap
                assert big.status_code == 413 and b"64 bytes" in big.content
    assert stores[0].live_entries("a1_s0") == 1 and stores[1].live_entries("a1_s0") == 0
    assert stores[1].live_entries("a5_s2") == 1 and stores[0].live_entries("a5_s2") == 0


def test_router_feeds_live_engines():
    """Two replica engines (stub runtimes, virtual time) behind the router: a wire submission for
    each engine's sequence, made while it reasons, turns that sequence's call into a full hit."""
    from fastapi.testclient import TestClient

    sims = [Simulator(), Simulator()]
    engines = [stub_factory(s, EngineConfig(prefill_rate=0.25, decode_rate=0.5, tool_cache=True)) for s in sims]
    router = ReplicaRouter(2)
    client = TestClient(create_router_app([e.store for e in engines], router))
    for i, (sim, eng) in enumerate(zip(sims, engines)):
        rid = f"resp-{i}"
        router.assign(rid, i)
        eng.submit_request(rid, S._script(API, [4], ['{"q": 1}']), 10, S.StubClient(sim, eng))
        sim.schedule(3.0, lambda rid=rid: client.post(f"/cache-tool-output/{rid}", content=json.dumps(BODY)))
        sim.run_until_idle()
        assert eng.sequences[rid].fates == ["full_hit"] and eng.evictions == 0
    assert engines[0].store.submissions == 1 and engines[1].store.submissions == 1
