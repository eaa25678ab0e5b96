"""The tool-cache endpoint in front of a LIVE wall-clock engine on the B200:
a real uvicorn server thread serves `create_app(engine.store)` while the main thread drives
`RealtimeLoop` + `BatchRuntime` (continuous batching, one flight in the air). A client thread
posts the speculated tool output over HTTP while the sequence is decoding its reasoning; the
engine validates the draft on the GPU (K4) and ingests the output in place: fate full_hit, no
eviction. Through the replica router front door as well (two replica stores, the second owning
the sequence)."""

import json
import threading
import time

import httpx
import pytest

pytestmark = pytest.mark.gpu

from oracle import scenarios as S  # noqa: E402
from test_service_router import BODY, Server  # noqa: E402

API = S.product_api()


@pytest.mark.parametrize("front", ["direct", "router"])
def test_http_submission_hits_live_wallclock_engine(front):
    from paper_2512_15834_b200.engine import B200Engine, EngineConfig, ToolCacheStore
    from paper_2512_15834_b200.modelcfg import TINY
    from paper_2512_15834_b200.runtime.executor import BatchRuntime
    from paper_2512_15834_b200.runtime.realtime import RealtimeLoop
    from paper_2512_15834_b200.service import ReplicaRouter, create_app, create_router_app

    rt = BatchRuntime(TINY, num_blocks=1024, max_slots=16, max_ctx=4096)
    loop = RealtimeLoop()
    engine = B200Engine(loop, EngineConfig(prefill_rate=0.0, decode_rate=0.0, tool_cache=True), runtime=rt)
    if front == "direct":
        app = create_app(engine.store)
    else:
        other = ToolCacheStore(time.monotonic)
        router = ReplicaRouter(2)
        router.assign("live-1", 1)
        app = create_router_app([other, engine.store], router)
    client = S.StubClient(loop, engine)
    started = threading.Event()
    orig = client.on_turn_start

    def on_turn_start(rid, turn):
        orig(rid, turn)
        started.set()

    client.on_turn_start = on_turn_start
    replies = []
    with Server(app) as url:
        def post():
            started.wait(timeout=60)
            with httpx.Client(base_url=url, timeout=10) as c:
                replies.append(c.post("/cache-tool-output/live-1", content=json.dumps(BODY)))

        th = threading.Thread(target=post, daemon=True)
        th.start()
        # 400 reasoning tokens: hundreds of GPU steps, so the post lands mid-reasoning
        engine.submit_request("live-1", S._script(API, [400], ['{"q": 1}']), 64, client)
        loop.run_until_idle()
        th.join(timeout=30)
    rt.drain()
    assert replies and replies[0].status_code == 200 and replies[0].content == b'{"cached": 1}'
    seq = engine.sequences["live-1"]
    assert seq.fates == ["full_hit"], seq.fates
    assert engine.evictions == 0
    assert any("phase=ingest" in e for e in engine.events)
