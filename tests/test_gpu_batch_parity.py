"""Numeric parity of the THROUGHPUT path (what bench.py times): `BatchRuntime` with one flight
in the air (pipeline=True), >= 8 concurrent agent sequences whose steps pack decode rows
together with prompt prefills, suffix re-prefills after misses, draft-verify passes (full and
partial acceptance, K4 + rollback) and in-place tool-output ingests, on a wall-clock fleet.

Every completed flight is replayed on the fp32 CPU oracle (`oracle/cpu_decoder.py`): each
sequence's fed run (rid, start, ids) is appended to its oracle KV cache at the same start (so
rollbacks / evictions truncate it exactly as the paged pool does) and the oracle's logits of the
sampled rows are compared with the GPU's: relative L2 <= 2e-2 per row (bf16 vs fp32, BASELINE
north star); the GPU's unforced raw argmax must be a near-max of the oracle's logits. The KV
allocator's op log is replayed on the oracle's LIFO allocator (`oracle/kv_alloc.py`) and every
sequence's block table at every flight completion must match it bit for bit.
(Reference: the engine hosts many concurrent sequences, `engine.py:172-180`; the fleet driver is
`workload.py:293-384`.)
"""

import dataclasses
import random

import pytest

pytestmark = pytest.mark.gpu

LOGIT_RTOL = 2e-2


def _run_fleet(shape, agents: int, steps: int, seed: int = 1, num_blocks: int = 4096):
    from harness.fleet import Fleet, TraceSpec, engine_config
    from paper_2512_15834_b200.domain import Token, TokenKind
    from paper_2512_15834_b200.engine import B200Engine
    from paper_2512_15834_b200.runtime.executor import BatchRuntime
    from paper_2512_15834_b200.runtime.realtime import RealtimeLoop

    rt = BatchRuntime(shape, num_blocks=num_blocks, max_slots=256, max_ctx=4096, max_step_tokens=1024, pipeline=True,
                      record=True)
    loop = RealtimeLoop()
    engine = B200Engine(loop, engine_config(agents), runtime=rt)
    rng = random.Random(seed)
    orig = engine.submit_tool_cache

    def submit(rid, entry):  # one draft in three: right key, wrong call tokens -> partial hit + rollback
        if entry.call_tokens and rng.random() < 0.33:
            toks = list(entry.call_tokens)
            k = rng.randrange(1, len(toks) - 1)
            toks[k] = Token(TokenKind.TEXT, toks[k].text + "~")
            entry = dataclasses.replace(entry, call_tokens=toks)
        return orig(rid, entry)

    engine.submit_tool_cache = submit
    spec = TraceSpec(prompt_tokens=40, reason=(3, 18), call_tokens=8, output=(2, 30), tool_latency=(0.002, 0.03),
                     tools=(1, 3), closing=(1, 3), draft_latency=0.004, accept_rate=0.8, seed=seed, library=16)
    fleet = Fleet(engine, loop, spec, agents)
    fleet.start()
    loop.run_until_idle(max_steps=steps)
    rt.drain()
    return rt, engine


def _replay(rt, shape, num_blocks=4096):
    """Oracle replay of every flight (logits, raw argmax) + LIFO-allocator replay (block tables)."""
    from oracle.cpu_decoder import CpuDecoder, RouteHints
    from oracle.kv_alloc import LifoAllocator

    ora = CpuDecoder(shape)
    if shape.moe:
        ora.bf16_points = True
        ora.route_hints = RouteHints().add_flights(rt.flights)
    alloc = LifoAllocator(num_blocks)
    ops, op_i, worst = rt.pool.log, 0, 0.0
    for f in rt.flights:
        k = 0
        for rid, start, ids, rows in f["items"]:
            want = ora.forward(rid, ids, start, rows)
            for j in range(len(rows)):
                got = f["logits"][k]
                worst = max(worst, float((got - want[j]).norm() / want[j].norm()))
                k += 1
        while op_i < f["pool_ops"]:
            op, slot, n = ops[op_i]
            getattr(alloc, op)(slot, n) if op != "release" else alloc.release(slot)
            op_i += 1
        for rid, slot in f["slots"].items():
            assert alloc.blocks(slot) == f["tables"][rid], (rid, slot)
    return worst


def test_batch_runtime_kv_preemption():
    """A KV pool far smaller than the fleet's working set: the step packer holds runs back and
    preempts decoding sequences (largest context first), recomputing their rows when blocks return
    (BatchRuntime._fit / _restore). The run completes; every sampled row — the recompute runs
    included — still matches the oracle within 2e-2 and the block tables match the LIFO replay."""
    from paper_2512_15834_b200.modelcfg import TINY

    rt, engine = _run_fleet(TINY, agents=12, steps=400, num_blocks=48)
    assert rt.spills > 0, "the pool never ran out: the test did not exercise preemption"
    assert _replay(rt, TINY, num_blocks=48) <= LOGIT_RTOL


@pytest.mark.parametrize("name", ["tiny", "qwen3-mini", "llama3-8b[L=2,V=32k]", "gpt-oss-mini"])
def test_batch_runtime_parity(name):
    from oracle.cpu_decoder import CpuDecoder
    from oracle.kv_alloc import LifoAllocator
    from paper_2512_15834_b200.modelcfg import GPT_OSS_MINI, SHAPES, QWEN3_MINI, TINY

    shape = {"tiny": TINY, "qwen3-mini": QWEN3_MINI, "gpt-oss-mini": GPT_OSS_MINI}.get(name) or dataclasses.replace(
        SHAPES["llama3-8b"], name=name, layers=2, vocab=32768)
    big = name.startswith("llama")
    rt, engine = _run_fleet(shape, agents=10 if big else 12, steps=140 if big else 260)
    ora = CpuDecoder(shape)
    if shape.moe:  # storage rounding as on the engine; the engine's choice on router near-ties only
        from oracle.cpu_decoder import RouteHints

        ora.bf16_points = True
        ora.route_hints = RouteHints().add_flights(rt.flights)
    alloc = LifoAllocator(4096)
    ops = rt.pool.log
    op_i = 0
    worst, rows_checked = 0.0, 0
    mixed = verify = multi_run = 0
    for f in rt.flights:
        k = 0
        runs = [it for it in f["items"] if len(it[2]) > 1 or it[3] != [0]]
        mixed += bool(runs) and len(runs) < len(f["items"])
        multi_run += len(runs) >= 2
        verify += any(len(rows) > 1 for _, _, _, rows in f["items"])
        for rid, start, ids, rows in f["items"]:
            want = ora.forward(rid, ids, start, rows)
            for j in range(len(rows)):
                got = f["logits"][k]
                err = float((got - want[j]).norm() / want[j].norm())
                worst = max(worst, err)
                raw = f["raw"][k]
                gap = float(want[j].max() - want[j][raw])
                assert gap <= 2e-2 * float(want[j].max() - want[j].min()), (rid, start, j, raw, gap)
                k += 1
                rows_checked += 1
        assert k == len(f["logits"])
        while op_i < f["pool_ops"]:
            op, slot, n = ops[op_i]
            getattr(alloc, op)(slot, n) if op != "release" else alloc.release(slot)
            op_i += 1
        for rid, slot in f["slots"].items():
            assert alloc.blocks(slot) == f["tables"][rid], (rid, slot)
    assert worst <= LOGIT_RTOL, worst
    assert ora.arbitrated <= max(2, 0.03 * ora.routed), (ora.arbitrated, ora.routed)
    fates = [x for s in engine.sequences.values() for x in s.fates]
    # the trace really exercised the packed mixed path
    assert len(rt.flights) >= 100 and rows_checked >= 500
    assert mixed >= 10 and verify >= 5 and multi_run >= 3, (mixed, verify, multi_run)
    assert {"full_hit", "partial_hit"} <= set(fates) and engine.evictions > 0, (set(fates), engine.evictions)


@pytest.mark.parametrize("name", ["tiny", "qwen3-mini", "llama3-8b[L=2,V=32k]"])
def test_batch_runtime_parity_verify_in_k3(name, monkeypatch):
    """The same wall-clock fleet with every step's short runs (verify passes, small ingests)
    folded into the decode attention launch as multi-query K3 entries (stb_attn_decode_mq) — the
    benchmarked path for steps with >= 16 decode rows, forced here for this fleet's smaller
    batches: sampled-row logits within 2e-2 of the oracle replay, raw argmax a near-max, block
    tables equal to the LIFO replay."""
    from paper_2512_15834_b200.modelcfg import QWEN3_MINI, SHAPES, TINY
    from paper_2512_15834_b200.runtime import decoder as D

    monkeypatch.setattr(D, "MQ_MIN_DECODE", 1)
    calls = {"mq": 0}
    orig = D.Decoder._mq_entries

    def counted(self, b):
        r = orig(self, b)
        calls["mq"] += r is not None
        return r

    monkeypatch.setattr(D.Decoder, "_mq_entries", counted)
    shape = {"tiny": TINY, "qwen3-mini": QWEN3_MINI}.get(name) or dataclasses.replace(
        SHAPES["llama3-8b"], name=name, layers=2, vocab=32768)
    big = name.startswith("llama")
    rt, engine = _run_fleet(shape, agents=10 if big else 12, steps=140 if big else 260)
    assert calls["mq"] >= 5, calls  # steps whose runs rode in K3
    assert _replay(rt, shape) <= LOGIT_RTOL
