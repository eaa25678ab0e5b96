"""Replicas (N > 1) on CPU with gloo, world size 2: each rank runs its shard of
the agents through the engine's host logic; the per-agent results equal the
single-process run and the reduced totals are exact (sessions are
independent, no collective on the data path)."""

import os
import socket

import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import scenarios as S
from paper_2512_15834_b200.runtime.replicas import reduce_run, shard_agents
from harness.workload import WorkloadConfig, _execute
from stub_runtime import stub_factory


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg_kw, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = WorkloadConfig(**cfg_kw)
    mine = shard_agents(cfg.agents, world, rank)
    run = _execute(cfg, stub_factory, agent_ids=mine)
    per_agent = {a.agent_index: (a.elapsed, a.tokens, a.tool_turns, a.hits) for a in run.agents}
    tokens, makespan = reduce_run([sum(a.tokens for a in run.agents), max(a.elapsed for a in run.agents)],
                                  ["sum", "max"], world)
    gathered = [None] * world
    dist.all_gather_object(gathered, per_agent)
    if rank == 0:
        merged = {}
        for g in gathered:
            merged.update(g)
        q.put((merged, tokens, makespan))
    dist.destroy_process_group()


def test_two_replicas_match_single_process():
    cfg_kw = dict(S.FLEETS["c1"])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg_kw, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, tokens, makespan = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = _execute(WorkloadConfig(**cfg_kw), stub_factory)
    want = {a.agent_index: (a.elapsed, a.tokens, a.tool_turns, a.hits) for a in full.agents}
    assert merged == want
    assert tokens == sum(a.tokens for a in full.agents)
    assert makespan == max(a.elapsed for a in full.agents)


def test_shard_map_partitions_agents():
    for world in (1, 2, 4, 8):
        shards = [shard_agents(64, world, r) for r in range(world)]
        assert sorted(a for s in shards for a in s) == list(range(64))
        assert max(len(s) for s in shards) - min(len(s) for s in shards) <= 1
