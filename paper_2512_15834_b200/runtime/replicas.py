"""Replica data parallelism: agent sessions share nothing, so a
box runs one engine replica per GPU and partitions agents across them. No
collective touches the data path; only end-of-run metrics are reduced
(max of times, sum of tokens) with one tiny all-reduce.
"""

from __future__ import annotations


def shard_agents(n_agents: int, world: int, rank: int) -> list[int]:
    """Static agent -> replica map: agent a lives on replica a mod world."""
    return [a for a in range(n_agents) if a % world == rank]


def reduce_run(values: list[float], ops: list[str], world: int, device="cpu") -> list[float]:
    """All-reduce a few run scalars; ops[i] in {"max", "sum"}."""
    if world == 1:
        return list(values)
    import torch
    import torch.distributed as dist

    out = []
    for v, op in zip(values, ops):
        t = torch.tensor([float(v)], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        out.append(float(t.item()))
    return out
