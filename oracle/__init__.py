"""ORACLE — test infrastructure only; never imported by the product path.

CPU restatement of the reference hot path (arXiv 2512.15834 package
`spectool`, engine-side tool cache) used as the parity checker for the B200
engine. Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` leg may import it.

  engine.py       the reference EngineSim control plane (engine.py:172-401),
                  restated, driving a CPU compute model per phase
  ids.py          token-id rules (intern table, fill ids) restated
  kv_alloc.py     the deterministic LIFO block allocator restated
  cpu_decoder.py  fp32 CPU decoder (same random-init weights, upcast)
  gen_golden.py   imports the REAL reference from /root/reference (this
                  container only) and writes tests/golden/*.json

Parity pinning: the control plane (event logs, fates, accepted counts,
evictions, closed-form windows, wire bytes, keys, rng draws) is pinned to
golden vectors produced by the reference itself (gen_golden.py). Attention /
logit values and block ids have no reference counterpart (the reference has
no decoder and no paged KV: SPEC.md:17,521) — those are "parity unpinned" by
the reference and checked against this fp32 restatement only.
"""
