"""Test / bench HARNESS — not part of the product.

Restatements of the reference's *caller side* of the engine (`spectool/sim.py`,
`mocks.py`, `orchestrator.py`, `workload.py`, the engine closed forms of
`model.py`), used only to DRIVE the product engine where the reference itself is
not installed: the CPU/GPU parity suites (through `oracle/scenarios.py`) and
`bench.py`'s wall-clock agent fleet (`harness/fleet.py`). The modules say
"Restates ..." in their docstrings; they carry no hot-path code.

With the reference installed, its own modules drive `B200Engine` directly
(`integration/spectool_b200.py`, `tests/test_reference_suite.py`),
so nothing here is needed for the drop-in.
"""
