"""ORACLE (test infrastructure). Generates tests/golden/reference_*.json by
running the REAL reference package (`/root/reference/pkg/src/spectool`,
imported in place, unmodified) through the scenario drivers in
oracle/scenarios.py. Run in the build container (the reference does not
exist on the GPU box); the JSON it writes is committed.

    python -m oracle.gen_golden
"""

from __future__ import annotations

import json
from pathlib import Path

from . import scenarios as S

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main() -> None:
    api = S.reference_api()
    factory = api.engine.EngineSim
    OUT.mkdir(parents=True, exist_ok=True)
    timelines = {c: S.run_timeline(api, c, factory)[0] for c in S.TIMELINE_CASES}
    windows = {f"{s}|{m}|{p}": S.run_window(api, s, m, p)[0] for s, m, p in S.WINDOW_CASES}
    clients = {c: S.run_client(api, c, factory)[0] for c in S.CLIENT_CASES}
    fleets = {n: S.run_fleet(api, n)[0] for n in S.FLEETS}
    M = api.model
    closed = {
        "two_turn": [M.time_vanilla_engine(S.two_turn(api)), M.time_prefix_cached_engine(S.two_turn(api)),
                     M.tool_cache_saving_terms(S.two_turn(api))],
        "uneven": [M.time_vanilla_engine(S.uneven(api)), M.time_prefix_cached_engine(S.uneven(api))],
    }
    doc = {"source": "/root/reference/pkg/src/spectool (unmodified, imported in place)",
           "timelines": timelines, "windows": windows, "clients": clients, "fleets": fleets,
           "closed_forms": closed, "domain": S.domain_vectors(api), "service": S.service_vectors(api)}
    path = OUT / "reference_control_plane.json"
    path.write_text(json.dumps(doc, indent=1, sort_keys=True))
    print(f"wrote {path} ({path.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
