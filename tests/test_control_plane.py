"""Control-plane parity (CPU): the B200 engine's host logic and the oracle's
restated engine against golden vectors produced by the REAL reference
(oracle/gen_golden.py). Event logs, fates, accepted counts, evictions,
client callbacks, closed-form windows and fleet results must be identical.
"""

import pytest

from oracle import scenarios as S
from oracle.engine import OracleEngine
from stub_runtime import stub_factory


def oracle_factory(sim, config):
    return OracleEngine(sim, config, model=None)


FACTORIES = {"b200_host": stub_factory, "oracle": oracle_factory}
API = S.product_api()


@pytest.mark.parametrize("impl", sorted(FACTORIES))
@pytest.mark.parametrize("case", S.TIMELINE_CASES)
def test_timelines(golden, impl, case):
    got, _ = S.run_timeline(API, case, FACTORIES[impl])
    assert got == golden["timelines"][case]


@pytest.mark.parametrize("impl", sorted(FACTORIES))
@pytest.mark.parametrize("case", S.WINDOW_CASES, ids=lambda c: str(c))
def test_windows(golden, impl, case):
    got, _ = S.run_window(API, *case, engine_factory=FACTORIES[impl])
    want = golden["windows"][f"{case[0]}|{case[1]}|{case[2]}"]
    assert got == want


@pytest.mark.parametrize("impl", sorted(FACTORIES))
@pytest.mark.parametrize("case", S.CLIENT_CASES)
def test_clients(golden, impl, case):
    got, _ = S.run_client(API, case, FACTORIES[impl])
    assert got == golden["clients"][case]


@pytest.mark.parametrize("impl", sorted(FACTORIES))
@pytest.mark.parametrize("name", sorted(S.FLEETS))
def test_fleets(golden, impl, name):
    got, _ = S.run_fleet(API, name, FACTORIES[impl])
    assert got == golden["fleets"][name]


def test_c1_fates_match_survey(golden):
    # C1 -> 32 sequences, fates {full_hit:70, late_hit:3, miss:20}, 20 evictions
    import collections

    c1 = golden["fleets"]["c1"]
    counts = collections.Counter(f for v in c1["fates"].values() for f in v)
    assert dict(counts) == {"full_hit": 70, "late_hit": 3, "miss": 20}
    assert c1["evictions"] == 20 and len(c1["fates"]) == 32


def test_domain_vectors(golden):
    assert S.domain_vectors(API) == golden["domain"]


def test_service_vectors(golden):
    assert S.service_vectors(API) == golden["service"]


def test_closed_forms(golden):
    M = API.model
    got = {"two_turn": [M.time_vanilla_engine(S.two_turn(API)), M.time_prefix_cached_engine(S.two_turn(API)),
                        M.tool_cache_saving_terms(S.two_turn(API))],
           "uneven": [M.time_vanilla_engine(S.uneven(API)), M.time_prefix_cached_engine(S.uneven(API))]}
    assert got == golden["closed_forms"]
    assert golden["windows"]["two_turn|vanilla|None"]["measured"] == pytest.approx(9.22, abs=1e-9)
    assert golden["windows"]["two_turn|prefix_cache|None"]["measured"] == pytest.approx(8.44, abs=1e-9)
    assert golden["windows"]["two_turn|tool_cache|[True, True]"]["measured"] == pytest.approx(5.48, abs=1e-9)
