"""K4b — the tool-cache key lookup on the device (`stb_key_match` via runtime/keyindex.py).

The reference looks a finished span's call up by canonical key (`engine.py:339-355`) in a host
dict keyed by (rid, key hex) (`engine.py:63-65`) with lazy, inclusive expiry (`engine.py:55-58`).
The device index hashes the canonical key bytes to 128-bit digests and matches them bit-exactly on
the GPU; these tests hold it to the host dict's answers (same entry object, or both misses) over a
store with overwrites, expiries and purges, and run the reference timelines with the engine's
`_span_end` lookups on the device: events and fates equal the reference goldens."""

import random

import pytest

pytestmark = pytest.mark.gpu


class _Clock:
    def __init__(self):
        self.t = 0.0

    def __call__(self):
        return self.t


def _build(seed):
    from paper_2512_15834_b200.domain import CanonicalKey
    from paper_2512_15834_b200.engine import CacheEntry, ToolCacheStore

    rng = random.Random(seed)
    clock = _Clock()
    store = ToolCacheStore(clock)
    keys = [CanonicalKey(f"tool{rng.randrange(6)}({{\"q\":{rng.randrange(10 ** 6)}}})".encode()) for _ in range(300)]
    rids = [f"r{i}" for i in range(12)]
    log = []
    for i in range(400):
        clock.t += 0.01
        rid, key = rng.choice(rids), rng.choice(keys)
        ka = rng.choice([None, 0.5, 2.0])
        store.submit(rid, CacheEntry(name=f"tool{i % 5}", output="x" * rng.randrange(40), key=key, keep_alive=ka))
        log.append((rid, key))
        if i % 97 == 96:
            store.purge_request(rng.choice(rids))
    return store, clock, keys, rids, log


def test_key_match_kernel_equals_host_dict():
    from paper_2512_15834_b200.domain import CanonicalKey
    from paper_2512_15834_b200.runtime.keyindex import DeviceKeyIndex

    host, hclock, keys, rids, log = _build(7)
    dev, dclock, _, _, _ = _build(7)  # same sequence: identical store
    index = DeviceKeyIndex(dev)
    rng = random.Random(3)
    probes = [p for p in log] + [(rng.choice(rids), rng.choice(keys)) for _ in range(300)]
    probes += [(rng.choice(rids), CanonicalKey(b"absent(" + bytes([rng.randrange(256)]) + b")")) for _ in range(50)]
    probes += [("nobody", k) for k in keys[:20]]
    hits = 0
    for step, (rid, key) in enumerate(probes):
        hclock.t = dclock.t = 4.0 + step * 0.003  # expiries happen during the probe sequence
        want = host.lookup_key(rid, key)
        got = index.lookup(rid, key)
        assert (got is None) == (want is None), (rid, key)
        if want is not None:
            assert got.name == want.name and got.output == want.output and got.key == want.key
            hits += 1
    assert hits > 50 and index.launches == len(probes)


def test_key_match_batch_and_first_slot():
    """A batch of probes in one launch; a digest present for several rids matches only its own."""
    import torch

    from paper_2512_15834_b200.domain import CanonicalKey
    from paper_2512_15834_b200.engine import CacheEntry, ToolCacheStore
    from paper_2512_15834_b200.runtime.keyindex import DeviceKeyIndex

    store = ToolCacheStore(lambda: 0.0)
    k = CanonicalKey(b'grep({"q":"x"})')
    for rid in ("a", "b", "c"):
        store.submit(rid, CacheEntry(name="grep", output=rid, key=k))
    store.submit("b", CacheEntry(name="ls", output="b2", key=CanonicalKey(b"ls({})")))
    index = DeviceKeyIndex(store)
    slots = index.match([("a", k.data), ("b", k.data), ("c", k.data), ("d", k.data), ("b", b"ls({})"), ("a", b"ls({})")])
    assert [index._entries[j].output if j >= 0 else None for j in slots] == ["a", "b", "c", None, "b2", None]
    assert index.launches == 1
    torch.cuda.synchronize()


@pytest.mark.parametrize("case", ["full_hit", "partial_hit", "two_turn_mixed", "late_hit", "expired"])
def test_timelines_with_device_key_lookup(golden, case):
    from oracle import scenarios as S
    from paper_2512_15834_b200.engine import B200Engine
    from paper_2512_15834_b200.modelcfg import TINY
    from paper_2512_15834_b200.runtime.executor import EagerRuntime

    if case not in S.TIMELINE_CASES:
        pytest.skip(f"{case} not among the golden timelines")
    engines = []

    def gpu(sim, cfg):
        e = B200Engine(sim, cfg, runtime=EagerRuntime(TINY, num_blocks=512), device_keys=True)
        engines.append(e)
        return e

    got, _ = S.run_timeline(S.product_api(), case, gpu)
    assert got == golden["timelines"][case]
    assert any(e.key_index is not None and e.key_index.launches > 0 for e in engines if e.store is not None)
