"""Device mirror of the tool-cache key index for the K4b digest match (`stb_key_match`).

The reference looks a finished span's call up by canonical key (`engine.py:339-355`, key bytes
from `domain.py:123-158`) in a host dict keyed by (rid, key hex) (`engine.py:63-65`). Here the
key bytes are hashed once to a 128-bit digest (BLAKE2b-128) and the live index is mirrored on the
device as int64 digest pairs plus an int32 request id per entry; a lookup is a bit-exact integer
compare on the GPU, the lowest matching slot wins (entries are uploaded in the host dict's order,
in which a (rid, key) pair is unique). The host keeps the reference's lazy expiry: a device hit is
re-checked with `ToolCacheStore.alive_or_drop`.
"""

from __future__ import annotations

import ctypes as C
import hashlib

import numpy as np
import torch

from . import lib


def key_digest(data: bytes) -> tuple[int, int]:
    """BLAKE2b-128 of the canonical key bytes as two little-endian uint64."""
    d = hashlib.blake2b(data, digest_size=16).digest()
    return int.from_bytes(d[:8], "little"), int.from_bytes(d[8:], "little")


def _as_i64(pairs: list[tuple[int, int]]) -> np.ndarray:
    a = np.array(pairs, dtype=np.uint64).reshape(-1, 2) if pairs else np.zeros((0, 2), dtype=np.uint64)
    return a.view(np.int64)


class DeviceKeyIndex:
    def __init__(self, store, device: str = "cuda"):
        self.store = store
        self.device = device
        self._version = None
        self._rid_ids: dict[str, int] = {}
        self._entries: list = []
        self._keys = torch.zeros(0, 2, dtype=torch.int64, device=device)
        self._key_rid = torch.zeros(0, dtype=torch.int32, device=device)
        self._out = torch.empty(64, dtype=torch.int32, device=device)
        self.launches = 0

    def _rid(self, rid: str) -> int:
        i = self._rid_ids.get(rid)
        if i is None:
            i = self._rid_ids[rid] = len(self._rid_ids)
        return i

    def _sync(self) -> None:
        if self._version == self.store.version:
            return
        items = self.store.key_items()
        self._entries = [e for _, e in items]
        digests = [key_digest(bytes.fromhex(hexkey)) for (_, hexkey), _ in items]
        rids = [self._rid(rid) for (rid, _), _ in items]
        self._keys = torch.from_numpy(_as_i64(digests)).to(self.device)
        self._key_rid = torch.tensor(rids, dtype=torch.int32, device=self.device)
        self._version = self.store.version

    def match(self, probes: list[tuple[str, bytes]]) -> list[int]:
        """Slot of each (rid, canonical key bytes) probe in the uploaded index, or -1."""
        self._sync()
        n = len(probes)
        if n == 0:
            return []
        probe = torch.from_numpy(_as_i64([key_digest(k) for _, k in probes])).to(self.device)
        prid = torch.tensor([self._rid(r) for r, _ in probes], dtype=torch.int32, device=self.device)
        if self._out.numel() < n:
            self._out = torch.empty(max(n, 2 * self._out.numel()), dtype=torch.int32, device=self.device)
        out = self._out[:n]
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        lib.call("stb_key_match", C.c_void_p(probe.data_ptr()), C.c_void_p(prid.data_ptr()), n,
                 C.c_void_p(self._keys.data_ptr()), C.c_void_p(self._key_rid.data_ptr()), int(self._key_rid.numel()),
                 C.c_void_p(out.data_ptr()), st)
        self.launches += 1
        return out.cpu().tolist()

    def lookup(self, rid: str, key):
        """`ToolCacheStore.lookup_key(rid, key)` through the device match (same result)."""
        j = self.match([(rid, key.data)])[0]
        if j < 0:
            return None
        return self.store.alive_or_drop(rid, self._entries[j])
