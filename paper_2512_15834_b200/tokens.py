"""Token ids: the int32 view of the reference's `Token` objects.

The reference compares `Token(kind, text)` objects (`domain.py:29-32`,
`engine.py:106`). The GPU compares int32 ids, so the engine keeps one
`TokenTable` per engine instance:

* ids 0, 1, 2 are TOOL_START, TOOL_END, EOS;
* every other distinct token gets the next free id in first-interned order.
  The engine interns a whole script at `submit_request` and a draft's tokens
  at `submit_tool_cache`, so in a deterministic run the table is a pure
  function of the submission order; equality of ids <=> equality of tokens,
  which is what makes device-side draft validation bit-exact.

Content the reference only counts — prompt tokens, tool-output tokens — gets
deterministic pseudo-random ids from `fill_ids(seed, rid, salt, start, n)`:
splitmix64 over (seed, fnv1a(rid), salt, position), mapped into [3, vocab).
The oracle restates both rules independently (`oracle/ids.py`).
"""

from __future__ import annotations

import numpy as np

from .domain import EOS, TOOL_END, TOOL_START, Token
from .errors import ConfigError

RESERVED = 3
SALT_PROMPT = 1
SALT_OUTPUT = 2

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


class TokenTable:
    def __init__(self, vocab: int):
        if vocab <= RESERVED:
            raise ConfigError("vocabulary too small")
        self.vocab = vocab
        self._ids: dict[Token, int] = {TOOL_START: 0, TOOL_END: 1, EOS: 2}
        self._tokens: list[Token] = [TOOL_START, TOOL_END, EOS]

    def intern(self, tok: Token) -> int:
        tid = self._ids.get(tok)
        if tid is None:
            tid = len(self._tokens)
            if tid >= self.vocab:
                raise ConfigError(f"more than {self.vocab} distinct tokens in the trace")
            self._ids[tok] = tid
            self._tokens.append(tok)
        return tid

    def ids(self, toks) -> list[int]:
        return [self.intern(t) for t in toks]

    def token(self, tid: int) -> Token:
        return self._tokens[tid]

    def __len__(self) -> int:
        return len(self._tokens)


def fnv1a64(text: str) -> int:
    h = 0xCBF29CE484222325
    for b in text.encode("utf-8"):
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def _splitmix(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
        x = ((x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        x = ((x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return x ^ (x >> np.uint64(31))


def fill_ids(seed: int, rid: str, salt: int, start: int, n: int, vocab: int) -> np.ndarray:
    """Deterministic ids for positions [start, start+n) of uncounted content."""
    if n <= 0:
        return np.zeros(0, dtype=np.int32)
    with np.errstate(over="ignore"):
        base = np.uint64(fnv1a64(rid)) ^ (np.uint64(seed & 0xFFFFFFFF) << np.uint64(32)) ^ np.uint64(salt)
        pos = np.arange(start, start + n, dtype=np.uint64)
        h = _splitmix(base ^ (pos * np.uint64(0x2545F4914F6CDD1D)) & _M64)
    return (np.uint64(RESERVED) + h % np.uint64(vocab - RESERVED)).astype(np.int32)
