"""Token ids: the int32 view of the reference's `Token` objects.

The reference compares `Token(kind, text)` objects (`domain.py:29-32`,
`engine.py:106`). The GPU compares int32 ids, so the engine keeps one
`TokenTable` per engine instance:

* ids 0, 1, 2 are TOOL_START, TOOL_END, EOS;
* every other distinct token gets the next free id in first-interned order.
  The engine interns a whole script at `submit_request`, so in a deterministic
  run the table is a pure function of the submission order; equality of ids
  <=> equality of tokens, which is what makes device-side draft validation
  bit-exact. Drafted tokens are looked up, never interned: a token no script
  holds compares as UNKNOWN (-2) and is fed as a hashed id (`feed`).
* identity is structural, (kind value, text), so the reference's own Token
  objects work as well as this package's.

Content the reference only counts — prompt tokens, tool-output tokens — gets
deterministic pseudo-random ids from `fill_ids(seed, rid, salt, start, n)`:
splitmix64 over (seed, fnv1a(rid), salt, position), mapped into [3, vocab).
A cached / speculated tool output that is ingested in place carries its text
(`CacheEntry.output`): its ids come from the text itself (`output_ids`: one
token per 4 UTF-8 bytes, the reference's `token_estimate`, domain.py:245-247),
so different outputs put different rows into the KV cache.
The oracle restates both rules independently (`oracle/ids.py`).
"""

from __future__ import annotations

import numpy as np

from .domain import EOS, TOOL_END, TOOL_START, Token
from .errors import ConfigError

RESERVED = 3
SALT_PROMPT = 1
SALT_OUTPUT = 2
SALT_TEXT = 3

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


UNKNOWN = -2  # compare id of a draft token the scripts never produce: equals no model id


def token_key(tok) -> tuple[str, str]:
    """Structural identity (kind value, text): the reference's own `Token`/`TokenKind`
    objects (`domain.py:22-32`) and this package's compare equal."""
    return tok.kind.value, tok.text


class TokenTable:
    def __init__(self, vocab: int):
        if vocab <= RESERVED:
            raise ConfigError("vocabulary too small")
        self.vocab = vocab
        self._ids: dict[tuple[str, str], int] = {token_key(t): i for i, t in enumerate((TOOL_START, TOOL_END, EOS))}
        self._tokens: list[Token] = [TOOL_START, TOOL_END, EOS]

    def intern(self, tok) -> int:
        key = token_key(tok)
        tid = self._ids.get(key)
        if tid is None:
            tid = len(self._tokens)
            if tid >= self.vocab:
                raise ConfigError(f"more than {self.vocab} distinct tokens in the trace")
            self._ids[key] = tid
            self._tokens.append(tok)
        return tid

    def ids(self, toks) -> list[int]:
        """Intern scripted tokens (the model can only ever be forced to these)."""
        return [self.intern(t) for t in toks]

    def lookup(self, toks) -> list[int]:
        """Compare ids of drafted tokens, never interning: a token no script holds gets
        UNKNOWN, so untrusted drafts (HTTP submissions) cannot grow the table."""
        get = self._ids.get
        return [get(token_key(t), UNKNOWN) for t in toks]

    def feed(self, toks) -> list[int]:
        """Input ids of drafted tokens for the verify forward: the interned id, else a
        deterministic hash of (kind, text) into [3, vocab) (it is never compared: acceptance
        stops at the first UNKNOWN, and rows past it are rolled back)."""
        out = []
        for t in toks:
            tid = self._ids.get(token_key(t))
            if tid is None:
                kind, text = token_key(t)
                tid = RESERVED + fnv1a64(kind + "\x00" + text) % (self.vocab - RESERVED)
            out.append(tid)
        return out

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


def output_ids(seed: int, rid: str, text: str | None, start: int, n: int, vocab: int) -> np.ndarray:
    """Ids of an ingested tool output of n tokens at positions [start, start+n): token i is the
    i-th 4-byte chunk of the output's UTF-8 bytes (ceil(bytes / 4) tokens, the reference's
    `token_estimate`, domain.py:245-247), id = 3 + splitmix64(fnv1a64(chunk) ^ seed << 32 ^
    SALT_TEXT) mod (V - 3): a text-only function, like a tokenizer. Tokens past the text (an
    entry whose output_tokens exceeds its text, or no text) are `fill_ids(..., SALT_OUTPUT)`."""
    out = fill_ids(seed, rid, SALT_OUTPUT, start, n, vocab)
    if not text or n <= 0:
        return out
    raw = text.encode("utf-8")
    m = min(n, -(-len(raw) // 4))
    with np.errstate(over="ignore"):
        h = np.array([fnv1a64_bytes(raw[4 * i:4 * i + 4]) for i in range(m)], dtype=np.uint64)
        h = _splitmix(h ^ (np.uint64(seed & 0xFFFFFFFF) << np.uint64(32)) ^ np.uint64(SALT_TEXT))
    out[:m] = (np.uint64(RESERVED) + h % np.uint64(vocab - RESERVED)).astype(np.int32)
    return out


def fnv1a64_bytes(data: bytes) -> int:
    h = 0xCBF29CE484222325
    for b in data:
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h
