"""ORACLE (test infrastructure). Token-id rules, restated independently of
paper_2512_15834_b200/tokens.py: ids 0/1/2 = TOOL_START/TOOL_END/EOS, other
tokens numbered in first-interned order; uncounted content (prompt / tool
output) ids = 3 + splitmix64(seed, fnv1a64(rid), salt, position) mod (V - 3); an
in-place-ingested tool output with text: token i = 3 + splitmix64(fnv1a64(bytes 4i..4i+3) ^
seed << 32 ^ 3) mod (V - 3) for the ceil(bytes / 4) chunks, the fill rule past them.
"""

from __future__ import annotations

MASK = (1 << 64) - 1
SALT_PROMPT, SALT_OUTPUT, SALT_TEXT = 1, 2, 3


class Interner:
    def __init__(self, vocab: int):
        self.vocab = vocab
        self.ids = {}

    def __call__(self, tok) -> int:
        kind = tok.kind.value
        fixed = {"tool_start": 0, "tool_end": 1, "eos": 2}
        if kind in fixed and tok.text == "":
            return fixed[kind]
        key = (kind, tok.text)
        if key not in self.ids:
            self.ids[key] = 3 + len(self.ids)
            assert self.ids[key] < self.vocab, "vocabulary exhausted"
        return self.ids[key]

    def many(self, toks) -> list[int]:
        return [self(t) for t in toks]

    def _known(self, tok):
        kind = tok.kind.value
        fixed = {"tool_start": 0, "tool_end": 1, "eos": 2}
        if kind in fixed and tok.text == "":
            return fixed[kind]
        return self.ids.get((kind, tok.text))

    def compare_ids(self, toks) -> list[int]:
        """Drafted tokens are never interned: unknown ones compare as -2 (equal to no id)."""
        return [-2 if (k := self._known(t)) is None else k for t in toks]

    def feed_ids(self, toks) -> list[int]:
        """Input ids of drafted tokens: known id, else 3 + fnv1a64(kind NUL text) mod (V - 3)."""
        out = []
        for t in toks:
            k = self._known(t)
            out.append(k if k is not None else 3 + _fnv(t.kind.value + "\x00" + t.text) % (self.vocab - 3))
        return out


def _fnv(text: str) -> int:
    h = 0xCBF29CE484222325
    for b in text.encode("utf-8"):
        h = ((h ^ b) * 0x100000001B3) & MASK
    return h


def _mix(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK
    return x ^ (x >> 31)


def fill(seed: int, rid: str, salt: int, start: int, n: int, vocab: int) -> list[int]:
    base = _fnv(rid) ^ ((seed & 0xFFFFFFFF) << 32) ^ salt
    return [3 + _mix(base ^ ((p * 0x2545F4914F6CDD1D) & MASK)) % (vocab - 3) for p in range(start, start + n)]


def text_ids(seed: int, rid: str, text, start: int, n: int, vocab: int) -> list[int]:
    out = fill(seed, rid, SALT_OUTPUT, start, n, vocab)
    if not text:
        return out
    raw = text.encode("utf-8")
    for i in range(min(n, (len(raw) + 3) // 4)):
        h = 0xCBF29CE484222325
        for b in raw[4 * i:4 * i + 4]:
            h = ((h ^ b) * 0x100000001B3) & MASK
        out[i] = 3 + _mix(h ^ ((seed & 0xFFFFFFFF) << 32) ^ SALT_TEXT) % (vocab - 3)
    return out
