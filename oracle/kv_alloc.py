"""ORACLE (test infrastructure). The paged-KV block allocator policy, restated
from DESIGN.md "H3" (the reference only counts tokens,
engine.py:151): block size 16; a LIFO stack of free ids initialised so that
pops return 0, 1, 2, ...; reserve(len) grows a slot to ceil(len/16) blocks;
truncate(len) pops blocks off the slot's tail onto the stack (last block
first); release = truncate(0).
"""

from __future__ import annotations


class LifoAllocator:
    def __init__(self, num_blocks: int, block: int = 16):
        self.block = block
        self.free = list(range(num_blocks - 1, -1, -1))
        self.slots: dict[int, list[int]] = {}

    def _need(self, n: int) -> int:
        return -(-n // self.block)

    def reserve(self, slot: int, n: int) -> None:
        bl = self.slots.setdefault(slot, [])
        while len(bl) < self._need(n):
            if not self.free:
                raise MemoryError("pool exhausted")
            bl.append(self.free.pop())

    def truncate(self, slot: int, n: int) -> None:
        bl = self.slots.setdefault(slot, [])
        while len(bl) > self._need(n):
            self.free.append(bl.pop())

    def release(self, slot: int) -> None:
        self.truncate(slot, 0)

    def blocks(self, slot: int) -> list[int]:
        return list(self.slots.get(slot, []))
