"""Wall-clock event loop: real timers interleaved with continuous-batching steps.

Stands in for the reference `Simulator` (`sim.py:29-66`) when the engine runs
for throughput: same `now` / `schedule(delay, fn, name)` / `clock()` /
`sleep()` surface, so `EngineClient`, `ToolRuntime` and the workload agents
drive it unchanged, but time is `time.monotonic()` and every engine phase
is a job of the attached `BatchRuntime`. `run_until_idle()` alternates:
fire every due timer (tool completions, draft arrivals, client/engine
hops), then run one packed GPU step if any sequence has work, else sleep
until the next timer.
"""

from __future__ import annotations

import heapq
import time
from typing import Callable

from ..errors import InvalidDelay


class Future:
    """Single-assignment value resolved by a timer (what `sleep` hands to a driving coroutine:
    the same `resolve` / `result` / `add_done_callback` surface as the reference `sim.Future`,
    `sim.py:69-97`); callbacks run on the loop thread."""

    __slots__ = ("done", "_value", "_callbacks")

    def __init__(self):
        self.done, self._value, self._callbacks = False, None, []

    def resolve(self, value) -> None:
        if self.done:
            raise RuntimeError("future resolved twice")
        self.done, self._value = True, value
        callbacks, self._callbacks = self._callbacks, []
        for cb in callbacks:
            cb(value)

    def result(self):
        if not self.done:
            raise RuntimeError("future not resolved yet")
        return self._value

    def add_done_callback(self, cb) -> None:
        if self.done:
            cb(self._value)
        else:
            self._callbacks.append(cb)


class RealtimeLoop:
    realtime = True

    def __init__(self):
        self._t0 = time.monotonic()
        self._heap: list = []
        self._seq = 0
        self.runtime = None
        self.steps = 0
        self.on_step: Callable | None = None  # (step_index, emitted_tokens) after each step

    @property
    def now(self) -> float:
        return time.monotonic() - self._t0

    def clock(self) -> float:
        return self.now

    def attach(self, runtime) -> None:
        self.runtime = runtime

    def schedule(self, delay: float, action: Callable[[], None], name: str = ""):
        if delay < 0:
            raise InvalidDelay(f"cannot schedule {delay} seconds into the past")
        heapq.heappush(self._heap, (self.now + delay, self._seq, action, name))
        self._seq += 1

    def sleep(self, delay: float) -> Future:
        fut = Future()
        self.schedule(delay, lambda: fut.resolve(None), name="sleep")
        return fut

    def _fire_due(self) -> None:
        now = self.now
        while self._heap and self._heap[0][0] <= now:
            _, _, action, name = heapq.heappop(self._heap)
            try:
                action()
            except Exception as exc:
                exc.add_note(f"while firing timer {name!r}")
                raise

    def run_until_idle(self, max_steps: int | None = None, deadline: float | None = None) -> float:
        rt = self.runtime
        while True:
            self._fire_due()
            if max_steps is not None and self.steps >= max_steps:
                break
            if deadline is not None and self.now >= deadline:
                break
            if rt is not None and rt.busy():
                emitted = rt.step()
                self.steps += 1
                if self.on_step is not None:
                    self.on_step(self.steps, emitted)
                continue
            if not self._heap:
                break
            wait = self._heap[0][0] - self.now
            if wait > 0:
                time.sleep(min(wait, 0.05))
        return self.now
