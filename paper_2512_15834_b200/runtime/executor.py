"""Per-sequence device state and the two ways phases reach the GPU.

State of a resident sequence:
  kv_len   physical KV rows written for it in the paged pool;
  pend     the last sampled token id, not yet fed (its KV row is written
           lazily by the next forward), or None;
  counted  whether `pend` is already emitted, i.e. counted in the
           reference's `kv_tokens` (engine.py:285,313,335).
Invariant: reference kv_tokens == kv_len + (1 if pend is counted else 0), and
the pool holds ceil(kv_tokens / 16) blocks for the slot between phases, so
block tables are a pure function of the reference's KV accounting.

Phase work (what each reference charge becomes):
  prefill  feed prompt ids [cached, P) -> sample the turn's first token (uncounted)
  emit     n tokens: an uncounted pend is emitted for free, every other token
           is one decode step (feed pend, sample the next scripted token)
  verify   one append-prefill over [pend?] + draft -> sampled ids at every
           draft position -> K4 LCP -> rollback (truncate) of rejected rows
  ingest   one append-prefill over [pend?] + tool-output ids, in place
  evict    truncate to the retained prefix (prefix cache) or release

`EagerRuntime` runs each phase to completion immediately, one sequence per
forward (virtual-time parity mode). `BatchRuntime` queues phases as jobs and
`step()` packs every runnable job of every resident sequence into one forward
(wall-clock continuous batching; decode jobs advance one token per step).
"""

from __future__ import annotations

import ctypes as C
from collections import deque
from dataclasses import dataclass, field

import numpy as np
import torch

from ..errors import ConfigError, KernelError
from ..modelcfg import TINY, ModelShape
from ..tokens import SALT_OUTPUT, SALT_PROMPT, TokenTable, fill_ids
from . import lib
from . import weights as W
from .decoder import Decoder, KVPool, StepBatch

BLOCK = 16


@dataclass
class SeqDev:
    slot: int
    kv_len: int = 0
    pend: int | None = None
    counted: bool = False
    hist: list[int] = field(default_factory=list)  # id fed at each physical row
    replay: list[int] = field(default_factory=list)

    @property
    def kv_tokens(self) -> int:
        return self.kv_len + (1 if (self.pend is not None and self.counted) else 0)


def _turn_first(seq, turn: int, table: TokenTable) -> int:
    turns = seq.script.turns
    if turn < len(turns) and turns[turn]:
        return table.intern(turns[turn][0])
    return -1


# ------------------------------------------------------------------- jobs

class Run:
    """A contiguous run of input ids appended at `start`; samples some rows."""

    __slots__ = ("seq", "ids", "start", "rows", "targets", "on_done")

    def __init__(self, seq, ids: list[int], start: int, rows: list[int], targets: list[int], on_done):
        self.seq, self.ids, self.start = seq, ids, start
        self.rows, self.targets, self.on_done = rows, targets, on_done


class Decode:
    """Emit `targets` one decode step at a time."""

    __slots__ = ("seq", "targets", "k", "on_done")

    def __init__(self, seq, targets: list[int], on_done):
        self.seq, self.targets, self.k, self.on_done = seq, targets, 0, on_done


class Runtime:
    """Common state machine; subclasses decide when forwards run."""

    def __init__(self, shape: ModelShape, *, seed: int = 0, num_blocks: int = 4096, max_slots: int = 1024,
                 max_ctx: int = 8192, init_device: str = "cpu", weights: dict | None = None,
                 record: bool = False):
        lib.load()
        self.shape = shape
        self.seed = seed
        self.table = TokenTable(shape.vocab)
        self.pool = KVPool(shape, num_blocks, max_slots, (max_ctx + BLOCK - 1) // BLOCK)
        self.w = weights if weights is not None else W.build(shape, seed, init_device=init_device)
        self.dec = Decoder(shape, self.w, self.pool)
        self.max_ctx = max_ctx
        self._free_slots = list(range(max_slots - 1, -1, -1))
        self.record = record
        self.trace: list[dict] = []     # per forward row: rid, pos, target, sampled, logits (if record)
        self.forwards = 0
        self.tokens_fed = 0
        self.emitted = 0                # tokens sampled and counted (reference kv_tokens += ...)
        self.h2d_bytes = 0              # per-step metadata uploads (ids, positions, tables, drafts)
        self.d2h_bytes = 0              # sampled ids / validation results read back

    # -- vocabulary ------------------------------------------------------------

    def intern(self, toks) -> list[int]:
        return self.table.ids(toks)

    # -- slots / blocks ----------------------------------------------------------

    def open(self, seq) -> None:
        for turn in seq.script.turns:
            self.table.ids(turn)
        if not self._free_slots:
            raise ConfigError("no free KV slot rows")
        seq.dev = SeqDev(self._free_slots.pop())

    def close(self, seq) -> None:
        d = seq.dev
        self.pool.release(d.slot)
        self._free_slots.append(d.slot)
        d.kv_len, d.pend, d.counted, d.hist = 0, None, False, []

    def can_admit(self, seq) -> bool:
        need = -(-(seq.prompt_tokens + 1) // BLOCK)
        return self.pool.free_blocks() >= need

    def _commit_blocks(self, d: SeqDev) -> None:
        """Hold exactly ceil(kv_tokens / 16) blocks (rollback / growth)."""
        self.pool.truncate(d.slot, d.kv_tokens)
        self.pool.reserve(d.slot, d.kv_tokens)

    def block_ids(self, seq) -> list[int]:
        return self.pool.blocks(seq.dev.slot)

    def precapture(self, max_batch: int) -> None:
        """Capture the decode-step CUDA graphs for B = 1..max_batch up front (timed and
        untimed variants) against a scratch slot, so no capture lands in a timed run."""
        scratch = self._free_slots.pop(0)  # highest slot id: the last one handed out
        self.pool.reserve(scratch, 16)
        z = np.zeros
        for B in range(1, max_batch + 1):
            one = np.full(B, scratch, dtype=np.int32)
            batch = StepBatch(z(B, np.int32), z(B, np.int32), one, one, np.ones(B, np.int32), z(0, np.int32),
                              z(1, np.int32), z(0, np.int32), np.arange(B, dtype=np.int32), np.full(B, -1, np.int32))
            saved = self.dec.timers
            for timers in (None, {}):
                self.dec.timers = timers
                self.dec.forward(batch)
                torch.cuda.synchronize()
                self.dec.collect()
            self.dec.timers = saved
        self.pool.release(scratch)
        self._free_slots.insert(0, scratch)

    # -- phase entry points (called by B200Engine) ------------------------------

    def prefill(self, seq, cached: int, next_turn: int, done) -> None:
        d = seq.dev
        P = seq.prompt_tokens
        if P < 1:
            raise ConfigError("the B200 engine needs prompt_tokens >= 1")
        if d.kv_len != cached:
            # vanilla re-prefill (cached == 0) or a resubmit that drops retained rows
            d.kv_len = min(d.kv_len, cached)
            self.pool.truncate(d.slot, d.kv_len)
        ids = self._prompt_ids(seq, P)
        d.pend, d.counted = None, False
        start = cached
        if start >= P:  # nothing new: recompute the last row to get next-token logits
            start = P - 1
            d.kv_len = P - 1
        run_ids = ids[start:P]
        target = _turn_first(seq, next_turn, self.table)

        def finish(sampled: list[int]) -> None:
            d.pend, d.counted = sampled[-1], False
            self._commit_blocks(d)
            done(None)

        self._submit_run(Run(seq, run_ids, start, [len(run_ids) - 1], [target], finish))

    def emit(self, seq, tokens, done) -> None:
        d = seq.dev
        targets = self.table.ids(tokens)
        if not targets:
            done(None)
            return
        k = 0
        if d.pend is not None and not d.counted:
            if d.pend != targets[0]:
                raise KernelError(f"{seq.rid}: sampled {d.pend} but the script says {targets[0]}")
            d.counted = True
            k = 1
            self.emitted += 1
            self._commit_blocks(d)
        if k == len(targets):
            done(None)
            return
        if d.pend is None:  # nothing to feed: recompute the last row first
            self._recompute_last(seq)
        self._submit_decode(Decode(seq, targets[k:], lambda: done(None)))

    def verify(self, seq, draft_tokens, span_tokens, done) -> None:
        d = seq.dev
        draft = self.table.ids(draft_tokens)
        span = self.table.ids(span_tokens)
        if d.pend is None:
            self._recompute_last(seq)
        lead = [d.pend] if d.counted else []
        inputs = lead + draft
        # row j predicts the token after inputs[j]; the model's token for draft slot i
        # is pend (uncounted case, i == 0) or the sample of the row feeding slot i-1
        off = 0 if d.counted else 1
        targets = [span[j + off] if j + off < len(span) else -1 for j in range(len(inputs))]
        rows = list(range(len(inputs)))
        pend_uncounted = None if d.counted else d.pend

        def finish(sampled: list[int], dev_sampled: torch.Tensor) -> None:
            model = ([pend_uncounted] if pend_uncounted is not None else []) + sampled
            accepted, consume, new_len = self._validate(d, draft, model, len(span), len(lead), dev_sampled,
                                                        pend_uncounted)
            valid = len(lead) + accepted
            d.kv_len = d.kv_len - len(inputs) + valid  # kv_len was advanced by the whole run
            assert d.kv_len == new_len, (d.kv_len, new_len)
            del d.hist[len(d.hist) - (len(inputs) - valid):]
            if accepted < len(span):
                d.pend, d.counted = model[accepted], True
            else:
                d.pend, d.counted = None, False
            self._commit_blocks(d)  # K1 rollback of the rejected rows' blocks
            self.emitted += consume
            done((accepted, consume))

        self._submit_run(Run(seq, inputs, d.kv_len, rows, targets, finish), want_device=True)

    def ingest(self, seq, n_out: int, next_turn: int, done) -> None:
        d = seq.dev
        if d.pend is not None and not d.counted:
            raise KernelError(f"{seq.rid}: ingest with an unemitted sampled token")
        if d.pend is None and n_out == 0:
            self._recompute_last(seq)
        lead = [d.pend] if d.pend is not None else []
        out = fill_ids(self.seed, seq.rid, SALT_OUTPUT, d.kv_len + len(lead), n_out, self.shape.vocab).tolist()
        inputs = lead + out
        target = _turn_first(seq, next_turn, self.table)

        def finish(sampled: list[int]) -> None:
            d.pend, d.counted = sampled[-1], False
            self._commit_blocks(d)
            done(None)

        self._submit_run(Run(seq, inputs, d.kv_len, [len(inputs) - 1], [target], finish))

    def evict(self, seq, keep: int) -> None:
        d = seq.dev
        d.kv_len = min(d.kv_len, keep)
        d.pend, d.counted = None, False
        del d.hist[seq.turn_base:]
        d.replay = self.table.ids(seq.replay)
        if keep == 0:
            self.pool.release(d.slot)
        else:
            self.pool.truncate(d.slot, keep)

    # -- helpers -----------------------------------------------------------------

    def _prompt_ids(self, seq, P: int) -> list[int]:
        d = seq.dev
        ids = list(d.hist[:P])
        if len(ids) < P:
            ids += d.replay[: P - len(ids)]
        if len(ids) < P:
            salt = SALT_OUTPUT if d.replay else SALT_PROMPT
            ids += fill_ids(self.seed, seq.rid, salt, len(ids), P - len(ids), self.shape.vocab).tolist()
        d.replay = []
        return ids

    def _recompute_last(self, seq) -> None:
        """No pending token: un-feed the last written row so the next forward
        re-feeds it (same KV row, identical values) and yields next-token logits."""
        d = seq.dev
        if d.kv_len < 1:
            raise KernelError(f"{seq.rid}: no context to decode from")
        d.kv_len -= 1
        d.pend, d.counted = d.hist.pop(), True

    def _validate(self, d, draft, model, span_len, lead, dev_sampled, pend_uncounted):
        """K4 on the device: LCP(draft, model ids) clamped to the span."""
        dev = self.dec.device
        draft_t = torch.tensor(draft if draft else [0], dtype=torch.int32, device=dev)[: len(draft)]
        if pend_uncounted is not None:
            model_t = torch.cat([torch.tensor([pend_uncounted], dtype=torch.int32, device=dev), dev_sampled])
        else:
            model_t = dev_sampled
        meta = torch.tensor([0, len(draft), 0, int(model_t.shape[0]), span_len, d.kv_len - len(draft) - lead, lead],
                            dtype=torch.int32, device=dev)
        out = torch.empty(3, dtype=torch.int32, device=dev)
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        lib.call("stb_spec_validate", p(draft_t), p(meta[0:2]), p(model_t), p(meta[2:4]), p(meta[4:5]),
                 p(meta[5:6]), p(meta[6:7]), 1, p(out[0:1]), p(out[1:2]), p(out[2:3]), st)
        a, c, n = out.tolist()
        self.h2d_bytes += 4 * (len(draft) + 7)
        self.d2h_bytes += 12
        return a, c, n

    # -- forward plumbing ----------------------------------------------------------

    def _build(self, decodes: list[Decode], runs: list[Run]) -> StepBatch:
        ids, pos, slot_of = [], [], []
        dec_slots, dec_ctx = [], []
        for j in decodes:
            d = j.seq.dev
            ids.append(d.pend)
            pos.append(d.kv_len)
            slot_of.append(d.slot)
            dec_slots.append(d.slot)
            dec_ctx.append(d.kv_len + 1)
        pre_slots, qstart, pre_ctx = [], [0], []
        sample_rows, targets = list(range(len(decodes))), [j.targets[j.k] for j in decodes]
        base = len(decodes)
        for r in runs:
            d = r.seq.dev
            n = len(r.ids)
            ids.extend(r.ids)
            pos.extend(range(r.start, r.start + n))
            slot_of.extend([d.slot] * n)
            pre_slots.append(d.slot)
            pre_ctx.append(r.start + n)
            sample_rows.extend(base + qstart[-1] + x for x in r.rows)
            targets.extend(r.targets)
            qstart.append(qstart[-1] + n)
        a = lambda v: np.asarray(v, dtype=np.int32)  # noqa: E731
        return StepBatch(a(ids), a(pos), a(slot_of), a(dec_slots), a(dec_ctx), a(pre_slots), a(qstart),
                         a(pre_ctx), a(sample_rows), a(targets))

    def _run_now(self, runs: list[Run], decodes: list[Decode] = (), want_device: bool = False):
        """One forward over `decodes` (one token each) + `runs`; applies results."""
        decodes = list(decodes)
        for j in decodes:
            d = j.seq.dev
            self.pool.reserve(d.slot, d.kv_len + 1)
        for r in runs:
            d = r.seq.dev
            if r.start + len(r.ids) > self.max_ctx:
                raise ConfigError(f"{r.seq.rid}: context {r.start + len(r.ids)} exceeds max_ctx {self.max_ctx}")
            self.pool.reserve(d.slot, r.start + len(r.ids))
        batch = self._build(decodes, runs)
        self.dec.keep_logits = self.record
        sampled_dev = self.dec.forward(batch)
        sampled = sampled_dev.tolist()
        self.dec.collect()
        self.h2d_bytes += self.dec.h2d_bytes
        self.d2h_bytes += 4 * batch.R
        self.forwards += 1
        self.tokens_fed += batch.T
        if self.record:
            logits = self.dec.last_logits.float().cpu()
            raw = self.dec.last_raw_argmax.cpu().tolist()
            for i in range(batch.R):
                row = int(batch.sample_rows[i])
                seq = (decodes[row].seq if row < len(decodes) else None)
                if seq is None:
                    acc = len(decodes)
                    for r in runs:
                        if row < acc + len(r.ids):
                            seq = r.seq
                            break
                        acc += len(r.ids)
                self.trace.append({"rid": seq.rid, "pos": int(batch.pos[row]), "fed": int(batch.ids[row]),
                                   "target": int(batch.targets[i]), "sampled": sampled[i], "raw_argmax": raw[i],
                                   "logits": logits[i]})
        # apply decode results
        for i, j in enumerate(decodes):
            d = j.seq.dev
            got, want = sampled[i], j.targets[j.k]
            if want >= 0 and got != want:
                raise KernelError(f"{j.seq.rid}: forced sample {got} != scripted {want}")
            del d.hist[d.kv_len:]
            d.hist.append(d.pend)
            d.kv_len += 1
            d.pend, d.counted = got, True
            j.k += 1
        self.emitted += len(decodes)
        off = len(decodes)
        results = []
        for r in runs:
            d = r.seq.dev
            del d.hist[r.start:]
            d.hist.extend(r.ids)
            d.kv_len = r.start + len(r.ids)
            got = sampled[off:off + len(r.rows)]
            for g, t in zip(got, r.targets):
                if t >= 0 and g != t:
                    raise KernelError(f"{r.seq.rid}: forced sample {g} != scripted {t}")
            results.append((r, got, sampled_dev[off:off + len(r.rows)] if want_device else None))
            off += len(r.rows)
        return results

    def _submit_run(self, run: Run, want_device: bool = False) -> None:
        raise NotImplementedError

    def _submit_decode(self, job: Decode) -> None:
        raise NotImplementedError


class EagerRuntime(Runtime):
    """Parity mode: each phase runs to completion now, batch of one."""

    def _submit_run(self, run: Run, want_device: bool = False) -> None:
        ((r, got, dev),) = self._run_now([run], want_device=want_device)
        if want_device:
            r.on_done(got, dev)
        else:
            r.on_done(got)

    def _submit_decode(self, job: Decode) -> None:
        while job.k < len(job.targets):
            d = job.seq.dev
            self._run_now([], [job])
            self._commit_blocks(d)
        job.on_done()


class BatchRuntime(Runtime):
    """Throughput mode: jobs queue up; `step()` runs one packed forward."""

    def __init__(self, *a, max_step_tokens: int = 8192, **kw):
        super().__init__(*a, **kw)
        self.max_step_tokens = max_step_tokens
        self.runs: deque = deque()
        self.decodes: list[Decode] = []
        self.step_tokens_emitted = 0

    def _submit_run(self, run: Run, want_device: bool = False) -> None:
        self.runs.append((run, want_device))

    def _submit_decode(self, job: Decode) -> None:
        self.decodes.append(job)

    def busy(self) -> bool:
        return bool(self.runs or self.decodes)

    def step(self) -> int:
        """One packed forward over every decode job + as many runs as fit."""
        decodes = list(self.decodes)
        budget = self.max_step_tokens - len(decodes)
        runs = []
        while self.runs and (not runs or len(self.runs[0][0].ids) <= budget):
            r, wd = self.runs.popleft()
            budget -= len(r.ids)
            runs.append((r, wd))
        if not decodes and not runs:
            return 0
        want = any(wd for _, wd in runs)
        results = self._run_now([r for r, _ in runs], decodes, want_device=want)
        emitted = len(decodes)
        self.decodes = []
        for j in decodes:
            self._commit_blocks(j.seq.dev)
            if j.k < len(j.targets):
                self.decodes.append(j)
        for j in decodes:
            if j.k >= len(j.targets):
                j.on_done()
        for (r, got, dev), (_, wd) in zip(results, runs):
            if wd:
                r.on_done(got, dev)
            else:
                r.on_done(got)
        return emitted


def default_runtime(config, shape: ModelShape = TINY, **kw) -> Runtime:
    """The runtime `B200Engine(sim, config)` builds: tiny C1 decoder, eager."""
    nb = config.num_blocks or 4096
    return EagerRuntime(shape, num_blocks=nb, **kw)
