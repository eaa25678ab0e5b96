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
           draft position -> K4 LCP on the device -> rollback (truncate) of the
           rejected rows' blocks
  ingest   one append-prefill over [pend?] + tool-output ids, in place
  evict    truncate to the retained prefix (prefix cache) or release

Every forward is a *flight*: `_launch` packs the step, enqueues the forward,
the K4 validation of its verify runs and one async D2H of the sampled ids
(+ K4 results) into pinned memory; `_complete` waits for that copy, checks
every forced sample against its script target and fires the phase
callbacks. `EagerRuntime` completes each flight at once (virtual-time parity
mode, one sequence per forward). `BatchRuntime` keeps one flight in the air:
decode tokens advance optimistically at launch (their targets are the
script; the completion check raises on any mismatch), so step k+1 is packed
and launched while step k runs; a sequence with a run in flight (prefill /
verify / ingest) sits out until that run completes.
"""

from __future__ import annotations

import ctypes as C
from collections import deque
from dataclasses import dataclass, field

import numpy as np
import torch

from ..errors import ConfigError, KernelError, KVCapacityError
from ..modelcfg import TINY, ModelShape
from ..tokens import SALT_OUTPUT, SALT_PROMPT, TokenTable, fill_ids, output_ids
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
    busy: bool = False                              # a run of this sequence is in flight
    spilled: int = 0                                # rows dropped by a KV preemption (recomputed on restore)

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
    """A contiguous run of input ids appended at `start`; samples some rows.

    With `verify` = (draft ids, span_len, lead, model_first) the run is a
    validation pass: K4 compares the draft with the model's ids (model_first
    if >= 0, then the sampled rows) and `on_done` receives
    (accepted, consume, new_len, sampled rows)."""

    __slots__ = ("seq", "ids", "start", "rows", "targets", "on_done", "verify")

    def __init__(self, seq, ids, start, rows, targets, on_done, verify=None):
        self.seq, self.ids, self.start = seq, ids, start
        self.rows, self.targets, self.on_done, self.verify = rows, targets, on_done, verify


class Decode:
    """Emit `targets` one decode step at a time."""

    __slots__ = ("seq", "targets", "k", "on_done")

    def __init__(self, seq, targets: list[int], on_done):
        self.seq, self.targets, self.k, self.on_done = seq, targets, 0, on_done


class Flight:
    __slots__ = ("batch", "decodes", "runs", "event", "host", "n_sampled", "n_verify", "logits", "raw", "finished",
                 "timers", "routes")


class Runtime:
    """Common state machine; subclasses decide when flights complete."""

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
        self.reclaimer = None           # engine hook: free retained prefixes under KV pressure
        self.trace: list[dict] = []     # per sampled row: rid, pos, fed, target, sampled, logits (record mode)
        # record mode, per completed flight: every fed run (rid, start, ids, sampled local rows) with the
        # sampled rows' logits / raw argmax, and the block list of every sequence it touched
        self.flights: list[dict] = []
        if record:
            self.pool.log = []
        self.forwards = 0
        self.tokens_fed = 0
        self.emitted = 0                # tokens sampled and counted (reference kv_tokens += ...)
        self.h2d_bytes = 0              # per-step metadata uploads (ids, positions, tables, drafts)
        self.d2h_bytes = 0              # sampled ids / validation results read back
        # double-buffered pinned results (one flight may be in the air) + K4 staging
        self._host = [torch.empty(1 << 16, dtype=torch.int32, pin_memory=True) for _ in range(2)]
        self._vstage = [torch.empty(1 << 16, dtype=torch.int32, pin_memory=True) for _ in range(2)]
        self._host_ev: list = [None, None]
        self._flip = 0
        self._vdev = torch.empty(1 << 16, dtype=torch.int32, device="cuda")   # K4 inputs
        self._vout = torch.empty(3 * 4096, dtype=torch.int32, device="cuda")  # K4 outputs

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
        """Blocks the prompt still needs (ceil((P + 1) / 16) minus what the slot already
        holds, e.g. a retained prefix) fit in the free list."""
        need = -(-(seq.prompt_tokens + 1) // BLOCK) - len(self.pool.blocks(seq.dev.slot))
        return self.pool.free_blocks() >= need

    def _reserve(self, slot: int, n: int) -> None:
        """pool.reserve; on KV exhaustion ask the engine to drop paused sequences' retained
        prefixes (`reclaimer`) and retry once before giving up."""
        try:
            self.pool.reserve(slot, n)
        except KVCapacityError:
            if self.reclaimer is None or not self.reclaimer():
                raise
            self.pool.reserve(slot, n)

    def _commit_blocks(self, d: SeqDev) -> None:
        """Hold exactly ceil(kv_tokens / 16) blocks (rollback / growth)."""
        self.pool.truncate(d.slot, d.kv_tokens)
        self._reserve(d.slot, d.kv_tokens)

    def block_ids(self, seq) -> list[int]:
        return self.pool.blocks(seq.dev.slot)

    def precapture(self, max_batch: int) -> None:
        """Capture the decode-step CUDA graphs for B = 1..max_batch up front (timed and
        untimed variants) against a scratch slot, so no capture lands in a timed run."""
        # size the step buffers for the largest packed step up front: growing them later would
        # drop every captured graph (they point at the buffers) and recapture them mid-run
        cap_t = getattr(self, "max_step_tokens", 0) + max_batch + 64
        self.dec._ensure(cap_t, min(cap_t, 512), max(max_batch, 64))
        scratch = self._free_slots.pop(0)  # highest slot id: the last one handed out
        self.pool.reserve(scratch, 16)
        z = np.zeros
        for B in range(1, max_batch + 1):
            one = np.full(B, scratch, dtype=np.int32)
            batch = StepBatch(z(B, np.int32), z(B, np.int32), one, one, np.ones(B, np.int32), z(0, np.int32),
                              z(1, np.int32), z(0, np.int32), np.arange(B, dtype=np.int32), np.full(B, -1, np.int32))
            saved = self.dec.timers
            for timers in (None, {}, {}):  # untimed + both timed parities
                self.dec.timers = timers
                self.dec.forward(batch)
                torch.cuda.synchronize()
                self.dec.collect()
            self.dec.timers = saved
        # the mixed-step kernels (K2, its KV-split merge and split scratch, prefill-shaped GEMMs)
        # are loaded and their buffers sized here as well: the first verify pass of a run used
        # to pay the split scratch allocation and lazy module loads inside a timed step (~57 ms)
        self.pool.reserve(scratch, 320)
        for n in (33, 320):
            pos = np.arange(n, dtype=np.int32)
            batch = StepBatch(z(n, np.int32), pos, np.full(n, scratch, np.int32), z(0, np.int32), z(0, np.int32),
                              np.array([scratch], np.int32), np.array([0, n], np.int32), np.array([n], np.int32),
                              np.array([n - 1], np.int32), np.full(1, -1, np.int32))
            self.dec.forward(batch)
            torch.cuda.synchronize()
            self.dec.collect()
        self.pool.release(scratch)
        self._free_slots.insert(0, scratch)

    def probe_logits(self, ids: list[int], taps: list | None = None, routes: list | None = None) -> torch.Tensor:
        """Self-check (the bench's canary): prefill `ids` at positions 0.. on a scratch slot
        and return the fp32 logits of the last row (host). Leaves no state behind. `taps` (a
        list) receives the residual stream [n, d] (fp32, host) after the embedding and after
        every layer, for the per-layer teacher-forced check."""
        if self._host_ev[0] is not None or self._host_ev[1] is not None:
            torch.cuda.synchronize()
        slot = self._free_slots.pop(0)
        n = len(ids)
        try:
            self.pool.reserve(slot, n)
            z = np.zeros
            batch = StepBatch(np.asarray(ids, np.int32), np.arange(n, dtype=np.int32), np.full(n, slot, np.int32),
                              z(0, np.int32), z(0, np.int32), np.array([slot], np.int32), np.array([0, n], np.int32),
                              np.array([n], np.int32), np.array([n - 1], np.int32), np.full(1, -1, np.int32))
            keep = self.dec.keep_logits
            self.dec.keep_logits = True
            self.dec.taps = [] if taps is not None else None
            self.dec.route_log = [] if routes is not None else None
            try:
                self.dec.forward(batch)
                torch.cuda.synchronize()
            finally:
                if taps is not None:
                    taps.extend(t.float().cpu() for t in self.dec.taps)
                if routes is not None and self.dec.route_log:
                    routes.extend(r.view(n, -1).cpu().numpy() for r in self.dec.route_log)
                self.dec.taps = self.dec.route_log = None
            out = self.dec.last_logits[0].float().cpu()
            self.dec.keep_logits = keep
            self.dec.collect()
        finally:
            self.pool.release(slot)
            self._free_slots.insert(0, slot)
        return out

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
        draft = self.table.lookup(draft_tokens)   # compare ids: never interned (UNKNOWN = -2)
        span = self.table.ids(span_tokens)
        if d.pend is None:
            self._recompute_last(seq)
        lead = [d.pend] if d.counted else []
        inputs = lead + self.table.feed(draft_tokens)
        # row j predicts the token after inputs[j]; the model's token for draft slot i
        # is pend (uncounted case, i == 0) or the sample of the row feeding slot i-1
        off = 0 if d.counted else 1
        targets = [span[j + off] if j + off < len(span) else -1 for j in range(len(inputs))]
        first = -1 if d.counted else d.pend
        start = d.kv_len

        def finish(res) -> None:
            accepted, consume, new_len, rows = res
            if new_len != start + len(lead) + accepted:
                raise KernelError(f"{seq.rid}: K4 kept {new_len} rows, expected {start + len(lead) + accepted}")
            d.kv_len = new_len
            del d.hist[new_len:]
            if accepted < len(span):
                model = ([first] if first >= 0 else []) + rows
                d.pend, d.counted = model[accepted], True  # the correction token, emitted
            else:
                d.pend, d.counted = None, False
            self._commit_blocks(d)  # K1 rollback of the rejected rows' blocks
            self.emitted += consume
            done((accepted, consume))

        self._submit_run(Run(seq, inputs, start, list(range(len(inputs))), targets, finish,
                             verify=(draft, len(span), len(lead), first)))

    def ingest(self, seq, n_out: int, next_turn: int, done, output: str | None = None) -> None:
        d = seq.dev
        if d.pend is not None and not d.counted:
            raise KernelError(f"{seq.rid}: ingest with an unemitted sampled token")
        if d.pend is None and n_out == 0:
            self._recompute_last(seq)
        lead = [d.pend] if d.pend is not None else []
        # the output's own text becomes its token ids (tokens.output_ids)
        out = output_ids(self.seed, seq.rid, output, d.kv_len + len(lead), n_out, self.shape.vocab).tolist()
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

    # -- flights -----------------------------------------------------------------

    def _build(self, decodes: list[Decode], runs: list[Run]) -> StepBatch:
        nd = len(decodes)
        ids = [j.seq.dev.pend for j in decodes]
        pos = [j.seq.dev.kv_len for j in decodes]
        slots = [j.seq.dev.slot for j in decodes]
        ctx = [p + 1 for p in pos]
        targets = [j.targets[j.k] for j in decodes]
        slot_of = list(slots)
        pre_slots, qstart, pre_ctx = [], [0], []
        sample_rows = list(range(nd))
        for r in runs:
            d = r.seq.dev
            n = len(r.ids)
            ids.extend(r.ids)
            pos.extend(range(r.start, r.start + n))
            slot_of.extend([d.slot] * n)
            pre_slots.append(d.slot)
            pre_ctx.append(r.start + n)
            base = nd + qstart[-1]
            sample_rows.extend(base + x for x in r.rows)
            targets.extend(r.targets)
            qstart.append(qstart[-1] + n)
        a = lambda v: np.asarray(v, dtype=np.int32)  # noqa: E731
        return StepBatch(a(ids), a(pos), a(slot_of), a(slots), a(ctx), a(pre_slots), a(qstart), a(pre_ctx),
                         a(sample_rows), a(targets))

    def _launch(self, runs: list[Run], decodes=()) -> Flight:
        """Pack and enqueue one forward (+ K4, + D2H); advance decode rows optimistically."""
        decodes = list(decodes)
        runs = sorted(runs, key=lambda r: r.verify is None)  # verify runs first: their samples are contiguous
        for j in decodes:
            d = j.seq.dev
            self._reserve(d.slot, d.kv_len + 1)
        for r in runs:
            d = r.seq.dev
            if r.start + len(r.ids) > self.max_ctx:
                raise ConfigError(f"{r.seq.rid}: context {r.start + len(r.ids)} exceeds max_ctx {self.max_ctx}")
            self._reserve(d.slot, r.start + len(r.ids))
        batch = self._build(decodes, runs)
        self.dec.keep_logits = self.record
        self.dec.route_log = [] if (self.record and self.shape.moe) else None
        k = self._flip
        self._flip ^= 1
        if self._host_ev[k] is not None:  # the pinned buffers of two flights ago are free again
            self._host_ev[k].synchronize()
        sampled = self.dec.forward(batch)
        R = batch.R
        nv = self._launch_validate(decodes, runs, sampled, k)
        host = self._host[k]
        host[:R].copy_(sampled, non_blocking=True)
        if nv:
            host[R:R + 3 * nv].copy_(self._vout[:3 * nv], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._host_ev[k] = ev
        f = Flight()
        f.batch, f.decodes, f.runs, f.n_sampled, f.n_verify = batch, decodes, runs, R, nv
        f.event, f.host, f.finished = ev, host, []
        f.timers = (self.dec.take_pending(), self.dec.timers)
        f.logits = self.dec.last_logits if self.record else None
        f.raw = self.dec.last_raw_argmax if self.record else None
        f.routes, self.dec.route_log = self.dec.route_log, None
        self.h2d_bytes += self.dec.h2d_bytes
        self.d2h_bytes += 4 * (R + 3 * nv)
        self.forwards += 1
        self.tokens_fed += batch.T
        # optimistic state: decode rows take their scripted target, checked at completion
        for j in decodes:
            d = j.seq.dev
            del d.hist[d.kv_len:]
            d.hist.append(d.pend)
            d.kv_len += 1
            d.pend, d.counted = j.targets[j.k], True
            j.k += 1
        self.emitted += len(decodes)
        for r in runs:
            d = r.seq.dev
            del d.hist[r.start:]
            d.hist.extend(r.ids)
            d.kv_len = r.start + len(r.ids)
            d.busy = True
        return f

    def _launch_validate(self, decodes, runs, sampled: torch.Tensor, k: int) -> int:
        """K4 for the flight's verify runs (the first runs), on the device, after the forward."""
        vr = [r for r in runs if r.verify is not None]
        if not vr:
            return 0
        nv = len(vr)
        drafts, d_off, m_off, firsts, spans, kvs, extra = [], [0], [len(decodes)], [], [], [], []
        for r in vr:
            draft, span_len, lead, first = r.verify
            drafts.extend(draft)
            d_off.append(len(drafts))
            m_off.append(m_off[-1] + len(r.rows))
            firsts.append(first)
            spans.append(span_len)
            kvs.append(r.start)
            extra.append(lead)
        parts = [drafts, d_off, m_off, firsts, spans, kvs, extra]
        host = self._vstage[k].numpy()
        offs, o = [], 0
        for p in parts:
            offs.append(o)
            host[o:o + len(p)] = p
            o += len(p)
        self._vdev[:o].copy_(self._vstage[k][:o], non_blocking=True)
        base = self._vdev.data_ptr()
        ptr = [C.c_void_p(base + 4 * x) for x in offs]
        out = self._vout.data_ptr()
        lib.call("stb_spec_validate", ptr[0], ptr[1], C.c_void_p(sampled.data_ptr()), ptr[2], ptr[3], ptr[4],
                 ptr[5], ptr[6], nv, C.c_void_p(out), C.c_void_p(out + 4 * nv), C.c_void_p(out + 8 * nv),
                 C.c_void_p(torch.cuda.current_stream().cuda_stream))
        self.h2d_bytes += 4 * o
        return nv

    def _complete(self, f: Flight) -> None:
        """Wait for the flight's results, check every forced sample, fire callbacks."""
        f.event.synchronize()
        R, nv = f.n_sampled, f.n_verify
        sampled = f.host[:R].tolist()
        vres = f.host[R:R + 3 * nv].tolist() if nv else []
        self.dec.fold(*f.timers)
        b = f.batch
        if self.record:
            logits = f.logits.float().cpu()
            raw = f.raw.cpu().tolist()
            owners = [j.seq for j in f.decodes]
            for r in f.runs:
                owners.extend([r.seq] * len(r.ids))
            items = [(j.seq.rid, int(b.pos[i]), [int(b.ids[i])], [0]) for i, j in enumerate(f.decodes)]
            off = len(f.decodes)
            for r in f.runs:
                items.append((r.seq.rid, r.start, list(r.ids), list(r.rows)))
                off += len(r.ids)
            slots = {j.seq.rid: j.seq.dev.slot for j in f.decodes}
            slots.update({r.seq.rid: r.seq.dev.slot for r in f.runs})
            # MoE: each layer's expert ids [T, k] of the step (row order = the items' order)
            routes = [r.view(b.T, -1).cpu().numpy() for r in f.routes] if f.routes else None
            self.flights.append({"items": items, "logits": logits, "raw": raw, "sampled": list(sampled),
                                 "pool_ops": len(self.pool.log), "slots": slots, "routes": routes,
                                 "tables": {rid: self.pool.blocks(sl) for rid, sl in slots.items()}})
            for i in range(R):
                row = int(b.sample_rows[i])
                self.trace.append({"rid": owners[row].rid, "pos": int(b.pos[row]), "fed": int(b.ids[row]),
                                   "target": int(b.targets[i]), "sampled": sampled[i], "raw_argmax": raw[i],
                                   "logits": logits[i]})
        for i, j in enumerate(f.decodes):
            want = int(b.targets[i])
            if want >= 0 and sampled[i] != want:
                raise KernelError(f"{j.seq.rid}: forced sample {sampled[i]} != scripted {want}")
        off, kv = len(f.decodes), 0
        done_runs = []
        for r in f.runs:
            got = sampled[off:off + len(r.rows)]
            for g, t in zip(got, r.targets):
                if t >= 0 and g != t:
                    raise KernelError(f"{r.seq.rid}: forced sample {g} != scripted {t}")
            r.seq.dev.busy = False
            if r.verify is not None:
                done_runs.append((r, (vres[kv], vres[nv + kv], vres[2 * nv + kv], got)))
                kv += 1
            else:
                done_runs.append((r, got))
            off += len(r.rows)
        for j in f.finished:
            j.on_done()
        for r, res in done_runs:
            r.on_done(res)

    def _submit_run(self, run: Run) -> None:
        raise NotImplementedError

    def _submit_decode(self, job: Decode) -> None:
        raise NotImplementedError


class EagerRuntime(Runtime):
    """Parity mode: each phase runs to completion now, batch of one."""

    def _submit_run(self, run: Run) -> None:
        self._complete(self._launch([run]))

    def _submit_decode(self, job: Decode) -> None:
        while job.k < len(job.targets):
            f = self._launch([], [job])
            self._commit_blocks(job.seq.dev)
            self._complete(f)
        job.on_done()


class BatchRuntime(Runtime):
    """Throughput mode: jobs queue up; `step()` launches one packed forward and then
    completes the previous one (one flight in the air)."""

    def __init__(self, *a, max_step_tokens: int = 8192, pipeline: bool = True, **kw):
        super().__init__(*a, **kw)
        self.max_step_tokens = max_step_tokens
        self.pipeline = pipeline
        self.runs: deque = deque()
        self.decodes: list[Decode] = []
        self.flight: Flight | None = None
        # KV preemption (the pool is finite, the reference's is not: SPEC.md:521): decode jobs
        # whose sequence was spilled to free blocks, restored FIFO by recomputing its rows
        self.spilled: deque = deque()
        self._in_step: set = set()  # slots of the step being packed (never preempted mid-launch)
        self.spills = 0        # sequences preempted
        self._prev_in_air = False  # step(): a packed forward is still in flight while this one packs
        self.deferred = 0      # steps that held a prefill / ingest run back for lack of blocks

    def _submit_run(self, run: Run) -> None:
        self.runs.append(run)

    def _submit_decode(self, job: Decode) -> None:
        self.decodes.append(job)

    def busy(self) -> bool:
        return bool(self.runs or self.decodes or self.spilled or self.flight is not None)

    def _pack(self):
        self._restore()
        decodes = [j for j in self.decodes if not j.seq.dev.busy]
        budget = self.max_step_tokens - len(decodes)
        runs = []
        while self.runs and (not runs or len(self.runs[0].ids) <= budget):
            r = self.runs.popleft()
            budget -= len(r.ids)
            runs.append(r)
        free = self.pool.free_blocks()
        if free < 2 * (len(decodes) + sum(-(-len(r.ids) // BLOCK) + 1 for r in runs)):  # cheap guard
            decodes, runs = self._fit(decodes, runs, free)
        return decodes, runs

    # -- KV pressure -------------------------------------------------------------

    def _need(self, decodes, runs) -> int:
        """Blocks the step adds: decode rows (+ the pending token the reference counts, H4) and
        every run's rows, beyond what each slot already holds."""
        need = 0
        for j in decodes:
            d = j.seq.dev
            need += max(0, -(-(d.kv_len + 2) // BLOCK) - len(self.pool.blocks(d.slot)))
        for r in runs:
            d = r.seq.dev
            need += max(0, -(-(r.start + len(r.ids) + 1) // BLOCK) - len(self.pool.blocks(d.slot)))
        return need

    def _fit(self, decodes, runs, free):
        """Make the step fit the free blocks: drop retained prefixes (engine reclaimer), hold
        prefill / ingest runs back (they wait in the queue), then preempt decoding sequences —
        largest context first — whose rows are recomputed when blocks return (`_restore`)."""
        need = self._need(decodes, runs)
        if need <= free:
            return decodes, runs
        if self.reclaimer is not None and self.reclaimer():
            free = self.pool.free_blocks()
        while need > free and runs and (decodes or len(runs) > 1):
            self.runs.appendleft(runs.pop())
            self.deferred += 1
            need = self._need(decodes, runs)
        while need > free and len(decodes) + len(runs) > 1 and decodes:
            victim = max(decodes, key=lambda j: j.seq.dev.kv_len)
            decodes.remove(victim)
            self._spill(victim)
            free = self.pool.free_blocks()
            need = self._need(decodes, runs)
        if need > free and self._prev_in_air:
            # the blocks still missing sit with the sequences of the step in the air (busy, so not
            # preemptible now): launch nothing, let step() complete that flight, and pack again on
            # the next call, when they can be preempted
            for r in reversed(runs):
                self.runs.appendleft(r)
            self.deferred += 1
            return [], []
        if need > free and decodes and self.runs:
            # the missing blocks sit with sequences whose prefill / ingest runs were held back above:
            # preempt the remaining decodes as well, so those runs fit on the next step (the decodes
            # are recomputed once blocks return, `_restore`)
            for j in list(decodes):
                self._spill(j)
            for r in reversed(runs):
                self.runs.appendleft(r)
            return [], []
        while need > free:
            # last resort: a held-back (queued) prefill / ingest run whose sequence holds KV gives its
            # blocks up and becomes a recompute run from row 0 (verify passes are never rewritten)
            keep = ({r.seq.dev.slot for r in runs} | {j.seq.dev.slot for j in decodes}
                    | {j.seq.dev.slot for j in self.decodes})
            cands = [r for r in self.runs if r.verify is None and r.start > 0 and not r.seq.dev.busy
                     and r.seq.dev.slot not in keep and self.pool.blocks(r.seq.dev.slot)]
            if not cands:
                break
            self._spill_run(max(cands, key=lambda r: r.start))
            free = self.pool.free_blocks()
        if need > free:
            raise KVCapacityError(f"KV pool exhausted: the step needs {need} blocks, {free} free, nothing left to "
                                  "preempt")
        return decodes, runs

    def _spill_run(self, r: Run) -> None:
        """Preempt the sequence of a queued run: release its KV and rewrite the run to recompute its
        rows [0, start) ahead of its own ids (sampled rows shift by `start`)."""
        d = r.seq.dev
        prefix = list(d.hist[:r.start])
        d.kv_len = 0
        self.pool.release(d.slot)
        r.rows = [x + r.start for x in r.rows]
        r.ids = prefix + list(r.ids)
        r.start = 0
        self.spills += 1

    def _reserve(self, slot: int, n: int) -> None:
        """pool.reserve; under KV pressure drop retained prefixes, then preempt decoding sequences
        outside the step being packed (largest context first) until the reservation fits."""
        try:
            self.pool.reserve(slot, n)
            return
        except KVCapacityError:
            if self.reclaimer is not None and self.reclaimer():
                try:
                    self.pool.reserve(slot, n)
                    return
                except KVCapacityError:
                    pass
        while True:
            cand = [j for j in self.decodes if j.seq.dev.slot != slot and j.seq.dev.slot not in self._in_step
                    and not j.seq.dev.busy]
            if not cand:
                raise KVCapacityError(f"KV pool exhausted reserving {n} rows for slot {slot}; nothing to preempt")
            self._spill(max(cand, key=lambda j: j.seq.dev.kv_len))
            try:
                self.pool.reserve(slot, n)
                return
            except KVCapacityError:
                continue

    def _spill(self, job: Decode) -> None:
        d = job.seq.dev
        d.spilled = d.kv_len
        d.kv_len = 0
        self.pool.release(d.slot)
        self.decodes.remove(job)
        self.spilled.append(job)
        self.spills += 1

    def _restore(self) -> None:
        """Bring back the oldest preempted sequence once its rows (and some headroom for the
        running batch) fit: one run recomputes its context, then its decode job resumes."""
        if not self.spilled:
            return
        job = self.spilled[0]
        d = job.seq.dev
        need = -(-(d.spilled + 2) // BLOCK) + len(self.decodes) + 2
        if self.pool.free_blocks() < need and (self.decodes or self.runs or self.flight is not None):
            return
        self.spilled.popleft()
        ids = d.hist[:d.spilled]
        d.spilled = 0
        self.runs.appendleft(Run(job.seq, ids, 0, [len(ids) - 1], [-1], lambda _s, job=job: self.decodes.append(job)))

    def step(self) -> int:
        """Launch the next packed forward (if any work), then complete the previous one."""
        prev, self.flight = self.flight, None
        self._prev_in_air = prev is not None
        decodes, runs = self._pack()
        emitted = 0
        if decodes or runs:
            self._in_step = {j.seq.dev.slot for j in decodes} | {r.seq.dev.slot for r in runs}
            f = self._launch(runs, decodes)
            emitted = len(decodes)
            for j in decodes:
                self._commit_blocks(j.seq.dev)
            self._in_step = set()
            f.finished = [j for j in decodes if j.k >= len(j.targets)]
            self.decodes = [j for j in self.decodes if j.k < len(j.targets)]
            if self.pipeline:
                self.flight = f
            else:
                self._complete(f)
        if prev is not None:
            self._complete(prev)
        return emitted

    def drain(self) -> None:
        if self.flight is not None:
            f, self.flight = self.flight, None
            self._complete(f)


def default_runtime(config, shape: ModelShape = TINY, **kw) -> Runtime:
    """The runtime `B200Engine(sim, config)` builds: tiny C1 decoder, eager."""
    nb = config.num_blocks or 4096
    return EagerRuntime(shape, num_blocks=nb, **kw)
