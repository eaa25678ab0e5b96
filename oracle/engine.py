"""ORACLE (test infrastructure). The reference engine's control plane, restated,
with an fp32 CPU compute model attached to every phase.

Control plane: `spectool/engine.py` — admission (:233-243), prefill (:245-264),
reasoning decode (:266-306), draft validation + consume rule (:96-111,
:289-323), span decode (:325-337), fate selection (:339-355), ingest
(:357-372), emit + evict with the turn_base prefix rule (:374-387), final
(:389-401). Costs and event strings are the reference's; the whole flow is
re-expressed here as a table of phase handlers.

Compute model (self-defined semantics of the B200 build, DESIGN.md "KV
off-by-one"): per sequence, `rows` = KV rows written, `pend` = last sampled
id not yet fed, `counted` = whether it is already emitted. Reference
kv_tokens == rows + counted-pend; the allocator keeps ceil(kv_tokens/16)
blocks after every phase. `trace` collects every sampled row (rid, pos, fed,
target, sampled) and its fp32 logits; `tables` the block list of each
sequence after each phase.
"""

from __future__ import annotations

from paper_2512_15834_b200.domain import TokenKind, canonical_key, extract_tool_call
from paper_2512_15834_b200.errors import ConfigError, InvalidScenario

from .ids import SALT_OUTPUT, SALT_PROMPT, Interner, fill, text_ids
from .kv_alloc import LifoAllocator


class _Seq:
    def __init__(self, rid, script, prompt, client, slot):
        self.rid, self.script, self.client, self.slot = rid, script, client, slot
        self.state = "new"
        self.turn = 0
        self.prompt_tokens = prompt
        self.cached_prefix = 0
        self.kv_tokens = 0
        self.turn_base = 0
        self.emit_pending = 0
        self.advance = False
        self.fates: list[str] = []
        self.accepted_counts: list[int] = []
        # compute model
        self.rows = 0
        self.pend = None
        self.counted = False
        self.hist: list[int] = []
        self.replay: list[int] = []


def _split(turn):
    starts = [i for i, t in enumerate(turn) if t.kind is TokenKind.TOOL_START]
    if not starts:
        return list(turn), None
    i = starts[0]
    ends = [j for j in range(i + 1, len(turn)) if turn[j].kind is TokenKind.TOOL_END]
    if not ends:
        raise InvalidScenario("scripted turn opens a span it never closes")
    if ends[0] != len(turn) - 1:
        raise InvalidScenario("scripted turn continues past TOOL_END")
    return turn[:i], turn[i:]


class OracleEngine:
    def __init__(self, sim, config, model=None, seed: int = 0, num_blocks: int = 4096, vocab: int | None = None):
        from paper_2512_15834_b200.engine import ToolCacheStore  # same store semantics (pinned by goldens)

        self.sim, self.cfg, self.model, self.seed = sim, config, model, seed
        self.store = ToolCacheStore(sim.clock) if config.tool_cache else None
        self.sequences: dict[str, _Seq] = {}
        self.events: list[str] = []
        self.observers = []
        self.evictions = 0
        self._resident = 0
        self._queue: list[_Seq] = []
        V = vocab if vocab is not None else (model.s.vocab if model is not None else 512)
        self.vocab = V
        self.ids = Interner(V)
        self.alloc = LifoAllocator(num_blocks)
        self._slots = list(range(1023, -1, -1))
        self.trace: list[dict] = []
        self.tables: list[tuple[str, str, list[int]]] = []

    # ---------------------------------------------------------------- helpers
    def _log(self, seq, phase, n):
        t = self.sim.now
        self.events.append(f"t={t!r} rid={seq.rid} phase={phase} tokens={n}")
        for cb in self.observers:
            cb(t, seq.rid, phase, n)

    def _blocks(self, seq, phase):
        kv = seq.rows + (1 if seq.pend is not None and seq.counted else 0)
        self.alloc.truncate(seq.slot, kv)
        self.alloc.reserve(seq.slot, kv)
        self.tables.append((seq.rid, phase, self.alloc.blocks(seq.slot)))

    def _fwd(self, seq, ids, start, rows, targets):
        """Append `ids` at `start`; return the forced samples of `rows`."""
        self.alloc.reserve(seq.slot, start + len(ids))
        del seq.hist[start:]
        seq.hist.extend(ids)
        seq.rows = start + len(ids)
        logits = self.model.forward(seq.rid, ids, start, rows) if self.model is not None else None
        out = []
        for k, (r, tgt) in enumerate(zip(rows, targets)):
            raw = int(logits[k].argmax()) if logits is not None else tgt
            got = tgt if tgt >= 0 else raw
            out.append(got)
            self.trace.append({"rid": seq.rid, "pos": start + r, "fed": ids[r], "target": tgt, "sampled": got,
                               "raw_argmax": raw, "logits": None if logits is None else logits[k].clone()})
        return out

    def _first(self, seq, turn):
        tt = seq.script.turns
        return self.ids(tt[turn][0]) if turn < len(tt) and tt[turn] else -1

    def _unfeed_last(self, seq):
        seq.rows -= 1
        seq.pend, seq.counted = seq.hist.pop(), True

    # compute bodies of the phases ------------------------------------------
    def _c_prefill(self, seq, cached, nxt):
        P = seq.prompt_tokens
        if P < 1:
            raise ConfigError("prompt_tokens >= 1 required")
        seq.rows = min(seq.rows, cached)
        self.alloc.truncate(seq.slot, seq.rows)
        ids = seq.hist[:P]
        ids += seq.replay[: P - len(ids)]
        if len(ids) < P:
            ids += fill(self.seed, seq.rid, SALT_OUTPUT if seq.replay else SALT_PROMPT, len(ids), P - len(ids),
                        self.vocab)
        seq.replay = []
        start = cached if cached < P else P - 1
        run = ids[start:P]
        (tok,) = self._fwd(seq, run, start, [len(run) - 1], [self._first(seq, nxt)])
        seq.pend, seq.counted = tok, False
        self._blocks(seq, "prefill")

    def _c_emit(self, seq, toks, phase):
        want = self.ids.many(toks)
        if want and seq.pend is not None and not seq.counted:
            assert seq.pend == want[0]
            seq.counted = True
            want = want[1:]
        if want and seq.pend is None:
            self._unfeed_last(seq)
        for t in want:
            (got,) = self._fwd(seq, [seq.pend], seq.rows, [0], [t])
            seq.pend, seq.counted = got, True
            self._blocks(seq, phase)
        self._blocks(seq, phase)

    def _c_verify(self, seq, draft_toks, span):
        draft, sp = self.ids.compare_ids(draft_toks), self.ids.many(span)
        feed = self.ids.feed_ids(draft_toks)
        if seq.pend is None:
            self._unfeed_last(seq)
        if seq.counted:
            lead, model_head, shift = [seq.pend], [], 0
        else:
            lead, model_head, shift = [], [seq.pend], 1
        inp = lead + feed
        base = seq.rows
        tg = [sp[j + shift] if j + shift < len(sp) else -1 for j in range(len(inp))]
        got = self._fwd(seq, inp, base, list(range(len(inp))), tg)
        model = model_head + got
        acc = 0
        while acc < min(len(draft), len(model), len(sp)) and draft[acc] == model[acc]:
            acc += 1
        consume = len(sp) if acc >= len(sp) else acc + 1
        keep = base + len(lead) + acc
        seq.rows = keep
        del seq.hist[keep:]
        if self.model is not None:
            self.model.truncate(seq.rid, keep)
        if acc < len(sp):
            seq.pend, seq.counted = model[acc], True
        else:
            seq.pend, seq.counted = None, False
        self._blocks(seq, "validate")
        return acc, consume

    def _c_ingest(self, seq, n_out, nxt, text=None):
        if seq.pend is None and n_out == 0:
            self._unfeed_last(seq)
        lead = [seq.pend] if seq.pend is not None else []
        out = text_ids(self.seed, seq.rid, text, seq.rows + len(lead), n_out, self.vocab)
        inp = lead + out
        (tok,) = self._fwd(seq, inp, seq.rows, [len(inp) - 1], [self._first(seq, nxt)])
        seq.pend, seq.counted = tok, False
        self._blocks(seq, "ingest")

    # ---------------------------------------------------------------- API
    def submit_request(self, rid, script, prompt_tokens, client):
        if rid in self.sequences:
            raise ConfigError(f"request id {rid!r} already submitted")
        seq = _Seq(rid, script, prompt_tokens, client, self._slots.pop())
        for turn in script.turns:
            self.ids.many(turn)
        self.sequences[rid] = seq
        self._admit(seq)

    def resubmit(self, rid, prompt_tokens, turn_resolved):
        seq = self.sequences[rid]
        if seq.state != "waiting":
            raise ConfigError(f"request {rid!r} is not waiting on a tool")
        seq.prompt_tokens, seq.advance, seq.state = prompt_tokens, turn_resolved, "new"
        self._admit(seq)

    def submit_tool_cache(self, rid, entry):
        if self.store is None:
            raise ConfigError("this engine has no tool cache")
        self.store.submit(rid, entry)
        return 1

    # ---------------------------------------------------------------- phases
    def _admit(self, seq):
        if self._resident >= self.cfg.batch_size:
            self._queue.append(seq)
            return
        self._resident += 1
        self._prefill(seq)

    def _release_slot(self):
        self._resident -= 1
        while self._queue and self._resident < self.cfg.batch_size:
            self._resident += 1
            self._prefill(self._queue.pop(0))

    def _prefill(self, seq):
        nxt = seq.turn + int(seq.advance)
        seq.client.on_turn_start(seq.rid, nxt)
        cached = seq.cached_prefix if self.cfg.prefix_cache else 0
        fresh = seq.prompt_tokens - cached
        if fresh < 0:
            raise InvalidScenario("resubmitted prompt shrank below the cached prefix")
        self._c_prefill(seq, cached, nxt)

        def landed():
            self._log(seq, "prefill", fresh)
            seq.kv_tokens = seq.prompt_tokens
            if seq.advance:
                seq.advance = False
                seq.turn += 1
            seq.state = "decode"
            self._turn(seq)

        self.sim.schedule(self.cfg.prefill_rate * fresh, landed, name=f"prefill_{seq.rid}")

    def _turn(self, seq):
        seq.turn_base = seq.kv_tokens
        reason, span = _split(seq.script.turns[seq.turn])
        self._c_emit(seq, reason, "decode")
        if span is None:
            self.sim.schedule(self.cfg.decode_rate * len(reason), lambda: self._final(seq, reason),
                              name=f"final_{seq.rid}")
        else:
            self.sim.schedule(self.cfg.decode_rate * len(reason), lambda: self._reasoned(seq, reason, span),
                              name=f"reason_{seq.rid}")

    def _reasoned(self, seq, reason, span):
        if reason:
            self._log(seq, "decode", len(reason))
        seq.kv_tokens += len(reason)
        seq.emit_pending += len(reason)
        call = extract_tool_call(span)
        bet = self.store.lookup_name(seq.rid, call.name) if self.store is not None else None
        if bet is None or not bet.call_tokens:
            self._c_emit(seq, span, "decode")
            self.sim.schedule(self.cfg.decode_rate * len(span), lambda: self._decoded(seq, span, call, None, len(span)),
                              name=f"call_{seq.rid}")
            return
        acc, consume = self._c_verify(seq, bet.call_tokens, span)
        cost = (self.cfg.decode_rate * (acc + 1) if self.cfg.validate_per_token
                else self.cfg.decode_rate + self.cfg.prefill_rate * acc)

        def validated():
            self._log(seq, "validate", acc)
            seq.accepted_counts.append(acc)
            seq.kv_tokens += consume
            seq.emit_pending += consume
            rest = len(span) - consume
            if rest <= 0:
                self._span_done(seq, span, call, acc)
                return
            self._c_emit(seq, span[consume:], "decode")
            self.sim.schedule(self.cfg.decode_rate * rest, lambda: self._decoded(seq, span, call, acc, rest),
                              name=f"call_rest_{seq.rid}")

        self.sim.schedule(cost, validated, name=f"validate_{seq.rid}")

    def _decoded(self, seq, span, call, validated, n):
        self._log(seq, "decode", n)
        seq.kv_tokens += n
        seq.emit_pending += n
        self._span_done(seq, span, call, validated)

    def _span_done(self, seq, span, call, validated):
        hit = self.store.lookup_key(seq.rid, canonical_key(call)) if self.store is not None else None
        if hit is None:
            seq.fates.append("miss")
            self._evict(seq, span, call)
            return
        if validated is None:
            seq.fates.append("late_hit")
        elif validated >= len(span):
            seq.fates.append("full_hit")
        else:
            seq.fates.append("partial_hit")
        self._c_ingest(seq, hit.output_tokens, seq.turn + 1, hit.output)

        def ingested():
            self._log(seq, "ingest", hit.output_tokens)
            seq.kv_tokens += hit.output_tokens
            seq.emit_pending += hit.output_tokens
            seq.prompt_tokens = seq.kv_tokens
            seq.turn += 1
            seq.client.on_ingest(seq.rid, seq.turn - 1, hit)
            seq.client.on_turn_start(seq.rid, seq.turn)
            self._turn(seq)

        self.sim.schedule(self.cfg.prefill_rate * hit.output_tokens, ingested, name=f"ingest_{seq.rid}")

    def _evict(self, seq, span, call):
        self._log(seq, "emit", seq.emit_pending)
        seq.emit_pending = 0
        self._log(seq, "evict", seq.kv_tokens)
        self.evictions += 1
        seq.cached_prefix = seq.turn_base
        keep = seq.turn_base if self.cfg.prefix_cache else 0
        seq.rows = min(seq.rows, keep)
        seq.pend, seq.counted = None, False
        del seq.hist[seq.turn_base:]
        seq.replay = self.ids.many(span)
        if keep == 0:
            self.alloc.release(seq.slot)
        else:
            self.alloc.truncate(seq.slot, keep)
        if self.model is not None:
            self.model.truncate(seq.rid, keep)
        self.tables.append((seq.rid, "evict", self.alloc.blocks(seq.slot)))
        seq.state = "waiting"
        seq.kv_tokens = 0
        self._release_slot()
        seq.client.on_emit(seq.rid, seq.turn, span, call, seq.turn_base)

    def _final(self, seq, toks):
        self._log(seq, "decode", len(toks))
        seq.kv_tokens += len(toks)
        self._log(seq, "emit", seq.emit_pending + len(toks))
        seq.emit_pending = 0
        seq.state = "done"
        self.alloc.release(seq.slot)
        self._slots.append(seq.slot)
        self.tables.append((seq.rid, "final", []))
        if self.model is not None:
            self.model.drop(seq.rid)
        self._release_slot()
        if self.store is not None:
            self.store.purge_request(seq.rid)
        seq.client.on_final(seq.rid, toks)
