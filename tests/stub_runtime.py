"""Test double for the B200 runtime: host-only bookkeeping, no compute.

Lets the CPU suite exercise `B200Engine`'s control plane (phase order, costs,
fates, event strings) against the reference goldens without a GPU. Draft
acceptance is the host LCP of interned ids — the same decision the device
K4 kernel makes. Never used by the product path.
"""

from paper_2512_15834_b200.tokens import TokenTable


class StubRuntime:
    def __init__(self, vocab=4096):
        self.table = TokenTable(vocab)
        self.calls = []
        self.reclaimer = None

    def intern(self, toks):
        return self.table.ids(toks)

    def open(self, seq):
        for t in seq.script.turns:
            self.table.ids(t)
        seq.dev = object()

    def close(self, seq):
        self.calls.append(("close", seq.rid))

    def can_admit(self, seq):
        return True

    def prefill(self, seq, cached, next_turn, done):
        self.calls.append(("prefill", seq.rid, cached, seq.prompt_tokens))
        done(None)

    def emit(self, seq, tokens, done):
        self.calls.append(("emit", seq.rid, len(tokens)))
        done(None)

    def verify(self, seq, draft, span, done):
        d, s = self.table.lookup(draft), self.table.ids(span)
        n = min(len(d), len(s))
        acc = next((i for i in range(n) if d[i] != s[i]), n)
        self.calls.append(("verify", seq.rid, acc))
        done((acc, len(s) if acc >= len(s) else acc + 1))

    def ingest(self, seq, n_out, next_turn, done, output=None):
        self.calls.append(("ingest", seq.rid, n_out))
        done(None)

    def evict(self, seq, keep):
        self.calls.append(("evict", seq.rid, keep))


def stub_factory(sim, config):
    from paper_2512_15834_b200.engine import B200Engine

    return B200Engine(sim, config, runtime=StubRuntime())
