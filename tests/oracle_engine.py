"""TEST-ONLY stand-in engine built on the oracle (the checker, never shipped).

Lets the CPU suite exercise the host scheduler / kv / radix logic of the
product against the reference transcripts without a GPU.  It evaluates the
reference copy-model rule with oracle/ds_oracle.c on a host token history.
The product InferenceCore always builds a GpuEngine; only tests inject this.
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import cpu  # noqa: E402
from paper_2605_26289_b200.engine import CostLedger, RowResult, VerifyResult  # noqa: E402


class OracleEngine:
    def __init__(self, vocab: int = 32768, min_match: int = 3):
        self.vocab = vocab
        self.mm = min_match
        self.ledger = CostLedger()
        self.hist: dict[int, list[int]] = {}

    def load_prompt(self, seq, tokens, cursor, prefix_hash):
        self.hist[seq] = list(tokens)

    def _write(self, seq, pos, toks):
        h = self.hist.setdefault(seq, [])
        if len(h) < pos + len(toks):
            h.extend([0] * (pos + len(toks) - len(h)))
        h[pos:pos + len(toks)] = toks

    def _row(self, seq, upto):
        tok, src = cpu.copy_policy(self.hist[seq][:upto], upto, self.mm, self.vocab)
        return RowResult(tok, None if src < 0 else src)

    def forward_prefill(self, seq, past, batch, tokens):
        self.ledger.count_forward(len(batch))
        self._write(seq, past, list(batch))
        return self._row(seq, past + len(batch))

    def forward_decode(self, seq, past, token, tokens):
        self.ledger.count_forward(1)
        self._write(seq, past, [token])
        return self._row(seq, past + 1)

    def forward_verify(self, seq, past, batch, tokens, hash_in=None):
        self.ledger.count_forward(len(batch))
        self._write(seq, past, list(batch))
        rows = [self._row(seq, past + r + 1) for r in range(len(batch))]
        acc = 0
        while acc < len(batch) - 1 and rows[acc].argmax_id == batch[1 + acc]:
            acc += 1
        return VerifyResult(acc, rows)

    def propose(self, slots, window, min_match):
        out = []
        for seq, tokens, cap in slots:
            self._write(seq, len(tokens) - 1, [tokens[-1]])
            ring = list(tokens[-window:])
            out.append(cpu.lookup_ngram(ring, ring, min_match, cap))
        return out

    # batched plan execution (InferenceCore with batched_forward=True)
    def run(self, reqs, count=True):
        from paper_2605_26289_b200 import _lib

        out = []
        for r in reqs:
            q = len(r.batch)
            if count:
                self.ledger.count_forward(q)
            self._write(r.seq, r.past, list(r.batch))
            if r.kind == _lib.ENTRY_VERIFY:
                rows = [self._row(r.seq, r.past + i + 1) for i in range(q)]
                acc = 0
                while acc < q - 1 and rows[acc].argmax_id == r.batch[1 + acc]:
                    acc += 1
                res = VerifyResult(acc, rows)
            else:
                res = self._row(r.seq, r.past + q)
            if r.scratch:
                res.scratch = list(range(-q, 0))
            out.append(res)
        return out

    def queue_copies(self, pairs):
        self.copies = getattr(self, "copies", 0) + len(list(pairs))
