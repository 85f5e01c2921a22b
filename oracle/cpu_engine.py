"""CPU fp32 transformer engine - the BASELINE.md section 3.2 CPU baseline
(test / measurement infrastructure only; never imported by the product).

It serves the same engine interface the product InferenceCore drives
(forward_prefill / forward_decode / forward_verify / propose, reference
call sites scheduler.py:711, :766, speculator.py:102) with the oracle's
decoder math (oracle/llama_ref.py: RMSNorm, RoPE, GQA attention, SwiGLU, LM
head, bf16 storage points) executed with torch on the host cores, over a
paged K/V store indexed by the core's own cell ids - so radix restores and
grouped followers reuse cached K/V exactly as on the GPU.  Tokens follow the
reference copy-model rule (engine.py:196-216, via oracle/ds_oracle.c), so a
replay is transcript-identical to the reference and to the GPU engine while
every FLOP of the model runs; the real greedy ids are computed too (argmax
of the LM head) and discarded, as the GPU copy-policy path does.
"""
from __future__ import annotations

import torch

from . import cpu
from .llama_ref import _bf, rmsnorm, rope, rope_tables, split_gate_up, unpermute_qk


class _Ledger:
    def __init__(self):
        self.prefill_tokens = self.decode_passes = self.forward_calls = self.batch_tokens = 0

    def count_forward(self, n):
        self.forward_calls += 1
        self.batch_tokens += n

    def charge_prefill(self, n):
        self.prefill_tokens += n

    def charge_decode(self):
        self.decode_passes += 1

    def snapshot(self):
        return {"prefill_tokens": self.prefill_tokens, "decode_passes": self.decode_passes,
                "forward_calls": self.forward_calls, "batch_tokens": self.batch_tokens}


class _Row:
    def __init__(self, tok, src):
        self.argmax_id = tok
        self.copy_source = None if src < 0 else src
        self.scratch = None


class _Verify:
    def __init__(self, acc, rows):
        self.accepted = acc
        self.rows = rows
        self.scratch = None


class CpuTransformerEngine:
    def __init__(self, shape, weights: dict, vocab: int, min_match: int, capacity: int,
                 max_pos: int = 1 << 16, threads: int | None = None):
        if threads:
            torch.set_num_threads(threads)
        self.s = shape
        self.w = weights  # fp32 CPU copies of the bf16 weights
        self.vocab, self.mm = vocab, min_match
        self.ledger = _Ledger()
        self.hist: dict[int, list[int]] = {}
        s = shape
        self.k = torch.zeros(s.layers, capacity, s.n_kv_heads, s.head_dim)
        self.v = torch.zeros_like(self.k)
        self.cos, self.sin = rope_tables(max_pos, s.head_dim, s.rope_theta)
        self.kv = None
        self.flops = 0.0

    def attach(self, kv) -> None:
        """The core's UnifiedKvCache: position -> cell mapping of every seq."""
        self.kv = kv

    # -- token history + copy rule (identical to the reference mock) --
    def load_prompt(self, seq, tokens, cursor, prefix_hash):
        self.hist[seq] = [int(t) for t in tokens]

    def _write(self, seq, pos, toks):
        h = self.hist.setdefault(seq, [])
        if len(h) < pos + len(toks):
            h.extend([0] * (pos + len(toks) - len(h)))
        h[pos:pos + len(toks)] = toks

    def _row(self, seq, upto):
        tok, src = cpu.copy_policy(self.hist[seq][:upto], upto, self.mm, self.vocab)
        return _Row(tok, src)

    # -- the fp32 decoder over the paged store --
    @torch.no_grad()
    def _model(self, seq, past, batch, out_rows):
        s, w = self.s, self.w
        q_len = len(batch)
        nh, nkv, d = s.n_heads, s.n_kv_heads, s.head_dim
        G = nh // nkv
        new = torch.tensor(self.kv.cell_ids(seq, past, past + q_len), dtype=torch.long)
        ctx = torch.tensor(self.kv.cell_ids(seq, 0, past + q_len), dtype=torch.long)
        cos, sin = self.cos[past:past + q_len], self.sin[past:past + q_len]
        x = w["embed"][torch.tensor(batch, dtype=torch.long)]
        kpos = torch.arange(past + q_len)[None, :]
        qpos = torch.arange(past, past + q_len)[:, None]
        mask = (kpos > qpos)[None]
        scale = 1.0 / d ** 0.5
        for l in range(s.layers):
            h = rmsnorm(x, w["attn_norm"][l], s.rms_eps)
            qkv = unpermute_qk(_bf(h @ w["wqkv"][l].T), nh, nkv, d)
            q = rope(qkv[:, : nh * d].view(q_len, nh, d), cos, sin)
            self.k[l, new] = rope(qkv[:, nh * d:(nh + nkv) * d].view(q_len, nkv, d), cos, sin)
            self.v[l, new] = qkv[:, (nh + nkv) * d:].view(q_len, nkv, d)
            kk = self.k[l, ctx].repeat_interleave(G, dim=1)
            vv = self.v[l, ctx].repeat_interleave(G, dim=1)
            sc = torch.einsum("qhd,khd->hqk", q, kk) * scale
            sc = sc.masked_fill(mask, float("-inf"))
            o = _bf(torch.einsum("hqk,khd->qhd", torch.softmax(sc, dim=-1), vv).reshape(q_len, -1))
            x = x + o @ w["wo"][l].T
            h = rmsnorm(x, w["mlp_norm"][l], s.rms_eps)
            g, u = split_gate_up(_bf(h @ w["w_gate_up"][l].T), s.ffn)
            x = x + _bf(torch.nn.functional.silu(g) * u) @ w["w_down"][l].T
        logits = rmsnorm(x[out_rows], w["final_norm"], s.rms_eps) @ w["lm_head"].T
        return logits.argmax(-1)  # the model's greedy ids (the copy rule decides)

    def forward_prefill(self, seq, past, batch, tokens):
        self.ledger.count_forward(len(batch))
        self._write(seq, past, list(batch))
        self._model(seq, past, list(batch), [len(batch) - 1])
        return self._row(seq, past + len(batch))

    def forward_decode(self, seq, past, token, tokens):
        self.ledger.count_forward(1)
        self._write(seq, past, [token])
        self._model(seq, past, [token], [0])
        return self._row(seq, past + 1)

    def forward_verify(self, seq, past, batch, tokens, hash_in=None):
        self.ledger.count_forward(len(batch))
        self._write(seq, past, list(batch))
        self._model(seq, past, list(batch), list(range(len(batch))))
        rows = [self._row(seq, past + r + 1) for r in range(len(batch))]
        acc = 0
        while acc < len(batch) - 1 and rows[acc].argmax_id == batch[1 + acc]:
            acc += 1
        return _Verify(acc, rows)

    def propose(self, slots, window, min_match):
        out = []
        for seq, tokens, cap in slots:
            self._write(seq, len(tokens) - 1, [tokens[-1]])
            ring = list(tokens[-window:])
            out.append(cpu.lookup_ngram(ring, ring, min_match, cap))
        return out
