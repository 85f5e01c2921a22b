"""GpuEngine: the device realisation of the reference engine boundary.

The reference ``MockEngine.forward(context, batch)`` (engine.py:268-281)
materialises the whole context on the host every call.  Here the context is
the resident paged KV store and the sequence's token history on the device;
a forward ships only the batch tokens plus a few int32 of metadata (one
pinned H2D), runs the whole Llama-shaped decoder in ONE native call
(``ds_model_forward``: cuBLAS GEMMs + our sm_100a kernels), evaluates the
token policy and the verify accept loop on device, and returns only the
chosen ids, copy sources and accept counts (one small D2H).

Token policies:
* ``copy``   - the reference copy-model rule (engine.py:196-216) evaluated by
  the K2 kernel over the device token history: bit-exact transcripts versus
  the reference InferenceCore while every FLOP and byte of the real model runs.
* ``argmax`` - greedy argmax of the real logits (K8, lowest id on ties).

The ledger keeps the reference's per-entry semantics (engine.py:72-102).
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _hostcore, _lib
from ._lib import check, lib
from .config import CoreConfig
from .kernels import FNV64_OFFSET, _as_i32, host_fnv1a64_tokens
from .kvcache import UnifiedKvCache

_ENTRY_DT = np.dtype([("seq", "<i4"), ("past", "<i4"), ("q_len", "<i4"), ("q_start", "<i4"),
                      ("kind", "<i4"), ("n_draft", "<i4"), ("out_start", "<i4"),
                      ("n_out", "<i4"), ("hash_in", "<u8")])
assert _ENTRY_DT.itemsize == 40


# packed query rows the decode kernel K7 takes (kDecodeMaxRows, csrc/attn_plan.h);
# entries with more go to the tcgen05 kernel K6 and are ordered first
DECODE_MAX_ROWS = 24
# forwards of at most this many rows (one entry) replay a captured CUDA graph in
# the native runtime (csrc/runtime.cu); their arguments sit at fixed offsets
GRAPH_MAX_ROWS = 32


class CostLedger:
    """Monotonic forward-pass counters (engine.py:72-102)."""

    def __init__(self):
        self._lock = threading.Lock()
        self.prefill_tokens = 0
        self.decode_passes = 0
        self.forward_calls = 0
        self.batch_tokens = 0

    def count_forward(self, batch_size: int) -> None:
        with self._lock:
            self.forward_calls += 1
            self.batch_tokens += batch_size

    def charge_prefill(self, n: int) -> None:
        with self._lock:
            self.prefill_tokens += n

    def charge_decode(self) -> None:
        with self._lock:
            self.decode_passes += 1

    def snapshot(self) -> dict:
        with self._lock:
            return {"prefill_tokens": self.prefill_tokens, "decode_passes": self.decode_passes,
                    "forward_calls": self.forward_calls, "batch_tokens": self.batch_tokens}


@dataclass(slots=True)
class RowResult:
    """One sampled position: the reference Logits' argmax_id / copy_source."""

    argmax_id: int
    copy_source: int | None
    scratch: list | None = None


@dataclass(slots=True)
class VerifyResult:
    accepted: int
    rows: list
    scratch: list | None = None


@dataclass(slots=True)
class EntryRequest:
    """One plan entry for a (possibly batched) forward."""

    kind: int          # _lib.ENTRY_*
    seq: int
    past: int
    batch: list        # tokens forwarded
    tokens: list       # full committed token list of the slot (for the prefix hash)
    n_draft: int = 0
    scratch: bool = False  # rows' K/V go to scratch cells (batched decode/verify)


class _Staging:
    """Growable pinned-host + device int32 buffer; one H2D per flush."""

    def __init__(self, device, words: int = 1 << 16):
        self.device = device
        self._alloc(words)
        self.reset()

    def _alloc(self, words):
        self.host = torch.empty(words, dtype=torch.int32, pin_memory=True)
        self.host_np = self.host.numpy()
        self.dev = torch.empty(words, dtype=torch.int32, device=self.device)

    def reset(self):
        self.parts: list[tuple[int, np.ndarray]] = []
        self.n = 0

    def add(self, arr: np.ndarray) -> int:
        a = np.ascontiguousarray(arr).view(np.int32).reshape(-1)
        off = self.n
        self.parts.append((off, a))
        self.n = off + ((a.size + 3) // 4) * 4  # 16-byte aligned parts
        return off

    def ensure(self) -> None:
        """Grow (before direct writes into host_np) if the staged parts need it."""
        if self.n > self.host.numel():
            torch.cuda.current_stream().synchronize()
            self._alloc(max(self.n, 2 * self.host.numel()))

    def upload(self) -> None:
        self.ensure()
        for off, a in self.parts:
            self.host_np[off:off + a.size] = a
        if self.n:
            self.dev[: self.n].copy_(self.host[: self.n], non_blocking=True)

    def add_fixed(self, arr: np.ndarray, words: int) -> int:
        """Like add(), but reserves `words` so the next part's offset does not
        depend on this part's length (stable pointers for CUDA-graph replay)."""
        a = np.ascontiguousarray(arr).view(np.int32).reshape(-1)
        if a.size > words:
            raise ValueError("part larger than its fixed slot")
        off = self.n
        self.parts.append((off, a))
        self.n = off + ((words + 3) // 4) * 4
        return off

    def dptr(self, off: int) -> int:
        return self.dev.data_ptr() + 4 * off

    def hptr(self, off: int) -> int:
        return self.host.data_ptr() + 4 * off


class GpuEngine:
    """Weights, paged KV store and the per-forward plumbing on one B200."""

    def __init__(self, cfg: CoreConfig, kv: UnifiedKvCache, n_seqs: int, device=None,
                 weights: dict | None = None, keep_logits: bool = False):
        if not torch.cuda.is_available():
            raise RuntimeError("GpuEngine needs a CUDA device (no CPU fallback)")
        self.cfg = cfg
        self.shape = s = cfg.shape
        self.kv = kv
        kv.record_ops = True
        self.ledger = CostLedger()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.policy = {"copy": _lib.POLICY_COPY, "argmax": _lib.POLICY_ARGMAX}[cfg.token_policy]
        self.n_seqs = n_seqs
        self.capacity = kv.capacity_cells
        self.pos_stride = self.capacity
        # batched plans park decode/verify rows in scratch cells past the
        # allocator's range until the accept count is known (cell-id parity)
        self.n_scratch = ((cfg.spec_max_lookahead + 1) * n_seqs) if cfg.batched_forward else 0
        self.head_stride = self.capacity + self.n_scratch
        dev = self.device
        L = lib()

        # ---- weights (random init N(0, 0.02), norms = 1) ----
        self.w = weights if weights is not None else self._init_weights(cfg.seed)
        # ---- RoPE tables (float64 angles -> fp32) ----
        inv = cfg.shape.rope_theta ** (-torch.arange(0, s.head_dim, 2, dtype=torch.float64,
                                                      device=dev) / s.head_dim)
        pos = torch.arange(self.pos_stride, dtype=torch.float64, device=dev)
        ang = pos[:, None] * inv[None, :]
        self.rope_cos = torch.cos(ang).float().contiguous()
        self.rope_sin = torch.sin(ang).float().contiguous()
        del ang, pos
        # ---- paged KV store ----
        # head-major [L][kv_head][cell][hd]: a run of consecutive cells of one head
        # is one contiguous block -> TMA boxes for the attention kernels
        self.k_pool = torch.zeros((s.layers, s.n_kv_heads, self.head_stride, s.head_dim),
                                  dtype=torch.bfloat16, device=dev)
        self.v_pool = torch.zeros_like(self.k_pool)
        self.pos2cell = torch.zeros((n_seqs, self.pos_stride), dtype=torch.int32, device=dev)
        self.hist = torch.zeros((n_seqs, self.pos_stride), dtype=torch.int32, device=dev)
        self.mask_words = (n_seqs + 31) // 32
        self.member = torch.zeros((self.capacity, self.mask_words), dtype=torch.int32, device=dev)
        self.trie_ref = torch.zeros(self.capacity, dtype=torch.int32, device=dev)
        # exact page-table mappings per cell (the refcount observable also when
        # a sequence maps one cell twice)
        self.map_ref = torch.zeros(self.capacity, dtype=torch.int32, device=dev)

        # ---- per-forward buffers ----
        self.max_out = (cfg.spec_max_lookahead + 1) * (n_seqs if cfg.batched_forward else 1)
        self.max_entries = n_seqs if cfg.batched_forward else 1
        self.max_rows = cfg.n_batch + self.max_out
        self.logits = torch.empty((self.max_out, s.vocab), dtype=torch.float32, device=dev)
        # False: no logits materialisation - the LM head reduces each sampled
        # row to its argmax in its epilogue (ds_forward_args.logits_out)
        self.keep_logits = keep_logits
        # next prompt-lookup proposal computed inside decode/verify forwards
        # (ds_forward_args.next_*): [e, len, draft_len][n] + drafts [n][cap] + scratch
        self.nd_cap = max(1, cfg.spec_max_lookahead)
        self.nd_off = 2 * self.max_out + self.max_entries
        self.nd_off += self.nd_off & 1
        nd_words = self.max_entries * (3 + self.nd_cap) + 4 * self.max_entries + 2
        self.res_dev = torch.zeros(self.nd_off + nd_words, dtype=torch.int32, device=dev)
        self._draft_cache: dict[int, tuple[int, list]] = {}  # seq -> (len(tokens), draft)
        self.fused_drafts = bool(cfg.speculation_enabled)
        self.res_host = torch.zeros_like(self.res_dev, device="cpu").pin_memory()
        self.stage = _Staging(dev)
        self.k1_dev = torch.zeros(4 * n_seqs + n_seqs * cfg.spec_max_lookahead + 16,
                                  dtype=torch.int32, device=dev)
        self.k1_host = torch.zeros_like(self.k1_dev, device="cpu").pin_memory()

        self.model_c = _lib.Model(
            s.layers, s.hidden, s.n_heads, s.n_kv_heads, s.head_dim, s.ffn, s.vocab, s.rms_eps,
            self.w["embed"].data_ptr(), self.w["attn_norm"].data_ptr(), self.w["wqkv"].data_ptr(),
            self.w["wo"].data_ptr(), self.w["mlp_norm"].data_ptr(), self.w["w_gate_up"].data_ptr(),
            self.w["w_down"].data_ptr(), self.w["final_norm"].data_ptr(),
            self.w["lm_head"].data_ptr(), self.rope_cos.data_ptr(), self.rope_sin.data_ptr(),
            self.pos_stride)
        self.kv_c = _lib.KvStore(self.k_pool.data_ptr(), self.v_pool.data_ptr(), self.head_stride,
                                 self.pos2cell.data_ptr(), self.hist.data_ptr(), self.pos_stride,
                                 n_seqs)
        self._model_ref = ctypes.byref(self.model_c)
        self._kv_ref = ctypes.byref(self.kv_c)
        ws = L.ds_forward_workspace_bytes(ctypes.byref(self.model_c), self.max_rows,
                                          self.max_out, self.max_entries)
        # zero once: the attention split-merge counters live here and self-reset
        self.workspace = torch.zeros(ws, dtype=torch.uint8, device=dev)
        self._hash: dict[int, tuple[int, int]] = {}   # seq -> (length, FNV64 of hist[:length])
        self._pending_hist: list[tuple[int, int, np.ndarray]] = []
        self._copies: list[tuple[int, int]] = []
        self.gpu_launches = 0
        self._ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        self.reset_counters()

    # -- instrumentation ------------------------------------------------------------

    def reset_counters(self) -> None:
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        # n, device seconds, rows, kv; "propose" = the K1 launches outside forwards
        self._fwd = {"prefill": [0, 0.0, 0, 0], "decode": [0, 0.0, 0, 0],
                     "propose": [0, 0.0, 0, 0]}

    def device_seconds(self) -> float:
        return sum(v[1] for v in self._fwd.values())

    def forward_stats(self) -> dict:
        return {k: {"n": v[0], "seconds": v[1], "rows": v[2],
                    "mean_kv_len": (v[3] / v[0]) if v[0] else 0.0} for k, v in self._fwd.items()}

    # -- weights ------------------------------------------------------------------

    def _init_weights(self, seed: int) -> dict:
        s, dev = self.shape, self.device
        g = torch.Generator(device=dev)
        g.manual_seed(seed)

        def randn(*shape):
            t = torch.empty(shape, dtype=torch.bfloat16, device=dev)
            t.normal_(0.0, 0.02, generator=g)
            return t

        ones = lambda *shape: torch.ones(shape, dtype=torch.bfloat16, device=dev)  # noqa: E731
        return {
            "embed": randn(s.vocab, s.hidden),
            "attn_norm": ones(s.layers, s.hidden),
            "wqkv": randn(s.layers, s.qkv_width, s.hidden),
            "wo": randn(s.layers, s.hidden, s.n_heads * s.head_dim),
            "mlp_norm": ones(s.layers, s.hidden),
            "w_gate_up": randn(s.layers, 2 * s.ffn, s.hidden),
            "w_down": randn(s.layers, s.hidden, s.ffn),
            "final_norm": ones(s.hidden),
            "lm_head": randn(s.vocab, s.hidden),
        }

    # -- host-side state ------------------------------------------------------------

    def load_prompt(self, seq: int, tokens, cursor: int, prefix_hash: int) -> None:
        """New request on `seq`: its token history is (re)uploaded with the next
        flush; the committed-prefix hash restarts from the scheduler's
        prefix_hash (scheduler.py:237)."""
        self._pending_hist.append((seq, 0, tokens if isinstance(tokens, np.ndarray)
                                   and tokens.dtype == np.int32 else _as_i32(tokens)))
        self._hash[seq] = (cursor, prefix_hash)
        self._draft_cache.pop(seq, None)

    def _hash_in(self, seq: int, past: int, tokens) -> int:
        ln, st = self._hash.get(seq, (0, FNV64_OFFSET))
        if ln > past:
            ln, st = 0, FNV64_OFFSET
        if past > ln:
            st = _hostcore.fnv1a64_tokens(tokens, ln, past, st)
        self._hash[seq] = (past, st)
        return st

    def queue_copies(self, pairs) -> None:
        """(src_cell, dst_cell) K/V row moves applied at the next flush."""
        self._copies.extend(pairs)

    def _stage_metadata(self, extra_ops=None) -> tuple:
        """Queue pending hist writes, cell copies and kv ops; offsets for the flush."""
        segs_off = ops_off = cp_off = -1
        n_segs = n_ops = n_cp = 0
        if self._copies:
            last = {}
            for src, dst in self._copies:  # a later owner of a cell wins
                last[dst] = src
            pairs = np.array([(src, dst) for dst, src in last.items()], dtype=np.int32)
            cp_off = self.stage.add(pairs)
            n_cp = len(pairs)
            self._copies = []
        if self._pending_hist:
            rows, data = [], []
            cur = 0
            for seq, start, toks in self._pending_hist:
                n = len(toks)
                rows.append((seq, start, n, cur))
                data.append(toks)
                cur += n
            segs = np.array(rows, dtype=np.int32)
            data_off = self.stage.add(np.concatenate(data) if cur else np.zeros(1, np.int32))
            segs[:, 3] += data_off
            segs_off = self.stage.add(segs)
            n_segs = len(segs)
            self._pending_hist = []
        ops = np.asarray(self.kv.take_ops(), dtype=np.int32).reshape(-1, 5)
        if extra_ops:
            ops = np.concatenate([ops, np.asarray(extra_ops, dtype=np.int32).reshape(-1, 5)])
        if len(ops):
            ops_off = self.stage.add(ops)
            n_ops = len(ops)
        return segs_off, n_segs, ops_off, n_ops, cp_off, n_cp

    def _apply_metadata(self, segs_off, n_segs, ops_off, n_ops, cp_off, n_cp, stream) -> None:
        L = lib()
        if n_cp:
            s = self.shape
            check(L.ds_kv_copy_cells(self.k_pool.data_ptr(), self.v_pool.data_ptr(), s.layers,
                                     s.n_kv_heads, self.head_stride, s.head_dim,
                                     self.stage.dptr(cp_off), n_cp, stream), "ds_kv_copy_cells")
            self.gpu_launches += 1
        if n_segs:
            check(L.ds_hist_write(self.stage.dev.data_ptr(), self.stage.dptr(segs_off), n_segs,
                                  self.hist.data_ptr(), self.pos_stride, stream), "ds_hist_write")
            self.gpu_launches += 1
        if n_ops:
            check(L.ds_kv_apply(self.stage.dptr(ops_off), n_ops, self.pos2cell.data_ptr(),
                                self.pos_stride, self.n_seqs, self.member.data_ptr(),
                                self.mask_words, self.trie_ref.data_ptr(),
                                self.map_ref.data_ptr(), stream), "ds_kv_apply")
            self.gpu_launches += 1

    def flush(self) -> None:
        """Push pending metadata (page-table ops, history writes) to the device."""
        stream = torch.cuda.current_stream()
        self.stage.reset()
        meta = self._stage_metadata()
        self.stage.upload()
        self._apply_metadata(*meta, stream.cuda_stream)

    # -- forward -------------------------------------------------------------------

    def run(self, reqs: list[EntryRequest], count: bool = True) -> list:
        """Execute entries in one native forward; returns RowResult / VerifyResult
        per request (in request order).  Requests with ``scratch`` get their rows'
        K/V in scratch cells; their cells are reported in ``result.scratch``."""
        n_e = len(reqs)
        if n_e == 0:
            return []
        if n_e == 1 and not reqs[0].scratch and len(reqs[0].batch) <= GRAPH_MAX_ROWS \
                and reqs[0].kind != _lib.ENTRY_PREFILL:
            return [self._run_one(reqs[0], count)]
        if n_e > self.max_entries:
            raise ValueError(f"{n_e} entries > engine max {self.max_entries}")
        G = self.shape.n_heads // self.shape.n_kv_heads
        # prefill-sized entries first (stable: the order of sorted() with a 0/1 key)
        lim = DECODE_MAX_ROWS // G
        order = [i for i, r in enumerate(reqs) if len(r.batch) > lim]
        if order:
            order += [i for i, r in enumerate(reqs) if len(r.batch) <= lim]
        else:
            order = list(range(n_e))
        # every per-entry column in ONE pass over the requests (a batched plan
        # has hundreds of entries: separate generator passes cost ~1 ms per forward)
        rs = [reqs[ri] for ri in order]
        PRE = _lib.ENTRY_PREFILL
        q_l, k_l, p_l, s_l, nd_l, h_l, final, tok_l = [], [], [], [], [], [], [], []
        hash_in = self._hash_in
        for r in rs:
            b = r.batch
            q, kd, pa, sq = len(b), r.kind, r.past, r.seq
            f = kd == PRE and pa + q == len(r.tokens)
            q_l.append(q)
            k_l.append(kd)
            p_l.append(pa)
            s_l.append(sq)
            final.append(f)
            # a chunk that ends its prompt (no generated token yet) also gets the
            # first decode step's proposal from the forward (n_draft = -1)
            nd_l.append(-1 if f else r.n_draft)
            h_l.append(hash_in(sq, pa, r.tokens))
            tok_l.extend(b)
        qs = np.array(q_l, dtype=np.int64)
        if n_e and qs.min() == 0:
            raise ValueError("batch must be non-empty")
        kinds = np.array(k_l, dtype=np.int64)
        pasts = np.array(p_l, dtype=np.int64)
        seqs = np.array(s_l, dtype=np.int64)
        n_outs = np.where(kinds == _lib.ENTRY_VERIFY, qs, 1)
        q_starts = np.concatenate(([0], np.cumsum(qs)[:-1]))
        out_starts = np.concatenate(([0], np.cumsum(n_outs)[:-1]))
        q_start, out_start = int(qs.sum()), int(n_outs.sum())
        if q_start > self.max_rows or out_start > self.max_out:
            raise ValueError("forward exceeds engine buffers")
        ents = np.zeros(n_e, dtype=_ENTRY_DT)
        ents["seq"], ents["past"], ents["q_len"], ents["q_start"] = seqs, pasts, qs, q_starts
        ents["kind"], ents["out_start"], ents["n_out"] = kinds, out_starts, n_outs
        ents["n_draft"] = nd_l
        ents["hash_in"] = np.array(h_l, dtype=np.uint64)
        row_entry = np.repeat(np.arange(n_e), qs)
        row_in = np.arange(q_start) - np.repeat(q_starts, qs)  # row index within its entry
        toks = [np.asarray(tok_l, dtype=np.int32)]
        rseq = [seqs[row_entry].astype(np.int32)]
        rpos = [(pasts[row_entry] + row_in).astype(np.int32)]
        # sampled rows: the last n_out rows of every entry
        orow = [np.nonzero(row_in >= (qs - n_outs)[row_entry])[0].astype(np.int32)]
        scratch_ops, scratch_of, s_off = [], {}, 0
        for i, ri in enumerate(order):
            r = rs[i]
            if r.scratch:
                q = int(qs[i])
                if s_off + q > self.n_scratch:
                    raise ValueError("scratch cells exhausted")
                cell = self.capacity + s_off
                scratch_ops.append((_lib.KV_MAP_SCRATCH, r.seq, r.past, cell, q))
                scratch_of[ri] = list(range(cell, cell + q))
                s_off += q
        if count:
            for q in qs.tolist():
                self.ledger.count_forward(q)
        st = self.stage
        st.reset()
        if q_start <= GRAPH_MAX_ROWS or n_e == 1:
            # the forward's arguments at fixed offsets (first in the buffer), so
            # the native runtime can replay its captured CUDA graph: a compact
            # layout for decode / verify, a max-rows one for a prefill chunk
            rows = GRAPH_MAX_ROWS if q_start <= GRAPH_MAX_ROWS else self.max_rows
            o_ent = st.add_fixed(ents.view(np.int32), GRAPH_MAX_ROWS * _ENTRY_DT.itemsize // 4)
            o_tok = st.add_fixed(np.concatenate(toks), rows)
            o_seq = st.add_fixed(np.concatenate(rseq), rows)
            o_pos = st.add_fixed(np.concatenate(rpos), rows)
            o_out = st.add_fixed(np.concatenate(orow), GRAPH_MAX_ROWS if rows == GRAPH_MAX_ROWS
                                 else self.max_out)
            meta = self._stage_metadata(scratch_ops)
        else:
            meta = self._stage_metadata(scratch_ops)
            o_ent = st.add(ents.view(np.int32))
            o_tok = st.add(np.concatenate(toks))
            o_seq = st.add(np.concatenate(rseq))
            o_pos = st.add(np.concatenate(rpos))
            o_out = st.add(np.concatenate(orow))
        st.upload()
        self.h2d_bytes += 4 * st.n
        stream = torch.cuda.current_stream()
        sp = stream.cuda_stream
        self._ev[0].record(stream)  # device time includes the metadata kernels
        self._apply_metadata(*meta, sp)
        res = self.res_dev
        # the next proposal of every decode / verify entry and prompt-ending
        # chunk rides in the same launch (other prefill chunks: empty ring)
        nd = self.fused_drafts and any(r.kind != _lib.ENTRY_PREFILL for r in reqs) or \
            (self.fused_drafts and any(final))
        args = _lib.ForwardArgs(
            n_e, q_start, out_start, self.policy, self.cfg.copy_min_match, self.cfg.vocab,
            st.hptr(o_ent), st.dptr(o_ent), st.dptr(o_tok), st.dptr(o_seq), st.dptr(o_pos),
            st.dptr(o_out), res.data_ptr(), res.data_ptr() + 4 * self.max_out,
            res.data_ptr() + 8 * self.max_out, self.logits.data_ptr(),
            self.workspace.data_ptr(), self.workspace.numel(),
            self.cfg.spec_buffer if nd else 0, self.cfg.spec_min_match, self.nd_cap if nd else 0,
            res.data_ptr() + 4 * self.nd_off, int(self.keep_logits))
        check(lib().ds_model_forward(ctypes.byref(self.model_c), ctypes.byref(self.kv_c),
                                     ctypes.byref(args), sp), "ds_model_forward")
        self.gpu_launches += self.launches_per_forward(reqs)
        self._ev[1].record(stream)
        self.res_host.copy_(res, non_blocking=True)
        self.d2h_bytes += 4 * res.numel()
        stream.synchronize()
        kind = "prefill" if any(r.kind == _lib.ENTRY_PREFILL for r in reqs) else "decode"
        f = self._fwd[kind]
        f[0] += 1
        f[1] += self._ev[0].elapsed_time(self._ev[1]) / 1000.0
        f[2] += q_start
        f[3] += int(pasts.sum()) + q_start
        h = self.res_host.numpy()
        tok, src, acc = h[: self.max_out], h[self.max_out: 2 * self.max_out], h[2 * self.max_out:]
        if nd:  # cache the proposals for the token lists the scheduler will hold next
            o = self.nd_off
            dlen = h[o + 2 * n_e: o + 3 * n_e].tolist()
            d0 = o + 3 * n_e
            cap = self.nd_cap
            acc_l = acc[:n_e].tolist()
            dc = self._draft_cache
            for i, r in enumerate(rs):
                if r.kind == _lib.ENTRY_PREFILL:
                    if final[i]:
                        dc[r.seq] = (r.past + len(r.batch) + 1,
                                     h[d0 + i * cap: d0 + i * cap + dlen[i]].tolist())
                    continue
                a = acc_l[i] if r.kind == _lib.ENTRY_VERIFY else 0
                dc[r.seq] = (r.past + a + 2, h[d0 + i * cap: d0 + i * cap + dlen[i]].tolist())
        out = [None] * n_e
        tok_all, src_all = tok[:out_start].tolist(), src[:out_start].tolist()
        acc_all = acc[:n_e].tolist()
        for i, (ri, o0, n_out) in enumerate(zip(order, out_starts.tolist(), n_outs.tolist())):
            r = rs[i]
            rows = [RowResult(tok_all[o0 + j], None if src_all[o0 + j] < 0 else src_all[o0 + j])
                    for j in range(n_out)]
            res = VerifyResult(acc_all[i], rows) if r.kind == _lib.ENTRY_VERIFY else rows[0]
            if r.scratch:
                res.scratch = scratch_of[ri]
            out[ri] = res
        return out

    # fixed argument layout of forwards with <= GRAPH_MAX_ROWS rows (staging words)
    _FX_ENT, _FX_TOK, _FX_SEQ, _FX_POS, _FX_OUT, _FX_END = 0, 320, 352, 384, 416, 448

    def _run_one(self, r: EntryRequest, count: bool):
        """run() for one decode / verify entry - the steady-state hot call - with
        the arguments written straight into the pinned staging buffer at their
        fixed offsets (same layout as run()'s add_fixed path, so the captured
        CUDA graph is the same) and a cached argument struct."""
        q = len(r.batch)
        if q == 0:
            raise ValueError("batch must be non-empty")
        verify = r.kind == _lib.ENTRY_VERIFY
        n_out = q if verify else 1
        if count:
            self.ledger.count_forward(q)
        st = self.stage
        st.reset()
        st.n = self._FX_END
        meta = self._stage_metadata(None)
        st.ensure()
        hv = st.host_np
        hu = hv.view(np.uint32)
        h_in = self._hash_in(r.seq, r.past, r.tokens)
        hv[0:8] = (r.seq, r.past, q, 0, r.kind, r.n_draft, 0, n_out)
        hu[8] = h_in & 0xFFFFFFFF
        hu[9] = h_in >> 32
        t0 = self._FX_TOK
        hv[t0:t0 + q] = r.batch
        hv[self._FX_SEQ:self._FX_SEQ + q] = r.seq
        hv[self._FX_POS:self._FX_POS + q] = np.arange(r.past, r.past + q, dtype=np.int32)
        hv[self._FX_OUT:self._FX_OUT + n_out] = np.arange(q - n_out, q, dtype=np.int32)
        st.upload()
        self.h2d_bytes += 4 * st.n
        stream = torch.cuda.current_stream()
        sp = stream.cuda_stream
        self._ev[0].record(stream)  # device time includes the metadata kernels
        self._apply_metadata(*meta, sp)
        res = self.res_dev
        nd = self.fused_drafts
        fa = getattr(self, "_fargs", None)
        if fa is None or self._fargs_key != (st.dev.data_ptr(), st.host.data_ptr()):
            fa = _lib.ForwardArgs(
                1, q, n_out, self.policy, self.cfg.copy_min_match, self.cfg.vocab,
                st.hptr(self._FX_ENT), st.dptr(self._FX_ENT), st.dptr(self._FX_TOK),
                st.dptr(self._FX_SEQ), st.dptr(self._FX_POS), st.dptr(self._FX_OUT),
                res.data_ptr(), res.data_ptr() + 4 * self.max_out,
                res.data_ptr() + 8 * self.max_out, self.logits.data_ptr(),
                self.workspace.data_ptr(), self.workspace.numel(), 0, self.cfg.spec_min_match,
                0, res.data_ptr() + 4 * self.nd_off, int(self.keep_logits))
            self._fargs, self._fargs_key = fa, (st.dev.data_ptr(), st.host.data_ptr())
            self._fargs_ref = ctypes.byref(fa)
        fa.n_rows = q
        fa.n_out = n_out
        fa.logits_out = int(self.keep_logits)
        fa.next_window = self.cfg.spec_buffer if nd else 0
        fa.next_cap = self.nd_cap if nd else 0
        check(lib().ds_model_forward(self._model_ref, self._kv_ref, self._fargs_ref, sp),
              "ds_model_forward")
        self.gpu_launches += self.launches_per_forward([r])
        self._ev[1].record(stream)
        self.res_host.copy_(res, non_blocking=True)
        self.d2h_bytes += 4 * res.numel()
        stream.synchronize()
        f = self._fwd["decode"]
        f[0] += 1
        f[1] += self._ev[0].elapsed_time(self._ev[1]) / 1000.0
        f[2] += q
        f[3] += r.past + q
        h = self.res_host.numpy()
        tok, src = h[:n_out], h[self.max_out:self.max_out + n_out]
        acc = int(h[2 * self.max_out]) if verify else 0
        if nd:
            o = self.nd_off
            self._draft_cache[r.seq] = (r.past + acc + 2,
                                        h[o + 3: o + 3 + int(h[o + 2])].tolist())
        rows = [RowResult(int(tok[j]), None if src[j] < 0 else int(src[j])) for j in range(n_out)]
        return VerifyResult(acc, rows) if verify else rows[0]

    def launches_per_forward(self, reqs) -> int:
        """Our kernels per ds_model_forward (cuBLAS GEMMs not counted): scatter,
        row-hash, embed; per layer 2 rmsnorm + rope/kv-store + attention (+combine)
        + silu_mul; final rmsnorm, token policy, verify-accept."""
        per_layer = 5 + (1 if any(r.past + len(r.batch) > 128 for r in reqs) else 0)
        return 3 + self.shape.layers * per_layer + 3

    # convenience wrappers used by the scheduler (one entry per call)
    def forward_prefill(self, seq, past, batch, tokens) -> RowResult:
        return self.run([EntryRequest(_lib.ENTRY_PREFILL, seq, past, list(batch), tokens)])[0]

    def forward_decode(self, seq, past, token, tokens) -> RowResult:
        return self.run([EntryRequest(_lib.ENTRY_DECODE, seq, past, [token], tokens)])[0]

    def forward_verify(self, seq, past, batch, tokens, hash_in=None) -> VerifyResult:
        return self.run([EntryRequest(_lib.ENTRY_VERIFY, seq, past, list(batch), tokens,
                                      n_draft=len(batch) - 1)])[0]

    # -- K1: batched prompt-lookup proposals -----------------------------------------

    def propose(self, slots: list[tuple[int, list, int]], window: int, min_match: int,
                use_cache: bool = True) -> list:
        """Drafts for many decoding slots in one launch.

        slots: (seq, tokens, cap) with tokens the full committed list (its last
        element is pending, not yet in the device history).  The ring is
        tokens[-window:] and the tail is the ring (scheduler.py:531-532).
        """
        n = len(slots)
        if n == 0:
            return []
        # proposals computed by the previous forward (the token list it assumed
        # is the one held now): a prefix of the max-cap draft, no launch
        out: list = [None] * n
        miss = []
        for i, (seq, tokens, cap) in enumerate(slots):
            hit = self._draft_cache.get(seq) if use_cache else None
            if hit is not None and hit[0] == len(tokens) and window == self.cfg.spec_buffer \
                    and min_match == self.cfg.spec_min_match and cap <= self.nd_cap:
                out[i] = hit[1][:cap]
            else:
                miss.append(i)
        if not miss:
            return out
        if len(miss) < n:
            sub = self.propose([slots[i] for i in miss], window, min_match, use_cache=False)
            for i, d in zip(miss, sub):
                out[i] = d
            return out
        for seq, tokens, _ in slots:
            self._pending_hist.append((seq, len(tokens) - 1, np.asarray(tokens[-1:], np.int32)))
        offs = np.zeros(n, dtype=np.int64)
        lens = np.zeros(n, dtype=np.int32)
        caps = np.zeros(n, dtype=np.int32)
        for i, (seq, tokens, cap) in enumerate(slots):
            ln = min(len(tokens), window)
            offs[i] = seq * self.pos_stride + len(tokens) - ln
            lens[i] = ln
            caps[i] = cap
        max_draft = max(1, int(caps.max()))
        st = self.stage
        st.reset()
        meta = self._stage_metadata()
        o_off = st.add(offs.view(np.int32))
        o_len = st.add(lens)
        o_cap = st.add(caps)
        st.upload()
        self.h2d_bytes += 4 * st.n
        stream = torch.cuda.current_stream()
        sp = stream.cuda_stream
        self._ev[0].record(stream)
        self._apply_metadata(*meta, sp)
        k1 = self.k1_dev
        need = 3 * n + n * max_draft
        if need > k1.numel():
            raise ValueError("too many slots for the K1 buffer")
        e_p, l_p, dl_p, d_p = (k1.data_ptr(), k1.data_ptr() + 4 * n, k1.data_ptr() + 8 * n,
                               k1.data_ptr() + 12 * n)
        hp = self.hist.data_ptr()
        check(lib().ds_longest_suffix_match(hp, st.dptr(o_off), st.dptr(o_len), hp,
                                            st.dptr(o_off), st.dptr(o_len), n, min_match,
                                            st.dptr(o_cap), max_draft, e_p, l_p, d_p, dl_p, sp),
              "ds_longest_suffix_match")
        self.gpu_launches += 1
        self._ev[1].record(stream)
        self.k1_host[:need].copy_(k1[:need], non_blocking=True)
        self.d2h_bytes += 4 * need
        stream.synchronize()
        f = self._fwd["propose"]
        f[0] += 1
        f[1] += self._ev[0].elapsed_time(self._ev[1]) / 1000.0
        h = self.k1_host.numpy()
        dl = h[2 * n: 3 * n]
        d = h[3 * n: 3 * n + n * max_draft].reshape(n, max_draft)
        return [d[i, : dl[i]].tolist() for i in range(n)]

    # -- prefix migration payload (dist.py) ------------------------------------------

    def _cells_dev(self, cells) -> torch.Tensor:
        return torch.as_tensor(np.asarray(cells, dtype=np.int32)).to(self.device,
                                                                    non_blocking=False)

    def pack_cells(self, cells) -> torch.Tensor:
        """K/V rows of `cells` (all layers) as one [L][2][nkv][n][hd] bf16 buffer
        (ds_kv_pack_cells); the message a prefix migration sends."""
        s = self.shape
        n = len(cells)
        buf = torch.empty((s.layers, 2, s.n_kv_heads, n, s.head_dim), dtype=torch.bfloat16,
                          device=self.device)
        self.flush()  # pending row copies land before the rows are read
        cd = self._cells_dev(cells)
        stream = torch.cuda.current_stream().cuda_stream
        check(lib().ds_kv_pack_cells(self.k_pool.data_ptr(), self.v_pool.data_ptr(), s.layers,
                                     s.n_kv_heads, self.head_stride, s.head_dim, cd.data_ptr(), n,
                                     buf.data_ptr(), 0, stream), "ds_kv_pack_cells")
        self.gpu_launches += 1
        return buf

    def unpack_cells(self, cells, buf: torch.Tensor) -> None:
        """Scatter a received [L][2][nkv][n][hd] buffer into `cells`."""
        s = self.shape
        n = len(cells)
        if tuple(buf.shape) != (s.layers, 2, s.n_kv_heads, n, s.head_dim) or \
                buf.dtype != torch.bfloat16 or not buf.is_contiguous():
            raise ValueError(f"migration payload shape {tuple(buf.shape)} does not match "
                             f"{n} cells")
        cd = self._cells_dev(cells)
        stream = torch.cuda.current_stream().cuda_stream
        check(lib().ds_kv_pack_cells(self.k_pool.data_ptr(), self.v_pool.data_ptr(), s.layers,
                                     s.n_kv_heads, self.head_stride, s.head_dim, cd.data_ptr(), n,
                                     buf.data_ptr(), 1, stream), "ds_kv_pack_cells")
        self.gpu_launches += 1

    def payload_buffer(self, n: int) -> torch.Tensor:
        s = self.shape
        return torch.empty((s.layers, 2, s.n_kv_heads, n, s.head_dim), dtype=torch.bfloat16,
                           device=self.device)

    # -- diagnostics -------------------------------------------------------------------

    def device_refcounts(self) -> tuple[np.ndarray, int]:
        """map_ref+trie_ref per cell (page-table mappings + radix holds) and the
        device occupancy."""
        self.flush()
        rc = torch.empty(self.capacity, dtype=torch.int32, device=self.device)
        occ = torch.zeros(1, dtype=torch.int32, device=self.device)
        check(lib().ds_kv_refcount(self.member.data_ptr(), self.mask_words,
                                   self.trie_ref.data_ptr(), self.map_ref.data_ptr(),
                                   self.capacity, rc.data_ptr(),
                                   occ.data_ptr(), torch.cuda.current_stream().cuda_stream),
              "ds_kv_refcount")
        return rc.cpu().numpy(), int(occ.item())

    def device_cells(self, seq: int, n: int) -> list[int]:
        self.flush()
        return self.pos2cell[seq, :n].cpu().tolist()

    def weights_cpu(self) -> dict:
        return {k: v.float().cpu() for k, v in self.w.items()}
