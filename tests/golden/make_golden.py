"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run here (the reference exists only in this container):

    bash oracle/build_ref.sh && python tests/golden/make_golden.py

It imports the unmodified reference (``deltaserve`` built into oracle/_ref from
/root/reference/pkg) and records its outputs on seeded inputs:

* ``kernels.json``   - FNV-1a 32/64, copy_continuation, longest_suffix_match,
                       lookup_ngram and copy-policy rows
                       (reference: _kernels/_native.pyx:18-119, engine.py:196-216,
                       speculator.py:52-65).
* ``kvcache_ops.json`` - random UnifiedKvCache op sequences with every observable
                       after each op (kvcache.py:71-293).
* ``radix_ops.json``  - random RadixTrie save/lookup/evict sequences (radix.py:81-222).
* ``traces/*.json.gz`` - scenario transcripts driven through the reference
                       ``InferenceCore`` (scheduler.py) for BASELINE configs C1-C5:
                       every request's prompt (delta coded), pieces, parameters and
                       the reference's result counters; used both for transcript
                       parity and as the bench workload.

The fixtures are committed; nothing on the GPU box reads /root/reference.
"""
from __future__ import annotations

import gzip
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

import numpy as np  # noqa: E402

from deltaserve import _kernels as K  # noqa: E402
from deltaserve.caches import prompt_seed  # noqa: E402
from deltaserve.config import ServerConfig  # noqa: E402
from deltaserve.engine import MockEngine, ModelConfig  # noqa: E402
from deltaserve.kvcache import CapacityExhausted, DonorRangeInvalid, UnifiedKvCache  # noqa: E402
from deltaserve.radix import BudgetExceeded, RadixTrie  # noqa: E402
from deltaserve.scenarios import (  # noqa: E402
    Scenario,
    agent_scenario,
    agentic_6turn,
    burst_prompts,
    deep_workflow,
    turn_tool_result,
)
from deltaserve.scheduler import (  # noqa: E402
    GenerationRequest, InferenceCore, RequestHandle, SessionHandle)
from deltaserve.speculator import lookup_ngram  # noqa: E402

assert K.BACKEND == "native"


def dump(name, obj, gz=False):
    path = os.path.join(HERE, name)
    os.makedirs(os.path.dirname(path), exist_ok=True)
    data = json.dumps(obj, separators=(",", ":")).encode()
    if gz:
        with gzip.GzipFile(path, "wb", mtime=0) as fh:
            fh.write(data)
    else:
        with open(path, "wb") as fh:
            fh.write(data)
    print(f"wrote {path} ({len(data)} bytes raw)")


# ---------------------------------------------------------------------------
# kernels
# ---------------------------------------------------------------------------

def rand_tokens(rng, n, alpha):
    return [rng.randrange(alpha) for _ in range(n)]


def gen_kernels():
    rng = random.Random(20251017)
    out = {"fnv_bytes": [], "fnv_tokens": [], "copy_continuation": [], "suffix_match": [],
           "lookup_ngram": [], "copy_policy": []}
    for data in [b"", b"a", b"hello world", bytes(range(256)), b'{"name"']:
        out["fnv_bytes"].append({"hex": data.hex(), "f32": K.fnv1a32_bytes(data),
                                 "f64": K.fnv1a64_bytes(data)})
    tok_cases = [[], [1], [70000], [-1, 0, 2**31 - 1, -2**31], [5, 6, 7, 5, 6]]
    for _ in range(60):
        tok_cases.append(rand_tokens(rng, rng.randrange(0, 300), rng.choice([8, 1000, 2**31 - 1])))
    for toks in tok_cases:
        st32 = rng.randrange(2**32)
        st64 = rng.randrange(2**64)
        out["fnv_tokens"].append({
            "tokens": toks, "f32": K.fnv1a32_tokens(toks), "f64": K.fnv1a64_tokens(toks),
            "state32": st32, "f32s": K.fnv1a32_tokens(toks, st32),
            "state64": st64, "f64s": K.fnv1a64_tokens(toks, st64)})
    # copy_continuation: known answer + random (sizes up to 4096)
    cc = [([5, 6, 7, 5, 6], 2), ([], 3), ([1, 2, 3], 3), ([1, 1, 1, 1], 0), ([7, 8, 9, 7, 8], 2)]
    for _ in range(400):
        n = rng.randrange(0, 48)
        cc.append((rand_tokens(rng, n, rng.choice([2, 3, 5, 8])), rng.randrange(1, 6)))
    for _ in range(40):
        n = rng.randrange(100, 4097)
        cc.append((rand_tokens(rng, n, rng.choice([4, 16, 64, 30000])), rng.randrange(1, 5)))
    for toks, mm in cc:
        out["copy_continuation"].append({"tokens": toks, "mm": mm,
                                         "e": K.copy_continuation(toks, mm)})
    # longest_suffix_match: self (ring == tail, as the scheduler uses it) + separate tails
    sm = [([10, 20, 30, 40, 10, 20], None, 2), ([1, 2, 3, 4, 5, 6], None, 3),
          ([1, 2, 7, 5, 1, 2, 9, 6, 1, 2], None, 2), ([4, 1, 2, 8, 8, 1, 2, 5, 4, 1, 2], None, 2)]
    for _ in range(400):
        ring = rand_tokens(rng, rng.randrange(0, 48), rng.choice([2, 3, 5, 8]))
        tail = None if rng.random() < 0.6 else rand_tokens(rng, rng.randrange(0, 20), 4)
        sm.append((ring, tail, rng.randrange(1, 5)))
    for _ in range(60):
        n = rng.choice([2048, rng.randrange(64, 2049)])
        ring = rand_tokens(rng, n, rng.choice([3, 16, 64, 30000]))
        if rng.random() < 0.5:  # plant long repeats the way agentic copies look
            span = ring[: rng.randrange(8, 64)]
            pos = rng.randrange(0, max(1, n - len(span)))
            ring[pos:pos + len(span)] = span
            ring[-len(span) // 2:] = span[: len(span) // 2]
            ring = ring[:n]
        sm.append((ring, None, rng.choice([1, 2, 3, 4])))
    for ring, tail, lmin in sm:
        t = ring if tail is None else tail
        e, ln = K.longest_suffix_match(ring, t, lmin)
        out["suffix_match"].append({"ring": ring, "tail": tail, "min_len": lmin, "e": e, "len": ln})
    # lookup_ngram known answers (test_speculator.py:22-46) + random with caps
    ln_cases = [([10, 20, 30, 40, 10, 20], 2, 2), ([1, 2, 3, 4, 5, 6], 3, 8),
                ([1, 2, 7, 5, 1, 2, 9, 6, 1, 2], 2, 1), ([4, 1, 2, 8, 8, 1, 2, 5, 4, 1, 2], 2, 1),
                ([1, 2, 3, 4, 5, 1, 2], 2, 2), ([1, 2, 1, 2], 2, 0)]
    for _ in range(200):
        ln_cases.append((rand_tokens(rng, rng.randrange(0, 40), rng.choice([2, 3, 6])),
                         rng.randrange(1, 4), rng.randrange(0, 18)))
    for ring, mm, cap in ln_cases:
        out["lookup_ngram"].append({"ring": ring, "mm": mm, "cap": cap,
                                    "draft": lookup_ngram(ring, ring, mm, cap)})
    # copy policy rows via the reference MockEngine forward (engine.py:268-281, 196-216)
    for vocab, mm in [(32768, 3), (32768, 2), (1000, 3)]:
        eng = MockEngine(ModelConfig(vocab=vocab, copy_min_match=mm))
        for _ in range(60):
            n = rng.randrange(1, 300)
            alpha = rng.choice([3, 20, 5000])
            full = rand_tokens(rng, n, alpha)
            c = rng.randrange(0, n)
            lb = eng.forward(full[:c], full[c:])
            rows = []
            for i in range(len(lb)):
                lg = lb[i]
                rows.append([lg.argmax_id, -1 if lg.copy_source is None else lg.copy_source])
            out["copy_policy"].append({"vocab": vocab, "mm": mm, "full": full, "ctx": c,
                                       "rows": rows})
    # test_engine.py:127-141 known answers
    eng = MockEngine(ModelConfig(copy_min_match=2))
    lb = eng.forward([7, 8, 9], [7, 8])
    out["copy_policy"].append({"vocab": 32768, "mm": 2, "full": [7, 8, 9, 7, 8], "ctx": 3,
                               "rows": [[lb[i].argmax_id, -1 if lb[i].copy_source is None
                                         else lb[i].copy_source] for i in range(2)]})
    dump("kernels.json.gz", out, gz=True)


# ---------------------------------------------------------------------------
# kv cache and radix op sequences
# ---------------------------------------------------------------------------

def kv_observe(kv, seqs):
    obs = {"occ": kv.occupancy, "free": kv.free_cells, "seqs": {}}
    for s in seqs:
        n = kv.seq_len(s)
        if n:
            obs["seqs"][str(s)] = {"len": n, "spans": kv.span_count(s), "cells": kv.cell_ids(s, 0, n)}
    obs["ref"] = {str(int(c)): int(kv._refcnt[c]) for c in np.flatnonzero(kv._refcnt)}
    return obs


def gen_kvcache():
    rng = random.Random(7)
    runs_out = []
    for case in range(60):
        cap = rng.choice([64, 128, 256])
        kv = UnifiedKvCache(cap)
        seqs = list(range(6))
        ops = []
        for _ in range(rng.randrange(10, 60)):
            kind = rng.choice(["append", "append", "append", "trim", "alias", "alias_runs",
                               "release", "decref"])
            s = rng.choice(seqs)
            op = {"op": kind, "seq": s}
            try:
                if kind == "append":
                    op["n"] = rng.randrange(1, 40)
                    op["ret"] = list(kv.append_cells(s, op["n"]))
                elif kind == "trim":
                    op["pos"] = rng.randrange(0, kv.seq_len(s) + 2)
                    op["ret"] = kv.trim(s, op["pos"])
                elif kind == "alias":
                    d = rng.choice(seqs)
                    op["dest"] = d
                    op["start"] = kv.seq_len(d) if rng.random() < 0.8 else rng.randrange(0, 5)
                    op["end"] = op["start"] + rng.randrange(0, max(1, kv.seq_len(s) + 3 - op["start"]))
                    kv.seq_alias(s, d, op["start"], op["end"])
                elif kind == "alias_runs":
                    n = kv.seq_len(s)
                    if n == 0:
                        op["runs"] = []
                    else:
                        a = rng.randrange(0, n)
                        b = rng.randrange(a, n + 1)
                        op["runs"] = [list(r) for r in kv.resolve_runs(s, a, b)]
                    d = rng.choice(seqs)
                    op["dest"] = d
                    kv.alias_runs(d, [tuple(r) for r in op["runs"]])
                    kv.incref_runs([tuple(r) for r in op["runs"]])  # mimic a radix hold
                    op["held"] = True
                elif kind == "decref":
                    n = kv.seq_len(s)
                    op["runs"] = [list(r) for r in kv.resolve_runs(s, 0, n)] if n and rng.random() < 0.3 else []
                    op["ret"] = kv.decref_runs([tuple(r) for r in op["runs"]])
                else:
                    op["ret"] = kv.release_sequence(s)
                op["err"] = None
            except CapacityExhausted:
                op["err"] = "CapacityExhausted"
            except DonorRangeInvalid:
                op["err"] = "DonorRangeInvalid"
            except ValueError:
                op["err"] = "ValueError"
            op["obs"] = kv_observe(kv, seqs)
            ops.append(op)
        runs_out.append({"capacity": cap, "ops": ops})
    dump("kvcache_ops.json.gz", runs_out, gz=True)


def gen_radix():
    rng = random.Random(11)
    out = []
    for case in range(40):
        cap = 512
        kv = UnifiedKvCache(cap)
        trie = RadixTrie(kv, cell_budget=rng.choice([64, 128, 256]))
        ops = []
        bases = [rand_tokens(rng, rng.randrange(5, 40), 50) for _ in range(3)]
        for step in range(rng.randrange(5, 30)):
            kind = rng.choice(["save", "save", "lookup", "lookup", "evict", "release"])
            s = rng.randrange(4)
            op = {"op": kind, "seq": s}
            try:
                if kind == "save":
                    toks = list(rng.choice(bases))[: rng.randrange(1, 41)] + rand_tokens(
                        rng, rng.randrange(0, 20), 50)
                    held = kv.seq_len(s)
                    if held < len(toks):
                        kv.append_cells(s, len(toks) - held)
                    op["tokens"] = toks
                    op["ret"] = trie.save(toks, s, 0)
                elif kind == "lookup":
                    toks = list(rng.choice(bases))[: rng.randrange(0, 41)] + rand_tokens(
                        rng, rng.randrange(0, 5), 50)
                    m = trie.longest_prefix(toks)
                    op["tokens"] = toks
                    op["ret"] = {"length": m.length, "runs": [list(r) for r in m.runs],
                                 "donor": m.donor}
                elif kind == "evict":
                    op["n"] = rng.randrange(1, 80)
                    op["ret"] = trie.evict(op["n"])
                else:
                    op["ret"] = kv.release_sequence(s)
                op["err"] = None
            except BudgetExceeded:
                op["err"] = "BudgetExceeded"
            except CapacityExhausted:
                op["err"] = "CapacityExhausted"
            op["dump"] = trie.dump()
            op["cells"] = trie.total_cells
            op["occ"] = kv.occupancy
            op["evicted_total"] = trie.evicted_cells_total
            ops.append(op)
        out.append({"budget": trie.cell_budget, "ops": ops})
    dump("radix_ops.json.gz", out, gz=True)


# ---------------------------------------------------------------------------
# scenario traces through the reference InferenceCore
# ---------------------------------------------------------------------------

RESULT_FIELDS = ("generated", "finish_reason", "n_t", "cached_prompt_tokens", "prefill_tokens",
                 "decode_passes", "spec_proposed", "spec_accepted", "spec_rejected",
                 "aliased_cells", "early_stopped", "text")


class Recorder:
    """Drives the reference core the way scenarios.run_core_scenario does, but
    records every request so a different engine can replay the same stream."""

    def __init__(self, core):
        self.core = core
        self.requests = []
        self.last_prompt = {}  # stream key -> (tokens, pieces) for delta coding
        self.wave = 0  # requests of one wave are submitted together, then run to completion
        self.chat = None  # (messages, tools) of the next submit, when recording chat input
        self.record_chat = False

    def submit(self, stream, tokens, pieces, max_tokens, tools, rid, session=None):
        # a session request holds no transient guard (server.py:300-318)
        guard = None if session is not None else self.core.pool.acquire("transient", timeout=1.0)
        declared = frozenset(t["function"]["name"] for t in tools if "function" in t)
        req = GenerationRequest(request_id=rid, prompt_tokens=list(tokens),
                                prompt_pieces=list(pieces), max_tokens=max_tokens,
                                temperature=0.0, seed=prompt_seed(tokens),
                                declared_tools=declared, guard=guard, session=session)
        h = RequestHandle(req)
        self.core.submit(h)
        prev_t, prev_p = self.last_prompt.get(stream, ([], []))
        c = 0
        while c < min(len(prev_t), len(tokens)) and prev_t[c] == tokens[c] and prev_p[c] == pieces[c]:
            c += 1
        self.last_prompt[stream] = (list(tokens), list(pieces))
        rec = {"id": rid, "wave": self.wave, "stream": stream, "common": c, "tokens": tokens[c:],
               "pieces": pieces[c:], "max_tokens": max_tokens, "tools": sorted(declared)}
        if session is not None:
            rec["session"] = session.session_id
        if self.record_chat and self.chat is not None:
            # the chat input the prompt was rendered + tokenized from
            # (scheduler.py:340-346), plus the caches' counters after it
            rec["messages"] = json.loads(json.dumps(self.chat[0]))
            rec["tool_defs"] = self.chat[1]
            rec["cache_stats"] = {"render": self.core.render_cache.stats(),
                                  "tokenize": self.core.tokenize_cache.stats()}
            self.chat = None
        self.requests.append((h, rec))
        return h

    def run_until_done(self, handles, max_iters=200_000):
        self.wave += 1
        pending = list(handles)
        for _ in range(max_iters):
            pending = [h for h in pending if not h.wait(timeout=0)]
            if not pending:
                return
            self.core.step()
        raise RuntimeError("unfinished")

    def finish_records(self):
        out = []
        for h, rec in self.requests:
            assert h.error is None, h.error
            r = h.result
            rec["expect"] = {f: getattr(r, f) for f in RESULT_FIELDS}
            rec["expect"]["finalize"] = r.finalize.kind
            out.append(rec)
        return out


def assistant_content(result):
    fin = result.finalize
    if fin.kind == "tool_calls":
        return "\n".join(json.dumps({"name": c.name, "parameters": c.parameters},
                                    separators=(",", ":")) for c in fin.calls)
    return result.text


class Conv:
    def __init__(self, sc: Scenario):
        self.sc = sc
        self.messages = [{"role": "system", "content": sc.system}]

    def prompt(self, core, t, rec=None):
        self.messages.append({"role": "user", "content": self.sc.user_texts[t]})
        _, toks, pieces = core.prepare_prompt(self.messages, self.sc.tools)
        if rec is not None:
            rec.chat = (list(self.messages), self.sc.tools)
        return toks, pieces

    def after(self, t, result):
        self.messages.append({"role": "assistant", "content": assistant_content(result)})
        if t < len(self.sc.tool_results):
            self.messages.append({"role": "tool", "content": self.sc.tool_results[t]})


def core_snapshot(core):
    return {"ledger": core.engine.ledger.snapshot(), "occ": core.kv.occupancy,
            "radix_cells": core.radix.total_cells, "radix_dump": core.radix.dump(),
            "iterations": core.iterations}


def trace_sequential(name, cfg_over, scenarios, interleave=True, bursts=(), chat=False):
    """Conversations turn by turn (interleaved A1 B1 C1 A2 ...), each turn run to
    completion; then optional bursts of concurrent single-turn requests.
    chat=True also records each request's chat messages / tools and the
    render / tokenize cache counters (host front-end parity)."""
    core = InferenceCore(ServerConfig(**cfg_over))
    rec = Recorder(core)
    rec.record_chat = chat
    convs = [Conv(sc) for sc in scenarios]
    turns = max(sc.turn_count for sc in scenarios)
    order = ([(t, i) for t in range(turns) for i in range(len(convs))] if interleave
             else [(t, i) for i in range(len(convs)) for t in range(turns)])
    snaps = []
    for t, i in order:
        conv = convs[i]
        if t >= conv.sc.turn_count:
            continue
        toks, pieces = conv.prompt(core, t, rec)
        h = rec.submit(f"s{i}", toks, pieces, conv.sc.max_tokens, conv.sc.tools,
                       f"{conv.sc.name}-t{t}")
        rec.run_until_done([h])
        conv.after(t, h.result)
        snaps.append(core_snapshot(core))
    for bsalt, width in bursts:
        system, tools, texts = burst_prompts(bsalt, width)
        handles = []
        for w, text in enumerate(texts):
            msgs = [{"role": "system", "content": system}, {"role": "user", "content": text}]
            _, toks, pieces = core.prepare_prompt(msgs, tools)
            rec.chat = (msgs, tools)
            handles.append(rec.submit(f"b{w}", toks, pieces, 80, tools, f"burst-{bsalt}-{w}"))
        rec.run_until_done(handles)
        snaps.append(core_snapshot(core))
    return {"name": name, "config": cfg_over, "mode": "sequential", "interleave": interleave,
            "requests": rec.finish_records(), "snapshots": snaps}


def trace_sessions(name, cfg_over, scenarios, session_convs):
    """Session path (server.py:367-387): conversations in
    `session_convs` run on a session-pool sequence bound once (POST
    /v1/sessions) - admission matches against session.tokens, trims the KV
    to the match and prefills only the delta (scheduler.py:431-458); the
    others are transient requests (radix path).  Turns interleaved; at the
    end every session is deleted (kv.release_sequence + guard.release)."""
    core = InferenceCore(ServerConfig(**cfg_over))
    rec = Recorder(core)
    convs = [Conv(sc) for sc in scenarios]
    sessions = {i: SessionHandle(session_id=f"sess-{i}", guard=core.pool.acquire("session"))
                for i in session_convs}
    snaps = []
    for t in range(max(sc.turn_count for sc in scenarios)):
        for i, conv in enumerate(convs):
            if t >= conv.sc.turn_count:
                continue
            toks, pieces = conv.prompt(core, t)
            h = rec.submit(f"s{i}", toks, pieces, conv.sc.max_tokens, conv.sc.tools,
                           f"{conv.sc.name}-c{i}-t{t}", session=sessions.get(i))
            rec.run_until_done([h])
            conv.after(t, h.result)
            snaps.append(core_snapshot(core))
    for i in sorted(sessions):
        core.kv.release_sequence(sessions[i].guard.seq)
        sessions[i].guard.release()
    snaps.append(core_snapshot(core))
    return {"name": name, "config": cfg_over, "mode": "sessions",
            "sessions": [sessions[i].session_id for i in sorted(sessions)],
            "requests": rec.finish_records(), "snapshots": snaps}


def trace_waves(name, cfg_over, scenarios):
    """Turn-synchronous waves: turn t of every session submitted together (C5)."""
    core = InferenceCore(ServerConfig(**cfg_over))
    rec = Recorder(core)
    convs = [Conv(sc) for sc in scenarios]
    snaps = []
    for t in range(max(sc.turn_count for sc in scenarios)):
        handles = []
        for i, conv in enumerate(convs):
            toks, pieces = conv.prompt(core, t)
            handles.append(rec.submit(f"s{i}", toks, pieces, conv.sc.max_tokens, conv.sc.tools,
                                      f"{conv.sc.name}-t{t}"))
        rec.run_until_done(handles)
        for conv, h in zip(convs, handles):
            conv.after(t, h.result)
        snaps.append(core_snapshot(core))
    return {"name": name, "config": cfg_over, "mode": "waves",
            "requests": rec.finish_records(), "snapshots": snaps}


def trace_failures(name, cfg_over, total=1000, seed=3, vocab_cap=30000):
    """Acceptance c11 (tests/test_acceptance.py:314-341): 1000 requests in waves
    of 10, ~10% with an injected fault after 1-3 tokens (InjectedFault ->
    _fail_slot, scheduler.py:630-634, 853-867).  Same rng call sequence as the
    reference test; prompt ids are folded into the vocabulary
    (`% vocab_cap`) so a real embedding table can serve them.  Every request's
    outcome (result fields, or failed) plus the pool / KV / radix state after
    each wave are recorded."""
    core = InferenceCore(ServerConfig(**cfg_over))
    rng = random.Random(seed)
    reqs, snaps, done, failures = [], [], 0, 0
    wave_no = 0
    while done < total:
        wave = []
        for _ in range(min(10, total - done)):
            inject = rng.random() < 0.10
            fail_after = rng.randint(1, 3) if inject else None
            failures += bool(inject)
            base = (rng.randint(1, 1_000_000) * 30) % vocab_cap
            toks = [(base + i) % vocab_cap for i in range(rng.randint(4, 24))]
            rid = f"s{done + len(wave)}"
            max_tokens = rng.randint(1, 6)
            guard = core.pool.acquire("transient", timeout=1.0)
            req = GenerationRequest(request_id=rid, prompt_tokens=list(toks),
                                    prompt_pieces=[f" w{t}" for t in toks], max_tokens=max_tokens,
                                    temperature=0.0, seed=prompt_seed(toks), guard=guard,
                                    fail_after_tokens=fail_after)
            h = RequestHandle(req)
            core.submit(h)
            wave.append(h)
            reqs.append((h, {"id": rid, "wave": wave_no, "stream": rid, "common": 0,
                             "tokens": toks, "pieces": [f" w{t}" for t in toks],
                             "max_tokens": max_tokens, "tools": [], "fail_after": fail_after}))
        pending = list(wave)
        while pending:
            core.step()
            pending = [h for h in pending if not h.wait(timeout=0)]
        done += len(wave)
        wave_no += 1
        snap = core_snapshot(core)
        snap["pool"] = core.pool.free_counts()
        snaps.append(snap)
    assert failures > total // 20  # the ~10% injection actually happened
    for snap in snaps[:-1]:  # the full radix dump only at the end (fixture size)
        snap.pop("radix_dump")
    assert core.pool.free_counts() == {"transient": 12, "session": 4}
    assert core.kv.occupancy == core.radix.total_cells
    out = []
    for h, rec in reqs:
        if h.error is not None:
            rec["expect"] = {"failed": type(h.error).__name__}
        else:
            rec["expect"] = {f: getattr(h.result, f) for f in RESULT_FIELDS}
            rec["expect"]["finalize"] = h.result.finalize.kind
        out.append(rec)
    return {"name": name, "config": cfg_over, "mode": "waves", "requests": out,
            "snapshots": snaps, "failures": failures}


def deep_c4(salt, turns, pieces=820):
    sc = deep_workflow(salt, turns)
    sc.tool_results = [turn_tool_result(salt, t, pieces=pieces) for t in range(turns)]
    sc.max_tokens = 128
    return sc


def gen_traces():
    c2 = agentic_6turn("c2")
    traces = [
        trace_sequential("c1", {}, [agent_scenario("travel", "c1")], chat=True),
        trace_sequential("c2", {"spec_max_lookahead": 4}, [c2], chat=True),
        trace_sequential("c2_nospec", {"spec_max_lookahead": 4, "speculation_enabled": False}, [c2]),
        trace_sequential("c3", {"pool_transient": 16},
                         [deep_workflow(s, 5) for s in ("c3a", "c3b", "c3c")],
                         bursts=[("c3burst", 16)], chat=True),
        trace_sequential("c3_nogroup", {"pool_transient": 16, "grouping_enabled": False},
                         [deep_workflow(s, 5) for s in ("c3a", "c3b", "c3c")],
                         bursts=[("c3burst", 16)]),
        trace_sequential("c4_small", {"spec_max_lookahead": 4, "capacity_cells": 65536},
                         [deep_c4("c4s", 8, pieces=200)]),
        trace_sequential("c4", {"spec_max_lookahead": 4, "capacity_cells": 262144},
                         [deep_c4("c4", 35)]),
        trace_sessions("sessions", {"spec_max_lookahead": 4, "radix_enabled": False},
                       [agentic_6turn("se1"), agentic_6turn("se2")], session_convs=(0, 1)),
        trace_sessions("sessions_radix", {"spec_max_lookahead": 4},
                       [agentic_6turn("sr1"), agentic_6turn("sr2"), agentic_6turn("sr1")],
                       session_convs=(0,)),
        trace_waves("c5_small", {"pool_transient": 8, "capacity_cells": 65536},
                    [agentic_6turn(f"c5s{i}") for i in range(8)]),
        trace_waves("c5", {"pool_transient": 256, "capacity_cells": 1 << 19},
                    [agentic_6turn(f"c5s{i}") for i in range(256)]),
        trace_failures("c11", {}),
        # the same under KV pressure: evictions and deferrals between faults
        trace_failures("c11_tight", {"capacity_cells": 256}, total=400, seed=11),
    ]
    only = [a for a in sys.argv[2:]] if len(sys.argv) > 2 and sys.argv[1] == "traces" else None
    for tr in traces:
        if only and tr["name"] not in only:
            continue
        n = len(tr["requests"])
        last = tr["requests"][-1]
        print(f"{tr['name']}: {n} requests, last n_t={last['expect'].get('n_t')}")
        dump(f"traces/{tr['name']}.json.gz", tr, gz=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["kernels", "kvcache", "radix", "traces"]
    if "kernels" in which:
        gen_kernels()
    if "kvcache" in which:
        gen_kvcache()
    if "radix" in which:
        gen_radix()
    if "traces" in which:
        gen_traces()
