"""Synthetic multi-turn workloads: replay of reference-generated traces.

The traces under tests/golden/traces/ were produced by driving the reference
InferenceCore with its own scenario generators (scenarios.py:121-188; see
tests/golden/make_golden.py).  Each request carries its full prompt token ids
and pieces (delta coded per conversation stream), its parameters, the wave it
was submitted in, and the reference's result counters.  Under the copy token
policy our engine regenerates the reference transcripts, so replaying the
recorded prompts is the same conversation; the recorded results are the
parity oracle.
"""
from __future__ import annotations

import gzip
import json
import os
import time
from dataclasses import dataclass

from .kernels import prompt_seed

TRACE_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                         "golden", "traces")

RESULT_FIELDS = ("generated", "finish_reason", "n_t", "cached_prompt_tokens", "prefill_tokens",
                 "decode_passes", "spec_proposed", "spec_accepted", "spec_rejected",
                 "aliased_cells", "early_stopped", "text")


@dataclass
class TraceRequest:
    id: str
    wave: int
    stream: str
    tokens: list
    pieces: list
    max_tokens: int
    tools: frozenset
    expect: dict
    session: str | None = None  # session id (session path) or None (transient + radix)
    fail_after: int | None = None  # injected fault after this many tokens (acceptance c11)
    messages: list | None = None   # chat input the prompt was rendered from (chat traces)
    tool_defs: list | None = None
    cache_stats: dict | None = None  # reference render / tokenize cache counters after it


def load_trace(name: str) -> dict:
    path = name if os.path.exists(name) else os.path.join(TRACE_DIR, f"{name}.json.gz")
    with gzip.open(path, "rb") as fh:
        tr = json.loads(fh.read())
    last: dict[str, tuple[list, list]] = {}
    reqs = []
    for r in tr["requests"]:
        pt, pp = last.get(r["stream"], ([], []))
        toks = pt[: r["common"]] + r["tokens"]
        pieces = pp[: r["common"]] + r["pieces"]
        last[r["stream"]] = (toks, pieces)
        reqs.append(TraceRequest(r["id"], r["wave"], r["stream"], toks, pieces, r["max_tokens"],
                                 frozenset(r["tools"]), r.get("expect", {}), r.get("session"),
                                 r.get("fail_after"), r.get("messages"), r.get("tool_defs"),
                                 r.get("cache_stats")))
    tr["reqs"] = reqs
    return tr


def waves(trace: dict) -> list[list[TraceRequest]]:
    out: dict[int, list] = {}
    for r in trace["reqs"]:
        out.setdefault(r.wave, []).append(r)
    return [out[k] for k in sorted(out)]


@dataclass
class TurnRecord:
    req: TraceRequest
    result: object
    latency_ms: float
    handle_error: Exception | None = None


class ChatMismatch(AssertionError):
    """prepare_prompt did not reproduce the reference's tokens / pieces."""


def replay(core, trace: dict, wave_limit: int | None = None, max_iters: int = 200_000,
           rid_suffix: str = "", via_chat: bool = False) -> list[TurnRecord]:
    """Submit each wave's requests together and step the core until they finish.
    Session traces (mode "sessions") bind one session per id first
    (`InferenceCore.open_session`, POST /v1/sessions) and delete them all after
    the last wave (`close_session`, DELETE /v1/sessions/{id}).

    via_chat: requests that carry their chat messages go through the host
    front end first - render + tokenize with the render / tokenize caches
    (InferenceCore.prepare_prompt, reference scheduler.py:340-346) - and the
    turn latency starts before it; the produced ids / pieces must equal the
    reference's recorded prompt."""
    from .scheduler import GenerationRequest, RequestHandle

    records: list[TurnRecord] = []
    sessions = {sid: core.open_session(sid) for sid in trace.get("sessions", [])}
    for wi, wave in enumerate(waves(trace)):
        if wave_limit is not None and wi >= wave_limit:
            break
        handles = []
        for r in wave:
            session = sessions[r.session] if r.session is not None else None
            t_start = time.monotonic()
            tokens, pieces = r.tokens, r.pieces
            if via_chat and r.messages is not None:
                _, tokens, pieces = core.prepare_prompt(r.messages, r.tool_defs)
                if tokens != r.tokens or pieces != r.pieces:
                    raise ChatMismatch(f"{r.id}: front end produced a different prompt")
            guard = None if session is not None else core.pool.acquire("transient", timeout=1.0)
            req = GenerationRequest(request_id=r.id + rid_suffix, prompt_tokens=list(tokens),
                                    prompt_pieces=list(pieces), max_tokens=r.max_tokens,
                                    temperature=0.0, seed=prompt_seed(tokens),
                                    declared_tools=r.tools, guard=guard, session=session,
                                    fail_after_tokens=r.fail_after)
            h = RequestHandle(req)
            h.submitted_at = t_start  # the turn starts at its chat input
            core.submit(h)
            handles.append((r, h))
        pending = [h for _, h in handles]
        it = 0
        while pending:
            core.step()
            it += 1
            now = time.monotonic()
            still = []
            for h in pending:
                if h._event.is_set():  # non-blocking poll (wait(0) costs a lock round trip)
                    h.completed_at = h.completed_at or now
                else:
                    still.append(h)
            pending = still
            if it > max_iters:
                raise RuntimeError("wave did not complete")
        for r, h in handles:
            if h.error is not None and not (r.fail_after is not None
                                            and type(h.error).__name__ == "InjectedFault"):
                raise h.error
            records.append(TurnRecord(r, h.result, (h.completed_at - h.submitted_at) * 1000.0,
                                      h.error))
    if wave_limit is None:
        for sid in sorted(sessions):
            core.close_session(sessions[sid])
    return records


def mismatches(records: list[TurnRecord]) -> list[str]:
    """Field-by-field comparison with the reference results (empty = parity)."""
    bad = []
    for rec in records:
        exp = rec.req.expect
        if "failed" in exp or rec.result is None:
            err = rec.handle_error
            if "failed" not in exp or err is None or type(err).__name__ != exp["failed"]:
                bad.append(f"{rec.req.id}: failed {err!r}, expected {exp.get('failed')}")
            continue
        for f in RESULT_FIELDS:
            got = getattr(rec.result, f)
            if f in exp and got != exp[f]:
                bad.append(f"{rec.req.id}.{f}: got {str(got)[:120]} expected {str(exp[f])[:120]}")
        if "finalize" in exp and rec.result.finalize.kind != exp["finalize"]:
            bad.append(f"{rec.req.id}.finalize: {rec.result.finalize.kind} != {exp['finalize']}")
    return bad


def core_config_for(trace: dict, **overrides):
    """CoreConfig with the reference ServerConfig overrides the trace ran with."""
    from .config import CoreConfig

    cfg = CoreConfig().with_overrides(**trace["config"])
    return cfg.with_overrides(**overrides) if overrides else cfg
