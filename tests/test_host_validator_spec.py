"""Streaming tool-call validator (its early stop shapes the
transcript) and the speculation acceptance EMA (a19/a21), differentially
against the unmodified reference built into oracle/_ref (test infrastructure;
skipped when that build is absent), plus fixed behaviours the reference's own
tests pin (test_validator.py, test_speculator.py)."""
from __future__ import annotations

import os
import random
import sys

import pytest

from paper_2605_26289_b200 import speculator as ours_spec
from paper_2605_26289_b200 import validator as ours

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


def _ref():
    if not os.path.isdir(os.path.join(REF, "deltaserve")):
        pytest.skip("oracle/_ref (the reference build) is absent")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from deltaserve import speculator, validator

    return validator, speculator


def _pieces(rng: random.Random) -> list[str]:
    """Random JSON-ish piece streams: tool-call objects (some malformed, some
    with braces/escapes inside strings), prose, splits across pieces."""
    names = ["get_weather", "search", "fly", "x"]
    out = []
    for _ in range(rng.randrange(1, 5)):
        kind = rng.random()
        if kind < 0.5:
            val = rng.choice(['"a}b"', '"q\\"}"', "1", '{"k":[1,2]}', '"{"'])
            obj = '{"name":"%s","parameters":{"p":%s}}' % (rng.choice(names), val)
            if rng.random() < 0.2:
                obj = obj[: rng.randrange(1, len(obj))]  # never closes
            if rng.random() < 0.1:
                obj = obj.replace(":", " ", 1)  # closes, does not parse
        elif kind < 0.8:
            obj = rng.choice([" plain", " text}", " {not json", " and then"])
        else:
            obj = '{"other":%d}' % rng.randrange(9)
        cuts = sorted(rng.sample(range(1, len(obj)), min(len(obj) - 1, rng.randrange(0, 4))))
        prev = 0
        for c in cuts + [len(obj)]:
            out.append(obj[prev:c])
            prev = c
    return out


def test_validator_matches_reference_on_random_streams():
    rv, _ = _ref()
    rng = random.Random(2605)
    declared = {"get_weather", "search"}
    for case in range(3000):
        pieces = _pieces(rng)
        grace = rng.randrange(0, 4)
        sent = rng.randrange(len(pieces)) if rng.random() < 0.1 else None
        a, b = ours.ValidatorState(grace_pieces=grace), rv.ValidatorState(grace_pieces=grace)
        acts_a = [ours.on_piece(a, p, is_sentinel=(i == sent)).name for i, p in enumerate(pieces)]
        acts_b = [rv.on_piece(b, p, is_sentinel=(i == sent)).name for i, p in enumerate(pieces)]
        assert acts_a == acts_b, (case, pieces)
        assert a.closed_objects == b.closed_objects, (case, pieces)
        assert a.chars_scanned == b.chars_scanned
        raw = "".join(pieces)
        fa, fb = ours.finalize(a, declared, raw), rv.finalize(b, declared, raw)
        assert (fa.kind, fa.reason, fa.text) == (fb.kind, fb.reason, fb.text), (case, pieces)
        assert [(c.name, c.parameters) for c in fa.calls] == \
            [(c.name, c.parameters) for c in fb.calls]


def test_validator_fixed_cases():
    st = ours.ValidatorState(grace_pieces=1)
    acts = [ours.on_piece(st, p) for p in ['{"na', 'me":"search","parameters":{"q":"}"}}', " x"]]
    assert [a.name for a in acts] == ["CONTINUE", "CONTINUE", "EARLY_STOP"]
    res = ours.finalize(st, {"search"}, "")
    assert res.kind == "tool_calls" and res.calls[0].parameters == {"q": "}"}
    st = ours.ValidatorState(grace_pieces=0)
    ours.on_piece(st, '{"name":"nope","parameters":{}}')
    assert ours.finalize(st, {"search"}, "").kind == "rejected"
    st = ours.ValidatorState()
    assert ours.on_piece(st, "just prose").name == "CONTINUE"
    assert ours.finalize(st, {"search"}, "just prose").kind == "text"


def test_acceptance_ema_matches_reference():
    _, rs = _ref()
    rng = random.Random(7)
    for _ in range(200):
        decay = rng.choice([0.0, 0.3, 0.8, 1.0])
        a = ours_spec.SpecState(ours_spec.SpecConfig(ema_decay=decay))
        b = rs.SpecState(rs.SpecConfig(ema_decay=decay))
        for _ in range(rng.randrange(1, 30)):
            k = rng.randrange(1, 17)
            acc = rng.randrange(0, k + 1)
            ours_spec.update_acceptance(a, ours_spec.SpecOutcome(proposed=k, accepted=acc))
            rs.update_acceptance(b, rs.SpecOutcome(proposed=k, accepted=acc))
            assert a.ema == b.ema
            assert 0.0 <= a.ema <= 1.0


def test_spec_cap_and_chunk_for_match_reference():
    """Planner helpers (SURVEY 8a a11 chunk_for, a19 spec_cap) over random
    configs, decoder counts, acceptance EMAs and prefill counts."""
    _ref()
    from deltaserve import scheduler as rsch

    from paper_2605_26289_b200 import scheduler as osch

    rng = random.Random(11)
    for _ in range(3000):
        cmin = rng.choice([16, 64, 128])
        fair = rng.choice([cmin, 256, 1024])
        cmax = rng.choice([fair, 2048, 4096])
        kw = dict(n_batch=rng.choice([cmax, 4096, 8192]), chunk_min=cmin, fair_chunk=fair,
                  chunk_max=cmax, spec_base_cap=rng.choice([4, 16, 32]),
                  spec_d0=rng.choice([1, 2, 4, 8]), spec_floor_cap=rng.choice([1, 2]))
        a, b = osch.SchedulerConfig(**kw), rsch.SchedulerConfig(**kw)
        n, lat = rng.randrange(0, 300), rng.random() < 0.5
        assert osch.chunk_for(a, n, lat) == rsch.chunk_for(b, n, lat)
        d, ema = rng.randrange(0, 600), rng.random()
        assert osch.spec_cap(d, ema, a) == rsch.spec_cap(d, ema, b)
