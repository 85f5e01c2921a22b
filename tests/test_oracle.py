"""The oracle (oracle/ds_oracle.c) pinned against the reference's golden vectors.

Golden vectors were produced by the reference itself (tests/golden/make_golden.py)
and include the reference's own known-answer tests (test_kernels.py:61-120,
test_speculator.py:22-46, test_engine.py:127-141).
"""
from __future__ import annotations

import random

from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import cpu


def test_fnv_bytes(golden_kernels):
    for case in golden_kernels["fnv_bytes"]:
        data = bytes.fromhex(case["hex"])
        assert cpu.fnv1a32_bytes(data) == case["f32"]
        assert cpu.fnv1a64_bytes(data) == case["f64"]


def test_fnv_tokens(golden_kernels):
    for case in golden_kernels["fnv_tokens"]:
        t = case["tokens"]
        assert cpu.fnv1a32_tokens(t) == case["f32"]
        assert cpu.fnv1a64_tokens(t) == case["f64"]
        assert cpu.fnv1a32_tokens(t, case["state32"]) == case["f32s"]
        assert cpu.fnv1a64_tokens(t, case["state64"]) == case["f64s"]


def test_known_answers():
    assert cpu.fnv1a32_bytes(b"") == 2166136261
    assert cpu.fnv1a64_bytes(b"") == 0xCBF29CE484222325
    assert cpu.copy_continuation([5, 6, 7, 5, 6], 2) == 2
    assert cpu.lookup_ngram([10, 20, 30, 40, 10, 20], [10, 20, 30, 40, 10, 20], 2, 2) == [30, 40]


def test_copy_continuation(golden_kernels):
    for case in golden_kernels["copy_continuation"]:
        assert cpu.copy_continuation(case["tokens"], case["mm"]) == case["e"], case


def test_suffix_match(golden_kernels):
    for case in golden_kernels["suffix_match"]:
        tail = case["ring"] if case["tail"] is None else case["tail"]
        assert cpu.longest_suffix_match(case["ring"], tail, case["min_len"]) == (
            case["e"], case["len"])


def test_lookup_ngram(golden_kernels):
    for case in golden_kernels["lookup_ngram"]:
        assert cpu.lookup_ngram(case["ring"], case["ring"], case["mm"], case["cap"]) == case["draft"]


def test_copy_policy(golden_kernels):
    for case in golden_kernels["copy_policy"]:
        full, c = case["full"], case["ctx"]
        for i, (tok, src) in enumerate(case["rows"]):
            assert cpu.copy_policy(full, c + i + 1, case["mm"], case["vocab"]) == (tok, src)


def _brute_suffix(ring, tail, lmin):  # test_kernels.py:44-54 formulation
    best = (-1, 0)
    n, t = len(ring), len(tail)
    for length in range(lmin, min(t, n) + 1):
        suffix = list(tail[t - length:])
        for e in range(n - 1, length - 1, -1):
            if list(ring[e - length:e]) == suffix:
                if length > best[1]:
                    best = (e, length)
                break
    return best


@given(st.lists(st.integers(0, 5), max_size=40), st.integers(1, 4))
@settings(max_examples=200, deadline=None)
def test_suffix_match_bruteforce(ring, lmin):
    assert cpu.longest_suffix_match(ring, ring, lmin) == _brute_suffix(ring, ring, lmin)


def test_large_inputs_consistent():
    rng = random.Random(3)
    ring = [rng.randrange(4) for _ in range(2048)]
    assert cpu.longest_suffix_match(ring, ring, 3) == _brute_suffix(ring, ring, 3)
