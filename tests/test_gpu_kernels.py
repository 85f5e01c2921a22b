"""Device integer kernels (K1 n-gram matcher, K2 copy scan, FNV) vs the
reference golden vectors and the oracle on large random inputs - bit exact."""
from __future__ import annotations

import random

import pytest

from oracle import cpu

pytestmark = pytest.mark.gpu


def test_fnv(cuda, golden_kernels):
    from paper_2605_26289_b200 import kernels as K

    for case in golden_kernels["fnv_bytes"]:
        data = bytes.fromhex(case["hex"])
        assert K.fnv1a32_bytes(data) == case["f32"]
        assert K.fnv1a64_bytes(data) == case["f64"]
    cases = golden_kernels["fnv_tokens"]
    toks = [c["tokens"] for c in cases]
    assert K.fnv1a_tokens_batched(toks, 64) == [c["f64"] for c in cases]
    assert K.fnv1a_tokens_batched(toks, 32) == [c["f32"] for c in cases]
    assert K.fnv1a_tokens_batched(toks, 64, [c["state64"] for c in cases]) == [c["f64s"] for c in cases]
    assert K.fnv1a_tokens_batched(toks, 32, [c["state32"] for c in cases]) == [c["f32s"] for c in cases]


def test_copy_continuation(cuda, golden_kernels):
    from paper_2605_26289_b200 import kernels as K

    by_mm = {}
    for c in golden_kernels["copy_continuation"]:
        by_mm.setdefault(c["mm"], []).append(c)
    for mm, cases in by_mm.items():
        got = K.copy_continuation_batched([c["tokens"] for c in cases], mm)
        assert got == [c["e"] for c in cases], mm


def test_suffix_match_and_drafts(cuda, golden_kernels):
    from paper_2605_26289_b200 import kernels as K

    by_l = {}
    for c in golden_kernels["suffix_match"]:
        by_l.setdefault(c["min_len"], []).append(c)
    for lmin, cases in by_l.items():
        rings = [c["ring"] for c in cases]
        tails = [c["ring"] if c["tail"] is None else c["tail"] for c in cases]
        e, ln = K.longest_suffix_match_batched(rings, tails, lmin)
        assert list(zip(e, ln)) == [(c["e"], c["len"]) for c in cases]
    by_mm = {}
    for c in golden_kernels["lookup_ngram"]:
        by_mm.setdefault(c["mm"], []).append(c)
    for mm, cases in by_mm.items():
        rings = [c["ring"] for c in cases]
        _, _, drafts = K.longest_suffix_match_batched(rings, None, mm, caps=[c["cap"] for c in cases],
                                                      max_draft=17)
        assert drafts == [c["draft"][:17] for c in cases]


def test_reference_api_single_calls(cuda):
    from paper_2605_26289_b200 import kernels as K

    assert K.BACKEND == "cuda-sm100a"
    assert K.copy_continuation([5, 6, 7, 5, 6], 2) == 2
    assert K.longest_suffix_match([10, 20, 30, 40, 10, 20], [10, 20, 30, 40, 10, 20], 2) == (2, 2)
    assert K.fnv1a32_bytes(b"") == 2166136261


@pytest.mark.parametrize("n,alpha", [(2048, 3), (2048, 64), (32768, 30000), (32768, 4)])
def test_large_random_vs_oracle(cuda, n, alpha):
    from paper_2605_26289_b200 import kernels as K

    rng = random.Random(n * 7 + alpha)
    seqs = []
    for _ in range(8):
        s = [rng.randrange(alpha) for _ in range(n)]
        span = s[100:140]
        s[-20:] = span[:20]  # recent copy, like an agent re-emitting a tool call
        seqs.append(s)
    for mm in (1, 2, 3, 4):
        assert K.copy_continuation_batched(seqs, mm) == [cpu.copy_continuation(s, mm) for s in seqs]
    rings = [s[-2048:] for s in seqs]
    e, ln = K.longest_suffix_match_batched(rings, None, 3)
    assert list(zip(e, ln)) == [cpu.longest_suffix_match(r, r, 3) for r in rings]
    assert K.fnv1a_tokens_batched(seqs, 64) == [cpu.fnv1a64_tokens(s) for s in seqs]


def test_empty_and_degenerate(cuda):
    from paper_2605_26289_b200 import kernels as K

    assert K.copy_continuation_batched([[], [1], [1, 1]], 3) == [-1, -1, -1]
    e, ln = K.longest_suffix_match_batched([[], [1, 2, 3]], None, 0)
    assert list(zip(e, ln)) == [(-1, 0), (-1, 0)]
    assert K.fnv1a_tokens_batched([[]], 64) == [cpu.fnv1a64_tokens([])]
