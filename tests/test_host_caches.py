"""Host front end: render / tokenize caches and the mock
tokenizer / renderer restated from the reference (caches.py, engine.py:104-264)
- prepare_prompt on the recorded chat messages must reproduce the reference's
prompt ids and pieces byte for byte, with the same render / tokenize cache
counters (hits, misses, entries, pieces_tokenized) after every request; plus
the LRU / prefix-delta unit semantics (reference tests/test_caches.py)."""
from __future__ import annotations

import pytest

from oracle_engine import OracleEngine
from paper_2605_26289_b200 import caches as C
from paper_2605_26289_b200.scheduler import InferenceCore
from paper_2605_26289_b200.workload import core_config_for, load_trace, mismatches, replay, waves


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_prepare_prompt_reproduces_reference(name):
    tr = load_trace(name)
    cfg = core_config_for(tr, model="tiny")
    core = InferenceCore(cfg, engine=OracleEngine(cfg.vocab, cfg.copy_min_match))
    n = 0
    for wave in waves(tr):
        for r in wave:
            assert r.messages is not None
            _, ids, pieces = core.prepare_prompt(r.messages, r.tool_defs)
            assert ids == r.tokens and pieces == r.pieces, r.id
            assert core.render_cache.stats() == r.cache_stats["render"], r.id
            assert core.tokenize_cache.stats() == r.cache_stats["tokenize"], r.id
            n += 1
    assert n == len(tr["reqs"])


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_replay_through_the_front_end(name):
    tr = load_trace(name)
    cfg = core_config_for(tr, model="tiny")
    core = InferenceCore(cfg, engine=OracleEngine(cfg.vocab, cfg.copy_min_match))
    recs = replay(core, tr, via_chat=True)
    assert mismatches(recs) == []
    assert core.tokenize_cache.stats()["pieces_tokenized"] < sum(len(r.tokens) for r in tr["reqs"])


def test_lru_and_prefix_delta_semantics():
    lru = C.LruCache(2)
    lru.put("a", 1)
    lru.put("b", 2)
    assert lru.get("a") == 1
    lru.put("c", 3)  # evicts b, the least recently used
    assert "b" not in lru and lru.get("a") == 1 and lru.get("c") == 3
    assert lru.stats() == {"hits": 3, "misses": 0, "entries": 2}
    tc = C.TokenizeCache(8)
    base = "<|system|>\nhello world<|end|>\n"
    ids1, p1, hit1 = tc.get_or_tokenize(base, lambda t: C.tokenize_with_pieces(t, 32768))
    ext = base + "<|user|>\nmore words<|end|>\n"
    ids2, p2, hit2 = tc.get_or_tokenize(ext, lambda t: C.tokenize_with_pieces(t, 32768))
    assert not hit1 and not hit2
    assert (ids2, p2) == C.tokenize_with_pieces(ext, 32768)
    assert ids2[: len(ids1)] == ids1
    assert tc.pieces_tokenized == len(p1) + (len(p2) - len(p1))  # only the suffix
    assert tc.get_or_tokenize(ext, None)[2] is True
    assert C.is_piece_boundary("ab cd", 2) and not C.is_piece_boundary("abcd", 2)
    assert C.split_pieces("a  b,c") == ["a", "  ", "b", ",", "c"]
    with pytest.raises(C.RenderError):
        C.render_chat([{"role": "robot", "content": "x"}])
    assert C.prompt_seed([]) == 2166136261  # reference test_caches.py:31-44
