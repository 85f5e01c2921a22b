"""The native host core (csrc_host/hostcore.cpp: cell allocator / page tables
and radix trie) against the Python restatement, which is itself pinned to the
reference (golden op logs in test_host_kvcache.py / test_host_radix.py):
random operation sequences - appends, aliases, trims, releases, radix saves /
lookups / evictions, error paths - must leave identical observables (cell
ids, refcounts, occupancy, span counts, device-op logs, radix dumps, eviction
totals), and whole reference traces replay identically on both."""
from __future__ import annotations

import random

import numpy as np
import pytest

from paper_2605_26289_b200 import kvcache as K
from paper_2605_26289_b200 import radix as R


def _observe(kv, trie, seqs):
    return {"occ": kv.occupancy, "free": kv.free_cells,
            "ref": np.asarray(kv._refcnt).tolist(),
            "tables": {s: (kv.seq_len(s), kv.span_count(s), kv.cell_ids(s, 0, kv.seq_len(s)))
                       for s in seqs},
            "radix": trie.dump(), "cells": trie.total_cells, "nodes": trie.node_count(),
            "evicted": trie.evicted_cells_total}


def _apply(kv, trie, op):
    kind = op[0]
    try:
        if kind == "append":
            return kv.append_cells(op[1], op[2])
        if kind == "trim":
            return kv.trim(op[1], op[2])
        if kind == "release":
            return kv.release_sequence(op[1])
        if kind == "alias":
            if op[3] is None:  # follower-style: dest's current end, a run of the donor
                a = kv.seq_len(op[2])
                return kv.seq_alias(op[1], op[2], a, a + op[4])
            return kv.seq_alias(op[1], op[2], op[3], op[4])
        if kind == "save":
            return trie.save(op[2], op[1], 0)
        if kind == "lookup":
            m = trie.longest_prefix(op[1])
            if m.length and op[2] is not None:  # restore like _admit
                kv.alias_runs(op[2], K.slice_runs(m.runs, 0, m.length))
            return (m.length, [tuple(r) for r in m.runs], m.donor)
        if kind == "evict":
            return trie.evict(op[1])
    except (K.CapacityExhausted, K.DonorRangeInvalid, R.BudgetExceeded, ValueError) as e:
        return type(e).__name__
    raise AssertionError(op)


def _ops(rng, n_seqs, alphabet):
    ops = []
    for _ in range(600):
        r = rng.random()
        s = rng.randrange(n_seqs)
        if r < 0.25:
            ops.append(("append", s, rng.randrange(1, 40)))
        elif r < 0.40:
            ops.append(("trim", s, rng.randrange(0, 60)))
        elif r < 0.45:
            ops.append(("release", s))
        elif r < 0.55:
            d = rng.randrange(n_seqs)
            if rng.random() < 0.7:
                ops.append(("alias", s, d, None, rng.randrange(1, 20)))
            else:
                a = rng.randrange(0, 30)
                ops.append(("alias", s, d, a, a + rng.randrange(0, 30)))
        elif r < 0.75:
            toks = [rng.randrange(alphabet) for _ in range(rng.randrange(1, 50))]
            ops.append(("save", s, toks))
        elif r < 0.92:
            toks = [rng.randrange(alphabet) for _ in range(rng.randrange(1, 50))]
            ops.append(("lookup", toks, rng.choice([None, s])))
        else:
            ops.append(("evict", rng.randrange(0, 80)))
    return ops


@pytest.mark.parametrize("seed", range(12))
def test_native_matches_python_restatement(seed):
    rng = random.Random(seed)
    cap = rng.choice([96, 256, 1024])
    budget = rng.choice([32, 64, 200])
    alphabet = rng.choice([2, 3, 6])  # small alphabets: shared prefixes, splits, ties
    n_seqs = 6
    impls = []
    for KvC, RtC in ((K.PyUnifiedKvCache, R.PyRadixTrie),
                     (K.NativeUnifiedKvCache, R.NativeRadixTrie)):
        kv = KvC(cap)
        kv.record_ops = True
        impls.append((kv, RtC(kv, budget)))
    for i, op in enumerate(_ops(rng, n_seqs, alphabet)):
        outs = [_apply(kv, trie, op) for kv, trie in impls]
        assert outs[0] == outs[1], (i, op, outs)
        if i % 25 == 0:
            a, b = (_observe(kv, trie, range(n_seqs)) for kv, trie in impls)
            assert a == b, (i, op)
            oa = np.asarray(impls[0][0].take_ops(), dtype=np.int32).reshape(-1, 5)
            ob = np.asarray(impls[1][0].take_ops(), dtype=np.int32).reshape(-1, 5)
            assert np.array_equal(oa, ob), i
    a, b = (_observe(kv, trie, range(n_seqs)) for kv, trie in impls)
    assert a == b


@pytest.mark.parametrize("name", ["c3", "c5_small", "c11_tight"])
def test_traces_identical_on_both_host_cores(name, monkeypatch):
    from oracle_engine import OracleEngine
    from paper_2605_26289_b200 import scheduler as S
    from paper_2605_26289_b200.workload import core_config_for, load_trace, mismatches, replay

    tr = load_trace(name)
    snaps = []
    for KvC, RtC in ((K.PyUnifiedKvCache, R.PyRadixTrie),
                     (K.NativeUnifiedKvCache, R.NativeRadixTrie)):
        monkeypatch.setattr(S, "UnifiedKvCache", KvC)
        monkeypatch.setattr(S, "RadixTrie", RtC)
        cfg = core_config_for(tr, model="tiny", batched_forward=True)
        core = S.InferenceCore(cfg, engine=OracleEngine(cfg.vocab, cfg.copy_min_match))
        recs = replay(core, tr)
        assert mismatches(recs) == []
        snaps.append((core.radix.dump(), np.asarray(core.kv._refcnt).tolist(),
                      core.engine.ledger.snapshot()))
    assert snaps[0] == snaps[1]


def test_native_is_the_default():
    assert K.UnifiedKvCache is K.NativeUnifiedKvCache
    assert R.RadixTrie is R.NativeRadixTrie
