"""SequencePool / SlotGuard (reference pool.py:24-116) and the
KV release policy the core hangs on it (scheduler `_release_hook`): the
behaviours the reference's test_pool.py / test_release_policy.py pin, checked
against the B200 build's host restatement (CPU, no GPU engine needed)."""
from __future__ import annotations

import random
import threading

import pytest

from oracle_engine import OracleEngine
from paper_2605_26289_b200.config import CoreConfig
from paper_2605_26289_b200.pool import AcquireTimeout, PoolConfig, SequencePool
from paper_2605_26289_b200.scheduler import InferenceCore


def test_transient_and_session_regions():
    pool = SequencePool(PoolConfig(5, 3))
    t = [pool.acquire("transient") for _ in range(5)]
    s = [pool.acquire("session") for _ in range(3)]
    assert sorted(g.seq for g in t) == list(range(5))
    assert sorted(g.seq for g in s) == [5, 6, 7]
    assert {pool.region_of(g.seq) for g in t} == {"transient"}
    assert {pool.region_of(g.seq) for g in s} == {"session"}
    for g in t + s:
        g.release()
    assert pool.free_counts() == {"transient": 5, "session": 3}


def test_acquire_timeout_is_backpressure():
    pool = SequencePool(PoolConfig(1, 1))
    g = pool.acquire("session")
    with pytest.raises(AcquireTimeout):
        pool.acquire("session", timeout=0.02)
    g.release()
    assert pool.acquire("session", timeout=0.02).seq == g.seq


def test_blocked_acquire_wakes_on_release():
    pool = SequencePool(PoolConfig(1, 1))
    held = pool.acquire("transient")
    out = []
    th = threading.Thread(target=lambda: out.append(pool.acquire("transient", timeout=5.0).seq))
    th.start()
    held.release()
    th.join(timeout=5.0)
    assert out == [held.seq]


def test_guard_context_and_idempotent_release():
    hook = []
    pool = SequencePool(PoolConfig(3, 1), release_hook=lambda seq, kind: hook.append((seq, kind)))
    with pytest.raises(KeyError):
        with pool.acquire("transient") as g:
            raise KeyError("failure inside the request")
    assert g.released and hook == [(g.seq, "transient")]
    g.release()  # second release: no hook, no double free
    assert hook == [(g.seq, "transient")]
    assert pool.free_counts() == {"transient": 3, "session": 1}


def test_hook_runs_before_the_id_is_reusable():
    order = []
    pool = SequencePool(PoolConfig(1, 1))

    def hook(seq, kind):
        order.append("hook")
        # the id is not yet back: a concurrent acquire would have to wait
        with pytest.raises(AcquireTimeout):
            pool.acquire("transient", timeout=0.01)

    pool._hook = hook
    g = pool.acquire("transient")
    g.release()
    order.append(pool.acquire("transient", timeout=0.01).seq)
    assert order == ["hook", g.seq]


def test_bad_region_and_bad_config():
    with pytest.raises(ValueError):
        SequencePool(PoolConfig(1, 1)).acquire("batch")
    with pytest.raises(ValueError):
        PoolConfig(0, 2)


def test_ids_conserved_under_threads():
    pool = SequencePool(PoolConfig(3, 2))

    def worker(seed):
        r = random.Random(seed)
        for _ in range(150):
            kind = "session" if r.random() < 0.3 else "transient"
            try:
                g = pool.acquire(kind, timeout=2.0)
            except AcquireTimeout:
                continue
            with g:
                assert pool.region_of(g.seq) == kind
    ths = [threading.Thread(target=worker, args=(i,)) for i in range(6)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=30)
        assert not t.is_alive()
    assert pool.free_counts() == {"transient": 3, "session": 2}


def _core():
    cfg = CoreConfig(model="tiny")
    return InferenceCore(cfg, engine=OracleEngine(cfg.vocab, cfg.copy_min_match))


def test_release_policy_transient_frees_uncommitted_cells():
    core = _core()
    g = core.pool.acquire("transient")
    core.kv.append_cells(g.seq, 37)
    occ = core.kv.occupancy
    g.release()
    assert occ - core.kv.occupancy == 37 and core.kv.seq_len(g.seq) == 0


def test_release_policy_transient_keeps_radix_cells():
    core = _core()
    g = core.pool.acquire("transient")
    toks = [3 * i + 1 for i in range(25)]
    core.kv.append_cells(g.seq, 25)
    core.radix.save(toks, g.seq, 0)
    g.release()
    assert core.kv.occupancy == 25  # held by the trie only
    assert core.radix.longest_prefix(toks).length == 25


def test_release_policy_session_retains_until_closed():
    core = _core()
    h = core.open_session("s")
    core.kv.append_cells(h.guard.seq, 19)
    h.guard.release()  # retention is the caller's policy (server DELETE)
    assert core.kv.occupancy == 19
    core.kv.release_sequence(h.guard.seq)
    assert core.kv.occupancy == 0
