"""End-to-end parity on the B200: the product InferenceCore + GpuEngine (real
random-init transformer on device, copy token policy) replays the reference
traces and must reproduce every result field bit-exactly (tokens, accepted
drafts, radix hits, aliased cells, ledger), and the device page tables /
membership refcounts must equal the host allocator's."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2605_26289_b200.scheduler import InferenceCore
from paper_2605_26289_b200.workload import core_config_for, load_trace, mismatches, replay

pytestmark = pytest.mark.gpu


def _device_invariants(core):
    eng = core.engine
    rc, occ = eng.device_refcounts()
    assert occ == core.kv.occupancy
    assert np.array_equal(rc, core.kv._refcnt)
    for seq in core.kv.sequences():
        if seq < eng.n_seqs:
            n = core.kv.seq_len(seq)
            assert eng.device_cells(seq, n) == core.kv.cell_ids(seq, 0, n)


@pytest.mark.parametrize("name,batched", [("c1", False), ("c2", False), ("c2_nospec", False),
                                          ("c3", False), ("c4_small", False), ("c5_small", False),
                                          ("c2", True), ("c3", True), ("c5_small", True),
                                          ("sessions", False), ("sessions_radix", False),
                                          ("sessions", True),
                                          # full BASELINE C4 (32,370-token prefix: split-KV
                                          # through the whole path) and C5 (256 sessions,
                                          # radix evictions on the device page tables)
                                          ("c4", False), ("c4", True), ("c5", False),
                                          ("c5", True),
                                          # acceptance c11: injected faults -> _fail_slot
                                          ("c11", False), ("c11", True),
                                          ("c11_tight", False), ("c11_tight", True)])
def test_trace_parity_gpu(cuda, name, batched):
    tr = load_trace(name)
    core = InferenceCore(core_config_for(tr, model="tiny", batched_forward=batched))
    recs = replay(core, tr)
    assert mismatches(recs) == []
    final = tr["snapshots"][-1]
    assert core.engine.ledger.snapshot() == final["ledger"]
    assert core.radix.dump() == final["radix_dump"]
    if name == "c5":  # the device page tables went through radix evictions
        assert core.radix.evicted_cells_total > 0
    if "pool" in final:  # c11: zero leaked sequence ids or cells after the faults
        assert core.pool.free_counts() == final["pool"]
        assert core.kv.occupancy == core.radix.total_cells == final["radix_cells"]
        assert not core._slots and not core._pending
        assert sum(1 for r in recs if r.handle_error is not None) > 20
    _device_invariants(core)


def test_batched_capacity_precheck_gpu(cuda):
    """KV pressure (session-held cells): batched plans fall back to the
    reference's check-then-forward order; results equal the sequential run
    and the device page tables / refcounts equal the host allocator's."""
    from test_host_scheduler import _pressure_run

    from paper_2605_26289_b200.engine import GpuEngine

    def gpu(cfg):
        return None  # InferenceCore builds its GpuEngine

    seq_out, seq_snap, _, c0 = _pressure_run(False, engine_factory=gpu)
    _device_invariants(c0)
    bat_out, bat_snap, tight, c1 = _pressure_run(True, engine_factory=gpu)
    _device_invariants(c1)
    assert tight > 0 and seq_snap[3] > 0
    assert bat_out == seq_out and bat_snap == seq_snap
    assert isinstance(c1.engine, GpuEngine)


@pytest.mark.parametrize("name,batched", [("c2", False), ("c4_small", False), ("c3", True),
                                          ("c5_small", True), ("c11_tight", True)])
def test_fused_next_proposal_matches_k1(cuda, name, batched):
    """The proposal computed inside each decode/verify forward (bonus token
    written on device, suffix match over the post-commit ring) equals a fresh
    K1 launch over the host's token list, for every proposal the scheduler
    makes; and every cached proposal is actually used (no silent misses).
    Batched plans: mixed prefill + decode / verify plans, scratch-cell rows and
    deferred commits (c11_tight: KV pressure) included."""
    from paper_2605_26289_b200 import engine as E

    tr = load_trace(name)
    core = InferenceCore(core_config_for(tr, model="tiny", batched_forward=batched))
    eng = core.engine
    stats = {"hits": 0, "calls": 0}
    orig = E.GpuEngine.propose

    def checked(self, slots, window, min_match, use_cache=True):
        got = orig(self, slots, window, min_match, use_cache)
        if use_cache:
            stats["calls"] += 1
            stats["hits"] += sum(1 for seq, toks, _ in slots
                                 if self._draft_cache.get(seq, (None,))[0] == len(toks))
            fresh = orig(self, slots, window, min_match, use_cache=False)
            assert got == fresh
        return got

    E.GpuEngine.propose = checked
    try:
        recs = replay(core, tr)
    finally:
        E.GpuEngine.propose = orig
    assert mismatches(recs) == []
    assert stats["calls"] > 0 and stats["hits"] >= stats["calls"] // 2, stats
    assert eng.fused_drafts
