"""Host scheduler parity: the product InferenceCore (admission, planning,
grouping, speculation caps, commit/finish, radix, kv) replays reference traces
with the TEST-ONLY oracle engine and must reproduce every reference result
field, the ledger and the radix dump.  The GPU version of this test
(test_gpu_transcripts.py) swaps in the real GpuEngine."""
from __future__ import annotations

import pytest

from oracle_engine import OracleEngine
from paper_2605_26289_b200.scheduler import InferenceCore, SchedulerConfig, chunk_for, spec_cap
from paper_2605_26289_b200.workload import core_config_for, load_trace, mismatches, replay

TRACES = ["c1", "c2", "c2_nospec", "c3", "c3_nogroup", "c4_small", "c5_small", "sessions",
          "sessions_radix", "c4", "c5", "c11", "c11_tight"]


@pytest.mark.parametrize("batched", [False, True])
@pytest.mark.parametrize("name", TRACES)
def test_trace_parity_host(name, batched):
    tr = load_trace(name)
    cfg = core_config_for(tr, model="tiny", batched_forward=batched)
    core = InferenceCore(cfg, engine=OracleEngine(cfg.vocab, cfg.copy_min_match))
    recs = replay(core, tr)
    assert mismatches(recs) == []
    final = tr["snapshots"][-1]
    assert core.engine.ledger.snapshot() == final["ledger"]
    assert core.kv.occupancy == final["occ"]
    assert core.radix.total_cells == final["radix_cells"]
    assert core.radix.dump() == final["radix_dump"]
    assert core.iterations == final["iterations"]
    if "pool" in final:  # acceptance c11: zero leaked ids / cells after injected faults
        assert core.pool.free_counts() == final["pool"]
        assert core.kv.occupancy == core.radix.total_cells
        assert not core._slots and not core._pending
        assert sum(1 for r in recs if r.handle_error is not None) > 20


CFG = SchedulerConfig()


def test_spec_cap_and_chunk():  # test_scheduler.py:20-68
    assert spec_cap(1, 0.9, CFG) == 16
    assert spec_cap(16, 0.9, CFG) == 4
    assert spec_cap(1, 0.1, CFG) == 2
    assert [spec_cap(n, 0.5, CFG) for n in (4, 5, 8, 9)] == [16, 8, 8, 4]
    assert spec_cap(1, 0.30, CFG) == 16
    assert chunk_for(CFG, 1, False) == 4096
    assert chunk_for(CFG, 64, False) == 128
    assert chunk_for(CFG, 4, True) == 1024
    assert chunk_for(CFG, 1, True) == 4096
    with pytest.raises(ValueError):
        SchedulerConfig(chunk_min=2048, fair_chunk=1024)


def test_temperature_rejected():
    from paper_2605_26289_b200.config import CoreConfig
    from paper_2605_26289_b200.scheduler import GenerationRequest, RequestHandle

    core = InferenceCore(CoreConfig(model="tiny"), engine=OracleEngine())
    g = core.pool.acquire("transient")
    h = RequestHandle(GenerationRequest("t", [1, 2, 3], [" a"] * 3, 4, 0.7, 0, guard=g))
    with pytest.raises(ValueError):
        core.submit(h)


def _pressure_run(batched: bool, engine_factory=None):
    """Session KV (held between turns, outside the admission charge) squeezes
    the free pool so decode/verify entries must evict radix leaves or defer."""
    from paper_2605_26289_b200 import scheduler as S
    from paper_2605_26289_b200.config import CoreConfig
    from paper_2605_26289_b200.kernels import prompt_seed
    from paper_2605_26289_b200.scheduler import GenerationRequest, RequestHandle
    import random

    cfg = CoreConfig(model="tiny", capacity_cells=256, spec_max_lookahead=4, pool_transient=12,
                     batched_forward=batched)
    core = InferenceCore(cfg, engine=(engine_factory or (
        lambda c: OracleEngine(c.vocab, c.copy_min_match)))(cfg))
    tight = {"n": 0}
    orig = S.InferenceCore._run_decode_entry

    def counting(self, entry, events):
        tight["n"] += 1
        return orig(self, entry, events)

    S.InferenceCore._run_decode_entry = counting
    rng = random.Random(5)
    sessions = [core.open_session(f"s{i}") for i in range(2)]
    out = []
    try:
        for rnd in range(12):
            hs = []
            for i, sess in enumerate(sessions):  # sessions grow by ~20 tokens a turn
                toks = list(sess.tokens) + [rng.randrange(50) for _ in range(20)]
                req = GenerationRequest(f"s{i}-{rnd}", toks, [f" w{t}" for t in toks], 6, 0.0,
                                        prompt_seed(toks), session=sess)
                hs.append(RequestHandle(req))
            for w in range(6):  # repetitive transient prompts: copy policy + long drafts
                base = [rng.randrange(6) for _ in range(6)]
                toks = (base * 5)[: 12 + rng.randrange(12)]
                req = GenerationRequest(f"t{rnd}-{w}", toks, [f" w{t}" for t in toks], 10, 0.0,
                                        prompt_seed(toks), guard=core.pool.acquire("transient"))
                hs.append(RequestHandle(req))
            for h in hs:
                core.submit(h)
            for _ in range(10_000):
                if all(h.wait(timeout=0) for h in hs):
                    break
                core.step()
            for h in hs:
                assert h.error is None, h.error
                r = h.result
                out.append((r.request_id, r.generated, r.decode_passes, r.spec_accepted,
                            r.cached_prompt_tokens))
            for i, sess in enumerate(sessions):
                if rnd % 3 == 2:  # reset the sessions now and then
                    core.close_session(sess)
                    sessions[i] = core.open_session(f"s{i}")
    finally:
        S.InferenceCore._run_decode_entry = orig
    snap = (core.engine.ledger.snapshot(), core.radix.dump(), core.kv.occupancy,
            core.radix.evicted_cells_total)
    return out, snap, tight["n"], core


def test_batched_capacity_precheck_matches_sequential():
    """Batched plans check capacity BEFORE the forward (scheduler.py:740/761
    order); under KV pressure they fall back to entry-by-entry execution and
    must produce exactly the sequential (reference-order) results."""
    seq_out, seq_snap, _, _ = _pressure_run(False)
    bat_out, bat_snap, tight, _ = _pressure_run(True)
    assert tight > 0  # the pre-check fired
    assert seq_snap[3] > 0  # radix evictions happened
    assert bat_out == seq_out
    assert bat_snap == seq_snap
