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
          "sessions_radix"]


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
