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
                                          ("c2", True), ("c3", True), ("c5_small", True)])
def test_trace_parity_gpu(cuda, name, batched):
    tr = load_trace(name)
    core = InferenceCore(core_config_for(tr, model="tiny", batched_forward=batched))
    recs = replay(core, tr)
    assert mismatches(recs) == []
    final = tr["snapshots"][-1]
    assert core.engine.ledger.snapshot() == final["ledger"]
    assert core.radix.dump() == final["radix_dump"]
    _device_invariants(core)
