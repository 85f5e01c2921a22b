"""Prefix migration on the device: core A (one B200 process) commits the shared
tool-schema prefix; core B imports those K/V cell rows (the payload an NCCL
send/recv carries between GPUs) into freshly allocated cells; B's next request
restores them by metadata-only aliasing and reproduces the reference result."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2605_26289_b200 import dist as D
from paper_2605_26289_b200.scheduler import InferenceCore
from paper_2605_26289_b200.workload import core_config_for, load_trace, mismatches, replay, waves

pytestmark = pytest.mark.gpu


def test_prefix_import_between_cores(cuda):
    tr = load_trace("c3")
    cfg = core_config_for(tr, model="tiny", capacity_cells=4096)
    a = InferenceCore(cfg)
    b = InferenceCore(cfg)
    w = waves(tr)
    first_a, first_b = w[0][0], w[1][0]
    assert mismatches(replay(a, {"reqs": [first_a]})) == []
    prefix = first_b.tokens[:224]
    src = D.export_prefix(a, prefix)
    payload = D.pack_cells(a.engine.k_pool, a.engine.v_pool, src)
    n = D.import_prefix(b, prefix,
                        lambda cells: D.unpack_cells(b.engine.k_pool, b.engine.v_pool, cells,
                                                     payload))
    assert n == 224
    dst = D.export_prefix(b, prefix)
    assert torch.equal(D.pack_cells(b.engine.k_pool, b.engine.v_pool, dst), payload)
    recs = replay(b, {"reqs": [first_b]})
    assert recs[0].result.cached_prompt_tokens == 224
    assert mismatches(recs) == []
    rc, occ = b.engine.device_refcounts()
    assert occ == b.kv.occupancy and np.array_equal(rc, b.kv._refcnt)
