"""Prefix migration on the device.

* One B200: the migration payload kernel (ds_kv_pack_cells) packs core A's
  cells into the [L][2][nkv][n][hd] message and scatters it into core B's
  freshly allocated cells; B's radix then restores the prefix by
  metadata-only aliasing and reproduces the reference result.
* Two B200s (skipped with fewer): the real thing - two processes, NCCL data
  group, rank 1's ADMISSION migrates rank 0's announced prefix over NVLink and
  reproduces the reference's 224-token C3 radix hit bit-exactly.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

from paper_2605_26289_b200.scheduler import InferenceCore
from paper_2605_26289_b200.workload import core_config_for, load_trace, mismatches, replay, waves

pytestmark = pytest.mark.gpu


def test_pack_unpack_cells_between_cores(cuda):
    tr = load_trace("c3")
    cfg = core_config_for(tr, model="tiny", capacity_cells=4096)
    a = InferenceCore(cfg)
    b = InferenceCore(cfg)
    w = waves(tr)
    first_a, first_b = w[0][0], w[1][0]
    assert mismatches(replay(a, {"reqs": [first_a]})) == []
    m = a.radix.longest_prefix(first_b.tokens)
    assert m.length == 224
    src = [c for s, n in m.runs for c in range(s, s + n)]
    payload = a.engine.pack_cells(src)
    idx = torch.as_tensor(src, device=cuda, dtype=torch.long)
    ref = torch.stack([a.engine.k_pool[:, :, idx], a.engine.v_pool[:, :, idx]], 1)
    assert torch.equal(payload, ref)
    # import into b: cells on the scratch sequence, scatter, radix commit
    seq = b.scratch_seq
    b.kv.append_cells(seq, 224)
    cells = b.kv.cell_ids(seq, 0, 224)
    b.engine.unpack_cells(cells, payload)
    b.radix.save(list(first_b.tokens[:224]), seq, 0)
    b.kv.release_sequence(seq)
    dst = [c for s, n in b.radix.longest_prefix(first_b.tokens).runs for c in range(s, s + n)]
    assert torch.equal(b.engine.pack_cells(dst), payload)
    recs = replay(b, {"reqs": [first_b]})
    assert recs[0].result.cached_prompt_tokens == 224
    assert mismatches(recs) == []
    rc, occ = b.engine.device_refcounts()
    assert occ == b.kv.occupancy and np.array_equal(rc, b.kv._refcnt)


def _nccl_worker(rank, port, q):
    import torch.distributed as dist

    from paper_2605_26289_b200 import dist as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=2,
                            device_id=torch.device("cuda", rank))
    mig = None
    try:
        tr = load_trace("c3")
        core = InferenceCore(core_config_for(tr, model="tiny", capacity_cells=4096))
        mig = D.PrefixMigrator(core)  # data over the default (NCCL) group
        w = waves(tr)
        first_a, first_b = w[0][0], w[1][0]
        if rank == 0:
            replay(core, {"reqs": [first_a]})
            src = [c for s, n in core.radix.longest_prefix(first_b.tokens).runs
                   for c in range(s, s + n)][:224]
            payload = core.engine.pack_cells(src).cpu()
            dist.send_object_list([payload], dst=1)
        else:
            got = [None]
            dist.recv_object_list(got, src=0)
            while not mig.directory.tries:
                mig.poll()
            recs = replay(core, {"reqs": [first_b]})
            assert mismatches(recs) == []
            cells = [c for s, n in core.radix.longest_prefix(first_b.tokens).runs
                     for c in range(s, s + n)][:224]
            assert torch.equal(core.engine.pack_cells(cells).cpu(), got[0])
            rc, occ = core.engine.device_refcounts()
            assert occ == core.kv.occupancy and np.array_equal(rc, core.kv._refcnt)
            q.put((recs[0].result.cached_prompt_tokens, mig.stats["fetches"],
                   mig.stats["bytes_in"]))
    finally:
        if mig is not None:
            mig.close(timeout_s=60)
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_nccl_prefix_migration_two_gpus(cuda):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_nccl_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    cached, fetches, nbytes = q.get()
    assert cached == 224 and fetches == 1 and nbytes > 0
