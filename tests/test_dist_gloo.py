"""Multi-GPU host logic on CPU (gloo, world_size 2): session routing, the prefix
directory, and prefix migration between two cores - the migrated prefix must
produce the same radix hit the reference core produces locally (C3: the
second agent restores the 224-token shared tool-schema prefix)."""
from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cpu
from paper_2605_26289_b200 import dist as D

L, NKV, HD, CAP = 2, 2, 8, 4096


def test_route_is_reference_fnv32():
    for sid in ["a", "session-17", "agent/coding/3", ""]:
        assert D.route(sid, 8) == cpu.fnv1a32_bytes(sid.encode()) % 8
    counts = [0] * 4
    for i in range(400):
        counts[D.route(f"c5s{i}", 4)] += 1
    assert min(counts) > 60  # roughly balanced


def test_pack_unpack_roundtrip():
    k = torch.randn(L, NKV, 64, HD)
    v = torch.randn(L, NKV, 64, HD)
    cells = [3, 9, 10, 40]
    buf = D.pack_cells(k, v, cells)
    assert buf.shape == (L, 2, NKV, 4, HD)
    k2, v2 = torch.zeros_like(k), torch.zeros_like(v)
    D.unpack_cells(k2, v2, [0, 1, 2, 3], buf)
    assert torch.equal(k2[:, :, :4], k[:, :, cells]) and torch.equal(v2[:, :, :4], v[:, :, cells])


def _make_core():
    from oracle_engine import OracleEngine
    from paper_2605_26289_b200.scheduler import InferenceCore
    from paper_2605_26289_b200.workload import core_config_for, load_trace

    tr = load_trace("c3")
    cfg = core_config_for(tr, model="tiny", capacity_cells=CAP)
    eng = OracleEngine(cfg.vocab, cfg.copy_min_match)
    eng.k_pool = torch.zeros(L, NKV, CAP, HD)
    eng.v_pool = torch.zeros(L, NKV, CAP, HD)
    return InferenceCore(cfg, engine=eng), tr


def _worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2605_26289_b200.workload import replay, waves

        core, tr = _make_core()
        w = waves(tr)
        first_a, first_b = w[0][0], w[1][0]  # agent A turn 0, agent B turn 0
        shared = 224  # reference C3: B's first turn restores 224 cached tokens
        prefix = first_b.tokens[:shared]
        if rank == 0:
            replay(core, {"reqs": [first_a]})  # A's turn commits the schema prefix
            cells = D.export_prefix(core, prefix)
            assert len(cells) == shared
            eng = core.engine
            for c in range(CAP):  # deterministic per-cell payload
                eng.k_pool[:, :, c, :] = c
                eng.v_pool[:, :, c, :] = -c
            dist.send_object_list([cells], dst=1)
        else:
            src_cells = [None]
            dist.recv_object_list(src_cells, src=0)
        directory = D.PrefixDirectory()
        if rank == 0:
            directory.publish_local(0, [(cpu.fnv1a64_tokens(prefix), shared)])
        directory.sync()
        owner = directory.owner(cpu.fnv1a64_tokens(prefix))
        assert owner is not None and owner.rank == 0 and owner.length == shared
        nbytes = D.migrate_prefix(core, core, prefix, 0, 1)
        assert nbytes == L * 2 * NKV * shared * HD * 4
        if rank == 1:
            got = D.export_prefix(core, prefix)
            assert len(got) == shared
            eng = core.engine
            exp = torch.tensor(src_cells[0], dtype=torch.float32)
            assert torch.equal(eng.k_pool[0, 0, got, 0], exp)
            assert torch.equal(eng.v_pool[1, 1, got, 3], -exp)
            recs = replay(core, {"reqs": [first_b]})
            q.put(("hit", recs[0].result.cached_prompt_tokens,
                   first_b.expect["cached_prompt_tokens"]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_prefix_migration_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    tag, got, expected = q.get()
    assert tag == "hit" and got == expected == 224
