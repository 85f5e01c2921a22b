"""K4 metadata kernels: the host UnifiedKvCache op log applied on the device
(ds_kv_apply) reproduces the reference page tables (cell ids) and refcounts
(popcount of the sequence-membership bitmask + radix holds) - with 0 KV bytes
moved."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import load_golden
from paper_2605_26289_b200.kvcache import CapacityExhausted, DonorRangeInvalid, UnifiedKvCache

pytestmark = pytest.mark.gpu


def _apply(cuda, ops, pos2cell, member, trie, n_seqs, map_ref=None):
    from paper_2605_26289_b200._lib import check, lib

    ops = np.asarray(ops, dtype=np.int32).reshape(-1, 5)
    if not len(ops):
        return
    o = torch.tensor(ops).to(cuda)
    check(lib().ds_kv_apply(o.data_ptr(), len(ops), pos2cell.data_ptr(), pos2cell.shape[1],
                            n_seqs, member.data_ptr(), member.shape[1], trie.data_ptr(),
                            None if map_ref is None else map_ref.data_ptr(),
                            torch.cuda.current_stream().cuda_stream))


def _refcount(cuda, member, trie, map_ref=None):
    """map_ref + trie_ref (exact), or popcount(member) + trie_ref without map_ref."""
    from paper_2605_26289_b200._lib import check, lib

    cap = member.shape[0]
    rc = torch.empty(cap, dtype=torch.int32, device=cuda)
    occ = torch.zeros(1, dtype=torch.int32, device=cuda)
    check(lib().ds_kv_refcount(member.data_ptr(), member.shape[1], trie.data_ptr(),
                               None if map_ref is None else map_ref.data_ptr(), cap,
                               rc.data_ptr(), occ.data_ptr(),
                               torch.cuda.current_stream().cuda_stream))
    return rc.cpu().numpy(), int(occ.item())


def test_golden_ops_on_device(cuda):
    cases = load_golden("kvcache_ops.json.gz")
    checked = dup_free = 0
    for case in cases:
        cap = case["capacity"]
        kv = UnifiedKvCache(cap)
        kv.record_ops = True
        pos2cell = torch.full((6, cap), -1, dtype=torch.int32, device=cuda)
        member = torch.zeros((cap, 1), dtype=torch.int32, device=cuda)
        trie = torch.zeros(cap, dtype=torch.int32, device=cuda)
        map_ref = torch.zeros(cap, dtype=torch.int32, device=cuda)
        ever_dup = False
        for op in case["ops"]:
            s = op["seq"]
            try:
                if op["op"] == "append":
                    kv.append_cells(s, op["n"])
                elif op["op"] == "trim":
                    kv.trim(s, op["pos"])
                elif op["op"] == "alias":
                    kv.seq_alias(s, op["dest"], op["start"], op["end"])
                elif op["op"] == "alias_runs":
                    runs = [tuple(r) for r in op["runs"]]
                    kv.alias_runs(op["dest"], runs)
                    kv.incref_runs(runs)
                elif op["op"] == "decref":
                    kv.decref_runs([tuple(r) for r in op["runs"]])
                else:
                    kv.release_sequence(s)
            except (CapacityExhausted, DonorRangeInvalid, ValueError):
                pass
            _apply(cuda, kv.take_ops(), pos2cell, member, trie, 6, map_ref)
            p2c = pos2cell.cpu().numpy()
            for seq in range(6):
                n = kv.seq_len(seq)
                cells = kv.cell_ids(seq, 0, n) if n else []
                assert p2c[seq, :n].tolist() == cells
                ever_dup |= len(set(cells)) != len(cells)
            # exact mappings per cell: the refcount holds after every op, also
            # once a sequence maps a cell twice
            rc, occ = _refcount(cuda, member, trie, map_ref)
            assert np.array_equal(rc, kv._refcnt)
            assert occ == int(np.count_nonzero(kv._refcnt))
            checked += 1
            if not ever_dup:  # the membership bits (one per sequence) until then
                rc, occ = _refcount(cuda, member, trie)
                assert np.array_equal(rc, kv._refcnt)
                dup_free += 1
    assert checked > 500 and dup_free > 500


@pytest.mark.parametrize("n_seqs", [300, 2000])
def test_many_sequences_large_flushes(cuda, n_seqs):
    """The per-sequence parallel apply (one warp per sequence across the grid,
    atomics on shared membership words and counters) over 300 sequences and
    flushes of thousands of ops, with cells trimmed and re-allocated inside one
    flush - page tables and exact refcounts equal the host allocator's."""
    import random

    rng = random.Random(11 + n_seqs)
    cap = 60000  # 2000 sequences: more than the grid's 1184 warps, a warp owns several
    kv = UnifiedKvCache(cap)
    kv.record_ops = True
    pos2cell = torch.full((n_seqs, 4096), -1, dtype=torch.int32, device=cuda)
    member = torch.zeros((cap, (n_seqs + 31) // 32), dtype=torch.int32, device=cuda)
    trie = torch.zeros(cap, dtype=torch.int32, device=cuda)
    map_ref = torch.zeros(cap, dtype=torch.int32, device=cuda)
    for flush in range(12):
        for _ in range(1500):
            s = rng.randrange(n_seqs)
            n = kv.seq_len(s)
            r = rng.random()
            try:
                if r < 0.55 and n < 3000:
                    kv.append_cells(s, rng.randrange(1, 40))
                elif r < 0.8 and n:
                    kv.trim(s, rng.randrange(n))
                elif r < 0.95 and n:
                    d = rng.randrange(n_seqs)
                    if d != s and kv.seq_len(d) == 0:
                        kv.seq_alias(s, d, 0, rng.randrange(1, n + 1))
                else:
                    kv.release_sequence(s)
            except (CapacityExhausted, DonorRangeInvalid, ValueError):
                pass
        ops = kv.take_ops()
        _apply(cuda, ops, pos2cell, member, trie, n_seqs, map_ref)
        p2c = pos2cell.cpu().numpy()
        for seq in range(n_seqs):
            n = kv.seq_len(seq)
            if n:
                assert p2c[seq, :n].tolist() == kv.cell_ids(seq, 0, n)
        rc, occ = _refcount(cuda, member, trie, map_ref)
        assert np.array_equal(rc, kv._refcnt)
        assert occ == int(np.count_nonzero(kv._refcnt))
