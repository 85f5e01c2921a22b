"""Host UnifiedKvCache vs the reference, op by op (golden kvcache_ops from the
reference kvcache.py), plus the device-op log replayed through a numpy model of
ds_kv_apply: the page table it builds must equal cell_ids and the membership
bitmask + trie refs must equal the host refcounts."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden
from paper_2605_26289_b200.kvcache import (CapacityExhausted, DonorRangeInvalid, UnifiedKvCache,
                                           estimate_bytes, slice_runs)

ERRS = {"CapacityExhausted": CapacityExhausted, "DonorRangeInvalid": DonorRangeInvalid,
        "ValueError": ValueError}


class DeviceModel:
    """numpy restatement of kv_apply_kernel (csrc/kvmeta.cu)."""

    def __init__(self, capacity, n_seqs):
        self.pos2cell = np.full((n_seqs, capacity), -1, dtype=np.int64)
        self.member = np.zeros((capacity, n_seqs), dtype=bool)
        self.trie = np.zeros(capacity, dtype=np.int64)
        self.map_ref = np.zeros(capacity, dtype=np.int64)  # exact mappings per cell

    def apply(self, ops):
        for kind, seq, pos, cell, ln in ops:
            if kind == 0:
                self.pos2cell[seq, pos:pos + ln] = np.arange(cell, cell + ln)
                self.member[cell:cell + ln, seq] = True
                self.map_ref[cell:cell + ln] += 1
            elif kind == 1:
                self.member[cell:cell + ln, seq] = False
                self.map_ref[cell:cell + ln] -= 1
            elif kind == 2:
                self.trie[cell:cell + ln] += 1
            else:
                self.trie[cell:cell + ln] -= 1

    def refcount(self):
        return self.member.sum(1) + self.trie

    def exact_refcount(self):
        return self.map_ref + self.trie


def _observe(kv, seqs):
    obs = {"occ": kv.occupancy, "free": kv.free_cells, "seqs": {}}
    for s in seqs:
        n = kv.seq_len(s)
        if n:
            obs["seqs"][str(s)] = {"len": n, "spans": kv.span_count(s),
                                   "cells": kv.cell_ids(s, 0, n)}
    obs["ref"] = {str(int(c)): int(kv._refcnt[c]) for c in np.flatnonzero(kv._refcnt)}
    return obs


def _run_case(case, check_device=True):
    kv = UnifiedKvCache(case["capacity"])
    kv.record_ops = True
    dev = DeviceModel(case["capacity"], 6)
    seqs = list(range(6))
    ever_dup = False  # a seq holding one cell twice breaks the 1-bit-per-seq model
    for op in case["ops"]:
        kind, s = op["op"], op["seq"]
        err = None
        try:
            if kind == "append":
                assert list(kv.append_cells(s, op["n"])) == op["ret"]
            elif kind == "trim":
                assert kv.trim(s, op["pos"]) == op["ret"]
            elif kind == "alias":
                kv.seq_alias(s, op["dest"], op["start"], op["end"])
            elif kind == "alias_runs":
                runs = [tuple(r) for r in op["runs"]]
                kv.alias_runs(op["dest"], runs)
                kv.incref_runs(runs)
            elif kind == "decref":
                assert kv.decref_runs([tuple(r) for r in op["runs"]]) == op["ret"]
            else:
                assert kv.release_sequence(s) == op["ret"]
        except (CapacityExhausted, DonorRangeInvalid, ValueError) as exc:
            err = type(exc).__name__
        assert err == op["err"], (op, err)
        assert _observe(kv, seqs) == op["obs"], op
        dev.apply(kv.take_ops())
        if check_device:
            dup = any(len(set(v["cells"])) != len(v["cells"]) for v in op["obs"]["seqs"].values())
            for s2, v in op["obs"]["seqs"].items():
                assert dev.pos2cell[int(s2), : v["len"]].tolist() == v["cells"]
            ever_dup |= dup
            # the op log mirrors every refcount change, failed ops included
            # (a failed decref logs the runs it dropped, a failed alias the
            # holds it left): exact after every op
            assert np.array_equal(dev.exact_refcount(), kv._refcnt), op
            if not ever_dup:
                assert np.array_equal(dev.refcount(), kv._refcnt), op


def test_golden_op_sequences():
    cases = load_golden("kvcache_ops.json.gz")
    assert len(cases) >= 50
    for case in cases:
        _run_case(case)


def test_reference_unit_cases():
    kv = UnifiedKvCache(30_000)
    kv.append_cells(1, 10_000)
    kv.seq_alias(1, 2, 0, 100)
    kv.seq_alias(1, 3, 0, 10_000)
    assert kv.span_count(2) == 1 and kv.span_count(3) == 1
    kv2 = UnifiedKvCache(8)
    with pytest.raises(CapacityExhausted):
        kv2.append_cells(1, 10)
    assert kv2.occupancy == 0
    assert estimate_bytes(32, 4096, 1000, 2) == 524_288_000
    runs = [(0, 4), (10, 3), (20, 5)]
    assert slice_runs(runs, 2, 4) == [(2, 2), (10, 2)]
    assert slice_runs(runs, 4, 8) == [(10, 3), (20, 5)]
    assert slice_runs(runs, 5, 1) == [(11, 1)]
