"""The C-ABI library loads and exports every symbol include/deltaserve_b200.h declares
(no compute calls - this runs without a GPU)."""
from __future__ import annotations

import ctypes
import os

import pytest

from paper_2605_26289_b200 import _lib


def test_library_built_for_sm100a():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build() first"


def test_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    declared = _lib.exported_symbols()
    assert len(declared) >= 20
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing


def test_struct_layouts():
    assert ctypes.sizeof(_lib.Entry) == 40
    assert ctypes.sizeof(_lib.KvOp) == 20


def test_host_hash_matches_oracle():
    from oracle import cpu
    from paper_2605_26289_b200 import kernels

    toks = [1, 2, 3, 70000, -5, 2**31 - 1]
    assert kernels.host_fnv1a64_tokens(toks) == cpu.fnv1a64_tokens(toks)
    assert kernels.host_fnv1a32_tokens(toks) == cpu.fnv1a32_tokens(toks)
    assert kernels.host_fnv1a64_tokens(toks[3:], kernels.host_fnv1a64_tokens(toks[:3])) == \
        cpu.fnv1a64_tokens(toks)


def test_no_cpu_fallback_in_product_kernels(monkeypatch):
    import torch

    from paper_2605_26289_b200 import kernels

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        kernels.copy_continuation([1, 2, 3, 1, 2], 2)
