"""Shared fixtures: golden fixtures, CUDA availability, the oracle engine."""
from __future__ import annotations

import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name: str):
    with gzip.open(os.path.join(GOLDEN, name), "rb") as fh:
        return json.loads(fh.read())


@pytest.fixture(scope="session")
def golden_kernels():
    return load_golden("kernels.json.gz")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_26289_b200 import _lib

    _lib.lib()  # fails loudly if the sm_100a library is missing
    return torch.device("cuda", 0)


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    """(Re)build the sm_100a library and the C oracle if sources are newer."""
    from oracle import cpu
    from paper_2605_26289_b200 import build

    build.build()
    cpu.build()


def record_numeric(name: str, **values) -> None:
    """Append one measured error record (max-abs, rel RMS, floor ...) to
    gpurun_out/numerics.jsonl - the evidence behind the tolerances stated in
    DESIGN.md section 4 (copied to profiles/ per round)."""
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "numerics.jsonl"), "a") as fh:
        fh.write(json.dumps({"case": name, **values}) + "\n")
