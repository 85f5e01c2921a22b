"""ctypes binding of oracle/ds_oracle.c (test infrastructure only).

Each function mirrors one reference kernel; citations are in ds_oracle.c.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libds_oracle.so")
_SRC = os.path.join(_HERE, "ds_oracle.c")


def build() -> str:
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", _SO, _SRC])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.oracle_fnv1a32_bytes.restype = ctypes.c_uint32
        L.oracle_fnv1a32_bytes.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
        L.oracle_fnv1a64_bytes.restype = ctypes.c_uint64
        L.oracle_fnv1a64_bytes.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
        L.oracle_fnv1a32_tokens.restype = ctypes.c_uint32
        L.oracle_fnv1a32_tokens.argtypes = [i32p, ctypes.c_size_t, ctypes.c_uint32]
        L.oracle_fnv1a64_tokens.restype = ctypes.c_uint64
        L.oracle_fnv1a64_tokens.argtypes = [i32p, ctypes.c_size_t, ctypes.c_uint64]
        L.oracle_copy_continuation.restype = ctypes.c_int64
        L.oracle_copy_continuation.argtypes = [i32p, ctypes.c_int64, ctypes.c_int64]
        L.oracle_longest_suffix_match.restype = None
        L.oracle_longest_suffix_match.argtypes = [
            i32p, ctypes.c_int64, i32p, ctypes.c_int64, ctypes.c_int64,
            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        L.oracle_copy_policy.restype = None
        L.oracle_copy_policy.argtypes = [i32p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                         i32p, i32p]
        _lib = L
    return _lib


FNV32_OFFSET = 0x811C9DC5
FNV64_OFFSET = 0xCBF29CE484222325


def _arr(tokens) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(tokens, dtype=np.int64).astype(np.int32))


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def fnv1a32_bytes(data: bytes) -> int:
    return int(lib().oracle_fnv1a32_bytes(data, len(data)))


def fnv1a64_bytes(data: bytes) -> int:
    return int(lib().oracle_fnv1a64_bytes(data, len(data)))


def fnv1a32_tokens(tokens, state=None) -> int:
    a = _arr(tokens)
    return int(lib().oracle_fnv1a32_tokens(_p(a), len(a), FNV32_OFFSET if state is None else state))


def fnv1a64_tokens(tokens, state=None) -> int:
    a = _arr(tokens)
    return int(lib().oracle_fnv1a64_tokens(_p(a), len(a), FNV64_OFFSET if state is None else state))


def copy_continuation(tokens, min_match: int) -> int:
    a = _arr(tokens)
    return int(lib().oracle_copy_continuation(_p(a), len(a), min_match))


def longest_suffix_match(ring, tail, min_len: int) -> tuple[int, int]:
    r, t = _arr(ring), _arr(tail)
    e, ln = ctypes.c_int64(), ctypes.c_int64()
    lib().oracle_longest_suffix_match(_p(r), len(r), _p(t), len(t), min_len,
                                      ctypes.byref(e), ctypes.byref(ln))
    return int(e.value), int(ln.value)


def copy_policy(full, upto: int, min_match: int, vocab: int) -> tuple[int, int]:
    """(token, copy_source or -1) for the row whose preceding sequence is full[:upto]."""
    a = _arr(full)
    tok, src = ctypes.c_int32(), ctypes.c_int32()
    lib().oracle_copy_policy(_p(a), upto, min_match, vocab, ctypes.byref(tok), ctypes.byref(src))
    return int(tok.value), int(src.value)


def lookup_ngram(ring, tail, min_match: int, max_tokens: int) -> list[int]:
    """speculator.py:52-65 restated on top of longest_suffix_match."""
    if max_tokens <= 0:
        return []
    e, ln = longest_suffix_match(ring, tail, min_match)
    if e < 0 or ln < min_match:
        return []
    take = min(max_tokens, len(ring) - e)
    return [int(x) for x in ring[e:e + take]]
