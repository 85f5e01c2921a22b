"""Device kernels behind the reference's ``deltaserve._kernels`` API.

Same names and semantics as the reference module (_kernels/__init__.py:21-73,
_native.pyx:18-119) - single call, host ints in and out - but every call runs
on the GPU through the C ABI (H2D, kernel, D2H).  There is no backend switch
and no CPU implementation: ``BACKEND`` is always ``"cuda-sm100a"``.  The
batched ``*_batched`` variants take device tensors and are what the engine and
scheduler use.

``host_fnv1a64_tokens`` / ``host_fnv1a32_tokens`` are the native host hashes the
scheduler uses for its own bookkeeping keys (Slot.prefix_hash, window hash;
scheduler.py:237, 489-490, 687, 715), exactly as the reference scheduler
hashes on the host.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from . import _hostcore
from ._lib import check, lib, stream_ptr

BACKEND = "cuda-sm100a"
FNV32_OFFSET = 0x811C9DC5
FNV32_PRIME = 0x01000193
FNV64_OFFSET = 0xCBF29CE484222325
FNV64_PRIME = 0x100000001B3


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("deltaserve_b200 kernels need a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _as_i32(tokens) -> np.ndarray:
    if isinstance(tokens, torch.Tensor):
        tokens = tokens.detach().cpu().numpy()
    if isinstance(tokens, list):
        try:  # ~30% faster than asarray on long token lists
            return np.fromiter(tokens, dtype=np.int32, count=len(tokens))
        except (OverflowError, TypeError, ValueError):
            pass
    a = np.asarray(tokens)
    if a.dtype != np.int32:
        a = a.astype(np.int64).astype(np.int32)
    return np.ascontiguousarray(a)


def _signed64(v: int) -> int:
    v &= 2**64 - 1
    return v - 2**64 if v >= 2**63 else v


def _pack(seqs) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Concatenate int32 sequences onto the device with offsets/lengths."""
    arrs = [_as_i32(s) for s in seqs]
    lengths = np.array([len(a) for a in arrs], dtype=np.int32)
    offsets = np.zeros(len(arrs), dtype=np.int64)
    if len(arrs) > 1:
        offsets[1:] = np.cumsum(lengths[:-1])
    flat = np.concatenate(arrs) if arrs and lengths.sum() else np.zeros(1, dtype=np.int32)
    dev = _device()
    return (torch.from_numpy(flat).to(dev), torch.from_numpy(offsets).to(dev),
            torch.from_numpy(lengths).to(dev))


# ---------------------------------------------------------------------------
# batched device API
# ---------------------------------------------------------------------------

def fnv1a_tokens_batched(seqs, bits: int = 64, states=None) -> list[int]:
    base, off, ln = _pack(seqs)
    n = len(seqs)
    out = torch.empty(max(n, 1), dtype=torch.int64, device=base.device)
    st = None
    if states is not None:
        st = torch.tensor([_signed64(int(s)) for s in states], dtype=torch.int64).to(base.device)
    check(lib().ds_fnv1a_tokens(base.data_ptr(), off.data_ptr(), ln.data_ptr(), n, bits,
                                _lib.ptr(st), out.data_ptr(), stream_ptr()), "ds_fnv1a_tokens")
    return [int(v) & (2**64 - 1) for v in out[:n].cpu().tolist()]


def copy_continuation_batched(seqs, min_match: int) -> list[int]:
    base, off, ln = _pack(seqs)
    n = len(seqs)
    out = torch.empty(max(n, 1), dtype=torch.int32, device=base.device)
    check(lib().ds_copy_continuation(base.data_ptr(), off.data_ptr(), ln.data_ptr(), n, min_match,
                                     out.data_ptr(), stream_ptr()), "ds_copy_continuation")
    return out[:n].cpu().tolist()


def longest_suffix_match_batched(rings, tails, min_len: int, caps=None, max_draft: int = 0):
    """K1 over many slots. Returns (e list, len list[, drafts list])."""
    rb, ro, rl = _pack(rings)
    if tails is None:
        tb, to, tl = rb, ro, rl
    else:
        tb, to, tl = _pack(tails)
    n = len(rings)
    e = torch.empty(max(n, 1), dtype=torch.int32, device=rb.device)
    ln = torch.empty_like(e)
    caps_t = drafts = dlen = None
    if caps is not None:
        caps_t = torch.tensor(list(caps), dtype=torch.int32).to(rb.device)
        max_draft = max(1, max_draft)
        drafts = torch.empty(max(n, 1) * max_draft, dtype=torch.int32, device=rb.device)
        dlen = torch.empty_like(e)
    check(lib().ds_longest_suffix_match(rb.data_ptr(), ro.data_ptr(), rl.data_ptr(), tb.data_ptr(),
                                        to.data_ptr(), tl.data_ptr(), n, min_len,
                                        _lib.ptr(caps_t), max_draft, e.data_ptr(), ln.data_ptr(),
                                        _lib.ptr(drafts), _lib.ptr(dlen), stream_ptr()),
          "ds_longest_suffix_match")
    es, ls = e[:n].cpu().tolist(), ln[:n].cpu().tolist()
    if caps is None:
        return es, ls
    d = drafts.view(-1, max_draft).cpu().tolist()
    dl = dlen[:n].cpu().tolist()
    return es, ls, [d[i][: dl[i]] for i in range(n)]


# ---------------------------------------------------------------------------
# reference-named single-call API (device-backed)
# ---------------------------------------------------------------------------

def _bytes_call(data: bytes, bits: int) -> int:
    dev = _device()
    buf = torch.frombuffer(bytearray(data or b"\0"), dtype=torch.uint8).to(dev)
    off = torch.zeros(1, dtype=torch.int64, device=dev)
    ln = torch.tensor([len(data)], dtype=torch.int32, device=dev)
    out = torch.empty(1, dtype=torch.int64, device=dev)
    check(lib().ds_fnv1a_bytes(buf.data_ptr(), off.data_ptr(), ln.data_ptr(), 1, bits,
                               out.data_ptr(), stream_ptr()), "ds_fnv1a_bytes")
    return int(out.item()) & (2**64 - 1)


def fnv1a32_bytes(data: bytes) -> int:
    return _bytes_call(bytes(data), 32)


def fnv1a64_bytes(data: bytes) -> int:
    return _bytes_call(bytes(data), 64)


def fnv1a32_tokens(tokens, state: int | None = None) -> int:
    return fnv1a_tokens_batched([tokens], 32, None if state is None else [state])[0]


def fnv1a64_tokens(tokens, state: int | None = None) -> int:
    return fnv1a_tokens_batched([tokens], 64, None if state is None else [state])[0]


def copy_continuation(tokens, min_match: int) -> int:
    return copy_continuation_batched([tokens], min_match)[0]


def longest_suffix_match(ring, tail, min_len: int) -> tuple[int, int]:
    e, ln = longest_suffix_match_batched([ring], [tail], min_len)
    return e[0], ln[0]


# ---------------------------------------------------------------------------
# native host hashing for scheduler bookkeeping
# ---------------------------------------------------------------------------

def host_fnv1a64_tokens(tokens, state: int | None = None) -> int:
    """Host bookkeeping hash (native host core; same function as the library's
    ds_host_fnv1a64_tokens, reference _native.pyx:47-59)."""
    return _hostcore.fnv1a64_tokens(tokens, 0, len(tokens),
                                    FNV64_OFFSET if state is None else state)


def host_fnv1a32_tokens(tokens, state: int | None = None) -> int:
    return _hostcore.fnv1a32_tokens(tokens, 0, len(tokens),
                                    FNV32_OFFSET if state is None else state)


def prompt_seed(tokens) -> int:
    """Sampler seed = FNV-1a32 of the prompt (caches.py:22-24)."""
    return host_fnv1a32_tokens(tokens)


__all__ = [
    "BACKEND", "fnv1a32_bytes", "fnv1a64_bytes", "fnv1a32_tokens", "fnv1a64_tokens",
    "copy_continuation", "longest_suffix_match", "fnv1a_tokens_batched",
    "copy_continuation_batched", "longest_suffix_match_batched", "host_fnv1a64_tokens",
    "host_fnv1a32_tokens", "prompt_seed", "ctypes",
]
