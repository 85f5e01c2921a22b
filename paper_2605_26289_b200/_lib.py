"""ctypes binding of the C ABI in include/deltaserve_b200.h.

The product path has no CPU fallback: if libdeltaserve_b200.so is missing or
no CUDA device is visible, calls fail loudly.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# DS_B200_LIB: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("DS_B200_LIB") or os.path.join(HERE, "libdeltaserve_b200.so")

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_vp = ctypes.c_void_p
c_f32 = ctypes.c_float


class KvOp(ctypes.Structure):
    _fields_ = [("kind", c_i32), ("seq", c_i32), ("pos", c_i32), ("cell", c_i32), ("len", c_i32)]


KV_MAP, KV_UNMAP, KV_TRIE_INC, KV_TRIE_DEC, KV_MAP_SCRATCH = 0, 1, 2, 3, 4


class Model(ctypes.Structure):
    _fields_ = [("layers", c_i32), ("hidden", c_i32), ("n_heads", c_i32), ("n_kv_heads", c_i32),
                ("head_dim", c_i32), ("ffn", c_i32), ("vocab", c_i32), ("rms_eps", c_f32),
                ("embed", c_vp), ("attn_norm", c_vp), ("wqkv", c_vp), ("wo", c_vp),
                ("mlp_norm", c_vp), ("w_gate_up", c_vp), ("w_down", c_vp), ("final_norm", c_vp),
                ("lm_head", c_vp), ("rope_cos", c_vp), ("rope_sin", c_vp),
                ("rope_max_pos", c_i32)]


class KvStore(ctypes.Structure):
    _fields_ = [("k_pool", c_vp), ("v_pool", c_vp), ("capacity", c_i64), ("pos2cell", c_vp),
                ("hist", c_vp), ("pos_stride", c_i64), ("n_seqs", c_i32)]


class Entry(ctypes.Structure):
    _fields_ = [("seq", c_i32), ("past", c_i32), ("q_len", c_i32), ("q_start", c_i32),
                ("kind", c_i32), ("n_draft", c_i32), ("out_start", c_i32), ("n_out", c_i32),
                ("hash_in", c_u64)]


ENTRY_PREFILL, ENTRY_DECODE, ENTRY_VERIFY = 0, 1, 2
POLICY_COPY, POLICY_ARGMAX = 0, 1




class SkinnyEpi(ctypes.Structure):
    """ds_skinny_epi: epilogue fusions of ds_gemm_skinny_ex."""
    _fields_ = [("row_ss", c_vp), ("eps", c_f32), ("ss_out", c_vp), ("ss_zero", c_vp),
                ("h_out", c_vp), ("h_w", c_vp), ("swiglu", c_i32), ("rope", c_i32),
                ("n_heads", c_i32), ("n_kv_heads", c_i32), ("row_seq", c_vp), ("row_pos", c_vp),
                ("pos2cell", c_vp), ("pos_stride", c_i64), ("rope_cos", c_vp),
                ("rope_sin", c_vp), ("k_pool_l", c_vp), ("v_pool_l", c_vp),
                ("kv_head_stride", c_i64), ("l2_next", c_vp), ("l2_next_bytes", c_i64),
                ("argmax_out", c_vp), ("l2_pre", c_vp), ("l2_pre_bytes", c_i64)]


class ForwardArgs(ctypes.Structure):
    _fields_ = [("n_entries", c_i32), ("n_rows", c_i32), ("n_out", c_i32), ("policy", c_i32),
                ("copy_min_match", c_i32), ("policy_vocab", c_i32), ("entries_host", c_vp),
                ("entries", c_vp), ("tokens", c_vp), ("row_seq", c_vp), ("row_pos", c_vp),
                ("out_rows", c_vp), ("out_tok", c_vp), ("out_src", c_vp), ("out_accept", c_vp),
                ("logits", c_vp), ("workspace", c_vp), ("workspace_bytes", ctypes.c_size_t),
                ("next_window", c_i32), ("next_min_match", c_i32), ("next_cap", c_i32),
                ("next_out", c_vp), ("logits_out", c_i32)]


assert ctypes.sizeof(Entry) == 40


class CudaLibraryMissing(RuntimeError):
    pass


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise CudaLibraryMissing(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    import torch  # noqa: F401  (load torch's CUDA/cuBLAS first so sonames are shared)

    L = ctypes.CDLL(LIB_PATH)
    P = c_vp
    sigs = {
        "ds_abi_version": (c_i32, []),
        "ds_status_string": (ctypes.c_char_p, [c_i32]),
        "ds_fnv1a_tokens": (c_i32, [P, P, P, c_i32, c_i32, P, P, P]),
        "ds_fnv1a_bytes": (c_i32, [P, P, P, c_i32, c_i32, P, P]),
        "ds_copy_continuation": (c_i32, [P, P, P, c_i32, c_i32, P, P]),
        "ds_longest_suffix_match": (c_i32, [P, P, P, P, P, P, c_i32, c_i32, P, c_i32, P, P, P, P,
                                            P]),
        "ds_host_fnv1a64_tokens": (c_u64, [P, c_i64, c_u64]),
        "ds_host_fnv1a32_tokens": (ctypes.c_uint32, [P, c_i64, ctypes.c_uint32]),
        "ds_kv_apply": (c_i32, [P, c_i32, P, c_i64, c_i32, P, c_i32, P, P, P]),
        "ds_hist_write": (c_i32, [P, P, c_i32, P, c_i64, P]),
        "ds_kv_copy_cells": (c_i32, [P, P, c_i32, c_i32, c_i64, c_i32, P, c_i32, P]),
        "ds_kv_refcount": (c_i32, [P, c_i32, P, P, c_i64, P, P, P]),
        "ds_kv_pack_cells": (c_i32, [P, P, c_i32, c_i32, c_i64, c_i32, P, c_i32, P, c_i32, P]),
        "ds_forward_workspace_bytes": (ctypes.c_size_t, [P, c_i32, c_i32, c_i32]),
        "ds_model_forward": (c_i32, [P, P, P, P]),
        "ds_rope_kv_store": (c_i32, [P, c_i32, P, P, P, c_i64, c_i32, c_i32, c_i32, P, P, P, P,
                                     c_i64, P]),
        "ds_attention_workspace_bytes": (ctypes.c_size_t, [c_i32, c_i32, c_i32, c_i32]),
        "ds_attention": (c_i32, [P, P, P, c_i32, c_i32, P, P, c_i64, P, c_i64, c_i32, c_i32,
                                 c_i32, c_f32, P, P, ctypes.c_size_t, c_i32, P]),
        "ds_rmsnorm": (c_i32, [P, c_i32, P, c_i32, c_i32, P, c_f32, P, P]),
        "ds_silu_mul": (c_i32, [P, c_i32, c_i32, P, P]),
        "ds_embed": (c_i32, [P, c_i32, P, c_i32, P, c_i32, P]),
        "ds_argmax": (c_i32, [P, c_i32, c_i32, P, P]),
        "ds_gemm_skinny": (c_i32, [P, P, P, c_i32, c_i32, c_i32, c_i32, c_i32, P]),
        "ds_gemm_skinny_ex": (c_i32, [P, P, P, c_i32, c_i32, c_i32, c_i32, c_i32, P, P]),
        "ds_gemm_stream": (c_i32, [P, P, P, c_i32, c_i32, c_i32, c_i32, c_i32, P, P]),
        "ds_gemm_pair": (c_i32, [P, P, P, c_i32, c_i32, c_i32, c_i32, c_i32, P, P]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def exported_symbols() -> list[str]:
    """Every function the C header declares (checked by the CPU test suite)."""
    import re

    hdr = os.path.join(os.path.dirname(HERE), "include", "deltaserve_b200.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"\b(ds_[a-z0-9_]+)\(", text)))


def check(status: int, what: str = "") -> None:
    if status != 0:
        msg = lib().ds_status_string(status).decode()
        raise RuntimeError(f"{what or 'deltaserve_b200'} failed: status {status} ({msg})")


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()
