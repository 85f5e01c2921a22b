"""ORACLE - CPU fp32 restatement of the decoder the GPU engine runs (test only).

The reference artifact has NO model (engine.py:1-17 is a copy-model mock;
SPEC.md:18 puts GPU execution out of scope), so attention / logits parity is
pinned only by this restatement of standard Llama-3 math (PAPER.md:293:
Llama-3.1-8B): RMSNorm (eps 1e-5), rotate-half RoPE (theta 500000, fp64
angles), GQA attention, SwiGLU MLP, untied LM head.  It rounds to bf16 at
exactly the tensor boundaries the GPU stores (norm outputs, projections,
roped q/k, KV cache, attention output, MLP activations) and keeps the
residual stream and every accumulation in fp32, so the tolerance budget is only the
accumulation-order / bf16-P difference.  Measured: per
attention kernel max-abs <= 1e-2 (9e-3 worst); logits through the 8B layer
shapes 4.6e-2 .. 5.6e-2 max-abs against this oracle's own fp32-vs-fp64 floor
of 2.5e-2 - the stated logits bound is 6e-2 (tests/test_gpu_numerics_8b.py).
"""
from __future__ import annotations

import torch




def qk_perm(d: int = 128) -> torch.Tensor:
    """perm[c] = head dim stored at column c of a q/k head in the wqkv layout
    (RoPE-pair interleaved, include/deltaserve_b200.h ds_model.wqkv)."""
    c = torch.arange(d)
    t, j = c // 16, c % 16
    return torch.where(j < 8, 8 * t + j, d // 2 + 8 * t + j - 8)


def unpermute_qk(qkv: torch.Tensor, nh: int, nkv: int, d: int) -> torch.Tensor:
    """qkv columns in wqkv order -> plain dim order for the q and k heads."""
    inv = torch.argsort(qk_perm(d))
    T = qkv.shape[0]
    qk = qkv[:, : (nh + nkv) * d].reshape(T, nh + nkv, d)[:, :, inv].reshape(T, -1)
    return torch.cat([qk, qkv[:, (nh + nkv) * d:]], dim=1)

def split_gate_up(gu, ffn: int):
    """gate, up from a gate|up projection whose weight rows are interleaved in
    8-unit blocks (row 16b+j: j<8 gate unit 8b+j, else up unit 8b+j-8) - the
    ds_model.w_gate_up layout (include/deltaserve_b200.h)."""
    v = gu.reshape(*gu.shape[:-1], ffn // 8, 2, 8)
    return v[..., 0, :].reshape(*gu.shape[:-1], ffn), v[..., 1, :].reshape(*gu.shape[:-1], ffn)

def _bf(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).float()


def rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    inv = torch.rsqrt((x * x).mean(-1, keepdim=True) + eps)
    return _bf(x * inv * w)


def rope_tables(n_pos: int, head_dim: int, theta: float):
    inv = theta ** (-torch.arange(0, head_dim, 2, dtype=torch.float64) / head_dim)
    ang = torch.arange(n_pos, dtype=torch.float64)[:, None] * inv[None, :]
    return torch.cos(ang).float(), torch.sin(ang).float()


def rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """x [T, H, d]; cos/sin [T, d/2] -> rotate-half RoPE rounded to bf16."""
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    c, s = cos[:, None, :], sin[:, None, :]
    return _bf(torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1))


@torch.no_grad()
def forward(w: dict, shape, tokens: list[int], out_rows: list[int] | None = None,
            threads: int | None = None) -> torch.Tensor:
    """Logits [len(out_rows), V] (fp32) for one causal sequence of `tokens`.

    w: fp32 CPU copies of the bf16 weights (GpuEngine.weights_cpu()).
    """
    if threads:
        torch.set_num_threads(threads)
    T = len(tokens)
    nh, nkv, d = shape.n_heads, shape.n_kv_heads, shape.head_dim
    G = nh // nkv
    cos, sin = rope_tables(T, d, shape.rope_theta)
    x = w["embed"][torch.tensor(tokens, dtype=torch.long)]
    mask = torch.full((T, T), float("-inf")).triu(1)
    scale = 1.0 / (d ** 0.5)
    for l in range(shape.layers):
        h = rmsnorm(x, w["attn_norm"][l], shape.rms_eps)
        qkv = unpermute_qk(_bf(h @ w["wqkv"][l].T), nh, nkv, d)
        q = qkv[:, : nh * d].view(T, nh, d)
        k = qkv[:, nh * d: (nh + nkv) * d].view(T, nkv, d)
        v = qkv[:, (nh + nkv) * d:].view(T, nkv, d)
        q, k = rope(q, cos, sin), rope(k, cos, sin)
        kr = k.repeat_interleave(G, dim=1)  # [T, nh, d]
        vr = v.repeat_interleave(G, dim=1)
        s = torch.einsum("qhd,khd->hqk", q, kr) * scale + mask
        p = torch.softmax(s, dim=-1)
        o = _bf(torch.einsum("hqk,khd->qhd", p, vr).reshape(T, nh * d))
        x = x + o @ w["wo"][l].T  # fp32 residual stream
        h = rmsnorm(x, w["mlp_norm"][l], shape.rms_eps)
        gu = _bf(h @ w["w_gate_up"][l].T)
        g, u = split_gate_up(gu, shape.ffn)
        a = _bf(torch.nn.functional.silu(g) * u)
        x = x + a @ w["w_down"][l].T
    rows = list(range(T)) if out_rows is None else out_rows
    hf = rmsnorm(x[rows], w["final_norm"], shape.rms_eps)
    return hf @ w["lm_head"].T


@torch.no_grad()
def forward_prefix(w: dict, shape, prefix_kv: list, tokens: list[int], start: int,
                   out_rows: list[int], dtype=torch.float32, q_chunk: int = 256) -> torch.Tensor:
    """Logits [len(out_rows), V] for `tokens` at positions start.. over an
    EXTERNAL cached prefix: prefix_kv[l] = (k, v), each [start, n_kv, d] with
    the values the paged store holds (k already rotated).  This is what the
    GPU forward computes for a delta-prefill chunk / verify over an aliased
    prefix - the prefix need not be re-run on the CPU, so
    the 8B layer shapes at 32k positions stay tractable.  `dtype` float64 gives
    the oracle's own accumulation-order noise floor.  Queries are processed in
    chunks of q_chunk (score memory)."""
    T = len(tokens)
    nh, nkv, d = shape.n_heads, shape.n_kv_heads, shape.head_dim
    G = nh // nkv
    cos, sin = rope_tables(start + T, d, shape.rope_theta)
    cos, sin = cos[start:], sin[start:]
    cast = (lambda t: t.to(dtype))  # noqa: E731
    x = cast(w["embed"][torch.tensor(tokens, dtype=torch.long)])
    scale = 1.0 / (d ** 0.5)
    kpos = torch.arange(start + T)
    for l in range(shape.layers):
        h = rmsnorm(x, cast(w["attn_norm"][l]), shape.rms_eps).to(dtype)
        qkv = unpermute_qk(_bf(h @ cast(w["wqkv"][l]).T).to(dtype), nh, nkv, d)
        q = qkv[:, : nh * d].view(T, nh, d)
        k = qkv[:, nh * d: (nh + nkv) * d].view(T, nkv, d)
        v = qkv[:, (nh + nkv) * d:].view(T, nkv, d)
        q, k = rope(q, cos, sin).to(dtype), rope(k, cos, sin).to(dtype)
        pk, pv = prefix_kv[l]
        kk = torch.cat([cast(pk), k]).repeat_interleave(G, dim=1)  # [S, nh, d]
        vv = torch.cat([cast(pv), v]).repeat_interleave(G, dim=1)
        o = torch.empty(T, nh, d, dtype=dtype)
        for a in range(0, T, q_chunk):
            b = min(T, a + q_chunk)
            s_ = torch.einsum("qhd,khd->hqk", q[a:b], kk) * scale
            qpos = torch.arange(start + a, start + b)[:, None]
            s_ = s_.masked_fill((kpos[None, :] > qpos)[None], float("-inf"))
            o[a:b] = torch.einsum("hqk,khd->qhd", torch.softmax(s_, dim=-1), vv)
        o = _bf(o.reshape(T, nh * d)).to(dtype)
        x = x + o @ cast(w["wo"][l]).T
        h = rmsnorm(x, cast(w["mlp_norm"][l]), shape.rms_eps).to(dtype)
        gu = _bf(h @ cast(w["w_gate_up"][l]).T).to(dtype)
        g, u = split_gate_up(gu, shape.ffn)
        a_ = _bf(torch.nn.functional.silu(g) * u).to(dtype)
        x = x + a_ @ cast(w["w_down"][l]).T
    hf = rmsnorm(x[out_rows], cast(w["final_norm"]), shape.rms_eps).to(dtype)
    return (hf @ cast(w["lm_head"]).T).float()


@torch.no_grad()
def paged_attention(q: torch.Tensor, k_cells: torch.Tensor, v_cells: torch.Tensor,
                    q_pos: list[int], kv_len: int, scale: float, q_chunk: int = 128) -> torch.Tensor:
    """Reference attention for one sequence: q [Tq, nh, d] (roped, bf16 values),
    k/v [kv_len, nkv, d] gathered in logical order; causal by absolute position.
    Queries in chunks of q_chunk (bounded score memory at 32k keys)."""
    Tq, nh, d = q.shape
    G = nh // k_cells.shape[1]
    kr = k_cells.float().repeat_interleave(G, dim=1)
    vr = v_cells.float().repeat_interleave(G, dim=1)
    kpos = torch.arange(kv_len)[None, :]
    out = torch.empty(Tq, nh, d)
    for a in range(0, Tq, q_chunk):
        b = min(Tq, a + q_chunk)
        s = torch.einsum("qhd,khd->hqk", q[a:b].float(), kr) * scale
        qpos = torch.tensor(q_pos[a:b])[:, None]
        s = s.masked_fill((kpos > qpos)[None], float("-inf"))
        out[a:b] = torch.einsum("hqk,khd->qhd", torch.softmax(s, dim=-1), vr)
    return out
