"""Element-wise kernels + K5 (RoPE/KV store) + K7 attention vs torch fp32."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

from oracle.llama_ref import paged_attention, qk_perm, rope_tables, split_gate_up, unpermute_qk

pytestmark = pytest.mark.gpu


def _bf(x):
    return x.to(torch.bfloat16)


def test_rmsnorm_silu_embed_argmax(cuda):
    from paper_2605_26289_b200._lib import check, lib

    L = lib()
    s = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device=cuda).manual_seed(0)
    x = torch.randn(7, 4096, device=cuda, generator=g).bfloat16()
    w = (1 + 0.1 * torch.randn(4096, device=cuda, generator=g)).bfloat16()
    out = torch.empty_like(x)
    rows = torch.tensor([6, 0, 3], dtype=torch.int32, device=cuda)
    check(L.ds_rmsnorm(x.data_ptr(), 0, rows.data_ptr(), 3, 4096, w.data_ptr(), 1e-5,
                       out.data_ptr(), s))
    out32 = torch.empty_like(x)
    x32 = x.float().contiguous()
    check(L.ds_rmsnorm(x32.data_ptr(), 1, rows.data_ptr(), 3, 4096,
                       w.data_ptr(), 1e-5, out32.data_ptr(), s))
    torch.cuda.synchronize()
    assert torch.equal(out32[:3], out[:3])
    xf = x.float()[[6, 0, 3]]
    ref = xf * torch.rsqrt((xf * xf).mean(-1, keepdim=True) + 1e-5) * w.float()
    assert torch.allclose(out[:3].float(), _bf(ref).float(), atol=2e-2, rtol=1e-2)
    gu = torch.randn(5, 2 * 2816, device=cuda, generator=g).bfloat16()
    act = torch.empty(5, 2816, device=cuda, dtype=torch.bfloat16)
    check(L.ds_silu_mul(gu.data_ptr(), 5, 2816, act.data_ptr(), s))
    gf = gu.float()
    gt, up = split_gate_up(gf, 2816)
    ref = torch.nn.functional.silu(gt) * up
    assert torch.allclose(act.float(), _bf(ref).float(), atol=1e-2, rtol=1e-2)
    table = torch.randn(100, 1024, device=cuda, generator=g).bfloat16()
    tok = torch.tensor([5, 99, 0], dtype=torch.int32, device=cuda)
    emb = torch.empty(3, 1024, device=cuda, dtype=torch.bfloat16)
    check(L.ds_embed(tok.data_ptr(), 3, table.data_ptr(), 1024, emb.data_ptr(), 0, s))
    assert torch.equal(emb, table[[5, 99, 0]])
    emb32 = torch.empty(3, 1024, device=cuda, dtype=torch.float32)
    check(L.ds_embed(tok.data_ptr(), 3, table.data_ptr(), 1024, emb32.data_ptr(), 1, s))
    assert torch.equal(emb32, table[[5, 99, 0]].float())
    logits = torch.randn(4, 128256, device=cuda, generator=g)
    logits[2, 77] = logits[2, 1000] = 1e4  # tie -> lowest index
    am = torch.empty(4, dtype=torch.int32, device=cuda)
    check(L.ds_argmax(logits.data_ptr(), 4, 128256, am.data_ptr(), s))
    ref = logits.argmax(-1)
    ref[2] = 77
    assert am.tolist() == ref.tolist()


def _setup_paged(cuda, seq_len, nkv=8, d=128, capacity=None, seed=0, contiguous=False):
    g = torch.Generator(device="cpu").manual_seed(seed)
    capacity = capacity or seq_len + 37
    if contiguous:  # first-fit style runs (TMA path) with one break in the middle
        cells = torch.cat([torch.arange(5, 5 + seq_len // 2),
                           torch.arange(seq_len // 2 + 17, seq_len + 17)]).to(torch.int32)
    else:  # fully fragmented (cell-by-cell gather path)
        cells = torch.randperm(capacity, generator=g)[:seq_len].to(torch.int32)
    k_pool = torch.randn(nkv, capacity, d, generator=g).bfloat16()  # head-major pool
    v_pool = torch.randn(nkv, capacity, d, generator=g).bfloat16()
    pos2cell = torch.zeros(2, seq_len + 64, dtype=torch.int32)
    pos2cell[1, :seq_len] = cells
    return (k_pool.to(cuda), v_pool.to(cuda), pos2cell.to(cuda), cells, k_pool, v_pool, capacity)


def _entries(entries):
    from paper_2605_26289_b200 import _lib

    arr = (_lib.Entry * len(entries))()
    for i, e in enumerate(entries):
        arr[i] = _lib.Entry(*e)
    return arr


# (4500, 5), (32768, 4), (8192, 3), (5000, 6), (20000, 5), (3000, 5), (2043, 5)
# run the tcgen05 K7 variant (R > 8 over >= 2k keys; (2040, 5) is the mma.sync
# side of the threshold); (20000, 5) also takes the > 8-split combine;
# (1100, 5), (3000, 5), (5000, 6), (8000, 5): R > 8 over <= 8k keys, capped at
# a cluster's worth of splits (attn_split_plan)
@pytest.mark.parametrize("past,q_len", [(0, 1), (5, 1), (1000, 1), (3000, 5), (31, 17), (2000, 8), (32768, 4),
                                        (4500, 5), (8192, 3), (5000, 6), (20000, 5), (777, 64), (1100, 5), (8000, 5),
                                        (0, 150), (2048, 300), (2040, 5), (2043, 5), (1023, 9)])
@pytest.mark.parametrize("contiguous", [False, True])
def test_attention_paged_vs_fp32(cuda, past, q_len, contiguous):
    _attention_case(cuda, past, q_len, contiguous, impl=1)


@pytest.mark.parametrize("past,q_len", [(300, 1), (301, 1), (302, 5), (64, 1), (127, 1)])
@pytest.mark.parametrize("contiguous", [False, True])
def test_attention_small_gqa(cuda, past, q_len, contiguous):
    """The tiny model's head shape (8 q / 2 kv heads): few CTAs, so short
    contexts still split and merge inline."""
    _attention_case(cuda, past, q_len, contiguous, impl=1, nh=8, nkv=2)


@pytest.mark.parametrize("past,q_len", [(0, 32), (0, 150), (100, 33), (2048, 300), (3000, 881),
                                        (127, 129), (5, 1)])
@pytest.mark.parametrize("contiguous", [False, True])
def test_attention_tcgen05_prefill_vs_fp32(cuda, past, q_len, contiguous):
    _attention_case(cuda, past, q_len, contiguous, impl=2)


# per-kernel attention tolerance (bf16 Q/K/V in, fp32 softmax and accumulate,
# P rounded to bf16 for the PV product, bf16 O out): measured max-abs at
# N(0,1) inputs is recorded per case (gpurun_out/numerics.jsonl ->
# profiles/round2/numerics.md); the bound is 1e-2
ATTN_TOL = 1e-2


# the BASELINE reference points on the 8B head shape: K6 at the C4 last turn
# (31,489 cached + 881 new) and K7 verify q = 5 over 32k keys
@pytest.mark.parametrize("past,q_len,impl", [(31489, 881, 2), (32768, 5, 1), (32768, 1, 1)])
def test_attention_bench_points(cuda, past, q_len, impl):
    _attention_case(cuda, past, q_len, True, impl)


def _attention_case(cuda, past, q_len, contiguous, impl, nh=32, nkv=8):
    from paper_2605_26289_b200._lib import check, lib

    d = 128
    kv_len = past + q_len
    k_pool, v_pool, pos2cell, cells, k_cpu, v_cpu, cap = _setup_paged(cuda, kv_len, nkv=nkv,
                                                                     seed=past + q_len,
                                                                     contiguous=contiguous)
    g = torch.Generator(device="cpu").manual_seed(1)
    qkv = torch.randn(q_len, (nh + 2 * nkv) * d, generator=g).bfloat16()
    ent = _entries([(1, past, q_len, 0, 0, 0, 0, 1, 0)])
    ent_dev = torch.frombuffer(bytearray(bytes(ent)), dtype=torch.uint8).to(cuda)
    out = torch.zeros(q_len, nh * d, dtype=torch.bfloat16, device=cuda)
    ws_bytes = lib().ds_attention_workspace_bytes(q_len, 1, nh, d)
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device=cuda)
    qkv_d = qkv.to(cuda)
    q = qkv[:, : nh * d].view(q_len, nh, d)
    ref = paged_attention(q, k_cpu[:, cells.long()].transpose(0, 1), v_cpu[:, cells.long()].transpose(0, 1),
                          list(range(past, kv_len)), kv_len, 1.0 / d ** 0.5)
    for _ in range(3):  # repeated launches: split-merge arrival counters must re-arm
        out.zero_()
        check(lib().ds_attention(qkv_d.data_ptr(), ctypes.addressof(ent), ent_dev.data_ptr(), 1,
                                 q_len, k_pool.data_ptr(), v_pool.data_ptr(), cap,
                                 pos2cell.data_ptr(), pos2cell.shape[1], nh, nkv, d, 1.0 / d ** 0.5,
                                 out.data_ptr(), ws.data_ptr(), ws_bytes, impl,
                                 torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        got = out.cpu().float().view(q_len, nh, d)
        err = (got - ref).abs().max().item()
        assert err < ATTN_TOL, err
    from conftest import record_numeric

    record_numeric(f"attention impl={impl} past={past} q={q_len} heads={nh}/{nkv} "
                   f"contiguous={contiguous}", max_abs=err, ref_max=ref.abs().max().item())


def test_rope_kv_store(cuda):
    from paper_2605_26289_b200._lib import check, lib

    nh, nkv, d, T = 8, 2, 128, 6
    cos, sin = rope_tables(64, d, 500000.0)
    g = torch.Generator(device="cpu").manual_seed(2)
    qkv = torch.randn(T, (nh + 2 * nkv) * d, generator=g).bfloat16()
    # the kernel takes q/k heads in the wqkv (RoPE-pair interleaved) column order
    perm = qk_perm(d)
    qkv_in = qkv.clone()
    qk = qkv_in[:, : (nh + nkv) * d].view(T, nh + nkv, d)
    qk[:] = qkv[:, : (nh + nkv) * d].view(T, nh + nkv, d)[:, :, perm]
    row_seq = torch.full((T,), 1, dtype=torch.int32)
    row_pos = torch.arange(10, 10 + T, dtype=torch.int32)
    pos2cell = torch.zeros(2, 64, dtype=torch.int32)
    pos2cell[1, 10:16] = torch.tensor([40, 3, 17, 8, 9, 60], dtype=torch.int32)
    kp = torch.zeros(nkv, 64, d, dtype=torch.bfloat16, device=cuda)
    vp = torch.zeros_like(kp)
    qd = qkv_in.to(cuda)
    keep = [t.to(cuda) for t in (row_seq, row_pos, pos2cell, cos, sin)]  # keep alive
    rs, rp, p2c, cd, sd = keep
    check(lib().ds_rope_kv_store(qd.data_ptr(), T, rs.data_ptr(), rp.data_ptr(), p2c.data_ptr(),
                                 64, nh, nkv, d, cd.data_ptr(), sd.data_ptr(), kp.data_ptr(),
                                 vp.data_ptr(), 64, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    from oracle.llama_ref import rope

    x = qkv.float()
    q = rope(x[:, : nh * d].view(T, nh, d), cos[10:16], sin[10:16])
    k = rope(x[:, nh * d:(nh + nkv) * d].view(T, nkv, d), cos[10:16], sin[10:16])
    v = x[:, (nh + nkv) * d:].view(T, nkv, d)
    # fp32 FMA contraction may flip a bf16 rounding: allow one bf16 ulp
    assert torch.allclose(qd.cpu().float()[:, : nh * d].view(T, nh, d), q, atol=1e-2, rtol=8e-3)
    cells = [40, 3, 17, 8, 9, 60]
    assert torch.allclose(kp.cpu().float()[:, cells].transpose(0, 1), k, atol=1e-2, rtol=8e-3)
    assert torch.equal(vp.cpu().float()[:, cells].transpose(0, 1), v)


# (6|8, 6144, 4096): two CTAs per SM with the ring wrapping - the shape that
# exposed a missing generic->async proxy fence before a stage is refilled
@pytest.mark.parametrize("M,N,K", [(1, 4096, 4096), (5, 6144, 4096), (17, 4096, 14336),
                                   (32, 1024, 2816 * 0 + 2048), (3, 128256 // 16 * 16, 1024),
                                   (6, 6144, 4096), (8, 6144, 4096), (7, 4096, 2816)])
@pytest.mark.parametrize("y_f32,acc", [(0, 0), (1, 1)])
def test_gemm_skinny_vs_fp32(cuda, M, N, K, y_f32, acc):
    from paper_2605_26289_b200._lib import check, lib

    g = torch.Generator(device=cuda).manual_seed(M + N + K)
    X = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    W = (0.02 * torch.randn(N, K, device=cuda, generator=g)).bfloat16()
    Y0 = torch.randn(M, N, device=cuda, generator=g)
    Y = Y0.clone() if y_f32 else Y0.bfloat16()
    check(lib().ds_gemm_skinny(X.data_ptr(), W.data_ptr(), Y.data_ptr(), M, N, K, y_f32, acc,
                               torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    ref = X.float() @ W.float().T
    if acc:
        ref = ref + (Y0 if y_f32 else Y0.bfloat16().float())
    err = (Y.float() - ref).abs().max().item()
    assert err < (1e-3 if y_f32 else 1e-2 * ref.abs().max().item()), err


def _gemm_ex(L, X, W, Y, M, N, K, y_f32, acc, epi, s, impl="auto"):
    """The forward's GEMM for M rows: skinny (M <= 32) or stream-K K10; with
    impl="pair" the CTA-pair K11 (M > 32)."""
    if impl == "pair":
        return L.ds_gemm_pair(X, W, Y, M, N, K, y_f32, acc, epi, s)
    f = L.ds_gemm_skinny_ex if M <= 32 else L.ds_gemm_stream
    return f(X, W, Y, M, N, K, y_f32, acc, epi, s)


def _skip_pair(impl, M, N):
    if impl == "pair" and (M <= 32 or N % 256):
        pytest.skip("K11 serves M > 32 rows, N % 256 == 0")


# K10 (persistent stream-K tcgen05, the product GEMM for M > 32): every shape
# the forward uses (8B qkv / wo / gate_up / down / LM head at prefill and
# batched row counts, the tiny model), ragged token tiles, plain bf16 and the
# fp32 residual accumulate; bit-identical on a repeat (fixed-order split-K).
@pytest.mark.parametrize("T,N,K", [(150, 4096, 4096), (150, 6144, 4096), (150, 28672, 4096),
                                   (150, 4096, 14336), (33, 1024, 1024), (415, 4096, 4096),
                                   (881, 1536, 1024), (881, 6144, 4096), (200, 5632, 1024),
                                   (100, 1024, 2816), (4096, 1024, 4096), (256, 4096, 4096),
                                   (257, 4096, 4096), (64, 128256, 4096), (512, 4096, 14336),
                                   (1300, 28672, 4096), (40, 128, 64)])
@pytest.mark.parametrize("y_f32,acc", [(0, 0), (1, 1)])
def test_gemm_stream_vs_fp32(cuda, T, N, K, y_f32, acc):
    from paper_2605_26289_b200._lib import check, lib

    g = torch.Generator(device=cuda).manual_seed(T + N + K)
    X = torch.randn(T, K, device=cuda, generator=g).bfloat16()
    W = (0.02 * torch.randn(N, K, device=cuda, generator=g)).bfloat16()
    Y0 = torch.randn(T, N, device=cuda, generator=g)
    Y = Y0.clone() if y_f32 else Y0.bfloat16()
    s = torch.cuda.current_stream().cuda_stream
    L = lib()
    check(L.ds_gemm_stream(X.data_ptr(), W.data_ptr(), Y.data_ptr(), T, N, K, y_f32, acc, None, s))
    torch.cuda.synchronize()
    ref = X.float() @ W.float().T
    if acc:
        ref = ref + (Y0 if y_f32 else Y0.bfloat16().float())
    err = (Y.float() - ref).abs().max().item()
    assert err < (2e-3 if y_f32 else 1e-2 * ref.abs().max().item()), err
    if y_f32:  # deterministic: partial tiles are added in fixed k order
        Y2 = Y0.clone()
        check(L.ds_gemm_stream(X.data_ptr(), W.data_ptr(), Y2.data_ptr(), T, N, K, 1, acc, None,
                               s))
        torch.cuda.synchronize()
        assert torch.equal(Y, Y2)


# K11 (CTA-pair tcgen05, persistent, split tail): the same shapes (N % 256),
# plus multi-wave row counts; deterministic (fixed-order tail partials).
@pytest.mark.parametrize("T,N,K", [(150, 4096, 4096), (150, 6144, 4096), (150, 28672, 4096),
                                   (150, 4096, 14336), (33, 1024, 1024), (415, 4096, 4096),
                                   (881, 1536, 1024), (881, 6144, 4096), (200, 5632, 1024),
                                   (100, 1024, 2816), (4096, 1024, 4096), (256, 4096, 4096),
                                   (257, 4096, 4096), (64, 128256, 4096), (512, 4096, 14336),
                                   (1300, 28672, 4096), (2048, 6144, 4096), (4096, 4096, 4096),
                                   # ragged token tiles + tails split 2-4 ways, a
                                   # single-tile GEMM, a 64-column K
                                   (300, 1536, 1024), (1025, 512, 2048), (64, 256, 64),
                                   (3000, 5632, 1024)])
@pytest.mark.parametrize("y_f32,acc", [(0, 0), (1, 1)])
def test_gemm_pair_vs_fp32(cuda, T, N, K, y_f32, acc):
    from paper_2605_26289_b200._lib import check, lib

    g = torch.Generator(device=cuda).manual_seed(T + N + K)
    X = torch.randn(T, K, device=cuda, generator=g).bfloat16()
    W = (0.02 * torch.randn(N, K, device=cuda, generator=g)).bfloat16()
    Y0 = torch.randn(T, N, device=cuda, generator=g)
    Y = Y0.clone() if y_f32 else Y0.bfloat16()
    s = torch.cuda.current_stream().cuda_stream
    L = lib()
    check(L.ds_gemm_pair(X.data_ptr(), W.data_ptr(), Y.data_ptr(), T, N, K, y_f32, acc, None, s))
    torch.cuda.synchronize()
    ref = X.float() @ W.float().T
    if acc:
        ref = ref + (Y0 if y_f32 else Y0.bfloat16().float())
    err = (Y.float() - ref).abs().max().item()
    assert err < (2e-3 if y_f32 else 1e-2 * ref.abs().max().item()), err
    if y_f32:
        Y2 = Y0.clone()
        check(L.ds_gemm_pair(X.data_ptr(), W.data_ptr(), Y2.data_ptr(), T, N, K, 1, acc, None, s))
        torch.cuda.synchronize()
        assert torch.equal(Y, Y2)


@pytest.mark.parametrize("M", [1, 5, 13, 20, 32, 33, 150, 300, 881])
@pytest.mark.parametrize("impl", ["auto", "pair"])
def test_gemm_skinny_epilogue_fusions(cuda, M, impl):
    """ds_gemm_skinny_ex: residual producer (y += X.W^T, h = bf16(y*w_norm),
    per-CTA partial sums of y^2) feeding a norm consumer (row scale
    rsqrt(mean(y^2)+eps)) and a SwiGLU consumer (8-row interleaved gate|up) -
    against the unfused RMSNorm -> GEMM -> SiLU*up chain in fp32 with the
    unfused path's bf16 storage points."""
    from paper_2605_26289_b200._lib import SkinnyEpi, check, lib

    _skip_pair(impl, M, 512)
    L = lib()
    s = torch.cuda.current_stream().cuda_stream
    H, F, Kin = 2048, 1024, 1024
    g = torch.Generator(device=cuda).manual_seed(M)
    Xin = torch.randn(M, Kin, device=cuda, generator=g).bfloat16()
    Wo = (0.05 * torch.randn(H, Kin, device=cuda, generator=g)).bfloat16()
    x0 = torch.randn(M, H, device=cuda, generator=g)
    nw = (1 + 0.1 * torch.randn(H, device=cuda, generator=g)).bfloat16()
    Wgu = (0.02 * torch.randn(2 * F, H, device=cuda, generator=g)).bfloat16()
    x = x0.clone()
    h = torch.empty(M, H, device=cuda, dtype=torch.bfloat16)
    R = max(32, M)
    ss = torch.zeros(R, device=cuda, dtype=torch.int64)
    other = torch.full((R,), 7, device=cuda, dtype=torch.int64)
    prod = SkinnyEpi(ss_out=ss.data_ptr(), ss_zero=other.data_ptr(), h_out=h.data_ptr(),
                     h_w=nw.data_ptr())
    check(_gemm_ex(L, Xin.data_ptr(), Wo.data_ptr(), x.data_ptr(), M, H, Kin, 1, 1,
                   ctypes.byref(prod), s, impl))
    act = torch.empty(M, F, device=cuda, dtype=torch.bfloat16)
    cons = SkinnyEpi(row_ss=ss.data_ptr(), eps=1e-5, swiglu=1)
    check(_gemm_ex(L, h.data_ptr(), Wgu.data_ptr(), act.data_ptr(), M, 2 * F, H, 0, 0,
                   ctypes.byref(cons), s, impl))
    q = torch.empty(M, 512, device=cuda, dtype=torch.bfloat16)
    cons2 = SkinnyEpi(row_ss=ss.data_ptr(), eps=1e-5)
    check(_gemm_ex(L, h.data_ptr(), Wgu[:512].contiguous().data_ptr(), q.data_ptr(), M,
                   512, H, 0, 0, ctypes.byref(cons2), s, impl))
    torch.cuda.synchronize()
    x_ref = x0 + Xin.float() @ Wo.float().T
    assert (x - x_ref).abs().max().item() < 1e-3
    assert torch.allclose(h.float(), _bf(x * nw.float()).float(), atol=0, rtol=0)
    assert torch.allclose(ss[:M].double() / 2**24, (x * x).sum(-1).double(), rtol=1e-5)
    assert other[:M].eq(0).all()
    hn = _bf(x_ref * torch.rsqrt((x_ref * x_ref).mean(-1, keepdim=True) + 1e-5) * nw.float())
    gu = _bf(hn.float() @ Wgu.float().T).float()
    gt, up = split_gate_up(gu, F)
    a_ref = torch.nn.functional.silu(gt) * up
    err = (act.float() - a_ref).abs().max().item()
    assert err < 2e-2 * a_ref.abs().max().item(), err
    q_ref = hn.float() @ Wgu[:512].float().T
    err = (q.float() - q_ref).abs().max().item()
    assert err < 2e-2 * q_ref.abs().max().item(), err


@pytest.mark.parametrize("M", [1, 5, 6, 17, 32, 33, 100, 300])
@pytest.mark.parametrize("impl", ["auto", "pair"])
def test_gemm_skinny_argmax_epilogue(cuda, M, impl):
    """Fused LM-head argmax (ds_skinny_epi.argmax_out): the
    packed per-row key decodes to np.argmax of the same kernel's fp32 product
    (largest value, lowest column on exact ties - duplicated weight rows make
    bit-identical columns), with and without the product stored."""
    from paper_2605_26289_b200._lib import SkinnyEpi, check, lib

    _skip_pair(impl, M, 128256)
    L = lib()
    s = torch.cuda.current_stream().cuda_stream
    V, H = 128256, 4096
    g = torch.Generator(device=cuda).manual_seed(100 + M)
    X = torch.randn(M, H, device=cuda, generator=g).bfloat16()
    W = (0.02 * torch.randn(V, H, device=cuda, generator=g)).bfloat16()
    W[77000] = W[90000] = W[5] = (0.5 * X[0].float() / X[0].float().norm()).bfloat16()
    Y = torch.empty(M, V, device=cuda)
    R = max(32, M)
    keys = torch.zeros(R, device=cuda, dtype=torch.int64)
    epi = SkinnyEpi(argmax_out=keys.data_ptr())
    check(_gemm_ex(L, X.data_ptr(), W.data_ptr(), Y.data_ptr(), M, V, H, 1, 0,
                   ctypes.byref(epi), s, impl))
    keys2 = torch.zeros(R, device=cuda, dtype=torch.int64)
    epi2 = SkinnyEpi(argmax_out=keys2.data_ptr())
    check(_gemm_ex(L, X.data_ptr(), W.data_ptr(), None, M, V, H, 1, 0,
                   ctypes.byref(epi2), s, impl))
    torch.cuda.synchronize()
    idx = (0xFFFFFFFF - (keys[:M] & 0xFFFFFFFF)).cpu()
    assert torch.equal(idx, Y.argmax(-1).cpu())  # torch: first maximal index
    assert torch.equal(keys, keys2)
    assert int(idx[0]) == 5  # three identical top columns: the lowest wins
    assert keys[M:].eq(0).all()
    ref = X.float() @ W.float().T
    assert (Y - ref).abs().max().item() < 1e-2


@pytest.mark.parametrize("M", [1, 5, 17, 32, 48, 150, 300])
@pytest.mark.parametrize("norm", [False, True])
@pytest.mark.parametrize("impl", ["auto", "pair"])
def test_gemm_skinny_rope_kv_epilogue(cuda, M, norm, impl):
    """ds_gemm_skinny_ex rope mode (wqkv projection + RoPE + KV store, the
    decode forward's K5 fusion) vs torch: qkv = bf16(X.W^T) in the wqkv
    RoPE-pair interleaved layout, un-permuted, rotated, q to Y, k/v into the
    head-major pools at pos2cell cells."""
    from paper_2605_26289_b200._lib import SkinnyEpi, check, lib

    nh, nkv, d, H = 8, 2, 128, 1024
    QKV = (nh + 2 * nkv) * d
    _skip_pair(impl, M, QKV)
    g = torch.Generator(device="cpu").manual_seed(M + 100 * norm)
    X = torch.randn(M, H, generator=g).bfloat16()
    W = (0.05 * torch.randn(QKV, H, generator=g)).bfloat16()
    cos, sin = rope_tables(4096, d, 500000.0)
    row_seq = torch.randint(0, 3, (M,), generator=g, dtype=torch.int32)
    row_pos = torch.randperm(4096, generator=g)[:M].to(torch.int32)  # distinct (seq, pos)
    cells = torch.randperm(1024, generator=g)[:M].to(torch.int32)
    pos2cell = torch.zeros(3, 4096, dtype=torch.int32)
    pos2cell[row_seq.long(), row_pos.long()] = cells
    head_stride = 1024
    kp = torch.zeros(nkv, head_stride, d, dtype=torch.bfloat16, device=cuda)
    vp = torch.zeros_like(kp)
    Y = torch.zeros(M, QKV, dtype=torch.bfloat16, device=cuda)
    dev = [t.to(cuda) for t in (X, W, cos, sin, row_seq, row_pos, pos2cell)]
    Xd, Wd, cd, sd, rsd, rpd, p2cd = dev
    R = max(32, M)
    ss = torch.zeros(R, dtype=torch.int64, device=cuda)
    scale = torch.ones(M)
    if norm:  # consumer row scale: X holds bf16(x * w); row sums of x^2 given
        x = torch.randn(M, H, generator=g) * 2
        fixed = ((x * x).double().sum(-1) * 2**24).round().long()
        ss.copy_(torch.nn.functional.pad(fixed, (0, R - M)).to(cuda))
        scale = torch.rsqrt((x * x).sum(-1) / H + 1e-5)
    epi = SkinnyEpi(row_ss=ss.data_ptr() if norm else None, eps=1e-5, rope=1, n_heads=nh,
                    n_kv_heads=nkv, row_seq=rsd.data_ptr(), row_pos=rpd.data_ptr(),
                    pos2cell=p2cd.data_ptr(), pos_stride=4096, rope_cos=cd.data_ptr(),
                    rope_sin=sd.data_ptr(), k_pool_l=kp.data_ptr(), v_pool_l=vp.data_ptr(),
                    kv_head_stride=head_stride)
    check(_gemm_ex(lib(), Xd.data_ptr(), Wd.data_ptr(), Y.data_ptr(), M, QKV, H, 0, 0,
                   ctypes.byref(epi), torch.cuda.current_stream().cuda_stream, impl))
    torch.cuda.synchronize()
    qkv = unpermute_qk(_bf((X.float() @ W.float().T) * scale[:, None]), nh, nkv, d).float()
    from oracle.llama_ref import rope

    c, s_ = cos[row_pos.long()], sin[row_pos.long()]
    q = rope(qkv[:, : nh * d].view(M, nh, d), c, s_)
    k = rope(qkv[:, nh * d:(nh + nkv) * d].view(M, nkv, d), c, s_)
    v = qkv[:, (nh + nkv) * d:].view(M, nkv, d)
    # fp32 accumulation order + FMA contraction: a bf16 ulp or two
    tol = dict(atol=2e-2, rtol=2e-2)
    assert torch.allclose(Y.cpu().float()[:, : nh * d].view(M, nh, d), q, **tol)
    cl = cells.long()
    assert torch.allclose(kp.cpu().float()[:, cl].transpose(0, 1), k, **tol)
    assert torch.allclose(vp.cpu().float()[:, cl].transpose(0, 1), v, **tol)
