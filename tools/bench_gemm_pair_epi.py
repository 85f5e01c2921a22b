"""K11 with vs without its fused epilogues (T rows, 8B shapes): plain bf16,
residual producer (fp32 x += , h = bf16(x * w), row sums), SwiGLU, RoPE + KV
store.  Usage: bench_gemm_pair_epi.py [T]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26289_b200._lib import SkinnyEpi, check, lib

dev = torch.device("cuda", 0)
L = lib()
s = torch.cuda.current_stream()
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
H, F, QKV = 4096, 14336, 6144


def timeit(fn, n=10):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        fn(i)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n * 1e3


for name, N, K in (("qkv", QKV, H), ("o", H, H), ("gate_up", 2 * F, H), ("down", H, F)):
    X = torch.randn(T, K, device=dev).bfloat16()
    Ws = [(0.02 * torch.randn(N, K, device=dev)).bfloat16() for _ in range(3)]
    Yb = torch.zeros(T, N, device=dev).bfloat16()
    res = {}
    res["plain"] = timeit(lambda i: check(L.ds_gemm_pair(X.data_ptr(), Ws[i % 3].data_ptr(), Yb.data_ptr(), T, N, K, 0, 0, None, s.cuda_stream)))
    ss = torch.zeros(T, dtype=torch.int64, device=dev)
    rs = torch.full((T,), 1 << 30, dtype=torch.int64, device=dev)
    if name in ("o", "down"):
        x = torch.zeros(T, N, device=dev)
        h = torch.empty(T, N, device=dev, dtype=torch.bfloat16)
        nw = torch.ones(N, device=dev, dtype=torch.bfloat16)
        e = SkinnyEpi(ss_out=ss.data_ptr(), h_out=h.data_ptr(), h_w=nw.data_ptr())
        res["fused"] = timeit(lambda i: check(L.ds_gemm_pair(X.data_ptr(), Ws[i % 3].data_ptr(), x.data_ptr(), T, N, K, 1, 1, ctypes.byref(e), s.cuda_stream)))
    elif name == "gate_up":
        act = torch.empty(T, N // 2, device=dev, dtype=torch.bfloat16)
        e = SkinnyEpi(row_ss=rs.data_ptr(), eps=1e-5, swiglu=1)
        res["fused"] = timeit(lambda i: check(L.ds_gemm_pair(X.data_ptr(), Ws[i % 3].data_ptr(), act.data_ptr(), T, N, K, 0, 0, ctypes.byref(e), s.cuda_stream)))
    else:
        cap = T + 64
        kp = torch.zeros(8, cap, 128, device=dev, dtype=torch.bfloat16)
        vp = torch.zeros_like(kp)
        cos = torch.rand(cap, 64, device=dev)
        sin = torch.rand(cap, 64, device=dev)
        rseq = torch.zeros(T, dtype=torch.int32, device=dev)
        rpos = torch.arange(T, dtype=torch.int32, device=dev)
        p2c = torch.randperm(cap, device=dev).to(torch.int32).view(1, cap)
        e = SkinnyEpi(row_ss=rs.data_ptr(), eps=1e-5, rope=1, n_heads=32, n_kv_heads=8,
                      row_seq=rseq.data_ptr(), row_pos=rpos.data_ptr(), pos2cell=p2c.data_ptr(),
                      pos_stride=cap, rope_cos=cos.data_ptr(), rope_sin=sin.data_ptr(),
                      k_pool_l=kp.data_ptr(), v_pool_l=vp.data_ptr(), kv_head_stride=cap)
        res["fused"] = timeit(lambda i: check(L.ds_gemm_pair(X.data_ptr(), Ws[i % 3].data_ptr(), Yb.data_ptr(), T, N, K, 0, 0, ctypes.byref(e), s.cuda_stream)))
    res["cublas"] = timeit(lambda i: torch.matmul(X, Ws[i % 3].T, out=Yb))
    print(f"T={T} {name:8s} " + "  ".join(f"{k} {v:7.1f} us" for k, v in res.items()), flush=True)
