"""Microbench: ds_gemm_skinny vs cuBLAS (torch) for the 8B decode projections."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ctypes
from paper_2605_26289_b200._lib import SkinnyEpi, check, lib

dev = torch.device("cuda", 0)
L = lib()
s = torch.cuda.current_stream()
for M in (1, 5, 17):
    for name, N, K in (("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096),
                       ("down", 4096, 14336), ("lm_head", 128256, 4096)):
        X = torch.randn(M, K, device=dev).bfloat16()
        Ws = [(0.02 * torch.randn(N, K, device=dev)).bfloat16() for _ in range(4)]  # > L2 rotation
        Y = torch.zeros(M, N, device=dev)
        def ours(i):
            check(L.ds_gemm_skinny(X.data_ptr(), Ws[i % 4].data_ptr(), Y.data_ptr(), M, N, K, 1, 0, s.cuda_stream))
        ss = torch.zeros(32, device=dev, dtype=torch.int64)
        hw = torch.ones(N, device=dev).bfloat16()
        hout = torch.empty(M, N, device=dev).bfloat16()
        if name == "gate_up":
            epi = SkinnyEpi(row_ss=ss.data_ptr(), eps=1e-5, swiglu=1)
            Yf, f32, acc = torch.empty(M, N // 2, device=dev).bfloat16(), 0, 0
        elif name in ("o", "down"):
            epi = SkinnyEpi(ss_out=ss.data_ptr(), h_out=hout.data_ptr(), h_w=hw.data_ptr())
            Yf, f32, acc = Y, 1, 1
        else:
            epi = SkinnyEpi(row_ss=ss.data_ptr(), eps=1e-5)
            Yf, f32, acc = Y, 1, 0
        def fused(i):
            check(L.ds_gemm_skinny_ex(X.data_ptr(), Ws[i % 4].data_ptr(), Yf.data_ptr(), M, N, K,
                                      f32, acc, ctypes.byref(epi), s.cuda_stream))
        def cub(i):
            torch.matmul(X, Ws[i % 4].T, out=None)
        res = {}
        for tag, fn in (("ours", ours), ("fused", fused), ("cublas", cub)):
            for i in range(3): fn(i)
            ts = []
            for i in range(20):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); fn(i); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
            t = statistics.median(ts) / 1e3
            res[tag] = (t * 1e6, N * K * 2 / t / 1e9)
        ref = (X.float() @ Ws[19 % 4].float().T)
        ours(19); torch.cuda.synchronize()
        err = (Y - ref).abs().max().item()
        print(f"M={M:2d} {name:8s} ours {res['ours'][0]:8.1f} us {res['ours'][1]:7.0f} GB/s | fused    {res['fused'][0]:8.1f} us | cublas {res['cublas'][0]:8.1f} us {res['cublas'][1]:7.0f} GB/s | err {err:.2e}")
