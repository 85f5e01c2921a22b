"""Microbench: ds_gemm_tc (K9, tcgen05) vs cuBLAS (torch) on the 8B projections
for prefill chunks / batched plans.  4 rotating weight copies (> L2)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26289_b200._lib import check, lib

dev = torch.device("cuda", 0)
L = lib()
s = torch.cuda.current_stream()
peak_bw, peak_tf = 6535e9, 1676e12
for T in [int(x) for x in (sys.argv[1:] or ["150", "415", "881"])]:
    for name, N, K in (("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096),
                       ("down", 4096, 14336)):
        X = torch.randn(T, K, device=dev).bfloat16()
        Ws = [(0.02 * torch.randn(N, K, device=dev)).bfloat16() for _ in range(4)]
        Y = torch.zeros(T, N, device=dev).bfloat16()
        def ours(i):
            check(L.ds_gemm_tc(X.data_ptr(), Ws[i % 4].data_ptr(), Y.data_ptr(), T, N, K, 0, 0,
                               s.cuda_stream))
        def cub(i):
            torch.matmul(X, Ws[i % 4].T, out=Y)
        res = {}
        for tag, fn in (("tc", ours), ("cublas", cub)):
            for i in range(3): fn(i)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for i in range(20): fn(i)
            b.record(); b.synchronize()
            t = a.elapsed_time(b) / 20 / 1e3
            res[tag] = t
        byt = N * K * 2 + T * K * 2 + T * N * 2
        fl = 2.0 * T * N * K
        print(f"T={T:4d} {name:8s} tc {res['tc']*1e6:7.1f} us ({byt/res['tc']/1e9:5.0f} GB/s, "
              f"{fl/res['tc']/1e12:5.0f} TF/s, {max(byt/res['tc']/peak_bw, fl/res['tc']/peak_tf)*100:4.0f}% roof) | "
              f"cublas {res['cublas']*1e6:7.1f} us ({max(byt/res['cublas']/peak_bw, fl/res['cublas']/peak_tf)*100:4.0f}% roof)")
