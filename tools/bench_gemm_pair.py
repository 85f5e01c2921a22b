"""Microbench + check: ds_gemm_pair (K11, CTA-pair tcgen05) vs cuBLAS (torch)
on the 8B projections at prefill / batched row counts.  4 rotating weight
copies (> L2), CUDA events on the launching stream, 20 launches after 3
warm-up.  Usage: bench_gemm_pair.py [T ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26289_b200._lib import check, lib

dev = torch.device("cuda", 0)
L = lib()
s = torch.cuda.current_stream()
peak_tf = 1676e12
tot = {"k11": 0.0, "cublas": 0.0}
for T in [int(x) for x in (sys.argv[1:] or ["256", "512", "881", "2048"])]:
    for name, N, K in (("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096),
                       ("down", 4096, 14336)):
        X = torch.randn(T, K, device=dev).bfloat16()
        Ws = [(0.02 * torch.randn(N, K, device=dev)).bfloat16() for _ in range(4)]
        Y = torch.zeros(T, N, device=dev).bfloat16()
        check(L.ds_gemm_pair(X.data_ptr(), Ws[0].data_ptr(), Y.data_ptr(), T, N, K, 0, 0, None,
                             s.cuda_stream))
        torch.cuda.synchronize()
        ref = X.float() @ Ws[0].float().T
        err = (Y.float() - ref).abs().max().item() / ref.abs().max().item()

        def ours(i):
            check(L.ds_gemm_pair(X.data_ptr(), Ws[i % 4].data_ptr(), Y.data_ptr(), T, N, K, 0, 0,
                                 None, s.cuda_stream))

        def cub(i):
            torch.matmul(X, Ws[i % 4].T, out=Y)

        res = {}
        for tag, fn in (("k11", ours), ("cublas", cub)):
            for i in range(3):
                fn(i)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for i in range(20):
                fn(i)
            b.record()
            b.synchronize()
            res[tag] = a.elapsed_time(b) / 20 / 1e3
            tot[tag] += res[tag]
        fl = 2.0 * T * N * K
        print(f"T={T:4d} {name:8s} k11 {res['k11']*1e6:7.1f} us ({fl/res['k11']/1e12:5.0f} TF/s, "
              f"{fl/res['k11']/peak_tf*100:4.0f}%) | cublas {res['cublas']*1e6:7.1f} us "
              f"({fl/res['cublas']/peak_tf*100:4.0f}%)  rel.err {err:.2e}", flush=True)
print(f"sum k11 {tot['k11']*1e6:.1f} us  cublas {tot['cublas']*1e6:.1f} us")
