"""Microbench: ds_gemm_stream (K10, stream-K tcgen05) vs cuBLAS (torch) on the
8B projections at prefill / batched row counts.  4 rotating weight copies
(> L2), CUDA events on the launching stream, 20 launches after 3 warm-up.
Usage: bench_gemm_stream.py [T ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26289_b200._lib import check, lib

dev = torch.device("cuda", 0)
L = lib()
s = torch.cuda.current_stream()
peak_bw, peak_tf = 6535e9, 1676e12
tot = {"k10": 0.0, "cublas": 0.0}
for T in [int(x) for x in (sys.argv[1:] or ["150", "512", "881"])]:
    for name, N, K in (("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096),
                       ("down", 4096, 14336)):
        X = torch.randn(T, K, device=dev).bfloat16()
        Ws = [(0.02 * torch.randn(N, K, device=dev)).bfloat16() for _ in range(4)]
        Y = torch.zeros(T, N, device=dev).bfloat16()

        def ours(i):
            check(L.ds_gemm_stream(X.data_ptr(), Ws[i % 4].data_ptr(), Y.data_ptr(), T, N, K, 0,
                                   0, None, s.cuda_stream))

        def cub(i):
            torch.matmul(X, Ws[i % 4].T, out=Y)

        res = {}
        for tag, fn in (("k10", ours), ("cublas", cub)):
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
        byt = N * K * 2 + T * K * 2 + T * N * 2
        fl = 2.0 * T * N * K
        roof = lambda t: max(byt / t / peak_bw, fl / t / peak_tf) * 100  # noqa: E731
        print(f"T={T:4d} {name:8s} k10 {res['k10']*1e6:7.1f} us ({byt/res['k10']/1e9:5.0f} GB/s, "
              f"{fl/res['k10']/1e12:5.0f} TF/s, {roof(res['k10']):4.0f}% roof) | "
              f"cublas {res['cublas']*1e6:7.1f} us ({roof(res['cublas']):4.0f}% roof)", flush=True)
print(f"sum k10 {tot['k10']*1e6:.1f} us  cublas {tot['cublas']*1e6:.1f} us")
