"""Run one projection shape through ds_gemm_stream (k10), ds_gemm_pair (k11) or cuBLAS a
few times - for ncu.  Usage: one_gemm.py T N K [reps] [k10|k11|cublas]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26289_b200._lib import check, lib

T, N, K = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
impl = sys.argv[5] if len(sys.argv) > 5 else "k10"
dev = torch.device("cuda", 0)
X = torch.randn(T, K, device=dev).bfloat16()
W = (0.02 * torch.randn(N, K, device=dev)).bfloat16()
Y = torch.zeros(T, N, device=dev).bfloat16()
s = torch.cuda.current_stream()
for _ in range(reps):
    if impl == "k10":
        check(lib().ds_gemm_stream(X.data_ptr(), W.data_ptr(), Y.data_ptr(), T, N, K, 0, 0, None,
                                   s.cuda_stream))
    elif impl == "k11":
        check(lib().ds_gemm_pair(X.data_ptr(), W.data_ptr(), Y.data_ptr(), T, N, K, 0, 0, None,
                                 s.cuda_stream))
    else:
        torch.matmul(X, W.T, out=Y)
torch.cuda.synchronize()
