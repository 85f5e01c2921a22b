"""cuBLASLt heuristic candidates vs the cublasGemmEx default on the 8B
projections at prefill / batched row counts (ds_debug_lt_sweep; 4 rotating
weight copies > L2).  Usage: bench_lt.py [T ...]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import subprocess
import torch

# measurement-only: tools/gemm_lt.cu is built into its own library here (it is
# not part of the product libdeltaserve_b200.so)
HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libgemm_lt.so")
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                       "-O2", "-shared", "-Xcompiler", "-fPIC",
                       "-I" + os.path.join(os.path.dirname(HERE), "include"),
                       os.path.join(HERE, "gemm_lt.cu"), "-o", SO, "-lcublasLt", "-lcublas"])
L = ctypes.CDLL(SO)
f = L.ds_debug_lt_sweep
P = ctypes.c_void_p
f.argtypes = [P, P, ctypes.c_int, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
              ctypes.c_int, P]
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
for T in [int(x) for x in (sys.argv[1:] or ["150"])]:
    for name, N, K, f32 in (("qkv", 6144, 4096, 0), ("o", 4096, 4096, 1),
                            ("gate_up", 28672, 4096, 0), ("down", 4096, 14336, 1)):
        X = torch.randn(T, K, device=dev).bfloat16()
        Ws = [(0.02 * torch.randn(N, K, device=dev)).bfloat16() for _ in range(4)]
        arr = (P * 4)(*[w.data_ptr() for w in Ws])
        Y = torch.zeros(T, N, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
        print(f"== T={T} {name}", file=sys.stderr, flush=True)
        rc = f(X.data_ptr(), arr, 4, Y.data_ptr(), T, N, K, f32, 20, s)
        assert rc == 0, rc
        del Ws
