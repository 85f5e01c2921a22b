import torch, sys
sys.path.insert(0, "/root/repo")
from paper_2605_26289_b200._lib import check, lib
cuda = torch.device("cuda", 0)
for (N, K) in [(6144, 4096), (4096, 4096), (2048, 4096), (6144, 1024), (4736, 4096), (4608, 4096)]:
    row = []
    for M in range(1, 9):
        g = torch.Generator(device=cuda).manual_seed(M + N + K)
        X = torch.randn(M, K, device=cuda, generator=g).bfloat16()
        W = (0.02 * torch.randn(N, K, device=cuda, generator=g)).bfloat16()
        Y = torch.zeros(M, N, device=cuda)
        check(lib().ds_gemm_skinny(X.data_ptr(), W.data_ptr(), Y.data_ptr(), M, N, K, 1, 0,
                                   torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        ref = X.float() @ W.float().T
        err = (Y - ref).abs()
        bad = (err > 1e-3).nonzero()
        row.append(f"M{M}:{'ok' if len(bad) == 0 else 'BAD n=%d rows=%s cols=%s..' % (len(bad), sorted(set(bad[:,0].tolist())), bad[:4,1].tolist())}")
    print(N, K, " ".join(row))
