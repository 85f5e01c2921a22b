"""Host launch cost vs device time of ds_gemm_stream (one shape)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26289_b200._lib import check, lib

T, N, K = (int(x) for x in sys.argv[1:4])
dev = torch.device("cuda", 0)
X = torch.randn(T, K, device=dev).bfloat16()
Ws = [(0.02 * torch.randn(N, K, device=dev)).bfloat16() for _ in range(4)]
Y = torch.zeros(T, N, device=dev).bfloat16()
s = torch.cuda.current_stream()
L = lib()
f = L.ds_gemm_stream
for i in range(5):
    check(f(X.data_ptr(), Ws[i % 4].data_ptr(), Y.data_ptr(), T, N, K, 0, 0, None, s.cuda_stream))
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(20):
    f(X.data_ptr(), Ws[i % 4].data_ptr(), Y.data_ptr(), T, N, K, 0, 0, None, s.cuda_stream)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e6*(t1-t0)/20:.1f} us/launch, wall incl. drain {1e6*(t2-t0)/20:.1f} us/launch")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(20_000_000)  # let the host run ahead: events then time the GPU only
a.record()
for i in range(20):
    f(X.data_ptr(), Ws[i % 4].data_ptr(), Y.data_ptr(), T, N, K, 0, 0, None, s.cuda_stream)
b.record()
b.synchronize()
print(f"device {a.elapsed_time(b)*1e3/20:.1f} us/launch (host ahead)")
# isolated launches (synchronize between), same weights / rotating
for rot in (False, True):
    ts = []
    for i in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f(X.data_ptr(), Ws[i % 4 if rot else 0].data_ptr(), Y.data_ptr(), T, N, K, 0, 0, None,
          s.cuda_stream)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(f"isolated rot={rot}: " + " ".join(f"{t:.1f}" for t in ts))
# back to back, same weights
torch.cuda._sleep(20_000_000)
a.record()
for i in range(20):
    f(X.data_ptr(), Ws[0].data_ptr(), Y.data_ptr(), T, N, K, 0, 0, None, s.cuda_stream)
b.record()
b.synchronize()
print(f"back-to-back same W {a.elapsed_time(b)*1e3/20:.1f} us/launch")
