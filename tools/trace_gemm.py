"""K10 per-CTA timeline (DS_STREAM_TRACE build path): stamps relative to the
earliest CTA start, in microseconds.  Usage: DS_STREAM_TRACE=1 trace_gemm.py T N K"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2605_26289_b200._lib import check, lib

T, N, K = (int(x) for x in sys.argv[1:4])
dev = torch.device("cuda", 0)
X = torch.randn(T, K, device=dev).bfloat16()
W = (0.02 * torch.randn(N, K, device=dev)).bfloat16()
Y = torch.zeros(T, N, device=dev).bfloat16()
s = torch.cuda.current_stream()
L = lib()
for i in range(4):
    check(L.ds_gemm_stream(X.data_ptr(), W.data_ptr(), Y.data_ptr(), T, N, K, 0, 0, None,
                           s.cuda_stream))
    if os.environ.get("ISOLATED"):
        torch.cuda.synchronize()
torch.cuda.synchronize()
stamps = torch.zeros(2, dtype=torch.int64, device=dev)
L.ds_debug_stamp.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
L.ds_debug_stamp(stamps.data_ptr(), s.cuda_stream)
check(L.ds_gemm_stream(X.data_ptr(), W.data_ptr(), Y.data_ptr(), T, N, K, 0, 0, None,
                       s.cuda_stream))
L.ds_debug_stamp(stamps.data_ptr() + 8, s.cuda_stream)
torch.cuda.synchronize()
st = stamps.cpu().numpy()
if os.environ.get("FLUSH"):
    junk = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    junk.zero_()
    torch.cuda.synchronize()
    L.ds_debug_stamp(stamps.data_ptr(), s.cuda_stream)
    check(L.ds_gemm_stream(X.data_ptr(), W.data_ptr(), Y.data_ptr(), T, N, K, 0, 0, None,
                           s.cuda_stream))
    L.ds_debug_stamp(stamps.data_ptr() + 8, s.cuda_stream)
    torch.cuda.synchronize()
    st = stamps.cpu().numpy()
P = int(os.environ.get("NCTA", "148"))
buf = (ctypes.c_ulonglong * (P * 16))()
L.ds_gemm_stream_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.ds_gemm_stream_trace(ctypes.addressof(buf), P)
a = np.array(buf, dtype=np.int64).reshape(P, 16)[:, :14]
t0 = a[:, 0].min()
print(f"stamp before -> first CTA start {(t0 - st[0]) / 1000:.2f} us; "
      f"last CTA end -> stamp after {(st[1] - a[:, 7].max()) / 1000:.2f} us; "
      f"total {(st[1] - st[0]) / 1000:.2f} us")
r = (a - t0) / 1000.0
r[a == 0] = np.nan
names = ["start", "setup", "prod", "mma", "contrib", "hwait0", "hwait1", "end", "hacc", "bulkN",
         "chunkN", "hdone", "bulk0", "batch0"]
print("cta " + " ".join(f"{n:>8s}" for n in names))
order = np.argsort(r[:, 0])
print("start-time deciles:", np.round(np.nanpercentile(r[:, 0], [0, 10, 50, 80, 90, 95, 100]), 2))
late = [int(c) for c in order[-12:]]
print("latest-starting CTAs:", late)
for c in list(range(0, P, 16)) + late[-4:]:
    print(f"{c:3d} " + " ".join(f"{x:8.2f}" for x in r[c]))
raw = np.array(buf, dtype=np.int64).reshape(P, 16)
if os.environ.get("PROBE"):
    print("probe ns (dsmem ld, local ld, 1000 dependent FFMA):", raw[:6, 11:14].tolist())
ok = raw[:, 14] > 0
if ok.any():
    print("SM clock MHz (head CTAs):", np.round(raw[ok, 15] / raw[ok, 14] * 1000, 0)[:8])
print("max end", np.nanmax(r[:, 7]), "mean setup", np.nanmean(r[:, 1]), "mean mma", np.nanmean(r[:, 3]),
      "mean wait", np.nanmean(r[:, 6] - r[:, 5]))
