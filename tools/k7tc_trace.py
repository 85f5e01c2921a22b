"""K7-tc phase timing in back-to-back launches (needs the DS_K7_TRACE build in
ab_trace/).  Stamps: 6 CTA start, 0 before / 1 after the dependency wait,
2 first S ready, 3 tile loop done, 5 exit."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("DS_B200_LIB", os.path.join(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))), "ab_trace", "libdeltaserve_b200.so"))
import numpy as np
import torch
from paper_2605_26289_b200 import _lib

past, q = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda", 0)
nh, nkv, d = 32, 8, 128
L = _lib.lib()
kv_len = past + q
cap = kv_len + 64
g = torch.Generator(device=dev).manual_seed(7)
pools = [(torch.randn(nkv, cap, d, device=dev, dtype=torch.bfloat16, generator=g),
          torch.randn(nkv, cap, d, device=dev, dtype=torch.bfloat16, generator=g)) for _ in range(2)]
p2c = torch.arange(cap, dtype=torch.int32, device=dev).view(1, cap)
qkv = torch.randn(q, (nh + 2 * nkv) * d, device=dev, dtype=torch.bfloat16, generator=g)
o = torch.empty(q, nh * d, device=dev, dtype=torch.bfloat16)
ent = (_lib.Entry * 1)(_lib.Entry(0, past, q, 0, 0, 0, 0, 1, 0))
ent_d = torch.frombuffer(bytearray(bytes(ent)), dtype=torch.uint8).to(dev)
wsb = L.ds_attention_workspace_bytes(q, 1, nh, d)
ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream()
def launch(i):
    kp, vp = pools[i & 1]
    _lib.check(L.ds_attention(qkv.data_ptr(), ctypes.addressof(ent), ent_d.data_ptr(), 1, q,
                              kp.data_ptr(), vp.data_ptr(), cap, p2c.data_ptr(), cap, nh, nkv, d,
                              1.0 / d ** 0.5, o.data_ptr(), ws.data_ptr(), wsb, 1, s.cuda_stream))
buf = (ctypes.c_ulonglong * (1024 * 8))()
for i in range(8):
    launch(i)
torch.cuda.synchronize()
L.ds_debug_k7tc_trace(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 8).astype(np.int64)
a = a[a[:, 6] > 0]
t0 = a[:, 6].min()
for i, nm in ((6, "start"), (0, "pre-wait"), (1, "waited"), (2, "S0 ready"), (3, "loop done"), (5, "exit")):
    v = (a[:, i] - t0) / 1000.0
    print(f"  {nm:10s} {v.min():7.2f} {np.median(v):7.2f} {v.max():7.2f}")
