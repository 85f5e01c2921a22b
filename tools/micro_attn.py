"""Run K7/K6 attention at one (past, q) point (8B-shape layer) for ncu / timing."""
import ctypes, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26289_b200 import _lib

past = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
q = int(sys.argv[2]) if len(sys.argv) > 2 else 5
impl = int(sys.argv[3]) if len(sys.argv) > 3 else 0
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 10
dev = torch.device("cuda", 0)
nh, nkv, d = 32, 8, 128
L = _lib.lib()
kv_len = past + q
cap = kv_len + 64
g = torch.Generator(device=dev).manual_seed(7)
# two pool copies, alternated, so a launch never finds the previous one's K/V in L2
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
def launch(i=0):
    kp, vp = pools[i & 1]
    _lib.check(L.ds_attention(qkv.data_ptr(), ctypes.addressof(ent), ent_d.data_ptr(), 1, q,
                              kp.data_ptr(), vp.data_ptr(), cap, p2c.data_ptr(), cap, nh, nkv, d,
                              1.0 / d ** 0.5, o.data_ptr(), ws.data_ptr(), wsb, impl, s.cuda_stream))
for _ in range(2):
    launch()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(iters):
    launch(i)
b.record(); b.synchronize()
t = a.elapsed_time(b) * 1e3 / iters  # back-to-back, alternating pools: K/V from HBM
byt = nkv * 2 * d * 2 * kv_len
fl = 4.0 * nh * d * q * (past + (q + 1) / 2)
print(f"past={past} q={q} impl={impl}: {t:.1f} us  {byt / t / 1e3:.0f} GB/s  {fl / t / 1e6:.1f} TFLOP/s")
