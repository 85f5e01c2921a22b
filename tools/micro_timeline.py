"""Kernel timeline (torch.profiler / CUPTI) of back-to-back K7 launches at one
(past, q) point: shows each launch's attention kernel and merge kernel."""
import ctypes, json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
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
for i in range(4): launch(i)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(6): launch(i)
    torch.cuda.synchronize()
tr = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(tr)
ev = sorted([e for e in json.load(open(tr))["traceEvents"] if e.get("cat") == "kernel"], key=lambda e: e["ts"])
t0 = ev[0]["ts"]
for e in ev:
    print(f"  {e['name'][:34]:34s} grid={str(e['args'].get('grid')):14s} start {e['ts']-t0:8.2f} end {e['ts']+e['dur']-t0:8.2f} dur {e['dur']:7.2f}")
