"""Kernel start/end timeline (CUPTI via torch.profiler) of one whole-model
forward at (past, q): prints the kernels of layers 4-5 relative to the first
kernel of layer 4.  Usage: timeline.py MODEL PAST Q"""
import json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2605_26289_b200 import _lib
from paper_2605_26289_b200.config import CoreConfig
from paper_2605_26289_b200.engine import EntryRequest, GpuEngine
from paper_2605_26289_b200.kvcache import UnifiedKvCache

model, past, q = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
edges = len(sys.argv) > 4 and sys.argv[4] == "edges"
cfg = CoreConfig(model=model, capacity_cells=past + q + 512)
kv = UnifiedKvCache(cfg.capacity_cells)
eng = GpuEngine(cfg, kv, n_seqs=1)
toks = [(7 * i + 3) % 30000 for i in range(past + q + 8)]
eng.load_prompt(0, toks, 0, 0xCBF29CE484222325)
kv.append_cells(0, past + q)
kind = _lib.ENTRY_PREFILL if q > 24 else _lib.ENTRY_VERIFY if q > 1 else _lib.ENTRY_DECODE
req = EntryRequest(kind, 0, past, toks[past:past + q], toks, n_draft=q - 1 if q > 1 else 0)
for _ in range(5):
    eng.run([req], count=False)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eng.run([req], count=False)
tr = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(tr)
ev = sorted([e for e in json.load(open(tr))["traceEvents"] if e.get("cat") == "kernel"],
            key=lambda e: e["ts"])
main = [e for e in ev if e["args"].get("stream") == max(set(x["args"].get("stream") for x in ev), key=lambda s: sum(1 for x in ev if x["args"].get("stream") == s))]
# layer boundaries: the wqkv projection is the grid with (nh+2nkv)*hd/16 CTAs
s = cfg.shape
g_qkv = s.qkv_width // 16
starts = [i - 1 for i, e in enumerate(main) if "attn_" in e["name"] and "combine" not in e["name"]]
i0, i1 = starts[4], starts[5]
if edges:  # the forward's head (up to layer 1) and tail (from the last layer's attention)
    sel = main[: starts[1]] + main[starts[-1]:]
    t0 = main[0]["ts"]
    print(f"past={past} q={q} forward {main[-1]['ts'] + main[-1]['dur'] - t0:.1f} us (edges)")
    for e in sorted(ev, key=lambda e: e["ts"]):
        if e in sel or e not in main:
            nm = e["name"].split("(")[0].replace("void ds::", "").replace("ds::", "")[:28]
            print(f"  s{e['args'].get('stream')} {nm:28s} grid={str(e['args'].get('grid')):16s} "
                  f"start {e['ts'] - t0:8.2f} end {e['ts'] + e['dur'] - t0:8.2f} dur {e['dur']:7.2f}")
    sys.exit(0)
t0 = main[i0]["ts"]
print(f"past={past} q={q} forward {main[-1]['ts'] + main[-1]['dur'] - main[0]['ts']:.1f} us")
t1 = main[i1]["ts"]
for e in [x for x in ev if main[i0]["ts"] - 50 <= x["ts"] < t1]:
    nm = e["name"].split("(")[0].replace("void ds::", "").replace("ds::", "")[:28]
    print(f"  s{e['args'].get('stream')} {nm:28s} grid={str(e['args'].get('grid')):16s} start {e['ts'] - t0:8.2f} "
          f"end {e['ts'] + e['dur'] - t0:8.2f} dur {e['dur']:7.2f}")
