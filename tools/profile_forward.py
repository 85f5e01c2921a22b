"""Per-kernel GPU time of one decode/verify forward (8B shape) via torch.profiler (CUPTI)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2605_26289_b200 import _lib
from paper_2605_26289_b200.config import CoreConfig
from paper_2605_26289_b200.engine import EntryRequest, GpuEngine
from paper_2605_26289_b200.kvcache import UnifiedKvCache

model = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"
past = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
q = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cfg = CoreConfig(model=model, capacity_cells=max(8192, past + 4096))
kv = UnifiedKvCache(cfg.capacity_cells)
eng = GpuEngine(cfg, kv, n_seqs=2)
toks = [int(x) for x in torch.randint(0, 30000, (past + q,))]
eng.load_prompt(0, toks, 0, 0xCBF29CE484222325)
done = 0
while done < past:
    n = min(4096, past - done)
    kv.append_cells(0, n)
    eng.run([EntryRequest(_lib.ENTRY_PREFILL, 0, done, toks[done:done + n], toks)])
    done += n
kv.append_cells(0, q)
kind = _lib.ENTRY_VERIFY if q > 1 else _lib.ENTRY_DECODE
req = EntryRequest(kind, 0, past, toks[past:past + q], toks, n_draft=q - 1 if q > 1 else 0)
for _ in range(3):
    eng.run([req])
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        eng.run([req])
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
st = eng.forward_stats()
print(st)

# critical-path attribution: with PDL a kernel launches early and waits, so its
# duration overstates its cost; the gap between consecutive kernel END times on
# the main stream is what each kernel adds to the forward.
import json, tempfile
from collections import defaultdict
tr = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(tr)
ev = [e for e in json.load(open(tr))["traceEvents"] if e.get("cat") == "kernel"]
streams = defaultdict(list)
for e in ev:
    streams[e["args"].get("stream")].append(e)
main = max(streams.values(), key=len)
main.sort(key=lambda e: e["ts"] + e["dur"])
inc = defaultdict(float)
cnt = defaultdict(int)
for a, b in zip(main, main[1:]):
    name = b["name"].split("(")[0].split("<")[0][:48]
    if "gemm_skinny" in name:  # split by shape (grid size)
        name += f" grid={b['args'].get('grid')}"
    inc[name] += (b["ts"] + b["dur"]) - (a["ts"] + a["dur"])
    cnt[name] += 1
tot = sum(inc.values())
print(f"\ncritical-path increments over {len(main)} kernels ({tot / 5:.1f} us per forward):")
for k, v in sorted(inc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:60s} {cnt[k] // 5:5d}/fwd {v / 5:9.1f} us/fwd {v / cnt[k]:7.2f} us each {v / tot * 100:5.1f}%")
