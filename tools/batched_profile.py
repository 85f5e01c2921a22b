"""Per-kernel GPU time of one batched decode forward (N sessions x 1 row, past m)
- the C5 shape - via torch.profiler."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2605_26289_b200 import _lib
from paper_2605_26289_b200.config import CoreConfig
from paper_2605_26289_b200.engine import EntryRequest, GpuEngine
from paper_2605_26289_b200.kvcache import UnifiedKvCache

n, past = int(sys.argv[1]), int(sys.argv[2])
cfg = CoreConfig(model="llama3-8b", capacity_cells=n * (past + 8) + 1024, batched_forward=True)
kv = UnifiedKvCache(cfg.capacity_cells)
eng = GpuEngine(cfg, kv, n_seqs=n)
toks = [(7 * i + 3) % 30000 for i in range(past + 4)]
reqs = []
for s in range(n):
    eng.load_prompt(s, toks, 0, 0xCBF29CE484222325)
    kv.append_cells(s, past + 1)
    reqs.append(EntryRequest(_lib.ENTRY_DECODE, s, past, toks[past:past + 1], toks))
for _ in range(3):
    eng.run(reqs, count=False)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        eng.run(reqs, count=False)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14, max_name_column_width=60))
st = eng.forward_stats()
print({k: (v["n"], round(v["seconds"] / max(v["n"], 1) * 1e3, 3)) for k, v in st.items()})
