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
