"""A/B of the M > 32 projection path on the 8B shape: whole-forward device time
of a delta-prefill chunk (prefix_curve points) and a batched decode plan of
many sequences (n_out > 32: the LM head with / without fp32 logits).
Run twice: DS_GEMM_STREAM=0 (cuBLAS + unfused) and DS_GEMM_STREAM=1 (K10)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26289_b200 import _lib
from paper_2605_26289_b200.config import CoreConfig
from paper_2605_26289_b200.curve import prefix_curve
from paper_2605_26289_b200.engine import EntryRequest, GpuEngine
from paper_2605_26289_b200.kvcache import UnifiedKvCache

tag = os.environ.get("DS_GEMM_STREAM", "0")
c = prefix_curve(prefixes=(0, 1024), delta=int(os.environ.get("DELTA", "150")), reps=5)
for p in c["points"]:
    print(f"[stream={tag}] m={p['m']} prefill {p['prefill_ms']} ms verify {p['verify_ms']} ms")
# batched decode plan: B sequences x 2 rows (verify k=1), m = 1024 each
B = int(os.environ.get("BATCH", "256"))
cfg = CoreConfig(model="llama3-8b", capacity_cells=B * 1100 + 4096, batched_forward=True,
                 spec_max_lookahead=1, n_batch=4096)
kv = UnifiedKvCache(cfg.capacity_cells)
eng = GpuEngine(cfg, kv, n_seqs=B + 1)
toks = [(11 * i + 5) % 30000 for i in range(1100)]
for s in range(B):
    eng.load_prompt(s, toks, 0, 0xCBF29CE484222325)
    kv.append_cells(s, 1024)
reqs = [EntryRequest(_lib.ENTRY_VERIFY, s, 1024, toks[1024:1026], toks, n_draft=1, scratch=True)
        for s in range(B)]
ts = []
for i in range(6):
    before = eng.device_seconds()
    eng.run(reqs, count=False)
    ts.append(eng.device_seconds() - before)
print(f"[stream={tag}] batched verify B={B} rows={2*B}: {1000*statistics.median(ts[1:]):.3f} ms")
