"""Median device time of one whole-model forward at (past, q) through GpuEngine
(CUDA events around ds_model_forward; no profiler).  Usage:
  fwd_time.py MODEL PAST:Q [PAST:Q ...]   (set DS_B200_LIB for an A/B build)"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_26289_b200 import _lib
from paper_2605_26289_b200.config import CoreConfig
from paper_2605_26289_b200.engine import EntryRequest, GpuEngine
from paper_2605_26289_b200.kvcache import UnifiedKvCache

model = sys.argv[1]
pts = [tuple(int(v) for v in a.split(":")) for a in sys.argv[2:]]
mx = max(p + q for p, q in pts)
cfg = CoreConfig(model=model, capacity_cells=mx + 512)
kv = UnifiedKvCache(cfg.capacity_cells)
eng = GpuEngine(cfg, kv, n_seqs=1, keep_logits=True)
toks = [(7 * i + 3) % 30000 for i in range(mx + 8)]
eng.load_prompt(0, toks, 0, 0xCBF29CE484222325)
tag = os.environ.get("DS_B200_LIB", "tree") + f" L2={os.environ.get('DS_L2_NEXT_MB', 'dflt')}"
for past, q in pts:
    kv.append_cells(0, past + q)
    kind = _lib.ENTRY_PREFILL if q > 24 else _lib.ENTRY_VERIFY if q > 1 else _lib.ENTRY_DECODE
    req = EntryRequest(kind, 0, past, toks[past:past + q], toks,
                       n_draft=q - 1 if kind == _lib.ENTRY_VERIFY else 0)
    ts = []
    for i in range(25):
        b = eng.device_seconds()
        eng.run([req], count=False)
        ts.append(eng.device_seconds() - b)
    kv.trim(0, 0)
    import torch
    lg = eng.logits[: (q if kind == _lib.ENTRY_VERIFY else 1)]
    fin = bool(torch.isfinite(lg).all())
    mag = float(lg.abs().max()) if fin else float("nan")
    ts = sorted(ts[5:])
    print(f"{tag:40s} past={past:6d} q={q:4d}: median {1e6 * statistics.median(ts):8.1f} us  "
          f"min {1e6 * ts[0]:8.1f}  max {1e6 * ts[-1]:8.1f}  logits finite={fin} max|.|={mag:.3g}", flush=True)
