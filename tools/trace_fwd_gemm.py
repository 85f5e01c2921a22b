"""K10 per-CTA timeline of the LAST K10 launch of one whole-model forward
(DS_GEMM_STREAM=1 DS_STREAM_TRACE=1): the layer-31 down projection of a
delta-prefill chunk, in place - compare with tools/trace_gemm.py (isolated).
Usage: DS_GEMM_STREAM=1 DS_STREAM_TRACE=1 trace_fwd_gemm.py PAST Q NCTA"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_26289_b200 import _lib
from paper_2605_26289_b200.config import CoreConfig
from paper_2605_26289_b200.engine import EntryRequest, GpuEngine
from paper_2605_26289_b200.kvcache import UnifiedKvCache

past, q, P = (int(x) for x in sys.argv[1:4])
cfg = CoreConfig(model="llama3-8b", capacity_cells=past + q + 512)
kv = UnifiedKvCache(cfg.capacity_cells)
eng = GpuEngine(cfg, kv, n_seqs=1)
toks = [(7 * i + 3) % 30000 for i in range(past + q + 8)]
eng.load_prompt(0, toks, 0, 0xCBF29CE484222325)
kv.append_cells(0, past + q)
req = EntryRequest(_lib.ENTRY_PREFILL, 0, past, toks[past:past + q], toks)
for i in range(3):
    eng.run([req], count=False)
L = _lib.lib()
buf = (ctypes.c_ulonglong * (P * 16))()
L.ds_gemm_stream_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.ds_gemm_stream_trace(ctypes.addressof(buf), P)
a = np.array(buf, dtype=np.int64).reshape(P, 16)
t0 = a[:, 0].min()
r = (a - t0) / 1000.0
r[a == 0] = np.nan
cols = {"start": 0, "setup": 1, "wprod": 2, "acc": 3, "part": 4, "csync": 5, "epi": 9, "end": 7}
print("cta " + " ".join(f"{n:>7s}" for n in cols))
for c in range(0, P, max(1, P // 12)):
    print(f"{c:3d} " + " ".join(f"{r[c, i]:7.2f}" for i in cols.values()))
for n, i in cols.items():
    print(f"{n:6s} min {np.nanmin(r[:, i]):7.2f} median {np.nanmedian(r[:, i]):7.2f} max {np.nanmax(r[:, i]):7.2f}")
