"""K7 phase timing inside a real forward (needs the DS_K7_TRACE build:
DS_LIB_OUT=ab_trace/libdeltaserve_b200.so DS_NVCC_EXTRA=-DDS_K7_TRACE).
Prints, for the LAST layer's K7 launch of one forward, per-CTA globaltimer
stamps relative to the earliest CTA start:
  6 CTA start, 0 before pdl_wait, 1 after pdl_wait, 2 first tile ready,
  3 main loop done, 4 warp merge + partials done, 5 exit (after cluster merge)."""
import ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("DS_B200_LIB", os.path.join(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))), "ab_trace", "libdeltaserve_b200.so"))
import numpy as np
from paper_2605_26289_b200 import _lib
from paper_2605_26289_b200.config import CoreConfig
from paper_2605_26289_b200.engine import EntryRequest, GpuEngine
from paper_2605_26289_b200.kvcache import UnifiedKvCache

model, past, q = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = CoreConfig(model=model, capacity_cells=past + q + 512)
kv = UnifiedKvCache(cfg.capacity_cells)
eng = GpuEngine(cfg, kv, n_seqs=1)
toks = [(7 * i + 3) % 30000 for i in range(past + q + 8)]
eng.load_prompt(0, toks, 0, 0xCBF29CE484222325)
kv.append_cells(0, past + q)
kind = _lib.ENTRY_VERIFY if q > 1 else _lib.ENTRY_DECODE
req = EntryRequest(kind, 0, past, toks[past:past + q], toks, n_draft=q - 1 if q > 1 else 0)
L = _lib.lib()
buf = (ctypes.c_ulonglong * (1024 * 8))()
cbuf = (ctypes.c_longlong * (1024 * 16))()
res = []
cres = []
for rep in range(6):
    ctypes.memset(buf, 0, ctypes.sizeof(buf))
    eng.run([req], count=False)
    L.ds_debug_k7_trace(buf)
    ctypes.memset(cbuf, 0, ctypes.sizeof(cbuf))
    L.ds_debug_k7_clk(cbuf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 8).astype(np.int64)
    a = a[a[:, 6] > 0]
    c = np.frombuffer(cbuf, dtype=np.int64).reshape(1024, 16)
    if rep:
        res.append(a)
        cres.append(c[: len(a)].copy())
a = res[-1]
t0 = a[:, 6].min()
names = {6: "start", 0: "pre-wait", 1: "waited", 2: "tile0", 3: "loop", 7: "osm-wr", 4: "merge", 5: "exit"}
print(f"past={past} q={q}: {len(a)} CTAs; times (us) relative to the first CTA start: "
      "min / median / max")
for i in (6, 0, 1, 2, 3, 7, 4, 5):
    v = (a[:, i] - t0) / 1000.0
    print(f"  {names[i]:9s} {v.min():7.2f} {np.median(v):7.2f} {v.max():7.2f}")

# SM-clock deltas of thread 0 from its dependency wait (cycles -> us at 1.965 GHz)
c = cres[-1]
c = c[c[:, 0] > 0]
cn = {1: "tile0", 2: "max-exch", 3: "P-exch", 4: "PV done", 9: "row sums", 10: "rows done",
      11: "branch out", 5: "rows out", 6: "csync1", 7: "merged", 8: "csync2"}
print("thread-0 SM-clock phase ends after the wait (us, median / max over CTAs):")
for i in (1, 2, 3, 4, 9, 10, 11, 5, 6, 7, 8):
    v = c[:, i]
    ok = v > 0
    if not ok.any():
        continue
    d = (v[ok] - c[ok, 0]) / 1965.0
    print(f"  {cn[i]:9s} {np.median(d):7.2f} {d.max():7.2f}")
