"""Per-forward latency and tok/s versus prefix length (BASELINE metric: "delta-prefill /
decode tok/s vs prefix length").

Drives the same GpuEngine forward the scheduler issues at scheduler.py:711
(delta-prefill chunk), :766 (decode) and speculator.py:102 (verify), over a
sequence whose first ``m`` positions are mapped cells of the paged store
(``append_cells`` = page-table writes only; the prefix K/V content does not
change the work).  Each point is the device time of the whole forward (all
layers, LM head, token policy) from the engine's CUDA events, median of
``reps`` forwards.  The per-turn model the north_star targets is
t_turn(m) = t_prefill(Delta, m) + n_pass * t_verify(k+1, m): flat in m means
O(Delta_t) per turn.
"""
from __future__ import annotations

import statistics

from . import _lib
from .config import CoreConfig
from .engine import EntryRequest, GpuEngine
from .kvcache import UnifiedKvCache

DEFAULT_PREFIXES = (0, 1024, 2048, 4096, 8192, 16384, 32768)


def prefix_curve(model: str = "llama3-8b", prefixes=DEFAULT_PREFIXES, delta: int = 150,
                 k: int = 4, reps: int = 5, weights: dict | None = None) -> dict:
    m_max = max(prefixes)
    cfg = CoreConfig(model=model, capacity_cells=m_max + delta + 512)
    kv = UnifiedKvCache(cfg.capacity_cells)
    eng = GpuEngine(cfg, kv, n_seqs=1, weights=weights)  # weights shared with the caller's engine
    toks = [(7 * i + 3) % 30000 for i in range(m_max + delta + 8)]
    eng.load_prompt(0, toks, 0, 0xCBF29CE484222325)
    points = []

    def timed(req: EntryRequest) -> float:
        ts = []
        for _ in range(reps + 1):
            before = eng.device_seconds()
            eng.run([req], count=False)
            ts.append(eng.device_seconds() - before)
        return statistics.median(ts[1:])

    cur = 0
    for m in sorted(prefixes):
        if m > cur:
            kv.append_cells(0, m - cur)  # the prefix: page-table mapping only
            cur = m
        row = {"m": m}
        for name, q, kind in (("prefill", delta, _lib.ENTRY_PREFILL),
                              ("verify", k + 1, _lib.ENTRY_VERIFY),
                              ("decode", 1, _lib.ENTRY_DECODE)):
            kv.append_cells(0, q)
            req = EntryRequest(kind, 0, m, toks[m:m + q], toks,
                               n_draft=q - 1 if kind == _lib.ENTRY_VERIFY else 0)
            t = timed(req)
            kv.trim(0, m)
            row[f"{name}_ms"] = round(1000 * t, 3)
            if name == "prefill":
                row["prefill_tok_s"] = round(q / t, 1)
        # greedy verify at 100% acceptance commits k+1 tokens per pass
        row["verify_tok_s_full_accept"] = round((k + 1) / (row["verify_ms"] / 1000), 1)
        row["decode_tok_s"] = round(1 / (row["decode_ms"] / 1000), 1)
        points.append(row)
    base = points[0]
    worst = max(points, key=lambda r: r["verify_ms"])
    return {"what": f"whole-model forward device time vs prefix length m (delta={delta} prefill, "
                    f"k={k} verify, decode), median of {reps}",
            "delta": delta, "k": k, "points": points,
            "verify_ms_ratio_mmax_vs_m0": round(points[-1]["verify_ms"] / base["verify_ms"], 3),
            "prefill_ms_ratio_mmax_vs_m0": round(points[-1]["prefill_ms"] / base["prefill_ms"], 3),
            "worst_verify_m": worst["m"]}
