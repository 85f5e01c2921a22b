"""Counter registry for the core (the subset of metrics.py:82-138 the hot path
touches); per-turn timings come from CUDA events, not a simulated cost model."""
from __future__ import annotations

import threading
from collections import Counter


class MetricsRegistry:
    def __init__(self):
        self._lock = threading.Lock()
        self._c: Counter = Counter()
        self.turns: list[dict] = []

    def add(self, name: str, n: int = 1) -> None:
        with self._lock:
            self._c[name] += n

    def counters(self) -> dict:
        with self._lock:
            return dict(self._c)

    def record_turn(self, row: dict) -> None:
        with self._lock:
            self.turns.append(row)

    def reset(self) -> None:
        with self._lock:
            self._c.clear()
            self.turns.clear()
