"""Where the wall clock between device forwards goes (GPU box): wraps
GpuEngine.run / propose and the stream sync with perf_counter stamps during C2
replays and prints per-forward averages."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26289_b200 import engine as E
from paper_2605_26289_b200.scheduler import InferenceCore
from paper_2605_26289_b200.workload import core_config_for, load_trace, replay

acc = {"in_run_pre": 0.0, "sync": 0.0, "in_run_post": 0.0, "between": 0.0, "propose": 0.0,
       "n": 0, "np": 0}
last_exit = [None]
orig_sync = torch.cuda.Stream.synchronize
cur = {}


def sync(self):
    t = time.perf_counter()
    cur["pre_end"] = t
    orig_sync(self)
    cur["sync_end"] = time.perf_counter()


torch.cuda.Stream.synchronize = sync
orig_run, orig_prop = E.GpuEngine.run, E.GpuEngine.propose


def run(self, *a, **k):
    t0 = time.perf_counter()
    if last_exit[0] is not None:
        acc["between"] += t0 - last_exit[0]
    r = orig_run(self, *a, **k)
    t1 = time.perf_counter()
    acc["in_run_pre"] += cur["pre_end"] - t0
    acc["sync"] += cur["sync_end"] - cur["pre_end"]
    acc["in_run_post"] += t1 - cur["sync_end"]
    acc["n"] += 1
    last_exit[0] = t1
    return r


def propose(self, *a, **k):
    t0 = time.perf_counter()
    r = orig_prop(self, *a, **k)
    acc["propose"] += time.perf_counter() - t0
    acc["np"] += 1
    return r


E.GpuEngine.run, E.GpuEngine.propose = run, propose
_real_lib = E.lib()
acc["native"] = 0.0
acc["apply_meta"] = 0.0


class _Proxy:
    def __getattr__(self, name):
        f = getattr(_real_lib, name)
        if name in ("ds_model_forward", "ds_kv_apply", "ds_hist_write", "ds_kv_copy_cells"):
            key = "native" if name == "ds_model_forward" else "apply_meta"

            def w(*a):
                t = time.perf_counter()
                r = f(*a)
                acc[key] += time.perf_counter() - t
                return r
            return w
        return f


_proxy = _Proxy()
E.lib = lambda: _proxy
tr = load_trace(sys.argv[1] if len(sys.argv) > 1 else "c2")
core = InferenceCore(core_config_for(tr, model=os.environ.get("DS_MODEL", "llama3-8b"),
                                    batched_forward=bool(int(os.environ.get("BATCHED", "0")))))
REPS = int(os.environ.get("REPS", "3"))
for _ in range(2 if REPS > 1 else 1):
    core.reset_state(); replay(core, tr)
for k in acc: acc[k] = 0 if k in ("n", "np") else 0.0
last_exit[0] = None
core.engine.reset_counters()
t0 = time.perf_counter()
for _ in range(REPS):
    core.reset_state(); replay(core, tr)
wall = time.perf_counter() - t0
n = acc["n"]
print(f"wall/step {wall / REPS * 1e3:.1f} ms, device/step {core.engine.device_seconds() / REPS * 1e3:.1f} ms, "
      f"forwards/step {n / REPS:.0f}, proposes/step {acc['np'] / REPS:.0f}")
for k in ("in_run_pre", "native", "apply_meta", "sync", "in_run_post", "between", "propose"):
    print(f"  {k:12s} {acc[k] / n * 1e6:8.1f} us per forward   ({acc[k] / REPS * 1e3:6.1f} ms/step)")
