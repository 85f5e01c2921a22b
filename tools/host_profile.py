"""cProfile of the host side of C2 replays (GPU box): where the wall-clock time
between device forwards goes."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26289_b200.scheduler import InferenceCore
from paper_2605_26289_b200.workload import core_config_for, load_trace, replay

tr = load_trace(sys.argv[1] if len(sys.argv) > 1 else "c2")
core = InferenceCore(core_config_for(tr, model=os.environ.get("DS_MODEL", "llama3-8b")))
for _ in range(2):
    core.reset_state(); replay(core, tr)
torch.cuda.synchronize()
core.engine.reset_counters()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(3):
    core.reset_state(); replay(core, tr)
pr.disable()
wall = time.perf_counter() - t0
dev = core.engine.device_seconds()
print(f"wall {wall * 1000 / 3:.1f} ms/step, device forwards {dev * 1000 / 3:.1f} ms/step")
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(40)
