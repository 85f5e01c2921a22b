"""cProfile of the host side of one C5 step (256 sessions, batched plans) on the GPU box."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26289_b200.scheduler import InferenceCore
from paper_2605_26289_b200.workload import core_config_for, load_trace, replay

tr = load_trace("c5")
core = InferenceCore(core_config_for(tr, model="llama3-8b", batched_forward=True))
core.reset_state(); replay(core, tr)
torch.cuda.synchronize()
core.engine.reset_counters()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
core.reset_state(); replay(core, tr)
pr.disable()
print(f"wall {time.perf_counter() - t0:.2f} s, device {core.engine.device_seconds():.2f} s")
st = pstats.Stats(pr)
for key in (sys.argv[1:] or ["tottime"]):
    st.sort_stats(key).print_stats(45)
