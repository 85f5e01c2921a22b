"""Debug: per-row logit error of the tiny model vs the CPU oracle variants."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import llama_ref
from paper_2605_26289_b200 import _lib
from paper_2605_26289_b200.config import CoreConfig
from paper_2605_26289_b200.engine import EntryRequest, GpuEngine
from paper_2605_26289_b200.kvcache import UnifiedKvCache

for layers in (1, 2):
    cfg = CoreConfig(model="tiny", token_policy="argmax", capacity_cells=4096)
    import dataclasses
    from paper_2605_26289_b200 import config as C
    C.SHAPES["tiny1"] = dataclasses.replace(C.SHAPES["tiny"], name="tiny1", layers=1)
    if layers == 1:
        cfg = cfg.with_overrides(model="tiny1")
    kv = UnifiedKvCache(cfg.capacity_cells)
    eng = GpuEngine(cfg, kv, n_seqs=4)
    w = eng.weights_cpu()
    g = torch.Generator().manual_seed(5)
    prompt = torch.randint(0, cfg.shape.vocab, (300,), generator=g).tolist()
    for T in (1, 2, 17, 64, 300):
        kv2 = kv
        eng.load_prompt(1, prompt[:T], 0, 0xCBF29CE484222325)
        kv.release_sequence(1)
        kv.append_cells(1, T)
        eng.run([EntryRequest(_lib.ENTRY_PREFILL, 1, 0, prompt[:T], prompt[:T])])
        gpu = eng.logits[:1].cpu()
        ref = llama_ref.forward(w, cfg.shape, prompt[:T], out_rows=[T - 1])
        print(f"layers={layers} T={T} max|gpu-ref|={(gpu-ref).abs().max().item():.5f} "
              f"ref_std={ref.std().item():.3f} ref_absmax={ref.abs().max().item():.3f}")
