"""Debug: tiny-model prefill + decodes, checking logits per step against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import llama_ref
from paper_2605_26289_b200 import _lib
from paper_2605_26289_b200.config import CoreConfig
from paper_2605_26289_b200.engine import EntryRequest, GpuEngine
from paper_2605_26289_b200.kvcache import UnifiedKvCache

cfg = CoreConfig(model="tiny", token_policy="argmax", capacity_cells=4096)
kv = UnifiedKvCache(cfg.capacity_cells)
eng = GpuEngine(cfg, kv, n_seqs=4)
w = eng.weights_cpu()
g = torch.Generator().manual_seed(5)
prompt = torch.randint(0, cfg.shape.vocab, (300,), generator=g).tolist()
seq = 1
kv.append_cells(3, 17)
eng.load_prompt(seq, prompt, 0, 0xCBF29CE484222325)
kv.append_cells(seq, 200)
kv.release_sequence(3)
kv.append_cells(seq, 100)
res = eng.run([EntryRequest(_lib.ENTRY_PREFILL, seq, 0, prompt, prompt)])
toks = list(prompt)
ref = llama_ref.forward(w, cfg.shape, toks, out_rows=[len(toks) - 1])
print("prefill err", (eng.logits[:1].cpu() - ref).abs().max().item(), res[0].argmax_id)
toks.append(res[0].argmax_id)
for i in range(2):
    kv.append_cells(seq, 1)
    r = eng.run([EntryRequest(_lib.ENTRY_DECODE, seq, len(toks) - 1, [toks[-1]], toks)])
    lg = eng.logits[:1].cpu()
    ref = llama_ref.forward(w, cfg.shape, toks, out_rows=[len(toks) - 1])
    print("decode", i, "finite", torch.isfinite(lg).all().item(), "err", (lg - ref).abs().max().item(), r[0].argmax_id)
    toks.append(r[0].argmax_id)
