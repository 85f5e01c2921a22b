"""Noise floor of bf16-storage numerics: the oracle against itself (fp32 vs fp64 accumulation)."""
import sys; import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, copy
from oracle import llama_ref as R
from paper_2605_26289_b200.config import SHAPES
s = SHAPES["tiny"]
g = torch.Generator().manual_seed(0)
def rn(*sh): return (torch.randn(*sh, generator=g)*0.02).bfloat16().float()
w = {"embed": rn(s.vocab, s.hidden), "attn_norm": torch.ones(s.layers, s.hidden), "wqkv": rn(s.layers, s.qkv_width, s.hidden),
     "wo": rn(s.layers, s.hidden, s.n_heads*s.head_dim), "mlp_norm": torch.ones(s.layers, s.hidden),
     "w_gate_up": rn(s.layers, 2*s.ffn, s.hidden), "w_down": rn(s.layers, s.hidden, s.ffn), "final_norm": torch.ones(s.hidden), "lm_head": rn(s.vocab, s.hidden)}
toks = torch.randint(0, s.vocab, (64,), generator=g).tolist()
a = R.forward(w, s, toks, out_rows=[63])
# same math in float64 (different rounding of accumulations, same bf16 storage points)
w64 = {k: v.double() for k, v in w.items()}
orig_bf = R._bf
R._bf = lambda x: x.to(torch.bfloat16).to(x.dtype)
b = R.forward(w64, s, toks, out_rows=[63]).float()
print("fp32 vs fp64-accum oracle: max abs", (a-b).abs().max().item(), "rel rms", ((a-b).norm()/b.norm()).item())
