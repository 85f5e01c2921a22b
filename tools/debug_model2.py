"""Debug: compare layer-0 intermediates (1-layer tiny model, T tokens) GPU vs oracle."""
import sys, os, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import llama_ref as R
from paper_2605_26289_b200 import _lib, config as C
from paper_2605_26289_b200.config import CoreConfig
from paper_2605_26289_b200.engine import EntryRequest, GpuEngine
from paper_2605_26289_b200.kvcache import UnifiedKvCache

C.SHAPES["tiny1"] = dataclasses.replace(C.SHAPES["tiny"], name="tiny1", layers=1)
cfg = CoreConfig(model="tiny1", token_policy="argmax", capacity_cells=4096)
s = cfg.shape
kv = UnifiedKvCache(cfg.capacity_cells)
eng = GpuEngine(cfg, kv, n_seqs=4)
w = eng.weights_cpu()
T = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = torch.Generator().manual_seed(5)
prompt = torch.randint(0, s.vocab, (T,), generator=g).tolist()
eng.load_prompt(1, prompt, 0, 0xCBF29CE484222325)
kv.append_cells(1, T)
eng.run([EntryRequest(_lib.ENTRY_PREFILL, 1, 0, prompt, prompt)])
torch.cuda.synchronize()
ws = eng.workspace
base = (ws.data_ptr() + 255) // 256 * 256 - ws.data_ptr()
off = [base]
H, F, QKV, A = s.hidden, s.ffn, s.qkv_width, s.n_heads * s.head_dim
sizes = [T * H * 4, T * H * 2, T * QKV * 2, T * A * 2, T * 2 * F * 2, T * F * 2, 1 * H * 2]
names = ["x", "h", "qkv", "attn", "gu", "act", "hf"]
bufs = {}
for n, sz in zip(names, sizes):
    o = off[-1]
    bufs[n] = ws[o:o + sz].view(torch.float32 if n == "x" else torch.bfloat16).float().cpu()
    off.append(o + (sz + 255) // 256 * 256)
# oracle step by step
_bf = R._bf
x = w["embed"][torch.tensor(prompt)]
h = R.rmsnorm(x, w["attn_norm"][0], s.rms_eps)
qkv = _bf(h @ w["wqkv"][0].T)
nh, nkv, d = s.n_heads, s.n_kv_heads, s.head_dim
cos, sin = R.rope_tables(T, d, s.rope_theta)
q = R.rope(qkv[:, :nh*d].view(T, nh, d), cos, sin)
k = R.rope(qkv[:, nh*d:(nh+nkv)*d].view(T, nkv, d), cos, sin)
v = qkv[:, (nh+nkv)*d:].view(T, nkv, d)
qkv_r = torch.cat([q.reshape(T, -1), k.reshape(T, -1), v.reshape(T, -1)], 1)
o = _bf(R.paged_attention(q, k, v, list(range(T)), T, 1/d**0.5).reshape(T, -1))
x1 = x + o @ w["wo"][0].T
h2 = R.rmsnorm(x1, w["mlp_norm"][0], s.rms_eps)
gu = _bf(h2 @ w["w_gate_up"][0].T)
act = _bf(torch.nn.functional.silu(gu[:, :F]) * gu[:, F:])
x2 = x1 + act @ w["w_down"][0].T
hf = R.rmsnorm(x2[-1:], w["final_norm"], s.rms_eps)
ref = {"x": x2, "h": h2, "qkv": qkv_r, "attn": o, "gu": gu, "act": act, "hf": hf}
for n in names:
    a, b = bufs[n].view_as(ref[n]), ref[n]
    diff = (a - b).abs()
    print(f"{n:5s} maxdiff={diff.max().item():.5f} frac_mismatch={(diff > 0).float().mean().item():.4f} absmax={b.abs().max().item():.3f}")
# GEMM-only check with GPU inputs: qkv = bf16(h_gpu @ Wqkv^T)
hq = _bf(bufs["h"].view(T, H) @ w["w_gate_up"][0].T)
print("gu from gpu h:", (hq - bufs["gu"].view(T, -1)).abs().max().item())
