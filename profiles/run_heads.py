"""576 GPT-2 S per-head slices (768 x 64 bf16) through the small path, a few calls (for ncu)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2505_16932_b200 as pe
hs = [(torch.randn((768, 64), device="cuda") * 0.02).bfloat16() for _ in range(576)]
ys = [torch.empty_like(h) for h in hs]
ctx = pe.Context(0)
for _ in range(2):
    ctx.polar(hs, ys, iters=5)
torch.cuda.synchronize()
print("ok")
