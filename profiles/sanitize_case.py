"""Small mixed batch (wide, tall, ragged, degenerate) for compute-sanitizer."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2505_16932_b200 as pe
shapes = [(256, 512), (512, 256), (200, 520), (37, 100), (64, 1), (300, 1100)]
xs = [(torch.randn(s, device="cuda") * 0.02).to(torch.bfloat16) for s in shapes]
ctx = pe.Context(0)
ys = ctx.polar(xs, iters=3)
xf = [torch.randn(128, 128, device="cuda")]
yf = ctx.polar(xf, iters=3)
torch.cuda.synchronize()
print("ok", [bool(torch.isfinite(y.float()).all()) for y in ys + yf])
