"""Scale invariance probe (P:494 normalises by the Frobenius norm): the same
matrix at scales 1e-30 .. 1e30 through pe_polar (bf16 folded path, bf16
unfolded cols % 8 != 0, fp32) vs the result at scale 1."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2505_16932_b200 as pe
ctx = pe.Context(0)
torch.manual_seed(0)
for shape in [(256, 768), (256, 770)]:
    base = torch.randn(shape, device="cuda")
    for dt in (torch.bfloat16, torch.float32):
        ref = ctx.polar([base.to(dt)])[0].float()
        row = []
        for e in (-36, -30, -20, -15, -10, 10, 15, 20, 30, 36):
            x = (base * 10.0 ** e).to(dt)
            y = ctx.polar([x])[0].float()
            ok = bool(torch.isfinite(y).all())
            err = float((y - ref).norm() / ref.norm()) if ok else float("nan")
            row.append(f"1e{e}:{err:.1e}")
        print(shape, str(dt).split(".")[-1], " ".join(row), flush=True)
