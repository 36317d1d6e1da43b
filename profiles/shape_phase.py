"""Per-phase device times of pe_polar on single matrices (profiling ABI).
Usage: python profiles/shape_phase.py RxC [RxC ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_16932_b200 as pe  # noqa: E402

ctx = pe.Context(0)
for arg in sys.argv[1:]:
    r, c = (int(v) for v in arg.split("x"))
    x = (torch.randn((r, c), device="cuda") * 0.02).to(torch.bfloat16)
    y = torch.empty_like(x)
    for _ in range(2):
        ctx.polar([x], [y], iters=5)
    torch.cuda.synchronize()
    ctx.profile_enable(True)
    n = 3
    for _ in range(n):
        ctx.polar([x], [y], iters=5)
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    fl = pe.pe_flops([(r, c)], 5)
    tot = sum(v[0] for v in prof.values()) / n
    print(f"{arg}: " + " ".join(f"{k}={v[0] / max(v[1], 1) * 1e3:.1f}us" for k, v in prof.items() if v[1])
          + f" | call {tot:.3f} ms, {fl / (tot * 1e-3) / 1e12:.0f} TF/s", flush=True)
    del x, y
    torch.cuda.empty_cache()
