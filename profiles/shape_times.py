"""Per-phase device times for one or more explicit shapes (profiling ABI).
Usage: python profiles/shape_times.py 4096x8192 [8192x4096 ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_16932_b200 as pe  # noqa: E402

ctx = pe.Context(0)
for arg in sys.argv[1:]:
    shapes = [tuple(int(v) for v in a.split("x")) for a in arg.split(",")]
    xs = [(torch.randn(s, device="cuda") * 0.02).to(torch.bfloat16) for s in shapes]
    ys = [torch.empty_like(x) for x in xs]
    for _ in range(3):
        ctx.polar(xs, ys, iters=5)
    torch.cuda.synchronize()
    ctx.profile_enable(True)
    for _ in range(5):
        ctx.polar(xs, ys, iters=5)
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    fl = pe.pe_flops(shapes, 5)
    tot = sum(v[0] for v in prof.values()) / 5
    print(arg, f"total={tot:.3f}ms TF/s={fl / (tot * 1e-3) / 1e12:.0f}",
          " ".join(f"{k}={v[0] / max(v[1], 1) * 1e3:.1f}us" for k, v in prof.items() if v[1]))
