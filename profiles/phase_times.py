"""Per-phase device times of pe_polar on a layer set (profiling ABI), for
kernel experiments.  Usage: python profiles/phase_times.py <workload> [calls]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_16932_b200 as pe  # noqa: E402
import pe_synth as syn  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "gpt2-small"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 5
shapes = syn.layer_set_shapes(wl)
g = torch.Generator(device="cuda")
xs = []
for i, (r, c) in enumerate(shapes):
    g.manual_seed(i)
    xs.append((torch.randn((r, c), generator=g, device="cuda") * 0.02).to(torch.bfloat16))
ys = [torch.empty_like(x) for x in xs]
ctx = pe.Context(0)
for _ in range(3):
    ctx.polar(xs, ys, iters=5)
torch.cuda.synchronize()
ctx.profile_enable(True)
for _ in range(calls):
    ctx.polar(xs, ys, iters=5)
torch.cuda.synchronize()
prof = ctx.profile_read()
tag = os.environ.get("PE_DEBUG_GEMM", "0") + "/" + os.environ.get("PE_FUSED", "0")
print(wl, tag, " ".join(f"{k}={v[0] / max(v[1], 1) * 1e3:.1f}us" for k, v in prof.items() if v[1]))
