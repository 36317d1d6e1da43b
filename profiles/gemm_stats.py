"""Wait-cycle breakdown of the GEMM phases (PE_DEBUG_GEMM=4): per CTA, MMA
warp total cycles / waiting for a free accumulator (epilogue-bound) /
waiting for operands (load-bound), epilogue warp waiting for the MMA.
Usage: PE_DEBUG_GEMM=4 python profiles/gemm_stats.py <workload>"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_16932_b200 as pe  # noqa: E402
import pe_synth as syn  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "gpt2-small"
shapes = syn.layer_set_shapes(wl)
xs = [(torch.randn((r, c), device="cuda") * 0.02).to(torch.bfloat16) for r, c in shapes]
ys = [torch.empty_like(x) for x in xs]
ctx = pe.Context(0)
for _ in range(2):
    ctx.polar(xs, ys, iters=5)
torch.cuda.synchronize()
L = pe.lib()
L.pe_debug_stats.restype = ctypes.c_int
buf = (ctypes.c_longlong * (8 * 1024))()
assert L.pe_debug_stats(ctx._h, buf) == 0
a = np.array(buf[:6144], dtype=np.int64).reshape(3, 256, 8)
for mode, name in enumerate(["gram", "poly", "update"]):
    lead = a[mode, 0:148:2]          # leader CTAs
    tot = lead[:, 0].astype(float)
    print(f"{wl} {os.environ.get('PE_FUSED','0')} {name}: total {tot.mean()/1e3:.1f}k cyc, "
          f"MMA waits tempty {100*lead[:,1].mean()/tot.mean():.1f}%, waits full {100*lead[:,2].mean()/tot.mean():.1f}%, "
          f"epi waits tfull {100*lead[:,3].mean()/tot.mean():.1f}%  (min/max total {tot.min()/1e3:.0f}k/{tot.max()/1e3:.0f}k)"
          f"  issue->full latency {lead[:,4].sum()/max(lead[:,5].sum(),1):.0f} cyc/stage over {lead[:,5].sum()/74:.0f} stages/CTA")
