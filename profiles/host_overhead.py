"""Host-side cost of one pe_polar call (enqueue only, no synchronisation)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2505_16932_b200 as pe
import pe_synth as syn
for wl in ("gpt2-small", "gpt2-large"):
    shapes = syn.layer_set_shapes(wl)
    xs = [(torch.randn(s, device="cuda") * 0.02).to(torch.bfloat16) for s in shapes]
    ys = [torch.empty_like(x) for x in xs]
    ctx = pe.Context(0)
    for _ in range(3):
        ctx.polar(xs, ys, iters=5)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); ctx.polar(xs, ys, iters=5); ts.append((time.perf_counter() - t0) * 1e3)
    torch.cuda.synchronize()
    print(wl, "host ms per call: min %.3f median %.3f" % (min(ts), sorted(ts)[5]))
    ctx.close()
