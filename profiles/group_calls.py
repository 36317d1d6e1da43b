"""L2 locality probe: the GPT-2 S set as G consecutive pe_polar calls of
72/G matrices each (every call runs all T iterations of its group) vs one
call.  Device time per set, L2 flushed before each set."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2505_16932_b200 as pe
import pe_synth as syn
shapes = syn.layer_set_shapes("gpt2-small")
xs = [(torch.randn(s, device="cuda") * 0.02).to(torch.bfloat16) for s in shapes]
ys = [torch.empty_like(x) for x in xs]
ctx = pe.Context(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for G in [1, 2, 3, 4, 6]:
    n = len(shapes) // G
    groups = [(xs[g * n:(g + 1) * n], ys[g * n:(g + 1) * n]) for g in range(G)]
    for _ in range(3):
        flush.zero_()
        for a, b in groups:
            ctx.polar(a, b)
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for a, b in groups:
            ctx.polar(a, b)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"G={G} ({n} matrices per call): median {ts[5]:.4f} ms  min {ts[0]:.4f}", flush=True)
