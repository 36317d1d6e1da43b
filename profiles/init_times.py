"""Cost of App. G's spectrum-aware first step (pe_set_spectrum_init):
device time per layer-set call with and without it (T = 5 in both; the step
adds one Gram + poly + update and `q` power-method passes over A_0)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2505_16932_b200 as pe
import pe_synth as syn
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for wl in sys.argv[1:] or ["gpt2-small", "gpt2-large"]:
    shapes = syn.layer_set_shapes(wl)
    xs = [(torch.randn(s, device="cuda") * 0.02).to(torch.bfloat16) for s in shapes]
    ys = [torch.empty_like(x) for x in xs]
    ctx = pe.Context(0)
    for q in (0, 2, 8):
        ctx.set_spectrum_init(q)
        for _ in range(3):
            flush.zero_()
            ctx.polar(xs, ys)
        ts = []
        for _ in range(5):
            flush.zero_()
            ctx.polar(xs, ys)               # pre-roll (no idle gap before the timed call)
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ctx.polar(xs, ys)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        print(f"{wl} power_iters={q}: {ts[2]:.3f} ms per call (median of 5)", flush=True)
    ctx.close()
    del xs, ys
    torch.cuda.empty_cache()
