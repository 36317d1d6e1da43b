"""NEXT row 4 (Muon-step fusion): device time of one Muon step over a layer
set with pe_muon_step (momentum in the norm pass, W update in the last
epilogue) vs the unfused composition (torch momentum update, pe_polar,
torch W update).  CUDA events, 3 warm-ups, median of 10, L2 flushed (256 MiB
write) before every step.  Usage: python profiles/muon_times.py [workload]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_16932_b200 as pe  # noqa: E402
import pe_synth as syn  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "gpt2-small"
shapes = syn.layer_set_shapes(wl)
gen = torch.Generator(device="cuda")
gen.manual_seed(0)
mk = lambda s: (torch.randn(s, generator=gen, device="cuda") * 0.02).to(torch.bfloat16)  # noqa: E731
W = [mk(s) for s in shapes]
M = [mk(s) for s in shapes]
G = [mk(s) for s in shapes]
X = [torch.empty_like(w) for w in W]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ctx = pe.Context(0)
beta, lr = 0.9, 0.02


def fused():
    ctx.muon_step(W, M, G, beta=beta, lr=lr, iters=5)


def unfused():
    torch._foreach_mul_(M, beta)
    torch._foreach_add_(M, G, alpha=1 - beta)
    ctx.polar(M, X, iters=5)
    torch._foreach_add_(W, X, alpha=-lr)


def timeit(fn):
    for _ in range(3):
        fn()
    ms = []
    for _ in range(10):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return statistics.median(ms)


f, u = timeit(fused), timeit(unfused)
print(f"{wl}: pe_muon_step {f:.3f} ms, unfused (torch momentum + pe_polar + torch W update) {u:.3f} ms, "
      f"saved {u - f:.3f} ms ({(u - f) / u * 100:.1f} %)")
