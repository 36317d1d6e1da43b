"""NEXT row 3 (small-matrix fused path): device time per pe_polar call for small
matrices, small path vs the large path (PE_SMALL=0), T = 1, 2, 5.  The GPU is
kept busy (torch.cuda._sleep) before the start event so host submission is
not timed.  Usage: python profiles/small_times.py; PE_SMALL=0 python profiles/small_times.py"""
import sys, statistics
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch, paper_2505_16932_b200 as pe
ctx = pe.Context(0)
import os
if os.environ.get("PE_SMALL_PLANES"):
    ctx.set_small_planes(int(os.environ["PE_SMALL_PLANES"]))
for dt in (torch.float32, torch.bfloat16):
    for shape in [(128, 128), (64, 64), (128, 512)]:
        x = (torch.randn(shape, device="cuda") * 0.02).to(dt)
        y = torch.empty_like(x)
        res = []
        for T in (1, 2, 5):
            for _ in range(3): ctx.polar([x], [y], iters=T)
            torch.cuda.synchronize(); ms = []
            for _ in range(20):
                a, b = torch.cuda.Event(True), torch.cuda.Event(True)
                torch.cuda._sleep(2000000); a.record(); ctx.polar([x], [y], iters=T); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
            res.append(statistics.median(ms) * 1e3)
        print(dt, shape, " ".join(f"T={T}:{v:.1f}us" for T, v in zip((1, 2, 5), res)), flush=True)

# per-head Muon slices: GPT-2 Small attention q, k, v, o split
# into 12 heads each (768 x 64), 12 layers -> 576 matrices in one call
hs = [(torch.randn((768, 64), device="cuda") * 0.02).bfloat16() for _ in range(576)]
ho = [torch.empty_like(h) for h in hs]
for _ in range(3):
    ctx.polar(hs, ho, iters=5)
torch.cuda.synchronize()
ms = []
for _ in range(10):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda._sleep(2000000); a.record(); ctx.polar(hs, ho, iters=5); b.record(); torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
m = statistics.median(ms)
print(f"per-head GPT-2 S attention slices (576 x 768x64 bf16), T=5: {m * 1e3:.1f} us, "
      f"{pe.pe_flops([(768, 64)] * 576, 5) / (m * 1e-3) / 1e12:.1f} TF/s", flush=True)
