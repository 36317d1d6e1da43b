"""fp32 (three-plane tensor-core path) vs bf16 device time per pe_polar call, T=5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2505_16932_b200 as pe, statistics  # noqa: E402
ctx=pe.Context(0)
for (r,c) in [(128,128),(1024,1024),(4096,4096),(768,3072),(4096,16384)]:
    x=(torch.randn(r,c,device="cuda")*0.02)
    for dt in ("f32","bf16"):
        xx = x if dt=="f32" else x.bfloat16()
        y=torch.empty_like(xx)
        for _ in range(2): ctx.polar([xx],[y],iters=5)
        torch.cuda.synchronize(); ms=[]
        for _ in range(5):
            a,b=torch.cuda.Event(True),torch.cuda.Event(True); a.record(); ctx.polar([xx],[y],iters=5); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
        m=statistics.median(ms); tf=pe.pe_flops([(r,c)],5)/(m*1e-3)/1e12
        print(f"{r}x{c} {dt} {m:.3f} ms {tf:.1f} TF/s")
