"""Wall time of pe_polar_host on the GPT-2 Small set (pinned host tensors)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2505_16932_b200 as pe
import pe_synth as syn
shapes = syn.layer_set_shapes(sys.argv[1] if len(sys.argv) > 1 else "gpt2-small")
ctx = pe.Context(0)
hin = [(torch.randn(s) * 0.02).to(torch.bfloat16).pin_memory() for s in shapes]
hout = [torch.empty_like(h).pin_memory() for h in hin]
for _ in range(2):
    ctx.polar_host(hin, hout, iters=5)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); ctx.polar_host(hin, hout, iters=5); ts.append((time.perf_counter() - t0) * 1e3)
print(os.environ.get("PE_HOST_GROUPS", "auto"), "nocompute" if os.environ.get("PE_HOST_NOCOMPUTE") else "", f"{min(ts):.3f} ms (min of 5)", f"{sorted(ts)[2]:.3f} median")
