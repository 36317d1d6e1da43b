"""Device time per pe_polar call: direct launches vs one CUDA-graph replay of
the same call (after pe_reserve).  CUDA events, 3 warm-ups, median of 20, L2
flushed before each call.  Usage: python profiles/graph_times.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_16932_b200 as pe  # noqa: E402
import pe_synth as syn  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ctx = pe.Context(0)


def timeit(fn):
    for _ in range(3):
        fn()
    ms = []
    for _ in range(20):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return statistics.median(ms)


cases = [("config 1: 128x128 fp32", [(128, 128)], torch.float32),
         ("128x128 bf16", [(128, 128)], torch.bfloat16),
         ("GPT-2 Small set bf16", syn.layer_set_shapes("gpt2-small"), torch.bfloat16)]
for name, shapes, dt in cases:
    xs = [(torch.randn(s, device="cuda") * 0.02).to(dt) for s in shapes]
    ys = [torch.empty_like(x) for x in xs]
    ctx.reserve(shapes, pe.PE_FP32 if dt == torch.float32 else pe.PE_BF16)
    direct = timeit(lambda: ctx.polar(xs, ys, iters=5))
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        ctx.polar(xs, ys, iters=5)
    graph = timeit(g.replay)
    print(f"{name}: direct {direct * 1e3:.1f} us, graph replay {graph * 1e3:.1f} us")
