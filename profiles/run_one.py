"""Run pe_polar on a (sub)layer set a few times -- a short command for ncu.
Usage: python profiles/run_one.py <workload> [layers] [calls] [T]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2505_16932_b200 as pe  # noqa: E402
import pe_synth as syn  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    calls = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    T = int(sys.argv[4]) if len(sys.argv) > 4 else 5
    shapes = syn.layer_set_shapes(wl, layers=layers)
    g = torch.Generator(device="cuda")
    xs = []
    for i, (r, c) in enumerate(shapes):
        g.manual_seed(i)
        xs.append((torch.randn((r, c), generator=g, device="cuda") * 0.02).to(torch.bfloat16))
    ctx = pe.Context(0)
    if os.environ.get("PE_RUN_RECT"):            # App. H Alg. 4 with this restart interval
        ctx.set_rect_iteration(int(os.environ["PE_RUN_RECT"]), 0.0, 1e-3)
    ys = [torch.empty_like(x) for x in xs]
    for _ in range(calls):
        ctx.polar(xs, ys, iters=T)
    torch.cuda.synchronize()
    print("ok", wl, layers, len(shapes), "launches/call", ctx.last_launch_count())


if __name__ == "__main__":
    main()
