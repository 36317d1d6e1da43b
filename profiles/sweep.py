"""BASELINE.json configs[4]: square sweep 1024-16384 and aspect ratios 1:1-1:8
(both orientations), bf16 vs fp32, iterations 3-8.  Device time per pe_polar
call (CUDA events, 3 warm-ups, median of 5), algorithmic TFLOP/s (pe_flops).
Usage: python profiles/sweep.py > profiles/r1_sweep.md"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_16932_b200 as pe  # noqa: E402


def time_call(ctx, xs, T, reps=5, warm=3):
    ys = [torch.empty_like(x) for x in xs]
    for _ in range(warm):
        ctx.polar(xs, ys, iters=T)
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ctx.polar(xs, ys, iters=T)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return statistics.median(ms)


def main():
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    ctx = pe.Context(0)
    rows = []
    cases = [((n, n), "square") for n in (1024, 2048, 4096, 8192, 16384)]
    cases += [((4096, n), "aspect wide") for n in (8192, 16384, 32768)]
    cases += [((n, 4096), "aspect tall") for n in (8192, 16384, 32768)]
    for (r, c), kind in cases:
        for dt in ("bf16", "fp32"):
            torch.manual_seed(0)
            x = torch.randn((r, c), device="cuda") * 0.02
            x = x.to(torch.bfloat16) if dt == "bf16" else x
            Ts = (3, 4, 5, 6, 7, 8) if (dt == "bf16" and (r, c) == (4096, 4096)) else (5,)
            for T in Ts:
                ms = time_call(ctx, [x], T, reps=3 if dt == "fp32" else 5, warm=1 if dt == "fp32" else 3)
                tf = pe.pe_flops([(r, c)], T) / (ms * 1e-3) / 1e12
                rows.append((f"{r}x{c}", kind, dt, T, ms, tf))
            del x
            torch.cuda.empty_cache()
    ctx.close()
    print("# Sweep (BASELINE configs[4]) -- one matrix per pe_polar call, device time\n")
    print(f"bf16 fraction against {peaks['bf16_tflops']} TFLOP/s (measured burst); fp32 runs six bf16 "
          "plane products per product (three-plane split), so its algorithmic rate is at most 1/6 of the bf16 one.\n")
    print("| shape | kind | dtype | T | ms / call | TFLOP/s (algorithmic) | frac of bf16 peak |")
    print("|---|---|---|---|---|---|---|")
    for shape, kind, dt, T, ms, tf in rows:
        print(f"| {shape} | {kind} | {dt} | {T} | {ms:.3f} | {tf:.1f} | {tf / peaks['bf16_tflops']:.3f} |")


if __name__ == "__main__":
    main()
