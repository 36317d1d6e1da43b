"""Small single matrices of BASELINE configs[4] (1024^2, 2048^2, 1024 x 4096):
device time per pe_polar call (CUDA events, median of 7 after 3 warm-ups)
and algorithmic TFLOP/s, for the current environment's knobs (run it with
PE_FUSED=0/1 to compare the phase-per-launch and the fused persistent
schedules).  Usage: python profiles/small_sweep.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_16932_b200 as pe  # noqa: E402


def main():
    ctx = pe.Context(0)
    tag = f"PE_FUSED={os.environ.get('PE_FUSED', '0')}"
    for shape in ((1024, 1024), (2048, 2048), (1024, 4096), (3072, 3072), (4096, 4096)):
        x = (torch.randn(shape, device="cuda") * 0.02).to(torch.bfloat16)
        y = torch.empty_like(x)
        for _ in range(3):
            ctx.polar([x], [y], iters=5)
        torch.cuda.synchronize()
        ms = []
        for _ in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ctx.polar([x], [y], iters=5)
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        t = statistics.median(ms)
        f = pe.pe_flops([shape], 5)
        print(f"{tag} {shape}: {t * 1e3:.1f} us  {f / t / 1e9:.1f} TFLOP/s", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
