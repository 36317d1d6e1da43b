"""Alg. 4 debug probe: one fuzz case against the R19 emulation, alone and in
batches.  Usage: python profiles/alg4_debug.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_16932_b200 as pe  # noqa: E402
import pe_synth as syn  # noqa: E402
from oracle import alg4 as a4, coeffs as oc, emulate, metrics as om  # noqa: E402

TABLE, _ = oc.pe_coeffs(1e-3, 5, 8, 1.01)


def dev(M):
    bits = syn.f32_to_bf16_bits(np.asarray(M, dtype=np.float32))
    return torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).cuda()


def sweep():
    """gpu vs R19 emulation across shapes near the 128 / 256 boundaries."""
    c = pe.Context(0)
    for T, restart in ((2, 2), (3, 3), (2, 1)):
        c.set_rect_iteration(restart, 1.0, 0.0)
        for shape in ((129, 244), (129, 300), (136, 260), (160, 400), (192, 400), (250, 500), (255, 600),
                      (256, 600), (257, 600), (300, 700), (384, 900), (512, 1100), (130, 1000)):
            M = syn.to_bf16_values(syn.gaussian(*shape, seed=7, std=0.02)).astype(np.float64)
            X = c.polar([dev(M)], iters=T)[0].float().cpu().numpy().astype(np.float64)
            emu = emulate.r19_alg4(M, TABLE, T, restart=restart, shift=0.0,
                                   folded=True).astype(np.float64)
            print(f"T={T} r={restart} {shape}: gpu-vs-emu {om.rel_frobenius(X, emu):.4f}", flush=True)
    c.close()


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "sweep":
        return sweep()
    shapes = [(129, 244), (255, 448), (1907, 513)]
    mats = [syn.to_bf16_values(syn.gaussian(r, c, seed=50000 + i, std=0.02)).astype(np.float64)
            for i, (r, c) in enumerate(shapes)]
    T, restart, shift = 5, 5, 1e-3
    c = pe.Context(0)
    c.set_rect_iteration(restart, 0.0, shift)
    for name, idx in (("mixed", [0, 1, 2]), ("alone0", [0]), ("alone2", [2]), ("pair02", [0, 2])):
        ys = c.polar([dev(mats[i]) for i in idx], iters=T)
        torch.cuda.synchronize()
        for i, y in zip(idx, ys):
            X = y.float().cpu().numpy().astype(np.float64)
            M = mats[i]
            emu = emulate.r19_alg4(M, TABLE, T, restart=restart, shift=shift,
                                   folded=True).astype(np.float64)
            ref = a4.alg4(M, TABLE, T, restart=restart, shift=shift)
            print(name, M.shape, f"gpu-vs-emu {om.rel_frobenius(X, emu):.4f}  gpu-vs-oracle {om.rel_frobenius(X, ref):.4f}"
                  f"  emu-vs-oracle {om.rel_frobenius(emu, ref):.4f}", flush=True)
    # diagonal versions
    for shape in ((129, 244), (1907, 513), (244, 129)):
        k = min(shape)
        sig = syn.to_bf16_values(np.linspace(1.0, 0.05, k)).astype(np.float64)
        M = syn.diagonal(*shape, sig)
        y = c.polar([dev(M)], iters=T)[0]
        torch.cuda.synchronize()
        X = y.float().cpu().numpy().astype(np.float64)
        emu = emulate.r19_alg4(M, TABLE, T, restart=restart, shift=shift, folded=True)
        d = np.abs(X - emu)
        print("diag", shape, "max |gpu - emu|", d.max(), "at", np.unravel_index(np.argmax(d), d.shape), flush=True)
    c.close()


if __name__ == "__main__":
    main()
