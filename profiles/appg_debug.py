"""App. G debug probe: the first case of the random-spikes fuzz test and
variants (orientation, folded / explicit X_0, T = 0..5) against the oracle's
exact step.  Usage: python profiles/appg_debug.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_16932_b200 as pe  # noqa: E402
import pe_synth as syn  # noqa: E402
from oracle import coeffs as oc, iteration as oi, metrics as om  # noqa: E402

TABLE, _ = oc.pe_coeffs(1e-3, 5, 8, 1.01)


def spiked(rows, cols, seed, top=1.0, tail=(0.05, 1e-2)):
    rng = np.random.default_rng(seed)
    k = min(rows, cols)
    U, _ = np.linalg.qr(rng.standard_normal((rows, k)))
    V, _ = np.linalg.qr(rng.standard_normal((cols, k)))
    s = np.concatenate([[top], np.geomspace(tail[0], tail[1], k - 1)])
    return (U * s) @ V.T * 0.01


def dev(M):
    bits = syn.f32_to_bf16_bits(np.asarray(M, dtype=np.float32))
    return torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).cuda()


def main():
    rng = np.random.default_rng(777)
    r, cc = int(rng.integers(8, 701)), int(rng.integers(8, 701))
    T, q = int(rng.integers(4, 8)), int(rng.integers(2, 13))
    rng.random()
    tail = tuple(sorted(rng.uniform(1e-4, 0.3, 2))[::-1])
    print("case", r, cc, T, q, tail, flush=True)
    c = pe.Context(0)
    for shape in ((r, cc), (cc, r), (r, 432), (432, r), (640, 432)):
        M = syn.to_bf16_values(spiked(*shape, seed=8000, tail=tail)).astype(np.float64)
        P = oi.exact_polar(M)
        for TT in (1, 2, 5):
            c.set_spectrum_init(q)
            X = c.polar([dev(M)], iters=TT)[0].float().cpu().numpy().astype(np.float64)
            c.set_spectrum_init(0)
            ref, z, ap = oi.polar_express_init(M, TABLE, TT, power_iters=q)
            print(shape, "T", TT, f"z {z:.6f} ap {ap} gpu-vs-ref {om.rel_frobenius(X, ref):.4f} "
                  f"truth gpu {om.rel_frobenius(X, P):.4f} ref {om.rel_frobenius(ref, P):.4f} "
                  f"|X|2 {np.linalg.norm(X, 2):.3f} |ref|2 {np.linalg.norm(ref, 2):.3f}", flush=True)
    c.close()


if __name__ == "__main__":
    main()
