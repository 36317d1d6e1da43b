"""App. G margin probe (reading R17): the GPU's spectrum-aware step with
margin m (p / (1 + |b| m)) against the paper's exact step (oracle, no
margin) on the inputs the tests use.  Prints, per margin, finiteness,
||X||_2 and relF to polar(M) next to the oracle's.  Usage:
  python profiles/appg_margin.py"""
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


def spiked(rows, cols, seed, top=1.0, tail=(0.05, 1e-2), law=None):
    rng = np.random.default_rng(seed)
    k = min(rows, cols)
    U, _ = np.linalg.qr(rng.standard_normal((rows, k)))
    V, _ = np.linalg.qr(rng.standard_normal((cols, k)))
    s = np.arange(1, k + 1, dtype=np.float64) ** -law if law else np.concatenate([[top], np.geomspace(tail[0], tail[1], k - 1)])
    return (U * s) @ V.T * 0.01


def run(c, M, T):
    bits = syn.f32_to_bf16_bits(np.asarray(M, dtype=np.float32))
    x = torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).cuda()
    y = c.polar([x], iters=T)[0]
    torch.cuda.synchronize()
    return y.float().cpu().numpy().astype(np.float64)


def sweep_m():
    """Smallest safe margin per size: sigma_j = j^-5 (z ~ 0.9995, |b| ~ 30),
    margins k * 2^-7 / sqrt(m)."""
    c = pe.Context(0)
    for m in (8, 16, 32, 64, 128, 256, 512, 1024):
        for seed in (11, 12, 13):
            M = syn.to_bf16_values(spiked(m, 3 * m, seed, law=5.0)).astype(np.float64)
            P = oi.exact_polar(M)
            ref, z, applied = oi.polar_express_init(M, TABLE, 5, power_iters=8)
            line = [f"m={m} seed={seed} z={z:.6f} oracle {om.rel_frobenius(ref, P):.4f}"]
            for k in (0.0, 0.125, 0.25, 0.5, 1.0, 2.0):
                c.set_spectrum_init(8, k * 2.0 ** -7 / np.sqrt(m))
                X = run(c, M, 5)
                fin = np.all(np.isfinite(X)) and np.abs(X).max() < 1e3
                line.append(f"k={k}: " + (f"{om.rel_frobenius(X, P):.4f}" if fin else "DIVERGED"))
            print(" | ".join(line), flush=True)
    c.close()


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "sweep":
        return sweep_m()
    rng = np.random.default_rng(3)
    cases = [("32x32 j^-5", spiked(32, 32, 11, law=5.0), (4, 5)),
             ("256x512 j^-3", spiked(256, 512, 11, law=3.0), (4, 5)),
             ("1536x512 j^-5", spiked(1536, 512, 11, law=5.0), (4, 5)),
             ("256x1024 tail 3e-3..1e-3", spiked(256, 1024, 1280, tail=(3e-3, 1e-3)), (5, 6)),
             ("256x1024 tail 2e-3..2e-4", spiked(256, 1024, 1280, tail=(2e-3, 2e-4)), (5, 6)),
             ("200x520 rank one", np.outer(rng.standard_normal(200), rng.standard_normal(520)) * 0.01, (5,))]
    c = pe.Context(0)
    for name, M, Ts in cases:
        M = syn.to_bf16_values(M).astype(np.float64)
        P = oi.exact_polar(M)
        for T in Ts:
            ref, z, applied = oi.polar_express_init(M, TABLE, T, power_iters=8)
            line = [f"{name} T={T} z={z:.6f} oracle {om.rel_frobenius(ref, P):.4f}"]
            for m in (2.0 ** -7, 2.0 ** -8, 2.0 ** -9, 2.0 ** -11, 0.0):
                c.set_spectrum_init(8, m)
                X = run(c, M, T)
                fin = np.all(np.isfinite(X))
                nrm = np.linalg.norm(X, 2) if fin else float("nan")
                e = om.rel_frobenius(X, P) if fin else float("nan")
                line.append(f"m={m:.2e}: {e:.4f} |X|={nrm:.3f} vsref {om.rel_frobenius(X, ref) if fin else float('nan'):.4f}")
            print(" | ".join(line), flush=True)
    c.close()


if __name__ == "__main__":
    main()
