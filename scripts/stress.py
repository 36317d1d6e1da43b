"""Randomised cross-feature stress run against the fp64 oracle (not part of the
test suite; seeds other than the tests').  Each call draws a batch of shapes
and a feature mix -- bf16 / fp32 / pe_polar_ex, T, App. G step, Alg. 4
restart, small-path planes, in place or not -- and checks every result with
the gates of tests/test_gpu_parity.py (G1 from the design's own spread when
that is wider, G3).  Usage: python scripts/stress.py <seed> <calls>"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_16932_b200 as pe  # noqa: E402
import pe_synth as syn  # noqa: E402
from oracle import alg4 as a4, coeffs as oc, emulate, iteration as oi, metrics as om  # noqa: E402

TABLE, _ = oc.pe_coeffs(1e-3, 5, 8, 1.01)


def g1_gate(m):
    return 2e-2 if m >= 128 else (2.5e-2 if m >= 64 else (4e-2 if m >= 16 else 1e-1))


def dev_bf16(M):
    bits = syn.f32_to_bf16_bits(np.asarray(M, dtype=np.float32))
    return torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).cuda()


def main():
    seed, calls = int(sys.argv[1]), int(sys.argv[2])
    rng = np.random.default_rng(seed)
    c = pe.Context(0)
    fails = 0
    for call in range(calls):
        T = int(rng.integers(1, 9))
        kind = rng.choice(["bf16", "bf16", "fp32", "ex"])
        rect = int(rng.choice([0, 0, 2, 3])) if kind == "bf16" else 0
        planes = int(rng.choice([1, 2])) if kind == "bf16" else 1
        inplace = bool(rng.random() < 0.3) and kind != "ex"
        c.set_rect_iteration(rect, 0.0, 1e-3)
        c.set_small_planes(planes)
        shapes = []
        for _ in range(int(rng.integers(1, 5))):
            r = int(rng.choice([1, 7, 8, 64, 100, 128, 129, 200, 256, 300, 511, 700]))
            cc = int(r * rng.uniform(0.3, 5.0)) + 1
            if kind == "fp32":
                r, cc = min(r, 400), min(cc, 400)
            shapes.append((r, cc) if rng.random() < 0.5 else (cc, r))
        mats = [syn.gaussian(r, cc, seed=90000 + 100 * call + i, std=0.02) for i, (r, cc) in enumerate(shapes)]
        if kind == "fp32":
            mats = [M.astype(np.float32).astype(np.float64) for M in mats]
            xs = [torch.from_numpy(M.astype(np.float32)).cuda() for M in mats]
        elif kind == "ex":
            mats = [M.astype(np.float32).astype(np.float64) for M in mats]
            xs = [torch.from_numpy(M.astype(np.float32)).cuda() for M in mats]
        else:
            mats = [syn.to_bf16_values(M).astype(np.float64) for M in mats]
            xs = [dev_bf16(M) for M in mats]
        if kind == "ex":
            ys = c.polar_ex(xs, [torch.empty(x.shape, dtype=torch.bfloat16, device="cuda") for x in xs], iters=T)
        elif inplace:
            ys = c.polar(xs, xs, iters=T)
        else:
            ys = c.polar(xs, iters=T)
        torch.cuda.synchronize()
        small = all(min(s) <= 128 and -(-max(s) // 64) * 64 <= (640 if planes == 2 else 768) for s in shapes)
        for y, M, s in zip(ys, mats, shapes):
            X = y.float().cpu().numpy().astype(np.float64)
            m, n = min(s), max(s)
            P = oi.exact_polar(M)
            use_rect = rect > 0 and m > 128 and T > 1 and n > 1.5 * T / (T - 1) * m
            if use_rect:
                ref = a4.alg4(M, TABLE, T, restart=rect, shift=1e-3)
                emu = emulate.r19_alg4(M, TABLE, T, restart=rect, shift=1e-3, folded=True)
            else:
                ref = oi.polar_express(M, TABLE, T)
                emu = emulate.r8_polar_express(M, TABLE, T, folded=kind == "bf16",
                                               ab_planes=2 if (planes == 2 and small and kind == "bf16") else 1)
            emu = emu.astype(np.float64)
            e_ref = om.rel_frobenius(ref, P)
            err = om.rel_frobenius(X, ref)
            if kind == "fp32":
                ok = err <= (1e-4 if m == 1 else 1e-5)
                g = 1e-5
            else:
                e_emu = om.rel_frobenius(emu, ref)
                g = max(5e-2 if m == 1 else g1_gate(m), 1.5 * e_emu + 2e-3, 1e-1 if use_rect else 0.0)
                g3 = max(1e-2, 1.5 * (om.rel_frobenius(emu, P) - e_ref) + 2e-3)
                ok = np.all(np.isfinite(X)) and err <= g and om.rel_frobenius(X, P) <= e_ref + g3
            if not ok:
                fails += 1
                print(f"FAIL call {call} kind {kind} T {T} rect {rect} planes {planes} inplace {inplace} "
                      f"shape {s}: relF {err:.4g} gate {g:.3g} truth {om.rel_frobenius(X, P):.4g} vs {e_ref:.4g}",
                      flush=True)
    print(f"seed {seed}: {calls} calls, {fails} failures", flush=True)
    c.close()


if __name__ == "__main__":
    main()
