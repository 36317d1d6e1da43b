"""Pins of the bf16 design's App. G step emulation (oracle.emulate.
r17_init_polar_express, reading R17) and of the exact
power-of-two prescale the GPU applies to bf16 inputs that go through an
oriented copy (readings R8 / R18).  CPU only."""
import numpy as np
import pytest

import pe_synth as syn
from oracle import coeffs as oc
from oracle import emulate
from oracle import iteration as oi
from oracle import metrics as om
from oracle.iteration import schedule

TABLE, _ = oc.pe_coeffs(1e-3, 5, 8, 1.01)


def _spiked(rows, cols, seed, top, tail):
    rng = np.random.default_rng(seed)
    k = min(rows, cols)
    U, _ = np.linalg.qr(rng.standard_normal((rows, k)))
    V, _ = np.linalg.qr(rng.standard_normal((cols, k)))
    s = np.concatenate([[top], np.geomspace(tail[0], tail[1], k - 1)])
    return syn.to_bf16_values((U * s) @ V.T * 0.01).astype(np.float64)


@pytest.mark.parametrize("shape", [(48, 80), (80, 48), (33, 70)])
@pytest.mark.parametrize("folded", [True, False])
def test_r17_not_applied_is_the_plain_design(shape, folded):
    """z < 1/sqrt(2) (flat spectrum): the step is the identity
    (a, b) = (1, 0), so the emulation must equal r8_polar_express with an
    explicit X_0 = bf16(M inv) bit for bit (X_1 = bf16((1 M + 0) inv))."""
    M = syn.to_bf16_values(syn.gaussian(*shape, seed=5, std=0.02)).astype(np.float64)
    for T in (1, 3, 5):
        X, z, applied = emulate.r17_init_polar_express(M, TABLE, T, 8, folded=folded)
        assert not applied and z < 1 / np.sqrt(2)
        ref = emulate.r8_polar_express(M, TABLE, T, folded=False)
        assert np.array_equal(X.view(np.uint32), ref.view(np.uint32)), T


@pytest.mark.parametrize("folded", [True, False])
def test_r17_applied_tracks_the_exact_step(folded):
    """A spike over a moderate tail (App. G's case): z agrees with the fp64
    step's to 1e-5 when X_0 = M (the Gram is formed from the same bf16
    values; only its fp32 rounding differs), to 1e-4 with an explicit
    X_0 = bf16(M inv) (fp32 input: sigma_1 of the rounded X_0 over the norm
    of the unrounded one), and the result to bf16 level (2e-2 relF)."""
    M = _spiked(96, 160, 3, 1.0, (0.2, 0.01))
    for T in (2, 5):
        X, z, applied = emulate.r17_init_polar_express(M, TABLE, T, 8, folded=folded)
        ref, zr, ar = oi.polar_express_init(M, TABLE, T, power_iters=8)
        assert applied and ar and abs(z - zr) <= (1e-5 if folded else 1e-4)
        assert om.rel_frobenius(X.astype(np.float64), ref) <= 2e-2, T


def _r8_prescaled(M, T):
    """The folded design's arithmetic with X_0 = bf16(M 2^e) stored by a copy
    and the residual 1/s 2^-e applied in iteration 1 (2^e the power-of-two
    part of inv = fp32(1/s)), written out independently of r8_polar_express."""
    M = np.asarray(M, dtype=np.float32)
    tall = M.shape[0] > M.shape[1]
    X = (M.T if tall else M).copy()
    nrm = np.sqrt(float(np.sum(X.astype(np.float64) ** 2))) * 1.01 + 1e-7
    inv = np.float32(1.0 / nrm)
    m_, e = np.frexp(inv)                    # inv = m_ 2^e, m_ in [0.5, 1)
    p2 = np.float32(np.ldexp(1.0, int(e) - 1))
    r = np.float32(inv / p2)                 # in [1, 2), exact
    X = emulate._bf16(np.float32(X * p2))
    for it, tup in enumerate(schedule(TABLE, T)):
        a, b, c = (np.float32(v) for v in tup)
        acc = (X.astype(np.float64) @ X.T.astype(np.float64)).astype(np.float32)
        A = emulate._bf16(np.float32(acc * np.float32(r * r))) if it == 0 else emulate._bf16(acc)
        B = emulate._bf16(np.float32(b * A) + np.float32(c * (A.astype(np.float64) @ A.astype(np.float64)).astype(np.float32)))
        BX = (B.astype(np.float64) @ X.astype(np.float64)).astype(np.float32)
        Xn = np.float32(np.float32(a * X) + BX)
        X = emulate._bf16(np.float32(Xn * r)) if it == 0 else emulate._bf16(Xn)
    return X.T if tall else X


@pytest.mark.parametrize("scale", [1.0, 3e-5, 7e12])
def test_pow2_prescale_is_bit_identical_to_folding(scale):
    """Reading R8/R18: storing X_0 = M 2^e and applying 1/s 2^-e in iteration
    1 gives the folded path's result bit for bit -- every fp32 product, sum
    and rounding commutes with an exponent shift -- at any input scale whose
    values stay normal (diagonal inputs make the accumulations exact too, so
    the equality also holds on the GPU, test_diagonal_bit_exact)."""
    for shape in ((40, 70), (70, 40)):
        k = min(shape)
        sig = syn.to_bf16_values(np.linspace(1.0, 0.02, k) * scale).astype(np.float64)
        M = syn.diagonal(*shape, sig)
        for T in (1, 3):
            ref = emulate.r8_polar_express(M, TABLE, T, folded=True)
            got = _r8_prescaled(M, T)
            assert np.array_equal(ref.view(np.uint32), got.view(np.uint32)), (scale, shape, T)
        G = syn.to_bf16_values(syn.gaussian(*shape, seed=2, std=0.02) * scale).astype(np.float64)
        assert np.array_equal(emulate.r8_polar_express(G, TABLE, 2, folded=True).view(np.uint32),
                              _r8_prescaled(G, 2).view(np.uint32))


def test_r17_explicit_x0_keeps_the_lower_bound():
    """Reading R17 on the fp32-input path (X_0 = bf16(M inv) rounded): z and F
    come from the same fp32 Gram (trace(acc) = ||X_0||^2), so z stays a lower
    bound of sigma_1(X_0) / ||X_0||_F up to the fp32 Gram's own
    rounding.  Taking F from the unrounded ||M|| inv instead overshoots it by
    up to 1.3e-4 on these power laws (the planted variant below)."""
    rng = np.random.default_rng(5)
    over_fixed, over_planted = 0.0, 0.0
    for _ in range(24):
        r, c = int(rng.integers(32, 300)), int(rng.integers(32, 300))
        k = min(r, c)
        U, _ = np.linalg.qr(rng.standard_normal((r, k)))
        V, _ = np.linalg.qr(rng.standard_normal((c, k)))
        M = ((U * np.arange(1, k + 1) ** -rng.uniform(2, 6)) @ V.T * 0.01).astype(np.float32).astype(np.float64)
        X = (M.T if r > c else M).astype(np.float32)
        ssq = float(np.sum(X.astype(np.float64) ** 2))
        inv = np.float32(1.0 / (np.sqrt(ssq) * 1.01 + 1e-7))
        X0 = emulate._bf16(X * inv).astype(np.float64)
        s = np.linalg.svd(X0, compute_uv=False)
        z_true = s[0] / np.sqrt(np.sum(s * s))
        _, z, _ = emulate.r17_init_polar_express(M, TABLE, 1, 12, folded=False)
        over_fixed = max(over_fixed, z - z_true)
        # planted: the Rayleigh quotient of the rounded X_0's Gram over ||M||^2 inv^2
        lam = (z ** 2) * float(np.sum(np.diag((X0 @ X0.T).astype(np.float32)).astype(np.float64)))
        over_planted = max(over_planted, np.sqrt(lam / (ssq * float(inv) ** 2)) - z_true)
    assert over_fixed <= 2e-6, over_fixed
    assert over_planted > 1e-5, over_planted
