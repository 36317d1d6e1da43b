"""Evidence for the size-dependent bf16 gates of tests/test_gpu_parity.py
(DESIGN.md "Tolerances"): how far the bf16 design's own rounding points
(reading R8, ``oracle.emulate.r8_polar_express``: bf16 operands, exact
products, fp32 accumulation) land from the fp64 oracle, over seeds.

north_star's G1 (relF <= 2e-2) holds for this design from m = 128 (and for
most smaller shapes), but on a few small shapes some seeds exceed it with no
kernel involved at all -- there are too few singular values to average the
bf16 roundings of A, B and X' -- so the GPU gates below m = 128 are the
design's spread with headroom, not a property of the kernels.  The tests
assert both halves: the widened gate covers the design's worst seed, and
2e-2 alone would not (so the widening is needed, not slack).
"""
import numpy as np
import pytest

import pe_synth as syn
from oracle import coeffs as oc
from oracle import emulate, iteration as oi, metrics as om

TABLE, _ = oc.pe_coeffs(1e-3, 5, 8, 1.01)


def g1_gate(m):
    """Same as tests/test_gpu_parity.g1_gate."""
    return 2e-2 if m >= 128 else (2.5e-2 if m >= 64 else (4e-2 if m >= 16 else 1e-1))


def spread(shape, seeds, T=5, ab_planes=1):
    out = []
    for seed in seeds:
        M = syn.to_bf16_values(syn.gaussian(*shape, seed=seed, std=0.02)).astype(np.float64)
        E = emulate.r8_polar_express(M, TABLE, T, folded=True, ab_planes=ab_planes).astype(np.float64)
        out.append(om.rel_frobenius(E, oi.polar_express(M, TABLE, T)))
    return np.array(out)


def test_r8_emulation_equals_diagonal_pin():
    """The general emulation reduces to the bit-pinned diagonal one
    (tests/test_emulate_pin.py) on diagonal inputs, folded and unfolded."""
    sig = syn.to_bf16_values(np.linspace(1.0, 0.03, 40)).astype(np.float64)
    for shape in ((40, 96), (96, 40), (40, 61)):
        M = syn.diagonal(*shape, sig)
        for T in (1, 3, 5):
            E = emulate.r8_polar_express(M, TABLE, T, folded=True)
            d = emulate.diagonal_bf16(sig, TABLE, T, folded=True)
            assert np.array_equal(np.diag(E)[:40], d)


@pytest.mark.parametrize("shape", [(8, 8), (8, 100), (16, 16), (16, 40), (32, 32), (37, 100), (48, 100),
                                   (64, 300), (300, 64), (64, 768), (71, 547), (100, 37), (127, 700)])
def test_small_m_spread_needs_and_fits_the_widened_gate(shape):
    """Small m, 24 seeds: the design's worst relF stays inside g1_gate(m)
    (measured maxima: 7.8e-2 at 8 x 8, 4.4e-2 at 8 x 100, 3.6e-2 at 16 x 40,
    2.9e-2 at 32 x 32, 2.5e-2 at 37 x 100, 1.97e-2 at 71 x 547)."""
    r = spread(shape, range(24))
    assert r.max() <= g1_gate(min(shape)), (shape, r.max())


def test_small_m_spread_exceeds_2e2_somewhere():
    """... and 2e-2 alone would fail the design itself on small shapes (so the
    widening below m = 128 is needed)."""
    for shape in ((8, 8), (16, 40), (37, 100)):
        assert spread(shape, range(24)).max() > 2e-2, shape


@pytest.mark.parametrize("shape", [(32, 32), (32, 500), (37, 100), (48, 100), (64, 64), (64, 300), (71, 547),
                                   (100, 37), (127, 600)])
def test_two_plane_small_path_meets_2e2_from_m32(shape):
    """The small path's precise variant (R8p: A and B as two bf16 planes,
    pe_set_small_planes(2), max side <= 640) meets north_star's 2e-2 from
    m = 32 on every seed (24 seeds; 16 x 40 reaches 1.16e-2, 16 x 16 3.5e-2,
    8 x 8 2.1e-2 -- X's own rounding then dominates)."""
    r = spread(shape, range(24), ab_planes=2)
    assert r.max() <= 2e-2, (shape, r.max())


def test_r8p_general_emulation_reduces_to_the_diagonal_one():
    sig = syn.to_bf16_values(np.linspace(1.0, 0.03, 40)).astype(np.float64)
    for shape in ((40, 96), (96, 40), (40, 61)):
        M = syn.diagonal(*shape, sig)
        for T in (1, 3, 5):
            E = emulate.r8_polar_express(M, TABLE, T, folded=True, ab_planes=2)
            d = emulate.diagonal_bf16(sig, TABLE, T, folded=True, ab_planes=2)
            assert np.array_equal(np.diag(E)[:40], d)


@pytest.mark.parametrize("shape", [(128, 128), (128, 512), (200, 520)])
def test_from_m128_the_design_meets_2e2(shape):
    """From m = 128 the same design stays within north_star's 2e-2 (8 seeds)."""
    r = spread(shape, range(8))
    assert r.max() <= 2e-2, (shape, r.max())


@pytest.mark.parametrize("T", [1, 2])
def test_early_iterates_spread(T):
    """T <= 2 (iterates on the steep part of the composite): the GPU gate
    3e-2 (test_iteration_counts) covers the design's spread at 256 x 768."""
    r = spread((256, 768), range(6), T=T)
    assert r.max() <= 3e-2, (T, r.max())


def test_rank_one_spread():
    """Rank one (1 x n): every normalised singular value at 1/1.01 where the
    T = 5 composite has slope ~160, so one bf16 rounding of A moves the result
    by a few percent: the GPU gate 5e-2 (test_gaussian_parity) covers the
    design's spread over 20 seeds, which does exceed 2e-2."""
    r = np.concatenate([spread((1, 64), range(10)), spread((64, 1), range(10, 20))])
    assert r.max() <= 5e-2 and r.max() > 2e-2, r.max()


# ---------------------------------------------------------------- App. H
def test_r19_alg4_emulation_pins():
    """oracle.emulate.r19_alg4 (the bf16 Alg. 4 design) reduces to the
    R8 emulation with restart 1 and no shift (restarting every
    iteration is the baseline), bit for bit, and tracks the fp64 Alg. 4
    oracle on a diagonal input to bf16 accuracy once converged."""
    from oracle import alg4 as a4
    for shape in ((64, 200), (200, 64), (60, 203)):
        M = syn.to_bf16_values(syn.gaussian(*shape, seed=5, std=0.02)).astype(np.float64)
        fold = shape[1] % 8 == 0
        for T in (1, 3, 5):
            assert np.array_equal(emulate.r19_alg4(M, TABLE, T, restart=1, shift=0.0, folded=fold),
                                  emulate.r8_polar_express(M, TABLE, T, folded=fold))
    sig = syn.to_bf16_values(np.linspace(1.0, 0.2, 30)).astype(np.float64)
    M = syn.diagonal(30, 90, sig)
    E = emulate.r19_alg4(M, TABLE, 8, restart=None, shift=0.0).astype(np.float64)
    assert np.abs(np.diag(E)[:30] - np.diag(a4.alg4(M, TABLE, 8, restart=None, shift=0.0))[:30]).max() < 2e-2


def alg4_spread(shape, seeds, restart, T=5, spectrum=None):
    from oracle import alg4 as a4
    g1, g3 = [], []
    for seed in seeds:
        if spectrum is None:
            M = syn.gaussian(*shape, seed=seed, std=0.02)
        else:
            M = syn.prescribed_spectrum(*shape, np.geomspace(1.0, 1.0 / spectrum, min(shape)), seed=seed) * 0.01
        M = syn.to_bf16_values(M).astype(np.float64)
        ref = a4.alg4(M, TABLE, T, restart=restart, shift=1e-3)
        E = emulate.r19_alg4(M, TABLE, T, restart=restart, shift=1e-3, folded=True).astype(np.float64)
        P = oi.exact_polar(M)
        g1.append(om.rel_frobenius(E, ref))
        g3.append(om.rel_frobenius(E, P) - om.rel_frobenius(ref, P))
    return np.array(g1), np.array(g3)


ALG4_G1 = {2: 3e-2, 3: 5e-2, None: 8e-2}     # tests/test_gpu_parity.py Alg. 4 gates


@pytest.mark.parametrize("restart", [2, 3, None])
def test_alg4_design_spread_on_gaussians(restart):
    """The bf16 Alg. 4 design against the fp64 Alg. 4 oracle on Gaussian
    inputs (T = 5, shift 1e-3): every bf16 rounding of Y, T, R, H and Q feeds
    the next m x m product, so the design lands further from the fp64 path
    than Listing 2's (up to 2.3e-2 / 4.2e-2 / 6.5e-2 for restarts 2 / 3 /
    none, vs <= 2e-2) -- the Alg. 4 G1 gates of the GPU test are these
    spreads with headroom, while its error to polar(M) stays within 3e-3 of
    the oracle's (G3, north_star's 1e-2)."""
    worst1, worst3 = 0.0, -1.0
    for shape in ((128, 512), (192, 768), (256, 1024), (300, 1100)):
        g1, g3 = alg4_spread(shape, range(3), restart)
        worst1, worst3 = max(worst1, g1.max()), max(worst3, g3.max())
    assert worst1 <= ALG4_G1[restart], worst1
    assert worst3 <= 3e-3, worst3
