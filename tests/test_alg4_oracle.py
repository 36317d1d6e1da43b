"""Pins of oracle/alg4.py (App. H, Alg. 4) against what the
paper and the mathematics fix, independently of the oracle's own code:

  * restarting after every iteration is exactly the baseline:
    Alg. 4 with restart 1 and no shift equals Listing 2 (oracle iteration);
  * without shift, one application equals the scalar composite map of the
    singular values (q_t recursion P:1319-1327: X Q_T = (p_T o..o p_1)(X)),
    computed through an SVD, to 1e-10;
  * with the shift s one application is the matrix function
    U diag(sigma p*(sqrt(sigma^2 + s)) / sqrt(sigma^2 + s)) V^T (Q_T is
    q_T(Y + s I), q_T(y) = p*(sqrt y) / sqrt y), and a restart composes such
    maps (the shift only in the first application);
  * Q_T -> Y^{-1/2} (footnote) via eigh;
  * the cost model and the selection rule alpha > 1.5 T / (T - 1)
    (P:1294-1295);
  * the shift does not change the polar factor: enough
    iterations converge to polar(M) with and without it.
"""
import numpy as np
import pytest

import pe_synth as syn
from oracle import alg4 as a4
from oracle import coeffs as oc
from oracle import iteration as oi
from oracle import metrics as om

TABLE, _ = oc.pe_coeffs(1e-3, 5, 8, 1.01)


def _svd_map(M, fn):
    U, s, Vt = np.linalg.svd(M, full_matrices=False)
    return (U * fn(s)) @ Vt


@pytest.mark.parametrize("shape", [(40, 10), (10, 40), (64, 16), (33, 33)])
def test_restart_every_iteration_is_the_baseline(shape):
    M = syn.gaussian(*shape, seed=sum(shape))
    for T in (1, 3, 5, 8):
        X = a4.alg4(M, TABLE, T, restart=1, shift=0.0)
        assert np.abs(X - oi.polar_express(M, TABLE, T)).max() < 1e-12


@pytest.mark.parametrize("shape", [(60, 15), (15, 60), (48, 12)])
def test_one_application_is_the_scalar_composite(shape):
    M = syn.gaussian(*shape, seed=7 + shape[0])
    nrm = np.linalg.norm(M) * 1.01 + 1e-7
    for T in (2, 5, 8):
        X = a4.alg4(M, TABLE, T, restart=None, shift=0.0)
        ref = _svd_map(M, lambda s: oi.composite(s / nrm, TABLE, T))
        assert np.abs(X - ref).max() < 1e-10, T


def _shifted_block(s, tuples, shift):
    """sigma -> sigma q(sigma^2 + shift), q(y) = p*(sqrt y) / sqrt y."""
    y = np.sqrt(s * s + shift)
    out = y.copy()
    for tup in tuples:
        out = oc.odd_poly(tup, out)
    return s * out / y


@pytest.mark.parametrize("restart", [None, 2, 3])
def test_shifted_applications_are_matrix_functions(restart):
    M = syn.gaussian(80, 20, seed=3)
    T = 5
    nrm = np.linalg.norm(M) * 1.01 + 1e-7
    tups = oi.schedule(TABLE, T)
    k = T if restart is None else restart

    def fn(s):
        s = s / nrm
        first = True
        for t0 in range(0, T, k):
            s = _shifted_block(s, tups[t0:t0 + k], 1e-3 if first else 0.0)
            first = False
        return s

    X = a4.alg4(M, TABLE, T, restart=restart, shift=1e-3)
    assert np.abs(X - _svd_map(M, fn)).max() < 1e-10


def test_Q_converges_to_inverse_square_root():
    """Footnote P:1332: Q_T -> Y^{-1/2} (singular values in [0.2, 1], T = 10)."""
    rng = np.random.default_rng(1)
    U, _ = np.linalg.qr(rng.standard_normal((50, 12)))
    V, _ = np.linalg.qr(rng.standard_normal((12, 12)))
    X = (U * np.linspace(1.0, 0.2, 12)) @ V.T
    _, Q = a4.alg4_block(X, oi.schedule(TABLE, 10))
    w, E = np.linalg.eigh(X.T @ X)
    assert np.abs(Q - (E / np.sqrt(w)) @ E.T).max() < 1e-8


def test_cost_model_and_selection_rule():
    """baseline (d-3)/2 + 2 alpha per iteration; Alg. 4 costs
    ((d+3)/2 T + 2 alpha) n^3; the crossover is alpha = 1.5 T / (T - 1)
     for d = 5.  The symmetric-aware counts (alg4_flops /
    baseline_flops) follow the same ordering at the BASELINE shapes."""
    for T in (3, 5, 6, 8):
        crit = 1.5 * T / (T - 1)
        for alpha in (crit * 0.9, crit * 1.1):
            base = ((5 - 3) / 2 + 2 * alpha) * T
            fast = (5 + 3) / 2 * T + 2 * alpha
            assert (fast < base) == (alpha > crit)
    # GPT-2 MLP (alpha = 4) and Llama MLP (alpha = 3.5), T = 5: fewer flops
    for m, n in ((768, 3072), (4096, 14336)):
        assert a4.alg4_flops(m, n, 5) < a4.baseline_flops(m, n, 5)
        assert a4.alg4_flops(m, n, 5, restart=1) > a4.baseline_flops(m, n, 5)


def test_shift_keeps_the_polar_factor_with_restarts():
    """the shift (first application only) changes early iterates,
    not the limit -- when a later, unshifted application follows (restart).
    A single shifted application converges to X (X^T X + s I)^{-1/2}
    instead (reading R20), whose singular values are sigma / sqrt(sigma^2 + s)."""
    M = syn.gaussian(120, 30, seed=11)
    P = oi.exact_polar(M)
    X = a4.alg4(M, TABLE, 12, restart=3, shift=1e-3)
    assert om.rel_frobenius(X, P) < 1e-12
    X5 = a4.alg4(M, TABLE, 5, restart=3, shift=1e-3)
    assert om.rel_frobenius(X5, oi.polar_express(M, TABLE, 5)) > 1e-3     # ... but it does move T = 5
    nrm = np.linalg.norm(M) * 1.01 + 1e-7
    lim = _svd_map(M, lambda s: (s / nrm) / np.sqrt((s / nrm) ** 2 + 1e-3))
    assert np.abs(a4.alg4(M, TABLE, 12, restart=None, shift=1e-3) - lim).max() < 1e-10
