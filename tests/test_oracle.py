"""Pins of the fp64 oracle against what the paper and the mathematics fix.

Nothing here compares the oracle with itself: every test checks it against a
value the paper prints (tests/golden/, cited), a closed form, an independent
decomposition (SVD / eigh), a brute-force linear program, or an invariant the
paper states.  Each docstring names the passage (P:<line> = PAPER.md line).
"""
import math
import os

import numpy as np
import pytest
from scipy.optimize import linprog

import pe_synth as syn
from oracle import coeffs as oc
from oracle import emulate, iteration as oi, metrics as om

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load_table(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(tuple(float(v) for v in line.split()))
    return rows


def load_constants():
    out = {}
    with open(os.path.join(GOLD, "paper_constants.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                k, v, _cite = line.split()
                out[k] = float(v)
    return out


PRINTED = load_table("listing2_coeffs_pre_safety.txt")
CONST = load_constants()


# --------------------------------------------------------------------------
# Offline stage
# --------------------------------------------------------------------------

def lp_minimax(l, u, degree, npts=6001):
    """Brute force: min_E s.t. |1 - p(x_i)| <= E on a dense grid of [l, u],
    p odd of the given degree (eq. (remez_goal)) -- a linear
    program with no Remez/equioscillation logic in it."""
    x = np.concatenate([np.linspace(l, u, npts),
                        l + (u - l) * (1 - np.cos(np.linspace(0, np.pi, npts))) / 2])
    nq = (degree + 1) // 2
    V = np.stack([x ** (2 * q + 1) for q in range(nq)], axis=1)
    ones = np.ones((len(x), 1))
    # variables: coeffs (nq), E ; minimize E
    A_ub = np.vstack([np.hstack([V, -ones]), np.hstack([-V, -ones])])
    b_ub = np.concatenate([np.ones(len(x)), -np.ones(len(x))])
    cvec = np.zeros(nq + 1)
    cvec[-1] = 1
    res = linprog(cvec, A_ub=A_ub, b_ub=b_ub, bounds=[(None, None)] * (nq + 1), method="highs")
    assert res.status == 0
    return res.x[:nq], res.x[-1]


@pytest.mark.parametrize("l,u", [(0.1, 1.0), (0.02407327424182761, 1.0), (0.3, 0.9), (0.5, 1.0), (0.8, 1.2)])
def test_quintic_is_minimax_vs_linear_program(l, u):
    """Remez output (Listing 1) equals the brute-force LP minimax
    solution of eq. (remez_goal)."""
    (a, b, c) = oc.optimal_quintic(l, u)
    cl, El = lp_minimax(l, u, 5)
    xs = np.linspace(l, u, 200001)
    E = np.max(np.abs(1 - oc.odd_poly((a, b, c), xs)))
    assert E <= El * (1 + 1e-6) + 1e-9          # Remez is at least as good as the LP
    assert E >= El * (1 - 1e-6) - 1e-9          # ... and the LP cannot beat it
    assert np.allclose((a, b, c), cl, rtol=2e-5, atol=1e-7)


@pytest.mark.parametrize("l,u", [(0.1, 1.0), (0.5, 1.0), (0.039, 1.0), (0.3, 2.0)])
def test_cubic_closed_form_is_minimax_vs_linear_program(l, u):
    """eq. (deg3_solution) equals the LP minimax cubic."""
    a, b = oc.optimal_cubic(l, u)
    cl, El = lp_minimax(l, u, 3)
    xs = np.linspace(l, u, 200001)
    E = np.max(np.abs(1 - oc.odd_poly((a, b), xs)))
    assert abs(E - El) <= 1e-6 * max(El, 1e-3)
    assert np.allclose((a, b), cl, rtol=2e-5, atol=1e-7)


def test_cubic_special_cases():
    """l=u=1 gives Newton-Schulz (3/2, -1/2);
    [0,1] gives alpha=sqrt(3), beta=2, i.e. (3 sqrt3, -3 sqrt3) with E=beta-1=1."""
    assert np.allclose(oc.optimal_cubic(1.0, 1.0), (1.5, -0.5), rtol=0, atol=1e-15)
    a, b = oc.optimal_cubic(0.0, 1.0)
    assert math.isclose(a, 3 * math.sqrt(3), rel_tol=1e-14)
    assert math.isclose(b, -3 * math.sqrt(3), rel_tol=1e-14)
    # equioscillation at l, 1/alpha, u
    l, u = 0.5, 1.0
    a, b = oc.optimal_cubic(l, u)
    xs = math.sqrt(-a / (3 * b))
    e = [1 - oc.odd_poly((a, b), v) for v in (l, xs, u)]
    assert abs(e[0] - e[2]) < 1e-14 and abs(e[0] + e[1]) < 1e-14 and e[0] > 0


def quintic_extrema(coef, l, u):
    a, b, c = coef
    disc = 9 * b * b - 20 * a * c
    ys = [(-3 * b - math.sqrt(disc)) / (10 * c), (-3 * b + math.sqrt(disc)) / (10 * c)]
    inner = sorted(math.sqrt(y) for y in ys if y > 0 and l < math.sqrt(y) < u)
    return [l] + inner + [u]


def test_equioscillation_of_each_greedy_step():
    """Lemma: the pre-recentre Remez polynomial on [l', u_t] has
    q+2 = 4 alternating extrema of equal amplitude E; cushioned steps have
    E = 9/11 (reading R3); recentred p_t has min p(l_t), max p(u_t) with
    1 - p(l_t) = p(u_t) - 1 (Lemma 2)."""
    l, u = 1e-3, 1.0
    raw, pade, trace = oc.greedy_composition(1e-3, 7)
    for t in range(7):
        lo = max(l, oc.CUSHION_QUINTIC * u)
        coef = oc.optimal_quintic(lo, u)
        pts = quintic_extrema(coef, lo, u)
        assert len(pts) == 4
        errs = [1 - float(oc.odd_poly(coef, p)) for p in pts]
        E = abs(errs[0])
        for i, e in enumerate(errs):
            assert abs(abs(e) - E) <= 1e-14 + 1e-12 * E
            assert np.sign(e) == (1 if i % 2 == 0 else -1)
        if t < 3:
            assert abs(E - 9 / 11) < 1e-12
        p = raw[t]
        assert abs((1 - oc.odd_poly(p, l)) - (oc.odd_poly(p, u) - 1)) < 1e-14
        if E > 1e-8:
            xs = np.linspace(l, u, 1_000_001)
            v = oc.odd_poly(p, xs)
            assert v.min() >= oc.odd_poly(p, l) - 1e-14
            assert v.max() <= oc.odd_poly(p, u) + 1e-14
        l = float(oc.odd_poly(p, l))
        u = 2 - l


def test_printed_table_reproduced():
    """The 8 pre-safety tuples printed in Listing 2 (produced by
    Listing 1): tuples 1-6 to 1e-12, tuple 7 to 1e-9 (conditioning,
    reading R4), tuple 8 exactly (Pade snap, R4)."""
    raw, pade, trace = oc.greedy_composition(1e-3, 8)
    for t, (mine, printed) in enumerate(zip(raw, PRINTED)):
        tol = 1e-14 if t < 6 else (1e-9 if t == 6 else 0.0)
        for m, p in zip(mine, printed):
            assert abs(m - p) <= tol * abs(p), (t, mine, printed)
    assert pade == [False] * 7 + [True]


def test_greedy_recurrence_and_certified_error():
    """Theorem 1: max_{[l,1]} |1 - p*(x)| = 1 - l_{T+1}, with
    l_{t+1} = p_t(l_t) and u_{t+1} = 2 - l_{t+1} (eq. (newbounds)),
    checked on a dense grid against the composite of the printed table."""
    _, _, trace = oc.greedy_composition(1e-3, 8)
    xs = np.concatenate([np.logspace(-3, 0, 400001)])
    for T in range(1, 8):
        err = np.max(np.abs(1 - oi.composite(xs, PRINTED, T)))
        assert abs(err - (1 - trace[T])) <= 1e-9 * max(1.0, 1 - trace[T]) + 1e-12, T
    # P:54 (SPEC S:54 derived): p_1(1) = 2 - l_2
    assert abs(oc.odd_poly(PRINTED[0], 1.0) - (2 - trace[1])) < 1e-12


def test_safety_semantics():
    """P:485-487 / App. F: the stored polynomial is x -> p_t(x/1.01)
    (checked by evaluation, not by coefficient formula), the Pade tail is
    stored unscaled, and the fixed point of the scaled Pade polynomial is
    ~0.999998."""
    tab, _ = oc.pe_coeffs(1e-3, 5, 8, CONST["safety"])
    xs = np.linspace(0, 1.2, 1001)
    for t in range(7):
        assert np.allclose(oc.odd_poly(tab[t], xs), oc.odd_poly(PRINTED[t], xs / 1.01),
                           rtol=1e-9, atol=1e-12)
    assert tab[7] == (1.875, -1.25, 0.375)
    safe_pade = oc.apply_safety([oc.NEWTON_SCHULZ_5], [False], 1.01)[0]
    x = 1.0
    for _ in range(200):
        x = float(oc.odd_poly(safe_pade, x))
    assert abs(x - CONST["safety_fixed_point"]) < 5e-7
    # flags: SAFETY_ALL also scales the tail, SAFETY_NOT_FINAL leaves the last one
    t2, _ = oc.pe_coeffs(1e-3, 5, 8, 1.01, flags=oc.SAFETY_ALL)
    assert np.allclose(oc.odd_poly(t2[7], xs), oc.odd_poly(PRINTED[7], xs / 1.01), rtol=1e-12)
    t3, _ = oc.pe_coeffs(1e-3, 5, 5, 1.01, flags=oc.SAFETY_NOT_FINAL)
    assert np.allclose(t3[4], PRINTED[4], rtol=1e-12)


def test_cushion_bounds_ratio():
    """App. F: with the cushion, p_t(x)/x stays bounded below
    (>= 0.236 for the u/10 cushion); Listing 1's cushion gives >= 0.236 too."""
    tab, _ = oc.pe_coeffs(1e-3, 5, 8, 1.0)
    xs = np.linspace(1e-6, 1.0, 100001)
    for t in range(3):
        assert np.min(oc.odd_poly(tab[t], xs) / xs) >= CONST["cushion_ratio_floor"]
    # Alg. 1's u/10 rule as a parameter
    tab10, _ = oc.pe_coeffs(1e-3, 5, 3, 1.0, cushion=0.1)
    assert np.min(oc.odd_poly(tab10[0], xs) / xs) >= CONST["cushion_ratio_floor"] - 1e-3


def test_cushion_constant_gives_output_ratio_ten():
    """Reading R3: Listing 1's cushion is where the minimax quintic on
    [c,1] has error 9/11, i.e. maps [c,1] onto [2/11, 20/11] (ratio 10,
    'The choice of 10').  Degree 3 analogue from P:808."""
    E = oc.remez_error(CONST["cushion"], 1.0)
    assert abs(E - 9 / 11) < 1e-13
    c3 = oc.CUSHION_CUBIC
    a, b = oc.optimal_cubic(c3, 1.0)
    xs = np.linspace(c3, 1, 200001)
    assert abs(np.max(np.abs(1 - oc.odd_poly((a, b), xs))) - 9 / 11) < 1e-9


def test_pade_branch_and_scale_covariance():
    """l/u >= 1-5e-6 returns (15/8, -10/8, 3/8)/u^k; the minimax
    problem is covariant under x -> x/u, so
    quintic(l,u) = quintic(l/u,1) with a/u, b/u^3, c/u^5."""
    assert oc.optimal_quintic(1.0, 1.0) == (1.875, -1.25, 0.375)
    a, b, c = oc.optimal_quintic(0.999999, 1.0)
    assert np.allclose((a, b, c), (1.875, -1.25, 0.375), rtol=1e-12)
    for (l, u) in [(0.05, 0.5), (0.2, 1.7)]:
        a1, b1, c1 = oc.optimal_quintic(l, u)
        a0, b0, c0 = oc.optimal_quintic(l / u, 1.0)
        assert np.allclose((a1, b1, c1), (a0 / u, b0 / u ** 3, c0 / u ** 5), rtol=1e-10)


def test_remez_iteration_count():
    """'we never observed Alg. 2 taking more than five iterations'."""
    g = syn.rng(0)
    for _ in range(200):
        l = float(g.uniform(1e-4, 0.99))
        _, it = oc.optimal_quintic(l, 1.0, return_iters=True)
        assert it <= 6


def test_theorem2_bound():
    """Theorem 2: error <= (1 - l^2)^((q+1)^T) (d=5: q=2; d=3: q=1),
    no cushion, no safety."""
    for l in (0.1, 0.3, 0.5, 0.9):
        for T in range(1, 6):
            for d, q in ((5, 2), (3, 1)):
                _, trace = oc.pe_coeffs(l, d, T, 1.0, cushion=0.0)
                assert 1 - trace[T] <= (1 - l * l) ** ((q + 1) ** T) + 1e-15


def test_section41_convergence_claims():
    """§4.1 on sigma in [1e-6, 1] (scalar replay):
    NS5 'almost no progress for the first 17 iterations'; Jordan '~0.3 after
    just 11 iterations' and no further; PE with l = sigma_min 'excellent
    accuracy after just 11 iterations'; with l off by 100x PE beats Jordan
    only from 'iteration 13 or 14'."""
    x = np.logspace(-6, 0, 20001)

    def err(tab, T):
        return float(np.max(np.abs(1 - oi.composite(x, tab, T))))
    assert all(err([oc.NEWTON_SCHULZ_5], T) > 0.95 for T in range(1, 18))
    jordan = [err([oc.JORDAN], T) for T in range(1, 26)]
    assert abs(jordan[10] - CONST["jordan_plateau"]) < 0.03
    assert min(jordan) > 0.3
    pe6, _ = oc.pe_coeffs(1e-6, 5, 25, 1.0)
    assert err(pe6, 11) < 1e-3
    firsts = []
    for ell in (1e-4, 1e-8):
        tab, _ = oc.pe_coeffs(ell, 5, 25, 1.0)
        firsts.append(next(T for T in range(10, 26) if err(tab, T) < jordan[T - 1]))
    assert sorted(firsts) == [13, 14]


def test_online_composite_suppression():
    """App. E.1: with T=5 the online table maps sigma >= 1e-3
    near 1 and sigma <= 1e-4 towards 0 (well below 1)."""
    tab, _ = oc.pe_coeffs(1e-3, 5, 5, 1.01)
    assert abs(oi.composite(1e-3, tab, 5) - 1) < 0.2
    assert oi.composite(1e-4, tab, 5) < 0.15
    xs = np.logspace(-3, 0, 100001)
    assert np.max(np.abs(1 - oi.composite(xs, tab, 5))) < 0.16


# --------------------------------------------------------------------------
# Online stage
# --------------------------------------------------------------------------

@pytest.mark.parametrize("shape", [(2, 2), (4, 7), (7, 4), (16, 32), (32, 16), (9, 9)])
def test_iteration_equals_scalar_map(shape):
    """p(M) = U p(Sigma) V^T with odd monomials through Gram products
    (P:113-117): the Listing-2 iteration equals the SVD route."""
    tab, _ = oc.pe_coeffs(1e-3, 5, 8, 1.01)
    M = syn.gaussian(*shape, seed=sum(shape))
    for T in (1, 3, 5, 8, 10):
        X = oi.polar_express(M, tab, T)
        Y = oi.via_scalar_map(M, tab, T)
        assert np.max(np.abs(X - Y)) <= 1e-12
    # degree 3 table too
    t3, _ = oc.pe_coeffs(1e-3, 3, 6, 1.01)
    assert np.max(np.abs(oi.polar_express(M, t3, 6) - oi.via_scalar_map(M, t3, 6))) <= 1e-12


def test_symmetric_input_gives_matrix_sign():
    """polar(M) = sign(M) for symmetric M, computed via eigh -- an
    independent decomposition -- for both exact_polar and the iteration."""
    g = syn.rng(3)
    Q = syn.haar_orthonormal(12, 12, g)
    lam = np.array([2.0, -1.0, 0.5, -0.3, 0.9, 1.5, -2.0, 0.7, -0.8, 1.1, -1.3, 0.6])
    M = (Q * lam) @ Q.T
    w, V = np.linalg.eigh(M)
    S = (V * np.sign(w)) @ V.T
    assert np.max(np.abs(oi.exact_polar(M) - S)) < 1e-12
    tab, _ = oc.pe_coeffs(1e-3, 5, 12, 1.0)
    X = oi.polar_express(M, tab, 12)
    assert np.max(np.abs(X - S)) < 1e-9


def test_exact_polar_properties():
    """polar(M) = U V^T: semi-orthogonal, and M = polar(M) H with
    H = polar(M)^T M symmetric positive semidefinite; 3I -> I."""
    for shape in [(16, 8), (8, 16), (10, 10)]:
        M = syn.gaussian(*shape, seed=7)
        P = oi.exact_polar(M)
        k = min(shape)
        G = P.T @ P if shape[0] >= shape[1] else P @ P.T
        assert np.max(np.abs(G - np.eye(k))) < 1e-12
        H = P.T @ M if shape[0] >= shape[1] else M @ P.T
        assert np.max(np.abs(H - H.T)) < 1e-12
        assert np.min(np.linalg.eigvalsh((H + H.T) / 2)) > -1e-12
    assert np.allclose(oi.exact_polar(3 * np.eye(5)), np.eye(5), atol=1e-15)


@pytest.mark.parametrize("rows,cols", [(64, 256), (256, 64), (128, 128)])
def test_hadamard_closed_form(rows, cols):
    """Equal singular values: rows of a Sylvester Hadamard matrix have
    all sigma = sqrt(n); after Listing-2 normalisation every sigma is
    sqrt(n)/(1.01 sqrt(mn) + 1e-7), so X_T = p*(sigma_hat) M / sqrt(n)."""
    tab, _ = oc.pe_coeffs(1e-3, 5, 8, 1.01)
    M = syn.hadamard_rows(rows, cols)
    m, n = min(rows, cols), max(rows, cols)
    sh = math.sqrt(n) / (1.01 * math.sqrt(m * n) + 1e-7)
    for T in (3, 5, 8):
        s = float(oi.composite(sh, tab, T))
        X = oi.polar_express(M, tab, T)
        assert np.max(np.abs(X - s * M / math.sqrt(n))) < 1e-13


def test_error_bound_on_prescribed_spectrum():
    """eq. (error): with sigma(X_0) in [l, 1] (normalisation
    bypassed), ||polar(M) - X_T||_2 <= 1 - l_{T+1} (safety = 1)."""
    tab, trace = oc.pe_coeffs(1e-3, 5, 6, 1.0)
    for seed in range(4):
        sig = np.concatenate([[1.0, 1e-3], syn.rng(seed).uniform(1e-3, 1, 14)])
        M = syn.prescribed_spectrum(24, 40, sig, seed)
        for T in range(1, 7):
            X = oi.polar_express(M, tab, T, norm=None)
            err = om.spectral(X, oi.exact_polar(M))
            assert err <= 1 - trace[T] + 1e-10


def test_normalization_and_symmetries():
    """X_0 = M/(||M||_F 1.01 + 1e-7) (I_3: ||I||_F = sqrt 3)
    alg1 mode; zero input returns zeros (R9); odd symmetry p(-M) = -p(M)
    (odd polynomials) and transpose trick."""
    assert np.allclose(oi.normalize(np.eye(3)), np.eye(3) / (math.sqrt(3) * 1.01 + 1e-7), rtol=1e-15)
    assert np.allclose(oi.normalize(np.eye(3), "alg1"), np.eye(3) / (math.sqrt(3) + 1e-2), rtol=1e-15)
    tab, _ = oc.pe_coeffs(1e-3, 5, 8, 1.01)
    assert np.all(oi.polar_express(np.zeros((4, 6)), tab, 5) == 0)
    M = syn.gaussian(12, 20, seed=5)
    X = oi.polar_express(M, tab, 5)
    assert np.array_equal(oi.polar_express(-M, tab, 5), -X)
    assert np.array_equal(oi.polar_express(M.T, tab, 5), X.T)
    # T past the table repeats the last tuple
    assert np.array_equal(oi.polar_express(M, tab[:3], 5),
                          oi.polar_express(M, tab[:3] + [tab[2]] * 2, 5))


def test_metrics_examples():
    """App. E.1 metrics: X = polar -> errors 0, cosine 1;
    X = -polar -> cosine -1; truncated polar of diag(1, 1e-4) at gamma=1e-3
    is diag(1, 0)."""
    M = syn.gaussian(10, 6, seed=1)
    P = oi.exact_polar(M)
    assert om.rel_frobenius(P, P) == 0 and om.spectral(P, P) == 0
    assert abs(om.cosine(P, P) - 1) < 1e-14 and abs(om.cosine(-P, P) + 1) < 1e-14
    D = np.diag([1.0, 1e-4])
    X = np.diag([1.0, 0.0])
    assert om.truncated_rel_frobenius(X, D, 1e-3) < 1e-15
    assert abs(om.spectral(X, oi.exact_polar(D)) - 1) < 1e-15
    Pg, _, _ = om.truncated_polar(D, 1e-3)
    assert np.allclose(Pg, X)


def test_bf16_diagonal_emulation_tracks_fp64_oracle():
    """The R8 rounding-point emulation (oracle/emulate.py) stays within bf16
    accuracy of the fp64 iteration on diagonal inputs (each singular
    value evolves under the scalar map)."""
    tab, _ = oc.pe_coeffs(1e-3, 5, 8, 1.01)
    sig = syn.to_bf16_values(np.linspace(1.0, 0.05, 64)).astype(np.float64)
    # intermediate iterates sit on the steep part of p_t (slope up to ~8 per
    # step), so bf16 rounding is amplified there; once converged (T >= 6 for
    # these sigma) the emulation must agree to bf16 resolution.
    for T, tol in ((1, 0.02), (3, 0.15), (5, 0.15), (6, 0.01), (8, 4e-3)):
        emu = emulate.diagonal_bf16(sig, tab, T).astype(np.float64)
        ref = np.diag(oi.polar_express(syn.diagonal(64, 96, sig), tab, T))
        assert np.max(np.abs(emu - ref)) < tol, T
        assert np.all(np.isfinite(emu))


def test_muon_step_pins():
    """oracle.iteration.muon_step against what P:41-49 fixes independently of
    the code: (i) the momentum recursion from M_0 = 0 unrolls to
    M_k = (1 - beta) sum_j beta^(k-j) G_j; (ii) on a diagonal gradient the
    step is W - lambda diag(p*(sigma_hat)) with p* the scalar composite
     and sigma_hat = sigma / (||sigma|| 1.01 + 1e-7);
    (iii) beta = 1 keeps M and moves W by -lambda polar_express(M); (iv) for a
    rank-one 1 x n gradient and enough iterations the step direction is the
    exact polar factor g / |g|."""
    table = oc.pe_coeffs(1e-3, 5, 8, 1.01)[0]
    rng = np.random.default_rng(3)
    beta = 0.9
    Gs = [rng.standard_normal((6, 9)) for _ in range(4)]
    M = np.zeros((6, 9))
    W = rng.standard_normal((6, 9))
    for G in Gs:
        W, M = oi.muon_step(W, M, G, beta, 0.01, table, 5)
    closed = (1 - beta) * sum(beta ** (len(Gs) - 1 - j) * G for j, G in enumerate(Gs))
    assert np.allclose(M, closed, rtol=0, atol=1e-14)
    # (ii) diagonal gradient, zero momentum, beta = 0
    sig = np.array([3.0, 1.0, 0.25, 0.01])
    G = np.zeros((4, 7))
    G[np.arange(4), np.arange(4)] = sig
    W0 = rng.standard_normal((4, 7))
    W1, M1 = oi.muon_step(W0, np.zeros_like(G), G, 0.0, 0.5, table, 5)
    shat = sig / (np.sqrt(np.sum(sig ** 2)) * 1.01 + 1e-7)
    expect = W0.copy()
    expect[np.arange(4), np.arange(4)] -= 0.5 * oi.composite(shat, table, 5)
    assert np.allclose(M1, G) and np.allclose(W1, expect, rtol=0, atol=1e-12)
    # (iii) beta = 1
    Mb = rng.standard_normal((5, 3))
    W2, M2 = oi.muon_step(np.zeros((5, 3)), Mb, rng.standard_normal((5, 3)), 1.0, 2.0, table, 5)
    assert np.array_equal(M2, Mb)
    assert np.allclose(W2, -2.0 * oi.polar_express(Mb, table, 5), rtol=0, atol=1e-14)
    # (iv) rank one: converges to g / |g|
    g = rng.standard_normal((1, 50))
    W3, _ = oi.muon_step(np.zeros((1, 50)), np.zeros((1, 50)), g, 0.0, 1.0, table, 12)
    assert np.allclose(-W3, g / np.linalg.norm(g), rtol=0, atol=1e-6)


def _mp_quintic(l, u, mp):
    """Listing 1's optimal_quintic in 60-digit arithmetic, with
    the Remez loop run to the high-precision fixed point (|dE| < 1e-50)."""
    if l / u >= mp.mpf(1) - mp.mpf("5e-6"):
        return (mp.mpf(15) / 8 / u, mp.mpf(-10) / 8 / u ** 3, mp.mpf(3) / 8 / u ** 5)
    q, r = (3 * l + u) / 4, (l + 3 * u) / 4
    E, old = mp.inf, None
    for _ in range(200):
        if old is not None and abs(old - E) < mp.mpf("1e-50"):
            break
        old = E
        M = mp.matrix([[l, l ** 3, l ** 5, 1], [q, q ** 3, q ** 5, -1],
                       [r, r ** 3, r ** 5, 1], [u, u ** 3, u ** 5, -1]])
        a, b, c, E = mp.lu_solve(M, mp.matrix([1, 1, 1, 1]))
        d = mp.sqrt(9 * b ** 2 - 20 * a * c)
        q, r = mp.sqrt((-3 * b - d) / (10 * c)), mp.sqrt((-3 * b + d) / (10 * c))
    return (a, b, c)


def test_coefficients_against_60_digit_replay():
    """SURVEY §8(c)1 cross-check: Listing 1's greedy composition (cushion,
    recentring) replayed in 60-digit mpmath arithmetic agrees with
    the fp64 oracle tuple by tuple (tuples 1-6 to 1e-14 relative, measured
    <= 1.6e-15; tuple 7 to
    1e-9, measured 5.7e-11, where the tiny interval makes the fp64 solve
    ill-conditioned; the
    Pade tail exactly, reading R4) -- i.e. the oracle's fp64 evaluation loses
    no accuracy that matters -- and the pre-safety table P:476-483 matches
    the high-precision values as well."""
    mpmath = pytest.importorskip("mpmath")
    mp = mpmath.mp
    mp.dps = 60
    l, u = mp.mpf("1e-3"), mp.mpf(1)
    cushion = mp.mpf("0.02407327424182761")
    hp = []
    for _ in range(8):
        a, b, c = _mp_quintic(max(l, cushion * u), u, mp)
        if max(l, cushion * u) / u < mp.mpf(1) - mp.mpf("5e-6"):
            p = lambda x: a * x + b * x ** 3 + c * x ** 5      # noqa: E731
            s = 2 / (p(l) + p(u))
            a, b, c = a * s, b * s, c * s
        else:
            a, b, c = mp.mpf(15) / 8, mp.mpf(-10) / 8, mp.mpf(3) / 8
        hp.append((a, b, c))
        l = a * l + b * l ** 3 + c * l ** 5
        u = 2 - l
    raw, pade, _ = oc.greedy_composition(1e-3, 8)
    printed = [tuple(float(v) for v in line.split()) for line in
               open(os.path.join(GOLD, "listing2_coeffs_pre_safety.txt")) if line.strip() and not line.startswith("#")]
    for t, (h, o, pr) in enumerate(zip(hp, raw, printed)):
        tol = 1e-14 if t < 6 else (1e-9 if t == 6 else 0.0)
        for hv, ov, pv in zip(h, o, pr):
            assert abs(float(hv) - ov) <= tol * abs(float(hv)), (t, float(hv), ov)
            if t < 7:
                assert abs(float(hv) - pv) <= max(tol, 1e-13) * abs(float(hv)) + 1e-14, (t, float(hv), pv)


# ---------------------------------------------------------------- App. G
def test_init_cubic_interpolates_and_bounds():
    """eq. (init_poly): p(sqrt(1-z^2)) = p(z) = 1; p(1) > 1/sqrt(2)
    (P:1262); p <= 1 on [0, sqrt(1-z^2)] and p([z, 1]) within [p(1), 1]
    (P:1260-1261), for z over [1/sqrt(2), 1)."""
    for z in np.linspace(0.7072, 0.99995, 60):
        a, b = oi.init_cubic(z)
        t = np.sqrt(1 - z * z)
        p = lambda x: a * x + b * x ** 3          # noqa: E731
        assert abs(p(t) - 1) < 1e-9 and abs(p(z) - 1) < 1e-9, z
        assert p(1.0) > 1 / np.sqrt(2)
        lo = np.linspace(0, t, 200)
        assert np.all(p(lo) <= 1 + 1e-9) and np.all(np.diff(p(lo)) >= -1e-12)      # concave-increasing
        hi = np.linspace(z, 1, 200)
        assert np.all(p(hi) <= 1 + 1e-9) and np.all(p(hi) >= p(1.0) - 1e-12)


def test_spectrum_init_is_the_scalar_map_and_a_lower_bound():
    """spectrum_init(X) = U p(Sigma/F) V^T with p = eq. (init_poly) at the z it
    found (matrix function, via an independent SVD route; no margin:
    P:1256-1263 has none); the result's largest singular value is <= 1
    ("the largest singular value of p(M) is still at most 1");
    z <= sigma_1 / F (Rayleigh
    quotient bound) and -> sigma_1 / F as the power method
    converges; no gap (Gaussian, z < 1/sqrt(2)) leaves X unchanged."""
    rng = np.random.default_rng(5)
    U, _ = np.linalg.qr(rng.standard_normal((40, 40)))
    V, _ = np.linalg.qr(rng.standard_normal((90, 40)))
    s = np.concatenate([[1.0], np.geomspace(0.2, 1e-3, 39)])
    X = (U * s) @ V.T * 0.37
    F = np.sqrt(np.sum(X * X))
    zs = []
    for q in (1, 2, 4, 8, 30):
        Y, z, applied = oi.spectrum_init(X, q)
        zs.append(z)
        assert z <= s[0] * 0.37 / F + 1e-12
        assert applied == (z >= 1 / np.sqrt(2)) and (applied or q < 8)
        if not applied:
            assert np.array_equal(Y, X)
            continue
        a, b = oi.init_cubic(z)
        sh = s * 0.37 / F
        ref = (U * (a * sh + b * sh ** 3)) @ V.T
        assert np.abs(Y - ref).max() <= 1e-12 * np.abs(ref).max()
        assert np.linalg.svd(Y, compute_uv=False)[0] <= 1 + 1e-9
    assert zs == sorted(zs) and abs(zs[-1] - s[0] * 0.37 / F) < 1e-12
    G = rng.standard_normal((64, 128))
    Y, z, applied = oi.spectrum_init(G, 8)
    assert not applied and z < 1 / np.sqrt(2) and np.array_equal(Y, G)


def test_spectrum_init_speeds_up_power_law_spectrum():
    """App. G's figure claim: on a 32 x 32 matrix with
    sigma_j = j^-5, the spectrum-aware step followed by T-1 Polar Express
    iterations beats T Polar Express iterations (the step counted as one)."""
    rng = np.random.default_rng(0)
    U, _ = np.linalg.qr(rng.standard_normal((32, 32)))
    V, _ = np.linalg.qr(rng.standard_normal((32, 32)))
    M = (U * np.arange(1, 33) ** -5.0) @ V.T
    P = oi.exact_polar(M)
    table, _ = oc.pe_coeffs(1e-3, 5, 8, 1.01)
    for T in range(3, 8):
        plain = om.rel_frobenius(oi.polar_express(M, table, T), P)
        X, z, applied = oi.polar_express_init(M, table, T - 1)
        assert applied and om.rel_frobenius(X, P) < plain - 1e-3, (T, plain)
