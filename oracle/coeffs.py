"""Offline stage of Polar Express in fp64 -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows, step by step and in the paper's order:
  * Listing 1 ``optimal_quintic`` / ``optimal_composition``, which
    implements Alg. 2 with Listing 1's constants (reading R6);
  * the degree-3 closed form, eq. (deg3_solution);
  * Listing 2's safety-factor comprehension;
  * the greedy recurrence of Theorem 1, eq. (newbounds).

Readings used: R3 (cushion constant of
Listing 1), R4 (Pade snap of the table tail), R5 (safety on every tuple except
the Pade tail), R6 (Listing 1's thresholds, iteration cap 50), R15 (degree-3
recentering about the interior maximum).
"""
from __future__ import annotations

import math

import numpy as np

# Listing 1 constants and Listing 2's safety.
PADE_THRESHOLD = 1 - 5e-6          # P:515  "if 1 - 5e-6 <= l / u"
REMEZ_TOL = 1e-15                  # P:523  "abs(old_E - E) > 1e-15"
CUSHION_QUINTIC = 0.02407327424182761  # P:537 default ``cushion``
SAFETY = 1.01                      # P:486  "a / 1.01, b / 1.01**3, c / 1.01**5"
REMEZ_MAX_ITERS = 50               # R6 (cap; the paper gives none)

# Flags (mirrored by value, not by code, in include/pe.h).
SAFETY_ALL = 1         # Alg.1 line 5: scale every p_t, Pade tail included
SAFETY_NOT_FINAL = 2   # App. F: omit the safety factor in the final iteration
NO_RECENTER = 4        # skip Listing 1's recentering


class NoConvergence(RuntimeError):
    pass


def odd_poly(coeffs, x):
    """p(x) = a x + b x^3 + c x^5 (odd monomials), summed term by term."""
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    for q, a in enumerate(coeffs):
        out = out + a * x ** (2 * q + 1)
    return out


def optimal_quintic(l, u, return_iters=False):
    """Listing 1 ``optimal_quintic`` = Alg. 2.

    Minimax odd quintic for the constant 1 on [l, u].  Pade branch when
    l/u >= 1 - 5e-6; otherwise Remez on the trial set
    {l, q, r, u} initialised at (3l+u)/4, (l+3u)/4, solving
    the 4x4 "Vandermonde + sign" system eq. (linearsystem) and
    moving q, r to the roots of 5c x^4 + 3b x^2 + a = 0.
    """
    assert 0 <= l <= u
    if PADE_THRESHOLD <= l / u:
        res = ((15 / 8) / u, (-10 / 8) / u ** 3, (3 / 8) / u ** 5)
        return (res, 0) if return_iters else res
    q = (3 * l + u) / 4
    r = (l + 3 * u) / 4
    E, old_E = math.inf, None
    iters = 0
    while not old_E or abs(old_E - E) > REMEZ_TOL:
        if iters >= REMEZ_MAX_ITERS:
            raise NoConvergence(f"Remez did not converge on [{l}, {u}]")
        old_E = E
        LHS = np.array([
            [l, l ** 3, l ** 5, 1],
            [q, q ** 3, q ** 5, -1],
            [r, r ** 3, r ** 5, 1],
            [u, u ** 3, u ** 5, -1],
        ])
        a, b, c, E = np.linalg.solve(LHS, np.ones(4))
        q, r = np.sqrt((-3 * b + np.array([-1, 1]) * math.sqrt(9 * b ** 2 - 20 * a * c)) / (10 * c))
        iters += 1
    res = (float(a), float(b), float(c))
    return (res, iters) if return_iters else res


def remez_error(l, u):
    """E of the minimax quintic on [l, u]: the last E of the Remez loop
    (= max |1 - p| on [l, u] at convergence, Lemma P:641-644)."""
    a, b, c = optimal_quintic(l, u)
    return float(1 - odd_poly((a, b, c), l))


def optimal_cubic(l, u):
    """Degree-3 closed form, eq. (deg3_solution):
    p(x) = beta * p_NS(alpha x), p_NS(x) = 3/2 x - 1/2 x^3,
    alpha = sqrt(3 / (u^2 + l u + l^2)), beta = 4 / (2 + l u (l + u) alpha^3)."""
    assert 0 <= l <= u and u > 0
    alpha = math.sqrt(3 / (u ** 2 + l * u + l ** 2))
    beta = 4 / (2 + l * u * (l + u) * alpha ** 3)
    return (beta * 1.5 * alpha, -beta * 0.5 * alpha ** 3)


def cubic_cushion_for_error(E_target=9 / 11):
    """Reading R3 for degree 3: the c in (0,1) at which the optimal cubic on
    [c, 1] has minimax error E_target (default 9/11, i.e. output ratio 10,
    the rule that reproduces Listing 1's quintic cushion).  Bisection on the
    closed form's error beta - 1, which decreases in c."""
    lo, hi = 1e-12, 1.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        alpha = math.sqrt(3 / (1 + mid + mid ** 2))
        beta = 4 / (2 + mid * (1 + mid) * alpha ** 3)
        if beta - 1 > E_target:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


CUSHION_CUBIC = cubic_cushion_for_error()


def greedy_composition(l, num_iters, degree=5, cushion=None, recenter=True):
    """Listing 1 ``optimal_composition`` generalised to degree 3.

    For each step: minimax polynomial on [max(l, cushion*u), u] (P:539,
    Alg.1 line 4 P:320), recentre so that 1 - p(l) = max p - 1,
    then l <- p(l), u <- 2 - l (eq. (newbounds)).

    Returns (pre-safety tuples, pade_flags, ell_trace[num_iters+1]).
    pade_flags[t] is True when the Pade branch produced tuple t (reading R4).
    """
    if cushion is None:
        cushion = CUSHION_QUINTIC if degree == 5 else CUSHION_CUBIC
    u = 1.0
    coefficients, pade, trace = [], [], [l]
    for _ in range(num_iters):
        lo = max(l, cushion * u)
        if degree == 5:
            is_pade = PADE_THRESHOLD <= lo / u
            if is_pade:
                # R4: the Pade branch emits the exact limit (15/8, -10/8, 3/8)
                # (Listing 2's printed tail, "subsequent coeffs equal
                # this numerically"); no recentering.
                coeffs = (15 / 8, -10 / 8, 3 / 8)
            else:
                coeffs = optimal_quintic(lo, u)
        elif degree == 3:
            is_pade = PADE_THRESHOLD <= lo / u
            coeffs = (1.5, -0.5) if is_pade else optimal_cubic(lo, u)
        else:
            raise ValueError("degree must be 3 or 5 (general Remez is out of scope, P:345)")
        if recenter and not is_pade:
            pl = float(odd_poly(coeffs, l))
            if degree == 5:
                pmax = float(odd_poly(coeffs, u))           # P:544  pu
            else:
                # R15: the cubic's maximum is at its interior extremum
                # x* = sqrt(-a/(3b)) when it lies in [l, u].
                a, b = coeffs
                xs = math.sqrt(-a / (3 * b))
                xs = min(max(xs, l), u)
                pmax = max(float(odd_poly(coeffs, xs)), float(odd_poly(coeffs, u)))
            rescalar = 2 / (pl + pmax)
            coeffs = tuple(x * rescalar for x in coeffs)
        coefficients.append(tuple(float(x) for x in coeffs))
        pade.append(is_pade)
        l = float(odd_poly(coeffs, l))
        u = 2 - l
        trace.append(l)
    return coefficients, pade, trace


def apply_safety(coeffs, pade_flags, safety=SAFETY, flags=0):
    """Listing 2's comprehension: p(x) -> p(x / safety), i.e.
    coefficient of x^(2q+1) divided by safety^(2q+1); reading R5 leaves the
    Pade tail unscaled.  SAFETY_ALL scales it too (Alg.1 line 5);
    SAFETY_NOT_FINAL leaves the final tuple unscaled (App. F)."""
    out = []
    T = len(coeffs)
    for t, (tup, is_pade) in enumerate(zip(coeffs, pade_flags)):
        scale = True
        if is_pade and not (flags & SAFETY_ALL):
            scale = False
        if (flags & SAFETY_NOT_FINAL) and t == T - 1:
            scale = False
        if scale:
            tup = tuple(x / safety ** (2 * q + 1) for q, x in enumerate(tup))
        out.append(tup)
    return out


def pe_coeffs(ell=1e-3, degree=5, T=8, safety=SAFETY, cushion=None, flags=0):
    """The oracle's version of the offline stage: T tuples ready for the
    online iteration (Alg. 1 offline box P:316-323 + Listing 2).
    Returns (tuples, ell_trace)."""
    if not (0 < ell <= 1) or T < 1 or safety < 1:
        raise ValueError("invalid argument")
    raw, pade, trace = greedy_composition(ell, T, degree, cushion,
                                          recenter=not (flags & NO_RECENTER))
    return apply_safety(raw, pade, safety, flags), trace


# Fixed polynomials the paper compares against (used with the same kernels).
NEWTON_SCHULZ_3 = (1.5, -0.5)
NEWTON_SCHULZ_5 = (15 / 8, -10 / 8, 3 / 8)
JORDAN = (3.4445, -4.7750, 2.0315)
