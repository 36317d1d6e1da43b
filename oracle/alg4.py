"""Fast polynomial iteration for rectangular matrices (App. H, Alg. 4,
P:1303-1316) in fp64 -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper states Alg. 4 for X in R^{m x n} with m >= n (tall; aspect ratio
alpha = m / n) and odd polynomials p_t(x) = x h_t(x^2):

    Y = X^T X                                   (the first application adds
                                                 10^-3 I)
    Q_0 = I
    for t = 1..T:  R_t = Q_{t-1}^T Y Q_{t-1}
                   Q_t = Q_{t-1} h_t(R_t)       (Horner)
    return X Q_T

with restarts: for T > k the algorithm is applied to X_0 with
p_1..p_k, giving X_k, then again to X_k with p_{k+1}..p_{2k}, and so on;
restarting after every iteration is the baseline (Listing 2).  The
normalisation is Listing 2's (reading R1) unless ``norm="app_h"`` asks for
App. H's ``||X||_F + 10^-3``.  Wide inputs are transposed to the
paper's tall orientation and back (the polar factor commutes with
transposition).
"""
from __future__ import annotations

import numpy as np

from .iteration import schedule


def horner(tup, R):
    """h(R) for p(x) = x h(x^2): h(y) = a + y (b [+ c y]) by Horner's rule
    (P:1291-1293)."""
    n = R.shape[0]
    eye = np.eye(n)
    if len(tup) == 3:
        a, b, c = tup
        return a * eye + R @ (b * eye + c * R)
    a, b = tup
    return a * eye + b * R


def alg4_block(X, tuples, shift=0.0):
    """One application of Alg. 4 to a tall X (m >= n) with the
    polynomials ``tuples``: returns (X Q_T, Q_T).  ``shift`` is the
    10^-3 I of P:1344 (first application only)."""
    X = np.asarray(X, dtype=np.float64)
    Y = X.T @ X + shift * np.eye(X.shape[1])          # mn^2
    Q = np.eye(X.shape[1])                              # Q_0 = I
    for tup in tuples:
        R = Q.T @ Y @ Q                                 # 2 n^3
        Q = Q @ horner(tup, R)                          # deg(h) n^3
    return X @ Q, Q                                     # mn^2


def alg4(M, table, T, restart=None, shift=1e-3, norm="listing2"):
    """(p_T o ... o p_1)(X_0) by Alg. 4 with a restart every ``restart``
    iterations (None: no restart), Y shifted by ``shift`` I in
    the first application only, X_0 the normalised M (R1 /
    ``norm="app_h"``: M / (||M||_F + 10^-3)).  Tuples past the table
    repeat the last one.  Returns the result in M's orientation."""
    M = np.asarray(M, dtype=np.float64)
    wide = M.shape[0] < M.shape[1]
    X = M.T if wide else M                              # the paper's m >= n
    nrm = np.sqrt(np.sum(X * X))
    if norm == "listing2":
        X = X / (nrm * 1.01 + 1e-7)
    elif norm == "app_h":
        X = X / (nrm + 1e-3)
    elif norm is not None:
        raise ValueError(norm)
    tups = schedule(table, T)
    k = T if restart is None else int(restart)
    first = True
    for t0 in range(0, T, k):
        X, _ = alg4_block(X, tups[t0:t0 + k], shift if first else 0.0)
        first = False
    return X.T if wide else X


def alg4_flops(m, n, T, restart=None, degree=5):
    """Algorithmic flops of Alg. 4 on an m x n matrix (min side s, long side
    l; symmetric products counted once as in SURVEY §8d): per application
    l s^2 (Y) + 2 l s^2 (X Q), per iteration 2 s^3 (Y Q) + s^3 (Q^T (Y Q),
    symmetric) + s^3 (R^2, symmetric, degree 5 only) + 2 s^3 (H Q)."""
    s, l = min(m, n), max(m, n)
    k = T if restart is None else int(restart)
    apps = (T + k - 1) // k
    per_it = (6 if degree == 5 else 5) * s ** 3
    return apps * 3 * l * s * s + T * per_it


def baseline_flops(m, n, T, degree=5):
    """Listing 2 / pe_flops: T [s(s+1) l + s^2 (s+1) + 2 s^2 l]."""
    s, l = min(m, n), max(m, n)
    return T * (s * (s + 1) * l + (s * s * (s + 1) if degree == 5 else 0) + 2 * s * s * l)
