"""Error measures of App. E.1 -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""
from __future__ import annotations

import numpy as np


def rel_frobenius(X, Y):
    """||X - Y||_F / ||Y||_F (App. E.1)."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    d = np.linalg.norm(Y)
    return float(np.linalg.norm(X - Y) / d) if d > 0 else float(np.linalg.norm(X - Y))


def spectral(X, Y):
    """||X - Y||_2 (eq. (matrix_minimax_problem))."""
    D = np.asarray(X, dtype=np.float64) - np.asarray(Y, dtype=np.float64)
    if D.size == 0:
        return 0.0
    return float(np.linalg.norm(D, 2))


def cosine(X, Y):
    """<X, Y>_F / (||X||_F ||Y||_F) (App. E.1)."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    return float(np.sum(X * Y) / (np.linalg.norm(X) * np.linalg.norm(Y)))


def truncated_polar(M, gamma):
    """polar_gamma(M) = U_1 V_1^T over singular values >= gamma * sigma_max
    (App. E.1).  Returns (polar_gamma, U_1, V_1)."""
    M = np.asarray(M, dtype=np.float64)
    U, s, Vt = np.linalg.svd(M, full_matrices=False)
    keep = s >= gamma * s[0]
    U1, V1 = U[:, keep], Vt[keep, :].T
    return U1 @ V1.T, U1, V1


def truncated_rel_frobenius(X, M, gamma, reference=None):
    """||P_gamma - U_1 U_1^T X V_1 V_1^T||_F / ||P_gamma||_F (App. E.1,
    P:1036-1037): error restricted to the singular directions of M with
    sigma >= gamma sigma_max.  If ``reference`` is given it replaces
    polar_gamma(M) as the target (restricted the same way), which is the
    restricted-parity gate G2(i) of DESIGN.md."""
    Pg, U1, V1 = truncated_polar(M, gamma)
    Xr = U1 @ (U1.T @ np.asarray(X, dtype=np.float64) @ V1) @ V1.T
    if reference is not None:
        Pg = U1 @ (U1.T @ np.asarray(reference, dtype=np.float64) @ V1) @ V1.T
    return float(np.linalg.norm(Xr - Pg) / np.linalg.norm(Pg))
