"""Online stage of Polar Express in fp64 -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

``polar_express`` is Listing 2 written out in numpy fp64 with no
rounding: normalise by ||X||_F * 1.01 + 1e-7 (reading R1), transpose
when rows > cols (reading R10), then for each tuple
A = X X^T; B = b A + c A A; X = a X + B X, repeating the last
tuple past the table (reading R11), transpose back.
"""
from __future__ import annotations

import numpy as np

from .coeffs import odd_poly


def schedule(table, T):
    """Listing 2 ``hs``: the first T tuples, last one repeated."""
    table = [tuple(t) for t in table]
    return table[:T] + [table[-1]] * max(0, T - len(table))


def normalize(M, mode="listing2"):
    """X_0 = M / (||M||_F * 1.01 + 1e-7) (Listing 2) -- reading R1;
    mode 'alg1' gives Alg. 1 line 9's M / (||M||_F + 1e-2)."""
    M = np.asarray(M, dtype=np.float64)
    nrm = np.sqrt(np.sum(M * M))
    if mode == "listing2":
        return M / (nrm * 1.01 + 1e-7)
    if mode == "alg1":
        return M / (nrm + 1e-2)
    raise ValueError(mode)


def polar_express(M, table, T, norm="listing2", return_all=False):
    """Listing 2 in fp64.  M: (rows, cols) array; table: list of
    (a, b, c) (or (a, b) for degree 3) tuples; T: iterations."""
    M = np.asarray(M, dtype=np.float64)
    assert M.ndim == 2
    tall = M.shape[0] > M.shape[1]                     # P:493 (strict, R10)
    X = M.T if tall else M
    X = normalize(X, norm) if norm else X.copy()
    iterates = [X]
    for tup in schedule(table, T):
        A = X @ X.T
        if len(tup) == 3:
            a, b, c = tup
            B = b * A + c * (A @ A)
        else:
            a, b = tup                                 # degree 3: B = b A
            B = b * A
        X = a * X + B @ X
        iterates.append(X)
    if tall:
        X = X.T
        iterates = [Y.T for Y in iterates]
    return (X, iterates) if return_all else X


def exact_polar(M, rtol=1e-13):
    """polar(M) = U V^T from the rank-reduced SVD (eq. (matrixsign), P:51-53;
    notation P:107), singular values below rtol * sigma_max dropped."""
    M = np.asarray(M, dtype=np.float64)
    U, s, Vt = np.linalg.svd(M, full_matrices=False)
    if s.size == 0 or s[0] == 0:
        return np.zeros_like(M)
    keep = s > rtol * s[0]
    return U[:, keep] @ Vt[keep, :]


def composite(x, table, T):
    """Scalar composite p* = p_T o ... o p_1 (eq. (composition))."""
    y = np.asarray(x, dtype=np.float64)
    for tup in schedule(table, T):
        y = odd_poly(tup, y)
    return y


def via_scalar_map(M, table, T, norm="listing2"):
    """X_T = U p*(Sigma_hat) V^T with Sigma_hat the normalised singular values
    (definition of p(M); odd monomials via Gram).  An
    independent route to polar_express's result, used as a pin."""
    M = np.asarray(M, dtype=np.float64)
    U, s, Vt = np.linalg.svd(M, full_matrices=False)
    nrm = np.sqrt(np.sum(s * s))
    if norm == "listing2":
        sh = s / (nrm * 1.01 + 1e-7)
    elif norm == "alg1":
        sh = s / (nrm + 1e-2)
    else:
        sh = s
    return (U * composite(sh, table, T)) @ Vt


def muon_step(W, M, G, beta, lr, table, T):
    """One Muon step in fp64, with polar(M_t) replaced by the Polar
    Express iteration exactly as ``polar_express`` computes it (the method's
    use inside Muon, Listing 2):
        M_t     = beta M_{t-1} + (1 - beta) G_t
        W_{t+1} = W_t - lambda polar(M_t)
    Returns (W_{t+1}, M_t)."""
    W = np.asarray(W, dtype=np.float64)
    Mt = beta * np.asarray(M, dtype=np.float64) + (1.0 - beta) * np.asarray(G, dtype=np.float64)
    return W - lr * polar_express(Mt, table, T), Mt


# ---------------------------------------------------------------- App. G
INIT_Z_MIN = 1.0 / np.sqrt(2.0)     # P:1252 "the intervals do not overlap ... z >= 1/sqrt(2)"
INIT_Z_MAX = 1.0 - 1e-6             # reading R17: numerically rank one -> no init


def power_start(m):
    """The deterministic power-method start vector both sides generate
    (counter based, reading R17): v0_i = frac((i + 1) * phi^-1) + 0.5."""
    i = np.arange(m, dtype=np.float64)
    return np.mod((i + 1) * 0.6180339887498949, 1.0) + 0.5


def init_cubic(z):
    """eq. (init_poly): the odd cubic p(x) = a x + b x^3 with
    p(sqrt(1 - z^2)) = p(z) = 1, for ||M||_F = 1 and sigma_1 in [z, 1]."""
    t = np.sqrt(1.0 - z * z)
    den = z * t * (2.0 * z * z - 1.0)
    return (z * z * (z + t) - t) / den, (t - z) / den


def spectrum_init(X, power_iters):
    """App. G, k = 1: for the normalised iterate X (Listing 2's
    X_0, ||X||_F = F), estimate z = sigma~_1 / F from below by the power
    method on A = X X^T (the k = 1 case of the footnote's subspace iteration,
    P:1237-1239: Rayleigh quotient of the last vector, sigma~_1 <= sigma_1),
    and if 1/sqrt(2) <= z apply p(x) = a (x/F) + b (x/F)^3 with
    (a, b) = init_cubic(z) exactly as eq. (init_poly) gives them (
    App. G assumes ||M||_F = 1, hence the x/F -- reading R17), i.e.
    X <- (a/F) X + (b/F^3) A X.  Nothing else: the product's bf16 margin
    (reading R17) is the product's own stabilisation and is gated against
    this step, not built into it.  Returns (X', z, applied)."""
    X = np.asarray(X, dtype=np.float64)
    F = np.sqrt(np.sum(X * X))
    A = X @ X.T
    v = power_start(A.shape[0])
    lam = 0.0
    for _ in range(power_iters):
        w = A @ v
        lam = float(v @ w) / float(v @ v)          # Rayleigh quotient <= lambda_max(A)
        v = w / np.sqrt(float(w @ w))
    z = np.sqrt(max(lam, 0.0)) / F if F > 0 else 0.0
    if not (INIT_Z_MIN <= z <= INIT_Z_MAX):
        return X, z, False
    a, b = init_cubic(z)                           # eq. (init_poly)
    return (a / F) * X + (b / F ** 3) * (A @ X), z, True


def polar_express_init(M, table, T, power_iters=8, norm="listing2"):
    """Polar Express with App. G's spectrum-aware first step: normalise and
    orient as Listing 2, apply ``spectrum_init``,
    then the T Listing 2 iterations, transpose back."""
    M = np.asarray(M, dtype=np.float64)
    tall = M.shape[0] > M.shape[1]
    X = M.T if tall else M
    X = normalize(X, norm)
    X, z, applied = spectrum_init(X, power_iters)
    for tup in schedule(table, T):
        A = X @ X.T
        a, b, c = tup
        X = a * X + (b * A + c * (A @ A)) @ X
    return (X.T if tall else X), z, applied
