"""Scalar emulation of the bf16 rounding points of the GPU design (DESIGN.md
reading R8) -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Used only where it is exact: diagonal inputs M = diag(sigma) (zero padded).
There every product the kernels form has at most one non-zero term, products
of two bf16 values are exact in fp32, and zeros stay zeros, so the diagonal
of the GPU result must equal this emulation bit for bit.  It is written from
the reading, not from the kernels (the two share no code):

  R2/R8 normalisation: s = sqrt(sum x^2) * 1.01 + 1e-7 in fp64,
        inv = fp32(1/s)
  bf16 inputs (``folded=True``; X_0 = M/s is never rounded -- rows of
  16-byte multiples are read in place, others through an exact copy
  M 2^e with 1/s 2^-e applied below, which is bit-identical):
        Gram 1:    A = bf16(fp32(x*x) * fp32(inv*inv))
        update 1:  X_1 = bf16(fp32(fp32(a*x) + B*x) * inv)
  fp32 inputs of pe_polar_ex (``folded=False``): X_0 = bf16(fp32(x) * inv),
  then the generic steps
  Gram:      A = bf16(x*x)
  poly:      B = bf16(fp32(b*A) + fp32(c*(A*A)))   (no FMA contraction)
  update:    X' = bf16(fp32(a*X) + (B*X))          (no FMA contraction)
  degree 3 (B = b A, eq. deg3_solution): B is never formed;
                     X' = bf16(fp32(a*X) + fp32(b*(A*X)))
with a, b, c the fp32-rounded table entries.
"""
from __future__ import annotations

import numpy as np

from .iteration import schedule


def _bf16(x):
    """Round float32 -> bfloat16 (RNE), returned as float32 values."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = x.view(np.uint32).astype(np.uint64)
    u = ((u + (((u >> 16) & 1) + 0x7FFF)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def _split2(v):
    """Two bf16 planes of fp32 values: (bf16(v), bf16(v - bf16(v)))."""
    v = np.asarray(v, dtype=np.float32)
    p0 = _bf16(v)
    return p0, _bf16(np.float32(v - p0))


def diagonal_bf16(sigmas_bf16, table, T, folded=True, ab_planes=1):
    """Diagonal of the GPU's bf16 result for M = diag(sigmas) (any padding).
    ``sigmas_bf16`` must already be bf16 values (the GPU input); ``folded``
    says whether the normalisation is folded into the first iteration (the
    path the GPU takes for every bf16 input; ``False``: an explicit rounded
    X_0, the fp32-input path).
    ``ab_planes = 2``: the small path's precise variant (reading R8p): A and
    B kept as two bf16 planes; a product with a two-plane operand is its big
    plane product plus the small ones, one fp32 add."""
    s = np.asarray(sigmas_bf16, dtype=np.float32)
    sumsq = float(np.sum(s.astype(np.float64) ** 2))
    nrm = np.sqrt(sumsq) * 1.01 + 1e-7
    inv = np.float32(1.0 / nrm)
    x = s.copy() if folded else _bf16(s * inv)
    for it, tup in enumerate(schedule(table, T)):
        a = np.float32(tup[0])
        b = np.float32(tup[1])
        first = folded and it == 0
        if ab_planes == 2:
            acc = np.float32(np.float32(x * x) * np.float32(inv * inv)) if first else np.float32(x * x)
            A0, A1 = _split2(acc)
            Af = np.float32(A0 + A1)
            if len(tup) == 3:
                c = np.float32(tup[2])
                w = np.float32(np.float32(A0 * A0) + np.float32(2.0 * np.float32(A1 * A0)))
                B0, B1 = _split2(np.float32(b * Af) + np.float32(c * w))
                BX = np.float32(np.float32(B0 * x) + np.float32(B1 * x))
            else:
                BX = np.float32(b * np.float32(np.float32(A0 * x) + np.float32(A1 * x)))
            if first:
                x = _bf16(np.float32(np.float32(a * x) + BX) * inv)
            else:
                x = _bf16(np.float32(a * x) + BX)
            continue
        A = _bf16(np.float32(x * x) * np.float32(inv * inv)) if first else _bf16(x * x)
        if len(tup) == 3:
            c = np.float32(tup[2])
            B = _bf16(np.float32(b * A) + np.float32(c * np.float32(A * A)))
            BX = np.float32(B * x)
        else:
            BX = np.float32(b * np.float32(A * x))
        if first:
            x = _bf16(np.float32(np.float32(a * x) + BX) * inv)
        else:
            x = _bf16(np.float32(a * x) + BX)
    return x


def r8_polar_express(M_bf16, table, T, folded=True, ab_planes=1):
    """The bf16 design of reading R8 on a general matrix: bf16 operands and an
    exact-products accumulation rounded once to fp32 (fp64 matmul of the
    bf16-valued operands, then fp32 -- the tensor cores' fp32 accumulation
    differs only in its order and truncation.),
    and the same rounding points as ``diagonal_bf16`` (which it equals bit for
    bit on diagonal inputs -- its pin).  Listing 2's orientation (P:493,
    P:501).  Used to measure how widely the design's own rounding points
    spread against the fp64 oracle (tests/test_r8_spread.py), i.e. what a
    bf16 gate can demand of the GPU at a given size.  ``ab_planes = 2`` is
    the small path's precise variant (R8p, as ``diagonal_bf16``)."""
    def mm(P, Q):
        return (P.astype(np.float64) @ Q.astype(np.float64)).astype(np.float32)

    M = np.asarray(M_bf16, dtype=np.float32)
    tall = M.shape[0] > M.shape[1]
    X = (M.T if tall else M).copy()
    nrm = np.sqrt(float(np.sum(X.astype(np.float64) ** 2))) * 1.01 + 1e-7
    inv = np.float32(1.0 / nrm)
    if not folded:
        X = _bf16(X * inv)
    for it, tup in enumerate(schedule(table, T)):
        a, b = np.float32(tup[0]), np.float32(tup[1])
        first = folded and it == 0
        acc = mm(X, X.T)
        if ab_planes == 2:
            A0, A1 = _split2(np.float32(acc * np.float32(inv * inv)) if first else acc)
            Af = np.float32(A0 + A1)
            if len(tup) == 3:
                c = np.float32(tup[2])
                w = np.float32(mm(A0, A0.T) + (mm(A1, A0.T) + mm(A0, A1.T)).astype(np.float32))
                B0, B1 = _split2(np.float32(b * Af) + np.float32(c * w))
                BX = np.float32(mm(B0, X) + mm(B1, X))
            else:
                BX = np.float32(b * np.float32(mm(A0, X) + mm(A1, X)))
            X = _bf16(np.float32(np.float32(a * X) + BX) * inv) if first else _bf16(np.float32(a * X) + BX)
            continue
        A = _bf16(acc * np.float32(inv * inv)) if first else _bf16(acc)
        if len(tup) == 3:
            c = np.float32(tup[2])
            B = _bf16(np.float32(b * A) + np.float32(c * mm(A, A)))
            BX = mm(B, X)
        else:
            BX = np.float32(b * mm(A, X))
        X = _bf16(np.float32(np.float32(a * X) + BX) * inv) if first else _bf16(np.float32(a * X) + BX)
    return X.T if tall else X


def _sym_upper(S, blk=256):
    """The symmetric matrix a kernel that stores only the blk x blk blocks on
    or above the block diagonal hands to its consumers: blocks below the
    diagonal are the transposes of the stored ones."""
    n = S.shape[0]
    bi = np.arange(n) // blk
    lower = bi[:, None] > bi[None, :]
    return np.where(lower, S.T, S)


def r19_alg4(M_bf16, table, T, restart=None, shift=1e-3, folded=True):
    """The bf16 design of Alg. 4 (App. H) on the GPU (DESIGN.md
    reading R19), in the wide orientation with products accumulated exactly
    and rounded once to fp32 (as r8_polar_express):
        Y   = bf16(fp32(acc [* inv^2]) + shift)   acc = X X^T (shift: first application)
        H_1 = bf16(fp32(b Y) + fp32(c acc))       acc = Y Y
        Q_1 = H_1, diagonal bf16(fp32(H_1) + a)
        then per further iteration t of the application:
        T   = bf16(acc)   acc = Y Q
        R   = bf16(acc)   acc = Q T   (upper blocks stored, symmetrised)
        H   = bf16(fp32(b R) + fp32(c acc))       acc = R R (the true product:
              R is not symmetric inside its diagonal blocks; upper blocks
              stored, symmetrised)
        Q   = bf16(fp32(a Q) + acc)               acc = H Q
        X'  = bf16(acc [* inv])                   acc = Q X
    An application of one iteration is Listing 2's step (r8).  Equal to the
    GPU bit for bit on diagonal inputs (every product has one term)."""
    def mm(P, Q):
        return (P.astype(np.float64) @ Q.astype(np.float64)).astype(np.float32)

    M = np.asarray(M_bf16, dtype=np.float32)
    tall = M.shape[0] > M.shape[1]
    X = (M.T if tall else M).copy()
    nrm = np.sqrt(float(np.sum(X.astype(np.float64) ** 2))) * 1.01 + 1e-7
    inv = np.float32(1.0 / nrm)
    inv2 = np.float32(inv * inv)
    if not folded:
        X = _bf16(X * inv)
    tups = schedule(table, T)
    k = T if restart is None else min(int(restart), T)
    m = X.shape[0]
    eye = np.eye(m, dtype=bool)
    for b, t0 in enumerate(range(0, T, k)):
        first = b == 0
        scaled = folded and first
        sh = np.float32(shift if first else 0.0)
        blk = tups[t0:t0 + k]
        a, bb, c = (np.float32(v) for v in blk[0])
        acc = mm(X, X.T)
        if scaled:
            acc = np.float32(acc * inv2)
        Y = _bf16(np.where(eye, np.float32(acc + sh), acc))
        H = _bf16(np.float32(bb * Y) + np.float32(c * mm(Y, Y)))
        if len(blk) == 1:
            Xn = np.float32(np.float32(a * X) + mm(H, X))
            X = _bf16(np.float32(Xn * inv) if scaled else Xn)
            continue
        Q = np.where(eye, _bf16(np.float32(H + a)), H)
        for tup in blk[1:]:
            a, bb, c = (np.float32(v) for v in tup)
            Tm = _bf16(mm(Y, Q))
            R = _sym_upper(_bf16(mm(Q, Tm)))
            H = _sym_upper(_bf16(np.float32(bb * R) + np.float32(c * mm(R, R))))
            Q = _bf16(np.float32(a * Q) + mm(H, Q))
        acc = mm(Q, X)
        X = _bf16(np.float32(acc * inv) if scaled else acc)
    return X.T if tall else X


def r17_init_polar_express(M_bf16, table, T, power_iters, folded=True):
    """App. G's first step at the GPU design's rounding points
    (reading R17), then ``T`` iterations as ``r8_polar_express``:
        acc = X X^T  (exact, rounded once to fp32; X = M when folded, else
                      X_0 = bf16(M inv))
        z   = sqrt(lambda / d): lambda the Rayleigh quotient of ``power_iters``
              power steps on the fp32 acc (start vector of iteration.power_start),
              d = ||M||^2 (folded) or trace(acc) = ||X_0||^2 of the rounded X_0
        (a, b) = eq. (init_poly) at z when 1/sqrt(2) <= z <= 1 - 1e-6,
              else (1, 0); F^2 = ||M||^2 inv^2 (folded) or trace(acc);
              a' = fp32(a / F), b' = fp32(b / F^3)
        A_0 = bf16(acc [* inv^2])
        X_1 = bf16(fp32(fp32(a' X) + fp32(b' (A_0 X))) [* inv])
    Used to measure how far the bf16 design's own rounding of this step
    (the b / F^3 ~ 1 / sqrt(1 - z^2) amplification of A_0's rounding as
    z -> 1) moves the result from the fp64 step.  Returns (X_T, z, applied)."""
    from .iteration import power_start, init_cubic, INIT_Z_MIN, INIT_Z_MAX

    def mm(P, Q):
        return (P.astype(np.float64) @ Q.astype(np.float64)).astype(np.float32)

    M = np.asarray(M_bf16, dtype=np.float32)
    tall = M.shape[0] > M.shape[1]
    X = (M.T if tall else M).copy()
    ssq = float(np.sum(X.astype(np.float64) ** 2))
    nrm = np.sqrt(ssq) * 1.01 + 1e-7
    inv = np.float32(1.0 / nrm)
    if not folded:
        X = _bf16(X * inv)
    acc = mm(X, X.T)
    if folded:
        f2 = ssq * float(inv) * float(inv)
        d = ssq
    else:                       # X_0 rounded: its norm from the same Gram (trace)
        f2 = d = float(np.sum(np.diag(acc).astype(np.float64)))
    A64 = acc.astype(np.float64)
    v = power_start(A64.shape[0])
    lam = 0.0
    for _ in range(power_iters):
        w = A64 @ v
        lam = float(v @ w) / float(v @ v)
        v = w / np.sqrt(float(w @ w))
    z = np.sqrt(lam / d) if d > 0 and lam > 0 else 0.0
    applied = INIT_Z_MIN <= z <= INIT_Z_MAX
    if applied:
        a, b = init_cubic(z)
        F = np.sqrt(f2)
        ca, cb = np.float32(a / F), np.float32(b / F ** 3)
    else:
        ca, cb = np.float32(1.0), np.float32(0.0)
    A0 = _bf16(np.float32(acc * np.float32(inv * inv))) if folded else _bf16(acc)
    X1 = np.float32(np.float32(ca * X) + np.float32(cb * mm(A0, X)))
    X = _bf16(np.float32(X1 * inv)) if folded else _bf16(X1)
    for tup in schedule(table, T):
        a, b = np.float32(tup[0]), np.float32(tup[1])
        A = _bf16(mm(X, X.T))
        if len(tup) == 3:
            c = np.float32(tup[2])
            B = _bf16(np.float32(b * A) + np.float32(c * mm(A, A)))
            BX = mm(B, X)
        else:
            BX = np.float32(b * mm(A, X))
        X = _bf16(np.float32(a * X) + BX)
    return (X.T if tall else X), z, applied
