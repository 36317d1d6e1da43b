"""Scalar emulation of the bf16 rounding points of the GPU design (DESIGN.md
reading R8) -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Used only where it is exact: diagonal inputs M = diag(sigma) (zero padded).
There every product the kernels form has at most one non-zero term, products
of two bf16 values are exact in fp32, and zeros stay zeros, so the diagonal
of the GPU result must equal this emulation bit for bit.  It is written from
the reading, not from the kernels (the two share no code):

  R2/R8 normalisation: s = sqrt(sum x^2) * 1.01 + 1e-7 in fp64,
        inv = fp32(1/s)
  folded inputs (rows of 16-byte multiples; X_0 = M/s is never rounded):
        Gram 1:    A = bf16(fp32(x*x) * fp32(inv*inv))
        update 1:  X_1 = bf16(fp32(fp32(a*x) + B*x) * inv)
  other inputs: X_0 = bf16(fp32(x) * inv), then the generic steps
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


def diagonal_bf16(sigmas_bf16, table, T, folded=True):
    """Diagonal of the GPU's bf16 result for M = diag(sigmas) (any padding).
    ``sigmas_bf16`` must already be bf16 values (the GPU input); ``folded``
    says whether the normalisation is folded into the first iteration (the
    path the GPU takes when the caller's rows are 16-byte multiples)."""
    s = np.asarray(sigmas_bf16, dtype=np.float32)
    sumsq = float(np.sum(s.astype(np.float64) ** 2))
    nrm = np.sqrt(sumsq) * 1.01 + 1e-7
    inv = np.float32(1.0 / nrm)
    x = s.copy() if folded else _bf16(s * inv)
    for it, tup in enumerate(schedule(table, T)):
        a = np.float32(tup[0])
        b = np.float32(tup[1])
        first = folded and it == 0
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
