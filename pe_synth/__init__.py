"""Seeded synthetic inputs for Polar Express -- shared by the oracle tests,
the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no normalisation, no
polynomials, no products of iterates): only random matrices, prescribed
spectra, the Muon layer-set shapes and the bf16 storage format the inputs are
handed over in.  The recipe is stated in DESIGN.md "Inputs".

Workload shapes follow the paper's Muon parameter rule (every >=2-D
parameter except embeddings, unembeddings and positional encodings) for
GPT-2 Small / Large and Llama-3-8B (BASELINE.json configs[3]),
reading R12 of DESIGN.md.
"""
from __future__ import annotations

import numpy as np

# --------------------------------------------------------------------------
# bf16 storage (round-to-nearest-even from float32), as bit patterns.
# --------------------------------------------------------------------------


def f32_to_bf16_bits(x):
    """Round float32 values to bfloat16 (RNE) and return the uint16 bits."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = x.view(np.uint32).astype(np.uint64)
    rounding_bias = ((u >> 16) & 1) + 0x7FFF
    out = ((u + rounding_bias) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        out[nan] = 0x7FC0
    return out


def bf16_bits_to_f32(b):
    b = np.ascontiguousarray(np.asarray(b, dtype=np.uint16))
    return (b.astype(np.uint32) << 16).view(np.float32)


def to_bf16_values(x):
    """float64/float32 array -> float32 array of bf16-representable values."""
    return bf16_bits_to_f32(f32_to_bf16_bits(np.asarray(x, dtype=np.float32)))


# --------------------------------------------------------------------------
# Matrices.
# --------------------------------------------------------------------------


def rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def gaussian(rows, cols, seed=0, std=1.0):
    """Entries N(0, std^2) (numpy PCG64), float64."""
    return rng(seed).standard_normal((rows, cols)) * std


def haar_orthonormal(rows, k, g):
    """rows x k matrix with orthonormal columns, Haar-distributed (QR of a
    Gaussian with the sign of diag(R) folded in)."""
    Z = g.standard_normal((rows, k))
    Q, R = np.linalg.qr(Z)
    d = np.sign(np.diag(R))
    d[d == 0] = 1
    return Q * d


def prescribed_spectrum(rows, cols, sigmas, seed=0):
    """U diag(sigmas) V^T with Haar U (rows x k), V (cols x k), k = len(sigmas)
    <= min(rows, cols)."""
    g = rng(seed)
    k = len(sigmas)
    U = haar_orthonormal(rows, k, g)
    V = haar_orthonormal(cols, k, g)
    return (U * np.asarray(sigmas, dtype=np.float64)) @ V.T


def logspaced(k, kappa):
    """k singular values log-spaced in [1/kappa, 1] (P:367 uses kappa=1e6)."""
    if k == 1:
        return np.ones(1)
    return np.logspace(0, -np.log10(kappa), k)


def power_law(k, p=5.0):
    """sigma_j = j^-p (App. G)."""
    return np.arange(1, k + 1, dtype=np.float64) ** (-p)


def sylvester_hadamard(n):
    """Sylvester Hadamard matrix H_n (n a power of two), entries +-1."""
    assert n >= 1 and (n & (n - 1)) == 0
    H = np.ones((1, 1))
    while H.shape[0] < n:
        H = np.block([[H, H], [H, -H]])
    return H


def hadamard_rows(rows, cols, dtype=np.float64):
    """First min(rows,cols) rows of H_max: all singular values equal to
    sqrt(max(rows, cols)); entries +-1 (exact in bf16).  Tall shapes are the
    transpose.  Built entry-wise from H[i, j] = (-1)^popcount(i & j) (the
    Sylvester recursion), so large shapes need only the m x n result."""
    m, n = min(rows, cols), max(rows, cols)
    assert n >= 1 and (n & (n - 1)) == 0
    i = np.arange(m, dtype=np.uint32)[:, None]
    H = np.empty((m, n), dtype=dtype)
    for j0 in range(0, n, 4096):
        par = np.bitwise_count(i & np.arange(j0, min(n, j0 + 4096), dtype=np.uint32)[None, :]) & 1
        H[:, j0:j0 + par.shape[1]] = 1.0 - 2.0 * par
    return H if rows <= cols else H.T.copy()


def diagonal(rows, cols, sigmas):
    M = np.zeros((rows, cols))
    k = min(rows, cols, len(sigmas))
    M[np.arange(k), np.arange(k)] = sigmas[:k]
    return M


# --------------------------------------------------------------------------
# Muon layer sets (reading R12).  Each entry: (rows, cols, count).
# --------------------------------------------------------------------------

LAYER_SETS = {
    # GPT-2 Small: d=768, 12 layers; q,k,v,o (768x768), c_fc 768x3072, c_proj 3072x768
    "gpt2-small": [(768, 768, 48), (768, 3072, 12), (3072, 768, 12)],
    # GPT-2 Small with the fused attention projection as stored by GPT-2
    # checkpoints (SURVEY §8d config 2 variant): c_attn 768x2304 (q,k,v),
    # attn c_proj 768x768, c_fc 768x3072, mlp c_proj 3072x768 per layer
    "gpt2-small-fused": [(768, 2304, 12), (768, 768, 12), (768, 3072, 12), (3072, 768, 12)],
    # GPT-2 Large: d=1280, 36 layers
    "gpt2-large": [(1280, 1280, 144), (1280, 5120, 36), (5120, 1280, 36)],
    # Llama-3-8B: q,o 4096^2; k,v 1024x4096 (GQA); gate,up 14336x4096; down 4096x14336
    "llama3-8b": [(4096, 4096, 64), (1024, 4096, 64), (14336, 4096, 64), (4096, 14336, 32)],
    # BASELINE.json configs[3] literal reading (no k/v)
    "llama3-8b-literal": [(4096, 4096, 64), (14336, 4096, 64), (4096, 14336, 32)],
    # BASELINE.json configs[0]
    "single-128": [(128, 128, 1)],
}


def layer_set_shapes(name, layers=None):
    """List of (rows, cols) in layer order.  ``layers`` truncates to the first
    k layers (parity subsets)."""
    spec = LAYER_SETS[name]
    if name.startswith("gpt2") or name.startswith("llama"):
        nl = {"gpt2-small": 12, "gpt2-small-fused": 12, "gpt2-large": 36}.get(name, 32)
        per_layer = []
        for r, c, cnt in spec:
            per_layer.append((r, c, cnt // nl))
        shapes = []
        for L in range(nl if layers is None else layers):
            for r, c, k in per_layer:
                shapes += [(r, c)] * k
        return shapes
    out = []
    for r, c, cnt in spec:
        out += [(r, c)] * cnt
    return out
