"""Independent bit-level pin of oracle/emulate.py (reading R8).

``emulate.diagonal_bf16`` predicts, bit for bit, the diagonal of the GPU's
bf16 result on diagonal inputs (the GPU test ``test_diagonal_bit_exact``
relies on it).  Here it is checked against a second implementation written
from the text of reading R8 alone, with no numpy float arithmetic at all:
every value is an exact ``fractions.Fraction`` and every rounding point the
reading names is an explicit round-to-nearest-even to the stated format
(fp64 = 53 significand bits, fp32 = 24, bf16 = 8).  Reading R8:

  s = sqrt(sum x^2) * 1.01 + 1e-7 in fp64, inv = fp32(1/s)
  folded first iteration:  A_1 = bf16(fp32(acc) * fp32(inv * inv)),  acc = x x
                           X_1 = bf16(fp32(fp32(a x) + acc) * inv),   acc = B_1 x
  explicit X_0 (unfolded): X_0 = bf16(fp32(x) * inv)
  Gram:          A  = bf16(acc),                           acc = x x
  poly:          B  = bf16(fp32(b A) + fp32(c acc)),       acc = A A
  update:          X' = bf16(fp32(a X) + acc),               acc = B X
  degree 3:        no B;  X' = bf16(fp32(a X) + fp32(b acc)), acc = A X
  a, b, c the table entries rounded to fp32; fp32 products of two bf16
  values are exact (on a diagonal every accumulator holds one product).

The planted-change tests show the pin is sharp: each one-rounding-point
variant of the reading (A or B or X_0 left in fp32, A rounded before the
folded 1/s^2 scale, an FMA-contracted update) disagrees
with ``emulate`` on some of the inputs on which the unplanted pin agrees.
"""
import math
from fractions import Fraction as Fr

import numpy as np
import pytest

import pe_synth as syn
from oracle import coeffs as oc
from oracle import emulate
from oracle.iteration import schedule

TABLE, _ = oc.pe_coeffs(1e-3, 5, 8, 1.01)


def rne(x, p, emin=-126):
    """Round the exact rational x to the nearest binary float with p
    significand bits and minimum normal exponent emin (ties to even)."""
    if x == 0:
        return Fr(0)
    sgn = -1 if x < 0 else 1
    x = abs(x)
    e = x.numerator.bit_length() - x.denominator.bit_length()      # 2^e <= x < 2^(e+2)
    if Fr(2) ** e > x:
        e -= 1
    while Fr(2) ** (e + 1) <= x:
        e += 1
    e = max(e, emin)
    ulp = Fr(2) ** (e - p + 1)
    q = x / ulp
    n = q.numerator // q.denominator
    r = q - n
    if r > Fr(1, 2) or (r == Fr(1, 2) and n % 2 == 1):
        n += 1
    return sgn * n * ulp


def f64(x):
    return rne(x, 53, -1022)


def f32(x):
    return rne(x, 24)


def bf16(x):
    return rne(x, 8)


def sqrt64(x):
    """Correctly rounded fp64 square root of a non-negative rational."""
    if x == 0:
        return Fr(0)
    k = 200                                   # 2^-200 resolution >> 53 bits
    n = (x.numerator << (2 * k)) // x.denominator
    lo = Fr(math.isqrt(n), 2 ** k)            # sqrt(x) in [lo, lo + 2^-k)
    a, b = f64(lo), f64(lo + Fr(1, 2 ** k))
    assert a == b                             # irrational or exact: no tie within 2^-200
    return a


def pin_trajectory_r8p(sig_bf16, tuples, folded):
    """Reading R8p (the small path's two-plane A/B variant) on
    M = diag(sig): A = split2(fp32 acc [* inv^2]); a product with a two-plane
    operand = fp32(big plane product + fp32(sum of the small ones));
    B = split2(fp32(b (A0 + A1)) + fp32(c (A A))); X' = bf16(fp32(a X) + B X)."""
    xs = [Fr(float(v)) for v in sig_bf16]
    sumsq = sum(x * x for x in xs)
    s = f64(f64(sqrt64(sumsq) * Fr(1.01)) + Fr(1e-7))
    inv = f32(f64(Fr(1) / s))
    inv2 = f32(inv * inv)
    x = list(xs) if folded else [bf16(f32(v * inv)) for v in xs]

    def split2(v):
        p0 = bf16(v)
        return p0, bf16(f32(v - p0))

    out = []
    for it, tup in enumerate(tuples):
        a, b = f32(Fr(tup[0])), f32(Fr(tup[1]))
        c = f32(Fr(tup[2])) if len(tup) == 3 else None
        first = folded and it == 0
        nx = []
        for v in x:
            acc = v * v
            A0, A1 = split2(f32(f32(acc) * inv2) if first else f32(acc))
            if c is not None:
                w = f32(A0 * A0 + f32(2 * A1 * A0))
                B0, B1 = split2(f32(f32(b * f32(A0 + A1)) + f32(c * w)))
                bx = f32(B0 * v + f32(B1 * v))
            else:
                bx = f32(b * f32(A0 * v + f32(A1 * v)))
            y = bf16(f32(f32(f32(a * v) + bx) * inv)) if first else bf16(f32(f32(a * v) + bx))
            nx.append(y)
        x = nx
        out.append(x)
    return out


def pin_trajectory(sig_bf16, tuples, folded, variant=None):
    """Reading R8 on M = diag(sig): the bf16 diagonal after each iteration
    (list of lists of Fractions).  ``variant`` plants one changed rounding
    point (for the sharpness tests)."""
    xs = [Fr(float(v)) for v in sig_bf16]
    sumsq = sum(x * x for x in xs)                 # exact; the GPU's fp64 sum is exact for these inputs
    s = f64(f64(sqrt64(sumsq) * Fr(1.01)) + Fr(1e-7))
    inv = f32(Fr(1) / s) if variant == "inv_direct" else f32(f64(Fr(1) / s))
    inv2 = f32(inv * inv)
    if folded:
        x = list(xs)
    elif variant == "X0_fp32":
        x = [f32(v * inv) for v in xs]
    else:
        x = [bf16(f32(v * inv)) for v in xs]
    cr = (lambda v: Fr(v)) if variant == "coeff_f64" else (lambda v: f32(Fr(v)))
    out = []
    for it, tup in enumerate(tuples):
        a, b = cr(tup[0]), cr(tup[1])
        c = cr(tup[2]) if len(tup) == 3 else None
        first = folded and it == 0
        nx = []
        for v in x:
            acc = v * v                                           # exact
            A = bf16(f32(f32(acc) * inv2)) if first else bf16(acc)
            if variant == "A_fp32":
                A = f32(f32(acc) * inv2) if first else f32(acc)
            elif variant == "A_round_then_scale" and first:
                A = bf16(f32(bf16(acc) * inv2))
            if c is None:
                B = None
            elif variant == "poly_fma":
                B = bf16(f32(b * A + c * (A * A)))
            elif variant == "B_fp32":
                B = f32(f32(b * A) + f32(c * (A * A)))
            else:
                B = bf16(f32(b * A) + f32(c * (A * A)))
            acc = B * v if B is not None else f32(b * (A * v))     # cubic: b (A X), B never formed
            if first:
                if variant == "inv_early":
                    y = bf16(f32(f32(a * v) * inv + f32(acc * inv)))
                else:
                    y = bf16(f32(f32(f32(a * v) + acc) * inv))
            elif variant == "update_fma":
                y = bf16(f32(a * v + acc))
            else:
                y = bf16(f32(f32(a * v) + acc))
            nx.append(y)
        x = nx
        out.append(x)
    return out


def _sigma_sets():
    """512 bf16 singular values in four sets: log-spaced over [2^-6, 1] (a
    wide spread of normalised values, most on the steep part of p_1), random
    in [2^-4, 2^3], clustered near the top (sigma-hat near 1/1.01 / sqrt(k)),
    and one with an outlier.  Squares of bf16 values in these ranges sum
    exactly in fp64 whatever the order (checked), so the GPU's and numpy's
    fp64 norms equal the exact one."""
    rng = np.random.default_rng(20260)
    sets = [np.geomspace(2.0 ** -6, 1.0, 128),
            rng.uniform(2.0 ** -4, 8.0, 128),
            1.0 - rng.uniform(0, 0.05, 128),
            np.concatenate([[40.0], rng.uniform(0.01, 1.0, 127)])]
    out = []
    for s in sets:
        b = syn.to_bf16_values(s).astype(np.float32)
        exact = sum(Fr(float(v)) ** 2 for v in b)
        assert Fr(float(np.sum(b.astype(np.float64) ** 2))) == exact
        out.append(b)
    return out


def _bits(v):
    return np.asarray(v, dtype=np.float32).view(np.uint32)


@pytest.mark.parametrize("folded", [True, False])
def test_emulation_bit_exact_against_fraction_pin(folded):
    """emulate.diagonal_bf16 == the Fraction pin, bit for bit, on 512 sigma
    values, T = 1..8 (degree-5 table of Listing 2 with safety)."""
    for sig in _sigma_sets():
        traj = pin_trajectory(sig, schedule(TABLE, 8), folded)
        for T in range(1, 9):
            emu = emulate.diagonal_bf16(sig, TABLE, T, folded=folded)
            pin = np.array([float(v) for v in traj[T - 1]], dtype=np.float32)
            assert np.array_equal(_bits(emu), _bits(pin)), (folded, T, np.flatnonzero(_bits(emu) != _bits(pin))[:5])


@pytest.mark.parametrize("folded", [True, False])
def test_r8p_emulation_bit_exact_against_fraction_pin(folded):
    """The two-plane small-path variant (R8p): emulate.diagonal_bf16(...,
    ab_planes=2) == its exact-rational pin bit for bit (256 sigma values,
    T = 1..6, degree 5 and 3)."""
    tab3, _ = oc.pe_coeffs(1e-3, 3, 8, 1.01)
    for sig in _sigma_sets()[:2]:
        for tab in (TABLE, tab3):
            traj = pin_trajectory_r8p(sig, schedule(tab, 6), folded)
            for T in range(1, 7):
                emu = emulate.diagonal_bf16(sig, tab, T, folded=folded, ab_planes=2)
                pin = np.array([float(v) for v in traj[T - 1]], dtype=np.float32)
                assert np.array_equal(_bits(emu), _bits(pin)), (folded, T, len(tab[0]))


def test_emulation_bit_exact_degree3_table():
    """Same pin for a degree-3 table (eq. deg3_solution; the product
    never forms B = b A: X' = a X + b (A X)), both paths."""
    tab3, _ = oc.pe_coeffs(1e-3, 3, 8, 1.01)
    sig = _sigma_sets()[0]
    for folded in (True, False):
        traj = pin_trajectory(sig, schedule(tab3, 6), folded)
        for T in range(1, 7):
            emu = emulate.diagonal_bf16(sig, tab3, T, folded=folded)
            pin = np.array([float(v) for v in traj[T - 1]], dtype=np.float32)
            assert np.array_equal(_bits(emu), _bits(pin)), (folded, T)


# A tuple under which an FMA-contracted update (a x + acc rounded once)
# flips a bf16 bit at T = 1 on the second sigma set (unfolded): found by a
# numpy search over random fp32 tuples (11k tries).  With Listing 2's own
# table the contraction changes no bit of these inputs -- it moves the fp32
# sum by <= 1 fp32 ulp, which survives the bf16 rounding only within ~2^-16
# of a bf16 midpoint -- so it is immaterial to accuracy; the pin still
# separates the two rounding orders whenever they differ.
FMA_TUPLE = (4.334741592407227, -1.6090689897537231, 12.14086627960205)


@pytest.mark.parametrize("variant,folded,table,T_max", [
    ("A_fp32", False, None, 8),               # A kept in fp32 (not rounded to bf16)
    ("A_round_then_scale", True, None, 2),    # folded Gram: round acc to bf16 before the 1/s^2 scale
    ("B_fp32", True, None, 3),                # B kept in fp32
    ("X0_fp32", False, None, 2),              # explicit X_0 not rounded to bf16
    ("update_fma", False, [FMA_TUPLE], 1),    # a x + acc contracted into one rounding
])
def test_planted_rounding_changes_are_caught(variant, folded, table, T_max):
    """Sharpness: moving one rounding point of reading R8 changes at least
    one predicted bit pattern on these inputs, while the unplanted pin agrees
    with ``emulate`` on the same inputs (so the bit-exact pin above, and the
    GPU's diagonal test, would catch that mistake in emulate.py or in the
    kernels)."""
    tab = TABLE if table is None else table
    differs = False
    for sig in _sigma_sets():
        planted = pin_trajectory(sig, schedule(tab, T_max), folded, variant=variant)
        clean = pin_trajectory(sig, schedule(tab, T_max), folded)
        for T in range(1, T_max + 1):
            emu = _bits(emulate.diagonal_bf16(sig, tab, T, folded=folded))
            assert np.array_equal(emu, _bits(np.array([float(v) for v in clean[T - 1]], dtype=np.float32)))
            if not np.array_equal(emu, _bits(np.array([float(v) for v in planted[T - 1]], dtype=np.float32))):
                differs = True
    assert differs, variant


def test_rne_helper_against_hardware_formats():
    """The pin's rounding helper agrees with numpy's IEEE fp32 conversion and
    the bf16 RNE conversion of pe_synth on random and tie cases."""
    rng = np.random.default_rng(1)
    for v in np.concatenate([rng.standard_normal(200) * 10.0 ** rng.integers(-8, 8, 200),
                             [1 + 2.0 ** -24, 1 + 3 * 2.0 ** -24, 1 + 2.0 ** -8, 1 + 3 * 2.0 ** -8]]):
        assert float(f32(Fr(float(v)))) == float(np.float32(v))
        assert float(bf16(Fr(float(np.float32(v))))) == float(syn.to_bf16_values(np.array([v], np.float32))[0])
    assert sqrt64(Fr(2)) == Fr(float(np.sqrt(2.0))) and sqrt64(Fr(9, 4)) == Fr(3, 2)
