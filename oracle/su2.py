"""Exact SU(2) data for the oracle (test infrastructure).

All spins are DOUBLED integers (J = 2j, M = 2m). Clebsch-Gordan coefficients
and 6j symbols are built exactly as  s * sqrt(r)  with s, r Fractions
(BASELINE cfg5: "computed independently by the oracle in exact rational
arithmetic"), then rounded once to float64.

  cg6 / cg   Condon-Shortley CG via the Racah closed form (textbook; these are
             the components of the splitting tensors X^{ab}_c)
  sixj       Racah sum for the Wigner 6j symbol
  fsymbol    the paper's Eq. SU2FSymbol, P:2318-2325 (reading C9 for the argument order)
  rsymbol    reading C8: R^{j1 j2}_{j3} = (-1)^{j1+j2-j3}; the printed (-1)^{j1+j2+j3}
              violates the unit axiom for half-integer j3 (C8)
  z_flip     reading C7: Z_j <j m| = (-1)^{j-m} |j,-m>
"""
from fractions import Fraction
from functools import lru_cache
import math

import numpy as np


@lru_cache(maxsize=None)
def _f(n):
    if n < 0:
        raise ValueError("negative factorial")
    return math.factorial(n)


def _half(x):
    if x % 2:
        raise ValueError("non-integer half")
    return x // 2


def triangle(a, b, c):
    """Doubled spins a, b, c admissible: |a-b| <= c <= a+b and a+b+c even."""
    return abs(a - b) <= c <= a + b and (a + b + c) % 2 == 0


@lru_cache(maxsize=None)
def cg_exact(j1, m1, j2, m2, J, M):
    """<j1 m1 j2 m2 | J M> as (s, r) with value s*sqrt(r), Fractions (Racah formula)."""
    if m1 + m2 != M or not triangle(j1, j2, J):
        return Fraction(0), Fraction(0)
    for j, m in ((j1, m1), (j2, m2), (J, M)):
        if abs(m) > j or (j - m) % 2:
            return Fraction(0), Fraction(0)
    r = Fraction((J + 1) * _f(_half(J + j1 - j2)) * _f(_half(J - j1 + j2)) * _f(_half(j1 + j2 - J)),
                 _f(_half(j1 + j2 + J) + 1))
    r *= _f(_half(J + M)) * _f(_half(J - M)) * _f(_half(j1 - m1)) * _f(_half(j1 + m1)) \
        * _f(_half(j2 - m2)) * _f(_half(j2 + m2))
    s = Fraction(0)
    for k in range(0, _half(j1 + j2 - J) + 1):
        args = (k, _half(j1 + j2 - J) - k, _half(j1 - m1) - k, _half(j2 + m2) - k,
                _half(J - j2 + m1) + k, _half(J - j1 - m2) + k)
        if min(args) < 0:
            continue
        den = 1
        for x in args:
            den *= _f(x)
        s += Fraction((-1) ** k, den)
    return s, r


def cg(j1, m1, j2, m2, J, M):
    s, r = cg_exact(j1, m1, j2, m2, J, M)
    return float(s) * math.sqrt(float(r)) if s != 0 else 0.0


def mvals(j):
    """Doubled magnetic numbers in basis order mu = 0..2j  <->  m = j - mu."""
    return [j - 2 * mu for mu in range(j + 1)]


@lru_cache(maxsize=None)
def cg_tensor(j1, j2, J):
    """Array X[mu1, mu2, muJ] = <j1 m1 j2 m2 | J M>: the splitting tensor V_J -> V_j1 (x) V_j2."""
    X = np.zeros((j1 + 1, j2 + 1, J + 1))
    for a, m1 in enumerate(mvals(j1)):
        for b, m2 in enumerate(mvals(j2)):
            M = m1 + m2
            if abs(M) <= J:
                X[a, b, _half(J - M)] = cg(j1, m1, j2, m2, J, M)
    X.setflags(write=False)
    return X


def _delta(a, b, c):
    return Fraction(_f(_half(a + b - c)) * _f(_half(a - b + c)) * _f(_half(-a + b + c)), _f(_half(a + b + c) + 1))


@lru_cache(maxsize=None)
def sixj_exact(j1, j2, j3, j4, j5, j6):
    """Wigner 6j {j1 j2 j3; j4 j5 j6} (doubled) as (s, r): value s*sqrt(r). Racah sum."""
    tri = ((j1, j2, j3), (j1, j5, j6), (j4, j2, j6), (j4, j5, j3))
    if not all(triangle(*t) for t in tri):
        return Fraction(0), Fraction(0)
    r = Fraction(1)
    for t in tri:
        r *= _delta(*t)
    lo = max(_half(sum(t)) for t in tri)
    hi = min(_half(j1 + j2 + j4 + j5), _half(j2 + j3 + j5 + j6), _half(j3 + j1 + j6 + j4))
    s = Fraction(0)
    for t in range(lo, hi + 1):
        den = 1
        for x in (t - _half(j1 + j2 + j3), t - _half(j1 + j5 + j6), t - _half(j4 + j2 + j6),
                  t - _half(j4 + j5 + j3), _half(j1 + j2 + j4 + j5) - t, _half(j2 + j3 + j5 + j6) - t,
                  _half(j3 + j1 + j6 + j4) - t):
            den *= _f(x)
        s += Fraction((-1) ** t * _f(t + 1), den)
    return s, r


def sixj(j1, j2, j3, j4, j5, j6):
    s, r = sixj_exact(j1, j2, j3, j4, j5, j6)
    return float(s) * math.sqrt(float(r)) if s != 0 else 0.0


def fsymbol_exact(j1, j2, j3, j4, e, f):
    """Eq. SU2FSymbol: F^{j1 j2 j3}_{j4}[e, f] = sqrt(d_e d_f) (-1)^{j1+j2+j3+j4} {j1 j2 e; j3 j4 f}.

    e = left inner label (j1 j2 -> e), f = right inner label (j2 j3 -> f) (reading C9).
    Returned exactly as (s, r).
    """
    s, r = sixj_exact(j1, j2, e, j3, j4, f)
    if s == 0:
        return Fraction(0), Fraction(0)
    sign = -1 if _half(j1 + j2 + j3 + j4) % 2 else 1
    return sign * s, r * (e + 1) * (f + 1)


def fsymbol(j1, j2, j3, j4, e, f):
    s, r = fsymbol_exact(j1, j2, j3, j4, e, f)
    return float(s) * math.sqrt(float(r)) if s != 0 else 0.0


def rsymbol(j1, j2, j3):
    """Reading C8: R^{j1 j2}_{j3} = (-1)^{j1+j2-j3} (0 if not admissible)."""
    if not triangle(j1, j2, j3):
        return 0.0
    return -1.0 if _half(j1 + j2 - j3) % 2 else 1.0


def rsymbol_printed(j1, j2, j3):
    """The formula as printed at P:2329, kept only to document reading C8 in tests."""
    if not triangle(j1, j2, j3):
        return 0.0
    x = j1 + j2 + j3
    return -1.0 if (x % 4) == 2 else (1.0 if x % 4 == 0 else float("nan"))


def z_flip(X, axis, j):
    """Apply Z^dagger (codomain dual leg) / Z (domain dual leg) along `axis` (reading C7).

    Both act on the tree tensor as  X'[.., mu, ..] = (-1)^{j-m} X[.., -m, ..]  with
    m = j - mu, i.e. (-1)^mu times the m -> -m flipped slice.
    """
    Xf = np.flip(X, axis=axis)
    shape = [1] * X.ndim
    shape[axis] = j + 1
    sgn = np.array([(-1.0) ** mu for mu in range(j + 1)]).reshape(shape)
    return Xf * sgn


def spin_matrices(j):
    """J_z, J_+, J_- in the basis mu = 0..2j (m = j - mu), for Wigner-D tests."""
    d = j + 1
    ms = [m / 2 for m in mvals(j)]
    jj = j / 2
    Jz = np.diag(ms)
    Jp = np.zeros((d, d))
    for mu in range(1, d):
        m = ms[mu]
        Jp[mu - 1, mu] = math.sqrt(jj * (jj + 1) - m * (m + 1))
    return Jz, Jp, Jp.T.copy()
