"""Pins of the oracle's SU(2) data against closed forms, textbook identities and the paper.

Nothing here re-types an oracle formula: each check compares two independent
computations (CG vs 6j, exact vs identity, oracle vs printed paper values).
"""
import math
import itertools

import numpy as np
import pytest

from oracle import su2

JMAX = 4  # doubled: spins up to 2


def spins(jmax=JMAX):
    return range(0, jmax + 1)


def test_cg_textbook_values():
    # Condon-Shortley values (any angular-momentum textbook table)
    assert su2.cg(1, 1, 1, -1, 2, 0) == pytest.approx(1 / math.sqrt(2), abs=1e-15)
    assert su2.cg(1, 1, 1, -1, 0, 0) == pytest.approx(1 / math.sqrt(2), abs=1e-15)
    assert su2.cg(1, -1, 1, 1, 0, 0) == pytest.approx(-1 / math.sqrt(2), abs=1e-15)
    assert su2.cg(2, 2, 2, -2, 0, 0) == pytest.approx(1 / math.sqrt(3), abs=1e-15)
    assert su2.cg(2, 0, 2, 0, 0, 0) == pytest.approx(-1 / math.sqrt(3), abs=1e-15)
    assert su2.cg(2, 2, 1, -1, 1, 1) == pytest.approx(math.sqrt(2 / 3), abs=1e-15)
    for j1, j2 in itertools.product(spins(6), repeat=2):
        assert su2.cg(j1, j1, j2, j2, j1 + j2, j1 + j2) == pytest.approx(1.0, abs=1e-15)


def test_cg_orthogonality_and_completeness():
    # eq. fusiontensororthogonality: the CG matrix is orthogonal
    for j1, j2 in itertools.product(spins(6), repeat=2):
        cols = []
        for J in range(abs(j1 - j2), j1 + j2 + 1, 2):
            X = su2.cg_tensor(j1, j2, J)
            cols.append(X.reshape((j1 + 1) * (j2 + 1), J + 1))
        U = np.concatenate(cols, axis=1)
        assert U.shape[0] == U.shape[1]
        assert np.abs(U.T @ U - np.eye(U.shape[0])).max() < 1e-14


def test_sixj_special_values_and_orthogonality():
    # {a b c; 0 c b} = (-1)^{a+b+c} / sqrt((2b+1)(2c+1))
    for a, b, c in itertools.product(spins(6), repeat=3):
        if su2.triangle(a, b, c):
            ref = (-1) ** ((a + b + c) // 2) / math.sqrt((b + 1) * (c + 1))
            assert su2.sixj(a, b, c, 0, c, b) == pytest.approx(ref, abs=1e-15)
    # sum_x (2x+1)(2p+1) {a b x; c d p}{c d x; a b q} = delta_pq  (textbook orthogonality)
    for a, b, c, d in itertools.product(spins(3), repeat=4):
        ps = [p for p in range(0, 8) if su2.triangle(a, d, p) and su2.triangle(c, b, p)]
        for p, q in itertools.product(ps, repeat=2):
            s = sum((x + 1) * (p + 1) * su2.sixj(a, b, x, c, d, p) * su2.sixj(c, d, x, a, b, q)
                    for x in range(0, 8))
            assert s == pytest.approx(1.0 if p == q else 0.0, abs=1e-13)


def _cg_overlap_F(j1, j2, j3, j4, e, f):
    """<((j1 j2)e, j3) j4 | (j1, (j2 j3) f) j4>, both trees built from CG tensors."""
    left = np.tensordot(su2.cg_tensor(j1, j2, e), su2.cg_tensor(e, j3, j4), axes=([2], [0]))   # m1 m2 m3 M
    inner = su2.cg_tensor(j2, j3, f)
    right = np.tensordot(su2.cg_tensor(j1, f, j4), inner, axes=([1], [2]))                     # m1 M m2 m3
    right = right.transpose(0, 2, 3, 1)
    return float(np.sum(left[..., 0] * right[..., 0]))


def test_fsymbol_formula_equals_cg_overlap():
    # Eq. SU2FSymbol vs the CG projection; reading C9
    n = 0
    for j1, j2, j3, j4 in itertools.product(spins(), repeat=4):
        for e in range(0, 9):
            for f in range(0, 9):
                if not (su2.triangle(j1, j2, e) and su2.triangle(e, j3, j4) and su2.triangle(j2, j3, f)
                        and su2.triangle(j1, f, j4)):
                    continue
                assert su2.fsymbol(j1, j2, j3, j4, e, f) == pytest.approx(_cg_overlap_F(j1, j2, j3, j4, e, f),
                                                                          abs=2e-15)
                n += 1
    assert n > 500


def test_fsymbol_unitary():
    # P:1566-1569
    for j1, j2, j3, j4 in itertools.product(spins(), repeat=4):
        es = [e for e in range(0, 9) if su2.triangle(j1, j2, e) and su2.triangle(e, j3, j4)]
        fs = [f for f in range(0, 9) if su2.triangle(j2, j3, f) and su2.triangle(j1, f, j4)]
        if not es:
            continue
        F = np.array([[su2.fsymbol(j1, j2, j3, j4, e, f) for f in fs] for e in es])
        assert np.abs(F @ F.T - np.eye(len(es))).max() < 1e-14


def _F(a, b, c, d, e, f):
    return su2.fsymbol(a, b, c, d, e, f)


def test_pentagon():
    # F^{fcd}_e[g,l] F^{abl}_e[f,k] = sum_h F^{abc}_g[f,h] F^{ahd}_e[g,k] F^{bcd}_k[h,l]
    r = range(0, 4)
    worst = 0.0
    for a, b, c, d in itertools.product(r, repeat=4):
        for e in range(0, 9):
            for f, g, k, l in itertools.product(range(0, 7), repeat=4):
                if not (su2.triangle(a, b, f) and su2.triangle(f, c, g) and su2.triangle(g, d, e)
                        and su2.triangle(c, d, l) and su2.triangle(b, l, k) and su2.triangle(a, k, e)
                        and su2.triangle(f, l, e)):
                    continue
                lhs = _F(f, c, d, e, g, l) * _F(a, b, l, e, f, k)
                rhs = sum(_F(a, b, c, g, f, h) * _F(a, h, d, e, g, k) * _F(b, c, d, k, h, l) for h in range(0, 9))
                worst = max(worst, abs(lhs - rhs))
    assert worst < 1e-13


def test_rsymbol_from_cg_exchange_and_unit_axiom():
    # R^{ab}_c defined by swapping the legs of the splitting tensor
    for j1, j2 in itertools.product(spins(6), repeat=2):
        for J in range(abs(j1 - j2), j1 + j2 + 1, 2):
            swapped = su2.cg_tensor(j2, j1, J).transpose(1, 0, 2)
            assert np.abs(swapped - su2.rsymbol(j1, j2, J) * su2.cg_tensor(j1, j2, J)).max() < 1e-14
    # unit axiom R^{aI}_a = 1 (reading C8); the printed formula fails it for half-integers
    for a in spins(6):
        assert su2.rsymbol(a, 0, a) == 1.0
    assert su2.rsymbol_printed(1, 0, 1) == -1.0


def test_hexagon():
    # symmetric-braiding hexagon:
    #   R^{ca}_e F^{acb}_d[e,g] R^{cb}_g = sum_f F^{cab}_d[e,f] R^{cf}_d F^{abc}_d[f,g]
    worst = 0.0
    r = range(0, 5)
    for a, b, c, d in itertools.product(r, repeat=4):
        for e, g in itertools.product(range(0, 9), repeat=2):
            if not (su2.triangle(c, a, e) and su2.triangle(e, b, d) and su2.triangle(c, b, g)
                    and su2.triangle(a, g, d)):
                continue
            lhs = su2.rsymbol(c, a, e) * _F(a, c, b, d, e, g) * su2.rsymbol(c, b, g)
            rhs = sum(_F(c, a, b, d, e, f) * su2.rsymbol(c, f, d) * _F(a, b, c, d, f, g)
                      for f in range(0, 9) if su2.triangle(a, b, f) and su2.triangle(c, f, d))
            worst = max(worst, abs(lhs - rhs))
    assert worst < 1e-13


def test_dimensions_and_frobenius_schur():
    # d_a d_b = sum_c N d_c; 1/d_a = |F^{a a a}_a[I, I]|, chi_a = sign
    for a, b in itertools.product(spins(8), repeat=2):
        assert (a + 1) * (b + 1) == sum(c + 1 for c in range(abs(a - b), a + b + 1, 2))
    for a in spins(8):
        F = su2.fsymbol(a, a, a, a, 0, 0)
        assert abs(F) == pytest.approx(1 / (a + 1), abs=1e-15)
        assert math.copysign(1, F) == (-1) ** a   # chi_j = (-1)^{2j}


def test_z_intertwines_dual_representation():
    # Reading C7: Z o rho*(g) = rho(g) o Z (eq. definitionZ)
    from scipy.linalg import expm
    rng = np.random.default_rng(1)
    for j in spins(6):
        Jz, Jp, Jm = su2.spin_matrices(j)
        Jx, Jy = (Jp + Jm) / 2, (Jp - Jm) / 2j
        th = rng.standard_normal(3)
        D = expm(-1j * (th[0] * Jx + th[1] * Jy + th[2] * Jz))
        Z = np.zeros((j + 1, j + 1))
        for mu in range(j + 1):  # Z <j m| = (-1)^{j-m} |j,-m>,  m = j - mu
            Z[j - mu, mu] = (-1.0) ** mu
        assert np.abs(Z @ D.conj() - D @ Z).max() < 1e-12
