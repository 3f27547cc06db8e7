"""Pins of the planar (anyonic) oracle, oracle/planar.py -- SURVEY NEXT-4, CPU only.

  * the planar moves (right bends with B-symbols, F-recoupling of the first leg to the top, the
    Frobenius-Schur factor of carrying it around) reproduce the DENSE SU(2) Clebsch-Gordan oracle for
    every cyclic transpose with dual legs, integer and half-integer spins;
  * the Fib / Ising F-symbols typed from P:2424-2437 satisfy the pentagon and are
    unitary; Ising restricted to {I, psi} has trivial F;
  * a full rotation of all legs is the identity; every transfer matrix preserves the inner product
    sum_c d_c |block|^2 (the moves are unitary).
"""
import itertools

import numpy as np
import pytest

from oracle import planar as OP, sectors
from workloads import configs as W


def cyclic(n1, N, r, n1p):
    S = list(range(n1)) + list(range(N - 1, n1 - 1, -1))
    T = [S[(i + r) % N] for i in range(N)]
    return T[:n1p], list(reversed(T[n1p:]))


SHAPES = [([0, 1], [0]), ([0, 0], [1, 0]), ([1, 0, 0], [0]), ([0], [0, 0]), ([0, 0], [0, 0])]


def _spaces(kind, secs, cd, dd):
    V = W.space(kind, secs)
    return [W.dual(V) if d else V for d in cd], [W.dual(V) if d else V for d in dd]


@pytest.mark.parametrize("secs,nshapes", [([((0,), 1), ((1,), 1), ((2,), 1)], 4),
                                         ([((1,), 1), ((2,), 1)], 3)])
def test_planar_moves_equal_dense_su2(secs, nshapes):
    from tests.test_library_host import oracle_transfer
    for cd, dd in SHAPES[:nshapes]:
        cod, dom = _spaces("SU2", secs, cd, dd)
        n1, N = len(cod), len(cod) + len(dom)
        for r in range(N):
            for n1p in range(N + 1):
                p, q = cyclic(n1, N, r, n1p)
                ref, _, _ = oracle_transfer("SU2", cod, dom, p, q)
                M, _, _ = OP.planar_transfer("SU2", cod, dom, p, q)
                assert np.abs(M - ref).max() < 1e-13, (cd, dd, p, q)


@pytest.mark.parametrize("kind,labels", [("Fib", [0, 1]), ("Ising", [0, 1, 2])])
def test_anyon_pentagon_and_unitarity(kind, labels):
    L = [(x,) for x in labels]
    F = lambda *a: OP.fsymbol(kind, *a)  # noqa: E731
    worst = 0.0
    for a, b, c, d, e in itertools.product(L, repeat=5):
        for f, g, k, l in itertools.product(L, repeat=4):
            lhs = F(f, c, d, e, g, l) * F(a, b, l, e, f, k)
            rhs = sum(F(a, b, c, g, f, h) * F(a, h, d, e, g, k) * F(b, c, d, k, h, l) for h in L)
            worst = max(worst, abs(lhs - rhs))
    assert worst < 1e-13
    for a, b, c, d in itertools.product(L, repeat=4):
        es = [e for e in L if OP.admissible(kind, a, b, e) and OP.admissible(kind, e, c, d)]
        fs = [f for f in L if OP.admissible(kind, b, c, f) and OP.admissible(kind, a, f, d)]
        assert len(es) == len(fs)
        M = np.array([[F(a, b, c, d, e, f) for f in fs] for e in es]).reshape(len(es), len(fs))
        if M.size:
            assert np.abs(M @ M.T - np.eye(len(es))).max() < 1e-14


def test_ising_psi_subcategory_trivial():
    for a, b, c, d, e, f in itertools.product([(0,), (2,)], repeat=6):
        x = OP.fsymbol("Ising", a, b, c, d, e, f)
        assert x in (0.0, 1.0)


@pytest.mark.parametrize("kind,secs", [("Fib", [((0,), 1), ((1,), 1)]), ("Ising", [((0,), 1), ((1,), 1), ((2,), 1)]),
                                       ("SU2", [((0,), 1), ((1,), 1), ((2,), 1)])])
def test_full_rotation_identity_and_unitarity(kind, secs):
    for cd, dd in SHAPES:
        cod, dom = _spaces(kind, secs, cd, dd)
        n1, N = len(cod), len(cod) + len(dom)
        # rotate by one position N times (keeping n1 codomain legs): the composition is the identity
        total = None
        c, d = cod, dom
        p, q = cyclic(n1, N, 1, n1)
        for _ in range(N):
            M, lt, ls = OP.planar_transfer(kind, c, d, p, q)
            # unitarity: d_c-weighted norm of tree-pair coefficients preserved
            wa = np.array([sectors.qdim(kind, sb.key[2]) for sb in lt.subblocks])
            wb = np.array([sectors.qdim(kind, sb.key[2]) for sb in ls.subblocks])
            assert np.abs(M @ np.diag(wb) @ M.T - np.diag(wa)).max() < 1e-12
            total = M if total is None else total @ M
            c, d = ls.cod, ls.dom
        assert np.abs(total - np.eye(total.shape[0])).max() < 1e-12


@pytest.mark.parametrize("secs", [[((0,), 2), ((1,), 1), ((2,), 1)], [((1,), 2), ((2,), 1)]])
def test_tree_trace_equals_dense_su2(secs):
    """The tree-level partial trace (close the end legs, d_c/d_e) equals the plain dense trace for SU(2)."""
    from oracle import dense as OD, contract as OC, layout as OL
    V = W.space("SU2", secs)
    Vd = W.dual(V)
    rng = np.random.default_rng(1)
    # planar traces (pairs nested in the cyclic leg order), closed at the tree ends
    cases = [([V, V], [V, V], [1], [3], [0], [2]), ([V, V], [V, V], [2], [0], [1, 3], []),
             ([V, V, V], [V, V], [2], [4], [0, 1], [3]), ([V, V], [V, V], [0, 1], [2, 3], [], []),
             ([Vd, V], [Vd, V], [1], [3], [0], [2])]
    for cod, dom, pt, qt, p, q in cases:
        lt = OL.homspace_layout("SU2", cod, dom)
        x = rng.standard_normal(lt.nelems)
        got, lc = OP.trace_planar("SU2", cod, dom, x, pt, qt, p, q)
        R, c2, d2 = OC.partial_trace_dense(OD.to_dense(lt, x), cod, dom, pt, qt, p, q)
        assert OC.rel_frobenius(OD.to_dense(lc, got), R) < 1e-13, (pt, qt, p, q)
