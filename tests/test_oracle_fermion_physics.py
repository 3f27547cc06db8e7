"""Physics pins of the oracle's fermionic convention (reading C13) -- anchors outside the oracle itself.

The paper prints no fermionic example (P:2355-2362 only states that exchanging two odd legs gives -1),
so the C13 partial pins in test_oracle_dense.py fix the sign of codomain permutes. These tests pin the
rest of the convention -- domain legs, bends, Alg. 4 with legs moving between codomain and domain --
against what the mathematics of super vector spaces (SVect) and the canonical
anticommutation relations fix, independently of the oracle's formula:

  1. the tensor product of two EVEN morphisms f (x) g in SVect carries no Koszul sign:
     (f (x) g)(v (x) w) = (-1)^{|g||v|} f(v) (x) g(w) = f(v) (x) g(w), so its matrix in the product basis is the
     Kronecker product. Building f (x) g with Alg. 4 (an empty contraction: A~ = permute(f, (all, ())),
     B~ = permute(g, ((), all)), then the output permute to (cod_f cod_g ; dom_f dom_g)) must give exactly
     that for random even tensors -- a convention that did not reverse the domain legs would give
     (-1)^{|dom_f||cod_g|} instead;
  2. Jordan-Wigner: an annihilation operator is an odd map, written as an even tensor map
     c^: V <- V (x) A with an odd one-dimensional auxiliary leg A. On L sites,
     C_j = id (x) ... (x) c^ (x) ... (x) id with A moved to the end of the domain, and
     c_i^dag c_j = (D_i o (C_j (x) id_A)) o (id (x) eta), eta the pairing state of the two aux legs, must equal
     the textbook Jordan-Wigner matrices sigma_i^+ Z...Z sigma_j^- (the string is the Koszul sign of moving A
     past the occupied sites) for EVERY i, j, with one global sign fixed by c_i^dag c_i = n_i. The
     Jordan-Wigner matrices are themselves checked against the CAR {c_i, c_j^dag} = delta_ij.
"""
import itertools

import numpy as np
import pytest

from oracle import contract as C, dense as Dn, layout as L
from workloads import configs as W


def _par(sps):
    return [Dn.parity_vector(s) for s in sps]


def tensor_product(f, fsp, fn, g, gsp, gn):
    """f (x) g through the oracle's Alg. 4 with nothing contracted (all signs from reading C13)."""
    Nf, Ng = f.ndim, g.ndim
    pA, qA = list(range(Nf)), []
    pB, qB = [], list(range(Ng))
    # C~ legs: f's legs 0..Nf-1, then g's legs (positions Nf..Nf+Ng-1)
    pAB = list(range(fn)) + [Nf + j for j in range(gn)]
    qAB = list(range(fn, Nf)) + [Nf + j for j in range(gn, Ng)]
    out = C.contract_alg4_tuples(f, fsp, fn, g, gsp, gn, pA, qA, pB, qB, pAB, qAB)
    sp = [fsp[i] for i in range(fn)] + [gsp[j] for j in range(gn)] + \
         [fsp[i] for i in range(fn, Nf)] + [gsp[j] for j in range(gn, Ng)]
    return out, sp, fn + gn


def compose(X, Xsp, nX, Y, Ysp, nY):
    """X o Y (dom X = cod Y) through Alg. 4: A~ = X, B~ = Y, C~ = A~ B~."""
    NX, NY = X.ndim, Y.ndim
    assert NX - nX == nY
    out = C.contract_alg4_tuples(X, Xsp, nX, Y, Ysp, nY, list(range(nX)), list(range(nX, NX)),
                                 list(range(nY)), list(range(nY, NY)), list(range(nX)),
                                 list(range(nX, nX + NY - nY)))
    return out, Xsp[:nX] + Ysp[nY:], nX


def _kron_expected(f, fn, g, gn):
    Nf, Ng = f.ndim, g.ndim
    o = np.multiply.outer(f, g)  # legs (f..., g...)
    order = list(range(fn)) + [Nf + j for j in range(gn)] + list(range(fn, Nf)) + [Nf + j for j in range(gn, Ng)]
    return np.transpose(o, order)


@pytest.mark.parametrize("kind,secs", [
    ("fZ2", [((0,), 2), ((1,), 3)]),
    ("fU1xU1", [((0, 0), 1), ((1, 1), 2), ((1, -1), 1), ((-1, 1), 2), ((2, 0), 1)]),
])
def test_tensor_product_of_even_maps_is_kronecker(kind, secs):
    V = W.space(kind, secs)
    Vd = W.dual(V)
    rng = np.random.default_rng(11)
    shapes = [(([V], [V, V]), ([V, Vd], [V])), (([V, V], [Vd]), ([V], [V, V])), (([V], [V]), ([Vd, V], [V, Vd])),
              (([V, V], []), ([V], [V, V]))]
    nontrivial = 0
    for (fc, fd), (gc, gd) in shapes:
        lf, lg = L.homspace_layout(kind, fc, fd), L.homspace_layout(kind, gc, gd)
        f = Dn.to_dense(lf, rng.standard_normal(lf.nelems))
        g = Dn.to_dense(lg, rng.standard_normal(lg.nelems))
        got, _, _ = tensor_product(f, fc + fd, len(fc), g, gc + gd, len(gc))
        want = _kron_expected(f, len(fc), g, len(gc))
        assert np.array_equal(got, want), (fc, fd, gc, gd)
        # the same result with the wrong (unreversed-domain) convention differs: the sign it would put,
        # (-1)^{|dom_f| |cod_g|}, is not identically +1 on these inputs
        pdf = sum(np.ix_(*[Dn.parity_vector(s) for s in fd])) if fd else 0
        pcg = sum(np.ix_(*[Dn.parity_vector(s) for s in gc])) if gc else 0
        nontrivial += int(np.any((np.multiply.outer(pdf, pcg) % 2) == 1) and np.abs(want).max() > 0)
    assert nontrivial >= 2


# ------------------------------------------------------------------ Jordan-Wigner / CAR
_SIG = np.array([[0.0, 1.0], [0.0, 0.0]])   # |0><1| (annihilator on one mode)
_Z = np.diag([1.0, -1.0])


def _jw(L, j, dag=False):
    """Textbook Jordan-Wigner operator with the string on the sites after j (dense 2^L x 2^L)."""
    ops = [np.eye(2)] * j + [_SIG.T if dag else _SIG] + [_Z] * (L - 1 - j)
    M = np.array([[1.0]])
    for o in ops:
        M = np.kron(M, o)
    return M


def _site_ops():
    V = W.space("fZ2", [((0,), 1), ((1,), 1)])   # |0> even (index 0), |1> odd (index 1)
    A = W.space("fZ2", [((1,), 1)])              # odd auxiliary leg
    c = np.zeros((2, 2, 1))
    c[0, 1, 0] = 1.0                             # c^: |0> <- |1> (x) |a>
    a = np.zeros((2, 2, 1))
    a[1, 0, 0] = 1.0                             # c^dag: |1> <- |0> (x) |a>
    return V, A, c, a


def _operator_with_aux(L, j, site_op):
    """O_j = id^(x)j (x) site_op (x) id^(x)(L-1-j), its aux leg moved to the end of the domain."""
    V, A, _, _ = _site_ops()
    I1 = np.eye(2)
    X, Xsp, nX = None, None, 0
    for s in range(L):
        if s == j:
            T, Tsp, nT = site_op, [V, V, A], 1
        else:
            T, Tsp, nT = I1, [V, V], 1
        if X is None:
            X, Xsp, nX = T, Tsp, nT
        else:
            X, Xsp, nX = tensor_product(X, Xsp, nX, T, Tsp, nT)
    # domain legs now: V_0 .. V_j A V_{j+1} .. V_{L-1}; move A to the end (a domain-internal permute)
    dom = list(range(nX, X.ndim))
    aux = nX + j + 1
    q = [d for d in dom if d != aux] + [aux]
    X = C.permute_dense(X, _par(Xsp), nX, list(range(nX)), q)
    return X, Xsp[:nX] + [Xsp[k] for k in q], nX


def _hopping(L, i, j):
    """c_i^dag c_j built from the graded local tensors through the oracle's permutes and Alg. 4."""
    V, A, c, a = _site_ops()
    Di, Dsp, nD = _operator_with_aux(L, i, a)
    Cj, Csp, nC = _operator_with_aux(L, j, c)
    idA = np.eye(1)
    Cx, Cxsp, nCx = tensor_product(Cj, Csp, nC, idA, [A, A], 1)      # V^L A <- V^L A A
    P, Psp, nP = compose(Di, Dsp, nD, Cx, Cxsp, nCx)                # V^L <- V^L A A
    eta = np.ones((1, 1))                                          # A A <- (unit): the pairing state
    idL = np.eye(2 ** L).reshape([2] * (2 * L))
    E, Esp, nE = tensor_product(idL, [V] * (2 * L), L, eta, [A, A], 2)  # V^L A A <- V^L
    M, _, _ = compose(P, Psp, nP, E, Esp, nE)                      # V^L <- V^L
    return M.reshape(2 ** L, 2 ** L)


def test_jordan_wigner_matrices_satisfy_car():
    L = 3
    for i, j in itertools.product(range(L), repeat=2):
        ci, cjd = _jw(L, i), _jw(L, j, dag=True)
        assert np.array_equal(ci @ cjd + cjd @ ci, np.eye(2 ** L) * (i == j))
        assert np.array_equal(ci @ _jw(L, j) + _jw(L, j) @ ci, np.zeros((2 ** L, 2 ** L)))


@pytest.mark.parametrize("L", [3, 4])
def test_graded_hopping_equals_jordan_wigner(L):
    s = None
    strings = 0
    for i, j in itertools.product(range(L), repeat=2):
        got = _hopping(L, i, j)
        want = _jw(L, i, dag=True) @ _jw(L, j)
        if s is None:  # global sign of the aux pairing, fixed by c_0^dag c_0 = n_0 (i = j = 0 comes first)
            assert i == j == 0
            s = 1.0 if np.array_equal(got, want) else -1.0
            assert np.array_equal(got, s * want), "c^dag c is not the number operator"
        assert np.array_equal(got, s * want), (i, j)
        # the string is really exercised: without it (sigma+_i sigma-_j) the matrix differs
        bare = [np.eye(2)] * L
        if i == j:
            continue
        bare[i] = _SIG.T
        bare[j] = _SIG
        B = np.array([[1.0]])
        for o in bare:
            B = np.kron(B, o)
        strings += int(not np.array_equal(B, want))
    assert strings > 0


def test_pins_reject_plausible_wrong_conventions(monkeypatch):
    """The two pins above are not vacuous: a convention that keeps the domain order (no reversal of q) fails
    the tensor-product pin, and dropping every Koszul sign (bosonic) fails the Jordan-Wigner pin."""
    def unreversed(n1, n2, p, q):
        N = n1 + n2
        ps = {leg: i for i, leg in enumerate(range(N))}
        pt = {leg: i for i, leg in enumerate(list(p) + list(q))}
        return [(x, y) for x in range(N) for y in range(x + 1, N) if (ps[x] < ps[y]) != (pt[x] < pt[y])]

    monkeypatch.setattr(C, "koszul_sign_pairs", unreversed)
    with pytest.raises(AssertionError):
        test_tensor_product_of_even_maps_is_kronecker("fZ2", [((0,), 2), ((1,), 3)])
    monkeypatch.setattr(C, "koszul_sign_pairs", lambda n1, n2, p, q: [])
    with pytest.raises(AssertionError):
        test_graded_hopping_equals_jordan_wigner(3)
