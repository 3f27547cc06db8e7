"""Planar (cyclic) transposes on fusion-tree pairs -- TEST INFRASTRUCTURE ONLY.

Anyonic categories (Fib, Ising) have no group representation, so there is no dense
embedding to compare against; their R-symbols are complex phases, so only planar operations stay
real. This module follows the paper's moves step by step, written from the text (it shares no code
with the library):

  1. bend every domain leg, last first, to the end of the splitting tree (eq. ftbendright):
     coefficient sqrt(d_c / d_e) B^{e b}_c, times chi_b when the bent leg carried a Z,
     with B^{ab}_c = sqrt(d_a d_b / d_c) F^{a b bbar}_a[c, I];
  2. rotate the all-codomain tree (unit coupled charge) cyclically: recouple the first leg a1 to the top
     by F-moves, ((a1 a2)e2 a3)e3... = sum prod F^{a1 f a_k}_{e_k}[e_{k-1}, f'] (a1 (a2 ... aN)_y)_I
     (P:1117-1123), then carry a1 around the unit vertex to the right end with the Frobenius-Schur
     indicator chi_{a1} (the left fold, followed by a right bend);
  3. bend the trailing legs back to the domain (step 1 in reverse order of legs).

Pins (tests/test_oracle_planar.py): for SU(2) the result equals the dense Clebsch-Gordan oracle for
every cyclic transpose with dual legs (so the moves and their normalisation are right); the Fib/Ising
F-symbols satisfy the pentagon and are unitary; a full rotation is the identity; transfer matrices
preserve the norm sum_c d_c |block|^2 (unitarity of the moves).
"""
import math

import numpy as np

from . import sectors, su2
from .layout import homspace_layout, underlying


# ------------------------------------------------------------------ topological data
def _fib_F(a, b, c, d, e, f):
    if (a, b, c, d) == (1, 1, 1, 1):
        phi = sectors.GOLDEN
        M = {(0, 0): 1 / phi, (0, 1): phi ** -0.5, (1, 0): phi ** -0.5, (1, 1): -1 / phi}
        return M[(e, f)]
    return 1.0


def _ising_F(a, b, c, d, e, f):
    if (a, b, c, d) == (1, 1, 1, 1):
        return (-1.0 if (e, f) == (2, 2) else 1.0) / math.sqrt(2)
    if (a, b, c, d) in ((1, 2, 1, 2), (2, 1, 2, 1)):
        return -1.0
    return 1.0


def admissible(kind, a, b, c):
    return tuple(c) in [tuple(x) for x in sectors.fuse(kind, a, b)]


def fsymbol(kind, a, b, c, d, e, f):
    """F^{abc}_d[e, f], e = a x b, f = b x c (zero when a vertex is not allowed)."""
    if not (admissible(kind, a, b, e) and admissible(kind, e, c, d) and admissible(kind, b, c, f)
            and admissible(kind, a, f, d)):
        return 0.0
    if kind == "SU2":
        return su2.fsymbol(a[0], b[0], c[0], d[0], e[0], f[0])
    if kind == "Fib":
        return _fib_F(a[0], b[0], c[0], d[0], e[0], f[0])
    if kind == "Ising":
        return _ising_F(a[0], b[0], c[0], d[0], e[0], f[0])
    raise ValueError(kind)


def chi(kind, a):
    if kind == "SU2":
        return -1.0 if a[0] % 2 else 1.0
    return 1.0  # Fib and Ising labels are all real


def bsymbol(kind, a, b, c):
    unit = sectors.unit(kind)
    return math.sqrt(sectors.qdim(kind, a) * sectors.qdim(kind, b) / sectors.qdim(kind, c)) * \
        fsymbol(kind, a, b, sectors.dual(kind, b), a, c, unit)


# ------------------------------------------------------------------ tree states
# A state is one splitting tree (all legs in the codomain after step 1) plus a fusion tree:
# (s_unc, s_chain, s_dual, s_ids, f_unc, f_chain, f_dual, f_ids); chains list the labels of the first
# k+1 legs (chain[-1] = coupled; () for an empty tree means the unit).
def _chain(kind, unc, inner, coupled):
    if not unc:
        return ()
    if len(unc) == 1:
        return (tuple(unc[0]),)
    return (tuple(unc[0]),) + tuple(tuple(x) for x in inner) + (tuple(coupled),)


def _coupled(kind, chain):
    return chain[-1] if chain else sectors.unit(kind)


def _bend_last(kind, frm, to, coef):
    """Move the last leg of tree `frm` to the end of tree `to` (eq. ftbendright)."""
    unc, ch, du, ids = frm
    tunc, tch, tdu, tids = to
    n = len(unc)
    c = _coupled(kind, ch)
    b = unc[-1]
    e = ch[n - 2] if n >= 2 else sectors.unit(kind)
    coef *= math.sqrt(sectors.qdim(kind, c) / sectors.qdim(kind, e)) * bsymbol(kind, e, b, c)
    if du[-1]:
        coef *= chi(kind, b)
    nfrm = (unc[:-1], ch[:n - 1] if n >= 2 else (), du[:-1], ids[:-1])
    bb = sectors.dual(kind, b)
    if not tunc:
        ntch = (bb,)
    else:
        ntch = tch + (e,)
    nto = (tunc + (bb,), ntch, tdu + (not du[-1],), tids + (ids[-1],))
    return nfrm, nto, coef


def _rotate(kind, s, coef):
    """(a1, ..., aN) -> (a2, ..., aN, a1) on a codomain tree with unit coupled charge: list of (s', c)."""
    unc, ch, du, ids = s
    n = len(unc)
    if n <= 1:
        return [(s, coef)]
    a1 = unc[0]
    paths = [((unc[1],), 1.0)]
    for k in range(2, n):
        nx = []
        for f, c in paths:
            for fnew in sectors.fuse(kind, f[-1], unc[k]):
                x = fsymbol(kind, a1, f[-1], unc[k], ch[k], ch[k - 1], fnew)
                if x != 0.0:
                    nx.append((f + (tuple(fnew),), c * x))
        paths = nx
    out = []
    for f, c in paths:
        if not admissible(kind, a1, f[-1], ch[n - 1]):
            continue
        ns = (unc[1:] + (a1,), f + (ch[n - 1],), du[1:] + (du[0],), ids[1:] + (ids[0],))
        out.append((ns, coef * c * chi(kind, a1)))
    return out


def transform_tree_pair(kind, key, cod, dom, p, q):
    """Terms {(cod_unc, cod_chain, dom_unc, dom_chain): coef} of permute((s, f), (p, q)) for a planar
    (cyclic) (p, q); key = (s_unc, s_inner, coupled, f_unc, f_inner) with tree labels."""
    s_unc, s_inn, c, f_unc, f_inn = key
    n1, n2 = len(s_unc), len(f_unc)
    N = n1 + n2
    S = list(range(n1)) + list(range(N - 1, n1 - 1, -1))
    T = list(p) + list(reversed(q))
    r = next((r for r in range(max(N, 1)) if all(T[i] == S[(i + r) % N] for i in range(N))), None) if N else 0
    if r is None:
        raise ValueError("not a planar (cyclic) transpose")
    s = (tuple(map(tuple, s_unc)), _chain(kind, s_unc, s_inn, c), tuple(sp["dual"] for sp in cod), tuple(range(n1)))
    f = (tuple(map(tuple, f_unc)), _chain(kind, f_unc, f_inn, c), tuple(sp["dual"] for sp in dom),
         tuple(range(n1, N)))
    coef = 1.0
    while f[0]:
        f, s, coef = _bend_last(kind, f, s, coef)
    states = [(s, coef)]
    for _ in range(r):
        states = [x for st, cf in states for x in _rotate(kind, st, cf)]
    out = {}
    n2p = len(q)
    for st, cf in states:
        ss, ff = st, ((), (), (), ())
        for _ in range(n2p):
            ss, ff, cf = _bend_last(kind, ss, ff, cf)
        k = (ss[0], ss[1], ff[0], ff[1])
        out[k] = out.get(k, 0.0) + cf
    return out


def _pair_key(sb_key):
    s_unc, s_inn, c, f_unc, f_inn = sb_key
    return (tuple(map(tuple, s_unc)), None, tuple(map(tuple, f_unc)), None)


def planar_transfer(kind, cod, dom, p, q):
    """Dense (n_sub(A) x n_sub(C)) matrix of the planar permute on tree pairs (layout order of
    oracle.layout), plus C's spaces."""
    from .contract import permuted_spaces
    lt = homspace_layout(kind, cod, dom)
    c2, d2 = permuted_spaces(cod, dom, p, q)
    ls = homspace_layout(kind, c2, d2)
    index = {}
    for j, sb in enumerate(ls.subblocks):
        s_unc, s_inn, cc, f_unc, f_inn = sb.key
        index[(tuple(map(tuple, s_unc)), _chain(kind, s_unc, s_inn, cc), tuple(map(tuple, f_unc)),
               _chain(kind, f_unc, f_inn, cc))] = j
    M = np.zeros((len(lt.subblocks), len(ls.subblocks)))
    for i, sb in enumerate(lt.subblocks):
        for k, cf in transform_tree_pair(kind, sb.key, cod, dom, p, q).items():
            M[i, index[k]] += cf
    return M, lt, ls


def apply_planar(kind, cod, dom, flat, p, q):
    """Reduced data of permute(A, (p, q)) for a planar (p, q): every destination subblock is the
    coefficient-weighted sum of its sources, transposed to (p..., q...) leg order."""
    M, lt, ls = planar_transfer(kind, cod, dom, p, q)
    from .dense import subblock_array
    out = np.zeros(ls.nelems, dtype=np.asarray(flat).dtype)
    order = list(p) + list(q)
    for i, sa in enumerate(lt.subblocks):
        x = np.transpose(np.asarray(subblock_array(lt, np.asarray(flat), sa)), order)
        for j in np.nonzero(M[i])[0]:
            subblock_array(ls, out, ls.subblocks[j])[...] += M[i, j] * x
    return out, ls


def contract_planar(kind, A_spec, xa, labA, B_spec, xb, labB, labC, n_cod_C):
    """Alg. 4 with planar permutes: A~ = permute(A), B~ = permute(B) (reading C2 tuples),
    one block product per coupled sector (composition = matmul), then permute C~ -> C."""
    from .contract import tuples_from_labels
    from .dense import subblock_array  # noqa: F401
    pA, qA, pB, qB, pAB, qAB = tuples_from_labels(labA, labB, labC, n_cod_C)
    At, la = apply_planar(kind, A_spec["cod"], A_spec["dom"], xa, pA, qA)
    Bt, lb = apply_planar(kind, B_spec["cod"], B_spec["dom"], xb, pB, qB)
    lc = homspace_layout(kind, la.cod, lb.dom)
    Ct = np.zeros(lc.nelems)
    ablk = {b[0]: b for b in la.blocks}
    bblk = {b[0]: b for b in lb.blocks}
    for (c, rows, cols, off) in lc.blocks:
        if c not in ablk or c not in bblk:
            continue
        _, ar, ac, ao = ablk[c]
        _, br, bc, bo = bblk[c]
        Ma = At[ao:ao + ar * ac].reshape(ar, ac, order="F")
        Mb = Bt[bo:bo + br * bc].reshape(br, bc, order="F")
        Ct[off:off + rows * cols] = (Ma @ Mb).reshape(-1, order="F")
    return apply_planar(kind, lc.cod, lc.dom, Ct, pAB, qAB)


def _peel_key(kind, unc, inner, coupled):
    """Tree without its last leg: (unc, inner, coupled)."""
    n = len(unc)
    if n == 1:
        return (), (), sectors.unit(kind)
    if n == 2:
        return (tuple(unc[0]),), (), tuple(unc[0])
    return tuple(map(tuple, unc[:-1])), tuple(map(tuple, inner[:-1])), tuple(inner[-1])


def trace_planar(kind, cod, dom, flat, pt, qt, p, q):
    """Partial trace by tree manipulations: permute so that the traced pairs close at the
    ends of the trees, (p..., pt... ; q..., qt...), then close the last splitting leg with the last
    fusion leg: both trees lose that leg, their new coupled labels must agree (e), and the loop leaves
    the factor d_c / d_e (the tadpole). Returns (reduced data of C, C's layout)."""
    from .dense import subblock_array
    nt = len(pt)
    At, la = apply_planar(kind, cod, dom, flat, list(p) + list(pt), list(q) + list(qt))
    from .contract import permuted_spaces
    c2, d2 = permuted_spaces(cod, dom, p, q)
    lc = homspace_layout(kind, c2, d2)
    index = {(tuple(map(tuple, sb.key[0])), tuple(map(tuple, sb.key[1])), tuple(sb.key[2]),
              tuple(map(tuple, sb.key[3])), tuple(map(tuple, sb.key[4]))): j for j, sb in enumerate(lc.subblocks)}
    out = np.zeros(lc.nelems)
    n1, n2 = len(p), len(q)
    for sb in la.subblocks:
        s_unc, s_inn, c, f_unc, f_inn = sb.key
        s = (list(s_unc), list(s_inn), tuple(c))
        f = (list(f_unc), list(f_inn), tuple(c))
        coef, ok = 1.0, True
        for _ in range(nt):
            if tuple(s[0][-1]) != tuple(f[0][-1]):
                ok = False
                break
            cc = s[2]
            s = _peel_key(kind, *s)
            f = _peel_key(kind, *f)
            if tuple(s[2]) != tuple(f[2]):
                ok = False
                break
            coef *= sectors.qdim(kind, cc) / sectors.qdim(kind, s[2])
            s = (list(s[0]), list(s[1]), s[2])
            f = (list(f[0]), list(f[1]), f[2])
        if not ok:
            continue
        key = (tuple(map(tuple, s[0])), tuple(map(tuple, s[1])), tuple(s[2]), tuple(map(tuple, f[0])),
               tuple(map(tuple, f[1])))
        j = index[key]
        x = np.asarray(subblock_array(la, At, sb))  # legs (p..., pt..., q..., qt...)
        letters = "abcdefghijklmnop"
        L = [letters[i] for i in range(x.ndim)]
        for r in range(nt):
            L[n1 + nt + n2 + r] = L[n1 + r]
        outl = "".join(L[:n1] + L[n1 + nt:n1 + nt + n2])
        y = np.einsum("".join(L) + "->" + outl, x)
        subblock_array(lc, out, lc.subblocks[j])[...] += coef * y
    return out, lc
